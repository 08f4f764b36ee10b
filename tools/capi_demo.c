/*
 * capi_demo.c -- a plain-C host driving the B200 path through the C ABI only
 * (no Python): load a bootstrapping key and a ciphertext tensor from the
 * reference's FDSN containers (serial.save_bootstrap_key / save_ciphertexts),
 * bootstrap every ciphertext through the sign table (neuron.g_fire: test
 * polynomial = Delta everywhere, bootstrap.py:90-96), write the results.
 *
 *   capi_demo BK.bin CT.bin PARAMS_DIGEST n N log2q p bg_log levels ks_log ks_levels OUT.bin
 *
 * OUT.bin: count, then count x n int64 masks, then count int64 bodies.
 * build: gcc -O2 -Iinclude tools/capi_demo.c -Lpaper_2309_09025_b200 -lfdsnn_b200 \
 *            -Wl,-rpath,$PWD/paper_2309_09025_b200 -o capi_demo
 */
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include "fdsnn_b200.h"

#define CHECK(call)                                                              \
    do {                                                                         \
        int rc_ = (call);                                                        \
        if (rc_ != FDSNN_OK) {                                                   \
            fprintf(stderr, "%s failed (%d): %s\n", #call, rc_, fdsnn_last_error()); \
            return 1;                                                            \
        }                                                                        \
    } while (0)

int main(int argc, char** argv) {
    if (argc != 13) {
        fprintf(stderr, "usage: %s BK CT DIGEST n N log2q p bg_log levels ks_log ks_levels OUT\n", argv[0]);
        return 2;
    }
    fdsnn_params prm = {atoi(argv[4]), atoi(argv[5]), atoi(argv[6]), atoi(argv[7]),
                        atoi(argv[8]), atoi(argv[9]), atoi(argv[10]), atoi(argv[11])};
    fdsnn_ctx* ctx = NULL;
    CHECK(fdsnn_ctx_create(&prm, 0, &ctx));
    CHECK(fdsnn_bsk_load_fdsn(ctx, argv[1], argv[3]));

    int64_t count = 0, shape[8];
    int32_t ndim = 0;
    CHECK(fdsnn_ciphertexts_load_fdsn(ctx, argv[2], argv[3], &count, &ndim, shape, NULL, NULL));
    const int64_t stride = fdsnn_row_stride(prm.n);
    void *d_in = NULL, *d_out = NULL;
    CHECK(fdsnn_dev_alloc(ctx, count * stride * 4, &d_in));
    CHECK(fdsnn_dev_alloc(ctx, count * stride * 4, &d_out));
    CHECK(fdsnn_ciphertexts_load_fdsn(ctx, argv[2], argv[3], &count, &ndim, shape, (uint32_t*)d_in, NULL));

    /* sign table: g(m) = +1 on [0, p/2) -> every slot holds Delta = q / p */
    int64_t* tp = (int64_t*)malloc(sizeof(int64_t) * prm.N);
    const int64_t delta = ((int64_t)1 << prm.log2_q) / prm.p;
    for (int i = 0; i < prm.N; ++i) tp[i] = delta;
    int32_t lut = -1;
    CHECK(fdsnn_lut_load(ctx, tp, &lut));

    CHECK(fdsnn_pbs_dev(ctx, 1, &lut, NULL, NULL, (const uint32_t*)d_in, NULL, count, (uint32_t*)d_out, NULL));
    int64_t* A = (int64_t*)malloc(sizeof(int64_t) * count * prm.n);
    int64_t* b = (int64_t*)malloc(sizeof(int64_t) * count);
    CHECK(fdsnn_rows_to_host(ctx, (const uint32_t*)d_out, count, A, b, NULL));
    CHECK(fdsnn_sync(ctx));

    FILE* f = fopen(argv[12], "wb");
    if (!f) return 3;
    fwrite(&count, sizeof(int64_t), 1, f);
    fwrite(A, sizeof(int64_t), (size_t)(count * prm.n), f);
    fwrite(b, sizeof(int64_t), (size_t)count, f);
    fclose(f);
    printf("bootstrapped %lld ciphertexts (tensor ndim %d)\n", (long long)count, ndim);
    CHECK(fdsnn_dev_free(ctx, d_in));
    CHECK(fdsnn_dev_free(ctx, d_out));
    CHECK(fdsnn_ctx_destroy(ctx));
    free(tp);
    free(A);
    free(b);
    return 0;
}
