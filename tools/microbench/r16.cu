// Warp-per-transform (fft16.cuh) check and throughput probe on B200.
//  1. exactness: negacyclic products d * k (digits |d| < 2^12, key |k| < 2^24,
//     N = 1024) through forward(d) x key_transform(k) -> inverse, vs the exact
//     integer product on the host; key-transform outputs vs a host DFT at the
//     documented (lane, register) -> frequency positions.
//  2. throughput: the CMux-step skeleton per warp (4 forward transforms, MAC
//     against a shared-memory key into 2 spectra, 2 inverse transforms),
//     8 warps/SM, twiddles from TMEM -> cycles per accumulator-step per SM
//     (8 vs 12 warps per SM: r16occ.cu).
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../../paper_2309_09025_b200/csrc -o r16 r16.cu
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>
#include <complex>
#include <random>
#include <cuda_runtime.h>
#include "fft16.cuh"
using namespace fdsnn;

constexpr int N = 1024, M = 512;

__global__ void k_polymul(const int32_t* dig, const int64_t* key, const double2* tab, int64_t* out,
                          double2* keyf, double* err) {
    __shared__ double2 xbuf[r16::XBUF];
    const int lane = threadIdx.x;
    const int test = blockIdx.x;
    const r16::TabGlobal tp{tab + lane * r16::TAB};
    const double2* t = tab + lane * r16::TAB;
    const int32_t* d = dig + test * N;
    const int64_t* k = key + test * N;
    double2 kv[16], dv[16];
    for (int j2 = 0; j2 < 16; ++j2) {
        const int p = lane + 32 * j2;
        kv[j2] = make_double2((double)k[p], (double)k[p + M]);
        dv[j2] = make_double2((double)d[p], (double)d[p + M]);
    }
    r16::forward(kv, lane, tp, xbuf);
    const int a = lane & 1;
    for (int r = 0; r < 8; ++r) {
        if (a) {  // odd lanes: back to the true basis (conj(s))
            const double2 z = t[8 * r16::BLK_ZJ + r];
            kv[r] = cmulc(kv[r], z);
            kv[r + 8] = cmulc(kv[r + 8], z);
            kv[r + 8] = make_double2(-kv[r + 8].x, -kv[r + 8].y);
        }
    }
    for (int i = 0; i < 16; ++i) keyf[(test * 16 + i) * 32 + lane] = kv[i];
    r16::forward(dv, lane, tp, xbuf);
    for (int i = 0; i < 16; ++i) dv[i] = cmul(dv[i], make_double2(kv[i].x / M, kv[i].y / M));
    r16::inverse(dv, lane, tp, xbuf);
    double e = 0;
    for (int j2 = 0; j2 < 16; ++j2) {
        const int p = lane + 32 * j2;
        const double2 z = cmulc(dv[j2], r16::g_twist(j2));  // register untwist (the lane factor is applied by inverse())
        const long long r0 = __double2ll_rn(z.x), r1 = __double2ll_rn(z.y);
        e = fmax(e, fabs(z.x - (double)r0));
        e = fmax(e, fabs(z.y - (double)r1));
        out[test * N + p] = r0;
        out[test * N + p + M] = r1;
    }
    err[test * 32 + lane] = e;
}

// ---- throughput skeleton ----
FDSNN_DEV void ld_c8(uint32_t taddr, double2 (&c)[8]) {
    uint32_t w[32];
    tmem_ld32_async(taddr, w);
    tmem_wait32(w);
#pragma unroll
    for (int i = 0; i < 8; ++i) c[i] = words_c(w, i);
}
FDSNN_DEV void ld_c16(uint32_t taddr, double2 (&c)[16]) {
    uint32_t w0[32], w1[32];
    tmem_ld32_async(taddr, w0);
    tmem_ld32_async(taddr + 32, w1);
    tmem_wait64(w0, w1);
#pragma unroll
    for (int i = 0; i < 8; ++i) { c[i] = words_c(w0, i); c[i + 8] = words_c(w1, i); }
}

template <int P1_TMEM>
__global__ void __launch_bounds__(256, 1) k_step(const double2* tab, const double2* gkey, double* out, int steps) {
    extern __shared__ __align__(128) unsigned char sm[];
    __shared__ uint32_t tslot;
    double2* key = reinterpret_cast<double2*>(sm);                 // 4 chunks x 1024
    double2* xb = key + 4 * 1024 + (threadIdx.x / 32) * r16::XBUF;
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    for (int i = threadIdx.x; i < 4096; i += 256) key[i] = gkey[i];
    if (warp == 0) tmem_alloc(&tslot, 512);
    tmem_fence_before();
    __syncthreads();
    tmem_fence_after();
    const uint32_t lb = tslot + ((uint32_t)((warp % 4) * 32) << 16);
    if (warp < 4) {
        const double2* t = tab + lane * r16::TAB;
        for (int c = 0; c < r16::TAB / 8; ++c) {
            uint32_t w[32];
            for (int i = 0; i < 8; ++i) put_words_c(w, i, t[8 * c + i]);
            tmem_st32(lb + 32 * c, w);
        }
        tmem_wait_st();
    }
    tmem_fence_before();
    __syncthreads();
    tmem_fence_after();
    const uint32_t pcol = lb + 224 + 64 * (warp / 4);
    const r16::TabTmem tp{lb};
    double sink = 0;
    for (int s = 0; s < steps; ++s) {
        double2 P0[16], P1[16];
        for (int d = 0; d < 4; ++d) {
            double2 v[16];
#pragma unroll
            for (int j = 0; j < 16; ++j) v[j] = make_double2((double)((lane + j + s + d) & 63) - 31.0, (double)(j - 7));
            r16::forward(v, lane, tp, xb);
            const double2* k = key + d * 1024;
#pragma unroll
            for (int i = 0; i < 16; ++i) {
                if (d == 0) P0[i] = make_double2(0, 0);
                cmac(P0[i], v[i], k[i * 32 + lane]);
            }
            if (P1_TMEM) {
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    uint32_t w[32];
                    double2 q[8];
                    if (d > 0) {
                        tmem_ld32_async(pcol + 32 * h, w);
                        tmem_wait32(w);
                    }
#pragma unroll
                    for (int i = 0; i < 8; ++i) {
                        q[i] = d > 0 ? words_c(w, i) : make_double2(0, 0);
                        cmac(q[i], v[8 * h + i], k[512 + (8 * h + i) * 32 + lane]);
                        put_words_c(w, i, q[i]);
                    }
                    tmem_st32(pcol + 32 * h, w);
                }
                tmem_wait_st();
            } else {
#pragma unroll
                for (int i = 0; i < 16; ++i) {
                    if (d == 0) P1[i] = make_double2(0, 0);
                    cmac(P1[i], v[i], k[512 + i * 32 + lane]);
                }
            }
        }
        r16::inverse(P0, lane, tp, xb);
        if (P1_TMEM) ld_c16(pcol, P1);
        r16::inverse(P1, lane, tp, xb);
#pragma unroll
        for (int i = 0; i < 16; ++i) sink += P0[i].x + P1[i].y;
    }
    out[blockIdx.x * 256 + threadIdx.x] = sink;
    tmem_fence_before();
    __syncthreads();
    if (warp == 0) { tmem_fence_after(); tmem_dealloc(tslot, 512); }
}


int main() {
    // ---- tables
    std::vector<double2> tab(32 * r16::TAB);
    r16::build_table(N, tab.data(), [](long double c, long double s) { return make_double2((double)c, (double)s); });
    double2* d_tab;
    cudaMalloc(&d_tab, tab.size() * sizeof(double2));
    cudaMemcpy(d_tab, tab.data(), tab.size() * sizeof(double2), cudaMemcpyHostToDevice);
    // ---- exactness
    const int TESTS = 64;
    std::mt19937_64 rng(7);
    std::vector<int32_t> dig(TESTS * N);
    std::vector<int64_t> key(TESTS * N);
    for (auto& x : dig) x = (int32_t)(rng() % 8191) - 4095;
    for (auto& x : key) x = (int64_t)(rng() % (1 << 24)) - (1 << 23);
    int32_t* d_dig; int64_t *d_key, *d_out; double2* d_kf; double* d_err;
    cudaMalloc(&d_dig, dig.size() * 4); cudaMalloc(&d_key, key.size() * 8); cudaMalloc(&d_out, key.size() * 8);
    cudaMalloc(&d_kf, TESTS * 512 * sizeof(double2)); cudaMalloc(&d_err, TESTS * 32 * 8);
    cudaMemcpy(d_dig, dig.data(), dig.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(d_key, key.data(), key.size() * 8, cudaMemcpyHostToDevice);
    k_polymul<<<TESTS, 32>>>(d_dig, d_key, d_tab, d_out, d_kf, d_err);
    cudaError_t ce = cudaDeviceSynchronize();
    if (ce != cudaSuccess) { printf("polymul: %s\n", cudaGetErrorString(ce)); return 1; }
    std::vector<int64_t> out(TESTS * N);
    std::vector<double2> kf(TESTS * 512);
    std::vector<double> err(TESTS * 32);
    cudaMemcpy(out.data(), d_out, out.size() * 8, cudaMemcpyDeviceToHost);
    cudaMemcpy(kf.data(), d_kf, kf.size() * sizeof(double2), cudaMemcpyDeviceToHost);
    cudaMemcpy(err.data(), d_err, err.size() * 8, cudaMemcpyDeviceToHost);
    long bad = 0;
    double emax = 0;
    for (double e : err) emax = std::max(emax, e);
    for (int t = 0; t < TESTS; ++t) {
        std::vector<int64_t> ref(N, 0);
        for (int i = 0; i < N; ++i)
            for (int j = 0; j < N; ++j) {
                const int64_t pr = (int64_t)dig[t * N + i] * key[t * N + j];
                if (i + j < N) ref[i + j] += pr; else ref[i + j - N] -= pr;
            }
        for (int m = 0; m < N; ++m) bad += ref[m] != out[t * N + m];
    }
    // key transform vs host DFT (test 0, a few frequencies per lane)
    double kdev = 0, kmag = 0;
    {
        const long double PI = 3.141592653589793238462643383279502884L;
        std::vector<std::complex<long double>> c(M);
        for (int j = 0; j < M; ++j)
            c[j] = std::complex<long double>((long double)key[j], (long double)key[j + M]) *
                   std::polar(1.0L, PI * j / N);
        for (int lane = 0; lane < 32; ++lane)
            for (int i = 0; i < 16; ++i) {
                const int r = i & 7, dd = i >> 3, k2p = lane >> 1, a = lane & 1;
                const int f = k2p + 16 * (r + 8 * a) + 256 * dd;
                std::complex<long double> X = 0;
                for (int j = 0; j < M; ++j) X += c[j] * std::polar(1.0L, 2.0L * PI * (long double)((j * f) % M) / M);
                const double2 g = kf[i * 32 + lane];
                kdev = std::max(kdev, (double)std::abs(X - std::complex<long double>(g.x, g.y)));
                kmag = std::max(kmag, (double)std::abs(X));
            }
    }
    printf("exactness: %d products x %d coefficients, mismatches %ld, max |x - round(x)| %.4g; key transform max dev %.3g (max |X| %.3g)\n",
           TESTS, N, bad, emax, kdev, kmag);
    // ---- throughput
    std::vector<double2> hk(4096);
    for (int i = 0; i < 4096; ++i) hk[i] = make_double2(1e-3 * (i % 17), -1e-3 * (i % 13));
    double2* d_k; double* d_o;
    cudaMalloc(&d_k, 4096 * sizeof(double2));
    cudaMalloc(&d_o, 148 * 4 * 256 * 8);
    double* d_o2;
    cudaMalloc(&d_o2, 148 * 4 * 512 * 8);
    cudaMemcpy(d_k, hk.data(), 4096 * sizeof(double2), cudaMemcpyHostToDevice);
    const size_t smem = 4 * 1024 * sizeof(double2) + 8 * r16::XBUF * sizeof(double2);
    auto run = [&](auto kern, const char* name) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        const int steps = 512;
        kern<<<148, 256, smem>>>(d_tab, d_k, d_o, 8);
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0); cudaEventCreate(&e1);
        cudaEventRecord(e0);
        kern<<<148 * 4, 256, smem>>>(d_tab, d_k, d_o, steps);
        cudaEventRecord(e1);
        cudaError_t ce2 = cudaEventSynchronize(e1);
        if (ce2 != cudaSuccess) { printf("%s: %s\n", name, cudaGetErrorString(ce2)); return; }
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        const double acc_steps_per_sm = 4.0 * 8 * steps;  // 4 CTAs per SM in sequence, 8 warps each
        const double cyc = ms * 1e-3 * 1.965e9;
        printf("%s: %.3f ms, %.0f cycles per accumulator-step per SM (current kernel: ~3050 incl. all overheads)\n",
               name, ms, cyc / acc_steps_per_sm);
    };
    run(k_step<0>, "skeleton P1 in registers");
    run(k_step<1>, "skeleton P1 in TMEM     ");
    return 0;
}
