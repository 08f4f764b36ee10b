/*
 * fdsnn_b200.h — C ABI of the B200-native FHE-DiCSNN hot path.
 *
 * The reference (/root/reference/pkg/src/fdsnn, pure Python + numba) has no
 * FFI layer: its boundary is the Python API on numpy int64 arrays.  Each entry
 * point below replaces one reference call (file:line cited per function); the
 * Python package `paper_2309_09025_b200` binds them with ctypes and keeps the
 * reference names and signatures on top.
 *
 * Conventions
 *  - Host arrays are int64 (the reference's numpy dtype); values are taken
 *    modulo q on entry (two's complement masking), so unreduced negatives are
 *    accepted exactly like `% q` in the reference.
 *  - Device ciphertext storage ("rows"): uint32 row-major, one LWE ciphertext
 *    per row, row = [a_0 .. a_{n-1}, b, pad...], row stride = fdsnn_row_stride().
 *  - Every function returns FDSNN_OK (0) or an error code; the message of the
 *    last error on the calling thread is available from fdsnn_last_error().
 *    The Python layer maps FDSNN_ERR_PARAMETER -> ParameterError and
 *    FDSNN_ERR_DOMAIN -> DomainError (reference errors.py:8-17).
 *  - Calls on one context are serialised on the context's CUDA stream unless a
 *    stream is passed explicitly (`*_dev` entry points).
 *  - There is no CPU fallback: without a usable sm_100 device ctx_create fails.
 *  - No C++ exception crosses this ABI: internal failures (including a
 *    malformed FDSN container) come back as error codes.
 */
#ifndef FDSNN_B200_H
#define FDSNN_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FDSNN_OK 0
#define FDSNN_ERR_PARAMETER 1   /* dimension / modulus mismatch (ParameterError) */
#define FDSNN_ERR_DOMAIN 2      /* value outside its domain (DomainError)        */
#define FDSNN_ERR_CUDA 3        /* CUDA runtime error                            */
#define FDSNN_ERR_STATE 4       /* key not loaded, bad handle, ...               */

/* Mirrors params.FheParams (params.py:36-106) restricted to what the path uses.
 * q, N, p, gadget base and key-switch base are powers of two (validated). */
typedef struct fdsnn_params {
    int32_t n;            /* LWE dimension                                  */
    int32_t N;            /* ring degree (512, 1024 or 2048)                */
    int32_t log2_q;       /* q = 2^log2_q, q <= 2^31                        */
    int32_t p;            /* message modulus                                */
    int32_t bg_log;       /* gadget base = 2^bg_log   (params.gadget.base)  */
    int32_t levels;       /* gadget levels l (2 or 3)                       */
    int32_t ks_log;       /* key-switch base = 2^ks_log                     */
    int32_t ks_levels;    /* key-switch levels                              */
} fdsnn_params;

typedef struct fdsnn_ctx fdsnn_ctx;

const char* fdsnn_last_error(void);
int32_t fdsnn_row_stride(int32_t n);          /* padded row length (words)   */

/* Context: owns device copies of the keys and the CUDA stream. */
int fdsnn_ctx_create(const fdsnn_params* prm, int32_t device, fdsnn_ctx** out);
int fdsnn_ctx_destroy(fdsnn_ctx* ctx);
/* Raw cudaStream_t of the context (for callers that share it). */
void* fdsnn_ctx_stream(fdsnn_ctx* ctx);

/* Load the bootstrapping key and the key-switch key.
 *   rows  : (n, 2l, 2, N) int64 residues — RGSW(s_i) rows [i][row][a|b][coef]
 *           (rgsw.py:141-157 layout, BootstrapKey._ek_fft input bootstrap.py:125-130)
 *   ksk_A : (N*ks_levels, n) int64, ksk_b : (N*ks_levels,) int64
 *           (KeySwitchKey bootstrap.py:99-110, row index j*levels+i)
 * The Fourier transform of the RGSW rows is computed on the device. */
int fdsnn_bsk_load(fdsnn_ctx* ctx, const int64_t* rows, const int64_t* ksk_A,
                   const int64_t* ksk_b);

/* Load only the key-switch key (bootstrap.key_switch_batch with a standalone
 * KeySwitchKey, bootstrap.py:303-316): enough for fdsnn_key_switch_batch,
 * no bootstrapping key is transformed or stored. */
int fdsnn_ksk_load(fdsnn_ctx* ctx, const int64_t* ksk_A, const int64_t* ksk_b);

/* Load the bootstrapping key straight from a reference "FDSN" BK container
 * (serial.save_bootstrap_key, reference serial.py:111-118): arrays ek_a,
 * ek_b (n, 2l, N), ksk_A, ksk_b.  `params_digest` (hex, may be NULL) must
 * equal FheParams.digest() of the context's parameters (serial.py:79-84). */
int fdsnn_bsk_load_fdsn(fdsnn_ctx* ctx, const char* path, const char* params_digest);

/* Read a reference "FDSN" CT container (serial.save_ciphertexts,
 * serial.py:132-137).  Always returns the ciphertext count and the tensor
 * shape (ndim <= 8); when d_rows is non-NULL also uploads the ciphertexts as
 * device rows (count * fdsnn_row_stride(n) words). */
int fdsnn_ciphertexts_load_fdsn(fdsnn_ctx* ctx, const char* path, const char* params_digest,
                                int64_t* count, int32_t* ndim, int64_t* shape,
                                uint32_t* d_rows, void* stream);

/* Register a test polynomial (bootstrap.test_polynomial, bootstrap.py:90-96):
 * N int64 residues.  Returns a LUT id usable by the PBS entry points. */
int fdsnn_lut_load(fdsnn_ctx* ctx, const int64_t* testpoly, int32_t* lut_id);

/* ---- host-buffer entry points (end-to-end; copies inside) ------------- */

/* bootstrap.bootstrap_batch (bootstrap.py:324-341): (count,n),(count,) ->
 * LWE(g(m)) under s, including sample extract and key switch. */
int fdsnn_pbs_batch(fdsnn_ctx* ctx, int32_t lut_id, const int64_t* A,
                    const int64_t* b, int64_t count, int64_t* outA,
                    int64_t* outb);

/* neuron.fhe_lif_step_batch (neuron.py:160-172): h = v + i; spike2 =
 * PBS_fire(h - Delta*v_th_hat) + Delta; v' = PBS_reset(h).  2*count PBS. */
int fdsnn_lif_step_batch(fdsnn_ctx* ctx, int32_t lut_fire, int32_t lut_reset,
                         int64_t v_th_hat, const int64_t* vA, const int64_t* vb,
                         const int64_t* iA, const int64_t* ib, int64_t count,
                         int64_t* sA, int64_t* sb, int64_t* nA, int64_t* nb);

/* bootstrap.blind_rotate_batch (bootstrap.py:252-282): acc (count,2,N) int64
 * residues rotated in place by a2N (count,n) residues mod 2N. */
int fdsnn_blind_rotate_batch(fdsnn_ctx* ctx, int64_t* acc, const int64_t* a2N,
                             int64_t count);

/* bootstrap.key_switch_batch (bootstrap.py:303-316): (count,N),(count,) under
 * z -> (count,n),(count,) under s. */
int fdsnn_key_switch_batch(fdsnn_ctx* ctx, const int64_t* A, const int64_t* b,
                           int64_t count, int64_t* outA, int64_t* outb);

/* network.layer_forward (network.py:409-421): out = M @ [A|b] mod q.
 * M is (out_cells, in_cells) int64 (small integers). */
int fdsnn_weight_sum(fdsnn_ctx* ctx, const int64_t* M, int64_t out_cells,
                     int64_t in_cells, const int64_t* A, const int64_t* b,
                     int64_t* outA, int64_t* outb);

/* ---- device-pointer entry points (device-resident pipeline) ----------- */
/* All `rows` pointers are uint32 device arrays of count * fdsnn_row_stride(n)
 * words.  `stream` may be NULL: the legacy default stream. */

/* Host int64 (A,b) -> device rows (with mod-q masking) and back.  Rows are
 * packed/unpacked on the host by a thread pool in page-locked slots that are
 * DMA'd while the next slot is packed; from_host returns once the host arrays
 * may be reused, to_host once they are complete.  Thread-safe per context. */
int fdsnn_rows_from_host(fdsnn_ctx* ctx, const int64_t* A, const int64_t* b,
                         int64_t count, uint32_t* d_rows, void* stream);
/* Several host arrays stacked in order into one device row buffer (the
 * batched network calls: no host-side concatenation).  counts[p] rows of
 * A[p] (counts[p], n) and b[p] (counts[p],). */
int fdsnn_rows_from_host_parts(fdsnn_ctx* ctx, int32_t nparts, const int64_t* const* A,
                               const int64_t* const* b, const int64_t* counts, uint32_t* d_rows,
                               void* stream);
int fdsnn_rows_to_host(fdsnn_ctx* ctx, const uint32_t* d_rows, int64_t count,
                       int64_t* A, int64_t* b, void* stream);

/* PBS over `count` input rows and `nlut` LUTs: virtual ciphertext v = u*count+r
 * (u < nlut) bootstraps row r (plus optional row r of d_in2: charge v+i) with
 * b shifted by in_boff[u]*Delta before the modulus switch and out_boff[u]*Delta
 * after the key switch; result row v of d_out (nlut*count rows). */
int fdsnn_pbs_dev(fdsnn_ctx* ctx, int32_t nlut, const int32_t* lut_ids,
                  const int64_t* in_boff, const int64_t* out_boff,
                  const uint32_t* d_in, const uint32_t* d_in2, int64_t count,
                  uint32_t* d_out, void* stream);

/* Dense or sparse integer operator on device rows (network.layer_forward).
 * The operator is uploaded once and referenced by id. */
int fdsnn_operator_load(fdsnn_ctx* ctx, const int64_t* M, int64_t out_cells,
                        int64_t in_cells, int32_t* op_id);
/* Applies op to `batch` stacked inputs (batch*in_cells rows) -> batch*out_cells
 * rows.  Exact mod 2^32 accumulation, masked to q. */
int fdsnn_operator_apply(fdsnn_ctx* ctx, int32_t op_id, const uint32_t* d_in,
                         int64_t batch, uint32_t* d_out, void* stream);

/* (x + y) mod q over rows (network.infer score accumulation, network.py:489). */
int fdsnn_rows_add(fdsnn_ctx* ctx, const uint32_t* d_x, const uint32_t* d_y,
                   int64_t count, uint32_t* d_out, void* stream);

/* ---- client-side encryption on the device -------------
 * The randomness is drawn by the caller in the reference's order (masks A on
 * the q/2N grid, rounded-Gaussian e: lwe.encrypt_batch, lwe.py:75-87); the
 * device computes b = <A, s> + e + Delta*m mod q into rows.  sk is the host
 * binary secret (n int64), A (count, n), e and m (count,) host int64.
 * Messages outside {-p/2+1..p/2} -> FDSNN_ERR_DOMAIN. */
int fdsnn_encrypt_rows(fdsnn_ctx* ctx, const int64_t* sk, const int64_t* A, const int64_t* e,
                       const int64_t* m, int64_t count, uint32_t* d_rows, void* stream);
/* lwe.decrypt_batch (lwe.py:89-96) of device rows into host m (count int64);
 * returns when m is on the host. */
int fdsnn_decrypt_rows(fdsnn_ctx* ctx, const int64_t* sk, const uint32_t* d_rows, int64_t count,
                       int64_t* m, void* stream);

/* ---- mod-p plaintext twin (oracle.plain_infer, oracle.py:44-78) ----
 * int64 device vectors, exact integer arithmetic as in the reference numpy. */
/* y[b] = M x[b] for a loaded operator (weight layer on plaintext values). */
int fdsnn_plain_apply(fdsnn_ctx* ctx, int32_t op_id, const int64_t* d_x, int64_t batch,
                      int64_t* d_y, void* stream);
/* neuron.plain_lif_step_batch (neuron.py:107-119): h = v + i; spike2 = 2 if
 * h >= v_th_hat else 0; v' = 0 if fired or h <= 0 else round_half_away(h *
 * leak_num / leak_den).  p > 0 adds the number of h outside [v_th_hat - p/2,
 * p/2) to *d_overflow (the reference raises OverflowViolation). */
int fdsnn_plain_lif(fdsnn_ctx* ctx, const int64_t* d_v, const int64_t* d_i, int64_t count,
                    int64_t v_th_hat, int64_t leak_num, int64_t leak_den, int64_t p,
                    int64_t* d_spike2, int64_t* d_v_next, uint64_t* d_overflow, void* stream);

/* Device memory helpers (so a caller without torch can drive the pipeline). */
int fdsnn_dev_alloc(fdsnn_ctx* ctx, int64_t bytes, void** ptr);
int fdsnn_dev_free(fdsnn_ctx* ctx, void* ptr);
int fdsnn_sync(fdsnn_ctx* ctx);

/* Instrumentation used by bench.py / tests.  `which`: 0 = blind rotation,
 * 1 = key switch, 2 = linear operators.  Returns the summed device time (ms)
 * of that kernel family since the last reset, measured with CUDA events on
 * the launching stream, and the number of kernels launched. */
int fdsnn_timing_enable(fdsnn_ctx* ctx, int32_t on);
int fdsnn_timing_read(fdsnn_ctx* ctx, int32_t which, double* ms, int64_t* launches);
int fdsnn_timing_reset(fdsnn_ctx* ctx);
/* Max |x - round(x)| seen by the inverse transform (exactness margin probe;
 * only tracked when enabled, costs an atomic per thread per step). */
int fdsnn_margin_enable(fdsnn_ctx* ctx, int32_t on);
int fdsnn_margin_read(fdsnn_ctx* ctx, double* max_err);

/* ---- ring / RGSW algebra (host buffers, synchronous, no context) ------
 * The reference's algebra layer for users outside the bootstrapping path
 * (tests, key tooling).  `device` selects the GPU; arrays are host memory.
 * ring.NegacyclicTransform.forward (ring.py:125-131): count real length-N
 * polynomials (float64) -> count x N/2 complex evaluations, interleaved
 * (re, im) float64.  N a power of two in [2, 4096]. */
int fdsnn_nt_forward(int32_t device, int32_t N, const double* coeffs, double* evals, int64_t count);
/* ring.NegacyclicTransform.inverse (ring.py:133-137): unrounded coefficients. */
int fdsnn_nt_inverse(int32_t device, int32_t N, const double* evals, double* coeffs, int64_t count);
/* Exact negacyclic multiply-accumulate mod q = 2^log2_q, replacing
 * ring.poly_mul / poly_mul_schoolbook / negacyclic_mul_raw (ring.py:200-223)
 * and the MAC of rgsw.external_product (rgsw.py:189-192):
 * out[b] = sum_{d<D} x[b][d] * y[b][d] mod (X^N + 1, q); x, y (count, D, N)
 * int64 (any representatives), out (count, N) in [0, q).  Exact at every
 * size (the reference's transform path is exact only while N max|x| max|y|
 * stays below 2^53; where it is, the results are identical). */
int fdsnn_negacyclic_mac(int32_t device, int32_t N, int32_t log2_q, int32_t D, const int64_t* x,
                         const int64_t* y, int64_t* out, int64_t count);
/* rgsw.gadget_decompose (rgsw.py:119-133): signed digits in (-B/2, B/2],
 * lowest level first; x (rows, len) -> digits (rows, levels, len). */
int fdsnn_gadget_decompose(int32_t device, int32_t log2_q, int32_t bg_log, int32_t levels, const int64_t* x,
                           int64_t rows, int64_t len, int64_t* digits);

/* Microbenchmarks for the roofline denominators (run on ctx's device). */
int fdsnn_probe_fp64_peak(fdsnn_ctx* ctx, double* tflops);
int fdsnn_flush_l2(fdsnn_ctx* ctx, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* FDSNN_B200_H */
