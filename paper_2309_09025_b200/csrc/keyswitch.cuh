// keyswitch.cuh — batched LWE key switching z (dim N) -> s (dim n).
//
// Reference: bootstrap.key_switch_batch (bootstrap.py:303-316) with
// rgsw.gadget_decompose (rgsw.py:119-133):
//   digits of centred a_j, base 2^ks_log, ks_L levels, lowest first,
//   flattened index j*ks_L + t;
//   out_a = -sum digit * kskA  (mod q),  out_b = b - sum digit * kskb (mod q).
// The reference evaluates the sums as exact float64 GEMMs; here they are
// int32 GEMMs with wrap-around modulo 2^32, which is exact modulo q = 2^k.
//
// Device KSK layout: (N*ks_L) x stride uint32, columns [kskA (n) | kskb | pad].
// The mask GEMM normally runs on the tensor cores (ks_umma.cuh); the CUDA-core
// ks_mask_kernel below serves parameter sets outside the int8 bounds.
#pragma once
#include "common.cuh"

namespace fdsnn {

constexpr int KS_ROWS = 64;   // ciphertexts per CTA tile
constexpr int KS_COLS = 128;  // output mask columns per CTA tile
constexpr int KS_CK = 8;      // ring coefficients per K chunk

struct KsArgs {
    DevParams prm;
    const uint32_t* ext;   // V x ext_stride (z-LWE rows, a'_0..a'_{N-1}, b')
    int64_t V;
    const uint32_t* ksk;   // (N*ks_L) x stride
    const uint32_t* kskb;  // (N*ks_L) body column, contiguous (coalesced reads)
    uint32_t* out;         // V x stride
    int64_t count;         // rows per LUT (for out_boff selection)
    uint32_t out_boff[4];  // added to the output body, per LUT (mod q)
};

FDSNN_DEV int32_t ks_digit(int32_t& x, int ks_log) {
    const int32_t half1 = (1 << (ks_log - 1)) - 1;
    const int32_t d = ((x + half1) & ((1 << ks_log) - 1)) - half1;
    x = (x - d) >> ks_log;
    return d;
}

// Mask columns: out[v][c] = -sum_k dig[v][k] * ksk[k][c]   (c < n)
template <int KSL>
__global__ void __launch_bounds__(256) ks_mask_kernel(const KsArgs args) {
    const DevParams& prm = args.prm;
    constexpr int KC = KS_CK * KSL;
    __shared__ __align__(16) int32_t dig[KC][KS_ROWS];
    __shared__ __align__(16) uint32_t key[KC][KS_COLS];
    const int tx = threadIdx.x % 32;  // column group: 4 columns
    const int ty = threadIdx.x / 32;  // row group: 8 rows
    const int64_t row0 = (int64_t)blockIdx.x * KS_ROWS;
    const int col0 = blockIdx.y * KS_COLS;
    const int n = prm.n;
    uint32_t acc[8][4];
#pragma unroll
    for (int a = 0; a < 8; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) acc[a][b] = 0u;

    for (int j0 = 0; j0 < prm.N; j0 += KS_CK) {
        // decompose KS_ROWS x KS_CK coefficients (2 per thread)
        for (int e = threadIdx.x; e < KS_ROWS * KS_CK; e += blockDim.x) {
            const int rr = e / KS_CK, cc = e % KS_CK;
            const int64_t v = row0 + rr;
            int32_t x = 0;
            if (v < args.V) x = center_q(args.ext[v * prm.ext_stride + j0 + cc], prm.log2q);
#pragma unroll
            for (int lv = 0; lv < KSL; ++lv) dig[cc * KSL + lv][rr] = ks_digit(x, prm.ks_log);
        }
        // key tile rows (j0*KSL .. +KC) x columns col0 .. col0+KS_COLS
        for (int e = threadIdx.x; e < KC * (KS_COLS / 4); e += blockDim.x) {
            const int kr = e / (KS_COLS / 4), kc = (e % (KS_COLS / 4)) * 4;
            const int col = col0 + kc;
            uint4 val = make_uint4(0, 0, 0, 0);
            if (col < prm.stride)
                val = *reinterpret_cast<const uint4*>(args.ksk + (size_t)(j0 * KSL + kr) * prm.stride + col);
            *reinterpret_cast<uint4*>(&key[kr][kc]) = val;
        }
        __syncthreads();
#pragma unroll 4
        for (int kk = 0; kk < KC; ++kk) {
            const int4 d0 = *reinterpret_cast<const int4*>(&dig[kk][ty * 8]);
            const int4 d1 = *reinterpret_cast<const int4*>(&dig[kk][ty * 8 + 4]);
            const uint4 kv = *reinterpret_cast<const uint4*>(&key[kk][tx * 4]);
            const int32_t dd[8] = {d0.x, d0.y, d0.z, d0.w, d1.x, d1.y, d1.z, d1.w};
            const uint32_t kk4[4] = {kv.x, kv.y, kv.z, kv.w};
#pragma unroll
            for (int a = 0; a < 8; ++a)
#pragma unroll
                for (int b = 0; b < 4; ++b) acc[a][b] += (uint32_t)dd[a] * kk4[b];
        }
        __syncthreads();
    }
#pragma unroll
    for (int a = 0; a < 8; ++a) {
        const int64_t v = row0 + ty * 8 + a;
        if (v >= args.V) continue;
#pragma unroll
        for (int b = 0; b < 4; ++b) {
            const int col = col0 + tx * 4 + b;
            if (col < n) args.out[v * prm.stride + col] = (0u - acc[a][b]) & prm.qmask;
            else if (col > n && col < prm.stride) args.out[v * prm.stride + col] = 0u;
        }
    }
}

// Body column: out[v][n] = b' - sum_k dig[v][k] * kskb[k] + out_boff (mod q),
// and the row padding (zeros).  One warp per ciphertext.
template <int KSL>
__global__ void __launch_bounds__(256) ks_body_kernel(const KsArgs args) {
    const DevParams& prm = args.prm;
    const int lane = threadIdx.x % 32;
    const int64_t v = (int64_t)blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
    if (v >= args.V) return;
    const uint32_t* e = args.ext + v * prm.ext_stride;
    uint32_t s = 0;
    for (int j = lane; j < prm.N; j += 32) {
        int32_t x = center_q(e[j], prm.log2q);
#pragma unroll
        for (int lv = 0; lv < KSL; ++lv) {
            const int32_t d = ks_digit(x, prm.ks_log);
            s += (uint32_t)d * __ldg(args.kskb + j * KSL + lv);
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) {
        const int u = (int)(v / args.count);
        args.out[v * prm.stride + prm.n] = (e[prm.N] - s + args.out_boff[u]) & prm.qmask;
    } else if (prm.n + lane < prm.stride) {
        args.out[v * prm.stride + prm.n + lane] = 0u;  // row padding
    }
}

}  // namespace fdsnn
