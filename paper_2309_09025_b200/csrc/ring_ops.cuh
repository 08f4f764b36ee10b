// ring_ops.cuh — device kernels behind the reference's ring / RGSW algebra
// API (ring.NegacyclicTransform, poly_mul, poly_mul_schoolbook,
// rgsw.gadget_decompose, rgsw.external_product).  These serve single
// polynomials and small batches (tests, key tooling, users of the algebra
// layer); the bootstrapping hot path has its own fused kernels (pbs.cuh).
#pragma once
#include "common.cuh"

namespace fdsnn {

// ---------------------------------------------------------------------------
// Negacyclic transform of one real length-N polynomial per CTA
// (ring.py:103-137): forward c_k = (a_k + i a_{k+M}) e^{i pi k/N}, then the
// unnormalised M-point DFT with the e^{+2 pi i jk/M} kernel; inverse: the
// e^{-} DFT / M, times e^{-i pi k/N}, real parts then imaginary parts.
// Iterative radix-2 in shared memory (bit-reversed load), twiddles from
// sincospi in FP64.  M <= 2048 (N <= 4096).
// ---------------------------------------------------------------------------
template <bool INV>
__global__ void nt_fft_kernel(int N, const double* __restrict__ in, double* __restrict__ out) {
    extern __shared__ double2 xs[];
    const int M = N / 2;
    const int logM = 31 - __clz(M);
    const int64_t poly = blockIdx.x;
    const double sgn = INV ? -1.0 : 1.0;
    for (int k = threadIdx.x; k < M; k += blockDim.x) {
        double2 c;
        if constexpr (!INV) {
            const double* a = in + poly * N;
            double s, co;
            sincospi((double)k / (double)N, &s, &co);  // twist e^{i pi k/N}
            const double re = a[k], im = a[k + M];
            c = make_double2(re * co - im * s, re * s + im * co);
        } else {
            const double* e = in + poly * 2 * M;
            c = make_double2(e[2 * k], e[2 * k + 1]);
        }
        const int r = logM ? (int)(__brev((unsigned)k) >> (32 - logM)) : 0;
        xs[r] = c;
    }
    __syncthreads();
    for (int len = 2; len <= M; len <<= 1) {
        const int half = len >> 1;
        for (int b = threadIdx.x; b < M / 2; b += blockDim.x) {
            const int pos = b & (half - 1);
            const int j0 = (b - pos) * 2 + pos, j1 = j0 + half;
            double s, co;
            sincospi(2.0 * (double)pos / (double)len, &s, &co);
            const double2 w = make_double2(co, sgn * s);
            const double2 u = xs[j0], v = cmul(xs[j1], w);
            xs[j0] = cadd(u, v);
            xs[j1] = csub(u, v);
        }
        __syncthreads();
    }
    for (int k = threadIdx.x; k < M; k += blockDim.x) {
        const double2 c = xs[k];
        if constexpr (!INV) {
            double* e = out + poly * 2 * M;
            e[2 * k] = c.x;
            e[2 * k + 1] = c.y;
        } else {
            double s, co;
            sincospi((double)k / (double)N, &s, &co);  // untwist e^{-i pi k/N}
            const double re = c.x / M, im = c.y / M;
            double* a = out + poly * N;
            a[k] = re * co + im * s;
            a[k + M] = im * co - re * s;
        }
    }
}

// ---------------------------------------------------------------------------
// Exact negacyclic multiply-accumulate mod q = 2^log2q (ring.py:200-223):
// out[b] = sum_{d<D} x[b][d] * y[b][d]  mod (X^N + 1, q).  Arithmetic is
// uint64 with wraparound, i.e. exact modulo 2^64 and therefore modulo q, so
// inputs may be any int64 representatives.  Grid (count, ceil(N/blockDim)):
// each thread owns one output coefficient j and runs the O(N) convolution
// sum from shared memory (x broadcast, y read at consecutive j - i).
// ---------------------------------------------------------------------------
__global__ void negacyclic_mac_kernel(int N, uint64_t qmask, int D, const int64_t* __restrict__ x,
                                      const int64_t* __restrict__ y, int64_t* __restrict__ out) {
    extern __shared__ uint64_t sm[];
    uint64_t* xs = sm;
    uint64_t* ys = sm + N;
    const int64_t b = blockIdx.x;
    const int j = blockIdx.y * blockDim.x + threadIdx.x;
    uint64_t acc = 0;
    for (int d = 0; d < D; ++d) {
        __syncthreads();
        for (int i = threadIdx.x; i < N; i += blockDim.x) {
            xs[i] = (uint64_t)x[(b * D + d) * N + i];
            ys[i] = (uint64_t)y[(b * D + d) * N + i];
        }
        __syncthreads();
        if (j < N) {
            uint64_t pos = 0, neg = 0;
            for (int i = 0; i <= j; ++i) pos += xs[i] * ys[j - i];
            for (int i = j + 1; i < N; ++i) neg += xs[i] * ys[N + j - i];
            acc += pos - neg;
        }
    }
    if (j < N) out[b * N + j] = (int64_t)(acc & qmask);
}

// ---------------------------------------------------------------------------
// Signed gadget digits (rgsw.py:119-133), lowest level first, digits in
// (-B/2, B/2]: with y = centred(x) + H, H = (B/2 - 1)(1 + B + ... +
// B^(levels-1)), digit i = ((y >> i*bg) & (B-1)) - (B/2 - 1) (the offset
// absorbs the carries).  x (rows, len) -> out (rows, levels, len).
// ---------------------------------------------------------------------------
__global__ void gadget_digits_kernel(int log2q, int bg, int levels, const int64_t* __restrict__ x,
                                     int64_t rows, int64_t len, int64_t* __restrict__ out) {
    const int64_t total = rows * len;
    const uint64_t qmask = (log2q >= 64) ? ~0ull : ((1ull << log2q) - 1);
    const int64_t half = (int64_t)1 << (bg - 1);
    int64_t H = 0;
    for (int i = 0; i < levels; ++i) H += (half - 1) << (bg * i);
    for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < total;
         g += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = g / len, c = g - r * len;
        const uint64_t v = (uint64_t)x[g] & qmask;
        const int64_t centred = v >= (qmask >> 1) + 1 ? (int64_t)v - (int64_t)(qmask + 1) : (int64_t)v;
        const uint64_t yy = (uint64_t)(centred + H);
        for (int i = 0; i < levels; ++i)
            out[(r * levels + i) * len + c] = (int64_t)((yy >> (bg * i)) & ((1ull << bg) - 1)) - (half - 1);
    }
}

}  // namespace fdsnn
