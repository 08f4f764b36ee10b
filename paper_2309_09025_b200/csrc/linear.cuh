// linear.cuh — homomorphic weighted sums (network.layer_forward,
// reference network.py:409-421): out = M @ [A | b] mod q for an integer
// operator M (conv / pool / linear, all lowered to (out_cells, in_cells)).
//
// The reference computes the product in float64 (asserted exact, :417) and
// reduces mod q.  Here: int32 multiply-accumulate with wrap-around mod 2^32,
// exact modulo q = 2^k, on the uint32 row layout.  Two kernels:
//   * dense tiled GEMM (fully connected layers), weight tile reused across a
//     128-column ciphertext tile, ciphertext tile reused across 64 rows;
//   * CSR gather (conv / pool lowered matrices are >95% zeros: 25 non-zeros
//     per conv row), one CTA per output row, 16-byte column vectors.
#pragma once
#include "common.cuh"

namespace fdsnn {

constexpr int LIN_ROWS = 64;
constexpr int LIN_COLS = 128;
constexpr int LIN_K = 16;

// Dense: Wm (out x in) int32 row-major; X batch-stacked rows (batch*in x stride).
// A CTA computes RPT*8 output rows x LIN_COLS columns (8 warps, each thread
// RPT rows x 4 columns); RPT = 8 for large operators, 4 when the grid would
// otherwise fill less than two waves of SMs.
template <int RPT = 8>
__global__ void __launch_bounds__(256)
linear_dense_kernel(const int32_t* __restrict__ Wm, int out_cells, int in_cells,
                    const uint32_t* __restrict__ X, uint32_t* __restrict__ Y,
                    int stride, uint32_t qmask) {
    constexpr int TR = 8 * RPT;
    constexpr int WE = (LIN_K * TR + 255) / 256;            // weight elements per thread per stage
    constexpr int XE = (LIN_K * (LIN_COLS / 4) + 255) / 256;  // 16-byte ciphertext vectors per thread
    __shared__ __align__(16) int32_t ws[2][LIN_K][TR];
    __shared__ __align__(16) uint32_t xs[2][LIN_K][LIN_COLS];
    const int tx = threadIdx.x % 32, ty = threadIdx.x / 32;
    const int r0 = blockIdx.x * TR;
    const int c0 = blockIdx.y * LIN_COLS;
    const int bidx = blockIdx.z;
    const uint32_t* Xb = X + (size_t)bidx * in_cells * stride;
    uint32_t* Yb = Y + (size_t)bidx * out_cells * stride;
    uint32_t acc[RPT][4];
#pragma unroll
    for (int a = 0; a < RPT; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) acc[a][b] = 0u;
    // stage k0's tiles are fetched into registers one stage ahead (the global
    // latency hides behind the current stage's multiply-adds), then stored
    // into the other shared-memory buffer
    int32_t wreg[WE];
    uint4 xreg[XE];
    auto fetch = [&](int k0) {
#pragma unroll
        for (int u = 0; u < WE; ++u) {
            const int e = threadIdx.x + u * 256;
            const int rr = e / LIN_K, kk = e % LIN_K;
            const int r = r0 + rr, k = k0 + kk;
            wreg[u] = (e < LIN_K * TR && r < out_cells && k < in_cells) ? __ldg(Wm + (size_t)r * in_cells + k) : 0;
        }
#pragma unroll
        for (int u = 0; u < XE; ++u) {
            const int e = threadIdx.x + u * 256;
            const int kk = e / (LIN_COLS / 4), cc = (e % (LIN_COLS / 4)) * 4;
            const int k = k0 + kk, c = c0 + cc;
            xreg[u] = (e < LIN_K * (LIN_COLS / 4) && k < in_cells && c < stride)
                          ? __ldg(reinterpret_cast<const uint4*>(Xb + (size_t)k * stride + c))
                          : make_uint4(0, 0, 0, 0);
        }
    };
    auto put = [&](int buf) {
#pragma unroll
        for (int u = 0; u < WE; ++u) {
            const int e = threadIdx.x + u * 256;
            if (e < LIN_K * TR) ws[buf][e % LIN_K][e / LIN_K] = wreg[u];
        }
#pragma unroll
        for (int u = 0; u < XE; ++u) {
            const int e = threadIdx.x + u * 256;
            if (e < LIN_K * (LIN_COLS / 4))
                *reinterpret_cast<uint4*>(&xs[buf][e / (LIN_COLS / 4)][(e % (LIN_COLS / 4)) * 4]) = xreg[u];
        }
    };
    fetch(0);
    put(0);
    __syncthreads();
    int buf = 0;
    for (int k0 = 0; k0 < in_cells; k0 += LIN_K, buf ^= 1) {
        const bool more = k0 + LIN_K < in_cells;
        if (more) fetch(k0 + LIN_K);
#pragma unroll
        for (int kk = 0; kk < LIN_K; ++kk) {
            int32_t wd[RPT];
#pragma unroll
            for (int a = 0; a < RPT; a += 4) {
                const int4 w4 = *reinterpret_cast<const int4*>(&ws[buf][kk][ty * RPT + a]);
                wd[a] = w4.x; wd[a + 1] = w4.y; wd[a + 2] = w4.z; wd[a + 3] = w4.w;
            }
            const uint4 xv = *reinterpret_cast<const uint4*>(&xs[buf][kk][tx * 4]);
            const uint32_t xd[4] = {xv.x, xv.y, xv.z, xv.w};
#pragma unroll
            for (int a = 0; a < RPT; ++a)
#pragma unroll
                for (int b = 0; b < 4; ++b) acc[a][b] += (uint32_t)wd[a] * xd[b];
        }
        if (more) put(buf ^ 1);  // the other buffer's last readers passed the previous barrier
        __syncthreads();
    }
#pragma unroll
    for (int a = 0; a < RPT; ++a) {
        const int r = r0 + ty * RPT + a;
        if (r >= out_cells) continue;
        const int c = c0 + tx * 4;
        if (c < stride) {
            uint4 o = make_uint4(acc[a][0] & qmask, acc[a][1] & qmask, acc[a][2] & qmask,
                                 acc[a][3] & qmask);
            *reinterpret_cast<uint4*>(Yb + (size_t)r * stride + c) = o;
        }
    }
}

// The last few columns of the rows ([c0, stride): the body b and the row
// padding when n is a multiple of the 128-column tile) as warp dot products,
// so the dense kernel's grid covers only full column tiles.  One warp per
// (batch, output row); each lane sums a strided slice of the input rows for
// up to 4 columns, then the warp reduces.
__global__ void __launch_bounds__(256)
linear_tail_kernel(const int32_t* __restrict__ Wm, int out_cells, int in_cells, const uint32_t* __restrict__ X,
                   uint32_t* __restrict__ Y, int stride, int c0, uint32_t qmask, int batch) {
    const int lane = threadIdx.x % 32;
    const int64_t wid = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / 32;
    if (wid >= (int64_t)batch * out_cells) return;
    const int bidx = (int)(wid / out_cells), r = (int)(wid % out_cells);
    const uint32_t* Xb = X + (size_t)bidx * in_cells * stride + c0;
    const int32_t* w = Wm + (size_t)r * in_cells;
    uint32_t s0 = 0, s1 = 0, s2 = 0, s3 = 0;
    for (int k = lane; k < in_cells; k += 32) {
        const uint32_t wk = (uint32_t)__ldg(w + k);
        const uint4 xv = __ldg(reinterpret_cast<const uint4*>(Xb + (size_t)k * stride));
        s0 += wk * xv.x; s1 += wk * xv.y; s2 += wk * xv.z; s3 += wk * xv.w;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        s0 += __shfl_xor_sync(0xffffffffu, s0, o);
        s1 += __shfl_xor_sync(0xffffffffu, s1, o);
        s2 += __shfl_xor_sync(0xffffffffu, s2, o);
        s3 += __shfl_xor_sync(0xffffffffu, s3, o);
    }
    if (lane == 0)
        *reinterpret_cast<uint4*>(Y + ((size_t)bidx * out_cells + r) * stride + c0) =
            make_uint4(s0 & qmask, s1 & qmask, s2 & qmask, s3 & qmask);
}

// CSR: row_ptr (out+1), col_idx/val (nnz).  grid = (out_cells, batch).
__global__ void __launch_bounds__(160)
linear_csr_kernel(const int32_t* __restrict__ row_ptr, const int32_t* __restrict__ col_idx,
                  const int32_t* __restrict__ val, int out_cells, int in_cells,
                  const uint32_t* __restrict__ X, uint32_t* __restrict__ Y, int stride,
                  uint32_t qmask) {
    const int r = blockIdx.x;
    const int bidx = blockIdx.y;
    const uint32_t* Xb = X + (size_t)bidx * in_cells * stride;
    uint32_t* Yb = Y + (size_t)bidx * out_cells * stride;
    const int beg = row_ptr[r], end = row_ptr[r + 1];
    for (int c = threadIdx.x * 4; c < stride; c += blockDim.x * 4) {
        uint32_t s0 = 0, s1 = 0, s2 = 0, s3 = 0;
        for (int e = beg; e < end; ++e) {
            const uint32_t w = (uint32_t)__ldg(val + e);
            const uint4 xv = __ldg(reinterpret_cast<const uint4*>(Xb + (size_t)__ldg(col_idx + e) * stride + c));
            s0 += w * xv.x; s1 += w * xv.y; s2 += w * xv.z; s3 += w * xv.w;
        }
        *reinterpret_cast<uint4*>(Yb + (size_t)r * stride + c) =
            make_uint4(s0 & qmask, s1 & qmask, s2 & qmask, s3 & qmask);
    }
}

__global__ void rows_add_kernel(const uint32_t* __restrict__ x, const uint32_t* __restrict__ y,
                                uint32_t* __restrict__ out, int64_t words, uint32_t qmask) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < words;
         i += (int64_t)gridDim.x * blockDim.x)
        out[i] = (x[i] + y[i]) & qmask;
}

// int64 host-layout (A,b) -> uint32 rows (mod q); pad columns zeroed.
__global__ void rows_pack_kernel(const int64_t* __restrict__ A, const int64_t* __restrict__ b,
                                 int64_t count, int n, int stride, uint32_t qmask,
                                 uint32_t* __restrict__ rows) {
    const int64_t total = count * stride;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = i / stride;
        const int c = (int)(i - r * stride);
        uint32_t v = 0;
        if (c < n) v = (uint32_t)(A[r * n + c]) & qmask;
        else if (c == n) v = (uint32_t)(b[r]) & qmask;
        rows[i] = v;
    }
}

__global__ void rows_unpack_kernel(const uint32_t* __restrict__ rows, int64_t count, int n,
                                   int stride, int64_t* __restrict__ A, int64_t* __restrict__ b) {
    const int64_t total = count * (n + 1);
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = i / (n + 1);
        const int c = (int)(i - r * (n + 1));
        const uint32_t v = rows[r * stride + c];
        if (c < n) A[r * n + c] = (int64_t)v;
        else b[r] = (int64_t)v;
    }
}

}  // namespace fdsnn
