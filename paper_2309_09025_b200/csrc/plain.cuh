// plain.cuh — the mod-p plaintext twin of the encrypted forward on the GPU
// (SURVEY §8(f)1): integer weight layers and the integer LIF update over a
// batch of images, used for fast full-batch parity of configs 2/4 and for
// spike-rate statistics.
//
// Reference semantics:
//   plain_infer                  oracle.py:44-78
//   plain_lif_step_batch         neuron.py:107-119  (spike2 = 2 on fire,
//                                v' = 0 if fired or h <= 0, else
//                                round_half_away(h*leak_num/leak_den))
//   div_round_half_away          ring.py:45-53
//   range check (when p given)   h in [v_th_hat - p/2, p/2)
// All arithmetic is exact int64, as in the reference's numpy.
#pragma once
#include "common.cuh"

namespace fdsnn {

// y[b][o] = sum_i W[o][i] * x[b][i]; one warp per (b, o).
__global__ void plain_dense_kernel(const int32_t* __restrict__ w, int out_cells, int in_cells,
                                   const int64_t* __restrict__ x, int64_t batch, int64_t* __restrict__ y) {
    const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) / 32;
    const int lane = threadIdx.x % 32;
    if (gw >= batch * out_cells) return;
    const int64_t b = gw / out_cells;
    const int o = (int)(gw % out_cells);
    const int32_t* wr = w + (size_t)o * in_cells;
    const int64_t* xr = x + b * in_cells;
    long long s = 0;
    for (int i = lane; i < in_cells; i += 32) s += (long long)wr[i] * xr[i];
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
    if (lane == 0) y[b * out_cells + o] = s;
}

__global__ void plain_csr_kernel(const int32_t* __restrict__ row_ptr, const int32_t* __restrict__ col_idx,
                                 const int32_t* __restrict__ val, int out_cells, int in_cells,
                                 const int64_t* __restrict__ x, int64_t batch, int64_t* __restrict__ y) {
    const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) / 32;
    const int lane = threadIdx.x % 32;
    if (gw >= batch * out_cells) return;
    const int64_t b = gw / out_cells;
    const int o = (int)(gw % out_cells);
    const int64_t* xr = x + b * in_cells;
    long long s = 0;
    for (int e = row_ptr[o] + lane; e < row_ptr[o + 1]; e += 32) s += (long long)val[e] * xr[col_idx[e]];
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
    if (lane == 0) y[b * out_cells + o] = s;
}

FDSNN_DEV long long div_round_half_away(long long num, long long den) {
    const long long mag = num < 0 ? -num : num;
    const long long r = (2 * mag + den) / (2 * den);
    return num >= 0 ? r : -r;
}

// h = v + i; spike2 = 2*[h >= vth]; v' = 0 if fired or h <= 0 else leak(h).
// p > 0: counts charged potentials outside [vth - p/2, p/2) into *overflow.
__global__ void plain_lif_kernel(const int64_t* __restrict__ v, const int64_t* __restrict__ in, int64_t count,
                                 long long vth, long long leak_num, long long leak_den, long long p,
                                 int64_t* __restrict__ spike2, int64_t* __restrict__ v_next,
                                 unsigned long long* __restrict__ overflow) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < count; e += (int64_t)gridDim.x * blockDim.x) {
        const long long h = v[e] + in[e];
        if (p > 0 && (h < vth - p / 2 || h >= p / 2)) atomicAdd(overflow, 1ull);
        const bool fired = h >= vth;
        spike2[e] = fired ? 2 : 0;
        v_next[e] = (fired || h <= 0) ? 0 : div_round_half_away(h * leak_num, leak_den);
    }
}

}  // namespace fdsnn
