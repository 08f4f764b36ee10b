// SHFL vs shared-memory throughput on B200: cycles per warp instruction per
// SM for 32-bit __shfl_xor_sync, LDS.32 and LDS.128, and SHFL mixed with
// LDS.128 (do they share a pipe?).
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o shfl shfl.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int MODE>
__global__ void __launch_bounds__(256) k(float* out, int iters) {
    __shared__ float4 buf[2048];
    for (int i = threadIdx.x; i < 2048; i += blockDim.x) buf[i] = make_float4(i, i, i, i);
    __syncthreads();
    const int lane = threadIdx.x & 31;
    float x = lane, y = 0;
    float4 acc = make_float4(0, 0, 0, 0);
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int r = 0; r < 8; ++r) {
            if (MODE == 0 || MODE == 3) x += __shfl_xor_sync(0xffffffffu, x, 1 + (r & 7));
            if (MODE == 1) y += reinterpret_cast<const float*>(buf)[(lane + 32 * r + it) & 8191];
            if (MODE == 2 || MODE == 3) {
                const float4 v = buf[(lane + 32 * r + it) & 2047];
                acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
            }
        }
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = x + y + acc.x + acc.y + acc.z + acc.w;
}

int main() {
    float* d;
    cudaMalloc(&d, 148 * 4 * 256 * 4);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const int iters = 4096;
    const char* names[4] = {"SHFL.32", "LDS.32", "LDS.128", "SHFL.32 + LDS.128"};
    for (int mode = 0; mode < 4; ++mode) {
        auto run = [&](int it) {
            if (mode == 0) k<0><<<148 * 4, 256>>>(d, it);
            if (mode == 1) k<1><<<148 * 4, 256>>>(d, it);
            if (mode == 2) k<2><<<148 * 4, 256>>>(d, it);
            if (mode == 3) k<3><<<148 * 4, 256>>>(d, it);
        };
        run(16);
        cudaEventRecord(a);
        run(iters);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        const double warp_instr_per_sm = 4.0 * 8 * iters * 8;  // CTAs/SM * warps * iters * per-iter
        const double cyc = ms * 1e-3 * 1.965e9;
        printf("%-20s %.2f cycles per warp instruction (group) per SM\n", names[mode], cyc / warp_instr_per_sm);
    }
}
