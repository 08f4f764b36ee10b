// Does FP64 mma.sync (DMMA, m8n8k4) run on B200 at useful throughput, and
// does it overlap with DFMA (separate pipe)?  Measures FP64 FLOP/s of
//   0: DFMA chains only, 1: DMMA only, 2: both interleaved in every warp.
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o dmma dmma.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(d[0]), "+d"(d[1]) : "d"(a), "d"(b));
}

template <int MODE>
__global__ void __launch_bounds__(256) k(double* out, int iters) {
    double x[8], acc[4][2];
    for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 1e-9 + i;
    for (int i = 0; i < 4; ++i) acc[i][0] = acc[i][1] = 0;
    const double a = 1.0000001, b = 0.9999999;
    for (int it = 0; it < iters; ++it) {
        if (MODE != 1) {
#pragma unroll
            for (int r = 0; r < 4; ++r)
#pragma unroll
                for (int i = 0; i < 8; ++i) x[i] = fma(x[i], a, b);
        }
        if (MODE != 0) {
#pragma unroll
            for (int r = 0; r < 2; ++r)
#pragma unroll
                for (int i = 0; i < 4; ++i) dmma(acc[i], a + i, b);
        }
    }
    double s = 0;
    for (int i = 0; i < 8; ++i) s += x[i];
    for (int i = 0; i < 4; ++i) s += acc[i][0] + acc[i][1];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
    double* d;
    cudaMalloc(&d, 148 * 8 * 256 * 8);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int iters = 2000;
    const char* names[3] = {"DFMA only", "DMMA only", "DFMA + DMMA"};
    for (int mode = 0; mode < 3; ++mode) {
        auto run = [&](int it) {
            if (mode == 0) k<0><<<148 * 4, 256>>>(d, it);
            if (mode == 1) k<1><<<148 * 4, 256>>>(d, it);
            if (mode == 2) k<2><<<148 * 4, 256>>>(d, it);
        };
        run(10);
        cudaEventRecord(e0);
        run(iters);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        const double threads = 148.0 * 4 * 256;
        const double fma_flops = (mode != 1) ? threads * iters * 32 * 2 : 0;          // 32 DFMA per iter
        const double mma_flops = (mode != 0) ? threads / 32 * iters * 8 * 256 * 2 : 0;  // 8 DMMA per warp-iter
        printf("%-12s %.3f ms  DFMA %.1f TF  DMMA %.1f TF  total %.1f TF  err=%s\n", names[mode], ms,
               fma_flops / (ms * 1e-3) / 1e12, mma_flops / (ms * 1e-3) / 1e12,
               (fma_flops + mma_flops) / (ms * 1e-3) / 1e12, cudaGetErrorString(cudaGetLastError()));
    }
}
