// FP64 pipe rate of the radix-8 butterfly code itself (fft.cuh pass bodies on
// register data, no exchanges), W warps/SM, one or two independent transforms
// per thread, vs the pure-DFMA rate.  Counts DP instructions from the SASS.
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../../paper_2309_09025_b200/csrc -o fp64_fft fp64_fft.cu
#include <cstdio>
#include <cuda_runtime.h>
#include "fft.cuh"
using namespace fdsnn;

template <int PAIRS>
__global__ void k(double* out, int iters) {
    double2 v[PAIRS][8], w[8];
#pragma unroll
    for (int r = 0; r < 8; ++r) {
        w[r] = make_double2(0.7 + 0.01 * r, 0.3 - 0.01 * threadIdx.x);
#pragma unroll
        for (int p = 0; p < PAIRS; ++p) v[p][r] = make_double2(threadIdx.x + r + p, r - 1.0 * p);
    }
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int p = 0; p < PAIRS; ++p) pass_body<512, 1, false>(v[p], w);
#pragma unroll
        for (int p = 0; p < PAIRS; ++p) pass_body<512, 2, true>(v[p], w);
    }
    double s = 0;
#pragma unroll
    for (int p = 0; p < PAIRS; ++p)
#pragma unroll
        for (int r = 0; r < 8; ++r) s += v[p][r].x + v[p][r].y;
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int PAIRS>
void run(double* d, int warps, int dp_per_iter) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int iters = 4096;
    k<PAIRS><<<148, warps * 32>>>(d, 16);
    cudaEventRecord(e0);
    k<PAIRS><<<148, warps * 32>>>(d, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double inst = 148.0 * warps * iters * dp_per_iter;
    const double cyc = ms * 1e-3 * 1.965e9;
    const double rate = inst / (148.0 * 4) / cyc;
    printf("transforms/thread=%d warps/SM=%2d: %.3f DP warp-instr/SMSP/cycle (%.0f%% of 0.5)\n", PAIRS, warps, rate,
           rate / 0.5 * 100);
}

int main(int argc, char** argv) {
    // DP instructions per loop iteration (two pass bodies per transform), from cuobjdump
    const int dp1 = argc > 1 ? atoi(argv[1]) : 144, dp2 = argc > 2 ? atoi(argv[2]) : 288;
    double* d;
    cudaMalloc(&d, 148 * 1024 * 8);
    for (int w : {4, 8, 12, 16}) {
        run<1>(d, w, dp1);
        run<2>(d, w, dp2);
    }
    printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
}
