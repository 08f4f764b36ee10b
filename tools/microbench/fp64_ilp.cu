// FP64 pipe throughput vs warps per scheduler and per-warp ILP on B200:
// W warps/SM (W/4 per SMSP), each thread runs ILP independent DFMA chains.
// Also a DADD-only and a 1:1 DFMA/DADD mix variant.
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_ilp fp64_ilp.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int ILP, int KIND>
__global__ void k(double* out, int iters, double a, double b) {
    double x[ILP];
#pragma unroll
    for (int i = 0; i < ILP; ++i) x[i] = threadIdx.x + i;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int u = 0; u < 8; ++u)
#pragma unroll
            for (int i = 0; i < ILP; ++i) {
                if (KIND == 0) x[i] = fma(x[i], a, b);
                if (KIND == 1) x[i] = x[i] + b;
                if (KIND == 2) x[i] = (u & 1) ? x[i] + b : fma(x[i], a, b);
            }
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < ILP; ++i) s += x[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int ILP, int KIND>
void run(double* d, int warps, const char* name) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int iters = 2048;
    k<ILP, KIND><<<148, warps * 32>>>(d, 8, 1.0000001, 1e-9);
    cudaEventRecord(e0);
    k<ILP, KIND><<<148, warps * 32>>>(d, iters, 1.0000001, 1e-9);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double inst = 148.0 * warps * iters * 8 * ILP;  // warp instructions
    const double per_smsp_cyc = ms * 1e-3 * 1.965e9;       // cycles
    const double rate = inst / (148.0 * 4) / per_smsp_cyc;  // warp-instr per SMSP-cycle
    printf("%-6s warps/SM=%2d ILP=%d: %.3f FP64 warp-instr/SMSP/cycle (%.0f%% of 0.5)\n", name, warps, ILP, rate,
           rate / 0.5 * 100);
}

int main() {
    double* d;
    cudaMalloc(&d, 148 * 1024 * 8);
    for (int w : {4, 8, 12, 16, 32}) {
        run<1, 0>(d, w, "dfma");
        run<2, 0>(d, w, "dfma");
        run<4, 0>(d, w, "dfma");
        run<8, 0>(d, w, "dfma");
        run<4, 1>(d, w, "dadd");
        run<4, 2>(d, w, "mix");
    }
    printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
}
