// Does a non-FP64 instruction issue "under" a DFMA on B200, or does every
// FP64 warp instruction hold the scheduler's dispatch for its 2 cycles?
// Each thread runs 8 independent DFMA chains interleaved with R integer
// (IMAD / LOP3), FP32 (FFMA) or shared-memory (LDS.32) instructions per DFMA.
// Reports cycles per DFMA per scheduler (2.0 = FP64 pipe bound).
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_mix fp64_mix.cu
#include <cstdio>
#include <cuda_runtime.h>

// KIND 0: IMAD, 1: LOP3 (xor+and), 2: FFMA, 3: LDS.32, 4: register moves (ptxas emits MOV / IMAD.MOV.U32)
template <int KIND, int RNUM, int RDEN>
__global__ void k(double* out, int iters, double a, double b, int ia, int ib, float fa) {
    __shared__ int sm[1024];
    sm[threadIdx.x] = threadIdx.x;
    __syncthreads();
    double x[8];
    int y[8];
    float z[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) { x[i] = threadIdx.x + i; y[i] = threadIdx.x * 3 + i; z[i] = y[i]; }
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int u = 0; u < 8; ++u) {
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                x[i] = fma(x[i], a, b);
                const int idx = u * 8 + i;
                const int n_here = ((idx + 1) * RNUM) / RDEN - (idx * RNUM) / RDEN;
#pragma unroll
                for (int r = 0; r < n_here; ++r) {
                    if (KIND == 0) y[i] = y[i] * ia + ib;
                    if (KIND == 1) y[i] = (y[i] ^ ia) & ib;
                    if (KIND == 2) z[i] = fmaf(z[i], fa, 1.0f);
                    if (KIND == 3) y[i] = sm[(y[i] + ib) & 1023];
                    if (KIND == 4) asm volatile("mov.b32 %0, %1;" : "=r"(y[i]) : "r"(y[(i + 1) & 7]));
                }
            }
        }
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += x[i] + y[i] + z[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int KIND, int RNUM, int RDEN>
void run(double* d, int warps, const char* name) {
    const int iters = 2000;
    k<KIND, RNUM, RDEN><<<148, warps * 32>>>(d, 10, 1.0000001, 0.5, 3, 0x7fffffff, 1.0001f);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    k<KIND, RNUM, RDEN><<<148, warps * 32>>>(d, iters, 1.0000001, 0.5, 3, 0x7fffffff, 1.0001f);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    int khz; cudaDeviceGetAttribute(&khz, cudaDevAttrClockRate, 0);
    const double cycles = ms * 1e-3 * khz * 1e3;
    const double dfma_per_smsp = (double)iters * 64 * (warps / 4.0);
    printf("%-6s other/DFMA = %d/%d  warps/SM %2d: %.2f cycles per DFMA per scheduler\n", name, RNUM, RDEN, warps,
           cycles / dfma_per_smsp);
}

int main() {
    double* d; cudaMalloc(&d, 148 * 1024 * 8);
    for (int w : {8, 12}) {
        run<0, 0, 1>(d, w, "none");
        run<0, 1, 2>(d, w, "IMAD"); run<0, 1, 1>(d, w, "IMAD"); run<0, 3, 2>(d, w, "IMAD"); run<0, 2, 1>(d, w, "IMAD");
        run<1, 1, 2>(d, w, "LOP3"); run<1, 1, 1>(d, w, "LOP3"); run<1, 2, 1>(d, w, "LOP3");
        run<2, 1, 1>(d, w, "FFMA"); run<2, 2, 1>(d, w, "FFMA");
        run<3, 1, 2>(d, w, "LDS"); run<3, 1, 1>(d, w, "LDS");
        run<4, 1, 4>(d, w, "MOV"); run<4, 1, 2>(d, w, "MOV"); run<4, 1, 1>(d, w, "MOV");
    }
    return 0;
}
