// Dependent-chain latencies (cycles) of FP64 ops and LDS on B200.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(double* out, long long* cyc, int iters) {
    __shared__ double s[1024];
    for (int i = threadIdx.x; i < 1024; i += blockDim.x) s[i] = 0.0;
    __syncthreads();
    double a = threadIdx.x * 1e-9, b = 1.0000001;
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) { a = fma(a, b, 1e-9); a = fma(a, b, 1e-9); a = fma(a, b, 1e-9); a = fma(a, b, 1e-9); }
    long long t1 = clock64();
    for (int i = 0; i < iters; ++i) { a = a + b; a = a + b; a = a + b; a = a + b; }
    long long t2 = clock64();
    int idx = threadIdx.x & 7;
    double x = 0;
    for (int i = 0; i < iters; ++i) { x = s[(idx + (int)x) & 1023]; x = s[(idx + (int)x) & 1023]; x = s[(idx + (int)x) & 1023]; x = s[(idx + (int)x) & 1023]; }
    long long t3 = clock64();
    if (threadIdx.x == 0) { cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; }
    out[threadIdx.x] = a + x;
}
int main() {
    double* o; long long* c; cudaMalloc(&o, 8 * 32); cudaMalloc(&c, 24);
    int iters = 10000;
    k<<<1, 32>>>(o, c, iters); cudaDeviceSynchronize();
    long long h[3]; cudaMemcpy(h, c, 24, cudaMemcpyDeviceToHost);
    printf("DFMA dep latency %.2f cyc, DADD %.2f cyc, LDS.64 dep %.2f cyc\n", h[0] / (4.0 * iters), h[1] / (4.0 * iters), h[2] / (4.0 * iters));
}
