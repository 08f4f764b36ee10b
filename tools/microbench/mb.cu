// Microbenchmarks informing the blind-rotation design (run on B200):
// shared-memory LDS.128 bandwidth, SHFL throughput, and whether they overlap.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k_lds(float4* out, int iters) {
    __shared__ float4 s[2048];
    for (int i = threadIdx.x; i < 2048; i += blockDim.x) s[i] = make_float4(i, i, i, i);
    __syncthreads();
    float4 acc = make_float4(0, 0, 0, 0);
    int base = threadIdx.x;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            float4 v = s[(base + u * 256 + it) & 2047];
            acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
        }
    }
    if (acc.x == 1.2345f) out[0] = acc;
}
__global__ void k_shfl(float4* out, int iters) {
    float a0 = threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            a0 = __shfl_xor_sync(~0u, a0, 1 + u); a1 = __shfl_xor_sync(~0u, a1, 2 + u);
            a2 = __shfl_xor_sync(~0u, a2, 3 + u); a3 = __shfl_xor_sync(~0u, a3, 4 + u);
            a4 = __shfl_xor_sync(~0u, a4, 5 + u); a5 = __shfl_xor_sync(~0u, a5, 6 + u);
            a6 = __shfl_xor_sync(~0u, a6, 7 + u); a7 = __shfl_xor_sync(~0u, a7, 8 + u);
        }
    }
    float s = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
    if (s == 1.2345f) out[0] = make_float4(s, 0, 0, 0);
}
// half the warps do LDS, half do SHFL
__global__ void k_mix(float4* out, int iters) {
    if ((threadIdx.x / 32) % 2 == 0) {
        __shared__ float4 s[2048];
        for (int i = threadIdx.x; i < 2048; i += blockDim.x) s[i] = make_float4(i, i, i, i);
        float4 acc = make_float4(0, 0, 0, 0);
        int base = threadIdx.x;
        for (int it = 0; it < iters; ++it) {
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                float4 v = s[(base + u * 256 + it) & 2047];
                acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
            }
        }
        if (acc.x == 1.2345f) out[0] = acc;
    } else {
        float a0 = threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
        for (int it = 0; it < iters * 2; ++it) {
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                a0 = __shfl_xor_sync(~0u, a0, 1 + u); a1 = __shfl_xor_sync(~0u, a1, 2 + u);
                a2 = __shfl_xor_sync(~0u, a2, 3 + u); a3 = __shfl_xor_sync(~0u, a3, 4 + u);
                a4 = __shfl_xor_sync(~0u, a4, 5 + u); a5 = __shfl_xor_sync(~0u, a5, 6 + u);
                a6 = __shfl_xor_sync(~0u, a6, 7 + u); a7 = __shfl_xor_sync(~0u, a7, 8 + u);
            }
        }
        float s = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
        if (s == 1.2345f) out[0] = make_float4(s, 0, 0, 0);
    }
}
__global__ void k_dfma(double* out, int iters) {
    double a[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-9 + i;
    for (int it = 0; it < iters; ++it)
#pragma unroll
        for (int u = 0; u < 8; ++u)
#pragma unroll
            for (int i = 0; i < 8; ++i) a[i] = fma(a[i], 0.999999, 1e-9);
    double s = 0;
    for (int i = 0; i < 8; ++i) s += a[i];
    if (s == 1.2345) out[0] = s;
}
__global__ void k_dadd(double* out, int iters) {
    double a[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-9 + i;
    for (int it = 0; it < iters; ++it)
#pragma unroll
        for (int u = 0; u < 8; ++u)
#pragma unroll
            for (int i = 0; i < 8; ++i) a[i] = a[i] + 1e-9;
    double s = 0;
    for (int i = 0; i < 8; ++i) s += a[i];
    if (s == 1.2345) out[0] = s;
}
__global__ void k_i2f(double* out, int iters) {
    int x = threadIdx.x;
    double acc[4] = {0, 0, 0, 0};
    for (int it = 0; it < iters; ++it)
#pragma unroll
        for (int u = 0; u < 16; ++u) { acc[u & 3] = (double)(x + u + it); }
    if (acc[0] + acc[1] + acc[2] + acc[3] == 1.2345) out[0] = acc[0];
}
__global__ void k_f2i(double* out, int iters) {
    double x = threadIdx.x + 0.3;
    long long acc = 0;
    for (int it = 0; it < iters; ++it)
#pragma unroll
        for (int u = 0; u < 16; ++u) { acc ^= __double2ll_rn(x + u); }
    if (acc == 12345) out[0] = (double)acc;
}
int main() {
    float4* o; cudaMalloc(&o, 64);
    double* od; cudaMalloc(&od, 64);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    const int SM = 148;
    for (int warps : {4, 8, 16}) {
        int threads = warps * 32, blocks = SM;
        int iters = 4096;
        float ms;
        k_lds<<<blocks, threads>>>(o, 16); cudaEventRecord(a); k_lds<<<blocks, threads>>>(o, iters); cudaEventRecord(b); cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b);
        double bytes = (double)blocks * threads * iters * 8 * 16;
        printf("warps/SM=%2d LDS.128: %.1f B/clk/SM (%.2f TB/s)\n", warps, bytes / SM / (ms * 1e-3 * 1.965e9), bytes / ms / 1e9);
        k_shfl<<<blocks, threads>>>(o, 16); cudaEventRecord(a); k_shfl<<<blocks, threads>>>(o, iters); cudaEventRecord(b); cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b);
        double sh = (double)blocks * threads * iters * 32;
        printf("warps/SM=%2d SHFL.32: %.1f lanes/clk/SM (%.1f B/clk)\n", warps, sh / SM / (ms * 1e-3 * 1.965e9), 4 * sh / SM / (ms * 1e-3 * 1.965e9));
        k_mix<<<blocks, threads>>>(o, 16); cudaEventRecord(a); k_mix<<<blocks, threads>>>(o, iters); cudaEventRecord(b); cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b);
        double mb = (double)blocks * threads / 2 * iters * 8 * 16 + (double)blocks * threads / 2 * iters * 2 * 32 * 4;
        printf("warps/SM=%2d MIX (LDS+SHFL bytes): %.1f B/clk/SM\n", warps, mb / SM / (ms * 1e-3 * 1.965e9));
        k_dfma<<<blocks, threads>>>(od, 16); cudaEventRecord(a); k_dfma<<<blocks, threads>>>(od, iters); cudaEventRecord(b); cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b);
        double fl = (double)blocks * threads * iters * 64;
        printf("warps/SM=%2d DFMA: %.1f /clk/SM  (%.1f TFLOPs)\n", warps, fl / SM / (ms * 1e-3 * 1.965e9), 2 * fl / ms / 1e9);
        k_dadd<<<blocks, threads>>>(od, 16); cudaEventRecord(a); k_dadd<<<blocks, threads>>>(od, iters); cudaEventRecord(b); cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b);
        printf("warps/SM=%2d DADD: %.1f /clk/SM\n", warps, fl / SM / (ms * 1e-3 * 1.965e9));
        k_i2f<<<blocks, threads>>>(od, 16); cudaEventRecord(a); k_i2f<<<blocks, threads>>>(od, iters); cudaEventRecord(b); cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b);
        double cv = (double)blocks * threads * iters * 16;
        printf("warps/SM=%2d I2F.F64: %.1f /clk/SM\n", warps, cv / SM / (ms * 1e-3 * 1.965e9));
        k_f2i<<<blocks, threads>>>(od, 16); cudaEventRecord(a); k_f2i<<<blocks, threads>>>(od, iters); cudaEventRecord(b); cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b);
        printf("warps/SM=%2d F2I.F64(+DADD): %.1f /clk/SM\n", warps, cv / SM / (ms * 1e-3 * 1.965e9));
    }
    printf("clock attr %d kHz, err=%s\n", clk, cudaGetErrorString(cudaGetLastError()));
}
