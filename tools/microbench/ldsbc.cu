// LDS.128 throughput vs address-duplication pattern across lanes (B200):
// does a warp-wide 128-bit shared load with only 16 distinct addresses cost
// fewer wavefronts than one with 32?
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ldsbc ldsbc.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int MODE>
__global__ void __launch_bounds__(256) k(double* out, int iters) {
    __shared__ double2 buf[2048];
    for (int i = threadIdx.x; i < 2048; i += blockDim.x) buf[i] = make_double2(i, -i);
    __syncthreads();
    const int lane = threadIdx.x % 32, w = threadIdx.x / 32;
    int idx;
    if (MODE == 0) idx = lane;                    // 32 distinct
    else if (MODE == 1) idx = lane & 15;          // lanes l and l+16 share
    else if (MODE == 2) idx = lane >> 1;          // adjacent lanes share
    else idx = 0;                                 // full broadcast
    idx += w * 64;
    double2 acc = make_double2(0, 0);
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int r = 0; r < 8; ++r) {
            const double2 v = buf[(idx + r * 256 + it) & 2047];
            acc.x += v.x;
            acc.y += v.y;
        }
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc.x + acc.y;
}

int main() {
    double* d;
    cudaMalloc(&d, 148 * 4 * 256 * 8);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const int iters = 4096;
    const char* names[4] = {"32 distinct", "l / l+16 shared", "adjacent shared", "broadcast"};
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
        const double inst = 148.0 * 4 * 8 * iters * 8;  // warp LDS.128 per SM... total
        const double cyc = ms * 1e-3 * 1.965e9;
        printf("%-18s %.2f cycles per warp LDS.128 per SM\n", names[mode], cyc / (inst / 148));
    }
}
