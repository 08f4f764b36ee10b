// Throughput/latency of tcgen05.cp 64x128b.warpx2::02_13 chunks (16 x 1 KB) with commit+wait.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t sdesc(const void* p) {
    uint64_t d = 0;
    d |= (uint64_t)((su32(p) >> 4) & 0x3FFF);
    d |= (uint64_t)((128 >> 4) & 0x3FFF) << 16;
    d |= (uint64_t)((128 >> 4) & 0x3FFF) << 32;
    d |= (uint64_t)1 << 46;
    return d;
}
template <int SHAPE>
__global__ void k(uint32_t* out, int iters, long long* cyc) {
    extern __shared__ __align__(1024) uint32_t blk[];  // 32 KB
    __shared__ uint32_t tbase;
    __shared__ __align__(8) uint64_t bar;
    const int warp = threadIdx.x / 32;
    for (int i = threadIdx.x; i < 8192; i += blockDim.x) blk[i] = i;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;" ::"r"(su32(&tbase)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tb = tbase;
    long long t0 = clock64();
    if (threadIdx.x == 0) {
        for (int it = 0; it < iters; ++it) {
            for (int b = 0; b < 16; ++b) {
                if (SHAPE == 0) {
                    uint64_t d = sdesc(&blk[b * 256]);  // 1 KB block -> 2 KB written (multicast)
                    asm volatile("tcgen05.cp.cta_group::1.64x128b.warpx2::02_13 [%0], %1;" ::"r"(tb + 4 * b), "l"(d) : "memory");
                } else if (SHAPE == 1) {
                    uint64_t d = sdesc(&blk[b * 512]);  // 2 KB block
                    asm volatile("tcgen05.cp.cta_group::1.128x128b [%0], %1;" ::"r"(tb + 4 * b), "l"(d) : "memory");
                } else if (SHAPE == 2) {
                    uint64_t d = sdesc(&blk[(b % 8) * 1024]);  // 4 KB block (128 rows x 32 B)
                    asm volatile("tcgen05.cp.cta_group::1.128x256b [%0], %1;" ::"r"(tb + 8 * (b % 8)), "l"(d) : "memory");
                } else {
                    uint64_t d = sdesc(&blk[b * 128]);  // 512 B block -> 2 KB written (x4 multicast)
                    asm volatile("tcgen05.cp.cta_group::1.32x128b.warpx4 [%0], %1;" ::"r"(tb + 4 * b), "l"(d) : "memory");
                }
            }
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar)) : "memory");
            asm volatile("{\n\t.reg .pred P1;\nW:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t@!P1 bra W;\n\t}" ::"r"(su32(&bar)), "r"(it & 1) : "memory");
        }
    }
    long long t1 = clock64();
    if (threadIdx.x == 0 && blockIdx.x == 0) cyc[0] = t1 - t0;
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;" ::"r"(tb));
}
int main() {
    uint32_t* d; long long* c; cudaMalloc(&d, 64); cudaMalloc(&c, 8);
    const double bytes_per_iter[4] = {16384, 32768, 32768, 8192};  // smem bytes read per iteration
    for (int shape = 0; shape < 4; ++shape) {
        for (int iters : {1, 100}) {
            if (shape == 0) k<0><<<148, 128, 32768>>>(d, iters, c);
            if (shape == 1) k<1><<<148, 128, 32768>>>(d, iters, c);
            if (shape == 2) k<2><<<148, 128, 32768>>>(d, iters, c);
            if (shape == 3) k<3><<<148, 128, 32768>>>(d, iters, c);
            cudaError_t e = cudaDeviceSynchronize();
            long long h; cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
            printf("shape %d iters %d: %.0f cycles per iter, smem read %.1f B/clk %s\n", shape, iters,
                   (double)h / iters, bytes_per_iter[shape] * iters / h, cudaGetErrorString(e));
            if (e != cudaSuccess) return 1;
        }
    }
}
