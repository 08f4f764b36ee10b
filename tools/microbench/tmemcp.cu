// Verify tcgen05.cp .64x128b.warpx2::02_13 (smem -> TMEM multicast) addressing
// with a plain K-major no-swizzle descriptor: row t of a contiguous 64x16B block
// must land in TMEM lanes t (quadrants 0/1) and 64+t (quadrants 2/3).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ uint64_t sdesc(const void* p, uint32_t lbo, uint32_t sbo) {
    uint64_t d = 0;
    d |= (uint64_t)((su32(p) >> 4) & 0x3FFF);
    d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
    d |= (uint64_t)1 << 46;  // descriptor version (sm_100)
    return d;                // base offset 0, lbo mode 0, swizzle none (0)
}

__global__ void k(uint32_t* out, int variant) {
    __shared__ __align__(1024) uint32_t blk[2][64 * 4];  // two 1 KB blocks
    __shared__ uint32_t tbase;
    __shared__ __align__(8) uint64_t bar;
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    for (int i = threadIdx.x; i < 2 * 64 * 4; i += blockDim.x) (&blk[0][0])[i] = 0xA0000000u + i;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 32;" ::"r"(su32(&tbase)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic smem writes -> async proxy
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tb = tbase;
    if (threadIdx.x == 0) {
        for (int b = 0; b < 2; ++b) {
            uint64_t d = sdesc(&blk[b][0], variant == 0 ? 128 : 1024, 128);
            asm volatile("tcgen05.cp.cta_group::1.64x128b.warpx2::02_13 [%0], %1;" ::"r"(tb + 4 * b), "l"(d) : "memory");
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar)) : "memory");
    }
    // wait for the copy
    asm volatile("{\n\t.reg .pred P1;\nW:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n\t@!P1 bra W;\n\t}" ::"r"(su32(&bar)) : "memory");
    asm volatile("tcgen05.fence::after_thread_sync;");
    uint32_t v[8];
    const uint32_t ta = tb + ((uint32_t)((warp % 4) * 32) << 16);
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n\ttcgen05.wait::ld.sync.aligned;"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]) : "r"(ta));
    for (int i = 0; i < 8; ++i) out[threadIdx.x * 8 + i] = v[i];
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;" ::"r"(tb));
}

int main() {
    uint32_t* d;
    cudaMalloc(&d, 256 * 8 * 4);
    uint32_t h[256 * 8];
    for (int variant = 0; variant < 2; ++variant) {
        cudaMemset(d, 0, sizeof h);
        k<<<1, 128>>>(d, variant);
        cudaError_t e = cudaDeviceSynchronize();
        cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
        printf("variant %d: %s\n", variant, cudaGetErrorString(e));
        int bad = 0;
        for (int th = 0; th < 128; ++th) {
            int lanei = th;  // TMEM lane of this thread (warp w covers lanes 32w..)
            int row = lanei % 64;
            for (int i = 0; i < 8; ++i) {
                int b = i / 4, word = i % 4;
                uint32_t want = 0xA0000000u + b * 256 + row * 4 + word;
                if (h[th * 8 + i] != want) ++bad;
            }
        }
        printf("  mismatches %d; thread0: %08x %08x %08x %08x | %08x; thread 64: %08x %08x; thread 100: %08x\n", bad,
               h[0], h[1], h[2], h[3], h[4], h[64 * 8], h[64 * 8 + 1], h[100 * 8]);
    }
}
