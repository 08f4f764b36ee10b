// Warp-local data exchange through tensor memory vs shared memory on B200.
//  1. layout check of tcgen05.ld.16x256b after a tcgen05.st.32x32b
//  2. per-warp cost (latency with 1 warp/SM, throughput with 8 warps/SM) of
//     exchanging 8 complex doubles per thread: shared memory (STS.128/LDS.128
//     transpose) vs one or two TMEM hops (st.32x32b.x32 -> ld.16x256b.x4 x2).
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tmemx tmemx.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void st32(uint32_t a, const uint32_t (&v)[32]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
        "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(a),
        "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]),
        "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]), "r"(v[16]), "r"(v[17]), "r"(v[18]),
        "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]), "r"(v[23]), "r"(v[24]), "r"(v[25]), "r"(v[26]), "r"(v[27]),
        "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31])
        : "memory");
}
// 16x256b.x4: 16 regs
__device__ __forceinline__ void ld16x256x4(uint32_t a, uint32_t* v) {
    asm volatile(
        "tcgen05.ld.sync.aligned.16x256b.x4.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
          "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
        : "r"(a)
        : "memory");
}
__device__ __forceinline__ void wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void fb() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fa() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

__device__ uint32_t tmem_setup(uint32_t* tbase) {
    if (threadIdx.x < 32) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(tbase)), "r"(256));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    fb();
    __syncthreads();
    fa();
    return *tbase;
}
__device__ void tmem_free(uint32_t t) {
    fb();
    __syncthreads();
    if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(t), "r"(256));
}

__global__ void k_layout(uint32_t* out) {
    __shared__ uint32_t tb;
    uint32_t t = tmem_setup(&tb);
    const int i = threadIdx.x;
    uint32_t v[32];
    for (int c = 0; c < 32; ++c) v[c] = i * 1000 + c;
    st32(t, v);
    wait_st();
    fb();
    __syncwarp();
    fa();
    uint32_t r[32];
    ld16x256x4(t, r);
    ld16x256x4(t + (16u << 16), r + 16);
    wait_ld();
    for (int c = 0; c < 32; ++c) out[i * 32 + c] = r[c];
    tmem_free(t);
}

// MODE 0: shared-memory exchange, 1: one TMEM hop, 2: two TMEM hops
template <int MODE0>
__global__ void __launch_bounds__(256, 1) k_ex(double* out, int iters) {
    __shared__ uint32_t tb;
    __shared__ double2 buf[8][288];  // per warp 256 complex + pad
    uint32_t t = tmem_setup(&tb);
    const int w = threadIdx.x / 32, i = threadIdx.x % 32;
    const uint32_t ta = t + ((uint32_t)((w % 4) * 32) << 16) + (uint32_t)((w / 4) * 64);
    double2 x[8];
    for (int r = 0; r < 8; ++r) x[r] = make_double2(i + r, i - r);
    // MODE0 3: half the warps exchange through smem, the other half hop through TMEM
    const int MODE = MODE0 == 3 ? (w < 4 ? 0 : 1) : MODE0;
    for (int it = 0; it < iters; ++it) {
        if (MODE == 0) {
            double2* b = buf[w];
#pragma unroll
            for (int r = 0; r < 8; ++r) { int a = 8 * i + r; b[a + (a >> 3)] = x[r]; }
            __syncwarp();
#pragma unroll
            for (int r = 0; r < 8; ++r) { int a = i + 32 * r; x[r] = b[a + (a >> 3)]; }
            __syncwarp();
        } else {
#pragma unroll
            for (int h = 0; h < (MODE0 == 3 ? 1 : MODE0); ++h) {
                uint32_t v[32];
#pragma unroll
                for (int r = 0; r < 8; ++r) {
                    v[2 * r] = __double2loint(x[r].x); v[2 * r + 1] = __double2hiint(x[r].x);
                    v[16 + 2 * r] = __double2loint(x[r].y); v[16 + 2 * r + 1] = __double2hiint(x[r].y);
                }
                st32(ta, v);
                wait_st();
                fb();
                __syncwarp();
                fa();
                uint32_t q[32];
                ld16x256x4(ta, q);
                ld16x256x4(ta + (16u << 16), q + 16);
                wait_ld();
                // q[4k+{0,1}] = dcol 4k+(i&3) lane i>>2 ; q[4k+{2,3}] = lane +8 ; second load lanes +16
#pragma unroll
                for (int r = 0; r < 8; ++r) {
                    const int ld = r >> 2, k = (r >> 1) & 1, hv = r & 1;  // real at k, imag at k+2
                    x[r].x = __hiloint2double(q[16 * ld + 4 * k + 2 * hv + 1], q[16 * ld + 4 * k + 2 * hv]);
                    x[r].y = __hiloint2double(q[16 * ld + 4 * (k + 2) + 2 * hv + 1], q[16 * ld + 4 * (k + 2) + 2 * hv]);
                }
                fb();
                __syncwarp();
                fa();
            }
        }
#pragma unroll
        for (int r = 0; r < 8; ++r) x[r].x += 1.0;
    }
    double s = 0;
    for (int r = 0; r < 8; ++r) s += x[r].x + x[r].y;
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    tmem_free(t);
}

int main() {
    uint32_t* o;
    cudaMalloc(&o, 32 * 32 * 4);
    k_layout<<<1, 32>>>(o);
    uint32_t h[32 * 32];
    cudaMemcpy(h, o, sizeof(h), cudaMemcpyDeviceToHost);
    printf("layout err=%s\n", cudaGetErrorString(cudaGetLastError()));
    int bad = 0;
    for (int i = 0; i < 32; ++i)
        for (int c = 0; c < 32; ++c) {
            int ld = c / 16, rr = c % 16, k = rr / 4, j = rr % 4;
            int lane = 16 * ld + (i >> 2) + (j >= 2 ? 8 : 0);
            int col = 8 * k + 2 * (i & 3) + (j & 1);
            if (h[i * 32 + c] != (uint32_t)(lane * 1000 + col)) ++bad;
        }
    printf("16x256b mapping mismatches: %d\n", bad);
    for (int i = 0; i < 6; ++i) {
        printf("thr %d:", i);
        for (int c = 0; c < 8; ++c) printf(" %u", h[i * 32 + c]);
        printf("\n");
    }
    double* d;
    cudaMalloc(&d, 148 * 256 * 8);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const int iters = 4000;
    const char* names[4] = {"smem", "tmem 1 hop", "tmem 2 hops", "4 warps smem + 4 warps tmem"};
    for (int mode = 0; mode < 4; ++mode)
        for (int threads : {32, 256}) {
            auto run = [&](int it) {
                if (mode == 0) k_ex<0><<<148, threads>>>(d, it);
                if (mode == 1) k_ex<1><<<148, threads>>>(d, it);
                if (mode == 2) k_ex<2><<<148, threads>>>(d, it);
                if (mode == 3) k_ex<3><<<148, threads>>>(d, it);
            };
            run(10);
            cudaEventRecord(a);
            run(iters);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            double cyc = ms * 1e-3 * 1.965e9 / iters;
            printf("%-12s warps/SM=%d: %.1f cycles per exchange iteration (%.2f per warp-exchange) err=%s\n", names[mode],
                   threads / 32, cyc, cyc / (threads / 32), cudaGetErrorString(cudaGetLastError()));
        }
}
