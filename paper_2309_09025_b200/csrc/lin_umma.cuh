// lin_umma.cuh — fully connected weight sums on the 5th-generation tensor
// cores (network.layer_forward, reference network.py:409-421):
//   Y[s][o][w] = sum_i W[o][i] * X[s][i][w]   (mod q)
// for every word w of the ciphertext rows (mask a_0..a_{n-1}, body b, pad).
// The reference forms the product in float64 (asserted exact, :417) and
// reduces mod q; here it is the same tcgen05 `kind::i8` GEMM construction as
// the key switch (ks_umma.cuh):
//   * A = W as s8 (every weight in [-128, 127], checked at operator load),
//     rows = output cells (UMMA M = 128 per CTA), K = input cells, tiled once
//     at operator load in the canonical K-major no-swizzle layout;
//   * B = the input ciphertext words split into 4 unsigned byte limbs, columns
//     = (sample, word) pairs, the limbs of 64 columns stacked along the MMA's
//     N (= 256); tiled per call by lin_prepare_b_kernel (one pass over X);
//   * s32 accumulation is exact (K * 128 * 255 < 2^31, checked on the host);
//     the epilogue recombines sum_j acc_j << 8j modulo 2^32 -- exact modulo
//     q = 2^k -- masks and writes 16-byte vectors into the output rows.
// Compared with the CUDA-core int32 GEMM (linear.cuh, IMAD-bound), the MMA
// work is 4 byte-limb products per multiply-add but runs on the tensor core,
// so the layer becomes a pass over its operands.
#pragma once
#include "ks_umma.cuh"

namespace fdsnn {

constexpr int LIN_LIMBS = 4;
constexpr int LINU_B_STEP = KSU_COLS * LIN_LIMBS * KSU_KSTEP;  // 8 KB per K step

// W (out x in, int32 on device) -> s8 A tiles [row block][K step] (4 KB each).
// One thread per 16-byte core-matrix row: (row block, K step, row, K half).
__global__ void lin_prepare_a_kernel(const int32_t* __restrict__ W, int out_cells, int in_cells, int ksteps,
                                     int rblocks, uint8_t* __restrict__ at) {
    const int64_t segs = (int64_t)rblocks * ksteps * KSU_M * 2;
    for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < segs; s += (int64_t)gridDim.x * blockDim.x) {
        const int half = (int)(s & 1);
        const int row = (int)((s >> 1) % KSU_M);
        const int64_t tk = (s >> 1) / KSU_M;  // rb * ksteps + ks
        const int ks = (int)(tk % ksteps);
        const int o = (int)(tk / ksteps) * KSU_M + row;
        uint8_t a[16];
#pragma unroll
        for (int e = 0; e < 16; ++e) {
            const int i = ks * KSU_KSTEP + half * 16 + e;
            a[e] = (uint8_t)(int8_t)((o < out_cells && i < in_cells) ? W[(size_t)o * in_cells + i] : 0);
        }
        *reinterpret_cast<uint4*>(at + (size_t)tk * KSU_A_STEP + ksu_tile_off(row, half * 16)) =
            *reinterpret_cast<const uint4*>(a);
    }
}

// X (batch x in x stride uint32) -> u8 limb tiles [column tile][K step]
// (8 KB each: B row = limb * 64 + column within the tile).  One thread per
// (column, 16-input group): 16 coalesced word loads, 4 limb rows written.
__global__ void lin_prepare_b_kernel(const uint32_t* __restrict__ X, int in_cells, int stride, int64_t ncols,
                                     int ksteps, int64_t ctiles, uint8_t* __restrict__ bt) {
    const int64_t segs = ctiles * KSU_COLS * (int64_t)ksteps * 2;
    for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < segs; s += (int64_t)gridDim.x * blockDim.x) {
        const int cc = (int)(s % KSU_COLS);        // column within the tile (fastest: coalesced loads)
        const int64_t r = s / KSU_COLS;
        const int half = (int)(r & 1);
        const int64_t tk = r >> 1;                  // ct * ksteps + ks
        const int ks = (int)(tk % ksteps);
        const int64_t col = (tk / ksteps) * KSU_COLS + cc;
        uint32_t x[16];
        if (col < ncols) {
            const int64_t smp = col / stride, w = col - smp * stride;
            const uint32_t* src = X + (smp * in_cells) * stride + w;
#pragma unroll
            for (int e = 0; e < 16; ++e) {
                const int i = ks * KSU_KSTEP + half * 16 + e;
                x[e] = i < in_cells ? __ldg(src + (size_t)i * stride) : 0u;
            }
        } else {
#pragma unroll
            for (int e = 0; e < 16; ++e) x[e] = 0u;
        }
        uint8_t* tile = bt + (size_t)tk * LINU_B_STEP;
#pragma unroll
        for (int j = 0; j < LIN_LIMBS; ++j) {
            uint8_t b[16];
#pragma unroll
            for (int e = 0; e < 16; ++e) b[e] = (uint8_t)(x[e] >> (8 * j));
            *reinterpret_cast<uint4*>(tile + ksu_tile_off(j * KSU_COLS + cc, half * 16)) =
                *reinterpret_cast<const uint4*>(b);
        }
    }
}

struct LinUmmaArgs {
    const uint8_t* at;  // [row block][K step] A tiles
    const uint8_t* bt;  // [column tile][K step] B tiles
    int ksteps;         // padded K / 32 (a multiple of KSU_KPS)
    int out_cells;
    int stride;
    int64_t ncols;      // batch * stride
    uint32_t qmask;
    uint32_t* Y;        // batch x out x stride
};

// One CTA = 128 output cells x 64 (sample, word) columns, all 4 limbs.
__global__ void __launch_bounds__(128, 1) lin_umma_kernel(const LinUmmaArgs args) {
    constexpr int NB = KSU_COLS * LIN_LIMBS;  // MMA N = 256
    constexpr int BSTEP = LINU_B_STEP;
    constexpr int ASTAGE = KSU_KPS * KSU_A_STEP, BSTAGE = KSU_KPS * BSTEP;
    constexpr uint32_t IDESC = (2u << 4)      // D = s32
                             | (1u << 7)      // A = s8
                             | (0u << 10)     // B = u8
                             | ((uint32_t)(NB >> 3) << 17) | ((uint32_t)(KSU_M >> 4) << 24);
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    uint64_t* full = reinterpret_cast<uint64_t*>(smem_raw);
    uint64_t* empty = full + KSU_STAGES;
    uint64_t* done = empty + KSU_STAGES;
    uint32_t* tslot = reinterpret_cast<uint32_t*>(done + 1);
    unsigned char* ring = smem_raw + 256;
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const int rb = blockIdx.y, ct = blockIdx.x;
    const int nstages = args.ksteps / KSU_KPS;

    if (threadIdx.x == 0) {
        for (int s = 0; s < KSU_STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        mbar_init(done, 1);
        fence_mbar_init();
    }
    if (warp == 0) tmem_alloc(tslot, 256);
    tmem_fence_before();
    __syncthreads();
    tmem_fence_after();
    const uint32_t tacc = *tslot;

    const uint8_t* a_src = args.at + (size_t)rb * args.ksteps * KSU_A_STEP;
    const uint8_t* b_src = args.bt + (size_t)ct * args.ksteps * BSTEP;
    if (threadIdx.x == 0) {  // producer: TMA bulk copies into the ring
        for (int st = 0; st < nstages; ++st) {
            const int s = st % KSU_STAGES;
            if (st >= KSU_STAGES) mbar_wait(&empty[s], (uint32_t)(((st / KSU_STAGES) - 1) & 1));
            unsigned char* sa = ring + (size_t)s * (ASTAGE + BSTAGE);
            mbar_arrive_expect_tx(&full[s], ASTAGE + BSTAGE);
            bulk_g2s(sa, a_src + (size_t)st * ASTAGE, ASTAGE, &full[s]);
            bulk_g2s(sa + ASTAGE, b_src + (size_t)st * BSTAGE, BSTAGE, &full[s]);
        }
    } else if (threadIdx.x == 32) {  // MMA issuer
        for (int st = 0; st < nstages; ++st) {
            const int s = st % KSU_STAGES;
            mbar_wait(&full[s], (uint32_t)((st / KSU_STAGES) & 1));
            tmem_fence_after();
            const unsigned char* sa = ring + (size_t)s * (ASTAGE + BSTAGE);
#pragma unroll
            for (int i = 0; i < KSU_KPS; ++i)
                umma_i8(tacc, ksu_desc(sa + i * KSU_A_STEP), ksu_desc(sa + ASTAGE + i * BSTEP), IDESC,
                        (st | i) != 0);
            tmem_commit(&empty[s]);
        }
        tmem_commit(done);
    }
    __syncwarp();
    mbar_wait(done, 0);
    tmem_fence_after();

    // epilogue: lane = output cell, 16 (sample, word) columns per chunk; the
    // row stride is a multiple of 4, so every 4-word group lies in one sample
    const int o = rb * KSU_M + warp * 32 + lane;
    const uint32_t lane_addr = tacc + ((uint32_t)(warp * 32) << 16);
#pragma unroll 1
    for (int c0 = 0; c0 < KSU_COLS; c0 += 16) {
        uint32_t sum[16];
#pragma unroll
        for (int e = 0; e < 16; ++e) sum[e] = 0u;
#pragma unroll
        for (int j = 0; j < LIN_LIMBS; ++j) {
            uint32_t w[16];
            tmem_ld16_async(lane_addr + (uint32_t)(j * KSU_COLS + c0), w);
            tmem_wait16(w);
#pragma unroll
            for (int e = 0; e < 16; ++e) sum[e] += w[e] << (8 * j);
        }
        if (o < args.out_cells) {
#pragma unroll
            for (int e = 0; e < 16; e += 4) {
                const int64_t col = (int64_t)ct * KSU_COLS + c0 + e;
                if (col < args.ncols) {
                    const int64_t smp = col / args.stride, wd = col - smp * args.stride;
                    uint32_t* dst = args.Y + (smp * args.out_cells + o) * args.stride + wd;
                    *reinterpret_cast<uint4*>(dst) =
                        make_uint4(sum[e] & args.qmask, sum[e + 1] & args.qmask, sum[e + 2] & args.qmask,
                                   sum[e + 3] & args.qmask);
                }
            }
        }
    }
    tmem_fence_before();
    __syncthreads();
    if (warp == 0) {
        tmem_fence_after();
        tmem_dealloc(tacc, 256);
    }
}

}  // namespace fdsnn
