// ks_umma.cuh — LWE key switching on the 5th-generation tensor cores.
//
// Reference: bootstrap.key_switch_batch (bootstrap.py:303-316) with the
// gadget rule of rgsw.gadget_decompose (rgsw.py:119-133):
//   out_a = -sum_k dig[v][k] * kskA[k][c]   (mod q),  k = j*ks_L + t.
// The mask part is an integer GEMM  C = D (V x K) . KSK (K x n)  with
// K = N*ks_L (DESK: 4096 x 5120 x 512 per bench launch).  It runs as a
// tcgen05 `kind::i8` GEMM:
//   * A = the signed base-2^ks_log digits, s8 (|d| <= 2^(ks_log-1) <= 64);
//   * B = the KSK split into LIMBS = ceil(log2 q / 8) unsigned byte limbs,
//     KSK = sum_j limb_j << 8j; the limbs of 64 output columns are stacked
//     along the MMA's N dimension (N = 64*LIMBS <= 256), so one CTA's TMEM
//     accumulator holds every limb of its 128 x 64 output tile;
//   * accumulation is exact in s32: K * 2^(ks_log-1) * 255 < 2^31 (checked on
//     the host); the epilogue recombines  sum_j acc_j << 8j  modulo 2^32,
//     which is exact modulo q = 2^k, negates and masks.
// Operands are pre-tiled in global memory in the canonical K-major
// no-swizzle UMMA layout (8-row x 16-byte core matrices, core matrix (r8, k16)
// at byte (r8*2 + k16)*128 inside each 32-byte K step), so every pipeline
// stage is two 1-D bulk copies (TMA engine) into a 4-deep shared-memory ring.
// One elected thread issues the MMAs; tcgen05.commit releases ring stages.
// The body column (b) and the row padding stay on ks_body_kernel.
#pragma once
#include "keyswitch.cuh"

namespace fdsnn {

constexpr int KSU_M = 128;       // ciphertexts per CTA (UMMA M, TMEM lanes)
constexpr int KSU_COLS = 64;     // output columns per CTA
constexpr int KSU_KSTEP = 32;    // K bytes per MMA (kind::i8)
constexpr int KSU_KPS = 4;       // K steps per ring stage
constexpr int KSU_STAGES = 4;    // ring depth
constexpr int KSU_A_STEP = KSU_M * KSU_KSTEP;  // 4 KB of digits per K step

__host__ __device__ constexpr int ksu_b_step(int limbs) { return KSU_COLS * limbs * KSU_KSTEP; }
__host__ __device__ constexpr size_t ksu_smem_bytes(int limbs) {
    return 256 + (size_t)KSU_STAGES * KSU_KPS * (KSU_A_STEP + ksu_b_step(limbs));
}

// byte offset of element (row, k) inside one K-step tile of the canonical
// K-major no-swizzle layout (rows x 32 bytes)
FDSNN_DEV int ksu_tile_off(int row, int k) {
    return ((row >> 3) * 2 + (k >> 4)) * 128 + (row & 7) * 16 + (k & 15);
}

struct KsUmmaArgs {
    DevParams prm;
    const uint8_t* dig;    // [row block][K step] 4 KB tiles (s8 digits)
    const uint8_t* bt;     // [column tile][K step] tiles (u8 key limbs)
    int ksteps;            // padded K / 32
    int limbs;
    int64_t V;
    uint32_t* out;         // V x stride
};

// KSK (K x stride uint32, device) -> limb tiles.  One thread per 16-byte
// core-matrix row: (column tile, K step, B row, K half).
__global__ void ksu_prepare_b_kernel(const uint32_t* __restrict__ ksk, int K, int n, int stride, int ksteps,
                                     int limbs, int ntiles, uint8_t* __restrict__ bt) {
    const int nb_rows = KSU_COLS * limbs;
    const int64_t segs = (int64_t)ntiles * ksteps * nb_rows * 2;
    for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < segs; s += (int64_t)gridDim.x * blockDim.x) {
        const int half = (int)(s & 1);
        const int64_t r = s >> 1;
        const int nb = (int)(r % nb_rows);
        const int64_t tk = r / nb_rows;
        const int ks = (int)(tk % ksteps);
        const int ct = (int)(tk / ksteps);
        const int limb = nb / KSU_COLS, col = ct * KSU_COLS + nb % KSU_COLS;
        uint8_t b[16];
#pragma unroll
        for (int e = 0; e < 16; ++e) {
            const int k = ks * KSU_KSTEP + half * 16 + e;
            const uint32_t v = (k < K && col < n) ? ksk[(size_t)k * stride + col] : 0u;
            b[e] = (uint8_t)(v >> (8 * limb));
        }
        uint8_t* dst = bt + (size_t)tk * ksu_b_step(limbs) + ksu_tile_off(nb, half * 16);
        *reinterpret_cast<uint4*>(dst) = *reinterpret_cast<const uint4*>(b);
    }
}

// z-LWE masks -> s8 digit tiles (rgsw.py:130-132 rule, k = j*ks_L + t).  One
// thread per 16-byte core-matrix row: (row block, K step, row, K half).
template <int KSL>
__global__ void ksu_digits_kernel(const KsArgs args, int ksteps, uint8_t* __restrict__ dig) {
    const DevParams& prm = args.prm;
    const int64_t rblocks = (args.V + KSU_M - 1) / KSU_M;
    const int64_t segs = rblocks * ksteps * KSU_M * 2;
    const int K = prm.N * KSL;
    for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < segs; s += (int64_t)gridDim.x * blockDim.x) {
        const int half = (int)(s & 1);
        const int row = (int)((s >> 1) % KSU_M);
        const int64_t tk = (s >> 1) / KSU_M;   // rb * ksteps + ks
        const int ks = (int)(tk % ksteps);
        const int64_t v = (tk / ksteps) * KSU_M + row;
        const int k0 = ks * KSU_KSTEP + half * 16;
        uint8_t d[16];
        int j = k0 / KSL, t = k0 % KSL;
        int32_t x = 0;
        // digits of coefficient j up to level t
        auto start = [&](int jj) {
            x = (v < args.V && jj < prm.N) ? center_q(args.ext[v * prm.ext_stride + jj], prm.log2q) : 0;
        };
        start(j);
        for (int lv = 0; lv < t; ++lv) ks_digit(x, prm.ks_log);
#pragma unroll
        for (int e = 0; e < 16; ++e) {
            const int k = k0 + e;
            d[e] = (uint8_t)(int8_t)(k < K ? ks_digit(x, prm.ks_log) : 0);
            if (++t == KSL) {
                t = 0;
                start(++j);
            }
        }
        uint8_t* dst = dig + (size_t)tk * KSU_A_STEP + ksu_tile_off(row, half * 16);
        *reinterpret_cast<uint4*>(dst) = *reinterpret_cast<const uint4*>(d);
    }
}

FDSNN_DEV void umma_i8(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc, uint32_t accum) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, {%5, %6, %7, %8}, p;\n\t}"
        ::"r"(tmem_d), "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accum), "r"(0), "r"(0), "r"(0), "r"(0)
        : "memory");
}

// K-major, no-swizzle descriptor of a 32-byte-wide K step tile: core matrices
// adjacent in K at +128 B (LBO), 8-row groups at +256 B (SBO).
FDSNN_DEV uint64_t ksu_desc(const void* p) { return smem_desc(p, 128, 256); }

// out[v][c] = -sum_k dig[v][k] * ksk[k][c] mod q for c in this CTA's 64 columns.
template <int LIMBS>
__global__ void __launch_bounds__(128, 1) ks_umma_kernel(const KsUmmaArgs args) {
    constexpr int NB = KSU_COLS * LIMBS;          // MMA N
    constexpr int BSTEP = ksu_b_step(LIMBS);
    constexpr int ASTAGE = KSU_KPS * KSU_A_STEP, BSTAGE = KSU_KPS * BSTEP;
    constexpr uint32_t IDESC = (2u << 4)          // D = s32
                             | (1u << 7)          // A = s8
                             | (0u << 10)         // B = u8
                             | ((uint32_t)(NB >> 3) << 17) | ((uint32_t)(KSU_M >> 4) << 24);
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    uint64_t* full = reinterpret_cast<uint64_t*>(smem_raw);
    uint64_t* empty = full + KSU_STAGES;
    uint64_t* done = empty + KSU_STAGES;
    uint32_t* tslot = reinterpret_cast<uint32_t*>(done + 1);
    unsigned char* ring = smem_raw + 256;
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const int rb = blockIdx.x, ct = blockIdx.y;
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

    const uint8_t* a_src = args.dig + (size_t)rb * args.ksteps * KSU_A_STEP;
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
            tmem_commit(&empty[s]);  // stage free once these MMAs have read it
        }
        tmem_commit(done);
    }
    __syncwarp();
    mbar_wait(done, 0);
    tmem_fence_after();

    // epilogue: lane = ciphertext row, 16 output columns per chunk
    const DevParams& prm = args.prm;
    const int64_t v = (int64_t)rb * KSU_M + warp * 32 + lane;
    const uint32_t lane_addr = tacc + ((uint32_t)(warp * 32) << 16);
#pragma unroll 1
    for (int c0 = 0; c0 < KSU_COLS; c0 += 16) {
        uint32_t sum[16];
#pragma unroll
        for (int e = 0; e < 16; ++e) sum[e] = 0u;
#pragma unroll
        for (int j = 0; j < LIMBS; ++j) {
            uint32_t w[16];
            tmem_ld16_async(lane_addr + (uint32_t)(j * KSU_COLS + c0), w);
            tmem_wait16(w);
#pragma unroll
            for (int e = 0; e < 16; ++e) sum[e] += w[e] << (8 * j);
        }
        const int col = ct * KSU_COLS + c0;
        if (v < args.V) {
            uint32_t* o = args.out + v * prm.stride + col;
            if (col + 16 <= prm.n) {
#pragma unroll
                for (int e = 0; e < 16; e += 4)
                    *reinterpret_cast<uint4*>(o + e) =
                        make_uint4((0u - sum[e]) & prm.qmask, (0u - sum[e + 1]) & prm.qmask,
                                   (0u - sum[e + 2]) & prm.qmask, (0u - sum[e + 3]) & prm.qmask);
            } else {
#pragma unroll
                for (int e = 0; e < 16; ++e)
                    if (col + e < prm.n) o[e] = (0u - sum[e]) & prm.qmask;
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
