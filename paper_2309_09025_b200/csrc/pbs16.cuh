// pbs16.cuh — throughput blind rotation, one warp per rotation (DESK rings:
// N = 1024, gadget levels l = 2).
//
// Same GINX CMux chain and arithmetic as pbs_blind_rotate_kernel (reference
// bootstrap.py:252-282: fold/twist _fold_twist_kernel :193-230, Fourier MAC
// :279, _untwist_round_add_kernel :232-249; rescale ring.py:56-67, accumulator
// init bootstrap.py:332-336, sample extract :291-295), reorganised around the
// warp-per-transform FFT of fft16.cuh:
//   * warp w of a CTA owns rotation v0 + w for all n steps: its accumulator
//     (2 x N int32) and exchange buffer in shared memory, its own accumulator
//     coefficients and the partial spectrum of output poly 1 in tensor memory.
//     No barrier couples the warps of a CTA -- only the key ring.
//   * per step and digit f = (poly cc, level lvl): digits of the centred
//     (X^k - 1) ACC_cc (rgsw.py:130-132 rule, offset form), forward transform,
//     MAC against the key chunk (step i, digit f) into the spectra of both
//     output polynomials (poly 0 in registers, poly 1 parked in TMEM);
//     then two inverse transforms, untwist, round, add.
//   * Key ring: S stages of 16 KB filled by the TMA engine (cp.async.bulk +
//     mbarrier), shared by the CTA's warps; the warp that releases a stage
//     last (smem atomic count) refills it, so no warp ever waits for another
//     warp except through the data it needs.
// Fourier key: chunk (i, f) = [h][16 registers][32 lanes] complex, scaled by
// 1/M and stored in the true frequency basis (bsk_forward16_kernel), so
// each lane's MAC reads 32 consecutive 16-byte words per register.
#pragma once
#include "pbs.cuh"
#include "fft16.cuh"

namespace fdsnn {

constexpr int BR16_MAXW = 8;   // warps (rotations) per CTA
constexpr int BR16_S = 4;      // key ring stages (3: 18% slower, 5: 0.7% slower)
constexpr uint32_t BR16_CHUNK = 2u * 512u * sizeof(double2);
// header: full[S], empty[S] mbarriers, release counters[S], TMEM address slot
constexpr size_t BR16_HDR = 128;
static_assert(20 * BR16_S + 8 <= BR16_HDR, "ring header");
// TMEM columns per lane quadrant: the lane table (3 x 32, shared by warps w
// and w + 4), then per warp (w / 4 = 0, 1) 192 columns: the partial spectra of
// output polynomials 0 and 1 (2 x 64) and the warp's own accumulator
// coefficients (2 x 32).
constexpr uint32_t BR16_TMEM_COLS = 512;
constexpr uint32_t BR16_COL_P = r16::NBLK * 32;
static_assert(BR16_COL_P + 2 * 192 <= BR16_TMEM_COLS, "TMEM columns");

__host__ __device__ constexpr size_t br16_warp_bytes(int n) {
    return 2 * 1024 * sizeof(int32_t) + r16::XBUF * sizeof(double2) + (((size_t)n * 2 + 15) & ~(size_t)15);
}
__host__ __device__ constexpr size_t br16_smem_bytes(int G, int n) {
    return BR16_HDR + (size_t)BR16_S * BR16_CHUNK + (size_t)G * br16_warp_bytes(n);
}

template <bool MODE_RAW, bool TRACK_MARGIN>
__global__ void __launch_bounds__(BR16_MAXW * 32, 1) pbs_br16_kernel(const PbsArgs args) {
    constexpr int M = 512, N = 1024, S = BR16_S, log2_2N = 11;
    constexpr uint32_t CHUNK = BR16_CHUNK;
    const DevParams& prm = args.prm;
    const int n = prm.n;
    const uint32_t qmask = prm.qmask;

    extern __shared__ __align__(128) unsigned char smem_raw[];
    uint64_t* full = reinterpret_cast<uint64_t*>(smem_raw);          // [S] stage landed
    uint64_t* empty = full + S;                                       // [S] stage released by every warp
    uint32_t* cnt = reinterpret_cast<uint32_t*>(smem_raw + 16 * S);   // [S] releases so far
    uint32_t* tslot = reinterpret_cast<uint32_t*>(smem_raw + BR16_HDR - 8);
    double2* ring = reinterpret_cast<double2*>(smem_raw + BR16_HDR);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int G = blockDim.x >> 5;
    unsigned char* mine = smem_raw + BR16_HDR + S * CHUNK + warp * br16_warp_bytes(n);
    int32_t* acc = reinterpret_cast<int32_t*>(mine);                  // [2][N]
    double2* xbuf = reinterpret_cast<double2*>(mine + 2 * N * sizeof(int32_t));
    uint16_t* a2N = reinterpret_cast<uint16_t*>(mine + 2 * N * sizeof(int32_t) + r16::XBUF * sizeof(double2));

    const int64_t V = (int64_t)args.nlut * args.count;
    const int64_t vb = args.v_base + (int64_t)blockIdx.x * G;
    const int nact = (int)((V - vb) < G ? (V - vb) : G);
    const bool active = warp < nact;
    const int nchunks = n * 4;
    if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], nact);
            cnt[s] = 0;
        }
        fence_mbar_init();
    }
    if (warp == 0) tmem_alloc(tslot, BR16_TMEM_COLS);
    tmem_fence_before();
    __syncthreads();
    tmem_fence_after();
    const uint32_t lb = *tslot + ((uint32_t)((warp & 3) * 32) << 16);
    if (warp < 4) {  // this lane's transform table -> TMEM (shared with warp + 4)
        const double2* t = args.tab16 + lane * r16::TAB;
#pragma unroll 1
        for (int b = 0; b < r16::NBLK; ++b) {
            uint32_t w[32];
#pragma unroll
            for (int i = 0; i < 8; ++i) put_words_c(w, i, __ldg(t + 8 * b + i));
            tmem_st32(lb + 32 * b, w);
        }
        tmem_wait_st();
    }
    tmem_fence_before();
    __syncthreads();
    tmem_fence_after();
    if (threadIdx.x == 0) {
        for (int s = 0; s < S && s < nchunks; ++s) {
            mbar_arrive_expect_tx(&full[s], CHUNK);
            bulk_g2s(ring + (size_t)s * 1024, args.bsk16 + (size_t)s * 1024, CHUNK, &full[s]);
        }
    }
    // Every active warp releases every chunk once; the warp whose release is
    // the stage's last (atomic count) waits for the stage's empty phase (all
    // arrivals, so it returns at once and orders the other warps' reads
    // before the copy) and refills it with chunk c + S.
    auto release = [&](int c) {
        __syncwarp();
        if (lane == 0) {
            const int s = c % S;
            const uint32_t use = (uint32_t)(c / S);
            mbar_arrive(&empty[s]);
            const uint32_t old = atomicAdd(&cnt[s], 1u);
            if (old == (use + 1) * (uint32_t)nact - 1 && c + S < nchunks) {
                mbar_wait(&empty[s], use & 1);
                mbar_arrive_expect_tx(&full[s], CHUNK);
                bulk_g2s(ring + (size_t)s * 1024, args.bsk16 + (size_t)(c + S) * 1024, CHUNK, &full[s]);
            }
        }
    };

    if (active) {
        const int64_t v = vb + warp;
        const r16::TabTmem tp{lb};
        const uint32_t p_col = lb + BR16_COL_P + 192 * (uint32_t)(warp >> 2);  // [poly 0 | poly 1] x 64 | own

        // ---------------- setup: modulus switch + accumulator init -------------
        if constexpr (!MODE_RAW) {
            const int u = (int)(v / args.count);
            const int64_t row = v - (int64_t)u * args.count;
            const uint32_t* a_in = args.in + row * prm.stride;
            const uint32_t* a_in2 = args.in2 ? args.in2 + row * prm.stride : nullptr;
            for (int i = lane; i < n; i += 32) {
                uint32_t a = a_in[i];
                if (a_in2) a += a_in2[i];
                a2N[i] = (uint16_t)rescale_q_to_2N(a, prm.log2q, log2_2N);
            }
            uint32_t b = a_in[n] + args.in_boff[u];
            if (a_in2) b += a_in2[n];
            const uint32_t b2N = (rescale_q_to_2N(b, prm.log2q, log2_2N) + prm.half_slot) & (2 * N - 1);
            const int32_t* lut = args.lut[u];
            // acc_b = X^{-b2N} * v  (monomial_rotate_raw with k = -b2N mod 2N)
            for (int j = lane; j < N; j += 32) {
                acc[j] = 0;
                const int src = (j + (int)b2N) & (2 * N - 1);
                const int32_t val = lut[src & (N - 1)];
                acc[N + j] = (int32_t)((uint32_t)(src >= N ? -val : val) & qmask);
            }
        } else {
            const int32_t* a_src = args.acc_io + v * 2 * N;
            for (int j = lane; j < 2 * N; j += 32) acc[j] = (int32_t)((uint32_t)a_src[j] & qmask);
            const int32_t* k_src = args.a2N_in + v * n;
            for (int i = lane; i < n; i += 32) a2N[i] = (uint16_t)(k_src[i] & (2 * N - 1));
        }
        __syncwarp();
        {  // own coefficients -> TMEM: word 2 j2 = coef lane + 32 j2, word 2 j2 + 1 = coef lane + 32 j2 + M
            const uint32_t own_col = p_col + 128;
#pragma unroll
            for (int cc = 0; cc < 2; ++cc) {
                uint32_t w[32];
#pragma unroll
                for (int j = 0; j < 16; ++j) {
                    w[2 * j] = (uint32_t)acc[cc * N + lane + 32 * j];
                    w[2 * j + 1] = (uint32_t)acc[cc * N + lane + 32 * j + M];
                }
                tmem_st32(own_col + 32 * cc, w);
            }
            tmem_wait_st();
        }
        const int bg = prm.bg_log;
        const int32_t halfB1 = (1 << (bg - 1)) - 1;  // B/2 - 1
        const int32_t bmask = (1 << bg) - 1;
        // signed digits by offset: y = x + H, H = (B/2-1)(1 + B), digit lvl =
        // ((y >> bg*lvl) & (B-1)) - (B/2-1)
        const int32_t hsum = halfB1 + (halfB1 << bg);
        const uint32_t halfq = 1u << (prm.log2q - 1);
        const int32_t yoff = hsum - (int32_t)halfq;
        double err_max = 0.0;

        int c = 0;  // chunk = 4 i + 2 cc + lvl
        const uint32_t own_col = p_col + 128;  // own accumulator coefficients (2 x 32 words)
#pragma unroll 1
        for (int i = 0; i < n; ++i) {
            const int k = a2N[i];
            if (k == 0) {  // X^0 ACC - ACC = 0: identity step; keep the key ring in step
#pragma unroll 1
                for (int d = 0; d < 4; ++d, ++c) {
                    mbar_wait(&full[c % S], (uint32_t)((c / S) & 1));
                    release(c);
                }
                continue;
            }
#pragma unroll
            for (int cc = 0; cc < 2; ++cc) {
                uint32_t dpk[16];  // level-1 digits, (coef p | coef p + M << 16)
                double2 vv[16];
                {
                    const int32_t* a = acc + cc * N;
                    const int base = lane - k;
#pragma unroll
                    for (int g = 0; g < 4; ++g) {  // 4 points (8 rotated reads + 8 own words) at a time
                        uint32_t ow[8];
                        tmem_ld8_async(own_col + 32 * cc + 8 * g, ow);
                        uint32_t rv[8];
#pragma unroll
                        for (int jj = 0; jj < 4; ++jj) {
#pragma unroll
                            for (int h = 0; h < 2; ++h) {
                                const int s = (base + 32 * (4 * g + jj) + h * M) & (2 * N - 1);
                                const uint32_t val = (uint32_t)a[s & (N - 1)];
                                rv[2 * jj + h] = (s & N) ? (uint32_t)(-val) : val;
                            }
                        }
                        tmem_wait8(ow);
#pragma unroll
                        for (int jj = 0; jj < 4; ++jj) {
                            const int j = 4 * g + jj;
                            const int32_t ylo = (int32_t)((rv[2 * jj] - ow[2 * jj] + halfq) & qmask) + yoff;
                            const int32_t yhi = (int32_t)((rv[2 * jj + 1] - ow[2 * jj + 1] + halfq) & qmask) + yoff;
                            vv[j] = make_double2((double)((ylo & bmask) - halfB1), (double)((yhi & bmask) - halfB1));
                            const uint32_t d1lo = (uint32_t)(((ylo >> bg) & bmask) - halfB1) & 0xFFFFu;
                            const uint32_t d1hi = (uint32_t)(((yhi >> bg) & bmask) - halfB1);
                            dpk[j] = d1lo | (d1hi << 16);
                        }
                    }
                }
#pragma unroll
                for (int lvl = 0; lvl < 2; ++lvl, ++c) {
                    const int f = 2 * cc + lvl;
                    if (lvl == 1) {
#pragma unroll
                        for (int j = 0; j < 16; ++j) {
                            asm volatile("" : "+r"(dpk[j]));  // keep the unpack after the level-0 MAC
                            vv[j] = make_double2((double)(int16_t)(dpk[j] & 0xFFFFu), (double)((int32_t)dpk[j] >> 16));
                        }
                    }
                    r16::forward(vv, lane, tp, xbuf);
                    const int s = c % S;
                    mbar_wait(&full[s], (uint32_t)((c / S) & 1));
                    const double2* K = ring + (size_t)s * 1024 + lane;
                    // MAC into both output spectra (TMEM, 64 columns each), 8
                    // frequencies (32 columns) at a time, one double per
                    // tcgen05.ld / st (no register staging, common.cuh)
                    // (the loads of piece hq + 1 are in flight while piece hq is
                    // multiplied)
                    uint32_t q[4][32];
                    if (f > 0) tmem_ld32_pairs_async(p_col, q[0]);
#pragma unroll
                    for (int hq = 0; hq < 4; ++hq) {
                        const uint32_t col = p_col + 32 * hq;
                        if (f > 0) {
                            tmem_wait32(q[hq]);
                            if (hq < 3) tmem_ld32_pairs_async(col + 32, q[hq + 1]);
                        }
#pragma unroll
                        for (int j = 0; j < 8; ++j) {
                            const int jj = 8 * (hq & 1) + j;
                            const double2 kk = K[512 * (hq >> 1) + 32 * jj];
                            double2 z;
                            if (f == 0) z = cmul(vv[jj], kk);
                            else {
                                z = words_c(q[hq], j);
                                cmac(z, vv[jj], kk);
                            }
                            tmem_st_c(col + 4 * j, z);
                        }
                    }
                    release(c);
                    tmem_wait_st();
                }
            }
            // ---- inverse transforms, untwist, round, add (poly 0 then 1)
#pragma unroll
            for (int cc = 0; cc < 2; ++cc) {
                double2 O[16];
                {
                    uint32_t w0[32], w1[32];
                    tmem_ld32_async(p_col + 64 * cc, w0);
                    tmem_ld32_async(p_col + 64 * cc + 32, w1);
                    tmem_wait64(w0, w1);
#pragma unroll
                    for (int j = 0; j < 8; ++j) {
                        O[j] = words_c(w0, j);
                        O[8 + j] = words_c(w1, j);
                    }
                }
                r16::inverse(O, lane, tp, xbuf);
                uint32_t ow[32];
                tmem_ld32_async(own_col + 32 * cc, ow);
                int32_t* a = acc + cc * N;
                tmem_wait32(ow);
#pragma unroll
                for (int j = 0; j < 16; ++j) {
                    const double2 z = cmulc(O[j], r16::g_twist(j));
                    uint32_t r0, r1;
                    if constexpr (TRACK_MARGIN) {
                        const long long e0 = round_product(z.x), e1 = round_product(z.y);
                        err_max = fmax(err_max, fabs(z.x - (double)e0));
                        err_max = fmax(err_max, fabs(z.y - (double)e1));
                        r0 = (uint32_t)e0;
                        r1 = (uint32_t)e1;
                    } else {
                        r0 = round_lo32_fp64(z.x);
                        r1 = round_lo32_fp64(z.y);
                    }
                    ow[2 * j] = (ow[2 * j] + r0) & qmask;
                    ow[2 * j + 1] = (ow[2 * j + 1] + r1) & qmask;
                    a[lane + 32 * j] = (int32_t)ow[2 * j];
                    a[lane + 32 * j + M] = (int32_t)ow[2 * j + 1];
                }
                tmem_st32(own_col + 32 * cc, ow);
            }
            tmem_wait_st();
            __syncwarp();  // the accumulator update is visible to the next step's rotated reads
        }
        if constexpr (TRACK_MARGIN) {
            if (args.margin) atomicMax(args.margin, (unsigned long long)__double_as_longlong(err_max));
        }
        if constexpr (MODE_RAW) {
            int32_t* a_dst = args.acc_io + v * 2 * N;
            for (int j = lane; j < 2 * N; j += 32) a_dst[j] = acc[j];
        } else {
            // sample extract (bootstrap.py:291-295): (a_0, -a_{N-1}, ..., -a_1), b = acc_b[0]
            uint32_t* out = args.ext_out + v * prm.ext_stride;
            for (int j = lane; j < N; j += 32)
                out[j] = (j == 0) ? (uint32_t)acc[0] : ((uint32_t)(-acc[N - j]) & qmask);
            if (lane == 0) out[N] = (uint32_t)acc[N];
        }
    }  // active
    tmem_fence_before();
    __syncthreads();
    if (warp == 0) {
        tmem_fence_after();
        tmem_dealloc(*tslot, BR16_TMEM_COLS);
    }
}

// Fourier transform of the bootstrapping key rows for pbs_br16_kernel
// (BootstrapKey.__init__, bootstrap.py:125-130): centred residues -> the
// fft16.cuh forward transform, odd lanes rotated back to the true frequency
// basis (conj(s)), scaled by 1/M, stored [poly][register][lane].
__global__ void __launch_bounds__(128) bsk_forward16_kernel(const int64_t* __restrict__ rows, int64_t npoly,
                                                            int log2q, const double2* __restrict__ tab16,
                                                            double2* __restrict__ out) {
    constexpr int M = 512;
    __shared__ double2 xb[4][r16::XBUF];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t poly = (int64_t)blockIdx.x * 4 + warp;
    if (poly >= npoly) return;
    const double2* t = tab16 + lane * r16::TAB;
    const int64_t* src = rows + poly * 2 * M;
    const int64_t qm = (1ll << log2q) - 1;
    double2 v[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) {
        const int p = lane + 32 * j;
        v[j] = make_double2((double)center_q((uint32_t)(src[p] & qm), log2q),
                            (double)center_q((uint32_t)(src[p + M] & qm), log2q));
    }
    r16::forward(v, lane, r16::TabGlobal{t}, xb[warp]);
    const double inv_m = 1.0 / M;
#pragma unroll
    for (int r = 0; r < 8; ++r) {
        double2 x0 = v[r], x1 = v[r + 8];
        if (lane & 1) {  // odd lanes hold s X: multiply by conj(s) (fft16.cuh header)
            const double2 z = __ldg(t + 8 * r16::BLK_ZJ + r);
            x0 = cmulc(x0, z);
            x1 = cmulc(x1, z);
            x1 = make_double2(-x1.x, -x1.y);
        }
        out[poly * M + 32 * r + lane] = make_double2(x0.x * inv_m, x0.y * inv_m);
        out[poly * M + 32 * (r + 8) + lane] = make_double2(x1.x * inv_m, x1.y * inv_m);
    }
}

}  // namespace fdsnn
