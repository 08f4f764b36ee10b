// pbs.cuh — programmable bootstrapping: modulus switch, accumulator init,
// GINX blind rotation, sample extract.  Key switching is keyswitch.cuh.
//
// Reference semantics (all bit-exact):
//   bootstrap_batch      bootstrap.py:324-341
//   rescale              ring.py:56-67   (a2N, b2N (+N//p half-slot, :526))
//   accumulator init     bootstrap.py:334-336, monomial_rotate_raw ring.py:226-242
//   CMux step i          _fold_twist_kernel bootstrap.py:193-230,
//                        einsum MAC :279, _untwist_round_add_kernel :232-249
//   sample extract       bootstrap.py:291-295
//
// Work decomposition: one group of T = M/8 threads owns one accumulator
// (2 x N int32 in shared memory) for all n CMux steps; G = 256/T groups per
// CTA.  Per step and accumulator: 2L forward transforms of the signed gadget
// digits of (X^k - 1)*ACC, a register MAC against the Fourier-domain key
// slice, 2 inverse transforms (interleaved), round and add back.
//
// Memory roles on sm_100a:
//   * shared memory: accumulators, FFT exchange buffers, and a ring of S key
//     chunks (one (step, digit) chunk = 2 polys x M complex) filled by the TMA
//     engine (cp.async.bulk + mbarrier full/empty) and shared by the G
//     accumulators of the CTA;
//   * tensor memory (TMEM, per-thread lanes, tcgen05.ld): the thread's
//     interior-pass twiddles and twist factors, fetched asynchronously ahead
//     of use so they cost neither registers nor shared-memory bandwidth;
//   * registers: the 8-point FFT vector and the 2 x 8 frequency accumulators.
// (Streaming the key chunks into TMEM with tcgen05.cp was measured too: it
// removes the key's shared-memory reads but the copy engine sustains only
// ~18 B/clk/SM with warpx2 multicast and the pipeline ran 25% slower.)
// The Fourier key is pre-scaled by 1/M (exact), so the inverse transform's
// untwist is a multiply by conj(twist).
#pragma once
#include "fft.cuh"
#ifndef FDSNN_SKIP_ENTRY
#define FDSNN_SKIP_ENTRY 1
#endif
#ifndef FDSNN_EARLY_KEYS
#define FDSNN_EARLY_KEYS 1
#endif
#ifndef FDSNN_SKEW
#define FDSNN_SKEW 2  // start half the accumulators of a CTA late: 1 = one transform pair, 2 = ~0.6 pair
#endif

namespace fdsnn {

struct PbsArgs {
    DevParams prm;
    // input mode A: LWE rows
    const uint32_t* in;    // count x stride (may be null in mode B)
    const uint32_t* in2;   // optional second operand added to `in` (LIF charge)
    int64_t count;         // rows per LUT
    int nlut;              // virtual ciphertexts = nlut * count
    int64_t v_base;        // first virtual ciphertext of this launch (a launch may cover a sub-range)
    const int32_t* lut[4]; // device test polynomials (N residues)
    uint32_t in_boff[4];   // added to b before the modulus switch (mod q)
    // input mode B: raw accumulators + rotation indices (blind_rotate_batch)
    int32_t* acc_io;       // count x 2 x N
    const int32_t* a2N_in; // count x n
    // key: (n, 2L, 2, M) Fourier-domain RGSW rows, scaled by 1/M
    const double2* bsk;
    // tables: twist[M] | interior twiddles (fft.cuh layout)
    const double2* tables;
    // output mode A: extracted z-LWE rows (virtual ct v at v*ext_stride)
    uint32_t* ext_out;
    unsigned long long* margin;  // optional max |x - round(x)| (as double bits)
    // warp-per-rotation kernel (pbs16.cuh, M = 512): key in its layout, lane table
    const double2* bsk16;
    const double2* tab16;
};

template <int M>
struct PbsShape {
    static constexpr int T = M / 8;
    // M = 1024: two 512-point regions, the odd one 4 slots (64 B) further so
    // that even and odd lanes of a quarter-warp hit different banks
    static constexpr int PADM = M == 1024 ? FFT1024_HALF + 576 : M + M / 8;
};

template <int M>
__host__ __device__ constexpr size_t pbs_group_bytes(int N, int n) {
    return 2 * PbsShape<M>::PADM * sizeof(double2)   // exchange buffers
           + 2 * (size_t)N * sizeof(int32_t)          // accumulator
           + (((size_t)n * sizeof(uint16_t) + 15) & ~(size_t)15);  // a2N
}

constexpr int PBS_THREADS = 256;
// Groups are PBS_GROUP_PAD bytes apart beyond their size (a multiple of 128 B),
// so two interleaved groups' 16-byte exchange accesses fall in opposite halves
// of the 32 banks.
constexpr size_t PBS_GROUP_PAD = 64;
#ifndef FDSNN_ILV
#define FDSNN_ILV 1  // M = 512, G = 4: accumulator pairs interleaved lane by lane (key loads broadcast)
#endif
#ifndef FDSNN_RING_S
#define FDSNN_RING_S 5
#endif
template <int M> struct PbsRing { static constexpr int S = (M == 1024) ? 3 : FDSNN_RING_S; };
static_assert(FDSNN_RING_S >= 2 && FDSNN_RING_S <= 7, "mbarriers live in the 120-byte ring header");
template <int M>
__host__ __device__ constexpr size_t pbs_chunk_bytes() { return (size_t)2 * M * sizeof(double2); }

// 6 rotations per CTA (12 warps) leave room for only 3 ring stages
template <int M>
__host__ __device__ constexpr int pbs_stages(int G) { return G >= 6 ? 3 : PbsRing<M>::S; }
template <int M>
__host__ __device__ constexpr size_t pbs_smem_bytes(int G, int N, int n) {
    return 128 + (size_t)pbs_stages<M>(G) * pbs_chunk_bytes<M>() + (size_t)G * (pbs_group_bytes<M>(N, n) + PBS_GROUP_PAD);
}

template <int M>
FDSNN_DEV void load_twist(double2 (&tw)[8], int t, const double2* __restrict__ tables) {
#pragma unroll
    for (int r = 0; r < 8; ++r) tw[r] = __ldg(tables + t + r * (M / 8));
}

// Per-thread transform constants.  M = 1024 (parity split, fft.cuh): the
// 512-point twiddles of t' = t >> 1 from the M = 512 table, then the radix-2
// factors w^{t' + 64 r}; host table layout [twist(M) | twiddles | radix-2].
template <int M>
FDSNN_DEV void load_tw_regs(TwiddlesInRegs<M>& tw, int t, const double2* __restrict__ tables) {
    if constexpr (M == 1024) {
        load_twiddles<512>(tw.half.tw, t >> 1, tables + 1024);
        const double2* r2 = tables + 1024 + twiddle_table_size<512>();
#pragma unroll
        for (int r = 0; r < 8; ++r) {  // join factors (fft.cuh r2_join): w^{t'+64r} (even), w^{-(t'+64(r+4))} (odd)
            if (r >= 4) {
                tw.r2[r] = make_double2(0.0, 0.0);
            } else if (t & 1) {
                const double2 w = __ldg(r2 + (t >> 1) + 64 * (r + 4));
                tw.r2[r] = make_double2(w.x, -w.y);
            } else {
                tw.r2[r] = __ldg(r2 + (t >> 1) + 64 * r);
            }
        }
    } else {
        load_twiddles<M>(tw.tw, t, tables + M);
    }
}

FDSNN_DEV void tmem_st_c8(uint32_t col, const double2 (&c)[8]) {
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        double d[8];
#pragma unroll
        for (int r = 0; r < 4; ++r) { d[2 * r] = c[4 * h + r].x; d[2 * r + 1] = c[4 * h + r].y; }
        tmem_st16(col + 16 * h, d);
    }
}

// interior-pass twiddles (cols 0..), M = 1024 also the radix-2 factors (64-95)
template <int M>
FDSNN_DEV void tmem_store_twiddles(uint32_t lane_base, int t, const double2* __restrict__ tables) {
    TwiddlesInRegs<M> twr;
    load_tw_regs<M>(twr, t, tables);
    constexpr int MS = M == 1024 ? 512 : M;
    const Twiddles<MS>& tt = [&]() -> const Twiddles<MS>& {
        if constexpr (M == 1024) return twr.half.tw; else return twr.tw;
    }();
#pragma unroll
    for (int p = 1; p < Schedule<MS>::P; ++p) {
        double2 c[8];
#pragma unroll
        for (int r = 0; r < 8; ++r) c[r] = tt.w[p][r < 7 ? r : 6];
        tmem_st_c8(lane_base + (p - 1) * 32, c);
    }
    if constexpr (M == 1024) tmem_st_c8(lane_base + 64, twr.r2);
}

// TMEM columns per lane (256 allocated): interior-pass twiddles of pass p at
// (p-1)*32 (8 complex), twist factors at 96 (8 complex) -- the warps sharing a
// lane quadrant (w, w+4) have the same in-group index t, so one copy each --
// and at 128 + 32*(w/4) the thread's own accumulator coefficients
// acc[c][t + rT + h*M] (word 16c + 8h + r): the unrotated operand of
// (X^k - 1)*ACC and the read half of the accumulator update come from TMEM,
// so shared memory only serves the rotated reads and the update stores.
constexpr uint32_t PBS_TMEM_COLS = 256;
constexpr uint32_t PBS_TMEM_TWIST = 96;
constexpr uint32_t PBS_TMEM_OWN = 128;

// PAIR (gadget levels L == 2): the two levels of a polynomial are transformed
// together (fft_group2: two independent transforms per thread, one barrier
// pair per exchange) and MAC'd together; the first polynomial's partial
// frequency accumulators wait in TMEM (columns 256 + 64*(w/4)) while the
// second polynomial is transformed.
template <int M, int G, bool MODE_RAW, bool TRACK_MARGIN, bool PAIR = false, int LQ = 2>
#ifdef FDSNN_MAXNREG
__global__ void __maxnreg__(FDSNN_MAXNREG)
#else
__global__ void __launch_bounds__(G * (M / 8), 1)
#endif
pbs_blind_rotate_kernel(const PbsArgs args) {
    constexpr uint32_t TMEM_COLS = PAIR ? 512 : PBS_TMEM_COLS;
    constexpr int NA = 2 * M;  // words per accumulator poly
    constexpr int T = M / 8;
    constexpr int PADM = PbsShape<M>::PADM;
    constexpr int S = pbs_stages<M>(G);
    constexpr uint32_t CHUNK = (uint32_t)pbs_chunk_bytes<M>();
    const DevParams& prm = args.prm;
    constexpr int N = 2 * M;
    const int n = prm.n;
    const int L = prm.L;
    const uint32_t qmask = prm.qmask;
    constexpr int log2_2N = (M == 256) ? 10 : (M == 512) ? 11 : 12;

    extern __shared__ __align__(128) unsigned char smem_raw[];
    uint64_t* full = reinterpret_cast<uint64_t*>(smem_raw);   // key chunk landed
    uint64_t* empty = full + S;                                // ring stage free (2S <= 15 slots)
    uint32_t* tmem_base_slot = reinterpret_cast<uint32_t*>(smem_raw + 120);
    double2* ring = reinterpret_cast<double2*>(smem_raw + 128);
    const int warp = threadIdx.x / 32;
    // ILV: groups 2h and 2h+1 share warps 4h..4h+3, lane parity = group, so
    // the two lanes of a pair hold the same t and their key-slice loads in the
    // MAC hit one address (a broadcast: half the shared-memory wavefronts).
    constexpr bool ILV = FDSNN_ILV && M == 512 && G == 4 && PAIR;
    const int g = ILV ? 2 * (threadIdx.x / (2 * T)) + (threadIdx.x & 1) : threadIdx.x / T;
    const int t = ILV ? (threadIdx.x % (2 * T)) >> 1 : threadIdx.x % T;
    unsigned char* mine = smem_raw + 128 + S * CHUNK + g * (pbs_group_bytes<M>(N, n) + PBS_GROUP_PAD);
    double2* buf0 = reinterpret_cast<double2*>(mine);
    double2* buf1 = buf0 + PADM;
    int32_t* acc = reinterpret_cast<int32_t*>(buf1 + PADM);  // [2][NA]
    uint16_t* a2N = reinterpret_cast<uint16_t*>(acc + 2 * NA);
    auto ax = [&](int j) { return j; };  // accumulator word of coefficient j
    auto coef = [&](int r, int h) { return t + r * T + h * M; };

    const int64_t V = (int64_t)args.nlut * args.count;
    const int64_t v0 = args.v_base + (int64_t)blockIdx.x * G;
    const int nact = (int)((V - v0) < G ? (V - v0) : G);  // active groups in this CTA
    // ILV runs an odd last group's partner as a shadow of it (same rotation,
    // no output) so both lanes of every pair take part in the pair barrier.
    const int nrun = ILV ? ((nact + 1) & ~1) : nact;
    const bool active = g < nrun;
    const int nchunks = n * 2 * L;  // 32-bit: stage index and phase by constant division
    const bool producer = threadIdx.x == 0;
    if (producer) {
        for (int s = 0; s < S; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], nrun * T);
        }
        fence_mbar_init();
    }
    if (warp == 0) tmem_alloc(tmem_base_slot, TMEM_COLS);
    tmem_fence_before();
    __syncthreads();
    tmem_fence_after();
    const uint32_t tbase = *tmem_base_slot;
    const uint32_t lane_base = tbase + ((uint32_t)((warp % 4) * 32) << 16);

    // ---- per-thread constants -> TMEM (warps 0-3 cover all lane quadrants)
    if (warp < 4 && active) {
        double2 twist[8];
        {
            tmem_store_twiddles<M>(lane_base, t, args.tables);
            load_twist<M>(twist, t, args.tables);
        }
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            double d[8];
#pragma unroll
            for (int r = 0; r < 4; ++r) { d[2 * r] = twist[4 * h + r].x; d[2 * r + 1] = twist[4 * h + r].y; }
            tmem_st16(lane_base + PBS_TMEM_TWIST + 16 * h, d);
        }
        tmem_wait_st();
    }
    tmem_fence_before();
    __syncthreads();
    tmem_fence_after();

    // ---- key ring: the producer (thread 0) fills S stages ahead; every
    // consumer thread arrives on `empty` after its MAC, and the producer then
    // refills that stage with chunk c+S.
    if (producer) {
        for (int s = 0; s < S && s < nchunks; ++s) {
            mbar_arrive_expect_tx(&full[s], CHUNK);
            bulk_g2s(ring + (size_t)s * 2 * M, args.bsk + (size_t)s * 2 * M, CHUNK, &full[s]);
        }
    }
    // With the phase skew the refills are issued by the last (trailing) group:
    // by the time it releases a stage every leading group has released it too,
    // so the refill never waits on a group that is half a step behind.
    const bool skewed = PAIR && FDSNN_SKEW && G == 4 && nrun > G / 2;
    const int last_tid = ILV ? 2 * T * ((nrun - 1) / 2) + ((nrun - 1) & 1) : (nact - 1) * T;
    const bool refiller = threadIdx.x == (skewed ? last_tid : 0);
    auto release = [&](int c) {
        const int s = (int)(c % S);
        mbar_arrive(&empty[s]);
        if (refiller && c + S < nchunks) {
            mbar_wait(&empty[s], (uint32_t)((c / S) & 1));
            mbar_arrive_expect_tx(&full[s], CHUNK);
            bulk_g2s(ring + (size_t)s * 2 * M, args.bsk + (size_t)(c + S) * 2 * M, CHUNK, &full[s]);
        }
    };

    if (active) {
        const int64_t v = v0 + (g < nact ? g : nact - 1);
        const GroupSync gs{ILV ? 1 + g / 2 : 1 + g, ILV ? 2 * T : T};
        const TwiddlesInTmem<M> tw{lane_base};

        // ---------------- setup: modulus switch + accumulator init -------------
        if constexpr (!MODE_RAW) {
            const int u = (int)(v / args.count);
            const int64_t row = v - (int64_t)u * args.count;
            const uint32_t* a_in = args.in + row * prm.stride;
            const uint32_t* a_in2 = args.in2 ? args.in2 + row * prm.stride : nullptr;
            for (int i = t; i < n; i += T) {
                uint32_t a = a_in[i];
                if (a_in2) a += a_in2[i];
                a2N[i] = (uint16_t)rescale_q_to_2N(a, prm.log2q, log2_2N);
            }
            uint32_t b = a_in[n] + args.in_boff[u];
            if (a_in2) b += a_in2[n];
            const uint32_t b2N = (rescale_q_to_2N(b, prm.log2q, log2_2N) + prm.half_slot) & (2 * N - 1);
            const int32_t* lut = args.lut[u];
            // acc_b = X^{-b2N} * v  (monomial_rotate_raw with k = -b2N mod 2N)
            for (int j = t; j < N; j += T) {
                acc[ax(j)] = 0;
                const int src = (j + (int)b2N) & (2 * N - 1);
                const int32_t val = lut[src & (N - 1)];
                acc[NA + ax(j)] = (int32_t)((uint32_t)(src >= N ? -val : val) & qmask);
            }
        } else {
            const int32_t* a_src = args.acc_io + v * 2 * N;
            for (int j = t; j < 2 * N; j += T) acc[(j >= N ? NA : 0) + ax(j & (N - 1))] = (int32_t)((uint32_t)a_src[j] & qmask);
            const int32_t* k_src = args.a2N_in + v * n;
            for (int i = t; i < n; i += T) a2N[i] = (uint16_t)(k_src[i] & (2 * N - 1));
        }
        gs.sync();
        const uint32_t own_col = lane_base + PBS_TMEM_OWN + 32 * (uint32_t)(warp / 4);
        const uint32_t o_col = lane_base + 256 + 64 * (uint32_t)(warp / 4);  // PAIR only
        {
            uint32_t w[32];
#pragma unroll
            for (int cc = 0; cc < 2; ++cc)
#pragma unroll
                for (int h = 0; h < 2; ++h)
#pragma unroll
                    for (int r = 0; r < 8; ++r) w[16 * cc + 8 * h + r] = (uint32_t)acc[cc * NA + ax(coef(0, 0)) + r * T + h * M];
            tmem_st32(own_col, w);
            tmem_wait_st();
        }

        const int bg = prm.bg_log;
        const int32_t halfB1 = (1 << (bg - 1)) - 1;  // B/2 - 1
        const int32_t bmask = (1 << bg) - 1;
        // Signed gadget digits by offset (rgsw.py:130-132 rule): with
        // y = x + H, H = (B/2-1)(1 + B + ... + B^(l-1)), digit lvl of the centred
        // x is ((y >> bg*lvl) & (B-1)) - (B/2-1) -- the offset absorbs the
        // carries, so each level costs a shift, a mask and a subtract.
        int32_t hsum = 0;
        for (int lvl = 0; lvl < L; ++lvl) hsum += halfB1 << (bg * lvl);
        const uint32_t halfq = 1u << (prm.log2q - 1);
        const int32_t yoff = hsum - (int32_t)halfq;
        int ex = 0;
        double err_max = 0.0;

        // Phase skew: the leading half of the accumulators signals after the
        // first pair of step 0 and the trailing half starts only then, so the
        // two warps of a scheduler (groups g and g + G/2) stay half a step
        // apart -- one in its exchanges while the other runs butterflies.
        const bool lead = g < G / 2;
        auto skew_arrive = [&]() {
            if (skewed && lead) asm volatile("bar.arrive 15, %0;" ::"r"(T * nrun) : "memory");
        };
        if (skewed && !lead) named_bar(15, T * nrun);

        int c = 0;      // chunk counter = i * 2L + digit
        for (int i = 0; i < n; ++i) {
            const int k = a2N[i];
            bool identity = k == 0;
            // ILV: the pair shares warps (and their barriers, warp-collective
            // TMEM accesses), so it skips only jointly; a k = 0 step run in
            // full adds exactly zero (zero digits, zero spectrum, zero rounding).
            if constexpr (ILV) identity = (k | __shfl_xor_sync(0xffffffffu, k, 1)) == 0;  // every lane shuffles
            if (identity) {  // X^0*ACC - ACC = 0: identity step; keep the key pipeline in sync
                for (int d = 0; d < 2 * L; ++d, ++c) {
                    mbar_wait(&full[c % S], (uint32_t)((c / S) & 1));
                    release(c);
                }
                if (i == 0) skew_arrive();
                continue;
            }
            double2 O0[8], O1[8];
            if constexpr (!PAIR) {
#pragma unroll
                for (int r = 0; r < 8; ++r) O0[r] = O1[r] = make_double2(0.0, 0.0);
            }

            // rotated reads X^k*ACC at {t + rT, t + rT + M} of poly cc.  Both
            // polys are read up front: the second set's shared-memory latency
            // hides behind the first poly's transforms.
            uint32_t rvs[2][16];
            const int rbase = ax((coef(0, 0) - k) & (2 * N - 1));
#pragma unroll
            for (int cc = 0; cc < 2; ++cc) {
                const int32_t* a = acc + cc * NA;
#pragma unroll
                for (int r = 0; r < 8; ++r) {
#pragma unroll
                    for (int half = 0; half < 2; ++half) {
                        const int s = (rbase + r * T + half * M) & (2 * N - 1);
                        const uint32_t val = (uint32_t)a[s & (N - 1)];
                        rvs[cc][8 * half + r] = (s & N) ? (uint32_t)(-val) : val;
                    }
                }
            }
            // y = centred((X^k - 1) ACC) + H of poly cc, lo/hi halves
            auto make_x = [&](int cc, int32_t (&xlo)[8], int32_t (&xhi)[8]) {
                uint32_t ow[16];
                tmem_ld16_async(own_col + 16 * cc, ow);
                const uint32_t (&rv)[16] = rvs[cc];
                tmem_wait16(ow);
#pragma unroll
                for (int r = 0; r < 8; ++r) {
                    xlo[r] = (int32_t)((rv[r] - ow[r] + halfq) & qmask) + yoff;
                    xhi[r] = (int32_t)((rv[8 + r] - ow[8 + r] + halfq) & qmask) + yoff;
                }
            };
            if constexpr (PAIR) {
                // The 2*LQ digit polynomials (poly cc, level lvl) in key-chunk
                // order f = cc*LQ + lvl, transformed two at a time; the
                // frequency sums of all but the last pair are parked in TMEM.
                int32_t xlo[2][8], xhi[2][8];
                make_x(0, xlo[0], xhi[0]);
#pragma unroll
                for (int pr = 0; pr < LQ; ++pr) {
                    const int fa = 2 * pr, fb = 2 * pr + 1;
                    const int ca = fa / LQ, la = fa % LQ, cb = fb / LQ, lb = fb % LQ;
                    if (pr == LQ / 2) make_x(1, xlo[1], xhi[1]);  // first pair touching poly 1
                    double2 v0[8], v1[8];
                    constexpr bool FT = FDSNN_FUSED_TW;
                    double2 twv[8];
                    {
                        uint32_t twr[32];
                        tmem_ld32_async(lane_base + PBS_TMEM_TWIST, twr);
                        auto i2d = [](int32_t d) { return (double)d; };
                        int32_t d1[8], d2[8], e1[8], e2[8];
#pragma unroll
                        for (int r = 0; r < 8; ++r) {
                            d1[r] = ((xlo[ca][r] >> (bg * la)) & bmask) - halfB1;
                            d2[r] = ((xhi[ca][r] >> (bg * la)) & bmask) - halfB1;
                            e1[r] = ((xlo[cb][r] >> (bg * lb)) & bmask) - halfB1;
                            e2[r] = ((xhi[cb][r] >> (bg * lb)) & bmask) - halfB1;
                        }
                        tmem_wait32(twr);
#pragma unroll
                        for (int r = 0; r < 8; ++r) {
                            const double2 tr = words_c(twr, r);
                            if constexpr (FT) {  // twist fused into the first pass
                                twv[r] = tr;
                                v0[r] = make_double2(i2d(d1[r]), i2d(d2[r]));
                                v1[r] = make_double2(i2d(e1[r]), i2d(e2[r]));
                            } else {
                                v0[r] = cmul(make_double2(i2d(d1[r]), i2d(d2[r])), tr);
                                v1[r] = cmul(make_double2(i2d(e1[r]), i2d(e2[r])), tr);
                            }
                        }
                    }
                    const int s0 = (int)(c % S), s1 = (int)((c + 1) % S);
                    // key chunks landed: waited for before the last pass, so
                    // the MAC's key loads may be scheduled into it
                    auto keys_ready = [&]() {
                        if (FDSNN_SKEW == 2 && i == 0 && pr == 0) skew_arrive();
                        mbar_wait(&full[s0], (uint32_t)((c / S) & 1));
                        mbar_wait(&full[s1], (uint32_t)(((c + 1) / S) & 1));
                    };
                    if constexpr (FDSNN_EARLY_KEYS) {
                        // the first pair of a step follows the step's closing
                        // barrier, which already fences the buffers' last readers
                        if (pr == 0 && FDSNN_SKIP_ENTRY)
                            fft_group2<M, false, TwiddlesInTmem<M>, decltype(keys_ready), false, FT>(
                                v0, v1, t, tw, buf0, buf1, gs, keys_ready, twv);
                        else
                            fft_group2<M, false, TwiddlesInTmem<M>, decltype(keys_ready), true, FT>(
                                v0, v1, t, tw, buf0, buf1, gs, keys_ready, twv);
                    } else {
                        fft_group2<M, false>(v0, v1, t, tw, buf0, buf1, gs);
                        keys_ready();
                    }
                    const double2* k0 = ring + (size_t)s0 * 2 * M;
                    const double2* k1 = ring + (size_t)s1 * 2 * M;
                    if (pr < LQ - 1) {  // partial sums -> TMEM
                        if (pr > 0) {
                            uint32_t oa[32], ob[32];
                            tmem_ld32_async(o_col, oa);
                            tmem_ld32_async(o_col + 32, ob);
                            tmem_wait64(oa, ob);
#pragma unroll
                            for (int r = 0; r < 8; ++r) {
                                O0[r] = words_c(oa, r);
                                O1[r] = words_c(ob, r);
                            }
                        }
#pragma unroll
                        for (int h = 0; h < 2; ++h) {
                            uint32_t ow2[32];
#pragma unroll
                            for (int r = 0; r < 8; ++r) {
                                double2 o = pr > 0 ? (h ? O1[r] : O0[r]) : make_double2(0.0, 0.0);
                                cmac(o, v0[r], k0[h * M + t + r * T]);
                                cmac(o, v1[r], k1[h * M + t + r * T]);
                                put_words_c(ow2, r, o);
                            }
                            tmem_st32(o_col + 32 * h, ow2);
                        }
                        tmem_wait_st();
                    } else {
                        uint32_t oa[32], ob[32];
                        tmem_ld32_async(o_col, oa);
                        tmem_ld32_async(o_col + 32, ob);
                        tmem_wait64(oa, ob);
#pragma unroll
                        for (int r = 0; r < 8; ++r) {
                            O0[r] = words_c(oa, r);
                            O1[r] = words_c(ob, r);
                            cmac(O0[r], v0[r], k0[t + r * T]);
                            cmac(O1[r], v0[r], k0[M + t + r * T]);
                            cmac(O0[r], v1[r], k1[t + r * T]);
                            cmac(O1[r], v1[r], k1[M + t + r * T]);
                        }
                    }
                    release(c);
                    release(c + 1);
                    c += 2;
                    if (FDSNN_SKEW == 1 && i == 0 && pr == 0) skew_arrive();
                }
            } else {
#pragma unroll
            for (int cc = 0; cc < 2; ++cc) {
                int32_t xlo[8], xhi[8];
                make_x(cc, xlo, xhi);
                for (int lvl = 0; lvl < L; ++lvl, ++c) {
                    double2 vv[8];
                    {
                        uint32_t twr[32];
                        tmem_ld32_async(lane_base + PBS_TMEM_TWIST, twr);
                        int32_t d1[8], d2[8];
#pragma unroll
                        for (int r = 0; r < 8; ++r) {
                            d1[r] = (xlo[r] & bmask) - halfB1;
                            d2[r] = (xhi[r] & bmask) - halfB1;
                            xlo[r] >>= bg;
                            xhi[r] >>= bg;
                        }
                        tmem_wait32(twr);
#pragma unroll
                        for (int r = 0; r < 8; ++r)
                            vv[r] = cmul(make_double2((double)d1[r], (double)d2[r]), words_c(twr, r));
                    }
                    fft_group<M, false>(vv, t, tw, buf0, buf1, ex, gs);
                    const int s = (int)(c % S);
                    mbar_wait(&full[s], (uint32_t)((c / S) & 1));
                    const double2* kd = ring + (size_t)s * 2 * M;
#pragma unroll
                    for (int r = 0; r < 8; ++r) {
                        cmac(O0[r], vv[r], kd[t + r * T]);
                        cmac(O1[r], vv[r], kd[M + t + r * T]);
                    }
                    release(c);
                }
            }
            }
            {
                uint32_t twr[32], own[32];
                auto fetch = [&]() {
                    tmem_ld32_async(lane_base + PBS_TMEM_TWIST, twr);
                    tmem_ld32_async(own_col, own);
                };
                fft_group2<M, true>(O0, O1, t, tw, buf0, buf1, gs, fetch);
                tmem_wait32(twr);
                tmem_touch32(own);
#pragma unroll
                for (int r = 0; r < 8; ++r) {
                    const int p = ax(coef(0, 0)) + r * T, pM = p + M;
                    const double2 tr = words_c(twr, r);
                    const double2 z0 = cmulc(O0[r], tr);
                    const double2 z1 = cmulc(O1[r], tr);
                    uint32_t r00, r01, r10, r11;
                    if constexpr (TRACK_MARGIN) {
                        const long long e00 = round_product(z0.x), e01 = round_product(z0.y);
                        const long long e10 = round_product(z1.x), e11 = round_product(z1.y);
                        err_max = fmax(err_max, fabs(z0.x - (double)e00));
                        err_max = fmax(err_max, fabs(z0.y - (double)e01));
                        err_max = fmax(err_max, fabs(z1.x - (double)e10));
                        err_max = fmax(err_max, fabs(z1.y - (double)e11));
                        r00 = (uint32_t)e00; r01 = (uint32_t)e01; r10 = (uint32_t)e10; r11 = (uint32_t)e11;
                    } else {
                        r00 = round_lo32(z0.x); r01 = round_lo32(z0.y);
                        r10 = round_lo32(z1.x); r11 = round_lo32(z1.y);
                    }
                    own[r] = (own[r] + r00) & qmask;
                    own[8 + r] = (own[8 + r] + r01) & qmask;
                    own[16 + r] = (own[16 + r] + r10) & qmask;
                    own[24 + r] = (own[24 + r] + r11) & qmask;
                    acc[p] = (int32_t)own[r];
                    acc[pM] = (int32_t)own[8 + r];
                    acc[NA + p] = (int32_t)own[16 + r];
                    acc[NA + pM] = (int32_t)own[24 + r];
                }
                tmem_st32(own_col, own);
                tmem_wait_st();
            }
            gs.sync();
        }
        if constexpr (TRACK_MARGIN) {
            if (args.margin) atomicMax(args.margin, (unsigned long long)__double_as_longlong(err_max));
        }

        if (g >= nact) {  // ILV shadow group: no output
        } else if constexpr (MODE_RAW) {
            int32_t* a_dst = args.acc_io + v * 2 * N;
            for (int j = t; j < 2 * N; j += T) a_dst[j] = acc[(j >= N ? NA : 0) + ax(j & (N - 1))];
        } else {
            // sample extract (bootstrap.py:291-295): (a_0, -a_{N-1}, ..., -a_1), b = acc_b[0]
            uint32_t* out = args.ext_out + v * prm.ext_stride;
            for (int j = t; j < N; j += T) {
                const uint32_t a = (j == 0) ? (uint32_t)acc[0] : ((uint32_t)(-acc[ax(N - j)]) & qmask);
                out[j] = a;
            }
            if (t == 0) out[N] = (uint32_t)acc[NA];
        }
    }  // active
    tmem_fence_before();
    __syncthreads();
    if (warp == 0) {
        tmem_fence_after();
        tmem_dealloc(tbase, TMEM_COLS);
    }
}

// ---------------------------------------------------------------------------
// Latency variant for small batches (fewer rotations than SMs): one CTA per
// accumulator, 2L warp-pairs (256 threads at l = 2), so the 2L forward
// transforms of a CMux step run in parallel instead of one after another.
// Warp-pair p transforms digit p = (poly cc = p / L, level p % L) and multiplies
// it with its key chunk into partial frequency sums (both output polys) in its
// own exchange buffers; after a CTA barrier warp-pairs 0 and 1 add the 2L
// partials of output poly 0 / 1, run its inverse transform and update that
// accumulator poly.  Same arithmetic, same rounding, same results as
// pbs_blind_rotate_kernel; only the work split differs.
template <int M, bool MODE_RAW, bool TRACK_MARGIN, int L2>
__global__ void __launch_bounds__(L2 * (M / 8), 1)
pbs_blind_rotate_wide_kernel(const PbsArgs args) {
    constexpr int T = M / 8;
    constexpr int PADM = PbsShape<M>::PADM;
    constexpr int S = L2;  // one ring stage per digit of a step
    constexpr uint32_t CHUNK = (uint32_t)pbs_chunk_bytes<M>();
    constexpr int NT = L2 * T;
    const DevParams& prm = args.prm;
    constexpr int N = 2 * M;
    const int n = prm.n;
    constexpr int L = L2 / 2;
    const uint32_t qmask = prm.qmask;
    constexpr int log2_2N = (M == 256) ? 10 : (M == 512) ? 11 : 12;

    extern __shared__ __align__(128) unsigned char smem_raw[];
    uint64_t* full = reinterpret_cast<uint64_t*>(smem_raw);
    uint64_t* empty = full + S;
    uint32_t* tmem_base_slot = reinterpret_cast<uint32_t*>(smem_raw + 120);
    double2* ring = reinterpret_cast<double2*>(smem_raw + 128);
    const int warp = threadIdx.x / 32;
    const int wp = threadIdx.x / T;  // warp-pair = digit index
    const int t = threadIdx.x % T;
    double2* bufs = reinterpret_cast<double2*>(smem_raw + 128 + S * CHUNK);
    double2* buf0 = bufs + (size_t)wp * 2 * PADM;
    double2* buf1 = buf0 + PADM;
    int32_t* acc = reinterpret_cast<int32_t*>(bufs + (size_t)L2 * 2 * PADM);  // [2][N]
    uint16_t* a2N = reinterpret_cast<uint16_t*>(acc + 2 * N);

    const int64_t v = args.v_base + blockIdx.x;
    const int64_t nchunks = (int64_t)n * L2;
    const bool producer = threadIdx.x == 0;
    if (producer) {
        for (int s = 0; s < S; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], T);  // a chunk is read by one warp-pair
        }
        fence_mbar_init();
    }
    if (warp == 0) tmem_alloc(tmem_base_slot, PBS_TMEM_COLS);
    tmem_fence_before();
    __syncthreads();
    tmem_fence_after();
    const uint32_t tbase = *tmem_base_slot;
    const uint32_t lane_base = tbase + ((uint32_t)((warp % 4) * 32) << 16);
    if (warp < 4) {  // per-lane twiddles + twist (t depends on the lane only)
        TwiddlesInRegs<M> twr;
        load_twiddles<M>(twr.tw, t, args.tables + M);
#pragma unroll
        for (int p = 1; p < Schedule<M>::P; ++p) {
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                double d[8];
#pragma unroll
                for (int r = 0; r < 4; ++r) {
                    const double2 w = twr.tw.w[p][4 * h + r < 7 ? 4 * h + r : 6];
                    d[2 * r] = w.x;
                    d[2 * r + 1] = w.y;
                }
                tmem_st16(lane_base + (p - 1) * 32 + 16 * h, d);
            }
        }
        double2 twist[8];
        load_twist<M>(twist, t, args.tables);
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            double d[8];
#pragma unroll
            for (int r = 0; r < 4; ++r) { d[2 * r] = twist[4 * h + r].x; d[2 * r + 1] = twist[4 * h + r].y; }
            tmem_st16(lane_base + PBS_TMEM_TWIST + 16 * h, d);
        }
        tmem_wait_st();
    }
    tmem_fence_before();
    __syncthreads();
    tmem_fence_after();

    if (producer) {
        for (int s = 0; s < S && s < nchunks; ++s) {
            mbar_arrive_expect_tx(&full[s], CHUNK);
            bulk_g2s(ring + (size_t)s * 2 * M, args.bsk + (size_t)s * 2 * M, CHUNK, &full[s]);
        }
    }
    // stage s always holds digit s of the current step; warp-pair s releases
    // it after its MAC, and after the step's CTA barrier the last warp-pair
    // (idle while pairs 0 and 1 run the inverse transforms, so the copies are
    // issued off the critical path) loads the next step's chunks
    const bool refiller = threadIdx.x == (L2 - 1) * T;
    auto refill = [&](int i) {
        if (refiller && (int64_t)(i + 1) * L2 < nchunks) {
            for (int s = 0; s < S; ++s) {
                mbar_wait(&empty[s], (uint32_t)(i & 1));
                mbar_arrive_expect_tx(&full[s], CHUNK);
                bulk_g2s(ring + (size_t)s * 2 * M, args.bsk + ((size_t)(i + 1) * L2 + s) * 2 * M, CHUNK, &full[s]);
            }
        }
    };

    const GroupSync gs{1 + wp, T};
    const TwiddlesInTmem<M> tw{lane_base};
    // ---------------- setup: modulus switch + accumulator init -------------
    if constexpr (!MODE_RAW) {
        const int u = (int)(v / args.count);
        const int64_t row = v - (int64_t)u * args.count;
        const uint32_t* a_in = args.in + row * prm.stride;
        const uint32_t* a_in2 = args.in2 ? args.in2 + row * prm.stride : nullptr;
        for (int i = threadIdx.x; i < n; i += NT) {
            uint32_t a = a_in[i];
            if (a_in2) a += a_in2[i];
            a2N[i] = (uint16_t)rescale_q_to_2N(a, prm.log2q, log2_2N);
        }
        uint32_t b = a_in[n] + args.in_boff[u];
        if (a_in2) b += a_in2[n];
        const uint32_t b2N = (rescale_q_to_2N(b, prm.log2q, log2_2N) + prm.half_slot) & (2 * N - 1);
        const int32_t* lut = args.lut[u];
        for (int j = threadIdx.x; j < N; j += NT) {
            acc[j] = 0;
            const int src = (j + (int)b2N) & (2 * N - 1);
            const int32_t val = lut[src & (N - 1)];
            acc[N + j] = (int32_t)((uint32_t)(src >= N ? -val : val) & qmask);
        }
    } else {
        const int32_t* a_src = args.acc_io + v * 2 * N;
        for (int j = threadIdx.x; j < 2 * N; j += NT) acc[j] = (int32_t)((uint32_t)a_src[j] & qmask);
        const int32_t* k_src = args.a2N_in + v * n;
        for (int i = threadIdx.x; i < n; i += NT) a2N[i] = (uint16_t)(k_src[i] & (2 * N - 1));
    }
    __syncthreads();

    const int bg = prm.bg_log;
    const int32_t halfB1 = (1 << (bg - 1)) - 1;
    const int32_t bmask = (1 << bg) - 1;
    int32_t hsum = 0;
#pragma unroll
    for (int lvl = 0; lvl < L; ++lvl) hsum += halfB1 << (bg * lvl);
    const uint32_t halfq = 1u << (prm.log2q - 1);
    const int32_t yoff = hsum - (int32_t)halfq;
    const int cc = wp / L, lvl = wp % L;
    int ex = 0;
    double err_max = 0.0;

    for (int i = 0; i < n; ++i) {
        const int k = a2N[i];
        if (k == 0) {
            mbar_wait(&full[wp], (uint32_t)(i & 1));
            mbar_arrive(&empty[wp]);
            __syncthreads();
            refill(i);
            continue;
        }
        // digit `lvl` of poly `cc` of (X^k - 1) * ACC
        double2 vv[8], twv[8];
        {
            const int32_t* a = acc + cc * N;
            uint32_t twr[32];
            tmem_ld32_async(lane_base + PBS_TMEM_TWIST, twr);
            int32_t d1[8], d2[8];
#pragma unroll
            for (int r = 0; r < 8; ++r) {
                const int p = t + r * T;
                const int s0 = (p - k) & (2 * N - 1), s1 = (p + M - k) & (2 * N - 1);
                const uint32_t r0 = (s0 >= N) ? (uint32_t)(-a[s0 - N]) : (uint32_t)a[s0];
                const uint32_t r1 = (s1 >= N) ? (uint32_t)(-a[s1 - N]) : (uint32_t)a[s1];
                const int32_t y0 = (int32_t)((r0 - (uint32_t)a[p] + halfq) & qmask) + yoff;
                const int32_t y1 = (int32_t)((r1 - (uint32_t)a[p + M] + halfq) & qmask) + yoff;
                d1[r] = ((y0 >> (bg * lvl)) & bmask) - halfB1;
                d2[r] = ((y1 >> (bg * lvl)) & bmask) - halfB1;
            }
            tmem_wait32(twr);
#pragma unroll
            for (int r = 0; r < 8; ++r) {  // the twist is fused into the first pass
                twv[r] = words_c(twr, r);
                vv[r] = make_double2((double)d1[r], (double)d2[r]);
            }
        }
        // the key chunk is waited for and read into registers before the
        // transform's last pass, so those loads overlap its butterflies
        const double2* kd = ring + (size_t)wp * 2 * M;
        double2 k0[8], k1[8];
        auto fetch_key = [&]() {
            mbar_wait(&full[wp], (uint32_t)(i & 1));
#pragma unroll
            for (int r = 0; r < 8; ++r) {
                k0[r] = kd[t + r * T];
                k1[r] = kd[M + t + r * T];
            }
        };
        fft_group<M, false, TwiddlesInTmem<M>, decltype(fetch_key), true>(vv, t, tw, buf0, buf1, ex, gs, fetch_key, twv);
        gs.sync();  // the transform's last exchange reads are done before the partials overwrite
#pragma unroll
        for (int r = 0; r < 8; ++r) {
            double2 o0 = make_double2(0.0, 0.0), o1 = make_double2(0.0, 0.0);
            cmac(o0, vv[r], k0[r]);
            cmac(o1, vv[r], k1[r]);
            buf0[t + r * T] = o0;  // partial sums of output poly 0
            buf1[t + r * T] = o1;  // and 1
        }
        mbar_arrive(&empty[wp]);
        __syncthreads();  // all partials written; every accumulator read of this step done
        refill(i);
        if (wp < 2) {  // warp-pair o inverse-transforms output poly o
            const int o = wp;
            double2 O[8];
#pragma unroll
            for (int r = 0; r < 8; ++r) {
                double2 sacc = bufs[(size_t)0 * 2 * PADM + o * PADM + t + r * T];
#pragma unroll
                for (int p = 1; p < L2; ++p) sacc = cadd(sacc, bufs[(size_t)p * 2 * PADM + o * PADM + t + r * T]);
                O[r] = sacc;
            }
            named_bar(1 + L2, 2 * T);  // partial reads of warp-pairs 0/1 done before their buffers are reused
            fft_group<M, true>(O, t, tw, buf0, buf1, ex, gs);
            uint32_t twr[32];
            tmem_ld32_async(lane_base + PBS_TMEM_TWIST, twr);
            tmem_wait32(twr);
            int32_t* a = acc + o * N;
#pragma unroll
            for (int r = 0; r < 8; ++r) {
                const int p = t + r * T;
                const double2 z = cmulc(O[r], words_c(twr, r));
                const long long r0 = round_product(z.x), r1 = round_product(z.y);
                if constexpr (TRACK_MARGIN) {
                    err_max = fmax(err_max, fabs(z.x - (double)r0));
                    err_max = fmax(err_max, fabs(z.y - (double)r1));
                }
                a[p] = (int32_t)(((uint32_t)a[p] + (uint32_t)r0) & qmask);
                a[p + M] = (int32_t)(((uint32_t)a[p + M] + (uint32_t)r1) & qmask);
            }
        }
        __syncthreads();  // accumulator updated before the next step's reads
    }
    if constexpr (TRACK_MARGIN) {
        if (args.margin) atomicMax(args.margin, (unsigned long long)__double_as_longlong(err_max));
    }
    if constexpr (MODE_RAW) {
        int32_t* a_dst = args.acc_io + v * 2 * N;
        for (int j = threadIdx.x; j < 2 * N; j += NT) a_dst[j] = acc[j];
    } else {
        uint32_t* out = args.ext_out + v * prm.ext_stride;
        for (int j = threadIdx.x; j < N; j += NT) {
            const uint32_t a = (j == 0) ? (uint32_t)acc[0] : ((uint32_t)(-acc[N - j]) & qmask);
            out[j] = a;
        }
        if (threadIdx.x == 0) out[N] = (uint32_t)acc[N];
    }
    tmem_fence_before();
    __syncthreads();
    if (warp == 0) {
        tmem_fence_after();
        tmem_dealloc(tbase, PBS_TMEM_COLS);
    }
}

template <int M>
__host__ __device__ constexpr size_t pbs_wide_smem_bytes(int L2, int N, int n) {
    return 128 + (size_t)L2 * pbs_chunk_bytes<M>() + (size_t)L2 * 2 * PbsShape<M>::PADM * sizeof(double2) +
           2 * (size_t)N * sizeof(int32_t) + (((size_t)n * sizeof(uint16_t) + 15) & ~(size_t)15);
}

// Fourier transform of the bootstrapping key rows (BootstrapKey.__init__,
// bootstrap.py:125-130): centred residues -> fold, twist, forward DFT, then
// scaled by 1/M (exact) for the untwist-free epilogue above.
// One group of T threads per polynomial; G polys per CTA.
template <int M, int G>
__global__ void __launch_bounds__(G * (M / 8))
bsk_forward_kernel(const int64_t* __restrict__ rows, int64_t npoly, int log2q,
                   const double2* __restrict__ tables, double2* __restrict__ out) {
    constexpr int T = M / 8;
    constexpr int PADM = PbsShape<M>::PADM;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int g = threadIdx.x / T, t = threadIdx.x % T;
    const int64_t poly = (int64_t)blockIdx.x * G + g;
    if (poly >= npoly) return;
    double2* buf0 = reinterpret_cast<double2*>(smem_raw) + g * 2 * PADM;
    double2* buf1 = buf0 + PADM;
    const GroupSync gs{1 + g, T};
    TwiddlesInRegs<M> tw;
    load_tw_regs<M>(tw, t, tables);
    const int64_t* src = rows + poly * 2 * M;
    const int64_t qm = (1ll << log2q) - 1;
    double2 vv[8];
#pragma unroll
    for (int r = 0; r < 8; ++r) {
        const int p = t + r * T;
        const int32_t lo = center_q((uint32_t)(src[p] & qm), log2q);
        const int32_t hi = center_q((uint32_t)(src[p + M] & qm), log2q);
        vv[r] = cmul(make_double2((double)lo, (double)hi), __ldg(tables + p));
    }
    int ex = 0;
    fft_group<M, false>(vv, t, tw, buf0, buf1, ex, gs);
    if constexpr (M == 1024) {
        // odd lanes hold s X, s = z_r (register r) / -z_r (r + 4): back to the
        // true basis (fft.cuh r2_join)
        if (t & 1) {
#pragma unroll
            for (int r = 0; r < 4; ++r) {
                vv[r] = cmulc(vv[r], tw.r2[r]);
                const double2 x = cmulc(vv[r + 4], tw.r2[r]);
                vv[r + 4] = make_double2(-x.x, -x.y);
            }
        }
    }
    const double inv_m = 1.0 / M;
#pragma unroll
    for (int r = 0; r < 8; ++r)
        out[poly * M + t + r * T] = make_double2(vv[r].x * inv_m, vv[r].y * inv_m);
}

}  // namespace fdsnn
