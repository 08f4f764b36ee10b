// pbs_cluster.cuh — latency-regime blind rotation: one rotation on a CTA pair.
//
// Same GINX CMux chain as pbs_blind_rotate_kernel (reference
// bootstrap.py:252-282, fold/twist :193-230, MAC :279, untwist/round/add
// :232-249), split across the two SMs of a thread-block cluster by
// accumulator polynomial: CTA c (c = 0 mask, 1 body) owns ACC_c.  Per step:
//   1. digits of (X^k - 1) ACC_c, both gadget levels (rgsw.py:130-132 rule);
//   2. the two digit transforms as one pipelined pair (fft_group2);
//   3. MAC against the key chunks of digit rows c*L + l: the thread's
//      frequencies of BOTH output polynomials, P_0 and P_1;
//   4. P_{1-c} goes to the partner CTA's receive buffer with st.async
//      (distributed shared memory, completion counted on the partner's
//      mbarrier), P_c stays;
//   5. O_c = P_c + partner's P_c, inverse transform, untwist, round, add into
//      ACC_c.
// The sum of the four digit products is formed in the frequency domain
// exactly as in the one-SM kernels, so the rounding and the results are
// identical.  Twice the SMs per rotation, half the serial transform work per
// SM per step: for batches below one wave of SM pairs this halves the
// latency of a bootstrap.  G rotations share a CTA pair (and its key ring).
#pragma once
#include "fft.cuh"

namespace fdsnn {

FDSNN_DEV uint32_t cluster_ctarank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
FDSNN_DEV void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// shared::cta address of `p` in CTA `rank` of this cluster (shared::cluster window)
FDSNN_DEV uint32_t mapa_shared(const void* p, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(smem_u32(p)), "r"(rank));
    return r;
}
// 16-byte asynchronous store into another CTA's shared memory; the bytes are
// counted on that CTA's mbarrier (complete_tx) when they have landed.
FDSNN_DEV void st_async_c(uint32_t raddr, double2 v, uint32_t rbar) {
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f64 [%0], {%1, %2}, [%3];"
                 ::"r"(raddr), "d"(v.x), "d"(v.y), "r"(rbar) : "memory");
}

#ifdef FDSNN_PHASE_PROF
__device__ unsigned long long g_pbsc_phase[8];
#define PHASE(k)                                                                  \
    do {                                                                          \
        if (blockIdx.x == 0 && threadIdx.x == 0) {                                \
            const long long now_ = clock64();                                     \
            atomicAdd(&g_pbsc_phase[k], (unsigned long long)(now_ - ph_t0));      \
            ph_t0 = now_;                                                         \
        }                                                                         \
    } while (0)
#else
#define PHASE(k) \
    do {         \
    } while (0)
#endif

constexpr int PBSC_T = 64;  // threads per rotation per CTA (M = 512: 8 points each)

template <int M>
__host__ __device__ constexpr size_t pbsc_group_bytes(int n) {
    return 2 * (size_t)PbsShape<M>::PADM * sizeof(double2)    // exchange buffers
           + 2 * (size_t)M * sizeof(double2)                   // receive buffers (2 exchanges in flight)
           + (size_t)2 * M * sizeof(int32_t)                    // own accumulator polynomial (N words)
           + (((size_t)n * sizeof(uint16_t) + 15) & ~(size_t)15);  // a2N
}
template <int M, int L>
__host__ __device__ constexpr size_t pbsc_smem_bytes(int G, int n) {
    return 128 + (size_t)2 * L * pbs_chunk_bytes<M>() + (size_t)G * pbsc_group_bytes<M>(n);
}

template <int M, int L, int G, bool MODE_RAW, bool TRACK_MARGIN>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(G * PBSC_T, 1)
pbs_blind_rotate_cluster_kernel(const PbsArgs args) {
    static_assert(M == 512 && L == 2, "paired-level CTA-pair kernel: DESK-shaped rings (M = 512, l = 2)");
    constexpr int T = PBSC_T;
    constexpr int N = 2 * M;
    constexpr int PADM = PbsShape<M>::PADM;
    constexpr int S = 2 * L;  // ring stages: this CTA's L chunks of two consecutive steps
    constexpr uint32_t CHUNK = (uint32_t)pbs_chunk_bytes<M>();
    constexpr uint32_t XBYTES = (uint32_t)M * sizeof(double2);
    constexpr int log2_2N = 11;
    const DevParams& prm = args.prm;
    const int n = prm.n;
    const uint32_t qmask = prm.qmask;

    extern __shared__ __align__(128) unsigned char smem_raw[];
    uint64_t* full = reinterpret_cast<uint64_t*>(smem_raw);  // [S] key stage landed
    uint64_t* xfull = full + S;                              // [G][2] partner partial landed
    double2* ring = reinterpret_cast<double2*>(smem_raw + 128);
    const int g = threadIdx.x / T;
    const int t = threadIdx.x % T;
    unsigned char* mine = smem_raw + 128 + S * CHUNK + (size_t)g * pbsc_group_bytes<M>(n);
    double2* buf0 = reinterpret_cast<double2*>(mine);
    double2* buf1 = buf0 + PADM;
    double2* recv = buf1 + PADM;  // [2][M]
    int32_t* acc = reinterpret_cast<int32_t*>(recv + 2 * M);
    uint16_t* a2N = reinterpret_cast<uint16_t*>(acc + N);

    auto a2N_of = [&](int gg) {
        unsigned char* base = smem_raw + 128 + S * CHUNK + (size_t)gg * pbsc_group_bytes<M>(n);
        return reinterpret_cast<const uint16_t*>(base + 2 * PADM * sizeof(double2) + 2 * M * sizeof(double2) +
                                                 (size_t)N * sizeof(int32_t));
    };
    const uint32_t cr = cluster_ctarank();  // polynomial owned by this CTA
    const uint32_t partner = cr ^ 1u;
    const int64_t V = (int64_t)args.nlut * args.count;
    const int64_t v = args.v_base + (int64_t)(blockIdx.x >> 1) * G + g;
    const bool active = v < V;
    const int nsteps_chunks = n * 2 * L;

    if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s) mbar_init(&full[s], 1);
        fence_mbar_init();
    }
    if (t == 0) {
        mbar_init(&xfull[2 * g], 1);
        mbar_init(&xfull[2 * g + 1], 1);
        fence_mbar_init();
        // arm the first two exchanges (partner bytes may land before or after)
        mbar_arrive_expect_tx(&xfull[2 * g], XBYTES);
        mbar_arrive_expect_tx(&xfull[2 * g + 1], XBYTES);
    }
    __syncthreads();
    cluster_sync_all();  // partner's mbarriers exist before any st.async targets them

    // key ring: stage (i & 1) * L + l holds row cr*L + l of step i
    auto chunk_of = [&](int i, int l) { return (size_t)i * 2 * L + cr * L + l; };
    if (threadIdx.x == 0) {
        for (int i = 0; i < 2 && i < n; ++i)
            for (int l = 0; l < L; ++l) {
                const int s = i * L + l;
                mbar_arrive_expect_tx(&full[s], CHUNK);
                bulk_g2s(ring + (size_t)s * 2 * M, args.bsk + chunk_of(i, l) * 2 * M, CHUNK, &full[s]);
            }
    }

    // per-thread transform constants in registers (a lone rotation per SM pair
    // leaves the register file mostly empty)
    TwiddlesInRegs<M> tw;
    load_twiddles<M>(tw.tw, t, args.tables + M);
    double2 twist[8];
    load_twist<M>(twist, t, args.tables);
    const GroupSync gs{1 + g, T};

    // ---------------- setup: modulus switch + this CTA's accumulator poly ---
    if (active) {
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
            for (int j = t; j < N; j += T) {
                if (cr == 0) {
                    acc[j] = 0;
                } else {  // acc_b = X^{-b2N} * v (monomial_rotate_raw, k = -b2N mod 2N)
                    const int src = (j + (int)b2N) & (2 * N - 1);
                    const int32_t val = lut[src & (N - 1)];
                    acc[j] = (int32_t)((uint32_t)(src >= N ? -val : val) & qmask);
                }
            }
        } else {
            const int32_t* a_src = args.acc_io + v * 2 * N + (size_t)cr * N;
            for (int j = t; j < N; j += T) acc[j] = (int32_t)((uint32_t)a_src[j] & qmask);
            const int32_t* k_src = args.a2N_in + v * n;
            for (int i = t; i < n; i += T) a2N[i] = (uint16_t)(k_src[i] & (2 * N - 1));
        }
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
    double err_max = 0.0;
    int xn = 0;  // exchanges done by this rotation (identity steps exchange nothing)
    // partner's receive buffers and mbarriers for this rotation
    const uint32_t r_recv = mapa_shared(recv, partner);
    const uint32_t r_bar = mapa_shared(&xfull[2 * g], partner);
#ifdef FDSNN_PHASE_PROF
    long long ph_t0 = clock64();
#endif

    for (int i = 0; i < n; ++i) {
        const int k = active ? (int)a2N[i] : 0;
        if (k != 0) {
            // ---- 1. digits of (X^k - 1) * ACC_cr at {t + rT, t + rT + M}
            double2 v0[8], v1[8];
#pragma unroll
            for (int r = 0; r < 8; ++r) {
                const int p = t + r * T;
                const int s0 = (p - k) & (2 * N - 1), s1 = (p + M - k) & (2 * N - 1);
                const uint32_t r0 = (s0 >= N) ? (uint32_t)(-acc[s0 - N]) : (uint32_t)acc[s0];
                const uint32_t r1 = (s1 >= N) ? (uint32_t)(-acc[s1 - N]) : (uint32_t)acc[s1];
                const int32_t y0 = (int32_t)((r0 - (uint32_t)acc[p] + halfq) & qmask) + yoff;
                const int32_t y1 = (int32_t)((r1 - (uint32_t)acc[p + M] + halfq) & qmask) + yoff;
                v0[r] = make_double2((double)((y0 & bmask) - halfB1), (double)((y1 & bmask) - halfB1));
                v1[r] = make_double2((double)(((y0 >> bg) & bmask) - halfB1),
                                     (double)(((y1 >> bg) & bmask) - halfB1));
            }
            PHASE(0);
            // ---- 2. both levels' forward transforms (twist fused into pass 0);
            // the key chunks are waited for before the last pass
            const int s0 = (i & 1) * L, s1 = s0 + 1;
            const uint32_t kpar = (uint32_t)((i >> 1) & 1);
            const double2* k0 = ring + (size_t)s0 * 2 * M;
            const double2* k1 = ring + (size_t)s1 * 2 * M;
            auto keys_ready = [&]() {
                mbar_wait(&full[s0], kpar);
                mbar_wait(&full[s1], kpar);
            };
            fft_group2<M, false, TwiddlesInRegs<M>, decltype(keys_ready), true, true>(v0, v1, t, tw, buf0, buf1, gs,
                                                                                    keys_ready, twist);
            PHASE(1);
            // ---- 3. MAC: this CTA's two digit rows into both output polys
            const int xp = xn & 1;
            const uint32_t xpar = (uint32_t)((xn >> 1) & 1);
            double2 O[8];
#pragma unroll
            for (int r = 0; r < 8; ++r) {
                const int f = t + r * T;
                double2 po = make_double2(0.0, 0.0), pp = make_double2(0.0, 0.0);
                cmac(po, v0[r], k0[cr * M + f]);  // own polynomial
                cmac(po, v1[r], k1[cr * M + f]);
                cmac(pp, v0[r], k0[(cr ^ 1) * M + f]);  // the partner's
                cmac(pp, v1[r], k1[(cr ^ 1) * M + f]);
                // ---- 4. the partner's share goes straight to its receive buffer
                st_async_c(r_recv + (uint32_t)((xp * M + f) * sizeof(double2)), pp,
                           r_bar + (uint32_t)(xp * sizeof(uint64_t)));
                O[r] = po;
            }
            PHASE(2);
            // ---- 5. own sum, inverse transform, untwist, round, add
            mbar_wait(&xfull[2 * g + xp], xpar);
            PHASE(3);
#pragma unroll
            for (int r = 0; r < 8; ++r) O[r] = cadd(O[r], recv[xp * M + t + r * T]);
            gs.sync();  // every thread of the rotation has read recv[xp]
            if (t == 0) mbar_arrive_expect_tx(&xfull[2 * g + xp], XBYTES);  // re-arm for exchange xn + 2
            ++xn;
            int ex = 0;
            PHASE(4);
            fft_group<M, true>(O, t, tw, buf0, buf1, ex, gs);
            PHASE(5);
#pragma unroll
            for (int r = 0; r < 8; ++r) {
                const int p = t + r * T;
                const double2 z = cmulc(O[r], twist[r]);
                const long long e0 = round_product(z.x), e1 = round_product(z.y);
                if constexpr (TRACK_MARGIN) {
                    err_max = fmax(err_max, fabs(z.x - (double)e0));
                    err_max = fmax(err_max, fabs(z.y - (double)e1));
                }
                acc[p] = (int32_t)(((uint32_t)acc[p] + (uint32_t)e0) & qmask);
                acc[p + M] = (int32_t)(((uint32_t)acc[p + M] + (uint32_t)e1) & qmask);
            }
        }
        PHASE(6);
        __syncthreads();  // accumulators updated; every reader of this step's key stages done
        if (threadIdx.x == 0 && i + 2 < n) {
            // a stage some rotation consumed this step has landed already;
            // otherwise (all identity steps) wait for the copy before re-arming
            bool consumed = false;
            for (int gg = 0; gg < G; ++gg)
                consumed |= (args.v_base + (int64_t)(blockIdx.x >> 1) * G + gg < V) &&
                            a2N_of(gg)[i] != 0;
            for (int l = 0; l < L; ++l) {
                const int s = (i & 1) * L + l;
                if (!consumed) mbar_wait(&full[s], (uint32_t)((i >> 1) & 1));
                mbar_arrive_expect_tx(&full[s], CHUNK);
                bulk_g2s(ring + (size_t)s * 2 * M, args.bsk + chunk_of(i + 2, l) * 2 * M, CHUNK, &full[s]);
            }
        }
    }
    PHASE(7);
    (void)nsteps_chunks;
    if constexpr (TRACK_MARGIN) {
        if (args.margin && active) atomicMax(args.margin, (unsigned long long)__double_as_longlong(err_max));
    }
    if (active) {
        if constexpr (MODE_RAW) {
            int32_t* a_dst = args.acc_io + v * 2 * N + (size_t)cr * N;
            for (int j = t; j < N; j += T) a_dst[j] = acc[j];
        } else {
            // sample extract (bootstrap.py:291-295): mask (a_0, -a_{N-1}, ..., -a_1) from CTA 0,
            // body acc_b[0] from CTA 1
            uint32_t* out = args.ext_out + v * prm.ext_stride;
            if (cr == 0) {
                for (int j = t; j < N; j += T)
                    out[j] = (j == 0) ? (uint32_t)acc[0] : ((uint32_t)(-acc[N - j]) & qmask);
            } else if (t == 0) {
                out[N] = (uint32_t)acc[0];
            }
        }
    }
    // no CTA leaves while its partner may still be writing into it
    cluster_sync_all();
}

}  // namespace fdsnn
