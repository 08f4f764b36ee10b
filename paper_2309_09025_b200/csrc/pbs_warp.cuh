// pbs_warp.cuh — warp-per-accumulator blind rotation for N = 1024 (M = 512).
//
// Same arithmetic as pbs.cuh (reference bootstrap.py:386-442, bit-exact), a
// different mapping: one warp owns one accumulator and transforms its
// polynomials alone (32 lanes x 16 points, fft16.cuh).  Every FFT exchange is
// warp-local (__syncwarp, no named barriers), so the 8 accumulators of a CTA
// progress independently and hide each other's shared-memory latency; the
// CTA only shares the TMA-fed key ring.
//
// Registers: the 16-point vector, the 16 mask-output frequency accumulators
// (O0) and the component's 32 centred differences.  Tensor memory (per-lane
// columns): pass twiddles + twist (shared by the two warps of a lane
// quadrant), the body-output accumulators O1 and the lane's own accumulator
// coefficients (private per warp).
#pragma once
#include "fft16.cuh"
#include "pbs.cuh"

namespace fdsnn {

constexpr int PBSW_THREADS = 256;  // 8 accumulators per CTA
constexpr int PBSW_S = 4;          // key ring stages
constexpr int PBSW_BUF = 512 + 32; // padded exchange buffer (complex)

__host__ __device__ constexpr size_t pbsw_warp_bytes(int n) {
    return (size_t)PBSW_BUF * sizeof(double2) + 2 * 1024 * sizeof(int32_t) +
           (((size_t)n * sizeof(uint16_t) + 15) & ~(size_t)15);
}
__host__ __device__ constexpr size_t pbsw_smem_bytes(int n) {
    return 128 + (size_t)PBSW_S * 2 * 512 * sizeof(double2) + 8 * pbsw_warp_bytes(n);
}

// TMEM columns per lane
constexpr uint32_t PW_TW1 = 0;      // 16 complex: pass-1 twiddles r = 1..15 (+pad)
constexpr uint32_t PW_TW2 = 64;     // 8 complex: pass-2 twiddles s = 0..7
constexpr uint32_t PW_TWIST = 96;   // 16 complex: twist of points t + 32m
constexpr uint32_t PW_O1 = 160;     // 16 complex per warp (x2 warps per lane)
constexpr uint32_t PW_OWN = 288;    // 64 words per warp: own acc [c][h][m]
constexpr uint32_t PW_COLS = 512;

FDSNN_DEV void tmem_st32d(uint32_t taddr, const double2 (&c)[8]) {
    uint32_t w[32];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        w[4 * i] = (uint32_t)__double2loint(c[i].x);
        w[4 * i + 1] = (uint32_t)__double2hiint(c[i].x);
        w[4 * i + 2] = (uint32_t)__double2loint(c[i].y);
        w[4 * i + 3] = (uint32_t)__double2hiint(c[i].y);
    }
    tmem_st32(taddr, w);
}

template <bool INV>
FDSNN_DEV void w16_fft(double2 (&v)[16], int t, double2* buf, uint32_t lane_base) {
    using namespace w16;
    dft16<INV>(v);
    __syncwarp();
    store0(v, t, buf);
    __syncwarp();
    load1(v, t, buf);
    {
        uint32_t a[32], b[32];
        tmem_ld32_async(lane_base + PW_TW1, a);
        tmem_ld32_async(lane_base + PW_TW1 + 32, b);
        tmem_wait64(a, b);
        double2 w[16];
#pragma unroll
        for (int r = 0; r < 8; ++r) { w[r] = words_c(a, r); w[8 + r] = words_c(b, r); }
        pass1<INV>(v, w);
    }
    __syncwarp();
    store1(v, t, buf);
    __syncwarp();
    load2(v, t, buf);
    {
        uint32_t a[32];
        tmem_ld32_async(lane_base + PW_TW2, a);
        tmem_wait32(a);
        double2 w[8];
#pragma unroll
        for (int s = 0; s < 8; ++s) w[s] = words_c(a, s);
        pass2<INV>(v, w);
    }
}

template <bool TRACK_MARGIN>
__global__ void __launch_bounds__(PBSW_THREADS, 1)
pbs_warp_kernel(const PbsArgs args) {
    using namespace w16;
    constexpr int N = 1024;
    constexpr uint32_t CHUNK = 2 * 512 * sizeof(double2);
    const DevParams& prm = args.prm;
    const int n = prm.n;
    const int L = prm.L;
    const uint32_t qmask = prm.qmask;

    extern __shared__ __align__(128) unsigned char smem_raw[];
    uint64_t* full = reinterpret_cast<uint64_t*>(smem_raw);
    uint64_t* empty = full + 4;
    uint32_t* tmem_base_slot = reinterpret_cast<uint32_t*>(smem_raw + 120);
    double2* ring = reinterpret_cast<double2*>(smem_raw + 128);
    const int warp = threadIdx.x / 32;
    const int t = threadIdx.x % 32;
    unsigned char* mine = smem_raw + 128 + PBSW_S * CHUNK + warp * pbsw_warp_bytes(n);
    double2* buf = reinterpret_cast<double2*>(mine);
    int32_t* acc = reinterpret_cast<int32_t*>(buf + PBSW_BUF);  // [2][N]
    uint16_t* a2N = reinterpret_cast<uint16_t*>(acc + 2 * N);

    const int64_t V = (int64_t)args.nlut * args.count;
    const int64_t v0 = (int64_t)blockIdx.x * 8;
    const int nact = (int)((V - v0) < 8 ? (V - v0) : 8);
    const bool active = warp < nact;
    const int nchunks = n * 2 * L;
    const bool producer = threadIdx.x == 0;
    if (producer) {
        for (int s = 0; s < PBSW_S; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], nact * 32);
        }
        fence_mbar_init();
    }
    if (warp == 0) tmem_alloc(tmem_base_slot, PW_COLS);
    tmem_fence_before();
    __syncthreads();
    tmem_fence_after();
    const uint32_t tbase = *tmem_base_slot;
    const uint32_t lane_base = tbase + ((uint32_t)((warp % 4) * 32) << 16);

    // per-lane constants (warps 0-3 cover the 4 lane quadrants; t = lane)
    if (warp < 4 && active) {
        double2 c[8];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                const int r = 1 + 8 * h + i;  // pass-1 twiddle w256^{(t%16) r}
                double s, co;
                sincospi((double)((t % 16) * (r < 16 ? r : 15)) / 128.0, &s, &co);
                c[i] = make_double2(co, s);
            }
            tmem_st32d(lane_base + PW_TW1 + 32 * h, c);
        }
#pragma unroll
        for (int s8 = 0; s8 < 8; ++s8) {  // pass-2 twiddle w512^{t + 32 s}
            double s, co;
            sincospi((double)(t + 32 * s8) / 256.0, &s, &co);
            c[s8] = make_double2(co, s);
        }
        tmem_st32d(lane_base + PW_TW2, c);
#pragma unroll
        for (int h = 0; h < 2; ++h) {
#pragma unroll
            for (int i = 0; i < 8; ++i) {  // twist e^{i pi (t + 32 m)/N}
                const int m = 8 * h + i;
                double s, co;
                sincospi((double)(t + 32 * m) / 1024.0, &s, &co);
                c[i] = make_double2(co, s);
            }
            tmem_st32d(lane_base + PW_TWIST + 32 * h, c);
        }
        tmem_wait_st();
    }
    tmem_fence_before();
    __syncthreads();
    tmem_fence_after();

    if (producer) {
        for (int s = 0; s < PBSW_S && s < nchunks; ++s) {
            mbar_arrive_expect_tx(&full[s], CHUNK);
            bulk_g2s(ring + (size_t)s * 1024, args.bsk + (size_t)s * 1024, CHUNK, &full[s]);
        }
    }
    auto release = [&](int c) {
        const int s = c & (PBSW_S - 1);
        mbar_arrive(&empty[s]);
        if (producer && c + PBSW_S < nchunks) {
            mbar_wait(&empty[s], (uint32_t)((c / PBSW_S) & 1));
            mbar_arrive_expect_tx(&full[s], CHUNK);
            bulk_g2s(ring + (size_t)s * 1024, args.bsk + (size_t)(c + PBSW_S) * 1024, CHUNK, &full[s]);
        }
    };

    if (active) {
        const int64_t v = v0 + warp;
        const uint32_t o1_col = lane_base + PW_O1 + 64 * (uint32_t)(warp / 4);
        const uint32_t own_col = lane_base + PW_OWN + 64 * (uint32_t)(warp / 4);
        // ---- modulus switch + accumulator init (bootstrap.py:524-529)
        {
            const int u = (int)(v / args.count);
            const int64_t row = v - (int64_t)u * args.count;
            const uint32_t* a_in = args.in + row * prm.stride;
            const uint32_t* a_in2 = args.in2 ? args.in2 + row * prm.stride : nullptr;
            for (int i = t; i < n; i += 32) {
                uint32_t a = a_in[i];
                if (a_in2) a += a_in2[i];
                a2N[i] = (uint16_t)rescale_q_to_2N(a, prm.log2q, 11);
            }
            uint32_t b = a_in[n] + args.in_boff[u];
            if (a_in2) b += a_in2[n];
            const uint32_t b2N = (rescale_q_to_2N(b, prm.log2q, 11) + prm.half_slot) & (2 * N - 1);
            const int32_t* lut = args.lut[u];
            uint32_t own[32], own2[32];
#pragma unroll
            for (int hm = 0; hm < 32; ++hm) {  // coefficient j = t + 32*hm (hm = 16h + m)
                const int j = t + 32 * hm;
                acc[j] = 0;
                own[hm] = 0u;
                const int src = (j + (int)b2N) & (2 * N - 1);
                const int32_t val = lut[src & (N - 1)];
                const uint32_t bv = (uint32_t)(src >= N ? -val : val) & qmask;
                acc[N + j] = (int32_t)bv;
                own2[hm] = bv;
            }
            tmem_st32(own_col, own);
            tmem_st32(own_col + 32, own2);
            tmem_wait_st();
        }
        __syncwarp();

        const int bg = prm.bg_log;
        const int32_t halfB1 = (1 << (bg - 1)) - 1;
        const int32_t bmask = (1 << bg) - 1;
        double err_max = 0.0;
        int c = 0;
        for (int i = 0; i < n; ++i) {
            const int k = a2N[i];
            if (k == 0) {
                for (int d = 0; d < 2 * L; ++d, ++c) {
                    mbar_wait(&full[c & (PBSW_S - 1)], (uint32_t)((c / PBSW_S) & 1));
                    release(c);
                }
                continue;
            }
            double2 O0[16];
#pragma unroll
            for (int m = 0; m < 16; ++m) O0[m] = make_double2(0.0, 0.0);
            bool first = true;
            for (int cc = 0; cc < 2; ++cc) {
                const int32_t* a = acc + cc * N;
                int32_t xs[32];  // [h*16 + m] centred (X^k - 1)*ACC at t + 32m + 512h
                {
                    uint32_t ow[32];
                    tmem_ld32_async(own_col + 32 * cc, ow);
                    uint32_t rv[32];
#pragma unroll
                    for (int hm = 0; hm < 32; ++hm) {
                        const int jj = t + 32 * hm;
                        const int s = (jj - k) & (2 * N - 1);
                        rv[hm] = (s >= N) ? (uint32_t)(-a[s - N]) : (uint32_t)a[s];
                    }
                    tmem_wait32(ow);
#pragma unroll
                    for (int hm = 0; hm < 32; ++hm) xs[hm] = center_q((rv[hm] - ow[hm]) & qmask, prm.log2q);
                }
                for (int lvl = 0; lvl < L; ++lvl, ++c) {
                    double2 vv[16];
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        uint32_t tw[32];
                        tmem_ld32_async(lane_base + PW_TWIST + 32 * h, tw);
                        int32_t d1[8], d2[8];
#pragma unroll
                        for (int i8 = 0; i8 < 8; ++i8) {
                            const int m = 8 * h + i8;
                            d1[i8] = ((xs[m] + halfB1) & bmask) - halfB1;
                            d2[i8] = ((xs[16 + m] + halfB1) & bmask) - halfB1;
                            xs[m] = (xs[m] - d1[i8]) >> bg;
                            xs[16 + m] = (xs[16 + m] - d2[i8]) >> bg;
                        }
                        tmem_wait32(tw);
#pragma unroll
                        for (int i8 = 0; i8 < 8; ++i8)
                            vv[8 * h + i8] = cmul(make_double2((double)d1[i8], (double)d2[i8]), words_c(tw, i8));
                    }
                    w16_fft<false>(vv, t, buf, lane_base);
                    const int s = c & (PBSW_S - 1);
                    mbar_wait(&full[s], (uint32_t)((c / PBSW_S) & 1));
                    const double2* kd = ring + (size_t)s * 1024;
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        uint32_t o1w[32];
                        if (!first) tmem_ld32_async(o1_col + 32 * h, o1w);
                        double2 o1[8];
#pragma unroll
                        for (int i8 = 0; i8 < 8; ++i8) {
                            const int m = 8 * h + i8;
                            const double2 d = vv[reg_of(m)];
                            cmac(O0[m], d, kd[t + 32 * m]);
                            o1[i8] = cmul(d, kd[512 + t + 32 * m]);
                        }
                        if (!first) {
                            tmem_wait32(o1w);
#pragma unroll
                            for (int i8 = 0; i8 < 8; ++i8) o1[i8] = cadd(o1[i8], words_c(o1w, i8));
                        }
                        tmem_st32d(o1_col + 32 * h, o1);
                    }
                    tmem_wait_st();
                    first = false;
                    release(c);
                }
            }
            // ---- inverse transforms, untwist, round, accumulate (bootstrap.py:425-442)
#pragma unroll
            for (int o = 0; o < 2; ++o) {
                double2 y[16];
                if (o == 0) {
#pragma unroll
                    for (int m = 0; m < 16; ++m) y[m] = O0[m];
                } else {
                    uint32_t a0[32], a1[32];
                    tmem_ld32_async(o1_col, a0);
                    tmem_ld32_async(o1_col + 32, a1);
                    tmem_wait64(a0, a1);
#pragma unroll
                    for (int i8 = 0; i8 < 8; ++i8) { y[i8] = words_c(a0, i8); y[8 + i8] = words_c(a1, i8); }
                }
                w16_fft<true>(y, t, buf, lane_base);
                uint32_t own[32];
                tmem_ld32_async(own_col + 32 * o, own);
                uint32_t tw0[32], tw1[32];
                tmem_ld32_async(lane_base + PW_TWIST, tw0);
                tmem_ld32_async(lane_base + PW_TWIST + 32, tw1);
                tmem_wait64(tw0, tw1);
                tmem_touch32(own);
#pragma unroll
                for (int m = 0; m < 16; ++m) {
                    const double2 tr = m < 8 ? words_c(tw0, m) : words_c(tw1, m - 8);
                    const double2 z = cmulc(y[reg_of(m)], tr);
                    const long long r0 = round_product(z.x), r1 = round_product(z.y);
                    if constexpr (TRACK_MARGIN) {
                        err_max = fmax(err_max, fabs(z.x - (double)r0));
                        err_max = fmax(err_max, fabs(z.y - (double)r1));
                    }
                    own[m] = (own[m] + (uint32_t)r0) & qmask;            // coefficient t + 32m
                    own[16 + m] = (own[16 + m] + (uint32_t)r1) & qmask;  // coefficient t + 32m + 512
                    acc[o * N + t + 32 * m] = (int32_t)own[m];
                    acc[o * N + t + 32 * m + 512] = (int32_t)own[16 + m];
                }
                tmem_st32(own_col + 32 * o, own);
            }
            tmem_wait_st();
            __syncwarp();
        }
        if constexpr (TRACK_MARGIN) {
            if (args.margin) atomicMax(args.margin, (unsigned long long)__double_as_longlong(err_max));
        }
        // sample extract (bootstrap.py:484-488)
        uint32_t* out = args.ext_out + v * prm.ext_stride;
        for (int j = t; j < N; j += 32) {
            const uint32_t aa = (j == 0) ? (uint32_t)acc[0] : ((uint32_t)(-acc[N - j]) & qmask);
            out[j] = aa;
        }
        if (t == 0) out[N] = (uint32_t)acc[N];
    }
    tmem_fence_before();
    __syncthreads();
    if (warp == 0) {
        tmem_fence_after();
        tmem_dealloc(tbase, PW_COLS);
    }
}

}  // namespace fdsnn
