// fft.cuh — register/shared-memory Stockham FFT for the folded negacyclic
// transform of ring.NegacyclicTransform (reference ring.py:103-137).
//
// The reference evaluates a real length-N polynomial by folding it into
// M = N/2 complex points c_j = (a_j + i a_{j+M}) * e^{i pi j / N} followed by a
// length-M DFT with the e^{+2 pi i jk/M} kernel (scipy ifft, norm="forward"),
// and inverts with the e^{-2 pi i} DFT, /M, untwist and unfold.
//
// B200 design: one polynomial is transformed by T = M/8 threads that each own
// the 8 points {t + r*T : r < 8}.  A Stockham autosort formulation (natural
// order in, natural order out) is used with radix-8 first and last passes, so
//   * the first pass reads exactly the points the thread computed itself
//     (digits of accumulator coefficients t + rT and t + rT + M),
//   * the last forward pass leaves frequencies {t + rT} in registers, which is
//     also the first inverse pass's input set -> the Fourier-domain MAC against
//     the bootstrapping key and the hand-off to the inverse transform need no
//     data exchange at all,
//   * the last inverse pass leaves coefficients {t + rT, t + rT + M} in
//     registers, i.e. exactly what the thread adds back into the accumulator.
// Only the interior pass boundaries exchange data through shared memory
// (padded a + a/8 to keep 16-byte accesses bank-conflict free).
#pragma once
#include "common.cuh"

namespace fdsnn {

// multiply by s*i where s = +1 (forward, e^{+}) or -1 (inverse)
template <bool INV>
FDSNN_DEV double2 mul_si(double2 a) {
    return INV ? make_double2(a.y, -a.x) : make_double2(-a.y, a.x);
}

template <bool INV>
FDSNN_DEV void dft2(double2& a, double2& b) {
    double2 t = a;
    a = cadd(t, b);
    b = csub(t, b);
}

// 4-point DFT with kernel e^{s 2 pi i/4}, natural order in/out.
template <bool INV>
FDSNN_DEV void dft4(double2& y0, double2& y1, double2& y2, double2& y3) {
    double2 c0 = cadd(y0, y2), c1 = csub(y0, y2);
    double2 c2 = cadd(y1, y3), c3 = mul_si<INV>(csub(y1, y3));
    y0 = cadd(c0, c2);
    y2 = csub(c0, c2);
    y1 = cadd(c1, c3);
    y3 = csub(c1, c3);
}

// Second half of the 8-point DFT from the first-stage sums a_r = x_r + x_{r+4}
// and differences b_r = x_r - x_{r+4}.
template <bool INV>
FDSNN_DEV void dft8_tail(double2* v, double2 a0, double2 a1, double2 a2, double2 a3,
                         double2 b0, double2 b1, double2 b2, double2 b3) {
    const double h = 0.70710678118654752440;  // sqrt(2)/2
    // odd outputs = DFT4(b0, b1 e^{s i pi/4}, b2 (s i), b3 e^{s 3i pi/4}).  The
    // sqrt(2)/2 of the two diagonal twiddles is folded into the final FMAs:
    // u1 = (1 + s i) b1, u3 = (-1 + s i) b3 cost additions only.
    const double2 u1 = INV ? make_double2(b1.x + b1.y, b1.y - b1.x)
                           : make_double2(b1.x - b1.y, b1.y + b1.x);
    const double2 u3 = INV ? make_double2(b3.y - b3.x, -(b3.y + b3.x))
                           : make_double2(-(b3.x + b3.y), b3.x - b3.y);
    b2 = mul_si<INV>(b2);
    dft4<INV>(a0, a1, a2, a3);
    v[0] = a0; v[2] = a1; v[4] = a2; v[6] = a3;
    const double2 c0 = cadd(b0, b2), c1 = csub(b0, b2);
    const double2 e = cadd(u1, u3);
    const double2 f = mul_si<INV>(csub(u1, u3));
    v[1] = make_double2(fma(h, e.x, c0.x), fma(h, e.y, c0.y));
    v[5] = make_double2(fma(-h, e.x, c0.x), fma(-h, e.y, c0.y));
    v[3] = make_double2(fma(h, f.x, c1.x), fma(h, f.y, c1.y));
    v[7] = make_double2(fma(-h, f.x, c1.x), fma(-h, f.y, c1.y));
}

// 8-point DFT with kernel e^{s 2 pi i/8}, natural order in/out.
template <bool INV>
FDSNN_DEV void dft8(double2* v) {
    dft8_tail<INV>(v, cadd(v[0], v[4]), cadd(v[1], v[5]), cadd(v[2], v[6]), cadd(v[3], v[7]),
                   csub(v[0], v[4]), csub(v[1], v[5]), csub(v[2], v[6]), csub(v[3], v[7]));
}

#ifndef FDSNN_FUSED_TW
#define FDSNN_FUSED_TW 1
#endif
// c + w v  (CONJ: c + conj(w) v), four DFMA
template <bool CONJ>
FDSNN_DEV double2 cfma(double2 c, double2 w, double2 v) {
    if constexpr (CONJ)
        return make_double2(fma(w.y, v.y, fma(w.x, v.x, c.x)), fma(-w.y, v.x, fma(w.x, v.y, c.y)));
    else
        return make_double2(fma(-w.y, v.y, fma(w.x, v.x, c.x)), fma(w.y, v.x, fma(w.x, v.y, c.y)));
}
// 2t - a, two DFMA
FDSNN_DEV double2 ctwo_minus(double2 t, double2 a) {
    return make_double2(fma(2.0, t.x, -a.x), fma(2.0, t.y, -a.y));
}

// 8-point DFT of the input-twiddled points x_r = w_r v_r with the twiddle
// products fused into the first butterfly stage:  a_r = t_r + w_{r+4} v_{r+4}
// (t_r = w_r v_r; four DFMA) and b_r = 2 t_r - a_r (two DFMA) instead of two
// complex products and two complex additions -- 8 fewer FP64 instructions
// per radix-8 pass.  W0 = false: v_0 is not twiddled (interior passes,
// w[r-1] = w_r); W0 = true: all eight are (the forward twist, w[r] = w_r).
template <bool INV, bool W0>
FDSNN_DEV void dft8_tw(double2* v, const double2* w) {
    auto wr = [&](int r) { return W0 ? w[r] : w[r - 1]; };
    auto tr = [&](int r) {
        if (r == 0 && !W0) return v[0];
        return INV ? cmulc(v[r], wr(r)) : cmul(v[r], wr(r));
    };
    const double2 t0 = tr(0), t1 = tr(1), t2 = tr(2), t3 = tr(3);
    const double2 a0 = cfma<INV>(t0, wr(4), v[4]), a1 = cfma<INV>(t1, wr(5), v[5]);
    const double2 a2 = cfma<INV>(t2, wr(6), v[6]), a3 = cfma<INV>(t3, wr(7), v[7]);
    dft8_tail<INV>(v, a0, a1, a2, a3, ctwo_minus(t0, a0), ctwo_minus(t1, a1), ctwo_minus(t2, a2),
                   ctwo_minus(t3, a3));
}

template <int R, bool INV>
FDSNN_DEV void dftR(double2* v) {
    if constexpr (R == 8) {
        dft8<INV>(v);
    } else if constexpr (R == 4) {
        dft4<INV>(v[0], v[1], v[2], v[3]);
    } else {
        dft2<INV>(v[0], v[1]);
    }
}

FDSNN_DEV int pad_idx(int a) { return a + (a >> 3); }

// Pass schedule per transform size (product of radices = M; first and last 8).
template <int M> struct Schedule;
template <> struct Schedule<256> { static constexpr int P = 3; static constexpr int R[4] = {8, 4, 8, 0}; };
template <> struct Schedule<512> { static constexpr int P = 3; static constexpr int R[4] = {8, 8, 8, 0}; };
template <> struct Schedule<1024> { static constexpr int P = 4; static constexpr int R[4] = {8, 4, 4, 8}; };

template <int M, int PASS>
struct PassInfo {
    static constexpr int R = Schedule<M>::R[PASS];
    static constexpr int NS = PASS == 0 ? 1 : PassInfo<M, PASS - 1>::NS * PassInfo<M, PASS - 1>::R;
};
template <int M>
struct PassInfo<M, -1> { static constexpr int R = 1; static constexpr int NS = 1; };

// Group-local synchronisation handle for the T threads transforming one poly.
struct GroupSync {
    int bar_id;
    int nthreads;
    FDSNN_DEV void sync() const { named_bar(bar_id, nthreads); }
};

// Per-thread twiddle factors: for pass p >= 1 the thread's groups all share
// jm = t mod NS_p (T is a multiple of NS_p for every interior pass), so each
// pass needs R_p - 1 constants e^{2 pi i r jm/(NS_p R_p)}.  They are loaded
// once per kernel into registers (no shared-memory traffic, no bank conflicts).
template <int M>
struct Twiddles {
    double2 w[4][7];
};

// Host/device table layout: for pass p (1..P-1), entries [r-1][jm], jm < NS_p.
template <int M>
__host__ __device__ constexpr int twiddle_offset(int pass) {
    int off = 0;
    for (int p = 1; p < pass; ++p) {
        int ns = 1;
        for (int k = 0; k < p; ++k) ns *= Schedule<M>::R[k];
        off += (Schedule<M>::R[p] - 1) * ns;
    }
    return off;
}
template <int M>
__host__ __device__ constexpr int twiddle_table_size() { return twiddle_offset<M>(Schedule<M>::P); }

template <int M, int PASS>
FDSNN_DEV void load_twiddles_pass(Twiddles<M>& tw, int t, const double2* __restrict__ tab) {
    if constexpr (PASS < Schedule<M>::P) {
        constexpr int R = PassInfo<M, PASS>::R;
        constexpr int NS = PassInfo<M, PASS>::NS;
        const double2* base = tab + twiddle_offset<M>(PASS);
#pragma unroll
        for (int r = 1; r < R; ++r) tw.w[PASS][r - 1] = __ldg(base + (r - 1) * NS + (t % NS));
        load_twiddles_pass<M, PASS + 1>(tw, t, tab);
    }
}
template <int M>
FDSNN_DEV void load_twiddles(Twiddles<M>& tw, int t, const double2* __restrict__ tab) {
    load_twiddles_pass<M, 1>(tw, t, tab);
}


// Twiddle providers.  issue<PASS>(raw) starts fetching the R-1 factors
// e^{2 pi i r jm/(NS R)} of this thread's interior pass PASS; finish<PASS>
// (raw, w) completes the fetch into w[r-1].  The FFT issues the fetch before
// the pass's exchange stores and completes it before the barrier, so the
// barrier wait hides its latency and the exchange loads issue right after it.
template <int M>
struct TwiddlesInRegs {
    Twiddles<M> tw;
    template <int PASS>
    FDSNN_DEV void issue(uint32_t (&)[32]) const {}
    template <int PASS>
    FDSNN_DEV void finish(uint32_t (&)[32], double2 (&w)[8]) const {
#pragma unroll
        for (int r = 0; r < 7; ++r) w[r] = tw.w[PASS][r];
    }
};

// Tensor-memory resident twiddles: pass p occupies columns (p-1)*32..+31 of
// the thread's TMEM lane (8 complex, entries r-1 = 0..6).
template <int M>
struct TwiddlesInTmem {
    uint32_t base;
    template <int PASS>
    FDSNN_DEV void issue(uint32_t (&raw)[32]) const { tmem_ld32_async(base + (PASS - 1) * 32, raw); }
    template <int PASS>
    FDSNN_DEV void finish(uint32_t (&raw)[32], double2 (&w)[8]) const {
        tmem_wait32(raw);
#pragma unroll
        for (int r = 0; r < 7; ++r) w[r] = words_c(raw, r);
    }
};

// Twiddles read from the (L1-resident) global table: issue<PASS> starts the
// loads before the exchange stores, finish<PASS> consumes them after the
// barrier, so their latency hides behind the exchange; no registers are held
// between passes.
template <int M>
struct TwiddlesFromGlobal {
    const double2* tab;  // interior-pass table (twiddle_offset layout)
    int t;
    template <int PASS>
    FDSNN_DEV void issue(uint32_t (&raw)[32]) const {
        constexpr int R = PassInfo<M, PASS>::R;
        constexpr int ns = PassInfo<M, PASS>::NS;
        const double2* base = tab + twiddle_offset<M>(PASS);
#pragma unroll
        for (int r = 1; r < R; ++r) {
            const double2 w = __ldg(base + (r - 1) * ns + (t % ns));
            raw[4 * (r - 1)] = (uint32_t)__double2loint(w.x);
            raw[4 * (r - 1) + 1] = (uint32_t)__double2hiint(w.x);
            raw[4 * (r - 1) + 2] = (uint32_t)__double2loint(w.y);
            raw[4 * (r - 1) + 3] = (uint32_t)__double2hiint(w.y);
        }
    }
    template <int PASS>
    FDSNN_DEV void finish(uint32_t (&raw)[32], double2 (&w)[8]) const {
#pragma unroll
        for (int r = 0; r < 7; ++r) w[r] = words_c(raw, r);
    }
};

// One Stockham pass.  v holds 8/R independent R-point groups.
template <int M, int PASS, bool INV>
FDSNN_DEV void pass_body(double2 (&v)[8], const double2 (&w)[8]) {
    constexpr int R = PassInfo<M, PASS>::R;
    constexpr int NS = PassInfo<M, PASS>::NS;
    if constexpr (FDSNN_FUSED_TW && R == 8 && NS > 1) {
        dft8_tw<INV, false>(v, w);
        return;
    }
#pragma unroll
    for (int s = 0; s < 8 / R; ++s) {
        if constexpr (NS > 1) {
#pragma unroll
            for (int r = 1; r < R; ++r)
                v[s * R + r] = INV ? cmulc(v[s * R + r], w[r - 1]) : cmul(v[s * R + r], w[r - 1]);
        }
        dftR<R, INV>(&v[s * R]);
    }
}

template <int M, int PASS>
FDSNN_DEV void pass_store(const double2 (&v)[8], int t, double2* __restrict__ buf) {
    constexpr int T = M / 8;
    constexpr int R = PassInfo<M, PASS>::R;
    constexpr int NS = PassInfo<M, PASS>::NS;
#pragma unroll
    for (int s = 0; s < 8 / R; ++s) {
        const int j = t + T * s;
        const int idxD = (j / NS) * NS * R + (j % NS);
#pragma unroll
        for (int r = 0; r < R; ++r) buf[pad_idx(idxD + r * NS)] = v[s * R + r];
    }
}

template <int M, int PASS>
FDSNN_DEV void pass_load(double2 (&v)[8], int t, const double2* __restrict__ buf) {
    constexpr int T = M / 8;
    constexpr int R = PassInfo<M, PASS>::R;
#pragma unroll
    for (int s = 0; s < 8 / R; ++s) {
        const int j = t + T * s;
#pragma unroll
        for (int r = 0; r < R; ++r) v[s * R + r] = buf[pad_idx(j + r * (M / R))];
    }
}

struct NoHook {
    FDSNN_DEV void operator()() const {}
};

// Full transform: v (points t + rT) -> v (frequencies t + rT).
// `ex` is the running exchange parity (alternates the two exchange buffers so
// that a single barrier per exchange is race free across consecutive FFTs).
// `pre_last` runs after the last exchange and twiddle fetch, before the last
// pass's arithmetic
// (used to start the key fetch of the following MAC).
template <int M, bool INV, class TW, class HOOK = NoHook, bool FT0 = false>
FDSNN_DEV void fft_stockham(double2 (&v)[8], int t, const TW& tw,
                            double2* __restrict__ buf0, double2* __restrict__ buf1,
                            int& ex, const GroupSync& gs, const HOOK& pre_last = HOOK(),
                            const double2* tw0 = nullptr) {
    constexpr int P = Schedule<M>::P;
    static_assert(!FT0 || Schedule<M>::R[0] == 8, "fused twist needs a radix-8 first pass");
    if constexpr (FT0) {
        dft8_tw<INV, true>(v, tw0);
    } else {
        double2 w[8];
        pass_body<M, 0, INV>(v, w);
    }
#define FDSNN_FFT_STEP(PS)                                        \
    if constexpr (PS < P) {                                       \
        uint32_t raw[32];                                         \
        tw.template issue<PS>(raw);                               \
        double2* b = ex ? buf1 : buf0;                            \
        pass_store<M, PS - 1>(v, t, b);                           \
        double2 w[8];                                             \
        tw.template finish<PS>(raw, w);                           \
        gs.sync();                                                \
        pass_load<M, PS>(v, t, b);                                \
        ex ^= 1;                                                  \
        if constexpr (PS == P - 1) pre_last();                    \
        pass_body<M, PS, INV>(v, w);                              \
    }
    FDSNN_FFT_STEP(1)
    FDSNN_FFT_STEP(2)
    FDSNN_FFT_STEP(3)
#undef FDSNN_FFT_STEP
}

// Two independent transforms interleaved (double ILP, shared barriers): v0
// exchanges through buf0, v1 through buf1.  Each exchange is fenced on both
// sides (write-after-read on the buffers), so it is safe whatever the buffers
// were last used for.
template <int M, bool INV, class TW, class HOOK = NoHook>
FDSNN_DEV void fft_stockham2(double2 (&v0)[8], double2 (&v1)[8], int t, const TW& tw,
                             double2* __restrict__ buf0, double2* __restrict__ buf1,
                             const GroupSync& gs, const HOOK& pre_last = HOOK()) {
    constexpr int P = Schedule<M>::P;
    {
        double2 w[8];
        pass_body<M, 0, INV>(v0, w);
        pass_body<M, 0, INV>(v1, w);
    }
#define FDSNN_FFT2_STEP(PS)                                       \
    if constexpr (PS < P) {                                       \
        uint32_t raw[32];                                         \
        tw.template issue<PS>(raw);                               \
        gs.sync();                                                \
        pass_store<M, PS - 1>(v0, t, buf0);                       \
        pass_store<M, PS - 1>(v1, t, buf1);                       \
        double2 w[8];                                             \
        tw.template finish<PS>(raw, w);                           \
        gs.sync();                                                \
        pass_load<M, PS>(v0, t, buf0);                            \
        pass_load<M, PS>(v1, t, buf1);                            \
        if constexpr (PS == P - 1) pre_last();                    \
        pass_body<M, PS, INV>(v0, w);                             \
        pass_body<M, PS, INV>(v1, w);                             \
    }
    FDSNN_FFT2_STEP(1)
    FDSNN_FFT2_STEP(2)
    FDSNN_FFT2_STEP(3)
#undef FDSNN_FFT2_STEP
}

// Software-pipelined pair: v1 runs half an exchange behind v0, so each batch
// of exchange loads is followed by the other transform's butterflies (which
// hide the load latency) instead of by its own consumer.  Each barrier is the
// read-after-write fence of one buffer and the write-after-read fence of the
// other: 2P-1 barriers per pair against 2(P-1) for fft_stockham2.
// FT0: the inputs still need the per-point factors tw0[r] (the forward
// twist); they are fused into the first pass (dft8_tw).
template <int M, bool INV, bool FT0>
FDSNN_DEV void first_pass(double2 (&v)[8], const double2* tw0) {
    if constexpr (FT0) {
        dft8_tw<INV, true>(v, tw0);
    } else {
        double2 w[8];
        pass_body<M, 0, INV>(v, w);
    }
}

template <int M, bool INV, class TW, class HOOK = NoHook, bool ENTRY_SYNC = true, bool FT0 = false>
FDSNN_DEV void fft_stockham2p(double2 (&v0)[8], double2 (&v1)[8], int t, const TW& tw,
                              double2* __restrict__ buf0, double2* __restrict__ buf1,
                              const GroupSync& gs, const HOOK& pre_last = HOOK(),
                              const double2* tw0 = nullptr) {
    constexpr int P = Schedule<M>::P;
    static_assert(P == 3, "pipelined pair written for three passes");
    static_assert(!FT0 || Schedule<M>::R[0] == 8, "fused twist needs a radix-8 first pass");
    {
        first_pass<M, INV, FT0>(v0, tw0);
        if constexpr (ENTRY_SYNC) gs.sync();  // previous readers of both buffers are done
        pass_store<M, 0>(v0, t, buf0);
        gs.sync();
        pass_load<M, 1>(v0, t, buf0);
        first_pass<M, INV, FT0>(v1, tw0);
    }
    {
        uint32_t raw[32];
        tw.template issue<1>(raw);
        pass_store<M, 0>(v1, t, buf1);
        double2 w[8];
        tw.template finish<1>(raw, w);
        gs.sync();
        pass_load<M, 1>(v1, t, buf1);
        pass_body<M, 1, INV>(v0, w);
        pass_store<M, 1>(v0, t, buf0);
        gs.sync();
        pass_load<M, 2>(v0, t, buf0);
        pass_body<M, 1, INV>(v1, w);
    }
    {
        uint32_t raw[32];
        tw.template issue<2>(raw);
        pass_store<M, 1>(v1, t, buf1);
        double2 w[8];
        tw.template finish<2>(raw, w);
        gs.sync();
        pass_load<M, 2>(v1, t, buf1);
        pre_last();
        pass_body<M, 2, INV>(v0, w);
        pass_body<M, 2, INV>(v1, w);
    }
}

#ifndef FDSNN_PIPE2
#define FDSNN_PIPE2 1
#endif

// ---------------------------------------------------------------------------
// M = 1024 as a parity split (C4, N = 2048): thread t = 2t' + p holds the
// points {t + 128 r} = {2(t' + 64 r) + p}, i.e. the 512-point subsequence of
// parity p at the positions the 64-thread M = 512 transform expects.  The two
// 512-point transforms (2 shared-memory exchanges each, run side by side by
// the even and odd lanes, each parity in its own half of the exchange
// buffers) are joined by one radix-2 step between lanes 2t' and 2t'+1 through
// warp shuffles:  X[k] = E[k] + w^k O[k],  X[k + 512] = E[k] - w^k O[k]
// (w = e^{+2 pi i/1024}; the inverse runs the mirrored steps with conj(w)),
// balanced so each lane ships 4 values (r2_join below).
// Against the 4-pass Stockham schedule (8,4,4,8) this trades one
// shared-memory exchange and its barrier for 16 shuffles per thread.
// Output layout: lane (t', p), register r < 4 / r + 4 holds (a unit multiple
// of) X[k] / X[k + 512], k = t' + 64 (r + 4p); the Fourier key is produced by
// the same transform (and scaled back to the true basis), so the MAC (thread
// t reads key index t + 128 r) pairs matching frequencies.
constexpr int FFT1024_HALF = 580;  // odd-parity region offset: 576 (padded 512 points) + 4 slots

template <>
struct TwiddlesInRegs<1024> {
    TwiddlesInRegs<512> half;
    double2 r2[8];  // w^{t' + 64 r}
    FDSNN_DEV const TwiddlesInRegs<512>& sub() const { return half; }
    FDSNN_DEV void issue_r2(uint32_t (&)[32]) const {}
    FDSNN_DEV void finish_r2(uint32_t (&)[32], double2 (&w)[8]) const {
#pragma unroll
        for (int r = 0; r < 8; ++r) w[r] = r2[r];
    }
};

// TMEM: the 512-point pass twiddles of t' at columns 0-63, w^{t'+64r} at 64-95
template <>
struct TwiddlesInTmem<1024> {
    uint32_t base;
    FDSNN_DEV TwiddlesInTmem<512> sub() const { return TwiddlesInTmem<512>{base}; }
    FDSNN_DEV void issue_r2(uint32_t (&raw)[32]) const { tmem_ld32_async(base + 64, raw); }
    FDSNN_DEV void finish_r2(uint32_t (&raw)[32], double2 (&w)[8]) const {
        tmem_wait32(raw);
#pragma unroll
        for (int r = 0; r < 8; ++r) w[r] = words_c(raw, r);
    }
};

FDSNN_DEV double2 shfl_xor1(double2 a) {
    return make_double2(__shfl_xor_sync(0xffffffffu, a.x, 1), __shfl_xor_sync(0xffffffffu, a.y, 1));
}

// Balanced, select-free radix-2 join (the fft16.cuh construction): the even
// lane finishes k = t' + 64 r for r < 4, the odd lane r >= 4, each sending 4
// of its 8 values.  The odd lane's 512-point inputs carry (-1)^{t'} (folded
// into the twist table: points j = 3 mod 4), which rotates its outputs by
// 4 registers, so every lane keeps registers 0-3 and ships 4-7; then
// out0 = P + z Q, out1 = P - z Q with z = w^k (even lane, k = t' + 64 r) or
// w^{-k} (odd lane, k = t' + 64 (r + 4)).  The odd lane thus holds
// w^{-k} X[k] and -w^{-k} X[k + 512]: the inverse's first step consumes
// exactly that scaling, and the Fourier key (bsk_forward_kernel) is stored in
// the true basis.  The provider returns the 4 factors z.
// forward: E (even lanes) / O (odd lanes) -> X, registers r < 4: k, r + 4: k + 512
template <class TW>
FDSNN_DEV void r2_join(double2 (&v)[8], int /*p*/, const TW& tw) {
    uint32_t raw[32];
    tw.issue_r2(raw);
    double2 z[8];
    tw.finish_r2(raw, z);
#pragma unroll
    for (int r = 0; r < 4; ++r) {
        const double2 q = shfl_xor1(v[r + 4]);
        const double2 y = cfma<false>(v[r], z[r], q);
        v[r + 4] = ctwo_minus(v[r], y);
        v[r] = y;
    }
}
// inverse: the join's output layout and scaling -> E' (even lanes) / O'
// rotated by 4 registers (odd lanes; its sign is cancelled by the twist)
template <class TW>
FDSNN_DEV void r2_split(double2 (&v)[8], int /*p*/, const TW& tw) {
    uint32_t raw[32];
    tw.issue_r2(raw);
    double2 z[8];
    tw.finish_r2(raw, z);
#pragma unroll
    for (int r = 0; r < 4; ++r) {
        const double2 mine = cadd(v[r], v[r + 4]);
        const double2 send = cmulc(csub(v[r], v[r + 4]), z[r]);
        v[r] = mine;
        v[r + 4] = shfl_xor1(send);
    }
}

template <int M, bool INV, class TW, class HOOK = NoHook, bool FT0 = false>
FDSNN_DEV void fft_group(double2 (&v)[8], int t, const TW& tw,
                         double2* __restrict__ buf0, double2* __restrict__ buf1,
                         int& ex, const GroupSync& gs, const HOOK& pre_last = HOOK(),
                         const double2* tw0 = nullptr) {
    static_assert(!FT0 || (M != 1024 && !INV), "fused twist: M <= 512 forward only");
    if constexpr (M == 1024) {
        const int p = t & 1;
        double2* b0 = buf0 + p * FFT1024_HALF;
        double2* b1 = buf1 + p * FFT1024_HALF;
        if constexpr (INV) {
            r2_split(v, p, tw);
            fft_stockham<512, true>(v, t >> 1, tw.sub(), b0, b1, ex, gs, pre_last);
        } else {
            fft_stockham<512, false>(v, t >> 1, tw.sub(), b0, b1, ex, gs, pre_last);
            r2_join(v, p, tw);
        }
    } else {
        fft_stockham<M, INV, TW, HOOK, FT0>(v, t, tw, buf0, buf1, ex, gs, pre_last, tw0);
    }
}

template <int M, bool INV, class TW, class HOOK = NoHook, bool ENTRY_SYNC = true, bool FT0 = false>
FDSNN_DEV void fft_group2(double2 (&v0)[8], double2 (&v1)[8], int t, const TW& tw,
                          double2* __restrict__ buf0, double2* __restrict__ buf1,
                          const GroupSync& gs, const HOOK& pre_last = HOOK(),
                          const double2* tw0 = nullptr) {
    static_assert(!FT0 || (FDSNN_PIPE2 && !INV), "fused twist: pipelined forward pairs only");
    if constexpr (M == 1024) {
        const int p = t & 1;
        double2* b0 = buf0 + p * FFT1024_HALF;
        double2* b1 = buf1 + p * FFT1024_HALF;
        if constexpr (INV) {
            r2_split(v0, p, tw);
            r2_split(v1, p, tw);
            if constexpr (FDSNN_PIPE2) fft_stockham2p<512, true, decltype(tw.sub()), HOOK, ENTRY_SYNC>(v0, v1, t >> 1, tw.sub(), b0, b1, gs, pre_last);
            else fft_stockham2<512, true>(v0, v1, t >> 1, tw.sub(), b0, b1, gs, pre_last);
        } else {
            if constexpr (FDSNN_PIPE2) fft_stockham2p<512, false, decltype(tw.sub()), HOOK, ENTRY_SYNC, FT0>(v0, v1, t >> 1, tw.sub(), b0, b1, gs, pre_last, tw0);
            else fft_stockham2<512, false>(v0, v1, t >> 1, tw.sub(), b0, b1, gs, pre_last);
            r2_join(v0, p, tw);
            r2_join(v1, p, tw);
        }
    } else if constexpr (FDSNN_PIPE2 && Schedule<M>::P == 3) {
        fft_stockham2p<M, INV, TW, HOOK, ENTRY_SYNC, FT0>(v0, v1, t, tw, buf0, buf1, gs, pre_last, tw0);
    } else {
        fft_stockham2<M, INV>(v0, v1, t, tw, buf0, buf1, gs, pre_last);
    }
}

}  // namespace fdsnn
