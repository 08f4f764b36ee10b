// fft16.cuh — warp-per-transform folded negacyclic transform, M = 512.
//
// Same transform as fft.cuh / ring.NegacyclicTransform (reference
// ring.py:103-137): fold c_j = (a_j + i a_{j+M}) e^{i pi j/N}, then the
// length-M DFT with the e^{+2 pi i jk/M} kernel; the inverse is the
// unnormalised e^{-2 pi i} DFT followed by the conjugate twist (the Fourier
// key carries the 1/M).
//
// B200 layout: ONE warp transforms one polynomial, 16 points per lane, so the
// only synchronisation a transform needs is __syncwarp.  M = 16 x 32:
//   pass A  lane l holds points p = l + 32 j2 (j2 < 16): 16-point DFT over j2
//           with the twist fused into its first butterflies -> Y[l][k2];
//   exchange through shared memory (16 STS.128 + 16 LDS.128 per lane, row
//           stride 34 x 16 B: conflict-free both ways);
//   pass B  lane L = 2 k2' + a holds Y[a + 2b][k2'] (b < 16): 16-point DFT
//           over b with the twiddles w512^{(a+2b) k2'} fused in -> W_a[c];
//   join    radix-2 between lanes 2k2' and 2k2'+1 over warp shuffles, each
//           lane sending 8 of its 16 values (half the bytes of a full swap):
//           X[k2' + 16c + 256d] = W_0[c] + (-1)^d w32^c W_1[c].
// Against the 64-thread, 8-points-per-lane radix-8 transform (two
// shared-memory exchanges and two group barriers), one transform moves 160
// instead of 256 cycles' worth of data through the L1/shared pipe and never
// waits on another warp.
//
// Select-free join.  Lane a = 0 finishes c = r (r < 8), lane a = 1 c = r + 8.
// Odd lanes receive their pass-B inputs sign-flipped for odd b (the twist of
// lanes l = 3 mod 4 carries a -1), which rotates their W_1 by 8 positions, so
// every lane keeps registers 0-7 and ships registers 8-15.  The join then
// computes out0 = P + z Q, out1 = P - z Q uniformly (P own, Q received) with
// z = w32^c on even lanes and w32^{-c} on odd lanes: odd lanes hold
// s X with the unit factor s = w32^{-c} (d = 0) / -w32^{-c} (d = 1).  The
// inverse's first step consumes exactly that scaling, so products formed
// against a key stored in the TRUE frequency basis come back right; the key
// transform (bsk_forward16_kernel) multiplies its odd-lane outputs by conj(s).
// The inverse's odd lanes see their inputs rotated by 8 as well, which
// leaves a (-1)^b on lanes l = 3 mod 4 after the return exchange -- cancelled
// by the conjugate of the same signed twist.
//
// Output / key layout: lane L, register r (d = 0) and r + 8 (d = 1) hold
// frequency k2' + 16 (r + 8a) + 256 d; the Fourier key is stored as
// [poly h][register r + 8d][lane] (one 16-byte word per lane: LDS.128,
// conflict-free).
#pragma once
#include "fft.cuh"

namespace fdsnn {
namespace r16 {

constexpr int M = 512;
constexpr int XSTRIDE = 34;            // exchange row stride (complex) per k2
constexpr int XBUF = 16 * XSTRIDE;     // complex per warp exchange buffer
// Twist factorisation.  The twist of point p = l + 32 j2 splits into a lane
// factor and a register factor: sigma_l e^{i pi p/N} = c_l g_{j2} with
// c_l = sigma_l e^{i pi l/N} (sigma = -1 for l = 3 mod 4, see the join) and
// g_{j2} = e^{i pi j2/32} (N = 1024).  Pass A (a DFT over j2 inside lane l)
// applies only g -- compile-time constants, no table -- and commutes with the
// lane constant c_l, which is folded into pass B's twiddles:
//   FB[L][b] = w512^{(a + 2b) k2'} c_{a + 2b}      (lane L = 2 k2' + a).
// The inverse mirrors the forward: its first DFT16 (over b in lane L) is
// followed by the conjugates of the same FB factors (the inter-pass twiddles
// of the inverse and the untwist's lane factor conj(c_l) at once), the return
// exchange, a twiddle-free DFT16 over k2 and the register untwist conj(g_j2).
// Per-lane constant table: 3 blocks of 8 complex (32 words = 32 TMEM columns
// each), lane-major [lane][TAB] in global memory.
constexpr int BLK_FB_E = 0;  // FB[L][b], even b
constexpr int BLK_FB_O = 1;  //   odd b
constexpr int BLK_ZJ = 2;    // a = 0: w32^r, a = 1: w32^{-(r+8)}, r < 8
constexpr int NBLK = 3;
constexpr int TAB = 8 * NBLK;

// g_j = e^{i pi j/32}, j < 16
FDSNN_DEV constexpr double g_cos(int j) {
    constexpr double c[16] = {1.0, 0.995184726672196886245, 0.980785280403230449126, 0.956940335732208864936,
                              0.923879532511286756128, 0.881921264348355029713, 0.831469612302545237079,
                              0.773010453362736960811, 0.707106781186547524401, 0.634393284163645498215,
                              0.555570233019602224743, 0.471396736825997648556, 0.382683432365089771728,
                              0.290284677254462367636, 0.195090322016128267848, 0.098017140329560601994};
    return c[j];
}
FDSNN_DEV constexpr double g_sin(int j) { return j == 0 ? 0.0 : g_cos(16 - j); }
FDSNN_DEV double2 g_twist(int j) { return make_double2(g_cos(j), j == 0 ? 0.0 : g_cos(16 - j)); }

// Table providers: issue(blk, raw) starts fetching block blk (8 complex),
// finish(raw, w) completes it.
struct TabGlobal {
    const double2* t;  // this lane's row
    FDSNN_DEV void issue(int blk, uint32_t (&raw)[32]) const {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const double2 w = __ldg(t + 8 * blk + i);
            raw[4 * i] = (uint32_t)__double2loint(w.x);
            raw[4 * i + 1] = (uint32_t)__double2hiint(w.x);
            raw[4 * i + 2] = (uint32_t)__double2loint(w.y);
            raw[4 * i + 3] = (uint32_t)__double2hiint(w.y);
        }
    }
    FDSNN_DEV void finish(uint32_t (&raw)[32], double2 (&w)[8]) const {
#pragma unroll
        for (int i = 0; i < 8; ++i) w[i] = words_c(raw, i);
    }
};
struct TabTmem {
    uint32_t col;  // this lane quadrant's first table column
    FDSNN_DEV void issue(int blk, uint32_t (&raw)[32]) const { tmem_ld32_async(col + 32 * blk, raw); }
    FDSNN_DEV void finish(uint32_t (&raw)[32], double2 (&w)[8]) const {
        tmem_wait32(raw);
#pragma unroll
        for (int i = 0; i < 8; ++i) w[i] = words_c(raw, i);
    }
};

// Y[k] = E[k] + w16^k O[k], Y[k+8] = E[k] - w16^k O[k]  (INV: conj(w16))
template <bool INV>
FDSNN_DEV void radix2_16(double2 (&v)[16], const double2 (&e)[8], const double2 (&o)[8]) {
    v[0] = cadd(e[0], o[0]);
    v[8] = csub(e[0], o[0]);
    {
        const double2 t = mul_si<INV>(o[4]);
        v[4] = cadd(e[4], t);
        v[12] = csub(e[4], t);
    }
    constexpr double C1 = 0.92387953251128675613, S1 = 0.38268343236508977173;  // cos, sin(pi/8)
    constexpr double H = 0.70710678118654752440;
#pragma unroll
    for (int k = 1; k < 8; ++k) {
        if (k == 4) continue;
        const double c = k == 1 ? C1 : k == 2 ? H : k == 3 ? S1 : k == 5 ? -S1 : k == 6 ? -H : -C1;
        const double s = k == 1 ? S1 : k == 2 ? H : k == 3 ? C1 : k == 5 ? C1 : k == 6 ? H : S1;
        const double2 y = cfma<INV>(e[k], make_double2(c, s), o[k]);
        v[k] = y;
        v[k + 8] = ctwo_minus(e[k], y);
    }
}

constexpr int TWIST_G = -2;  // dft16 BLK value: input twiddles g_j (constants)

// 16-point DFT, natural order in/out, kernel e^{+2 pi i/16} (INV: e^{-}).
// BLK >= 0: the input twiddles of table blocks BLK (even points) and BLK + 1
// (odd points) are fused into the first butterflies (conjugated when INV),
// as dft8_tw does for radix 8; BLK == TWIST_G: the constants g_j instead
// (g_0 = 1 is skipped).
template <bool INV, int BLK, class TP>
FDSNN_DEV void dft16(double2 (&v)[16], const TP& tp) {
    double2 e[8], o[8];
#pragma unroll
    for (int r = 0; r < 8; ++r) {
        e[r] = v[2 * r];
        o[r] = v[2 * r + 1];
    }
    if constexpr (BLK >= 0) {
        // one block in flight at a time (registers): the odd block's fetch
        // overlaps the even half's butterflies
        double2 w[8];
        {
            uint32_t re[32];
            tp.issue(BLK, re);
            tp.finish(re, w);
        }
        uint32_t ro[32];
        tp.issue(BLK + 1, ro);
        dft8_tw<INV, true>(e, w);
        tp.finish(ro, w);
        dft8_tw<INV, true>(o, w);
    } else if constexpr (BLK == TWIST_G) {
        double2 we[7], wo[8];
#pragma unroll
        for (int r = 0; r < 8; ++r) {
            if (r > 0) we[r - 1] = g_twist(2 * r);
            wo[r] = g_twist(2 * r + 1);
        }
        dft8_tw<INV, false>(e, we);
        dft8_tw<INV, true>(o, wo);
    } else {
        dft8<INV>(e);
        dft8<INV>(o);
    }
    radix2_16<INV>(v, e, o);
}

FDSNN_DEV double2 shfl_xor1c(double2 a) {
    return make_double2(__shfl_xor_sync(0xffffffffu, a.x, 1), __shfl_xor_sync(0xffffffffu, a.y, 1));
}

// Forward transform of one polynomial by one warp.
//   in:  v[j2] = folded point l + 32 j2 (digits, before the twist)
//   out: v[r] / v[r+8] = frequency k2' + 16 (r + 8a) (+ 256), odd lanes scaled (header)
// xbuf: the warp's exchange buffer.
template <class TP>
FDSNN_DEV void forward(double2 (&v)[16], int lane, const TP& tp, double2* __restrict__ xbuf) {
    dft16<false, TWIST_G>(v, tp);
    __syncwarp();  // the previous transform's readers of xbuf are done
#pragma unroll
    for (int k = 0; k < 16; ++k) xbuf[k * XSTRIDE + lane] = v[k];
    __syncwarp();
    const int row = (lane >> 1) * XSTRIDE + (lane & 1);
#pragma unroll
    for (int b = 0; b < 16; ++b) v[b] = xbuf[row + 2 * b];
    dft16<false, BLK_FB_E>(v, tp);
    double2 zj[8];
    {
        uint32_t rz[32];
        tp.issue(BLK_ZJ, rz);
        tp.finish(rz, zj);
    }
#pragma unroll
    for (int r = 0; r < 8; ++r) {
        const double2 q = shfl_xor1c(v[r + 8]);
        const double2 y = cfma<false>(v[r], zj[r], q);
        v[r + 8] = ctwo_minus(v[r], y);
        v[r] = y;
    }
}

// Inverse transform (unnormalised, kernel e^{-2 pi i jk/M}) of one polynomial.
//   in:  v in the forward's output layout and scaling
//   out: v[j2] = M * point l + 32 j2 times g_{j2} (the caller untwists with
//        conj(g_{j2}); the lane factor conj(c_l) is already applied)
template <class TP>
FDSNN_DEV void inverse(double2 (&v)[16], int lane, const TP& tp, double2* __restrict__ xbuf) {
    {
        uint32_t rz[32];
        tp.issue(BLK_ZJ, rz);
        double2 zj[8];
        tp.finish(rz, zj);
#pragma unroll
        for (int r = 0; r < 8; ++r) {
            const double2 mine = cadd(v[r], v[r + 8]);
            const double2 send = cmulc(csub(v[r], v[r + 8]), zj[r]);
            v[r] = mine;
            v[r + 8] = shfl_xor1c(send);
        }
    }
    dft16<true, -1>(v, tp);
    {  // output twiddles conj(FB[L][b]): even b, then odd b
        uint32_t re[32], ro[32];
        double2 w[8];
        tp.issue(BLK_FB_E, re);
        tp.issue(BLK_FB_O, ro);
        tp.finish(re, w);
#pragma unroll
        for (int r = 0; r < 8; ++r) v[2 * r] = cmulc(v[2 * r], w[r]);
        tp.finish(ro, w);
#pragma unroll
        for (int r = 0; r < 8; ++r) v[2 * r + 1] = cmulc(v[2 * r + 1], w[r]);
    }
    __syncwarp();
    const int row = (lane >> 1) * XSTRIDE + (lane & 1);
#pragma unroll
    for (int b = 0; b < 16; ++b) xbuf[row + 2 * b] = v[b];
    __syncwarp();
#pragma unroll
    for (int k = 0; k < 16; ++k) v[k] = xbuf[k * XSTRIDE + lane];
    dft16<true, -1>(v, tp);
}

// Host-side construction of the per-lane table (long double, ring.py:115-118
// conventions): out[lane * TAB + e].
template <class C, class MK>
inline void build_table(int N, C* out, MK make) {
    const long double PI = 3.141592653589793238462643383279502884L;
    auto at = [&](int l, int blk, int i) -> C& { return out[l * TAB + 8 * blk + i]; };
    for (int L = 0; L < 32; ++L) {
        const int k2p = L >> 1, a = L & 1;
        for (int b = 0; b < 16; ++b) {
            const int l = a + 2 * b;  // source lane of register b
            const long double sg = (l % 4 == 3) ? -1.0L : 1.0L;
            // w512^{l k2'} c_l, c_l = sigma_l e^{i pi l / N}
            const long double ang = 2.0L * PI * (long double)((l * k2p) % M) / M + PI * l / N;
            at(L, BLK_FB_E + (b & 1), b >> 1) = make(sg * cosl(ang), sg * sinl(ang));
        }
        for (int r = 0; r < 8; ++r) {
            const int e = a ? -(r + 8) : r;
            const long double ang = 2.0L * PI * e / 32.0L;
            at(L, BLK_ZJ, r) = make(cosl(ang), sinl(ang));
        }
    }
}

}  // namespace r16
}  // namespace fdsnn
