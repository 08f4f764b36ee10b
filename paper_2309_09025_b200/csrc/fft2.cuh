// fft2.cuh — "layout 2" folded negacyclic transform pair for M = 512 (DESK),
// used by the paired-level blind rotation.  Same transform as fft.cuh
// (reference ring.py:103-137: forward DFT with e^{+2 pi i jk/M}, inverse with
// e^{-}, unnormalised); a different distribution of points over the 64
// threads of a group so that the FIRST exchange of a forward transform (and
// the LAST of an inverse one) is warp-local:
//
//   fA (coefficients, forward input / inverse output): thread t = 32 t5 + l
//       holds n = 64 r + 8 n1 + n0 with n1 = l >> 2, n0 = 4 t5 + (l & 3)
//   pass 0: dft8 over r -> k0
//   E1 (warp-local): the 3 bits n1 (lane) and k0 (register) trade places
//   fB: lane i holds k0 = 4 ((i >> 1) & 1) + ((i >> 2) & 3),
//       n0 = 4 t5 + 2 (i & 1) + (i >> 4); registers n1 = 0..7
//   pass 1: twiddle w64^(n1 k0), dft8 over n1 -> k1; twiddle w512^(n0 (k0 + 8 k1))
//   E2 (shared memory, cross-warp, padded a + a/8, conflict-free both ways)
//   fC: thread t'' = 8 k1 + k0, registers n0 -> pass 2: dft8 -> k2:
//       natural frequencies t'' + 64 k2 (the key layout is unchanged)
// The inverse runs the forward backwards (dft8 inverse, conjugate twiddles
// after the butterflies, exchanges mirrored), ending in fA.
//
// Of the two transforms of a pair, the first takes E1 through a warp-local
// shared-memory transpose (__syncwarp only) and the second through two
// tensor-memory hops (tcgen05.st 32x32b -> ld 16x256b, then st 32x32b -> ld
// 16x64b; inverse: st 16x64b -> ld 32x32b, st 16x256b -> ld 32x32b), so the
// two exchanges run on different data paths at the same time.  Index maps
// are checked in tools/layout2_model.py.
#pragma once
#include "fft.cuh"

namespace fdsnn {

namespace l2 {

FDSNN_DEV int fa_n(int t, int r) { return 64 * r + 8 * ((t & 31) >> 2) + 4 * (t >> 5) + (t & 3); }
FDSNN_DEV int fb_k0(int t) { const int i = t & 31; return 4 * ((i >> 1) & 1) + ((i >> 2) & 3); }
FDSNN_DEV int fb_n0(int t) { const int i = t & 31; return 4 * (t >> 5) + 2 * (i & 1) + (i >> 4); }
FDSNN_DEV int pad(int a) { return a + (a >> 3); }

// ---- E1 through shared memory (warp region of 288 complex) ----
FDSNN_DEV void e1_smem_fwd(double2 (&v)[8], int t, double2* __restrict__ wreg) {
    const int l = t & 31;
    __syncwarp();  // previous readers of this region are done
#pragma unroll
    for (int k = 0; k < 8; ++k) wreg[pad(8 * l + k)] = v[k];
    __syncwarp();
    const int k0 = fb_k0(t), a = fb_n0(t) & 3;
#pragma unroll
    for (int n1 = 0; n1 < 8; ++n1) v[n1] = wreg[pad(32 * n1 + 8 * a + k0)];
}
FDSNN_DEV void e1_smem_inv(double2 (&v)[8], int t, double2* __restrict__ wreg) {
    const int l = t & 31;
    const int k0 = fb_k0(t), a = fb_n0(t) & 3;
    __syncwarp();
#pragma unroll
    for (int n1 = 0; n1 < 8; ++n1) wreg[pad(32 * n1 + 8 * a + k0)] = v[n1];
    __syncwarp();
#pragma unroll
    for (int k = 0; k < 8; ++k) v[k] = wreg[pad(8 * l + k)];
}

// ---- E1 through tensor memory ----
// word layout of 8 complex in 32 columns: re of c at (2c, 2c+1), im at (16+2c, 17+2c)
FDSNN_DEV void pack32(const double2 (&v)[8], uint32_t (&w)[32]) {
#pragma unroll
    for (int c = 0; c < 8; ++c) {
        w[2 * c] = (uint32_t)__double2loint(v[c].x);
        w[2 * c + 1] = (uint32_t)__double2hiint(v[c].x);
        w[16 + 2 * c] = (uint32_t)__double2loint(v[c].y);
        w[17 + 2 * c] = (uint32_t)__double2hiint(v[c].y);
    }
}
FDSNN_DEV void unpack32(const uint32_t (&w)[32], double2 (&v)[8]) {
#pragma unroll
    for (int c = 0; c < 8; ++c)
        v[c] = make_double2(__hiloint2double((int)w[2 * c + 1], (int)w[2 * c]),
                            __hiloint2double((int)w[17 + 2 * c], (int)w[16 + 2 * c]));
}
FDSNN_DEV void tm_sync_st() {
    tmem_wait_st();
    tmem_fence_before();
    __syncwarp();
    tmem_fence_after();
}
#define FDSNN_Q16(q, o) "=r"(q[o]), "=r"(q[o + 1]), "=r"(q[o + 2]), "=r"(q[o + 3]), "=r"(q[o + 4]), "=r"(q[o + 5]), \
    "=r"(q[o + 6]), "=r"(q[o + 7]), "=r"(q[o + 8]), "=r"(q[o + 9]), "=r"(q[o + 10]), "=r"(q[o + 11]), "=r"(q[o + 12]), \
    "=r"(q[o + 13]), "=r"(q[o + 14]), "=r"(q[o + 15])
#define FDSNN_R16(q, o) "r"(q[o]), "r"(q[o + 1]), "r"(q[o + 2]), "r"(q[o + 3]), "r"(q[o + 4]), "r"(q[o + 5]), \
    "r"(q[o + 6]), "r"(q[o + 7]), "r"(q[o + 8]), "r"(q[o + 9]), "r"(q[o + 10]), "r"(q[o + 11]), "r"(q[o + 12]), \
    "r"(q[o + 13]), "r"(q[o + 14]), "r"(q[o + 15])
// 16 lanes x N columns shapes at lane offsets 0 and 16 of the warp's quadrant
FDSNN_DEV void ld_16x256(uint32_t a, uint32_t (&q)[32]) {
    asm volatile("tcgen05.ld.sync.aligned.16x256b.x4.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%32];\n\t"
                 "tcgen05.ld.sync.aligned.16x256b.x4.b32 {%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%33];"
                 : FDSNN_Q16(q, 0), FDSNN_Q16(q, 16) : "r"(a), "r"(a + (16u << 16)) : "memory");
}
FDSNN_DEV void st_16x256(uint32_t a, const uint32_t (&q)[32]) {
    asm volatile("tcgen05.st.sync.aligned.16x256b.x4.b32 [%0], {%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17};\n\t"
                 "tcgen05.st.sync.aligned.16x256b.x4.b32 [%1], {%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32,%33};"
                 :: "r"(a), "r"(a + (16u << 16)), FDSNN_R16(q, 0), FDSNN_R16(q, 16) : "memory");
}
FDSNN_DEV void ld_16x64(uint32_t a, uint32_t (&q)[32]) {
    asm volatile("tcgen05.ld.sync.aligned.16x64b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%32];\n\t"
                 "tcgen05.ld.sync.aligned.16x64b.x16.b32 {%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%33];"
                 : FDSNN_Q16(q, 0), FDSNN_Q16(q, 16) : "r"(a), "r"(a + (16u << 16)) : "memory");
}
FDSNN_DEV void st_16x64(uint32_t a, const uint32_t (&q)[32]) {
    asm volatile("tcgen05.st.sync.aligned.16x64b.x16.b32 [%0], {%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17};\n\t"
                 "tcgen05.st.sync.aligned.16x64b.x16.b32 [%1], {%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32,%33};"
                 :: "r"(a), "r"(a + (16u << 16)), FDSNN_R16(q, 0), FDSNN_R16(q, 16) : "memory");
}
#undef FDSNN_Q16
#undef FDSNN_R16

// 16x256b.x4 register q[16 Lh + 4 k + 2 hh + {0,1}]: word col 8k + 2(i&3) + {0,1}
// of lane 16 Lh + 8 hh + (i >> 2).  With re(c) at words (2c, 2c+1) and im(c) at
// (16+2c, 17+2c): k = 0,1 hold re of c = 4k + (i&3), k = 2,3 the matching im.
// H-register 4 Lh + 2 k + hh  <->  complex c = 4k + (i&3) of that lane.
FDSNN_DEV void h_unpack(const uint32_t (&q)[32], double2 (&h)[8]) {
#pragma unroll
    for (int Lh = 0; Lh < 2; ++Lh)
#pragma unroll
        for (int k = 0; k < 2; ++k)
#pragma unroll
            for (int hh = 0; hh < 2; ++hh) {
                const int o = 16 * Lh + 4 * k + 2 * hh;
                h[4 * Lh + 2 * k + hh] = make_double2(__hiloint2double((int)q[o + 1], (int)q[o]),
                                                      __hiloint2double((int)q[o + 9], (int)q[o + 8]));
            }
}
FDSNN_DEV void h_pack(const double2 (&h)[8], uint32_t (&q)[32]) {
#pragma unroll
    for (int Lh = 0; Lh < 2; ++Lh)
#pragma unroll
        for (int k = 0; k < 2; ++k)
#pragma unroll
            for (int hh = 0; hh < 2; ++hh) {
                const int o = 16 * Lh + 4 * k + 2 * hh;
                const double2 c = h[4 * Lh + 2 * k + hh];
                q[o] = (uint32_t)__double2loint(c.x);
                q[o + 1] = (uint32_t)__double2hiint(c.x);
                q[o + 8] = (uint32_t)__double2loint(c.y);
                q[o + 9] = (uint32_t)__double2hiint(c.y);
            }
}
// 16x64b.x16 register q[16 Lh + j]: word col 2j + ((i >> 1) & 1) of lane
// (i >> 2) + 8 (i & 1) + 16 Lh.  With re(c) at words (2c, 2c+1), im(c) at
// (16+2c, 17+2c), the lo/hi words of one double land in different threads;
// so for this hop doubles are stored split: lo words in cols 0-15, hi words in
// cols 16-31 (double d = re(c) for d = c, im(c) for d = 8 + c).  Then register
// q[16 Lh + j] (j < 8) is the lo word of double 2j + b (b = (i>>1)&1) and
// q[16 Lh + 8 + j] its hi word: complex c = 2j' + b for j' = j < 4 (re) and
// j - 4 (im).  G-register 4 Lh + j'  <->  complex 2 j' + b of that lane.
FDSNN_DEV void pack_split(const double2 (&v)[8], uint32_t (&w)[32]) {
#pragma unroll
    for (int c = 0; c < 8; ++c) {
        w[c] = (uint32_t)__double2loint(v[c].x);
        w[16 + c] = (uint32_t)__double2hiint(v[c].x);
        w[8 + c] = (uint32_t)__double2loint(v[c].y);
        w[24 + c] = (uint32_t)__double2hiint(v[c].y);
    }
}
FDSNN_DEV void unpack_split(const uint32_t (&w)[32], double2 (&v)[8]) {
#pragma unroll
    for (int c = 0; c < 8; ++c)
        v[c] = make_double2(__hiloint2double((int)w[16 + c], (int)w[c]),
                            __hiloint2double((int)w[24 + c], (int)w[8 + c]));
}
FDSNN_DEV void g_unpack(const uint32_t (&q)[32], double2 (&g)[8]) {
#pragma unroll
    for (int Lh = 0; Lh < 2; ++Lh)
#pragma unroll
        for (int jp = 0; jp < 4; ++jp)
            g[4 * Lh + jp] = make_double2(__hiloint2double((int)q[16 * Lh + 8 + jp], (int)q[16 * Lh + jp]),
                                          __hiloint2double((int)q[16 * Lh + 12 + jp], (int)q[16 * Lh + 4 + jp]));
}
FDSNN_DEV void g_pack(const double2 (&g)[8], uint32_t (&q)[32]) {
#pragma unroll
    for (int Lh = 0; Lh < 2; ++Lh)
#pragma unroll
        for (int jp = 0; jp < 4; ++jp) {
            const double2 c = g[4 * Lh + jp];
            q[16 * Lh + jp] = (uint32_t)__double2loint(c.x);
            q[16 * Lh + 8 + jp] = (uint32_t)__double2hiint(c.x);
            q[16 * Lh + 4 + jp] = (uint32_t)__double2loint(c.y);
            q[16 * Lh + 12 + jp] = (uint32_t)__double2hiint(c.y);
        }
}
// register renaming between the hops: G-complex c = 2 (2 Lh + hh) + k holds
// H-register 4 Lh + 2 k + hh (tools/layout2_model.py `ren`)
__host__ __device__ constexpr int kRen(int c) { return (c & 4) | ((c & 1) << 1) | ((c >> 1) & 1); }  // c -> H register {0,2,1,3,4,6,5,7}
// after G, register j holds n1 = kN1[j]
__host__ __device__ constexpr int kN1(int j) { return ((j & 3) << 1) | (j >> 2); }  // {0,2,4,6,1,3,5,7}

FDSNN_DEV void e1_tmem_fwd(double2 (&v)[8], uint32_t col) {
    uint32_t w[32], q[32];
    pack32(v, w);
    tmem_st32(col, w);
    tm_sync_st();
    ld_16x256(col, q);
    tmem_wait32(q);
    double2 h[8], g[8];
    h_unpack(q, h);
#pragma unroll
    for (int c = 0; c < 8; ++c) g[c] = h[kRen(c)];
    tmem_fence_before();
    __syncwarp();  // everyone's H loads done before the region is overwritten
    tmem_fence_after();
    pack_split(g, w);
    tmem_st32(col, w);
    tm_sync_st();
    ld_16x64(col, q);
    tmem_wait32(q);
    g_unpack(q, h);
#pragma unroll
    for (int j = 0; j < 8; ++j) v[kN1(j)] = h[j];
    tmem_fence_before();
    __syncwarp();
    tmem_fence_after();
}
FDSNN_DEV void e1_tmem_inv(double2 (&v)[8], uint32_t col) {
    uint32_t q[32], w[32];
    double2 h[8], g[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) g[j] = v[kN1(j)];
    g_pack(g, q);
    st_16x64(col, q);
    tm_sync_st();
    tmem_ld32_async(col, w);
    tmem_wait32(w);
    unpack_split(w, g);  // g[c], c = G-complex
#pragma unroll
    for (int c = 0; c < 8; ++c) h[kRen(c)] = g[c];
    tmem_fence_before();
    __syncwarp();
    tmem_fence_after();
    h_pack(h, q);
    st_16x256(col, q);
    tm_sync_st();
    tmem_ld32_async(col, w);
    tmem_wait32(w);
    unpack32(w, v);  // v[k0]
    tmem_fence_before();
    __syncwarp();
    tmem_fence_after();
}

// ---- E2 through shared memory ----
FDSNN_DEV void e2_store_fwd(const double2 (&v)[8], int t, double2* __restrict__ buf) {
    const int k0 = fb_k0(t), n0 = fb_n0(t);
#pragma unroll
    for (int k1 = 0; k1 < 8; ++k1) buf[pad(8 * (k0 + 8 * k1) + n0)] = v[k1];
}
FDSNN_DEV void e2_load_fwd(double2 (&v)[8], int t, const double2* __restrict__ buf) {
#pragma unroll
    for (int n0 = 0; n0 < 8; ++n0) v[n0] = buf[pad(8 * t + n0)];
}
FDSNN_DEV void e2_store_inv(const double2 (&v)[8], int t, double2* __restrict__ buf) {
#pragma unroll
    for (int n0 = 0; n0 < 8; ++n0) buf[pad(8 * t + n0)] = v[n0];
}
FDSNN_DEV void e2_load_inv(double2 (&v)[8], int t, const double2* __restrict__ buf) {
    const int k0 = fb_k0(t), n0 = fb_n0(t);
#pragma unroll
    for (int k1 = 0; k1 < 8; ++k1) v[k1] = buf[pad(8 * (k0 + 8 * k1) + n0)];
}

}  // namespace l2

// Twiddles of layout 2, per lane in TMEM: w64^(n1 k0) for n1 = 1..7 at
// column 0 (entries n1 - 1), w512^(n0 (k0 + 8 k1)) for k1 = 0..7 at column 32.
struct TwiddlesL2 {
    uint32_t base;
    FDSNN_DEV void issue1(uint32_t (&raw)[32]) const { tmem_ld32_async(base, raw); }
    FDSNN_DEV void issue2(uint32_t (&raw)[32]) const { tmem_ld32_async(base + 32, raw); }
    FDSNN_DEV void finish(uint32_t (&raw)[32], double2 (&w)[8]) const {
        tmem_wait32(raw);
#pragma unroll
        for (int r = 0; r < 8; ++r) w[r] = words_c(raw, r);
    }
};

// Forward pair: v0, v1 in fA (points) -> natural frequencies.  xbuf: the
// group's E1 region (2 warps x 288 complex), buf0/buf1: E2 buffers, xcol: the
// warp's TMEM hop columns.
FDSNN_DEV void fft2_fwd_pair(double2 (&v0)[8], double2 (&v1)[8], int t, const TwiddlesL2& tw,
                             double2* __restrict__ xbuf, double2* __restrict__ buf0,
                             double2* __restrict__ buf1, uint32_t xcol, const GroupSync& gs) {
    dft8<false>(v0);
    dft8<false>(v1);
    uint32_t raw1[32];
    tw.issue1(raw1);
    l2::e1_smem_fwd(v0, t, xbuf + (t >> 5) * 288);
    l2::e1_tmem_fwd(v1, xcol);
    double2 w[8];
    tw.finish(raw1, w);
#pragma unroll
    for (int n1 = 1; n1 < 8; ++n1) {
        v0[n1] = cmul(v0[n1], w[n1 - 1]);
        v1[n1] = cmul(v1[n1], w[n1 - 1]);
    }
    dft8<false>(v0);
    dft8<false>(v1);
    uint32_t raw2[32];
    tw.issue2(raw2);
    tw.finish(raw2, w);
#pragma unroll
    for (int k1 = 0; k1 < 8; ++k1) {
        v0[k1] = cmul(v0[k1], w[k1]);
        v1[k1] = cmul(v1[k1], w[k1]);
    }
    gs.sync();  // the previous users of buf0/buf1 are done
    l2::e2_store_fwd(v0, t, buf0);
    l2::e2_store_fwd(v1, t, buf1);
    gs.sync();
    l2::e2_load_fwd(v0, t, buf0);
    l2::e2_load_fwd(v1, t, buf1);
    dft8<false>(v0);
    dft8<false>(v1);
}

// Inverse pair: natural frequencies -> fA points (unnormalised; the 1/M is in
// the key).  `pre_last` runs before the last butterflies (fetch hook).
template <class HOOK = NoHook>
FDSNN_DEV void fft2_inv_pair(double2 (&v0)[8], double2 (&v1)[8], int t, const TwiddlesL2& tw,
                             double2* __restrict__ xbuf, double2* __restrict__ buf0,
                             double2* __restrict__ buf1, uint32_t xcol, const GroupSync& gs,
                             const HOOK& pre_last = HOOK()) {
    dft8<true>(v0);
    dft8<true>(v1);
    uint32_t raw2[32];
    tw.issue2(raw2);
    gs.sync();
    l2::e2_store_inv(v0, t, buf0);
    l2::e2_store_inv(v1, t, buf1);
    double2 w[8];
    tw.finish(raw2, w);
    gs.sync();
    l2::e2_load_inv(v0, t, buf0);
    l2::e2_load_inv(v1, t, buf1);
#pragma unroll
    for (int k1 = 0; k1 < 8; ++k1) {
        v0[k1] = cmulc(v0[k1], w[k1]);
        v1[k1] = cmulc(v1[k1], w[k1]);
    }
    dft8<true>(v0);
    dft8<true>(v1);
    uint32_t raw1[32];
    tw.issue1(raw1);
    tw.finish(raw1, w);
#pragma unroll
    for (int n1 = 1; n1 < 8; ++n1) {
        v0[n1] = cmulc(v0[n1], w[n1 - 1]);
        v1[n1] = cmulc(v1[n1], w[n1 - 1]);
    }
    l2::e1_smem_inv(v0, t, xbuf + (t >> 5) * 288);
    l2::e1_tmem_inv(v1, xcol);
    pre_last();
    dft8<true>(v0);
    dft8<true>(v1);
}

}  // namespace fdsnn
