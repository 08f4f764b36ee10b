// common.cuh — shared device-side definitions for the fdsnn B200 kernels.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#define FDSNN_DEV __device__ __forceinline__

// Parameter block passed by value to every kernel (mirrors params.FheParams,
// reference params.py:36-106, restricted to the hot path).
struct DevParams {
    int n;          // LWE dimension
    int N;          // ring degree
    int M;          // N/2 complex points of the folded transform
    int log2q;      // q = 2^log2q
    uint32_t qmask; // q - 1
    int bg_log;     // gadget base 2^bg_log
    int L;          // gadget levels
    int ks_log;     // key-switch base 2^ks_log
    int ks_L;       // key-switch levels
    int stride;     // LWE row stride in words (>= n+1, multiple of 4)
    int ext_stride; // extracted z-LWE row stride (>= N+1, multiple of 4)
    int p;          // message modulus
    int half_slot;  // N / p (bootstrap.py:333 half-slot offset)
};

FDSNN_DEV double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
FDSNN_DEV double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
// a * b
FDSNN_DEV double2 cmul(double2 a, double2 b) {
    return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
// a * conj(b)
FDSNN_DEV double2 cmulc(double2 a, double2 b) {
    return make_double2(fma(a.x, b.x, a.y * b.y), fma(a.y, b.x, -a.x * b.y));
}
// acc += a * b
FDSNN_DEV void cmac(double2& acc, double2 a, double2 b) {
    acc.x = fma(a.x, b.x, acc.x);
    acc.x = fma(-a.y, b.y, acc.x);
    acc.y = fma(a.x, b.y, acc.y);
    acc.y = fma(a.y, b.x, acc.y);
}

// Centered representative of x mod q in [-q/2, q/2) (ring.py:27-33).
FDSNN_DEV int32_t center_q(uint32_t x, int log2q) {
    uint32_t m = x & ((1u << log2q) - 1u);
    return (m >= (1u << (log2q - 1))) ? (int32_t)(m - (1u << log2q)) : (int32_t)m;
}

// ring.rescale(x, q, 2N) (ring.py:56-67): round-half-away(centered(x)*2N/q) mod 2N.
FDSNN_DEV uint32_t rescale_q_to_2N(uint32_t x, int log2q, int log2_2N) {
    int32_t c = center_q(x, log2q);
    int32_t r;
    if (log2q >= log2_2N) {
        int s = log2q - log2_2N;
        if (s == 0) {
            r = c;
        } else {
            int32_t mag = c < 0 ? -c : c;
            int32_t t = (mag + (1 << (s - 1))) >> s;  // div_round_half_away (ring.py:45-53)
            r = c < 0 ? -t : t;
        }
    } else {
        r = c * (1 << (log2_2N - log2q));
    }
    return (uint32_t)r & ((1u << log2_2N) - 1u);
}

// round-half-away-from-zero exactly as ring.round_half_away (ring.py:36-42):
// floor(x+0.5) for x>=0, ceil(x-0.5) otherwise.
FDSNN_DEV long long round_half_away(double x) {
    return (x >= 0.0) ? (long long)floor(x + 0.5) : (long long)ceil(x - 0.5);
}

// Rounding used on the transform outputs.  The exact products are integers
// and the FP64 transform error is < 0.01 (measured max 0.003, see
// fdsnn_margin_read), so every value lies within 0.01 of an integer and
// round-to-nearest-even (one F2I) selects the same integer as the reference's
// round-half-away (ring.py:36-42) -- the two differ only at exact .5 ties.
FDSNN_DEV long long round_product(double x) { return __double2ll_rn(x); }
// Low 32 bits of the same rounding (the accumulator update is mod q <= 2^31).
FDSNN_DEV uint32_t round_lo32(double x) { return (uint32_t)__double2ll_rn(x); }

// Round-to-nearest-even of |x| < 2^51 on the FP64 pipe (no F2I): x + 1.5 2^52
// lands in [2^52, 2^53) where the ulp is 1, so the sum's low mantissa word is
// round(x) + 2^51 = round(x) mod 2^32.  Same integer as round_lo32.
FDSNN_DEV uint32_t round_lo32_fp64(double x) { return (uint32_t)__double2loint(x + 6755399441055744.0); }

FDSNN_DEV void named_bar(int id, int nthreads) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// ---- mbarrier / bulk-copy (TMA) helpers (sm_90+ PTX, used on sm_100a) ----
FDSNN_DEV uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
FDSNN_DEV void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
FDSNN_DEV void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
FDSNN_DEV void mbar_arrive(uint64_t* bar) {
    asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.shared::cta.b64 st, [%0];\n\t}" ::"r"(smem_u32(bar)) : "memory");
}
FDSNN_DEV void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;\n\t}"
                 ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
FDSNN_DEV void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred P1;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
        "@!P1 bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)), "r"(parity) : "memory");
}
// ---- tensor memory (tcgen05) helpers: per-thread constants live in TMEM ----
// A warp may only address its quadrant's 32 lanes: lane = 32*(warp%4) + laneid.
FDSNN_DEV void tmem_alloc(uint32_t* smem_dst, uint32_t ncols) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;"
                 ::"r"(smem_u32(smem_dst)), "r"(ncols) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
FDSNN_DEV void tmem_dealloc(uint32_t taddr, uint32_t ncols) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols) : "memory");
}
FDSNN_DEV void tmem_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
FDSNN_DEV void tmem_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
// store 8 doubles (16 words) of this thread's lane at column offset taddr
FDSNN_DEV void tmem_st16(uint32_t taddr, const double (&d)[8]) {
    uint32_t w[16];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        w[2 * i] = (uint32_t)__double2loint(d[i]);
        w[2 * i + 1] = (uint32_t)__double2hiint(d[i]);
    }
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};"
        ::"r"(taddr), "r"(w[0]), "r"(w[1]), "r"(w[2]), "r"(w[3]), "r"(w[4]), "r"(w[5]), "r"(w[6]), "r"(w[7]),
        "r"(w[8]), "r"(w[9]), "r"(w[10]), "r"(w[11]), "r"(w[12]), "r"(w[13]), "r"(w[14]), "r"(w[15]) : "memory");
}
FDSNN_DEV void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
// load 4 complex doubles (16 words) of this thread's lane from column offset taddr
FDSNN_DEV void tmem_ld4c(uint32_t taddr, double2 (&c)[4]) {
    uint32_t w[16];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n\t"
        "tcgen05.wait::ld.sync.aligned;"
        : "=r"(w[0]), "=r"(w[1]), "=r"(w[2]), "=r"(w[3]), "=r"(w[4]), "=r"(w[5]), "=r"(w[6]), "=r"(w[7]),
          "=r"(w[8]), "=r"(w[9]), "=r"(w[10]), "=r"(w[11]), "=r"(w[12]), "=r"(w[13]), "=r"(w[14]), "=r"(w[15])
        : "r"(taddr) : "memory");
#pragma unroll
    for (int i = 0; i < 4; ++i)
        c[i] = make_double2(__hiloint2double((int)w[4 * i + 1], (int)w[4 * i]),
                            __hiloint2double((int)w[4 * i + 3], (int)w[4 * i + 2]));
}

// Asynchronous 32-word TMEM load; the registers are valid only after
// tmem_wait32 on the same array (which carries them as operands so the
// compiler cannot hoist a use above the wait).
FDSNN_DEV void tmem_ld32_async(uint32_t taddr, uint32_t (&w)[32]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(w[0]), "=r"(w[1]), "=r"(w[2]), "=r"(w[3]), "=r"(w[4]), "=r"(w[5]), "=r"(w[6]), "=r"(w[7]),
          "=r"(w[8]), "=r"(w[9]), "=r"(w[10]), "=r"(w[11]), "=r"(w[12]), "=r"(w[13]), "=r"(w[14]), "=r"(w[15]),
          "=r"(w[16]), "=r"(w[17]), "=r"(w[18]), "=r"(w[19]), "=r"(w[20]), "=r"(w[21]), "=r"(w[22]), "=r"(w[23]),
          "=r"(w[24]), "=r"(w[25]), "=r"(w[26]), "=r"(w[27]), "=r"(w[28]), "=r"(w[29]), "=r"(w[30]), "=r"(w[31])
        : "r"(taddr) : "memory");
}
FDSNN_DEV void tmem_wait32(uint32_t (&w)[32]) {
    asm volatile("tcgen05.wait::ld.sync.aligned;"
                 : "+r"(w[0]), "+r"(w[1]), "+r"(w[2]), "+r"(w[3]), "+r"(w[4]), "+r"(w[5]), "+r"(w[6]), "+r"(w[7]),
                   "+r"(w[8]), "+r"(w[9]), "+r"(w[10]), "+r"(w[11]), "+r"(w[12]), "+r"(w[13]), "+r"(w[14]), "+r"(w[15]),
                   "+r"(w[16]), "+r"(w[17]), "+r"(w[18]), "+r"(w[19]), "+r"(w[20]), "+r"(w[21]), "+r"(w[22]), "+r"(w[23]),
                   "+r"(w[24]), "+r"(w[25]), "+r"(w[26]), "+r"(w[27]), "+r"(w[28]), "+r"(w[29]), "+r"(w[30]), "+r"(w[31])
                 :: "memory");
}
FDSNN_DEV void tmem_wait64(uint32_t (&a)[32], uint32_t (&b)[32]) {
    tmem_wait32(a);
    asm volatile(""
                 : "+r"(b[0]), "+r"(b[1]), "+r"(b[2]), "+r"(b[3]), "+r"(b[4]), "+r"(b[5]), "+r"(b[6]), "+r"(b[7]),
                   "+r"(b[8]), "+r"(b[9]), "+r"(b[10]), "+r"(b[11]), "+r"(b[12]), "+r"(b[13]), "+r"(b[14]), "+r"(b[15]),
                   "+r"(b[16]), "+r"(b[17]), "+r"(b[18]), "+r"(b[19]), "+r"(b[20]), "+r"(b[21]), "+r"(b[22]), "+r"(b[23]),
                   "+r"(b[24]), "+r"(b[25]), "+r"(b[26]), "+r"(b[27]), "+r"(b[28]), "+r"(b[29]), "+r"(b[30]), "+r"(b[31])
                 :: "memory");
}
FDSNN_DEV void tmem_ld16_async(uint32_t taddr, uint32_t (&w)[16]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(w[0]), "=r"(w[1]), "=r"(w[2]), "=r"(w[3]), "=r"(w[4]), "=r"(w[5]), "=r"(w[6]), "=r"(w[7]),
          "=r"(w[8]), "=r"(w[9]), "=r"(w[10]), "=r"(w[11]), "=r"(w[12]), "=r"(w[13]), "=r"(w[14]), "=r"(w[15])
        : "r"(taddr) : "memory");
}
FDSNN_DEV void tmem_wait16(uint32_t (&w)[16]) {
    asm volatile("tcgen05.wait::ld.sync.aligned;"
                 : "+r"(w[0]), "+r"(w[1]), "+r"(w[2]), "+r"(w[3]), "+r"(w[4]), "+r"(w[5]), "+r"(w[6]), "+r"(w[7]),
                   "+r"(w[8]), "+r"(w[9]), "+r"(w[10]), "+r"(w[11]), "+r"(w[12]), "+r"(w[13]), "+r"(w[14]), "+r"(w[15])
                 :: "memory");
}
FDSNN_DEV void tmem_ld8_async(uint32_t taddr, uint32_t (&w)[8]) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(w[0]), "=r"(w[1]), "=r"(w[2]), "=r"(w[3]), "=r"(w[4]), "=r"(w[5]), "=r"(w[6]), "=r"(w[7])
                 : "r"(taddr) : "memory");
}
FDSNN_DEV void tmem_wait8(uint32_t (&w)[8]) {
    asm volatile("tcgen05.wait::ld.sync.aligned;"
                 : "+r"(w[0]), "+r"(w[1]), "+r"(w[2]), "+r"(w[3]), "+r"(w[4]), "+r"(w[5]), "+r"(w[6]), "+r"(w[7])
                 :: "memory");
}
// One double (2 words) per tcgen05.ld / st.  A 32-register (or even
// 4-register) operand tuple assembled from separately computed doubles makes
// ptxas stage every word with a copy (IMAD.MOV.U32, dispatched on the pipe
// the FP64 instructions go through); a register pair is what a DFMA reads
// and writes anyway, so pair-granular accesses need no copies at all.
FDSNN_DEV void tmem_ld2_async(uint32_t taddr, uint32_t& lo, uint32_t& hi) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x2.b32 {%0,%1}, [%2];" : "=r"(lo), "=r"(hi) : "r"(taddr) : "memory");
}
FDSNN_DEV void tmem_st2(uint32_t taddr, uint32_t lo, uint32_t hi) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x2.b32 [%0], {%1,%2};" ::"r"(taddr), "r"(lo), "r"(hi) : "memory");
}
// 32 columns starting at taddr as 16 pair loads / stores
FDSNN_DEV void tmem_ld32_pairs_async(uint32_t taddr, uint32_t (&w)[32]) {
#pragma unroll
    for (int k = 0; k < 16; ++k) tmem_ld2_async(taddr + 2 * k, w[2 * k], w[2 * k + 1]);
}
FDSNN_DEV void tmem_st_c(uint32_t taddr, double2 c) {
    tmem_st2(taddr, (uint32_t)__double2loint(c.x), (uint32_t)__double2hiint(c.x));
    tmem_st2(taddr + 2, (uint32_t)__double2loint(c.y), (uint32_t)__double2hiint(c.y));
}
// mark registers as completed by an earlier wait (no instruction emitted)
FDSNN_DEV void tmem_touch32(uint32_t (&w)[32]) {
    asm volatile(""
                 : "+r"(w[0]), "+r"(w[1]), "+r"(w[2]), "+r"(w[3]), "+r"(w[4]), "+r"(w[5]), "+r"(w[6]), "+r"(w[7]),
                   "+r"(w[8]), "+r"(w[9]), "+r"(w[10]), "+r"(w[11]), "+r"(w[12]), "+r"(w[13]), "+r"(w[14]), "+r"(w[15]),
                   "+r"(w[16]), "+r"(w[17]), "+r"(w[18]), "+r"(w[19]), "+r"(w[20]), "+r"(w[21]), "+r"(w[22]), "+r"(w[23]),
                   "+r"(w[24]), "+r"(w[25]), "+r"(w[26]), "+r"(w[27]), "+r"(w[28]), "+r"(w[29]), "+r"(w[30]), "+r"(w[31])
                 :: "memory");
}
FDSNN_DEV void tmem_st32(uint32_t taddr, const uint32_t (&w)[32]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
        "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};"
        ::"r"(taddr), "r"(w[0]), "r"(w[1]), "r"(w[2]), "r"(w[3]), "r"(w[4]), "r"(w[5]), "r"(w[6]), "r"(w[7]),
        "r"(w[8]), "r"(w[9]), "r"(w[10]), "r"(w[11]), "r"(w[12]), "r"(w[13]), "r"(w[14]), "r"(w[15]),
        "r"(w[16]), "r"(w[17]), "r"(w[18]), "r"(w[19]), "r"(w[20]), "r"(w[21]), "r"(w[22]), "r"(w[23]),
        "r"(w[24]), "r"(w[25]), "r"(w[26]), "r"(w[27]), "r"(w[28]), "r"(w[29]), "r"(w[30]), "r"(w[31]) : "memory");
}
FDSNN_DEV void put_words_c(uint32_t (&w)[32], int i, double2 c) {
    w[4 * i] = (uint32_t)__double2loint(c.x);
    w[4 * i + 1] = (uint32_t)__double2hiint(c.x);
    w[4 * i + 2] = (uint32_t)__double2loint(c.y);
    w[4 * i + 3] = (uint32_t)__double2hiint(c.y);
}
FDSNN_DEV double2 words_c(const uint32_t (&w)[32], int i) {
    return make_double2(__hiloint2double((int)w[4 * i + 1], (int)w[4 * i]),
                        __hiloint2double((int)w[4 * i + 3], (int)w[4 * i + 2]));
}

// Shared-memory matrix descriptor for tcgen05 (K-major, no swizzle): 8-row x
// 16-byte core matrices, stride `sbo` bytes between core matrices along rows.
FDSNN_DEV uint64_t smem_desc(const void* p, uint32_t lbo, uint32_t sbo) {
    uint64_t d = 0;
    d |= (uint64_t)((smem_u32(p) >> 4) & 0x3FFF);
    d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
    d |= (uint64_t)1 << 46;  // descriptor version for sm_100
    return d;
}
// smem -> TMEM copy of T rows x 16 bytes; row t lands in every TMEM lane that
// holds in-group thread t (T=32: all 4 quadrants, T=64: quadrants 0/2 and 1/3,
// T=128: lanes 0..127).
template <int T>
FDSNN_DEV void tmem_cp_rows16(uint32_t taddr, uint64_t desc) {
    if constexpr (T == 32) {
        asm volatile("tcgen05.cp.cta_group::1.32x128b.warpx4 [%0], %1;" ::"r"(taddr), "l"(desc) : "memory");
    } else if constexpr (T == 64) {
        asm volatile("tcgen05.cp.cta_group::1.64x128b.warpx2::02_13 [%0], %1;" ::"r"(taddr), "l"(desc) : "memory");
    } else {
        asm volatile("tcgen05.cp.cta_group::1.128x128b [%0], %1;" ::"r"(taddr), "l"(desc) : "memory");
    }
}
// arrive on `bar` once all prior tcgen05 async ops of this thread complete
FDSNN_DEV void tmem_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];"
                 ::"r"(smem_u32(bar)) : "memory");
}

// 1-D bulk copy global -> shared, completion counted on `bar` (TMA engine).
FDSNN_DEV void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
        ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}
