// pbs.cuh — programmable bootstrapping: modulus switch, accumulator init,
// GINX blind rotation, sample extract.  Key switching is keyswitch.cuh.
//
// Reference semantics (all bit-exact):
//   bootstrap_batch      bootstrap.py:517-534
//   rescale              ring.py:56-67   (a2N, b2N (+N//p half-slot, :526))
//   accumulator init     bootstrap.py:527-529, monomial_rotate_raw ring.py:226-242
//   CMux step i          _fold_twist_kernel bootstrap.py:386-423,
//                        einsum MAC :472, _untwist_round_add_kernel :425-442
//   sample extract       bootstrap.py:484-488
//
// Work decomposition: one group of T = M/8 threads owns one accumulator
// (2 x N int32 in shared memory) for all n CMux steps; G groups per CTA.
// Per step and accumulator: 2L forward transforms of the signed gadget digits
// of (X^k - 1)*ACC, a register-resident MAC against the Fourier-domain key
// slice, 2 inverse transforms, round and add back.  The accumulator never
// leaves shared memory until the final sample extraction.
#pragma once
#include "fft.cuh"

namespace fdsnn {

struct PbsArgs {
    DevParams prm;
    // input mode A: LWE rows
    const uint32_t* in;    // count x stride (may be null in mode B)
    const uint32_t* in2;   // optional second operand added to `in` (LIF charge)
    int64_t count;         // rows per LUT
    int nlut;              // virtual ciphertexts = nlut * count
    const int32_t* lut[4]; // device test polynomials (N residues)
    uint32_t in_boff[4];   // added to b before the modulus switch (mod q)
    // input mode B: raw accumulators + rotation indices (blind_rotate_batch)
    int32_t* acc_io;       // count x 2 x N
    const int32_t* a2N_in; // count x n
    // key
    const double2* bsk;    // (n, 2L, 2, M) Fourier-domain RGSW rows
    // tables (global, copied to smem): W[M] = e^{2 pi i k/M}, twist[M], untw[M]=conj(twist)/M
    const double2* tables;
    // output mode A: extracted z-LWE rows (virtual ct v at v*ext_stride)
    uint32_t* ext_out;
    unsigned long long* margin;  // optional max |x - round(x)| (as double bits)
};

template <int M>
struct PbsShape {
    static constexpr int T = M / 8;
    static constexpr int PADM = M + M / 8;
};

// shared-memory bytes for G groups
template <int M>
__host__ __device__ constexpr size_t pbs_smem_bytes(int G, int N, int n) {
    return (size_t)3 * M * sizeof(double2)                               // W, twist, untw
           + (size_t)G * (2 * PbsShape<M>::PADM * sizeof(double2)       // exchange buffers
                          + 2 * (size_t)N * sizeof(int32_t)             // accumulator
                          + (((size_t)n * sizeof(uint16_t) + 15) & ~(size_t)15));  // a2N
}

template <int M, int G, bool MODE_RAW, bool TRACK_MARGIN>
__global__ void __launch_bounds__(G * (M / 8))
pbs_blind_rotate_kernel(const PbsArgs args) {
    constexpr int T = M / 8;
    constexpr int PADM = PbsShape<M>::PADM;
    const DevParams& prm = args.prm;
    const int N = 2 * M;
    const int n = prm.n;
    const int L = prm.L;
    const uint32_t qmask = prm.qmask;
    const int log2_2N = __ffs(2 * N) - 1;

    extern __shared__ __align__(16) unsigned char smem_raw[];
    double2* W = reinterpret_cast<double2*>(smem_raw);
    double2* twist = W + M;
    double2* untw = twist + M;
    unsigned char* gbase = reinterpret_cast<unsigned char*>(untw + M);
    const size_t gbytes = 2 * PADM * sizeof(double2) + 2 * (size_t)N * sizeof(int32_t) +
                          (((size_t)n * sizeof(uint16_t) + 15) & ~(size_t)15);

    for (int k = threadIdx.x; k < 3 * M; k += blockDim.x) W[k] = args.tables[k];

    const int g = threadIdx.x / T;
    const int t = threadIdx.x % T;
    unsigned char* mine = gbase + g * gbytes;
    double2* buf0 = reinterpret_cast<double2*>(mine);
    double2* buf1 = buf0 + PADM;
    int32_t* acc = reinterpret_cast<int32_t*>(buf1 + PADM);  // [2][N]
    uint16_t* a2N = reinterpret_cast<uint16_t*>(acc + 2 * N);
    __syncthreads();

    const int64_t V = (int64_t)args.nlut * args.count;
    const int64_t v = (int64_t)blockIdx.x * G + g;
    if (v >= V) return;  // only group barriers below
    const GroupSync gs{1 + g, T};

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
            acc[j] = 0;
            const int src = (j + (int)b2N) & (2 * N - 1);
            const int32_t val = lut[src & (N - 1)];
            acc[N + j] = (int32_t)((uint32_t)(src >= N ? -val : val) & qmask);
        }
    } else {
        const int32_t* a_src = args.acc_io + v * 2 * N;
        for (int j = t; j < 2 * N; j += T) acc[j] = (int32_t)((uint32_t)a_src[j] & qmask);
        const int32_t* k_src = args.a2N_in + v * n;
        for (int i = t; i < n; i += T) a2N[i] = (uint16_t)(k_src[i] & (2 * N - 1));
    }
    gs.sync();

    // per-thread constant tables for its 8 points p_r = t + r*T
    const int bg = prm.bg_log;
    const int32_t halfB1 = (1 << (bg - 1)) - 1;  // B/2 - 1
    const int32_t bmask = (1 << bg) - 1;
    int ex = 0;
    double err_max = 0.0;

    for (int i = 0; i < n; ++i) {
        const int k = a2N[i];
        if (k == 0) continue;  // X^0*ACC - ACC = 0: the step is the identity
        double2 O0[8], O1[8];
#pragma unroll
        for (int r = 0; r < 8; ++r) O0[r] = O1[r] = make_double2(0.0, 0.0);

        const double2* key_i = args.bsk + (size_t)i * (2 * L) * 2 * M;
        for (int c = 0; c < 2; ++c) {
            const int32_t* a = acc + c * N;
            int32_t xlo[8], xhi[8];
#pragma unroll
            for (int r = 0; r < 8; ++r) {
#pragma unroll
                for (int half = 0; half < 2; ++half) {
                    const int jj = t + r * T + half * M;
                    const int s = (jj - k) & (2 * N - 1);
                    const uint32_t val = (s >= N) ? (uint32_t)(-a[s - N]) : (uint32_t)a[s];
                    const uint32_t d = (val - (uint32_t)a[jj]) & qmask;
                    const int32_t xc = center_q(d, prm.log2q);
                    if (half == 0) xlo[r] = xc; else xhi[r] = xc;
                }
            }
            for (int lvl = 0; lvl < L; ++lvl) {
                double2 vv[8];
#pragma unroll
                for (int r = 0; r < 8; ++r) {
                    const int32_t d1 = ((xlo[r] + halfB1) & bmask) - halfB1;
                    const int32_t d2 = ((xhi[r] + halfB1) & bmask) - halfB1;
                    xlo[r] = (xlo[r] - d1) >> bg;
                    xhi[r] = (xhi[r] - d2) >> bg;
                    vv[r] = cmul(make_double2((double)d1, (double)d2), twist[t + r * T]);
                }
                fft_group<M, false>(vv, t, W, buf0, buf1, ex, gs);
                const double2* kd = key_i + (size_t)(c * L + lvl) * 2 * M;
#pragma unroll
                for (int r = 0; r < 8; ++r) {
                    const double2 k0 = __ldg(kd + t + r * T);
                    const double2 k1 = __ldg(kd + M + t + r * T);
                    cmac(O0[r], vv[r], k0);
                    cmac(O1[r], vv[r], k1);
                }
            }
        }
        fft_group<M, true>(O0, t, W, buf0, buf1, ex, gs);
        fft_group<M, true>(O1, t, W, buf0, buf1, ex, gs);
#pragma unroll
        for (int r = 0; r < 8; ++r) {
            const int p = t + r * T;
            const double2 uw = untw[p];
            const double2 z0 = cmul(O0[r], uw);
            const double2 z1 = cmul(O1[r], uw);
            const long long r00 = round_half_away(z0.x), r01 = round_half_away(z0.y);
            const long long r10 = round_half_away(z1.x), r11 = round_half_away(z1.y);
            if constexpr (TRACK_MARGIN) {
                err_max = fmax(err_max, fabs(z0.x - (double)r00));
                err_max = fmax(err_max, fabs(z0.y - (double)r01));
                err_max = fmax(err_max, fabs(z1.x - (double)r10));
                err_max = fmax(err_max, fabs(z1.y - (double)r11));
            }
            acc[p] = (int32_t)(((uint32_t)acc[p] + (uint32_t)r00) & qmask);
            acc[p + M] = (int32_t)(((uint32_t)acc[p + M] + (uint32_t)r01) & qmask);
            acc[N + p] = (int32_t)(((uint32_t)acc[N + p] + (uint32_t)r10) & qmask);
            acc[N + p + M] = (int32_t)(((uint32_t)acc[N + p + M] + (uint32_t)r11) & qmask);
        }
        gs.sync();
    }
    if constexpr (TRACK_MARGIN) {
        if (args.margin) atomicMax(args.margin, (unsigned long long)__double_as_longlong(err_max));
    }

    if constexpr (MODE_RAW) {
        int32_t* a_dst = args.acc_io + v * 2 * N;
        for (int j = t; j < 2 * N; j += T) a_dst[j] = acc[j];
    } else {
        // sample extract (bootstrap.py:484-488): (a_0, -a_{N-1}, ..., -a_1), b = acc_b[0]
        uint32_t* out = args.ext_out + v * prm.ext_stride;
        for (int j = t; j < N; j += T) {
            const uint32_t a = (j == 0) ? (uint32_t)acc[0] : ((uint32_t)(-acc[N - j]) & qmask);
            out[j] = a;
        }
        if (t == 0) out[N] = (uint32_t)acc[N];
    }
}

// Fourier transform of the bootstrapping key rows (BootstrapKey.__init__,
// bootstrap.py:319-323): centred residues -> fold, twist, forward DFT.
// One group of T threads per polynomial; G polys per CTA.
template <int M, int G>
__global__ void __launch_bounds__(G * (M / 8))
bsk_forward_kernel(const int64_t* __restrict__ rows, int64_t npoly, int log2q,
                   const double2* __restrict__ tables, double2* __restrict__ out) {
    constexpr int T = M / 8;
    constexpr int PADM = PbsShape<M>::PADM;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    double2* W = reinterpret_cast<double2*>(smem_raw);
    double2* twist = W + M;
    double2* bufs = twist + 2 * M;  // skip untw
    for (int k = threadIdx.x; k < 3 * M; k += blockDim.x) W[k] = tables[k];
    __syncthreads();
    const int g = threadIdx.x / T, t = threadIdx.x % T;
    const int64_t poly = (int64_t)blockIdx.x * G + g;
    if (poly >= npoly) return;
    double2* buf0 = bufs + g * 2 * PADM;
    double2* buf1 = buf0 + PADM;
    const GroupSync gs{1 + g, T};
    const int64_t* src = rows + poly * 2 * M;
    const int64_t qm = (1ll << log2q) - 1;
    double2 vv[8];
#pragma unroll
    for (int r = 0; r < 8; ++r) {
        const int p = t + r * T;
        const int32_t lo = center_q((uint32_t)(src[p] & qm), log2q);
        const int32_t hi = center_q((uint32_t)(src[p + M] & qm), log2q);
        vv[r] = cmul(make_double2((double)lo, (double)hi), twist[p]);
    }
    int ex = 0;
    fft_group<M, false>(vv, t, W, buf0, buf1, ex, gs);
#pragma unroll
    for (int r = 0; r < 8; ++r) out[poly * M + t + r * T] = vv[r];
}

}  // namespace fdsnn
