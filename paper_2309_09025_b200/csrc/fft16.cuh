// fft16.cuh — one-warp transforms of the folded negacyclic FFT (M = 512):
// 32 lanes x 16 points, Stockham passes (16, 16, 2), natural order in/out.
//
// Lane t owns points {t + 32m : m < 16}.  Pass 0 (radix 16) reads exactly
// those points; pass 2 (radix 2, 8 butterflies per lane) leaves frequencies
// {t + 32m} in registers with register index reg(m) = 2*(m % 8) + m / 8.
// Both exchanges stay inside the warp (__syncwarp), padded a + a/16 so every
// 16-byte shared access of a quarter warp hits 8 distinct bank groups.
#pragma once
#include "fft.cuh"

namespace fdsnn {
namespace w16 {

constexpr int M = 512;
constexpr int T = 32;

FDSNN_DEV int pad16(int a) { return a + (a >> 4); }
FDSNN_DEV constexpr int reg_of(int m) { return 2 * (m % 8) + m / 8; }

// 16-point DFT (kernel e^{s 2 pi i/16}), natural order in/out, as 4 x 4:
// n = 4 n1 + n2, k = k1 + 4 k2.
template <bool INV>
FDSNN_DEV void dft16(double2* v) {
    const double c1 = 0.92387953251128675613;  // cos(pi/8)
    const double s1 = 0.38268343236508977173;  // sin(pi/8)
    const double h = 0.70710678118654752440;
    double2 y[16];
#pragma unroll
    for (int n2 = 0; n2 < 4; ++n2) {
        double2 a0 = v[n2], a1 = v[4 + n2], a2 = v[8 + n2], a3 = v[12 + n2];
        dft4<INV>(a0, a1, a2, a3);
        y[4 * n2 + 0] = a0;  // k1 = 0..3
        y[4 * n2 + 1] = a1;
        y[4 * n2 + 2] = a2;
        y[4 * n2 + 3] = a3;
    }
    // twiddles w16^{n2 k1} with w16 = e^{s i pi/8}
    const double sg = INV ? -1.0 : 1.0;
    auto rot = [&](double2 z, double c, double s) {  // z * (c + i*sg*s)
        return make_double2(fma(z.x, c, -sg * s * z.y), fma(z.y, c, sg * s * z.x));
    };
    // n2 = 1: k1 = 1,2,3 -> w^1, w^2, w^3
    y[5] = rot(y[5], c1, s1);
    y[6] = rot(y[6], h, h);
    y[7] = rot(y[7], s1, c1);
    // n2 = 2: w^2, w^4, w^6
    y[9] = rot(y[9], h, h);
    y[10] = mul_si<INV>(y[10]);
    y[11] = rot(y[11], -h, h);
    // n2 = 3: w^3, w^6, w^9
    y[13] = rot(y[13], s1, c1);
    y[14] = rot(y[14], -h, h);
    y[15] = rot(y[15], -c1, -s1);
#pragma unroll
    for (int k1 = 0; k1 < 4; ++k1) {
        double2 b0 = y[k1], b1 = y[4 + k1], b2 = y[8 + k1], b3 = y[12 + k1];
        dft4<INV>(b0, b1, b2, b3);
        v[k1] = b0;
        v[k1 + 4] = b1;
        v[k1 + 8] = b2;
        v[k1 + 12] = b3;
    }
}

// pass 0 (NS=1, R=16): in = own points (register m), out to position 16t + r
FDSNN_DEV void store0(const double2 (&v)[16], int t, double2* buf) {
#pragma unroll
    for (int r = 0; r < 16; ++r) buf[pad16(16 * t + r)] = v[r];
}
// pass 1 (NS=16, R=16): in data[t + 32r]
FDSNN_DEV void load1(double2 (&v)[16], int t, const double2* buf) {
#pragma unroll
    for (int r = 0; r < 16; ++r) v[r] = buf[pad16(t + 32 * r)];
}
FDSNN_DEV void store1(const double2 (&v)[16], int t, double2* buf) {
    const int base = (t / 16) * 256 + (t % 16);
#pragma unroll
    for (int r = 0; r < 16; ++r) buf[pad16(base + 16 * r)] = v[r];
}
// pass 2 (NS=256, R=2): butterfly s uses data[t + 32s + 256r], r = 0,1 -> v[2s + r]
FDSNN_DEV void load2(double2 (&v)[16], int t, const double2* buf) {
#pragma unroll
    for (int s = 0; s < 8; ++s)
#pragma unroll
        for (int r = 0; r < 2; ++r) v[2 * s + r] = buf[pad16(t + 32 * s + 256 * r)];
}

// twiddle sources for a lane: pass 1 w256^{(t%16) r}, r = 1..15 (15 values),
// pass 2 w512^{t + 32 s}, s = 0..7 (8 values).
template <bool INV>
FDSNN_DEV void pass1(double2 (&v)[16], const double2 (&w)[16]) {
#pragma unroll
    for (int r = 1; r < 16; ++r) v[r] = INV ? cmulc(v[r], w[r - 1]) : cmul(v[r], w[r - 1]);
    dft16<INV>(v);
}
template <bool INV>
FDSNN_DEV void pass2(double2 (&v)[16], const double2 (&w)[8]) {
#pragma unroll
    for (int s = 0; s < 8; ++s) {
        const double2 b = INV ? cmulc(v[2 * s + 1], w[s]) : cmul(v[2 * s + 1], w[s]);
        const double2 a = v[2 * s];
        v[2 * s] = cadd(a, b);
        v[2 * s + 1] = csub(a, b);
    }
}

// Inverse-transform input: forward outputs sit at reg_of(m); pass 0 wants m.
FDSNN_DEV void to_natural(double2 (&v)[16]) {
    double2 tmp[16];
#pragma unroll
    for (int m = 0; m < 16; ++m) tmp[m] = v[reg_of(m)];
#pragma unroll
    for (int m = 0; m < 16; ++m) v[m] = tmp[m];
}

}  // namespace w16
}  // namespace fdsnn
