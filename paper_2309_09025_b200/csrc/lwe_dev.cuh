// lwe_dev.cuh — client-side LWE encryption / decryption on the device
// (SURVEY §8(f)4).  The randomness (masks A, rounded-Gaussian noise e) is
// drawn on the host by the caller's numpy Generator in the reference's order
// (lwe.py:75-87), so ciphertexts are bit-identical to the reference's; the
// device does the <A, s> inner products.
//   encrypt: b = (<A, s> + e + Delta*m) mod q                 (lwe.py:84-86)
//   decrypt: phase = centre((b - <A, s>) mod q);
//            m = round_half_away(phase*p/q) mod p -> {-p/2+1..p/2} (lwe.py:89-96)
// Inner products are exact: uint32 wrap-around arithmetic, masked to q = 2^k.
#pragma once
#include "common.cuh"

namespace fdsnn {

// one warp per ciphertext row: sum_i a_i s_i mod 2^32
FDSNN_DEV uint32_t row_dot_s(const uint32_t* __restrict__ a, const int32_t* __restrict__ s, int n, int lane) {
    uint32_t acc = 0;
    for (int i = lane; i < n; i += 32) acc += a[i] * (uint32_t)s[i];
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
    return acc;
}

// rows already hold A (masked); writes b.
__global__ void lwe_encrypt_kernel(uint32_t* __restrict__ rows, int64_t count, int stride, int n,
                                   const int32_t* __restrict__ s, const int64_t* __restrict__ e,
                                   const int64_t* __restrict__ m, uint32_t qmask, uint32_t delta) {
    const int64_t v = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) / 32;
    const int lane = threadIdx.x % 32;
    if (v >= count) return;
    uint32_t* r = rows + v * stride;
    const uint32_t dot = row_dot_s(r, s, n, lane);
    if (lane == 0) r[n] = (dot + (uint32_t)e[v] + delta * (uint32_t)m[v]) & qmask;
}

__global__ void lwe_decrypt_kernel(const uint32_t* __restrict__ rows, int64_t count, int stride, int n,
                                   const int32_t* __restrict__ s, int log2q, long long p,
                                   int64_t* __restrict__ out) {
    const int64_t v = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) / 32;
    const int lane = threadIdx.x % 32;
    if (v >= count) return;
    const uint32_t* r = rows + v * stride;
    const uint32_t dot = row_dot_s(r, s, n, lane);
    if (lane == 0) {
        const long long q = 1ll << log2q;
        const long long ph = (long long)((r[n] - dot) & (uint32_t)(q - 1));
        const long long c = ph >= q / 2 ? ph - q : ph;                  // centre (ring.py:27-33)
        const long long num = c * p;                                    // div_round_half_away(num, q)
        const long long mag = num < 0 ? -num : num;
        const long long rq = (2 * mag + q) / (2 * q);
        long long mm = num >= 0 ? rq : -rq;
        mm = ((mm % p) + p) % p;
        const long long half = p / 2;
        out[v] = ((mm + half - 1) % p) - (half - 1);
    }
}

}  // namespace fdsnn
