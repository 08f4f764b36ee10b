"""CPU oracle for the FHE-DiCSNN hot path — TEST INFRASTRUCTURE ONLY.

A plain numpy restatement of the reference algorithm (/root/reference/pkg/src/
fdsnn, cited file:line per function).  Only `tests/`, `__graft_entry__.smoke()`
and `bench.py`'s CPU-baseline leg may import this module, and only as the
checker / the timed CPU baseline — never as part of the product path.

Pinning: `tests/test_oracle_pin.py` checks every function here against golden
vectors produced by running the reference itself in the build container
(`tests/golden/make_golden.py`, fixtures under `tests/golden/`), and against
the reference's own known-answer tests.

Arithmetic notes
  * Keys and ciphertexts are int64 residues mod q (reference layout).
  * The negacyclic products use the reference's folded FFT formulation
    (ring.py:103-137): fold+twist, length-M DFT with the e^{+} kernel, MAC in
    the Fourier domain, e^{-} DFT, /M, untwist, round half away from zero.
  * Key switching and weight sums are exact int64 (the reference uses float64
    GEMMs asserted exact, bootstrap.py:311-315, network.py:416-420).
"""

from __future__ import annotations

import numpy as np

# ---------------------------------------------------------------- ring.py


def center(v, q):
    """ring.py:27-33"""
    v = np.asarray(v, dtype=np.int64)
    return np.where(v >= q // 2, v - q, v)


def round_half_away(x):
    """ring.py:36-42"""
    x = np.asarray(x)
    return np.where(x >= 0, np.floor(x + 0.5), np.ceil(x - 0.5)).astype(np.int64)


def div_round_half_away(num, den):
    """ring.py:45-53"""
    num = np.asarray(num, dtype=np.int64)
    r = (2 * np.abs(num) + den) // (2 * den)
    return np.where(num >= 0, r, -r)


def rescale(x, q1, q2):
    """ring.py:56-67 (q -> 2N modulus switch)."""
    c = center(np.asarray(x, dtype=np.int64) % q1, q1)
    if q1 >= q2:
        return div_round_half_away(c * q2, q1) % q2
    return (c * (q2 // q1)) % q2


def monomial_rotate(coeffs, k, N):
    """X^k * p(X), k per row (ring.py:226-242)."""
    k = np.asarray(k, dtype=np.int64) % (2 * N)
    src = (np.arange(N)[None, :] - k[:, None]) % (2 * N)
    sign = np.where(src >= N, -1, 1)
    coeffs = np.broadcast_to(coeffs, src.shape) if np.ndim(coeffs) == 1 else coeffs
    return sign * np.take_along_axis(coeffs, src % N, axis=-1)


class Transform:
    """Folded negacyclic transform (ring.py:103-137)."""

    def __init__(self, N):
        self.N = N
        self.M = N // 2
        k = np.arange(self.M)
        self.twist = np.exp(1j * np.pi * k / N)
        self.untwist = np.conj(self.twist)

    def forward(self, a):
        a = np.asarray(a, dtype=np.float64)
        c = (a[..., : self.M] + 1j * a[..., self.M:]) * self.twist
        return np.fft.ifft(c, axis=-1, norm="forward")  # e^{+2 pi i jk/M}, no scaling

    def inverse(self, y):
        c = np.fft.fft(y, axis=-1) / self.M * self.untwist
        return np.concatenate([c.real, c.imag], axis=-1)


def gadget_decompose(x, q, base, levels):
    """Signed digits in (-B/2, B/2], lowest first (rgsw.py:119-133)."""
    x = center(np.asarray(x, dtype=np.int64) % q, q)
    out = np.empty(x.shape[:-1] + (levels, x.shape[-1]), dtype=np.int64)
    for i in range(levels):
        d = ((x + base // 2 - 1) % base) - (base // 2 - 1)
        out[..., i, :] = d
        x = (x - d) // base
    return out


def negacyclic_mul(a, b, q):
    """Exact a*b mod (X^N + 1, q) of integer vectors (ring.py:200-207 schoolbook;
    the reference's transform path ring.py:210-223 equals it at preset sizes).
    int64 convolution: exact while N*max|a|*max|b| < 2^63."""
    a = center(np.asarray(a, dtype=np.int64) % q, q)
    b = np.asarray(b, dtype=np.int64)
    N = a.shape[-1]
    full = np.convolve(a, b)
    out = full[:N].copy()
    out[: len(full) - N] -= full[N:]
    return out % q


def external_product(ct_a, ct_b, rows_a, rows_b, q, base, levels):
    """RLWE x RGSW (rgsw.py:179-193): digits of (a, b) stacked (2l, N), then
    sum_d digit_d * row_d for the a and the b component, mod q."""
    digits = np.concatenate([gadget_decompose(np.asarray(ct_a)[None], q, base, levels)[0],
                             gadget_decompose(np.asarray(ct_b)[None], q, base, levels)[0]])
    out_a = sum(negacyclic_mul(r, d, q) for r, d in zip(rows_a, digits)) % q
    out_b = sum(negacyclic_mul(r, d, q) for r, d in zip(rows_b, digits)) % q
    return out_a, out_b


# --------------------------------------------------------- bootstrap.py


class OracleKey:
    """Keys as plain arrays: rows (n,2l,2,N), ksk_A (N*ks_l, n), ksk_b."""

    def __init__(self, prm, rows, ksk_A, ksk_b):
        self.prm = prm  # dict: n q N p Bg l ks_base ks_l
        self.rows = np.asarray(rows, dtype=np.int64)
        self.ksk_A = np.asarray(ksk_A, dtype=np.int64)
        self.ksk_b = np.asarray(ksk_b, dtype=np.int64)
        self.tr = Transform(prm["N"])
        # BootstrapKey._ek_fft (bootstrap.py:125-130)
        self.ek_f = self.tr.forward(center(self.rows, prm["q"]))


def params_dict(p):
    """Plain-dict view of an FheParams-like object."""
    return dict(n=p.n, q=p.q, N=p.N, p=p.p, Bg=p.gadget.base, l=p.gadget.levels,
                ks_base=p.ks_base, ks_l=p.ks_levels)


def program_table(pos_values, p):
    """make_program (bootstrap.py:74-87): antisymmetric fill, centred table."""
    half = p // 2
    t = np.concatenate([np.asarray(pos_values, np.int64), -np.asarray(pos_values, np.int64)]) % p
    return ((t + half - 1) % p) - (half - 1)


def test_polynomial(table, prm):
    """bootstrap.py:90-96"""
    N, p, q = prm["N"], prm["p"], prm["q"]
    slots = (np.arange(N) * p) // (2 * N)
    return ((q // p) * table[slots]) % q


test_polynomial.__test__ = False


def blind_rotate(acc, a2N, key: OracleKey):
    """GINX CMux chain, numpy restatement of bootstrap.py:169-190 / 445-475."""
    prm = key.prm
    q, N, Bg, l = prm["q"], prm["N"], prm["Bg"], prm["l"]
    acc = np.array(acc, dtype=np.int64)
    B = acc.shape[0]
    j = np.arange(N)
    for i in range(a2N.shape[1]):
        k = np.asarray(a2N[:, i], dtype=np.int64)
        if not k.any():
            continue
        src = (j[None, :] - k[:, None]) % (2 * N)
        sign = np.where(src >= N, -1, 1)[:, None, :]
        idx = np.broadcast_to((src % N)[:, None, :], acc.shape)
        diff = (sign * np.take_along_axis(acc, idx, axis=2) - acc) % q
        dig = gadget_decompose(diff, q, Bg, l).reshape(B, 2 * l, N)  # row c*l+lvl
        dig_f = key.tr.forward(dig)
        prod = np.einsum("bdm,dom->bom", dig_f, key.ek_f[i])
        acc = (acc + round_half_away(key.tr.inverse(prod))) % q
    return acc


def sample_extract(acc):
    """bootstrap.py:291-295"""
    a = acc[:, 0, :]
    return np.concatenate([a[:, :1], -a[:, -1:0:-1]], axis=1), acc[:, 1, 0].copy()


def key_switch(ea, eb, key: OracleKey):
    """bootstrap.py:303-316 with exact int64 sums."""
    prm = key.prm
    q = prm["q"]
    dig = gadget_decompose(ea, q, prm["ks_base"], prm["ks_l"])  # (B, l, N)
    flat = np.swapaxes(dig, -2, -1).reshape(ea.shape[0], -1)   # index j*l + i
    out_a = (-(flat @ key.ksk_A)) % q
    out_b = (np.asarray(eb, dtype=np.int64) - flat @ key.ksk_b) % q
    return out_a, out_b


def bootstrap_batch(table, A, b, key: OracleKey):
    """bootstrap.py:324-341"""
    prm = key.prm
    N, p, q = prm["N"], prm["p"], prm["q"]
    a2N = rescale(A, q, 2 * N)
    b2N = (rescale(b, q, 2 * N) + N // p) % (2 * N)
    v = test_polynomial(table, prm)
    acc_b = monomial_rotate(v, (-b2N) % (2 * N), N) % q
    acc = np.stack([np.zeros_like(acc_b), acc_b], axis=1)
    acc = blind_rotate(acc, a2N, key)
    ea, eb = sample_extract(acc)
    return key_switch(ea, eb, key)


# ------------------------------------------------------------ neuron.py


def fire_table(p):
    """g_fire (neuron.py:122-124)"""
    return program_table(np.ones(p // 2, dtype=np.int64), p)


def reset_table(v_th_hat, leak_num, leak_den, p):
    """g_reset (neuron.py:127-133)"""
    m = np.arange(p // 2)
    leak = div_round_half_away(m * leak_num, leak_den)
    return program_table(np.where(m >= v_th_hat, 0, leak), p)


def lif_step(vA, vb, iA, ib, v_th_hat, leak_num, leak_den, key: OracleKey):
    """fhe_lif_step_batch (neuron.py:160-172): charge, fire (+shifts), reset."""
    prm = key.prm
    q, p = prm["q"], prm["p"]
    delta = q // p
    hA = (np.asarray(vA) + np.asarray(iA)) % q
    hb = (np.asarray(vb) + np.asarray(ib)) % q
    sA, sb = bootstrap_batch(fire_table(p), hA, (hb - delta * v_th_hat) % q, key)
    sb = (sb + delta) % q
    nA, nb = bootstrap_batch(reset_table(v_th_hat, leak_num, leak_den, p), hA, hb, key)
    return sA, sb, nA, nb


def plain_lif_step(v, i, v_th_hat, leak_num, leak_den):
    """plain_lif_step_batch (neuron.py:107-119) without the strict range check."""
    h = np.asarray(v, dtype=np.int64) + np.asarray(i, dtype=np.int64)
    fired = h >= v_th_hat
    leak = div_round_half_away(h * leak_num, leak_den)
    return np.where(fired, 2, 0), np.where(fired | (h <= 0), 0, leak)


def twin_lif_step(v, i, v_th_hat, leak_num, leak_den, p):
    """Mod-p plaintext twin of the encrypted step: what the
    ciphertexts decrypt to, including deterministic wrap-around."""
    half = p // 2
    h = ((np.asarray(v) + np.asarray(i) + half - 1) % p) - (half - 1)  # centred Z_p
    ft = fire_table(p)
    rt = reset_table(v_th_hat, leak_num, leak_den, p)
    spike = ((ft[(h - v_th_hat) % p] + 1 + half - 1) % p) - (half - 1)
    return spike, rt[h % p]


# ------------------------------------------------------------ network.py


def layer_forward(Mx, A, b, q):
    """network.py:409-421 with exact int64 products."""
    Mx = np.asarray(Mx, dtype=np.int64)
    return (Mx @ np.asarray(A, np.int64)) % q, (Mx @ np.asarray(b, np.int64)) % q


def infer(A, b, layers, key: OracleKey, T, observer=None):
    """network.infer (network.py:459-491) on one image; layers are
    ("weight", matrix) or ("spike", v_th_hat, leak_num, leak_den)."""
    q, n = key.prm["q"], key.prm["n"]
    states = {}
    scores = None
    for t in range(T):
        xA, xb = np.asarray(A, np.int64), np.asarray(b, np.int64)
        for li, layer in enumerate(layers):
            if layer[0] == "weight":
                xA, xb = layer_forward(layer[1], xA, xb, q)
            else:
                cnt = len(xb)
                vA, vb = states.get(li, (np.zeros((cnt, n), np.int64), np.zeros(cnt, np.int64)))
                sA, sb, nA, nb = lif_step(vA, vb, xA, xb, *layer[1:], key)
                states[li] = (nA, nb)
                xA, xb = sA, sb
                if observer is not None:
                    observer(li, t, xA, xb)
        scores = (xA, xb) if scores is None else ((scores[0] + xA) % q, (scores[1] + xb) % q)
    return scores


def twin_infer(x, layers, T, p):
    """Mod-p twin of `infer` on decrypted values (x: input messages)."""
    half = p // 2

    def cz(v):
        return ((np.asarray(v) + half - 1) % p) - (half - 1)

    states = {}
    score = None
    spikes_log = []
    for t in range(T):
        v = np.asarray(x, dtype=np.int64)
        for li, layer in enumerate(layers):
            if layer[0] == "weight":
                v = cz(np.asarray(layer[1], np.int64) @ v)
            else:
                st = states.get(li, np.zeros(len(v), np.int64))
                s, nv = twin_lif_step(st, v, *layer[1:], p)
                states[li] = nv
                v = s
                spikes_log.append((li, t, v.copy()))
        score = v if score is None else cz(score + v)
    return score, spikes_log


def plain_infer(x, layers, T, p=None):
    """oracle.plain_infer (oracle.py:44-78): exact integer forward (no wrap)
    on the quantized input x.  Returns (scores, per-spiking-layer spike counts
    summed over T, number of out-of-range charges at p)."""
    states, counts = {}, {}
    scores = None
    overflow = 0
    for t in range(T):
        v = np.asarray(x, dtype=np.int64)
        for li, layer in enumerate(layers):
            if layer[0] == "weight":
                v = np.asarray(layer[1], np.int64) @ v
            else:
                vth, ln, ld = layer[1:]
                st = states.get(li, np.zeros(len(v), np.int64))
                if p is not None:
                    h = st + v
                    overflow += int(np.count_nonzero((h < vth - p // 2) | (h >= p // 2)))
                s, nv = plain_lif_step(st, v, vth, ln, ld)
                states[li] = nv
                counts[li] = counts.get(li, 0) + s // 2
                v = s
        scores = v if scores is None else scores + v
    return scores, [counts[k] for k in sorted(counts)], overflow


# --------------------------------------------------------- keygen / lwe.py


def lwe_decrypt(A, b, s, q, p):
    """lwe.py:90-96"""
    phase = center((np.asarray(b, np.int64) - np.asarray(A, np.int64) @ s) % q, q)
    m = div_round_half_away(phase * p, q) % p
    half = p // 2
    return ((m + half - 1) % p) - (half - 1)


# ------------------------------------------------- compiled CPU baseline path
# The reference accelerates the two elementwise stages of its CMux step with
# numba (bootstrap.py:193-249).  The CPU-baseline leg of bench.py times the
# same algorithm with the same library stack, so this module provides numba
# versions of those two stages (written for this oracle); `blind_rotate_fast`
# is checked bit-exact against `blind_rotate` in tests/test_oracle_pin.py.

try:  # pragma: no cover - optional
    import numba as _nb
except Exception:  # pragma: no cover
    _nb = None

if _nb is not None:

    @_nb.njit(cache=True)
    def _digits_twisted(acc, k, twist, out, q, base, levels):
        # powers of two throughout: reductions are masks, digit division a shift
        B, _, N = acc.shape
        M = N // 2
        qm, half_q, m2n = q - 1, q // 2, 2 * N - 1
        bm, hb = base - 1, base // 2 - 1
        shift = 0
        while (1 << shift) < base:
            shift += 1
        for bi in range(B):
            kk = k[bi]
            for c in range(2):
                a = acc[bi, c]
                for j in range(M):
                    s0 = (j - kk) & m2n
                    v0 = -a[s0 - N] if s0 >= N else a[s0]
                    x0 = (v0 - a[j]) & qm
                    if x0 >= half_q:
                        x0 -= q
                    s1 = (j + M - kk) & m2n
                    v1 = -a[s1 - N] if s1 >= N else a[s1]
                    x1 = (v1 - a[j + M]) & qm
                    if x1 >= half_q:
                        x1 -= q
                    tw = twist[j]
                    for lv in range(levels):
                        d0 = ((x0 + hb) & bm) - hb
                        d1 = ((x1 + hb) & bm) - hb
                        x0 = (x0 - d0) >> shift
                        x1 = (x1 - d1) >> shift
                        out[bi, c * levels + lv, j] = complex(d0, d1) * tw

    @_nb.njit(cache=True)
    def _round_add(acc, y, untw, q):
        B, _, N = acc.shape
        M = N // 2
        qm = q - 1
        for bi in range(B):
            for c in range(2):
                for j in range(M):
                    z = y[bi, c, j] * untw[j]
                    r0 = np.floor(z.real + 0.5) if z.real >= 0 else np.ceil(z.real - 0.5)
                    r1 = np.floor(z.imag + 0.5) if z.imag >= 0 else np.ceil(z.imag - 0.5)
                    acc[bi, c, j] = (acc[bi, c, j] + np.int64(r0)) & qm
                    acc[bi, c, j + M] = (acc[bi, c, j + M] + np.int64(r1)) & qm


def blind_rotate_fast(acc, a2N, key: OracleKey):
    """Same CMux chain as `blind_rotate`, numba-compiled digit/round stages."""
    if _nb is None:
        return blind_rotate(acc, a2N, key)
    prm = key.prm
    q, N, Bg, l = prm["q"], prm["N"], prm["Bg"], prm["l"]
    M = N // 2
    acc = np.array(acc, dtype=np.int64)
    B = acc.shape[0]
    dig = np.empty((B, 2 * l, M), dtype=np.complex128)
    untw = key.tr.untwist / M
    for i in range(a2N.shape[1]):
        k = np.ascontiguousarray(a2N[:, i], dtype=np.int64)
        if not k.any():
            continue
        _digits_twisted(acc, k, key.tr.twist, dig, q, Bg, l)
        dig_f = np.fft.ifft(dig, axis=-1, norm="forward")
        prod = np.einsum("bdm,dom->bom", dig_f, key.ek_f[i])
        _round_add(acc, np.fft.fft(prod, axis=-1), untw, q)
    return acc


def key_switch_fast(ea, eb, key: OracleKey):
    """`key_switch` as float64 BLAS products, exact below 2^52 like the
    reference's own assertion (bootstrap.py:311-315)."""
    prm = key.prm
    q = prm["q"]
    if not hasattr(key, "_ksk_Af"):
        key._ksk_Af = key.ksk_A.astype(np.float64)
        key._ksk_bf = key.ksk_b.astype(np.float64)
    dig = gadget_decompose(ea, q, prm["ks_base"], prm["ks_l"])
    flat = np.swapaxes(dig, -2, -1).reshape(ea.shape[0], -1).astype(np.float64)
    out_a = (-(flat @ key._ksk_Af)).astype(np.int64) % q
    out_b = (np.asarray(eb, dtype=np.int64) - (flat @ key._ksk_bf).astype(np.int64)) % q
    return out_a, out_b


def lif_step_fast(vA, vb, iA, ib, v_th_hat, leak_num, leak_den, key: OracleKey):
    """`lif_step` with the compiled blind rotation and BLAS key switch (CPU
    baseline leg of bench.py; bit-exact with `lif_step`)."""
    global blind_rotate, key_switch
    saved = blind_rotate, key_switch
    try:
        blind_rotate, key_switch = blind_rotate_fast, key_switch_fast  # looked up at call time
        return lif_step(vA, vb, iA, ib, v_th_hat, leak_num, leak_den, key)
    finally:
        blind_rotate, key_switch = saved
