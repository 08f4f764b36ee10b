"""Numpy model of the "layout 2" 512-point transform (design aid for a
blind-rotation variant whose first forward exchange is warp-local):

  fA  (coefficients): thread t = 32*t5 + l holds n = 64 r + 8 (l >> 2) + 4 t5 + (l & 3)
  pass 0: dft8 over r -> k0
  E1  warp-local: two TMEM hops (16x256b, then 16x64b) or a warp-local smem transpose
  pass 1: twiddle w64^(n1 k0), dft8 over n1 -> k1; twiddle w512^(n0 (k0 + 8 k1))
  E2  cross-warp smem: thread t'' = 8 k1 + k0 gets the 8 values n0
  pass 2: dft8 over n0 -> k2: natural order X[t'' + 64 k2]

Checks the transform against numpy and the shared-memory bank pattern of E2
(and of the smem version of E1).  Prints the fB layout (per lane: k0, n0 and
the register -> n1 map) the kernel tables are built from.
"""
import numpy as np

W8 = np.exp(2j * np.pi * np.arange(8)[:, None] * np.arange(8)[None, :] / 8)  # forward e^{+}


def dft8(v):
    return W8 @ v


def fa_index(t, r):
    t5, l = t >> 5, t & 31
    return 64 * r + 8 * (l >> 2) + 4 * t5 + (l & 3)


def hop_H(lanes):
    """lanes: (32, 8) complex per warp (thread = lane, 8 registers).
    32x32b store (re of complex c at dcol c, im at 8 + c) + 16x256b reload:
    thread i gets complex c = 4k + (i & 3) of lane 16 Lh + 8 hh + (i >> 2),
    register 4 Lh + 2 k + hh."""
    out = np.zeros_like(lanes)
    src = np.zeros((32, 8, 2), dtype=int)
    for i in range(32):
        for Lh in range(2):
            for k in range(2):
                for hh in range(2):
                    lane = 16 * Lh + 8 * hh + (i >> 2)
                    c = 4 * k + (i & 3)
                    out[i, 4 * Lh + 2 * k + hh] = lanes[lane, c]
                    src[i, 4 * Lh + 2 * k + hh] = (lane, c)
    return out, src


def hop_G(lanes):
    """32x32b store (lo/hi words of double dd in cols dd / 16 + dd; re of
    complex c = double c, im = double 8 + c) + 16x64b reload: thread i gets
    double dd = ((i >> 1) & 1) + 2 j from lane (i >> 2) + 8 (i & 1) + 16 Lh.
    Complexes: c = 2 j' + ((i >> 1) & 1), j' < 4, register 4 Lh + j'."""
    out = np.zeros_like(lanes)
    for i in range(32):
        b = (i >> 1) & 1
        for Lh in range(2):
            lane = (i >> 2) + 8 * (i & 1) + 16 * Lh
            for jp in range(4):
                out[i, 4 * Lh + jp] = lanes[lane, 2 * jp + b]
    return out


def main():
    rng = np.random.default_rng(0)
    x = rng.normal(size=512) + 1j * rng.normal(size=512)
    want = np.array([np.sum(x * np.exp(2j * np.pi * np.arange(512) * k / 512)) for k in range(512)])

    # tags: which (n1, n0) / k0 each value carries, to derive layouts
    v = np.zeros((64, 8), complex)
    n_of = np.zeros((64, 8), int)
    for t in range(64):
        for r in range(8):
            v[t, r] = x[fa_index(t, r)]
            n_of[t, r] = fa_index(t, r)
    # pass 0: dft8 over r (n2) -> register k0
    for t in range(64):
        v[t] = dft8(v[t])
    n1_of = lambda t: (t & 31) >> 2
    n0_of = lambda t: 4 * (t >> 5) + (t & 3)
    tag = np.zeros((64, 8, 3), int)  # (k0, n1, n0)
    for t in range(64):
        for k0 in range(8):
            tag[t, k0] = (k0, n1_of(t), n0_of(t))

    # E1 by two hops per warp; register renaming between hops chosen so
    # that H's output register (Lh, k, hh) feeds G's complex index c:
    # G moves c bit 0 into a thread bit and keeps (c2, c1) in registers.
    # H register 4 Lh + 2 k + hh holds lane bits (l4 = Lh, l3 = hh) and
    # k0 bit 2 (= k); we want k0 bit 2 -> thread, l4 l3 (n1 bits) -> registers:
    # c = 2 * (2 Lh + hh) + k  (c0 = k0 bit 2, c2 c1 = Lh hh).
    ren = [None] * 8
    for Lh in range(2):
        for k in range(2):
            for hh in range(2):
                ren[2 * (2 * Lh + hh) + k] = 4 * Lh + 2 * k + hh
    vb = np.zeros_like(v)
    tb = np.zeros_like(tag)
    for w in range(2):
        lanes = v[32 * w:32 * w + 32]
        ltag = tag[32 * w:32 * w + 32]
        h, _ = hop_H(lanes)
        htag = np.zeros_like(ltag)
        for i in range(32):
            for Lh in range(2):
                for k in range(2):
                    for hh in range(2):
                        htag[i, 4 * Lh + 2 * k + hh] = ltag[16 * Lh + 8 * hh + (i >> 2), 4 * k + (i & 3)]
        h2 = h[:, ren]
        ht2 = htag[:, ren]
        g = hop_G(h2)
        gtag = np.zeros_like(ht2)
        for i in range(32):
            b = (i >> 1) & 1
            for Lh in range(2):
                lane = (i >> 2) + 8 * (i & 1) + 16 * Lh
                for jp in range(4):
                    gtag[i, 4 * Lh + jp] = ht2[lane, 2 * jp + b]
        vb[32 * w:32 * w + 32] = g
        tb[32 * w:32 * w + 32] = gtag
    # fB: every thread holds one (k0, n0) and n1 = 0..7 in some register order
    fb = []
    for t in range(64):
        k0s, n0s = set(tb[t, :, 0]), set(tb[t, :, 2])
        assert len(k0s) == 1 and len(n0s) == 1, (t, tb[t])
        order = list(tb[t, :, 1])
        assert sorted(order) == list(range(8)), (t, order)
        fb.append((k0s.pop(), n0s.pop(), order))
    orders = {tuple(o) for _, _, o in fb}
    print("E1 by hops OK; register->n1 maps used:", orders)
    # put registers in natural n1 order
    for t in range(64):
        perm = np.argsort(fb[t][2])
        vb[t] = vb[t][perm]
    # pass 1 + twiddles
    for t in range(64):
        k0, n0, _ = fb[t]
        vb[t] = vb[t] * np.exp(2j * np.pi * np.arange(8) * k0 / 64)
        vb[t] = dft8(vb[t])  # -> k1
        vb[t] = vb[t] * np.exp(2j * np.pi * n0 * (k0 + 8 * np.arange(8)) / 512)
    # E2 through smem: idx = 8 (k0 + 8 k1) + n0, padded a + a / 8
    pad = lambda a: a + a // 8
    smem = np.zeros(576, complex)
    bad = 0
    for k1 in range(8):  # one STS.128 per register k1
        for w in range(2):
            for q in range(4):
                slots = [pad(8 * (fb[32 * w + 8 * q + j][0] + 8 * k1) + fb[32 * w + 8 * q + j][1]) % 8 for j in range(8)]
                bad += len(slots) - len(set(slots))
        for t in range(64):
            k0, n0, _ = fb[t]
            smem[pad(8 * (k0 + 8 * k1) + n0)] = vb[t, k1]
    print("E2 store bank conflicts (extra wavefronts):", bad)
    vc = np.zeros_like(v)
    bad = 0
    for n0 in range(8):
        for w in range(2):
            for q in range(4):
                slots = [pad(8 * (32 * w + 8 * q + j) + n0) % 8 for j in range(8)]
                bad += len(slots) - len(set(slots))
        for t in range(64):
            vc[t, n0] = smem[pad(8 * t + n0)]
    print("E2 load bank conflicts:", bad)
    for t in range(64):
        vc[t] = dft8(vc[t])  # -> k2
    got = np.zeros(512, complex)
    for t in range(64):
        for k2 in range(8):
            got[t + 64 * k2] = vc[t, k2]
    err = np.abs(got - want).max()
    print("forward transform max error:", err)
    assert err < 1e-9
    print("fB per lane (warp 0): k0, n0 =", [(fb[t][0], fb[t][1]) for t in range(32)])


if __name__ == "__main__":
    main()
