"""GPU parity of the algebra layer (ring.NegacyclicTransform, poly_mul,
poly_mul_schoolbook, rgsw.gadget_decompose, rgsw.external_product) against
the reference's own outputs (tests/golden/ring.npz) and the CPU oracle; the
semantic checks mirror the reference's test_ring.py / test_rgsw.py."""
import os

import numpy as np
import pytest

from conftest import GOLDEN, O
from paper_2309_09025_b200 import params, rgsw, ring
from paper_2309_09025_b200.errors import ParameterError

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def g():
    return np.load(os.path.join(GOLDEN, "ring.npz"))


def small_ring(p=8):
    return params.FheParams(n=4, q=1 << 12, N=64, p=p, sigma=1e-9,
                            gadget=params.GadgetParams(base=1 << 6, levels=2),
                            ks_base=8, ks_levels=4, sigma_bk=1e-9, sigma_ks=1e-9)


# FP64 transform: agreement with the reference's pocketfft to rounding
@pytest.mark.parametrize("N", [2, 8, 64, 1024, 2048])
def test_transform_matches_reference(g, N):
    tr = ring.get_transform(N)
    f = tr.forward(g[f"nt{N}_in"])
    scale = np.abs(g[f"nt{N}_fwd"]).max()
    assert f.shape == g[f"nt{N}_fwd"].shape and f.dtype == np.complex128
    assert np.abs(f - g[f"nt{N}_fwd"]).max() <= 1e-12 * scale
    inv = tr.inverse(g[f"nt{N}_fwd"])
    assert np.abs(inv - g[f"nt{N}_inv"]).max() <= 1e-9 * max(1.0, np.abs(g[f"nt{N}_inv"]).max() * 1e-3)


@pytest.mark.parametrize("N", [4, 32, 512, 4096])
def test_transform_roundtrip_and_oracle(N):
    rng = np.random.default_rng(N)
    a = rng.integers(-(1 << 20), 1 << 20, (3, N))
    tr = ring.NegacyclicTransform(N)
    f = tr.forward(a)
    want = O.Transform(N).forward(a)
    assert np.abs(f - want).max() <= 1e-12 * np.abs(want).max()
    assert np.abs(tr.inverse(f) - a).max() < 1e-6


def test_transform_product_is_exact_negacyclic_product():
    """FFT == schoolbook at DESK size (reference test_ring.py:91-110)."""
    N, q = 1024, 1 << 25
    rng = np.random.default_rng(3)
    a = rng.integers(-(1 << 24), 1 << 24, N)
    b = rng.integers(-(1 << 12), 1 << 12, N)
    tr = ring.get_transform(N)
    prod = ring.round_half_away(tr.inverse(tr.forward(a) * tr.forward(b))) % q
    assert np.array_equal(prod, O.negacyclic_mul(a, b, q))


@pytest.mark.parametrize("name", ["desk", "c4", "tiny"])
def test_poly_mul_matches_reference(g, name):
    q = int(g[f"mul_{name}_q"][0])
    a = ring.NegacyclicPoly(g[f"mul_{name}_a"], q)
    b = ring.NegacyclicPoly(g[f"mul_{name}_b"], q)
    assert np.array_equal(ring.poly_mul(a, b).coeffs, g[f"mul_{name}_out"])
    assert np.array_equal(ring.poly_mul_schoolbook(a, b).coeffs, g[f"mul_{name}_out"])


def test_poly_mul_algebra():
    """Associativity, X*p = rotation, modulus mismatch (reference test_ring.py:112-130)."""
    N, q = 256, 1 << 20
    rng = np.random.default_rng(4)
    a, b, c = (ring.NegacyclicPoly(rng.integers(0, q, N), q) for _ in range(3))
    assert ring.poly_mul(ring.poly_mul(a, b), c) == ring.poly_mul(a, ring.poly_mul(b, c))
    x = np.zeros(N, dtype=np.int64)
    x[1] = 1
    assert ring.poly_mul(ring.NegacyclicPoly(x, q), a) == ring.monomial_rotate(a, 1)
    with pytest.raises(ParameterError):
        ring.poly_mul(a, ring.NegacyclicPoly(a.coeffs, 2 * q))
    # batched MAC against the oracle, random sizes incl. N = 1 and 4096
    for n in (1, 2, 4096):
        x = rng.integers(-(1 << 30), 1 << 30, (2, 3, n))
        y = rng.integers(-(1 << 12), 1 << 12, (2, 3, n))
        got = ring.negacyclic_mac_device(x, y, 1 << 32)
        for bi in range(2):
            want = sum(O.negacyclic_mul(x[bi, d] % (1 << 32), y[bi, d], 1 << 32) for d in range(3)) % (1 << 32)
            assert np.array_equal(got[bi], want)


@pytest.mark.parametrize("name", ["desk", "c4", "small"])
def test_gadget_decompose_matches_reference(g, name):
    q, base, levels = (int(v) for v in g[f"dig_{name}_prm"])
    d = rgsw.gadget_decompose(g[f"dig_{name}_x"], q, params.GadgetParams(base=base, levels=levels))
    assert np.array_equal(d, g[f"dig_{name}_out"])


def test_gadget_decompose_edges():
    """Known pattern 2048 -> [0, 0, 8] (reference test_rgsw.py:79-84), zero,
    recompose identity, digit range, leading batch axes, B^l < q."""
    assert list(rgsw.gadget_decompose(np.array([2048]), 1 << 12, params.GadgetParams(16, 3)).ravel()) == [0, 0, 8]
    gp = params.GadgetParams(base=1 << 6, levels=2)
    assert not rgsw.gadget_decompose(np.zeros(64, dtype=np.int64), 1 << 12, gp).any()
    rng = np.random.default_rng(8)
    x = rng.integers(0, 1 << 12, (2, 3, 64))
    d = rgsw.gadget_decompose(x, 1 << 12, gp)
    assert d.shape == (2, 3, 2, 64) and d.min() >= -31 and d.max() <= 32
    assert np.array_equal(rgsw.gadget_recompose(d, gp) % (1 << 12), x)
    short = params.GadgetParams(base=1 << 4, levels=2)  # B^l < q: lossy, same digits as the oracle
    x = rng.integers(0, 1 << 20, 500)
    assert np.array_equal(rgsw.gadget_decompose(x, 1 << 20, short), O.gadget_decompose(x, 1 << 20, 16, 2))


@pytest.mark.parametrize("name", ["small", "desk"])
def test_external_product_matches_reference(g, name):
    q, base, levels, N = (int(v) for v in g[f"ext_{name}_gadget"])
    gp = params.GadgetParams(base=base, levels=levels)
    ct = rgsw.RlweCiphertext(g[f"ext_{name}_ct"][0], g[f"ext_{name}_ct"][1], q)
    gct = rgsw.RgswCiphertext(g[f"ext_{name}_rows"][0], g[f"ext_{name}_rows"][1], q, gp)
    prm = small_ring() if name == "small" else params.preset("DESK").with_p(1024)
    out = rgsw.external_product(ct, gct, prm)
    assert np.array_equal(np.stack([out.a, out.b]), g[f"ext_{name}_out"])


def test_external_product_semantics():
    """identity / absorbing bit, monomial shift, CMux (reference test_rgsw.py:87-152)."""
    prm = small_ring()
    rng = np.random.default_rng(0)
    zk = rgsw.rlwe_keygen(prm, rng)
    m = ring.NegacyclicPoly(rng.integers(0, prm.p, prm.N), prm.p)
    ct = rgsw.rlwe_encrypt(m, zk, prm, rng)
    one = rgsw.rgsw_encrypt_bit(1, zk, prm, rng)
    zero = rgsw.rgsw_encrypt_bit(0, zk, prm, rng)
    assert rgsw.rlwe_decrypt(rgsw.external_product(ct, one, prm), zk, prm) == m
    assert not rgsw.rlwe_decrypt(rgsw.external_product(ct, zero, prm), zk, prm).coeffs.any()
    for k in (3, 64, 100):
        gk = rgsw.rgsw_encrypt_monomial(k, zk, prm, rng)
        out = rgsw.rlwe_decrypt(rgsw.external_product(ct, gk, prm), zk, prm)
        assert out == ring.NegacyclicPoly(ring.monomial_rotate(m, k).coeffs, prm.p)
    for bit in (0, 1):
        gb = rgsw.rgsw_encrypt_bit(bit, zk, prm, rng)
        c0 = rgsw.rlwe_encrypt(ring.NegacyclicPoly.constant(2, prm.N, prm.p), zk, prm, rng)
        c1 = rgsw.rlwe_encrypt(ring.NegacyclicPoly.constant(3, prm.N, prm.p), zk, prm, rng)
        diff = rgsw.RlweCiphertext(c1.a - c0.a, c1.b - c0.b, prm.q)
        dec = rgsw.rlwe_decrypt(c0 + rgsw.external_product(diff, gb, prm), zk, prm)
        assert dec.coeffs[0] == (3 if bit else 2)


def test_algebra_errors():
    with pytest.raises(ParameterError):
        ring.NegacyclicTransform(12)
    with pytest.raises(ParameterError):
        ring.NegacyclicTransform(8192)
    with pytest.raises(ParameterError):
        ring.get_transform(8).forward(np.zeros(16))
    prm = small_ring()
    ct = rgsw.RlweCiphertext(np.zeros(64), np.zeros(64), 1 << 12)
    gct = rgsw.RgswCiphertext(np.zeros((4, 64)), np.zeros((4, 64)), 1 << 13, prm.gadget)
    with pytest.raises(ParameterError):
        rgsw.external_product(ct, gct, prm)
