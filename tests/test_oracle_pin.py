"""Pin the CPU oracle: golden vectors produced by the reference itself
(tests/golden/make_golden.py) and the reference's own known-answer tests.
CPU only (no GPU needed)."""
import os

import numpy as np
import pytest

from conftest import GOLDEN, O, oracle_key
from paper_2309_09025_b200 import lwe, neuron, params


def load(name):
    path = os.path.join(GOLDEN, name + ".npz")
    if not os.path.exists(path):
        pytest.skip(f"golden fixture {name} not generated")
    return np.load(path)


# ---------------------------------------------------------------- KATs

def test_rounding_known_answers():
    """ring.py:36-53 rules (reference test_ring.py:15-34)."""
    assert O.round_half_away(np.array(0.5)) == 1 and O.round_half_away(np.array(-0.5)) == -1
    assert O.round_half_away(np.array(1.4)) == 1 and O.round_half_away(np.array(-2.6)) == -3
    assert O.div_round_half_away(5, 2) == 3 and O.div_round_half_away(-5, 2) == -3
    assert list(O.div_round_half_away(np.array([19, -19]), 2)) == [10, -10]


def test_rescale_known_answers():
    """reference test_ring.py:37-54."""
    assert O.rescale(np.array([4095]), 4096, 1024)[0] == 0
    xs = np.arange(4096)
    want = np.array([O.round_half_away(np.array(O.center(np.array(x), 4096) * 256 / 4096)) % 256 for x in xs])
    assert np.array_equal(O.rescale(xs, 4096, 256), want)


def test_gadget_known_pattern():
    """2048 -> [0, 0, 8] for B=16, l=3, q=2^12 (reference test_rgsw.py:79-84)."""
    assert list(O.gadget_decompose(np.array([2048]), 1 << 12, 16, 3).ravel()) == [0, 0, 8]
    rng = np.random.default_rng(4)
    x = rng.integers(0, 1 << 25, (4, 64))
    d = O.gadget_decompose(x, 1 << 25, 1 << 13, 2)
    back = (d[..., 0, :] + (1 << 13) * d[..., 1, :]) % (1 << 25)
    assert np.array_equal(back, x)
    assert d.min() >= -(1 << 12) + 1 and d.max() <= 1 << 12


def test_reset_lut_probes():
    """reference test_bootstrap.py:24-32 (theta=10, tau=2, p=1024)."""
    t = O.reset_table(20, 1, 2, 1024)
    assert t[0] == 0 and t[5] == 3 and t[19] == 10 and t[20] == 0 and t[(-3) % 1024] == 0
    ft = O.fire_table(64)
    assert ft[0] == 1 and ft[31] == 1 and ft[(-1) % 64] == -1 and ft[(-32) % 64] == -1


def test_plain_lif_known_answers():
    """reference test_neuron.py:37-51 (tau=2, theta=10 -> v_th_hat=20)."""
    cases = [((0, 25), (2, 0)), ((0, 10), (0, 5)), ((5, -8), (0, 0)), ((0, 20), (2, 0))]
    for (v, i), want in cases:
        s, nv = O.plain_lif_step(np.array([v]), np.array([i]), 20, 1, 2)
        assert (int(s[0]), int(nv[0])) == want


def test_twin_equals_plain_inside_range():
    p, vth = 1024, 128
    rng = np.random.default_rng(0)
    v = rng.integers(0, vth, 2000)
    i = rng.integers(vth - p // 2 - v.min(), p // 2 - vth, 2000)
    h = v + i
    ok = (h >= vth - p // 2) & (h < p // 2)
    s1, n1 = O.plain_lif_step(v[ok], i[ok], vth, 1, 2)
    s2, n2 = O.twin_lif_step(v[ok], i[ok], vth, 1, 2, p)
    assert np.array_equal(s1, s2) and np.array_equal(n1, n2)


def test_select_p_known_answers():
    """reference test_params.py:35-60."""
    assert params.select_p(40, 36.13) == 4096
    assert params.select_p(10, 23.00) == 512
    assert params.select_p(40, 0.0) == 8
    assert params.select_p(1, 256) == 512 and params.select_p(1, 257) == 1024
    assert params.select_p(10, 23.0, safety_margin=True) == 1024


# ------------------------------------------------------- golden vectors

def test_oracle_toy_bootstrap_golden(toy, toy_keys):
    g = load("toy")
    sk, zk, bsk = toy_keys
    key = oracle_key(toy, bsk)
    fA, fb = O.bootstrap_batch(O.fire_table(toy.p), g["A"], g["b"], key)
    assert np.array_equal(fA, g["fire_A"]) and np.array_equal(fb, g["fire_b"])
    rA, rb = O.bootstrap_batch(g["lut"], g["A"], g["b"], key)
    assert np.array_equal(rA, g["lut_A"]) and np.array_equal(rb, g["lut_b"])
    assert np.array_equal(O.blind_rotate(g["acc"], g["a2N"], key), g["br"])
    kA, kb = O.key_switch(g["ks_in_A"], g["ks_in_b"], key)
    assert np.array_equal(kA, g["ks_A"]) and np.array_equal(kb, g["ks_b"])
    # decrypted sign outputs
    assert np.array_equal(lwe.decrypt_batch(fA, fb, sk, toy), neuron.g_fire(toy.p)(g["ms"]))


def test_oracle_toy64_lif_golden(toy64, toy64_keys):
    g = load("toy64")
    sk, zk, bsk = toy64_keys
    key = oracle_key(toy64, bsk)
    got = O.lif_step(g["vA"], g["vb"], g["iA"], g["ib"], 10, 1, 2, key)
    for a, name in zip(got, ("sA", "sb", "nA", "nb")):
        assert np.array_equal(a, g[name])


def test_oracle_toy64_infer_golden(toy64, toy64_keys):
    g = load("toy64")
    sk, zk, bsk = toy64_keys
    key = oracle_key(toy64, bsk)
    lif = neuron.LifParams(tau=float("inf"), theta=int(g["theta"]))
    layers = [("weight", g["m1"]), ("spike", lif.v_th_hat, lif.leak_num, lif.leak_den),
              ("weight", g["m2"]), ("spike", lif.v_th_hat, lif.leak_num, lif.leak_den)]
    for k in range(g["img_A"].shape[0]):
        sA, sb = O.infer(g["img_A"][k], g["img_b"][k], layers, key, T=2)
        assert np.array_equal(sA, g["score_A"][k]) and np.array_equal(sb, g["score_b"][k])


@pytest.mark.parametrize("name,which", [("desk_lif", "desk"), ("c4_lif", "c4prm")])
def test_oracle_lif_golden(name, which, request):
    g = load(name)
    prm = request.getfixturevalue(which)
    sk, zk, bsk = request.getfixturevalue("desk_keys" if which == "desk" else "c4_keys")
    lif = neuron.LifParams(tau=2, theta=256 if prm.p == 4096 else 64)
    key = oracle_key(prm, bsk)
    got = O.lif_step(g["vA"], g["vb"], g["iA"], g["ib"], lif.v_th_hat, lif.leak_num, lif.leak_den, key)
    for a, nm in zip(got, ("sA", "sb", "nA", "nb")):
        assert np.array_equal(a, g[nm])
    s, v = O.twin_lif_step(g["v"], g["i"], lif.v_th_hat, lif.leak_num, lif.leak_den, prm.p)
    assert np.array_equal(s, g["spike"]) and np.array_equal(v, g["state"])


def test_oracle_layer_golden(desk):
    g = load("layer")
    for kind in ("conv", "dense"):
        A, b = O.layer_forward(g[kind + "_m"], g["A"], g["b"], desk.q)
        assert np.array_equal(A, g[kind + "_A"]) and np.array_equal(b, g[kind + "_b"])


def test_oracle_compiled_path_matches(toy64, toy64_keys):
    """The numba/BLAS CPU-baseline path (bench.py reference leg) is bit-exact with
    the plain restatement."""
    g = load("toy64")
    sk, zk, bsk = toy64_keys
    key = oracle_key(toy64, bsk)
    a = O.lif_step_fast(g["vA"], g["vb"], g["iA"], g["ib"], 10, 1, 2, key)
    for x, nm in zip(a, ("sA", "sb", "nA", "nb")):
        assert np.array_equal(x, g[nm])


def _plain_case(tag, prm):
    import sys
    sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tools"))
    import workloads as W
    import paper_2309_09025_b200 as api
    lif = W.lif_for(api, prm)
    net = (W.config2_network if tag == "c2" else W.config4_network)(api, lif)
    imgs = W.synth_images(32)
    return net, imgs, W.layers_for_oracle(net)


@pytest.mark.parametrize("tag", ["c2", "c4"])
def test_oracle_plain_infer_golden(tag, desk, c4prm):
    """oracle.plain_infer restatement == the reference's plain_infer (scores,
    per-layer spike counts, range-check failures at p) on configs 2 and 4."""
    g = load("plain")
    prm = desk if tag == "c2" else c4prm
    net, imgs, layers = _plain_case(tag, prm)
    overflowing = 0
    for k, img in enumerate(imgs):
        x = (img.astype(np.float64) / 255.0 >= 0.5).astype(np.int64).ravel()
        sc, counts, over = O.plain_infer(x, layers, net.T, prm.p)
        assert np.array_equal(sc, g[f"{tag}_scores"][k]), k
        for li, c in enumerate(counts):
            assert np.array_equal(c, g[f"{tag}_counts{li}"][k]), (k, li)
        overflowing += over > 0
    assert overflowing == int(g[f"{tag}_overflow_images"][0])


@pytest.mark.parametrize("tag", ["c2", "c4"])
def test_oracle_twin_matches_reference_encrypted_run(tag, desk, c4prm):
    """The mod-p twin (the checker for every full-batch GPU test) equals the
    reference's ENCRYPTED infer (network.py:459-491) on image 0 of configs 2
    and 4: every spiking layer's decrypted spikes at every timestep and the
    decrypted scores (config2_img0.npz / config4_img0.npz)."""
    name = "config2_img0" if tag == "c2" else "config4_img0"
    path = os.path.join(GOLDEN, name + ".npz")
    g = np.load(path)
    prm = desk if tag == "c2" else c4prm
    net, imgs, layers = _plain_case(tag, prm)
    x = (imgs[0].astype(np.float64) / 255.0 >= 0.5).astype(np.int64).ravel()
    score, log = O.twin_infer(x, layers, net.T, prm.p)
    assert np.array_equal(score, g["scores"])
    assert len(log) == sum(1 for k in g.files if k.startswith("l"))
    for li, t, v in log:
        assert np.array_equal(v, g[f"l{li}_t{t}"]), (li, t)


# ---------------------------------------------------- algebra layer (ring.npz)

def test_oracle_transform_matches_reference():
    """oracle.Transform vs the reference's NegacyclicTransform outputs."""
    g = load("ring")
    for N in (2, 8, 64, 1024, 2048):
        tr = O.Transform(N)
        f = tr.forward(g[f"nt{N}_in"])
        scale = np.abs(g[f"nt{N}_fwd"]).max()
        assert np.abs(f - g[f"nt{N}_fwd"]).max() <= 1e-12 * scale
        assert np.abs(tr.inverse(g[f"nt{N}_fwd"]) - g[f"nt{N}_inv"]).max() <= 1e-9


def test_oracle_products_and_digits_match_reference():
    g = load("ring")
    for name in ("desk", "c4", "tiny"):
        q = int(g[f"mul_{name}_q"][0])
        assert np.array_equal(O.negacyclic_mul(g[f"mul_{name}_a"], g[f"mul_{name}_b"], q), g[f"mul_{name}_out"])
    for name in ("desk", "c4", "small"):
        q, base, levels = (int(v) for v in g[f"dig_{name}_prm"])
        assert np.array_equal(O.gadget_decompose(g[f"dig_{name}_x"], q, base, levels), g[f"dig_{name}_out"])
    for name in ("small", "desk"):
        q, base, levels, _ = (int(v) for v in g[f"ext_{name}_gadget"])
        ct, rows = g[f"ext_{name}_ct"], g[f"ext_{name}_rows"]
        oa, ob = O.external_product(ct[0], ct[1], rows[0], rows[1], q, base, levels)
        assert np.array_equal(np.stack([oa, ob]), g[f"ext_{name}_out"])
