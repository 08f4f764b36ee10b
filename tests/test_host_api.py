"""Host-side mirror of the reference API (CPU only): key generation parity,
parameter validation, LUTs, encryption, network lowering, error types."""
import hashlib
import json
import math
import os

import numpy as np
import pytest

from conftest import GOLDEN, O, make_keys
from paper_2309_09025_b200 import bootstrap, errors, lwe, network, neuron, params, rgsw, ring


def sha(*arrays):
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(np.asarray(a, dtype=np.int64)).tobytes())
    return h.hexdigest()


def test_key_generation_matches_reference_digests(toy, toy64, desk, c4prm):
    """Keys from a seed are bit-identical to the reference's (keys.json written by
    running the reference's gen_bootstrap_key)."""
    path = os.path.join(GOLDEN, "keys.json")
    want = json.load(open(path))
    for name, prm in (("toy", toy), ("toy64", toy64), ("desk1024", desk), ("c4", c4prm)):
        w = want[name]
        sk, zk, bsk = make_keys(prm, w["seed"])
        assert sha(sk.s) == w["sk"] and sha(zk.z) == w["zk"]
        assert sha(bsk.rows) == w["rows"]
        assert sha(bsk.ksk.A) == w["ksk_A"] and sha(bsk.ksk.b) == w["ksk_b"]
        assert prm.digest() == w["params_digest"]


def test_params_validation():
    with pytest.raises(errors.ParameterError):
        params.FheParams(n=8, q=1000, N=512, p=8, sigma=1, gadget=params.GadgetParams(64, 2),
                         ks_base=8, ks_levels=4, sigma_bk=0.1, sigma_ks=0.1)
    with pytest.raises(errors.ParameterError):  # gadget must cover q
        params.FheParams(n=8, q=1 << 25, N=1024, p=8, sigma=1, gadget=params.GadgetParams(1 << 7, 3),
                         ks_base=4, ks_levels=8, sigma_bk=0.1, sigma_ks=0.1)
    with pytest.raises(errors.ParameterError):
        params.preset("TOY").with_p(12)
    with pytest.raises(errors.ConfigurationError):
        params.preset("nope")
    d = params.preset("DESK")
    assert (d.grid, d.delta, d.noise_bound) == (1 << 14, 1 << 14, 1 << 13)
    assert params.FheParams.from_dict(d.to_dict()) == d


def test_program_functions():
    g = neuron.g_fire(8)
    assert all(g(m) == 1 for m in range(4)) and all(g(m) == -1 for m in range(-4, 0))
    with pytest.raises((errors.DomainError, errors.ParameterError)):
        bootstrap.ProgramFunction([1] * 8, 8)
    lif = neuron.LifParams(tau=2, theta=10)
    gr = neuron.g_reset(lif, 1024)
    assert (gr(0), gr(5), gr(19), gr(20), gr(-3)) == (0, 3, 10, 0, 0)
    with pytest.raises(errors.ParameterError):
        neuron.g_reset(neuron.LifParams(tau=2, theta=100), 64)
    rng = np.random.default_rng(0)
    for p in (8, 64, 1024):
        g = bootstrap.make_program(dict(enumerate(rng.integers(-p // 2 + 1, p // 2 + 1, p // 2))), p)
        for v in range(p // 2):
            assert (g(v - p // 2) + g(v)) % p == 0


def test_test_polynomial_and_accumulator(toy):
    g = neuron.g_fire(toy.p)
    v = bootstrap.test_polynomial(g, toy)
    want = np.array([(toy.delta * g((i * toy.p) // (2 * toy.N))) % toy.q for i in range(toy.N)])
    assert np.array_equal(v, want)
    acc = bootstrap.initialize_accumulator(g, 0, toy)
    assert np.array_equal(acc.b, want) and not np.any(acc.a)
    z = bootstrap.make_program(lambda m: 0, toy.p)
    for b2N in (0, 17, 511, 1023):
        a = bootstrap.initialize_accumulator(z, b2N, toy)
        assert not np.any(a.a) and not np.any(a.b)


def test_lif_params_and_plain_steps():
    lif = neuron.LifParams(tau=2, theta=10)
    assert lif.v_th_hat == 20 and (lif.leak_num, lif.leak_den) == (1, 2)
    assert neuron.LifParams(tau=math.inf, theta=10).v_th_hat == 10
    assert (neuron.LifParams(tau=2, theta=10, leak_convention="theta").leak_num) == 9
    with pytest.raises(errors.ParameterError):
        neuron.LifParams(tau=1, theta=10)
    s, nxt = neuron.plain_lif_step(neuron.PlainLifState(0), 25, lif)
    assert (s, nxt.v_hat) == (2, 0)
    s, nxt = neuron.plain_lif_step(neuron.PlainLifState(0), 10, lif)
    assert (s, nxt.v_hat) == (0, 5)
    with pytest.raises(errors.OverflowViolation):
        neuron.plain_lif_step(neuron.PlainLifState(0), 600, lif, p=1024)


def test_encrypt_decrypt_roundtrip(toy64, toy64_keys):
    sk, _, _ = toy64_keys
    rng = np.random.default_rng(3)
    ms = rng.integers(-31, 33, 500)
    A, b = lwe.encrypt_batch(ms, sk, toy64, rng)
    assert np.array_equal(lwe.decrypt_batch(A, b, sk, toy64), ms)
    assert np.all(A % toy64.grid == 0)
    with pytest.raises(errors.DomainError):
        lwe.encrypt_batch(np.array([-32]), sk, toy64, rng)
    ct = lwe.weight_sum([lwe.encrypt(1, sk, toy64, rng), lwe.encrypt(2, sk, toy64, rng)], [3, -1])
    assert lwe.decrypt(ct, sk, toy64) == 1


@pytest.mark.gpu
def test_gadget_device_rule(desk):
    rng = np.random.default_rng(5)
    x = rng.integers(0, desk.q, (3, 16))
    d = rgsw.gadget_decompose(x, desk.q, desk.gadget)
    assert np.array_equal(rgsw.gadget_recompose(d, desk.gadget) % desk.q, x)
    assert list(rgsw.gadget_decompose(np.array([2048]), 1 << 12, params.GadgetParams(16, 3)).ravel()) == [0, 0, 8]


def test_ring_helpers():
    assert ring.rescale(4095, 4096, 1024) == 0
    assert ring.round_half_away(0.5) == 1 and ring.round_half_away(-0.5) == -1
    a = np.random.default_rng(1).integers(-100, 100, 64)
    z = np.random.default_rng(2).integers(0, 2, 64)
    full = np.convolve(a, z)
    want = (full[:64] - np.concatenate([full[64:], [0]])) % 4096
    assert np.array_equal(ring.negacyclic_mul_raw(a, z, 4096), want)


def test_conv_and_pool_lowering():
    rng = np.random.default_rng(6)
    w = rng.integers(-3, 4, (2, 1, 3, 3))
    m, shape = network.conv_matrix(w, (1, 5, 6), (2, 1), (1, 0))
    x = rng.integers(0, 5, (1, 5, 6))
    # naive conv
    oh, ow = shape[1], shape[2]
    xp = np.pad(x, ((0, 0), (1, 1), (0, 0)))
    want = np.zeros(shape, np.int64)
    for o in range(2):
        for y in range(oh):
            for xx in range(ow):
                want[o, y, xx] = (w[o, 0] * xp[0, 2 * y:2 * y + 3, xx:xx + 3]).sum()
    assert shape == (2, 3, 4) and np.array_equal(m @ x.ravel(), want.ravel())
    pm, ps = network.pool_matrix((2, 4, 4), (2, 2))
    assert ps == (2, 2, 2) and np.all(pm.sum(axis=1) == 4) and np.all(pm.sum(axis=0) == 1)


def test_discretize_scale_rules():
    lin = network.CsnnModel(
        arch=({"type": "linear", "out_features": 4}, {"type": "spiking"},
              {"type": "linear", "out_features": 2}, {"type": "spiking"}),
        weights=(np.full((4, 4), 0.5), np.full((2, 4), 0.126)), input_shape=(1, 2, 2), T=1, L=1, tau=None)
    net = network.discretize(lin, 40)
    second = [l for l in net.layers if isinstance(l, network.WeightLayer)][1]
    assert second.scale == 20 and np.all(second.matrix == 3)
    assert net.bootstrap_count() == 2 * (4 + 2)
    doc = lin.to_dict()
    again = network.CsnnModel.from_dict(doc)
    assert again.T == 1 and np.array_equal(again.weights[1], lin.weights[1])
    doc["format"] = "fdsnn-model/999"
    with pytest.raises(errors.SerializationError):
        network.CsnnModel.from_dict(doc)


def test_ciphertext_tensor_checks(toy):
    with pytest.raises(errors.ParameterError):
        network.CiphertextTensor((3,), np.zeros((2, toy.n)), np.zeros(2), toy.q)
    z = network.zero_states(5, toy)
    assert z.count == 5 and not np.any(z.A)


def test_fdsn_containers_byte_identical_to_reference(toy, toy_keys, tmp_path):
    """Our FDSN writer produces the reference's exact bytes (sha256 recorded by
    running the reference's serial.save_* on the same objects)."""
    from paper_2309_09025_b200 import serial
    want = json.load(open(os.path.join(GOLDEN, "fdsn.json")))
    sk, zk, bsk = toy_keys
    rng = np.random.default_rng(want["ct_seed"])
    A, b = lwe.encrypt_batch(rng.integers(-3, 5, 12), sk, toy, rng)
    ct = network.CiphertextTensor((3, 4), A, b, toy.q)
    serial.save_secret_key(tmp_path / "sk.bin", sk, zk, toy)
    serial.save_bootstrap_key(tmp_path / "bk.bin", bsk)
    serial.save_ciphertexts(tmp_path / "ct.bin", ct, toy)
    for k in ("sk", "bk", "ct"):
        assert serial.file_digest(tmp_path / f"{k}.bin") == want[k], k
    sk2, zk2 = serial.load_secret_key(tmp_path / "sk.bin", toy)
    assert np.array_equal(sk2.s, sk.s) and np.array_equal(zk2.z, zk.z)
    bk2 = serial.load_bootstrap_key(tmp_path / "bk.bin", toy)
    assert np.array_equal(bk2.rows, bsk.rows) and np.array_equal(bk2.ksk.A, bsk.ksk.A)
    ct2 = serial.load_ciphertexts(tmp_path / "ct.bin", toy)
    assert ct2.shape == (3, 4) and np.array_equal(ct2.A, A) and np.array_equal(ct2.b, b)
    with pytest.raises(errors.SerializationError):
        serial.load_ciphertexts(tmp_path / "ct.bin", params.preset("DESK"))
    with pytest.raises(errors.SerializationError):
        serial.load_secret_key(tmp_path / "ct.bin", toy)


def test_fdsn_truncated_containers_raise_serialization_error(toy, toy_keys, tmp_path):
    """A container cut at any byte (header, tag, shape or payload) raises the
    reference's SerializationError, never IndexError/struct.error; negative
    extents are rejected too."""
    import struct
    from paper_2309_09025_b200 import serial
    sk, zk, bsk = toy_keys
    rng = np.random.default_rng(3)
    A, b = lwe.encrypt_batch(rng.integers(-3, 5, 3), sk, toy, rng)
    path = tmp_path / "ct.bin"
    serial.save_ciphertexts(path, network.CiphertextTensor((3,), A, b, toy.q), toy)
    blob = path.read_bytes()
    # array boundaries: a cut there is a well-formed shorter container, whose
    # missing array is a KeyError in the reference too (serial.py:140-145)
    bounds, pos = {9 + blob[8]}, 9 + blob[8]
    while pos < len(blob):
        tl = blob[pos]
        nd = blob[pos + 1 + tl]
        shape = struct.unpack_from(f"<{nd}q", blob, pos + 2 + tl)
        pos += 2 + tl + 8 * nd + 8 * int(np.prod(shape))
        bounds.add(pos)
    cut = tmp_path / "cut.bin"
    for n in range(len(blob)):
        cut.write_bytes(blob[:n])
        want = (errors.SerializationError, KeyError) if n in bounds else errors.SerializationError
        try:
            serial.load_ciphertexts(cut, toy)
        except want:
            continue
        except Exception as e:  # pragma: no cover - the failure being tested
            raise AssertionError(f"cut at {n}: {type(e).__name__}: {e}")
        raise AssertionError(f"cut at {n} loaded")
    # a negative extent in the first array header
    hdr = 9 + blob[8]
    bad = bytearray(blob)
    tl = bad[hdr]
    struct.pack_into("<q", bad, hdr + 1 + tl + 1, -1)
    cut.write_bytes(bytes(bad))
    with pytest.raises(errors.SerializationError):
        serial.load_ciphertexts(cut, toy)


def _paper_model():
    from paper_2309_09025_b200 import network as N
    m = np.load(os.path.join(GOLDEN, "paper_model.npz"))
    arch = ({"type": "conv2d", "out_channels": 10, "kernel": [8, 8], "stride": [2, 2], "padding": [1, 1]},
            {"type": "spiking"}, {"type": "avgpool", "window": [2, 2]},
            {"type": "linear", "out_features": 160}, {"type": "spiking"},
            {"type": "linear", "out_features": 10}, {"type": "spiking"})
    return N.CsnnModel(arch=arch, weights=(m["w0"], m["w1"], m["w2"]), input_shape=(1, 28, 28),
                       T=int(m["T"][0]), L=int(m["L"][0]), tau=None, v_th=float(m["v_th"][0]))


def test_paper_model_lowering_known_answers():
    """The paper's network (reference fixture model_if_t2.json, weights in
    tests/golden/paper_model.npz) discretized at theta=40: 3220 PBS per step
    (reference test_oracle.py:175) and the reference's plain_infer scores."""
    from paper_2309_09025_b200 import network as N
    net = N.discretize(_paper_model(), 40)
    assert net.bootstrap_count(1) == 3220 and net.bootstrap_count(2) == 6440
    g = np.load(os.path.join(GOLDEN, "paper.npz"))
    import sys
    sys.path.insert(0, os.path.join(os.path.dirname(GOLDEN), os.pardir, "tools"))
    import workloads as W
    from conftest import O
    layers = W.layers_for_oracle(net)
    for k, img in enumerate(W.synth_images(2)):
        x = (img.astype(np.float64) / 255.0 >= 0.5).astype(np.int64).ravel()
        sc, _, over = O.plain_infer(x, layers, net.T, 2048)
        assert over == 0 and np.array_equal(sc, g[f"plain{k}"])


def test_ring_value_types():
    """ZqElement / NegacyclicPoly / monomial_rotate semantics (ring.py:71-100,
    146-196, 245-247; reference test_ring.py:58-89)."""
    from paper_2309_09025_b200 import ring
    a, b = ring.ZqElement(13, 16), ring.ZqElement(7, 16)
    assert (a + b).value == 4 and (a - b).value == 6 and (a * b).value == 11 and a.centered == -3
    with pytest.raises(errors.ParameterError):
        a + ring.ZqElement(1, 32)
    N, q = 16, 1 << 10
    p = ring.NegacyclicPoly(np.arange(N) * 7, q)
    assert ring.monomial_rotate(p, N) == ring.NegacyclicPoly(-p.coeffs, q)      # half turn negates
    assert ring.monomial_rotate(p, 2 * N) == p                                   # full turn
    assert ring.monomial_rotate(ring.monomial_rotate(p, 5), -5) == p
    assert ring.monomial_rotate(p, 3) == ring.NegacyclicPoly(O.monomial_rotate(p.coeffs, [3], N)[0], q)
    assert (p + p) - p == p and ring.NegacyclicPoly.zero(N, q) + p == p
    with pytest.raises(errors.ParameterError):
        p + ring.NegacyclicPoly.zero(N, 2 * q)


def test_reference_architecture_topology():
    """network.py:214-233: conv 10x8x8/2 (pad 1) -> spike -> pool 2 -> 360->160 -> spike -> 160->10."""
    from paper_2309_09025_b200 import network
    m = network.reference_architecture()
    assert m.shape_chain() == [(10, 12, 12), (10, 12, 12), (10, 6, 6), (160,), (160,), (10,), (10,)]
    assert [w.shape for w in m.weights] == [(10, 1, 8, 8), (160, 360), (10, 160)]
    w0 = np.random.default_rng(0).normal(0, 0.1, (10, 1, 8, 8))
    assert np.array_equal(m.weights[0], w0)
