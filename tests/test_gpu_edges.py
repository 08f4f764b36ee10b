"""GPU edge cases: empty and ragged batches, identity rotations, error
behaviour, determinism, and the FP64 exactness margin of the transform."""
import numpy as np
import pytest

from conftest import O, oracle_key
from paper_2309_09025_b200 import bootstrap, errors, lwe, network, neuron

pytestmark = pytest.mark.gpu


def test_empty_batches(desk, desk_keys):
    sk, _, bsk = desk_keys
    A = np.zeros((0, desk.n), np.int64)
    b = np.zeros(0, np.int64)
    oA, ob = bootstrap.bootstrap_batch(neuron.g_fire(desk.p), A, b, bsk)
    assert oA.shape == (0, desk.n) and ob.shape == (0,)
    out = neuron.fhe_lif_step_batch(A, b, A, b, neuron.LifParams(tau=2, theta=64), bsk)
    assert all(x.shape[0] == 0 for x in out)


@pytest.mark.parametrize("count", [1, 3, 5, 7])
def test_ragged_batches_match_oracle(desk, desk_keys, count):
    """Batch sizes that leave part of the last CTA idle."""
    sk, _, bsk = desk_keys
    rng = np.random.default_rng(count)
    ms = rng.integers(-511, 513, count)
    A, b = lwe.encrypt_batch(ms, sk, desk, rng)
    g = neuron.g_fire(desk.p)
    oA, ob = bootstrap.bootstrap_batch(g, A, b, bsk)
    wA, wb = O.bootstrap_batch(g.table, A, b, oracle_key(desk, bsk))
    assert np.array_equal(oA, wA) and np.array_equal(ob, wb)


def test_identity_rotation_steps(toy, toy_keys):
    """Masks with many zero coordinates exercise the k == 0 skip path per ciphertext."""
    sk, _, bsk = toy_keys
    rng = np.random.default_rng(2)
    acc = rng.integers(0, toy.q, (9, 2, toy.N))
    a2N = rng.integers(0, 2 * toy.N, (9, toy.n))
    a2N[:, ::2] = 0
    a2N[3] = 0
    orig = acc.copy()
    got = bootstrap.blind_rotate_batch(acc, a2N, bsk)
    assert np.array_equal(got, O.blind_rotate(orig, a2N, oracle_key(toy, bsk)))
    assert np.array_equal(got[3], orig[3])


def test_deterministic(desk, desk_keys):
    sk, _, bsk = desk_keys
    rng = np.random.default_rng(5)
    A, b = lwe.encrypt_batch(rng.integers(-511, 513, 33), sk, desk, rng)
    g = neuron.g_fire(desk.p)
    r1 = bootstrap.bootstrap_batch(g, A, b, bsk)
    r2 = bootstrap.bootstrap_batch(g, A, b, bsk)
    assert np.array_equal(r1[0], r2[0]) and np.array_equal(r1[1], r2[1])


def test_parameter_errors(desk, desk_keys):
    sk, _, bsk = desk_keys
    g = neuron.g_fire(desk.p)
    with pytest.raises(errors.ParameterError):
        bootstrap.bootstrap_batch(g, np.zeros((2, desk.n + 1), np.int64), np.zeros(2, np.int64), bsk)
    with pytest.raises(errors.ParameterError):
        bootstrap.bootstrap_batch(neuron.g_fire(64), np.zeros((2, desk.n), np.int64), np.zeros(2, np.int64), bsk)
    with pytest.raises(errors.ParameterError):
        bootstrap.key_switch_batch(np.zeros((1, 10), np.int64), np.zeros(1, np.int64), bsk.ksk, desk)
    layer = network.WeightLayer("linear", np.ones((3, 4), np.int64), None, 1.0, (3,))
    x = network.zero_states(5, desk)
    with pytest.raises(errors.ParameterError):
        network.layer_forward(x, layer, desk)


@pytest.mark.parametrize("which,count,bound", [("desk", 64, 0.01), ("desk", 1184, 0.01), ("c4prm", 64, 0.01)])
def test_transform_exactness_margin(which, count, bound, request):
    """max |x - round(x)| over every rounded product of every CMux step stays far
    below 0.5 (the condition under which FP64 transforms are exact and the
    device's round-to-nearest equals the reference's round-half-away).  DESK
    64: the CTA-pair kernel; DESK 1184: one wave of the warp-per-rotation
    kernel (fft16.cuh); C4: the 4-per-SM kernel's parity-split transform."""
    prm = request.getfixturevalue(which)
    sk, _, bsk = request.getfixturevalue("desk_keys" if which == "desk" else "c4_keys")
    rng = np.random.default_rng(9)
    A, b = lwe.encrypt_batch(rng.integers(-prm.p // 2 + 1, prm.p // 2 + 1, count), sk, prm, rng)
    dev = bsk.device
    dev.margin(True)
    try:
        bootstrap.bootstrap_batch(neuron.g_fire(prm.p), A, b, bsk)
        m = dev.margin()
    finally:
        dev.margin(False)
    assert 0.0 < m < bound, m


def test_device_rows_roundtrip(desk, desk_keys):
    sk, _, bsk = desk_keys
    rng = np.random.default_rng(11)
    A = rng.integers(-desk.q, 2 * desk.q, (17, desk.n))
    b = rng.integers(-desk.q, 2 * desk.q, 17)
    dev = bsk.device
    rows = dev.rows_from_host(A, b)
    A2, b2 = dev.rows_to_host(rows)
    assert np.array_equal(A2, A % desk.q) and np.array_equal(b2, b % desk.q)
    assert rows.shape == (17, 516)


def test_fdsn_containers_to_device(toy, toy_keys, tmp_path):
    """Keys and ciphertexts loaded from FDSN files by the C library give the
    same bootstraps as the in-memory path."""
    from paper_2309_09025_b200 import serial
    sk, _, bsk = toy_keys
    rng = np.random.default_rng(13)
    ms = rng.integers(-3, 5, 24)
    A, b = lwe.encrypt_batch(ms, sk, toy, rng)
    serial.save_bootstrap_key(tmp_path / "bk.bin", bsk)
    serial.save_ciphertexts(tmp_path / "ct.bin", network.CiphertextTensor((2, 12), A, b, toy.q), toy)
    dev = serial.load_bootstrap_key_device(tmp_path / "bk.bin", toy)
    rows, shape = serial.load_ciphertexts_device(tmp_path / "ct.bin", dev)
    assert shape == (2, 12) and rows.shape[0] == 24
    g = neuron.g_fire(toy.p)
    lut = dev.lut(bootstrap.test_polynomial(g, toy))
    got = dev.rows_to_host(dev.pbs_dev([lut], [0], [0], rows))
    want = bootstrap.bootstrap_batch(g, A, b, bsk)
    assert np.array_equal(got[0], want[0]) and np.array_equal(got[1], want[1])
    with pytest.raises(errors.ParameterError):
        serial.load_bootstrap_key_device(tmp_path / "ct.bin", toy)


@pytest.mark.parametrize("count", [148, 149, 296, 297, 445, 446, 447, 600, 740, 1040, 1100, 1184, 1185, 1333, 2303, 2668])
def test_launch_regime_boundaries(desk, desk_keys, count):
    """Batches either side of the launch-split points give oracle-identical
    outputs (first and last 6 checked): waves of 8 rotations per SM on the
    warp-per-rotation kernel (1184 = one wave; 1185, 1333, 2668 add a
    remainder; 1100 and 2303 end in a partial wave whose last CTA has 4 and 7
    active warps); below that, and for small remainders, rounds of 4 rotations per SM
    then SM pairs (148, 1185), 2-3 per SM (149-447, 1333, 2668) or a
    4-rotation launch ending in a CTA of 1, 2 and 3 active rotations
    (445-447; 3 is the phase-skewed case with a single trailing group, which
    also refills the key ring)."""
    sk, _, bsk = desk_keys
    rng = np.random.default_rng(count)
    A, b = lwe.encrypt_batch(rng.integers(-511, 513, count), sk, desk, rng)
    g = neuron.g_fire(desk.p)
    oA, ob = bootstrap.bootstrap_batch(g, A, b, bsk)
    key = oracle_key(desk, bsk)
    for sl in (slice(0, 6), slice(count - 6, count)):
        wA, wb = O.bootstrap_batch(g.table, A[sl], b[sl], key)
        assert np.array_equal(oA[sl], wA) and np.array_equal(ob[sl], wb)


def test_large_preset_bit_exact():
    """The reference's LARGE preset (n=1024, q=2^27, N=2048, Bg=2^10 l=3, KS
    2^5x6): a different modulus, gadget and key-switch shape from every other
    test (4-limb tensor-core key switch with K=12288, n=1024 columns)."""
    from conftest import make_keys
    from paper_2309_09025_b200 import params
    prm = params.preset("LARGE")
    sk, _, bsk = make_keys(prm, 3)
    rng = np.random.default_rng(3)
    A, b = lwe.encrypt_batch(rng.integers(-prm.p // 2 + 1, prm.p // 2 + 1, 3), sk, prm, rng)
    g = neuron.g_fire(prm.p)
    oA, ob = bootstrap.bootstrap_batch(g, A, b, bsk)
    wA, wb = O.bootstrap_batch(g.table, A, b, oracle_key(prm, bsk))
    assert np.array_equal(oA, wA) and np.array_equal(ob, wb)


def test_n1024_three_level_gadget_paths():
    """N=1024 with a 3-level gadget (Bg=2^9): the single-level transform
    kernels at M=512 (1-rotation CTAs below 297 rotations, 4-rotation CTAs
    above), which the DESK gadget (l=2) never selects."""
    from dataclasses import replace
    from conftest import make_keys
    from paper_2309_09025_b200 import params
    prm = replace(params.preset("DESK").with_p(1024), gadget=params.GadgetParams(1 << 9, 3), preset_name="custom")
    sk, _, bsk = make_keys(prm, 4)
    key = oracle_key(prm, bsk)
    g = neuron.g_fire(prm.p)
    rng = np.random.default_rng(4)
    for count in (5, 300):
        A, b = lwe.encrypt_batch(rng.integers(-511, 513, count), sk, prm, rng)
        oA, ob = bootstrap.bootstrap_batch(g, A, b, bsk)
        for sl in (slice(0, 3), slice(count - 3, count)):
            wA, wb = O.bootstrap_batch(g.table, A[sl], b[sl], key)
            assert np.array_equal(oA[sl], wA) and np.array_equal(ob[sl], wb), count


@pytest.mark.parametrize("count", [5, 400, 599, 1300])
def test_desk_blind_rotate_raw_mode(desk, desk_keys, count):
    """blind_rotate_batch at DESK through the CTA-pair kernel (5), the paired
    kernel at 3 rotations per CTA (400), the phase-skewed 4-rotation kernel
    plus a CTA-pair tail (599) and a warp-per-rotation wave plus a CTA-pair
    tail (1300), raw accumulators in and out, vs the oracle.  Every third
    rotation starts with an identity step (rotation 0): the skew's signalling
    path when it falls on a leading accumulator, and a warp that skips a step
    but still takes part in the key ring."""
    sk, _, bsk = desk_keys
    rng = np.random.default_rng(40 + count)
    acc = rng.integers(0, desk.q, (count, 2, desk.N))
    a2N = rng.integers(0, 2 * desk.N, (count, desk.n))
    a2N[::3, 0] = 0
    orig = acc.copy()
    got = bootstrap.blind_rotate_batch(acc, a2N, bsk)
    key = oracle_key(desk, bsk)
    for j in sorted({0, 1, 3, count // 2, count - 1}):
        want = O.blind_rotate(orig[j:j + 1], a2N[j:j + 1], key)
        assert np.array_equal(got[j:j + 1], want), j


@pytest.mark.gpu
def test_fdsn_hostile_containers_fail_cleanly(toy, toy_keys, tmp_path):
    """The C reader checks every extent against the bytes left in the file and
    the body array against the mask count: a bogus shape is a ParameterError,
    not an abort (bad_alloc) or a heap over-read."""
    import struct
    from paper_2309_09025_b200 import serial
    from paper_2309_09025_b200.device import DeviceContext
    sk, _, bsk = toy_keys
    rng = np.random.default_rng(14)
    A, b = lwe.encrypt_batch(rng.integers(-3, 5, 6), sk, toy, rng)
    good = tmp_path / "ct.bin"
    serial.save_ciphertexts(good, network.CiphertextTensor((6,), A, b, toy.q), toy)
    blob = good.read_bytes()
    dev = DeviceContext(toy)

    def header_end():
        return 9 + blob[8]

    # 1. first array declares 2^40 x 2^20 elements
    bad = bytearray(blob)
    pos = header_end()
    tl = bad[pos]
    struct.pack_into("<q", bad, pos + 2 + tl, 1 << 40)
    (tmp_path / "huge.bin").write_bytes(bytes(bad))
    with pytest.raises(errors.ParameterError):
        serial.load_ciphertexts_device(tmp_path / "huge.bin", dev)
    # 2. body array "b" of shape (6, 0): zero payload but 6 ciphertexts claimed
    ct = tmp_path / "b0.bin"
    with open(ct, "wb") as f:
        serial._header(f, serial.KIND_CIPHERTEXTS, toy)
        serial._put(f, "shape", np.asarray([6]))
        serial._put(f, "A", A)
        serial._put(f, "b", np.zeros((6, 0), np.int64))
    with pytest.raises(errors.ParameterError):
        serial.load_ciphertexts_device(ct, dev)
    # 3. truncated key container
    bk = tmp_path / "bk.bin"
    serial.save_bootstrap_key(bk, bsk)
    kb = bk.read_bytes()
    (tmp_path / "bk_cut.bin").write_bytes(kb[: len(kb) // 2])
    with pytest.raises(errors.ParameterError):
        serial.load_bootstrap_key_device(tmp_path / "bk_cut.bin", toy)
    # the context still works afterwards
    rows, shape = serial.load_ciphertexts_device(good, dev)
    assert shape == (6,)
    A2, b2 = dev.rows_to_host(rows)
    assert np.array_equal(A2, A % toy.q) and np.array_equal(b2, b % toy.q)


@pytest.mark.gpu
def test_host_boundary_concurrent_streams(desk, desk_keys):
    """int64 host <-> device rows from several host threads on different
    streams at once (each stream has its own page-locked slots), sizes that
    span several slots, interleaved with bootstraps on the context stream."""
    import threading
    import torch
    sk, _, bsk = desk_keys
    dev = bsk.device
    rng = np.random.default_rng(15)
    sizes = [1, 5000, 9000, 777]
    data = [(rng.integers(-(1 << 40), 1 << 40, (c, desk.n)), rng.integers(-(1 << 40), 1 << 40, c)) for c in sizes]
    errs = []

    def work(k):
        try:
            st = torch.cuda.Stream()
            with torch.cuda.stream(st):
                for _ in range(3):
                    A, b = data[k]
                    rows = dev.rows_from_host(A, b)
                    A2, b2 = dev.rows_to_host(rows)
                    assert np.array_equal(A2, A % desk.q) and np.array_equal(b2, b % desk.q)
        except Exception as e:  # pragma: no cover
            errs.append(e)

    g = neuron.g_fire(desk.p)
    mA, mb = lwe.encrypt_batch(rng.integers(-511, 513, 40), sk, desk, rng)
    want = bootstrap.bootstrap_batch(g, mA, mb, bsk)
    ths = [threading.Thread(target=work, args=(k,)) for k in range(len(sizes))]
    for t in ths:
        t.start()
    got = bootstrap.bootstrap_batch(g, mA, mb, bsk)
    for t in ths:
        t.join()
    assert not errs, errs
    assert np.array_equal(got[0], want[0]) and np.array_equal(got[1], want[1])


@pytest.mark.parametrize("count", [1, 2, 37, 74, 75, 111, 148])
def test_cluster_latency_regime(desk, desk_keys, count):
    """Batches up to the SM count run on the CTA-pair kernel (one rotation per
    SM pair up to 74, two per pair above): bootstraps (with key switch) and
    raw-mode rotations bit-exact against the oracle, first/middle/last."""
    sk, _, bsk = desk_keys
    rng = np.random.default_rng(70 + count)
    A, b = lwe.encrypt_batch(rng.integers(-511, 513, count), sk, desk, rng)
    g = neuron.g_fire(desk.p)
    oA, ob = bootstrap.bootstrap_batch(g, A, b, bsk)
    key = oracle_key(desk, bsk)
    idx = sorted({0, count // 2, count - 1})
    wA, wb = O.bootstrap_batch(g.table, A[idx], b[idx], key)
    assert np.array_equal(oA[idx], wA) and np.array_equal(ob[idx], wb)
    acc = rng.integers(0, desk.q, (count, 2, desk.N))
    a2N = rng.integers(0, 2 * desk.N, (count, desk.n))
    a2N[:, 1::7] = 0  # identity steps inside the chain
    orig = acc.copy()
    got = bootstrap.blind_rotate_batch(acc, a2N, bsk)
    for j in idx:
        assert np.array_equal(got[j:j + 1], O.blind_rotate(orig[j:j + 1], a2N[j:j + 1], key)), j
