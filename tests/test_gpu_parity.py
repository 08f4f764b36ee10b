"""GPU parity: every device entry point vs the CPU oracle, bit-exact."""
import numpy as np
import pytest

from conftest import O, oracle_key
from paper_2309_09025_b200 import bootstrap, lwe, network, neuron

pytestmark = pytest.mark.gpu


def _enc(prm, sk, count, seed, lo=None, hi=None):
    rng = np.random.default_rng(seed)
    lo = -prm.p // 2 + 1 if lo is None else lo
    hi = prm.p // 2 if hi is None else hi
    ms = rng.integers(lo, hi + 1, count)
    A, b = lwe.encrypt_batch(ms, sk, prm, rng)
    return ms, A, b


@pytest.mark.parametrize("which", ["toy", "toy64", "desk"])
def test_bootstrap_batch_bit_exact(which, request):
    prm = request.getfixturevalue(which)
    sk, _, bsk = request.getfixturevalue(which + "_keys")
    ms, A, b = _enc(prm, sk, 48, 11)
    g = neuron.g_fire(prm.p)
    outA, outb = bootstrap.bootstrap_batch(g, A, b, bsk)
    key = oracle_key(prm, bsk)
    wA, wb = O.bootstrap_batch(g.table, A, b, key)
    assert np.array_equal(outA, wA) and np.array_equal(outb, wb)
    assert np.array_equal(lwe.decrypt_batch(outA, outb, sk, prm), g(ms))


def test_random_lut_and_counter(toy64, toy64_keys):
    sk, _, bsk = toy64_keys
    rng = np.random.default_rng(3)
    g = bootstrap.make_program(dict(enumerate(rng.integers(-31, 33, 32))), toy64.p)
    ms, A, b = _enc(toy64, sk, 64, 12)
    before = bsk.bootstrap_count
    outA, outb = bootstrap.bootstrap_batch(g, A, b, bsk)
    assert bsk.bootstrap_count == before + 64
    wA, wb = O.bootstrap_batch(g.table, A, b, oracle_key(toy64, bsk))
    assert np.array_equal(outA, wA) and np.array_equal(outb, wb)


def test_blind_rotate_batch(toy, toy_keys):
    sk, zk, bsk = toy_keys
    rng = np.random.default_rng(4)
    acc = rng.integers(0, toy.q, (5, 2, toy.N))
    a2N = rng.integers(0, 2 * toy.N, (5, toy.n))
    a2N[0] = 0  # identity rotation
    want = O.blind_rotate(acc.copy(), a2N, oracle_key(toy, bsk))
    got = bootstrap.blind_rotate_batch(acc, a2N, bsk)
    assert np.array_equal(got, want)
    assert got is acc  # C-contiguous int64: rotated in place (bootstrap.py:263,281)


def test_blind_rotate_batch_ownership(toy, toy_keys):
    """The reference's ownership rules (bootstrap.py:252-282): a C-contiguous
    int64 accumulator is rotated in place; a non-contiguous one is copied and
    left alone; when every rotation index is 0 mod 2N no step runs and the
    accumulators come back unreduced."""
    sk, zk, bsk = toy_keys
    rng = np.random.default_rng(41)
    acc = rng.integers(0, toy.q, (4, 2, toy.N))
    a2N = rng.integers(0, 2 * toy.N, (4, toy.n))
    want = O.blind_rotate(acc.copy(), a2N, oracle_key(toy, bsk))
    wide = np.zeros((4, 2, 2 * toy.N), np.int64)
    view = wide[:, :, ::2]  # non-contiguous view
    view[...] = acc
    got = bootstrap.blind_rotate_batch(view, a2N, bsk)
    assert got is not view and np.array_equal(got, want)
    assert np.array_equal(view, acc)  # caller's strided array untouched
    raw = acc.copy()
    raw[0, 0, :3] = [-5, toy.q + 7, 3 * toy.q]  # unreduced values
    zero = np.zeros_like(a2N)
    zero[1, 0] = 2 * toy.N  # == 0 mod 2N
    kept = raw.copy()
    assert bootstrap.blind_rotate_batch(raw, zero, bsk) is raw
    assert np.array_equal(raw, kept)


def test_key_switch_batch(toy, toy_keys):
    sk, zk, bsk = toy_keys
    rng = np.random.default_rng(5)
    A = rng.integers(-toy.q, toy.q, (9, toy.N))
    b = rng.integers(0, toy.q, 9)
    got = bootstrap.key_switch_batch(A, b, bsk.ksk, toy)
    want = O.key_switch(A, b, oracle_key(toy, bsk))
    assert np.array_equal(got[0], want[0]) and np.array_equal(got[1], want[1])
    # bsk.ksk is served by the bootstrapping key's own context
    assert bootstrap._key_device(bsk.ksk, toy) is bsk.device


def test_key_switch_standalone_key(toy, toy_keys):
    """A KeySwitchKey not attached to a loaded BootstrapKey gets a context that
    holds only the key-switch key; the cache entry dies with the key."""
    import gc
    sk, zk, bsk = toy_keys
    ksk = bootstrap.KeySwitchKey(bsk.ksk.A.copy(), bsk.ksk.b.copy(), bsk.ksk.base, bsk.ksk.levels, bsk.ksk.N)
    rng = np.random.default_rng(6)
    A = rng.integers(-toy.q, toy.q, (7, toy.N))
    b = rng.integers(0, toy.q, 7)
    got = bootstrap.key_switch_batch(A, b, ksk, toy)
    want = O.key_switch(A, b, oracle_key(toy, bsk))
    assert np.array_equal(got[0], want[0]) and np.array_equal(got[1], want[1])
    ctx = bootstrap._key_device(ksk, toy)
    assert ctx is not bsk.device and not ctx.keys_loaded
    before = len(bootstrap._KS_DEVICES)
    del ksk, ctx
    gc.collect()
    assert len(bootstrap._KS_DEVICES) == before - 1


@pytest.mark.parametrize("which,count", [("toy", 9), ("desk", 130), ("c4prm", 257)])
def test_key_switch_tensor_core_path(which, count, request, monkeypatch):
    """The tcgen05 int8 GEMM key switch (4 / 3 byte limbs, ragged 128-row
    blocks, partial 64-column tiles at n=742) equals the CUDA-core kernels and
    the oracle bit for bit, including the extreme residues 0 and q-1."""
    from paper_2309_09025_b200.device import DeviceContext
    prm = request.getfixturevalue(which)
    sk, zk, bsk = request.getfixturevalue({"toy": "toy_keys", "desk": "desk_keys", "c4prm": "c4_keys"}[which])
    rng = np.random.default_rng(17)
    A = rng.integers(0, prm.q, (count, prm.N))
    b = rng.integers(0, prm.q, count)
    A[0] = 0
    A[1] = prm.q - 1
    A[2] = prm.q // 2
    results = []
    for force in ("0", "1"):
        monkeypatch.setenv("FDSNN_KS_CUDACORE", force)
        dev = DeviceContext(prm)
        dev.load_keys(np.zeros((prm.n, 2 * prm.gadget.levels, 2, prm.N), np.int64), bsk.ksk.A, bsk.ksk.b)
        results.append(dev.key_switch_batch(A, b))
        dev.close()
    want = O.key_switch(A, b, oracle_key(prm, bsk))
    for got in results:
        assert np.array_equal(got[0], want[0]) and np.array_equal(got[1], want[1])


@pytest.mark.parametrize("which", ["toy64", "desk"])
def test_lif_step_bit_exact(which, request):
    prm = request.getfixturevalue(which)
    sk, _, bsk = request.getfixturevalue(which + "_keys")
    lif = neuron.LifParams(tau=2, theta=max(1, prm.p // 16))
    _, vA, vb = _enc(prm, sk, 40, 21, 0, lif.v_th_hat - 1)
    _, iA, ib = _enc(prm, sk, 40, 22)
    got = neuron.fhe_lif_step_batch(vA, vb, iA, ib, lif, bsk)
    want = O.lif_step(vA, vb, iA, ib, lif.v_th_hat, lif.leak_num, lif.leak_den, oracle_key(prm, bsk))
    for g, w in zip(got, want):
        assert np.array_equal(g, w)


def test_c4_lif_step_bit_exact(c4prm, c4_keys):
    sk, _, bsk = c4_keys
    lif = neuron.LifParams(tau=2, theta=256)
    _, iA, ib = _enc(c4prm, sk, 4, 23)
    zA, zb = np.zeros_like(iA), np.zeros_like(ib)
    got = neuron.fhe_lif_step_batch(zA, zb, iA, ib, lif, bsk)
    want = O.lif_step(zA, zb, iA, ib, lif.v_th_hat, lif.leak_num, lif.leak_den, oracle_key(c4prm, bsk))
    for g, w in zip(got, want):
        assert np.array_equal(g, w)


@pytest.mark.parametrize("dense", [True, False])
def test_layer_forward(desk, desk_keys, dense):
    sk, _, _ = desk_keys
    rng = np.random.default_rng(6)
    if dense:
        M = rng.integers(-15, 16, (37, 50))
        shape = (37,)
    else:
        w = rng.integers(-7, 8, (3, 1, 3, 3))
        M, shape = network.conv_matrix(w, (1, 5, 10), (1, 1), (0, 0))
    ms, A, b = _enc(desk, sk, M.shape[1], 7, 0, 1)
    layer = network.WeightLayer("linear", M, None, 1.0, shape)
    out = network.layer_forward(network.CiphertextTensor((M.shape[1],), A, b, desk.q), layer, desk)
    wA, wb = O.layer_forward(M, A, b, desk.q)
    assert np.array_equal(out.A, wA) and np.array_equal(out.b, wb)


@pytest.mark.parametrize("wmax,cudacore", [(127, False), (127, True), (200, False)])
def test_layer_forward_tensor_core_and_fallback(desk, desk_keys, wmax, cudacore, monkeypatch):
    """Dense weight sums: s8 weights run on the tcgen05 kind::i8 GEMM
    (lin_umma.cuh: 4 byte limbs of every ciphertext word, exact s32 sums);
    FDSNN_LIN_CUDACORE=1, or any weight outside [-128, 127], selects the
    CUDA-core int32 GEMM.  Shapes exercise every padding: 130 outputs (a
    partial second row block), 300 inputs (K padded to 384), 3 samples (1548
    columns: a partial last column tile), extreme weights +-127 / -128."""
    from paper_2309_09025_b200.device import DeviceContext
    if cudacore:
        monkeypatch.setenv("FDSNN_LIN_CUDACORE", "1")
    sk, _, _ = desk_keys
    rng = np.random.default_rng(60 + wmax)
    M = rng.integers(-wmax, wmax + 1, (130, 300))
    M[0, :4] = [127, -128, 127, -128] if wmax == 127 else [wmax, -wmax, 1, -1]
    xs = []
    for s in range(3):
        ms, A, b = _enc(desk, sk, 300, 70 + s, 0, 1)
        xs.append(network.CiphertextTensor((300,), A, b, desk.q))
    dev = DeviceContext(desk)  # fresh context: the operator is loaded under this test's environment
    op = dev.operator(M)
    rows = dev.rows_from_host_parts([(x.A, x.b) for x in xs])
    A, b = dev.rows_to_host(dev.apply(op, rows, 3, 130))
    for s in range(3):
        wA, wb = O.layer_forward(M, xs[s].A, xs[s].b, desk.q)
        assert np.array_equal(A[s * 130:(s + 1) * 130], wA) and np.array_equal(b[s * 130:(s + 1) * 130], wb), s
