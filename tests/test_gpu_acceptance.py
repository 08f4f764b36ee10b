"""The reference's acceptance sweeps for this path, on the device (toy64:
TOY shape, p=64, sigma=2): every program table on every message, and the
full LIF step over every admissible (state, input) pair.
Follows reference tests test_acceptance.py:82-101 and test_neuron.py:107-121."""
import numpy as np
import pytest

from paper_2309_09025_b200 import bootstrap, lwe, neuron

pytestmark = pytest.mark.gpu


def test_bootstrap_exhaustive_program_sweep(toy64, toy64_keys):
    """sign, the reset table and 5 random negacyclic tables, each message
    50 times with fresh noise: zero decryption failures (22,400 PBS)."""
    p = toy64.p
    sk, _, bsk = toy64_keys
    rng = np.random.default_rng(99)
    programs = [neuron.g_fire(p), neuron.g_reset(neuron.LifParams(tau=2, theta=10), p)]
    for _ in range(5):
        programs.append(bootstrap.make_program(rng.integers(-p // 2 + 1, p // 2 + 1, p // 2).__getitem__, p))
    ms = np.repeat(np.arange(-p // 2 + 1, p // 2 + 1), 50)
    failures = 0
    for g in programs:
        A, b = lwe.encrypt_batch(ms, sk, toy64, rng)
        oA, ob = bootstrap.bootstrap_batch(g, A, b, bsk)
        failures += int(np.sum(lwe.decrypt_batch(oA, ob, sk, toy64) != g(ms)))
    assert failures == 0


def test_full_lif_step_exhaustive_inputs(toy64, toy64_keys):
    """Every i_hat in [-p/4, p/4) from states 0, 4, 9 (inside the representable
    range): decrypted spike and next state equal the integer LIF step."""
    sk, _, bsk = toy64_keys
    lif = neuron.LifParams(tau=2, theta=5)  # v_th_hat = 10 at p=64
    p = toy64.p
    rng = np.random.default_rng(3)
    vs, ins = [], []
    for i_hat in range(-p // 4, p // 4):
        for v0 in (0, 4, 9):
            if lif.v_th_hat - p // 2 <= v0 + i_hat < p // 2:
                vs.append(v0)
                ins.append(i_hat)
    vs, ins = np.array(vs), np.array(ins)
    vA, vb = lwe.encrypt_batch(vs, sk, toy64, rng)
    iA, ib = lwe.encrypt_batch(ins, sk, toy64, rng)
    sA, sb, nA, nb = neuron.fhe_lif_step_batch(vA, vb, iA, ib, lif, bsk)
    want_s, want_v = neuron.plain_lif_step_batch(vs, ins, lif)
    assert np.array_equal(lwe.decrypt_batch(sA, sb, sk, toy64), want_s)
    assert np.array_equal(lwe.decrypt_batch(nA, nb, sk, toy64), want_v)


# ---- reference test_bootstrap.py / test_neuron.py semantics on the device ----

def test_rotation_amount_matches_key_dot_product(toy, toy_keys):
    """Blind rotation rotates the test polynomial by <a2N, s> (test_bootstrap.py:78-90)."""
    from paper_2309_09025_b200 import rgsw, ring
    sk, zk, bsk = toy_keys
    rng = np.random.default_rng(3)
    base = bootstrap.initialize_accumulator(neuron.g_fire(toy.p), 0, toy)
    a2N = rng.integers(0, 2 * toy.N, (5, toy.n))
    acc = np.broadcast_to(np.stack([base.a, base.b])[None], (5, 2, toy.N)).copy()
    out = bootstrap.blind_rotate_batch(acc, a2N, bsk)
    for j in range(5):
        rot = int((a2N[j] @ sk.s) % (2 * toy.N))
        phase = rgsw.rlwe_phase(rgsw.RlweCiphertext(out[j, 0], out[j, 1], toy.q), zk, toy)
        want = ring.monomial_rotate_raw(base.b[None, :], np.array([rot]), toy.N)[0] % toy.q
        err = ring.center((phase - want) % toy.q, toy.q)
        assert np.abs(err).max() <= toy.noise_bound // 4


def test_trivial_ciphertext_through_key_switch(toy, toy_keys):
    """(0, Delta*2) key-switches to an encryption of 2 (test_bootstrap.py:150-155)."""
    sk, _, bsk = toy_keys
    A, b = bootstrap.key_switch_batch(np.zeros((1, toy.N), np.int64), np.array([toy.delta * 2]), bsk.ksk, toy)
    assert lwe.decrypt_batch(A, b, sk, toy)[0] == 2


def test_sign_idempotent_and_noise_independent_of_input(toy, toy_keys):
    """sign(sign(m)) == sign(m) (test_bootstrap.py:183-190) and the output noise
    does not depend on the input noise (test_bootstrap.py:199-215)."""
    from dataclasses import replace
    sk, _, bsk = toy_keys
    rng = np.random.default_rng(10)
    g = neuron.g_fire(toy.p)
    ms = np.array([-3, -1, 1, 3] * 8)
    A, b = lwe.encrypt_batch(ms, sk, toy, rng)
    oA, ob = bootstrap.bootstrap_batch(g, A, b, bsk)
    tA, tb = bootstrap.bootstrap_batch(g, oA, ob, bsk)
    assert np.array_equal(lwe.decrypt_batch(tA, tb, sk, toy), g(ms))
    assert np.array_equal(lwe.decrypt_batch(oA, ob, sk, toy), g(ms))

    def regime_max(sigma, trials=200):
        A, b = lwe.encrypt_batch(np.ones(trials, np.int64), sk, replace(toy, sigma=sigma), rng)
        oA, ob = bootstrap.bootstrap_batch(g, A, b, bsk)
        return int(np.abs(lwe.noise_of_batch(oA, ob, sk, np.ones(trials, np.int64), toy)).max())

    fresh, loud = regime_max(1.0), regime_max(toy.noise_bound / 8)
    assert abs(loud - fresh) <= max(0.1 * max(fresh, loud), 1)


def test_chained_lif_steps_and_if_mode(toy64, toy64_keys):
    """10 chained encrypted LIF steps track the integer neuron with bounded
    noise (test_neuron.py:131-143); integrate-and-fire mode (tau = inf,
    test_neuron.py:145-156)."""
    import math
    sk, _, bsk = toy64_keys
    lif = neuron.LifParams(tau=2, theta=5)
    rng = np.random.default_rng(5)
    count = 16
    vA, vb = lwe.encrypt_batch(np.zeros(count, np.int64), sk, toy64, rng)
    plain = np.zeros(count, np.int64)
    for t in range(10):
        i_hat = rng.integers(-5, 12, count)
        iA, ib = lwe.encrypt_batch(i_hat, sk, toy64, rng)
        sA, sb, vA, vb = neuron.fhe_lif_step_batch(vA, vb, iA, ib, lif, bsk)
        s_ref, plain = neuron.plain_lif_step_batch(plain, i_hat, lif)
        assert np.array_equal(lwe.decrypt_batch(sA, sb, sk, toy64), s_ref)
        assert np.array_equal(lwe.decrypt_batch(vA, vb, sk, toy64), plain)
        assert np.abs(lwe.noise_of_batch(vA, vb, sk, plain, toy64)).max() < toy64.noise_bound
    lif_if = neuron.LifParams(tau=math.inf, theta=8)
    v0 = np.array([0, 3, 5, 7])
    ih = np.array([8, 4, -9, 1])
    vA, vb = lwe.encrypt_batch(v0, sk, toy64, rng)
    iA, ib = lwe.encrypt_batch(ih, sk, toy64, rng)
    sA, sb, nA, nb = neuron.fhe_lif_step_batch(vA, vb, iA, ib, lif_if, bsk)
    s_ref, v_ref = neuron.plain_lif_step_batch(v0, ih, lif_if)
    assert np.array_equal(lwe.decrypt_batch(sA, sb, sk, toy64), s_ref)
    assert np.array_equal(lwe.decrypt_batch(nA, nb, sk, toy64), v_ref)
