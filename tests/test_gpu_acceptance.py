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
