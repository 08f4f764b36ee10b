"""Client-side encryption / decryption on the device: same
ciphertexts as the host path for the same generator state, same decryptions."""
import numpy as np
import pytest

from paper_2309_09025_b200 import bootstrap, errors, lwe, neuron

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("which", ["toy", "desk", "c4prm"])
def test_encrypt_rows_bit_identical(which, request):
    prm = request.getfixturevalue(which)
    sk = lwe.lwe_keygen(prm, np.random.default_rng(3))
    ms = np.random.default_rng(4).integers(-prm.p // 2 + 1, prm.p // 2 + 1, 777)
    ms[:2] = (-prm.p // 2 + 1, prm.p // 2)
    A, b = lwe.encrypt_batch(ms, sk, prm, np.random.default_rng(5))
    rows = lwe.encrypt_batch_device(ms, sk, prm, np.random.default_rng(5))
    from paper_2309_09025_b200.network import _params_device
    dA, db = _params_device(prm).rows_to_host(rows)
    assert np.array_equal(dA, A) and np.array_equal(db, b)
    assert np.array_equal(lwe.decrypt_rows(rows, sk, prm), ms)


@pytest.mark.parametrize("which", ["toy", "desk", "c4prm"])
def test_decrypt_rows_matches_host_on_arbitrary_phases(which, request):
    """Arbitrary (A, b) -- every phase, including the rounding boundaries."""
    prm = request.getfixturevalue(which)
    sk = lwe.lwe_keygen(prm, np.random.default_rng(6))
    rng = np.random.default_rng(7)
    A = rng.integers(0, prm.q, (2000, prm.n))
    b = rng.integers(0, prm.q, 2000)
    # force phases onto the exact half-way points between messages
    ph = (np.arange(2000) * (prm.q // prm.p) + prm.q // (2 * prm.p)) % prm.q
    b[:2000:2] = ((A @ sk.s)[:2000:2] + ph[:2000:2]) % prm.q
    from paper_2309_09025_b200.network import _params_device
    rows = _params_device(prm).rows_from_host(A, b)
    assert np.array_equal(lwe.decrypt_rows(rows, sk, prm), lwe.decrypt_batch(A, b, sk, prm))


def test_device_client_round_trip_through_pbs(desk, desk_keys):
    sk, zk, bsk = desk_keys
    dev = bsk.device
    ms = np.random.default_rng(8).integers(-511, 513, 300)
    rows = lwe.encrypt_batch_device(ms, sk, desk, np.random.default_rng(9), device=dev)
    g = neuron.g_fire(desk.p)
    out = dev.pbs_dev([dev.lut(bootstrap.test_polynomial(g, desk))], [0], [0], rows)
    assert np.array_equal(lwe.decrypt_rows(out, sk, desk, device=dev), g(ms))


def test_encrypt_rows_domain_error(desk):
    sk = lwe.lwe_keygen(desk, np.random.default_rng(1))
    with pytest.raises(errors.DomainError):
        lwe.encrypt_batch_device(np.array([desk.p // 2 + 1]), sk, desk, np.random.default_rng(2))
