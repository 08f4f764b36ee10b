"""The reference's network-level semantics (reference test_network.py:78-215)
through the device path: weight sums on the GPU, encrypted inference vs the
integer plain path, bootstrap counts and score ranges, batch/serial
invariance, argument errors."""
import numpy as np
import pytest

from paper_2309_09025_b200 import errors, lwe, network

pytestmark = pytest.mark.gpu


def test_layer_forward_identity_pool_and_conv(toy, toy_keys, toy64, toy64_keys):
    sk, _, _ = toy_keys
    rng = np.random.default_rng(4)
    m, shape = network.conv_matrix(np.ones((1, 1, 1, 1), dtype=np.int64), (1, 3, 3), (1, 1), (0, 0))
    msgs = rng.integers(0, 2, 9)
    A, b = lwe.encrypt_batch(msgs, sk, toy, rng)
    out = network.layer_forward(network.CiphertextTensor((1, 3, 3), A, b, toy.q),
                                network.WeightLayer("conv2d", m, m.astype(float), 1.0, shape), toy)
    assert np.array_equal(lwe.decrypt_batch(out.A, out.b, sk, toy), msgs)
    m, shape = network.pool_matrix((1, 2, 2), (2, 2))
    A, b = lwe.encrypt_batch(np.array([0, 2, 2, 0]), sk, toy, rng)
    out = network.layer_forward(network.CiphertextTensor((1, 2, 2), A, b, toy.q),
                                network.WeightLayer("avgpool", m, m.astype(float), 1.0, shape), toy)
    assert lwe.decrypt_batch(out.A, out.b, sk, toy)[0] == 4
    sk64, _, _ = toy64_keys
    w = rng.integers(-2, 3, (2, 1, 2, 2))
    m, shape = network.conv_matrix(w, (1, 4, 4), (2, 2), (0, 0))
    layer = network.WeightLayer("conv2d", m, m.astype(float), 1.0, shape)
    xs = []
    for _ in range(10):
        msgs = rng.integers(0, 3, 16)
        A, b = lwe.encrypt_batch(msgs, sk64, toy64, rng)
        xs.append((msgs, network.CiphertextTensor((1, 4, 4), A, b, toy64.q)))
    outs = network.layer_forward_batch([x for _, x in xs], layer, toy64)
    for (msgs, _), out in zip(xs, outs):
        assert np.array_equal(lwe.decrypt_batch(out.A, out.b, sk64, toy64), m @ msgs)
    st = network.layer_forward_batch([x for _, x in xs], layer, toy64, stack=True)
    assert st.shape == (10, *layer.out_shape)
    assert np.array_equal(st.A, np.concatenate([o.A for o in outs])) and np.array_equal(st.b, np.concatenate([o.b for o in outs]))


@pytest.fixture(scope="module")
def small_net():
    """input 1x2x2 -> linear 4 -> spiking -> linear 3 -> spiking (IF), T=2."""
    rng = np.random.default_rng(7)
    model = network.CsnnModel(
        arch=({"type": "linear", "out_features": 4}, {"type": "spiking"},
              {"type": "linear", "out_features": 3}, {"type": "spiking"}),
        weights=(rng.normal(0, 0.5, (4, 4)), rng.normal(0, 0.5, (3, 4))),
        input_shape=(1, 2, 2), T=2, L=1, tau=None)
    return network.discretize(model, 4)


def test_inference_semantics(toy64, toy64_keys, small_net):
    sk, _, bsk = toy64_keys
    rng = np.random.default_rng(9)
    # zero input -> zero spikes
    enc = network.encrypt_image(np.zeros((2, 2)), 1, sk, toy64, rng)
    scores, _ = network.infer(enc, small_net, bsk)
    assert not np.any(lwe.decrypt_batch(scores.A, scores.b, sk, toy64))
    # matches the integer plain path (device twin) on random images, batched
    imgs = [rng.random((2, 2)) for _ in range(5)]
    encs = [network.encrypt_image(img, 1, sk, toy64, rng) for img in imgs]
    batch_scores, _ = network.infer_batch(encs, small_net, bsk)
    plain, _ = network.plain_infer_batch(np.stack(imgs), small_net, toy64, p=toy64.p)
    for k in range(5):
        assert np.array_equal(lwe.decrypt_batch(batch_scores[k].A, batch_scores[k].b, sk, toy64), plain[k])
        # batch position does not change the ciphertexts (serial single-image run)
        single, _ = network.infer(encs[k], small_net, bsk)
        assert np.array_equal(single.A, batch_scores[k].A) and np.array_equal(single.b, batch_scores[k].b)
    # bootstrap counts and the score range for T = 1, 2, 3
    for T in (1, 2, 3):
        s, stats = network.infer(encs[0], small_net, bsk, T=T)
        assert stats.bootstrap_count == 2 * (4 + 3) * T
        dec = lwe.decrypt_batch(s.A, s.b, sk, toy64)
        assert np.all(dec % 2 == 0) and np.all((0 <= dec) & (dec <= 2 * T))
    with pytest.raises(errors.ParameterError):
        network.infer(encs[0], small_net, bsk, T=0)


def test_classify_ties_and_unique_max(toy, toy_keys):
    sk, _, _ = toy_keys
    rng = np.random.default_rng(13)
    A, b = lwe.encrypt_batch(np.zeros(10, dtype=np.int64), sk, toy, rng)
    assert network.classify(network.CiphertextTensor((10,), A, b, toy.q), sk, toy) == 0
    scores = np.zeros(10, dtype=np.int64)
    scores[7] = 2
    A, b = lwe.encrypt_batch(scores, sk, toy, rng)
    assert network.classify(network.CiphertextTensor((10,), A, b, toy.q), sk, toy) == 7
