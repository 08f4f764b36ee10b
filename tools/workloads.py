"""Seeded synthetic workloads for BASELINE.json configs 0-4.

The reference's own datasets (pkg/data, MNIST) are absent; these generators
stand in for them with the shapes, sizes and value distributions the configs
name.  They depend only on numpy and take an `api` module bundle, so the same
code builds the inputs for the reference package (golden generation, build
container only) and for this package (tests, bench) with identical RNG draws.

RNG streams: keys seed 0, plaintext inputs seed 1, weights seed 2,
encryption randomness seed 3, images seed 4.
"""

from __future__ import annotations

import numpy as np

KEY_SEED, INPUT_SEED, WEIGHT_SEED, ENC_SEED, IMAGE_SEED = 0, 1, 2, 3, 4


def desk1024(api):
    return api.params.preset("DESK").with_p(1024)


def c4_params(api):
    """Config-4 parameters; q = 2^24 forced by Bg^l >= q (params.py:71-74)."""
    P = api.params
    return P.FheParams(n=742, q=1 << 24, N=2048, p=4096, sigma=0.25,
                       gadget=P.GadgetParams(1 << 8, 3), ks_base=1 << 3, ks_levels=8,
                       sigma_bk=1.0 / 64, sigma_ks=1.0 / 64)


def keys(api, prm, seed=KEY_SEED):
    """lwe_keygen, rlwe_keygen, gen_bootstrap_key in the CLI order (cli.py:61-64)."""
    rng = np.random.default_rng(seed)
    sk = api.lwe.lwe_keygen(prm, rng)
    zk = api.rgsw.rlwe_keygen(prm, rng)
    bsk = api.bootstrap.gen_bootstrap_key(sk, zk, prm, rng)
    return sk, zk, bsk


def lif_for(api, prm):
    theta = 256 if prm.p == 4096 else 64
    return api.neuron.LifParams(tau=2, theta=theta)  # v_th_hat = P/8


# ---------------------------------------------------------------- config 0/3

def pbs_messages(prm, count, seed=INPUT_SEED):
    """m ~ U{-p/2 .. p/2-1}, -p/2 mapped to +p/2 (same residue; lwe.py:79-80)."""
    rng = np.random.default_rng(seed)
    m = rng.integers(-prm.p // 2, prm.p // 2, count)
    m[m == -prm.p // 2] = prm.p // 2
    return m


def encrypt(api, prm, sk, msgs, seed=ENC_SEED):
    return api.lwe.encrypt_batch(np.asarray(msgs), sk, prm, np.random.default_rng(seed))


# ------------------------------------------------------------------ config 1

def config1_inputs(T=4, batch=16, cells=784, p_spike=0.15, seed=INPUT_SEED):
    rng = np.random.default_rng(seed)
    return (rng.random((T, batch, cells)) < p_spike).astype(np.int64)


def config1_weights(out=128, cells=784, seed=WEIGHT_SEED):
    return np.random.default_rng(seed).integers(-15, 16, (out, cells)).astype(np.int64)


# ---------------------------------------------------------------- config 2/4

def synth_images(count, seed=IMAGE_SEED, size=28, target=0.20):
    """Zero canvas, 3-6 thick random polyline strokes (brush radius 1-2 px),
    stroke pixels U{128..255}, strokes added until ~20% of pixels are set."""
    rng = np.random.default_rng(seed)
    imgs = np.zeros((count, size, size), dtype=np.uint8)
    yy, xx = np.mgrid[0:size, 0:size]
    for k in range(count):
        img = imgs[k]
        strokes = int(rng.integers(3, 7))
        s = 0
        while s < strokes or (img > 0).mean() < target - 0.02:
            if (img > 0).mean() >= target + 0.02:
                break
            radius = float(rng.integers(1, 3))
            pt = rng.uniform(4, size - 4, 2)
            for _ in range(int(rng.integers(2, 5))):
                ang = rng.uniform(0, 2 * np.pi)
                length = rng.uniform(3, 9)
                end = np.clip(pt + length * np.array([np.sin(ang), np.cos(ang)]), 2, size - 3)
                for f in np.linspace(0, 1, 12):
                    cy, cx = pt + f * (end - pt)
                    mask = (yy - cy) ** 2 + (xx - cx) ** 2 <= radius ** 2
                    img[mask & (img == 0)] = rng.integers(128, 256, int((mask & (img == 0)).sum()))
                pt = end
            s += 1
    return imgs


def _conv(api, w, in_shape):
    m, shape = api.network.conv_matrix(w, in_shape, (1, 1), (0, 0))
    return m.astype(np.int64), shape


def config2_network(api, lif, seed=WEIGHT_SEED):
    """conv 8x1x5x5 [-7,7] -> spiking -> fc 4608->128 [-15,15] -> spiking -> fc 128->10 -> spiking."""
    N = api.network
    rng = np.random.default_rng(seed)
    w_conv = rng.integers(-7, 8, (8, 1, 5, 5))
    w1 = rng.integers(-15, 16, (128, 4608))
    w2 = rng.integers(-15, 16, (10, 128))
    mc, shape = _conv(api, w_conv, (1, 28, 28))
    layers = (N.WeightLayer("conv2d", mc, None, 1.0, shape), N.SpikingLayer(lif, shape),
              N.WeightLayer("linear", w1.astype(np.int64), None, 1.0, (128,)), N.SpikingLayer(lif, (128,)),
              N.WeightLayer("linear", w2.astype(np.int64), None, 1.0, (10,)), N.SpikingLayer(lif, (10,)))
    return N.DiscretizedNetwork(layers, lif.theta, 1, lif, 4)


def config4_network(api, lif, seed=WEIGHT_SEED):
    """conv 8x5x5 [-63,63] -> spiking -> 4608->256 -> spiking -> 256->128 -> spiking -> 128->10 -> spiking."""
    N = api.network
    rng = np.random.default_rng(seed)
    w_conv = rng.integers(-63, 64, (8, 1, 5, 5))
    ws = [rng.integers(-63, 64, s) for s in ((256, 4608), (128, 256), (10, 128))]
    mc, shape = _conv(api, w_conv, (1, 28, 28))
    layers = [N.WeightLayer("conv2d", mc, None, 1.0, shape), N.SpikingLayer(lif, shape)]
    for w in ws:
        layers += [N.WeightLayer("linear", w.astype(np.int64), None, 1.0, (w.shape[0],)),
                   N.SpikingLayer(lif, (w.shape[0],))]
    return N.DiscretizedNetwork(tuple(layers), lif.theta, 1, lif, 8)


def encrypt_images(api, prm, sk, imgs, seed=ENC_SEED):
    """Quantize with L=1 (pixel/255 -> {0,1}) and encrypt cell-wise, one rng for all images."""
    rng = np.random.default_rng(seed)
    return [api.network.encrypt_image(img.astype(np.float64) / 255.0, 1, sk, prm, rng) for img in imgs]


def layers_for_oracle(net):
    """DiscretizedNetwork -> oracle layer tuples."""
    out = []
    for layer in net.layers:
        if hasattr(layer, "matrix"):
            out.append(("weight", np.asarray(layer.matrix, np.int64)))
        else:
            lif = layer.lif
            out.append(("spike", lif.v_th_hat, lif.leak_num, lif.leak_den))
    return out
