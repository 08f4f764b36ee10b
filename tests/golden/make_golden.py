"""Generate golden vectors by running the REFERENCE implementation.

Build-container only: imports the read-only reference package from
/root/reference/pkg/src (it does not exist on the GPU box).  Writes small
.npz fixtures next to this script; the parity tests load them without the
reference.  Run:

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \
        python tests/golden/make_golden.py [section ...]

Sections: keys toy toy64 desk c4 layer config0 config1 config2 config4 fdsn plain paper ring
"""

from __future__ import annotations

import hashlib
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, os.path.join(ROOT, "tools"))
sys.path.insert(0, "/root/reference/pkg/src")

import fdsnn  # noqa: E402  (the reference)
import workloads as W  # noqa: E402
from dataclasses import replace  # noqa: E402


def sha(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(np.asarray(a, dtype=np.int64)).tobytes())
    return h.hexdigest()


def key_rows(bsk):
    return np.stack([np.stack([e.rows_a, e.rows_b], axis=1) for e in bsk.ek])


def save(name, **arrays):
    path = os.path.join(HERE, name + ".npz")
    np.savez_compressed(path, **arrays)
    print(f"wrote {path} ({os.path.getsize(path) / 1024:.1f} KiB)")


def toy():
    return fdsnn.params.preset("TOY")


def toy64():
    return replace(fdsnn.params.preset("TOY"), p=64, sigma=2.0, preset_name="custom")


def sec_keys():
    """Key digests per (params, seed): pins the host key generator's RNG order."""
    out = {}
    for name, prm, seed in (("toy", toy(), 1), ("toy64", toy64(), 2),
                            ("desk1024", W.desk1024(fdsnn), 0), ("c4", W.c4_params(fdsnn), 0)):
        sk, zk, bsk = W.keys(fdsnn, prm, seed)
        out[name] = {"seed": seed, "sk": sha(sk.s), "zk": sha(zk.z), "rows": sha(key_rows(bsk)),
                     "ksk_A": sha(bsk.ksk.A), "ksk_b": sha(bsk.ksk.b), "params_digest": prm.digest()}
    with open(os.path.join(HERE, "keys.json"), "w") as f:
        json.dump(out, f, indent=1)
    print("wrote keys.json")


def sec_toy():
    prm = toy()
    sk, zk, bsk = W.keys(fdsnn, prm, 1)
    rng = np.random.default_rng(11)
    ms = np.repeat(np.arange(-prm.p // 2 + 1, prm.p // 2 + 1), 8)
    A, b = fdsnn.lwe.encrypt_batch(ms, sk, prm, rng)
    g = fdsnn.neuron.g_fire(prm.p)
    fA, fb = fdsnn.bootstrap.bootstrap_batch(g, A, b, bsk)
    rl = fdsnn.bootstrap.make_program(dict(enumerate(rng.integers(-3, 5, prm.p // 2))), prm.p)
    rA, rb = fdsnn.bootstrap.bootstrap_batch(rl, A, b, bsk)
    acc = rng.integers(0, prm.q, (5, 2, prm.N))
    a2N = rng.integers(0, 2 * prm.N, (5, prm.n))
    a2N[0] = 0
    br = fdsnn.bootstrap.blind_rotate_batch(acc.copy(), a2N, bsk)
    kA = rng.integers(-prm.q, prm.q, (9, prm.N))
    kb = rng.integers(0, prm.q, 9)
    ksA, ksb = fdsnn.bootstrap.key_switch_batch(kA, kb, bsk.ksk, prm)
    save("toy", ms=ms, A=A, b=b, fire_A=fA, fire_b=fb, lut=rl.table, lut_A=rA, lut_b=rb,
         acc=acc, a2N=a2N, br=br, ks_in_A=kA, ks_in_b=kb, ks_A=ksA, ks_b=ksb)


def sec_toy64():
    prm = toy64()
    sk, zk, bsk = W.keys(fdsnn, prm, 2)
    rng = np.random.default_rng(21)
    lif = fdsnn.neuron.LifParams(tau=2, theta=5)
    v = rng.integers(0, lif.v_th_hat, 64)
    i = rng.integers(-20, 21, 64)
    vA, vb = fdsnn.lwe.encrypt_batch(v, sk, prm, rng)
    iA, ib = fdsnn.lwe.encrypt_batch(i, sk, prm, rng)
    sA, sb, nA, nb = fdsnn.neuron.fhe_lif_step_batch(vA, vb, iA, ib, lif, bsk)
    # tiny network (test_network.py:166-175 shape): 2x2 -> linear 4 -> spiking -> linear 3 -> spiking
    model = fdsnn.network.CsnnModel(
        arch=({"type": "linear", "out_features": 4}, {"type": "spiking"},
              {"type": "linear", "out_features": 3}, {"type": "spiking"}),
        weights=(np.random.default_rng(7).normal(0, 0.5, (4, 4)),
                 np.random.default_rng(8).normal(0, 0.5, (3, 4))),
        input_shape=(1, 2, 2), T=2, L=1, tau=None)
    net = fdsnn.network.discretize(model, 4)
    imgs = rng.random((3, 2, 2))
    encs = [fdsnn.network.encrypt_image(im, 1, sk, prm, rng) for im in imgs]
    scores = [fdsnn.network.infer(e, net, bsk) for e in encs]
    mats = [l.matrix for l in net.layers if hasattr(l, "matrix")]
    save("toy64", v=v, i=i, vA=vA, vb=vb, iA=iA, ib=ib, sA=sA, sb=sb, nA=nA, nb=nb,
         m1=mats[0], m2=mats[1], theta=net.theta,
         img_A=np.stack([e.A for e in encs]), img_b=np.stack([e.b for e in encs]),
         score_A=np.stack([s[0].A for s in scores]), score_b=np.stack([s[0].b for s in scores]),
         boots=np.array([s[1].bootstrap_count for s in scores]))


def sec_lif(prm, name, count, seed_in=31):
    sk, zk, bsk = W.keys(fdsnn, prm, 0)
    lif = W.lif_for(fdsnn, prm)
    rng = np.random.default_rng(seed_in)
    v = rng.integers(0, lif.v_th_hat, count)
    i = rng.integers(-prm.p // 2 + 1, prm.p // 2 - lif.v_th_hat, count)
    vA, vb = fdsnn.lwe.encrypt_batch(v, sk, prm, rng)
    iA, ib = fdsnn.lwe.encrypt_batch(i, sk, prm, rng)
    t0 = time.time()
    sA, sb, nA, nb = fdsnn.neuron.fhe_lif_step_batch(vA, vb, iA, ib, lif, bsk)
    print(f"{name}: {2 * count} PBS in {time.time() - t0:.1f}s")
    save(name, v=v, i=i, vA=vA.astype(np.int32), vb=vb, iA=iA.astype(np.int32), ib=ib,
         sA=sA.astype(np.int32), sb=sb, nA=nA.astype(np.int32), nb=nb,
         spike=fdsnn.lwe.decrypt_batch(sA, sb, sk, prm), state=fdsnn.lwe.decrypt_batch(nA, nb, sk, prm))


def sec_layer():
    prm = W.desk1024(fdsnn)
    sk, zk, bsk = W.keys(fdsnn, prm, 0)
    rng = np.random.default_rng(41)
    w = rng.integers(-7, 8, (3, 1, 3, 3))
    mc, shape = fdsnn.network.conv_matrix(w, (1, 6, 6), (1, 1), (0, 0))
    md = rng.integers(-15, 16, (20, 36))
    ms = rng.integers(0, 2, 36)
    A, b = fdsnn.lwe.encrypt_batch(ms, sk, prm, rng)
    x = fdsnn.network.CiphertextTensor((1, 6, 6), A, b, prm.q)
    conv = fdsnn.network.layer_forward(x, fdsnn.network.WeightLayer("conv2d", mc, None, 1.0, shape), prm)
    dense = fdsnn.network.layer_forward(x, fdsnn.network.WeightLayer("linear", md, None, 1.0, (20,)), prm)
    save("layer", conv_m=mc, dense_m=md, ms=ms, A=A.astype(np.int32), b=b,
         conv_A=conv.A.astype(np.int32), conv_b=conv.b, dense_A=dense.A.astype(np.int32), dense_b=dense.b)


def sec_config0():
    """Config 0: 1024 LIF bootstraps (fire + reset = 2048 PBS) at DESK p=1024."""
    prm = W.desk1024(fdsnn)
    sk, zk, bsk = W.keys(fdsnn, prm, 0)
    lif = W.lif_for(fdsnn, prm)
    ms = W.pbs_messages(prm, 1024)
    A, b = W.encrypt(fdsnn, prm, sk, ms)
    t0 = time.time()
    sA, sb = fdsnn.neuron.fhe_fire_batch(A, b, lif, bsk)
    nA, nb = fdsnn.neuron.fhe_reset_batch(A, b, lif, bsk)
    dt = time.time() - t0
    print(f"config0: 2048 PBS in {dt:.1f}s ({2048 / dt:.1f} PBS/s)")
    save("config0", ms=ms, in_digest=np.frombuffer(bytes.fromhex(sha(A, b)), np.uint8),
         out_digest=np.frombuffer(bytes.fromhex(sha(sA, sb, nA, nb)), np.uint8),
         spike=fdsnn.lwe.decrypt_batch(sA, sb, sk, prm), state=fdsnn.lwe.decrypt_batch(nA, nb, sk, prm),
         sA64=sA[:64].astype(np.int32), sb64=sb[:64], nA64=nA[:64].astype(np.int32), nb64=nb[:64],
         ref_seconds=np.array([dt]))


def sec_config1():
    """Config 1: 16 samples x 784 Bernoulli(0.15) spikes per t, FC 784->128 [-15,15], LIF, T=4."""
    prm = W.desk1024(fdsnn)
    sk, zk, bsk = W.keys(fdsnn, prm, 0)
    lif = W.lif_for(fdsnn, prm)
    x = W.config1_inputs()
    Wm = W.config1_weights()
    T, B, C = x.shape
    A, b = W.encrypt(fdsnn, prm, sk, x.ravel())
    A = A.reshape(T, B, C, prm.n)
    b = b.reshape(T, B, C)
    layer = fdsnn.network.WeightLayer("linear", Wm, None, 1.0, (128,))
    states = [fdsnn.network.zero_states(128, prm) for _ in range(B)]
    spikes = np.zeros((T, B, 128), np.int64)
    digests = []
    t0 = time.time()
    for t in range(T):
        outs = []
        for s in range(B):
            cur = fdsnn.network.layer_forward(
                fdsnn.network.CiphertextTensor((C,), A[t, s], b[t, s], prm.q), layer, prm)
            sp, states[s] = fdsnn.network.spiking_forward(cur, states[s], lif, bsk)
            spikes[t, s] = fdsnn.lwe.decrypt_batch(sp.A, sp.b, sk, prm)
            outs += [sp.A, sp.b, states[s].A, states[s].b]
        digests.append(sha(*outs))
    dt = time.time() - t0
    print(f"config1: {2 * 128 * B * T} PBS in {dt:.1f}s")
    final_state = np.stack([fdsnn.lwe.decrypt_batch(s.A, s.b, sk, prm) for s in states])
    save("config1", spikes=spikes, final_state=final_state,
         step_digests=np.stack([np.frombuffer(bytes.fromhex(d), np.uint8) for d in digests]),
         ref_seconds=np.array([dt]))


def sec_config2():
    """Config 2: one synthetic image through conv(8x5x5)->LIF->FC 4608->128->LIF->FC 128->10->LIF, T=4."""
    prm = W.desk1024(fdsnn)
    sk, zk, bsk = W.keys(fdsnn, prm, 0)
    lif = W.lif_for(fdsnn, prm)
    net = W.config2_network(fdsnn, lif)
    imgs = W.synth_images(32)
    encs = W.encrypt_images(fdsnn, prm, sk, imgs[:1])
    spikes = {}

    def obs(li, t, x):
        spikes[f"l{li}_t{t}"] = fdsnn.lwe.decrypt_batch(x.A, x.b, sk, prm)

    t0 = time.time()
    scores, stats = fdsnn.network.infer(encs[0], net, bsk, workers=8, observer=obs)
    dt = time.time() - t0
    print(f"config2 image 0: {stats.bootstrap_count} PBS in {dt:.1f}s")
    save("config2_img0", scores=fdsnn.lwe.decrypt_batch(scores.A, scores.b, sk, prm),
         score_digest=np.frombuffer(bytes.fromhex(sha(scores.A, scores.b)), np.uint8),
         boots=np.array([stats.bootstrap_count]), ref_seconds=np.array([dt]), **spikes)


def sec_config4():
    """Config 4 (C4 params, p=4096): one synthetic image through
    conv(8x5x5)->LIF->FC 4608->256->LIF->256->128->LIF->128->10->LIF, T=8,
    through the reference's encrypted infer (network.py:459-491), 80,032 PBS."""
    prm = W.c4_params(fdsnn)
    sk, zk, bsk = W.keys(fdsnn, prm, 0)
    lif = W.lif_for(fdsnn, prm)
    net = W.config4_network(fdsnn, lif)
    imgs = W.synth_images(32)
    encs = W.encrypt_images(fdsnn, prm, sk, imgs[:1])
    spikes = {}

    def obs(li, t, x):
        spikes[f"l{li}_t{t}"] = fdsnn.lwe.decrypt_batch(x.A, x.b, sk, prm)

    t0 = time.time()
    scores, stats = fdsnn.network.infer(encs[0], net, bsk, workers=8, observer=obs)
    dt = time.time() - t0
    print(f"config4 image 0: {stats.bootstrap_count} PBS in {dt:.1f}s")
    save("config4_img0", scores=fdsnn.lwe.decrypt_batch(scores.A, scores.b, sk, prm),
         score_digest=np.frombuffer(bytes.fromhex(sha(scores.A, scores.b)), np.uint8),
         boots=np.array([stats.bootstrap_count]), ref_seconds=np.array([dt]), **spikes)


def sec_plain():
    """Reference oracle.plain_infer (oracle.py:44-78) on the config 2 network
    (32 synthetic images, T=4) and the config 4 network (32 images, T=8):
    integer scores and per-layer spike counts, plus whether the strict range
    check at p raises."""
    out = {}
    for tag, prm, mk, nimg in (("c2", W.desk1024(fdsnn), W.config2_network, 32),
                               ("c4", W.c4_params(fdsnn), W.config4_network, 32)):
        lif = W.lif_for(fdsnn, prm)
        net = mk(fdsnn, lif)
        imgs = W.synth_images(nimg).astype(np.float64) / 255.0
        scores, counts = [], None
        for img in imgs:
            sc, tr = fdsnn.oracle.plain_infer(net, img)
            scores.append(sc)
            c = [np.asarray(s2).sum(axis=0) // 2 for s2 in tr.spike2]
            counts = [[x] for x in c] if counts is None else [a + [x] for a, x in zip(counts, c)]
        out[f"{tag}_scores"] = np.stack(scores)
        for li, c in enumerate(counts):
            out[f"{tag}_counts{li}"] = np.stack(c)
        raised = 0
        for img in imgs:
            try:
                fdsnn.oracle.plain_infer(net, img, p=prm.p)
            except fdsnn.errors.OverflowViolation:
                raised += 1
        out[f"{tag}_overflow_images"] = np.array([raised])
        print(tag, "scores", out[f"{tag}_scores"][0], "overflowing images at p:", raised)
    save("plain", **out)


def sec_paper():
    """The paper's own network: the reference fixture model model_if_t2.json
    (conv 10x8x8/2 -> IF -> avgpool 2 -> fc 360->160 -> IF -> fc 160->10 -> IF,
    T=2) discretized at theta=40 on DESK with p=2048 (the parameter set of the
    reference's desk_eval.json, digest d71006c1...), keys seed 0, two synthetic
    images.  Saves the model weights (with the fixture's sha256) and the
    reference's encrypted-inference outputs."""
    path = "/root/reference/pkg/tests/fixtures/model_if_t2.json"
    with open(path, "rb") as f:
        model_sha = hashlib.sha256(f.read()).hexdigest()
    model = fdsnn.network.CsnnModel.load(path)
    net = fdsnn.network.discretize(model, 40)
    prm = fdsnn.params.preset("DESK").with_p(2048)
    sk, zk, bsk = W.keys(fdsnn, prm, 0)
    imgs = W.synth_images(2)
    encs = W.encrypt_images(fdsnn, prm, sk, imgs)
    out = {}
    for k, enc in enumerate(encs):
        t0 = time.time()
        scores, stats = fdsnn.network.infer(enc, net, bsk, workers=8)
        print(f"paper image {k}: {stats.bootstrap_count} PBS in {time.time() - t0:.1f}s")
        out[f"score_digest{k}"] = np.frombuffer(bytes.fromhex(sha(scores.A, scores.b)), np.uint8)
        out[f"scores{k}"] = fdsnn.lwe.decrypt_batch(scores.A, scores.b, sk, prm)
        out[f"boots{k}"] = np.array([stats.bootstrap_count])
        plain, _ = fdsnn.oracle.plain_infer(net, imgs[k].astype(np.float64) / 255.0, p=prm.p)
        out[f"plain{k}"] = plain
    save("paper", model_sha256=np.frombuffer(bytes.fromhex(model_sha), np.uint8),
         params_digest=np.frombuffer(bytes.fromhex(prm.digest()), np.uint8), **out)
    w = {f"w{i}": np.asarray(x, np.float64) for i, x in enumerate(model.weights)}
    save("paper_model", T=np.array([model.T]), L=np.array([model.L]), v_th=np.array([model.v_th]),
         model_sha256=np.frombuffer(bytes.fromhex(model_sha), np.uint8), **w)


def sec_fdsn():
    """sha256 of FDSN containers written by the reference (TOY keys seed 1)."""
    import tempfile
    prm = toy()
    sk, zk, bsk = W.keys(fdsnn, prm, 1)
    rng = np.random.default_rng(51)
    A, b = fdsnn.lwe.encrypt_batch(rng.integers(-3, 5, 12), sk, prm, rng)
    ct = fdsnn.network.CiphertextTensor((3, 4), A, b, prm.q)
    out = {}
    with tempfile.TemporaryDirectory() as d:
        paths = {"sk": os.path.join(d, "sk.bin"), "bk": os.path.join(d, "bk.bin"),
                 "ct": os.path.join(d, "ct.bin")}
        fdsnn.serial.save_secret_key(paths["sk"], sk, zk, prm)
        fdsnn.serial.save_bootstrap_key(paths["bk"], bsk)
        fdsnn.serial.save_ciphertexts(paths["ct"], ct, prm)
        for k, pth in paths.items():
            out[k] = fdsnn.serial.file_digest(pth)
    out["ct_seed"] = 51
    with open(os.path.join(HERE, "fdsn.json"), "w") as f:
        json.dump(out, f, indent=1)
    print("wrote fdsn.json")


def sec_ring():
    """Algebra layer: negacyclic transform, products, digits, external product."""
    from fdsnn import params as P, rgsw, ring
    rng = np.random.default_rng(61)
    out = {}
    for N in (2, 8, 64, 1024, 2048):
        a = rng.integers(-(1 << 24), 1 << 24, (2 if N < 1024 else 1, N))
        tr = ring.NegacyclicTransform(N)
        f = tr.forward(a)
        out[f"nt{N}_in"], out[f"nt{N}_fwd"], out[f"nt{N}_inv"] = a, f, tr.inverse(f)
    for name, N, q, bmax in (("desk", 1024, 1 << 25, 1 << 12), ("c4", 2048, 1 << 24, 1 << 7), ("tiny", 8, 1 << 12, 1 << 12)):
        a = rng.integers(0, q, N)
        b = rng.integers(-bmax, bmax + 1, N)
        pa, pb = ring.NegacyclicPoly(a, q), ring.NegacyclicPoly(b, q)
        out[f"mul_{name}_a"], out[f"mul_{name}_b"] = a, b
        out[f"mul_{name}_q"] = np.array([q])
        out[f"mul_{name}_out"] = ring.poly_mul(pa, pb).coeffs
    for name, q, base, levels in (("desk", 1 << 25, 1 << 13, 2), ("c4", 1 << 24, 1 << 8, 3), ("small", 1 << 12, 1 << 6, 2)):
        x = np.concatenate([rng.integers(0, q, 4000), [0, 1, q - 1, q // 2, q // 2 - 1, q // 2 + 1]])
        out[f"dig_{name}_x"] = x
        out[f"dig_{name}_prm"] = np.array([q, base, levels])
        out[f"dig_{name}_out"] = rgsw.gadget_decompose(x, q, P.GadgetParams(base=base, levels=levels))
    small = P.FheParams(n=4, q=1 << 12, N=64, p=8, sigma=1e-9, gadget=P.GadgetParams(base=1 << 6, levels=2),
                        ks_base=8, ks_levels=4, sigma_bk=1e-9, sigma_ks=1e-9)
    for name, prm, k in (("small", small, 37), ("desk", W.desk1024(fdsnn), 700)):
        erng = np.random.default_rng(62)
        zk = rgsw.rlwe_keygen(prm, erng)
        m = ring.NegacyclicPoly(erng.integers(0, prm.p, prm.N), prm.p)
        ct = rgsw.rlwe_encrypt(m, zk, prm, erng)
        g = rgsw.rgsw_encrypt_monomial(k, zk, prm, erng)
        res = rgsw.external_product(ct, g, prm)
        out[f"ext_{name}_ct"] = np.stack([ct.a, ct.b])
        out[f"ext_{name}_rows"] = np.stack([g.rows_a, g.rows_b])
        out[f"ext_{name}_gadget"] = np.array([prm.q, prm.gadget.base, prm.gadget.levels, prm.N])
        out[f"ext_{name}_out"] = np.stack([res.a, res.b])
        out[f"ext_{name}_z"] = zk.z
    save("ring", **out)


SECTIONS = {
    "fdsn": sec_fdsn,
    "keys": sec_keys, "toy": sec_toy, "toy64": sec_toy64,
    "desk": lambda: sec_lif(W.desk1024(fdsnn), "desk_lif", 32),
    "c4": lambda: sec_lif(W.c4_params(fdsnn), "c4_lif", 4),
    "layer": sec_layer, "config0": sec_config0, "config1": sec_config1, "config2": sec_config2,
    "config4": sec_config4,
    "plain": sec_plain, "paper": sec_paper, "ring": sec_ring,
}

if __name__ == "__main__":
    for name in sys.argv[1:] or [k for k in SECTIONS if k not in ("config2", "config4")]:
        SECTIONS[name]()
