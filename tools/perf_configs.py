"""Throughput of configs 2-4 on the device (development/report aid):
config 3 PBS sweep, config 2 (32 images, T=4) and config 4 (C4 params, T=8)
encrypted inferences per second, and the C4 LIF PBS rate."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tools"))
import numpy as np
import torch
import workloads as W
import paper_2309_09025_b200 as api
from paper_2309_09025_b200 import bootstrap, network, neuron

out = {}
which = sys.argv[1:] or ["c0", "c3", "c2", "c4"]
if "c0" in which or "c3" in which or "c2" in which:
    prm = W.desk1024(api)
    sk, zk, bsk = W.keys(api, prm)
    dev = bsk.device
    g = neuron.g_fire(prm.p)
    lut = dev.lut(bootstrap.test_polynomial(g, prm))
if "c0" in which:
    # config 0: 1024 LIF bootstraps (fire + reset = 2048 PBS with key switch), one fused launch
    lif0 = W.lif_for(api, prm)
    A0, b0 = W.encrypt(api, prm, sk, W.pbs_messages(prm, 1024))
    zeros = np.zeros_like(A0), np.zeros_like(b0)
    neuron.fhe_lif_step_batch(zeros[0], zeros[1], A0, b0, lif0, bsk)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    reps = 5
    for _ in range(reps):
        neuron.fhe_lif_step_batch(zeros[0], zeros[1], A0, b0, lif0, bsk)
    dt = (time.perf_counter() - t0) / reps
    out["config0"] = {"pbs": 2048, "ms_host_to_host": dt * 1e3, "pbs_per_s": 2048 / dt}
if "c3" in which:
    peak_tf = dev.fp64_peak_tflops()
    hbm_gbs, hbm_src = 7400.0, "B200_PROFILING.md fallback"
    mp = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")
    if os.path.exists(mp):
        try:
            d = json.load(open(mp))
            for k, v in d.items():
                if "hbm" in k.lower() and isinstance(v, (int, float)):
                    hbm_gbs, hbm_src = float(v), f"MEASURED_PEAKS.json:{k}"
                    break
        except Exception:
            pass
    sweep = {}
    for B in (1, 64, 1024, 16384, 131072):
        ms = W.pbs_messages(prm, B, seed=B)
        A, b = W.encrypt(api, prm, sk, ms)
        rows = dev.rows_from_host(A, b)
        dev.pbs_dev([lut], [0], [0], rows)
        torch.cuda.synchronize()
        reps = 3 if B <= 16384 else 1
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            dev.pbs_dev([lut], [0], [0], rows)
        e1.record(); torch.cuda.synchronize()
        ms_ = e0.elapsed_time(e1) / reps
        # roofline of the whole PBS launch (blind rotation + key switch): FP64
        # work 87.56 MFLOP/PBS vs the live DFMA peak; bytes = BSK + KSK read
        # once per launch + input/output ciphertext rows
        flops = B * 87556096
        nbytes = (prm.n * 2 * prm.gadget.levels * 2 * (prm.N // 2) * 16
                  + prm.N * prm.ks_levels * (prm.n + 1) * 4 + B * 2 * dev.stride * 4)
        t_fp64 = flops / (peak_tf * 1e12)
        t_hbm = nbytes / (hbm_gbs * 1e9)
        sweep[B] = {"ms": ms_, "pbs_per_s": B / ms_ * 1e3,
                    "fp64_tflops": flops / (ms_ * 1e-3) / 1e12, "hbm_gbs": nbytes / (ms_ * 1e-3) / 1e9,
                    "bound": "fp64" if t_fp64 >= t_hbm else "hbm",
                    "roofline_frac": max(t_fp64, t_hbm) / (ms_ * 1e-3)}
    out["config3_sweep"] = sweep
    out["config3_peaks"] = {"fp64_tflops": peak_tf, "hbm_gbs": hbm_gbs, "hbm_source": hbm_src}
if "c2" in which:
    lif = W.lif_for(api, prm)
    net = W.config2_network(api, lif)
    imgs = W.synth_images(32)
    encs = W.encrypt_images(api, prm, sk, imgs)
    network.infer_batch(encs[:2], net, bsk)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    scores, stats = network.infer_batch(encs, net, bsk)
    dt = time.perf_counter() - t0
    out["config2"] = {"images": 32, "seconds": dt, "inferences_per_s": 32 / dt, "pbs": stats.bootstrap_count,
                      "pbs_per_s": stats.bootstrap_count / dt}
if "c4" in which:
    prm4 = W.c4_params(api)
    sk4, zk4, bsk4 = W.keys(api, prm4)
    lif4 = W.lif_for(api, prm4)
    net4 = W.config4_network(api, lif4)
    imgs = W.synth_images(32)
    encs = W.encrypt_images(api, prm4, sk4, imgs)
    network.infer_batch(encs[:1], net4, bsk4, T=1)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    scores, stats = network.infer_batch(encs, net4, bsk4)
    dt = time.perf_counter() - t0
    out["config4"] = {"images": 32, "seconds": dt, "inferences_per_s": 32 / dt, "pbs": stats.bootstrap_count,
                      "pbs_per_s": stats.bootstrap_count / dt}
print(json.dumps(out))
