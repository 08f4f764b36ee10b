#!/usr/bin/env python
"""Benchmark: LIF programmable bootstrapping (with key switching) and encrypted
inference on one B200 -- BASELINE.json's metric on its configs.

Headline workload (BASELINE.json configs[1], DESK p=1024): one encrypted fully
connected LIF layer, 16 samples x 784 encrypted Bernoulli(0.15) input spikes
per timestep, int weights U[-15,15] for 128 neurons, T=4 timesteps, state
carried.  One "step" = the whole T=4 forward = 4 x (weight sum 784->128 for 16
samples + fused LIF step on 2048 neurons = 4096 PBS) = 16,384 PBS incl. key
switch.  `value` is device-timed (inputs resident in HBM); `e2e` is the same
step through the reference-signature calls on host int64 arrays
(network.layer_forward_batch + network.spiking_forward per timestep, every
copy and host<->device conversion inside the timed region).

The same JSON line carries the other configs, each measured once after a
warm-up (`configs`): config 0 (1024 LIF bootstraps, host int64 API), config 2
(32-image conv CSNN, T=4) and config 4 (C4 params, 32 images, T=8) as
encrypted inferences/s both device-timed and end to end from host
CiphertextTensors, and the config 3 PBS sweep B = 1 .. 131072 with the
roofline fraction at every batch size.

    python bench.py [--gpus N --steps K --warmup W] [--impl reference] [--quick]

N>1 (torchrun, one process per GPU): every rank runs its own replica of the
headline workload (the path shards by sample with no data-path collective) ->
weak scaling; value = PBS of all ranks / max-over-ranks device time.  The
per-config block runs on rank 0 only at N=1.

`--impl reference` times the reference algorithm's CPU implementation (the
numba/numpy oracle port in oracle/ -- the Python reference itself does not
travel to the GPU box) on all host cores, on bounded samples of the headline
workload: each step is one sample (48 LIF neurons = 96 PBS per core).
"""

from __future__ import annotations

import argparse
import hashlib
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))

METRIC = "LIF PBS/sec (incl. key switch) and encrypted inferences/sec on 1 B200 vs roofline"
GOLDEN = os.path.join(ROOT, "tests", "golden")


def flops_per_pbs(n, N, levels):
    """n * [(2l+2) * 5 M log2 M + 2l * 2 * M * 8], M = N/2."""
    M = N // 2
    lg = M.bit_length() - 1
    return n * ((2 * levels + 2) * 5 * M * lg + 2 * levels * 2 * M * 8)


FLOPS_PER_PBS_DESK = flops_per_pbs(512, 1024, 2)  # 87.56 MFLOP
FLOPS_PER_PBS_C4 = flops_per_pbs(742, 2048, 3)    # 376.86 MFLOP
T_STEPS, BATCH, CELLS, NEURONS = 4, 16, 784, 128
PBS_PER_STEP = T_STEPS * BATCH * NEURONS * 2
HEADLINE_CONFIG = {"workload": "config1: FC 784->128 LIF layer (weight sum + fused fire/reset PBS "
                               "with key switch), 16 samples, T=4, 16384 PBS per step",
                   "params": "DESK n=512 q=2^25 N=1024 Bg=2^13 l=2 KS 2^5x5 p=1024"}


# ----------------------------------------------------------------- helpers

class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self._stop = threading.Event()
        self._thr = None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), "--query-gpu=" + self.FIELDS,
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                     timeout=5).stdout.strip()
                if out:
                    self.samples.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._thr = threading.Thread(target=self._run, daemon=True)
        self._thr.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._thr.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for s in self.samples for k in range(4)
                          if len(s) > 2 + k and s[2 + k].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


def dist_setup():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def shard_range(total: int, rank: int, world: int):
    """Contiguous [lo, hi) share of `total` independent items for `rank` (replica /
    sample sharding: PBS batches and images are independent, no collective)."""
    if not 0 <= rank < world:
        raise ValueError(f"rank {rank} outside world of {world}")
    base, extra = divmod(total, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def max_over_ranks(x: float, world: int, device=None) -> float:
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(x: float, world: int, device=None) -> float:
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


def sha(*arrays) -> bytes:
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(np.asarray(a, dtype=np.int64)).tobytes())
    return h.digest()


def golden(name):
    path = os.path.join(GOLDEN, name + ".npz")
    return np.load(path) if os.path.exists(path) else None


def hbm_peak():
    """Measured HBM copy bandwidth of this pool (MEASURED_PEAKS.json), else the
    profiling recipe's fallback."""
    mp = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        return float(json.load(open(mp))["hbm_gbs"]), "MEASURED_PEAKS.json:hbm_gbs"
    except Exception:
        return 7400.0, "B200_PROFILING.md fallback"


def build_workload(api):
    """Keys (seed 0), config-1 inputs (seed 1), weights (seed 2), encryption (seed 3)."""
    import workloads as W
    prm = W.desk1024(api)
    sk, zk, bsk = W.keys(api, prm)
    lif = W.lif_for(api, prm)
    x = W.config1_inputs(T=T_STEPS, batch=BATCH, cells=CELLS)
    Wm = W.config1_weights(out=NEURONS, cells=CELLS)
    A, b = W.encrypt(api, prm, sk, x.ravel())
    return prm, sk, bsk, lif, x, Wm, A.reshape(T_STEPS, BATCH * CELLS, prm.n), b.reshape(T_STEPS, BATCH * CELLS)


# ------------------------------------------------------------- CPU oracle leg

def _oracle_worker(args):
    """One host process: the numpy oracle (reference algorithm) on `count` neurons."""
    count, seed = args
    import workloads as W
    import paper_2309_09025_b200 as api
    from oracle import fdsnn_oracle as O
    prm = W.desk1024(api)
    sk, zk, bsk = W.keys(api, prm)
    lif = W.lif_for(api, prm)
    key = O.OracleKey(O.params_dict(prm), bsk.rows, bsk.ksk.A, bsk.ksk.b)
    rng = np.random.default_rng(seed)
    v = rng.integers(0, lif.v_th_hat, count)
    i = rng.integers(-200, 200, count)
    vA, vb = api.lwe.encrypt_batch(v, sk, prm, rng)
    iA, ib = api.lwe.encrypt_batch(i, sk, prm, rng)
    # JIT warm-up on one neuron (untimed)
    O.lif_step_fast(vA[:1], vb[:1], iA[:1], ib[:1], lif.v_th_hat, lif.leak_num, lif.leak_den, key)
    t0 = time.perf_counter()
    O.lif_step_fast(vA, vb, iA, ib, lif.v_th_hat, lif.leak_num, lif.leak_den, key)
    return 2 * count, time.perf_counter() - t0


def _pin_single_thread():
    for var in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS", "NUMBA_NUM_THREADS"):
        os.environ[var] = "1"
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/fdsnn_numba_cache")


class OraclePool:
    """One single-threaded process per host core running the oracle port of the
    reference's LIF step (each with its own key copy and a shard)."""

    def __init__(self):
        from multiprocessing import get_context
        self.cores = len(os.sched_getaffinity(0))
        _pin_single_thread()  # inherited by the spawned workers: one thread per process
        self.pool = get_context("spawn").Pool(self.cores)

    def sample(self, neurons_per_core: int, seed0: int = 100):
        t0 = time.perf_counter()
        res = self.pool.map(_oracle_worker, [(neurons_per_core, seed0 + c) for c in range(self.cores)])
        wall = time.perf_counter() - t0
        compute = max(r[1] for r in res)
        pbs = sum(r[0] for r in res)
        return {"value": pbs / compute, "unit": "PBS/s", "cores": self.cores, "kind": "port",
                "sample": f"{pbs} PBS: fused LIF step (fire+reset, with key switch) on {neurons_per_core} "
                          f"DESK p=1024 neurons per core, {self.cores} processes, numba+numpy oracle port of "
                          f"bootstrap.py:324-341 / neuron.py:160-172; timed region = the slowest process's "
                          f"LIF step (keygen and JIT warm-up excluded)",
                "pbs": pbs, "compute_s": compute, "wall_s": round(wall, 2)}

    def close(self):
        self.pool.close()
        self.pool.join()


def cpu_oracle_pbs_per_s(neurons_per_core: int = 48):
    pool = OraclePool()
    try:
        pool.sample(2)  # spawn + JIT warm-up
        return pool.sample(neurons_per_core)
    finally:
        pool.close()


def run_reference(args, world, rank):
    """Reference arm: same metric, unit and config as the B200 arm; each step is
    one bounded sample of the headline workload on all host cores."""
    if rank != 0:
        return
    pool = OraclePool()
    try:
        for _ in range(args.warmup):
            pool.sample(4)
        samples = [pool.sample(48) for _ in range(args.steps)]
    finally:
        pool.close()
    pbs = sum(s["pbs"] for s in samples)
    secs = sum(s["compute_s"] for s in samples)
    value = pbs / secs
    info = dict(samples[-1])
    info.update(value=value, sample=info["sample"] + f"; {args.steps} samples, value = total PBS / total time")
    line = {"metric": METRIC, "impl": "reference", "value": value, "unit": "PBS/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": secs / args.steps * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "int64/f64", "data": "synthetic",
            "config": dict(HEADLINE_CONFIG),
            "step": "one bounded sample of the config-1 LIF step per step (48 neurons = 96 PBS per core)",
            "cpu_baseline": info,
            "e2e": {"value": value, "unit": "PBS/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line))


# ------------------------------------------------------------------ GPU leg

class KernelClock:
    """Per-family device time from the library's event timers (launching stream)."""

    def __init__(self, dev):
        self.dev = dev

    def __enter__(self):
        self.dev.timing(True)
        self.dev.timing_reset()
        return self

    def __exit__(self, *a):
        self.br = self.dev.timing_read(0)
        self.ks = self.dev.timing_read(1)
        self.lin = self.dev.timing_read(2)
        self.dev.timing(False)

    @property
    def launches(self):
        return int(self.br[1] + self.ks[1] + self.lin[1])


def run_b200(args, world, rank, local):
    import torch
    import paper_2309_09025_b200 as api
    from paper_2309_09025_b200.bootstrap import test_polynomial

    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    dev_t = torch.device(f"cuda:{local}")
    prm, sk, bsk, lif, x, Wm, A, b = build_workload(api)
    from paper_2309_09025_b200.device import DeviceContext
    dev = DeviceContext(prm, device=local)
    dev.load_keys(bsk.rows, bsk.ksk.A, bsk.ksk.b)
    bsk._device = dev
    lf = dev.lut(test_polynomial(api.neuron.g_fire(prm.p), prm))
    lr = dev.lut(test_polynomial(api.neuron.g_reset(lif, prm.p), prm))
    op = dev.operator(Wm)
    rows = [dev.rows_from_host(A[t], b[t]) for t in range(T_STEPS)]
    torch.cuda.synchronize()

    def step():
        states = dev.zero_rows(BATCH * NEURONS)
        outs = []
        for t in range(T_STEPS):
            cur = dev.apply(op, rows[t], BATCH, NEURONS)
            out = dev.pbs_dev([lf, lr], [-lif.v_th_hat, 0], [1, 0], states, cur)
            states = out[BATCH * NEURONS:]
            outs.append(out)
        return outs

    # correctness of the benchmarked workload vs the reference's golden run
    outs = step()
    torch.cuda.synchronize()
    parity = None
    g1 = golden("config1")
    if g1 is not None:
        spikes = np.stack([api.lwe.decrypt_batch(*dev.rows_to_host(o[:BATCH * NEURONS]), sk, prm)
                           .reshape(BATCH, NEURONS) for o in outs])
        parity = bool(np.array_equal(spikes, g1["spikes"]))

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk, KernelClock(dev) as kc:
        for k in range(args.steps):
            evs[k][0].record()
            step()
            evs[k][1].record()
            dev.flush_l2()  # untimed: L2 flushed between timed iterations
        torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    step_ms = [a.elapsed_time(bb) for a, bb in evs]
    br_ms, br_n = kc.br
    total_ms = max_over_ranks(sum(step_ms), world, dev_t)
    ms_per_step = total_ms / args.steps
    value = PBS_PER_STEP * world / (ms_per_step * 1e-3)

    # ---- end to end through the reference-signature calls (host int64)
    e2e = run_e2e_int64(args, api, prm, bsk, lif, Wm, A, b, sk, g1)
    e2e_ms = max_over_ranks(e2e["ms_per_step"], world, dev_t)
    packed = run_e2e_packed(args, api, prm, bsk, lif, Wm, A, b)

    # ---- roofline of the dominant kernel (blind rotation)
    peak = dev.fp64_peak_tflops()
    # one blind-rotation call per fused LIF call (T_STEPS per step); a call
    # may be served by more than one kernel launch (br_n counts launches)
    br_calls = T_STEPS * args.steps
    br_launch_ms = br_ms / max(br_calls, 1)
    pbs_per_launch = BATCH * NEURONS * 2
    achieved = FLOPS_PER_PBS_DESK * pbs_per_launch / (br_launch_ms * 1e-3) / 1e12
    traffic, pipe_active, traffic_pbs = None, None, None
    tpath = os.path.join(ROOT, "profiles", "roofline_traffic.json")
    if os.path.exists(tpath):
        tj = json.load(open(tpath))
        traffic = tj.get("bytes_per_launch")
        pipe_active = tj.get("fp64_pipe_active")
        traffic_pbs = tj.get("pbs_per_launch")

    configs = None
    if world == 1 and not args.no_configs:
        configs = run_configs(args, api, dev, prm, sk, bsk, lif, peak)
    if rank != 0:
        return
    line = {
        "metric": METRIC, "value": value, "unit": "PBS/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64+u32", "data": "synthetic",
        "config": {**HEADLINE_CONFIG, "parallelism": f"replicas x{world}",
                   "l2": "flushed between timed steps (256 MiB memset)"},
        "layer_forwards_per_s": BATCH * world / (ms_per_step * 1e-3),
        "parity_vs_reference_golden": parity,
        "kernel_ms_per_step": {"blind_rotate": br_ms / args.steps, "key_switch": kc.ks[0] / args.steps,
                               "weight_sum": kc.lin[0] / args.steps},
        "gpu_launches": kc.launches,
        "roofline": {"bound": "fp64", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                     "frac": achieved / peak, "traffic": traffic,
                     "traffic_note": f"DRAM bytes of one pbs_br16_kernel launch ({traffic_pbs} PBS) from the committed "
                                     "ncu capture (profiles/roofline_traffic.json); the key is read from DRAM about once "
                                     "per launch (L2-resident), the rest is ciphertext rows",
                     "fp64_pipe_active": pipe_active,
                     "kernel": "blind rotation per fused LIF call (4096 PBS): pbs_br16_kernel, 3 waves of 8 "
                               "rotations per SM (3552) + pbs_blind_rotate_kernel<512,4,..> for the 544-rotation "
                               "remainder (4 per SM); achieved = flops of the call / the call's device time",
                     "br_kernel_launches_per_call": br_n / max(br_calls, 1),
                     "flops_per_pbs": FLOPS_PER_PBS_DESK, "pbs_per_launch": pbs_per_launch,
                     "peak_source": "DFMA loop measured live in this run (fdsnn_probe_fp64_peak); "
                                    "MEASURED_PEAKS.json has no FP64 entry"},
        "e2e": {"value": PBS_PER_STEP * world / (e2e_ms * 1e-3), "unit": "PBS/s",
                "h2d_bytes_per_step": e2e["h2d"], "d2h_bytes_per_step": e2e["d2h"],
                "path": "reference signatures on host int64 arrays: per timestep "
                        "network.layer_forward_batch(16 x CiphertextTensor(784)) + "
                        "network.spiking_forward(CiphertextTensor(2048), states) -- host packing, "
                        "copies and unpacking inside the timed region; wall clock, median step",
                "ms_per_step": e2e_ms, "ms_all": e2e["ms_all"], "parity_vs_reference_golden": e2e["parity"]},
        "e2e_packed": {"value": PBS_PER_STEP * world / (packed["ms_per_step"] * 1e-3), "unit": "PBS/s",
                       "h2d_bytes_per_step": packed["h2d"], "d2h_bytes_per_step": packed["d2h"],
                       "path": "network.infer_sequence (extension): pinned uint32 host rows in, pinned rows out",
                       "ms_per_step": packed["ms_per_step"]},
        "clocks": clk.summary(),
    }
    if configs is not None:
        line["configs"] = configs
    if world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_oracle_pbs_per_s()
    print(json.dumps(line))


def run_e2e_int64(args, api, prm, bsk, lif, Wm, A, b, sk, g1):
    """The headline step through the reference's own call signatures on host
    int64 arrays: per timestep, the 16 samples' weight sums
    (network.layer_forward_batch: each result equals layer_forward, network.py:409-421,
    returned stacked as one (16, 128) tensor) then one spiking_forward over the
    2048 cells (network.py:430-436) carrying the states; results come back as
    host CiphertextTensors."""
    import torch
    N = api.network
    layer = N.WeightLayer("linear", Wm, None, 1.0, (NEURONS,))
    xs = [[N.CiphertextTensor((CELLS,), A[t, s * CELLS:(s + 1) * CELLS], b[t, s * CELLS:(s + 1) * CELLS], prm.q)
           for s in range(BATCH)] for t in range(T_STEPS)]
    n = prm.n
    h2d = T_STEPS * (BATCH * CELLS + 2 * BATCH * NEURONS) * (n + 1) * 8  # int64 (A, b) handed in
    d2h = T_STEPS * (BATCH * NEURONS + 2 * BATCH * NEURONS) * (n + 1) * 8

    def once():
        states = N.zero_states(BATCH * NEURONS, prm)
        spikes = []
        for t in range(T_STEPS):
            stacked = N.layer_forward_batch(xs[t], layer, prm, stack=True)  # (16, 128) cells
            sp, states = N.spiking_forward(stacked, states, lif, bsk)
            spikes.append(sp)
        return spikes

    for _ in range(max(1, min(args.warmup, 2))):
        sp = once()
    parity = None
    if g1 is not None:
        parity = all(np.array_equal(api.lwe.decrypt_batch(sp[t].A, sp[t].b, sk, prm).reshape(BATCH, NEURONS),
                                    g1["spikes"][t]) for t in range(T_STEPS))
    torch.cuda.synchronize()
    times = []
    for _ in range(max(5, args.steps)):
        t0 = time.perf_counter()
        once()  # every call returns host arrays: the step ends with its results on the host
        times.append(time.perf_counter() - t0)
    return {"ms_per_step": float(np.median(times)) * 1e3, "h2d": h2d, "d2h": d2h,
            "ms_all": [round(t * 1e3, 3) for t in times], "parity": parity}


def run_e2e_packed(args, api, prm, bsk, lif, Wm, A, b):
    """Same workload through the extension `network.infer_sequence`: inputs as
    pinned uint32 device-format rows, per-timestep spikes + scores back into
    pinned host rows; membrane states stay on the device."""
    import torch
    N = api.network
    layers = (N.WeightLayer("linear", Wm, None, 1.0, (NEURONS,)), N.SpikingLayer(lif, (NEURONS,)))
    net = N.DiscretizedNetwork(layers, lif.theta, 1, lif, T_STEPS)
    inputs = [N.PackedCiphertexts.pack(N.CiphertextTensor((BATCH * CELLS,), A[t], b[t], prm.q), prm)
              for t in range(T_STEPS)]
    h2d = sum(int(x.rows.numel()) * 4 for x in inputs)

    def once():
        outs, scores, _ = N.infer_sequence(inputs, net, bsk)
        return sum(int(o.rows.numel()) * 4 for o in outs) + int(scores.rows.numel()) * 4

    for _ in range(max(1, min(args.warmup, 2))):
        once()
    torch.cuda.synchronize()
    times = []
    for _ in range(max(5, args.steps)):
        t0 = time.perf_counter()
        d2h = once()
        times.append(time.perf_counter() - t0)
    return {"ms_per_step": float(np.median(times)) * 1e3, "h2d": h2d, "d2h": d2h}


# ------------------------------------------------------- the other configs

def _timed(fn, reps=1):
    """(device ms per call via CUDA events on the current stream, result)."""
    import torch
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(reps):
        out = fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps, out


def run_configs(args, api, dev, prm, sk, bsk, lif, peak):
    import torch
    import workloads as W
    from paper_2309_09025_b200 import bootstrap, network, neuron
    out = {}
    hbm, hbm_src = hbm_peak()
    g = neuron.g_fire(prm.p)
    lut = dev.lut(bootstrap.test_polynomial(g, prm))

    # ---- config 0: 1024 LIF bootstraps through the reference-signature host call
    ms0 = W.pbs_messages(prm, 1024)
    A0, b0 = W.encrypt(api, prm, sk, ms0)
    z = (np.zeros_like(A0), np.zeros_like(b0))
    neuron.fhe_lif_step_batch(z[0], z[1], A0, b0, lif, bsk)
    t0 = time.perf_counter()
    reps = 5
    for _ in range(reps):
        res = neuron.fhe_lif_step_batch(z[0], z[1], A0, b0, lif, bsk)
    dt = (time.perf_counter() - t0) / reps
    g0 = golden("config0")
    out["config0"] = {"pbs": 2048, "ms_host_to_host": dt * 1e3, "pbs_per_s": 2048 / dt,
                      "path": "neuron.fhe_lif_step_batch on host int64 arrays (neuron.py:160-172)",
                      "parity_vs_reference_golden": None if g0 is None else
                      sha(res[0], res[1], res[2], res[3]) == bytes(g0["out_digest"])}

    # ---- config 3: PBS + key switch sweep, device-resident rows
    sweep = {}
    for B in (1, 64, 1024, 16384, 131072):
        ms = W.pbs_messages(prm, B, seed=B)
        rows = dev.encrypt_rows(ms, sk, np.random.default_rng(B))
        dev.pbs_dev([lut], [0], [0], rows)
        reps = 5 if B <= 1024 else (2 if B <= 16384 else 1)
        with KernelClock(dev) as kc:
            ms_, o = _timed(lambda: dev.pbs_dev([lut], [0], [0], rows), reps)
        dec = dev.decrypt_rows(o, sk)
        ok = bool(np.array_equal(dec, g(ms)))
        flops = B * FLOPS_PER_PBS_DESK
        nbytes = (prm.n * 2 * prm.gadget.levels * 2 * (prm.N // 2) * 16
                  + prm.N * prm.ks_levels * (prm.n + 1) * 4 + B * 2 * dev.stride * 4)
        t_fp64 = flops / (peak * 1e12)
        t_hbm = nbytes / (hbm * 1e9)
        br_ms = kc.br[0] / reps
        sweep[str(B)] = {"ms": ms_, "pbs_per_s": B / ms_ * 1e3,
                         "bound": "fp64" if t_fp64 >= t_hbm else "hbm",
                         "roofline_frac": max(t_fp64, t_hbm) / (ms_ * 1e-3),
                         "fp64_tflops": flops / (ms_ * 1e-3) / 1e12,
                         "hbm_gbs": nbytes / (ms_ * 1e-3) / 1e9,
                         "blind_rotate_ms": br_ms, "key_switch_ms": kc.ks[0] / reps,
                         "decrypts_to_sign_lut": ok}
        del rows, o
    out["config3_sweep"] = {"points": sweep, "peaks": {"fp64_tflops": peak, "hbm_gbs": hbm, "hbm_source": hbm_src},
                            "bytes_model": "BSK (Fourier, 16 B/coef) + KSK (uint32) once per launch + input "
                                           "and output rows; flops 87.56 MFLOP/PBS (SURVEY 8(d))"}

    # ---- configs 2 and 4: encrypted inference of 32 images
    def net_config(tag, prm_c, sk_c, bsk_c, lif_c, net, T, flops):
        imgs = W.synth_images(32)
        encs = W.encrypt_images(api, prm_c, sk_c, imgs)
        network.infer_batch(encs[:2], net, bsk_c, T=1)  # warm-up (plans, LUTs, operators)
        torch.cuda.synchronize()
        dctx = bsk_c.device
        with KernelClock(dctx) as kc:
            t0 = time.perf_counter()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record()
            scores, stats = network.infer_batch(encs, net, bsk_c)  # host CiphertextTensors in and out
            e1.record()
            torch.cuda.synchronize()
            wall = time.perf_counter() - t0
        dev_s = e0.elapsed_time(e1) * 1e-3
        ref = golden(f"{tag}_img0")
        preds = [network.classify(s, sk_c, prm_c) for s in scores]
        in_bytes = sum(e.count for e in encs) * (prm_c.n + 1) * 8
        res = {"images": 32, "T": T, "pbs": stats.bootstrap_count,
               "inferences_per_s": 32 / dev_s, "inferences_per_s_e2e": 32 / wall,
               "pbs_per_s": stats.bootstrap_count / dev_s, "seconds_device": dev_s, "seconds_e2e": wall,
               "e2e_path": "network.infer_batch on host int64 CiphertextTensors (network.py:459-491 "
                           "semantics, batched), int64 scores back on the host",
               "h2d_bytes": in_bytes, "d2h_bytes": 32 * 10 * (prm_c.n + 1) * 8,
               "blind_rotate_ms": kc.br[0], "blind_rotate_launches": kc.br[1],
               "blind_rotate_frac_of_fp64_peak": stats.bootstrap_count * flops / (kc.br[0] * 1e-3) / 1e12 / peak,
               "predictions": preds,
               "parity_img0_vs_reference_encrypted_run": None if ref is None else
               sha(scores[0].A, scores[0].b) == bytes(ref["score_digest"])}
        return res

    net2 = W.config2_network(api, lif)
    out["config2"] = net_config("config2", prm, sk, bsk, lif, net2, 4, FLOPS_PER_PBS_DESK)
    if not args.quick:
        prm4 = W.c4_params(api)
        sk4, zk4, bsk4 = W.keys(api, prm4)
        lif4 = W.lif_for(api, prm4)
        net4 = W.config4_network(api, lif4)
        out["config4"] = net_config("config4", prm4, sk4, bsk4, lif4, net4, 8, FLOPS_PER_PBS_C4)
        bsk4._device.close()
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-configs", action="store_true", help="headline config only")
    ap.add_argument("--quick", action="store_true", help="skip config 4 (the 32-image C4 run)")
    args = ap.parse_args()
    world, rank, local = dist_setup()
    if args.impl == "reference":
        run_reference(args, world, rank)
        return
    import __graft_entry__
    __graft_entry__.build()
    run_b200(args, world, rank, local)


if __name__ == "__main__":
    main()
