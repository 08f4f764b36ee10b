#!/usr/bin/env python
"""Benchmark: LIF programmable bootstrapping (with key switching) on one B200.

Workload (BASELINE.json configs[1], DESK p=1024): one encrypted fully connected
LIF layer, 16 samples x 784 encrypted Bernoulli(0.15) input spikes per
timestep, int weights U[-15,15] for 128 neurons, T=4 timesteps, state carried.
One "step" = the whole T=4 forward = 4 x (weight sum 784->128 for 16 samples
+ fused LIF step on 2048 neurons = 4096 PBS) = 16,384 PBS incl. key switch.

    python bench.py [--gpus N --steps K --warmup W] [--impl reference]

N>1 (torchrun, one process per GPU): every rank runs its own replica of the
workload (the path shards by sample with no data-path collective) -> weak
scaling; value = PBS of all ranks / max-over-ranks device time.

`--impl reference` times the reference algorithm's CPU implementation (the
numpy oracle port in oracle/, since the Python reference does not travel to
the GPU box) on all host cores, on a bounded sample of the same workload.
"""

from __future__ import annotations

import argparse
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
FLOPS_PER_PBS_DESK = 512 * ((2 * 2 + 2) * 5 * 512 * 9 + 2 * 2 * 2 * 512 * 8)  # 87.56 MFLOP
T_STEPS, BATCH, CELLS, NEURONS = 4, 16, 784, 128
PBS_PER_STEP = T_STEPS * BATCH * NEURONS * 2


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


def cpu_oracle_pbs_per_s(neurons_per_core: int = 48):
    """Time the oracle port of the reference's LIF step on all host cores
    (one process per core, each with its own key copy and a shard)."""
    from multiprocessing import get_context
    cores = len(os.sched_getaffinity(0))
    _pin_single_thread()  # inherited by the spawned workers: one thread per process
    with get_context("spawn").Pool(cores) as pool:
        # best of two passes: host-side noise (other tenants, frequency ramps)
        # otherwise swings the slowest-process time by +-30 % between runs
        best = None
        for _ in range(2):
            t0 = time.perf_counter()
            res = pool.map(_oracle_worker, [(neurons_per_core, 100 + c) for c in range(cores)])
            wall = time.perf_counter() - t0
            compute = max(r[1] for r in res)
            if best is None or compute < best[1]:
                best = (res, compute, wall)
        res, compute, wall = best
    pbs = sum(r[0] for r in res)
    return {"value": pbs / compute, "unit": "PBS/s", "cores": cores, "kind": "port",
            "sample": f"{pbs} PBS: fused LIF step (fire+reset, with key switch) on {neurons_per_core} "
                      f"DESK p=1024 neurons per core, {cores} processes, numba+numpy oracle port of "
                      f"bootstrap.py:324-341 / neuron.py:160-172; timed region excludes keygen; "
                      f"slowest process of the better of two passes",
            "wall_s": round(wall, 2)}


def run_reference(args, world, rank):
    if rank != 0:
        return
    vals = []
    info = None
    for k in range(args.warmup + args.steps):
        info = cpu_oracle_pbs_per_s(neurons_per_core=8 if k < args.warmup else 48)
        if k >= args.warmup:
            vals.append(info["value"])
    value = statistics.mean(vals)
    line = {"metric": METRIC, "impl": "reference", "value": value, "unit": "PBS/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": PBS_PER_STEP / value * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "int64/f64", "data": "synthetic",
            "config": {"workload": "config1: FC 784->128 LIF layer, 16 samples, T=4, DESK p=1024 (sampled)",
                       "params": "DESK n=512 q=2^25 N=1024 Bg=2^13 l=2 KS 2^5x5 p=1024"},
            "cpu_baseline": {**info, "value": value},
            "e2e": {"value": value, "unit": "PBS/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line))


# ------------------------------------------------------------------ GPU leg

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
    bsk._device = None
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
    gpath = os.path.join(ROOT, "tests", "golden", "config1.npz")
    if os.path.exists(gpath):
        g = np.load(gpath)
        spikes = np.stack([api.lwe.decrypt_batch(*dev.rows_to_host(o[:BATCH * NEURONS]), sk, prm)
                           .reshape(BATCH, NEURONS) for o in outs])
        parity = bool(np.array_equal(spikes, g["spikes"]))

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    dev.timing(True)
    dev.timing_reset()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        for k in range(args.steps):
            evs[k][0].record()
            step()
            evs[k][1].record()
            dev.flush_l2()  # untimed: L2 flushed between timed iterations
        torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    step_ms = [a.elapsed_time(bb) for a, bb in evs]
    br_ms, br_n = dev.timing_read(0)
    ks_ms, ks_n = dev.timing_read(1)
    lin_ms, lin_n = dev.timing_read(2)
    dev.timing(False)
    total_ms = max_over_ranks(sum(step_ms), world, dev_t)
    ms_per_step = total_ms / args.steps
    value = PBS_PER_STEP * world / (ms_per_step * 1e-3)

    # ---- end-to-end through the reference-facing API with host buffers
    e2e = run_e2e(args, api, prm, bsk, lif, Wm, A, b)
    e2e_ms = max_over_ranks(e2e["ms_per_step"], world, dev_t)

    # ---- roofline of the dominant kernel (blind rotation)
    peak = dev.fp64_peak_tflops()
    br_launch_ms = br_ms / max(br_n, 1)
    pbs_per_launch = BATCH * NEURONS * 2
    achieved = FLOPS_PER_PBS_DESK * pbs_per_launch / (br_launch_ms * 1e-3) / 1e12
    traffic, pipe_active = None, None
    tpath = os.path.join(ROOT, "profiles", "roofline_traffic.json")
    if os.path.exists(tpath):
        tj = json.load(open(tpath))
        traffic = tj.get("bytes_per_launch")
        pipe_active = tj.get("fp64_pipe_active")
    if rank != 0:
        return
    line = {
        "metric": METRIC, "value": value, "unit": "PBS/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64+u32", "data": "synthetic",
        "config": {"workload": "config1: FC 784->128 LIF layer (weight sum + fused fire/reset PBS "
                               "with key switch), 16 samples, T=4, 16384 PBS per step",
                   "params": "DESK n=512 q=2^25 N=1024 Bg=2^13 l=2 KS 2^5x5 p=1024",
                   "parallelism": f"replicas x{world}", "l2": "flushed between timed steps (256 MiB memset)"},
        "inferences_per_s": BATCH * world / (ms_per_step * 1e-3),
        "parity_vs_reference_golden": parity,
        "kernel_ms_per_step": {"blind_rotate": br_ms / args.steps, "key_switch": ks_ms / args.steps,
                               "weight_sum": lin_ms / args.steps},
        "gpu_launches": int(br_n + ks_n + lin_n),
        "roofline": {"bound": "fp64", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                     "frac": achieved / peak, "traffic": traffic,
                     "fp64_pipe_active": pipe_active,
                     "kernel": "pbs_blind_rotate_kernel<512,4>",
                     "flops_per_pbs": FLOPS_PER_PBS_DESK, "pbs_per_launch": pbs_per_launch,
                     "peak_source": "DFMA loop measured live in this run (fdsnn_probe_fp64_peak); "
                                    "MEASURED_PEAKS.json has no FP64 entry"},
        "e2e": {"value": PBS_PER_STEP * world / (e2e_ms * 1e-3), "unit": "PBS/s",
                "h2d_bytes_per_step": e2e["h2d"], "d2h_bytes_per_step": e2e["d2h"],
                "path": "network.infer_sequence: pinned host rows -> device -> pinned host spikes/scores, "
                        "wall clock, median of the timed calls",
                "ms_per_step": e2e_ms, "ms_all": e2e.get("ms_all")},
        "clocks": clk.summary(),
    }
    if world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_oracle_pbs_per_s()
    print(json.dumps(line))


def run_e2e(args, api, prm, bsk, lif, Wm, A, b):
    """Same workload through the public API `network.infer_sequence`: every step
    DMAs that step's encrypted inputs (all T timesteps) from pinned host memory
    and reads the result (per-timestep spike ciphertexts + scores) back into
    pinned host memory; membrane states stay on the device."""
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
    n = max(5, args.steps)
    times = []
    for _ in range(n):
        t0 = time.perf_counter()
        d2h = once()  # returns after the results are in host memory
        times.append(time.perf_counter() - t0)
    # median step: host-side hiccups (allocator, GC, scheduling) of single
    # steps do not define the end-to-end rate
    return {"ms_per_step": float(np.median(times)) * 1e3, "h2d": h2d, "d2h": d2h,
            "ms_all": [t * 1e3 for t in times]}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
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
