"""Break the int64 reference-signature e2e step (bench.run_e2e_int64) into its
host / device pieces on the GPU box."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import numpy as np
import torch
import bench
import paper_2309_09025_b200 as api
N = api.network
prm, sk, bsk, lif, x, Wm, A, b = bench.build_workload(api)
layer = N.WeightLayer("linear", Wm, None, 1.0, (128,))
xs = [[N.CiphertextTensor((784,), A[t, s * 784:(s + 1) * 784], b[t, s * 784:(s + 1) * 784], prm.q)
       for s in range(16)] for t in range(4)]
dev = bsk.device
_, LF, LR = api.neuron._luts(lif, bsk)
T = {}
def tic(k, t0):
    torch.cuda.synchronize(); T[k] = T.get(k, 0) + time.perf_counter() - t0
for rep in range(4):
    if rep == 1: T.clear()
    states = N.zero_states(2048, prm)
    for t in range(4):
        t0 = time.perf_counter(); cur = N.layer_forward_batch(xs[t], layer, prm); tic("layer_forward_batch", t0)
        t0 = time.perf_counter()
        stacked = N.CiphertextTensor((2048,), np.concatenate([c.A for c in cur]), np.concatenate([c.b for c in cur]), prm.q)
        tic("concat", t0)
        t0 = time.perf_counter(); r1 = dev.rows_from_host(states.A, states.b); r2 = dev.rows_from_host(stacked.A, stacked.b); tic("upload2", t0)
        t0 = time.perf_counter(); sp, states = N.spiking_forward(stacked, states, lif, bsk); tic("spiking_forward", t0)
        rows = dev.empty_rows(4096)
        t0 = time.perf_counter(); o = dev.pbs_dev([LF, LR], [-128, 0], [1, 0], r1, r2, out=rows); tic("pbs_dev only", t0)
        t0 = time.perf_counter(); dev.rows_to_host(o[:2048]); dev.rows_to_host(o[2048:]); tic("download2", t0)
for k, v in T.items(): print(f"{k:24s} {v / 3 * 1e3:8.2f} ms per step")
