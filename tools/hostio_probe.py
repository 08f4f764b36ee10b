"""Host boundary throughput probe (int64 <-> device rows) on the GPU box."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2309_09025_b200 as api
from paper_2309_09025_b200.device import DeviceContext
prm = api.params.preset("DESK").with_p(1024)
dev = DeviceContext(prm)
print("cpus", os.cpu_count(), "affinity", len(os.sched_getaffinity(0)))
print(open("/proc/cpuinfo").read().split("model name")[1].split("\n")[0])
rng = np.random.default_rng(0)
for count in (2048, 12544):
    A = rng.integers(0, 1 << 25, (count, prm.n)); b = rng.integers(0, 1 << 25, count)
    rows = dev.empty_rows(count)
    for rep in range(3):
        torch.cuda.synchronize(); t0 = time.perf_counter(); dev.rows_from_host(A, b, out=rows); torch.cuda.synchronize(); t1 = time.perf_counter()
    MB = A.nbytes / 1e6
    print(f"upload {count}: {(t1-t0)*1e3:.2f} ms  ({MB / (t1-t0) / 1e3:.1f} GB/s of int64 input)")
    for rep in range(3):
        t0 = time.perf_counter(); dev.rows_to_host(rows); t1 = time.perf_counter()
    print(f"download {count}: {(t1-t0)*1e3:.2f} ms ({MB / (t1-t0) / 1e3:.1f} GB/s of int64 output)")
    outA = np.empty((count, prm.n), np.int64); outA.fill(0)
    t0 = time.perf_counter(); x = np.empty((count, prm.n), np.int64); x[...] = 1; t1 = time.perf_counter()
    print(f"  numpy fresh alloc+fill: {(t1-t0)*1e3:.2f} ms")
    t0 = time.perf_counter(); outA[...] = 2; t1 = time.perf_counter()
    print(f"  numpy fill faulted: {(t1-t0)*1e3:.2f} ms")
    t0 = time.perf_counter(); y = (A & (prm.q - 1)).astype(np.uint32); t1 = time.perf_counter()
    print(f"  numpy pack-like: {(t1-t0)*1e3:.2f} ms")
