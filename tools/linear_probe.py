"""Weight-sum kernels alone: config-1 FC 784->128 x 16 samples and config-2 FC 4608->128 x 32."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2309_09025_b200 import params
from paper_2309_09025_b200.device import DeviceContext
for name, prm, out, inn, batch in (("c1 fc 784->128 x16", params.preset("DESK").with_p(1024), 128, 784, 16),
                                    ("c2 fc 4608->128 x32", params.preset("DESK").with_p(1024), 128, 4608, 32),
                                    ("c4 fc 4608->256 x32", params.c4(), 256, 4608, 32)):
    dev = DeviceContext(prm)
    rng = np.random.default_rng(0)
    W = rng.integers(-15, 16, (out, inn))
    op = dev.operator(W)
    A = rng.integers(0, prm.q, (batch * inn, prm.n)); b = rng.integers(0, prm.q, batch * inn)
    rows = dev.rows_from_host(A, b)
    y = dev.apply(op, rows, batch, out); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10): dev.apply(op, rows, batch, out, out=y)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    yA, yb = dev.rows_to_host(y)
    k = 3
    ok = np.array_equal(yA[:out * k], np.concatenate([(W @ A[s * inn:(s + 1) * inn]) % prm.q for s in range(k)])) and \
        np.array_equal(yb[:out * k], np.concatenate([(W @ b[s * inn:(s + 1) * inn]) % prm.q for s in range(k)]))
    byts = (batch * inn + batch * out) * dev.stride * 4 + W.size * 4
    macs = batch * out * inn * (prm.n + 1)
    print(f"{name}: {ms * 1e3:.1f} us  {byts / ms / 1e6:.0f} GB/s  {macs / ms / 1e9:.2f} TMAC/s  exact={ok}")
