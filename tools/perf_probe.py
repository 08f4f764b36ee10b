"""Quick device timing probe (development aid): fused LIF step on DESK p=1024."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2309_09025_b200 import bootstrap, lwe, neuron, params, rgsw
from paper_2309_09025_b200.bootstrap import test_polynomial

prm = params.c4() if os.environ.get("PROBE_PARAMS") == "c4" else params.preset("DESK").with_p(1024)
rng = np.random.default_rng(0)
sk = lwe.lwe_keygen(prm, rng); zk = rgsw.rlwe_keygen(prm, rng)
t = time.time(); bsk = bootstrap.gen_bootstrap_key(sk, zk, prm, rng); print("keygen s", time.time() - t)
dev = bsk.device
print("fp64 peak TF", dev.fp64_peak_tflops())
lif = neuron.LifParams(tau=2, theta=256 if prm.p == 4096 else 64)
lf = dev.lut(test_polynomial(neuron.g_fire(prm.p), prm)); lr = dev.lut(test_polynomial(neuron.g_reset(lif, prm.p), prm))
for B in (int(x) for x in sys.argv[1:] or ["4096"]):
    ms = rng.integers(-prm.p // 2 + 1, prm.p // 2 + 1, B)
    A, b = lwe.encrypt_batch(ms, sk, prm, rng)
    rows = dev.rows_from_host(A, b)
    zero = dev.zero_rows(B)
    dev.pbs_dev([lf, lr], [-lif.v_th_hat, 0], [1, 0], zero, rows)
    torch.cuda.synchronize()
    dev.timing(True); dev.timing_reset()
    s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(3):
        dev.pbs_dev([lf, lr], [-lif.v_th_hat, 0], [1, 0], zero, rows)
    e.record(); torch.cuda.synchronize()
    ms_tot = s.elapsed_time(e) / 3
    br = dev.timing_read(0); ks = dev.timing_read(1)
    dev.timing(False)
    print(f"B={B} neurons ({2*B} PBS): {ms_tot:.2f} ms/step -> {2*B/ms_tot*1e3:.0f} PBS/s; BR {br[0]/br[1]:.2f} ms, KS {ks[0]/ks[1]:.3f} ms")
