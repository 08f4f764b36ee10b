"""Minimal ncu target: one fused LIF launch (2*B PBS) at DESK p=1024."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2309_09025_b200 import bootstrap, lwe, neuron, params, rgsw
from paper_2309_09025_b200.bootstrap import test_polynomial

B = int(sys.argv[1]) if len(sys.argv) > 1 else 1184
prm = params.c4() if os.environ.get("PROBE_PARAMS") == "c4" else params.preset("DESK").with_p(1024)
rng = np.random.default_rng(0)
sk = lwe.lwe_keygen(prm, rng); zk = rgsw.rlwe_keygen(prm, rng)
bsk = bootstrap.gen_bootstrap_key(sk, zk, prm, rng)
dev = bsk.device
lif = neuron.LifParams(tau=2, theta=256 if prm.p == 4096 else 64)
lf = dev.lut(test_polynomial(neuron.g_fire(prm.p), prm))
lr = dev.lut(test_polynomial(neuron.g_reset(lif, prm.p), prm))
A, b = lwe.encrypt_batch(rng.integers(-prm.p // 2 + 1, prm.p // 2 + 1, B), sk, prm, rng)
rows = dev.rows_from_host(A, b)
zero = dev.zero_rows(B)
for _ in range(2):
    out = dev.pbs_dev([lf, lr], [-lif.v_th_hat, 0], [1, 0], zero, rows)
torch.cuda.synchronize()
print("ok", out.shape)
