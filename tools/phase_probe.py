"""Per-phase cycle split of the CTA-pair kernel (build with -DFDSNN_PHASE_PROF)."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2309_09025_b200 import bootstrap, lwe, neuron, params, rgsw, _lib
from paper_2309_09025_b200.bootstrap import test_polynomial
prm = params.preset("DESK").with_p(1024)
rng = np.random.default_rng(0)
sk = lwe.lwe_keygen(prm, rng); zk = rgsw.rlwe_keygen(prm, rng)
bsk = bootstrap.gen_bootstrap_key(sk, zk, prm, rng)
dev = bsk.device
lf = dev.lut(test_polynomial(neuron.g_fire(prm.p), prm))
B = int(sys.argv[1]) if len(sys.argv) > 1 else 1
A, b = lwe.encrypt_batch(rng.integers(-511, 513, B), sk, prm, rng)
rows = dev.rows_from_host(A, b)
dev.pbs_dev([lf], [0], [0], rows); torch.cuda.synchronize()
import cuda.bindings.runtime as rt  # noqa
lib = ctypes.CDLL(_lib.LIB_PATH)
fn = lib.fdsnn_debug_phase_read
buf = (ctypes.c_ulonglong * 8)()
fn(buf)
dev.pbs_dev([lf], [0], [0], rows); torch.cuda.synchronize()
fn(buf)
names = ["digits", "fwd pair", "MAC+send", "wait partner", "recv add", "inverse", "update", "bar+refill"]
tot = sum(buf)
for k in range(8):
    print(f"{names[k]:14s} {buf[k] / 512:8.0f} cycles/step  {100 * buf[k] / max(tot, 1):5.1f}%")
print("total", tot / 512)
