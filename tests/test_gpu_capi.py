"""A plain-C host (tools/capi_demo.c) drives the path through the C ABI only:
FDSN key + ciphertext containers in, bootstrapped ciphertexts out, equal to
the Python drop-in's (and hence the reference's) results."""
import os
import subprocess

import numpy as np
import pytest

from conftest import ROOT
from paper_2309_09025_b200 import bootstrap, lwe, network, neuron, serial

pytestmark = pytest.mark.gpu


def test_c_host_end_to_end(toy, toy_keys, tmp_path):
    sk, _, bsk = toy_keys
    rng = np.random.default_rng(21)
    ms = rng.integers(-toy.p // 2 + 1, toy.p // 2 + 1, 40)
    A, b = lwe.encrypt_batch(ms, sk, toy, rng)
    serial.save_bootstrap_key(tmp_path / "bk.bin", bsk)
    serial.save_ciphertexts(tmp_path / "ct.bin", network.CiphertextTensor((5, 8), A, b, toy.q), toy)
    exe = tmp_path / "capi_demo"
    lib = os.path.join(ROOT, "paper_2309_09025_b200")
    subprocess.run(["gcc", "-O2", "-I", os.path.join(ROOT, "include"), os.path.join(ROOT, "tools", "capi_demo.c"),
                    "-L", lib, "-lfdsnn_b200", f"-Wl,-rpath,{lib}", "-o", str(exe)], check=True)
    lg = lambda x: int(x).bit_length() - 1
    args = [str(exe), str(tmp_path / "bk.bin"), str(tmp_path / "ct.bin"), toy.digest(), toy.n, toy.N, lg(toy.q),
            toy.p, lg(toy.gadget.base), toy.gadget.levels, lg(toy.ks_base), toy.ks_levels, str(tmp_path / "out.bin")]
    res = subprocess.run([str(a) for a in args], capture_output=True, text=True, timeout=120)
    assert res.returncode == 0, res.stderr
    raw = np.fromfile(tmp_path / "out.bin", dtype=np.int64)
    count = int(raw[0])
    oA = raw[1:1 + count * toy.n].reshape(count, toy.n)
    ob = raw[1 + count * toy.n:]
    wA, wb = bootstrap.bootstrap_batch(neuron.g_fire(toy.p), A, b, bsk)
    assert count == 40 and np.array_equal(oA, wA) and np.array_equal(ob, wb)
