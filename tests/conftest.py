import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

from paper_2309_09025_b200 import bootstrap, lwe, params, rgsw  # noqa: E402
from oracle import fdsnn_oracle as O  # noqa: E402  (checker only)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and the built CUDA library")
    config.addinivalue_line("markers", "slow: long-running parity sweep")


def _gpu_ok():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


def pytest_collection_modifyitems(config, items):
    if _gpu_ok():
        return
    skip = pytest.mark.skip(reason="no CUDA device in this container")
    for it in items:
        if "gpu" in it.keywords:
            it.add_marker(skip)


def make_keys(prm, seed):
    rng = np.random.default_rng(seed)
    sk = lwe.lwe_keygen(prm, rng)
    zk = rgsw.rlwe_keygen(prm, rng)
    bsk = bootstrap.gen_bootstrap_key(sk, zk, prm, rng)
    return sk, zk, bsk


def oracle_key(prm, bsk):
    return O.OracleKey(O.params_dict(prm), bsk.rows, bsk.ksk.A, bsk.ksk.b)


@pytest.fixture(scope="session")
def toy():
    return params.preset("TOY")


@pytest.fixture(scope="session")
def toy_keys(toy):
    return make_keys(toy, 1)


@pytest.fixture(scope="session")
def toy64():
    from dataclasses import replace
    return replace(params.preset("TOY"), p=64, sigma=2.0, preset_name="custom")


@pytest.fixture(scope="session")
def toy64_keys(toy64):
    return make_keys(toy64, 2)


@pytest.fixture(scope="session")
def desk():
    return params.preset("DESK").with_p(1024)


@pytest.fixture(scope="session")
def desk_keys(desk):
    return make_keys(desk, 0)


@pytest.fixture(scope="session")
def c4prm():
    return params.c4()


@pytest.fixture(scope="session")
def c4_keys(c4prm):
    return make_keys(c4prm, 0)
