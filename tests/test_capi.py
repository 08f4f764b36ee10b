"""The C-ABI library loads and exports every symbol include/fdsnn_b200.h
declares (no compute calls: this runs on the CPU-only build container)."""
import ctypes
import os
import re

import pytest

from conftest import ROOT
from paper_2309_09025_b200 import _lib

HEADER = os.path.join(ROOT, "include", "fdsnn_b200.h")


def declared_symbols():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(fdsnn_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_the_binding_table():
    syms = declared_symbols()
    assert len(syms) >= 25
    assert set(syms) == set(_lib.SIGNATURES), set(syms) ^ set(_lib.SIGNATURES)


def test_library_exports_every_declared_symbol():
    if not os.path.exists(_lib.LIB_PATH):
        pytest.skip("library not built (run __graft_entry__.build())")
    lib = ctypes.CDLL(_lib.LIB_PATH)
    missing = [s for s in declared_symbols() if not hasattr(lib, s)]
    assert not missing, missing


def test_library_binds_and_reports_errors_without_gpu():
    if not os.path.exists(_lib.LIB_PATH):
        pytest.skip("library not built")
    lib = _lib.load()
    assert lib.fdsnn_row_stride(512) == 516 and lib.fdsnn_row_stride(742) == 744
    # invalid parameters are rejected before any device call
    prm = _lib.FdsnnParams(512, 1000, 25, 1024, 13, 2, 5, 5)
    h = ctypes.c_void_p()
    rc = lib.fdsnn_ctx_create(ctypes.byref(prm), 0, ctypes.byref(h))
    assert rc == _lib.FDSNN_ERR_PARAMETER
    assert b"ring degree" in lib.fdsnn_last_error()
    prm = _lib.FdsnnParams(512, 1024, 25, 1024, 7, 3, 5, 5)  # gadget does not cover q
    assert lib.fdsnn_ctx_create(ctypes.byref(prm), 0, ctypes.byref(h)) == _lib.FDSNN_ERR_PARAMETER
    # covers q, but y = centred(x) + (B/2-1)(1+B+B^2) overflows the int32
    # digit arithmetic of the rotation kernels: rejected, not silently wrong
    prm = _lib.FdsnnParams(512, 1024, 27, 1024, 11, 3, 3, 9)
    assert lib.fdsnn_ctx_create(ctypes.byref(prm), 0, ctypes.byref(h)) == _lib.FDSNN_ERR_PARAMETER
    assert b"int32 digit range" in lib.fdsnn_last_error()


def test_no_device_fails_loudly():
    """Without a CUDA device the accelerated path raises; there is no fallback."""
    try:
        import torch
        if torch.cuda.is_available():
            pytest.skip("GPU present")
    except ImportError:
        pass
    if not os.path.exists(_lib.LIB_PATH):
        pytest.skip("library not built")
    from paper_2309_09025_b200 import errors, params
    from paper_2309_09025_b200.device import DeviceContext
    with pytest.raises(errors.DeviceError):
        DeviceContext(params.preset("TOY"))
