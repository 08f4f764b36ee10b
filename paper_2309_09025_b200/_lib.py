"""ctypes binding of libfdsnn_b200.so (C ABI: include/fdsnn_b200.h).

The shared library is built in-tree by `__graft_entry__.build()` (nvcc,
sm_100a).  Loading fails loudly: there is no CPU fallback anywhere on the
accelerated path.
"""

from __future__ import annotations

import ctypes
import os

from .errors import DeviceError, DomainError, ParameterError

LIB_NAME = "libfdsnn_b200.so"
LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), LIB_NAME)

FDSNN_OK = 0
FDSNN_ERR_PARAMETER = 1
FDSNN_ERR_DOMAIN = 2
FDSNN_ERR_CUDA = 3
FDSNN_ERR_STATE = 4

# Every symbol declared in include/fdsnn_b200.h, with its ctypes signature.
_c_int = ctypes.c_int
_i32 = ctypes.c_int32
_i64 = ctypes.c_int64
_vp = ctypes.c_void_p
_dp = ctypes.POINTER(ctypes.c_double)
_i64p = ctypes.POINTER(ctypes.c_int64)
_i32p = ctypes.POINTER(ctypes.c_int32)


class FdsnnParams(ctypes.Structure):
    _fields_ = [("n", _i32), ("N", _i32), ("log2_q", _i32), ("p", _i32),
                ("bg_log", _i32), ("levels", _i32), ("ks_log", _i32), ("ks_levels", _i32)]


SIGNATURES = {
    "fdsnn_last_error": (ctypes.c_char_p, []),
    "fdsnn_row_stride": (_i32, [_i32]),
    "fdsnn_ctx_create": (_c_int, [ctypes.POINTER(FdsnnParams), _i32, ctypes.POINTER(_vp)]),
    "fdsnn_ctx_destroy": (_c_int, [_vp]),
    "fdsnn_ctx_stream": (_vp, [_vp]),
    "fdsnn_bsk_load": (_c_int, [_vp, _vp, _vp, _vp]),
    "fdsnn_ksk_load": (_c_int, [_vp, _vp, _vp]),
    "fdsnn_bsk_load_fdsn": (_c_int, [_vp, ctypes.c_char_p, ctypes.c_char_p]),
    "fdsnn_ciphertexts_load_fdsn": (_c_int, [_vp, ctypes.c_char_p, ctypes.c_char_p, _i64p, _i32p,
                                             _i64p, _vp, _vp]),
    "fdsnn_lut_load": (_c_int, [_vp, _vp, _i32p]),
    "fdsnn_pbs_batch": (_c_int, [_vp, _i32, _vp, _vp, _i64, _vp, _vp]),
    "fdsnn_lif_step_batch": (_c_int, [_vp, _i32, _i32, _i64, _vp, _vp, _vp, _vp, _i64,
                                      _vp, _vp, _vp, _vp]),
    "fdsnn_blind_rotate_batch": (_c_int, [_vp, _vp, _vp, _i64]),
    "fdsnn_key_switch_batch": (_c_int, [_vp, _vp, _vp, _i64, _vp, _vp]),
    "fdsnn_weight_sum": (_c_int, [_vp, _vp, _i64, _i64, _vp, _vp, _vp, _vp]),
    "fdsnn_rows_from_host": (_c_int, [_vp, _vp, _vp, _i64, _vp, _vp]),
    "fdsnn_rows_from_host_parts": (_c_int, [_vp, _i32, _vp, _vp, _vp, _vp, _vp]),
    "fdsnn_rows_to_host": (_c_int, [_vp, _vp, _i64, _vp, _vp, _vp]),
    "fdsnn_pbs_dev": (_c_int, [_vp, _i32, _i32p, _i64p, _i64p, _vp, _vp, _i64, _vp, _vp]),
    "fdsnn_operator_load": (_c_int, [_vp, _vp, _i64, _i64, _i32p]),
    "fdsnn_operator_apply": (_c_int, [_vp, _i32, _vp, _i64, _vp, _vp]),
    "fdsnn_rows_add": (_c_int, [_vp, _vp, _vp, _i64, _vp, _vp]),
    "fdsnn_plain_apply": (_c_int, [_vp, _i32, _vp, _i64, _vp, _vp]),
    "fdsnn_encrypt_rows": (_c_int, [_vp, _vp, _vp, _vp, _vp, _i64, _vp, _vp]),
    "fdsnn_decrypt_rows": (_c_int, [_vp, _vp, _vp, _i64, _vp, _vp]),
    "fdsnn_plain_lif": (_c_int, [_vp, _vp, _vp, _i64, _i64, _i64, _i64, _i64, _vp, _vp, _vp, _vp]),
    "fdsnn_dev_alloc": (_c_int, [_vp, _i64, ctypes.POINTER(_vp)]),
    "fdsnn_dev_free": (_c_int, [_vp, _vp]),
    "fdsnn_sync": (_c_int, [_vp]),
    "fdsnn_timing_enable": (_c_int, [_vp, _i32]),
    "fdsnn_timing_read": (_c_int, [_vp, _i32, _dp, _i64p]),
    "fdsnn_timing_reset": (_c_int, [_vp]),
    "fdsnn_margin_enable": (_c_int, [_vp, _i32]),
    "fdsnn_margin_read": (_c_int, [_vp, _dp]),
    "fdsnn_probe_fp64_peak": (_c_int, [_vp, _dp]),
    "fdsnn_flush_l2": (_c_int, [_vp, _vp]),
    "fdsnn_nt_forward": (_c_int, [_i32, _i32, _vp, _vp, _i64]),
    "fdsnn_nt_inverse": (_c_int, [_i32, _i32, _vp, _vp, _i64]),
    "fdsnn_negacyclic_mac": (_c_int, [_i32, _i32, _i32, _i32, _vp, _vp, _vp, _i64]),
    "fdsnn_gadget_decompose": (_c_int, [_i32, _i32, _i32, _i32, _vp, _i64, _i64, _vp]),
}

_lib = None


def load(path: str = LIB_PATH):
    """Load (once) and return the ctypes library; raises DeviceError if absent."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise DeviceError(
            f"{path} not built: run `python -c 'import __graft_entry__ as g; g.build()'` "
            "(the accelerated path has no CPU fallback)")
    lib = ctypes.CDLL(path)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def check(rc: int) -> None:
    """Map a C status code to the reference's exception types."""
    if rc == FDSNN_OK:
        return
    msg = _lib.fdsnn_last_error().decode(errors="replace") if _lib else "library error"
    if rc == FDSNN_ERR_PARAMETER:
        raise ParameterError(msg)
    if rc == FDSNN_ERR_DOMAIN:
        raise DomainError(msg)
    raise DeviceError(msg)
