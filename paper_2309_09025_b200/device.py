"""Device context: the Python face of one `fdsnn_ctx` (C ABI, include/fdsnn_b200.h).

A context owns, on one B200, the Fourier-domain bootstrapping key (computed on
the device from the integer RGSW rows), the key-switch key, the registered
test polynomials and the integer weight operators.  Host-buffer calls
(`pbs_batch`, `lif_step_batch`, ...) copy in and out inside the C library;
device calls (`*_dev`) operate on device-resident ciphertext rows held in
torch tensors (torch is used only as the device allocator / stream source).
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _lib
from .errors import DeviceError, DomainError, ParameterError
from .params import FheParams


def _i64(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.int64))


def _ptr(a: np.ndarray):
    return ctypes.c_void_p(a.ctypes.data)


def _tptr(t):
    return ctypes.c_void_p(t.data_ptr()) if t is not None else None


def _log2(x: int) -> int:
    return int(x).bit_length() - 1


class DeviceContext:
    """Owns one C context; all methods raise DeviceError/ParameterError on failure."""

    def __init__(self, params: FheParams, device: int = 0):
        self.lib = _lib.load()
        self.params = params
        self.device = device
        prm = _lib.FdsnnParams(params.n, params.N, _log2(params.q), params.p,
                               params.gadget.log2_base, params.gadget.levels,
                               _log2(params.ks_base), params.ks_levels)
        h = ctypes.c_void_p()
        _lib.check(self.lib.fdsnn_ctx_create(ctypes.byref(prm), device, ctypes.byref(h)))
        self.h = h
        self.stride = int(self.lib.fdsnn_row_stride(params.n))
        self._luts: dict[bytes, int] = {}
        self._ops: dict[int, tuple] = {}
        self.keys_loaded = False

    def close(self):
        if getattr(self, "h", None):
            self.lib.fdsnn_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ---------------------------------------------------------------- keys
    def load_keys(self, rows: np.ndarray, ksk_A: np.ndarray, ksk_b: np.ndarray) -> None:
        p = self.params
        rows = _i64(rows)
        if rows.shape != (p.n, 2 * p.gadget.levels, 2, p.N):
            raise ParameterError(f"RGSW rows shape {rows.shape} does not match params")
        ksk_A, ksk_b = _i64(ksk_A), _i64(ksk_b)
        if ksk_A.shape != (p.N * p.ks_levels, p.n) or ksk_b.shape != (p.N * p.ks_levels,):
            raise ParameterError("key-switch key shape does not match params")
        _lib.check(self.lib.fdsnn_bsk_load(self.h, _ptr(rows), _ptr(ksk_A), _ptr(ksk_b)))
        self.keys_loaded = True

    def load_key_switch_key(self, ksk_A: np.ndarray, ksk_b: np.ndarray) -> None:
        """Only the key-switch key (no bootstrapping key is stored or transformed)."""
        p = self.params
        ksk_A, ksk_b = _i64(ksk_A), _i64(ksk_b)
        if ksk_A.shape != (p.N * p.ks_levels, p.n) or ksk_b.shape != (p.N * p.ks_levels,):
            raise ParameterError("key-switch key shape does not match params")
        _lib.check(self.lib.fdsnn_ksk_load(self.h, _ptr(ksk_A), _ptr(ksk_b)))

    def load_keys_fdsn(self, path: str) -> None:
        """Bootstrapping + key-switch key straight from a reference FDSN BK file."""
        _lib.check(self.lib.fdsnn_bsk_load_fdsn(self.h, str(path).encode(),
                                                self.params.digest().encode()))
        self.keys_loaded = True

    def ciphertexts_fdsn(self, path: str):
        """(device rows, tensor shape) of a reference FDSN CT file."""
        cnt = ctypes.c_int64()
        nd = ctypes.c_int32()
        shape = (ctypes.c_int64 * 8)()
        args = (self.h, str(path).encode(), self.params.digest().encode(), ctypes.byref(cnt),
                ctypes.byref(nd), shape)
        _lib.check(self.lib.fdsnn_ciphertexts_load_fdsn(*args, None, None))
        rows = self.empty_rows(int(cnt.value))
        _lib.check(self.lib.fdsnn_ciphertexts_load_fdsn(*args, _tptr(rows), self._stream()))
        return rows, tuple(int(shape[i]) for i in range(nd.value))

    def lut(self, testpoly: np.ndarray) -> int:
        tp = _i64(testpoly)
        if tp.shape != (self.params.N,):
            raise ParameterError("test polynomial must have N coefficients")
        key = tp.tobytes()
        lid = self._luts.get(key)
        if lid is None:
            out = ctypes.c_int32()
            _lib.check(self.lib.fdsnn_lut_load(self.h, _ptr(tp), ctypes.byref(out)))
            lid = self._luts[key] = int(out.value)
        return lid

    # ------------------------------------------------ host-buffer entry points
    def pbs_batch(self, lut_id: int, A, b):
        A, b = _i64(A), _i64(b)
        cnt = len(b)
        outA = np.empty((cnt, self.params.n), dtype=np.int64)
        outb = np.empty(cnt, dtype=np.int64)
        _lib.check(self.lib.fdsnn_pbs_batch(self.h, lut_id, _ptr(A), _ptr(b), cnt,
                                            _ptr(outA), _ptr(outb)))
        return outA, outb

    def lif_step_batch(self, lut_fire: int, lut_reset: int, v_th_hat: int, vA, vb, iA, ib):
        vA, vb, iA, ib = _i64(vA), _i64(vb), _i64(iA), _i64(ib)
        cnt = len(vb)
        n = self.params.n
        out = [np.empty((cnt, n), np.int64), np.empty(cnt, np.int64),
               np.empty((cnt, n), np.int64), np.empty(cnt, np.int64)]
        _lib.check(self.lib.fdsnn_lif_step_batch(
            self.h, lut_fire, lut_reset, int(v_th_hat), _ptr(vA), _ptr(vb), _ptr(iA), _ptr(ib),
            cnt, *[_ptr(o) for o in out]))
        return tuple(out)

    def blind_rotate_batch(self, acc: np.ndarray, a2N):
        """Rotates the C-contiguous int64 `acc` in place (the C entry point
        writes the results back into the caller's buffer) and returns it."""
        if acc.dtype != np.int64 or not acc.flags.c_contiguous or not acc.flags.writeable:
            raise ParameterError("accumulator must be a writeable C-contiguous int64 array")
        a2N = _i64(a2N)
        _lib.check(self.lib.fdsnn_blind_rotate_batch(self.h, _ptr(acc), _ptr(a2N), acc.shape[0]))
        return acc

    def key_switch_batch(self, A, b):
        A, b = _i64(A), _i64(b)
        cnt = len(b)
        outA = np.empty((cnt, self.params.n), np.int64)
        outb = np.empty(cnt, np.int64)
        _lib.check(self.lib.fdsnn_key_switch_batch(self.h, _ptr(A), _ptr(b), cnt,
                                                   _ptr(outA), _ptr(outb)))
        return outA, outb

    def weight_sum(self, M, A, b):
        M, A, b = _i64(M), _i64(A), _i64(b)
        out_cells, in_cells = M.shape
        outA = np.empty((out_cells, self.params.n), np.int64)
        outb = np.empty(out_cells, np.int64)
        _lib.check(self.lib.fdsnn_weight_sum(self.h, _ptr(M), out_cells, in_cells, _ptr(A),
                                             _ptr(b), _ptr(outA), _ptr(outb)))
        return outA, outb

    # ------------------------------------------------- device-resident path
    @staticmethod
    def _torch():
        import torch
        if not torch.cuda.is_available():
            raise DeviceError("CUDA device not available to torch")
        return torch

    def _stream(self):
        torch = self._torch()
        return ctypes.c_void_p(torch.cuda.current_stream(self.device).cuda_stream)

    def empty_rows(self, count: int):
        torch = self._torch()
        return torch.empty((max(count, 0), self.stride), dtype=torch.int32,
                           device=f"cuda:{self.device}")

    def zero_rows(self, count: int):
        t = self.empty_rows(count)
        t.zero_()
        return t

    def rows_from_host(self, A, b, out=None):
        """int64 host (A, b) -> device rows (a new tensor, or the rows of `out`)."""
        A, b = _i64(A), _i64(b)
        if A.ndim != 2 or A.shape != (len(b), self.params.n):
            raise ParameterError("ciphertext arrays do not match params")
        rows = self.empty_rows(len(b)) if out is None else out
        if rows.shape[0] != len(b):
            raise ParameterError("output rows do not match the ciphertext count")
        _lib.check(self.lib.fdsnn_rows_from_host(self.h, _ptr(A), _ptr(b), len(b),
                                                 _tptr(rows), self._stream()))
        return rows

    def rows_from_host_parts(self, parts, out=None):
        """[(A, b), ...] int64 host arrays -> device rows stacked in order."""
        arrs = []
        for A, b in parts:
            A, b = _i64(A), _i64(b)
            if A.ndim != 2 or A.shape != (len(b), self.params.n):
                raise ParameterError("ciphertext arrays do not match params")
            arrs.append((A, b))
        total = sum(len(b) for _, b in arrs)
        rows = self.empty_rows(total) if out is None else out
        if rows.shape[0] != total:
            raise ParameterError("output rows do not match the ciphertext count")
        k = len(arrs)
        pa = (ctypes.c_void_p * k)(*[a.ctypes.data for a, _ in arrs])
        pb = (ctypes.c_void_p * k)(*[b.ctypes.data for _, b in arrs])
        cnt = (ctypes.c_int64 * k)(*[len(b) for _, b in arrs])
        _lib.check(self.lib.fdsnn_rows_from_host_parts(self.h, k, pa, pb, cnt, _tptr(rows), self._stream()))
        return rows

    def rows_to_host(self, rows):
        cnt = rows.shape[0]
        A = np.empty((cnt, self.params.n), np.int64)
        b = np.empty(cnt, np.int64)
        _lib.check(self.lib.fdsnn_rows_to_host(self.h, _tptr(rows), cnt, _ptr(A), _ptr(b),
                                               self._stream()))
        return A, b

    def pbs_dev(self, lut_ids, in_boff, out_boff, rows, rows2=None, out=None):
        nl = len(lut_ids)
        cnt = rows.shape[0]
        if out is None:
            out = self.empty_rows(nl * cnt)
        ids = (ctypes.c_int32 * nl)(*[int(x) for x in lut_ids])
        ib = (ctypes.c_int64 * nl)(*[int(x) for x in in_boff])
        ob = (ctypes.c_int64 * nl)(*[int(x) for x in out_boff])
        _lib.check(self.lib.fdsnn_pbs_dev(self.h, nl, ids, ib, ob, _tptr(rows), _tptr(rows2),
                                          cnt, _tptr(out), self._stream()))
        return out

    def operator(self, matrix) -> int:
        key = id(matrix)
        hit = self._ops.get(key)
        if hit is not None and hit[0] is matrix:
            return hit[1]
        M = _i64(matrix)
        out = ctypes.c_int32()
        _lib.check(self.lib.fdsnn_operator_load(self.h, _ptr(M), M.shape[0], M.shape[1],
                                                ctypes.byref(out)))
        self._ops[key] = (matrix, int(out.value))
        return int(out.value)

    def apply(self, op_id: int, rows, batch: int, out_cells: int, out=None):
        if out is None:
            out = self.empty_rows(batch * out_cells)
        _lib.check(self.lib.fdsnn_operator_apply(self.h, op_id, _tptr(rows), batch, _tptr(out),
                                                 self._stream()))
        return out

    def rows_add(self, x, y, out=None):
        if out is None:
            out = self.empty_rows(x.shape[0])
        _lib.check(self.lib.fdsnn_rows_add(self.h, _tptr(x), _tptr(y), x.shape[0], _tptr(out),
                                           self._stream()))
        return out

    # ------------------------------------------- client side on device (8(f)4)
    def encrypt_rows(self, ms, sk, rng, sigma=None):
        """lwe.encrypt_batch with the device computing b = <A,s> + e + Delta*m.
        A and e are drawn from `rng` exactly as the reference draws them, so the
        rows equal the reference's (A, b) for the same generator state."""
        from .lwe import sample_noise
        p = self.params
        ms = _i64(np.asarray(ms).ravel())
        if np.any(ms < -p.p // 2 + 1) or np.any(ms > p.p // 2):
            raise DomainError("message outside centered Z_p")  # before any draw, as lwe.py:79-80
        grid = p.grid
        A = _i64(rng.integers(0, p.q // grid, size=(ms.size, p.n)) * grid)
        sig = p.sigma if sigma is None else sigma
        e = _i64(sample_noise(rng, sig, ms.size) if sig > 0 else np.zeros(ms.size, dtype=np.int64))
        rows = self.empty_rows(ms.size)
        _lib.check(self.lib.fdsnn_encrypt_rows(self.h, _ptr(_i64(sk.s)), _ptr(A), _ptr(e), _ptr(ms), ms.size,
                                               _tptr(rows), self._stream()))
        return rows

    def decrypt_rows(self, rows, sk) -> np.ndarray:
        """lwe.decrypt_batch of device rows (lwe.py:89-96)."""
        out = np.empty(rows.shape[0], dtype=np.int64)
        _lib.check(self.lib.fdsnn_decrypt_rows(self.h, _ptr(_i64(sk.s)), _tptr(rows), rows.shape[0], _ptr(out),
                                               self._stream()))
        return out

    # ------------------------------------------ mod-p plaintext twin (8(f)1)
    def plain_apply(self, op_id: int, x, batch: int, out_cells: int):
        """int64 device vectors: y[b] = M x[b] (oracle.plain_infer weight layer)."""
        torch = self._torch()
        y = torch.empty((batch, out_cells), dtype=torch.int64, device=x.device)
        _lib.check(self.lib.fdsnn_plain_apply(self.h, op_id, _tptr(x), batch, _tptr(y), self._stream()))
        return y

    def plain_lif(self, v, i, lif, p: int | None, overflow=None):
        """neuron.plain_lif_step_batch on int64 device tensors -> (spike2, v_next).
        With p, out-of-range charges are counted into `overflow` (int64[1])."""
        torch = self._torch()
        spike2 = torch.empty_like(v)
        v_next = torch.empty_like(v)
        _lib.check(self.lib.fdsnn_plain_lif(self.h, _tptr(v), _tptr(i), v.numel(), int(lif.v_th_hat),
                                            int(lif.leak_num), int(lif.leak_den), int(p or 0),
                                            _tptr(spike2), _tptr(v_next),
                                            _tptr(overflow) if overflow is not None else None,
                                            self._stream()))
        return spike2, v_next

    # ------------------------------------------------------ instrumentation
    def sync(self):
        _lib.check(self.lib.fdsnn_sync(self.h))

    def timing(self, on: bool):
        _lib.check(self.lib.fdsnn_timing_enable(self.h, 1 if on else 0))

    def timing_read(self, which: int):
        ms = ctypes.c_double()
        n = ctypes.c_int64()
        _lib.check(self.lib.fdsnn_timing_read(self.h, which, ctypes.byref(ms), ctypes.byref(n)))
        return ms.value, n.value

    def timing_reset(self):
        _lib.check(self.lib.fdsnn_timing_reset(self.h))

    def margin(self, on: bool | None = None):
        if on is not None:
            _lib.check(self.lib.fdsnn_margin_enable(self.h, 1 if on else 0))
            return None
        v = ctypes.c_double()
        _lib.check(self.lib.fdsnn_margin_read(self.h, ctypes.byref(v)))
        return v.value

    def fp64_peak_tflops(self) -> float:
        v = ctypes.c_double()
        _lib.check(self.lib.fdsnn_probe_fp64_peak(self.h, ctypes.byref(v)))
        return v.value

    def flush_l2(self):
        _lib.check(self.lib.fdsnn_flush_l2(self.h, self._stream()))
