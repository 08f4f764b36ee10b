"""Host-side integer helpers for Z_q and Z_q[X]/(X^N+1) (reference ring.py).

These are the rounding rules the device kernels reproduce bit for bit
(round-half-away on centred representatives, ring.py:27-67), the small host
utilities the key generator needs (`negacyclic_mul_raw` for RLWE bodies,
`monomial_rotate_raw` for test polynomials) and the value types
(`ZqElement`, `NegacyclicPoly`).  The algebra API that does real polynomial
arithmetic -- `NegacyclicTransform`, `poly_mul`, `poly_mul_schoolbook` --
runs on the GPU through the C library (csrc/ring_ops.cuh) and, like every
compute path of this package, has no CPU fallback.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass
from functools import lru_cache

import numpy as np

from . import _lib
from .errors import ParameterError


def is_power_of_two(x: int) -> bool:
    return x > 0 and (x & (x - 1)) == 0


def center(values, q: int):
    """Residues in [0,q) -> centred representatives in [-q/2, q/2) (ring.py:27-33)."""
    v = np.asarray(values, dtype=np.int64)
    out = np.where(v >= q // 2, v - q, v)
    return int(out) if out.ndim == 0 else out


def round_half_away(x):
    """Round to nearest, ties away from zero (ring.py:36-42)."""
    x = np.asarray(x)
    out = np.where(x >= 0, np.floor(x + 0.5), np.ceil(x - 0.5))
    return int(out) if out.ndim == 0 else out.astype(np.int64)


def div_round_half_away(num, den: int):
    """Exact integer round-half-away of num/den, den > 0 (ring.py:45-53)."""
    num = np.asarray(num, dtype=np.int64)
    r = (2 * np.abs(num) + den) // (2 * den)
    out = np.where(num >= 0, r, -r)
    return int(out) if out.ndim == 0 else out


def rescale(x, q1: int, q2: int):
    """round(x*q2/q1) mod q2 on the centred representative of x mod q1 (ring.py:56-67)."""
    if not (is_power_of_two(q1) and is_power_of_two(q2)):
        raise ParameterError("moduli must be powers of two")
    c = center(np.asarray(x, dtype=np.int64) % q1, q1)
    if q1 >= q2:
        out = div_round_half_away(np.asarray(c) * q2, q1) % q2
    else:
        out = (np.asarray(c) * (q2 // q1)) % q2
    return int(np.asarray(out)) if np.ndim(x) == 0 else out


def monomial_rotate_raw(coeffs: np.ndarray, k, N: int) -> np.ndarray:
    """X^k * p(X) with the X^N = -1 wrap; k scalar or one per leading row (ring.py:226-242)."""
    k = np.asarray(k, dtype=np.int64) % (2 * N)
    src = (np.arange(N, dtype=np.int64) - k[..., None]) % (2 * N)
    sign = np.where(src >= N, -1, 1)
    coeffs = np.asarray(coeffs)
    if coeffs.ndim < sign.ndim:
        coeffs = np.broadcast_to(coeffs, sign.shape[:-1] + coeffs.shape[-1:])
    return sign * np.take_along_axis(coeffs, src % N, axis=-1)


def negacyclic_mul_raw(a: np.ndarray, b: np.ndarray, q: int) -> np.ndarray:
    """Exact negacyclic product of centred int arrays (..., N), reduced mod q.

    Host utility for key generation (RLWE bodies a*z).  It uses a length-2N
    real FFT of the zero-padded operands followed by the X^N = -1 fold; the
    result is exact whenever N*max|a|*max|b| << 2^52, which holds for every
    preset (binary z, |a| < q/2 <= 2^30).
    """
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    N = a.shape[-1]
    fa = np.fft.rfft(a, 2 * N, axis=-1)
    fb = np.fft.rfft(b, 2 * N, axis=-1)
    full = np.fft.irfft(fa * fb, 2 * N, axis=-1)
    prod = full[..., :N] - full[..., N:]
    return round_half_away(prod) % q


@dataclass(frozen=True)
class NegacyclicPoly:
    """Element of Z_q[X]/(X^N + 1), coefficients reduced into [0, q)."""

    coeffs: np.ndarray
    q: int

    def __post_init__(self):
        c = np.asarray(self.coeffs, dtype=np.int64) % self.q
        if not is_power_of_two(len(c)) or not is_power_of_two(self.q):
            raise ParameterError("N and q must be powers of two")
        c.setflags(write=False)
        object.__setattr__(self, "coeffs", c)

    @property
    def N(self) -> int:
        return len(self.coeffs)

    @property
    def centered(self) -> np.ndarray:
        return center(self.coeffs, self.q)

    @staticmethod
    def constant(c: int, N: int, q: int) -> "NegacyclicPoly":
        coeffs = np.zeros(N, dtype=np.int64)
        coeffs[0] = c % q
        return NegacyclicPoly(coeffs, q)

    @staticmethod
    def zero(N: int, q: int) -> "NegacyclicPoly":
        return NegacyclicPoly(np.zeros(N, dtype=np.int64), q)

    def _check(self, other: "NegacyclicPoly") -> None:
        if self.q != other.q or self.N != other.N:
            raise ParameterError("ring parameters mismatch")

    def __add__(self, other: "NegacyclicPoly") -> "NegacyclicPoly":
        self._check(other)
        return NegacyclicPoly(self.coeffs + other.coeffs, self.q)

    def __sub__(self, other: "NegacyclicPoly") -> "NegacyclicPoly":
        self._check(other)
        return NegacyclicPoly(self.coeffs - other.coeffs, self.q)

    def __eq__(self, other) -> bool:
        return (isinstance(other, NegacyclicPoly) and self.q == other.q
                and np.array_equal(self.coeffs, other.coeffs))

    __hash__ = None


@dataclass(frozen=True)
class ZqElement:
    """Scalar of Z_q, q a power of two (ring.py:71-100)."""

    value: int
    q: int

    def __post_init__(self):
        if not is_power_of_two(self.q):
            raise ParameterError("q must be a power of two")
        object.__setattr__(self, "value", int(self.value) % self.q)

    @property
    def centered(self) -> int:
        return center(self.value, self.q)

    def _same(self, other: "ZqElement") -> None:
        if self.q != other.q:
            raise ParameterError("modulus mismatch")

    def __add__(self, other: "ZqElement") -> "ZqElement":
        self._same(other)
        return ZqElement(self.value + other.value, self.q)

    def __sub__(self, other: "ZqElement") -> "ZqElement":
        self._same(other)
        return ZqElement(self.value - other.value, self.q)

    def __mul__(self, other: "ZqElement") -> "ZqElement":
        self._same(other)
        return ZqElement(self.value * other.value, self.q)


def monomial_rotate(p: NegacyclicPoly, k: int) -> NegacyclicPoly:
    """X^k * p with the X^N = -1 sign wrap, k modulo 2N (ring.py:245-247)."""
    return NegacyclicPoly(monomial_rotate_raw(p.coeffs, int(k), p.N), p.q)


# --------------------------------------------------------------------------
# device algebra (csrc/ring_ops.cuh)
# --------------------------------------------------------------------------
def _dev() -> int:
    import torch  # noqa: F401  (device index of the current torch device, if any)
    return int(torch.cuda.current_device()) if torch.cuda.is_available() else 0


def _f64(x) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(x, dtype=np.float64))


class NegacyclicTransform:
    """Length-N negacyclic transform through a half-size complex DFT
    (ring.py:103-137), evaluated on the GPU.

    forward: c_k = (a_k + i a_{k+N/2}) e^{i pi k/N}, then the unnormalised
    N/2-point DFT with the e^{+2 pi i jk/(N/2)} kernel; inverse: the e^{-}
    DFT divided by N/2, times e^{-i pi k/N}, real parts then imaginary parts
    (unrounded).  FP64 throughout; agrees with the reference's pocketfft
    transform to rounding (tests/test_gpu_ring.py).
    """

    def __init__(self, N: int):
        if not is_power_of_two(N) or N < 2:
            raise ParameterError("N must be a power of two >= 2")
        if N > 4096:
            raise ParameterError("device negacyclic transform supports N <= 4096")
        self.N = N
        k = np.arange(N // 2)
        self.twist = np.exp(1j * np.pi * k / N)
        self.untwist = np.conj(self.twist)

    def forward(self, coeffs: np.ndarray) -> np.ndarray:
        """(..., N) int/float -> (..., N/2) complex evaluations."""
        a = _f64(coeffs)
        if a.shape[-1] != self.N:
            raise ParameterError(f"expected trailing length {self.N}")
        lead = a.shape[:-1]
        out = np.empty(lead + (self.N,), dtype=np.float64)  # N/2 interleaved complex
        lib = _lib.load()
        _lib.check(lib.fdsnn_nt_forward(_dev(), self.N, ctypes.c_void_p(a.ctypes.data),
                                        ctypes.c_void_p(out.ctypes.data), int(np.prod(lead, dtype=np.int64))))
        return out.view(np.complex128)

    def inverse(self, evals: np.ndarray) -> np.ndarray:
        """(..., N/2) complex -> (..., N) float coefficients (unrounded)."""
        e = np.ascontiguousarray(np.asarray(evals, dtype=np.complex128))
        if e.shape[-1] != self.N // 2:
            raise ParameterError(f"expected trailing length {self.N // 2}")
        lead = e.shape[:-1]
        out = np.empty(lead + (self.N,), dtype=np.float64)
        lib = _lib.load()
        _lib.check(lib.fdsnn_nt_inverse(_dev(), self.N, ctypes.c_void_p(e.ctypes.data),
                                        ctypes.c_void_p(out.ctypes.data), int(np.prod(lead, dtype=np.int64))))
        return out


@lru_cache(maxsize=None)
def get_transform(N: int) -> NegacyclicTransform:
    return NegacyclicTransform(N)


def negacyclic_mac_device(x: np.ndarray, y: np.ndarray, q: int) -> np.ndarray:
    """sum_d x[..., d, :] * y[..., d, :] mod (X^N + 1, q), exact, on the GPU.

    x, y (..., D, N) int64 (any representatives) -> (..., N) in [0, q)."""
    if not is_power_of_two(q):
        raise ParameterError("q must be a power of two")
    x = np.ascontiguousarray(np.asarray(x, dtype=np.int64))
    y = np.ascontiguousarray(np.asarray(y, dtype=np.int64))
    if x.shape != y.shape or x.ndim < 2:
        raise ParameterError("operand shapes differ")
    D, N = x.shape[-2:]
    lead = x.shape[:-2]
    out = np.empty(lead + (N,), dtype=np.int64)
    lib = _lib.load()
    _lib.check(lib.fdsnn_negacyclic_mac(_dev(), N, q.bit_length() - 1, D, ctypes.c_void_p(x.ctypes.data),
                                        ctypes.c_void_p(y.ctypes.data), ctypes.c_void_p(out.ctypes.data),
                                        int(np.prod(lead, dtype=np.int64))))
    return out


def poly_mul_schoolbook(a: NegacyclicPoly, b: NegacyclicPoly) -> NegacyclicPoly:
    """Exact negacyclic product (ring.py:200-207), computed on the GPU."""
    a._check(b)
    return NegacyclicPoly(negacyclic_mac_device(a.coeffs[None], b.coeffs[None], a.q), a.q)


def poly_mul(a: NegacyclicPoly, b: NegacyclicPoly) -> NegacyclicPoly:
    """Negacyclic product (ring.py:218-223).  The reference's transform path
    is exact at the preset sizes; the device computes the exact product
    directly, so the results are identical there and exact everywhere."""
    return poly_mul_schoolbook(a, b)

