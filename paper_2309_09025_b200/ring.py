"""Host-side integer helpers for Z_q and Z_q[X]/(X^N+1) (reference ring.py).

These are the rounding rules the device kernels reproduce bit for bit
(round-half-away on centred representatives, ring.py:27-67) plus the small
host utilities the key generator needs.  Nothing here is on the accelerated
path: ciphertext-batch work goes through the CUDA library.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

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
