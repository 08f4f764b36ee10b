"""Programmable bootstrapping (drop-in for reference bootstrap.py).

Initialize -> BlindRotate -> Extract -> KeySwitch, evaluated on the B200 by
`csrc/pbs.cuh` + `csrc/keyswitch.cuh` through the C ABI.  Host code here
builds the lookup tables and test polynomials (bootstrap.py:42-96), runs
key generation with the reference's RNG order (bootstrap.py:137-155), and
keeps the reference call signatures:

    bootstrap_batch(g, A, b, bsk) -> (A', b')          bootstrap.py:324-341
    blind_rotate_batch(acc, a2N, bsk) -> acc            bootstrap.py:252-282
    sample_extract_batch(acc) -> (ea, eb)               bootstrap.py:291-295
    key_switch_batch(A, b, ksk, params) -> (A', b')     bootstrap.py:303-316

Outputs are bit-identical to the reference for identical keys and inputs.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .errors import DomainError, ParameterError
from .lwe import LweCiphertext, LweSecretKey, sample_noise
from .params import FheParams
from .rgsw import RgswCiphertext, RlweCiphertext, RlweSecretKey, rgsw_encrypt_bit
from .ring import monomial_rotate_raw


class ProgramFunction:
    """Negacyclic LUT g: Z_p -> Z_p with g(v + p/2) = -g(v) (bootstrap.py:42-71)."""

    def __init__(self, table, p: int):
        table = np.asarray(table, dtype=np.int64)
        if table.shape != (p,):
            raise ParameterError(f"program table must have length p={p}")
        self.p = p
        half = p // 2
        resid = table % p
        if not np.array_equal(np.roll(resid, -half), (-resid) % p):
            raise DomainError("program function violates g(v + p/2) = -g(v)")
        self.table = ((resid + half - 1) % p) - (half - 1)
        self.table.setflags(write=False)

    def __call__(self, m):
        return self.table[np.asarray(m) % self.p]

    def __eq__(self, other):
        return (isinstance(other, ProgramFunction) and self.p == other.p
                and np.array_equal(self.table, other.table))

    __hash__ = None


def make_program(g_values, p: int) -> ProgramFunction:
    """LUT from values on [0, p/2); negative half by antisymmetry (bootstrap.py:74-87)."""
    half = p // 2
    get = g_values if callable(g_values) else g_values.__getitem__
    pos = np.array([int(get(v)) for v in range(half)], dtype=np.int64)
    return ProgramFunction(np.concatenate([pos, -pos]), p)


def test_polynomial(g: ProgramFunction, params: FheParams) -> np.ndarray:
    """v_i = Delta * g(floor(i*p/2N)) mod q (bootstrap.py:90-96)."""
    if g.p != params.p:
        raise ParameterError("program function is for a different message modulus")
    slots = (np.arange(params.N, dtype=np.int64) * params.p) // (2 * params.N)
    return (params.delta * g.table[slots]) % params.q


test_polynomial.__test__ = False  # not a pytest test


@dataclass(frozen=True)
class KeySwitchKey:
    """LWE encryptions of z_j*base^i under s, row j*levels+i (bootstrap.py:99-110)."""

    A: np.ndarray  # (N*levels, n)
    b: np.ndarray  # (N*levels,)
    base: int
    levels: int
    N: int

    def digest_arrays(self):
        return [self.A, self.b]


class BootstrapKey:
    """n RGSW(s_i) plus the key-switch key; read-only after generation.

    Accepts the reference constructor signature BootstrapKey(ek, ksk, params).
    The Fourier-domain key lives on the device (computed there on first use,
    `device` property); `bootstrap_count` counts ciphertexts bootstrapped.
    """

    def __init__(self, ek, ksk: KeySwitchKey, params: FheParams, *, rows: np.ndarray | None = None):
        self.params = params
        self.ksk = ksk
        self.bootstrap_count = 0
        if rows is None:
            rows = np.stack([np.stack([e.rows_a, e.rows_b], axis=1) for e in ek])
        self.rows = np.ascontiguousarray(rows, dtype=np.int64)  # (n, 2l, 2, N)
        self._ek = list(ek) if ek is not None else None
        self._device = None

    @property
    def n(self) -> int:
        return self.rows.shape[0]

    @property
    def ek(self) -> list:
        if self._ek is None:
            g = self.params.gadget
            self._ek = [RgswCiphertext(r[:, 0, :], r[:, 1, :], self.params.q, g) for r in self.rows]
        return self._ek

    @property
    def device(self):
        """The DeviceContext holding this key (created and loaded on first use)."""
        if self._device is None:
            from .device import DeviceContext
            ctx = DeviceContext(self.params)
            ctx.load_keys(self.rows, self.ksk.A, self.ksk.b)
            self._device = ctx
            _register_ks_device(self.ksk, self.params, ctx)
        return self._device

    def __getstate__(self):
        d = dict(self.__dict__)
        d["_device"] = None
        return d


def gen_key_switch_key(zk: RlweSecretKey, sk: LweSecretKey, params: FheParams,
                       rng: np.random.Generator) -> KeySwitchKey:
    """RNG order as bootstrap.py:137-148: mask grid draw, noise draw."""
    N, n = params.N, params.n
    base, levels = params.ks_base, params.ks_levels
    count = N * levels
    grid = params.grid
    A = (rng.integers(0, params.q // grid, size=(count, n)) * grid).astype(np.int64)
    e = sample_noise(rng, params.sigma_ks, count)
    payload = (zk.z[:, None] * (base ** np.arange(levels, dtype=np.int64))[None, :]).ravel()
    b = (A @ sk.s + e + payload) % params.q
    return KeySwitchKey(A, b.astype(np.int64), base, levels, N)


def gen_bootstrap_key(sk: LweSecretKey, zk: RlweSecretKey, params: FheParams,
                      rng: np.random.Generator) -> BootstrapKey:
    """n RGSW bit encryptions then the KSK, in the reference's order (bootstrap.py:151-155)."""
    ek = [rgsw_encrypt_bit(int(s_i), zk, params, rng) for s_i in sk.s]
    ksk = gen_key_switch_key(zk, sk, params, rng)
    return BootstrapKey(ek, ksk, params)


def initialize_accumulator(g: ProgramFunction, b2N: int, params: FheParams) -> RlweCiphertext:
    """Noiseless RLWE of X^{-b2N} * testpoly(g) (bootstrap.py:158-166)."""
    v = test_polynomial(g, params)
    rotated = monomial_rotate_raw(v, -int(b2N) % (2 * params.N), params.N)
    return RlweCiphertext(np.zeros(params.N, dtype=np.int64), rotated, params.q)


def _device_of(bsk):
    """Device context for our BootstrapKey or a reference-package key object."""
    if isinstance(bsk, BootstrapKey):
        return bsk.device
    dev = getattr(bsk, "_b200_device", None)
    if dev is None:
        from .device import DeviceContext
        params = bsk.params
        rows = np.stack([np.stack([e.rows_a, e.rows_b], axis=1) for e in bsk.ek])
        dev = DeviceContext(params)
        dev.load_keys(rows, bsk.ksk.A, bsk.ksk.b)
        bsk._b200_device = dev
    return dev


def blind_rotate_batch(acc: np.ndarray, a2N: np.ndarray, bsk) -> np.ndarray:
    """Rotate (B,2,N) accumulators by the encrypted phases a2N (B,n) (bootstrap.py:252-282).

    Same ownership as the reference: `acc` goes through np.ascontiguousarray,
    so a C-contiguous int64 array is rotated in place and returned (the
    reference's numba kernels write into it, bootstrap.py:263,281); any other
    array is copied first.  When no step rotates anything (every a2N entry is
    0 mod 2N: the reference skips every step, bootstrap.py:274-276) the
    accumulators come back untouched, unreduced values included.
    """
    params = bsk.params
    acc = np.ascontiguousarray(acc)
    a2N = np.asarray(a2N, dtype=np.int64)
    if acc.ndim != 3 or acc.shape[1:] != (2, params.N) or a2N.shape != (acc.shape[0], params.n):
        raise ParameterError("accumulator / rotation shapes do not match params")
    if not (a2N % (2 * params.N)).any():
        return acc
    if acc.dtype != np.int64 or not acc.flags.writeable:
        acc = acc.astype(np.int64)
    return _device_of(bsk).blind_rotate_batch(acc, a2N)


def blind_rotate(acc: RlweCiphertext, a2N, bsk) -> RlweCiphertext:
    arr = np.stack([acc.a, acc.b])[None, ...]
    out = blind_rotate_batch(arr, np.asarray(a2N, dtype=np.int64)[None, :], bsk)
    return RlweCiphertext(out[0, 0], out[0, 1], bsk.params.q)


def sample_extract_batch(acc: np.ndarray):
    """(B,2,N) -> LWE under z: (a_0, -a_{N-1}, ..., -a_1), b = body_0 (bootstrap.py:291-295).

    Pure index permutation of host arrays (the device path fuses it into the
    blind-rotation epilogue).
    """
    acc = np.asarray(acc)
    a = acc[:, 0, :]
    ea = np.concatenate([a[:, :1], -a[:, -1:0:-1]], axis=1)
    return ea, acc[:, 1, 0].copy()


def sample_extract(acc: RlweCiphertext) -> LweCiphertext:
    ea, eb = sample_extract_batch(np.stack([acc.a, acc.b])[None, ...])
    return LweCiphertext(ea[0], int(eb[0]), acc.q)


# Device contexts able to key-switch with a given KeySwitchKey, keyed by
# (id(ksk), params digest).  A bootstrapping key's context registers its own
# key-switch key when it is created, so key_switch_batch(..., bsk.ksk, ...)
# reuses it; a standalone key gets a context holding only the key-switch key.
# Entries die with their key (weakref.finalize), so nothing accumulates.
_KS_DEVICES: dict = {}


def _register_ks_device(ksk, params: FheParams, ctx) -> None:
    import weakref
    key = (id(ksk), params.digest())
    if key in _KS_DEVICES:
        return
    try:
        ref = weakref.ref(ksk)
    except TypeError:  # not weak-referenceable: do not cache
        return
    _KS_DEVICES[key] = (ref, weakref.ref(ctx))
    weakref.finalize(ksk, _KS_DEVICES.pop, key, None)


def _key_device(ksk: KeySwitchKey, params: FheParams):
    hit = _KS_DEVICES.get((id(ksk), params.digest()))
    if hit is not None and hit[0]() is ksk:
        ctx = hit[1]()
        if ctx is not None and getattr(ctx, "h", None):
            return ctx
        _KS_DEVICES.pop((id(ksk), params.digest()), None)
    from .device import DeviceContext
    ctx = DeviceContext(params)
    ctx.load_key_switch_key(ksk.A, ksk.b)
    ksk_ctxs = getattr(ksk, "__dict__", None)
    if ksk_ctxs is not None:  # the key owns its standalone context (frozen dataclass: bypass setattr)
        object.__setattr__(ksk, "_b200_ks_ctx", ctx)
    _register_ks_device(ksk, params, ctx)
    return ctx


def key_switch_batch(A: np.ndarray, b: np.ndarray, ksk: KeySwitchKey,
                     params: FheParams):
    """LWE under z (dim N) -> LWE under s (dim n) on the device (bootstrap.py:303-316)."""
    A = np.asarray(A, dtype=np.int64)
    if A.shape[-1] != ksk.N:
        raise ParameterError("ciphertext dimension does not match key-switch key")
    if ksk.base != params.ks_base or ksk.levels != params.ks_levels or ksk.N != params.N:
        raise ParameterError("key-switch key does not match params")
    return _key_device(ksk, params).key_switch_batch(A, np.asarray(b, dtype=np.int64))


def key_switch(ct: LweCiphertext, ksk: KeySwitchKey, params: FheParams) -> LweCiphertext:
    A, b = key_switch_batch(ct.a[None, :], np.asarray([ct.b]), ksk, params)
    return LweCiphertext(A[0], int(b[0]), params.q)


def bootstrap_batch(g: ProgramFunction, A: np.ndarray, b: np.ndarray, bsk):
    """LWE(m) -> LWE(g(m)) for a batch, on the B200 (bootstrap.py:324-341)."""
    params = bsk.params
    A = np.asarray(A, dtype=np.int64)
    b = np.asarray(b, dtype=np.int64)
    if A.ndim != 2 or A.shape[1] != params.n or b.shape != (A.shape[0],):
        raise ParameterError("ciphertext arrays do not match params")
    dev = _device_of(bsk)
    out = dev.pbs_batch(dev.lut(test_polynomial(g, params)), A, b)
    bsk.bootstrap_count += len(b)
    return out


def bootstrap(g: ProgramFunction, ct: LweCiphertext, bsk) -> LweCiphertext:
    A, b = bootstrap_batch(g, ct.a[None, :], np.asarray([ct.b]), bsk)
    return LweCiphertext(A[0], int(b[0]), bsk.params.q)
