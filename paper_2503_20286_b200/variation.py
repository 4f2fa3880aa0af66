"""Mating, SBX and polynomial mutation on the GPU -- drop-in for ``temo.variation`` (variation.py:17-120).

With a NumPy ``Generator`` over ``Philox`` (what ``RngStream`` builds) the
uniforms are produced on the device from the Generator's state and the host
Generator is advanced past them, so the stream stays identical to the
reference's.  Any other duck-typed RNG (``ForcedRng``, ``PlannedShuffleRng``
in the reference tests) is called on the host exactly like the reference and
its draws are uploaded.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _lib
from .rng import DeviceDraws, is_philox
from .rng import permutation as rng_permutation


class VariationStruct(ctypes.Structure):
    """Mirror of ``temo_variation`` (include/temo_b200.h)."""

    _fields_ = [("eta_c", ctypes.c_double), ("eta_m", ctypes.c_double), ("p_m", ctypes.c_double),
                ("gene_swap", ctypes.c_int32), ("reserved", ctypes.c_int32),
                ("lower", ctypes.c_void_p), ("upper", ctypes.c_void_p)]


@dataclass(frozen=True)
class VariationParams:
    """SBX / PM parameters and bounds (variation.py:17-45); gene_swap defaults True like the code."""

    eta_c: float = 20.0
    eta_m: float = 20.0
    p_m: float | None = None
    lower: np.ndarray = None
    upper: np.ndarray = None
    gene_swap: bool = True

    def __post_init__(self):
        if self.eta_c <= 0 or self.eta_m <= 0:
            raise ValueError("distribution indices must be positive")
        if self.p_m is not None and not 0.0 <= self.p_m <= 1.0:
            raise ValueError("p_m must lie in [0, 1]")
        lower = np.asarray(self.lower, dtype=np.float64)
        upper = np.asarray(self.upper, dtype=np.float64)
        if not np.all(lower < upper):
            raise ValueError("lower bounds must be strictly below upper bounds")
        object.__setattr__(self, "lower", lower)
        object.__setattr__(self, "upper", upper)

    def mutation_prob(self, d: int) -> float:
        return 1.0 / d if self.p_m is None else self.p_m

    def struct(self, d: int, dev=None) -> VariationStruct:
        """C struct with cached device copies of the bounds (broadcast to length d)."""
        t = _lib.torch()
        dv = _lib.device(dev)
        cache = self.__dict__.setdefault("_dev", {})
        key = (str(dv), d)
        if key not in cache:
            lo = np.broadcast_to(self.lower, (d,)).astype(np.float64)
            hi = np.broadcast_to(self.upper, (d,)).astype(np.float64)
            cache[key] = (t.from_numpy(np.ascontiguousarray(lo)).to(dv),
                          t.from_numpy(np.ascontiguousarray(hi)).to(dv))
        lo_d, hi_d = cache[key]
        s = VariationStruct()
        s.eta_c, s.eta_m, s.p_m = self.eta_c, self.eta_m, self.mutation_prob(d)
        s.gene_swap = 1 if self.gene_swap else 0
        s.lower, s.upper = lo_d.data_ptr(), hi_d.data_ptr()
        s._keep = (lo_d, hi_d)  # the struct owns its bound arrays (no dangling device pointers)
        return s


def pair_parents(rng, n: int):
    """Split a random permutation into two mating halves (variation.py:48-54)."""
    if n < 2:
        raise ValueError("need at least two individuals to pair")
    perm = rng_permutation(rng, n)
    half = n // 2
    return perm[:half], perm[half: 2 * half]


def _upload(rng, shape, dev):
    t = _lib.torch()
    return t.from_numpy(np.ascontiguousarray(rng.random(shape), dtype=np.float64)).to(dev)


def sbx(rng, X1, X2, params: VariationParams):
    """Simulated binary crossover; returns clipped [C1; C2] (variation.py:57-91)."""
    t = _lib.torch()
    is_np = not isinstance(X1, t.Tensor)
    A, _ = _lib.as_device(X1, t.float64)
    B, _ = _lib.as_device(X2, t.float64, A.device)
    if A.shape != B.shape:
        raise ValueError("parent blocks must share a shape")
    q, d = A.shape
    C = t.empty((2 * q, d), dtype=t.float64, device=A.device)
    var = params.struct(d, A.device)
    L = _lib.lib()
    if is_philox(rng):
        draws = DeviceDraws(rng)
        off = draws.take(q * d * (3 if params.gene_swap else 1))
        rc = L.temo_sbx(_lib.sptr(var), _lib.ptr(A), _lib.ptr(B), q, d, _lib.sptr(draws.state), off,
                        None, None, None, _lib.ptr(C), _lib.stream_handle(A.device))
        draws.commit()
    else:
        u_mu = _upload(rng, (q, d), A.device)
        u_sw = _upload(rng, (q, d), A.device) if params.gene_swap else None
        u_cr = _upload(rng, (q, d), A.device) if params.gene_swap else None
        rc = L.temo_sbx(_lib.sptr(var), _lib.ptr(A), _lib.ptr(B), q, d, None, 0, _lib.ptr(u_mu),
                        _lib.ptr(u_sw), _lib.ptr(u_cr), _lib.ptr(C), _lib.stream_handle(A.device))
    _lib.check(rc, "sbx")
    return C.cpu().numpy() if is_np else C


def polynomial_mutation(rng, X, params: VariationParams):
    """Bounded polynomial mutation with probability p_m per gene (variation.py:94-120)."""
    t = _lib.torch()
    is_np = not isinstance(X, t.Tensor)
    A, _ = _lib.as_device(X, t.float64)
    rows, d = A.shape
    Y = t.empty_like(A)
    var = params.struct(d, A.device)
    L = _lib.lib()
    if is_philox(rng):
        draws = DeviceDraws(rng)
        off = draws.take(2 * rows * d)
        rc = L.temo_pm(_lib.sptr(var), _lib.ptr(A), rows, d, _lib.sptr(draws.state), off, None, None,
                       _lib.ptr(Y), _lib.stream_handle(A.device))
        draws.commit()
    else:
        u_mu = _upload(rng, (rows, d), A.device)
        u_hit = _upload(rng, (rows, d), A.device)
        rc = L.temo_pm(_lib.sptr(var), _lib.ptr(A), rows, d, None, 0, _lib.ptr(u_mu), _lib.ptr(u_hit),
                       _lib.ptr(Y), _lib.stream_handle(A.device))
    _lib.check(rc, "polynomial_mutation")
    return Y.cpu().numpy() if is_np else Y


def uniform_device(rng, shape, dev=None):
    """``rng.random(shape)`` generated on the device (host Generator advanced)."""
    t = _lib.torch()
    count = int(np.prod(shape))
    out = t.empty(shape, dtype=t.float64, device=_lib.device(dev))
    draws = DeviceDraws(rng)
    off = draws.take(count)
    rc = _lib.lib().temo_uniform(_lib.sptr(draws.state), off, count, _lib.ptr(out),
                                 _lib.stream_handle(out.device))
    _lib.check(rc, "uniform")
    draws.commit()
    return out
