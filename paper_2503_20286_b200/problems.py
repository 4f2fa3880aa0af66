"""Benchmark problems -- drop-in for ``temo.problems`` (problems.py:21-184) plus LSMOP1-9.

Evaluation runs on the GPU (``temo_evaluate``; fused into offspring generation
by ``temo_offspring`` for DTLZ and LSMOP1, a warp-per-row pass over the children
for LSMOP2-9).  DTLZ1-7 follow problems.py:69-136 op for op; results agree with
NumPy to the last few ulps (transcendentals differ), inside the north star's 1e-5
relative tolerance.  LSMOP1-9 are new (the reference has no LSMOP):
the standard definitions of Cheng et al. 2017 in the PlatEMO formulation --
linkage x^s_j <- (1 + j/D) x^s_j - 10 x_1 (LSMOP1-4) or (1 + cos(j/D pi/2)) x^s_j
- 10 x_1 (LSMOP5-9), chaotic subcomponent sizes (c <- 3.8 c (1 - c), nk = 5),
eta1 on odd / eta2 on even objectives (Sphere, Griewank, Schwefel 2.21, Rastrigin,
Rosenbrock, Ackley per problem), and the linear (1-4), concave (5-8) or
disconnected (9) front.  As in PlatEMO, the requested dimension only sizes the
subcomponents; the problem then has D = m - 1 + nk * sum(sublen) variables
(``make_problem("lsmop1", 3, 1000)`` has D = 992) and the linkage divides by
that D.
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .directions import largest_h_for, simplex_lattice

DTLZ = ("dtlz1", "dtlz2", "dtlz3", "dtlz4", "dtlz5", "dtlz6", "dtlz7")
LSMOP = tuple(f"lsmop{k}" for k in range(1, 10))
_NAMES = DTLZ + LSMOP
PROB_LSMOP1 = 101


class ProblemStruct(ctypes.Structure):
    """Mirror of ``temo_problem`` (include/temo_b200.h)."""

    _fields_ = [("id", ctypes.c_int32), ("m", ctypes.c_int32), ("d", ctypes.c_int64),
                ("nk", ctypes.c_int32), ("sublen", ctypes.c_int32 * 16),
                ("offset", ctypes.c_int32 * 17)]


def lsmop_groups(m: int, d: int, nk: int = 5):
    """Subcomponent lengths per objective and group offsets within x^s."""
    c = [3.8 * 0.1 * (1.0 - 0.1)]
    for _ in range(m - 1):
        c.append(3.8 * c[-1] * (1.0 - c[-1]))
    c = np.asarray(c)
    sublen = np.floor(c / c.sum() * (d - m + 1) / nk).astype(np.int64)
    offset = np.concatenate([[0], np.cumsum(sublen * nk)])
    return sublen, offset


def lsmop_dimension(m: int, d_request: int, nk: int = 5):
    """PlatEMO's D for a requested dimension: (D, sublen, offset); D = m - 1 + offset[m]."""
    sublen, offset = lsmop_groups(m, d_request, nk)
    return m - 1 + int(offset[m]), sublen, offset


def lsmop_groups_for(m: int, D: int, nk: int = 5):
    """(sublen, offset) of an LSMOP problem with D variables.

    Every requested dimension that yields D yields the same groups (each floor
    is monotone in the request), so D alone determines them."""
    for d0 in range(D, D + nk * m + 2):
        Dd, sublen, offset = lsmop_dimension(m, d0, nk)
        if Dd == D:
            return sublen, offset
        if Dd > D:
            break
    raise ValueError(f"{D} is not an LSMOP dimension for m={m} (use make_problem with the requested D)")


@dataclass(frozen=True)
class ProblemSpec:
    """A DTLZ/LSMOP instance: name, decision dimension d, objective count m (problems.py:21-50)."""

    name: str
    d: int
    m: int
    lower: np.ndarray = field(default=None)
    upper: np.ndarray = field(default=None)

    def __post_init__(self):
        if self.name not in _NAMES:
            raise ValueError(f"unknown problem {self.name!r}")
        if self.m < 2:
            raise ValueError("need at least 2 objectives")
        if self.d < self.m:
            raise ValueError("DTLZ needs d >= m")
        if self.name in LSMOP:
            sub, _ = lsmop_groups_for(self.m, self.d)
            if (sub < 1).any():
                raise ValueError("LSMOP needs d large enough for every subcomponent")
            dl = np.zeros(self.d)
            du = np.concatenate([np.ones(self.m - 1), np.full(self.d - self.m + 1, 10.0)])
        else:
            dl, du = np.zeros(self.d), np.ones(self.d)
        lower = dl if self.lower is None else np.asarray(self.lower, dtype=np.float64)
        upper = du if self.upper is None else np.asarray(self.upper, dtype=np.float64)
        if lower.shape != (self.d,) or upper.shape != (self.d,):
            raise ValueError("bounds must be length-d vectors")
        if not np.all(lower < upper):
            raise ValueError("lower bounds must be strictly below upper bounds")
        object.__setattr__(self, "lower", lower)
        object.__setattr__(self, "upper", upper)

    @property
    def k(self) -> int:
        return self.d - self.m + 1

    def struct(self) -> ProblemStruct:
        s = ProblemStruct()
        s.m, s.d = self.m, self.d
        if self.name in LSMOP:
            s.id = PROB_LSMOP1 + LSMOP.index(self.name)
            s.nk = 5
            sub, off = lsmop_groups_for(self.m, self.d, 5)
            for i in range(self.m):
                s.sublen[i] = int(sub[i])
            for i in range(self.m + 1):
                s.offset[i] = int(off[i])
        else:
            s.id = DTLZ.index(self.name) + 1
        return s


def default_dimension(name: str, m: int) -> int:
    """problems.py:53-59; LSMOP: D = 100 m (PlatEMO default)."""
    if name == "dtlz1":
        return m + 4
    if name == "dtlz7":
        return m + 19
    if name in LSMOP:
        return 100 * m
    return m + 9


def make_problem(name: str, m: int = 3, d: int | None = None) -> ProblemSpec:
    name = name.lower()
    if d is None:
        d = default_dimension(name, m)
    if name in LSMOP:  # d is PlatEMO's requested D; the instance has D = m - 1 + nk * sum(sublen)
        if d < m:
            raise ValueError("DTLZ needs d >= m")
        sub, _ = lsmop_groups(m, d)
        if (sub < 1).any():
            raise ValueError("LSMOP needs d large enough for every subcomponent")
        d = lsmop_dimension(m, d)[0]
    return ProblemSpec(name, d, m)


def evaluate_device(spec: ProblemSpec, Xd, out=None):
    """Enqueue evaluation of a CUDA (n, d) float64 tensor; returns (n, m) tensor."""
    t = _lib.torch()
    n = Xd.shape[0]
    F = out if out is not None else t.empty((n, spec.m), dtype=t.float64, device=Xd.device)
    ps = spec.struct()  # keep the struct alive across the call
    rc = _lib.lib().temo_evaluate(_lib.sptr(ps), _lib.ptr(Xd), n, _lib.ptr(F),
                                  _lib.stream_handle(Xd.device))
    _lib.check(rc, "evaluate")
    return F


def evaluate(spec: ProblemSpec, X):
    """Batch-evaluate n x d decision rows to n x m objectives (problems.py:105-136)."""
    t = _lib.torch()
    is_np = not isinstance(X, t.Tensor)
    A = np.asarray(X, dtype=np.float64) if is_np else X
    if A.ndim != 2 or A.shape[1] != spec.d:
        raise ValueError(f"expected n x {spec.d} input, got {tuple(A.shape)}")
    Xd, _ = _lib.as_device(A, t.float64)
    F = evaluate_device(spec, Xd)
    return F.cpu().numpy() if is_np else F


def true_front(spec: ProblemSpec, count: int) -> np.ndarray:
    """Analytic Pareto-front sample for IGD (problems.py:151-184; setup-time host data)."""
    if count < spec.m:
        raise ValueError("count must be at least m")
    m = spec.m
    if spec.name in ("dtlz1",):
        return 0.5 * simplex_lattice(m, largest_h_for(count, m))
    if spec.name in ("lsmop1", "lsmop2", "lsmop3", "lsmop4"):  # linear front
        return simplex_lattice(m, largest_h_for(count, m))
    if spec.name in ("lsmop5", "lsmop6", "lsmop7", "lsmop8"):  # concave front
        pts = simplex_lattice(m, largest_h_for(count, m))
        return pts / np.linalg.norm(pts, axis=1, keepdims=True)
    if spec.name == "lsmop9":  # disconnected: f_M = 2 (M - sum f_k / 2 (1 + sin 3 pi f_k)), non-dominated
        return _disconnected_front(m, count, 1.0)
    if spec.name in ("dtlz2", "dtlz3", "dtlz4"):
        pts = simplex_lattice(m, largest_h_for(count, m))
        return pts / np.linalg.norm(pts, axis=1, keepdims=True)
    if spec.name in ("dtlz5", "dtlz6"):
        theta = np.full((count, m - 1), math.pi / 4.0)
        theta[:, 0] = np.linspace(0.0, math.pi / 2.0, count)
        out = np.empty((count, m))
        for i in range(m):
            p = np.prod(np.cos(theta[:, : m - 1 - i]), axis=1)
            if i:
                p = p * np.sin(theta[:, m - 1 - i])
            out[:, i] = p
        return out
    raise ValueError(f"true_front not provided for {spec.name}")


def _disconnected_front(m: int, count: int, G: float) -> np.ndarray:
    """Non-dominated sample of the DTLZ7-type front f_M = (1 + G) (M - sum_k f_k / (1 + G) (1 + sin 3 pi f_k))
    over a grid of the first m - 1 objectives (LSMOP9: G = 1 at the optimum)."""
    per = max(2, int((max(count, 6000) + 0.5) ** (1.0 / max(m - 1, 1))))  # grid of <= ~6000 points
    axes = np.meshgrid(*([np.linspace(0.0, 1.0, per)] * (m - 1)), indexing="ij")
    pos = np.stack([a.reshape(-1) for a in axes], axis=1)
    h = m - np.sum(pos / (1.0 + G) * (1.0 + np.sin(3.0 * np.pi * pos)), axis=1)
    P = np.concatenate([pos, ((1.0 + G) * h)[:, None]], axis=1)
    keep = np.ones(len(P), dtype=bool)
    for a in range(0, len(P), 512):  # q dominates p: q <= p everywhere and q < p somewhere
        blk = P[a: a + 512, None, :]
        le = np.all(P[None, :, :] <= blk, axis=2)
        lt = np.any(P[None, :, :] < blk, axis=2)
        keep[a: a + 512] = ~np.any(le & lt, axis=1)
    F = P[keep]
    if len(F) > count:
        F = F[np.linspace(0, len(F) - 1, count).astype(np.int64)]
    return F
