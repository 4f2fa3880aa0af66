"""Device-resident generation loop -- the caller of the hot path (``temo.harness``, harness.py:39-319).

``_Stepper`` keeps the reference protocol ``init(gen)`` / ``step(state, g, gen)
-> (state, seconds)`` (harness.py:164-248) and the reference RNG call order
(SURVEY App. B): permutations and integer draws happen on the host with the
run's NumPy Generator, every uniform block is produced on the device from the
same Philox stream, and the population never leaves HBM.

Decision variables live in ONE row pool of N = n + 2h rows (no survivor
copy): ``phys`` (device int64, N) maps the logical merged order -- parents
[0, n), offspring [n, N), the reference's [X; O] order (harness.py:221-222) --
to pool rows.  The offspring kernel reads parents through ``phys`` and writes
children into the pool rows ``phys[n:]``; after selection ``temo_pool_update``
rewrites ``phys`` (survivors first, freed rows after), so X[perm][keep]
(nsga3.py:218) is a 3.2 GB copy the generation never makes.  Objectives are
small and stay in logical order (ping-pong buffers).
"""

from __future__ import annotations

import ctypes
import dataclasses
import math
import time
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .directions import DirectionSet, das_dennis, largest_h_for, neighbors
from .nsga3 import Nsga3Selector
from .problems import ProblemSpec, make_problem
from .rng import DeviceDraws, RngStream
from .rng import permutation as rng_permutation
from .variation import VariationParams

ALGORITHMS = ("nsga3", "moead", "hype")


class ConfigError(ValueError):
    """Invalid or unsupported run configuration (harness.py:35-36)."""


@dataclass(frozen=True)
class RunConfig:
    """Everything needed to reproduce one experiment (harness.py:39-82 field names)."""

    algorithm: str = "nsga3"
    problem: str = "dtlz2"
    objectives: int = 3
    dim: int | None = None
    pop_size: int = 100
    generations: int = 100
    seed: int = 0
    repeats: int = 1
    eta_c: float = 20.0
    eta_m: float = 20.0
    pm: float | None = None
    theta: float = 5.0
    neighborhood: int | None = None
    divisions: int | None = None
    hv_samples: int | None = None
    hv_ref: str = "auto"
    time_selection_only: bool = False
    aggregation: str = "pbi"  # MOEA/D: "pbi" (reference) or "tch" (Tchebycheff, new)
    device: str | None = None

    def validate(self) -> None:
        if self.algorithm not in ALGORITHMS:
            raise ConfigError(f"unknown algorithm {self.algorithm!r}")
        if self.objectives < 2 or self.pop_size < 2 or self.repeats < 1:
            raise ConfigError("objectives >= 2, pop-size >= 2, repeats >= 1 required")
        if self.generations < 0:
            raise ConfigError("generations must be non-negative")
        if self.aggregation not in ("pbi", "tch"):
            raise ConfigError(f"unknown aggregation {self.aggregation!r}")


def _resolve(config: RunConfig):
    """Problem spec, direction set and effective population size (harness.py:147-161)."""
    spec = make_problem(config.problem, m=config.objectives, d=config.dim)
    if config.divisions is not None:
        if config.divisions < 1:
            raise ConfigError("divisions must be positive")
        H = config.divisions
    else:
        if config.pop_size < config.objectives:
            raise ConfigError("pop-size below objective count leaves no directions")
        H = largest_h_for(config.pop_size, config.objectives)
    R = das_dennis(config.objectives, H)
    n_eff = R.count if config.algorithm == "moead" else config.pop_size
    return spec, R, n_eff


@dataclass
class PopBuffers:
    """One merged population buffer: X (cap x d), F (cap x m)."""

    X: object
    F: object


@dataclass
class DeviceState:
    """Current population: logical rows [0, n); X rows live in the pool at ``phys``."""

    cur: PopBuffers
    nxt: PopBuffers
    n: int
    extra: dict = field(default_factory=dict)
    phys: object = None  # device int64 (N): logical merged row -> pool row (None: identity)

    def rows(self, lo: int, hi: int):
        """X of logical rows [lo, hi) (materialised from the pool)."""
        if self.phys is None:
            return self.cur.X[lo:hi]
        return self.cur.X.index_select(0, self.phys[lo:hi])

    @property
    def X(self):
        return self.rows(0, self.n)

    @property
    def F(self):
        return self.cur.F[: self.n]


class _Stepper:
    """Per-algorithm generation step on the device (harness.py:164-248)."""

    def __init__(self, config: RunConfig, spec: ProblemSpec, R: DirectionSet, n: int):
        t = _lib.torch()
        self.config, self.spec, self.R, self.n = config, spec, R, n
        self.dev = _lib.device(config.device)
        self.params = VariationParams(eta_c=config.eta_c, eta_m=config.eta_m, p_m=config.pm,
                                      lower=spec.lower, upper=spec.upper)
        self.var = self.params.struct(spec.d, self.dev)
        self.prob = spec.struct()
        self.h = n // 2
        self.N = n + 2 * self.h
        self.ring = _lib.HostRing()
        d, m = spec.d, spec.m
        pool = t.empty((self.N, d), dtype=t.float64, device=self.dev)  # the single X row pool
        mk = lambda: PopBuffers(pool, t.empty((self.N, m), dtype=t.float64, device=self.dev))  # noqa: E731
        self.bufs = (mk(), mk())
        self.phys = [t.arange(self.N, dtype=t.int64, device=self.dev),
                     t.empty(self.N, dtype=t.int64, device=self.dev)]
        self.pool_ws = t.empty(max(int(_lib.lib().temo_pool_update_ws_bytes(self.N)), 256),
                               dtype=t.uint8, device=self.dev)
        self.i12 = t.empty(2 * self.h, dtype=t.int64, device=self.dev)
        # two-phase offspring workspace (h x d SBX betas + per-quad flags), owned by the stepper
        self.off_ws = t.empty(max(int(_lib.lib().temo_offspring_ws_bytes(self.h, d)), 256),
                              dtype=t.uint8, device=self.dev)
        self.perm = t.empty(self.N, dtype=t.int64, device=self.dev)
        alg = config.algorithm
        if alg == "nsga3":
            dist_rank = None
            import torch.distributed as dist

            if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
                from .parallel import DistRank

                dist_rank = DistRank(self.N, m, dist.get_rank(), dist.get_world_size(), self.dev)
            self.selector = Nsga3Selector(self.N, m, R, n, self.dev, dist_rank=dist_rank)
        elif alg == "hype":
            from .hype import HypeSelector

            ref = None if config.hv_ref == "auto" else np.asarray(
                [float(v) for v in str(config.hv_ref).split(",")])
            s = config.hv_samples or 10 * n
            self.selector = HypeSelector(self.N, m, n, s, ref, self.dev)
        elif alg == "moead":
            from .moead import MoeadEngine, default_neighborhood

            T = config.neighborhood or default_neighborhood(n)
            if not 2 <= T <= n:
                raise ConfigError(f"neighborhood {T} out of range [2, {n}]")
            self.table = neighbors(R, T)
            self.engine = MoeadEngine(spec, R, self.table, self.params, config.theta,
                                      config.aggregation, self.dev)

    # -- init (harness.py:187-194)
    def init(self, gen) -> DeviceState:
        draws = DeviceDraws(gen)
        off = draws.take(self.n * self.spec.d)
        cur = self.bufs[0]
        lo, hi = self.var.lower, self.var.upper
        rc = _lib.lib().temo_init_population(_lib.sptr(draws.state), off, self.n, self.spec.d,
                                             ctypes.c_void_p(lo), ctypes.c_void_p(hi), _lib.ptr(cur.X),
                                             _lib.stream_handle(self.dev))
        _lib.check(rc, "init")
        draws.commit()
        from .problems import evaluate_device

        evaluate_device(self.spec, cur.X[: self.n], out=cur.F[: self.n])
        st = DeviceState(cur, self.bufs[1], self.n)
        if self.config.algorithm != "moead":
            st.phys = self.phys[0]  # identity at init: parents in pool rows [0, n)
            st.extra["pool_identity"] = True
        if self.config.algorithm == "moead":
            st.extra["moead"] = self.engine.init_state(cur.X[: self.n], cur.F[: self.n])
        return st

    # -- offspring of NSGA-III / HypE (harness.py:201-204, 218-222) into rows [n, N)
    def _offspring(self, st: DeviceState, gen):
        i1, i2 = (lambda p, h: (p[:h], p[h: 2 * h]))(rng_permutation(gen, self.n), self.h)
        self.ring.upload(np.concatenate([i1, i2]).astype(np.int64), self.i12)
        draws = DeviceDraws(gen)
        hd = self.h * self.spec.d
        off = draws.take((3 if self.params.gene_swap else 1) * hd + 4 * hd)
        cur = st.cur
        pooled = ((self.h * self.spec.d) % 4 == 0 and self.spec.d <= 3000  # two-phase path (row maps)
                  and not getattr(self, "force_unpooled", False))
        if pooled:
            src, dst, obase = _lib.ptr(st.phys), _lib.ptr(st.phys[self.n:]), _lib.ptr(cur.X)
        else:  # fused fallback: children into logical rows; make the pool the identity first
            self._pool_identity(st)
            src, dst, obase = None, None, _lib.ptr(cur.X[self.n:])
        rc = _lib.lib().temo_offspring_ws(_lib.sptr(self.prob), _lib.sptr(self.var), _lib.ptr(cur.X),
                                          _lib.ptr(self.i12), _lib.ptr(self.i12[self.h:]), self.h,
                                          _lib.sptr(draws.state), off, obase,
                                          _lib.ptr(cur.F[self.n:]), src, dst,
                                          _lib.ptr(self.off_ws), self.off_ws.numel(),
                                          _lib.stream_handle(self.dev))
        _lib.check(rc, "offspring")
        draws.commit()

    def _pool_identity(self, st: DeviceState):
        """Materialise the parents into pool rows [0, n) (fused-offspring fallback only)."""
        if st.phys is not None and st.extra.get("pool_identity") is not True:
            X = st.rows(0, self.n)
            st.cur.X[: self.n].copy_(X)
            st.phys.copy_(_lib.torch().arange(self.N, dtype=_lib.torch().int64, device=self.dev))
        st.extra["pool_identity"] = True

    def _pool_update(self, st: DeviceState, perm, keep):
        """phys' = survivors' pool rows, then the freed rows (temo_pool_update)."""
        out = self.phys[1] if st.phys.data_ptr() == self.phys[0].data_ptr() else self.phys[0]
        rc = _lib.lib().temo_pool_update(_lib.ptr(st.phys), _lib.ptr(perm), _lib.ptr(keep), self.N, self.n,
                                         _lib.ptr(out), _lib.ptr(self.selector.status),
                                         _lib.ptr(self.pool_ws), self.pool_ws.numel(),
                                         _lib.stream_handle(self.dev))
        _lib.check(rc, "pool_update")
        st.phys = out
        st.extra["pool_identity"] = False

    def offspring_rows(self, st: DeviceState):
        """X of the current offspring (logical rows [n, N))."""
        return st.rows(self.n, self.N)

    def step(self, st: DeviceState, g: int, gen):
        alg = self.config.algorithm
        t0 = time.perf_counter()
        if alg == "moead":
            st.extra["moead"] = self.engine.step(st.extra["moead"], gen)
            return st, time.perf_counter() - t0
        self._offspring(st, gen)
        ts = time.perf_counter()
        cur, nxt = st.cur, st.nxt
        n = self.n
        if alg == "nsga3":
            self.ring.upload(rng_permutation(gen, self.N), self.perm)
            keep = self.selector.select(cur.F, self.perm)
            self._pool_update(st, self.perm, keep)  # survivors' X rows stay where they are
            _lib.gather_rows(self.selector.Fs, keep, nxt.F[:n])
        else:  # hype (no shuffle; hype.py:135-163)
            keep = self.selector.select(cur.F, gen)
            self._pool_update(st, None, keep)
            _lib.gather_rows(cur.F, keep, nxt.F[:n])
        st.cur, st.nxt = nxt, cur
        return st, time.perf_counter() - ts

    def check(self):
        """Raise the reference's exception if a selection failed (device status word)."""
        if self.config.algorithm != "moead":
            self.selector.check()

    def objectives(self, st: DeviceState):
        """F of the current population (device, logical order) -- no X materialisation."""
        if self.config.algorithm == "moead":
            return st.extra["moead"].F1
        return st.F

    def population(self, st: DeviceState):
        if self.config.algorithm == "moead":
            ms = st.extra["moead"]
            return ms.X, ms.F1
        return st.X, st.F


@dataclass
class GenRow:
    generation: int
    time_s: float
    ideal: list


@dataclass
class RunRecord:
    config: dict
    rows: list
    mean_gen_time_s: float
    final_F: np.ndarray


def run(config: RunConfig, sync_every_step: bool = True) -> RunRecord:
    """Execute one repeat of a configured run (harness.py:270-319, timing per generation).

    Each generation is timed from launch to the host read of the new ideal
    point (the reference records ``F.min(axis=0)`` per generation)."""
    config.validate()
    spec, R, n_eff = _resolve(config)
    stepper = _Stepper(config, spec, R, n_eff)
    gen = RngStream(config.seed).split(0).generator()
    st = stepper.init(gen)
    rows = []
    for g in range(1, config.generations + 1):
        t0 = time.perf_counter()
        st, sel_s = stepper.step(st, g, gen)
        F = stepper.objectives(st)
        ideal = F.min(dim=0).values.cpu().numpy().tolist() if sync_every_step else []
        total = time.perf_counter() - t0
        if sync_every_step:
            stepper.check()
        rows.append(GenRow(g, sel_s if config.time_selection_only else total, ideal))
    F = stepper.objectives(st)
    Fh = F.cpu().numpy()
    stepper.check()
    mean = float(np.mean([r.time_s for r in rows])) if rows else math.nan
    return RunRecord(dataclasses.asdict(config), rows, mean, Fh)
