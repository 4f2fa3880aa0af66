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
import json
import math
import platform
import queue
import threading
import time
from dataclasses import dataclass, field
from pathlib import Path

import numpy as np

from . import _lib
from .directions import DirectionSet, das_dennis, largest_h_for, neighbors
from .indicators import hv_indicator, igd
from .nsga3 import Nsga3Selector
from .problems import ProblemSpec, make_problem, true_front
from .rng import DeviceDraws, RngStream
from .rng import permutation as rng_permutation
from .variation import VariationParams

ALGORITHMS = ("nsga3", "moead", "hype", "rvea")
HOST_ONLY = ("nsga3-seq", "moead-seq")  # the reference's sequential baselines (baselines.py)
CSV_COLUMNS = ("generation", "time_s", "igd", "hv")


class ConfigError(ValueError):
    """Invalid or unsupported run configuration (harness.py:35-36)."""


@dataclass(frozen=True)
class RunConfig:
    """Everything needed to reproduce one experiment (harness.py:39-82: same fields, defaults and
    validation) plus ``aggregation`` (MOEA/D "pbi" | "tch") and ``device``."""

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
    alpha: float = 2.0
    hv_samples: int | None = None
    hv_ref: str = "auto"
    indicators: tuple = ("igd", "hv")
    indicator_every: int = 1
    ref_front_size: int = 1000
    time_selection_only: bool = False
    out: str | None = None
    aggregation: str = "pbi"  # MOEA/D: "pbi" (reference) or "tch" (Tchebycheff, new)
    device: str | None = None

    def validate(self) -> None:
        if self.algorithm not in ALGORITHMS:
            if self.algorithm in HOST_ONLY:
                raise ConfigError(f"{self.algorithm!r} is the reference's sequential CPU baseline, "
                                  "not part of the GPU hot path")
            raise ConfigError(f"unknown algorithm {self.algorithm!r}")
        if self.objectives < 2 or self.pop_size < 2 or self.repeats < 1:
            raise ConfigError("objectives >= 2, pop-size >= 2, repeats >= 1 required")
        if self.generations < 0 or self.indicator_every < 0:
            raise ConfigError("generations and indicator-every must be non-negative")
        if self.ref_front_size < self.objectives:
            raise ConfigError("ref-front-size must be at least the objective count")
        for name in self.indicators:
            if name not in ("igd", "hv", "eu"):
                raise ConfigError(f"unknown indicator {name!r}")
        if self.hv_ref != "auto":
            try:
                _parse_ref_vector(self.hv_ref, self.objectives)
            except ValueError as exc:
                raise ConfigError(str(exc)) from None
        if self.aggregation not in ("pbi", "tch"):
            raise ConfigError(f"unknown aggregation {self.aggregation!r}")


def _parse_ref_vector(text: str, m: int) -> np.ndarray:
    """harness.py:85-89."""
    parts = [float(v) for v in str(text).split(",")]
    if len(parts) != m:
        raise ValueError(f"hv-ref needs {m} comma-separated values")
    return np.asarray(parts)


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
    n_eff = R.count if config.algorithm in ("moead", "rvea") else config.pop_size
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


@dataclass
class HostInputs:
    """One generation's host-drawn inputs: the parent pairing i1 ++ i2 (2h int64), the Philox
    state + offset of the offspring's device uniforms, and NSGA-III's shuffle permutation."""

    i12: object
    state: object
    off: int
    shuffle: object = None


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
        # TEMO_OVERLAP_RAND=1|2 (default 1): run the next generation's offspring randomness on a
        # low-priority side stream (needs its host inputs drawn ahead: pre-drawn lists or the host
        # pipeline), overlapping this generation's apply + selection (1) or apply only (2).  The
        # generation itself then runs on a high-priority stream (joined to the caller's stream at
        # both ends) and the randomness kernel is split into short (pair, 128-gene) units, so the
        # block scheduler hands SMs back to the latency-bound selection kernels within one unit:
        # 4.24 vs 5.0 ms per generation at pop 200k (profiles/r02_overlap_ab.txt).  Without the
        # priority stream and short units the overlap was slower (7.4-11 ms): long persistent
        # randomness CTAs took the SMs from the K0 sorts and the cooperative peel.
        import os

        self.overlap = int(os.environ.get("TEMO_OVERLAP_RAND", "1"))
        # launch the next generation's randomness after (1) or before (0) this generation's apply
        self._rand_after_apply = os.environ.get("TEMO_RAND_AFTER_APPLY", "0") == "1"
        # ... and only once this generation's apply has finished (overlap the selection only)
        self._rand_wait_apply = os.environ.get("TEMO_RAND_WAIT_APPLY", "0") == "1"
        if self._rand_wait_apply:
            self._rand_after_apply = True
        self._gen_k, self._rand_ahead, self._apply_done, self._side, self._hp = 0, None, None, None, None
        alg = config.algorithm
        # multi-GPU: one process per GPU, every rank runs the same host RNG stream;
        # offspring rows and HypE sample columns are sharded, the bitmap ND sort (m >= 4) too
        import torch.distributed as dist

        self.shard = None
        if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1 and alg in ("nsga3", "hype"):
            from .parallel import RowExchange

            self.shard = (dist.get_rank(), dist.get_world_size())
            self.xchg = RowExchange()
        if alg == "nsga3":
            dist_rank = None
            if self.shard is not None and m >= 4:  # m <= 3: the staircase sort runs on every rank
                from .parallel import DistRank

                dist_rank = DistRank(self.N, m, self.shard[0], self.shard[1], self.dev)
            self.selector = Nsga3Selector(self.N, m, R, n, self.dev, dist_rank=dist_rank)
        elif alg == "hype":
            from .hype import HypeSelector
            from .parallel import ColumnExchange

            ref = None if config.hv_ref == "auto" else np.asarray(
                [float(v) for v in str(config.hv_ref).split(",")])
            s = config.hv_samples or 10 * n
            shard = None if self.shard is None else (self.shard[0], self.shard[1], ColumnExchange())
            self.selector = HypeSelector(self.N, m, n, s, ref, self.dev, shard=shard)
        elif alg == "rvea":
            from .rvea import RveaSelector

            self.selector = RveaSelector(self.N, m, R, config.alpha, self.dev)
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

    # -- offspring of NSGA-III / HypE / RVEA (harness.py:201-204, 218-222) into rows [n, N)
    def draw_host_inputs(self, gen, n: int | None = None, shuffle: bool = True) -> HostInputs:
        """The host Generator's part of one NSGA-III / HypE / RVEA generation, drawn in the
        reference's order (harness.py:201-204 pairing permutation, the offspring's uniforms
        reserved for the device, then the NSGA-III shuffle permutation nsga3.py:190)."""
        n = self.n if n is None else n
        h = n // 2
        p = rng_permutation(gen, n)
        draws = DeviceDraws(gen)
        hd = h * self.spec.d
        off = draws.take((3 if self.params.gene_swap else 1) * hd + 4 * hd)
        state = draws.state
        draws.commit()
        perm = rng_permutation(gen, n + 2 * h) if shuffle and self.config.algorithm == "nsga3" else None
        return HostInputs(p[: 2 * h].astype(np.int64), state, off, perm)

    def _side_stream(self):
        if self._side is None:
            self._side = _lib.torch().cuda.Stream(device=self.dev)
        return self._side

    def start_host_pipeline(self, gen, steps: int, depth: int = 3) -> None:
        """NSGA-III: draw the host inputs of the next ``steps`` generations on a worker thread
        (in the reference's order; the permutations run in native code without the GIL), so
        the host's sequential shuffles overlap the GPU's generations.  Opt-in: at pop 200k the
        worker's NumPy work contends with the launching thread for the GIL and the e2e loop
        measured 143-153 gen/s with it vs 163 without.  ``step`` consumes them
        in order; the Generator must not be used elsewhere until they are consumed (after
        ``steps`` generations it is in exactly the state the sequential loop leaves)."""
        if self.config.algorithm != "nsga3" or steps <= 0:
            return
        self.stop_host_pipeline()
        q: queue.Queue = queue.Queue(maxsize=depth)
        stop = threading.Event()

        def work():
            for _ in range(steps):
                if stop.is_set():
                    return
                q.put(self.draw_host_inputs(gen))

        th = threading.Thread(target=work, daemon=True)
        th.start()
        self._pipe = [q, th, stop, steps]

    def stop_host_pipeline(self) -> None:
        self._look = None
        pipe = getattr(self, "_pipe", None)
        if pipe is None:
            return
        q, th, stop, _ = pipe
        stop.set()
        while th.is_alive():  # unblock a worker waiting on a full queue
            try:
                q.get(timeout=0.01)
            except queue.Empty:
                pass
        self._pipe = None

    def _pipe_get(self):
        pipe = self._pipe
        hi = pipe[0].get()
        pipe[3] -= 1
        if pipe[3] == 0:
            pipe[1].join()
            self._pipe = None
        return hi

    def _next_piped(self):
        """(this generation's pipelined host inputs uploaded through the pinned ring, the next
        generation's host inputs or None); (None, None) without a pipeline."""
        look = getattr(self, "_look", None)
        if getattr(self, "_pipe", None) is None and look is None:
            return None, None
        hi = look if look is not None else self._pipe_get()
        self._look = self._pipe_get() if getattr(self, "_pipe", None) is not None else None
        h = self.n // 2
        self.ring.upload(hi.i12, self.i12[: 2 * h])
        self.ring.upload(hi.shuffle, self.perm)
        return HostInputs(self.i12, hi.state, hi.off, self.perm), self._look

    def upload_host_inputs(self, inputs: list) -> list:
        """Device-resident copies of pre-drawn host inputs (bench: inputs in HBM before timing)."""
        t = _lib.torch()
        out = []
        for hi in inputs:
            i12 = t.from_numpy(hi.i12).to(self.dev)
            sh = None if hi.shuffle is None else t.from_numpy(hi.shuffle.astype(np.int64)).to(self.dev)
            out.append(HostInputs(i12, hi.state, hi.off, sh))
        return out

    def _rand_ws(self, k: int):
        """Offspring randomness workspace of generation k (two, alternating, when the next
        generation's randomness runs ahead on the side stream)."""
        t = _lib.torch()
        if k % 2 == 0:
            return self.off_ws
        if getattr(self, "off_ws_b", None) is None:
            self.off_ws_b = t.empty_like(self.off_ws)
        return self.off_ws_b

    def _launch_rand(self, hi: HostInputs, h: int, q0: int, q1: int, k: int, stream) -> None:
        ws = self._rand_ws(k)
        rc = _lib.lib().temo_offspring_rand_ws(_lib.sptr(self.var), self.spec.d, h, q0, q1, _lib.sptr(hi.state),
                                               hi.off, _lib.ptr(ws), ws.numel(), stream)
        _lib.check(rc, "offspring_rand")

    def _offspring(self, st: DeviceState, gen, pre: HostInputs | None = None, pre_next: HostInputs | None = None):
        n = st.n  # RVEA's population is the number of non-empty partitions (<= self.n)
        if n < 2:
            return self._mutate_in_place(st, gen)
        h = n // 2
        if pre is None:
            pre = self.draw_host_inputs(gen, n, shuffle=False)
            self.ring.upload(pre.i12, self.i12[: 2 * h])
            i12 = self.i12
        else:
            i12 = pre.i12
        off = pre.off
        cur = st.cur
        pooled = ((h * self.spec.d) % 4 == 0 and self.spec.d <= 3000  # two-phase path (row maps)
                  and not getattr(self, "force_unpooled", False))
        if pooled:
            src, dst, obase = _lib.ptr(st.phys), _lib.ptr(st.phys[n:]), _lib.ptr(cur.X)
        else:  # fused fallback: children into logical rows; make the pool the identity first
            self._pool_identity(st)
            src, dst, obase = None, None, _lib.ptr(cur.X[n:])
        q0, q1 = 0, h
        if self.shard is not None and pooled:
            from .parallel import shard_range

            q0, q1 = shard_range(h, *self.shard)
        t = _lib.torch()
        L = _lib.lib()
        if pooled and n == self.n and L.temo_offspring_two_phase(h, self.spec.d):
            # randomness of generation k (launched ahead on the side stream, or now), then this
            # generation's apply; the next generation's randomness (inputs drawn ahead) goes to
            # the side stream at once -- it needs no parent data, so it overlaps the apply and
            # the selection (SM time the latency-bound selection leaves idle)
            k = self._gen_k
            main = t.cuda.current_stream(self.dev)
            ahead = self._rand_ahead
            if ahead is not None and ahead[0] == k and ahead[2].state is pre.state and ahead[2].off == pre.off:
                main.wait_event(ahead[1])
            else:
                self._launch_rand(pre, h, q0, q1, k, _lib.stream_handle(self.dev))
            self._rand_ahead = None

            def ahead():
                side = self._side_stream()
                if self._apply_done is not None:  # the workspace of k + 1 was last read by apply k - 1
                    side.wait_event(self._apply_done)
                self._launch_rand(pre_next, h, q0, q1, k + 1, side.cuda_stream)
                ev = t.cuda.Event()
                ev.record(side)
                self._rand_ahead = (k + 1, ev, pre_next)

            late = self._rand_after_apply
            ov = self._overlap_on()
            if pre_next is not None and ov and not late:
                ahead()
            ws = self._rand_ws(k)
            rc = L.temo_offspring_apply_ws(_lib.sptr(self.prob), _lib.sptr(self.var), _lib.ptr(cur.X),
                                           _lib.ptr(i12), _lib.ptr(i12[h:]), h, q0, q1, _lib.sptr(pre.state), off,
                                           obase, _lib.ptr(cur.F[n:]), src, dst, _lib.ptr(ws), ws.numel(),
                                           _lib.stream_handle(self.dev))
            _lib.check(rc, "offspring")
            if pre_next is not None and ov and late:
                if self._rand_wait_apply:  # overlap the selection only: start after this apply
                    ev_a = t.cuda.Event()
                    ev_a.record(main)
                    self._side_stream().wait_event(ev_a)
                ahead()
            if ov and self.overlap == 2 and self._rand_ahead is not None:  # overlap the apply only
                main.wait_event(self._rand_ahead[1])
            self._apply_done = t.cuda.Event()
            self._apply_done.record(main)
            self._gen_k = k + 1
        else:
            rc = L.temo_offspring_ws_range(_lib.sptr(self.prob), _lib.sptr(self.var), _lib.ptr(cur.X),
                                           _lib.ptr(i12), _lib.ptr(i12[h:]), h, q0, q1,
                                           _lib.sptr(pre.state), off, obase,
                                           _lib.ptr(cur.F[n:]), src, dst,
                                           _lib.ptr(self.off_ws), self.off_ws.numel(),
                                           _lib.stream_handle(self.dev))
            _lib.check(rc, "offspring")
        st.extra["N_cur"] = n + 2 * h
        if (q0, q1) != (0, h):
            self._exchange_children(st, n, h)

    def _exchange_children(self, st: DeviceState, n: int, h: int):
        """Every rank's children (X rows and objectives of its pair range) to every rank: one
        all-gather of [X | F] rows (NCCL over NVLink), scattered into the replicated pool."""
        from .parallel import shard_range

        t = _lib.torch()
        G = self.shard[1]
        cur = st.cur
        ranges = [shard_range(h, g, G) for g in range(G)]
        lo, hi = ranges[self.shard[0]]
        rows = t.cat([st.phys[n + lo: n + hi], st.phys[n + h + lo: n + h + hi]])
        logical = t.cat([t.arange(n + lo, n + hi, device=self.dev), t.arange(n + h + lo, n + h + hi, device=self.dev)])
        local = t.cat([cur.X.index_select(0, rows), cur.F.index_select(0, logical)], dim=1)
        full = self.xchg(local, [2 * (b - a) for a, b in ranges])
        all_rows = t.cat([t.cat([st.phys[n + a: n + b], st.phys[n + h + a: n + h + b]]) for a, b in ranges])
        all_logical = t.cat([t.cat([t.arange(n + a, n + b, device=self.dev), t.arange(n + h + a, n + h + b, device=self.dev)])
                             for a, b in ranges])
        d = self.spec.d
        cur.X.index_copy_(0, all_rows, full[:, :d].contiguous())
        cur.F.index_copy_(0, all_logical, full[:, d:].contiguous())

    def _mutate_in_place(self, st: DeviceState, gen):
        """A shrunken population of one row: O = polynomial_mutation(X) (harness.py:223-226)."""
        from .problems import evaluate_device

        n, d = st.n, self.spec.d
        self._pool_identity(st)
        draws = DeviceDraws(gen)
        off = draws.take(2 * n * d)  # mu then hit (variation.py:107-108)
        X = st.cur.X
        rc = _lib.lib().temo_pm(_lib.sptr(self.var), _lib.ptr(X[:n]), n, d, _lib.sptr(draws.state), off,
                                None, None, _lib.ptr(X[n: 2 * n]), _lib.stream_handle(self.dev))
        _lib.check(rc, "polynomial_mutation")
        draws.commit()
        evaluate_device(self.spec, X[n: 2 * n], out=st.cur.F[n: 2 * n])
        st.extra["N_cur"] = 2 * n

    def _pool_identity(self, st: DeviceState):
        """Materialise the parents into pool rows [0, n) (fused-offspring fallback only)."""
        if st.phys is not None and st.extra.get("pool_identity") is not True:
            X = st.rows(0, st.n)
            st.cur.X[: st.n].copy_(X)
            st.phys.copy_(_lib.torch().arange(self.N, dtype=_lib.torch().int64, device=self.dev))
        st.extra["pool_identity"] = True

    def _pool_update(self, st: DeviceState, perm, keep, n_new: int | None = None):
        """phys' = survivors' pool rows, then the freed rows (temo_pool_update)."""
        n_new = self.n if n_new is None else n_new
        out = self.phys[1] if st.phys.data_ptr() == self.phys[0].data_ptr() else self.phys[0]
        rc = _lib.lib().temo_pool_update(_lib.ptr(st.phys), _lib.ptr(perm), _lib.ptr(keep), self.N, n_new,
                                         _lib.ptr(out), _lib.ptr(self.selector.status),
                                         _lib.ptr(self.pool_ws), self.pool_ws.numel(),
                                         _lib.stream_handle(self.dev))
        _lib.check(rc, "pool_update")
        st.phys = out
        st.extra["pool_identity"] = False

    def offspring_rows(self, st: DeviceState):
        """X of the current offspring (logical rows [n, N))."""
        return st.rows(st.n, st.extra.get("N_cur", self.N))

    def step(self, st: DeviceState, g: int, gen, timed: bool = True, pre: HostInputs | None = None,
             pre_next: HostInputs | None = None):
        """One generation (see ``_step``).  With the randomness overlap on (NSGA-III), the
        generation's kernels run on a high-priority stream that waits for the caller's current
        stream on entry and is waited for on exit, so stream order for the caller is unchanged."""
        if not self._overlap_on():
            return self._step(st, g, gen, timed, pre, pre_next)
        t = _lib.torch()
        if self._hp is None:
            self._hp = t.cuda.Stream(device=self.dev, priority=-1)
        caller = t.cuda.current_stream(self.dev)
        self._hp.wait_stream(caller)
        with t.cuda.stream(self._hp):
            out = self._step(st, g, gen, timed, pre, pre_next)
        caller.wait_stream(self._hp)
        return out

    def _sel_graph_on(self) -> bool:
        """Small NSGA-III populations are host-launch bound (~50 launches per selection): the
        selection (shuffle gather, ND sort, normalize/associate/niche, pool update, survivor
        objectives) is replayed as one CUDA graph per buffer parity.  TEMO_SEL_GRAPH=0: off."""
        import os

        if getattr(self, "_sel_graph_env", None) is None:
            self._sel_graph_env = os.environ.get("TEMO_SEL_GRAPH", "1") != "0"
        return (self._sel_graph_env and self.config.algorithm == "nsga3" and self.shard is None
                and self.N <= 16384 and getattr(self.selector, "dist_rank", None) is None)

    def _select_graph(self, st: DeviceState, perm):
        """The NSGA-III selection of this generation as a graph replay.  The graph is keyed by
        the buffers it touches (current/next objective buffers and row maps alternate with
        period 2); the shuffle goes to the fixed ``self.perm`` first.  The first use of a key
        runs eagerly (workspaces settle), the second captures."""
        t = _lib.torch()
        if perm.data_ptr() != self.perm.data_ptr():
            self.perm.copy_(perm)
        cur, nxt, n = st.cur, st.nxt, self.n
        out = self.phys[1] if st.phys.data_ptr() == self.phys[0].data_ptr() else self.phys[0]
        key = (cur.F.data_ptr(), nxt.F.data_ptr(), st.phys.data_ptr())
        graphs = self.__dict__.setdefault("_sel_graphs", {})
        seen = self.__dict__.setdefault("_sel_seen", set())

        def body():
            keep = self.selector.select(cur.F, self.perm)
            self._pool_update(st, self.perm, keep)
            _lib.gather_rows(self.selector.Fs, keep, nxt.F[:n])

        g = graphs.get(key)
        if g is None and key in seen:
            g = t.cuda.CUDAGraph()
            phys_in = st.phys
            try:
                with t.cuda.graph(g, capture_error_mode="thread_local"):
                    body()
            except Exception:  # capture not possible here: eager from now on (nothing ran)
                self._sel_graph_env = False
                g = None
                t.cuda.synchronize(self.dev)
            st.phys = phys_in  # capture does not run the work: replay below (or eager)
            if g is not None:
                graphs[key] = g
        if g is None:
            seen.add(key)
            body()
            return
        g.replay()
        st.phys = out
        st.extra["pool_identity"] = False

    def _overlap_on(self) -> bool:
        """The randomness overlap pays off only when the randomness is large: at small populations
        the extra stream hand-offs cost more host time than they hide (pop 100: 1.6 vs 1.7 kgen/s)."""
        return bool(self.overlap) and self.config.algorithm == "nsga3" and self.n * self.spec.d >= (1 << 20)

    def _step(self, st: DeviceState, g: int, gen, timed: bool = True, pre: HostInputs | None = None,
              pre_next: HostInputs | None = None):
        """One generation (harness.py:206-248); returns (state, seconds).

        ``seconds`` is the device time of the whole step -- or of the selection alone with
        ``time_selection_only`` -- from CUDA events on the launching stream (the call waits for
        the step).  ``timed=False`` returns at once with ``seconds = None`` (launch-ahead loops).
        ``pre``: this generation's host inputs drawn ahead by ``draw_host_inputs`` and made
        device-resident by ``upload_host_inputs`` (NSGA-III; the Generator must already be past
        them); ``pre_next``: the next generation's (its offspring randomness is then launched on
        the side stream during this step)."""
        t = _lib.torch()
        alg = self.config.algorithm
        ev = [t.cuda.Event(enable_timing=True) for _ in range(3)] if timed else None
        if timed:
            ev[0].record()
        if alg == "moead":
            st.extra["moead"] = self.engine.step(st.extra["moead"], gen)
            if timed:
                ev[1].record()
                ev[2].record()
        else:
            if pre is not None and alg != "nsga3":
                raise ValueError("pre-drawn host inputs are supported for NSGA-III only")
            if pre is None and alg == "nsga3":
                pre, pre_next = self._next_piped()
            if pre is None:
                self._offspring(st, gen)
            else:
                self._offspring(st, gen, pre, pre_next)
            if timed:
                ev[1].record()
            cur, nxt = st.cur, st.nxt
            n = self.n
            if alg == "nsga3":
                if pre is None:  # nsga3.py:190 shuffle, drawn after the offspring's uniforms
                    perm = self.ring.upload(rng_permutation(gen, self.N), self.perm)
                else:
                    perm = pre.shuffle
                if self._sel_graph_on():
                    self._select_graph(st, perm)
                else:
                    keep = self.selector.select(cur.F, perm)
                    self._pool_update(st, perm, keep)  # survivors' X rows stay where they are
                    _lib.gather_rows(self.selector.Fs, keep, nxt.F[:n])
            elif alg == "hype":  # no shuffle (hype.py:135-163)
                # launch-ahead loops (timed=False) defer the selection's RNG decision: the next
                # generation's host draws were made from the speculatively advanced Generator;
                # if the speculation was wrong, redo this generation's offspring from the
                # restored state (children rows are rewritten; parents are untouched)
                if self.selector.pending() and not self.selector.resolve():
                    self._offspring(st, gen)
                    cur = st.cur
                keep = self.selector.select(cur.F, gen, defer=not timed)
                self._pool_update(st, None, keep)
                _lib.gather_rows(cur.F, keep, nxt.F[:n])
            else:  # rvea: apd_select over [parents; offspring] (rvea.py:33-68, harness.py:240-244)
                keep = self.selector.select(cur.F, g, max(self.config.generations, 1), st.extra["N_cur"])
                k = int(keep.shape[0])
                self._pool_update(st, None, keep, k)
                _lib.gather_rows(cur.F, keep, nxt.F[:k])
                st.n = k
            st.cur, st.nxt = nxt, cur
            if timed:
                ev[2].record()
        if not timed:
            return st, None
        ev[2].synchronize()
        first = 1 if self.config.time_selection_only else 0
        return st, ev[first].elapsed_time(ev[2]) * 1e-3

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
    """harness.py:92-98."""

    generation: int
    time_s: float
    igd: float
    hv: float
    ideal: list


@dataclass
class RepeatRecord:
    """harness.py:101-110."""

    repeat: int
    initial: dict
    rows: list = field(default_factory=list)
    mean_gen_time_s: float = math.nan
    final_igd: float = math.nan
    final_hv: float = math.nan
    timed_out: bool = False


@dataclass
class RunRecord:
    """harness.py:113-118."""

    config: dict
    metadata: dict
    repeats: list
    summary: dict


@dataclass
class ScaleCell:
    size: int
    mean_gen_time_s: float
    generations_done: int
    status: str  # "ok" | "timeout"


@dataclass
class ScaleResult:
    kind: str
    config: dict
    metadata: dict
    cells: list


def _metadata() -> dict:
    from . import __version__

    t = _lib.torch()
    dev = t.cuda.get_device_name(t.cuda.current_device()) if t.cuda.is_available() else "none"
    return {"library": f"temo {__version__} (paper_2503_20286_b200)", "platform": platform.platform(),
            "python": platform.python_version(), "numpy": np.__version__, "device": dev}


class _Indicators:
    """Cached reference front and HV corner for per-generation metrics (harness.py:250-268);
    the indicators themselves run on the device (indicators.py)."""

    def __init__(self, config: RunConfig, spec: ProblemSpec):
        self.want_igd = "igd" in config.indicators
        self.want_hv = "hv" in config.indicators
        self.front = None
        self.hv_ref = None
        if self.want_igd or self.want_hv:
            self.front = true_front(spec, config.ref_front_size)
            self.hv_ref = 1.1 * self.front.max(axis=0)
            self.hv_ref[self.hv_ref <= 0] = 1e-6
            self.front_d = _lib.torch().from_numpy(np.ascontiguousarray(self.front)).to(_lib.device(config.device))

    def measure(self, F) -> tuple:
        gi = igd(F, self.front_d) if self.want_igd else math.nan
        gh = hv_indicator(F, self.hv_ref) if self.want_hv else math.nan
        return gi, gh


def run(config: RunConfig, deadline: float | None = None) -> RunRecord:
    """Execute all repeats of a configured run (harness.py:270-319), optionally up to a deadline.

    Every generation's ``time_s`` is the device time of the step (or of the selection with
    ``time_selection_only``) from CUDA events; indicators run on the device every
    ``indicator_every`` generations; ``ideal`` is the objective-wise minimum (one host read per
    generation, as the reference records it).  The device status word is checked every
    generation, so a failed selection raises the reference's exception at once."""
    config.validate()
    spec, R, n_eff = _resolve(config)
    stepper = _Stepper(config, spec, R, n_eff)
    metrics = _Indicators(config, spec)
    root = RngStream(config.seed)
    repeats = []
    for rep in range(config.repeats):
        gen = root.split(rep).generator()
        st = stepper.init(gen)
        F = stepper.objectives(st)
        gi, gh = metrics.measure(F)
        record = RepeatRecord(rep, {"igd": gi, "hv": gh, "ideal": F.min(dim=0).values.cpu().numpy().tolist()})
        for g in range(1, config.generations + 1):
            st, time_s = stepper.step(st, g, gen)
            stepper.check()
            F = stepper.objectives(st)
            every = config.indicator_every
            if every > 0 and g % every == 0:
                gi, gh = metrics.measure(F)
            else:
                gi, gh = math.nan, math.nan
            record.rows.append(GenRow(g, time_s, gi, gh, F.min(dim=0).values.cpu().numpy().tolist()))
            if deadline is not None and time.perf_counter() > deadline:
                record.timed_out = True
                break
        stepper.stop_host_pipeline()
        F = stepper.objectives(st)
        record.final_igd, record.final_hv = metrics.measure(F)
        if record.rows:
            record.mean_gen_time_s = float(np.mean([r.time_s for r in record.rows]))
        repeats.append(record)
        if deadline is not None and time.perf_counter() > deadline:
            break
    summary = {
        "median_final_igd": float(np.median([r.final_igd for r in repeats])),
        "median_final_hv": float(np.median([r.final_hv for r in repeats])),
        "mean_gen_time_s": float(np.mean([r.mean_gen_time_s for r in repeats])),
        "effective_pop_size": n_eff,
        "directions": R.count,
    }
    rec = RunRecord(dataclasses.asdict(config), _metadata(), repeats, summary)
    if config.out:
        emit(rec, "json", config.out)
    return rec


def scaling_experiment(kind: str, base: RunConfig, steps: int, timeout_s: float | None = None) -> ScaleResult:
    """Double the population or the dimension per step and time each cell (harness.py:322-361)."""
    if kind not in ("population", "dimension"):
        raise ConfigError("scale kind must be 'population' or 'dimension'")
    if steps < 1:
        raise ConfigError("steps must be at least 1")
    base.validate()
    cells = []
    for step_idx in range(steps):
        if kind == "population":
            size = base.pop_size * (2 ** step_idx)
            cfg = dataclasses.replace(base, pop_size=size, out=None)
        else:
            start = base.dim if base.dim is not None else 1024
            size = start * (2 ** step_idx)
            cfg = dataclasses.replace(base, dim=size, out=None)
        dl = None if timeout_s is None else time.perf_counter() + timeout_s
        record = run(cfg, deadline=dl)
        timed_out = any(r.timed_out for r in record.repeats) or len(record.repeats) < cfg.repeats
        done = sum(len(r.rows) for r in record.repeats)
        if timed_out:
            cells.append(ScaleCell(size, math.nan, done, "timeout"))
        else:
            cells.append(ScaleCell(size, float(np.mean([r.mean_gen_time_s for r in record.repeats])), done, "ok"))
    return ScaleResult(kind, dataclasses.asdict(base), _metadata(), cells)


def _fmt(x: float) -> str:
    return f"{x:.17g}"


def emit(record: RunRecord, fmt: str, out_dir) -> list:
    """Write a RunRecord as per-repeat CSVs or a single JSON mirror (harness.py:368-395)."""
    out = Path(out_dir)
    out.mkdir(parents=True, exist_ok=True)
    written = []
    if fmt == "csv":
        for rep in record.repeats:
            path = out / f"run_rep{rep.repeat}.csv"
            with open(path, "w") as fh:
                for key in ("algorithm", "problem", "seed"):
                    fh.write(f"# {key}={record.config[key]}\n")
                fh.write(f"# library={record.metadata['library']}\n")
                fh.write(f"# repeat={rep.repeat}\n")
                fh.write(",".join(CSV_COLUMNS) + "\n")
                for row in rep.rows:
                    fh.write(f"{row.generation},{_fmt(row.time_s)},{_fmt(row.igd)},{_fmt(row.hv)}\n")
            written.append(path)
    elif fmt == "json":
        path = out / "run.json"
        with open(path, "w") as fh:
            json.dump(dataclasses.asdict(record), fh, indent=2)
        written.append(path)
    else:
        raise ConfigError(f"unknown emit format {fmt!r}")
    return written


def emit_scale(result: ScaleResult, out_dir) -> list:
    """scale.csv plus a JSON mirror (harness.py:398-413)."""
    out = Path(out_dir)
    out.mkdir(parents=True, exist_ok=True)
    csv_path = out / "scale.csv"
    with open(csv_path, "w") as fh:
        fh.write(f"# kind={result.kind}\n")
        fh.write(f"# algorithm={result.config['algorithm']}\n")
        fh.write(f"# library={result.metadata['library']}\n")
        fh.write("size,mean_gen_time_s,generations,status\n")
        for cell in result.cells:
            fh.write(f"{cell.size},{_fmt(cell.mean_gen_time_s)},{cell.generations_done},{cell.status}\n")
    json_path = out / "scale.json"
    with open(json_path, "w") as fh:
        json.dump(dataclasses.asdict(result), fh, indent=2)
    return [csv_path, json_path]


def parse_run_csv(path) -> tuple:
    """Read back an emitted per-repeat CSV: (metadata, data rows) (harness.py:416-431)."""
    meta, rows = {}, []
    with open(path) as fh:
        for line in fh:
            line = line.strip()
            if not line:
                continue
            if line.startswith("#"):
                key, _, value = line[1:].strip().partition("=")
                meta[key] = value
                continue
            if line.startswith("generation"):
                continue
            g, t, gi, gh = line.split(",")
            rows.append((int(g), float(t), float(gi), float(gh)))
    return meta, rows
