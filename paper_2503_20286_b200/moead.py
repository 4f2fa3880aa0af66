"""Decoupled MOEA/D on the GPU -- drop-in for ``temo.moead`` (moead.py:24-174).

PBI follows the reference bit for bit (moead.py:43-67, App. A4b); Tchebycheff
(``kind="tch"``) is the new aggregation of the north star (no reference:
parity unpinned, self-oracle in oracle/moead.py).  The elite selection uses the
O(n T) reverse-CSR rule of SURVEY App. A5 instead of the reference's O(n^2)
column scan; the n x n ``UpdateIndexMatrix`` is materialised only on request.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _lib
from .rng import DeviceDraws, is_philox
from .rng import PhiloxState as _PhiloxState

KINDS = {"pbi": 0, "tch": 1}


@dataclass(frozen=True)
class MoeadState:
    """Population, objectives, ideal point, weights, neighbourhoods, penalty (moead.py:24-33)."""

    X: object
    F1: object
    z: object
    W: object
    I_nb: object
    theta: float = 5.0


class UpdateIndexMatrix:
    """moead.py:36-40: row i of I_new is arange(n) with -1 where offspring i replaces.

    Stored compactly as ``improves`` (n x T) over ``I_nb``; ``I_new`` materialises."""

    def __init__(self, improves, I_nb, g_new=None):
        self.improves = improves
        self.I_nb = I_nb
        self.g_new = g_new

    @property
    def I_new(self):
        t = _lib.torch()
        imp = self.improves.bool() if isinstance(self.improves, t.Tensor) else \
            t.from_numpy(np.asarray(self.improves, dtype=bool))
        nb = self.I_nb if isinstance(self.I_nb, t.Tensor) else t.from_numpy(np.asarray(self.I_nb))
        n, T = nb.shape
        out = t.arange(n, dtype=t.int64, device=imp.device).expand(n, n).clone()
        rows = t.arange(n, device=imp.device).repeat_interleave(T)
        mask = imp.reshape(-1)
        out[rows[mask], nb.reshape(-1).to(imp.device)[mask]] = -1
        return out.cpu().numpy()


def _t():
    return _lib.torch()


def pbi(f, w, z, theta, normalize_direction=True):
    """d1 + theta*d2 with broadcasting over leading axes (moead.py:43-67)."""
    return _aggregate(f, w, z, theta, "pbi", normalize_direction)


def tchebycheff(f, w, z, theta=None):
    """max_k w_k |f_k - z_k| (Zhang & Li 2007); the north star's MOEA/D aggregation."""
    return _aggregate(f, w, z, 0.0, "tch", True)


def _aggregate(f, w, z, theta, kind, normalize):
    t = _t()
    fa, wa, za = (np.asarray(a, dtype=np.float64) for a in (f, w, z))
    if kind == "pbi" and np.any(np.sqrt(np.sum(wa * wa, axis=-1)) == 0):
        raise ValueError("zero weight vector in PBI")
    fb, wb, zb = np.broadcast_arrays(fa, wa, za)
    shape = fb.shape[:-1]
    m = fb.shape[-1]
    rows = int(np.prod(shape)) if shape else 1
    dev = _lib.device()
    up = lambda a: t.from_numpy(np.ascontiguousarray(a.reshape(rows, m))).to(dev)  # noqa: E731
    F, Wd, Z = up(fb), up(wb), up(zb)
    out = t.empty(rows, dtype=t.float64, device=dev)
    rc = _lib.lib().temo_aggregate_rows(_lib.ptr(F), _lib.ptr(Wd), _lib.ptr(Z), rows, m, float(theta),
                                        KINDS[kind], 1 if normalize else 0, _lib.ptr(out),
                                        _lib.stream_handle(dev))
    _lib.check(rc, kind)
    res = out.cpu().numpy().reshape(shape)
    return res if shape else float(res)


class MoeadEngine:
    """Device-resident MOEA/D generation (moead.py:148-158) for a ProblemSpec.

    Per step: two ``integers`` draws on the host Generator (reference order,
    App. B), then one fused offspring+evaluation kernel drawing its uniforms
    from the same Philox stream, the compare kernel and the elite kernel."""

    def __init__(self, spec, R, table, params, theta=5.0, aggregation="pbi", dev=None):
        t = _t()
        self.dev = _lib.device(dev)
        self.spec, self.R, self.params, self.theta = spec, R, params, float(theta)
        self.kind = KINDS[aggregation]
        self.n, self.T = table.I_nb.shape
        if self.T < 2:
            raise ValueError("neighborhood size must be at least 2 for mating")
        I_nb = np.ascontiguousarray(table.I_nb, dtype=np.int64)
        self.I_nb_host = I_nb
        self.I_nb = t.from_numpy(I_nb.astype(np.int32)).to(self.dev)
        # reverse CSR: for each direction j the entries q = i*T + t with I_nb[i,t] == j, ascending i
        flat = I_nb.reshape(-1)
        order = np.argsort(flat, kind="stable")
        counts = np.bincount(flat, minlength=self.n)
        self.rptr = t.from_numpy(np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)).to(self.dev)
        self.rcol = t.from_numpy(order.astype(np.int32)).to(self.dev)
        self.W = R.device(self.dev)
        d, m = spec.d, spec.m
        z = lambda *s, dt=t.float64: t.empty(*s, dtype=dt, device=self.dev)  # noqa: E731
        self.O, self.F2 = z((self.n, d)), z((self.n, m))
        self.zmin = z(m)
        self.g_new = z((self.n, self.T))
        self.improves = z((self.n, self.T), dt=t.uint8)
        self.winner = z(self.n, dt=t.int32)
        self.parents = z(2 * self.n, dt=t.int64)
        self.ring = _lib.HostRing()
        self.var = params.struct(d, self.dev)
        self.prob = spec.struct()
        # one CUDA graph per state parity (TEMO_MOEAD_GRAPH=0: plain launches)
        import os

        self.graph = os.environ.get("TEMO_MOEAD_GRAPH", "1") != "0"
        self._gbuf, self._graphs = None, [None, None]

    def init_state(self, X, F1):
        t = _t()
        z0 = F1.min(dim=0).values.clone()
        return MoeadState(X.clone(), F1.clone(), z0, self.W, self.I_nb, self.theta)

    def step(self, st: MoeadState, gen):
        t = _t()
        n, T = self.n, self.T
        a = gen.integers(0, T, size=n)
        b = gen.integers(0, T - 1, size=n)
        draws = DeviceDraws(gen)
        off = draws.take(5 * n * self.spec.d if self.params.gene_swap else 3 * n * self.spec.d)
        if self.graph and off == 0 and (n * self.spec.d) % 4 == 0 and self.spec.d <= 3000:
            # the neighbour lookup I_nb[i, a_i], I_nb[i, b_i + (b_i >= a_i)] runs inside the graph:
            # only the raw draws go up (2n int32 instead of the host fancy-indexing + 2n int64)
            ab = np.empty(2 * n, dtype=np.int32)
            ab[:n] = a
            ab[n:] = b
            if getattr(self, "_ab", None) is None:
                self._ab = t.empty(2 * n, dtype=t.int32, device=self.dev)
            self.ring.upload(ab, self._ab)
            out = self._step_graph(st, draws)
            draws.commit()
            return out
        b = b + (b >= a)
        rows = np.arange(n)
        par = np.concatenate([self.I_nb_host[rows, a], self.I_nb_host[rows, b]]).astype(np.int64)
        self.ring.upload(par, self.parents)
        L = _lib.lib()
        p = _lib.ptr
        rc = L.temo_moead_offspring(_lib.sptr(self.prob), _lib.sptr(self.var), p(st.X), p(self.parents),
                                    p(self.parents[n:]), n, _lib.sptr(draws.state), off, p(self.O), p(self.F2),
                                    _lib.stream_handle(self.dev))
        _lib.check(rc, "moead_offspring")
        draws.commit()
        return self.select(st, self.O, self.F2)

    # -- CUDA-graph generation (moead.py:148-158 as one graph replay per step)
    def _graph_buffers(self, st: MoeadState):
        t = _t()
        if self._gbuf is None:
            self._gbuf = ([t.empty_like(st.X) for _ in range(2)], [t.empty_like(st.F1) for _ in range(2)],
                          [t.empty_like(self.zmin) for _ in range(2)],
                          t.zeros(ctypes.sizeof(_PhiloxState), dtype=t.uint8, device=self.dev))
        gX, gF, gz, _ = self._gbuf
        for p in (0, 1):  # the state already lives in a graph buffer: replay that parity's graph
            if st.X.data_ptr() == gX[p].data_ptr() and st.F1.data_ptr() == gF[p].data_ptr() \
                    and st.z.data_ptr() == gz[p].data_ptr():
                return p
        gX[0].copy_(st.X)
        gF[0].copy_(st.F1)
        gz[0].copy_(st.z)
        return 0

    def _capture(self, p: int):
        t = _t()
        gX, gF, gz, st_dev = self._gbuf
        q = 1 - p
        L, ptr = _lib.lib(), _lib.ptr
        g = t.cuda.CUDAGraph()
        with t.cuda.graph(g, capture_error_mode="thread_local"):
            h = _lib.stream_handle(self.dev)
            n = self.n
            a = self._ab[:n].long()
            b = self._ab[n:].long()
            b = b + (b >= a).long()
            rows = t.arange(n, device=self.dev)
            self.parents[:n].copy_(self.I_nb[rows, a])
            self.parents[n:].copy_(self.I_nb[rows, b])
            rc = L.temo_moead_offspring_dev(_lib.sptr(self.prob), _lib.sptr(self.var), ptr(gX[p]), ptr(self.parents),
                                            ptr(self.parents[self.n:]), self.n, ptr(st_dev), 0, ptr(self.O),
                                            ptr(self.F2), h)
            _lib.check(rc, "moead_offspring")
            self._select_into(gX[p], gF[p], gz[p], self.O, self.F2, gX[q], gF[q], h)
            gz[q].copy_(self.zmin)
        return g

    def _step_graph(self, st: MoeadState, draws):
        """One generation as a CUDA-graph replay: the pairing indices and the Philox state are
        uploaded to fixed device buffers (stream-ordered), then one graph runs offspring +
        compare + elite.  The state ping-pongs between two buffer sets, one graph per parity;
        a returned state stays valid until two more steps have run."""
        p = self._graph_buffers(st)
        gX, gF, gz, st_dev = self._gbuf
        raw = np.frombuffer(ctypes.string_at(ctypes.addressof(draws.state), ctypes.sizeof(draws.state)),
                            dtype=np.uint8)
        self.ring.upload(raw, st_dev)
        if self._graphs[p] is None:
            self._graphs[p] = self._capture(p)
        self._graphs[p].replay()
        q = 1 - p
        return MoeadState(gX[q], gF[q], gz[q], st.W, st.I_nb, st.theta)

    def _select_into(self, X, F1, z, O, F2, Xn, Fn, h):
        L, p = _lib.lib(), _lib.ptr
        n, T = self.n, self.T
        m, d = F2.shape[1], O.shape[1]
        rc = L.temo_moead_compare(p(F1), p(F2), p(self.W), p(self.I_nb), n, T, m, p(z), self.theta, self.kind,
                                  p(self.zmin), p(self.g_new), p(self.improves), h)
        _lib.check(rc, "compare_update")
        rc = L.temo_moead_elite(p(X), p(F1), p(self.W), p(O), p(F2), n, d, T, m, p(self.zmin), self.theta,
                                self.kind, p(self.rptr), p(self.rcol), p(self.g_new), p(self.improves),
                                p(self.winner), p(Xn), p(Fn), h)
        _lib.check(rc, "elite_select")

    def select(self, st: MoeadState, O, F2):
        """compare_update + elite_select + z update on device tensors."""
        t = _t()
        n, T = self.n, self.T
        L = _lib.lib()
        p = _lib.ptr
        m, d = F2.shape[1], O.shape[1]
        rc = L.temo_moead_compare(p(st.F1), p(F2), p(self.W), p(self.I_nb), n, T, m, p(st.z), st.theta,
                                  self.kind, p(self.zmin), p(self.g_new), p(self.improves),
                                  _lib.stream_handle(self.dev))
        _lib.check(rc, "compare_update")
        Xn = t.empty_like(st.X)
        Fn = t.empty_like(st.F1)
        rc = L.temo_moead_elite(p(st.X), p(st.F1), p(self.W), p(O), p(F2), n, d, T, m, p(self.zmin),
                                st.theta, self.kind, p(self.rptr), p(self.rcol), p(self.g_new),
                                p(self.improves), p(self.winner), p(Xn), p(Fn), _lib.stream_handle(self.dev))
        _lib.check(rc, "elite_select")
        return MoeadState(Xn, Fn, self.zmin.clone(), st.W, st.I_nb, st.theta)


# ------------------------------------------------------------------ reference-shaped API
class _Table:
    def __init__(self, I_nb):
        self.I_nb = np.asarray(I_nb)


def _engine_for(state: MoeadState, kind="pbi"):
    from .directions import DirectionSet

    W = np.asarray(state.W.cpu().numpy() if hasattr(state.W, "cpu") else state.W, dtype=np.float64)
    I_nb = np.asarray(state.I_nb.cpu().numpy() if hasattr(state.I_nb, "cpu") else state.I_nb)
    R = DirectionSet.__new__(DirectionSet)
    object.__setattr__(R, "W", W)
    object.__setattr__(R, "kind", "simplex")

    class _Spec:  # shapes only; the engine's fused offspring path is not used here
        d = np.asarray(state.X).shape[1] if not hasattr(state.X, "shape") else state.X.shape[1]
        m = W.shape[1]

        @staticmethod
        def struct():
            return None

    class _Params:
        gene_swap = True

        @staticmethod
        def struct(d, dev):
            return None

    return MoeadEngine(_Spec, R, _Table(I_nb), _Params, state.theta, kind)


def _dev(x):
    t = _t()
    return _lib.as_device(x, t.float64)[0]


def compare_update(state: MoeadState, F2, aggregation="pbi"):
    """Batched neighbourhood comparison (moead.py:70-92) -> (UpdateIndexMatrix, z_min)."""
    t = _t()
    eng = _engine_for(state, aggregation)
    st = MoeadState(_dev(state.X), _dev(state.F1), _dev(state.z), eng.W, eng.I_nb, state.theta)
    F2d = _dev(F2)
    n, T = eng.n, eng.T
    L = _lib.lib()
    p = _lib.ptr
    rc = L.temo_moead_compare(p(st.F1), p(F2d), p(eng.W), p(eng.I_nb), n, T, F2d.shape[1], p(st.z),
                              state.theta, eng.kind, p(eng.zmin), p(eng.g_new), p(eng.improves),
                              _lib.stream_handle(eng.dev))
    _lib.check(rc, "compare_update")
    upd = UpdateIndexMatrix(eng.improves.cpu().numpy().astype(bool), eng.I_nb_host, eng.g_new.cpu().numpy())
    return upd, eng.zmin.cpu().numpy()


def elite_select(state: MoeadState, O, F2, update: UpdateIndexMatrix, z_min, block: int = 256,
                 aggregation="pbi"):
    """Per-direction elite pick (moead.py:95-124) -> (X_next, F_next)."""
    del block
    t = _t()
    eng = _engine_for(state, aggregation)
    st = MoeadState(_dev(state.X), _dev(state.F1), _dev(z_min), eng.W, eng.I_nb, state.theta)
    eng.improves.copy_(t.from_numpy(np.asarray(update.improves, dtype=np.uint8)).to(eng.dev))
    if update.g_new is not None:
        eng.g_new.copy_(t.from_numpy(np.asarray(update.g_new, dtype=np.float64)).to(eng.dev))
    eng.zmin.copy_(_dev(z_min))
    Od, F2d = _dev(O), _dev(F2)
    n, T = eng.n, eng.T
    L = _lib.lib()
    p = _lib.ptr
    if update.g_new is None:  # recompute g_new with the identical ops
        rc = L.temo_moead_compare(p(st.F1), p(F2d), p(eng.W), p(eng.I_nb), n, T, F2d.shape[1], p(st.z),
                                  state.theta, eng.kind, p(eng.zmin), p(eng.g_new), p(eng.improves),
                                  _lib.stream_handle(eng.dev))
        _lib.check(rc, "elite_select")
        eng.improves.copy_(t.from_numpy(np.asarray(update.improves, dtype=np.uint8)).to(eng.dev))
        eng.zmin.copy_(_dev(z_min))
    Xn, Fn = t.empty_like(st.X), t.empty_like(st.F1)
    rc = L.temo_moead_elite(p(st.X), p(st.F1), p(eng.W), p(Od), p(F2d), n, Od.shape[1], T, F2d.shape[1],
                            p(eng.zmin), state.theta, eng.kind, p(eng.rptr), p(eng.rcol), p(eng.g_new),
                            p(eng.improves), p(eng.winner), p(Xn), p(Fn), _lib.stream_handle(eng.dev))
    _lib.check(rc, "elite_select")
    return Xn.cpu().numpy(), Fn.cpu().numpy()


def moead_offspring(state: MoeadState, rng, params, evaluate_fn):
    """One offspring per subproblem from two distinct random neighbours (moead.py:127-145)."""
    from .variation import polynomial_mutation, sbx

    I_nb = np.asarray(state.I_nb.cpu().numpy() if hasattr(state.I_nb, "cpu") else state.I_nb)
    n, T = I_nb.shape
    if T < 2:
        raise ValueError("neighborhood size must be at least 2 for mating")
    a = rng.integers(0, T, size=n)
    b = rng.integers(0, T - 1, size=n)
    b = b + (b >= a)
    rows = np.arange(n)
    X = state.X
    t = _t()
    if isinstance(X, t.Tensor):
        p1, p2 = X[t.as_tensor(I_nb[rows, a], device=X.device)], X[t.as_tensor(I_nb[rows, b], device=X.device)]
    else:
        X = np.asarray(X)
        p1, p2 = X[I_nb[rows, a]], X[I_nb[rows, b]]
    kids = sbx(rng, p1, p2, params)[:n]
    O = polynomial_mutation(rng, kids, params)
    return O, evaluate_fn(O)


def step(state: MoeadState, rng, params, evaluate_fn, aggregation="pbi"):
    """Reproduce, compare/update, elite-select, move z (moead.py:148-158)."""
    O, F2 = moead_offspring(state, rng, params, evaluate_fn)
    update, z_min = compare_update(state, F2, aggregation)
    Xn, Fn = elite_select(state, O, F2, update, z_min, aggregation=aggregation)
    return MoeadState(Xn, Fn, z_min, state.W, state.I_nb, state.theta)


def init_state(X, F1, W, table, theta: float = 5.0) -> MoeadState:
    """moead.py:161-169."""
    F1 = np.asarray(F1)
    return MoeadState(np.asarray(X), F1, F1.min(axis=0), np.asarray(W), table.I_nb, theta)


def default_neighborhood(n: int) -> int:
    """max(2, ceil(n/10)) capped at 20 (moead.py:172-174)."""
    return min(20, max(2, -(-n // 10)))
