"""NSGA-III environmental selection on the GPU -- drop-in for ``temo.nsga3`` (nsga3.py:26-218).

``environmental_selection`` draws ``rng.permutation(N)`` on the host exactly
like the reference (nsga3.py:204), then runs rank (SELECT mode), normalize,
associate, niche fill, repair and keep on the device in one stream with no
host round trip (``temo_rank`` + ``temo_nsga3_select``).  The standalone
functions map one-to-one onto C-ABI entry points for stage-level parity.

``Nsga3Selector`` is the allocation-free device form used by the harness and
the benchmark: inputs and outputs stay in HBM.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _lib
from .directions import DirectionSet
from .ndsort import SELECT, rank_device
from .rng import permutation as rng_permutation

BIG = np.finfo(np.float64).max  # tensorops.py:18


@dataclass(frozen=True)
class NormalizedObjectives:
    Fp: object
    ideal: object
    intercepts: object


@dataclass(frozen=True)
class AssociationResult:
    pi: object
    dist: object


@dataclass(frozen=True)
class NicheState:
    rho: object
    rho_l: object
    n_s: int


@dataclass(frozen=True)
class NicheSelection:
    rank: object
    promoted: object
    n_selected: int


def _t():
    return _lib.torch()


def _out(x, as_numpy):
    return x.cpu().numpy() if as_numpy else x


def _ws(N, m, nr, dev):
    return _lib.workspace.get(_lib.lib().temo_nsga3_select_ws_bytes(N, m, nr), dev)


def normalize(F) -> NormalizedObjectives:
    """Ideal shift + hyperplane intercepts (nsga3.py:61-93); NaN rows are excluded rows."""
    t = _t()
    Fd, was_np = _lib.as_device(F, t.float64)
    N, m = Fd.shape
    if bool(t.isnan(Fd).all(dim=0).any()):
        raise ValueError("a column is all-NaN: no retained rows to normalize")
    Fp = t.empty_like(Fd)
    ideal = t.empty(m, dtype=t.float64, device=Fd.device)
    icpt = t.empty(m, dtype=t.float64, device=Fd.device)
    ws = _ws(N, m, 1, Fd.device)
    rc = _lib.lib().temo_nsga3_normalize(_lib.ptr(Fd), N, m, _lib.ptr(Fp), _lib.ptr(ideal),
                                         _lib.ptr(icpt), None, _lib.ptr(ws), ws.numel(),
                                         _lib.stream_handle(Fd.device))
    _lib.check(rc, "normalize")
    return NormalizedObjectives(_out(Fp, was_np), _out(ideal, was_np), _out(icpt, was_np))


def associate(Fp, R: DirectionSet, lattice: bool = True) -> AssociationResult:
    """Perpendicular-nearest direction, first index on ties (nsga3.py:96-116).

    For das_dennis direction sets the exact lattice search is used (``lattice``
    False forces the filtered full scan; both are bit-identical)."""
    t = _t()
    Fd, was_np = _lib.as_device(Fp, t.float64)
    N, m = Fd.shape
    Wd = R.device(Fd.device)
    pi = t.empty(N, dtype=t.int32, device=Fd.device)
    dist = t.empty(N, dtype=t.float64, device=Fd.device)
    ws = _ws(N, m, R.count, Fd.device)
    rc = _lib.lib().temo_associate(_lib.ptr(Fd), N, m, _lib.ptr(Wd), R.count,
                                   R.lattice_H if lattice else 0, _lib.ptr(pi),
                                   _lib.ptr(dist), _lib.ptr(ws), ws.numel(), _lib.stream_handle(Fd.device))
    _lib.check(rc, "associate")
    return AssociationResult(_out(pi.to(t.int64), was_np), _out(dist, was_np))


def niche_counts(r, pi, l: int, n_r: int) -> NicheState:
    """Occupancy over ranks < l and == l (nsga3.py:119-123)."""
    t = _t()
    rd, was_np = _lib.as_device(r, t.int32)
    pd, _ = _lib.as_device(pi, t.int32, rd.device)
    N = rd.numel()
    rho = t.empty(n_r, dtype=t.int32, device=rd.device)
    rho_l = t.empty(n_r, dtype=t.int32, device=rd.device)
    ws = _ws(N, 1, n_r, rd.device)
    rc = _lib.lib().temo_niche_counts(_lib.ptr(rd), _lib.ptr(pd), N, int(l), n_r, _lib.ptr(rho),
                                      _lib.ptr(rho_l), _lib.ptr(ws), ws.numel(),
                                      _lib.stream_handle(rd.device))
    _lib.check(rc, "niche_counts")
    rho64, rho_l64 = rho.to(t.int64), rho_l.to(t.int64)
    return NicheState(_out(rho64, was_np), _out(rho_l64, was_np), int(rho64.sum().item()))


def niche_select(state: NicheState, r, pi, dist, l: int, n: int) -> NicheSelection:
    """Fill empty niches with their closest rank-l member (nsga3.py:126-167)."""
    del n
    t = _t()
    rd, was_np = _lib.as_device(r, t.int32)
    rd = rd.clone()
    pd, _ = _lib.as_device(pi, t.int32, rd.device)
    dd, _ = _lib.as_device(dist, t.float64, rd.device)
    rho, _ = _lib.as_device(state.rho, t.int32, rd.device)
    N, nr = rd.numel(), rho.numel()
    promoted = t.empty(max(nr, 1), dtype=t.int32, device=rd.device)
    counts = t.zeros(8, dtype=t.int32, device=rd.device)
    ws = _ws(N, 1, nr, rd.device)
    rc = _lib.lib().temo_niche_select(_lib.ptr(rd), _lib.ptr(pd), _lib.ptr(dd), N, int(l), _lib.ptr(rho),
                                      nr, _lib.ptr(promoted), _lib.ptr(counts), _lib.ptr(ws),
                                      ws.numel(), _lib.stream_handle(rd.device))
    _lib.check(rc, "niche_select")
    k = int(counts[0].item())
    prom = promoted[:k].to(t.int64)
    return NicheSelection(_out(rd.to(t.int64), was_np), _out(prom, was_np), int(state.n_s) + k)


def update_rank(r, selected, n_dif: int, l: int):
    """Promote by index order or demote the most recent promotions (nsga3.py:170-183)."""
    t = _t()
    rd, was_np = _lib.as_device(r, t.int32)
    rd = rd.clone()
    sel, _ = _lib.as_device(np.asarray(selected, dtype=np.int64) if not isinstance(selected, t.Tensor)
                            else selected, t.int32, rd.device)
    N = rd.numel()
    status = _lib.new_status(rd.device)
    ws = _ws(N, 1, 1, rd.device)
    sel_ptr = _lib.ptr(sel) if sel.numel() else _lib.ptr(rd)
    rc = _lib.lib().temo_update_rank(_lib.ptr(rd), N, sel_ptr, sel.numel(), int(n_dif), int(l),
                                     _lib.ptr(status), _lib.ptr(ws), ws.numel(),
                                     _lib.stream_handle(rd.device))
    _lib.check(rc, "update_rank")
    _lib.sync_status(status, "update_rank")
    return _out(rd.to(t.int64), was_np)


class Nsga3Selector:
    """Device-resident selection of n rows out of N merged rows (nsga3.py:207-218).

    Buffers are allocated once; ``select`` only enqueues kernels.  ``keep`` are
    indices into the shuffled order (ascending), like ``flatnonzero(rank < l)``.
    """

    def __init__(self, N: int, m: int, R: DirectionSet, n: int, dev=None, record=False, lattice=True,
                 dist_rank=None):
        t = _t()
        self.lattice_H = R.lattice_H if lattice else 0
        self.dist_rank = dist_rank  # parallel.DistRank: column-sharded ND sort across ranks
        self.dev = _lib.device(dev)
        self.N, self.m, self.n = N, m, n
        self.R = R
        self.W = R.device(self.dev)
        nr = R.count
        z = lambda *s, dt=t.int32: t.empty(*s, dtype=dt, device=self.dev)  # noqa: E731
        self.Fs = z((N, m), dt=t.float64)
        self.rank = z(N)
        self.l = z(1)
        self.nfronts = z(1)
        self.keep = z(n)
        self.pi = z(N)
        self.dist = z(N, dt=t.float64)
        self.icpt = z(m, dt=t.float64)
        self.ideal = z(m, dt=t.float64)
        self.promoted = z(max(nr, 1))
        self.counts = z(8)
        self.status = t.zeros(1, dtype=t.int32, device=self.dev)
        self.record = record
        self.Fp = z((N, m), dt=t.float64) if record else None
        self.extreme = z(m, dt=t.int64) if record else None
        self.rho = z(nr) if record else None
        self.rho_l = z(nr) if record else None
        L = _lib.lib()
        self.ws_sel = L.temo_nsga3_select_ws_bytes(N, m, nr)

    def select_shuffled(self, Fs=None):
        """Run on ``self.Fs`` (or copy ``Fs`` in first); returns the keep tensor."""
        if Fs is not None:
            self.Fs.copy_(Fs)
        if self.dist_rank is not None:
            r, l, nf = self.dist_rank(self.Fs, self.n, SELECT)
            self.status.bitwise_or_(self.dist_rank.status)  # K0's NaN flag of the sharded rank
            self.rank.copy_(r)
            self.l.fill_(l)
            self.nfronts.fill_(nf)
        else:
            rank_device(self.Fs, self.n, SELECT, self.status, out=(self.rank, self.l, self.nfronts))
        L = _lib.lib()
        ws = _lib.workspace.get(self.ws_sel, self.dev)
        p = _lib.ptr
        rc = L.temo_nsga3_select(p(self.Fs), self.N, self.m, p(self.W), self.R.count, self.lattice_H,
                                 self.n, p(self.rank),
                                 p(self.l), p(self.keep), p(self.pi), p(self.dist), p(self.Fp),
                                 p(self.ideal), p(self.icpt), p(self.extreme), p(self.rho), p(self.rho_l),
                                 p(self.promoted), p(self.counts), p(self.status), p(ws), ws.numel(),
                                 _lib.stream_handle(self.dev))
        _lib.check(rc, "environmental_selection")
        return self.keep

    def select(self, Fm, perm):
        """Shuffle by ``perm`` (int64 device tensor) then select; returns keep."""
        _lib.gather_rows(Fm, perm, self.Fs)
        return self.select_shuffled()

    def check(self):
        _lib.sync_status(self.status, "environmental_selection")


def environmental_selection(X, F, R: DirectionSet, n: int, rng):
    """Select exactly n rows; returned in shuffled order (nsga3.py:186-218)."""
    t = _t()
    is_np = not isinstance(X, t.Tensor)
    Xd, _ = _lib.as_device(X, t.float64)
    Fd, _ = _lib.as_device(F, t.float64, Xd.device)
    N = Xd.shape[0]
    if Fd.shape[0] != N or N < n:
        raise ValueError("need matching X/F with at least n rows")
    # the reference draws the shuffle first (nsga3.py:204) and raises inside rank_assign
    perm = t.as_tensor(rng_permutation(rng, N)).to(Xd.device)
    if is_np and np.isnan(np.asarray(F, dtype=np.float64)).any():
        raise ValueError("objective matrix contains NaN rows")
    sel = Nsga3Selector(N, Fd.shape[1], R, n, Xd.device)
    keep = sel.select(Fd, perm)
    Xn = t.empty((n, Xd.shape[1]), dtype=t.float64, device=Xd.device)
    Fn = t.empty((n, Fd.shape[1]), dtype=t.float64, device=Xd.device)
    _lib.gather_rows2(Xd, perm, keep, Xn)
    _lib.gather_rows(sel.Fs, keep, Fn)
    sel.check()
    return (Xn.cpu().numpy(), Fn.cpu().numpy()) if is_np else (Xn, Fn)
