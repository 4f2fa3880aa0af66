"""HypE Monte-Carlo hypervolume fitness and selection on the GPU -- drop-in for ``temo.hype`` (hype.py:21-163).

Estimation runs in ``libtemo_b200.so`` (csrc/hype.cu): sample-bitmap pass,
per-sample dominator counts, and the contribution sums in the OpenBLAS dgemv_t
order of SURVEY App. A7 so that estimates are bit-identical to the reference
run with single-threaded OpenBLAS.  Uniform samples come from the caller's
NumPy Philox Generator state on the device; the host Generator is advanced only
when the reference would have drawn (k >= 1 and a non-degenerate box).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _lib
from .ndsort import SELECT, rank_device
from .rng import DeviceDraws, advance, is_philox

BIG = np.finfo(np.float64).max


@dataclass(frozen=True)
class HvEstimateParams:
    """Sampling-box corner, removal parameter k, sample count (hype.py:21-34)."""

    v_ref: np.ndarray
    k: int
    s: int

    def __post_init__(self):
        if self.s < 1:
            raise ValueError("need at least one sample")
        if self.k < 1:
            raise ValueError("k must be at least 1")
        object.__setattr__(self, "v_ref", np.asarray(self.v_ref, dtype=np.float64))


def _t():
    return _lib.torch()


def shared_alpha(n1: int, k: int):
    """alpha_1..alpha_k padded with zeros to n1 (hype.py:37-51)."""
    if not 1 <= k <= n1:
        raise ValueError("k must lie in [1, n1]")
    t = _t()
    dev = _lib.device()
    out = t.empty(n1, dtype=t.float64, device=dev)
    _lib.check(_lib.lib().temo_hype_alpha(n1, k, _lib.ptr(out), _lib.stream_handle(dev)), "shared_alpha")
    return out.cpu().numpy()


def auto_reference(F):
    """Columnwise max + 10% of the range (hype.py:129-132)."""
    t = _t()
    Fd, was_np = _lib.as_device(F, t.float64)
    n, m = Fd.shape
    out = t.empty(m, dtype=t.float64, device=Fd.device)
    scratch = t.empty(32, dtype=t.float64, device=Fd.device)
    _lib.check(_lib.lib().temo_auto_reference(_lib.ptr(Fd), n, m, _lib.ptr(out), _lib.ptr(scratch),
                                              _lib.stream_handle(Fd.device)), "auto_reference")
    return out.cpu().numpy() if was_np else out


def _host_draws(rng, s, m, Fd, v_ref):
    """Duck-typed RNGs: draw on the host exactly like the reference, only if the box is valid."""
    t = _t()
    span = v_ref.cpu().numpy() - Fd.min(dim=0).values.cpu().numpy()
    if np.any(span <= 0):
        return None
    blocks, left = [], s
    while left > 0:
        b = min(65536, left)
        blocks.append(np.asarray(rng.random((b, Fd.shape[1])), dtype=np.float64))
        left -= b
    return t.from_numpy(np.ascontiguousarray(np.concatenate(blocks))).to(Fd.device)


def hv_estimate(F, params: HvEstimateParams, rng, sample_block: int = 65536):
    """Per-row MC hypervolume contribution (hype.py:54-85)."""
    if sample_block != 65536:
        raise ValueError("only the reference's 65536-sample blocks are supported")
    t = _t()
    Fd, was_np = _lib.as_device(F, t.float64)
    n1, m = Fd.shape
    if not params.k <= n1:
        raise ValueError("k exceeds the number of rows")
    vref = t.from_numpy(np.ascontiguousarray(params.v_ref)).to(Fd.device)
    out = t.empty(n1, dtype=t.float64, device=Fd.device)
    drew = t.zeros(1, dtype=t.int32, device=Fd.device)
    L = _lib.lib()
    ws = _lib.workspace.get(L.temo_hv_estimate_ws_bytes(n1, m, params.s), Fd.device)
    if is_philox(rng):
        draws = DeviceDraws(rng)
        rc = L.temo_hv_estimate(_lib.ptr(Fd), n1, m, _lib.ptr(vref), params.k, params.s,
                                _lib.sptr(draws.state), 0, None, _lib.ptr(out), _lib.ptr(drew),
                                _lib.ptr(ws), ws.numel(), _lib.stream_handle(Fd.device))
        _lib.check(rc, "hv_estimate")
        if int(drew.item()):
            advance(rng, params.s * m)
    else:
        U = _host_draws(rng, params.s, m, Fd, vref)
        if U is None:
            res = t.zeros(n1, dtype=t.float64, device=Fd.device)
            return res.cpu().numpy() if was_np else res
        rc = L.temo_hv_estimate(_lib.ptr(Fd), n1, m, _lib.ptr(vref), params.k, params.s, None, 0,
                                _lib.ptr(U), _lib.ptr(out), _lib.ptr(drew), _lib.ptr(ws), ws.numel(),
                                _lib.stream_handle(Fd.device))
        _lib.check(rc, "hv_estimate")
    return out.cpu().numpy() if was_np else out


class HypeSelector:
    """Device-resident HypE selection of n out of N rows (hype.py:135-163).

    ``select(F, rng)`` returns keep (n int32, lexsort order).  One small device->host
    read per call decides whether the Generator advances (the reference draws
    samples only when k >= 1 and the box is non-degenerate)."""

    def __init__(self, N: int, m: int, n: int, s: int, v_ref=None, dev=None, shard=None):
        """``shard = (rank, world, exchange)`` splits the Monte-Carlo work by exchange column
        (SURVEY 8e): this rank computes columns [C rank / world, C (rank + 1) / world) of the
        contribution partials and ``exchange(segment, counts)`` all-gathers them (NCCL); the
        combine then runs the reference's summation order on every rank (bit-identical)."""
        t = _t()
        self.dev = _lib.device(dev)
        self.N, self.m, self.n, self.s = N, m, n, s
        z = lambda *sh, dt=t.int32: t.empty(*sh, dtype=dt, device=self.dev)  # noqa: E731
        self.rank, self.l, self.nf = z(N), z(1), z(1)
        self.keep = z(n)
        self.v_hv = z(N, dt=t.float64)
        self.info = t.zeros(4, dtype=t.int32, device=self.dev)
        self.info_host = t.zeros(4, dtype=t.int32).pin_memory()
        self.status = t.zeros(1, dtype=t.int32, device=self.dev)
        self.v_ref = None if v_ref is None else t.from_numpy(np.asarray(v_ref, dtype=np.float64)).to(self.dev)
        self.ws_bytes = _lib.lib().temo_hype_select_ws_bytes(N, m, s)
        self.shard = shard
        if shard is not None:
            r, G, _ = shard
            C = int(_lib.lib().temo_hype_columns(s))
            self.col_bounds = [(C * g // G, C * (g + 1) // G) for g in range(G)]
            lo, hi = self.col_bounds[r]
            self.Tseg = z((max(hi - lo, 1), N), dt=t.float64)

    def select(self, F, rng, U=None, defer: bool = False):
        """``defer=True`` (launch-ahead loops): no host sync for the RNG decision -- the Generator
        is advanced speculatively (the samples are drawn whenever the last front must be cut,
        hype.py:154-158, i.e. almost always) and ``resolve()`` checks the device flag later,
        undoing the advance if no samples were drawn."""
        self.resolve()
        rank_device(F, self.n, SELECT, self.status, out=(self.rank, self.l, self.nf))
        L = _lib.lib()
        ws = _lib.workspace.get(self.ws_bytes, self.dev)
        p = _lib.ptr
        if U is None:
            draws = DeviceDraws(rng)
            st = _lib.sptr(draws.state)
        else:
            st = None
        sh = _lib.stream_handle(self.dev)
        if self.shard is None:
            rc = L.temo_hype_select(p(F), self.N, self.m, self.n, self.s, p(self.v_ref), p(self.rank), p(self.l),
                                    st, 0, p(U), p(self.keep), p(self.v_hv), p(self.info), p(ws), ws.numel(), sh)
            _lib.check(rc, "hype.environmental_selection")
        else:
            r, G, exchange = self.shard
            lo, hi = self.col_bounds[r]
            rc = L.temo_hype_select_begin(p(F), self.N, self.m, self.n, self.s, p(self.v_ref), p(self.rank),
                                          p(self.l), p(ws), ws.numel(), sh)
            _lib.check(rc, "hype.environmental_selection")
            rc = L.temo_hype_select_columns(p(F), self.N, self.m, self.s, lo, hi, st, 0, p(U), p(self.Tseg),
                                            p(ws), ws.numel(), sh)
            _lib.check(rc, "hype.environmental_selection")
            Tg = exchange(self.Tseg[: hi - lo], [b - a for a, b in self.col_bounds])
            rc = L.temo_hype_select_end(p(F), self.N, self.m, self.n, self.s, p(self.rank), p(self.l), p(Tg),
                                        p(self.keep), p(self.v_hv), p(self.info), p(ws), ws.numel(), sh)
            _lib.check(rc, "hype.environmental_selection")
        self.info_host.copy_(self.info, non_blocking=True)
        if defer and U is None:
            t = _lib.torch()
            ev = t.cuda.Event()
            ev.record(t.cuda.current_stream(self.dev))
            saved = rng.bit_generator.state
            advance(rng, self.s * self.m)
            self._pending = (ev, rng, saved)
            return self.keep
        _lib.torch().cuda.current_stream(self.dev).synchronize()
        if U is None and int(self.info_host[3]):
            advance(rng, self.s * self.m)
        return self.keep

    def pending(self) -> bool:
        return getattr(self, "_pending", None) is not None

    def resolve(self) -> bool:
        """Settle a deferred RNG decision: True if the speculative advance was right (or nothing
        was pending); False if it was undone (the Generator is back at the selection's end)."""
        pend = getattr(self, "_pending", None)
        if pend is None:
            return True
        ev, rng, saved = pend
        self._pending = None
        ev.synchronize()
        if int(self.info_host[3]):
            return True
        rng.bit_generator.state = saved
        return False

    def check(self):
        self.resolve()
        _lib.sync_status(self.status, "hype.environmental_selection")


def environmental_selection(X, F, v_ref, n: int, s: int, rng):
    """Keep the first n rows of lexsort(rank, -contribution) (hype.py:135-163)."""
    t = _t()
    is_np = not isinstance(X, t.Tensor)
    Xd, _ = _lib.as_device(X, t.float64)
    Fd, _ = _lib.as_device(F, t.float64, Xd.device)
    N, m = Fd.shape
    if N < n:
        raise ValueError("need at least n rows")
    if is_np and np.isnan(np.asarray(F, dtype=np.float64)).any():
        raise ValueError("objective matrix contains NaN rows")
    sel = HypeSelector(N, m, n, s, v_ref, Xd.device)
    if is_philox(rng):
        keep = sel.select(Fd, rng)
    else:
        # duck-typed RNG: rank first to know k, then draw on the host like the reference
        rank, l, _ = rank_device(Fd, n, SELECT)
        k = int((rank <= l).sum().item()) - n
        U = None
        if k >= 1:
            ref = t.from_numpy(np.asarray(v_ref, dtype=np.float64)).to(Xd.device) if v_ref is not None \
                else auto_reference(Fd)
            U = _host_draws(rng, s, m, Fd, ref)
        if U is None:
            U = t.zeros((s, m), dtype=t.float64, device=Xd.device)  # never read: no estimation
        keep = sel.select(Fd, None, U=U)
    sel.check()
    Xn = t.empty((n, Xd.shape[1]), dtype=t.float64, device=Xd.device)
    Fn = t.empty((n, m), dtype=t.float64, device=Xd.device)
    _lib.gather_rows(Xd, keep, Xn)
    _lib.gather_rows(Fd, keep, Fn)
    return (Xn.cpu().numpy(), Fn.cpu().numpy()) if is_np else (Xn, Fn)


def exact_hype_fitness_oracle(F, v_ref, k: int, moments: bool = False):
    """Exact shared-contribution fitness by cell decomposition (hype.py:88-126; n1 <= 8, m <= 3):
    the grid of point and box coordinates makes dominance constant on every cell, so the fitness
    integral is a finite sum.  Host code (a test oracle for the Monte-Carlo estimate)."""
    import itertools

    F = np.asarray(F.cpu().numpy() if hasattr(F, "cpu") else F, dtype=np.float64)
    v_ref = np.asarray(v_ref, dtype=np.float64)
    n1, m = F.shape
    if n1 > 8 or m > 3:
        raise ValueError("oracle is limited to n1 <= 8, m <= 3")
    f_l = F.min(axis=0)
    if np.any(v_ref - f_l <= 0):
        zero = np.zeros(n1)
        return (zero, zero.copy()) if moments else zero
    alpha = shared_alpha(n1, k)
    axes = []
    for a in range(m):
        vals = np.unique(np.concatenate([[f_l[a]], F[:, a], [v_ref[a]]]))
        axes.append(vals[(vals >= f_l[a]) & (vals <= v_ref[a])])
    fitness = np.zeros(n1)
    second = np.zeros(n1)
    for cell in itertools.product(*(range(len(ax) - 1) for ax in axes)):
        lo = np.array([axes[a][cell[a]] for a in range(m)])
        hi = np.array([axes[a][cell[a] + 1] for a in range(m)])
        vol = np.prod(hi - lo)
        dom = np.all(F <= lo, axis=1)
        c = int(dom.sum())
        if c >= 1:
            fitness[dom] += vol * alpha[c - 1]
            second[dom] += vol * alpha[c - 1] ** 2
    return (fitness, second) if moments else fitness
