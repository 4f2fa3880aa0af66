"""RVEA angle-penalized-distance selection on the GPU -- drop-in for ``temo.rvea`` (rvea.py:1-68).

``apd_select`` keeps one elite per non-empty direction partition (smallest APD, ties to the
lower row), in direction order, like the reference; ``RveaSelector`` is the device-resident
form the harness uses (population size = number of non-empty partitions, read back each
generation).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _lib
from .directions import DirectionSet


@dataclass(frozen=True)
class ApdParams:
    """Penalty growth exponent and generation progress t / t_max (rvea.py:19-30)."""

    alpha: float
    t: int
    t_max: int

    def __post_init__(self):
        if self.alpha <= 0:
            raise ValueError("alpha must be positive")
        if self.t_max < 1 or not 0 <= self.t <= self.t_max:
            raise ValueError("need 0 <= t <= t_max with t_max >= 1")

    @property
    def mp_factor(self) -> float:
        return (self.t / self.t_max) ** self.alpha  # rvea.py:59, host float like the reference


class RveaSelector:
    """Prepared directions (unit vectors, minimal angles) + workspace for apd_select on the device."""

    def __init__(self, N_max: int, m: int, V: DirectionSet, alpha: float = 2.0, dev=None):
        t = _lib.torch()
        self.dev = _lib.device(dev)
        self.m, self.alpha = m, float(alpha)
        self.r = V.count
        W = t.from_numpy(np.ascontiguousarray(V.W, dtype=np.float64)).to(self.dev)
        self.Vn = t.empty_like(W)
        self.gamma = t.empty(self.r, dtype=t.float64, device=self.dev)
        rc = _lib.lib().temo_rvea_prep(_lib.ptr(W), self.r, m, _lib.ptr(self.Vn), _lib.ptr(self.gamma),
                                       _lib.stream_handle(self.dev))
        _lib.check(rc, "apd_select")
        self.keep = t.empty(self.r, dtype=t.int32, device=self.dev)
        self.count = t.zeros(1, dtype=t.int32, device=self.dev)
        self.count_host = t.zeros(1, dtype=t.int32).pin_memory()
        self.status = t.zeros(1, dtype=t.int32, device=self.dev)
        self.N_max = N_max

    def select(self, F, t_gen: int, t_max: int, N: int | None = None):
        """Winners of F[:N] (device int32 tensor of length count); count read back to the host."""
        params = ApdParams(self.alpha, t_gen, t_max)
        N = F.shape[0] if N is None else N
        L = _lib.lib()
        ws = _lib.workspace.get(L.temo_rvea_select_ws_bytes(N, self.m, self.r), self.dev)
        rc = L.temo_rvea_select(_lib.ptr(F), N, self.m, _lib.ptr(self.Vn), _lib.ptr(self.gamma), self.r,
                                self.m * params.mp_factor, _lib.ptr(self.keep), _lib.ptr(self.count), None, None,
                                _lib.ptr(ws), ws.numel(), _lib.stream_handle(self.dev))
        _lib.check(rc, "apd_select")
        self.count_host.copy_(self.count)
        k = int(self.count_host.item())
        return self.keep[:k]

    def check(self):
        _lib.sync_status(self.status, "apd_select")


def apd_select(X, F, V: DirectionSet, params: ApdParams):
    """One elite per non-empty direction partition, by smallest APD (rvea.py:33-68)."""
    t = _lib.torch()
    is_np = not isinstance(F, t.Tensor)
    Fd, _ = _lib.as_device(F, t.float64)
    Xd, _ = _lib.as_device(X, t.float64, Fd.device)
    n, m = Fd.shape
    sel = RveaSelector(n, m, V, params.alpha, Fd.device)
    L = _lib.lib()
    ws = _lib.workspace.get(L.temo_rvea_select_ws_bytes(n, m, sel.r), Fd.device)
    rc = L.temo_rvea_select(_lib.ptr(Fd), n, m, _lib.ptr(sel.Vn), _lib.ptr(sel.gamma), sel.r,
                            m * params.mp_factor, _lib.ptr(sel.keep), _lib.ptr(sel.count), None, None,
                            _lib.ptr(ws), ws.numel(), _lib.stream_handle(Fd.device))
    _lib.check(rc, "apd_select")
    k = int(sel.count.item())
    keep = sel.keep[:k].long()
    Xn, Fn = Xd.index_select(0, keep), Fd.index_select(0, keep)
    return (Xn.cpu().numpy(), Fn.cpu().numpy()) if is_np else (Xn, Fn)
