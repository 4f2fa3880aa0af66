"""Non-dominated sorting on the GPU -- drop-in for ``temo.ndsort`` (ndsort.py:17-106).

``rank_assign`` / ``dominance_matrix`` keep the reference signatures and
exceptions; NumPy inputs return NumPy outputs, CUDA tensors stay on the
device.  The work runs in ``libtemo_b200.so`` (csrc/ndsort.cu): column ranks,
triangular dominance bitmap (K1) and on-device front peeling (K2).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _lib

SORT = 0
SELECT = 1


@dataclass(frozen=True)
class RankResult:
    """Non-domination ranks (0 = best front) and the last retained rank l (ndsort.py:17-22)."""

    r: object
    l: int


def _check_objectives(F, what):
    t = _lib.torch()
    if isinstance(F, t.Tensor):
        if F.dim() != 2 or F.shape[0] < 1:
            raise ValueError(f"{what}: expected a non-empty n x m objective matrix")
        return
    A = np.asarray(F, dtype=np.float64)
    if A.ndim != 2 or A.shape[0] < 1:
        raise ValueError(f"{what}: expected a non-empty n x m objective matrix")
    if np.isnan(A).any():
        raise ValueError(f"{what}: objective matrix contains NaN rows")


def rank_device(Fd, n: int, mode: int = SORT, status=None, out=None):
    """Enqueue the GPU sort of a CUDA float64 (N, m) tensor; no host sync.

    Returns ``(rank int32[N], l int32[1], nfronts int32[1])`` device tensors
    (written into ``out`` if given).  Data-dependent errors are OR-ed into
    ``status`` (int32[1]) if given.
    """
    t = _lib.torch()
    N, m = Fd.shape
    if not 1 <= n <= N:
        raise ValueError(f"population size {n} out of range [1, {N}]")
    L = _lib.lib()
    dev = Fd.device
    if out is None:
        rank = t.empty(N, dtype=t.int32, device=dev)
        l = t.empty(1, dtype=t.int32, device=dev)
        nf = t.empty(1, dtype=t.int32, device=dev)
    else:
        rank, l, nf = out
    nbytes = L.temo_rank_ws_bytes(N, m)
    if nbytes == 0:
        raise ValueError(f"unsupported problem size N={N}, m={m}")
    ws = _lib.workspace.get(nbytes, dev)
    rc = L.temo_rank(_lib.ptr(Fd), N, m, n, mode, _lib.ptr(rank), _lib.ptr(l), _lib.ptr(nf),
                     _lib.ptr(status), _lib.ptr(ws), ws.numel(), _lib.stream_handle(dev))
    _lib.check(rc, "rank_assign")
    return rank, l, nf


def rank_assign(F, n: int) -> RankResult:
    """Ranks by front peeling and l = sort(r)[n-1] (ndsort.py:47-71)."""
    _check_objectives(F, "rank_assign")
    Fd, was_np = _lib.as_device(F, _lib.torch().float64)
    N = Fd.shape[0]
    if not 1 <= n <= N:
        raise ValueError(f"population size {n} out of range [1, {N}]")
    status = _lib.new_status(Fd.device)
    rank, l, _ = rank_device(Fd, n, SORT, status)
    _lib.sync_status(status, "rank_assign")
    r = rank.to(_lib.torch().int64)
    return RankResult(r.cpu().numpy() if was_np else r, int(l.item()))


def dominance_matrix(F, block: int = 2048):
    """N x N int64 mask, (i, j) = 1 iff row i dominates row j (ndsort.py:25-44).

    Materialised only for parity at small N (the reference's own limit);
    ``block`` is accepted for signature compatibility.
    """
    del block
    _check_objectives(F, "dominance_matrix")
    t = _lib.torch()
    Fd, was_np = _lib.as_device(F, t.float64)
    N, m = Fd.shape
    L = _lib.lib()
    Wd = (N + 31) // 32
    words = t.empty((N, Wd), dtype=t.int32, device=Fd.device)
    status = _lib.new_status(Fd.device)
    nbytes = L.temo_dominance_ws_bytes(N, m)
    ws = _lib.workspace.get(nbytes, Fd.device)
    rc = L.temo_dominance(_lib.ptr(Fd), N, m, _lib.ptr(words), _lib.ptr(status), _lib.ptr(ws),
                          ws.numel(), _lib.stream_handle(Fd.device))
    _lib.check(rc, "dominance_matrix")
    _lib.sync_status(status, "dominance_matrix")
    shifts = t.arange(32, device=Fd.device, dtype=t.int32)
    bits = (words.unsqueeze(-1) >> shifts) & 1
    D = bits.reshape(N, Wd * 32)[:, :N].to(t.int64)
    return D.cpu().numpy() if was_np else D


def ndsort_oracle(F, n: int) -> RankResult:
    """Sequential domination-count sorting (ndsort.py:74-106): the host oracle the batched sort
    must equal.  Same algorithm and front order as the reference (pairwise counts, then fronts
    peeled in list order); O(N^2) host work, meant for small N."""
    A = np.asarray(F.cpu().numpy() if hasattr(F, "cpu") else F, dtype=np.float64)
    if A.ndim != 2:
        raise ValueError("objective matrix must be 2-D")
    N, _ = A.shape
    dominated_by = np.zeros(N, dtype=np.int64)
    dominates = []
    for i in range(N):
        le_ij = (A[i] <= A).all(axis=1)
        lt_ij = (A[i] < A).any(axis=1)
        le_ji = (A <= A[i]).all(axis=1)
        lt_ji = (A < A[i]).any(axis=1)
        d_ij = le_ij & lt_ij
        d_ij[i] = False
        d_ji = le_ji & lt_ji
        d_ji[i] = False
        dominates.append(np.flatnonzero(d_ij))
        dominated_by[i] = int((d_ji & ~d_ij).sum())
    r = np.zeros(N, dtype=np.int64)
    front = [i for i in range(N) if dominated_by[i] == 0]
    k = 0
    while front:
        nxt = []
        for i in front:
            r[i] = k
            for j in dominates[i]:
                dominated_by[j] -= 1
                if dominated_by[j] == 0:
                    nxt.append(int(j))
        front = nxt
        k += 1
    if not 1 <= n <= N:
        raise ValueError(f"population size {n} out of range [1, {N}]")
    return RankResult(r, int(np.sort(r)[n - 1]))
