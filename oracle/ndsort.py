"""Oracle: non-dominated sorting (restates ``temo/ndsort.py``). Test infrastructure only."""

from __future__ import annotations

import numpy as np


def _as_objectives(F) -> np.ndarray:
    A = np.asarray(F, dtype=np.float64)
    # ndsort.py:33-36 -- non-empty 2-D, no NaN
    if A.ndim != 2 or A.shape[0] < 1:
        raise ValueError("objective matrix must be 2-D with at least one row")
    if np.isnan(A).any():
        raise ValueError("NaN objective values")
    return A


def dominance_matrix(F, block: int = 2048) -> np.ndarray:
    """D[i, j] = 1 iff row i Pareto-dominates row j (ndsort.py:25-44).

    Built block-row by block-row exactly like the reference so that the CPU
    timing of the ``port`` baseline reflects the reference's memory traffic.
    """
    A = _as_objectives(F)
    N = A.shape[0]
    out = np.empty((N, N), dtype=np.int64)  # ndsort.py:38 int64 matrix
    for lo in range(0, N, block):
        rows = A[lo : lo + block, None, :]
        no_worse = (rows <= A[None]).all(axis=2)
        better_somewhere = (rows < A[None]).any(axis=2)
        out[lo : lo + block] = no_worse & better_somewhere
    return out


def rank_assign(F, n: int):
    """Peel fronts with ``c <- c - p@D - p`` (ndsort.py:47-71).

    Returns ``(r, l)``: int64 ranks (0 = first front) and the rank of the
    n-th best row, ``l = sort(r)[n-1]`` (ndsort.py:70).
    """
    A = np.asarray(F, dtype=np.float64)
    N = A.shape[0]
    if n < 1 or n > N:  # ndsort.py:56-57
        raise ValueError(f"n={n} outside [1, {N}]")
    D = dominance_matrix(A)
    count = D.sum(axis=0)
    rank = np.zeros(N, dtype=np.int64)
    front_id = 0
    front = count == 0
    while front.any():
        if front_id >= N:  # ndsort.py:64-65
            raise RuntimeError("peeling did not terminate")
        rank[front] = front_id
        count = count - front @ D - front
        front_id += 1
        front = count == 0
    last = int(np.sort(rank)[n - 1])
    return rank, last


def rank_loop(F, n: int):
    """Sequential Deb domination-count sort (ndsort.py:74-106), pure Python.

    Independent of the batched formulation above; only for small N.
    """
    A = np.asarray(F, dtype=np.float64)
    N, m = A.shape
    beats = [[] for _ in range(N)]
    beaten_by = [0] * N
    for i in range(N):
        for j in range(N):
            if i == j:
                continue
            ij_le = all(A[i, k] <= A[j, k] for k in range(m))
            ij_lt = any(A[i, k] < A[j, k] for k in range(m))
            if ij_le and ij_lt:
                beats[i].append(j)
                beaten_by[j] += 1
    rank = np.zeros(N, dtype=np.int64)
    current = [i for i in range(N) if beaten_by[i] == 0]
    k = 0
    while current:
        nxt = []
        for i in current:
            rank[i] = k
            for j in beats[i]:
                beaten_by[j] -= 1
                if beaten_by[j] == 0:
                    nxt.append(j)
        current = nxt
        k += 1
    return rank, int(np.sort(rank)[n - 1])


def rank_fast(F, n: int):
    """Exact ranks via lexicographic presort + longest-chain recursion.

    Same output as ``rank_assign`` (integer work, so any correct algorithm is
    bit-identical); O(N^2) time but O(N) memory, used by tests to check large
    CUDA sorts where the N x N int64 matrix of the reference does not fit.
    """
    A = _as_objectives(F)
    A = np.where(A == 0.0, 0.0, A)  # -0.0 == +0.0
    N = A.shape[0]
    order = np.lexsort(A.T[::-1])
    S = A[order]
    rank_sorted = np.zeros(N, dtype=np.int64)
    for j in range(1, N):
        prev = S[:j]
        le = (prev <= S[j]).all(axis=1)
        lt = (prev < S[j]).any(axis=1)
        dom = le & lt
        if dom.any():
            rank_sorted[j] = rank_sorted[:j][dom].max() + 1
    rank = np.empty(N, dtype=np.int64)
    rank[order] = rank_sorted
    if not 1 <= n <= N:
        raise ValueError(f"n={n} outside [1, {N}]")
    return rank, int(np.sort(rank)[n - 1])
