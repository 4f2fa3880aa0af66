"""Oracle: NSGA-III environmental selection (restates ``temo/nsga3.py``). Test infrastructure only.

Where the reference calls BLAS/LAPACK (``Fp @ W.T`` at nsga3.py:108 and
``np.linalg.solve`` at nsga3.py:86) the oracle uses the C restatements in
``oracle/csrc/oracle.c`` so its bits do not depend on the
OpenBLAS core of the host.  The rank/condition gate (nsga3.py:85) only needs
the same *decision* and uses NumPy's SVD.
"""

from __future__ import annotations

import numpy as np

from . import _clib
from .ndsort import rank_assign

BIG = np.finfo(np.float64).max  # tensorops.py:18
ASF_EPS = 1e-6                  # nsga3.py:21
COND_LIMIT = 1e8                # nsga3.py:22
INTERCEPT_FLOOR = 1e-10         # nsga3.py:23


def solve_ones(E: np.ndarray):
    """``np.linalg.solve(E, ones(m))`` restated as the App. A4 LU (None if singular)."""
    E = _clib.c_double(E)
    m = E.shape[0]
    y = np.empty(m)
    if _clib.lib().orc_lu_solve(_clib.ptr(E), m, _clib.ptr(y)) != 0:
        return None
    return y


def normalize(F):
    """Ideal shift + hyperplane intercepts (nsga3.py:61-93). Returns (Fp, ideal, intercepts, E_rows)."""
    A = np.asarray(F, dtype=np.float64)
    m = A.shape[1]
    if np.isnan(A).all(axis=0).any():  # nsga3.py:77-78
        raise ValueError("all-NaN objective column")
    ideal = np.nanmin(A, axis=0)
    shifted = A - ideal
    asf_w = np.maximum(np.eye(m), ASF_EPS)
    extreme = np.zeros(m, dtype=np.int64)
    for axis in range(m):
        asf = (shifted / asf_w[axis]).max(axis=1)
        extreme[axis] = np.argmin(np.where(np.isnan(asf), BIG, asf))
    E = shifted[extreme]
    icpt = None
    if np.linalg.matrix_rank(E) == m and np.linalg.cond(E) <= COND_LIMIT:  # nsga3.py:85
        plane = solve_ones(E)
        if plane is not None:
            with np.errstate(divide="ignore"):
                cand = 1.0 / plane
            if (cand > INTERCEPT_FLOOR).all():
                icpt = cand
    if icpt is None:  # nsga3.py:92 (unshifted masked max)
        icpt = np.maximum(np.nanmax(A, axis=0), INTERCEPT_FLOOR)
    return shifted / icpt, ideal, icpt, extreme


def associate(Fp, W):
    """Perpendicular-nearest direction (nsga3.py:96-116). Returns (pi int64, dist f64)."""
    Fp = _clib.c_double(Fp)
    W = _clib.c_double(W)
    N, m = Fp.shape
    pi = np.empty(N, dtype=np.int64)
    dist = np.empty(N)
    _clib.lib().orc_associate(_clib.ptr(Fp), N, m, _clib.ptr(W), W.shape[0],
                              _clib.ptr(pi), _clib.ptr(dist))
    return pi, dist


def niche_counts(r, pi, l, n_r):
    """(rho, rho_l, n_s) per nsga3.py:119-123."""
    r = np.asarray(r)
    pi = np.asarray(pi)
    rho = np.bincount(pi[r < l], minlength=n_r)
    rho_l = np.bincount(pi[r == l], minlength=n_r)
    return rho, rho_l, int(rho.sum())


def niche_select(rho, n_s, r, pi, dist, l):
    """Batched niche fill (nsga3.py:126-167). Returns (rank, promoted, n_selected).

    Each round: for every direction still empty, its (dist, index)-smallest
    rank-l candidate is promoted to l-1; rounds repeat until none claims.
    """
    rank = np.array(r, dtype=np.int64, copy=True)
    occ = np.array(rho, copy=True)
    pi = np.asarray(pi)
    dist = np.asarray(dist)
    promoted = []
    while True:
        cand = np.flatnonzero(rank == l)
        if cand.size == 0:
            break
        order = np.lexsort((cand, dist[cand], pi[cand]))
        dirs = pi[cand][order]
        head = np.ones(dirs.size, dtype=bool)
        head[1:] = dirs[1:] != dirs[:-1]
        claim_dir = dirs[head]
        claim_row = cand[order][head]
        ok = occ[claim_dir] == 0
        claim_dir, claim_row = claim_dir[ok], claim_row[ok]
        if claim_row.size == 0:
            break
        # one candidate has one direction, so claims are unique (nsga3.py:160-162)
        rank[claim_row] = l - 1
        occ[claim_dir] += 1
        promoted.extend(claim_row.tolist())
    return rank, np.asarray(promoted, dtype=np.int64), n_s + len(promoted)


def update_rank(rank, promoted, n_dif, l):
    """Count repair (nsga3.py:170-183)."""
    out = np.array(rank, dtype=np.int64, copy=True)
    promoted = np.asarray(promoted, dtype=np.int64)
    if n_dif > 0:
        rest = np.flatnonzero(out == l)
        if rest.size < n_dif:
            raise RuntimeError("not enough last-front rows")
        out[rest[:n_dif]] = l - 1
    elif n_dif < 0:
        if promoted.size < -n_dif:
            raise RuntimeError("demotion exceeds promotions")
        out[promoted[promoted.size + n_dif:]] = l
    return out


def select_shuffled(Fs, W, n, rank_fn=rank_assign):
    """The selection pipeline on already-shuffled objectives (nsga3.py:207-218).

    Returns a dict of every intermediate; ``keep`` are indices into Fs.
    """
    Fs = np.asarray(Fs, dtype=np.float64)
    r, l = rank_fn(Fs, n)
    masked = Fs.copy()
    masked[r > l] = np.nan
    Fp, ideal, icpt, extreme = normalize(masked)
    pi, dist = associate(Fp, W)
    rho, rho_l, n_s = niche_counts(r, pi, l, W.shape[0])
    rank, promoted, n_sel = niche_select(rho, n_s, r, pi, dist, l)
    rank = update_rank(rank, promoted, n - n_sel, l)
    keep = np.flatnonzero(rank < l)
    if keep.size != n:
        raise RuntimeError(f"selected {keep.size} rows, wanted {n}")
    return dict(r=r, l=l, Fp=Fp, ideal=ideal, intercepts=icpt, extreme=extreme, pi=pi,
                dist=dist, rho=rho, rho_l=rho_l, promoted=promoted, rank=rank, keep=keep)


def environmental_selection(X, F, W, n, rng, rank_fn=rank_assign):
    """nsga3.py:186-218: shuffle by ``rng.permutation(N)`` then select n rows."""
    X = np.asarray(X, dtype=np.float64)
    F = np.asarray(F, dtype=np.float64)
    N = X.shape[0]
    if F.shape[0] != N or N < n:
        raise ValueError("X/F row mismatch or fewer than n rows")
    perm = rng.permutation(N)
    out = select_shuffled(F[perm], W, n, rank_fn)
    keep = out["keep"]
    return X[perm][keep], F[perm][keep]
