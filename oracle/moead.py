"""Oracle: decoupled MOEA/D generation (restates ``temo/moead.py``). Test infrastructure only.

PBI parity is pinned (moead.py:43-67 and tests/golden/moead.npz).  The
Tchebycheff aggregation g(f|w,z) = max_k w_k |f_k - z_k| (Zhang & Li 2007) has
no reference implementation (the reference is PBI-only) -- self-oracle,
*parity unpinned*; it reuses the PBI compare/elite structure unchanged.
"""

from __future__ import annotations

import numpy as np

from .variation import polynomial_mutation, sbx


def pbi(f, w, z, theta, normalize_direction=True):
    """moead.py:43-67, same elementwise op order (sums over the last axis)."""
    f = np.asarray(f, dtype=np.float64)
    w = np.asarray(w, dtype=np.float64)
    v = f - z
    wn = np.sqrt(np.sum(w * w, axis=-1))
    if np.any(wn == 0):
        raise ValueError("zero weight vector")
    d1 = np.abs(np.sum(v * w, axis=-1)) / wn
    dirv = w / wn[..., None] if normalize_direction else w
    res = v - d1[..., None] * dirv
    return d1 + theta * np.sqrt(np.sum(res * res, axis=-1))


def tchebycheff(f, w, z, theta=None):
    """max_k w_k * |f_k - z_k| (self-oracle)."""
    f = np.asarray(f, dtype=np.float64)
    w = np.asarray(w, dtype=np.float64)
    return np.max(w * np.abs(f - z), axis=-1)


def _agg(kind):
    return pbi if kind == "pbi" else tchebycheff


def compare(F1, W, I_nb, z, F2, theta, kind="pbi"):
    """moead.py:70-92 without the n x n matrix: returns (improves (n,T) bool, z_min)."""
    g = _agg(kind)
    F2 = np.asarray(F2, dtype=np.float64)
    z_min = np.minimum(z, F2.min(axis=0))
    nb_w = W[I_nb]
    g_old = g(F1[I_nb], nb_w, z_min, theta)
    g_new = g(F2[:, None, :], nb_w, z_min, theta)
    return (g_old - g_new) >= 0, z_min


def update_matrix(improves, I_nb):
    """The reference's n x n int64 I_new (moead.py:87-91)."""
    n = I_nb.shape[0]
    I_new = np.broadcast_to(np.arange(n, dtype=np.int64), (n, n)).copy()
    rows = np.repeat(np.arange(n), I_nb.shape[1])
    flat = improves.ravel()
    I_new[rows[flat], I_nb.ravel()[flat]] = -1
    return I_new


def elite_select(X, F1, W, O, F2, I_new, z_min, theta, kind="pbi", block=256):
    """moead.py:95-124 literally (O(n^2)); returns (X_next, F_next, winners, from_off)."""
    g = _agg(kind)
    n = F1.shape[0]
    winners = np.empty(n, dtype=np.int64)
    g_old = g(F1, W, z_min, theta)
    for lo in range(0, n, block):
        hi = min(lo + block, n)
        g_new = g(F2[:, None, :], W[None, lo:hi, :], z_min, theta)
        scores = np.where(I_new[:, lo:hi] == -1, g_new, g_old[None, lo:hi])
        winners[lo:hi] = np.argmin(scores, axis=0)
    from_off = I_new[winners, np.arange(n)] == -1
    X_next = np.where(from_off[:, None], O[winners], X)
    F_next = np.where(from_off[:, None], F2[winners], F1)
    return X_next, F_next, winners, from_off


def offspring(X, I_nb, rng, eta_c, eta_m, p_m, lower, upper, gene_swap=True):
    """moead.py:127-145: one child per subproblem from two distinct neighbours."""
    n, T = I_nb.shape
    if T < 2:
        raise ValueError("T must be >= 2")
    a = rng.integers(0, T, size=n)
    b = rng.integers(0, T - 1, size=n)
    b = b + (b >= a)
    rows = np.arange(n)
    kids = sbx(rng, X[I_nb[rows, a]], X[I_nb[rows, b]], eta_c, lower, upper, gene_swap)[:n]
    pm = 1.0 / X.shape[1] if p_m is None else p_m
    return polynomial_mutation(rng, kids, eta_m, pm, lower, upper)


def step(X, F1, z, W, I_nb, theta, rng, evaluate, eta_c, eta_m, p_m, lower, upper,
         kind="pbi", gene_swap=True):
    """moead.py:148-158. Returns (X_next, F_next, z_min)."""
    O = offspring(X, I_nb, rng, eta_c, eta_m, p_m, lower, upper, gene_swap)
    F2 = evaluate(O)
    improves, z_min = compare(F1, W, I_nb, z, F2, theta, kind)
    I_new = update_matrix(improves, I_nb)
    Xn, Fn, _, _ = elite_select(X, F1, W, O, F2, I_new, z_min, theta, kind)
    return Xn, Fn, z_min


def default_neighborhood(n):
    """moead.py:172-174."""
    return min(20, max(2, -(-n // 10)))
