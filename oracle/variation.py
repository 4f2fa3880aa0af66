"""Oracle: mating, SBX, polynomial mutation (restates ``temo/variation.py``). Test infrastructure only.

Op sequences follow SURVEY App. A8; uniforms come from ``rng.random`` in the
reference's call order (App. B).  Branches are selected with ``np.where`` on
both evaluated sides, as ``masked_blend`` does (tensorops.py:26-36).
"""

from __future__ import annotations

import numpy as np


def pair_parents(rng, n):
    """variation.py:48-54."""
    if n < 2:
        raise ValueError("need two or more rows to pair")
    perm = rng.permutation(n)
    h = n // 2
    return perm[:h], perm[h:2 * h]


def sbx(rng, X1, X2, eta_c, lower, upper, gene_swap=True):
    """variation.py:57-91 -> stacked [c1; c2], clipped."""
    X1 = np.asarray(X1, dtype=np.float64)
    X2 = np.asarray(X2, dtype=np.float64)
    if X1.shape != X2.shape:
        raise ValueError("parent shapes differ")
    u = rng.random(X1.shape)
    e = 1.0 / (eta_c + 1.0)
    with np.errstate(divide="ignore", invalid="ignore"):
        beta = np.where(0.5 - u >= 0, np.power(2.0 * u, e), np.power(1.0 / (2.0 - 2.0 * u), e))
    if gene_swap:
        flip = (rng.random(X1.shape) < 0.5).astype(np.float64)
        beta = beta * (1.0 - 2.0 * flip)
        cross = rng.random(X1.shape) < 0.5
        beta = np.where(cross, beta, 1.0)
    half = 0.5 * (1.0 - beta)
    c1 = X1 + half * (X2 - X1)
    c2 = X2 + half * (X1 - X2)
    return np.clip(np.concatenate([c1, c2], axis=0), lower, upper)


def polynomial_mutation(rng, X, eta_m, p_m, lower, upper):
    """variation.py:94-120 (p_m already resolved: None -> 1/d)."""
    X = np.asarray(X, dtype=np.float64)
    span = upper - lower
    eta = eta_m + 1.0
    u = rng.random(X.shape)
    hit = (p_m - rng.random(X.shape)) >= 0
    lo_gap = (X - lower) / span
    hi_gap = (upper - X) / span
    with np.errstate(invalid="ignore"):
        down = np.power(2.0 * u + (1.0 - 2.0 * u) * np.power(1.0 - lo_gap, eta), 1.0 / eta) - 1.0
        up = 1.0 - np.power(2.0 - 2.0 * u + (2.0 * u - 1.0) * np.power(1.0 - hi_gap, eta), 1.0 / eta)
    step = np.where(0.5 - u >= 0, down, up)
    moved = X + step * span
    return np.clip(np.where(hit, moved, X), lower, upper)


def offspring(rng, X, eta_c, eta_m, p_m, lower, upper, gene_swap=True):
    """harness.py:201-204: pair, SBX, PM -> (2h, d)."""
    i1, i2 = pair_parents(rng, X.shape[0])
    kids = sbx(rng, X[i1], X[i2], eta_c, lower, upper, gene_swap)
    pm = 1.0 / X.shape[1] if p_m is None else p_m
    return polynomial_mutation(rng, kids, eta_m, pm, lower, upper)
