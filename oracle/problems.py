"""Oracle: DTLZ1-7 (restates ``temo/problems.py``) and LSMOP1-9 (self-oracle). Test infrastructure only.

DTLZ parity vs the reference is by tolerance (1e-5 rel, BASELINE north star):
NumPy's vectorised cos/sin/pow and CUDA's differ in the last ulp.

LSMOP1-9 have no reference implementation (problems.py:18): this is a
NumPy restatement of the standard definitions (Cheng et al. 2017, cited at
PAPER.md:518) in the PlatEMO formulation -- *parity unpinned*.
"""

from __future__ import annotations

import numpy as np

DTLZ = ("dtlz1", "dtlz2", "dtlz3", "dtlz4", "dtlz5", "dtlz6", "dtlz7")


def _rastrigin_g(xm):
    """problems.py:69-71."""
    z = xm - 0.5
    return 100.0 * (xm.shape[1] + np.sum(z * z - np.cos(20.0 * np.pi * z), axis=1))


def _sphere_g(xm):
    """problems.py:74-76."""
    z = xm - 0.5
    return np.sum(z * z, axis=1)


def _linear_front(pos, g, scale=0.5):
    """problems.py:79-89 (scale 0.5 for DTLZ1)."""
    n, m1 = pos.shape
    m = m1 + 1
    out = np.empty((n, m))
    for i in range(m):
        p = np.prod(pos[:, : m - 1 - i], axis=1)
        if i:
            p = p * (1.0 - pos[:, m - 1 - i])
        out[:, i] = scale * (1.0 + g) * p
    return out


def _sphere_front(theta, g):
    """problems.py:92-102."""
    n, m1 = theta.shape
    m = m1 + 1
    out = np.empty((n, m))
    for i in range(m):
        p = np.prod(np.cos(theta[:, : m - 1 - i]), axis=1)
        if i:
            p = p * np.sin(theta[:, m - 1 - i])
        out[:, i] = (1.0 + g) * p
    return out


def evaluate_dtlz(name, X, m):
    """problems.py:105-136."""
    X = np.asarray(X, dtype=np.float64)
    pos, xm = X[:, : m - 1], X[:, m - 1:]
    if name == "dtlz1":
        return _linear_front(pos, _rastrigin_g(xm))
    if name == "dtlz2":
        return _sphere_front(pos * (np.pi / 2.0), _sphere_g(xm))
    if name == "dtlz3":
        return _sphere_front(pos * (np.pi / 2.0), _rastrigin_g(xm))
    if name == "dtlz4":
        return _sphere_front(np.power(pos, 100.0) * (np.pi / 2.0), _sphere_g(xm))
    if name in ("dtlz5", "dtlz6"):
        g = _sphere_g(xm) if name == "dtlz5" else np.sum(np.power(xm, 0.1), axis=1)
        theta = np.empty_like(pos)
        theta[:, 0] = pos[:, 0] * (np.pi / 2.0)
        if m > 2:
            bend = np.pi / (4.0 * (1.0 + g))[:, None]
            theta[:, 1:] = bend * (1.0 + 2.0 * g[:, None] * pos[:, 1:])
        return _sphere_front(theta, g)
    if name == "dtlz7":
        k = X.shape[1] - m + 1
        g = 1.0 + 9.0 / k * np.sum(xm, axis=1)
        out = np.empty((X.shape[0], m))
        out[:, : m - 1] = pos
        h = m - np.sum(pos / (1.0 + g)[:, None] * (1.0 + np.sin(3.0 * np.pi * pos)), axis=1)
        out[:, m - 1] = (1.0 + g) * h
        return out
    raise ValueError(name)


def lsmop_groups(m, d, nk=5):
    """Chaotic subcomponent sizes: c_{j+1} = 3.8 c_j (1 - c_j), c_1 = 3.8*0.1*0.9.

    Returns (sublen[m], offset[m+1]) where objective i's nk segments start at
    column (m-1) + offset[i] + j*sublen[i].
    """
    c = [3.8 * 0.1 * (1.0 - 0.1)]
    for _ in range(m - 1):
        c.append(3.8 * c[-1] * (1.0 - c[-1]))
    c = np.asarray(c)
    sublen = np.floor(c / c.sum() * (d - m + 1) / nk).astype(np.int64)
    offset = np.concatenate([[0], np.cumsum(sublen * nk)])
    return sublen, offset


def lsmop_dimension(m, d_request, nk=5):
    """PlatEMO resets D = M - 1 + len(end) after sizing the subcomponents from the request."""
    sublen, offset = lsmop_groups(m, d_request, nk)
    return m - 1 + int(offset[m])


def lsmop_groups_for(m, D, nk=5):
    """Groups of the instance with D variables (D determines them: floors are monotone in the request)."""
    for d0 in range(D, D + nk * m + 2):
        if lsmop_dimension(m, d0, nk) == D:
            return lsmop_groups(m, d0, nk)
    raise ValueError(f"{D} is not an LSMOP dimension for m={m}")


def lsmop_bounds(m, d):
    lower = np.zeros(d)
    upper = np.concatenate([np.ones(m - 1), np.full(d - m + 1, 10.0)])
    return lower, upper


def evaluate_lsmop1(X, m, nk=5):
    """LSMOP1: linear linkage, Sphere g on every group, linear (DTLZ1-type) front."""
    X = np.asarray(X, dtype=np.float64)
    n, d = X.shape
    sublen, offset = lsmop_groups_for(m, d, nk)
    idx = np.arange(m, d + 1, dtype=np.float64)  # 1-based indices of x^s
    xs = (1.0 + idx / d) * X[:, m - 1:] - 10.0 * X[:, :1]
    G = np.zeros((n, m))
    for i in range(m):
        for j in range(nk):
            a = offset[i] + j * sublen[i]
            seg = xs[:, a:a + sublen[i]]
            G[:, i] = G[:, i] + np.sum(seg * seg, axis=1)
    G = G / sublen / nk
    ones = np.ones((n, 1))
    head = np.cumprod(np.concatenate([ones, X[:, : m - 1]], axis=1), axis=1)[:, ::-1]
    tail = np.concatenate([ones, 1.0 - X[:, m - 2::-1]], axis=1) if m > 1 else ones
    return (1.0 + G) * head * tail


# LSMOP1-9 (Cheng, Jin, Olhofer, Sendhoff 2017, "Test problems for large-scale multiobjective
# and many-objective optimization", IEEE T-Cyb 47(12)), restated from the PlatEMO
# formulation (LSMOP*.m CalObj): eta1 on odd objectives, eta2 on even ones.
_ETA = {1: ("sphere", "sphere"), 2: ("griewank", "schwefel"), 3: ("rastrigin", "rosenbrock"),
        4: ("ackley", "griewank"), 5: ("sphere", "sphere"), 6: ("rosenbrock", "schwefel"),
        7: ("ackley", "rosenbrock"), 8: ("griewank", "sphere"), 9: ("sphere", "ackley")}


def _eta(fn, z):
    L = z.shape[1]
    if fn == "sphere":
        return np.sum(z ** 2, axis=1)
    if fn == "griewank":
        return np.sum(z ** 2, axis=1) / 4000.0 - np.prod(np.cos(z / np.sqrt(np.arange(1, L + 1))), axis=1) + 1.0
    if fn == "schwefel":
        return np.max(np.abs(z), axis=1)
    if fn == "rastrigin":
        return np.sum(z ** 2 - 10.0 * np.cos(2.0 * np.pi * z) + 10.0, axis=1)
    if fn == "rosenbrock":
        return np.sum(100.0 * (z[:, :-1] ** 2 - z[:, 1:]) ** 2 + (z[:, :-1] - 1.0) ** 2, axis=1)
    if fn == "ackley":
        return (20.0 - 20.0 * np.exp(-0.2 * np.sqrt(np.sum(z ** 2, axis=1) / L))
                - np.exp(np.sum(np.cos(2.0 * np.pi * z), axis=1) / L) + np.exp(1.0))
    raise ValueError(fn)


def evaluate_lsmop(k, X, m, nk=5):
    """LSMOP k: linkage (linear k <= 4, cos k >= 5), per-subcomponent eta, front linear (1-4),
    concave (5-8: (1 + G_i + G_{i+1}) cos/sin) or disconnected (9)."""
    if k == 1:
        return evaluate_lsmop1(X, m, nk)
    X = np.asarray(X, dtype=np.float64)
    n, d = X.shape
    sublen, offset = lsmop_groups_for(m, d, nk)
    idx = np.arange(m, d + 1, dtype=np.float64) / d
    c = np.cos(idx * np.pi / 2.0) if k >= 5 else idx
    xs = (1.0 + c) * X[:, m - 1:] - 10.0 * X[:, :1]
    G = np.zeros((n, m))
    for i in range(m):
        fn = _ETA[k][i % 2]
        for j in range(nk):
            a = offset[i] + j * sublen[i]
            G[:, i] = G[:, i] + _eta(fn, xs[:, a:a + sublen[i]])
    G = G / sublen / nk
    ones = np.ones((n, 1))
    if k <= 4:
        head = np.cumprod(np.concatenate([ones, X[:, : m - 1]], axis=1), axis=1)[:, ::-1]
        tail = np.concatenate([ones, 1.0 - X[:, m - 2::-1]], axis=1)
        return (1.0 + G) * head * tail
    if k <= 8:
        head = np.cumprod(np.concatenate([ones, np.cos(X[:, : m - 1] * np.pi / 2.0)], axis=1), axis=1)[:, ::-1]
        tail = np.concatenate([ones, np.sin(X[:, m - 2::-1] * np.pi / 2.0)], axis=1)
        Gn = np.concatenate([G[:, 1:], np.zeros((n, 1))], axis=1)
        return (1.0 + G + Gn) * head * tail
    Gs = 1.0 + np.sum(G, axis=1)
    F = np.empty((n, m))
    F[:, : m - 1] = X[:, : m - 1]
    F[:, m - 1] = (1.0 + Gs) * (m - np.sum(F[:, : m - 1] / (1.0 + Gs)[:, None]
                                         * (1.0 + np.sin(3.0 * np.pi * F[:, : m - 1])), axis=1))
    return F


def evaluate(name, X, m):
    if name.startswith("lsmop"):
        return evaluate_lsmop(int(name[5:]), X, m)
    return evaluate_dtlz(name, X, m)
