"""Oracle: simplex-lattice directions and neighbour tables (restates ``temo/directions.py``). Test infrastructure only."""

from __future__ import annotations

import itertools
import math

import numpy as np


def simplex_lattice(m, H):
    """directions.py:64-82: compositions of H in itertools.combinations order, last column 1-sum."""
    rows = []
    for cuts in itertools.combinations(range(H + m - 1), m - 1):
        parts, prev = [], -1
        for c in cuts:
            parts.append(c - prev - 1)
            prev = c
        parts.append(H + m - 2 - prev)
        rows.append(parts)
    W = np.asarray(rows, dtype=np.float64) / H
    W[:, -1] = 1.0 - W[:, :-1].sum(axis=1)
    return W


def largest_h_for(count, m):
    """directions.py:94-101."""
    h = 1
    while math.comb(h + 1 + m - 1, m - 1) <= count:
        h += 1
    return h


def neighbors(W, T):
    """directions.py:104-114: T nearest rows by sqrt(sum diff^2), stable ties."""
    W = np.asarray(W, dtype=np.float64)
    diff = W[:, None, :] - W[None, :, :]
    dist = np.sqrt(np.sum(diff * diff, axis=-1))
    return np.argsort(dist, axis=1, kind="stable")[:, :T].astype(np.int64)
