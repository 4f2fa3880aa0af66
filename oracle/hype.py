"""Oracle: HypE Monte-Carlo HV fitness and selection (restates ``temo/hype.py``). Test infrastructure only.

``hv_estimate`` replaces the reference's ``dominates @ weight`` (hype.py:83,
OpenBLAS dgemv_t) by the C restatement of its summation order
(``orc_hv_block``).  Pinned against reference output made with
``OPENBLAS_NUM_THREADS=1`` (tests/golden/hype.npz).
"""

from __future__ import annotations

import numpy as np

from . import _clib
from .ndsort import rank_assign

BIG = np.finfo(np.float64).max


def shared_alpha(n1: int, k: int) -> np.ndarray:
    """alpha_c = prod_{l<c} (k-l)/(n1-l) / c, zero past k (hype.py:37-51)."""
    if k < 1 or k > n1:
        raise ValueError("k outside [1, n1]")
    lam = np.ones(n1)
    if n1 > 1:
        idx = np.arange(1, n1)
        lam[1:] = (k - idx) / (n1 - idx)
    alpha = np.zeros(n1)
    alpha[:k] = np.cumprod(lam[:k]) / np.arange(1, k + 1)
    return alpha


def auto_reference(F) -> np.ndarray:
    """max + 0.1*(max - min) over all rows (hype.py:129-132)."""
    F = np.asarray(F, dtype=np.float64)
    hi = F.max(axis=0)
    return hi + 0.1 * (hi - F.min(axis=0))


def hv_estimate(F, v_ref, k, s, rng, sample_block=65536, samples=None):
    """Per-row MC hypervolume contribution (hype.py:54-85).

    ``samples``, if given, is the (s, m) uniform matrix the reference would
    draw with ``rng.random`` (blocks concatenate into one stream, App. A9);
    otherwise it is drawn from ``rng`` block by block like the reference.
    """
    F = _clib.c_double(F)
    v_ref = np.asarray(v_ref, dtype=np.float64)
    n1, m = F.shape
    if s < 1 or k < 1:
        raise ValueError("need s >= 1 and k >= 1")
    if k > n1:
        raise ValueError("k exceeds rows")
    lo = F.min(axis=0)
    span = v_ref - lo
    if (span <= 0).any():  # hype.py:72-73: no draws
        return np.zeros(n1)
    alpha = shared_alpha(n1, k)
    contrib = np.zeros(n1)
    done = 0
    lib = _clib.lib()
    while done < s:
        b = min(sample_block, s - done)
        U = rng.random((b, m)) if samples is None else samples[done:done + b]
        S = _clib.c_double(lo + U * span)
        counts = np.empty(b, dtype=np.int64)
        scratch = np.empty(n1 * b, dtype=np.uint8)
        lib.orc_hv_block(_clib.ptr(F), n1, m, _clib.ptr(S), b, _clib.ptr(alpha),
                         _clib.ptr(contrib), _clib.ptr(counts), _clib.ptr(scratch))
        done += b
    return contrib * np.prod(span) / s


def select(F, v_ref, n, s, rng, samples=None, rank_fn=rank_assign):
    """Selection core (hype.py:153-163). Returns dict with r, l, k, v_hv, keep."""
    F = np.asarray(F, dtype=np.float64)
    if F.shape[0] < n:
        raise ValueError("fewer than n rows")
    r, l = rank_fn(F, n)
    retained = r <= l
    k = int(retained.sum()) - n
    ref = None
    if k >= 1:
        ref = auto_reference(F) if v_ref is None else np.asarray(v_ref, dtype=np.float64)
        v_hv = hv_estimate(F, ref, k, s, rng, samples=samples)
    else:
        v_hv = np.zeros(F.shape[0])
    d = np.where(retained, v_hv, -BIG)
    neg = -d
    # lexsort by (r, -d, index): np.lexsort keys are least-significant first
    keep = np.lexsort((np.arange(F.shape[0]), neg, r))[:n]
    return dict(r=r, l=l, k=k, v_ref=ref, v_hv=v_hv, keep=keep)


def environmental_selection(X, F, v_ref, n, s, rng, samples=None):
    out = select(F, v_ref, n, s, rng, samples=samples)
    keep = out["keep"]
    return np.asarray(X)[keep], np.asarray(F)[keep]
