"""Quality indicators on the GPU -- drop-in for ``temo.indicators`` (indicators.py:19-100).

``igd``, ``hv_indicator`` (exact for m <= 3, Monte-Carlo above) and ``eu`` run in
``csrc/indicators.cu`` with the reference's operation order (NumPy's last-axis and pairwise
summation, OpenBLAS's dgemm FMA chain), so they return the reference's value; inputs may be
NumPy arrays or CUDA tensors, the result is a Python float.  The m > 3 hypervolume draws its
10^6 box samples on the host from the same Generator the reference uses and tests them on
the device.
"""

from __future__ import annotations

import numpy as np

from . import _lib
from .directions import DirectionSet

_MC_SAMPLES = 1_000_000


def _dev2(A):
    t = _lib.torch()
    Ad, _ = _lib.as_device(A, t.float64)
    if Ad.dim() != 2:
        raise ValueError("expected a 2-D array")
    return Ad.contiguous()


def _scalar(out):
    return float(out.item())


def igd(F, Fstar) -> float:
    """Mean distance from each reference-front point to its nearest solution (indicators.py:19-26)."""
    t = _lib.torch()
    if np.size(F) == 0 or np.size(Fstar) == 0:
        raise ValueError("igd needs non-empty inputs")
    Fd = _dev2(F)
    Sd = _dev2(Fstar).to(Fd.device)
    n, m = Fd.shape
    r = Sd.shape[0]
    out = t.empty(1, dtype=t.float64, device=Fd.device)
    L = _lib.lib()
    ws = _lib.workspace.get(L.temo_igd_ws_bytes(r), Fd.device)
    rc = L.temo_igd(_lib.ptr(Fd), n, m, _lib.ptr(Sd), r, _lib.ptr(out), _lib.ptr(ws), ws.numel(),
                    _lib.stream_handle(Fd.device))
    _lib.check(rc, "igd")
    return _scalar(out)


def hv_indicator(F, ref, rng: np.random.Generator | None = None) -> float:
    """Volume dominated by F and bounded by ``ref`` (indicators.py:49-66); exact for m <= 3."""
    t = _lib.torch()
    Fd = _dev2(F)
    ref_h = np.asarray(ref.cpu().numpy() if hasattr(ref, "cpu") else ref, dtype=np.float64)
    n, m = Fd.shape
    if n == 0:
        return 0.0
    dev = Fd.device
    L = _lib.lib()
    refd = t.from_numpy(ref_h.copy()).to(dev)
    if m in (2, 3):
        out = t.zeros(1, dtype=t.float64, device=dev)
        ws = _lib.workspace.get(L.temo_hv_ws_bytes(n, m), dev)
        rc = L.temo_hv(_lib.ptr(Fd), n, m, _lib.ptr(refd), _lib.ptr(out), _lib.ptr(ws), ws.numel(),
                       _lib.stream_handle(dev))
        _lib.check(rc, "hv_indicator")
        return _scalar(out)
    keep = (Fd < refd).all(dim=1)
    Fk = Fd[keep].contiguous()
    if Fk.shape[0] == 0:
        return 0.0
    rng = np.random.default_rng(0) if rng is None else rng
    lo = Fk.min(dim=0).values.cpu().numpy()
    span = ref_h - lo
    S = t.from_numpy(lo + rng.random((_MC_SAMPLES, m)) * span).to(dev)
    hits = t.empty(_MC_SAMPLES, dtype=t.int32, device=dev)
    rc = L.temo_hv_mc_hits(_lib.ptr(Fk), Fk.shape[0], m, _lib.ptr(S), _MC_SAMPLES, _lib.ptr(hits),
                           _lib.stream_handle(dev))
    _lib.check(rc, "hv_indicator")
    frac = float(np.mean(hits.cpu().numpy().astype(bool)))
    return float(frac * np.prod(span))


def eu(F, W, maximize: bool = False, literal: bool = False) -> float:
    """Expected utility under weight rows (indicators.py:69-100)."""
    t = _lib.torch()
    weights = W.W if isinstance(W, DirectionSet) else W
    if np.size(F) == 0 or np.size(weights) == 0:
        raise ValueError("eu needs non-empty inputs")
    Fd = _dev2(F)
    Wd = _dev2(weights).to(Fd.device)
    U = (Fd if maximize else -Fd).contiguous()
    n, m = U.shape
    r = Wd.shape[0]
    out = t.empty(1, dtype=t.float64, device=Fd.device)
    L = _lib.lib()
    ws = _lib.workspace.get(L.temo_eu_ws_bytes(n, r, 1 if literal else 0), Fd.device)
    rc = L.temo_eu(_lib.ptr(U), n, m, _lib.ptr(Wd), r, 1 if literal else 0, _lib.ptr(out), _lib.ptr(ws),
                   ws.numel(), _lib.stream_handle(Fd.device))
    _lib.check(rc, "eu")
    return _scalar(out)
