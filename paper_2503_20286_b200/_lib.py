"""ctypes binding of the C ABI (``include/temo_b200.h``) and the host-side plumbing.

PyTorch is used only for device memory, streams and (multi-GPU) process
groups.  There is no CPU fallback: if ``libtemo_b200.so`` cannot be loaded or
built, or no CUDA device is visible, every hot-path call raises.
"""

from __future__ import annotations

import ctypes
import os
import threading
from pathlib import Path

import numpy as np

from . import build as _build

_P = ctypes.c_void_p
_I64 = ctypes.c_int64
_I32 = ctypes.c_int
_SZ = ctypes.c_size_t
_D = ctypes.c_double
_U64 = ctypes.c_uint64


def sptr(struct):
    """Address of a ctypes Structure as a void* argument (valid for the call)."""
    return _P(ctypes.addressof(struct))

# name -> (restype, argtypes); must mirror include/temo_b200.h
SIGNATURES = {
    "temo_abi_version": (_I32, []),
    "temo_strerror": (ctypes.c_char_p, [_I32]),
    "temo_rank_ws_bytes": (_SZ, [_I64, _I32]),
    "temo_rank": (_I32, [_P, _I64, _I32, _I64, _I32, _P, _P, _P, _P, _P, _SZ, _P]),
    "temo_rank_force_bitmap": (None, [_I32]),
    "temo_host_permutation": (_I32, [_P, _I64, _P]),
    "temo_stair_prof_enable": (None, [_I32]),
    "temo_stair_prof_read": (_I32, [_P, _I64]),
    "temo_dominance_ws_bytes": (_SZ, [_I64, _I32]),
    "temo_dominance": (_I32, [_P, _I64, _I32, _P, _P, _P, _SZ, _P]),
    "temo_rank_shard_bounds": (None, [_I64, _I32, _P]),
    "temo_rank_shard_ws_bytes": (_SZ, [_I64, _I32, _I64, _I64]),
    "temo_rank_shard_build": (_I32, [_P, _I64, _I32, _I64, _I64, _P, _P, _SZ, _P]),
    "temo_rank_shard_detect": (_I32, [_I64, _I32, _I64, _I64, _P, _P, _P, _SZ, _P]),
    "temo_rank_shard_apply": (_I32, [_I64, _I32, _I64, _I64, _P, _I32, _P, _P, _SZ, _P]),
    "temo_rank_shard_finish": (_I32, [_I64, _I32, _I64, _I64, _P, _P, _P, _SZ, _P]),
    "temo_nsga3_select_ws_bytes": (_SZ, [_I64, _I32, _I64]),
    "temo_nsga3_select": (_I32, [_P, _I64, _I32, _P, _I64, _I32, _I64, _P, _P, _P, _P, _P, _P, _P, _P,
                                 _P, _P, _P, _P, _P, _P, _P, _SZ, _P]),
    "temo_nsga3_normalize": (_I32, [_P, _I64, _I32, _P, _P, _P, _P, _P, _SZ, _P]),
    "temo_associate": (_I32, [_P, _I64, _I32, _P, _I64, _I32, _P, _P, _P, _SZ, _P]),
    "temo_niche_counts": (_I32, [_P, _P, _I64, _I32, _I64, _P, _P, _P, _SZ, _P]),
    "temo_niche_select": (_I32, [_P, _P, _P, _I64, _I32, _P, _I64, _P, _P, _P, _SZ, _P]),
    "temo_update_rank": (_I32, [_P, _I64, _P, _I64, _I64, _I32, _P, _P, _SZ, _P]),
    "temo_gather_rows": (_I32, [_P, _P, _P, _I64, _I64, _P, _P]),
    "temo_lu_solve_batch": (_I32, [_P, _P, _P, _I64, _P, _P, _P, _P]),
    "temo_rvea_prep": (_I32, [_P, _I64, _I32, _P, _P, _P]),
    "temo_rvea_select_ws_bytes": (_SZ, [_I64, _I32, _I64]),
    "temo_rvea_select": (_I32, [_P, _I64, _I32, _P, _P, _I64, _D, _P, _P, _P, _P, _P, _SZ, _P]),
    "temo_igd_ws_bytes": (_SZ, [_I64]),
    "temo_igd": (_I32, [_P, _I64, _I32, _P, _I64, _P, _P, _SZ, _P]),
    "temo_hv_ws_bytes": (_SZ, [_I64, _I32]),
    "temo_hv": (_I32, [_P, _I64, _I32, _P, _P, _P, _SZ, _P]),
    "temo_hv_mc_hits": (_I32, [_P, _I64, _I32, _P, _I64, _P, _P]),
    "temo_eu_ws_bytes": (_SZ, [_I64, _I64, _I32]),
    "temo_eu": (_I32, [_P, _I64, _I32, _P, _I64, _I32, _P, _P, _SZ, _P]),
    "temo_gather_rows2": (_I32, [_P, _P, _P, _I64, _I64, _P, _P]),
    "temo_neighbors": (_I32, [_P, _I64, _I32, _I32, _P, _P]),
    "temo_evaluate": (_I32, [_P, _P, _I64, _P, _P]),
    "temo_evaluate_rows": (_I32, [_P, _P, _P, _I64, _P, _P]),
    "temo_uniform": (_I32, [_P, _U64, _I64, _P, _P]),
    "temo_sbx_beta": (_I32, [_P, _I64, _D, _I32, _P, _P]),
    "temo_sbx": (_I32, [_P, _P, _P, _I64, _I64, _P, _U64, _P, _P, _P, _P, _P]),
    "temo_pm": (_I32, [_P, _P, _I64, _I64, _P, _U64, _P, _P, _P, _P]),
    "temo_offspring": (_I32, [_P, _P, _P, _P, _P, _I64, _P, _U64, _P, _P, _P]),
    "temo_offspring_ws_bytes": (_SZ, [_I64, _I64]),
    "temo_offspring_ws": (_I32, [_P, _P, _P, _P, _P, _I64, _P, _U64, _P, _P, _P, _P, _P, _SZ, _P]),
    "temo_offspring_two_phase": (_I32, [_I64, _I64]),
    "temo_offspring_rand_ws": (_I32, [_P, _I64, _I64, _I64, _I64, _P, _U64, _P, _SZ, _P]),
    "temo_offspring_apply_ws": (_I32, [_P, _P, _P, _P, _P, _I64, _I64, _I64, _P, _U64, _P, _P, _P, _P, _P, _SZ, _P]),
    "temo_offspring_ws_range": (_I32, [_P, _P, _P, _P, _P, _I64, _I64, _I64, _P, _U64, _P, _P, _P, _P, _P, _SZ,
                                       _P]),
    "temo_pool_update_ws_bytes": (_SZ, [_I64]),
    "temo_pool_update": (_I32, [_P, _P, _P, _I64, _I64, _P, _P, _P, _SZ, _P]),
    "temo_init_population": (_I32, [_P, _U64, _I64, _I64, _P, _P, _P, _P]),
    "temo_moead_offspring_dev": (_I32, [_P, _P, _P, _P, _P, _I64, _P, _U64, _P, _P, _P]),
    "temo_moead_offspring": (_I32, [_P, _P, _P, _P, _P, _I64, _P, _U64, _P, _P, _P]),
    "temo_moead_compare": (_I32, [_P, _P, _P, _P, _I64, _I32, _I32, _P, _D, _I32, _P, _P, _P, _P]),
    "temo_moead_elite": (_I32, [_P, _P, _P, _P, _P, _I64, _I64, _I32, _I32, _P, _D, _I32, _P, _P, _P,
                                _P, _P, _P, _P, _P]),
    "temo_aggregate_rows": (_I32, [_P, _P, _P, _I64, _I32, _D, _I32, _I32, _P, _P]),
    "temo_hype_alpha": (_I32, [_I64, _I64, _P, _P]),
    "temo_auto_reference": (_I32, [_P, _I64, _I32, _P, _P, _P]),
    "temo_hv_estimate_ws_bytes": (_SZ, [_I64, _I32, _I64]),
    "temo_hv_estimate": (_I32, [_P, _I64, _I32, _P, _I64, _I64, _P, _U64, _P, _P, _P, _P, _SZ, _P]),
    "temo_hype_select_ws_bytes": (_SZ, [_I64, _I32, _I64]),
    "temo_hype_columns": (_I64, [_I64]),
    "temo_hype_select_begin": (_I32, [_P, _I64, _I32, _I64, _I64, _P, _P, _P, _P, _SZ, _P]),
    "temo_hype_select_columns": (_I32, [_P, _I64, _I32, _I64, _I64, _I64, _P, _U64, _P, _P, _P, _SZ, _P]),
    "temo_hype_select_end": (_I32, [_P, _I64, _I32, _I64, _I64, _P, _P, _P, _P, _P, _P, _P, _SZ, _P]),
    "temo_hype_select": (_I32, [_P, _I64, _I32, _I64, _I64, _P, _P, _P, _P, _U64, _P, _P, _P, _P, _P,
                                _SZ, _P]),
    "temo_probe_philox_rate": (_D, [_I32, _I32, _P, _P]),
    "temo_probe_packed_rate": (_D, [_I32, _I32, _P, _P]),
    "temo_probe_dsub_rate": (_D, [_I32, _I32, _P, _P]),
    "temo_probe_rows_rate": (_D, [_P, _P, _P, _P, _P, _I64, _I64, _P, _I32, _P]),
    "temo_timing_enable": (None, [_I32]),
    "temo_timing_name": (ctypes.c_char_p, [_I32]),
    "temo_timing_read": (_I32, [_P, _P, _I32]),
}
STAGE_COUNT = 16

TEMO_OK, TEMO_EINVAL, TEMO_ENAN, TEMO_ERUNTIME, TEMO_EWORKSPACE, TEMO_ECUDA = range(6)
ST_NAN, ST_PEEL, ST_FILL, ST_DEMOTE, ST_COUNT, ST_KRANGE = 1, 2, 4, 8, 16, 32

_lock = threading.Lock()
_handle = None


class TemoError(RuntimeError):
    pass


def lib_path() -> Path:
    return _build.LIB


def lib():
    """Load (building first if the in-tree .so is missing or stale) the CUDA library."""
    global _handle
    if _handle is not None:
        return _handle
    with _lock:
        if _handle is None:
            path = _build.LIB
            override = os.environ.get("TEMO_LIB")  # A/B experiments: an alternative build of the library
            if override:
                path = Path(override).resolve()
            elif not _build.up_to_date() and os.environ.get("TEMO_NO_BUILD") != "1":
                _build.build()
            if not path.exists():
                raise TemoError(f"CUDA library missing: {path} (run __graft_entry__.build())")
            h = ctypes.CDLL(str(path))
            for name, (res, args) in SIGNATURES.items():
                fn = getattr(h, name)
                fn.restype = res
                fn.argtypes = args
            _handle = h
    return _handle


def check(rc: int, what: str):
    if rc == TEMO_OK:
        return
    msg = lib().temo_strerror(rc).decode()
    if rc in (TEMO_EINVAL, TEMO_ENAN):
        raise ValueError(f"{what}: {msg}")
    if rc == TEMO_ERUNTIME:
        raise RuntimeError(f"{what}: {msg}")
    raise TemoError(f"{what}: {msg} (code {rc})")


def raise_status(bits: int, what: str):
    """Map device status bits to the reference's exceptions."""
    if not bits:
        return
    if bits & ST_NAN:
        raise ValueError(f"{what}: objective matrix contains NaN rows")
    if bits & ST_KRANGE:
        raise ValueError(f"{what}: k out of range")
    if bits & ST_PEEL:
        raise RuntimeError(f"{what}: front peeling failed to terminate")
    if bits & ST_FILL:
        raise RuntimeError(f"{what}: not enough last-front rows to reach n")
    if bits & ST_DEMOTE:
        raise RuntimeError(f"{what}: cannot demote more rows than were promoted")
    if bits & ST_COUNT:
        raise RuntimeError(f"{what}: selection produced the wrong number of rows")
    raise RuntimeError(f"{what}: device status {bits:#x}")


# ------------------------------------------------------------------ torch plumbing
def torch():
    import torch as _t

    return _t


def device(dev=None):
    t = torch()
    if not t.cuda.is_available():
        raise TemoError("no CUDA device: the temo_b200 hot path has no CPU fallback")
    if dev is None:
        return t.device("cuda", t.cuda.current_device())
    return t.device(dev)


def stream_handle(dev=None):
    t = torch()
    return _P(t.cuda.current_stream(dev).cuda_stream)


def ptr(x):
    if x is None:
        return None
    return _P(x.data_ptr())


class _Workspace:
    """Per-device grow-only scratch buffer handed to the C ABI."""

    def __init__(self):
        self.bufs = {}

    def get(self, nbytes: int, dev):
        t = torch()
        key = (str(dev), threading.get_ident())
        buf = self.bufs.get(key)
        if buf is None or buf.numel() < nbytes:
            self.bufs[key] = None
            buf = t.empty(max(int(nbytes), 256), dtype=t.uint8, device=dev)
            self.bufs[key] = buf
        return buf

    def release(self):
        self.bufs.clear()


workspace = _Workspace()


def as_device(x, dtype, dev=None):
    """numpy/tensor -> contiguous CUDA tensor of ``dtype``; returns (tensor, was_numpy)."""
    t = torch()
    if isinstance(x, t.Tensor):
        d = x.device if x.is_cuda else device(dev)
        return x.to(device=d, dtype=dtype).contiguous(), False
    arr = np.ascontiguousarray(np.asarray(x), dtype=_np_dtype(dtype))
    return t.from_numpy(arr).to(device(dev), non_blocking=False), True


def _np_dtype(tdtype):
    t = torch()
    return {t.float64: np.float64, t.int64: np.int64, t.int32: np.int32,
            t.uint8: np.uint8, t.uint32: np.uint32}[tdtype]


def new_status(dev):
    t = torch()
    return t.zeros(1, dtype=t.int32, device=dev)


def sync_status(status, what):
    bits = int(status.item())
    raise_status(bits, what)


def timing_enable(on: bool = True):
    lib().temo_timing_enable(1 if on else 0)


def timing_read(reset: bool = True) -> dict:
    """{stage name: (ms, calls)} accumulated since the last reset (syncs the events)."""
    ms = np.zeros(STAGE_COUNT, dtype=np.float64)
    calls = np.zeros(STAGE_COUNT, dtype=np.int64)
    L = lib()
    L.temo_timing_read(_P(ms.ctypes.data), _P(calls.ctypes.data), 1 if reset else 0)
    return {L.temo_timing_name(i).decode(): (float(ms[i]), int(calls[i]))
            for i in range(STAGE_COUNT) if calls[i]}


def gather_rows(src, idx, dst):
    """dst[r] = src[idx[r]] on the device (int32 or int64 idx)."""
    t = torch()
    rows, cols = dst.shape[0], src.shape[1]
    i32 = idx if idx.dtype == t.int32 else None
    i64 = idx if idx.dtype == t.int64 else None
    check(lib().temo_gather_rows(ptr(src), ptr(i32), ptr(i64), rows, cols, ptr(dst),
                                 stream_handle(dst.device)), "gather_rows")
    return dst


def gather_rows2(src, idx_a, idx_b, dst):
    """dst[r] = src[idx_a[idx_b[r]]] (idx_a int64, idx_b int32)."""
    rows, cols = dst.shape[0], src.shape[1]
    check(lib().temo_gather_rows2(ptr(src), ptr(idx_a), ptr(idx_b), rows, cols, ptr(dst),
                                  stream_handle(dst.device)), "gather_rows2")
    return dst


class HostRing:
    """Pinned host staging buffers for per-step H2D uploads (no host/GPU serialisation)."""

    def __init__(self, slots: int = 4):
        self.slots = slots
        self.bufs = {}
        self.next = {}

    def upload(self, arr: np.ndarray, dst):
        t = torch()
        arr = np.ascontiguousarray(arr)
        key = (arr.dtype.str, arr.size)
        ring = self.bufs.setdefault(key, [None] * self.slots)
        k = self.next.get(key, 0)
        self.next[key] = (k + 1) % self.slots
        slot = ring[k]
        if slot is None:
            host = t.from_numpy(np.empty(arr.shape, dtype=arr.dtype)).pin_memory()
            slot = ring[k] = [host, t.cuda.Event()]
        else:
            slot[1].synchronize()  # previous copy out of this slot has finished
        host, ev = slot
        host.numpy().reshape(-1)[:] = arr.reshape(-1)
        dst.view(-1).copy_(host.view(-1), non_blocking=True)
        ev.record(t.cuda.current_stream(dst.device))
        return dst
