"""Build + load the oracle's C helpers (oracle/csrc/oracle.c). Test infrastructure only."""

from __future__ import annotations

import ctypes
import os
import subprocess
from pathlib import Path

import numpy as np

_HERE = Path(__file__).resolve().parent
_SRC = _HERE / "csrc" / "oracle.c"
_LIB = _HERE / "_lib" / "liboracle.so"
_handle = None


def build(force: bool = False) -> Path:
    """Compile liboracle.so with FMA contraction off (explicit fma() only)."""
    if _LIB.exists() and not force and _LIB.stat().st_mtime >= _SRC.stat().st_mtime:
        return _LIB
    _LIB.parent.mkdir(parents=True, exist_ok=True)
    tmp = _LIB.with_suffix(f".{os.getpid()}.tmp")
    subprocess.check_call(
        ["gcc", "-O2", "-fPIC", "-shared", "-ffp-contract=off", "-fno-fast-math",
         str(_SRC), "-lm", "-o", str(tmp)]
    )
    os.replace(tmp, _LIB)
    return _LIB


def lib():
    global _handle
    if _handle is None:
        _handle = ctypes.CDLL(str(build()))
        P = ctypes.c_void_p
        I64 = ctypes.c_int64
        _handle.orc_associate.argtypes = [P, I64, ctypes.c_int, P, I64, P, P]
        _handle.orc_lu_solve.argtypes = [P, ctypes.c_int, P]
        _handle.orc_lu_solve.restype = ctypes.c_int
        _handle.orc_hv_block.argtypes = [P, I64, ctypes.c_int, P, I64, P, P, P, P]
        _handle.orc_fma.argtypes = [P, P, P, P, I64]
    return _handle


def ptr(a: np.ndarray):
    return ctypes.c_void_p(a.ctypes.data)


def c_double(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)
