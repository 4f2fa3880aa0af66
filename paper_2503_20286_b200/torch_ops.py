"""``torch.ops.temo.*`` -- TORCH_LIBRARY registration of the C ABI.

The ops call the same entry points as the ctypes binding (``_lib.py``) on the current CUDA
stream, with torch-allocated outputs and workspace, so they can be captured in CUDA graphs
(``torch.cuda.graph``) and traced by ``torch.compile`` (Meta kernels give the shapes):

    torch.ops.temo.rank(F, n, mode) -> (rank int32, l, nfronts, status)   # ndsort.py:47-71
    torch.ops.temo.evaluate(X, problem_id, m, nk, sublen, offset) -> F    # problems.py:105-136
    torch.ops.temo.igd(F, Fstar) -> (1,)                                  # indicators.py:19-26

``load()`` builds ``_lib/libtemo_torch.so`` in-tree if needed (g++ against torch's headers,
linked to ``libtemo_b200.so``) and registers it.
"""

from __future__ import annotations

import hashlib
import subprocess
from pathlib import Path

from . import _lib
from . import build as _build

SRC = _build.PKG / "torchops" / "temo_ops.cpp"
LIB = _build.OUT_DIR / "libtemo_torch.so"
STAMP = _build.OUT_DIR / "libtemo_torch.stamp"
_loaded = False


def _cmd():
    import torch
    import torch.utils.cpp_extension as ce

    tdir = Path(torch.__file__).resolve().parent
    inc = [f"-I{p}" for p in ce.include_paths()] + ["-I/usr/local/cuda/include", f"-I{_build.ROOT / 'include'}"]
    abi = f"-D_GLIBCXX_USE_CXX11_ABI={int(torch._C._GLIBCXX_USE_CXX11_ABI)}"
    libs = [f"-L{tdir / 'lib'}", "-lc10", "-lc10_cuda", "-ltorch", "-ltorch_cpu", "-ltorch_cuda",
            f"-L{_build.OUT_DIR}", "-ltemo_b200", f"-Wl,-rpath,{tdir / 'lib'}", "-Wl,-rpath,$ORIGIN",
            "-L/usr/local/cuda/lib64", "-lcudart"]
    return ["g++", "-O2", "-std=c++17", "-shared", "-fPIC", abi, *inc, str(SRC), "-o", str(LIB), *libs]


def build(force: bool = False) -> Path:
    _build.build()
    cmd = _cmd()
    h = hashlib.sha256(SRC.read_bytes() + (_build.ROOT / "include" / "temo_b200.h").read_bytes()
                       + " ".join(cmd).encode()).hexdigest()
    if not force and LIB.exists() and STAMP.exists() and STAMP.read_text() == h:
        return LIB
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"building libtemo_torch.so failed:\n{res.stderr[-4000:]}")
    STAMP.write_text(h)
    return LIB


def load():
    """Register torch.ops.temo.* (builds the op library if needed); returns torch.ops.temo."""
    global _loaded
    import torch

    if not _loaded:
        _lib.lib()  # libtemo_b200.so first (the op library links against it)
        torch.ops.load_library(str(build()))
        _loaded = True
    return torch.ops.temo
