"""Build the in-tree CUDA library ``libtemo_b200.so`` for sm_100a.

One shared object exports the C ABI declared in ``include/temo_b200.h``.  It is
built in-tree (``paper_2503_20286_b200/_lib/``) so it travels to the GPU box
with the repo snapshot.  ``--fmad=false`` keeps every double expression
separately rounded, like NumPy; explicit ``fma()`` calls remain fused.
"""

from __future__ import annotations

import hashlib
import os
import shutil
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
OUT_DIR = PKG / "_lib"
LIB = OUT_DIR / "libtemo_b200.so"
STAMP = OUT_DIR / "libtemo_b200.stamp"

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ["-O3", "-std=c++17", "-lineinfo", "--fmad=false", "-Xcompiler", "-fPIC",
              "-Xptxas", "-v", "-I", str(ROOT / "include")]


M_SPLIT = tuple(range(2, 17))  # objective counts of the per-M translation units


def _nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found: cannot build libtemo_b200.so")


def _sources():
    return sorted(CSRC.glob("*.cu"))


def _digest() -> str:
    h = hashlib.sha256()
    for p in sorted(list(CSRC.glob("*")) + [ROOT / "include" / "temo_b200.h"]):
        if p.is_file():
            h.update(p.name.encode())
            h.update(p.read_bytes())
    h.update(" ".join(ARCH + NVCC_FLAGS).encode())
    return h.hexdigest()


def up_to_date() -> bool:
    return LIB.exists() and STAMP.exists() and STAMP.read_text().strip() == _digest()


def build(force: bool = False, verbose: bool = False) -> Path:
    if not force and up_to_date():
        return LIB
    nvcc = _nvcc()
    OUT_DIR.mkdir(parents=True, exist_ok=True)
    objs = []

    def compile_one(job):
        src, m_only = job
        tag = src.stem if m_only is None else f"{src.stem}_m{m_only}"
        obj = OUT_DIR / (tag + ".o")
        extra = [] if m_only is None else [f"-DTEMO_M_ONLY={m_only}"]
        cmd = [nvcc, *ARCH, *NVCC_FLAGS, *extra, "-c", str(src), "-o", str(obj)]
        # incremental: an object is reused when its source, the shared headers and the flags match
        h = hashlib.sha256(src.read_bytes() + hdrs + " ".join(cmd).encode()).hexdigest()
        ostamp = OUT_DIR / (tag + ".ostamp")
        if not force and obj.exists() and ostamp.exists() and ostamp.read_text() == h:
            return obj
        res = subprocess.run(cmd, capture_output=True, text=True)
        if res.returncode != 0:
            raise RuntimeError(f"nvcc failed for {tag}:\n{res.stderr}")
        (OUT_DIR / (tag + ".ptxas.txt")).write_text(res.stderr)
        ostamp.write_text(h)
        if verbose:
            sys.stderr.write(res.stderr)
        return obj

    hdrs = b"".join(p.read_bytes() for p in sorted(CSRC.glob("*.cuh")) + [ROOT / "include" / "temo_b200.h"])
    # sources that guard their M-templated launchers with TEMO_M_ONLY are split into a
    # base unit plus one unit per objective count, so the heavy instantiations build in parallel
    jobs = []
    for src in _sources():
        jobs.append((src, None))
        if "TEMO_M_ONLY" in src.read_text():
            jobs.extend((src, m) for m in M_SPLIT)
    jobs.sort(key=lambda j: (j[1] is None, j[1] or 0), reverse=True)  # heavy per-M units first
    with ThreadPoolExecutor(max_workers=max(1, os.cpu_count() or 1)) as ex:
        objs = list(ex.map(compile_one, jobs))
    tmp = LIB.with_suffix(f".{os.getpid()}.tmp")
    cmd = [nvcc, *ARCH, "-shared", "-o", str(tmp), *map(str, objs), "-lcudart"]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"link failed:\n{res.stderr}")
    os.replace(tmp, LIB)
    STAMP.write_text(_digest())
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
