"""CPU-side checks of the C ABI: the library builds, loads and exports every declared symbol."""

import ctypes
import re
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]


def declared_functions():
    text = (ROOT / "include" / "temo_b200.h").read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(temo_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_entry_points():
    names = declared_functions()
    assert "temo_rank" in names and "temo_abi_version" in names


def test_library_exports_every_declared_symbol():
    from paper_2503_20286_b200 import _lib

    L = _lib.lib()
    for name in declared_functions():
        assert hasattr(L, name), name
        assert name in _lib.SIGNATURES, f"{name} has no ctypes signature"


def test_abi_version_and_errors_without_gpu():
    from paper_2503_20286_b200 import _lib

    L = _lib.lib()
    assert L.temo_abi_version() == 1
    assert L.temo_strerror(1) == b"invalid argument"
    # argument validation happens on the host, before any launch
    assert L.temo_rank(None, 0, 3, 1, 0, None, None, None, None, None, 0, None) == _lib.TEMO_EINVAL
    assert L.temo_rank_ws_bytes(1000, 3) > 1000 * 1000 // 16


def test_workspace_sizes_monotone():
    from paper_2503_20286_b200 import _lib

    L = _lib.lib()
    sizes = [L.temo_rank_ws_bytes(n, 3) for n in (100, 1000, 10000, 100000)]
    assert sizes == sorted(sizes)


def test_product_does_not_import_oracle():
    for p in (ROOT / "paper_2503_20286_b200").rglob("*.py"):
        src = p.read_text()
        assert not re.search(r"^\s*(from|import)\s+oracle", src, flags=re.M), p


def test_no_gpu_means_loud_failure():
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import numpy as np

    from paper_2503_20286_b200 import rank_assign

    with pytest.raises(Exception, match="CUDA"):
        rank_assign(np.random.default_rng(0).random((10, 3)), 5)
