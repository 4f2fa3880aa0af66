"""Achievable bandwidth of the offspring apply phase's access pattern (temo_probe_rows_rate)
at the headline size (h = 100k pairs of d = 992 doubles; random parent rows, scattered children)
next to the same kernel on identity rows, and the apply kernel's own rate from the bench."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2503_20286_b200 import _lib  # noqa: E402

h, d = 100_000, 992
N = 4 * h
dev = torch.device("cuda", 0)
X = torch.rand((N, d), dtype=torch.float64, device=dev)
B = torch.rand((h, d), dtype=torch.float64, device=dev)
O = torch.empty((N, d), dtype=torch.float64, device=dev)
r = np.random.default_rng(0)
for name, (pa, pb, dst) in {
    "random rows (as the harness)": (r.integers(0, N, h), r.integers(0, N, h), r.permutation(N)[: 2 * h]),
    "identity rows": (np.arange(h), np.arange(h, 2 * h), np.arange(2 * h)),
}.items():
    t = [torch.from_numpy(np.asarray(v, dtype=np.int64)).to(dev) for v in (pa, pb, dst)]
    rate = _lib.lib().temo_probe_rows_rate(_lib.ptr(X), _lib.ptr(t[0]), _lib.ptr(t[1]), _lib.ptr(B), _lib.ptr(t[2]),
                                           h, d, _lib.ptr(O), 10, _lib.stream_handle(dev))
    print(f"{name}: {rate / 1e9:.0f} GB/s  ({5 * 8 * h * d / rate * 1e3:.3f} ms per pass of {5 * 8 * h * d / 1e9:.2f} GB)")
