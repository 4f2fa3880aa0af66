"""Phase timeline of the staircase peel (block 0, %globaltimer) at one size."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2503_20286_b200 import _lib  # noqa: E402
from paper_2503_20286_b200.ndsort import SELECT, rank_device  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 400000
m = int(sys.argv[2]) if len(sys.argv) > 2 else 3
F = torch.from_numpy(np.random.default_rng(0).random((N, m))).cuda()
rank_device(F, N // 2, SELECT)
L = _lib.lib()
blk = int(sys.argv[3]) if len(sys.argv) > 3 else 0
L.temo_stair_prof_enable(blk + 1)
r, l, nf = rank_device(F, N // 2, SELECT)
torch.cuda.synchronize()
f = int(nf.item())
buf = np.zeros(8 * min(f, 2048), dtype=np.uint64)
L.temo_stair_prof_read(_lib._P(buf.ctypes.data), buf.size)
t = buf.reshape(-1, 8).astype(np.int64)
names = ["phaseA", "sync1", "tileld", "high", "low", "front", "sync2"]
d = np.diff(t[:, :8], axis=1) / 1e3
print(f"N={N} m={m} block={blk} fronts={f}  per-front us (median / mean):")
for i, nm in enumerate(names):
    print(f"  {nm:7s} {np.median(d[:, i]):7.2f} {d[:, i].mean():7.2f}")
tot = (t[1:, 0] - t[:-1, 0]) / 1e3
print(f"  front-to-front {np.median(tot):7.2f} {tot.mean():7.2f}")
print("first fronts (us):")
for i in range(min(6, len(d))):
    print("  ", np.round(d[i], 2))
