"""One warm-up + one ND sort call at a given size (for ncu launch lists)."""
import sys, os
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2503_20286_b200.ndsort import rank_device, SORT, SELECT
N = int(sys.argv[1]); mode = int(sys.argv[2]) if len(sys.argv) > 2 else SELECT
F = torch.from_numpy(np.random.default_rng(0).random((N, 3))).cuda()
for _ in range(2):
    r, l, nf = rank_device(F, N // 2, mode)
torch.cuda.synchronize()
print("fronts", int(nf.item()))
