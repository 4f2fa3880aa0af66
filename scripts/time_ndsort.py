"""Time the GPU ND sort at several sizes (CUDA events on the launching stream)."""

import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2503_20286_b200 import _lib  # noqa: E402
from paper_2503_20286_b200.ndsort import SELECT, SORT, rank_device  # noqa: E402


def main():
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    sizes = [int(a) for a in args] or [20000, 100000, 400000]
    ms_list = [int(x) for x in os.environ.get("MS", "3").split(",")]
    if "--bitmap" in sys.argv:
        _lib.lib().temo_rank_force_bitmap(1)
    for m in ms_list:
        for N in sizes:
            F = torch.from_numpy(np.random.default_rng(0).random((N, m))).cuda()
            for mode in (SORT, SELECT):
                rank_device(F, N // 2, mode)
                torch.cuda.synchronize()
                s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                s.record()
                reps = 3
                for _ in range(reps):
                    r, l, nf = rank_device(F, N // 2, mode)
                e.record()
                torch.cuda.synchronize()
                ms = s.elapsed_time(e) / reps
                _lib.timing_enable(True)
                rank_device(F, N // 2, mode)
                stages = _lib.timing_read()
                _lib.timing_enable(False)
                print(json.dumps(dict(N=N, m=m, mode=mode, ms=round(ms, 3), fronts=int(nf.item()),
                                      l=int(l.item()), pairs_per_s=N * (N - 1) / ms * 1e3,
                                      stages={k: round(v[0], 3) for k, v in stages.items()})))


if __name__ == "__main__":
    main()
