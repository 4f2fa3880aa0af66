"""Compare the offspring paths (fused k_offspring_s, fused TMA, two-phase) on one case."""
import sys, os
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2503_20286_b200 import _lib
from paper_2503_20286_b200.problems import make_problem
from paper_2503_20286_b200.rng import DeviceDraws
from paper_2503_20286_b200.variation import VariationParams

name, m, d, h, pre = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4]), int(sys.argv[5])
spec = make_problem(name, m=m, d=d); d = spec.d
dev = torch.device("cuda", 0)
var = VariationParams(lower=spec.lower, upper=spec.upper).struct(d, dev)
prob = spec.struct()
gen = np.random.Generator(np.random.Philox(7)); gen.random(pre)
X = torch.from_numpy(spec.lower + np.random.default_rng(1).random((2 * h, d)) * (spec.upper - spec.lower)).to(dev)
idx = torch.from_numpy(np.random.default_rng(2).permutation(2 * h).astype(np.int64)).to(dev)
draws = DeviceDraws(gen); off = draws.take(7 * h * d)
outs = {}
for path in ("fused", "ws-tma", "ws-two-phase"):
    O = torch.full((2 * h, d), np.nan, dtype=torch.float64, device=dev)
    FO = torch.full((2 * h, m), np.nan, dtype=torch.float64, device=dev)
    L, s = _lib.lib(), _lib.stream_handle(dev)
    args = (_lib.sptr(prob), _lib.sptr(var), _lib.ptr(X), _lib.ptr(idx), _lib.ptr(idx[h:]), h,
            _lib.sptr(draws.state), off, _lib.ptr(O), _lib.ptr(FO))
    if path.startswith("ws"):
        L.temo_offspring_set_path(1 if path == "ws-tma" else 0)
        ws = torch.empty(max(L.temo_offspring_ws_bytes(h, d), 256), dtype=torch.uint8, device=dev)
        rc = L.temo_offspring_ws(*args, None, None, _lib.ptr(ws), ws.numel(), s)
        L.temo_offspring_set_path(1)
    else:
        rc = L.temo_offspring(*args, s)
    torch.cuda.synchronize()
    o, f = O.cpu().numpy(), FO.cpu().numpy()
    outs[path] = (o, f)
    bad = np.isnan(o)
    print(path, "rc", rc, "nan rows", np.unique(np.nonzero(bad)[0])[:10], "count", bad.sum(), "F nan", np.isnan(f).sum())
ref = outs["ws-two-phase"]
for k, (o, f) in outs.items():
    dif = ~np.isclose(o, ref[0], rtol=0, atol=0, equal_nan=True)
    print(k, "differs from two-phase at", dif.sum(), "genes; rows", np.unique(np.nonzero(dif)[0])[:10])
