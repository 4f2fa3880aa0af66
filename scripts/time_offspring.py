"""Time temo_offspring_ws (fused TMA path and two-phase) at pop 200k, LSMOP1 d=1000 (D=992), CUDA events."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2503_20286_b200 import _lib
from paper_2503_20286_b200.problems import make_problem
from paper_2503_20286_b200.rng import DeviceDraws
from paper_2503_20286_b200.variation import VariationParams

n = int(sys.argv[1]) if len(sys.argv) > 1 else 200000
spec = make_problem("lsmop1", m=3, d=1000); d = spec.d; h = n // 2
dev = torch.device("cuda", 0)
var = VariationParams(lower=spec.lower, upper=spec.upper).struct(d, dev)
prob = spec.struct()
gen = np.random.Generator(np.random.Philox(7))
X = torch.from_numpy(spec.lower + np.random.default_rng(1).random((2 * h, d)) * (spec.upper - spec.lower)).to(dev)
idx = torch.from_numpy(np.random.default_rng(2).permutation(2 * h).astype(np.int64)).to(dev)
O = torch.empty((2 * h, d), dtype=torch.float64, device=dev)
FO = torch.empty((2 * h, 3), dtype=torch.float64, device=dev)
draws = DeviceDraws(gen); off = draws.take(7 * h * d)
L, s = _lib.lib(), _lib.stream_handle(dev)
ws = torch.empty(max(L.temo_offspring_ws_bytes(h, d), 256), dtype=torch.uint8, device=dev)
args = (_lib.sptr(prob), _lib.sptr(var), _lib.ptr(X), _lib.ptr(idx), _lib.ptr(idx[h:]), h,
        _lib.sptr(draws.state), off, _lib.ptr(O), _lib.ptr(FO), None, None, _lib.ptr(ws), ws.numel(), s)
res = {}
for path in (1, 0):
    L.temo_offspring_set_path(path)
    for _ in range(2):
        L.temo_offspring_ws(*args)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(5):
        assert L.temo_offspring_ws(*args) == 0
    b.record(); torch.cuda.synchronize()
    res[path] = (a.elapsed_time(b) / 5, O[:, :8].clone(), FO.clone())
print(os.environ.get("TEMO_LIB", "default"), "tma %.3f ms  two-phase %.3f ms  equal %s" % (
    res[1][0], res[0][0], bool(torch.equal(res[1][1], res[0][1]) and torch.equal(res[1][2], res[0][2]))))
