"""Host-side cost of the headline generation loop: wall time per _Stepper.step call (launch
only, timed=False) with and without the host-input pipeline, and the loop's wall rate."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2503_20286_b200.harness import RunConfig, _resolve, _Stepper  # noqa: E402
from paper_2503_20286_b200.rng import RngStream  # noqa: E402

pop = int(sys.argv[1]) if len(sys.argv) > 1 else 200_000
cfg = RunConfig(algorithm="nsga3", problem="lsmop1", objectives=3, dim=1000, pop_size=pop, seed=0)
spec, R, n = _resolve(cfg)
st_ = _Stepper(cfg, spec, R, n)
gen = RngStream(0).split(0).generator()
st = st_.init(gen)
for g in range(3):
    st, _ = st_.step(st, g, gen)
torch.cuda.synchronize()
K = 20
for mode in ("plain", "pipeline", "pipeline", "plain"):
    if mode == "pipeline":
        st_.start_host_pipeline(gen, K)
    t = []
    t0 = time.perf_counter()
    for g in range(K):
        a = time.perf_counter()
        st, _ = st_.step(st, g, gen, timed=False)
        t.append(time.perf_counter() - a)
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    print(f"{mode:9s} step() call median {np.median(t)*1e3:.2f} ms  max {np.max(t)*1e3:.2f}  loop {wall/K*1e3:.2f} ms/gen")
# pieces
a = time.perf_counter()
for _ in range(5):
    hi = st_.draw_host_inputs(gen)
print("draw_host_inputs", (time.perf_counter() - a) / 5 * 1e3, "ms")
a = time.perf_counter()
for _ in range(5):
    st_.ring.upload(hi.shuffle, st_.perm)
print("ring.upload 400k int64", (time.perf_counter() - a) / 5 * 1e3, "ms")
