"""cProfile of 10 launch-only headline generations (host side of _Stepper.step)."""
import cProfile
import os
import pstats
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2503_20286_b200.harness import RunConfig, _resolve, _Stepper  # noqa: E402
from paper_2503_20286_b200.rng import RngStream  # noqa: E402

cfg = RunConfig(algorithm="nsga3", problem="lsmop1", objectives=3, dim=1000, pop_size=200_000, seed=0)
spec, R, n = _resolve(cfg)
st_ = _Stepper(cfg, spec, R, n)
gen = RngStream(0).split(0).generator()
st = st_.init(gen)
for g in range(3):
    st, _ = st_.step(st, g, gen)
torch.cuda.synchronize()
box = [st]


def run():
    for g in range(10):
        box[0], _ = st_.step(box[0], g, gen, timed=False)
    torch.cuda.synchronize()


cProfile.run("run()", "/tmp/prof.out")
pstats.Stats("/tmp/prof.out").sort_stats("tottime").print_stats(25)
