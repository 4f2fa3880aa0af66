"""Oracle: one full reference generation (harness.py:206-248) built from the oracle pieces.

Test infrastructure and the CPU baseline of bench.py (``cpu_baseline`` leg and
``--impl reference`` arm) -- never the product path.
"""

from __future__ import annotations

import numpy as np

from . import nsga3, problems, variation


def nsga3_generation(X, F, W, n, rng, problem, m, lower, upper, eta_c=20.0, eta_m=20.0, p_m=None):
    """harness._Stepper.step for algorithm="nsga3": offspring, evaluate, select."""
    O = variation.offspring(rng, X, eta_c, eta_m, p_m, lower, upper)
    FO = problems.evaluate(problem, O, m)
    Xm = np.concatenate([X, O])
    Fm = np.concatenate([F, FO])
    return nsga3.environmental_selection(Xm, Fm, W, n, rng)
