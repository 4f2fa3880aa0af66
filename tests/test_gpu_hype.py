"""GPU parity: HypE (alpha, MC hypervolume contributions in the dgemv_t order, selection)."""

import numpy as np
import pytest

from conftest import cases, load_golden
from oracle import hype as ohype

pytestmark = pytest.mark.gpu


def gen(seed):
    return np.random.Generator(np.random.Philox(np.random.SeedSequence(seed)))


def test_alpha_golden(cuda):
    from paper_2503_20286_b200.hype import shared_alpha

    z = load_golden("hype")
    for j in range(int(z["alpha_count"])):
        n1, k = z[f"alpha{j}_nk"]
        assert np.array_equal(shared_alpha(int(n1), int(k)), z[f"alpha{j}"])


@pytest.mark.parametrize("idx", range(7))
def test_selection_golden_bit_exact(cuda, idx):
    """v_hv and survivor order bit-identical to the reference (OPENBLAS_NUM_THREADS=1)."""
    import torch

    from paper_2503_20286_b200.hype import HypeSelector

    c = cases(load_golden("hype"))[idx]
    F = c["F"]
    N, m = F.shape
    sel = HypeSelector(N, m, int(c["n"]), int(c["s"]))
    g = gen(int(c["seed"]))
    keep = sel.select(torch.from_numpy(F).cuda(), g).cpu().numpy()
    sel.check()
    info = sel.info_host.numpy()
    assert info[1] == int(c["k"])
    if int(c["k"]) >= 1:
        assert np.array_equal(sel.v_hv.cpu().numpy(), c["v_hv"])
    assert np.array_equal(keep, c["keep"])
    # the Generator advanced exactly as the reference's did
    ref = gen(int(c["seed"]))
    if int(c["k"]) >= 1:
        ref.random((int(c["s"]), m))
    assert np.array_equal(g.random(5), ref.random(5))


@pytest.mark.parametrize("n1,m,s,k", [(401, 3, 70001, 17), (402, 3, 4099, 50), (403, 2, 2050, 3),
                                      (1000, 4, 65536, 100), (7, 3, 9000, 2), (2000, 3, 130001, 381)])
def test_hv_estimate_vs_oracle(cuda, n1, m, s, k):
    from paper_2503_20286_b200.hype import HvEstimateParams, hv_estimate

    r = np.random.default_rng(n1 + s)
    F = r.random((n1, m)) ** 2
    F[: n1 // 5] = np.round(F[: n1 // 5], 1)  # boundary ties with samples and between points
    ref = ohype.auto_reference(F)
    got = hv_estimate(F, HvEstimateParams(ref, k, s), gen(s))
    want = ohype.hv_estimate(F, ref, k, s, gen(s))
    assert np.array_equal(got, want)


def test_degenerate_box_draws_nothing(cuda):
    from paper_2503_20286_b200.hype import HvEstimateParams, hv_estimate

    F = np.random.default_rng(0).random((50, 3))
    g = gen(4)
    out = hv_estimate(F, HvEstimateParams(F.min(axis=0), 5, 1000), g)  # span == 0
    assert np.all(out == 0)
    assert np.array_equal(g.random(3), gen(4).random(3))


def test_environmental_selection_dropin(cuda):
    from paper_2503_20286_b200.hype import environmental_selection

    c = cases(load_golden("hype"))[0]
    N = c["F"].shape[0]
    X = np.arange(N, dtype=float)[:, None]
    Xk, Fk = environmental_selection(X, c["F"], None, int(c["n"]), int(c["s"]), gen(int(c["seed"])))
    assert np.array_equal(Xk[:, 0].astype(int), c["keep"])
    assert np.array_equal(Fk, c["F"][c["keep"]])


def test_auto_reference(cuda):
    from paper_2503_20286_b200.hype import auto_reference

    F = np.random.default_rng(1).random((300, 4)) * 5 - 1
    assert np.array_equal(auto_reference(F), ohype.auto_reference(F))


def test_config_c_golden_bit_exact(cuda):
    """BASELINE config C at full size (merged N = 20k, n = 10k, s = 100k samples): ranks, l,
    the HV contributions and the survivor order equal the reference's bits (hype.py:54-163;
    golden from the reference itself, OPENBLAS_NUM_THREADS=1)."""
    import torch

    from paper_2503_20286_b200.hype import HypeSelector

    z = dict(load_golden("hype_c"))
    F = z["F"]
    N, m = F.shape
    sel = HypeSelector(N, m, int(z["n"]), int(z["s"]))
    g = gen(int(z["seed"]))
    keep = sel.select(torch.from_numpy(F).cuda(), g).cpu().numpy()
    sel.check()
    assert int(sel.l.item()) == int(z["l"])
    r = sel.rank.cpu().numpy()
    live = z["r"] <= int(z["l"])
    assert np.array_equal(r[live], z["r"][live])
    assert sel.info_host.numpy()[1] == int(z["k"])
    assert np.array_equal(sel.v_hv.cpu().numpy(), z["v_hv"])
    assert np.array_equal(keep, z["keep"])


def test_deferred_rng_decision_equals_synced_loop(cuda):
    """Launch-ahead loops (step(timed=False)) advance the Generator speculatively after each HypE
    selection and settle the device's drew-samples flag one generation later, redoing the
    offspring when no samples were drawn; populations and the final Generator state equal the
    synced loop's.  Small populations make exact front fits (no samples drawn) frequent, so the
    undo path runs."""
    import json

    import torch

    from paper_2503_20286_b200.harness import RunConfig, _resolve, _Stepper
    from paper_2503_20286_b200.rng import RngStream

    undone = 0
    for seed, pop in ((1, 6), (2, 8), (3, 10), (4, 12)):
        cfg = RunConfig(algorithm="hype", problem="dtlz2", objectives=2, dim=6, pop_size=pop, seed=seed,
                        hv_samples=1001)
        spec, R, n = _resolve(cfg)
        outs = []
        for timed in (True, False):
            st_ = _Stepper(cfg, spec, R, n)
            gen = RngStream(seed).split(0).generator()
            st = st_.init(gen)
            flags = []
            for g in range(12):
                st, _ = st_.step(st, g, gen, timed=timed)
                if timed:
                    flags.append(int(st_.selector.info_host[3]))
            st_.check()
            X, F = st_.population(st)
            outs.append((X.cpu().numpy(), F.cpu().numpy(),
                         json.dumps(gen.bit_generator.state, default=lambda a: np.asarray(a).tolist())))
            if timed:
                undone += flags.count(0)
        assert np.array_equal(outs[0][0], outs[1][0]) and np.array_equal(outs[0][1], outs[1][1]), (seed, pop)
        assert outs[0][2] == outs[1][2], (seed, pop)
    assert undone > 0, "no generation exercised the undo path"
