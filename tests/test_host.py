"""CPU tests of the host-side logic (no GPU): RNG bridge, direction sets, problem descriptors."""

import numpy as np
import pytest

from oracle import directions as odir
from oracle import philox as ophilox
from oracle import problems as oprob


@pytest.mark.parametrize("pre", range(9))
@pytest.mark.parametrize("count", [1, 2, 3, 4, 5, 7, 8, 9, 100, 1001])
def test_rng_advance_equals_draws(pre, count):
    from paper_2503_20286_b200.rng import advance

    a = np.random.Generator(np.random.Philox(np.random.SeedSequence(3)))
    b = np.random.Generator(np.random.Philox(np.random.SeedSequence(3)))
    a.random(pre)
    b.random(pre)
    a.random(count)
    advance(b, count)
    assert np.array_equal(a.random(13), b.random(13))
    assert np.array_equal(a.permutation(50), b.permutation(50))


def test_device_draw_offsets_match_stream():
    """DeviceDraws offsets index the same raw outputs the oracle's Philox restatement produces."""
    from paper_2503_20286_b200.rng import DeviceDraws

    g = np.random.Generator(np.random.Philox(np.random.SeedSequence(8)))
    g.random(3)
    st = g.bit_generator.state
    dd = DeviceDraws(g)
    o1 = dd.take(10)
    o2 = dd.take(7)
    assert (o1, o2) == (0, 10)
    want = ophilox.doubles(st, 17)
    dd.commit()
    ref = np.random.Generator(np.random.Philox(np.random.SeedSequence(8)))
    ref.random(3)
    assert np.array_equal(ref.random(17), want)
    assert np.array_equal(g.random(5), ref.random(5))


@pytest.mark.parametrize("m,H", [(2, 40), (3, 12), (3, 630), (4, 7), (5, 6), (8, 3), (10, 3)])
def test_simplex_lattice_and_lattice_H(m, H):
    from paper_2503_20286_b200.directions import das_dennis, largest_h_for, simplex_lattice

    W = simplex_lattice(m, H)
    assert np.array_equal(W, odir.simplex_lattice(m, H))
    assert das_dennis(m, H).lattice_H == H
    assert largest_h_for(W.shape[0], m) == H


def test_lattice_H_rejects_other_sets():
    from paper_2503_20286_b200.directions import DirectionSet, das_dennis

    W = das_dennis(3, 5).W.copy()
    assert DirectionSet(W[::-1].copy(), "simplex").lattice_H == 0  # different row order
    assert DirectionSet(W[:-1], "simplex").lattice_H == 0
    assert DirectionSet(np.random.default_rng(0).random((10, 3)) + 0.1, "simplex").lattice_H == 0


def test_lsmop_descriptor_matches_self_oracle():
    from paper_2503_20286_b200.problems import lsmop_groups, make_problem

    for m, d in ((3, 1000), (2, 300), (5, 700)):
        a = lsmop_groups(m, d)
        b = oprob.lsmop_groups(m, d)
        assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
        spec = make_problem("lsmop1", m=m, d=d)
        # PlatEMO: the request sizes the groups, then D = m - 1 + nk * sum(sublen)
        assert spec.d == m - 1 + a[1][m] == oprob.lsmop_dimension(m, d)
        lo, hi = oprob.lsmop_bounds(m, spec.d)
        assert np.array_equal(spec.lower, lo) and np.array_equal(spec.upper, hi)
        s = spec.struct()
        assert s.id == 101 and s.nk == 5 and s.sublen[0] == a[0][0] and s.offset[m] == a[1][m]
        b2 = oprob.lsmop_groups_for(m, spec.d)
        assert np.array_equal(a[0], b2[0]) and np.array_equal(a[1], b2[1])
    assert make_problem("lsmop1", m=3, d=1000).d == 992


def test_run_config_validation():
    from paper_2503_20286_b200.harness import ConfigError, RunConfig, _resolve

    with pytest.raises(ConfigError):
        RunConfig(algorithm="nope").validate()
    with pytest.raises(ConfigError):
        RunConfig(aggregation="x").validate()
    spec, R, n = _resolve(RunConfig(algorithm="moead", problem="dtlz2", pop_size=100))
    assert n == R.count == 91
    spec, R, n = _resolve(RunConfig(algorithm="nsga3", problem="lsmop1", dim=1000, pop_size=200_000))
    assert R.count == 199_396 and n == 200_000 and spec.d == 992  # PlatEMO D for the request 1000


def test_moead_default_neighborhood():
    from paper_2503_20286_b200.moead import default_neighborhood

    assert default_neighborhood(10) == 2 and default_neighborhood(91) == 10 and default_neighborhood(1000) == 20


def test_variation_params_validation():
    from paper_2503_20286_b200.variation import VariationParams

    with pytest.raises(ValueError):
        VariationParams(eta_c=0.0, lower=np.zeros(2), upper=np.ones(2))
    with pytest.raises(ValueError):
        VariationParams(p_m=1.5, lower=np.zeros(2), upper=np.ones(2))
    with pytest.raises(ValueError):
        VariationParams(lower=np.ones(3), upper=np.zeros(3))
    assert VariationParams(lower=np.zeros(4), upper=np.ones(4)).mutation_prob(4) == 0.25


def test_host_permutation_bit_exact_with_numpy():
    """temo_host_permutation (native Fisher-Yates + random_interval over Philox next_uint32)
    equals Generator.permutation and leaves the identical Generator state, for every buffer
    position / pending-half-word state and across mask classes (variation.py:52, nsga3.py:204)."""
    from paper_2503_20286_b200 import rng as R

    def same(sa, sb):
        return (all(np.array_equal(sa["state"][k], sb["state"][k]) for k in ("counter", "key"))
                and np.array_equal(sa["buffer"], sb["buffer"])
                and all(sa[k] == sb[k] for k in ("buffer_pos", "has_uint32", "uinteger")))

    for seed in range(4):
        for pre in range(5):
            for n in (2, 3, 17, 64, 65, 1025, 4097, 65537, 200_003):
                a = np.random.Generator(np.random.Philox(seed))
                b = np.random.Generator(np.random.Philox(seed))
                a.random(pre)
                b.random(pre)
                a.integers(0, 7, pre)  # leaves a pending 32-bit half for odd counts
                b.integers(0, 7, pre)
                assert np.array_equal(a.permutation(n), R.permutation(b, n)), (seed, pre, n)
                assert same(a.bit_generator.state, b.bit_generator.state), (seed, pre, n)
                assert np.array_equal(a.random(3), b.random(3))


def test_ndsort_oracle_host_matches_reference_golden():
    """ndsort_oracle (ndsort.py:74-106) is provided as a host oracle: same ranks as the reference."""
    from conftest import load_golden, unpack
    from paper_2503_20286_b200.ndsort import ndsort_oracle

    z = dict(load_golden("ndsort"))
    for i in range(0, len(z["N"]), 5):
        N, m, n = int(z["N"][i]), int(z["m"][i]), int(z["n"][i])
        if N > 400:
            continue
        F = unpack(z["F"], z["F_off"], i).reshape(N, m)
        res = ndsort_oracle(F, n)
        assert np.array_equal(res.r, unpack(z["r"], z["r_off"], i)) and res.l == int(z["l"][i])


def test_run_config_fields_match_reference():
    import dataclasses

    from paper_2503_20286_b200.harness import ConfigError, RunConfig

    names = {f.name for f in dataclasses.fields(RunConfig)}
    for f in ("algorithm", "problem", "objectives", "dim", "pop_size", "generations", "seed", "repeats",
              "eta_c", "eta_m", "pm", "theta", "neighborhood", "divisions", "alpha", "hv_samples", "hv_ref",
              "indicators", "indicator_every", "ref_front_size", "time_selection_only", "out"):
        assert f in names
    with pytest.raises(ConfigError):
        RunConfig(indicators=("nope",)).validate()
    with pytest.raises(ConfigError):
        RunConfig(ref_front_size=2).validate()
    with pytest.raises(ConfigError):
        RunConfig(hv_ref="1,2").validate()
    with pytest.raises(ConfigError):
        RunConfig(algorithm="nsga3-seq").validate()
    RunConfig(algorithm="rvea").validate()


def test_lsmop_family_known_answers():
    """Self-oracle LSMOP1-9 (PlatEMO form): every eta vanishes at z = 0 except Rosenbrock
    (L - 1 per subcomponent), so rows whose linkage maps x^s to 0 land on the linear (1-4),
    concave (5-8) or disconnected (9) front, shifted by the Rosenbrock groups exactly."""
    import math

    from paper_2503_20286_b200.problems import LSMOP, make_problem

    assert LSMOP == tuple(f"lsmop{k}" for k in range(1, 10))
    m, nk = 3, 5
    for k in range(1, 10):
        spec = make_problem(f"lsmop{k}", m=m, d=300)
        assert spec.struct().id == 100 + k
        d = spec.d
        sub, off = oprob.lsmop_groups_for(m, d)
        pos = np.array([[0.3, 0.6], [0.0, 1.0], [0.9, 0.2]])
        j = np.arange(m, d + 1) / d
        c = np.cos(j * np.pi / 2.0) if k >= 5 else j
        X = np.zeros((len(pos), d))
        X[:, : m - 1] = pos
        X[:, m - 1:] = 10.0 * pos[:, :1] / (1.0 + c)
        F = oprob.evaluate_lsmop(k, X, m)
        eta = oprob._ETA[k]
        G = np.array([(nk * (sub[i] - 1) if eta[i % 2] == "rosenbrock" else 0.0) / sub[i] / nk for i in range(m)])
        for r, p in enumerate(pos):
            if k <= 4:
                want = (1.0 + G) * np.array([p[0] * p[1], p[0] * (1 - p[1]), 1 - p[0]])
            elif k <= 8:
                a, b = p * math.pi / 2.0
                Gn = np.append(G[1:], 0.0)
                want = (1.0 + G + Gn) * np.array([math.cos(a) * math.cos(b), math.cos(a) * math.sin(b), math.sin(a)])
            else:
                gs = 1.0 + G.sum()
                want = np.array([p[0], p[1], (1 + gs) * (m - np.sum(p / (1 + gs) * (1 + np.sin(3 * np.pi * p))))])
            assert np.allclose(F[r], want, rtol=1e-9, atol=1e-9), (k, r, F[r], want)


def test_lsmop_true_fronts():
    from paper_2503_20286_b200.problems import make_problem, true_front

    for k in range(1, 10):
        F = true_front(make_problem(f"lsmop{k}", m=3, d=300), 200)
        assert F.shape[1] == 3 and 3 <= len(F) <= 200
        if k <= 4:
            assert np.allclose(F.sum(axis=1), 1.0)
        elif k <= 8:
            assert np.allclose((F ** 2).sum(axis=1), 1.0)
        else:
            assert np.all(F[:, 2] >= 2.0 * 1.0)  # f_M = 2 (M - ...) >= 2 on the optimal front
