"""GPU parity: MOEA/D (PBI pinned to golden vectors; Tchebycheff vs the self-oracle)."""

import numpy as np
import pytest

from conftest import cases, load_golden
from oracle import moead as omoead
from oracle import problems as oprob

pytestmark = pytest.mark.gpu


def restore_gen(c):
    g = np.random.Generator(np.random.Philox())
    st = g.bit_generator.state
    st["state"]["counter"] = c["counter"]
    st["state"]["key"] = c["key"]
    st["buffer"] = c["buffer"]
    st["buffer_pos"] = int(c["buffer_pos"])
    g.bit_generator.state = st
    return g


def engine_for(c):
    from paper_2503_20286_b200.directions import DirectionSet, NeighborTable
    from paper_2503_20286_b200.moead import MoeadEngine
    from paper_2503_20286_b200.problems import make_problem
    from paper_2503_20286_b200.variation import VariationParams

    name, d = str(c["name"]), int(c["d"])
    m = c["W"].shape[1]
    spec = make_problem(name, m=m, d=d)
    R = DirectionSet(c["W"], "simplex")
    params = VariationParams(lower=spec.lower, upper=spec.upper)
    return MoeadEngine(spec, R, NeighborTable(c["I_nb"]), params, 5.0, "pbi"), spec


@pytest.mark.parametrize("idx", range(3))
def test_moead_step_golden(cuda, idx):
    import torch

    from paper_2503_20286_b200.moead import MoeadState

    c = cases(load_golden("moead"))[idx]
    eng, spec = engine_for(c)
    dev = eng.dev
    st = MoeadState(torch.from_numpy(c["X"]).to(dev), torch.from_numpy(c["F1"]).to(dev),
                    torch.from_numpy(c["z"]).to(dev), eng.W, eng.I_nb, 5.0)
    g = restore_gen(c)
    nxt = eng.step(st, g)
    O = eng.O.cpu().numpy()
    assert np.allclose(O, c["O"], rtol=1e-13, atol=1e-14)          # pow ulps (App. A8)
    assert np.allclose(eng.F2.cpu().numpy(), c["F2"], rtol=1e-10, atol=1e-12)
    # selection stages on the reference's exact offspring: bit-exact
    nxt = eng.select(st, torch.from_numpy(c["O"]).to(dev), torch.from_numpy(c["F2"]).to(dev))
    assert np.array_equal(eng.zmin.cpu().numpy(), c["z_min"])
    assert np.array_equal(eng.improves.cpu().numpy().astype(bool), c["improves"])
    assert np.array_equal(nxt.X.cpu().numpy(), c["Xn"])
    assert np.array_equal(nxt.F1.cpu().numpy(), c["Fn"])
    # the host Generator consumed exactly the reference's draws
    ref = restore_gen(c)
    n, T = c["I_nb"].shape
    ref.integers(0, T, size=n)
    ref.integers(0, T - 1, size=n)
    ref.random((5 * n, int(c["d"])))
    assert np.array_equal(g.random(4), ref.random(4))


def random_state(n_dirs_H, m, T, seed, grid=False):
    from paper_2503_20286_b200.directions import das_dennis, neighbors

    R = das_dennis(m, n_dirs_H)
    tab = neighbors(R, T)
    r = np.random.default_rng(seed)
    n = R.count
    X = r.random((n, 4))
    F1 = r.integers(0, 4, size=(n, m)).astype(float) if grid else r.random((n, m))
    return R, tab, X, F1, F1.min(axis=0)


@pytest.mark.parametrize("kind", ["pbi", "tch"])
@pytest.mark.parametrize("seed", range(6))
def test_elite_rule_equals_dense_argmin(cuda, kind, seed):
    """App. A5 reverse-CSR rule == the reference's n x n column argmin, with exact ties."""
    from paper_2503_20286_b200.moead import MoeadState, compare_update, elite_select

    R, tab, X, F1, z = random_state(9, 3, 6, seed, grid=seed % 2 == 0)
    n = R.count
    r = np.random.default_rng(100 + seed)
    F2 = r.integers(0, 4, size=(n, 3)).astype(float) if seed % 2 == 0 else r.random((n, 3))
    F2[::5] = F1[::5]  # copied incumbents -> exact g ties
    O = r.random((n, 4))
    st = MoeadState(X, F1, z, R.W, tab.I_nb, 5.0)
    upd, zmin = compare_update(st, F2, aggregation=kind)
    improves, want_z = omoead.compare(F1, R.W, tab.I_nb, z, F2, 5.0, kind)
    assert np.array_equal(zmin, want_z) and np.array_equal(upd.improves, improves)
    assert np.array_equal(upd.I_new, omoead.update_matrix(improves, tab.I_nb))
    Xn, Fn = elite_select(st, O, F2, upd, zmin, aggregation=kind)
    Xw, Fw, _, _ = omoead.elite_select(X, F1, R.W, O, F2, omoead.update_matrix(improves, tab.I_nb), want_z,
                                       5.0, kind)
    assert np.array_equal(Xn, Xw) and np.array_equal(Fn, Fw)


def test_pbi_known_answers(cuda):
    """Ports of test_moead.py:30-62."""
    from paper_2503_20286_b200.moead import pbi

    z = np.array([0.5, 0.5])
    for w in (np.array([1.0, 0.0]), np.array([0.3, 0.7])):
        assert pbi(z, w, z, theta=7.0) == 0.0
    w = np.array([3.0, 4.0])
    assert np.isclose(pbi(2.0 * w / np.linalg.norm(w), w, np.zeros(2), theta=5.0), 2.0)
    assert np.isclose(pbi(np.array([1.0, 1.0]), np.array([1.0, 0.0]), np.zeros(2), theta=5.0), 6.0)
    with pytest.raises(ValueError):
        pbi(np.ones(2), np.zeros(2), np.zeros(2), theta=5.0)
    f, w2 = np.array([1.0, 1.0]), np.array([2.0, 0.0])
    assert np.isclose(pbi(f, w2, np.zeros(2), 5.0, normalize_direction=False), 1.0 + 5.0 * np.linalg.norm(f - w2))
    r = np.random.default_rng(3)
    F, W, Z = r.random((7, 5, 3)), r.random((7, 5, 3)) + 0.1, r.random(3)
    assert np.array_equal(pbi(F, W, Z, 5.0), omoead.pbi(F, W, Z, 5.0))


def test_forced_identity_offspring(cuda):
    """test_moead.py:164-173: ForcedRng(0.5) gives the first neighbour of each row."""
    from paper_2503_20286_b200.moead import init_state, moead_offspring
    from paper_2503_20286_b200.directions import das_dennis, neighbors
    from paper_2503_20286_b200.variation import VariationParams

    class ForcedRng:
        def random(self, size=None):
            return np.full(size, 0.5)

        def integers(self, low, high=None, size=None):
            return np.full(size, 0 if high is None else low, dtype=np.int64)

    ds = das_dennis(2, 5)
    tab = neighbors(ds, 3)
    r = np.random.default_rng(6)
    st = init_state(r.random((6, 4)), r.random((6, 2)), ds.W, tab)
    params = VariationParams(lower=np.zeros(4), upper=np.ones(4))
    O, F2 = moead_offspring(st, ForcedRng(), params, lambda X: X[:, :2])
    first = st.X[st.I_nb[:, 0]]
    assert np.array_equal(O, first) and np.array_equal(F2, first[:, :2])


def test_z_monotone_and_tch_runs(cuda):
    import torch

    from paper_2503_20286_b200.harness import RunConfig, _resolve, _Stepper

    for agg in ("pbi", "tch"):
        cfg = RunConfig(algorithm="moead", problem="dtlz1", objectives=3, dim=7, pop_size=21, aggregation=agg)
        spec, R, n = _resolve(cfg)
        s = _Stepper(cfg, spec, R, n)
        g = np.random.Generator(np.random.Philox(np.random.SeedSequence(86)))
        st = s.init(g)
        prev = st.extra["moead"].z.cpu().numpy()
        for k in range(25):
            st, _ = s.step(st, k, g)
            z = st.extra["moead"].z.cpu().numpy()
            assert np.all(z <= prev + 1e-15)
            prev = z
        torch.cuda.synchronize()


def test_config_b_golden(cuda):
    """BASELINE config B at full size: DTLZ2 m=3 d=12, n = 9870 directions (H = 139), T = 20, with
    19 % exact T-th neighbour ties.  Offspring within pow ulps; z_min, improves and the elite
    selection on the reference's offspring bit-exact (moead.py:70-158)."""
    import torch

    from paper_2503_20286_b200.directions import DirectionSet, NeighborTable, das_dennis
    from paper_2503_20286_b200.moead import MoeadEngine, MoeadState
    from paper_2503_20286_b200.problems import make_problem
    from paper_2503_20286_b200.variation import VariationParams

    z = dict(load_golden("moead_b"))
    spec = make_problem("dtlz2", m=3, d=12)
    R = das_dennis(3, 139)
    I_nb = z["I_nb"].astype(np.int64)
    eng = MoeadEngine(spec, R, NeighborTable(I_nb), VariationParams(lower=spec.lower, upper=spec.upper), 5.0, "pbi")
    dev = eng.dev
    st = MoeadState(torch.from_numpy(z["X"]).to(dev), torch.from_numpy(z["F1"]).to(dev),
                    torch.from_numpy(z["z"]).to(dev), eng.W, eng.I_nb, 5.0)
    g = np.random.Generator(np.random.Philox())
    s = g.bit_generator.state
    s["state"]["counter"], s["state"]["key"] = z["counter"], z["key"]
    s["buffer"], s["buffer_pos"] = z["buffer"], int(z["buffer_pos"])
    s["has_uint32"], s["uinteger"] = int(z["has_uint32"]), int(z["uinteger"])
    g.bit_generator.state = s
    eng.step(st, g)
    assert np.allclose(eng.O.cpu().numpy(), z["O"], rtol=1e-13, atol=1e-14)
    assert np.allclose(eng.F2.cpu().numpy(), z["F2"], rtol=1e-10, atol=1e-12)
    nxt = eng.select(st, torch.from_numpy(z["O"]).to(dev), torch.from_numpy(z["F2"]).to(dev))
    assert np.array_equal(eng.zmin.cpu().numpy(), z["z_min"])
    assert np.array_equal(eng.improves.cpu().numpy().astype(bool), z["improves"])
    assert np.array_equal(nxt.X.cpu().numpy(), z["Xn"])
    assert np.array_equal(nxt.F1.cpu().numpy(), z["Fn"])


def test_graph_generation_equals_plain_launches(cuda):
    """MOEA/D generations replayed from the captured CUDA graph (offspring with the Philox state
    in device memory + compare + elite) equal plain launches bit for bit, and the host
    Generator ends in the same state."""
    import json

    from paper_2503_20286_b200.harness import RunConfig, _resolve, _Stepper
    from paper_2503_20286_b200.rng import RngStream

    cfg = RunConfig(algorithm="moead", problem="dtlz2", objectives=3, dim=12, pop_size=300, seed=4, neighborhood=10)
    spec, R, n = _resolve(cfg)
    outs = []
    for graph in (False, True):
        st_ = _Stepper(cfg, spec, R, n)
        st_.engine.graph = graph
        gen = RngStream(4).split(0).generator()
        st = st_.init(gen)
        traj = []
        for g in range(5):
            st, _ = st_.step(st, g, gen)
            X, F = st_.population(st)
            traj.append((X.cpu().numpy().copy(), F.cpu().numpy().copy(), st.extra["moead"].z.cpu().numpy().copy()))
        outs.append((traj, json.dumps(gen.bit_generator.state, default=lambda a: np.asarray(a).tolist())))
    for a, b in zip(outs[0][0], outs[1][0]):
        for x, y in zip(a, b):
            assert np.array_equal(x, y)
    assert outs[0][1] == outs[1][1]
