"""GPU parity: device Philox stream, SBX/PM, DTLZ/LSMOP evaluation, fused offspring kernel."""

import numpy as np
import pytest

from conftest import load_golden
from oracle import problems as oprob
from oracle import variation as ovar

pytestmark = pytest.mark.gpu


def philox_gen(seed):
    return np.random.Generator(np.random.Philox(np.random.SeedSequence(seed)))


class ForcedRng:
    """The reference tests' ForcedRng (oracles.py:108-121)."""

    def __init__(self, value=0.5):
        self.value = value

    def random(self, size=None):
        return self.value if size is None else np.full(size, self.value)

    def integers(self, low, high=None, size=None):
        lo = 0 if high is None else low
        return np.full(size, lo, dtype=np.int64) if size is not None else lo


@pytest.mark.parametrize("pre", [0, 1, 2, 3, 5, 17])
def test_uniform_stream_bit_exact(cuda, pre):
    from paper_2503_20286_b200.variation import uniform_device

    a, b = philox_gen(9), philox_gen(9)
    a.random(pre)
    b.random(pre)
    got = uniform_device(a, (1001, 3)).cpu().numpy()
    assert np.array_equal(got, b.random((1001, 3)))
    assert np.array_equal(a.permutation(77), b.permutation(77))  # host stream continues identically


def test_sbx_pm_golden(cuda):
    from paper_2503_20286_b200.variation import VariationParams, pair_parents, polynomial_mutation, sbx

    z = load_golden("variation")
    d = 12
    rng = philox_gen(int(z["seed"]))
    i1, i2 = pair_parents(rng, 101)
    assert np.array_equal(i1, z["i1"]) and np.array_equal(i2, z["i2"])
    p = VariationParams(lower=np.zeros(d), upper=np.ones(d))
    kids = sbx(rng, z["X"][i1], z["X"][i2], p)
    # pow differs from NumPy's in the last ulp for a few inputs
    assert np.allclose(kids, z["kids"], rtol=1e-13, atol=1e-15)
    assert np.mean(kids == z["kids"]) > 0.9
    mut = polynomial_mutation(rng, z["kids"], p)
    assert np.allclose(mut, z["mut"], rtol=1e-13, atol=1e-15)
    rng = philox_gen(int(z["seed2"]))
    p2 = VariationParams(lower=np.full(6, -2.0), upper=np.full(6, 3.0), eta_c=5.0, eta_m=7.0, p_m=0.5,
                         gene_swap=False)
    kids2 = sbx(rng, z["X2"][:20], z["X2"][20:], p2)
    assert np.allclose(kids2, z["kids2"], rtol=1e-13, atol=1e-15)
    assert np.allclose(polynomial_mutation(rng, z["kids2"], p2), z["mut2"], rtol=1e-13, atol=1e-15)


def test_forced_rng_identities(cuda):
    """test_variation.py:49-145 identities through the injected-draw path."""
    from paper_2503_20286_b200.variation import VariationParams, polynomial_mutation, sbx

    p = VariationParams(lower=np.zeros(4), upper=np.ones(4))
    rng = np.random.default_rng(45)
    X1, X2 = rng.random((5, 4)), rng.random((5, 4))
    out = sbx(ForcedRng(0.5), X1, X2, p)
    assert np.array_equal(out[:5], X1) and np.array_equal(out[5:], X2)
    X = rng.random((6, 4))
    assert np.array_equal(polynomial_mutation(ForcedRng(0.5), X, p), X)
    p1 = VariationParams(lower=np.zeros(4), upper=np.ones(4), p_m=1.0)
    Z = np.zeros((4, 4))
    assert np.array_equal(polynomial_mutation(ForcedRng(0.3), Z, p1), Z)
    # identical parents are a fixed point; bounds respected; child-sum identity
    g = philox_gen(47)
    same = sbx(g, X, X.copy(), p)
    assert np.array_equal(same[:6], X) and np.array_equal(same[6:], X)
    wide = VariationParams(lower=np.full(4, -100.0), upper=np.full(4, 100.0))
    A, B = rng.random((20, 4)), rng.random((20, 4))
    c = sbx(philox_gen(46), A, B, wide)
    assert np.allclose(c[:20] + c[20:], A + B, rtol=0, atol=1e-12)


def test_evaluate_golden(cuda):
    from paper_2503_20286_b200.problems import evaluate, make_problem

    z = load_golden("problems")
    for key in z.files:
        if not key.endswith("_X"):
            continue
        name, mm = key.split("_")[:2]
        m = int(mm[1:])
        spec = make_problem(name, m=m)
        F = evaluate(spec, z[key])
        want = z[key[:-1] + "F"]
        assert np.allclose(F, want, rtol=1e-12, atol=1e-12), key  # north star: 1e-5 rel


@pytest.mark.parametrize("m,d", [(3, 1000), (2, 300), (5, 700)])
def test_lsmop1_vs_self_oracle(cuda, m, d):
    from paper_2503_20286_b200.problems import evaluate, make_problem

    spec = make_problem("lsmop1", m=m, d=d)
    d = spec.d  # PlatEMO's D for the requested dimension
    rng = np.random.default_rng(d)
    X = spec.lower + rng.random((200, d)) * (spec.upper - spec.lower)
    assert np.allclose(evaluate(spec, X), oprob.evaluate_lsmop1(X, m), rtol=1e-12, atol=0)


@pytest.mark.parametrize("k", range(2, 10))
@pytest.mark.parametrize("m,d", [(3, 1000), (2, 300), (5, 700)])
def test_lsmop_k_vs_self_oracle(cuda, k, m, d):
    """LSMOP2-9 (warp-per-row kernel) vs the PlatEMO-form NumPy restatement."""
    from paper_2503_20286_b200.problems import evaluate, make_problem

    spec = make_problem(f"lsmop{k}", m=m, d=d)
    d = spec.d
    rng = np.random.default_rng(d + k)
    X = spec.lower + rng.random((150, d)) * (spec.upper - spec.lower)
    X[:5, m - 1:] = 10.0 * X[:5, :1] / (1.0 + np.arange(m, d + 1) / d)  # linkage-optimal rows (k <= 4)
    want = oprob.evaluate_lsmop(k, X, m)
    got = evaluate(spec, X)
    assert np.allclose(got, want, rtol=1e-11, atol=1e-12 * np.abs(want).max())


def test_evaluate_rows_map(cuda):
    import torch

    from paper_2503_20286_b200 import _lib
    from paper_2503_20286_b200.problems import make_problem

    for name in ("dtlz2", "lsmop1", "lsmop7"):
        spec = make_problem(name, m=3, d=300 if name.startswith("lsmop") else 12)
        X = torch.from_numpy(spec.lower + np.random.default_rng(3).random((64, spec.d)) * (spec.upper - spec.lower)).cuda()
        rows = torch.from_numpy(np.random.default_rng(4).permutation(64)[:40].astype(np.int64)).cuda()
        F = torch.empty((40, 3), dtype=torch.float64, device="cuda")
        ps = spec.struct()
        assert _lib.lib().temo_evaluate_rows(_lib.sptr(ps), _lib.ptr(X), _lib.ptr(rows), 40, _lib.ptr(F),
                                             _lib.stream_handle(X.device)) == 0
        want = oprob.evaluate(name, X[rows].cpu().numpy(), 3)
        assert np.allclose(F.cpu().numpy(), want, rtol=1e-11, atol=0)


@pytest.mark.parametrize("name,m,d,n", [("dtlz1", 3, 12, 100), ("lsmop1", 3, 1000, 64), ("dtlz2", 5, 40, 33),
                                        ("lsmop3", 3, 1000, 64), ("lsmop9", 4, 400, 40)])
def test_fused_offspring_matches_oracle(cuda, name, m, d, n):
    import torch

    from paper_2503_20286_b200.harness import RunConfig, _Stepper
    from paper_2503_20286_b200.problems import make_problem
    from paper_2503_20286_b200.directions import das_dennis

    spec = make_problem(name, m=m, d=d)
    cfg = RunConfig(algorithm="nsga3", problem=name, objectives=m, dim=d, pop_size=n)
    d = spec.d
    st_ = _Stepper(cfg, spec, das_dennis(m, 4), n)
    g_dev, g_ref = philox_gen(3), philox_gen(3)
    state = st_.init(g_dev)
    X0 = g_ref.random((n, d))
    X0 = spec.lower + X0 * (spec.upper - spec.lower)
    assert np.array_equal(state.X.cpu().numpy(), X0)
    st_._offspring(state, g_dev)
    torch.cuda.synchronize()
    O_ref = ovar.offspring(g_ref, X0, 20.0, 20.0, None, spec.lower, spec.upper)
    h = n // 2
    O = st_.offspring_rows(state).cpu().numpy()
    assert np.allclose(O, O_ref, rtol=1e-13, atol=1e-13)
    FO = state.cur.F[n:n + 2 * h].cpu().numpy()
    assert np.allclose(FO, oprob.evaluate(name, O_ref, m), rtol=1e-10, atol=1e-12)
    assert np.array_equal(g_dev.permutation(50), g_ref.permutation(50))


def test_sbx_beta_fast_vs_numpy(cuda):
    """The exp/log SBX spread factor used by the fused offspring kernel (csrc/sbx_pow.cuh)
    against np.power on the reference's expression (variation.py:77-78): 10^6 Philox draws
    plus the edge cases of the U grid.  Bound: 4e-15 relative (the exp/log form loses about
    |e log(base)| ulp, up to 24 at eta_c = 0.5 and U = 2^-53; the offspring
    parity tests need 1e-13)."""
    import torch

    from paper_2503_20286_b200 import _lib

    u = np.random.default_rng(0).random(1_000_000)
    ulp = 2.0 ** -53
    edges = np.array([0.0, ulp, 2 * ulp, 0.25, 0.5 - ulp, 0.5, 0.5 + ulp, 0.75, 1 - 2 * ulp, 1 - ulp])
    mu = np.concatenate([edges, u])
    for eta_c in (20.0, 15.0, 2.0, 0.5):
        e = 1.0 / (eta_c + 1.0)
        want = np.where(0.5 - mu >= 0.0, np.power(2.0 * mu, e), np.power(1.0 / (2.0 - 2.0 * mu), e))
        d_mu = torch.from_numpy(mu).cuda()
        out = torch.empty_like(d_mu)
        for fast in (1, 0):
            rc = _lib.lib().temo_sbx_beta(_lib.ptr(d_mu), mu.size, eta_c, fast, _lib.ptr(out),
                                          _lib.stream_handle(d_mu.device))
            assert rc == 0
            got = out.cpu().numpy()
            rel = np.abs(got - want) / np.where(want == 0, 1.0, want)
            assert got[0] == 0.0 and np.all(np.isfinite(got))
            assert rel.max() < 4e-15, (eta_c, fast, rel.max())


@pytest.mark.parametrize("name,m,d,h,pre", [("lsmop1", 3, 1000, 40, 0), ("lsmop1", 3, 1000, 40, 3),
                                            ("lsmop1", 3, 1000, 517, 1), ("lsmop1", 5, 700, 33, 2),
                                            ("dtlz1", 3, 12, 50, 1), ("dtlz2", 5, 40, 16, 2),
                                            ("dtlz2", 3, 12, 1000, 3), ("dtlz7", 3, 13, 3, 0),
                                            ("lsmop6", 3, 1000, 40, 1), ("lsmop8", 5, 700, 33, 0)])
def test_offspring_two_phase_equals_fused(cuda, name, m, d, h, pre):
    """temo_offspring_ws (randomness kernel + streaming apply kernel, the harness path) gives
    bit-identical children to the fused temo_offspring for every stream alignment (``pre``
    shifts the host Generator's buffered words) and falls back to the fused kernel when
    h*d % 4 != 0; objectives are bit-identical too below d = 128 (same lane layout) and agree
    to 1e-13 above it (the gene-major apply kernel sums the groups in another order)."""
    import torch

    from paper_2503_20286_b200 import _lib
    from paper_2503_20286_b200.problems import make_problem
    from paper_2503_20286_b200.rng import DeviceDraws
    from paper_2503_20286_b200.variation import VariationParams

    spec = make_problem(name, m=m, d=d)
    d = spec.d
    dev = torch.device("cuda", 0)
    var = VariationParams(lower=spec.lower, upper=spec.upper).struct(d, dev)
    prob = spec.struct()
    gen = philox_gen(7)
    gen.random(pre)
    X = torch.from_numpy(spec.lower + np.random.default_rng(1).random((2 * h, d)) * (spec.upper - spec.lower)).to(dev)
    idx = torch.from_numpy(np.random.default_rng(2).permutation(2 * h).astype(np.int64)).to(dev)
    draws = DeviceDraws(gen)
    off = draws.take(7 * h * d)
    outs = []
    for path in ("fused", "ws-two-phase"):
        O = torch.full((2 * h, d), np.nan, dtype=torch.float64, device=dev)
        FO = torch.full((2 * h, m), np.nan, dtype=torch.float64, device=dev)
        L, s = _lib.lib(), _lib.stream_handle(dev)
        args = (_lib.sptr(prob), _lib.sptr(var), _lib.ptr(X), _lib.ptr(idx), _lib.ptr(idx[h:]), h,
                _lib.sptr(draws.state), off, _lib.ptr(O), _lib.ptr(FO))
        if path.startswith("ws"):
            ws = torch.empty(max(L.temo_offspring_ws_bytes(h, d), 256), dtype=torch.uint8, device=dev)
            rc = L.temo_offspring_ws(*args, None, None, _lib.ptr(ws), ws.numel(), s)
        else:
            rc = L.temo_offspring(*args, s)
        assert rc == 0
        outs.append((O.cpu().numpy(), FO.cpu().numpy()))
    (O1, F1) = outs[0]
    assert not np.isnan(O1).any() and not np.isnan(F1).any()
    for O2, F2 in outs[1:]:
        assert np.array_equal(O1, O2)
        if path_d := (d >= 128 and (h * d) % 4 == 0):  # gene-major apply kernel: sums in another order
            assert np.allclose(F1, F2, rtol=1e-13, atol=0), path_d
        else:
            assert np.array_equal(F1, F2)


@pytest.mark.parametrize("alg", ["nsga3", "hype"])
def test_row_pool_equals_survivor_copy(cuda, alg):
    """The harness keeps X in one row pool (temo_pool_update instead of the X[perm][keep]
    copy of nsga3.py:218 / hype.py:163).  Over several generations the pooled population
    equals (1) a torch restatement that materialises [X; O][perm][keep] every step and
    (2) the unpooled path (fused offspring kernel writing contiguous rows), bit for bit."""
    import torch

    from paper_2503_20286_b200.directions import das_dennis
    from paper_2503_20286_b200.harness import RunConfig, _Stepper
    from paper_2503_20286_b200.problems import make_problem

    name, m, d, n = "dtlz2", 3, 40, 64
    spec = make_problem(name, m=m, d=d)
    cfg = RunConfig(algorithm=alg, problem=name, objectives=m, dim=d, pop_size=n, hv_samples=4000)
    runs = []
    for unpooled in (False, True):
        st_ = _Stepper(cfg, spec, das_dennis(m, 6), n)
        st_.force_unpooled = unpooled
        captured = []
        orig = st_._offspring

        def offspring_and_capture(state, gen, orig=orig, st_=st_, captured=captured):
            orig(state, gen)
            captured.append(st_.offspring_rows(state).clone())

        st_._offspring = offspring_and_capture
        gen = philox_gen(11)
        state = st_.init(gen)
        X_ref = state.X.clone()
        traj = []
        for g in range(4):
            state, _ = st_.step(state, g, gen)
            merged = torch.cat([X_ref, captured[-1]])
            keep = st_.selector.keep.long()
            X_ref = merged[st_.perm][keep] if alg == "nsga3" else merged[keep]
            assert torch.equal(state.X, X_ref), (unpooled, g)
            traj.append((state.X.cpu().numpy(), state.F.cpu().numpy()))
        runs.append(traj)
    for (Xa, Fa), (Xb, Fb) in zip(*runs):
        assert np.array_equal(Xa, Xb) and np.array_equal(Fa, Fb)


@pytest.mark.parametrize("overlap", [0, 1])
def test_host_pipeline_and_overlap_equivalence(cuda, overlap):
    """The opt-in host-input pipeline (worker thread) and the side-stream randomness overlap
    give the sequential loop's populations and leave the Generator in the same state."""
    import json

    from paper_2503_20286_b200.harness import RunConfig, _resolve, _Stepper
    from paper_2503_20286_b200.rng import RngStream

    cfg = RunConfig(algorithm="nsga3", problem="lsmop1", objectives=3, dim=300, pop_size=400, seed=2)
    spec, R, n = _resolve(cfg)
    outs = []
    for mode in ("plain", "pipe"):
        st_ = _Stepper(cfg, spec, R, n)
        st_.overlap = overlap if mode == "pipe" else 0
        gen = RngStream(2).split(0).generator()
        st = st_.init(gen)
        if mode == "pipe":
            st_.start_host_pipeline(gen, 4)
        for g in range(4):
            st, _ = st_.step(st, g, gen, timed=False)
        X, F = st_.population(st)
        state = json.dumps(gen.bit_generator.state, default=lambda a: np.asarray(a).tolist())
        outs.append((X.cpu().numpy(), F.cpu().numpy(), state))
    assert np.array_equal(outs[0][0], outs[1][0]) and np.array_equal(outs[0][1], outs[1][1])
    assert outs[0][2] == outs[1][2]


def test_predrawn_overlap_priority_stream_equivalence(cuda):
    """bench.py's device-resident loop (pre-drawn inputs, the next generation's randomness on the
    low-priority side stream while this one runs on the high-priority stream) gives the plain
    loop's populations bit for bit (pop 3000: units of several CTAs in flight at once)."""
    import torch

    from paper_2503_20286_b200.harness import RunConfig, _resolve, _Stepper
    from paper_2503_20286_b200.rng import RngStream

    cfg = RunConfig(algorithm="nsga3", problem="lsmop1", objectives=3, dim=500, pop_size=3000, seed=5)
    spec, R, n = _resolve(cfg)
    outs = []
    for overlap in (0, 1):
        st_ = _Stepper(cfg, spec, R, n)
        st_.overlap = overlap
        gen = RngStream(5).split(0).generator()
        st = st_.init(gen)
        K = 5
        pre = st_.upload_host_inputs([st_.draw_host_inputs(gen) for _ in range(K)])
        for g in range(K):
            st, _ = st_.step(st, g, gen, timed=False, pre=pre[g], pre_next=pre[g + 1] if g + 1 < K else None)
        torch.cuda.synchronize()
        st_.check()
        X, F = st_.population(st)
        outs.append((X.cpu().numpy(), F.cpu().numpy()))
    assert np.array_equal(outs[0][0], outs[1][0]) and np.array_equal(outs[0][1], outs[1][1])
