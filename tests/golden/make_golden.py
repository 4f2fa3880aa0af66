"""Generate golden vectors by running the REAL reference (``temo`` 0.1.0) in the build container.

Usage (build container only -- /root/reference does not exist on the GPU box):

    OPENBLAS_NUM_THREADS=1 python tests/golden/make_golden.py

Writes ``tests/golden/*.npz``.  Single-threaded OpenBLAS is required: the
reference's HypE bits depend on the BLAS thread count.
Stochastic inputs are recorded from a ``RecordingRng`` proxy (App. B) so the
tests can replay them exactly; large uniform blocks are not stored, only the
Philox seed that regenerates them.
"""

from __future__ import annotations

import os
import sys
from pathlib import Path

os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
REF = Path("/root/reference/pkg/src")
sys.path.insert(0, str(REF))

import numpy as np  # noqa: E402

from temo import directions, hype, moead, ndsort, nsga3, problems, variation  # noqa: E402
from temo.harness import RunConfig, _resolve, _Stepper  # noqa: E402
from temo.rng import RngStream  # noqa: E402

OUT = Path(__file__).resolve().parent


class RecordingRng:
    """Forward to a Generator and log every call's result."""

    def __init__(self, gen):
        self.gen = gen
        self.log = []

    def permutation(self, n):
        v = self.gen.permutation(n)
        self.log.append(("permutation", v))
        return v

    def random(self, size=None):
        v = self.gen.random(size)
        self.log.append(("random", v))
        return v

    def integers(self, low, high=None, size=None):
        v = self.gen.integers(low, high, size=size)
        self.log.append(("integers", v))
        return v


def pack(arrs, dtype):
    flat = np.concatenate([np.asarray(a, dtype=dtype).ravel() for a in arrs]) if arrs else np.zeros(0, dtype)
    off = np.concatenate([[0], np.cumsum([np.asarray(a).size for a in arrs])]).astype(np.int64)
    return flat, off


def gen_ndsort():
    Fs, Ns, ms, ns, rs, ls = [], [], [], [], [], []

    def add(F, n):
        res = ndsort.rank_assign(F, n)
        Fs.append(F)
        Ns.append(F.shape[0])
        ms.append(F.shape[1])
        ns.append(n)
        rs.append(res.r)
        ls.append(res.l)

    rng = np.random.default_rng(62)  # test_ndsort.py:47-57 generator
    for _ in range(200):
        N = int(rng.integers(2, 64))
        m = int(rng.integers(2, 6))
        F = rng.integers(0, 5, size=(N, m)).astype(float)
        add(F, int(rng.integers(1, N + 1)))
    rng = np.random.default_rng(1000)  # SPEC acceptance #1 style extra instances
    for _ in range(300):
        N = int(rng.integers(2, 200))
        m = int(rng.integers(2, 11))
        kind = rng.integers(0, 3)
        if kind == 0:
            F = rng.integers(0, 4, size=(N, m)).astype(float)
        elif kind == 1:
            F = rng.random((N, m))
        else:
            F = np.round(rng.random((N, m)), 1) * rng.choice([-1.0, 1.0], size=(N, m))
        add(F, int(rng.integers(1, N + 1)))
    # signed zeros and infinities
    add(np.array([[0.0, 1.0], [-0.0, 1.0], [np.inf, -np.inf], [1.0, 0.0], [-np.inf, 2.0]]), 3)
    for N, m, seed in ((1500, 3, 1), (1200, 5, 2), (800, 8, 3), (2000, 2, 4)):
        r = np.random.default_rng(seed)
        add(r.random((N, m)), N // 2)
    spec = problems.make_problem("dtlz1", m=3, d=30)
    X = np.random.default_rng(7).random((2000, 30))
    add(problems.evaluate(spec, X), 1000)
    F, Foff = pack([f.ravel() for f in Fs], np.float64)
    r, roff = pack(rs, np.int64)
    np.savez_compressed(OUT / "ndsort.npz", F=F, F_off=Foff, N=np.array(Ns), m=np.array(ms),
                        n=np.array(ns), r=r, r_off=roff, l=np.array(ls))


def selection_case(Fm, Xm, R, n, perm):
    """Run nsga3.environmental_selection's internals on an injected permutation."""
    Fs = Fm[perm]
    res = ndsort.rank_assign(Fs, n)
    masked = Fs.copy()
    masked[res.r > res.l] = np.nan
    norm = nsga3.normalize(masked)
    assoc = nsga3.associate(norm.Fp, R)
    state = nsga3.niche_counts(res.r, assoc.pi, res.l, R.count)
    picked = nsga3.niche_select(state, res.r, assoc.pi, assoc.dist, res.l, n)
    rank = nsga3.update_rank(picked.rank, picked.promoted, n - picked.n_selected, res.l)
    keep = np.flatnonzero(rank < res.l)

    class Planned:
        def permutation(self, N):
            return perm.copy()

    Xs, Fsel = nsga3.environmental_selection(Xm, Fm, R, n, Planned())
    assert np.array_equal(Fsel, Fs[keep])
    return dict(F=Fm, W=R.W, n=n, perm=perm, r=res.r, l=res.l, Fp=norm.Fp, ideal=norm.ideal,
                intercepts=norm.intercepts, pi=assoc.pi, dist=assoc.dist, promoted=picked.promoted,
                rank=rank, keep=keep)


def gen_nsga3():
    cases = []
    # config A inputs: merged population of the reference harness, DTLZ1 m=3 d=12 pop 100
    cfg = RunConfig(algorithm="nsga3", problem="dtlz1", objectives=3, dim=12, pop_size=100, seed=0)
    spec, R, n = _resolve(cfg)
    st = _Stepper(cfg, spec, R, n)
    gen = RngStream(0).split(0).generator()
    X, F = st.init(gen)
    captured = []
    real = nsga3.environmental_selection

    def spy(Xm, Fm, R_, n_, rng):
        captured.append((Xm.copy(), Fm.copy()))
        return real(Xm, Fm, R_, n_, rng)

    nsga3.environmental_selection = spy
    try:
        state = (X, F)
        for g in range(1, 31):
            state, _ = st.step(state, g, gen)
    finally:
        nsga3.environmental_selection = real
    pr = np.random.default_rng(11)
    for g in (0, 1, 9, 29):
        Xm, Fm = captured[g]
        cases.append(selection_case(Fm, Xm, R, n, pr.permutation(Fm.shape[0])))
    # random objective clouds, several m and lattice sizes
    for seed, (N, m, H, n) in enumerate(((600, 3, 12, 300), (1000, 3, 23, 500), (400, 2, 40, 200),
                                         (500, 4, 7, 250), (300, 5, 5, 150), (400, 8, 3, 200),
                                         (300, 10, 3, 150))):
        r = np.random.default_rng(100 + seed)
        Fm = r.random((N, m)) ** 2
        cases.append(selection_case(Fm, np.zeros((N, 1)), directions.das_dennis(m, H), n,
                                    r.permutation(N)))
    # heavy ties: integer grid objectives; and DTLZ2 objectives
    r = np.random.default_rng(200)
    Fm = r.integers(0, 6, size=(400, 3)).astype(float)
    cases.append(selection_case(Fm, np.zeros((400, 1)), directions.das_dennis(3, 6), 200, r.permutation(400)))
    spec2 = problems.make_problem("dtlz2", m=3)
    Fm = problems.evaluate(spec2, r.random((1200, spec2.d)))
    cases.append(selection_case(Fm, np.zeros((1200, 1)), directions.das_dennis(3, 33), 600, r.permutation(1200)))
    # many objectives with well-conditioned extremes: the hyperplane (np.linalg.solve) branch at
    # m = 6, 8, 10 (OpenBLAS getf2) and 12 (blocked getrf), not the nadir fallback
    for k, (N, m, H, n) in enumerate(((400, 6, 4, 200), (400, 8, 3, 200), (360, 10, 3, 180), (300, 12, 2, 150))):
        r2 = np.random.default_rng(500 + k)
        Fm = r2.dirichlet(np.ones(m), N) * (1.0 + 0.5 * r2.random((N, 1))) + 1e-3 * r2.random((N, m))
        c = selection_case(Fm, np.zeros((N, 1)), directions.das_dennis(m, H), n, r2.permutation(N))
        live = c["r"] <= c["l"]
        fallback = np.maximum(np.nanmax(Fm[c["perm"]][live], axis=0), 1e-10)
        assert not np.array_equal(c["intercepts"], fallback), "expected the solve branch"
        cases.append(c)
    # degenerate extremes -> fallback intercepts
    Fm = np.repeat(np.array([[1.0, 1.0, 1.0], [2.0, 2.0, 2.0]]), 30, axis=0) + np.linspace(0, 1e-3, 60)[:, None]
    cases.append(selection_case(Fm, np.zeros((60, 1)), directions.das_dennis(3, 4), 30, r.permutation(60)))
    out = {}
    for i, c in enumerate(cases):
        for k, v in c.items():
            out[f"c{i}_{k}"] = np.asarray(v)
    out["count"] = np.array(len(cases))
    np.savez_compressed(OUT / "nsga3.npz", **out)


def gen_linalg():
    """np.linalg.solve(E, ones) bits (nsga3.py:86) for m = 2..16: random and NSGA-III-shaped E
    (extreme points of shifted objectives: nonnegative, dominant diagonal).  m <= 9 is OpenBLAS's
    unblocked getf2; m >= 10 its blocked getrf_single."""
    r = np.random.default_rng(300)
    Es, ys, ms = [], [], []
    for k in range(3000 + 15 * 240):
        m = int(r.integers(2, 6)) if k < 3000 else 2 + (k - 3000) // 240
        E = r.random((m, m)) * r.choice([1e-3, 1.0, 1e3])
        if r.random() < 0.3:
            E = E + np.diag(r.random(m)) * 5
        if k >= 3000 and (k % 3) == 0:  # extreme-point shaped: near-diagonal, scaled axes
            E = np.diag(1.0 + r.random(m) * 10) + r.random((m, m)) * 1e-3 * r.choice([1.0, 10.0, 100.0])
        Es.append(E)
        ys.append(np.linalg.solve(E, np.ones(m)))
        ms.append(m)
    E, Eoff = pack(Es, np.float64)
    y, yoff = pack(ys, np.float64)
    np.savez_compressed(OUT / "linalg.npz", E=E, E_off=Eoff, y=y, y_off=yoff, m=np.array(ms))


def gen_associate():
    out = {}
    r = np.random.default_rng(400)
    for i, (m, H, N) in enumerate(((3, 20, 3000), (3, 99, 400), (4, 8, 800), (5, 6, 600),
                                   (8, 3, 500), (10, 3, 400), (2, 50, 500))):
        R = directions.das_dennis(m, H)
        Fp = r.random((N, m)) * r.choice([0.5, 2.0])
        Fp[::37] = np.nan
        Fp[5] = 0.0
        a = nsga3.associate(Fp, R)
        out[f"c{i}_Fp"], out[f"c{i}_W"], out[f"c{i}_pi"], out[f"c{i}_dist"] = Fp, R.W, a.pi, a.dist
    out["count"] = np.array(7)
    np.savez_compressed(OUT / "associate.npz", **out)


def gen_hype():
    out = {}
    cases = []
    for N, m, n, s, seed in ((400, 3, 200, 20000, 1), (401, 3, 200, 70000, 2), (402, 3, 200, 5000, 3),
                             (403, 3, 200, 8193, 4), (200, 2, 100, 65537, 5), (150, 4, 75, 12345, 6),
                             (1000, 3, 500, 100000, 7)):
        r = np.random.default_rng(500 + seed)
        spec = problems.make_problem("dtlz2", m=m)
        F = problems.evaluate(spec, r.random((N, spec.d)))
        if seed == 3:
            F = np.round(F, 1)  # ties between points and with box samples
        X = r.random((N, 2))
        res = ndsort.rank_assign(F, n)
        k = int((res.r <= res.l).sum()) - n
        rec = RecordingRng(np.random.Generator(np.random.Philox(np.random.SeedSequence(seed))))
        Xk, Fk = hype.environmental_selection(X, F, None, n, s, rec)
        # recompute v_hv directly with the recorded samples to store it
        v_hv = np.zeros(N)
        if k >= 1:
            ref = hype.auto_reference(F)
            v_hv = hype.hv_estimate(F, hype.HvEstimateParams(ref, k, s),
                                    np.random.Generator(np.random.Philox(np.random.SeedSequence(seed))))
        d = np.where(res.r <= res.l, v_hv, -np.finfo(float).max)
        keep = np.lexsort((np.arange(N), -d, res.r))[:n]
        assert np.array_equal(Fk, F[keep])
        cases.append(dict(F=F, n=n, s=s, seed=seed, r=res.r, l=res.l, k=k, v_hv=v_hv, keep=keep))
    for i, c in enumerate(cases):
        for key, v in c.items():
            out[f"c{i}_{key}"] = np.asarray(v)
    # shared_alpha pins
    for j, (n1, k) in enumerate(((10, 3), (2000, 381), (20000, 381), (5, 5), (1, 1))):
        out[f"alpha{j}"] = hype.shared_alpha(n1, k)
        out[f"alpha{j}_nk"] = np.array([n1, k])
    out["count"] = np.array(len(cases))
    out["alpha_count"] = np.array(5)
    np.savez_compressed(OUT / "hype.npz", **out)


def gen_variation():
    out = {}
    d = 12
    lo, hi = np.zeros(d), np.ones(d)
    r = np.random.default_rng(600)
    X = r.random((101, d))
    p = variation.VariationParams(lower=lo, upper=hi)
    gen = np.random.Generator(np.random.Philox(np.random.SeedSequence(61)))
    i1, i2 = variation.pair_parents(gen, 101)
    kids = variation.sbx(gen, X[i1], X[i2], p)
    mut = variation.polynomial_mutation(gen, kids, p)
    out.update(X=X, i1=i1, i2=i2, kids=kids, mut=mut, seed=np.array(61))
    p2 = variation.VariationParams(lower=np.full(6, -2.0), upper=np.full(6, 3.0), eta_c=5.0, eta_m=7.0,
                                   p_m=0.5, gene_swap=False)
    gen = np.random.Generator(np.random.Philox(np.random.SeedSequence(62)))
    X2 = r.random((40, 6)) * 5 - 2
    kids2 = variation.sbx(gen, X2[:20], X2[20:], p2)
    mut2 = variation.polynomial_mutation(gen, kids2, p2)
    out.update(X2=X2, kids2=kids2, mut2=mut2, seed2=np.array(62))
    np.savez_compressed(OUT / "variation.npz", **out)


def gen_problems():
    out = {}
    r = np.random.default_rng(700)
    for name in problems._NAMES:
        for m in (2, 3, 5):
            spec = problems.make_problem(name, m=m)
            X = r.random((64, spec.d))
            X[0] = 0.0
            X[1] = 1.0
            X[2, m - 1:] = 0.5
            out[f"{name}_m{m}_X"] = X
            out[f"{name}_m{m}_F"] = problems.evaluate(spec, X)
    np.savez_compressed(OUT / "problems.npz", **out)


def gen_moead():
    out = {}
    for i, (name, m, H, T, d, seed) in enumerate((("dtlz2", 3, 12, 10, 12, 1), ("dtlz1", 3, 20, 20, 7, 2),
                                                  ("dtlz2", 2, 60, 6, 10, 3))):
        spec = problems.make_problem(name, m=m, d=d)
        ds = directions.das_dennis(m, H)
        table = directions.neighbors(ds, T)
        r = np.random.default_rng(800 + seed)
        X = r.random((ds.count, d))
        F1 = problems.evaluate(spec, X)
        st = moead.init_state(X, F1, ds.W, table)
        params = variation.VariationParams(lower=spec.lower, upper=spec.upper)
        # a few steps to make the state non-trivial, then record one step
        gen = np.random.Generator(np.random.Philox(np.random.SeedSequence(seed)))
        for _ in range(3):
            st = moead.step(st, gen, params, lambda A: problems.evaluate(spec, A))
        state_before = gen.bit_generator.state
        rec = RecordingRng(gen)
        O, F2 = moead.moead_offspring(st, rec, params, lambda A: problems.evaluate(spec, A))
        upd, z_min = moead.compare_update(st, F2)
        Xn, Fn = moead.elite_select(st, O, F2, upd, z_min)
        ints = [v for kind, v in rec.log if kind == "integers"]
        out.update({f"c{i}_X": st.X, f"c{i}_F1": st.F1, f"c{i}_z": st.z, f"c{i}_W": st.W,
                    f"c{i}_I_nb": st.I_nb, f"c{i}_O": O, f"c{i}_F2": F2, f"c{i}_z_min": z_min,
                    f"c{i}_Xn": Xn, f"c{i}_Fn": Fn, f"c{i}_pick1": ints[0], f"c{i}_pick2": ints[1],
                    f"c{i}_improves": (upd.I_new[np.repeat(np.arange(ds.count), T), st.I_nb.ravel()] == -1).reshape(ds.count, T),
                    f"c{i}_seed": np.array(seed), f"c{i}_name": np.array(name), f"c{i}_d": np.array(d),
                    f"c{i}_counter": state_before["state"]["counter"], f"c{i}_key": state_before["state"]["key"],
                    f"c{i}_buffer": state_before["buffer"], f"c{i}_buffer_pos": np.array(state_before["buffer_pos"])})
    out["count"] = np.array(3)
    np.savez_compressed(OUT / "moead.npz", **out)


def gen_hype_c():
    """HypE at BASELINE config C: DTLZ2 m=3, merged N = 20k, n = 10k, s = 100k samples
    (hype.py:54-163 at the workload size; rank_assign, auto reference, hv_estimate, lexsort)."""
    seed = 77
    r = np.random.default_rng(900)
    spec = problems.make_problem("dtlz2", m=3)
    N, n, s = 20000, 10000, 100000
    F = problems.evaluate(spec, r.random((N, spec.d)))
    res = ndsort.rank_assign(F, n)
    k = int((res.r <= res.l).sum()) - n
    ref = hype.auto_reference(F)
    v_hv = hype.hv_estimate(F, hype.HvEstimateParams(ref, k, s),
                            np.random.Generator(np.random.Philox(np.random.SeedSequence(seed))))
    d = np.where(res.r <= res.l, v_hv, -np.finfo(float).max)
    keep = np.lexsort((np.arange(N), -d, res.r))[:n]
    np.savez_compressed(OUT / "hype_c.npz", F=F, n=np.array(n), s=np.array(s), seed=np.array(seed), r=res.r.astype(np.int32),
                        l=np.array(res.l), k=np.array(k), v_ref=ref, v_hv=v_hv, keep=keep.astype(np.int32))


def gen_moead_b():
    """MOEA/D at BASELINE config B: DTLZ2 m=3 d=12, das_dennis(3, 139) -> n = 9870, T = 20,
    PBI theta = 5; one recorded step after one warm-up step (moead.py:70-158)."""
    spec = problems.make_problem("dtlz2", m=3, d=12)
    ds = directions.das_dennis(3, 139)
    table = directions.neighbors(ds, 20)
    r = np.random.default_rng(901)
    X = r.random((ds.count, spec.d))
    F1 = problems.evaluate(spec, X)
    st = moead.init_state(X, F1, ds.W, table)
    params = variation.VariationParams(lower=spec.lower, upper=spec.upper)
    gen = np.random.Generator(np.random.Philox(np.random.SeedSequence(42)))
    st = moead.step(st, gen, params, lambda A: problems.evaluate(spec, A))
    state_before = gen.bit_generator.state
    rec = RecordingRng(gen)
    O, F2 = moead.moead_offspring(st, rec, params, lambda A: problems.evaluate(spec, A))
    upd, z_min = moead.compare_update(st, F2)
    Xn, Fn = moead.elite_select(st, O, F2, upd, z_min)
    ints = [v for kind, v in rec.log if kind == "integers"]
    n, T = ds.count, 20
    improves = (upd.I_new[np.repeat(np.arange(n), T), st.I_nb.ravel()] == -1).reshape(n, T)
    np.savez_compressed(OUT / "moead_b.npz", X=st.X, F1=st.F1, z=st.z, I_nb=st.I_nb.astype(np.int16),
                        O=O, F2=F2, z_min=z_min, Xn=Xn, Fn=Fn, pick1=np.asarray(ints[0]).astype(np.int8),
                        pick2=np.asarray(ints[1]).astype(np.int8), improves=improves,
                        counter=state_before["state"]["counter"], key=state_before["state"]["key"],
                        buffer=state_before["buffer"], buffer_pos=np.array(state_before["buffer_pos"]),
                        has_uint32=np.array(state_before["has_uint32"]), uinteger=np.array(state_before["uinteger"]))


def gen_neighbors():
    out = {}
    for i, (m, H, T) in enumerate(((3, 12, 10), (3, 30, 20), (2, 99, 7), (4, 6, 15))):
        ds = directions.das_dennis(m, H)
        out[f"c{i}_W"] = ds.W
        out[f"c{i}_I"] = directions.neighbors(ds, T).I_nb
    out["count"] = np.array(4)
    np.savez_compressed(OUT / "neighbors.npz", **out)


def gen_config_a():
    """Config A end-to-end reference trajectory summary (seed 0, 100 gens)."""
    from temo.harness import run
    cfg = RunConfig(algorithm="nsga3", problem="dtlz1", objectives=3, dim=12, pop_size=100,
                    generations=100, seed=0, indicators=("igd",))
    rec = run(cfg)
    rows = rec.repeats[0].rows
    np.savez_compressed(OUT / "config_a.npz", igd=np.array([r.igd for r in rows]),
                        ideal=np.array([r.ideal for r in rows]),
                        final_igd=np.array(rec.repeats[0].final_igd))


def gen_config_a_traj():
    """Config A trajectory, every generation (harness.py:206-248, seed 0, 100 gens): the merged
    objectives handed to environmental_selection, the shuffle it drew and the objectives it kept,
    so each generation's selection can be replayed bit for bit on the reference's own inputs."""
    cfg = RunConfig(algorithm="nsga3", problem="dtlz1", objectives=3, dim=12, pop_size=100, seed=0)
    spec, R, n = _resolve(cfg)
    st = _Stepper(cfg, spec, R, n)
    gen = RngStream(0).split(0).generator()
    X, F = st.init(gen)
    Fms, perms, Fsel = [], [], []
    real = nsga3.environmental_selection

    def spy(Xm, Fm, R_, n_, rng):
        rec = RecordingRng(rng)
        Xs, Fs = real(Xm, Fm, R_, n_, rec)
        Fms.append(Fm.copy())
        perms.append(np.asarray([v for kind, v in rec.log if kind == "permutation"][0]))
        Fsel.append(Fs.copy())
        return Xs, Fs

    nsga3.environmental_selection = spy
    try:
        state = (X, F)
        for g in range(1, 101):
            state, _ = st.step(state, g, gen)
    finally:
        nsga3.environmental_selection = real
    np.savez_compressed(OUT / "config_a_traj.npz", Fm=np.stack(Fms), perm=np.stack(perms).astype(np.int16),
                        Fsel=np.stack(Fsel), W=R.W, n=np.array(n))


def gen_indicators():
    """indicators.py:19-100 values from the reference: igd, exact hv (m = 2, 3), Monte-Carlo hv
    (m = 4, default seeded rng), eu (both readings), on DTLZ fronts and random clouds."""
    from temo import indicators

    out = {}
    r = np.random.default_rng(950)
    cases = []
    for k, (name, m, n) in enumerate((("dtlz2", 3, 120), ("dtlz1", 3, 300), ("dtlz2", 2, 90), ("dtlz2", 4, 60),
                                      ("dtlz1", 2, 200), ("dtlz2", 3, 1000))):
        spec = problems.make_problem(name, m=m)
        F = problems.evaluate(spec, r.random((n, spec.d)))
        if k == 4:
            F[:20] = F[20:40]  # duplicate rows
            F[40:50, 0] = F[50:60, 0]  # shared x coordinates
        front = problems.true_front(spec, 200 if m <= 3 else 100)
        ref = 1.1 * front.max(axis=0)
        ref[ref <= 0] = 1e-6
        W = directions.das_dennis(m, 5 if m <= 3 else 3)
        c = dict(F=F, front=front, ref=ref, W=W.W, igd=indicators.igd(F, front),
                 hv=indicators.hv_indicator(F, ref), eu=indicators.eu(F, W), eu_lit=indicators.eu(F, W, literal=True),
                 eu_max=indicators.eu(F, W, maximize=True))
        cases.append(c)
    for i, c in enumerate(cases):
        for key, v in c.items():
            out[f"c{i}_{key}"] = np.asarray(v)
    out["count"] = np.array(len(cases))
    np.savez_compressed(OUT / "indicators.npz", **out)


def gen_rvea():
    """rvea.apd_select (rvea.py:33-68): SPEC acceptance #5 shapes (n <= 32, r <= 16, t = 0 and
    theta = 0 cases) plus DTLZ-sized instances; winners as row indices."""
    from temo import rvea

    out = {}
    r = np.random.default_rng(960)
    cases = []
    for k in range(80):
        m = int(r.integers(2, 5))
        H = int(r.integers(1, 5))
        V = directions.das_dennis(m, H)
        n = int(r.integers(1, 33))
        F = r.random((n, m))
        if k % 5 == 0:  # rows collinear with a direction (theta = 0)
            j = int(r.integers(0, V.count))
            F[: max(n // 3, 1)] = V.W[j] * r.random((max(n // 3, 1), 1)) * 2 + F.min(axis=0)
        t_max = int(r.integers(1, 100))
        t = 0 if k % 7 == 0 else int(r.integers(0, t_max + 1))
        alpha = float(r.choice([1.0, 2.0, 3.5]))
        X = np.arange(n, dtype=float)[:, None]
        Xw, Fw = rvea.apd_select(X, F, V, rvea.ApdParams(alpha, t, t_max))
        cases.append(dict(F=F, W=V.W, t=t, t_max=t_max, alpha=alpha, keep=Xw[:, 0].astype(np.int64)))
    for k, (name, m, H, n) in enumerate((("dtlz2", 3, 12, 182), ("dtlz1", 3, 23, 600), ("dtlz2", 5, 4, 140))):
        spec = problems.make_problem(name, m=m)
        V = directions.das_dennis(m, H)
        F = problems.evaluate(spec, r.random((n, spec.d)))
        X = np.arange(n, dtype=float)[:, None]
        Xw, Fw = rvea.apd_select(X, F, V, rvea.ApdParams(2.0, 37, 100))
        cases.append(dict(F=F, W=V.W, t=37, t_max=100, alpha=2.0, keep=Xw[:, 0].astype(np.int64)))
    for i, c in enumerate(cases):
        for key, v in c.items():
            out[f"c{i}_{key}"] = np.asarray(v)
    out["count"] = np.array(len(cases))
    np.savez_compressed(OUT / "rvea.npz", **out)


def gen_exact_hype():
    """hype.exact_hype_fitness_oracle (hype.py:88-126) on small instances (n1 <= 8, m <= 3)."""
    out = {}
    r = np.random.default_rng(970)
    cases = []
    for k in range(12):
        n1, m = int(r.integers(2, 9)), int(r.integers(2, 4))
        F = np.round(r.random((n1, m)), 2)
        ref = F.max(axis=0) + 0.1
        kk = int(r.integers(1, n1 + 1))
        fit, sec = hype.exact_hype_fitness_oracle(F, ref, kk, moments=True)
        cases.append(dict(F=F, ref=ref, k=kk, fit=fit, sec=sec))
    for i, c in enumerate(cases):
        for key, v in c.items():
            out[f"c{i}_{key}"] = np.asarray(v)
    out["count"] = np.array(len(cases))
    np.savez_compressed(OUT / "exact_hype.npz", **out)


if __name__ == "__main__":
    wanted = set(sys.argv[1:])  # e.g. "gen_linalg": regenerate only those sets
    for fn in (gen_ndsort, gen_nsga3, gen_linalg, gen_associate, gen_hype, gen_variation, gen_problems,
               gen_moead, gen_neighbors, gen_config_a, gen_hype_c, gen_moead_b, gen_config_a_traj,
               gen_indicators, gen_rvea, gen_exact_hype):
        if wanted and fn.__name__ not in wanted:
            continue
        fn()
        print("wrote", fn.__name__)
