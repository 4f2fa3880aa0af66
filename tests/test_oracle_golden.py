"""Pin the CPU oracle against golden vectors produced by the real reference (CPU-only)."""

import numpy as np
import pytest

from conftest import cases, load_golden, unpack
from oracle import directions, hype, moead, ndsort, nsga3, problems, variation


def test_ndsort_golden():
    z = load_golden("ndsort")
    for i in range(len(z["N"])):
        N, m, n = int(z["N"][i]), int(z["m"][i]), int(z["n"][i])
        F = unpack(z["F"], z["F_off"], i).reshape(N, m)
        want_r = unpack(z["r"], z["r_off"], i)
        if N <= 2000:
            r, l = ndsort.rank_assign(F, n)
            assert np.array_equal(r, want_r) and l == int(z["l"][i])
        r2, l2 = ndsort.rank_fast(F, n)
        assert np.array_equal(r2, want_r) and l2 == int(z["l"][i])


def test_ndsort_loop_matches_on_small():
    z = load_golden("ndsort")
    for i in range(60):
        N, m, n = int(z["N"][i]), int(z["m"][i]), int(z["n"][i])
        F = unpack(z["F"], z["F_off"], i).reshape(N, m)
        r, l = ndsort.rank_loop(F, n)
        assert np.array_equal(r, unpack(z["r"], z["r_off"], i)) and l == int(z["l"][i])


def test_lu_solve_matches_lapack_bits():
    """np.linalg.solve bits (OpenBLAS getf2 for m <= 9, blocked getrf for m >= 10) for m = 2..16."""
    z = dict(load_golden("linalg"))  # decompress once
    bad = 0
    for i in range(len(z["m"])):
        m = int(z["m"][i])
        E = unpack(z["E"], z["E_off"], i).reshape(m, m)
        y = nsga3.solve_ones(E)
        bad += not np.array_equal(y, unpack(z["y"], z["y_off"], i))
    assert bad == 0
    assert set(np.unique(z["m"]).tolist()) == set(range(2, 17))


def test_associate_golden():
    z = load_golden("associate")
    for c in cases(z):
        pi, dist = nsga3.associate(c["Fp"], c["W"])
        assert np.array_equal(pi, c["pi"])
        assert np.array_equal(dist, c["dist"], equal_nan=True)


@pytest.mark.parametrize("idx", range(18))
def test_nsga3_selection_golden(idx):
    z = load_golden("nsga3")
    cs = cases(z)
    c = cs[idx]
    Fs = c["F"][c["perm"]]
    out = nsga3.select_shuffled(Fs, c["W"], int(c["n"]))
    assert np.array_equal(out["r"], c["r"]) and out["l"] == int(c["l"])
    assert np.array_equal(out["ideal"], c["ideal"])
    assert np.array_equal(out["intercepts"], c["intercepts"])
    assert np.array_equal(out["Fp"], c["Fp"], equal_nan=True)
    assert np.array_equal(out["pi"], c["pi"])
    if Fs.shape[1] <= 4:
        assert np.array_equal(out["dist"], c["dist"], equal_nan=True)
    else:  # m >= 5: dgemm edge-kernel columns (n_r mod 8) within tolerance
        assert np.allclose(out["dist"], c["dist"], rtol=1e-12, atol=0, equal_nan=True)
    assert np.array_equal(out["promoted"], c["promoted"])
    assert np.array_equal(out["keep"], c["keep"])


def test_hype_alpha_golden():
    z = load_golden("hype")
    for j in range(int(z["alpha_count"])):
        n1, k = z[f"alpha{j}_nk"]
        assert np.array_equal(hype.shared_alpha(int(n1), int(k)), z[f"alpha{j}"])


@pytest.mark.parametrize("idx", range(7))
def test_hype_selection_golden(idx):
    c = cases(load_golden("hype"))[idx]
    seed = int(c["seed"])
    rng = np.random.Generator(np.random.Philox(np.random.SeedSequence(seed)))
    out = hype.select(c["F"], None, int(c["n"]), int(c["s"]), rng)
    assert np.array_equal(out["r"], c["r"]) and out["k"] == int(c["k"])
    assert np.array_equal(out["v_hv"], c["v_hv"])
    assert np.array_equal(out["keep"], c["keep"])


def test_variation_golden():
    z = load_golden("variation")
    d = 12
    rng = np.random.Generator(np.random.Philox(np.random.SeedSequence(int(z["seed"]))))
    i1, i2 = variation.pair_parents(rng, 101)
    assert np.array_equal(i1, z["i1"]) and np.array_equal(i2, z["i2"])
    X = z["X"]
    kids = variation.sbx(rng, X[i1], X[i2], 20.0, np.zeros(d), np.ones(d))
    assert np.array_equal(kids, z["kids"])
    mut = variation.polynomial_mutation(rng, kids, 20.0, 1.0 / d, np.zeros(d), np.ones(d))
    assert np.array_equal(mut, z["mut"])
    rng = np.random.Generator(np.random.Philox(np.random.SeedSequence(int(z["seed2"]))))
    X2 = z["X2"]
    lo, hi = np.full(6, -2.0), np.full(6, 3.0)
    kids2 = variation.sbx(rng, X2[:20], X2[20:], 5.0, lo, hi, gene_swap=False)
    assert np.array_equal(kids2, z["kids2"])
    assert np.array_equal(variation.polynomial_mutation(rng, kids2, 7.0, 0.5, lo, hi), z["mut2"])


def test_problems_golden():
    z = load_golden("problems")
    for key in z.files:
        if not key.endswith("_X"):
            continue
        name, mm = key.split("_")[:2]
        m = int(mm[1:])
        F = problems.evaluate(name, z[key], m)
        assert np.array_equal(F, z[key[:-1] + "F"]), key


def test_moead_golden():
    for c in cases(load_golden("moead")):
        name, d = str(c["name"]), int(c["d"])
        lo, hi = np.zeros(d), np.ones(d)
        gen = np.random.Generator(np.random.Philox())
        st = gen.bit_generator.state
        st["state"]["counter"] = c["counter"]
        st["state"]["key"] = c["key"]
        st["buffer"] = c["buffer"]
        st["buffer_pos"] = int(c["buffer_pos"])
        gen.bit_generator.state = st
        m = c["W"].shape[1]
        O = moead.offspring(c["X"], c["I_nb"], gen, 20.0, 20.0, None, lo, hi)
        assert np.array_equal(O, c["O"])
        F2 = problems.evaluate(name, O, m)
        assert np.array_equal(F2, c["F2"])
        improves, z_min = moead.compare(c["F1"], c["W"], c["I_nb"], c["z"], F2, 5.0)
        assert np.array_equal(improves, c["improves"]) and np.array_equal(z_min, c["z_min"])
        I_new = moead.update_matrix(improves, c["I_nb"])
        Xn, Fn, _, _ = moead.elite_select(c["X"], c["F1"], c["W"], O, F2, I_new, z_min, 5.0)
        assert np.array_equal(Xn, c["Xn"]) and np.array_equal(Fn, c["Fn"])


def test_neighbors_golden():
    for c in cases(load_golden("neighbors")):
        I = directions.neighbors(c["W"], c["I"].shape[1])
        assert np.array_equal(I, c["I"])


def test_simplex_lattice_rows():
    W = directions.simplex_lattice(3, 12)
    assert W.shape == (91, 3)
    assert np.array_equal(W[0], [0.0, 0.0, 1.0])
    assert directions.largest_h_for(200000, 3) == 630
