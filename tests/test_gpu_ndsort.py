"""GPU parity: ND sort (K0-K2) against golden reference vectors and the CPU oracle."""

import numpy as np
import pytest

from conftest import load_golden, unpack
from oracle import ndsort as ond

pytestmark = pytest.mark.gpu


def test_rank_golden_all(cuda):
    from paper_2503_20286_b200 import rank_assign

    z = load_golden("ndsort")
    for i in range(len(z["N"])):
        N, m, n = int(z["N"][i]), int(z["m"][i]), int(z["n"][i])
        F = unpack(z["F"], z["F_off"], i).reshape(N, m)
        res = rank_assign(F, n)
        assert np.array_equal(res.r, unpack(z["r"], z["r_off"], i)), i
        assert res.l == int(z["l"][i]), i


def test_dominance_matrix_golden_small(cuda):
    from paper_2503_20286_b200 import dominance_matrix

    z = load_golden("ndsort")
    for i in range(0, 500, 7):
        N, m = int(z["N"][i]), int(z["m"][i])
        F = unpack(z["F"], z["F_off"], i).reshape(N, m)
        assert np.array_equal(dominance_matrix(F), ond.dominance_matrix(F)), i


def _np_dominance(F, block=512):
    N = F.shape[0]
    D = np.zeros((N, N), dtype=np.int64)
    for a in range(0, N, block):
        X = F[a:a + block, None, :]
        D[a:a + block] = ((X <= F[None]).all(-1) & (X < F[None]).any(-1))
    return D


@pytest.mark.parametrize("N,m,kind", [(5000, 3, "u"), (4500, 4, "i"), (6145, 2, "i"), (4200, 3, "dup")])
def test_dominance_matrix_multi_supertile(cuda, N, m, kind):
    """The packed K1 (local ranks per 2048-column super-tile, two columns per
    subtraction) against a blocked NumPy restatement of ndsort.py:37-43, across
    several super-tiles, with ties and duplicate rows straddling tile borders."""
    from paper_2503_20286_b200 import dominance_matrix

    rng = np.random.default_rng(N * m)
    if kind == "u":
        F = rng.random((N, m))
    elif kind == "i":
        F = rng.integers(0, 9, size=(N, m)).astype(float)
    else:  # many exact duplicate rows, plus -0.0 / +0.0
        base = rng.random((N // 7, m))
        F = base[rng.integers(0, len(base), N)]
        F[rng.random(N) < 0.05, 0] = -0.0
        F[rng.random(N) < 0.05, 1] = 0.0
    assert np.array_equal(dominance_matrix(F), _np_dominance(F))


# -- ports of the reference's own tests (test_ndsort.py) ---------------------
def test_known_answers(cuda):
    from paper_2503_20286_b200 import dominance_matrix, rank_assign

    assert dominance_matrix(np.array([[1.0, 1.0], [1.0, 1.0]])).sum() == 0
    D = dominance_matrix(np.array([[0.0, 0.0], [1.0, 2.0], [2.0, 1.0]]))
    assert D.tolist() == [[0, 1, 1], [0, 0, 0], [0, 0, 0]]
    res = rank_assign(np.array([[0.0, 0.0], [1.0, 1.0], [2.0, 2.0]]), 2)
    assert res.r.tolist() == [0, 1, 2] and res.l == 1
    res = rank_assign(np.array([[0.0, 0.0], [1.0, 2.0], [2.0, 1.0]]), 2)
    assert res.r.tolist() == [0, 1, 1] and res.l == 1
    r = rank_assign(np.array([[1.0, 2.0], [1.0, 2.0], [0.5, 3.0]]), 2).r
    assert r.tolist() == [0, 0, 0]
    assert rank_assign(np.array([[0.0, 1.0], [1.0, 0.0]]), 2).l == 0


def test_errors(cuda):
    from paper_2503_20286_b200 import dominance_matrix, rank_assign

    with pytest.raises(ValueError):
        dominance_matrix(np.array([[0.0, np.nan]]))
    with pytest.raises(ValueError):
        rank_assign(np.array([[0.0, np.nan], [1.0, 1.0]]), 1)
    with pytest.raises(ValueError):
        rank_assign(np.zeros((3, 2)), 4)
    with pytest.raises(ValueError):
        rank_assign(np.zeros((3, 2)), 0)


def test_nan_on_device_tensor_flags_status(cuda):
    import torch

    from paper_2503_20286_b200 import rank_assign

    F = torch.rand(100, 3, dtype=torch.float64, device=cuda)
    F[17, 1] = float("nan")
    with pytest.raises(ValueError):
        rank_assign(F, 10)


def test_permutation_equivariance_and_contiguity(cuda):
    from paper_2503_20286_b200 import rank_assign

    rng = np.random.default_rng(65)
    F = rng.integers(0, 4, size=(25, 3)).astype(float)
    base = rank_assign(F, 10).r
    for _ in range(10):
        perm = rng.permutation(25)
        assert np.array_equal(rank_assign(F[perm], 10).r, base[perm])
    for _ in range(20):
        r = rank_assign(rng.random((300, 3)), 10).r
        assert set(r.tolist()) == set(range(int(r.max()) + 1))


@pytest.mark.parametrize("N,m,kind", [(3000, 3, "u"), (5000, 2, "u"), (4097, 5, "i"), (2000, 10, "u"),
                                      (1025, 16, "u"), (6000, 3, "dtlz2"), (257, 1, "i"),
                                      (10241, 3, "u"), (9000, 4, "i")])
def test_rank_vs_oracle_mid(cuda, N, m, kind):
    from paper_2503_20286_b200 import rank_assign

    rng = np.random.default_rng(N + m)
    if kind == "u":
        F = rng.random((N, m))
    elif kind == "i":
        F = rng.integers(0, 7, size=(N, m)).astype(float)
    else:
        from oracle.problems import evaluate_dtlz

        F = evaluate_dtlz("dtlz2", rng.random((N, m + 9)), m)
    n = N // 2
    got = rank_assign(F, n)
    want_r, want_l = ond.rank_fast(F, n)
    assert np.array_equal(got.r, want_r) and got.l == want_l


def test_select_mode_matches_sort_below_l(cuda):
    import torch

    from paper_2503_20286_b200.ndsort import SELECT, SORT, rank_device

    rng = np.random.default_rng(5)
    F = torch.from_numpy(rng.random((50000, 3))).cuda()
    n = 25000
    r_sort, l_sort, nf_sort = rank_device(F, n, SORT)
    r_sel, l_sel, nf_sel = rank_device(F, n, SELECT)
    l = int(l_sort.item())
    assert l == int(l_sel.item())
    rs, rl = r_sort.cpu().numpy(), r_sel.cpu().numpy()
    keep = rs <= l
    assert np.array_equal(rs[keep], rl[keep])
    assert np.all(rl[~keep] == l + 1)
    assert int(nf_sel.item()) == l + 1 <= int(nf_sort.item())


def test_large_property_equivariance(cuda):
    """N=200k (beyond the reference's memory limit): ranks are permutation-equivariant,
    contiguous, and rank 0 == rows not dominated by any rank-0 row (size-independent checks)."""
    import torch

    from paper_2503_20286_b200.ndsort import SORT, rank_device

    rng = np.random.default_rng(11)
    N = 200_000
    F = rng.random((N, 3))
    perm = rng.permutation(N)
    r1 = rank_device(torch.from_numpy(F).cuda(), N // 2, SORT)[0].cpu().numpy()
    r2 = rank_device(torch.from_numpy(F[perm]).cuda(), N // 2, SORT)[0].cpu().numpy()
    assert np.array_equal(r2, r1[perm])
    assert set(np.unique(r1).tolist()) == set(range(int(r1.max()) + 1))
    # spot-check 300 random rows against the definition of rank
    for j in rng.choice(N, 300, replace=False):
        dom = np.all(F <= F[j], axis=1) & np.any(F < F[j], axis=1)
        want = 0 if not dom.any() else int(r1[dom].max()) + 1
        assert r1[j] == want


def _rank_both(Fd, n, mode):
    """(staircase, bitmap) results of temo_rank for the same input."""
    from paper_2503_20286_b200 import _lib
    from paper_2503_20286_b200.ndsort import rank_device

    outs = []
    for force in (0, 1):
        _lib.lib().temo_rank_force_bitmap(force)
        try:
            r, l, nf = rank_device(Fd, n, mode)
            outs.append((r.cpu().numpy(), int(l.item()), int(nf.item())))
        finally:
            _lib.lib().temo_rank_force_bitmap(0)
    return outs


@pytest.mark.parametrize("N,m,kind", [(1, 3, "u"), (2, 2, "u"), (3, 3, "i"), (2047, 3, "u"), (2048, 3, "i"),
                                      (2049, 2, "u"), (4097, 3, "dup"), (30000, 3, "i"), (65537, 3, "u"),
                                      (70000, 2, "i"), (131072, 3, "dup"), (400_000, 3, "lsmop"),
                                      (300_001, 2, "u"), (500_000, 3, "u")])
def test_staircase_equals_bitmap(cuda, N, m, kind):
    """The m <= 3 staircase sort (ndsort_stair.cuh) against the O(N^2) bitmap path (K1 + peel):
    identical ranks, l and front counts in SORT and SELECT mode, across tile (2048) and level
    boundaries, integer ties, exact duplicate rows (-0.0 / +0.0) and the LSMOP1 distribution."""
    import torch

    from paper_2503_20286_b200.ndsort import SELECT, SORT

    rng = np.random.default_rng(N * 7 + m)
    if kind == "u":
        F = rng.random((N, m))
    elif kind == "i":
        F = rng.integers(0, 40, size=(N, m)).astype(float)
    elif kind == "dup":
        base = rng.random((max(N // 5, 1), m))
        F = base[rng.integers(0, len(base), N)]
        F[rng.random(N) < 0.05, 0] = -0.0
        F[rng.random(N) < 0.05, 1] = 0.0
    else:  # LSMOP1-like objectives: (1 + g) * linear front
        x = rng.random((N, 2))
        g = rng.random(N)[:, None] * 50
        F = (1 + g) * np.stack([x[:, 0] * x[:, 1], x[:, 0] * (1 - x[:, 1]), 1 - x[:, 0]], 1)
    Fd = torch.from_numpy(F).cuda()
    for mode in (SORT, SELECT):
        if mode == SORT and N > 131072:
            continue  # the bitmap SORT at 400k+ is slow; SELECT covers the headline
        n = max(N // 2, 1)
        (ra, la, fa), (rb, lb, fb) = _rank_both(Fd, n, mode)
        assert la == lb and fa == fb, (mode, la, lb, fa, fb)
        assert np.array_equal(ra, rb), mode
