"""torch.ops.temo.* (TORCH_LIBRARY registration of the C ABI): schemas and Meta
shapes on CPU; results equal to the ctypes path and CUDA-graph capture on the GPU."""

import numpy as np
import pytest


def test_ops_registered_with_meta_shapes():
    import torch

    from paper_2503_20286_b200 import torch_ops

    ops = torch_ops.load()
    F = torch.empty((10, 3), dtype=torch.float64, device="meta")
    assert [t.shape for t in ops.rank(F, 5, 0)] == [(10,), (1,), (1,), (1,)]
    assert ops.evaluate(torch.empty((7, 12), dtype=torch.float64, device="meta"), 2, 3, 0, [], []).shape == (7, 3)
    assert ops.igd(F, torch.empty((4, 3), dtype=torch.float64, device="meta")).shape == (1,)


@pytest.mark.gpu
def test_ops_match_ctypes_path(cuda):
    import torch

    from paper_2503_20286_b200 import torch_ops
    from paper_2503_20286_b200.indicators import igd
    from paper_2503_20286_b200.ndsort import SELECT, SORT, rank_device
    from paper_2503_20286_b200.problems import evaluate, make_problem

    ops = torch_ops.load()
    r = np.random.default_rng(5)
    for N, m in ((5000, 3), (3000, 5), (2000, 2)):
        F = torch.from_numpy(np.round(r.random((N, m)), 2)).cuda()
        for mode in (SORT, SELECT):
            a = ops.rank(F, N // 2, mode)
            b = rank_device(F, N // 2, mode)
            assert torch.equal(a[0], b[0]) and int(a[1]) == int(b[1]) and int(a[3]) == 0
    for name, d in (("dtlz2", 12), ("lsmop1", 300), ("lsmop7", 300)):
        spec = make_problem(name, m=3, d=d)
        X = spec.lower + r.random((64, spec.d)) * (spec.upper - spec.lower)
        ps = spec.struct()
        got = ops.evaluate(torch.from_numpy(X).cuda(), ps.id, ps.m, ps.nk, list(ps.sublen)[: ps.m],
                           list(ps.offset)[: ps.m + 1])
        assert np.array_equal(got.cpu().numpy(), evaluate(spec, X))
    Fs, R = r.random((500, 3)), r.random((300, 3))
    assert float(ops.igd(torch.from_numpy(Fs).cuda(), torch.from_numpy(R).cuda())) == igd(Fs, R)


@pytest.mark.gpu
def test_rank_captured_in_cuda_graph(cuda):
    """The staircase sort (one cooperative kernel per sort) and the m >= 4 bitmap sort run inside
    a captured CUDA graph; replays on new objectives give the direct call's ranks."""
    import torch

    from paper_2503_20286_b200 import torch_ops
    from paper_2503_20286_b200.ndsort import SELECT, rank_device

    ops = torch_ops.load()
    r = np.random.default_rng(9)
    for N, m in ((20000, 3), (8000, 4)):
        static = torch.from_numpy(r.random((N, m))).cuda()
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            for _ in range(2):
                ops.rank(static, N // 2, SELECT)  # warm-up outside capture
        torch.cuda.current_stream().wait_stream(s)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            out = ops.rank(static, N // 2, SELECT)
        for _ in range(3):
            F = torch.from_numpy(np.round(r.random((N, m)), 2)).cuda()
            static.copy_(F)
            g.replay()
            want = rank_device(F, N // 2, SELECT)
            torch.cuda.synchronize()
            assert torch.equal(out[0], want[0]) and int(out[1]) == int(want[1])
