"""GPU: column-sharded ND-sort kernels, G shards simulated in lockstep on one device.

Every shard must reproduce the single-GPU ranks bit for bit (the multi-GPU path
differs only in that the mask assembly is an NCCL all-gather)."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("N,m,G,mode", [(5000, 3, 2, 0), (20000, 3, 4, 1), (20000, 5, 3, 0),
                                        (100_000, 3, 8, 1), (1500, 2, 8, 0), (60_000, 3, 2, 0)])
def test_lockstep_shards_equal_single_gpu(cuda, N, m, G, mode):
    import torch

    from paper_2503_20286_b200.ndsort import rank_device
    from paper_2503_20286_b200.parallel import CudaShardBackend, run_lockstep, shard_bounds

    rng = np.random.default_rng(N + G)
    F = rng.random((N, m))
    if G % 2:
        F = np.round(F, 2)
    Fd = torch.from_numpy(F).cuda()
    n = N // 2
    want, l_want, nf_want = rank_device(Fd, n, mode)
    bounds = shard_bounds(N, G)
    backends = [CudaShardBackend(N, m, lo, hi) for lo, hi in bounds]
    for b in backends:
        b.build(Fd)
    w = want.cpu().numpy()
    for batch in (1, 8):  # host read per front / per batch of fronts
        for b in backends:
            b.build(Fd)
        ranks, l, nf = run_lockstep(backends, bounds, N, n, mode, batch=batch)
        assert l == int(l_want.item()) and nf == int(nf_want.item())
        for r in ranks:
            assert np.array_equal(r.cpu().numpy(), w)
