"""Multi-GPU sharding parity on one GPU: the sharded generation loop -- offspring
pair ranges + row all-gather, HypE exchange-column split + all-gather, bitmap ND sort column
shards (m >= 4) -- gives bit-identical populations to the unsharded loop.  Ranks share cuda:0
and talk over gloo (parallel.all_gather_into stages through host memory); on an NVLink node
the same code runs one rank per GPU over NCCL."""

import json
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
WORKER = os.path.join(ROOT, "tests", "shard_worker.py")

CASES = [
    dict(algorithm="nsga3", problem="dtlz2", objectives=3, pop_size=210, generations=4, seed=3),
    dict(algorithm="nsga3", problem="dtlz1", objectives=5, pop_size=126, generations=3, seed=4),
    dict(algorithm="nsga3", problem="lsmop1", objectives=3, pop_size=92, generations=2, seed=5),
    # bench.py's sharded loop at a size with the randomness overlap on (n * D >= 2^20)
    dict(algorithm="nsga3", problem="lsmop1", objectives=3, pop_size=1100, dim=1000, generations=3, seed=8,
         predrawn=True),
    dict(algorithm="hype", problem="dtlz2", objectives=3, pop_size=64, generations=3, seed=6, hv_samples=140001),
    dict(algorithm="hype", problem="dtlz7", objectives=4, pop_size=50, generations=2, seed=7, hv_samples=70001),
]


def _run(cfg, out, world, port):
    env = dict(os.environ, PYTHONPATH=ROOT + os.pathsep + os.environ.get("PYTHONPATH", ""))
    if world == 1:
        cmd = [sys.executable, WORKER, json.dumps(cfg), out]
    else:
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
               "--master-addr", "127.0.0.1", "--master-port", str(port), WORKER, json.dumps(cfg), out]
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]


@pytest.mark.parametrize("idx", range(len(CASES)))
def test_sharded_loop_bit_identical(cuda, tmp_path, idx):
    cfg = CASES[idx]
    base = str(tmp_path / "w1")
    _run(cfg, base, 1, 0)
    want = dict(np.load(base + ".r0.npz"))
    for world in (2, 3):
        out = str(tmp_path / f"w{world}")
        _run(cfg, out, world, 29600 + 10 * idx + world)
        for r in range(world):
            got = np.load(f"{out}.r{r}.npz")
            for key in ("X", "F", "ideals", "tail"):
                assert np.array_equal(got[key], want[key]), (cfg, world, r, key)


@pytest.mark.parametrize("N,m,n,s,G", [(400, 3, 200, 300001, 8), (1001, 4, 500, 65536, 3), (64, 2, 32, 5000, 4),
                                       (2000, 3, 1000, 200000, 5)])
def test_hype_column_split_lockstep(cuda, N, m, n, s, G):
    """temo_hype_select_begin / _columns over G column ranges / _end == temo_hype_select, bitwise."""
    import torch

    from paper_2503_20286_b200 import _lib
    from paper_2503_20286_b200.hype import HypeSelector

    r = np.random.default_rng(N + s)
    F = torch.from_numpy(np.round(r.random((N, m)) ** 2, 3)).cuda()
    seed = np.random.SeedSequence(s)
    full = HypeSelector(N, m, n, s)
    g1 = np.random.Generator(np.random.Philox(seed))
    want_keep = full.select(F, g1).cpu().numpy()
    want_v = full.v_hv.cpu().numpy()
    state = lambda g: json.dumps(g.bit_generator.state, default=lambda a: np.asarray(a).tolist())  # noqa: E731
    want_state = state(g1)

    class Lockstep:
        """Stands in for the all-gather: the segments of the other G - 1 shards are computed here."""

        def __init__(self):
            self.sel = None

        def __call__(self, seg, counts):
            sel = self.sel
            L, p = _lib.lib(), _lib.ptr
            C = int(L.temo_hype_columns(s))
            Tg = torch.empty((C, N), dtype=torch.float64, device="cuda")
            ws = _lib.workspace.get(sel.ws_bytes, sel.dev)
            from paper_2503_20286_b200.rng import DeviceDraws

            for g, (lo, hi) in enumerate(sel.col_bounds):
                if g == sel.shard[0]:
                    Tg[lo:hi] = seg
                elif hi > lo:
                    draws = DeviceDraws(np.random.Generator(np.random.Philox(seed)))
                    rc = L.temo_hype_select_columns(p(F), N, m, s, lo, hi, _lib.sptr(draws.state), 0, None,
                                                    p(Tg[lo:]), p(ws), ws.numel(), _lib.stream_handle(sel.dev))
                    _lib.check(rc, "columns")
            return Tg

    for me in (0, G - 1):
        ex = Lockstep()
        sel = HypeSelector(N, m, n, s, shard=(me, G, ex))
        ex.sel = sel
        g2 = np.random.Generator(np.random.Philox(seed))
        keep = sel.select(F, g2).cpu().numpy()
        assert np.array_equal(sel.v_hv.cpu().numpy(), want_v)
        assert np.array_equal(keep, want_keep)
        assert state(g2) == want_state
