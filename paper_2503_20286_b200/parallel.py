"""Multi-GPU plumbing: row-sharded offspring, column-sharded HypE sampling, and the
column-sharded bitmap ND sort (m >= 4) with a per-front mask all-gather.

Sharding used by the generation loop (harness._Stepper under torch.distributed):
  * offspring + evaluation: rank g computes the pairs ``shard_range(h, g, G)`` with exactly the
    draws the full call gives them (temo_offspring_ws_range), then ``RowExchange`` all-gathers
    the children's X rows and objective rows so every rank holds the merged population;
  * HypE: rank g computes its range of Monte-Carlo exchange columns; ``ColumnExchange``
    all-gathers them and every rank combines in the reference's order (bit-identical);
  * ND sort: m <= 3 runs the staircase sort on every rank (latency-bound, ~1 ms); m >= 4 shards
    the O(N^2) bitmap by column tiles (DistRank below).


One process per GPU (``torch.distributed``, NCCL over NVLink).  Every rank
holds the same objectives F, runs K0 identically and owns a contiguous range
of sorted column tiles (``shard_bounds``: equal triangle area).  K1 builds only
the rank's bitmap columns and their dominated-by counts -- no exchange.  Each
front step exchanges one N-bit mask:

    detect (own columns)  ->  all-gather of the mask segments  ->  apply (rank the
    front everywhere, subtract its rows from the own columns' counts)

``run_sharded`` is written against two small interfaces -- a backend
(``CudaShardBackend`` here; a NumPy backend in tests) and an exchange
(``TorchDistExchange`` for NCCL/gloo, ``LockstepExchange`` to run G shards in one
process) -- so the orchestration is tested on CPU with gloo and the kernels on
one GPU with simulated shards.
"""

from __future__ import annotations

import numpy as np

from . import _lib

SORT, SELECT = 0, 1


def all_gather_into(recv, send, group=None):
    """``dist.all_gather_into_tensor`` (NCCL over NVLink on GPUs).  Under gloo (CPU tests, or
    several ranks sharing one GPU in the sharding parity test) CUDA buffers are staged through
    host memory, since gloo's all-gather runs on host tensors."""
    import torch.distributed as dist

    if recv.is_cuda and dist.get_backend(group) == "gloo":
        r = recv.cpu()
        dist.all_gather_into_tensor(r, send.cpu(), group=group)
        recv.copy_(r)
    else:
        dist.all_gather_into_tensor(recv, send, group=group)


def shard_range(total: int, rank: int, world: int):
    """[lo, hi) of an even split of range(total) (rank g of world G)."""
    return total * rank // world, total * (rank + 1) // world


class RowExchange:
    """All-gather of per-rank row blocks of unequal length (padded to the longest for NCCL's
    all_gather_into_tensor); returns the concatenation in rank order."""

    def __init__(self, group=None):
        self.group = group
        self.buf = {}

    def __call__(self, local, counts):
        t = _lib.torch()
        G = len(counts)
        mx = max(max(counts), 1)
        tail = tuple(local.shape[1:])
        key = (mx, tail, local.dtype, str(local.device))
        if key not in self.buf:
            self.buf[key] = (t.zeros((mx,) + tail, dtype=local.dtype, device=local.device),
                             t.zeros((G * mx,) + tail, dtype=local.dtype, device=local.device))
        send, recv = self.buf[key]
        send[: local.shape[0]].copy_(local)
        all_gather_into(recv, send, self.group)
        return t.cat([recv[g * mx: g * mx + c] for g, c in enumerate(counts)])


class ColumnExchange(RowExchange):
    """HypE exchange columns: per-rank (columns x N) blocks -> the full column-major (C x N) buffer."""


def shard_bounds(N: int, G: int):
    """[(jt_lo, jt_hi)] column-tile ranges (256 sorted columns per tile) for G shards."""
    out = np.zeros(2 * G, dtype=np.int64)
    _lib.lib().temo_rank_shard_bounds(N, G, _lib._P(out.ctypes.data))
    return [(int(out[2 * g]), int(out[2 * g + 1])) for g in range(G)]


def mask_words(N: int) -> int:
    """Words of the full front mask (sorted index space, padded to 1024 rows)."""
    return ((N + 1023) // 1024) * 32


class CudaShardBackend:
    """One rank's shard of the sorted columns on its GPU (C ABI temo_rank_shard_*)."""

    def __init__(self, N: int, m: int, lo: int, hi: int, dev=None):
        t = _lib.torch()
        self.N, self.m, self.lo, self.hi = N, m, lo, hi
        self.dev = _lib.device(dev)
        self.empty = hi <= lo
        self.seg = t.zeros(max(8 * (hi - lo), 1), dtype=t.int32, device=self.dev)
        self.count = t.zeros(1, dtype=t.int32, device=self.dev)
        self.total = t.zeros(1, dtype=t.int32, device=self.dev)
        self.fill = t.zeros(1, dtype=t.int32, device=self.dev)
        self.rank = t.empty(N, dtype=t.int32, device=self.dev)
        self.totals = t.zeros(N + 64, dtype=t.int32, device=self.dev)  # row count of front k at [k] (+ batch slack)
        self.status = t.zeros(1, dtype=t.int32, device=self.dev)
        L = _lib.lib()
        # empty shards still need K0 + rank bookkeeping: give them a one-block dummy range
        self.plo, self.phi = (lo, hi) if not self.empty else (0, 4)
        self.ws = t.empty(L.temo_rank_shard_ws_bytes(N, m, self.plo, self.phi), dtype=t.uint8,
                          device=self.dev)
        self._empty_seg = t.zeros(1, dtype=t.int32, device=self.dev)

    def _a(self):
        return (self.N, self.m, self.plo, self.phi)

    def build(self, Fd):
        L = _lib.lib()
        rc = L.temo_rank_shard_build(_lib.ptr(Fd), self.N, self.m, self.plo, self.phi, _lib.ptr(self.status),
                                     _lib.ptr(self.ws), self.ws.numel(), _lib.stream_handle(self.dev))
        _lib.check(rc, "rank_shard_build")

    def detect(self, k: int):
        if self.empty:
            return self.seg[:0], self.count
        rc = _lib.lib().temo_rank_shard_detect(*self._a(), _lib.ptr(self.seg), _lib.ptr(self.count),
                                               _lib.ptr(self.ws), self.ws.numel(),
                                               _lib.stream_handle(self.dev))
        _lib.check(rc, "rank_shard_detect")
        return self.seg, self.count

    def apply(self, full, k: int):
        """Rank front k everywhere and subtract its rows; returns its row count (device, [k])."""
        out = self.totals[k: k + 1]
        rc = _lib.lib().temo_rank_shard_apply(*self._a(), _lib.ptr(full), int(k), _lib.ptr(out),
                                              _lib.ptr(self.ws), self.ws.numel(),
                                              _lib.stream_handle(self.dev))
        _lib.check(rc, "rank_shard_apply")
        return out

    def finish(self, fill: int):
        self.fill.fill_(int(fill))
        rc = _lib.lib().temo_rank_shard_finish(*self._a(), _lib.ptr(self.fill), _lib.ptr(self.rank),
                                               _lib.ptr(self.ws), self.ws.numel(),
                                               _lib.stream_handle(self.dev))
        _lib.check(rc, "rank_shard_finish")
        return self.rank


class TorchDistExchange:
    """All-gather of per-rank mask segments through torch.distributed (NCCL on GPUs, gloo on CPU)."""

    def __init__(self, bounds, W: int, device, group=None):
        t = _lib.torch()
        self.bounds = bounds
        self.W = W
        self.S = max(max(8 * (hi - lo) for lo, hi in bounds), 1)
        self.group = group
        self.send = t.zeros(self.S, dtype=t.int32, device=device)
        self.recv = t.zeros(len(bounds) * self.S, dtype=t.int32, device=device)
        self.full = t.zeros(W, dtype=t.int32, device=device)

    def __call__(self, seg):
        self.send.zero_()
        self.send[: seg.numel()].copy_(seg)
        all_gather_into(self.recv, self.send, self.group)
        for g, (lo, hi) in enumerate(self.bounds):
            n = 8 * (hi - lo)
            if n:
                self.full[8 * lo: 8 * hi].copy_(self.recv[g * self.S: g * self.S + n])
        return self.full


def assemble(bounds, segs, W, like):
    """Full mask from per-shard segments (used by the lockstep exchange and tests)."""
    full = like.new_zeros(W)
    for (lo, hi), seg in zip(bounds, segs):
        if hi > lo:
            full[8 * lo: 8 * hi] = seg[: 8 * (hi - lo)]
    return full


def _front_loop(round_fn, N: int, n: int, mode: int, batch: int):
    """Host side of the sharded peel: enqueue rounds (detect -> mask exchange -> apply) for
    fronts k, k+1, ... in batches of 1, 2, 4 .. ``batch`` and read their row counts back once per
    batch (one host sync per batch instead of per front).  Rounds past the end are no-ops (no
    unranked row has a zero count); in SELECT mode rows ranked past the stop front are reset to
    l + 1 by the finish kernel (SORT passes the front count, which no rank reaches).  Returns (l, number of fronts)."""
    t = _lib.torch()
    k, ranked, l, B = 0, 0, -1, 1
    while True:
        outs = [round_fn(k + b) for b in range(B)]
        vals = t.cat([o.reshape(-1)[:1] for o in outs]).cpu().tolist()
        for b, total in enumerate(vals):
            kk = k + b
            if total == 0:
                if ranked < N:
                    raise RuntimeError("front peeling failed to terminate")
                return l, kk
            ranked += int(total)
            if l < 0 and ranked >= n:
                l = kk
            if (mode == SELECT and ranked >= n) or ranked >= N:
                return l, kk + 1
        k += B
        B = min(2 * B, max(int(batch), 1))


def run_sharded(backend, exchange, N: int, n: int, mode: int = SORT, batch: int = 8):
    """Front loop of one rank; returns (rank in original order, l, number of fronts)."""

    def round_fn(k):
        seg, _ = backend.detect(k)
        return backend.apply(exchange(seg), k)

    l, nf = _front_loop(round_fn, N, n, mode, batch)
    return backend.finish(l + 1 if mode == SELECT else nf), l, nf


def run_lockstep(backends, bounds, N: int, n: int, mode: int = SORT, batch: int = 8):
    """G shards in one process, advanced together (single-GPU test of the shard kernels)."""
    W = mask_words(N)
    t = _lib.torch()

    def round_fn(k):
        segs = [b.detect(k)[0] for b in backends]
        full = assemble(bounds, segs, W, segs[0] if segs[0].numel() else backends[0].seg)
        totals = t.cat([b.apply(full, k).reshape(-1)[:1] for b in backends])
        return totals

    def checked(k):
        tot = round_fn(k)
        assert bool((tot == tot[0]).all())
        return tot[:1]

    l, nf = _front_loop(checked, N, n, mode, batch)
    return [b.finish(l + 1 if mode == SELECT else nf) for b in backends], l, nf


class DistRank:
    """Sharded replacement of ``rank_device`` for one rank of a process group."""

    def __init__(self, N: int, m: int, rank: int, world: int, dev=None, group=None):
        self.N, self.m = N, m
        self.bounds = shard_bounds(N, world)
        lo, hi = self.bounds[rank]
        self.backend = CudaShardBackend(N, m, lo, hi, dev)
        self.exchange = TorchDistExchange(self.bounds, mask_words(N), self.backend.dev, group)

    @property
    def status(self):
        """Device status word of the shard (K0 flags NaN objectives here)."""
        return self.backend.status

    def __call__(self, Fd, n: int, mode: int = SELECT):
        self.backend.build(Fd)
        rank, l, nf = run_sharded(self.backend, self.exchange, self.N, n, mode)
        return rank, l, nf
