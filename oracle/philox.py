"""Oracle: NumPy's Philox4x64-10 bit generator restated in pure Python. Test infrastructure only.

Used to check the device stream of ``paper_2503_20286_b200`` against
``np.random.Philox`` (rng.py:17-31 backs every reference stream with it).
``Generator.random`` returns ``(raw >> 11) * 2**-53`` per 64-bit output
(SURVEY App. A9); outputs come four per counter increment.
"""

from __future__ import annotations

import numpy as np

M0 = 0xD2E7470EE14C6C93
M1 = 0xCA5A826395121157
W0 = 0x9E3779B97F4A7C15
W1 = 0xBB67AE8584CAA73B
MASK = (1 << 64) - 1


def block(ctr, key, rounds=10):
    """philox4x64_R: one 4-word output block for a 4-word counter and 2-word key."""
    c0, c1, c2, c3 = ctr
    k0, k1 = key
    for r in range(rounds):
        if r:
            k0 = (k0 + W0) & MASK
            k1 = (k1 + W1) & MASK
        p0 = M0 * c0
        p1 = M1 * c2
        hi0, lo0 = p0 >> 64, p0 & MASK
        hi1, lo1 = p1 >> 64, p1 & MASK
        c0, c1, c2, c3 = hi1 ^ c1 ^ k0, lo1, hi0 ^ c3 ^ k1, lo0
    return (c0, c1, c2, c3)


def raw_stream(state: dict, count: int):
    """The next ``count`` 64-bit outputs of a Philox state dict (does not mutate it)."""
    st = state["state"]
    ctr = [int(v) for v in st["counter"]]
    key = [int(v) for v in st["key"]]
    buf = [int(v) for v in state["buffer"]]
    pos = int(state["buffer_pos"])
    out = []
    while len(out) < count:
        if pos < 4:
            out.append(buf[pos])
            pos += 1
            continue
        for w in range(4):  # 256-bit counter increment with carry
            ctr[w] = (ctr[w] + 1) & MASK
            if ctr[w]:
                break
        buf = list(block(ctr, key))
        pos = 0
    return np.array(out, dtype=np.uint64)


def doubles(state: dict, count: int) -> np.ndarray:
    raw = raw_stream(state, count)
    return (raw >> np.uint64(11)).astype(np.float64) * (1.0 / 9007199254740992.0)
