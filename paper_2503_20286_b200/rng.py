"""Reproducible streams (``temo.rng``, rng.py:17-31) and the host<->device Philox bridge.

Every reference stream is ``Generator(Philox(SeedSequence(seed, spawn_key=path)))``.
``Generator.random`` consumes one 64-bit output per double, so a draw of k
uniforms starting at the Generator's current state can be produced on the
device element by element (``temo_philox_state``).  ``DeviceDraws`` hands the
device the state, and advances the host Generator by exactly the number of
outputs the reference would have consumed, so subsequent host draws
(``permutation``, ``integers``) continue the identical stream.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import numpy as np

_M0 = 0xD2E7470EE14C6C93
_M1 = 0xCA5A826395121157
_W0 = 0x9E3779B97F4A7C15
_W1 = 0xBB67AE8584CAA73B
_MASK = (1 << 64) - 1


@dataclass(frozen=True)
class RngStream:
    """Reproducible random stream addressed by (seed, path) (rng.py:17-31)."""

    seed: int
    path: tuple = field(default=())

    def split(self, key: int) -> "RngStream":
        return RngStream(self.seed, self.path + (int(key),))

    def generator(self) -> np.random.Generator:
        seq = np.random.SeedSequence(self.seed, spawn_key=self.path)
        return np.random.Generator(np.random.Philox(seq))


class PhiloxState(ctypes.Structure):
    """Mirror of ``temo_philox_state`` (include/temo_b200.h)."""

    _fields_ = [("counter", ctypes.c_uint64 * 4), ("key", ctypes.c_uint64 * 2),
                ("buffer", ctypes.c_uint64 * 4), ("buffer_pos", ctypes.c_int32),
                ("reserved", ctypes.c_int32)]


class PhiloxHostState(ctypes.Structure):
    """Mirror of ``temo_philox_host`` (include/temo_b200.h): the full NumPy Philox state."""

    _fields_ = [("counter", ctypes.c_uint64 * 4), ("key", ctypes.c_uint64 * 2),
                ("buffer", ctypes.c_uint64 * 4), ("buffer_pos", ctypes.c_int32),
                ("has_uint32", ctypes.c_int32), ("uinteger", ctypes.c_uint32),
                ("reserved", ctypes.c_uint32)]


def permutation(rng, n: int) -> np.ndarray:
    """``rng.permutation(n)`` (int64), drawn by the native replica for Philox Generators.

    Bit-identical to NumPy (``temo_host_permutation``) and the Generator ends in the
    same state; any other RNG object is called directly (duck-typed test RNGs)."""
    n = int(n)
    if not is_philox(rng) or n < 2:
        return np.asarray(rng.permutation(n), dtype=np.int64)
    from . import _lib

    st = rng.bit_generator.state
    s = PhiloxHostState()
    for i in range(4):
        s.counter[i] = int(st["state"]["counter"][i])
        s.buffer[i] = int(st["buffer"][i])
    s.key[0], s.key[1] = int(st["state"]["key"][0]), int(st["state"]["key"][1])
    s.buffer_pos = int(st["buffer_pos"])
    s.has_uint32 = int(st["has_uint32"])
    s.uinteger = int(st["uinteger"])
    out = np.empty(n, dtype=np.int64)
    rc = _lib.lib().temo_host_permutation(ctypes.byref(s), n, out.ctypes.data_as(ctypes.c_void_p))
    _lib.check(rc, "permutation")
    st["state"]["counter"] = np.array(list(s.counter), dtype=np.uint64)
    st["buffer"] = np.array(list(s.buffer), dtype=np.uint64)
    st["buffer_pos"] = int(s.buffer_pos)
    st["has_uint32"] = int(s.has_uint32)
    st["uinteger"] = int(s.uinteger)
    rng.bit_generator.state = st
    return out


def is_philox(rng) -> bool:
    return isinstance(rng, np.random.Generator) and isinstance(rng.bit_generator, np.random.Philox)


def _block(ctr, key):
    c0, c1, c2, c3 = ctr
    k0, k1 = key
    for r in range(10):
        if r:
            k0 = (k0 + _W0) & _MASK
            k1 = (k1 + _W1) & _MASK
        p0, p1 = _M0 * c0, _M1 * c2
        c0, c1, c2, c3 = (p1 >> 64) ^ c1 ^ k0, p1 & _MASK, (p0 >> 64) ^ c3 ^ k1, p0 & _MASK
    return [c0, c1, c2, c3]


def snapshot(rng) -> PhiloxState:
    st = rng.bit_generator.state
    s = PhiloxState()
    for i in range(4):
        s.counter[i] = int(st["state"]["counter"][i])
        s.buffer[i] = int(st["buffer"][i])
    s.key[0], s.key[1] = int(st["state"]["key"][0]), int(st["state"]["key"][1])
    s.buffer_pos = int(st["buffer_pos"])
    return s


def advance(rng, count: int) -> None:
    """Move ``rng`` forward by ``count`` 64-bit outputs exactly as ``count`` doubles would."""
    if count <= 0:
        return
    st = rng.bit_generator.state
    pos = int(st["buffer_pos"])
    avail = 4 - pos
    if count <= avail:
        st["buffer_pos"] = pos + count
        rng.bit_generator.state = st
        return
    rest = count - avail
    blocks = (rest + 3) // 4
    ctr = sum(int(v) << (64 * i) for i, v in enumerate(st["state"]["counter"]))
    ctr = (ctr + blocks) & ((1 << 256) - 1)
    words = [(ctr >> (64 * i)) & _MASK for i in range(4)]
    key = [int(v) for v in st["state"]["key"]]
    st["state"]["counter"] = np.array(words, dtype=np.uint64)
    st["buffer"] = np.array(_block(words, key), dtype=np.uint64)
    st["buffer_pos"] = rest - 4 * (blocks - 1)
    rng.bit_generator.state = st


class DeviceDraws:
    """Reserve consecutive uniform draws for the device.

    ``take(k)`` returns the raw offset (relative to ``self.state``) of the next
    k uniforms; ``commit()`` advances the host Generator past all of them.
    """

    def __init__(self, rng):
        self.rng = rng
        self.state = snapshot(rng)
        self.used = 0

    def take(self, count: int) -> int:
        off = self.used
        self.used += int(count)
        return off

    def commit(self):
        advance(self.rng, self.used)
        self.used = 0
        self.state = snapshot(self.rng)
