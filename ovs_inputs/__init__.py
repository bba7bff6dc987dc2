"""Seeded synthetic input generators shared by the oracle tests, the GPU tests and bench.py.

This module holds NONE of the method's arithmetic (no sampling, no splitters, no
classification, no sorting).  It only produces input keys/values, deterministically
from a data seed, with the shapes and distributions of BASELINE.json's configs
(SURVEY.md §8(d) "Synthetic inputs").  The paper itself measures on random 32-byte
strings; BASELINE.json replaces that workload with the integer and
float key sets below, so these generators stand in for it.

Every key i is a function of u_i = SplitMix64 output number i of the data seed,
i.e. mix64(seed + GAMMA*(i+1)) (stream 0), so shards of a distributed input can be
generated independently from their global index range.  Gaussian keys use
Box-Muller and are generated here on the host once; the identical bytes feed both
the GPU path and the oracle (never regenerated on the device: libm != CUDA math).
"""
from __future__ import annotations

import numpy as np

GAMMA = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)

_CHUNK = 1 << 22


def _mix64(z: np.ndarray) -> np.ndarray:
    z = (z ^ (z >> np.uint64(30))) * _M1
    z = (z ^ (z >> np.uint64(27))) * _M2
    return z ^ (z >> np.uint64(31))


def data_u64(seed: int, start: int, count: int, stream: int = 0) -> np.ndarray:
    """u_i for global indices i in [start, start+count) of the data stream."""
    out = np.empty(count, dtype=np.uint64)
    base = np.uint64((int(seed) + (int(stream) << 40) * int(GAMMA)) & (2**64 - 1))
    with np.errstate(over="ignore"):
        for c0 in range(0, count, _CHUNK):
            c1 = min(count, c0 + _CHUNK)
            i = np.arange(start + c0 + 1, start + c1 + 1, dtype=np.uint64)
            out[c0:c1] = _mix64(base + GAMMA * i)
    return out


def _u01_open(u: np.ndarray) -> np.ndarray:
    """(0,1]: 53-bit uniform, never 0 (log argument of Box-Muller)."""
    return ((u >> np.uint64(11)).astype(np.float64) + 1.0) * (2.0 ** -53)


def _u01(u: np.ndarray) -> np.ndarray:
    """[0,1): exact 53-bit uniform."""
    return (u >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)


def _box_muller(seed: int, start: int, count: int) -> np.ndarray:
    u1 = data_u64(seed, 2 * start, 2 * count)
    a = _u01_open(u1[0::2])
    b = _u01(u1[1::2])
    return np.sqrt(-2.0 * np.log(a)) * np.cos(2.0 * np.pi * b)


def keys(dist: str, n: int, seed: int, start: int = 0, world: int = 1, rank: int = 0) -> np.ndarray:
    """Return keys for global indices [start, start+n).

    dist names:
      u32_u31      uint32 uniform on [0, 2^31)            (C1)
      u32          uint32 uniform on [0, 2^32)            (C5 uniform)
      i32_uniform  int32 uniform on [0, 2^31)             (C2 uniform)
      i32_gauss    int32 round-half-even(2^30 + 2^28 z), clamped to [0, 2^31-1] (C2 Gaussian)
      i32_sorted / i32_reverse  uniform i32 sorted ascending / descending (C2)
      i32_few      u mod 1024                              (C2 few-distinct)
      f64_uniform  (u >> 11) * 2^-53 in [0,1)              (C3)
      f64_normal   Box-Muller N(0,1), -0.0 -> +0.0          (C3)
      u16key       uint32 key = u >> 48 (uniform [0,2^16))  (C4 keys)
      u32_const    all keys equal (42)
      u32_r26      uint32 uniform on [0, 2^26) (tests: dense bucket ranges with duplicates)
      u32_few4     u mod 4
      u32_staggered / u32_bucketsorted  C5 multi-GPU distributions (need world, rank)
      s32          32-byte strings of uniform random bytes (the paper's workload):
                   string i = the little-endian bytes of u_{4i} .. u_{4i+3}; numpy dtype V32
      s32_prefix   s32 whose first 8 bytes take only 4 values (ties on the 8-byte prefix)
      s32_few      8 distinct strings (u mod 8 picks one of 8 fixed s32 strings)
    """
    if dist in ("s32", "s32_prefix", "s32_few"):
        w = data_u64(seed, 4 * start, 4 * n).reshape(n, 4)
        if dist == "s32_prefix":
            w[:, 0] = w[:, 0] % np.uint64(4)
        elif dist == "s32_few":
            pick = w[:, 0] % np.uint64(8)
            base = data_u64(seed + 1, 0, 32).reshape(8, 4)
            w = base[pick.astype(np.int64)]
        return np.ascontiguousarray(w).view("V32").reshape(n)
    if dist in ("i32_sorted", "i32_reverse") and start != 0:
        raise ValueError("sorted distributions are defined on the whole array only")
    u = None if dist in ("i32_gauss", "f64_normal") else data_u64(seed, start, n)
    if dist == "u32_u31":
        return (u >> np.uint64(33)).astype(np.uint32)
    if dist == "u32_r26":  # uniform on [0, 2^26): dense bucket ranges with duplicates (tests)
        return (u >> np.uint64(38)).astype(np.uint32)
    if dist == "u32":
        return (u >> np.uint64(32)).astype(np.uint32)
    if dist == "i32_uniform":
        return (u >> np.uint64(33)).astype(np.int32)
    if dist == "i32_sorted":
        return np.sort((u >> np.uint64(33)).astype(np.int32))
    if dist == "i32_reverse":
        return np.sort((u >> np.uint64(33)).astype(np.int32))[::-1].copy()
    if dist == "i32_few":
        return (u % np.uint64(1024)).astype(np.int32)
    if dist == "i32_gauss":
        z = _box_muller(seed, start, n)
        x = np.rint(2.0 ** 30 + 2.0 ** 28 * z)  # rint = round half to even
        return np.clip(x, 0, 2 ** 31 - 1).astype(np.int32)
    if dist == "f64_uniform":
        return _u01(u)
    if dist == "f64_normal":
        z = _box_muller(seed, start, n)
        z[z == 0.0] = 0.0  # -0.0 -> +0.0
        return z
    if dist == "u16key":
        return (u >> np.uint64(48)).astype(np.uint32)
    if dist == "u32_const":
        return np.full(n, 42, dtype=np.uint32)
    if dist == "u32_few4":
        return (u % np.uint64(4)).astype(np.uint32)
    if dist == "u32_staggered":
        # rank g's keys are uniform in slice (g + world//2) mod world of width 2^32/world
        sl = (rank + world // 2) % world
        w = (1 << 32) // world
        return (np.uint64(sl * w) + (u % np.uint64(w))).astype(np.uint32)
    if dist == "u32_bucketsorted":
        # rank's shard = world equal contiguous chunks; chunk c uniform in [c*2^32/world, (c+1)*2^32/world)
        w = (1 << 32) // world
        c = (np.arange(n, dtype=np.uint64) * np.uint64(world)) // np.uint64(max(n, 1))
        return (c * np.uint64(w) + (u % np.uint64(w))).astype(np.uint32)
    raise ValueError(f"unknown distribution {dist!r}")


def index_values(n: int, start: int = 0) -> np.ndarray:
    """uint32 value = original (global) index (C4: makes stability observable)."""
    return np.arange(start, start + n, dtype=np.uint32)


# The BASELINE.json configurations (readings Q7/Q14).
CONFIGS = {
    "C1": dict(n=1 << 20, dists=[("u32_u31", 1)], method="ros", p=64, s=32, seed=1, kv=False),
    "C2": dict(n=1 << 24, dists=[("i32_uniform", 21), ("i32_gauss", 22), ("i32_sorted", 23),
                                 ("i32_reverse", 24), ("i32_few", 25)],
               method="dro", p=256, s=24, seed=0, kv=False),
    "C3": dict(n=1 << 27, dists=[("f64_uniform", 31), ("f64_normal", 32)], method="ros", p=1024,
               s=64, seed=1, kv=False),
    "C4": dict(n=1 << 27, dists=[("u16key", 41)], method="dro", p=512, s=27, seed=0, kv=True),
    "C5": dict(n=1 << 27, dists=[("u32", 51)], method="ros", p=4096, s=64, seed=1, kv=False),
}
