"""ctypes wrapper of the CPU oracle (oracle/ovs_oracle.cpp).

TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / ``--impl reference`` legs may import this package.  The product path
(paper_1608_08648_b200) never imports it and shares no code with it.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "ovs_oracle.cpp")
_LIB = os.path.join(_HERE, "libovs_oracle.so")

OK, EINVAL, EDTYPE, ESAMPLE = 0, 1, 2, 3
DTYPES = {np.dtype(np.uint32): 0, np.dtype(np.int32): 1, np.dtype(np.float64): 2,
          np.dtype("V32"): 3}  # 32-byte strings in memcmp order (np.void, 32 bytes per key)
DRO_PADDED_POSITIONS = 1


def build(force: bool = False) -> str:
    """Compile the oracle (plain g++, -O2, no fast-math: IEEE compares, Q18)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["g++", "-O2", "-std=c++17", "-pthread", "-fPIC", "-shared", "-o", _LIB, _SRC])
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        # OVS_ORACLE_LIB: load a deliberately mutated build (tests/test_oracle_mutations.py)
        _lib = ctypes.CDLL(os.environ.get("OVS_ORACLE_LIB") or build())
        u64, u32, vp, i32 = ctypes.c_uint64, ctypes.c_uint32, ctypes.c_void_p, ctypes.c_int
        _lib.orc_splitmix64.restype = u64
        _lib.orc_splitmix64.argtypes = [u64, u64, u64]
        _lib.orc_draw_index.restype = u64
        _lib.orc_draw_index.argtypes = [u64, u64]
        _lib.orc_ros_sample_indices.restype = i32
        _lib.orc_ros_sample_indices.argtypes = [u64, u32, u32, u64, vp, vp]
        sig = [i32, vp, vp, u64, u32, u32, u64, vp, vp, vp, vp, vp]
        for f in (_lib.orc_ros_sort, _lib.orc_sqran_literal):
            f.restype = i32
            f.argtypes = sig
        _lib.orc_mcran_sort.restype = i32
        _lib.orc_mcran_sort.argtypes = [i32, vp, vp, u64, u32, u32, u64, u32, vp, vp, vp, vp, vp]
        _lib.orc_dro_sample_positions.restype = i32
        _lib.orc_dro_sample_positions.argtypes = [u64, u32, u32, u32, u32, vp]
        _lib.orc_dro_sort.restype = i32
        _lib.orc_dro_sort.argtypes = [i32, vp, vp, u64, u32, u32, u32, vp, vp, vp, vp, vp]
    return _lib


class OracleError(RuntimeError):
    def __init__(self, code: int):
        super().__init__(f"oracle status {code}")
        self.code = code


@dataclass
class Result:
    keys: np.ndarray
    vals: np.ndarray | None
    split_keys: np.ndarray
    split_tags: np.ndarray
    counts: np.ndarray


def _ptr(a):
    return None if a is None else a.ctypes.data


def splitmix64(seed: int, stream: int, j: int) -> int:
    return int(lib().orc_splitmix64(seed, stream, j))


def draw_index(u: int, n: int) -> int:
    return int(lib().orc_draw_index(u, n))


def ros_sample_indices(n: int, p: int, s: int, seed: int):
    m = p * s - 1
    out = np.empty(max(m, 0), dtype=np.uint64)
    draws = np.zeros(1, dtype=np.uint64)
    rc = lib().orc_ros_sample_indices(n, p, s, seed, _ptr(out), _ptr(draws))
    if rc != OK:
        raise OracleError(rc)
    return out, int(draws[0])


def dro_sample_positions(n: int, p: int, r: int, k: int, padded: bool = False) -> np.ndarray:
    out = np.empty(r * p, dtype=np.uint64)
    rc = lib().orc_dro_sample_positions(n, p, r, DRO_PADDED_POSITIONS if padded else 0, k, _ptr(out))
    if rc != OK:
        raise OracleError(rc)
    return out


def _run(fn, keys, vals, n, p, s, extra):
    keys = np.ascontiguousarray(keys)
    if keys.dtype not in DTYPES:
        raise OracleError(EDTYPE)
    vals = None if vals is None else np.ascontiguousarray(vals, dtype=np.uint32)
    out = np.empty_like(keys)
    outv = None if vals is None else np.empty_like(vals)
    sk = np.zeros(max(p - 1, 0), dtype=keys.dtype)  # n = 0: no splitters drawn, reported as 0
    st = np.zeros(max(p - 1, 0), dtype=np.uint64)
    cnt = np.zeros(max(p, 1), dtype=np.uint64)
    rc = fn(DTYPES[keys.dtype], _ptr(keys), _ptr(vals), n, p, s, *extra, _ptr(out), _ptr(outv), _ptr(sk), _ptr(st),
            _ptr(cnt))
    if rc != OK:
        raise OracleError(rc)
    return Result(out, outv, sk, st, cnt[:p])


def ros_sort(keys, p: int, s: int, seed: int, vals=None) -> Result:
    """ROS, partition-first."""
    return _run(lib().orc_ros_sort, keys, vals, len(keys), p, s, (seed,))


def sqran_literal(keys, p: int, s: int, seed: int, vals=None) -> Result:
    """Algorithm 2 (SqRan) as written."""
    return _run(lib().orc_sqran_literal, keys, vals, len(keys), p, s, (seed,))


def mcran_sort(keys, p: int, s: int, seed: int, threads: int, vals=None) -> Result:
    """McRan: Algorithm 2 with step 1's sorts, step 4's splits and step 5's merges on `threads`
    threads; the multi-core CPU baseline."""
    return _run(lib().orc_mcran_sort, keys, vals, len(keys), p, s, (seed, threads))


def dro_sort(keys, p: int, r: int, vals=None, padded: bool = False) -> Result:
    """Algorithm 1 (SqDet) as written."""
    return _run(lib().orc_dro_sort, keys, vals, len(keys), p, r, (DRO_PADDED_POSITIONS if padded else 0,))


def lemma1_bound(n: int, p: int, r: int) -> int:
    """ceil((1 + 1/r)(n/p) + r p)  (Lemma 1), exact integers."""
    num = (r + 1) * n + r * r * p * p  # (1+1/r) n/p + r p  =  ((r+1) n + r^2 p^2) / (r p)
    den = r * p
    return -(-num // den)


def tight_bound(n: int, p: int, r: int) -> int:
    """s*x + (p-1)(x-1), x = ceil(ceil(n/p)/s), s = r p  (reading Q10 of the Lemma 1 proof)."""
    s = r * p
    x = -(-(-(-n // p)) // s)
    return s * x + (p - 1) * (x - 1)
