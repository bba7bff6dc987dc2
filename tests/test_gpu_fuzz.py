"""Randomised parity sweep (GPU): 128 seeded random configurations (size, dtype, distribution,
method, p, s or r, key-value or not) compared bit for bit with the oracle, so that the many
internal paths (refinement, windows, level 1, CTA re-split, direct digits, misaligned heads) are
hit in combinations the hand-written cases do not list."""
import numpy as np
import pytest
import torch

import ovs_inputs

pytestmark = pytest.mark.gpu

DISTS = {np.uint32: ["u32", "u32_u31", "u32_few4", "u32_const", "u16key"], np.int32: ["i32_uniform", "i32_gauss", "i32_few", "i32_sorted", "i32_reverse"],
         np.float64: ["f64_uniform", "f64_normal"]}


def cases(seed, count, base):
    rng = np.random.default_rng(seed)
    out = []
    for i in range(base, base + count):
        dt = [np.uint32, np.int32, np.float64][i % 3]
        dist = DISTS[dt][rng.integers(len(DISTS[dt]))]
        n = int(rng.choice([1, 17, 5000, 200_000, 1_000_003, 2_500_000, 8_000_000, 20_000_011],
                           p=[0.06, 0.06, 0.12, 0.16, 0.16, 0.16, 0.16, 0.12]))
        kv = bool(rng.integers(2))
        method = "ros" if rng.random() < 0.6 else "dro"
        p = int(2 ** rng.integers(0, 12)) + int(rng.integers(0, 3))
        if method == "ros":
            s = int(rng.choice([1, 3, 8, 33, 64, 150]))
            p = max(1, min(p, 4096))
            while p > 1 and p * s - 1 > n:
                p //= 2
        else:
            s = int(rng.integers(1, 6))
            p = max(1, min(p, 1024))
            while p > 1 and s * p > n // p:
                p //= 2
        padded = method == "dro" and bool(rng.integers(2))
        out.append((i, dist, n, kv, method, p, s, padded))
    return out


@pytest.mark.parametrize("i,dist,n,kv,method,p,s,padded", cases(20261020, 64, 0) + cases(7, 64, 64))
def test_fuzz(orc, i, dist, n, kv, method, p, s, padded):
    import paper_1608_08648_b200 as ovs
    x = ovs_inputs.keys(dist, n, seed=100 + i)
    v = ovs_inputs.index_values(n) if kv else None
    ref = orc.ros_sort(x, p, s, 7 + i, vals=v) if method == "ros" else orc.dro_sort(x, p, s, vals=v, padded=padded)
    off = i % 3  # some calls on buffers that start past a 16-byte boundary
    kb = torch.empty(n + off, dtype={np.dtype(np.uint32): torch.uint32, np.dtype(np.int32): torch.int32,
                                     np.dtype(np.float64): torch.float64}[x.dtype], device="cuda")
    kt = kb[off:]
    kt.copy_(torch.from_numpy(x))
    vt = torch.from_numpy(v).cuda() if kv else None
    srt = ovs.Sorter(n, kt.dtype, kv, method, p, s, 7 + i, padded=padded)
    rep = srt(kt, vt, report=True)
    torch.cuda.synchronize()
    assert rep.device_status == 0
    np.testing.assert_array_equal(kt.cpu().numpy(), ref.keys)
    if kv:
        np.testing.assert_array_equal(vt.cpu().numpy(), ref.vals)
    np.testing.assert_array_equal(rep.counts, ref.counts)
    if p > 1:
        np.testing.assert_array_equal(rep.splitter_keys, ref.split_keys)
        np.testing.assert_array_equal(rep.splitter_tags, ref.split_tags)
