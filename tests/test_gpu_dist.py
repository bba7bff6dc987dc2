"""Multi-GPU kernels (ovs_dist_*) on one B200: G virtual ranks driven by one process
(dist.dist_sort_virtual; collectives emulated by device copies), and the real torch.distributed
path (NCCL) with world_size 1.  Every result equals the single-process oracle on the
rank-ordered concatenation of the shards: output, values, bucket counts."""
import os
import socket

import numpy as np
import pytest
import torch

import ovs_inputs

pytestmark = pytest.mark.gpu


def shards_of(dist_name, G, n_per, seed):
    xs = [ovs_inputs.keys(dist_name, n_per, seed=seed, start=r * n_per, world=G, rank=r) for r in range(G)]
    return xs


@pytest.mark.parametrize("G", [1, 2, 4, 8])
@pytest.mark.parametrize("dist_name", ["u32", "u32_staggered", "u32_bucketsorted"])
def test_virtual_ranks_u32(orc, G, dist_name):
    from paper_1608_08648_b200.dist import dist_sort_virtual
    n_per, p, s = 1 << 18, 64 * G, 32
    xs = shards_of(dist_name, G, n_per, 51)
    out, _, counts = dist_sort_virtual([torch.from_numpy(x).cuda() for x in xs], None, p, s, 1)
    ref = orc.ros_sort(np.concatenate(xs), p, s, 1)
    np.testing.assert_array_equal(out.cpu().numpy(), ref.keys)
    np.testing.assert_array_equal(counts, ref.counts)


@pytest.mark.parametrize("dist_name,G", [("u16key", 4), ("f64_normal", 2), ("i32_gauss", 8), ("u32_few4", 2)])
def test_virtual_ranks_kv_and_dtypes(orc, dist_name, G):
    from paper_1608_08648_b200.dist import dist_sort_virtual
    n_per, p, s = 200_000, 32 * G, 16
    xs = shards_of(dist_name, G, n_per, 5)
    vs = [ovs_inputs.index_values(n_per, r * n_per) for r in range(G)]
    out, vout, counts = dist_sort_virtual([torch.from_numpy(x).cuda() for x in xs],
                                          [torch.from_numpy(v).cuda() for v in vs], p, s, 2)
    ref = orc.ros_sort(np.concatenate(xs), p, s, 2, vals=np.concatenate(vs))
    np.testing.assert_array_equal(out.cpu().numpy(), ref.keys)
    np.testing.assert_array_equal(vout.cpu().numpy(), ref.vals)
    np.testing.assert_array_equal(counts, ref.counts)


def _random_dist_cases():
    rng = np.random.default_rng(4242)
    out = []
    for i in range(12):
        G = int(rng.choice([2, 3, 4, 8]))
        dist_name = ["u32", "i32_few", "f64_uniform", "u16key", "u32_const"][i % 5]
        sizes = [int(rng.integers(0, 400_000)) for _ in range(G)]
        kv = bool(rng.integers(2))
        p = G * int(rng.choice([1, 4, 16, 64, 256]))
        s = int(rng.choice([2, 8, 33]))
        while p > G and p * s - 1 > sum(sizes):
            p //= 2
            p = max(G, p // G * G)
        out.append((i, G, dist_name, sizes, kv, p, s))
    return out


@pytest.mark.parametrize("i,G,dist_name,sizes,kv,p,s", _random_dist_cases())
def test_virtual_ranks_random(orc, i, G, dist_name, sizes, kv, p, s):
    """Seeded random world sizes, unequal (also empty) shards, dtypes, key-value or not."""
    from paper_1608_08648_b200.dist import dist_sort_virtual
    n = sum(sizes)
    if p < 2 or p * s - 1 > n:
        pytest.skip("sample larger than the input")
    x = ovs_inputs.keys(dist_name, n, seed=30 + i)
    offs = np.concatenate([[0], np.cumsum(sizes)])
    xs = [x[offs[r]:offs[r + 1]] for r in range(G)]
    v = ovs_inputs.index_values(n) if kv else None
    vs = [v[offs[r]:offs[r + 1]] for r in range(G)] if kv else None
    out, vout, counts = dist_sort_virtual([torch.from_numpy(np.ascontiguousarray(a)).cuda() for a in xs],
                                          [torch.from_numpy(np.ascontiguousarray(a)).cuda() for a in vs] if kv else None,
                                          p, s, 9)
    ref = orc.ros_sort(x, p, s, 9, vals=v)
    np.testing.assert_array_equal(out.cpu().numpy(), ref.keys)
    if kv:
        np.testing.assert_array_equal(vout.cpu().numpy(), ref.vals)
    np.testing.assert_array_equal(counts, ref.counts)


def test_nccl_world1(orc):
    import torch.distributed as dist
    from paper_1608_08648_b200.dist import dist_sort
    s_ = socket.socket()
    s_.bind(("127.0.0.1", 0))
    port = s_.getsockname()[1]
    s_.close()
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK="0", WORLD_SIZE="1")
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        x = ovs_inputs.keys("u32", 1 << 20, seed=3)
        res = dist_sort(torch.from_numpy(x).cuda(), None, 256, 32, 4)
        ref = orc.ros_sort(x, 256, 32, 4)
        np.testing.assert_array_equal(res.keys.cpu().numpy(), ref.keys)
        np.testing.assert_array_equal(res.counts, ref.counts)
    finally:
        dist.destroy_process_group()
