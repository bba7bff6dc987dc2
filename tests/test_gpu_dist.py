"""Multi-GPU path on one B200.

- G ranks emulated by one library call (ovs_dist_sort_virtual): the same phases and kernels as
  the NCCL path; the fused scatter stores every key into the emulated owner's window; phases run
  rank after rank, so no kernel waits on another (B200_PROFILING.md: never run waiting ranks on
  one GPU).
- The real communicator path (ovs_comm_create + ovs_dist_sort_keys: NCCL window, NVLink peer
  pointers, LSA barriers) with world_size 1.
Every result equals the single-process oracle on the rank-ordered concatenation of the shards:
output, values, bucket counts and the splitters (keys and tags; north_star: the same splitters
as the oracle for the same seeds).
"""
import os
import socket

import numpy as np
import pytest
import torch

import ovs_inputs

pytestmark = pytest.mark.gpu


def shards_of(dist_name, G, n_per, seed):
    return [ovs_inputs.keys(dist_name, n_per, seed=seed, start=r * n_per, world=G, rank=r) for r in range(G)]


def check(ref, out, vout, counts, sk, st):
    np.testing.assert_array_equal(out.cpu().numpy(), ref.keys)
    if vout is not None:
        np.testing.assert_array_equal(vout.cpu().numpy(), ref.vals)
    np.testing.assert_array_equal(counts, ref.counts)
    np.testing.assert_array_equal(sk, ref.split_keys)
    np.testing.assert_array_equal(st, ref.split_tags)


@pytest.mark.parametrize("G", [1, 2, 4, 8])
@pytest.mark.parametrize("dist_name", ["u32", "u32_staggered", "u32_bucketsorted"])
def test_virtual_ranks_u32(orc, G, dist_name):
    from paper_1608_08648_b200.dist import dist_sort_virtual
    n_per, p, s = 1 << 18, 64 * G, 32
    xs = shards_of(dist_name, G, n_per, 51)
    out, _, counts, sk, st, _ = dist_sort_virtual([torch.from_numpy(x).cuda() for x in xs], None, p, s, 1)
    ref = orc.ros_sort(np.concatenate(xs), p, s, 1)
    check(ref, out, None, counts, sk, st)


@pytest.mark.parametrize("dist_name,G", [("u16key", 4), ("f64_normal", 2), ("i32_gauss", 8), ("u32_few4", 2)])
def test_virtual_ranks_kv_and_dtypes(orc, dist_name, G):
    from paper_1608_08648_b200.dist import dist_sort_virtual
    n_per, p, s = 200_000, 32 * G, 16
    xs = shards_of(dist_name, G, n_per, 5)
    vs = [ovs_inputs.index_values(n_per, r * n_per) for r in range(G)]
    out, vout, counts, sk, st, _ = dist_sort_virtual([torch.from_numpy(x).cuda() for x in xs],
                                                     [torch.from_numpy(v).cuda() for v in vs], p, s, 2)
    ref = orc.ros_sort(np.concatenate(xs), p, s, 2, vals=np.concatenate(vs))
    check(ref, out, vout, counts, sk, st)


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
    out, vout, counts, sk, st, _ = dist_sort_virtual(
        [torch.from_numpy(np.ascontiguousarray(a)).cuda() for a in xs],
        [torch.from_numpy(np.ascontiguousarray(a)).cuda() for a in vs] if kv else None, p, s, 9)
    ref = orc.ros_sort(x, p, s, 9, vals=v)
    check(ref, out, vout, counts, sk, st)


def _full_size_check(G, dist_name, n_per, p, s, seed):
    """Full-size C5 shards (oracle too slow at 2^28): per-rank slices equal the slices of the
    global sort of the concatenation (numpy, a library sort: the unique sorted output), counts sum
    to n and are consistent with the slices, splitters are sorted (key, tag) pairs whose counts
    match a brute classification of the keys around each splitter."""
    from paper_1608_08648_b200.dist import dist_sort_virtual, owned
    xs = shards_of(dist_name, G, n_per, seed)
    out, _, counts, sk, st, n_out = dist_sort_virtual([torch.from_numpy(x).cuda() for x in xs], None, p, s, 1)
    x = np.concatenate(xs)
    ref = np.sort(x)
    np.testing.assert_array_equal(out.cpu().numpy(), ref)
    assert int(counts.sum()) == len(x)
    for r in range(G):
        b0, b1 = owned(G, p, r)
        assert int(n_out[r]) == int(counts[b0:b1].sum())
    # bucket j = (S[j-1], S[j]] in (key, global index) order: the count up to splitter q is the
    # number of (key, index) pairs <= (sk[q], st[q])
    below = np.searchsorted(ref, sk, side="left").astype(np.int64)  # keys < sk[q]
    eq_before = np.array([int(np.count_nonzero((x == sk[q])[:int(st[q]) + 1])) for q in range(0, p - 1, max(1, p // 16))])
    cum = np.cumsum(counts)[:-1]
    idx = np.arange(0, p - 1, max(1, p // 16))
    np.testing.assert_array_equal(cum[idx], below[idx] + eq_before)
    assert np.all(x[st.astype(np.int64)] == sk)


@pytest.mark.slow
@pytest.mark.parametrize("dist_name", ["u32_staggered", "u32_bucketsorted"])
def test_virtual_ranks_c5_full_size(dist_name):
    """C5 staggered and bucket-sorted distributions at 2^27 keys per rank, G = 2 (the bench's
    p = 4096 and s = 64): sorted output, counts, ownership and splitter consistency."""
    _full_size_check(2, dist_name, 1 << 27, 4096, 64, 52 if dist_name == "u32_staggered" else 53)


def _free_port():
    s_ = socket.socket()
    s_.bind(("127.0.0.1", 0))
    port = s_.getsockname()[1]
    s_.close()
    return port


@pytest.fixture(scope="module")
def nccl_world1():
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(_free_port()), RANK="0", WORLD_SIZE="1")
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    yield dist
    dist.destroy_process_group()


@pytest.mark.parametrize("dist_name,n,p,s,kv", [("u32", 1 << 20, 256, 32, False), ("f64_normal", 300_001, 64, 16, True),
                                                ("i32_few", 1 << 21, 1024, 64, False)])
def test_nccl_comm_world1(orc, nccl_world1, dist_name, n, p, s, kv):
    """The real path: NCCL communicator, symmetric window (ncclMemAlloc + window registration),
    NVLink/LSA peer pointers and LSA barriers, world_size 1."""
    from paper_1608_08648_b200.dist import DistSorter
    x = ovs_inputs.keys(dist_name, n, seed=3)
    v = ovs_inputs.index_values(n) if kv else None
    ds = DistSorter(n, torch.from_numpy(x).dtype, kv, p, s, 4)
    xt = torch.from_numpy(x).cuda()
    res = ds(xt, torch.from_numpy(v).cuda() if kv else None, report=True)
    ref = orc.ros_sort(x, p, s, 4, vals=v)
    check(ref, res.keys, res.vals, res.counts, res.splitter_keys, res.splitter_tags)
    assert res.n_before == 0 and res.exchange_bytes == 0
    # a second call on the same communicator (window reuse across calls)
    res2 = ds(xt, torch.from_numpy(v).cuda() if kv else None)
    np.testing.assert_array_equal(res2.keys.cpu().numpy(), ref.keys)
    np.testing.assert_array_equal(xt.cpu().numpy(), x)  # the input shard is not modified
    ds.close()


def test_nccl_capacity_retry(orc, nccl_world1):
    """A window / output too small for the received items: OVS_ECAPACITY with the requirement,
    then DistSorter grows both (ovs_comm_reserve) and the sort succeeds."""
    from paper_1608_08648_b200.dist import DistSorter
    n, p, s = 500_000, 64, 16
    x = ovs_inputs.keys("u32", n, seed=8)
    ds = DistSorter(n, torch.uint32, False, p, s, 2, out_capacity=1000, window_bytes=1 << 20)
    res = ds(torch.from_numpy(x).cuda(), report=True)
    ref = orc.ros_sort(x, p, s, 2)
    check(ref, res.keys, None, res.counts, res.splitter_keys, res.splitter_tags)
    assert ds.out_cap >= n and ds.window_bytes() >= 4 * n
    ds.close()


# ---------------------------------------------------------------- DRO across GPUs (§8(e) DRO steps)
@pytest.mark.parametrize("G,dist_name,n_per,p,r,kv,padded", [
    (1, "i32_uniform", 1 << 18, 64, 4, False, False), (2, "i32_gauss", 1 << 18, 64, 4, False, False),
    (4, "u16key", 1 << 17, 32, 3, True, False), (2, "f64_normal", 1 << 17, 16, 5, True, True),
    (8, "u32_few4", 1 << 16, 64, 2, False, False), (4, "u32", 1 << 20, 256, 8, False, True)])
def test_virtual_ranks_dro(orc, G, dist_name, n_per, p, r, kv, padded):
    """Rank g holds the p/G whole sequences of its shard; samples, splitters, split, exchange and the
    owners' sorts equal the single-process Algorithm 1 on the concatenation (keys, values,
    splitters, counts)."""
    from paper_1608_08648_b200.dist import dist_sort_virtual
    n = G * n_per
    x = ovs_inputs.keys(dist_name, n, seed=19) if dist_name in ("i32_sorted",) else \
        np.concatenate([ovs_inputs.keys(dist_name, n_per, seed=19, start=g * n_per) for g in range(G)])
    v = ovs_inputs.index_values(n) if kv else None
    xs = [torch.from_numpy(np.ascontiguousarray(x[g * n_per:(g + 1) * n_per])).cuda() for g in range(G)]
    vs = [torch.from_numpy(np.ascontiguousarray(v[g * n_per:(g + 1) * n_per])).cuda() for g in range(G)] if kv else None
    out, vout, counts, sk, st, _ = dist_sort_virtual(xs, vs, p, r, 0, method="dro", padded=padded)
    ref = orc.dro_sort(x, p, r, vals=v, padded=padded)
    check(ref, out, vout, counts, sk, st)


def test_nccl_comm_world1_dro(orc, nccl_world1):
    from paper_1608_08648_b200.dist import DistSorter
    n, p, r = 1 << 20, 128, 6
    x = ovs_inputs.keys("i32_gauss", n, seed=4)
    v = ovs_inputs.index_values(n)
    ds = DistSorter(n, torch.int32, True, p, r, 0, method="dro")
    res = ds(torch.from_numpy(x).cuda(), torch.from_numpy(v).cuda(), report=True)
    ref = orc.dro_sort(x, p, r, vals=v)
    check(ref, res.keys, res.vals, res.counts, res.splitter_keys, res.splitter_tags)
    ds.close()
