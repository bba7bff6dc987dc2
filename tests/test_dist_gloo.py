"""The multi-GPU exchange protocol with world_size 2 and 3 over gloo on CPU (no GPU needed).

Each process is one rank holding a ragged shard.  It computes what the library's device steps
compute (the global sample, the splitters and its bucket counts, here from the oracle's sample
index set and a plain lexicographic classification: test infrastructure), all-gathers the count
matrix, and takes the exchange plan from the LIBRARY's host code (ovs_dist_plan, the function
ovs_dist_sort_* runs).  Every rank then sends each key to its owner (bucket j on rank
floor(j*world/p)) at the position the plan gives (all_to_all over gloo, in place
of the NVLink stores), the owner checks that the runs of all senders tile its receive region
exactly, sorts every owned bucket by (key, global index), and the concatenation over ranks must
equal the single-process oracle (output, values, counts, splitters)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import ovs_inputs


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _classify(x, gidx, sk, st):
    """bucket = #{q : (sk[q], st[q]) <lex (x, gidx)} (reading Q5), vectorised."""
    b = np.searchsorted(sk, x, side="left")
    hi = np.searchsorted(sk, x, side="right")
    for i in np.nonzero(hi > b)[0]:
        b[i] += int(np.sum(st[b[i]:hi[i]] < gidx[i]))
    return b


def _worker(rank, world, port, dist_name, n_per, p, s, kv, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle
    from paper_1608_08648_b200.dist import exchange_plan, owned
    sizes = [n_per + r for r in range(world)]  # ragged shards
    start = sum(sizes[:rank])
    n_local, n_global = sizes[rank], sum(sizes)
    x = ovs_inputs.keys(dist_name, n_local, seed=7, start=start, world=world, rank=rank)
    v = ovs_inputs.index_values(n_local, start) if kv else None
    gidx = start + np.arange(n_local, dtype=np.int64)
    # the global sample (same on every rank) and this shard's records, assembled by all-gather
    I, _ = oracle.ros_sample_indices(n_global, p, s, 3)
    I = I.astype(np.int64)
    mine = (I >= start) & (I < start + n_local)
    rec = np.zeros((len(I), 2), dtype=np.float64 if x.dtype == np.float64 else np.int64)
    rec[mine, 0] = x[I[mine] - start]
    rec[mine, 1] = I[mine]
    got = [torch.zeros_like(torch.from_numpy(rec)) for _ in range(world)]
    dist.all_gather(got, torch.from_numpy(rec))
    T = sum(g.numpy() for g in got)  # every slot filled by exactly one rank
    order = np.lexsort((T[:, 1], T[:, 0]))
    S = T[order][np.arange(1, p) * s - 1]
    sk, st = S[:, 0].astype(x.dtype), S[:, 1].astype(np.int64)
    b = _classify(x, gidx, sk, st)
    counts = np.bincount(b, minlength=p).astype(np.uint32)
    allc = [torch.zeros(p, dtype=torch.int64) for _ in range(world)]
    dist.all_gather(allc, torch.from_numpy(counts.astype(np.int64)))
    C = np.stack([c.numpy() for c in allc]).astype(np.uint32)
    dst_off, recv = exchange_plan(C, world, p, rank)  # the library's host plan
    # positions inside the owners' receive regions: dst_off[b] + rank of the key in this rank's run
    o = np.argsort(b, kind="stable")
    run_start = np.concatenate([[0], np.cumsum(counts)[:-1]]).astype(np.int64)
    pos = np.empty(n_local, dtype=np.int64)
    pos[o] = dst_off[b[o]].astype(np.int64) + (np.arange(n_local) - run_start[b[o]])
    owner = (b.astype(np.int64) * world) // p
    send, recv_sizes = [], [int(C[r, slice(*owned(world, p, rank))].sum()) for r in range(world)]
    payload = [np.stack([pos[owner == d], gidx[owner == d], (v[owner == d] if kv else np.zeros(int((owner == d).sum()))).astype(np.int64),
                         x[owner == d].view(np.int64) if x.dtype == np.float64 else x[owner == d].astype(np.int64)], 1)
               for d in range(world)]
    send = torch.from_numpy(np.concatenate(payload).astype(np.int64)) if n_local else torch.zeros((0, 4), dtype=torch.int64)
    out = torch.zeros((sum(recv_sizes), 4), dtype=torch.int64)
    dist.all_to_all_single(out, send, recv_sizes, [len(pp) for pp in payload])
    R = out.numpy()
    n_out = int(recv[rank])
    assert n_out == len(R)
    hit = np.zeros(n_out, dtype=np.int64)
    np.add.at(hit, R[:, 0], 1)
    assert np.all(hit == 1), "the senders' runs must tile the receive region exactly"
    region = np.empty_like(R)
    region[R[:, 0]] = R
    keys = region[:, 3].view(np.float64) if x.dtype == np.float64 else region[:, 3].astype(x.dtype)
    # every owned bucket (contiguous in the region) sorted by (key, global index)
    b0, b1 = owned(world, p, rank)
    tot = C.sum(axis=0).astype(np.int64)
    ok, ov = [], []
    at = 0
    for j in range(b0, b1):
        seg = slice(at, at + int(tot[j]))
        oo = np.lexsort((region[seg, 1], keys[seg]))
        ok.append(keys[seg][oo])
        ov.append(region[seg, 2][oo])
        at += int(tot[j])
    q.put((rank, np.concatenate(ok) if ok else keys[:0], np.concatenate(ov).astype(np.uint32) if ov else None,
           C.sum(axis=0), sk, st))
    dist.destroy_process_group()


@pytest.mark.parametrize("world,dist_name,kv", [(2, "u32_u31", False), (2, "u32_few4", True), (3, "i32_gauss", False),
                                                (2, "f64_normal", True), (3, "u32_staggered", False)])
def test_dist_exchange_protocol_matches_oracle(orc, world, dist_name, kv):
    n_per, p, s = 2000, 6 * world, 8
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, dist_name, n_per, p, s, kv, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    got = sorted([q.get(timeout=180) for _ in range(world)], key=lambda t: t[0])
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    xs, vs = [], []
    start = 0
    for r in range(world):
        n_local = n_per + r
        xs.append(ovs_inputs.keys(dist_name, n_local, seed=7, start=start, world=world, rank=r))
        vs.append(ovs_inputs.index_values(n_local, start))
        start += n_local
    ref = orc.ros_sort(np.concatenate(xs), p, s, 3, vals=np.concatenate(vs) if kv else None)
    np.testing.assert_array_equal(np.concatenate([g[1] for g in got]), ref.keys)
    if kv:
        np.testing.assert_array_equal(np.concatenate([g[2] for g in got]), ref.vals)
    for g in got:
        np.testing.assert_array_equal(g[3], ref.counts)
        np.testing.assert_array_equal(g[4], ref.split_keys)
        np.testing.assert_array_equal(g[5], ref.split_tags)


def test_exchange_plan_closed_form():
    """ovs_dist_plan against its definition on a hand-checkable matrix (4 ranks, 8 buckets)."""
    from paper_1608_08648_b200.dist import exchange_plan, owned
    world, p = 4, 8
    C = np.arange(1, world * p + 1, dtype=np.uint32).reshape(world, p)
    assert [owned(world, p, r) for r in range(world)] == [(0, 2), (2, 4), (4, 6), (6, 8)]
    tot = C.sum(axis=0)
    for rank in range(world):
        dst, recv = exchange_plan(C, world, p, rank)
        for b in range(p):
            d = b * world // p
            b0 = owned(world, p, d)[0]
            assert dst[b] == tot[b0:b].sum() + C[:rank, b].sum()
        assert recv.tolist() == [int(tot[slice(*owned(world, p, d))].sum()) for d in range(world)]
