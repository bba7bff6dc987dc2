"""The multi-GPU host logic (paper_1608_08648_b200/dist.py) with world_size 2 and 3 over gloo
on CPU: shard offsets, the all-reduce that assembles the global sample, the all-gather of the
count matrix, the all-to-all split sizes, bucket ownership (p a multiple of world,
PAPER.md:669-670) and the per-rank output slices.  The device steps are replaced by a CPU test
backend implementing the same contract from the oracle's pieces; the result must equal the
single-process oracle on the rank-ordered concatenation (splitters, counts, output)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import ovs_inputs


class CpuBackend:
    """Test double of dist.CudaBackend on CPU tensors (test infrastructure)."""

    def __init__(self, n_local, n_global, p, s, seed, kv):
        import oracle
        self.orc = oracle
        self.n_local, self.n_global, self.p, self.s, self.seed, self.kv = n_local, n_global, p, s, seed, kv

    def sample(self, keys, offset):
        I, _ = self.orc.ros_sample_indices(self.n_global, self.p, self.s, self.seed)
        I = np.sort(I.astype(np.int64))
        rec = torch.zeros(2 * len(I), dtype=torch.int64)
        x = keys.numpy()
        for t, gi in enumerate(I):
            if offset <= gi < offset + self.n_local:
                rec[2 * t] = int(np.float64(x[gi - offset]).view(np.int64)) if x.dtype == np.float64 else int(x[gi - offset])
                rec[2 * t + 1] = int(gi)
        return rec

    def partition(self, keys, vals, offset, rec):
        x = keys.numpy()
        r = rec.numpy().reshape(-1, 2)
        tk = r[:, 0].view(np.float64) if x.dtype == np.float64 else r[:, 0]
        order = np.lexsort((r[:, 1], tk))
        T = [(tk[i], int(r[i, 1])) for i in order]
        self.S = [T[(q + 1) * self.s - 1] for q in range(self.p - 1)]
        gi = offset + np.arange(len(x))
        sk = np.array([k for k, _ in self.S]) if self.S else np.zeros(0)
        st = np.array([t for _, t in self.S], dtype=np.int64)
        # bucket = #{q : S[q] <lex (x, gi)}
        b = np.searchsorted(sk, x, side="left")
        hi = np.searchsorted(sk, x, side="right")
        for i in range(len(x)):
            b[i] += int(np.sum(st[b[i]:hi[i]] < gi[i]))
        o = np.argsort(b, kind="stable")
        counts = np.bincount(b, minlength=self.p).astype(np.int32)
        sv = torch.from_numpy(vals.numpy()[o].copy()) if vals is not None else None
        si = torch.from_numpy(gi[o].astype(np.uint32)) if self.kv else None
        return torch.from_numpy(x[o].copy()), sv, si, torch.from_numpy(counts)

    def reserve(self, n):
        pass

    def finish(self, rk, rv, ri, C, rank, n_recv):
        k = rk.numpy()
        if self.kv:
            o = np.lexsort((ri.numpy(), k))
            return torch.from_numpy(k[o].copy()), torch.from_numpy(rv.numpy()[o].copy())
        return torch.from_numpy(np.sort(k)), None


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, dist_name, n_per, p, s, kv, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1608_08648_b200.dist import dist_sort
    n_local = n_per + rank  # ragged shards
    start = sum(n_per + r for r in range(rank))
    x = ovs_inputs.keys(dist_name, n_local, seed=7, start=start, world=world, rank=rank)
    v = ovs_inputs.index_values(n_local, start) if kv else None
    n_global = sum(n_per + r for r in range(world))
    be = CpuBackend(n_local, n_global, p, s, 3, kv)
    res = dist_sort(torch.from_numpy(x), torch.from_numpy(v) if kv else None, p, s, 3, backend=be)
    q.put((rank, res.keys.numpy(), None if res.vals is None else res.vals.numpy(), res.counts, res.n_before,
           [be.S[i] for i in range(len(be.S))]))
    dist.destroy_process_group()


@pytest.mark.parametrize("world,dist_name,kv", [(2, "u32_u31", False), (2, "u32_few4", True), (3, "i32_gauss", False),
                                                (2, "f64_normal", True)])
def test_dist_host_logic_matches_oracle(orc, world, dist_name, kv):
    n_per, p, s = 2000, 6 * world, 8
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, dist_name, n_per, p, s, kv, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    got = sorted([q.get(timeout=120) for _ in range(world)], key=lambda t: t[0])
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    # the single-process oracle on the concatenation
    xs, vs = [], []
    start = 0
    for r in range(world):
        n_local = n_per + r
        xs.append(ovs_inputs.keys(dist_name, n_local, seed=7, start=start, world=world, rank=r))
        vs.append(ovs_inputs.index_values(n_local, start))
        start += n_local
    x = np.concatenate(xs)
    ref = orc.ros_sort(x, p, s, 3, vals=np.concatenate(vs) if kv else None)
    np.testing.assert_array_equal(np.concatenate([g[1] for g in got]), ref.keys)
    if kv:
        np.testing.assert_array_equal(np.concatenate([g[2] for g in got]), ref.vals)
    for g in got:
        np.testing.assert_array_equal(g[3], ref.counts)
        assert [t for _, t in g[5]] == ref.split_tags.tolist()
    assert got[0][4] == 0 and got[-1][4] + len(got[-1][1]) == len(x)


def test_exchange_plan_ownership():
    from paper_1608_08648_b200.dist import exchange_plan, owned
    world, p = 4, 8
    C = np.arange(world * p).reshape(world, p)
    assert [owned(world, p, r) for r in range(world)] == [(0, 2), (2, 4), (4, 6), (6, 8)]
    send, recv = exchange_plan(C, world, p, 1)
    assert send == [C[1, 0:2].sum(), C[1, 2:4].sum(), C[1, 4:6].sum(), C[1, 6:8].sum()]
    assert recv == [C[s, 2:4].sum() for s in range(world)]
