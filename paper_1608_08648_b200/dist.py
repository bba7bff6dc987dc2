"""Multi-GPU sort (ROS): one process per GPU, NCCL collectives through torch.distributed.

The work is split the way the paper's multi-core method splits it (SURVEY.md
§8(e)): every GPU samples its shard, the sample is assembled on every GPU (all-reduce), every
GPU classifies its keys against the same splitters and scatters them into destination order
(kernels), the bucket counts are all-gathered, the buckets are exchanged (all-to-all-v over
NVLink/NVSwitch), and every GPU sorts the buckets it received (kernels).  Bucket j lives on
rank floor(j*world/p) (p must be a multiple of world).  Rank r's output is
exactly its slice of the single-GPU sort of the rank-ordered concatenation of the shards.

Only argument marshalling and the collectives live here; every compute step runs in the
library's kernels (include/ovs.h, ovs_dist_*).  `Backend` is the seam the CPU gloo tests use
to exercise this host logic without a GPU.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import (OVS_F64, OVS_I32, OVS_OK, OVS_U32, OvsError, lib, params)


def _ensure_sigs():
    L = lib()
    if getattr(L, "_dist_sigs", False):
        return L
    vp, sz, i32, u64 = ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int, ctypes.c_uint64
    from . import Params
    P = ctypes.POINTER(Params)
    L.ovs_dist_workspace_bytes.restype = sz
    L.ovs_dist_workspace_bytes.argtypes = [sz, u64, i32, i32, P, i32, sz]
    L.ovs_dist_sample_words.restype = sz
    L.ovs_dist_sample_words.argtypes = [u64, i32, P]
    L.ovs_dist_sample.restype = i32
    L.ovs_dist_sample.argtypes = [vp, sz, u64, u64, i32, i32, P, i32, sz, vp, vp, sz, vp]
    L.ovs_dist_partition.restype = i32
    L.ovs_dist_partition.argtypes = [vp, vp, sz, u64, u64, i32, P, i32, sz, vp, vp, vp, vp, vp, vp, sz, vp]
    L.ovs_dist_finish.restype = i32
    L.ovs_dist_finish.argtypes = [vp, vp, vp, sz, u64, i32, P, i32, i32, sz, vp, vp, vp, vp, sz, vp]
    L._dist_sigs = True
    return L


def _dtcode(dt):
    import torch
    m = {torch.uint32: OVS_U32, torch.int32: OVS_I32, torch.float64: OVS_F64}
    return m[dt]


def _ptr(t):
    return None if t is None else t.data_ptr()


def owned(world: int, p: int, r: int):
    """Buckets [b0, b1) owned by rank r."""
    return (r * p) // world, ((r + 1) * p) // world


def exchange_plan(C: np.ndarray, world: int, p: int, rank: int):
    """Split sizes of the all-to-all from the all-gathered count matrix C (world x p):
    send_split[d] = this rank's items of d's buckets; recv_split[s] = s's items of ours."""
    send = [int(C[rank, slice(*owned(world, p, d))].sum()) for d in range(world)]
    recv = [int(C[s, slice(*owned(world, p, rank))].sum()) for s in range(world)]
    return send, recv


class CudaBackend:
    """The product backend: the three C-ABI steps on CUDA tensors."""

    def __init__(self, n_local, n_global, dtype, kv, p, s, seed, world, recv_capacity, device):
        import torch
        self.L = _ensure_sigs()
        self.prm = params("ros", p, s, seed)
        self.dt = _dtcode(dtype)
        self.dtype, self.kv, self.world, self.device = dtype, kv, world, device
        self.n_local, self.n_global = n_local, n_global
        self.p = p
        self.cap = max(int(recv_capacity), 1)
        nb = self._ws_bytes(self.cap)
        if nb == 0:
            raise OvsError(1, self.L.ovs_last_error().decode() or "invalid distributed arguments")
        self.ws = torch.empty(nb, dtype=torch.uint8, device=device)
        self.words = int(self.L.ovs_dist_sample_words(n_global, self.dt, ctypes.byref(self.prm)))

    def _ws_bytes(self, cap):
        return int(self.L.ovs_dist_workspace_bytes(self.n_local, self.n_global, self.dt, 1 if self.kv else 0,
                                                   ctypes.byref(self.prm), self.world, cap))

    def _check(self, rc):
        if rc != OVS_OK:
            raise OvsError(rc, self.L.ovs_last_error().decode())

    def _stream(self):
        import torch
        return ctypes.c_void_p(torch.cuda.current_stream(self.device).cuda_stream)

    def sample(self, keys, offset):
        import torch
        rec = torch.empty(self.words, dtype=torch.int64, device=self.device)
        self._check(self.L.ovs_dist_sample(keys.data_ptr(), self.n_local, offset, self.n_global, self.dt,
                                           1 if self.kv else 0, ctypes.byref(self.prm), self.world, self.cap,
                                           rec.data_ptr(), self.ws.data_ptr(), self.ws.numel(), self._stream()))
        return rec

    def partition(self, keys, vals, offset, rec):
        import torch
        sk = torch.empty_like(keys)
        sv = torch.empty_like(vals) if self.kv else None
        si = torch.empty(self.n_local, dtype=torch.uint32, device=self.device) if self.kv else None
        counts = torch.empty(self.p, dtype=torch.int32, device=self.device)
        self._check(self.L.ovs_dist_partition(keys.data_ptr(), _ptr(vals), self.n_local, offset, self.n_global,
                                              self.dt, ctypes.byref(self.prm), self.world, self.cap, rec.data_ptr(),
                                              sk.data_ptr(), _ptr(sv), _ptr(si), counts.data_ptr(),
                                              self.ws.data_ptr(), self.ws.numel(), self._stream()))
        return sk, sv, si, counts

    def reserve(self, n_recv):
        """Grow recv_capacity: the workspace prefix (sample, splitters) keeps its layout."""
        import torch
        if n_recv <= self.cap:
            return
        nb = self._ws_bytes(n_recv)
        ws = torch.empty(nb, dtype=torch.uint8, device=self.device)
        ws[: self.ws.numel()].copy_(self.ws)
        self.ws, self.cap = ws, n_recv

    def finish(self, rk, rv, ri, C, rank, n_recv):
        import torch
        ok = torch.empty(n_recv, dtype=self.dtype, device=self.device)
        ov = torch.empty(n_recv, dtype=torch.uint32, device=self.device) if self.kv else None
        self._check(self.L.ovs_dist_finish(rk.data_ptr(), _ptr(rv), _ptr(ri), self.n_local, self.n_global, self.dt,
                                           ctypes.byref(self.prm), self.world, rank, self.cap, C.data_ptr(),
                                           ok.data_ptr(), _ptr(ov), self.ws.data_ptr(), self.ws.numel(),
                                           self._stream()))
        return ok, ov


@dataclass
class DistResult:
    keys: object            # this rank's sorted slice (torch tensor)
    vals: object            # values (key-value sorts) or None
    counts: np.ndarray      # the p global bucket counts
    n_before: int           # number of keys on lower ranks (this slice's global offset)
    exchange_bytes: int     # bytes this rank sent to other ranks


def _as_comm(t):
    """Bit-identical view with a dtype every backend's collectives accept."""
    import torch
    if t is None:
        return None
    if t.dtype == torch.uint32:
        return t.view(torch.int32)
    return t


def dist_sort(keys, vals=None, p: int = 1024, s: int = 64, seed: int = 1, group=None, backend=None,
              recv_capacity=None) -> DistResult:
    """Sort the rank-ordered concatenation of every rank's `keys` (and `vals`) across the
    process group; returns this rank's slice.  Collective: every rank must call it."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    dev = keys.device
    kv = vals is not None
    n_local = keys.numel()
    # shard sizes -> global offsets (ranks in index order)
    sizes = torch.zeros(world, dtype=torch.int64, device=dev)
    mine = torch.tensor([n_local], dtype=torch.int64, device=dev)
    dist.all_gather_into_tensor(sizes, mine, group=group)
    sizes_h = sizes.cpu().tolist()
    offset, n_global = int(sum(sizes_h[:rank])), int(sum(sizes_h))
    if backend is None:
        backend = CudaBackend(n_local, n_global, keys.dtype, kv, p, s, seed, world,
                              recv_capacity or max(2 * n_local, 1024), dev)
    # 1. sample: this shard's records of the global sample; all-reduce assembles T
    rec = backend.sample(keys, offset)
    dist.all_reduce(rec, op=dist.ReduceOp.SUM, group=group)
    # 2. splitters, local counts, destination-ordered send buffers
    sk, sv, si, counts = backend.partition(keys, vals, offset, rec)
    C = torch.empty(world * p, dtype=torch.int32, device=dev)
    dist.all_gather_into_tensor(C, counts, group=group)
    Ch = C.view(world, p).cpu().numpy().astype(np.int64)
    send, recv = exchange_plan(Ch, world, p, rank)
    n_recv = int(sum(recv))
    # 3. all-to-all-v of the buckets
    rk = torch.empty(n_recv, dtype=keys.dtype, device=dev)
    dist.all_to_all_single(_as_comm(rk), _as_comm(sk), recv, send, group=group)
    rv = ri = None
    if kv:
        rv = torch.empty(n_recv, dtype=torch.uint32, device=dev)
        ri = torch.empty(n_recv, dtype=torch.uint32, device=dev)
        dist.all_to_all_single(_as_comm(rv), _as_comm(sv), recv, send, group=group)
        dist.all_to_all_single(_as_comm(ri), _as_comm(si), recv, send, group=group)
    # 4. gather every owned bucket's runs (source order) and sort them
    backend.reserve(n_recv)
    ok, ov = backend.finish(rk, rv, ri, C, rank, n_recv)
    counts_g = Ch.sum(axis=0)
    b0, _ = owned(world, p, rank)
    item = keys.element_size() + (8 if kv else 0)
    sent_out = sum(send) - send[rank]
    return DistResult(ok, ov, counts_g, int(counts_g[:b0].sum()), int(sent_out * item))


def dist_sort_virtual(shards, vals=None, p: int = 1024, s: int = 64, seed: int = 1):
    """The same three steps for G shards held by ONE process on one GPU (the collectives are
    emulated with device copies, one rank after the other; no kernel waits on another).
    Used to test the multi-rank kernels on a single GPU.  Returns the concatenated output,
    values and the global counts."""
    import torch
    world = len(shards)
    kv = vals is not None
    dev = shards[0].device
    sizes = [int(x.numel()) for x in shards]
    n_global = sum(sizes)
    offs = [sum(sizes[:r]) for r in range(world)]
    bes = [CudaBackend(sizes[r], n_global, shards[0].dtype, kv, p, s, seed, world, max(2 * sizes[r], 1024), dev)
           for r in range(world)]
    recs = [bes[r].sample(shards[r], offs[r]) for r in range(world)]
    rec = torch.stack(recs).sum(0)
    parts = [bes[r].partition(shards[r], vals[r] if kv else None, offs[r], rec.clone()) for r in range(world)]
    C = torch.cat([pp[3] for pp in parts])
    Ch = C.view(world, p).cpu().numpy().astype(np.int64)
    outs, vouts = [], []
    for r in range(world):
        pieces_k, pieces_v, pieces_i = [], [], []
        for src in range(world):
            send, _ = exchange_plan(Ch, world, p, src)
            a = sum(send[:r])
            pieces_k.append(parts[src][0][a:a + send[r]])
            if kv:
                pieces_v.append(parts[src][1][a:a + send[r]])
                pieces_i.append(parts[src][2][a:a + send[r]])
        rk = torch.cat(pieces_k)
        rv = torch.cat(pieces_v) if kv else None
        ri = torch.cat(pieces_i) if kv else None
        bes[r].reserve(rk.numel())
        ok, ov = bes[r].finish(rk, rv, ri, C, r, rk.numel())
        outs.append(ok)
        vouts.append(ov)
    torch.cuda.synchronize(dev)
    return torch.cat(outs), (torch.cat(vouts) if kv else None), Ch.sum(axis=0)
