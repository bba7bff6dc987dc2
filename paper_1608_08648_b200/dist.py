"""Multi-GPU sort (ROS) through the library's communicator (include/ovs.h, ovs_comm_* and
ovs_dist_*): argument marshalling only.

One process per GPU.  The library owns the NCCL communicator and its symmetric window; every
step, including the exchange (the scatter stores each key straight into its owner's window over
NVLink) and the barriers between the phases, runs inside libovs.  Python only
hands the NCCL unique id from rank 0 to the others (torch.distributed broadcast) and allocates
the tensors.  Rank r's output is exactly its slice of the single-GPU sort of the rank-ordered
concatenation of the shards (bucket j lives on rank floor(j*world/p), p a
multiple of world).
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import (OVS_ECAPACITY, OVS_F64, OVS_I32, OVS_OK, OVS_U32, OvsError, Params, Report, _NP, lib, params)


def _ensure_sigs():
    L = lib()
    if getattr(L, "_dist_sigs", False):
        return L
    vp, sz, i32, u32 = ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int, ctypes.c_uint32
    P = ctypes.POINTER(Params)
    L.ovs_comm_unique_id.restype = i32
    L.ovs_comm_unique_id.argtypes = [vp]
    L.ovs_comm_create.restype = i32
    L.ovs_comm_create.argtypes = [ctypes.POINTER(vp), vp, i32, i32, i32, sz]
    L.ovs_comm_reserve.restype = i32
    L.ovs_comm_reserve.argtypes = [vp, sz, vp]
    L.ovs_comm_destroy.restype = i32
    L.ovs_comm_destroy.argtypes = [vp]
    L.ovs_comm_window_bytes.restype = sz
    L.ovs_comm_window_bytes.argtypes = [vp]
    L.ovs_dist_window_bytes.restype = sz
    L.ovs_dist_window_bytes.argtypes = [sz, i32, i32, P, i32]
    L.ovs_dist_workspace_bytes.restype = sz
    L.ovs_dist_workspace_bytes.argtypes = [vp, sz, i32, i32, P, sz, vp]
    L.ovs_dist_sort_keys.restype = i32
    L.ovs_dist_sort_keys.argtypes = [vp, vp, sz, i32, P, vp, sz, ctypes.POINTER(sz), vp, sz, vp,
                                     ctypes.POINTER(Report)]
    L.ovs_dist_sort_pairs_stable.restype = i32
    L.ovs_dist_sort_pairs_stable.argtypes = [vp, vp, vp, sz, i32, P, vp, vp, sz, ctypes.POINTER(sz), vp, sz, vp,
                                             ctypes.POINTER(Report)]
    L.ovs_dist_plan.restype = i32
    L.ovs_dist_plan.argtypes = [vp, i32, u32, i32, vp, vp]
    L.ovs_dist_sort_virtual.restype = i32
    L.ovs_dist_sort_virtual.argtypes = [i32, vp, vp, vp, i32, P, vp, vp, vp, vp, vp, vp, vp, sz, vp, vp, vp, vp, vp]
    L.ovs_dist_virtual_workspace_bytes.restype = sz
    L.ovs_dist_virtual_workspace_bytes.argtypes = [i32, vp, i32, i32, P, vp, sz]
    L._dist_sigs = True
    return L


def _dtcode(dt):
    import torch
    m = {torch.uint32: OVS_U32, torch.int32: OVS_I32, torch.float64: OVS_F64}
    if dt not in m:
        raise OvsError(2, f"unsupported dtype {dt}")
    return m[dt]


def owned(world: int, p: int, r: int):
    """Buckets [b0, b1) owned by rank r (bucket j on rank floor(j*world/p))."""
    return (r * p) // world, ((r + 1) * p) // world


def exchange_plan(C: np.ndarray, world: int, p: int, rank: int):
    """ovs_dist_plan (the library's host plan): dst_off[b] = where `rank`'s run of bucket b starts
    inside its owner's receive region; recv[r] = items rank r receives.  C = world x p counts."""
    L = _ensure_sigs()
    C = np.ascontiguousarray(C, dtype=np.uint32)
    dst = np.zeros(p, dtype=np.uint32)
    recv = np.zeros(world, dtype=np.uint64)
    rc = L.ovs_dist_plan(C.ctypes.data, world, p, rank, dst.ctypes.data, recv.ctypes.data)
    if rc != OVS_OK:
        raise OvsError(rc, "ovs_dist_plan")
    return dst, recv


@dataclass
class DistResult:
    keys: object            # this rank's sorted slice (torch tensor, n_out items)
    vals: object            # values (key-value sorts) or None
    counts: np.ndarray      # the p global bucket counts (report) or None
    n_before: int           # keys on lower ranks (this slice's global offset), or -1 without report
    splitter_keys: np.ndarray
    splitter_tags: np.ndarray
    exchange_bytes: int     # bytes this rank stored into other ranks' windows (report) or -1
    phase_ms: list
    kernel_launches: int = -1  # kernels the call enqueued (report)


class DistSorter:
    """One rank's handle: the library communicator (NCCL + symmetric window), the workspace and
    the output buffers, sized for shards of n_local keys; collective like NCCL (every rank of
    `group` constructs it and calls it the same number of times)."""

    def __init__(self, n_local: int, dtype, with_values: bool = False, p: int = 1024, s: int = 64, seed: int = 1,
                 group=None, device=None, out_capacity: int | None = None, window_bytes: int | None = None,
                 method: str = "ros", padded: bool = False):
        import torch
        import torch.distributed as dist
        self.L = _ensure_sigs()
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.dtype, self.dt, self.kv = dtype, _dtcode(dtype), with_values
        self.prm = params(method, p, s, seed, padded)  # DRO: s = r, equal shards of whole sequences
        self.p = p
        self.n_local = n_local
        # the NCCL unique id: rank 0 draws it, the process group broadcasts the 128 bytes
        idb = np.zeros(128, dtype=np.uint8)
        if self.rank == 0:
            self._check(self.L.ovs_comm_unique_id(idb.ctypes.data))
        backend = dist.get_backend(group)
        t = torch.from_numpy(idb)
        if backend == "nccl":
            t = t.to(self.device)
        dist.broadcast(t, src=dist.get_global_rank(group, 0) if group is not None else 0, group=group)
        idb = t.cpu().numpy().copy()
        self.out_cap = int(out_capacity or (n_local + n_local // 4 + 4096))
        win = int(window_bytes or self.L.ovs_dist_window_bytes(self.out_cap, self.dt, int(with_values),
                                                               ctypes.byref(self.prm), self.world))
        self.comm = ctypes.c_void_p()
        with torch.cuda.device(self.device):
            self._check(self.L.ovs_comm_create(ctypes.byref(self.comm), idb.ctypes.data, self.rank, self.world,
                                               self.device.index, win))
        self._alloc()

    def _check(self, rc):
        if rc != OVS_OK:
            raise OvsError(rc, self.L.ovs_last_error().decode())

    def _stream(self):
        import torch
        return ctypes.c_void_p(torch.cuda.current_stream(self.device).cuda_stream)

    def _alloc(self):
        import torch
        with torch.cuda.device(self.device):
            nb = int(self.L.ovs_dist_workspace_bytes(self.comm, self.n_local, self.dt, int(self.kv),
                                                     ctypes.byref(self.prm), self.out_cap, self._stream()))
            if nb == 0:
                raise OvsError(1, self.L.ovs_last_error().decode() or "invalid distributed arguments")
            self.ws = torch.empty(nb, dtype=torch.uint8, device=self.device)
            self.ws[:16].zero_()
            self.out_k = torch.empty(self.out_cap, dtype=self.dtype, device=self.device)
            self.out_v = torch.empty(self.out_cap, dtype=torch.uint32, device=self.device) if self.kv else None

    def window_bytes(self) -> int:
        return int(self.L.ovs_comm_window_bytes(self.comm))

    def __call__(self, keys, vals=None, report: bool = False) -> DistResult:
        import torch
        assert keys.is_cuda and keys.is_contiguous() and keys.numel() == self.n_local and keys.dtype == self.dtype
        with torch.cuda.device(self.device):
            for _ in range(3):
                rc, res = self._call(keys, vals, report)
                if rc != OVS_ECAPACITY:
                    self._check(rc)
                    return res
                # every rank got OVS_ECAPACITY (decided from the all-gathered counts): grow the
                # output and the (symmetric, collective) window, then call again
                need = int(self._n_out.value)
                self.out_cap = max(self.out_cap, need + need // 8 + 4096)
                win = int(self.L.ovs_dist_window_bytes(self.out_cap, self.dt, int(self.kv), ctypes.byref(self.prm),
                                                       self.world))
                self._check(self.L.ovs_comm_reserve(self.comm, win, self._stream()))
                self._alloc()
            self._check(rc)

    def _call(self, keys, vals, report):
        p = self.p
        rep = None
        kbuf = np.zeros(p - 1, dtype=_NP[self.dt])
        tbuf = np.zeros(p - 1, dtype=np.uint64)
        cbuf = np.zeros(p, dtype=np.uint64)
        if report:
            rep = Report(kbuf.ctypes.data, tbuf.ctypes.data, cbuf.ctypes.data)
        rp = ctypes.byref(rep) if rep is not None else None
        self._n_out = ctypes.c_size_t(0)
        if self.kv:
            assert vals is not None and vals.dtype.itemsize == 4 and vals.numel() == self.n_local
            rc = self.L.ovs_dist_sort_pairs_stable(self.comm, keys.data_ptr(), vals.data_ptr(), self.n_local, self.dt,
                                                   ctypes.byref(self.prm), self.out_k.data_ptr(),
                                                   self.out_v.data_ptr(), self.out_cap, ctypes.byref(self._n_out),
                                                   self.ws.data_ptr(), self.ws.numel(), self._stream(), rp)
        else:
            rc = self.L.ovs_dist_sort_keys(self.comm, keys.data_ptr(), self.n_local, self.dt, ctypes.byref(self.prm),
                                           self.out_k.data_ptr(), self.out_cap, ctypes.byref(self._n_out),
                                           self.ws.data_ptr(), self.ws.numel(), self._stream(), rp)
        if rc != OVS_OK:
            return rc, None
        n = int(self._n_out.value)
        n_before, xbytes, phases, counts = -1, -1, [], None
        if report:
            counts = cbuf
            b0, b1 = owned(self.world, p, self.rank)
            n_before = int(cbuf[:b0].sum())
            phases = list(rep.phase_ms)
            xbytes = int(rep.exchange_bytes)
        res = DistResult(self.out_k[:n], self.out_v[:n] if self.kv else None, counts, n_before, kbuf, tbuf, xbytes,
                         phases, int(rep.kernel_launches) if report else -1)
        return rc, res

    def close(self):
        if getattr(self, "comm", None) and self.comm.value:
            self.L.ovs_comm_destroy(self.comm)
            self.comm = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def dist_sort_virtual(shards, vals=None, p: int = 1024, s: int = 64, seed: int = 1, win_items=None,
                      method: str = "ros", padded: bool = False):
    """G ranks emulated on ONE GPU by one library call (ovs_dist_sort_virtual: the same phases
    and kernels, the fused scatter storing into the other emulated ranks' windows, phases run
    rank after rank so no kernel waits on another).  Returns (concatenated output, values,
    global counts, splitter keys, splitter tags, per-rank output sizes)."""
    import torch
    L = _ensure_sigs()
    world = len(shards)
    kv = vals is not None
    dev = shards[0].device
    dt = _dtcode(shards[0].dtype)
    prm = params(method, p, s, seed, padded)
    n_local = np.array([int(x.numel()) for x in shards], dtype=np.uint64)
    n_global = int(n_local.sum())
    cap = int(win_items or (n_global // world + n_global // (2 * world) + 8192))
    for _ in range(3):
        res = _virtual_call(L, shards, vals, dt, prm, n_local, cap, world, kv, dev, p)
        if isinstance(res, tuple):
            return res
        cap = max(cap, res + res // 8 + 4096)  # OVS_ECAPACITY: the largest requirement
    raise OvsError(OVS_ECAPACITY, "dist_sort_virtual: capacity")


def _virtual_call(L, shards, vals, dt, prm, n_local, cap, world, kv, dev, p):
    import torch
    out_cap = np.full(world, cap, dtype=np.uint64)
    win_bytes = int(L.ovs_dist_window_bytes(cap, dt, int(kv), ctypes.byref(prm), world))
    wsb = int(L.ovs_dist_virtual_workspace_bytes(world, n_local.ctypes.data, dt, int(kv), ctypes.byref(prm),
                                                 out_cap.ctypes.data, win_bytes))
    if wsb == 0:
        raise OvsError(1, "invalid virtual distributed arguments")
    wins = [torch.empty(win_bytes, dtype=torch.uint8, device=dev) for _ in range(world)]
    wss = [torch.zeros(wsb, dtype=torch.uint8, device=dev) for _ in range(world)]
    outs = [torch.empty(cap, dtype=shards[0].dtype, device=dev) for _ in range(world)]
    vouts = [torch.empty(cap, dtype=torch.uint32, device=dev) for _ in range(world)] if kv else None

    def arr(ts):
        return (ctypes.c_void_p * world)(*[t.data_ptr() for t in ts])

    n_out = np.zeros(world, dtype=np.uint64)
    rank_ms = np.zeros(world, dtype=np.float32)
    ws_bytes = np.full(world, wsb, dtype=np.uint64)
    counts = np.zeros(p, dtype=np.uint64)
    sk = np.zeros(p - 1, dtype=_NP[dt])
    st = np.zeros(p - 1, dtype=np.uint64)
    rc = L.ovs_dist_sort_virtual(world, arr(shards), arr(vals) if kv else None, n_local.ctypes.data, dt,
                                 ctypes.byref(prm), arr(outs), arr(vouts) if kv else None, out_cap.ctypes.data,
                                 n_out.ctypes.data, arr(wss), ws_bytes.ctypes.data, arr(wins), win_bytes,
                                 ctypes.c_void_p(torch.cuda.current_stream(dev).cuda_stream), counts.ctypes.data,
                                 sk.ctypes.data, st.ctypes.data, rank_ms.ctypes.data)
    if rc == OVS_ECAPACITY:
        return int(n_out.max())
    if rc != OVS_OK:
        raise OvsError(rc, L.ovs_last_error().decode())
    torch.cuda.synchronize(dev)
    out = torch.cat([outs[r][:int(n_out[r])] for r in range(world)])
    vout = torch.cat([vouts[r][:int(n_out[r])] for r in range(world)]) if kv else None
    dist_sort_virtual.last_rank_ms = rank_ms.tolist()  # each emulated rank's device time
    return out, vout, counts, sk, st, n_out
