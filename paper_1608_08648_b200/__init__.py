"""Thin ctypes binding of libovs.so (include/ovs.h): argument marshalling only.

Every step of the sort runs in the library's sm_100a kernels.  PyTorch is used for device
memory (tensors, the workspace) and streams only.  There is no CPU fallback: if the
extension is missing or no CUDA device is present the calls raise.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("OVS_LIB_PATH") or os.path.join(_HERE, "libovs.so")  # override: A/B experiments

OVS_OK, OVS_EINVAL, OVS_EDTYPE, OVS_ESAMPLE, OVS_EWORKSPACE, OVS_ECUDA, OVS_ECAPACITY, OVS_EINTERNAL = 0, 1, 2, 3, 4, 5, 7, 8
OVS_U32, OVS_I32, OVS_F64, OVS_S32 = 0, 1, 2, 3
OVS_ROS, OVS_DRO = 0, 1
OVS_DRO_PADDED_POSITIONS = 1
OVS_DRO_MERGE = 2
METHODS = {"ros": OVS_ROS, "dro": OVS_DRO}


_NP = {OVS_U32: np.uint32, OVS_I32: np.int32, OVS_F64: np.float64, OVS_S32: np.dtype("V32")}


class Params(ctypes.Structure):
    _fields_ = [("method", ctypes.c_uint32), ("p", ctypes.c_uint32), ("s", ctypes.c_uint32),
                ("flags", ctypes.c_uint32), ("seed", ctypes.c_uint64)]


class Report(ctypes.Structure):
    _fields_ = [("splitter_keys", ctypes.c_void_p), ("splitter_tags", ctypes.c_void_p),
                ("bucket_counts", ctypes.c_void_p), ("phase_ms", ctypes.c_float * 8),
                ("max_bucket", ctypes.c_uint32), ("kernel_launches", ctypes.c_uint32),
                ("device_status", ctypes.c_uint32), ("reserved", ctypes.c_uint32),
                ("exchange_bytes", ctypes.c_uint64)]


class OvsError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"ovs status {code}: {msg}")
        self.code = code


_lib = None


def lib() -> ctypes.CDLL:
    """Load the in-tree libovs.so; raise loudly if it has not been built."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: run `python -c 'import __graft_entry__ as g; g.build()'`")
        L = ctypes.CDLL(LIB_PATH)
        vp, sz, i32 = ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int
        L.ovs_workspace_bytes.restype = sz
        L.ovs_workspace_bytes.argtypes = [sz, i32, i32, ctypes.POINTER(Params)]
        L.ovs_sort_keys.restype = i32
        L.ovs_sort_keys.argtypes = [vp, sz, i32, ctypes.POINTER(Params), vp, sz, vp, ctypes.POINTER(Report)]
        L.ovs_sort_pairs_stable.restype = i32
        L.ovs_sort_pairs_stable.argtypes = [vp, vp, sz, i32, ctypes.POINTER(Params), vp, sz, vp,
                                            ctypes.POINTER(Report)]
        L.ovs_set_phase_events.restype = None
        L.ovs_set_phase_events.argtypes = [ctypes.POINTER(ctypes.c_void_p), ctypes.c_int]
        L.ovs_auto_params.restype = i32
        L.ovs_auto_params.argtypes = [sz, i32, i32, i32, ctypes.POINTER(Params)]
        L.ovs_device_status.restype = i32
        L.ovs_device_status.argtypes = [vp, vp, ctypes.POINTER(ctypes.c_uint32), i32]
        L.ovs_host_pipe_create.restype = i32
        L.ovs_host_pipe_create.argtypes = [ctypes.POINTER(vp), sz, i32, ctypes.POINTER(Params),
                                           ctypes.POINTER(vp), i32, vp, sz]
        L.ovs_host_pipe_submit.restype = i32
        L.ovs_host_pipe_submit.argtypes = [vp, vp, vp]
        L.ovs_host_pipe_wait.restype = i32
        L.ovs_host_pipe_wait.argtypes = [vp, ctypes.POINTER(ctypes.c_float)]
        L.ovs_host_pipe_destroy.restype = i32
        L.ovs_host_pipe_destroy.argtypes = [vp]
        L.ovs_last_error.restype = ctypes.c_char_p
        L.ovs_version.restype = ctypes.c_char_p
        _lib = L
    return _lib


def version() -> str:
    return lib().ovs_version().decode()


PHASES = ("sample", "sample_sort", "classify_hist", "scatter", "bucket_sort")


def set_phase_events(events) -> None:
    """Record torch.cuda.Event objects (enable_timing=True) at the phase boundaries of every
    following sort call on this thread: 0 start, 1 sample drawn, 2 splitters, 3 histogram done,
    4 scatter done, 5 bucket sort done (6 events, PHASES between them).  None / [] disables."""
    events = list(events or [])
    for e in events:
        if e.cuda_event == 0:  # torch creates the event lazily
            e.record()
    arr = (ctypes.c_void_p * max(len(events), 1))(*[e.cuda_event for e in events])
    lib().ovs_set_phase_events(arr, len(events))


def _dtype_code(dt) -> int:
    """torch dtype -> ovs dtype; "s32" = 32-byte string records (a uint8 tensor of 32 n bytes)."""
    import torch
    if dt == "s32":
        return OVS_S32
    m = {torch.uint32: OVS_U32, torch.int32: OVS_I32, torch.float64: OVS_F64}
    if dt not in m:
        raise OvsError(OVS_EDTYPE, f"unsupported dtype {dt}")
    return m[dt]


def params(method: str = "ros", p: int = 64, s: int = 32, seed: int = 1, padded: bool = False,
           merge: bool = False) -> Params:
    flags = (OVS_DRO_PADDED_POSITIONS if padded else 0) | (OVS_DRO_MERGE if merge else 0)
    return Params(METHODS[method], p, s, flags, seed)


def auto_params(n: int, dtype, with_values: bool = False, method: str = "ros") -> Params:
    """ovs_auto_params: p (and s or r) for which the buckets fit on chip in one level."""
    prm = Params()
    rc = lib().ovs_auto_params(n, _dtype_code(dtype), int(with_values), 0 if method == "ros" else 1, ctypes.byref(prm))
    if rc != OVS_OK:
        raise OvsError(rc, "ovs_auto_params")
    return prm


def workspace_bytes(n: int, dtype_code: int, with_values: bool, prm: Params) -> int:
    return int(lib().ovs_workspace_bytes(n, dtype_code, 1 if with_values else 0, ctypes.byref(prm)))


@dataclass
class SortReport:
    splitter_keys: np.ndarray
    splitter_tags: np.ndarray
    counts: np.ndarray
    total_ms: float
    max_bucket: int
    kernel_launches: int
    device_status: int
    phase_ms: list = field(default_factory=list)


class Sorter:
    """Holds a workspace tensor sized for (n, dtype, kv, params) and sorts tensors in place."""

    def __init__(self, n: int, dtype, with_values: bool = False, method: str = "ros", p: int = 64, s: int = 32,
                 seed: int = 1, padded: bool = False, device=None, merge: bool = False):
        import torch
        self.prm = params(method, p, s, seed, padded, merge)
        self.dt = _dtype_code(dtype)
        self.kv = with_values
        self.n = n
        nb = workspace_bytes(n, self.dt, with_values, self.prm)
        if n > 0 and nb == 0:
            self._raise(OVS_EINVAL)
        self.ws = torch.empty(max(nb, 1), dtype=torch.uint8, device=device or "cuda")
        self.ws[:16].zero_()  # the status words (include/ovs.h ovs_device_status): sticky bits start clear
        self.ws_bytes = nb

    def _raise(self, rc):
        raise OvsError(rc, lib().ovs_last_error().decode())

    def __call__(self, keys, vals=None, stream=None, report: bool = False):
        import torch
        assert keys.is_cuda and keys.is_contiguous() and keys.numel() == self.n * (32 if self.dt == OVS_S32 else 1)
        assert keys.device == self.ws.device, "keys and the workspace must be on the same device"
        with torch.cuda.device(keys.device):
            return self._call(keys, vals, stream, report)

    def status(self, stream=None, reset: bool = True) -> int:
        """ovs_device_status: synchronise the stream and return the sticky device-status bits of every
        sort run on this workspace since the last reset (0 = no device-side check failed)."""
        import torch
        with torch.cuda.device(self.ws.device):
            st = ctypes.c_void_p(stream.cuda_stream if stream is not None
                                 else torch.cuda.current_stream(self.ws.device).cuda_stream)
            out = ctypes.c_uint32(0)
            rc = lib().ovs_device_status(self.ws.data_ptr(), st, ctypes.byref(out), 1 if reset else 0)
            if rc not in (OVS_OK, OVS_EINTERNAL):
                self._raise(rc)
            return int(out.value)

    def _call(self, keys, vals, stream, report):
        import torch
        if self.dt == OVS_S32:
            assert keys.dtype == torch.uint8 and keys.numel() == 32 * self.n, "s32: 32 n bytes of uint8"
        st = ctypes.c_void_p(stream.cuda_stream if stream is not None
                             else torch.cuda.current_stream(keys.device).cuda_stream)
        rep = None
        p = self.prm.p
        kbuf = tbuf = cbuf = None
        if report:
            kbuf = np.zeros(max(p - 1, 0), dtype=_NP[self.dt])
            tbuf = np.zeros(max(p - 1, 0), dtype=np.uint64)
            cbuf = np.zeros(p, dtype=np.uint64)
            rep = Report(kbuf.ctypes.data if kbuf.size else None, tbuf.ctypes.data if tbuf.size else None,
                         cbuf.ctypes.data)
        rp = ctypes.byref(rep) if rep is not None else None
        if self.kv:
            assert vals is not None and vals.is_cuda and vals.dtype == torch.uint32 and vals.numel() == self.n
            rc = lib().ovs_sort_pairs_stable(keys.data_ptr(), vals.data_ptr(), self.n, self.dt, ctypes.byref(self.prm),
                                             self.ws.data_ptr(), self.ws_bytes, st, rp)
        else:
            rc = lib().ovs_sort_keys(keys.data_ptr(), self.n, self.dt, ctypes.byref(self.prm), self.ws.data_ptr(),
                                     self.ws_bytes, st, rp)
        if rc != OVS_OK:
            self._raise(rc)
        if report:
            return SortReport(kbuf, tbuf, cbuf, rep.phase_ms[7], rep.max_bucket, rep.kernel_launches,
                              rep.device_status, list(rep.phase_ms))
        return None

    def graph(self, keys, vals=None):
        """Capture this sorter's call on these exact buffers into a CUDA graph (the library only
        enqueues on the stream, so the whole sort is capturable) and return a callable that
        replays it on the current stream: one launch instead of ~20, no per-kernel host work.
        The buffers' contents may change between replays, their addresses may not."""
        import torch
        side = torch.cuda.Stream(device=keys.device)
        side.wait_stream(torch.cuda.current_stream(keys.device))
        with torch.cuda.stream(side):
            self(keys, vals)  # warm-up outside the capture (first-use host setup)
        torch.cuda.current_stream(keys.device).wait_stream(side)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=side):
            self(keys, vals)
        return g.replay


class HostPipeline:
    """ovs_host_pipe_* (include/ovs.h): sorts a stream of pinned host key arrays (n keys each) with one
    Sorter's parameters and workspace.  The library runs step k's host->device copy, the sorts and step
    k-1's device->host copy on its own three streams over nbuf rotating device buffers (allocated here
    as torch tensors; three let a copy-in never wait), so a stream of host sorts is bound by the slower
    PCIe direction instead of the sum of both copies and the sort.  This class only marshals arguments."""

    def __init__(self, sorter: "Sorter", dtype, nbuf: int = 3):
        import torch
        assert not sorter.kv, "keys-only sorter"
        dev = sorter.ws.device
        self.sorter = sorter
        self.bytes = sorter.n * {OVS_F64: 8, OVS_S32: 32}.get(sorter.dt, 4)
        with torch.cuda.device(dev):
            self.buf = [torch.empty(self.bytes, dtype=torch.uint8, device=dev) for _ in range(nbuf)]
            torch.cuda.synchronize(dev)  # the pipe's streams do not wait for torch's
            ptrs = (ctypes.c_void_p * nbuf)(*[b.data_ptr() for b in self.buf])
            self.h = ctypes.c_void_p()
            rc = lib().ovs_host_pipe_create(ctypes.byref(self.h), sorter.n, sorter.dt, ctypes.byref(sorter.prm), ptrs,
                                            nbuf, sorter.ws.data_ptr(), sorter.ws_bytes)
        if rc != OVS_OK:
            sorter._raise(rc)

    def submit(self, host_in, host_out) -> None:
        """Enqueue: host_in -> device, sort, device -> host_out (pinned host tensors of n keys each);
        returns at once.  host_out is valid after wait()."""
        assert host_in.is_pinned() and host_out.is_pinned() and host_in.is_contiguous() and host_out.is_contiguous()
        assert host_in.numel() * host_in.element_size() == self.bytes == host_out.numel() * host_out.element_size()
        rc = lib().ovs_host_pipe_submit(self.h, host_in.data_ptr(), host_out.data_ptr())
        if rc != OVS_OK:
            self.sorter._raise(rc)

    def wait(self) -> float:
        """Block until every submitted result is in host memory; returns the device time (ms) from the
        first copy-in submitted since the previous wait to the last copy-out.  Raises if a device-side
        check of any of those sorts failed."""
        ms = ctypes.c_float(0.0)
        rc = lib().ovs_host_pipe_wait(self.h, ctypes.byref(ms))
        if rc != OVS_OK:
            self.sorter._raise(rc)
        return float(ms.value)

    def close(self) -> None:
        if getattr(self, "h", None):
            lib().ovs_host_pipe_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def sort_keys(keys, method: str = "ros", p: int = 64, s: int = 32, seed: int = 1, padded: bool = False,
              report: bool = True):
    """Sort a CUDA tensor (uint32 / int32 / float64) in place; returns the report."""
    return Sorter(keys.numel(), keys.dtype, False, method, p, s, seed, padded, keys.device)(keys, report=report)


def sort_pairs_stable(keys, vals, method: str = "ros", p: int = 64, s: int = 32, seed: int = 1,
                      padded: bool = False, report: bool = True):
    """Stable key-value sort (uint32 values) in place; returns the report."""
    return Sorter(keys.numel(), keys.dtype, True, method, p, s, seed, padded, keys.device)(keys, vals, report=report)


def sort_strings32(recs, p: int = 64, s: int = 32, seed: int = 1, report: bool = True):
    """Sort 32-byte string records (a CUDA uint8 tensor of 32 n bytes, memcmp order; the paper's
    workload) in place with ROS; returns the report (splitter keys as V32)."""
    n = recs.numel() // 32
    return Sorter(n, "s32", False, "ros", p, s, seed, device=recs.device)(recs, report=report)
