"""The C-ABI library loads and exports every symbol include/ovs.h declares; host-side argument
validation (no kernel launches: these run without a GPU)."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_functions():
    src = open(os.path.join(ROOT, "include", "ovs.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(ovs_[a-z_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    import paper_1608_08648_b200 as ovs
    L = ovs.lib()
    names = header_functions()
    assert {"ovs_sort_keys", "ovs_sort_pairs_stable", "ovs_workspace_bytes", "ovs_last_error", "ovs_device_status",
            "ovs_comm_create", "ovs_comm_destroy", "ovs_dist_sort_keys", "ovs_dist_sort_pairs_stable"} <= set(names)
    for nm in names:
        assert hasattr(L, nm), nm
    assert ovs.version().startswith("ovs")


def test_library_is_sm100a():
    out = os.popen(f"cuobjdump --list-elf {os.path.join(ROOT, 'paper_1608_08648_b200', 'libovs.so')}").read()
    assert "sm_100a" in out


def _prm(ovs, method="ros", p=64, s=32):
    return ovs.params(method, p, s, 1)


def test_workspace_bytes_validation():
    import paper_1608_08648_b200 as ovs
    P = lambda **kw: _prm(ovs, **kw)
    assert ovs.workspace_bytes(1 << 20, ovs.OVS_U32, False, P()) > 4 * (1 << 20)
    assert ovs.workspace_bytes(1 << 20, ovs.OVS_F64, True, P()) > 16 * (1 << 20)
    assert ovs.workspace_bytes(100, ovs.OVS_U32, False, P(p=11, s=10)) == 0     # ps-1 > n
    assert ovs.workspace_bytes(100, ovs.OVS_U32, False, P(p=0)) == 0            # p == 0
    assert ovs.workspace_bytes(100, 7, False, P()) == 0                          # dtype
    assert ovs.workspace_bytes(100, ovs.OVS_U32, False, P(method="dro", p=8, s=2)) == 0  # rp > n/p
    assert ovs.workspace_bytes(0, ovs.OVS_U32, False, P()) == 0                  # nothing to do


def test_sort_rejects_bad_arguments_before_any_launch():
    import paper_1608_08648_b200 as ovs
    L = ovs.lib()
    prm = _prm(ovs, p=11, s=10)
    rc = L.ovs_sort_keys(None, 100, ovs.OVS_U32, ctypes.byref(prm), None, 0, None, None)
    assert rc == ovs.OVS_ESAMPLE
    prm = _prm(ovs, p=0)
    assert L.ovs_sort_keys(None, 100, ovs.OVS_U32, ctypes.byref(prm), None, 0, None, None) == ovs.OVS_EINVAL
    prm = _prm(ovs)
    assert L.ovs_sort_keys(None, 100, 9, ctypes.byref(prm), None, 0, None, None) == ovs.OVS_EDTYPE
    prm = _prm(ovs, p=4, s=8)
    assert L.ovs_sort_keys(None, 1000, ovs.OVS_U32, ctypes.byref(prm), None, 0, None, None) == ovs.OVS_EINVAL  # NULL
    assert L.ovs_sort_keys(None, 0, ovs.OVS_U32, ctypes.byref(prm), None, 0, None, None) == ovs.OVS_OK
    assert L.ovs_last_error() is not None


def test_binding_raises_without_cuda():
    import torch
    if torch.cuda.is_available():
        pytest.skip("has a GPU")
    import paper_1608_08648_b200 as ovs
    with pytest.raises(Exception):
        ovs.Sorter(1000, torch.uint32, False, "ros", 4, 8, 1)


def test_auto_params():
    """ovs_auto_params (host only): buckets of n/p keys fit the on-chip capacity with margin, p within
    the one-level limits, the sample-size preconditions of PAPER.md:566 (ps-1 <= n) and of the DRO
    regular sample (r*p <= n/p) hold."""
    import paper_1608_08648_b200 as ovs
    import torch
    for n in (1000, 1 << 20, 1 << 24, 1 << 27, 3_000_017):
        for dt in (torch.uint32, torch.float64):
            for kv in (False, True):
                pr = ovs.auto_params(n, dt, kv, "ros")
                assert pr.method == 0 and pr.p >= 1 and pr.p & (pr.p - 1) == 0
                if pr.p > 1:
                    assert pr.p * pr.s - 1 <= n and pr.s >= 1
                    assert ovs.workspace_bytes(n, ovs._dtype_code(dt), kv, pr) > 0
                pd = ovs.auto_params(n, dt, kv, "dro")
                if pd.p > 1:
                    assert pd.s >= 1 and pd.s * pd.p <= n // pd.p
    small = ovs.auto_params(1000, torch.uint32)
    assert small.p == 1
    big = ovs.auto_params(1 << 27, torch.uint32)
    assert big.p == 4096 and big.s == 64          # the metric's configuration
    assert ovs.auto_params(1 << 27, torch.float64).p < 1 << 27


def test_dist_plan_validation():
    """ovs_dist_plan (host only): p must be a multiple of world, rank in range."""
    import numpy as np
    from paper_1608_08648_b200.dist import exchange_plan
    C = np.ones((2, 6), dtype=np.uint32)
    dst, recv = exchange_plan(C, 2, 6, 1)
    assert dst.tolist() == [1, 3, 5, 1, 3, 5] and recv.tolist() == [6, 6]
    with pytest.raises(Exception):
        exchange_plan(np.ones((2, 5), dtype=np.uint32), 2, 5, 0)


def test_workspace_bytes_new_dtypes_and_flags():
    """Round-2 surface (host-only checks): 32-byte strings (OVS_S32) are ROS keys-only; the DRO merge
    flag (OVS_DRO_MERGE) is accepted for DRO; unknown flags are rejected; every ps - 1 <= n is valid
    (samples up to the whole input)."""
    import paper_1608_08648_b200 as ovs
    P = lambda **kw: _prm(ovs, **kw)
    assert ovs.workspace_bytes(1 << 20, ovs.OVS_S32, False, P(p=256, s=32)) > 32 * (1 << 20)
    assert ovs.workspace_bytes(1 << 20, ovs.OVS_S32, True, P(p=256, s=32)) == 0          # values
    assert ovs.workspace_bytes(1 << 20, ovs.OVS_S32, False, P(method="dro", p=16, s=2)) == 0  # DRO
    m = ovs.params("dro", 16, 2, 1, merge=True)
    assert m.flags == ovs.OVS_DRO_MERGE
    assert ovs.workspace_bytes(1 << 20, ovs.OVS_U32, False, m) > 0
    bad = ovs.params("dro", 16, 2, 1)
    bad.flags = 8
    assert ovs.workspace_bytes(1 << 20, ovs.OVS_U32, False, bad) == 0
    assert ovs.workspace_bytes(1 << 20, ovs.OVS_U32, False, P(p=64, s=(1 << 20) // 64)) > 0  # ps - 1 = n - 1
    assert ovs.workspace_bytes(1 << 20, ovs.OVS_U32, False, P(p=1, s=1)) > 0
    assert ovs.workspace_bytes((1 << 32) - 20, ovs.OVS_U32, False, P()) == 0            # n + 32 >= 2^32


def test_device_status_rejects_null():
    import paper_1608_08648_b200 as ovs
    L = ovs.lib()
    st = ctypes.c_uint32(7)
    assert L.ovs_device_status(None, None, ctypes.byref(st), 0) == ovs.OVS_EINVAL


def test_host_pipe_rejects_bad_arguments_before_any_cuda_call():
    """ovs_host_pipe_* (host-buffer entry): argument checks run before the first CUDA call."""
    import paper_1608_08648_b200 as ovs
    L = ovs.lib()
    prm = _prm(ovs)
    h = ctypes.c_void_p()
    bufs = (ctypes.c_void_p * 2)(0x1000, 0x2000)  # never dereferenced: every call below fails validation
    ws = ctypes.c_void_p(0x3000)
    need = ovs.workspace_bytes(1 << 16, ovs.OVS_U32, False, prm)
    C = L.ovs_host_pipe_create
    assert C(None, 1 << 16, ovs.OVS_U32, ctypes.byref(prm), bufs, 2, ws, need) == ovs.OVS_EINVAL
    assert C(ctypes.byref(h), 0, ovs.OVS_U32, ctypes.byref(prm), bufs, 2, ws, need) == ovs.OVS_EINVAL
    assert C(ctypes.byref(h), 1 << 16, ovs.OVS_U32, ctypes.byref(prm), bufs, 0, ws, need) == ovs.OVS_EINVAL
    assert C(ctypes.byref(h), 1 << 16, ovs.OVS_U32, ctypes.byref(prm), bufs, 17, ws, need) == ovs.OVS_EINVAL
    assert C(ctypes.byref(h), 1 << 16, 9, ctypes.byref(prm), bufs, 2, ws, need) == ovs.OVS_EDTYPE
    assert C(ctypes.byref(h), 1 << 16, ovs.OVS_U32, ctypes.byref(prm), bufs, 2, ws, need - 1) == ovs.OVS_EWORKSPACE
    assert L.ovs_last_error().decode() == "workspace too small"
    hole = (ctypes.c_void_p * 2)(0x1000, None)
    assert C(ctypes.byref(h), 1 << 16, ovs.OVS_U32, ctypes.byref(prm), hole, 2, ws, need) == ovs.OVS_EINVAL
    bad = _prm(ovs, p=0)
    assert C(ctypes.byref(h), 1 << 16, ovs.OVS_U32, ctypes.byref(bad), bufs, 2, ws, need) == ovs.OVS_EINVAL
    assert not h.value
    assert L.ovs_host_pipe_submit(None, None, None) == ovs.OVS_EINVAL
    assert L.ovs_host_pipe_wait(None, None) == ovs.OVS_EINVAL
    assert L.ovs_host_pipe_destroy(None) == ovs.OVS_OK
