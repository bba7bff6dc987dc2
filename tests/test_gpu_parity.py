"""Parity of the CUDA path (called through the C ABI) with the CPU oracle.

Bit-exact comparison: sorted output, values of stable key-value sorts,
the p-1 splitters (key AND tag) and the p bucket counts, element by element, on seeded
inputs from ovs_inputs.  Sizes span several tiles, sub-tiles and buckets with ragged tails;
the full-size BASELINE.json configurations run in the launch configuration bench.py times.
"""
import numpy as np
import pytest
import torch

import ovs_inputs

pytestmark = pytest.mark.gpu

TORCH = {np.dtype(np.uint32): torch.uint32, np.dtype(np.int32): torch.int32, np.dtype(np.float64): torch.float64}


@pytest.fixture(scope="module")
def ovs():
    import paper_1608_08648_b200 as m
    assert torch.cuda.is_available()
    m.lib()
    return m


def gpu_sort(ovs, x, method, p, s, seed, vals=None, stream=None):
    xt = torch.from_numpy(x).cuda()
    if vals is not None:
        vt = torch.from_numpy(vals).cuda()
        srt = ovs.Sorter(len(x), xt.dtype, True, method, p, s, seed)
        rep = srt(xt, vt, stream=stream, report=True)
        torch.cuda.synchronize()
        return xt.cpu().numpy(), vt.cpu().numpy(), rep
    srt = ovs.Sorter(len(x), xt.dtype, False, method, p, s, seed)
    rep = srt(xt, stream=stream, report=True)
    torch.cuda.synchronize()
    return xt.cpu().numpy(), None, rep


def check(ref, out, vout, rep, p):
    assert rep.device_status == 0
    np.testing.assert_array_equal(out, ref.keys)
    if vout is not None:
        np.testing.assert_array_equal(vout, ref.vals)
    np.testing.assert_array_equal(rep.counts, ref.counts)
    if p > 1:
        np.testing.assert_array_equal(rep.splitter_keys, ref.split_keys)
        np.testing.assert_array_equal(rep.splitter_tags, ref.split_tags)


def ros_case(ovs, orc, dist, n, p, s, seed=1, kv=False, dseed=3):
    x = ovs_inputs.keys(dist, n, seed=dseed)
    v = ovs_inputs.index_values(n) if kv else None
    ref = orc.ros_sort(x, p, s, seed, vals=v)
    out, vout, rep = gpu_sort(ovs, x, "ros", p, s, seed, v)
    check(ref, out, vout, rep, p)
    return rep


def test_c1_full(ovs, orc):
    """BASELINE configs[0]: n=2^20 u32 uniform [0,2^31) seed 1, ROS p=64 s=32."""
    c = ovs_inputs.CONFIGS["C1"]
    ros_case(ovs, orc, "u32_u31", c["n"], c["p"], c["s"], c["seed"], dseed=1)


EDGE = [
    ("u32_u31", 1, 1, 1), ("u32_u31", 2, 1, 1), ("u32_u31", 2, 2, 1), ("u32_u31", 7, 4, 2), ("u32_u31", 1000, 4, 8),
    ("u32", 4097, 64, 64), ("u32_const", 100_000, 64, 32), ("u32_few4", 300_001, 16, 8), ("u32_few4", 70_000, 256, 16),
    ("i32_gauss", 100_003, 16, 16), ("i32_sorted", 500_000, 128, 32), ("i32_reverse", 500_000, 128, 32),
    ("i32_few", 1_000_003, 1000, 16), ("f64_normal", 200_000, 64, 32), ("f64_uniform", 1_000_003, 7, 64),
    ("u32_u31", 100_000, 1, 1), ("f64_normal", 300_000, 1, 1), ("u32", 3_000_017, 4096, 64), ("u32_u31", 65_536, 2, 1),
    ("u32", 2_000_000, 2, 1_000_000),
    # refinement of oversized contract buckets with s not a multiple of the refinement factor
    ("u32", 1_500_000, 8, 37), ("f64_uniform", 2_000_000, 16, 51), ("i32_few", 3_000_000, 32, 129),
]


@pytest.mark.parametrize("dist,n,p,s", EDGE)
def test_ros_keys_edge_matrix(ovs, orc, dist, n, p, s):
    ros_case(ovs, orc, dist, n, p, s, seed=n % 97 + 1)


KV_EDGE = [("u16key", 100_000, 8, 8), ("u32_few4", 200_000, 16, 16), ("f64_uniform", 100_000, 32, 16),
           ("u32_const", 150_000, 64, 8), ("i32_sorted", 300_000, 16, 16), ("f64_normal", 400_001, 1, 1),
           ("u16key", 1_000_000, 512, 32), ("u32_few4", 5, 2, 2)]


@pytest.mark.parametrize("dist,n,p,s", KV_EDGE)
def test_ros_pairs_stable_edge_matrix(ovs, orc, dist, n, p, s):
    rep = ros_case(ovs, orc, dist, n, p, s, seed=5, kv=True)
    assert rep.device_status == 0


@pytest.mark.parametrize("dist,n,p,s", [("u32", 1_000_001, 4096, 16), ("i32_few", 777_777, 2000, 8),
                                        ("f64_uniform", 500_001, 512, 16)])
def test_ros_misaligned_input(ovs, orc, dist, n, p, s):
    """The caller's keys start one element past a 16-byte boundary: the scalar head/tail paths of
    the vectorised histogram, scatter and bucket-sort passes."""
    x = ovs_inputs.keys(dist, n, seed=9)
    ref = orc.ros_sort(x, p, s, 2)
    buf = torch.empty(n + 1, dtype=TORCH[x.dtype], device="cuda")
    xt = buf[1:]
    xt.copy_(torch.from_numpy(x))
    srt = ovs.Sorter(n, xt.dtype, False, "ros", p, s, 2)
    rep = srt(xt, report=True)
    torch.cuda.synchronize()
    check(ref, xt.cpu().numpy(), None, rep, p)


@pytest.mark.parametrize("dist,n,p,s", [("u32", 2_000_003, 8192, 4), ("u32_few4", 1_500_000, 6000, 4),
                                        ("i32_gauss", 3_000_000, 5000, 8)])
def test_ros_large_p(ovs, orc, dist, n, p, s):
    """p beyond the write-combining scatter's shared-memory limit: the generic staged scatter
    with a classifier table of fewer than one entry per splitter (multi-splitter entries)."""
    ros_case(ovs, orc, dist, n, p, s, seed=4)


def test_exhaustive_sample_closed_form(ovs, orc):
    """ps-1 = n: splitter q is the element of rank (q+1)s; counts = [s,..,s,s-1]."""
    n, p, s = 4095, 64, 64
    x = ovs_inputs.keys("u32_few4", n, seed=9)
    out, _, rep = gpu_sort(ovs, x, "ros", p, s, 2)
    assert rep.counts.tolist() == [s] * (p - 1) + [s - 1]
    np.testing.assert_array_equal(out, np.sort(x))


def test_determinism_and_streams(ovs):
    x = ovs_inputs.keys("u32", 1 << 22, seed=4)
    st = torch.cuda.Stream()
    a = gpu_sort(ovs, x, "ros", 512, 32, 7, stream=st)
    b = gpu_sort(ovs, x, "ros", 512, 32, 7)
    np.testing.assert_array_equal(a[0], b[0])
    np.testing.assert_array_equal(a[2].counts, b[2].counts)
    np.testing.assert_array_equal(a[2].splitter_tags, b[2].splitter_tags)


@pytest.mark.parametrize("nbuf", [1, 2, 3])
def test_host_pipeline(ovs, orc, nbuf):
    """ovs.HostPipeline = ovs_host_pipe_* of the C ABI (the e2e path bench.py times): seven different host arrays streamed through
    nbuf rotating device buffers (3 is the default) and three streams; every host result equals the
    oracle's output for its input (no step reads another step's buffer)."""
    n, p, s, seed = (1 << 20) + 77, 64, 32, 3
    srt = ovs.Sorter(n, torch.uint32, False, "ros", p, s, seed)
    pipe = ovs.HostPipeline(srt, torch.uint32, nbuf)
    xs = [ovs_inputs.keys(d, n, seed=10 + i)
          for i, d in enumerate(["u32", "u32_u31", "u32_few4", "u32", "u32_const", "u32_u31", "u32"])]
    hin = [torch.from_numpy(x).pin_memory() for x in xs]
    hout = [torch.empty_like(h).pin_memory() for h in hin]
    for a, b in zip(hin, hout):
        pipe.submit(a, b)
    assert pipe.wait() > 0.0
    assert pipe.wait() == 0.0  # nothing submitted since
    for x, h in zip(xs, hout):
        np.testing.assert_array_equal(h.numpy(), orc.ros_sort(x, p, s, seed).keys)
    pipe.submit(hin[1], hin[1])  # in place in host memory, after a wait
    pipe.wait()
    np.testing.assert_array_equal(hin[1].numpy(), orc.ros_sort(xs[1], p, s, seed).keys)
    pipe.close()


def test_host_pipeline_f64_dro(ovs, orc):
    """The host pipe with 8-byte keys and DRO (Algorithm 1) parameters: three host arrays through two
    device buffers, each result equal to the oracle's DRO output."""
    n, p, r = 64 * 4099, 64, 12
    srt = ovs.Sorter(n, torch.float64, False, "dro", p, r, 1)
    pipe = ovs.HostPipeline(srt, torch.float64, 2)
    xs = [ovs_inputs.keys(d, n, seed=40 + i) for i, d in enumerate(["f64_uniform", "f64_normal", "f64_uniform"])]
    hin = [torch.from_numpy(x).pin_memory() for x in xs]
    hout = [torch.empty_like(h).pin_memory() for h in hin]
    for a, b in zip(hin, hout):
        pipe.submit(a, b)
    pipe.wait()
    for x, h in zip(xs, hout):
        np.testing.assert_array_equal(h.numpy(), orc.dro_sort(x, p, r).keys)
    pipe.close()


def test_error_codes(ovs):
    x = torch.zeros(100, dtype=torch.uint32, device="cuda")
    with pytest.raises(ovs.OvsError) as e:
        ovs.Sorter(100, torch.uint32, False, "ros", 11, 10, 1)
    assert e.value.code in (ovs.OVS_EINVAL, ovs.OVS_ESAMPLE)
    import ctypes
    prm = ovs.params("ros", 4, 8, 1)
    ws = torch.empty(16, dtype=torch.uint8, device="cuda")
    rc = ovs.lib().ovs_sort_keys(x.data_ptr(), 100, ovs.OVS_U32, ctypes.byref(prm), ws.data_ptr(), 16, None, None)
    assert rc == ovs.OVS_EWORKSPACE


def test_c5_metric_full(ovs, orc):
    """The bench workload (metric): 2^27 u32 uniform [0,2^32) data seed 51, ROS p=4096 s=64,
    same launch configuration as bench.py; full element-wise comparison with the oracle."""
    c = ovs_inputs.CONFIGS["C5"]
    ros_case(ovs, orc, "u32", c["n"], c["p"], c["s"], c["seed"], dseed=51)


@pytest.mark.parametrize("dist,dseed", [("f64_uniform", 31), ("f64_normal", 32)])
def test_c3_full(ovs, orc, dist, dseed):
    """BASELINE configs[2]: 2^27 f64, ROS p=1024 s=64 (uniform [0,1) and N(0,1))."""
    c = ovs_inputs.CONFIGS["C3"]
    ros_case(ovs, orc, dist, c["n"], c["p"], c["s"], c["seed"], dseed=dseed)


# ---------------------------------------------------------------- DRO (Algorithm 1, SqDet)
def dro_case(ovs, orc, x, p, r, kv=False, padded=False, merge=False):
    n = len(x)
    v = ovs_inputs.index_values(n) if kv else None
    ref = orc.dro_sort(x, p, r, vals=v, padded=padded)
    xt = torch.from_numpy(x).cuda()
    if kv:
        vt = torch.from_numpy(v).cuda()
        rep = ovs.Sorter(n, xt.dtype, True, "dro", p, r, 0, padded, merge=merge)(xt, vt, report=True)
    else:
        vt = None
        rep = ovs.Sorter(n, xt.dtype, False, "dro", p, r, 0, padded, merge=merge)(xt, report=True)
    torch.cuda.synchronize()
    check(ref, xt.cpu().numpy(), None if vt is None else vt.cpu().numpy(), rep, p)
    # Lemma 1 on the GPU's own bucket counts
    assert int(rep.counts.max()) <= orc.lemma1_bound(n, p, r)
    return rep


DRO_EDGE = [("u32_u31", 1000, 4, 1), ("u32_u31", 1003, 5, 2), ("i32_gauss", 100_003, 16, 3), ("u32_const", 65_536, 8, 4),
            ("u32_few4", 200_000, 32, 5), ("f64_normal", 300_001, 64, 2), ("i32_few", 1_000_000, 100, 24),
            ("u32", 3_000_000, 256, 8), ("f64_uniform", 50_000, 2, 1), ("u32_u31", 10, 1, 1)]


@pytest.mark.parametrize("dist,n,p,r", DRO_EDGE)
@pytest.mark.parametrize("padded", [False, True])
def test_dro_keys_edge_matrix(ovs, orc, dist, n, p, r, padded):
    dro_case(ovs, orc, ovs_inputs.keys(dist, n, seed=n % 31), p, r, padded=padded)


@pytest.mark.parametrize("dist,n,p,r", [("u16key", 200_000, 16, 3), ("u32_few4", 100_000, 8, 8),
                                         ("f64_normal", 150_000, 32, 2), ("u32_const", 70_000, 4, 2)])
def test_dro_pairs_stable_edge_matrix(ovs, orc, dist, n, p, r):
    dro_case(ovs, orc, ovs_inputs.keys(dist, n, seed=3), p, r, kv=True)


@pytest.mark.parametrize("dist", ["u32", "i32_gauss", "f64_normal"])
@pytest.mark.parametrize("method", ["ros", "dro"])
@pytest.mark.parametrize("kv", [False, True])
def test_empty_input(ovs, orc, dist, method, kv):
    """n = 0: nothing to sort; the oracle's report is p zero counts (and the call must succeed)."""
    x = ovs_inputs.keys(dist, 0, seed=1)
    v = ovs_inputs.index_values(0) if kv else None
    ref = orc.ros_sort(x, 4, 2, 1, vals=v) if method == "ros" else orc.dro_sort(x, 4, 2, vals=v)
    xt = torch.from_numpy(x).cuda()
    srt = ovs.Sorter(0, xt.dtype, kv, method, 4, 2, 1)
    rep = srt(xt, torch.from_numpy(v).cuda(), report=True) if kv else srt(xt, report=True)
    torch.cuda.synchronize()
    assert rep.device_status == 0 and xt.numel() == 0
    np.testing.assert_array_equal(rep.counts, ref.counts)  # p zero counts; no splitters are drawn


@pytest.mark.parametrize("dist,n,p,r,kv", [("u32", 2_000_003, 8, 2, False), ("i32_few", 1_600_000, 4, 3, False),
                                           ("u16key", 600_001, 4, 2, True), ("f64_normal", 900_000, 4, 2, False)])
def test_dro_level1(ovs, orc, dist, n, p, r, kv):
    """Sequences and buckets of n/p keys far over the on-chip capacity: both go through the
    GPU-wide level-1 re-split (segment-aware histogram and scatter) before the bucket sorter."""
    x = ovs_inputs.keys(dist, n, seed=13)
    v = ovs_inputs.index_values(n) if kv else None
    ref = orc.dro_sort(x, p, r, vals=v)
    out, vout, rep = gpu_sort(ovs, x, "dro", p, r, 0, v)
    check(ref, out, vout, rep, p)


@pytest.mark.parametrize("method,dist,n,p,s", [("dro", "u16key", 400_003, 8, 3), ("ros", "u32_few4", 600_000, 16, 8),
                                               ("ros", "f64_normal", 500_000, 8, 8), ("dro", "i32_gauss", 700_000, 4, 5)])
def test_pairs_windows(ovs, orc, method, dist, n, p, s):
    """Key-value buckets of 1.1-4x the on-chip capacity (no refinement possible with these s):
    the windowed bucket sorter (k_bucket_sort<..., WIN>) with values and indices."""
    x = ovs_inputs.keys(dist, n, seed=17)
    v = ovs_inputs.index_values(n)
    ref = orc.ros_sort(x, p, s, 3, vals=v) if method == "ros" else orc.dro_sort(x, p, s, vals=v)
    out, vout, rep = gpu_sort(ovs, x, method, p, s, 3, v)
    check(ref, out, vout, rep, p)


def test_dro_closed_forms(ovs):
    """Sorted input: counts = m_j; reverse: m_{p-1-j}; constant: m_j (tags order equal keys)."""
    n, p, r = 1_000_003, 64, 3
    m = [n // p + (1 if k < n % p else 0) for k in range(p)]
    base = np.sort(ovs_inputs.keys("i32_uniform", n, seed=8))
    for x, want in [(base, m), (base[::-1].copy(), m[::-1]), (np.full(n, 5, np.int32), m)]:
        xt = torch.from_numpy(x).cuda()
        rep = ovs.Sorter(n, xt.dtype, False, "dro", p, r, 0)(xt, report=True)
        assert rep.counts.tolist() == want
        np.testing.assert_array_equal(xt.cpu().numpy(), np.sort(x))


@pytest.mark.parametrize("dist,dseed", [("i32_uniform", 21), ("i32_gauss", 22), ("i32_sorted", 23),
                                        ("i32_reverse", 24), ("i32_few", 25)])
def test_c2_full(ovs, orc, dist, dseed):
    """BASELINE configs[1]: 2^24 i32, DRO p=256, r=log2 n=24 (reading Q7), five distributions."""
    c = ovs_inputs.CONFIGS["C2"]
    dro_case(ovs, orc, ovs_inputs.keys(dist, c["n"], seed=dseed), c["p"], c["s"])


def test_c4_full(ovs, orc):
    """BASELINE configs[3]: 2^27 stable key-value pairs (u32 key uniform [0,2^16), value =
    original index), DRO p=512, r=ceil(log2 n)=27; checks stability element by element."""
    c = ovs_inputs.CONFIGS["C4"]
    dro_case(ovs, orc, ovs_inputs.keys("u16key", c["n"], seed=41), c["p"], c["s"], kv=True)


@pytest.mark.parametrize("force,dist,dseed", [("0", None, 41), ("1", "i32_uniform", 21), ("1", "f64_normal", 2)])
def test_dro_sample_merge_and_sort(ovs, orc, monkeypatch, force, dist, dseed):
    """a11 both ways (Algorithm 1 step 2: the p sorted T_k "merged or sorted" into T,
    PAPER.md:359-364): C4 with its sample merged (it is sorted by default, 56.6 MB > L2/4), and
    C2 / an f64 case with their samples sorted (merged by default); same splitters and output."""
    monkeypatch.setenv("OVS_DRO_SAMPLE_SORT", force)
    if dist is None:
        c = ovs_inputs.CONFIGS["C4"]
        dro_case(ovs, orc, ovs_inputs.keys("u16key", c["n"], seed=dseed), c["p"], c["s"], kv=True)
    elif dist == "f64_normal":
        dro_case(ovs, orc, ovs_inputs.keys(dist, 300_001, seed=dseed), 64, 2)
    else:
        c = ovs_inputs.CONFIGS["C2"]
        dro_case(ovs, orc, ovs_inputs.keys(dist, c["n"], seed=dseed), c["p"], c["s"])


# ---------------------------------------------------------------- samples that are a large fraction of n
@pytest.mark.parametrize("dist,n,p,s,kv", [
    ("u32", 1_000_000, 64, 12_000, False),      # ps-1 = 0.77 n: the direct-address sample table
    ("i32_few", 300_000, 16, 18_750, True),     # ps-1 = n - 1
    ("f64_normal", 200_000, 40, 5_000, False),  # ps-1 = n - 1, 64-bit keys
    ("u32_u31", 1_048_575, 64, 16_384, False),  # ps-1 = n exactly
    ("u32", 2_000_000, 1000, 1_000, False),     # ps-1 = n/2 - 1 (hash-set form)
])
def test_ros_large_sample_fraction(ovs, orc, dist, n, p, s, kv):
    """ps-1 up to n is valid (ps >= n/2 allowed, Claim 1's precondition only);
    the GPU takes the same first ps-1 distinct draws as the oracle (reading Q1)."""
    ros_case(ovs, orc, dist, n, p, s, seed=9, kv=kv)


def _closed_form_exhaustive(x, p, s):
    """ps-1 = n: T is the whole input, splitter q is the element of rank (q+1)s in (key, index)
    order and the counts are [s, ..., s, s-1] (closed form)."""
    order = np.argsort(x, kind="stable")
    idx = order[np.arange(1, p) * s - 1]
    return x[idx], idx.astype(np.uint64), np.array([s] * (p - 1) + [s - 1], dtype=np.uint64)


@pytest.mark.slow
def test_ros_sample_equals_input_full_size(ovs):
    """n = 2^27 u32 with ps-1 = n (p = 1539, s = 87211, ps = 2^27 + 1): ~2.6e9 draws through the
    direct-address table; splitters and counts equal the closed form, output sorted."""
    n, p, s = 1 << 27, 1539, 87211
    assert p * s - 1 == n
    x = ovs_inputs.keys("u32", n, seed=51)
    out, _, rep = gpu_sort(ovs, x, "ros", p, s, 5)
    assert rep.device_status == 0
    sk, st, cnt = _closed_form_exhaustive(x, p, s)
    np.testing.assert_array_equal(rep.splitter_keys, sk)
    np.testing.assert_array_equal(rep.splitter_tags, st)
    np.testing.assert_array_equal(rep.counts, cnt)
    np.testing.assert_array_equal(out, np.sort(x))


@pytest.mark.slow
def test_ros_half_sample_full_size(ovs, orc):
    """n = 2^27 u32 with ps-1 = n/2 (p = 4096, s = 16384): ~9.3e7 draws (beyond the round-1
    2^26-draw cap); splitters, counts and output equal the oracle's."""
    n, p, s = 1 << 27, 4096, 16384
    x = ovs_inputs.keys("u32", n, seed=51)
    ref = orc.ros_sort(x, p, s, 5)
    out, _, rep = gpu_sort(ovs, x, "ros", p, s, 5)
    check(ref, out, None, rep, p)


def test_sticky_status_after_graph_replays(ovs):
    """ovs_device_status: the sticky status word after CUDA-graph replays (no report) is 0, and
    the per-phase report events are filled (phase_ms[0..4] and the total)."""
    n = 3_000_017
    x = torch.from_numpy(ovs_inputs.keys("u32", n, seed=3)).cuda()
    w = x.clone()
    srt = ovs.Sorter(n, torch.uint32, False, "ros", 1024, 64, 1)
    replay = srt.graph(w)
    for _ in range(3):
        w.copy_(x)
        replay()
    assert srt.status() == 0
    h = w.cpu().numpy()
    assert bool(np.all(h[1:] >= h[:-1]))
    w.copy_(x)
    rep = srt(w, report=True)
    assert rep.device_status == 0
    assert all(v >= 0 for v in rep.phase_ms[:5]) and rep.phase_ms[7] > 0
    assert abs(sum(rep.phase_ms[:5]) - rep.phase_ms[7]) < 0.05 * rep.phase_ms[7] + 0.01


# ---------------------------------------------------------------- f2: DRO step 5 as a p-way merge
@pytest.mark.parametrize("dist,n,p,r,kv", DRO_MERGE_CASES := [
    ("u32_u31", 1000, 4, 1, False), ("i32_gauss", 100_003, 16, 3, False), ("u32_const", 65_536, 8, 4, True),
    ("u32_few4", 200_000, 32, 5, True), ("f64_normal", 300_001, 64, 2, False), ("f64_uniform", 250_000, 16, 3, True),
    ("i32_few", 1_000_000, 100, 24, False), ("u32", 3_000_000, 256, 8, False),
    # fine buckets over the merge capacity (s small): gather + bucket sorter fallback
    ("u32", 2_000_003, 8, 2, False), ("u16key", 600_001, 4, 2, True), ("i32_few", 1_600_000, 4, 3, False)])
@pytest.mark.parametrize("padded", [False, True])
def test_dro_merge_step5(ovs, orc, dist, n, p, r, kv, padded):
    """OVS_DRO_MERGE: fine split by the regular sample, every fine bucket's p sorted runs merged
    on chip (ties to the lower sequence): output, values (stability), splitters and the
    contract counts (folded from the fine counts) equal the oracle's p-way merge."""
    dro_case(ovs, orc, ovs_inputs.keys(dist, n, seed=n % 29), p, r, kv=kv, padded=padded, merge=True)


@pytest.mark.parametrize("dist,dseed", [("i32_uniform", 21), ("i32_gauss", 22), ("i32_sorted", 23), ("i32_reverse", 24),
                                        ("i32_few", 25)])
def test_c2_full_merge(ovs, orc, dist, dseed):
    c = ovs_inputs.CONFIGS["C2"]
    dro_case(ovs, orc, ovs_inputs.keys(dist, c["n"], seed=dseed), c["p"], c["s"], merge=True)


@pytest.mark.slow
def test_c4_full_merge(ovs, orc):
    c = ovs_inputs.CONFIGS["C4"]
    dro_case(ovs, orc, ovs_inputs.keys("u16key", c["n"], seed=41), c["p"], c["s"], kv=True, merge=True)


@pytest.mark.parametrize("dist,n,p,s", [("u32_r26", 1 << 21, 64, 32), ("u32_r26", 3_000_001, 100, 16),
                                        ("i32_few", 2_000_000, 512, 8), ("u32", 1 << 22, 2048, 64)])
def test_dense_range_buckets(ovs, orc, dist, n, p, s):
    """Dense bucket key ranges with hundreds of duplicate keys per bucket (u32 uniform on [0, 2^26))
    and few-distinct keys: the digit-group bucket sorter against the oracle."""
    ros_case(ovs, orc, dist, n, p, s, seed=4, dseed=8)


@pytest.mark.parametrize("dist,n,p,s", [
    ("u32", 1 << 20, 64, 32),          # ps-1 = 2047: one coarse bucket
    ("u32", 1 << 20, 1025, 2),         # 2049: two
    ("i32_gauss", 1 << 20, 2049, 64),  # 131135: 128 coarse buckets of ~1K records
    ("u32_few4", 1 << 20, 4096, 64),   # 262143 (the metric's sample): 128 buckets of ~2K, 4 key values
    ("u32_const", 1 << 20, 4096, 64),  # every record has the same key word: ordered by index alone
    ("u32", 1 << 21, 4097, 64),        # 262207 > 128 * 2048: the multi-launch sample sort instead
])
def test_fused_sample_sort_bounds(ovs, orc, dist, n, p, s):
    """a3+a4 in one cooperative launch (k_sel_fused) at the edges of its coarse-bucket count
    and past its limit: splitters (key and tag), counts and output against the oracle."""
    ros_case(ovs, orc, dist, n, p, s, seed=6)
