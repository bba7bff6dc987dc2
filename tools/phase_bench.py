"""Phase timing of the metric sort for one or more library variants (experiments only):
python tools/phase_bench.py [lib.so ...]   (default: the in-tree libovs.so)"""
import statistics, sys
sys.path.insert(0, ".")
import numpy as np
import torch
import ovs_inputs
import paper_1608_08648_b200 as ovs

libs = sys.argv[1:] or [None]
n, p, s = 1 << 27, 4096, 64
x = torch.from_numpy(ovs_inputs.keys("u32", n, seed=51)).cuda()
ref = None
for path in libs:
    if path:
        ovs.LIB_PATH = path
        ovs._lib = None
    srt = ovs.Sorter(n, torch.uint32, False, "ros", p, s, 1)
    w = x.clone()
    srt(w)
    torch.cuda.synchronize()
    h = w[:: 1 << 12].cpu().numpy()
    ok = bool(np.all(np.diff(w.cpu().numpy().astype(np.int64)) >= 0))
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(6)] for _ in range(10)]
    for k in range(13):
        w.copy_(x)
        if k >= 3:
            ovs.set_phase_events(evs[k - 3])
        srt(w)
    ovs.set_phase_events(None)
    torch.cuda.synchronize()
    ph = [statistics.median(e[i].elapsed_time(e[i + 1]) for e in evs) for i in range(5)]
    tot = statistics.median(e[0].elapsed_time(e[5]) for e in evs)
    print(f"{path or 'libovs.so'}: sorted={ok} total {tot:.3f} ms ({n / tot / 1e6:.1f} Gkeys/s)  "
          + "  ".join(f"{nm} {v:.3f}" for nm, v in zip(ovs.PHASES, ph)), flush=True)
    del srt

# bucket-sorter phase profile (libraries built with -DOVS_BS_PROF)
import ctypes
for path in libs:
    L = ctypes.CDLL(path or ovs.LIB_PATH)
    if not hasattr(L, "ovs_debug_bsprof_u32_k"):
        continue
    arr = (ctypes.c_ulonglong * 16)()
    for dt in ("u32_k", "u32_v", "i32_k", "i32_v", "f64_k", "f64_v"):
        if hasattr(L, "ovs_debug_bsprof_" + dt):
            getattr(L, "ovs_debug_bsprof_" + dt)(arr, 1)
    srt = ovs.Sorter(n, torch.uint32, False, "ros", p, s, 1) if False else None
    names = ["resplit-push", "loose", "setup", "hist", "scan", "scatter", "net8", "net16+warp", "huge", "write", "rs-sample", "rs-count", "rs-scatter"]
    tot = arr[15]
    print("bucket sorter cycles (sum over CTAs, thread 0), share of kernel:",
          "  ".join(f"{nm} {arr[i] / tot * 100:.1f}%" for i, nm in enumerate(names)),
          f" other {(tot - sum(arr[:13])) / tot * 100:.1f}%")


# fused sample-sort phase cycles (libraries built with -DOVS_SF_PROF)
for path in libs:
    L = ctypes.CDLL(path or ovs.LIB_PATH)
    if hasattr(L, "ovs_debug_sfprof"):
        a = (ctypes.c_ulonglong * 8)()
        L.ovs_debug_sfprof(a)
        print("k_sel_fused cycles (sum over CTAs and sorts, thread 0):", [a[i] for i in range(7)])
