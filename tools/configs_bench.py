"""Device time of one sort for each BASELINE.json configuration (C1-C4; C5 is bench.py):
python tools/configs_bench.py [reps]   -> one JSON line per config (median of reps, after 2 warm-ups)"""
import json, os, statistics, sys
sys.path.insert(0, ".")
import torch
import ovs_inputs
import paper_1608_08648_b200 as ovs

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 5
only = sys.argv[2].split(",") if len(sys.argv) > 2 else None
CASES = [  # name, dist, data seed, n, method, p, s/r, kv, algorithmic bytes per key
    ("C1", "u32_u31", 1, 1 << 20, "ros", 64, 32, False, 20),
    ("C2-uniform", "i32_uniform", 21, 1 << 24, "dro", 256, 24, False, 16),
    ("C2-few", "i32_few", 25, 1 << 24, "dro", 256, 24, False, 16),
    ("C3-uniform", "f64_uniform", 31, 1 << 27, "ros", 1024, 64, False, 40),
    ("C4", "u16key", 41, 1 << 27, "dro", 512, 27, True, 32),
]
for name, dist, dseed, n, method, p, s, kv, bpk in CASES:
    if only and name not in only:
        continue
    x = torch.from_numpy(ovs_inputs.keys(dist, n, seed=dseed)).cuda()
    v = torch.from_numpy(ovs_inputs.index_values(n)).cuda() if kv else None
    merge = os.environ.get("OVS_BENCH_MERGE") == "1" and method == "dro"  # f2: DRO step 5 as a p-way merge
    srt = ovs.Sorter(n, x.dtype, kv, method, p, s, 1, merge=merge)
    wk, wv = x.clone(), (v.clone() if kv else None)
    ms, ph = [], []
    for r in range(reps + 2):
        wk.copy_(x)
        if kv:
            wv.copy_(v)
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(6)]
        ovs.set_phase_events(ev)
        srt(wk, wv) if kv else srt(wk)
        ovs.set_phase_events(None)
        ev[5].synchronize()
        if r >= 2:
            ms.append(ev[0].elapsed_time(ev[5]))
            ph.append([ev[i].elapsed_time(ev[i + 1]) for i in range(5)])
    t = statistics.median(ms)
    phases = {nm: round(statistics.median(q[i] for q in ph), 3) for i, nm in enumerate(ovs.PHASES)}
    print(json.dumps({"config": name + ("+merge" if merge else ""), "n": n, "dtype": str(x.dtype).replace("torch.", ""), "method": method, "p": p,
                      "s_or_r": s, "kv": kv, "ms": round(t, 4), "Gkeys_per_s": round(n / t / 1e6, 2),
                      "algorithmic_GBps": round(n * bpk / t / 1e6, 1), "phases_ms": phases}), flush=True)
    del srt, x, v, wk, wv
    torch.cuda.empty_cache()

import ctypes
L = ovs.lib()
if hasattr(L, "ovs_debug_bsprof_u32_k"):
    arr = (ctypes.c_ulonglong * 16)()
    for dt in ("u32_k", "u32_v", "i32_k", "i32_v", "f64_k", "f64_v"):
        getattr(L, "ovs_debug_bsprof_" + dt)(arr, 1)
    names = ["resplit-push", "loose", "setup", "hist", "scan", "scatter", "net8", "net16+warp", "huge", "write", "rs-sample", "rs-count", "rs-scatter"]
    tot = arr[15] or 1
    print("bucket sorter cycles:", "  ".join(f"{nm} {arr[i] / tot * 100:.1f}%" for i, nm in enumerate(names)),
          f" other {(tot - sum(arr[:13])) / tot * 100:.1f}%")
