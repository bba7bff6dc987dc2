"""Multi-GPU path emulated on one B200 (ovs_dist_sort_virtual): G ranks x 2^27 uint32 keys (C5 shards),
p = 4096, s = 64.  The emulation runs every phase rank after rank, so the device time of one call divided
by G is the per-rank work (its fused scatter stores into local memory instead of NVLink); compare it with
the single-GPU sort of 2^27 keys.  Outputs are checked sorted.  One JSON line per G.
python tools/dist_virtual_bench.py [G ...]"""
import json
import statistics
import sys

sys.path.insert(0, ".")
import numpy as np
import torch

import ovs_inputs
import paper_1608_08648_b200 as ovs
from paper_1608_08648_b200.dist import dist_sort_virtual

Gs = [int(a) for a in sys.argv[1:]] or [1, 2, 4, 8]
n, p, s = 1 << 27, 4096, 64
x1 = torch.from_numpy(ovs_inputs.keys("u32", n, seed=51)).cuda()
srt = ovs.Sorter(n, torch.uint32, False, "ros", p, s, 1)
w = x1.clone()
ms = []
for _ in range(4):
    w.copy_(x1)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); srt(w); b.record(); b.synchronize()
    ms.append(a.elapsed_time(b))
single = statistics.median(ms[1:])
print(json.dumps({"G": 1, "mode": "single-GPU sort", "ms": round(single, 4)}), flush=True)
del srt, w
for G in Gs:
    xs = [torch.from_numpy(ovs_inputs.keys("u32", n, seed=51, start=r * n)).cuda() for r in range(G)]
    t, rk = [], []
    for it in range(3):
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        out, _, counts, _, _, n_out = dist_sort_virtual(xs, None, p, s, 1)
        b.record()
        b.synchronize()
        t.append(a.elapsed_time(b))
        rk.append(max(dist_sort_virtual.last_rank_ms))
        if it == 0:
            h = out[:: 1 << 10].cpu().numpy()
            ok = bool(np.all(h[1:] >= h[:-1])) and int(counts.sum()) == G * n
        del out
    tm = statistics.median(t[1:])
    rmax = statistics.median(rk[1:])
    print(json.dumps({"G": G, "mode": "emulated ranks (ovs_dist_sort_virtual)", "call_ms_all_ranks": round(tm, 3),
                      "max_rank_device_ms": round(rmax, 4), "single_gpu_ms": round(single, 4),
                      "rank_over_single": round(rmax / single, 3), "sorted_sampled": ok,
                      "max_owned_items_over_n": round(float(max(n_out)) / n, 4),
                      "note": "max_rank_device_ms: one rank's kernels (sample, select+count, fused scatter, local sort) "
                              "timed with events; the call time adds the emulation's allocations and host plan; "
                              "the scatter's stores are local instead of NVLink"}),
          flush=True)
    del xs
    torch.cuda.empty_cache()
