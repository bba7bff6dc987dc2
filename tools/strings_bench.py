"""f3 measurement: ROS on 32-byte random strings (the paper's workload) over the
paper's n grid (1.024M .. 32.768M keys ~ 2^20 .. 2^25) and p in {4, 16, 64, 256} with the paper's
default s = ceil(lg^2 n) (reading Q13).  Device time of one sort (median of 5);
algorithmic bytes = 32 B read (classify + histogram) + 64 B (scatter) + 64 B (bucket sort) per key.
One JSON line per run.   python tools/strings_bench.py [max lg n]"""
import json
import math
import statistics
import sys

sys.path.insert(0, ".")
import numpy as np
import torch

import ovs_inputs
import paper_1608_08648_b200 as ovs

top = int(sys.argv[1]) if len(sys.argv) > 1 else 25
for lg in range(20, top + 1):
    n = 1 << lg
    x = torch.from_numpy(np.frombuffer(ovs_inputs.keys("s32", n, seed=71).tobytes(), dtype=np.uint8).copy()).cuda()
    w = x.clone()
    for p in (4, 16, 64, 256):
        s = math.ceil(lg * lg)
        srt = ovs.Sorter(n, "s32", False, "ros", p, s, 1)
        w.copy_(x)
        rep = srt(w, report=True)
        h = w.view(-1, 32)[:: max(1, n // 4096)].cpu().numpy()
        ok = rep.device_status == 0 and all(bytes(h[i]) <= bytes(h[i + 1]) for i in range(len(h) - 1))
        ms = []
        for _ in range(6):
            w.copy_(x)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            srt(w)
            b.record()
            b.synchronize()
            ms.append(a.elapsed_time(b))
        t = statistics.median(ms[1:])
        print(json.dumps({"workload": "s32 uniform random bytes", "n": n, "p": p, "s": s, "ms": round(t, 4),
                          "Mkeys_per_s": round(n / t / 1e3, 1), "algorithmic_GBps": round(160 * n / t / 1e6, 1),
                          "max_bucket_over_n_p": round(float(rep.counts.max()) * p / n, 4), "sorted_sampled": ok}),
              flush=True)
        del srt
    del x, w
    torch.cuda.empty_cache()
