"""Device time of one sort per input distribution (looking for slow distributions; experiments):
python tools/dist_sweep.py [reps]  -> one JSON line per (method, distribution), median of reps after 2 warm-ups"""
import json, statistics, sys
sys.path.insert(0, ".")
import torch
import ovs_inputs
import paper_1608_08648_b200 as ovs

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 5
CASES = [  # method, p, s/r, n, distributions
    ("ros", 4096, 64, 1 << 27, ["u32", "u32_u31", "u32_r26", "u32_few4", "u32_const", "i32_sorted", "i32_reverse",
                                "i32_gauss", "i32_few"]),
    ("dro", 256, 24, 1 << 24, ["i32_uniform", "i32_gauss", "i32_sorted", "i32_reverse", "i32_few"]),
]
for method, p, s, n, dists in CASES:
    for dist in dists:
        x = torch.from_numpy(ovs_inputs.keys(dist, n, seed=7)).cuda()
        srt = ovs.Sorter(n, x.dtype, False, method, p, s, 1)
        w = x.clone()
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps + 2)]
        for a, b in ev:
            w.copy_(x)
            a.record()
            srt(w)
            b.record()
        torch.cuda.synchronize()
        ms = statistics.median(a.elapsed_time(b) for a, b in ev[2:])
        print(json.dumps({"method": method, "dist": dist, "n": n, "p": p, "s_or_r": s, "ms": round(ms, 4),
                          "Gkeys_per_s": round(n / ms / 1e6, 2)}), flush=True)
        del srt
