"""Small sorts for compute-sanitizer (one tool per GPU call):
   compute-sanitizer --tool {memcheck|racecheck|synccheck} python tools/sanitize_one.py
Covers: C1 (ROS u32), ROS key-value with oversized buckets (windows), the direct-address sample,
DRO keys-only, DRO key-value, the DRO merge (f2), and an emulated 2-rank distributed sort (f1)."""
import sys
sys.path.insert(0, ".")
import numpy as np
import torch

import ovs_inputs
import paper_1608_08648_b200 as ovs
from paper_1608_08648_b200.dist import dist_sort_virtual


def run(dist, n, method, p, s, kv=False, merge=False):
    x = torch.from_numpy(ovs_inputs.keys(dist, n, seed=5)).cuda()
    v = torch.from_numpy(ovs_inputs.index_values(n)).cuda() if kv else None
    srt = ovs.Sorter(n, x.dtype, kv, method, p, s, 1, merge=merge)
    rep = srt(x, v, report=True) if kv else srt(x, report=True)
    h = x.cpu().numpy()
    ok = bool(np.all(h[1:] >= h[:-1])) and rep.device_status == 0
    print(f"{dist} n={n} {method} p={p} s={s} kv={kv} merge={merge}: sorted={ok}", flush=True)
    assert ok


run("u32_u31", 1 << 20, "ros", 64, 32)                 # C1
run("u16key", 300_000, "ros", 8, 8, kv=True)           # key-value, windows
run("u32", 200_000, "ros", 16, 11_000)                 # direct-address sample (ps-1 = 0.88 n)
run("i32_gauss", 1 << 20, "dro", 64, 4)                # DRO keys
run("u16key", 400_000, "dro", 16, 3, kv=True)          # DRO key-value
run("i32_few", 500_000, "dro", 32, 4, merge=True)      # f2 merge
xs = [torch.from_numpy(ovs_inputs.keys("u32", 200_000, seed=7, start=r * 200_000)).cuda() for r in range(2)]
out, _, counts, _, _, _ = dist_sort_virtual(xs, None, 64, 16, 3)
h = out.cpu().numpy()
assert bool(np.all(h[1:] >= h[:-1])) and int(counts.sum()) == 400_000
print("emulated 2-rank distributed sort: sorted=True", flush=True)
print("sanitize_one: done")
