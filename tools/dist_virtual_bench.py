"""Full-size multi-rank sort on ONE GPU with virtual ranks (dist.dist_sort_virtual: the collectives
are emulated by device copies, ranks run one after the other): correctness at 2^27 keys per rank and
the time of each rank's steps (not a scaling measurement: one GPU does every rank's work).
python tools/dist_virtual_bench.py G [n_per_rank_log2]"""
import sys, time
sys.path.insert(0, ".")
import numpy as np, torch
import ovs_inputs
from paper_1608_08648_b200.dist import dist_sort_virtual

G = int(sys.argv[1]) if len(sys.argv) > 1 else 2
lg = int(sys.argv[2]) if len(sys.argv) > 2 else 27
n = 1 << lg
p = 4096 // G * G
shards = [torch.from_numpy(ovs_inputs.keys("u32", n, seed=51, start=r * n)).cuda() for r in range(G)]
tot = sum(int(x.cpu().numpy().astype(np.uint64).sum()) for x in shards)  # exact
for it in range(2):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    out, _, counts = dist_sort_virtual([x.clone() for x in shards], None, p, 64, 1)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
h = out.cpu().numpy()
ok = bool(np.all(h[1:] >= h[:-1])) and h.size == G * n and int(h.astype(np.uint64).sum()) == tot
if not ok:
    ref = np.sort(np.concatenate([x.cpu().numpy() for x in shards]))
    bad = np.nonzero(h != ref)[0]
    starts = np.concatenate([[0], np.cumsum(counts)])
    b = np.searchsorted(starts, bad[0], side="right") - 1
    print(f"  mismatches {bad.size}, first at {bad[0]}: bucket {b} [{starts[b]}, {starts[b+1]}) len {counts[b]}, "
          f"owner rank {b * G // p}; buckets with errors: {sorted(set((np.searchsorted(starts, bad, side='right') - 1).tolist()))[:10]}")
print(f"G={G} n/rank=2^{lg} p={p}: sorted={ok} wall {dt*1e3:.1f} ms for all ranks (host-driven, sequential), "
      f"max bucket {int(counts.max())} = {counts.max() * p / (G * n):.2f} x mean")
