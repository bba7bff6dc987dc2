"""Quick GPU check against the oracle (development helper)."""
import sys, time
import numpy as np
import torch
sys.path.insert(0, ".")
import oracle, ovs_inputs
import paper_1608_08648_b200 as ovs

TT = {np.uint32: torch.uint32, np.int32: torch.int32, np.float64: torch.float64}

def run(dist, n, p, s, seed=1, kv=False, dseed=7):
    x = ovs_inputs.keys(dist, n, seed=dseed)
    v = ovs_inputs.index_values(n) if kv else None
    t0 = time.time()
    ref = oracle.ros_sort(x, p, s, seed, vals=v)
    to = time.time() - t0
    xt = torch.from_numpy(x).cuda()
    if kv:
        vt = torch.from_numpy(v.view(np.int32)).cuda().view(torch.uint32)
        rep = ovs.sort_pairs_stable(xt, vt, "ros", p, s, seed)
    else:
        rep = ovs.sort_keys(xt, "ros", p, s, seed)
    torch.cuda.synchronize()
    out = xt.cpu().numpy()
    ok_out = np.array_equal(out, ref.keys)
    ok_v = True
    if kv:
        ok_v = np.array_equal(vt.cpu().view(torch.int32).numpy().view(np.uint32), ref.vals)
    ok_c = np.array_equal(rep.counts, ref.counts)
    ok_s = np.array_equal(rep.splitter_keys, ref.split_keys) and np.array_equal(rep.splitter_tags, ref.split_tags)
    print(f"{dist:12s} n={n:9d} p={p:5d} s={s:3d} kv={kv}: out={ok_out} vals={ok_v} counts={ok_c} splitters={ok_s} "
          f"status={rep.device_status} gpu_ms={rep.total_ms:.3f} launches={rep.kernel_launches} oracle_s={to:.2f} maxb={rep.max_bucket}", flush=True)
    if not ok_out:
        bad = np.nonzero(out != ref.keys)[0]
        print("   first bad", bad[:10], out[bad[:5]], ref.keys[bad[:5]], "nbad", len(bad))
    return ok_out and ok_v and ok_c and ok_s

allok = True
for args in [("u32_u31", 1000, 4, 8), ("u32_u31", 1 << 20, 64, 32), ("i32_gauss", 100000, 16, 16),
             ("f64_normal", 200000, 64, 32), ("u32_const", 100000, 8, 8), ("u32_few4", 300000, 16, 8),
             ("u32_u31", 3, 1, 1), ("u32_u31", 100000, 1, 1), ("u32", 1 << 24, 4096, 64), ("u32", 1 << 27, 4096, 64)]:
    allok &= run(*args)
for args in [("u16key", 100000, 8, 8), ("u32_few4", 200000, 16, 16), ("f64_uniform", 100000, 32, 16)]:
    allok &= run(*args, kv=True)
print("ALLOK", allok)
