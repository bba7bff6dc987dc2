"""Debug driver for the fused sample sort: one sort per config, flushed progress."""
import sys, time
sys.path.insert(0, ".")
import numpy as np, torch
import ovs_inputs, oracle
import paper_1608_08648_b200 as ovs
for (n, p, s) in [(1 << 16, 64, 32), (1 << 20, 64, 32), (1 << 22, 256, 64), (1 << 24, 1024, 64), (1 << 27, 4096, 64)]:
    x = ovs_inputs.keys("u32", n, seed=5)
    xt = torch.from_numpy(x).cuda()
    t = time.time()
    rep = ovs.sort_keys(xt, "ros", p, s, 1)
    torch.cuda.synchronize()
    out = xt.cpu().numpy()
    ok = bool(np.all(out[1:] >= out[:-1]))
    line = f"n={n} p={p} s={s} sorted={ok} {time.time() - t:.2f}s status={getattr(rep, 'device_status', None)}"
    if n <= 1 << 22:
        ref = oracle.ros_sort(x, p, s, 1)
        line += f" split_ok={np.array_equal(rep.splitter_keys, ref.split_keys) and np.array_equal(rep.splitter_tags, ref.split_tags)}"
    print(line, flush=True)
