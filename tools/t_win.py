import sys; sys.path.insert(0, ".")
import numpy as np, torch, ovs_inputs, oracle, paper_1608_08648_b200 as ovs
if len(sys.argv) > 1:
    ovs.LIB_PATH = sys.argv[1]; ovs._lib = None
oracle.build()
for dist, n, p, r in (("u32", 1_600_000, 12, 2), ("u32", 2_400_000, 16, 2), ("u32", 1_000_000, 6, 2)):
    x = ovs_inputs.keys(dist, n, seed=7)
    ref = oracle.dro_sort(x, p, r)
    xt = torch.from_numpy(x).cuda()
    rep = ovs.Sorter(n, xt.dtype, False, "dro", p, r, 0)(xt, report=True)
    torch.cuda.synchronize()
    out = xt.cpu().numpy()
    bad = np.nonzero(out != ref.keys)[0]
    print(dist, n, p, r, "n/p", n // p, "ok" if bad.size == 0 else f"MISMATCH {bad.size} first {bad[:3]}", "status", rep.device_status, flush=True)
