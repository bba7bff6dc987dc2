"""Metric sort launched eagerly vs replayed from a CUDA graph (experiment)."""
import statistics, sys
sys.path.insert(0, ".")
import torch, numpy as np
import ovs_inputs
import paper_1608_08648_b200 as ovs

n, p, s = 1 << 27, 4096, 64
x = torch.from_numpy(ovs_inputs.keys("u32", n, seed=51)).cuda()
w = x.clone()
srt = ovs.Sorter(n, torch.uint32, False, "ros", p, s, 1)
st = torch.cuda.Stream()
with torch.cuda.stream(st):
    for _ in range(3):
        w.copy_(x); srt(w)
torch.cuda.synchronize()
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g, stream=st):
    srt(w)
torch.cuda.synchronize()
def timeit(fn, reps=20):
    ts = []
    for _ in range(reps):
        w.copy_(x)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record(); b.synchronize()
        ts.append(a.elapsed_time(b))
    return statistics.median(ts)
te = timeit(lambda: srt(w))
tg = timeit(lambda: g.replay())
h = w.cpu().numpy()
print(f"eager {te:.3f} ms  graph {tg:.3f} ms  sorted={bool(np.all(h[1:] >= h[:-1]))}")
for lgn, pp, ss in ((20, 64, 32), (24, 1024, 64)):
    nn = 1 << lgn
    xx = torch.from_numpy(ovs_inputs.keys("u32", nn, seed=1)).cuda(); ww = xx.clone()
    ss2 = ovs.Sorter(nn, torch.uint32, False, "ros", pp, ss, 1)
    with torch.cuda.stream(st):
        for _ in range(3): ww.copy_(xx); ss2(ww)
    torch.cuda.synchronize()
    g2 = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g2, stream=st):
        ss2(ww)
    def tm(fn):
        ts = []
        for _ in range(20):
            ww.copy_(xx); torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(); fn(); b.record(); b.synchronize(); ts.append(a.elapsed_time(b))
        return statistics.median(ts)
    print(f"n=2^{lgn}: eager {tm(lambda: ss2(ww)):.4f} ms  graph {tm(lambda: g2.replay()):.4f} ms")
