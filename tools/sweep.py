"""Sample-parameter sweeps (the paper's Tables 2, 5, 6, 8 vary a, r and p,
PAPER.md:728-737): device time, bucket expansion max|Y_j| / (n/p), and for DRO the Lemma 1 bound
ceil((1 + 1/r) n/p + r p) and the proof's tight form s x + (p-1)(x-1) with
x = ceil(ceil(n/p)/s), s = rp (Q10).  One JSON line per run.
python tools/sweep.py [log2 n]"""
import json, math, statistics, sys
sys.path.insert(0, ".")
import torch
import ovs_inputs
import paper_1608_08648_b200 as ovs

lg = int(sys.argv[1]) if len(sys.argv) > 1 else 24
n = 1 << lg
x = torch.from_numpy(ovs_inputs.keys("u32", n, seed=61)).cuda()


def run(method, p, s, reps=5):
    srt = ovs.Sorter(n, torch.uint32, False, method, p, s, 1)
    w = x.clone()
    rep = srt(w, report=True)
    ms = []
    for _ in range(reps + 1):
        w.copy_(x)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); srt(w); b.record(); b.synchronize()
        ms.append(a.elapsed_time(b))
    t = statistics.median(ms[1:])
    return t, int(rep.counts.max())


out = []
for p in (256, 1024, 4096):
    for a in (0.2, 0.6, 1.0):
        s = math.ceil(lg ** (1 + a))
        while p * s - 1 > n // 2:
            s //= 2
        t, mx = run("ros", p, s)
        out.append({"method": "ros", "n": n, "p": p, "a": a, "s": s, "ms": round(t, 4), "Gkeys_per_s": round(n / t / 1e6, 2),
                    "expansion": round(mx * p / n, 4)})
for s in (8, 16, 32, 64, 128):
    t, mx = run("ros", 4096, s)
    out.append({"method": "ros", "n": n, "p": 4096, "a": None, "s": s, "ms": round(t, 4),
                "Gkeys_per_s": round(n / t / 1e6, 2), "expansion": round(mx * 4096 / n, 4)})
for p in (64, 256):
    for r in (1, 2, 3, 4, 5):
        if r * p > n // p:
            continue
        t, mx = run("dro", p, r)
        S = r * p
        xx = -(-(-(-n // p)) // S)
        lemma = math.ceil((1 + 1 / r) * n / p + r * p)
        tight = S * xx + (p - 1) * (xx - 1)
        out.append({"method": "dro", "n": n, "p": p, "r": r, "ms": round(t, 4), "Gkeys_per_s": round(n / t / 1e6, 2),
                    "max_bucket": mx, "expansion": round(mx * p / n, 4), "lemma1_bound": lemma, "tight_bound": tight,
                    "max_over_lemma1": round(mx / lemma, 4)})
ap = ovs.auto_params(n, torch.uint32, False, "ros")
t, mx = run("ros", ap.p, ap.s)
out.append({"method": "ros", "n": n, "auto_params": True, "p": ap.p, "s": ap.s, "ms": round(t, 4),
            "Gkeys_per_s": round(n / t / 1e6, 2), "expansion": round(mx * ap.p / n, 4)})
for o in out:
    print(json.dumps(o), flush=True)
