"""Sample-parameter sweeps, the GPU analog of the paper's Tables 2, 5, 6
(ROS: s = ceil(lg^(1+a) n) for a in {0.2, 0.6, 1.0, 1.4, 1.8}) and Table 8
(DRO: r = 1..5), over a p grid 4 ... 8192, on 2^lg uniform u32 keys.

Per run: device time, Gkeys/s, the bucket expansion max|Y_j| / (n/p) and
- ROS: Claim 1 (log = natural log, reading Q12): the epsilon for which the
  claim's condition on s holds with equality at rho = 1,
      s = (1+eps)/eps^2 * L,  L = 2 rho ln n + ln(2 pi p^2 (ps-1) e^(1/(3(ps-1)))),
  i.e. eps = (L + sqrt(L^2 + 4 s L)) / (2 s), the claim's bucket bound ceil((1+eps)(n-p+1)/p)
  (every bucket at most this with probability >= 1 - 1/n when ps < n/2), the largest bucket
  over `seeds` sample seeds, and how many of those runs exceeded the bound;
- DRO: Lemma 1's bound ceil((1+1/r) n/p + r p) and the proof's tight form
  s x + (p-1)(x-1), x = ceil(ceil(n/p)/s), s = rp (reading Q10).
One JSON line per run.   python tools/sweep.py [lg n] [seeds]"""
import json
import math
import statistics
import sys

sys.path.insert(0, ".")
import torch

import ovs_inputs
import paper_1608_08648_b200 as ovs

lg = int(sys.argv[1]) if len(sys.argv) > 1 else 27
seeds = int(sys.argv[2]) if len(sys.argv) > 2 else 5
n = 1 << lg
x = torch.from_numpy(ovs_inputs.keys("u32", n, seed=61)).cuda()
w = x.clone()


def claim1(n, p, s, rho=1.0):
    m = p * s - 1
    L = 2 * rho * math.log(n) + math.log(2 * math.pi * p * p * m * math.exp(1 / (3 * m)))
    eps = (L + math.sqrt(L * L + 4 * s * L)) / (2 * s)
    return eps, math.ceil((1 + eps) * (n - p + 1) / p)


def timed(srt, reps=5):
    ms = []
    for _ in range(reps + 1):
        w.copy_(x)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        srt(w)
        b.record()
        b.synchronize()
        ms.append(a.elapsed_time(b))
    return statistics.median(ms[1:])


def ros(p, s, a):
    mxs = []
    t = None
    for sd in range(1, seeds + 1):
        srt = ovs.Sorter(n, torch.uint32, False, "ros", p, s, sd)
        w.copy_(x)
        rep = srt(w, report=True)
        mxs.append(int(rep.counts.max()))
        if sd == 1:
            t = timed(srt)
        del srt
    eps, bound = claim1(n, p, s)
    return {"method": "ros", "n": n, "p": p, "a": a, "s": s, "ms": round(t, 4), "Gkeys_per_s": round(n / t / 1e6, 2),
            "expansion": round(max(mxs) * p / n, 4), "max_bucket": max(mxs), "seeds": seeds,
            "claim1_eps": round(eps, 4), "claim1_bound": bound, "claim1_precondition_ps_lt_n_over_2": p * s < n / 2,
            "runs_over_claim1_bound": sum(1 for v in mxs if v > bound)}


def dro(p, r):
    srt = ovs.Sorter(n, torch.uint32, False, "dro", p, r, 1)
    w.copy_(x)
    rep = srt(w, report=True)
    mx = int(rep.counts.max())
    t = timed(srt)
    S = r * p
    xx = -(-(-(-n // p)) // S)
    lemma = math.ceil((1 + 1 / r) * n / p + r * p)
    tight = S * xx + (p - 1) * (xx - 1)
    return {"method": "dro", "n": n, "p": p, "r": r, "ms": round(t, 4), "Gkeys_per_s": round(n / t / 1e6, 2),
            "max_bucket": mx, "expansion": round(mx * p / n, 4), "lemma1_bound": lemma, "tight_bound": tight,
            "max_over_lemma1": round(mx / lemma, 4), "within_tight": mx <= tight}


for p in (4, 16, 64, 256, 1024, 4096, 8192):
    for a in (0.2, 0.6, 1.0, 1.4, 1.8):
        s = math.ceil(lg ** (1 + a))
        if p * s - 1 > n:
            print(json.dumps({"method": "ros", "n": n, "p": p, "a": a, "s": s, "skipped": "ps-1 > n"}), flush=True)
            continue
        try:
            print(json.dumps(ros(p, s, a)), flush=True)
        except Exception as e:  # p beyond the one-level classifier's shared memory
            print(json.dumps({"method": "ros", "n": n, "p": p, "a": a, "s": s, "error": str(e)[:200]}), flush=True)
        torch.cuda.empty_cache()
for p in (64, 256, 1024):
    for r in (1, 2, 3, 4, 5):
        if r * p > n // p:
            continue
        print(json.dumps(dro(p, r)), flush=True)
        torch.cuda.empty_cache()
ap = ovs.auto_params(n, torch.uint32, False, "ros")
o = ros(ap.p, ap.s, None)
o["auto_params"] = True
print(json.dumps(o), flush=True)
