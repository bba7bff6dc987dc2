"""Per CUDA source line: stall %, inst %, shared wavefronts and excess (bank-conflict) wavefronts.
python tools/ncu_lines2.py file.csv [top] [sort-col: stall|inst|wf|ex]"""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
sk = sys.argv[3] if len(sys.argv) > 3 else "stall"
agg, h = {}, None
for r in rows:
    if not r:
        continue
    if r[0] == "Line No":
        h = r
        ie = h.index("Instructions Executed"); ws = h.index("Warp Stall Sampling (All Samples)")
        wf = h.index("L1 Wavefronts Shared"); ex = h.index("L1 Wavefronts Shared Excessive")
        continue
    if h is None or len(r) < len(h) or not r[0].isdigit() or r[2] not in ("-", ""):
        continue
    a = agg.setdefault(r[0], [r[1], 0.0, 0.0, 0.0, 0.0])
    for j, c in enumerate((ws, ie, wf, ex)):
        try:
            a[1 + j] += float(r[c] or 0)
        except ValueError:
            pass
tot = [sum(a[j] for a in agg.values()) or 1 for j in range(1, 5)]
print(f"stall samples {tot[0]:.0f} warp-inst {tot[1]:.3e} smem wavefronts {tot[2]:.3e} excess {tot[3]:.3e}")
col = {"stall": 1, "inst": 2, "wf": 3, "ex": 4}[sk]
for k, a in sorted(agg.items(), key=lambda kv: -kv[1][col])[:top]:
    print(f"{a[1]/tot[0]*100:5.1f}%st {a[2]/tot[1]*100:5.1f}%in {a[3]/tot[2]*100:5.1f}%wf {a[4]/tot[2]*100:5.1f}%ex L{k:>5} {a[0].strip()[:80]}")
