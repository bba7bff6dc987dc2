"""Aggregate an ncu source-page CSV (`--page source --csv --print-source cuda,sass`) per CUDA
source line: python tools/ncu_lines.py file.csv [top]"""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
agg = {}
h = None
for r in rows:
    if not r:
        continue
    if r[0] == "Line No":
        h = r
        ie = h.index("Instructions Executed")
        ws = h.index("Warp Stall Sampling (All Samples)")
        continue
    if h is None or len(r) < len(h) or not r[0].isdigit() or r[2] not in ("-", ""):
        continue
    try:
        key = r[0]
        a = agg.setdefault(key, [r[1], 0.0, 0.0])
        a[1] += float(r[ws] or 0)
        a[2] += float(r[ie] or 0)
    except ValueError:
        continue
ti = sum(a[2] for a in agg.values()) or 1
ts = sum(a[1] for a in agg.values()) or 1
print(f"total warp-inst {ti:.3e}  stall samples {ts:.0f}")
for k, a in sorted(agg.items(), key=lambda kv: -kv[1][1])[:top]:
    print(f"{a[1]/ts*100:5.1f}% stall {a[2]/ti*100:5.1f}% inst  L{k:>5} {a[0].strip()[:90]}")
