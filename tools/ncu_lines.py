"""Aggregate an ncu 'source --print-source cuda,sass' CSV per CUDA source line:
python tools/ncu_lines.py file.csv [top]"""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
lines = []
h = None
fname = ""
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        h = r
        ie = h.index("Instructions Executed")
        ws = h.index("Warp Stall Sampling (All Samples)")
        continue
    if h is None or len(r) < len(h) or r[0] == "" or not r[0].isdigit():
        continue
    try:
        lines.append([fname + ":" + r[0], r[1], float(r[ws] or 0), float(r[ie] or 0)])
    except ValueError:
        continue
ti = sum(l[3] for l in lines) or 1
ts = sum(l[2] for l in lines) or 1
print(f"total warp-inst {ti:.3e}  stall samples {ts:.0f}")
for l in sorted(lines, key=lambda l: -l[2])[:top]:
    print(f"{l[2]/ts*100:5.1f}% stall {l[3]/ti*100:5.1f}% inst  {l[0]:>22} {l[1].strip()[:90]}")
