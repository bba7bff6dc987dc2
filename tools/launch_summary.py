"""Summarise an ncu launch-list CSV (--metrics gpu__time_duration.sum,dram__bytes_read.sum,
dram__bytes_write.sum --csv) of one bench run: per-launch table of the LAST sort (the timed
step) and per-kernel share of that sort's time.
python tools/launch_summary.py launches.csv launches_per_sort [title]"""
import csv, sys
from collections import OrderedDict
path, per = sys.argv[1], int(sys.argv[2])
title = sys.argv[3] if len(sys.argv) > 3 else path
L = OrderedDict()
for r in csv.reader(open(path)):
    if len(r) < 15 or r[0] == "ID":
        continue
    d = L.setdefault(int(r[0]), {"name": r[4].split("(")[0], "grid": r[8], "block": r[7]})
    v = float(r[14].replace(",", ""))
    unit = r[13]
    if r[12] == "gpu__time_duration.sum":
        d["ns"] = v * {"ns": 1, "us": 1e3, "usecond": 1e3, "nsecond": 1, "ms": 1e6, "msecond": 1e6}.get(unit, 1)
    elif r[12].startswith("dram__bytes_read"):
        d["rd"] = v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
    elif r[12].startswith("dram__bytes_write"):
        d["wr"] = v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
ids = sorted(L)
# the launches of one sort: find the last run of `per` launches that starts at the first kernel name
first = L[ids[0]]["name"]
starts = [i for i in ids if L[i]["name"] == first]
last = [i for i in ids if i >= starts[-1]][:per]
tot = sum(L[i].get("ns", 0) for i in last)
print(f"# {title}")
print(f"# ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none")
print(f"# one sort = {len(last)} launches, sum of serialised cold-cache launch times {tot/1e3:.1f} us")
print("# id | kernel | grid | ns | share | dram read B | dram write B")
for i in last:
    d = L[i]
    print(f"{i} | {d['name']} | {d['grid']} | {d.get('ns',0):.0f} | {d.get('ns',0)/tot*100:.1f}% | {d.get('rd',0):.0f} | {d.get('wr',0):.0f}")
agg = OrderedDict()
for i in last:
    n = L[i]["name"]
    agg[n] = agg.get(n, 0) + L[i].get("ns", 0)
print("# per kernel: share of the sort")
for n, v in sorted(agg.items(), key=lambda kv: -kv[1]):
    print(f"#   {v/tot*100:5.1f}%  {v/1e3:8.1f} us  {n}")
