"""Print selected metrics per kernel from `ncu -i X.ncu-rep --page raw --csv`:
python tools/ncu_raw.py raw.csv [metric-substring ...]"""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
h, units, data = rows[0], rows[1], rows[2:]
want = sys.argv[2:] or ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
                         "sm__warps_active.avg.pct_of_peak", "smsp__inst_executed.sum",
                         "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "lts__t_sectors.sum",
                         "smsp__average_warp_latency_issue_stalled", "sm__throughput.avg.pct",
                         "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"]
cols = [i for i, c in enumerate(h) if any(c.startswith(w) or c == w for w in want)]
for r in data:
    name = r[h.index("Kernel Name")][:60]
    print(f"== {r[0]} {name}")
    for i in cols:
        print(f"   {h[i]:70s} {r[i]:>18s} {units[i]}")
