"""Per kernel, the warp-stall reasons of an `ncu --set full` capture, largest first, plus the shared-memory
pipe's share of the kernel's time:  ncu -i X.ncu-rep --page raw --csv > raw.csv; python tools/ncu_stalls.py raw.csv

Stall reasons: smsp__average_warps_issue_stalled_<reason>_per_issue_active.ratio (warps waiting for <reason> per
issued instruction; their sum + 1 is the average number of resident warps per scheduler per issue).
Shared pipe: l1tex__data_pipe_lsu_wavefronts_mem_shared.sum / (SMs x sm cycles) = wavefronts per cycle per SM
(the pipe retires one wavefront per cycle)."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
h, units, data = rows[0], rows[1], rows[2:]
PRE, SUF = "smsp__average_warps_issue_stalled_", "_per_issue_active.ratio"
stall_cols = [(i, c[len(PRE):-len(SUF)]) for i, c in enumerate(h) if c.startswith(PRE) and c.endswith(SUF)
              and not c[len(PRE):].startswith("not_issued")]


def col(name):
    return h.index(name) if name in h else None


def num(r, i):
    try:
        return float(r[i].replace(",", ""))
    except (TypeError, ValueError, AttributeError):
        return float("nan")


c_name, c_dur = col("Kernel Name"), col("gpu__time_duration.sum")
c_wf = col("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum")
c_bc = col("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum")
c_cyc = col("sm__cycles_elapsed.max")
c_sms = col("launch__sm_count") if "launch__sm_count" in h else col("device__attribute_multiprocessor_count")
for r in data:
    st = sorted(((num(r, i), n) for i, n in stall_cols), reverse=True)
    tot = sum(v for v, _ in st if v == v)
    dur, wf, bc, cyc = num(r, c_dur), num(r, c_wf), num(r, c_bc), num(r, c_cyc)
    sms = num(r, c_sms) if c_sms is not None else 148.0
    print(f"== {r[c_name][:70]} | {dur / 1e3 if units[c_dur] in ('ns', 'nsecond') else dur:.1f} us")
    print("   stalled warps per issue: " + ", ".join(f"{n} {v:.2f} ({v / tot * 100:.0f}%)" for v, n in st[:6]))
    if wf == wf and cyc == cyc and cyc > 0:
        print(f"   shared wavefronts {wf / 1e6:.1f}M ({bc / 1e6:.1f}M bank-conflict replays), "
              f"{wf / (sms * cyc) * 100:.0f}% of the shared pipe's cycles")
