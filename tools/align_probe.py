"""Sensitivity of the device time to where the workspace sits relative to the caller's key array:
python tools/align_probe.py [config ...]  -> one JSON line per (config, workspace offset).
The workspace is a slice of one larger allocation at a chosen byte offset (experiments only)."""
import json, statistics, sys
sys.path.insert(0, ".")
import torch
import ovs_inputs
import paper_1608_08648_b200 as ovs

CASES = {
    "C2-uniform": ("i32_uniform", 21, 1 << 24, "dro", 256, 24),
    "C5": ("u32", 51, 1 << 27, "ros", 4096, 64),
}
OFFS = [0, 1 << 16, 1 << 19, 1 << 20, 3 << 20, 1 << 22, 5 << 20, 1 << 23, 13 << 20, 1 << 24, 1 << 25, 1 << 26]
names = sys.argv[1:] or list(CASES)
for name in names:
    dist, dseed, n, method, p, s = CASES[name]
    x = torch.from_numpy(ovs_inputs.keys(dist, n, seed=dseed)).cuda()
    wk = x.clone()
    srt = ovs.Sorter(n, x.dtype, False, method, p, s, 1)
    nb = srt.ws_bytes
    big = torch.empty(nb + OFFS[-1] + 4096, dtype=torch.uint8, device="cuda")
    for off in OFFS:
        srt.ws = big[off:off + nb]
        srt.ws[:16].zero_()
        ms, ph = [], []
        for r in range(7):
            wk.copy_(x)
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(6)]
            ovs.set_phase_events(ev)
            srt(wk)
            ovs.set_phase_events(None)
            ev[5].synchronize()
            if r >= 2:
                ms.append(ev[0].elapsed_time(ev[5]))
                ph.append([ev[i].elapsed_time(ev[i + 1]) for i in range(5)])
        phases = {nm: round(statistics.median(q[i] for q in ph), 3) for i, nm in enumerate(ovs.PHASES)}
        print(json.dumps({"config": name, "ws_offset": off, "ws_minus_keys_mod_64MiB": (srt.ws.data_ptr() - wk.data_ptr()) % (1 << 26),
                          "ms": round(statistics.median(ms), 4), "phases_ms": phases}), flush=True)
    del srt, big, x, wk
    torch.cuda.empty_cache()
