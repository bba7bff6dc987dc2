#!/usr/bin/env python3
"""Benchmark of the B200-native oversampling sort (arXiv 1608.08648) — BASELINE.json metric:
Gkeys/s for 2^27 uint32 keys per GPU, plus the HBM-roofline fraction of the dominant kernel.

  python bench.py [--gpus N --steps K --warmup W]            # our CUDA path (one JSON line)
  python bench.py --impl reference [--steps K --warmup W]    # the CPU oracle, bounded sample
  torchrun --nproc-per-node N ... bench.py --gpus N ...      # one rank per GPU

A step is one whole sort (every row of SURVEY.md §8(a): sample, sample sort, splitters,
classify + histogram + scan, scatter, bucket sort) of 2^27 resident uint32 keys.  The input is
restored from a pristine copy before each step (outside the timed events); the 512 MiB
input and the 512 MiB restore copy exceed the 126 MB L2, so no step starts L2-warm.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

WORKLOAD = dict(workload="C5/metric: 2^27 uint32 keys per GPU, uniform on [0,2^32) (data seed 51), "
                         "ROS p=4096 s=64 (sample seed 1)",
                n=1 << 27, dist="u32", data_seed=51, method="ros", p=4096, s=64, seed=1)
METRIC = "sort throughput (BASELINE.json: Gkeys/s for 2^27 uint32 keys per B200)"
# algorithmic HBM bytes per key of each timed phase, u32 keys
PHASE_BYTES = {"classify_hist": 4, "scatter": 8, "bucket_sort": 8}


def measured_peak_gbs():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 100 ms while running."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.rows = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) == 6:
                self.rows.append(parts)

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        sm, mx, reasons = [], [], set()
        for r in self.rows:
            try:
                sm.append(float(r[0]))
                mx.append(float(r[1]))
            except ValueError:
                continue
            for nm, v in zip(names, r[2:]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def dist_info():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def run_reference(args):
    """The base contract's reference arm: the CPU oracle as it stands, on the box's host cores,
    each step a bounded sample of the workload (n_s keys, p scaled to keep n/p)."""
    rank, world, _ = dist_info()
    if rank != 0:
        return
    import oracle
    import ovs_inputs
    oracle.build()
    n_s = args.ref_n
    p_s = max(2, WORKLOAD["p"] * n_s // WORKLOAD["n"])
    x = ovs_inputs.keys(WORKLOAD["dist"], n_s, seed=WORKLOAD["data_seed"])
    for _ in range(args.warmup):
        oracle.ros_sort(x, p_s, WORKLOAD["s"], WORKLOAD["seed"])
    ts = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        oracle.ros_sort(x, p_s, WORKLOAD["s"], WORKLOAD["seed"])
        ts.append(time.perf_counter() - t0)
    sec = sum(ts) / len(ts)
    v = n_s / sec / 1e9
    sample = f"first {n_s} keys of the workload, ROS p={p_s} s={WORKLOAD['s']} (n/p kept), 1 thread"
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "Gkeys/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": sec * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "u32", "data": "synthetic",
            "config": {"workload": WORKLOAD["workload"], "global_batch": n_s, "seq_len": None,
                       "parallelism": "cpu oracle, 1 thread"},
            "cpu_baseline": {"value": v, "unit": "Gkeys/s", "cores": 1, "kind": "oracle", "sample": sample},
            "e2e": {"value": v, "unit": "Gkeys/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def run_dist(args, x, src, work, dev, rank, world, local):
    """N > 1: weak scaling, 2^27 keys per GPU; the library's distributed ROS sort (ovs_dist_sort_keys:
    sample records and count rows stored into every rank's NCCL window, the scatter storing every
    key straight into its owner's window over NVLink, LSA barriers, local bucket sort).  Device
    time per step with CUDA events, max over ranks."""
    import torch
    import torch.distributed as dist
    from paper_1608_08648_b200.dist import DistSorter
    n = args.n
    p = args.p // world * world  # 4096 buckets at every N (the write-combining scatter's range)
    s, seed = args.s, WORKLOAD["seed"]
    ds = DistSorter(n, torch.uint32, False, p, s, seed, device=dev)
    res = ds(src, report=True)
    host = res.keys.cpu().numpy()
    assert bool(np.all(host[1:] >= host[:-1]))
    nvlink = torch.tensor([float(res.exchange_bytes)], device=dev, dtype=torch.float64)
    dist.all_reduce(nvlink, op=dist.ReduceOp.SUM)
    for _ in range(args.warmup):
        ds(src)
    torch.cuda.synchronize(dev)
    sampler = ClockSampler(local)
    sampler.start()
    ms = []
    for _ in range(args.steps):
        dist.barrier()
        torch.cuda.synchronize(dev)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        ds(src)
        b.record()
        b.synchronize()
        ms.append(a.elapsed_time(b))
    t = torch.tensor([sum(ms)], device=dev, dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_per_step = float(t.item()) / args.steps
    value = n * world / (ms_per_step * 1e-3) / 1e9
    # end to end: pinned host shard -> device -> distributed sort -> host slice
    hx = torch.from_numpy(x).pin_memory()
    hout = torch.empty(ds.out_cap, dtype=torch.uint32).pin_memory()
    e2e, d2h = [], 0
    for k in range(args.e2e_steps + 1):
        dist.barrier()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        work.copy_(hx, non_blocking=True)
        r = ds(work)
        nk = r.keys.numel()
        hout[:nk].copy_(r.keys, non_blocking=True)
        b.record()
        b.synchronize()
        d2h = nk * 4
        if k > 0:
            e2e.append(a.elapsed_time(b))
    clocks = sampler.stop()
    te = torch.tensor([statistics.mean(e2e)], device=dev, dtype=torch.float64)
    dist.all_reduce(te, op=dist.ReduceOp.MAX)
    if rank == 0:
        line = {"metric": METRIC,
                "value": value, "unit": "Gkeys/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
                "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
                "dtype": "u32", "data": "synthetic (ovs_inputs, seeded)",
                "config": {"workload": f"C5: 2^27 uint32 keys per GPU x {world}, uniform on [0,2^32) (data seed 51), "
                                       f"ROS p={p} s={s}", "global_batch": n * world, "seq_len": None,
                           "parallelism": f"dp{world}: ovs_dist_sort_keys (NCCL symmetric window; sample, counts "
                                          f"and items stored into peer windows over NVLink; LSA barriers)",
                           "n_per_gpu": n, "p": p, "s": s,
                           "l2": "input 512 MiB per GPU > 126 MB L2"},
                "nvlink_bytes_per_step": float(nvlink.item()),
                "roofline": None, "cpu_baseline": None,
                "e2e": {"value": n * world / (float(te.item()) * 1e-3) / 1e9, "unit": "Gkeys/s",
                        "h2d_bytes_per_step": int(n * 4), "d2h_bytes_per_step": int(d2h),
                        "note": "per rank; value = all ranks' keys / max-over-ranks time"},
                "gpu_launches": res.kernel_launches * args.steps, "launches_per_step": res.kernel_launches,
                "phases_ms_rank0": dict(zip(["sample+records", "sample_sort", "hist+counts", "fused_scatter",
                                              "bucket_sort"], res.phase_ms[:5])),
                "clocks": clocks}
        print(json.dumps(line), flush=True)
    ds.close()
    dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--p", type=int, default=WORKLOAD["p"])
    ap.add_argument("--s", type=int, default=WORKLOAD["s"])
    ap.add_argument("--n", type=int, default=WORKLOAD["n"])
    ap.add_argument("--ref-n", type=int, default=1 << 22)
    ap.add_argument("--cpu-n", type=int, default=1 << 27, help="keys of the cpu_baseline oracle run (default: "
                    "the whole workload, ~20 s on one core)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=8)
    ap.add_argument("--force-dist", action="store_true", help="run the distributed path even at N=1 (tests)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.impl == "reference":
        run_reference(args)
        return

    import torch
    import ovs_inputs
    import paper_1608_08648_b200 as ovs

    rank, world, local = dist_info()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1 or args.force_dist:
        import torch.distributed as dist
        if world == 1:
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            os.environ.setdefault("MASTER_PORT", "29533")
            os.environ.setdefault("RANK", "0")
            os.environ.setdefault("WORLD_SIZE", "1")
        dist.init_process_group("nccl", device_id=dev)
    n, p, s, seed = args.n, args.p, args.s, WORKLOAD["seed"]

    x = ovs_inputs.keys(WORKLOAD["dist"], n, seed=WORKLOAD["data_seed"], start=rank * n)
    src = torch.from_numpy(x).to(dev)
    work = torch.empty_like(src)
    stream = torch.cuda.current_stream(dev)
    if world > 1 or args.force_dist:
        run_dist(args, x, src, work, dev, rank, world, local)
        return
    sorter = ovs.Sorter(n, torch.uint32, False, "ros", p, s, seed, device=dev)

    # one reported call: launch count, device status, and a correctness spot check
    work.copy_(src)
    rep = sorter(work, report=True)
    launches_per_step = rep.kernel_launches
    host = work.cpu().numpy()
    assert rep.device_status == 0, f"device status {rep.device_status}"
    assert bool(np.all(host[1:] >= host[:-1])) and int(host.astype(np.uint64).sum()) == int(x.astype(np.uint64).sum())

    for _ in range(args.warmup):
        work.copy_(src)
        sorter(work)
    torch.cuda.synchronize(dev)
    # the timed step replays the whole sort from a CUDA graph (captured once on these buffers)
    replay = sorter.graph(work)
    for _ in range(args.warmup):
        work.copy_(src)
        replay()
    torch.cuda.synchronize(dev)
    rep2 = None

    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(5)] for _ in range(args.steps)]
    sampler = ClockSampler(local)
    sampler.start()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    sorter.status(reset=True)  # clear the sticky device-status word before the timed replays
    for k in range(args.steps):
        work.copy_(src)
        evs[k][0].record(stream)
        replay()
        evs[k][4].record(stream)
    torch.cuda.synchronize(dev)
    # every timed replay ran its device-side checks (work lists, sample size) without a failure
    dev_status = sorter.status(reset=True)
    assert dev_status == 0, f"device status {dev_status} after the timed replays"
    # phase split of the same sort (eager launches with the library's phase events)
    pevs = [[torch.cuda.Event(enable_timing=True) for _ in range(6)] for _ in range(args.steps)]
    for k in range(args.steps):
        work.copy_(src)
        ovs.set_phase_events(pevs[k])
        sorter(work)
    ovs.set_phase_events(None)
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    step_ms = [evs[k][0].elapsed_time(evs[k][4]) for k in range(args.steps)]
    ph_names = list(ovs.PHASES)  # sample, sample_sort, classify_hist, scatter, bucket_sort
    phase_ms = {nm: statistics.mean(pevs[k][i].elapsed_time(pevs[k][i + 1]) for k in range(args.steps))
                for i, nm in enumerate(ph_names)}
    tot_ms = sum(step_ms)
    if world > 1:
        t = torch.tensor([tot_ms], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        tot_ms = float(t.item())
    ms_per_step = tot_ms / args.steps
    value = n * world / (ms_per_step * 1e-3) / 1e9

    # end to end through the public API: pinned host input -> device -> sort -> host result
    hx = torch.from_numpy(x).pin_memory()
    hout = torch.empty_like(hx).pin_memory()
    e2e = []
    for k in range(args.e2e_steps + 1):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        work.copy_(hx, non_blocking=True)
        sorter(work)
        hout.copy_(work, non_blocking=True)
        b.record(stream)
        b.synchronize()
        if k > 0:
            e2e.append(a.elapsed_time(b))
    e2e_serial_ms = statistics.mean(e2e)
    # the same host-to-host sorts as a stream through ovs.HostPipeline: step k's H2D copy overlaps step
    # k-1's D2H copy and sort; every step still copies its whole input in and its whole result out
    pipe = ovs.HostPipeline(sorter, torch.uint32)
    pipe.submit(hx, hout)
    pipe.wait()
    for k in range(args.e2e_steps):
        pipe.submit(hx, hout)
    e2e_ms = pipe.wait() / args.e2e_steps  # device time, first copy-in start to last copy-out end
    pipe.close()
    ho = hout.numpy()
    assert bool(np.all(ho[1:] >= ho[:-1])) and int(ho.astype(np.uint64).sum()) == int(x.astype(np.uint64).sum())
    clocks = sampler.stop()
    e2e_v = n * world / (e2e_ms * 1e-3) / 1e9

    # roofline of the dominant kernel (algorithmic bytes / event-timed duration)
    peak, peak_src = measured_peak_gbs()
    dom = max(PHASE_BYTES, key=lambda k: phase_ms[k])
    achieved = PHASE_BYTES[dom] * n / (phase_ms[dom] * 1e-3) / 1e9
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tpath):
        try:
            with open(tpath) as f:
                traffic = json.load(f).get(dom)
        except Exception:
            traffic = None
    roofline = {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": achieved / peak, "traffic": traffic, "peak_source": peak_src,
                "phases_ms": phase_ms,
                "phases_frac": {k: PHASE_BYTES[k] * n / (phase_ms[k] * 1e-3) / 1e9 / peak for k in PHASE_BYTES}}

    cpu = None
    cpu_extra = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        import oracle
        oracle.build()
        n_c = min(args.cpu_n, n)
        p_c = max(2, p * n_c // n)
        t0 = time.perf_counter()
        oracle.ros_sort(x[:n_c], p_c, s, seed)
        dt = time.perf_counter() - t0
        cpu = {"value": n_c / dt / 1e9, "unit": "Gkeys/s", "cores": 1, "kind": "oracle",
               "sample": f"{n_c} keys of the workload, ROS p={p_c} s={s}, one run, {dt:.1f} s"}
        # the paper's multi-core variant (McRan) on every core of the process, and the
        # standalone library sort column on one core: context for the oracle line
        cores = len(os.sched_getaffinity(0))
        t0 = time.perf_counter()
        oracle.mcran_sort(x[:n_c], p_c, s, seed, cores)
        dt_mc = time.perf_counter() - t0
        t0 = time.perf_counter()
        np.sort(x[:n_c])
        dt_np = time.perf_counter() - t0
        cpu_extra = {"mcran": {"value": n_c / dt_mc / 1e9, "unit": "Gkeys/s", "cores": cores, "kind": "oracle-mcran",
                               "sample": f"{n_c} keys, SqRan with steps 1/4/5 on {cores} threads, {dt_mc:.1f} s"},
                     "standalone": {"value": n_c / dt_np / 1e9, "unit": "Gkeys/s", "cores": 1,
                                    "kind": "numpy.sort", "sample": f"{n_c} keys, {dt_np:.1f} s"}}

    if rank == 0:
        line = {"metric": METRIC,
                "value": value, "unit": "Gkeys/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
                "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
                "dtype": "u32", "data": "synthetic (ovs_inputs, seeded)",
                "config": {"workload": WORKLOAD["workload"] if (p, s, n) == (WORKLOAD["p"], WORKLOAD["s"], WORKLOAD["n"])
                           else f"{n} uint32 uniform, ROS p={p} s={s}",
                           "global_batch": n * world, "seq_len": None,
                           "parallelism": "single GPU" if world == 1 else f"{world} independent replicas",
                           "n_per_gpu": n, "p": p, "s": s,
                           "l2": "input 512 MiB > 126 MB L2; 512 MiB restore copy before every step",
                           "launch": "timed steps replay the whole sort from a CUDA graph captured once "
                                     "(Sorter.graph); phases_ms from eager launches with phase events"},
                "roofline": roofline, "cpu_baseline": cpu, "cpu_baselines_context": cpu_extra,
                "e2e": {"value": e2e_v, "unit": "Gkeys/s", "h2d_bytes_per_step": int(n * 4),
                        "d2h_bytes_per_step": int(n * 4), "ms_per_step": e2e_ms,
                        "how": f"{args.e2e_steps} host-to-host sorts streamed through the C ABI's ovs_host_pipe_* (ovs.HostPipeline; three rotating "
                               "device buffers: H2D of step k overlaps D2H of step k-1 and the sorts), device-timed "
                               "first H2D start to last D2H end",
                        "serial_ms_per_step": e2e_serial_ms,
                        "serial_value": n * world / (e2e_serial_ms * 1e-3) / 1e9},
                "gpu_launches": launches_per_step * args.steps, "launches_per_step": launches_per_step,
                "device_status": dev_status,
                "clocks": clocks}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
