#!/usr/bin/env python
"""Benchmark of the diagonal-multigrid V-cycle on B200 (BASELINE.json metric).

    python bench.py [--gpus N --steps K --warmup W] [--workload 2d_8193] [--dtype f64]
    python bench.py --impl reference ...      # the CPU oracle arm

One *step* is one V-cycle (every row of SURVEY.md 8(a)) on the workload's
seeded synthetic right-hand side.  `value` is fine-grid unknowns x V-cycles
per second over all ranks (GDOF*V/s), timed with CUDA events on the stream
the work is ordered on, inputs resident in HBM (each 537 MB field is larger
than the 126 MB L2).  Prints ONE JSON line on rank 0.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_math_9907190_b200 import workloads as W  # noqa: E402

METRIC = "GDOF·V-cycles/s (fine unknowns × cycles/sec) and % HBM roofline, 1-8 B200"
UNIT = "GDOF*V-cycles/s"


def _peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as fh:
            d = json.load(fh)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy read+write)"
    return 6650.0, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 100 ms in the background."""
    FIELDS = ("timestamp,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.rows = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits", "-lms", "100",
                 "-i", str(self.gpu)], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
            return
        self.t = threading.Thread(target=self._read, daemon=True)
        self.t.start()

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append((time.time(), [x.strip() for x in line.split(",")]))

    def stop(self):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self, t0, t1):
        rows = [r for (t, r) in self.rows if t0 - 0.05 <= t <= t1 + 0.15]
        if not rows:
            rows = [r for (_, r) in self.rows]
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if len(r) > 5 + i and r[5 + i] == "Active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows)}


def _dist():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def run_reference(args, w, ws, rank):
    """The oracle (plain single-threaded C) as the reference arm, on the host."""
    if rank != 0:
        return
    import oracle
    oracle.build()
    dtype = np.float64 if args.dtype == "f64" else np.float32
    f = W.workload_rhs(w.name, dtype)
    u = np.zeros_like(f)
    N = (w.n - 2) ** w.dim
    t0 = time.perf_counter()
    oracle.vcycle(u, f, w.p, 1, order=w.order)       # one warm-up cycle (allocation, page faults)
    t_one = time.perf_counter() - t0
    budget = 150.0
    steps = max(1, min(args.steps, int(budget / max(t_one, 1e-3))))
    t0 = time.perf_counter()
    oracle.vcycle(u, f, w.p, steps, order=w.order)
    dt = time.perf_counter() - t0
    value = N * steps / dt / 1e9
    sample = f"{steps} V-cycle(s) of the full {w.name} workload (requested {args.steps}; capped to ~{budget:.0f} s)"
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": steps, "warmup": 1, "ms_per_step": dt / steps * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": args.dtype, "data": "synthetic",
        "config": {"workload": w.name, "dim": w.dim, "n": w.n, "order": w.order, "p": list(w.p),
                   "unknowns": N},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": 1, "kind": "oracle", "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def cpu_baseline(w, dtype, seconds=20.0):
    """Oracle throughput on a bounded sample of the same workload (1 host core)."""
    import oracle
    oracle.build()
    f = W.workload_rhs(w.name, dtype)
    u = np.zeros_like(f)
    N = (w.n - 2) ** w.dim
    t0 = time.perf_counter()
    oracle.vcycle(u, f, w.p, 1, order=w.order)
    t1 = time.perf_counter() - t0
    cyc = max(1, min(w.cycles, int(seconds / max(t1, 1e-3))))
    t0 = time.perf_counter()
    oracle.vcycle(u, f, w.p, cyc, order=w.order)
    dt = time.perf_counter() - t0
    return {"value": N * cyc / dt / 1e9, "unit": UNIT, "cores": 1, "kind": "oracle",
            "sample": f"{cyc} V-cycle(s) of the full {w.name} workload, single-threaded C oracle "
                      f"({dt:.1f} s; host has {os.cpu_count()} cores)"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=400)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--impl", default="libmg", choices=["libmg", "reference"])
    ap.add_argument("--workload", default="2d_8193", choices=sorted(W.WORKLOADS))
    ap.add_argument("--dtype", default="f64", choices=["f64", "f32"])
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--profile-only", action="store_true", help="short run for ncu (no sampler/e2e/cpu)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    w = W.WORKLOADS[args.workload]
    ws, rank, local = _dist()

    if args.impl == "reference":
        run_reference(args, w, ws, rank)
        return

    import torch
    import torch.distributed as dist
    from paper_math_9907190_b200.mg import Solver

    torch.cuda.set_device(local)
    if ws > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    tdt = torch.float64 if args.dtype == "f64" else torch.float32
    npdt = np.float64 if args.dtype == "f64" else np.float32

    # Multi-GPU: the slab solver over NCCL -- 2D y-slabs, 3D z-slabs, per-level
    # halo exchange, all-gather agglomeration of the coarse octaves (strong
    # scaling: the one global grid is split over the ranks).
    slabs = ws > 1
    if slabs:
        s = Solver(w.dim, w.n, order=w.order, p=w.p, dtype=tdt, group=dist.group.WORLD)
    else:
        s = Solver(w.dim, w.n, order=w.order, p=w.p, dtype=tdt)
    f_full = W.workload_rhs(w.name, npdt)
    if slabs:
        from paper_math_9907190_b200.mg import split_rows
        f_host = split_rows(f_full, s.lo, s.hi, s.ghost)
    else:
        f_host = f_full
    u = s.alloc()
    f = s.alloc(f_host)
    N = (w.n - 2) ** w.dim
    stream = torch.cuda.current_stream()

    s.vcycle(u, f, args.warmup)
    torch.cuda.synchronize()
    if args.profile_only:
        # ncu --profile-from-start off captures exactly these cycles
        torch.cuda.profiler.start()
        s.vcycle(u, f, args.steps)
        torch.cuda.synchronize()
        torch.cuda.profiler.stop()
        if rank == 0:
            print(json.dumps({"profile_only": True, "workload": w.name, "steps": args.steps}))
        return

    sampler = ClockSampler(local)
    sampler.start()
    # keep the GPU busy while nvidia-smi starts, so the samples are under load
    t_end = time.time() + 1.0
    while time.time() < t_end:
        s.vcycle(u, f, 20)
        torch.cuda.synchronize()

    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if ws > 1:
        dist.barrier()
    torch.cuda.synchronize()
    t0 = time.time()
    torch.cuda.profiler.start()      # ncu --profile-from-start off: the timed region only
    ev0.record(stream)
    s.vcycle(u, f, args.steps)
    ev1.record(stream)
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()
    t1 = time.time()
    if ws > 1:
        dist.barrier()
    ms = ev0.elapsed_time(ev1)
    sampler.stop()
    if ws > 1:
        t = torch.tensor([ms], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    ms_per_step = ms / args.steps
    units = N if slabs else ws * N   # strong scaling: one grid; replicas: ws grids
    value = units * args.steps / (ms / 1e3) / 1e9
    clocks = sampler.summary(t0, t1)

    # per-step CUDA-event profile (separate, un-graphed pass) for the roofline
    prof = s.profile(u, f, 10)
    peak, peak_src = _peaks()
    top = max(prof, key=lambda r: r["ms"])
    achieved = top["alg_bytes"] / (top["ms"] / top["launches"] * 1e-3) / 1e9 / top["launches"]
    total_bytes = sum(r["alg_bytes"] for r in prof)
    cycle_gbs = total_bytes / (ms_per_step * 1e-3) / 1e9
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tpath):
        with open(tpath) as fh:
            tr = json.load(fh)
        key = f"{w.name}/{args.dtype}/{top['name']}"
        if key in tr:
            traffic = tr[key]
    prof_ms = sum(r["ms"] for r in prof)
    roofline = {
        "bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
        "traffic": traffic, "kernel": top["name"], "kernel_launches": top["launches"],
        "kernel_ms": top["ms"], "kernel_alg_bytes": top["alg_bytes"],
        "kernel_share_of_step": top["ms"] / prof_ms,
        "peak_source": peak_src,
        "cycle": {"alg_bytes": total_bytes, "achieved": cycle_gbs, "frac": cycle_gbs / peak},
        "steps": [{k: (round(v, 5) if isinstance(v, float) else v) for k, v in r.items()} for r in prof],
    }

    e2e = None
    if not args.no_e2e:
        # the user-facing call on HOST buffers: copy u, f in, run the workload's
        # cycles, copy u out -- all inside the CUDA-event timed region
        uh = torch.zeros(s.shape, dtype=tdt).pin_memory()
        fh = torch.zeros(s.shape, dtype=tdt).pin_memory()
        s.view(fh).copy_(torch.from_numpy(np.ascontiguousarray(f_host)))
        s.vcycle_host(uh, fh, w.cycles)
        times = []
        for _ in range(3):
            uh.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            s.vcycle_host(uh, fh, w.cycles)
            e1.record(stream)
            torch.cuda.synchronize()
            times.append(e0.elapsed_time(e1))
        t_e2e = float(np.median(times))
        fb = uh.numel() * uh.element_size()
        if ws > 1:
            t = torch.tensor([t_e2e], device="cuda", dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            t_e2e = float(t.item())
        e2e = {"value": units * w.cycles / (t_e2e / 1e3) / 1e9, "unit": UNIT,
               "h2d_bytes_per_step": 2 * fb * ws, "d2h_bytes_per_step": fb * ws,
               "step": f"one mg_vcycle_host call: H2D u,f (pinned) + {w.cycles} V-cycles + D2H u",
               "ms_per_step": t_e2e}

    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu:
        cpu = cpu_baseline(w, npdt)

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
        "scaling": "strong" if slabs else "weak", "vs_baseline": None, "dtype": args.dtype, "data": "synthetic",
        "config": {"workload": w.name, "dim": w.dim, "n": w.n, "order": w.order, "p": list(w.p),
                   "unknowns": N, "rhs": w.note,
                   "parallelism": (f"{'y' if w.dim == 2 else 'z'}-slabs x{ws} (NCCL halo exchange, all-gather agglomeration)" if slabs
                                   else ("replicas" if ws > 1 else "single")),
                   "l2": "inputs larger than L2 (u and f are %.0f MB each vs 126 MB L2)" %
                         (s.view(u).numel() * u.element_size() / 1e6),
                   "levels": s.levels},
        "roofline": roofline,
        "cpu_baseline": cpu,
        "e2e": e2e,
        # per call: K steady-state cycles, plus the first cycle's finest descent when the 2D single-GPU cycles
        # are fused; tests/test_gpu_launches.py checks this count against the CUDA profiler
        "gpu_launches": s.launches_per_cycle * args.steps + (
            1 if (w.dim == 2 and not slabs and os.environ.get("MG_2D_NOXFUSE", "0") in ("", "0")) else 0),
        "clocks": clocks,
    }
    if rank == 0:
        print(json.dumps(line), flush=True)
    if ws > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
