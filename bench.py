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


def _cpu_model():
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


class _OneCore:
    """Pin this process to one host core for the oracle timing (SURVEY 8(d):
    single thread pinned with os.sched_setaffinity); restore afterwards."""

    def __enter__(self):
        self.prev = os.sched_getaffinity(0)
        self.core = min(self.prev)
        os.sched_setaffinity(0, {self.core})
        return self

    def __exit__(self, *exc):
        os.sched_setaffinity(0, self.prev)


def _oracle_rate(w, dtype, budget_s, max_cycles, warmup=1, warm_budget_s=30.0):
    """Oracle cycles of the full workload within ~budget_s on one pinned core, after
    min(warmup, ~warm_budget_s worth) untimed warm-up cycles (at least one)."""
    import oracle
    oracle.build()
    f = W.workload_rhs(w.name, dtype)
    u = np.zeros_like(f)
    N = (w.n - 2) ** w.dim
    with _OneCore() as pin:
        t0 = time.perf_counter()
        oracle.vcycle(u, f, w.p, 1, order=w.order)       # one warm-up cycle (allocation, page faults)
        t_one = time.perf_counter() - t0
        wu = max(1, min(warmup, int(warm_budget_s / max(t_one, 1e-3)) + 1))
        if wu > 1:
            oracle.vcycle(u, f, w.p, wu - 1, order=w.order)
        cyc = max(1, min(max_cycles, int(budget_s / max(t_one, 1e-3))))
        t0 = time.perf_counter()
        oracle.vcycle(u, f, w.p, cyc, order=w.order)
        dt = time.perf_counter() - t0
    sample = (f"{cyc} V-cycle(s) of the full {w.name} workload ({N} unknowns), single-threaded C oracle pinned "
              f"to host core {pin.core} ({dt:.1f} s; host: {os.cpu_count()} cores, {_cpu_model()})")
    return N * cyc / dt / 1e9, cyc, dt, sample, wu


def run_reference(args, w, ws, rank):
    """The oracle (plain single-threaded C) as the reference arm, on the host."""
    if rank != 0:
        return
    dtype = np.float64 if args.dtype == "f64" else np.float32
    value, steps, dt, sample, wu = _oracle_rate(w, dtype, 150.0, args.steps, args.warmup)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": steps, "warmup": wu, "ms_per_step": dt / steps * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": args.dtype, "data": "synthetic",
        "config": {"workload": w.name, "dim": w.dim, "n": w.n, "order": w.order, "p": list(w.p),
                   "unknowns": (w.n - 2) ** w.dim},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": 1, "kind": "oracle",
                         "sample": sample + f" (requested {args.steps} steps and {args.warmup} warm-up steps; "
                                             "capped to ~150 s timed and ~30 s of warm-up)"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def cpu_baseline(w, dtype, seconds=20.0):
    """Oracle throughput on a bounded sample of the same workload (1 pinned host core)."""
    value, _, _, sample, _ = _oracle_rate(w, dtype, seconds, w.cycles)
    return {"value": value, "unit": UNIT, "cores": 1, "kind": "oracle", "sample": sample}


def _spawn(args):
    """--gpus N without a launcher: re-run this command under torch.distributed.run
    (one rank per GPU, rendezvous on 127.0.0.1) and pass its exit code on."""
    import torch
    have = torch.cuda.device_count()
    if have < args.gpus:
        sys.exit(f"bench.py: --gpus {args.gpus} requested but only {have} CUDA device(s) are visible")
    import socket
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    sys.exit(subprocess.call(cmd))


def _roofline(s, u, f, ms_per_step, w, dtype_tag):
    """Dominant step of a separate, un-graphed per-step profile (CUDA events)."""
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
        traffic = tr.get(f"{w.name}/{dtype_tag}/{top['name']}")
    prof_ms = sum(r["ms"] for r in prof)
    return {
        "bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
        "traffic": traffic, "kernel": top["name"], "kernel_launches": top["launches"],
        "kernel_ms": top["ms"], "kernel_alg_bytes": top["alg_bytes"],
        "kernel_share_of_step": top["ms"] / prof_ms,
        "peak_source": peak_src,
        "cycle": {"alg_bytes": total_bytes, "achieved": cycle_gbs, "frac": cycle_gbs / peak},
        "steps": [{k: (round(v, 5) if isinstance(v, float) else v) for k, v in r.items()} for r in prof],
    }


def _b_alg(s, itemsize):
    """SURVEY 8(d) B_alg per V-cycle: w [5 N_0 + 5 sum_{l=1}^{L-2} N_l + 4 N_{L-1}]
    (every array once per producer/consumer, interior nodes only)."""
    L = s.levels
    pts = [s.level_points(l) for l in range(L)]
    return itemsize * (5 * pts[0] + 5 * sum(pts[1:L - 1]) + 4 * pts[L - 1])


def measure(args, w, tdt, ws, rank, local, slabs, dist, sampler_ok=True):
    """Time args.steps V-cycles of workload w in one mg_vcycle call (CUDA events
    on the calling stream, barrier + synchronize on both sides, max over ranks)."""
    import torch
    from paper_math_9907190_b200.mg import Solver
    npdt = np.float64 if tdt == torch.float64 else np.float32
    dtag = "f64" if tdt == torch.float64 else "f32"
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
        return None

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
    # SURVEY 8(d) headline fraction: B_alg per cycle (~10 values per unknown) over nominal 8 TB/s per GPU
    b_alg = _b_alg(s, u.element_size()) * (1 if slabs else ws)
    res = {"s": s, "u": u, "f": f, "f_host": f_host, "N": N, "units": units, "ms_per_step": ms_per_step,
           "value": value, "clocks": sampler.summary(t0, t1), "launches": s.launches_per_cycle,
           "levels": s.levels, "survey_frac_nominal": b_alg / (ms_per_step * 1e-3) / (8.0e12 * ws),
           "b_alg_per_cycle": b_alg}
    res["roofline"] = _roofline(s, u, f, ms_per_step, w, dtag)
    return res


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
    ap.add_argument("--no-sub", action="store_true", help="skip the 3D 513^3 sub-record")
    ap.add_argument("--profile-only", action="store_true", help="short run for ncu (no sampler/e2e/cpu)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    w = W.WORKLOADS[args.workload]
    ws, rank, local = _dist()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ and args.impl != "reference":
        _spawn(args)
    if args.impl == "reference":
        run_reference(args, w, ws, rank)
        return

    import torch
    import torch.distributed as dist

    torch.cuda.set_device(local)
    if ws > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    tdt = torch.float64 if args.dtype == "f64" else torch.float32

    # Multi-GPU: the slab solver over NCCL -- 2D y-slabs, 3D z-slabs, per-level
    # halo exchange, all-gather agglomeration of the coarse octaves (strong
    # scaling: the one global grid is split over the ranks).
    slabs = ws > 1
    m = measure(args, w, tdt, ws, rank, local, slabs, dist)
    if m is None:
        if rank == 0:
            print(json.dumps({"profile_only": True, "workload": w.name, "steps": args.steps}))
        return
    s, u, f, f_host, units = m["s"], m["u"], m["f"], m["f_host"], m["units"]
    stream = torch.cuda.current_stream()

    e2e = None
    if not args.no_e2e:
        # the user-facing calls on HOST buffers, the workload as BASELINE states it
        # ("V-cycles from u=0"): every step uploads its f, starts u at 0 on the
        # device, runs the workload's cycles and downloads its u -- all inside the
        # CUDA-event timed region.  Headline: mg_solve_host_batch over E2E_PROBLEMS
        # steps (each step's upload / download overlapping another step's cycles:
        # three streams, two device slots); single: one mg_solve_host call.
        E2E_PROBLEMS = 32   # the pipeline's fill and drain (one upload, one compute + download) amortised over 32
        uh = torch.zeros(s.shape, dtype=tdt).pin_memory()
        fh = torch.zeros(s.shape, dtype=tdt).pin_memory()
        s.view(fh).copy_(torch.from_numpy(np.ascontiguousarray(f_host)))
        s.solve_host_batch([uh] * 2, [fh] * 2, w.cycles)   # warm: graphs of both slots, staging, streams
        times = []
        for _ in range(2):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            s.solve_host_batch([uh] * E2E_PROBLEMS, [fh] * E2E_PROBLEMS, w.cycles)
            e1.record(stream)
            torch.cuda.synchronize()
            times.append(e0.elapsed_time(e1) / E2E_PROBLEMS)
        t_e2e = float(np.median(times))
        fb = uh.numel() * uh.element_size()
        if ws > 1:
            t = torch.tensor([t_e2e], device="cuda", dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            t_e2e = float(t.item())
        e2e = {"value": units * w.cycles / (t_e2e / 1e3) / 1e9, "unit": UNIT,
               "h2d_bytes_per_step": fb * ws, "d2h_bytes_per_step": fb * ws,
               "step": f"one solve: H2D f (pinned), u = 0 on the device, {w.cycles} V-cycles, D2H u; "
                       f"{E2E_PROBLEMS} steps per mg_solve_host_batch call, uploads and downloads overlapping "
                       "other steps' cycles",
               "ms_per_step": t_e2e}
        # the link's bound: the step's upload and download moved at once on two streams, no compute
        # (pinned, same sizes; best of 3) -- e2e cannot beat max(this, the cycles' device time)
        d_a, d_b = torch.empty_like(uh, device="cuda"), torch.empty_like(uh, device="cuda")
        s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
        tl = []
        for _ in range(3):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            s1.wait_stream(stream)
            s2.wait_stream(stream)
            with torch.cuda.stream(s1):
                d_a.copy_(fh, non_blocking=True)
            with torch.cuda.stream(s2):
                uh.copy_(d_b, non_blocking=True)
            stream.wait_stream(s1)
            stream.wait_stream(s2)
            e1.record(stream)
            torch.cuda.synchronize()
            tl.append(e0.elapsed_time(e1))
        del d_a, d_b
        t_link = max(min(tl), m["ms_per_step"] * w.cycles)
        e2e["bound"] = {"ms_per_step": t_link, "what": "max(H2D f + D2H u at once on two streams, measured; the "
                        "step's V-cycles at the device-timed rate)", "frac": t_link / t_e2e}
        s.solve_host(uh, fh, w.cycles)
        t1 = []
        for _ in range(2):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            s.solve_host(uh, fh, w.cycles)
            e1.record(stream)
            torch.cuda.synchronize()
            t1.append(e0.elapsed_time(e1))
        e2e["single"] = {"call": "mg_solve_host (one solve, nothing to overlap)", "ms_per_step": float(np.median(t1)),
                         "value": units * w.cycles / (float(np.median(t1)) / 1e3) / 1e9}
        # the warm-start variant (u uploaded as well), for reference
        s.vcycle_host(uh, fh, w.cycles)
        tw = []
        for _ in range(2):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            s.vcycle_host(uh, fh, w.cycles)
            e1.record(stream)
            torch.cuda.synchronize()
            tw.append(e0.elapsed_time(e1))
        e2e["warm_start"] = {"call": "mg_vcycle_host (H2D u, f; D2H u)", "ms_per_step": float(np.median(tw)),
                             "value": units * w.cycles / (float(np.median(tw)) / 1e3) / 1e9}

    pitch_n = None
    if not slabs and not args.no_e2e:
        pitch_n = _pitch_n_rate(s, w, tdt, args)

    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu:
        cpu = cpu_baseline(w, np.float64 if args.dtype == "f64" else np.float32)

    # BASELINE configs[4] (3D 513^3 fp64) and configs[2]'s "fp32 variant also timed"
    # (2D 8193^2 fp32) ride along as sub-records on one GPU, so the driver's single
    # line carries every north-star workload
    sub = []
    if not slabs and not args.no_sub:
        extra = []
        if w.name != "3d_513":
            extra.append(("3d_513", torch.float64))
        if w.name == "2d_8193" and tdt == torch.float64:
            extra.append(("2d_8193", torch.float32))
        if extra:
            for key in ("s", "u", "f"):
                m.pop(key)
            del s, u, f
            torch.cuda.empty_cache()
        for wname, sdt in extra:
            wx = W.WORKLOADS[wname]
            mx = measure(args, wx, sdt, ws, rank, local, False, dist)
            sub.append({"workload": wx.name, "dtype": "f64" if sdt == torch.float64 else "f32",
                        "value": mx["value"], "unit": UNIT,
                        "ms_per_step": mx["ms_per_step"], "steps": args.steps, "warmup": args.warmup,
                        "unknowns": mx["N"], "survey_frac_of_nominal_8tbs": mx["survey_frac_nominal"],
                        "gpu_launches": mx["s"].launches_per_cycle * args.steps,
                        "roofline": mx["roofline"], "clocks": mx["clocks"]})
            del mx
            torch.cuda.empty_cache()

    line = {
        "metric": METRIC, "value": m["value"], "unit": UNIT, "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": m["ms_per_step"], "higher_is_better": True,
        "scaling": "strong" if slabs else "weak", "vs_baseline": None, "dtype": args.dtype, "data": "synthetic",
        "config": {"workload": w.name, "dim": w.dim, "n": w.n, "order": w.order, "p": list(w.p),
                   "unknowns": m["N"], "rhs": w.note,
                   "parallelism": (f"{'y' if w.dim == 2 else 'z'}-slabs x{ws} (NCCL halo exchange, all-gather agglomeration)" if slabs
                                   else ("replicas" if ws > 1 else "single")),
                   "l2": "inputs larger than L2 (u and f are %.0f MB each vs 126 MB L2)" %
                         (s_bytes(w, tdt) / 1e6),
                   "levels": m["levels"]},
        "survey_frac_of_nominal_8tbs": m["survey_frac_nominal"],
        "roofline": m["roofline"],
        "cpu_baseline": cpu,
        "e2e": e2e,
        "pitch_n": pitch_n,
        # per call: K steady-state cycles, plus the first cycle's finest descent when the 2D single-GPU cycles
        # are fused; tests/test_gpu_launches.py checks this count against the CUDA profiler
        "gpu_launches": m["launches"] * args.steps + (
            1 if (w.dim == 2 and not slabs and os.environ.get("MG_2D_NOXFUSE", "0") in ("", "0")) else 0),
        "clocks": m["clocks"],
        "sub": sub or None,
    }
    if rank == 0:
        print(json.dumps(line), flush=True)
    if ws > 1:
        dist.destroy_process_group()


def s_bytes(w, tdt):
    import torch
    return w.n ** w.dim * (8 if tdt == torch.float64 else 4)


def _pitch_n_rate(s, w, tdt, args):
    """The C-ABI default layout (mg_create: pitch = n, unpadded device arrays):
    same cycles through the same kernels, u and f staged into the work layout
    once per call (include/mg.h).  One call of the workload's cycle count, timed
    with CUDA events; reported next to the headline."""
    import torch
    from paper_math_9907190_b200 import mg as M
    npdt = np.float64 if tdt == torch.float64 else np.float32
    cfg = M.mg_config()
    cfg.dim, cfg.n, cfg.order = w.dim, w.n, w.order
    cfg.dtype = M.MG_F64 if tdt == torch.float64 else M.MG_F32
    pp = list(w.p) + [0.0] * (4 - len(w.p))
    cfg.p = (M.ctypes.c_double * 4)(*pp)
    cfg.pitch = 0
    stream = torch.cuda.current_stream()
    cfg.stream = stream.cuda_stream
    cfg.device = torch.cuda.current_device()
    cfg.nranks, cfg.rank = 1, 0
    h = M.mg_create_ex(cfg)
    try:
        shape = (w.n,) * w.dim
        u = torch.zeros(shape, dtype=tdt, device="cuda")
        f = torch.from_numpy(W.workload_rhs(w.name, npdt)).cuda()
        M.mg_vcycle(h, u.data_ptr(), f.data_ptr(), 3)
        times = []
        for _ in range(3):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            M.mg_vcycle(h, u.data_ptr(), f.data_ptr(), w.cycles)
            e1.record(stream)
            torch.cuda.synchronize()
            times.append(e0.elapsed_time(e1))
        t = float(np.median(times))
        N = (w.n - 2) ** w.dim
        return {"value": N * w.cycles / (t / 1e3) / 1e9, "unit": UNIT, "ms_per_call": t, "cycles_per_call": w.cycles,
                "call": "mg_create(dim, n, order, p) + mg_vcycle on (n, n[, n]) device arrays: pitch = n, staged"}
    finally:
        M.mg_destroy(h)
        del u, f
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
