#!/usr/bin/env python
"""Kernel timeline of graph-replayed V-cycles from CUPTI (torch.profiler):
per-kernel durations inside the graph and the idle gaps between consecutive
kernels (launch latency + ramp), i.e. what the per-step profile cannot see.

    python tools/graph_timeline.py --dim 3 --n 513 [--dtype f32] [--cycles 3]
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_math_9907190_b200 import workloads as W  # noqa: E402
from paper_math_9907190_b200.mg import Solver  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--dim", type=int, default=3)
    ap.add_argument("--n", type=int, default=513)
    ap.add_argument("--dtype", default="f64")
    ap.add_argument("--cycles", type=int, default=3)
    a = ap.parse_args()
    p = (1.052,) if a.dim == 2 else (1.11, 1.42, 1.08, 0.99)
    tdt = torch.float64 if a.dtype == "f64" else torch.float32
    s = Solver(a.dim, a.n, order=2, p=p, dtype=tdt)
    f = W.random_field(a.dim, a.n, seed=1).astype(np.float64 if a.dtype == "f64" else np.float32)
    u, fd = s.alloc(), s.alloc(f)
    s.vcycle(u, fd, 2 + a.cycles)   # the graphs of this call pattern exist
    torch.cuda.synchronize()
    from torch.profiler import ProfilerActivity, profile
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        s.vcycle(u, fd, 2 + a.cycles)
        torch.cuda.synchronize()
    ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA and "Memcpy" not in e.name
          and "Memset" not in e.name]
    ev.sort(key=lambda e: e.time_range.start)
    rows = []
    for i, e in enumerate(ev):
        gap = (e.time_range.start - ev[i - 1].time_range.end) if i else 0.0
        rows.append((e.name.split("(")[0].replace("void ", "")[:48], e.time_range.elapsed_us(), gap))
    total = (ev[-1].time_range.end - ev[0].time_range.start)
    busy = sum(r[1] for r in rows)
    gaps = sum(r[2] for r in rows)
    print(json.dumps({"dim": a.dim, "n": a.n, "dtype": a.dtype, "kernels": len(rows), "span_us": total,
                      "busy_us": busy, "gap_us": gaps}))
    for r in rows:
        print(f"  {r[1]:9.1f} us  gap {r[2]:6.1f}  {r[0]}")


if __name__ == "__main__":
    main()
