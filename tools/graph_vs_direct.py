#!/usr/bin/env python
"""ms per V-cycle: graph replay (mg_vcycle) vs the un-graphed per-step profile
(mg_profile, CUDA events between steps), interleaved; plus the per-step list.

    python tools/graph_vs_direct.py --dim 3 --n 513 [--dtype f32] [--cycles 100]
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
    ap.add_argument("--cycles", type=int, default=100)
    ap.add_argument("--rounds", type=int, default=3)
    a = ap.parse_args()
    p = (1.052,) if a.dim == 2 else (1.11, 1.42, 1.08, 0.99)
    tdt = torch.float64 if a.dtype == "f64" else torch.float32
    s = Solver(a.dim, a.n, order=2, p=p, dtype=tdt)
    f = W.random_field(a.dim, a.n, seed=1).astype(np.float64 if a.dtype == "f64" else np.float32)
    u, fd = s.alloc(), s.alloc(f)
    s.vcycle(u, fd, 5)
    torch.cuda.synchronize()
    g, d, dw = [], [], []
    steps = None
    for _ in range(a.rounds):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        s.vcycle(u, fd, a.cycles)
        e1.record()
        torch.cuda.synchronize()
        g.append(e0.elapsed_time(e1) / a.cycles)
        e0.record()
        prof = s.profile(u, fd, a.cycles)
        e1.record()
        torch.cuda.synchronize()
        dw.append(e0.elapsed_time(e1) / a.cycles)
        d.append(sum(x["ms"] for x in prof))
        steps = prof
    out = {"dim": a.dim, "n": a.n, "dtype": a.dtype, "graph_ms": float(np.median(g)),
           "direct_sum_ms": float(np.median(d)), "direct_wall_ms": float(np.median(dw)),
           "steps": [(x["name"], x["level"], round(x["ms"] * 1000, 1)) for x in steps]}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
