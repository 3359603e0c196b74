#!/usr/bin/env python
"""ms per V-cycle of the library's variants (order, dtype) at the big sizes.

    python tools/variants.py [--cycles 20]
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


def time_variant(dim, n, order, dtype, cycles):
    p = ((1.052 if order == 2 else 1.20),) if dim == 2 else (0.91, 0.80, 0.70, 1.77)
    tdt = torch.float64 if dtype == "f64" else torch.float32
    s = Solver(dim, n, order=order, p=p, dtype=tdt)
    f = W.random_field(dim, n, seed=1).astype(np.float64 if dtype == "f64" else np.float32)
    u, fd = s.alloc(), s.alloc(f)
    s.vcycle(u, fd, 4)
    torch.cuda.synchronize()
    ts = []
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        s.vcycle(u, fd, cycles)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) / cycles)
    ms = float(np.median(ts))
    return {"dim": dim, "n": n, "order": order, "dtype": dtype, "ms": ms, "gdof_v_s": (n - 2) ** dim / ms * 1e-6}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cycles", type=int, default=20)
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    res = []
    for dim, n, order, dtype in [(3, 513, 2, "f64"), (3, 513, 2, "f32"), (3, 513, 4, "f64"), (3, 513, 4, "f32"),
                                 (2, 8193, 4, "f64"), (2, 8193, 4, "f32")]:
        r = time_variant(dim, n, order, dtype, args.cycles)
        print(json.dumps(r), flush=True)
        res.append(r)
        torch.cuda.empty_cache()
    if args.out:
        json.dump(res, open(args.out, "w"), indent=1)


if __name__ == "__main__":
    main()
