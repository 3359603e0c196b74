#!/usr/bin/env python
"""SURVEY 8(f) NEXT-1 measurement: rho-bar on the GPU (mg_convergence_factor)
for the paper's Tables 1-3 and at the BASELINE sizes, Nelder-Mead tuning of
the relaxation parameters, each timed; the oracle's power iteration timed
beside it at the paper's sizes.  Writes one JSON document.

    python tools/rates_bench.py > profiles/r1_rates.json
"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402  (test infrastructure: the timed CPU baseline)
import torch  # noqa: E402
from paper_math_9907190_b200 import rates  # noqa: E402
from paper_math_9907190_b200 import workloads as W  # noqa: E402
from paper_math_9907190_b200.mg import Solver  # noqa: E402


def timed(fn):
    torch.cuda.synchronize()
    t = time.perf_counter()
    out = fn()
    torch.cuda.synchronize()
    return out, time.perf_counter() - t


def main():
    out = {"tables": [], "large": [], "tuning": [], "device": torch.cuda.get_device_name(0)}
    rows = []
    for line in open(os.path.join(ROOT, "tests", "golden", "paper_tables.txt")):
        line = line.split("#")[0].split()
        if line:
            rows.append(line)
    for r in rows:
        dim, n, order = int(r[0]), int(r[1]), int(r[2])
        pv = [float(t) for t in r[3].split(",")]
        p = pv[0] if dim == 2 else tuple(pv)
        s = Solver(dim, n, order=order, p=p, dtype=torch.float64)
        rates.convergence_factor(dim, n, p, order, 20, solver=s)   # graph capture, warm-up
        (rho, _), tg = timed(lambda: rates.convergence_factor(dim, n, p, order, 200, solver=s))
        t = time.perf_counter()
        rho_o, _ = oracle.convergence_factor(W.random_field(dim, n, seed=3), p, 200, order=order)
        to = time.perf_counter() - t
        out["tables"].append(dict(dim=dim, n=n, order=order, p=pv, rho_gpu=rho, rho_oracle=rho_o,
                                  rho_paper=float(r[4]), window=float(r[5]), iters=200, gpu_s=tg,
                                  oracle_s=to, oracle_cores=1))
    for dim, n, order, p in [(2, 8193, 2, 1.052), (2, 8193, 4, 1.20), (2, 8193, 2, 1.0),
                             (3, 513, 2, (1.11, 1.42, 1.08, 0.99)), (3, 513, 2, (1.0, 1.0, 1.0, 1.0)),
                             (3, 257, 4, (0.91, 0.80, 0.70, 1.77))]:
        s = Solver(dim, n, order=order, p=p, dtype=torch.float64)
        rates.convergence_factor(dim, n, p, order, 5, solver=s)
        (rho, ratios), tg = timed(lambda: rates.convergence_factor(dim, n, p, order, 150, solver=s))
        out["large"].append(dict(dim=dim, n=n, order=order, p=list(p) if dim == 3 else [p], rho_gpu=rho,
                                 last_ratios=[float(x) for x in ratios[-4:]], iters=150, gpu_s=tg))
        del s
        torch.cuda.empty_cache()
    for dim, n, order, p0 in [(2, 65, 2, [1.0]), (2, 65, 4, [1.0]), (2, 1025, 2, [1.0]),
                              (3, 17, 2, [1.0] * 4), (3, 33, 2, [1.0] * 4), (3, 65, 2, [1.0] * 4),
                              (3, 17, 4, [1.0] * 4)]:
        res, tt = timed(lambda: rates.tune(dim, n, order, p0, iters=120, dtype=torch.float64, maxfev=300))
        res.update(dim=dim, n=n, order=order, p0=p0, seconds=tt)
        out["tuning"].append(res)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
