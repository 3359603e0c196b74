#!/usr/bin/env python
"""SURVEY 8(f) NEXT-3 measurement: the paper's "twice as fast" claim (P:270-275,
Tables 1-3 "per dig" columns) as time per decimal digit of error reduction on
one B200 -- the diagonal V-cycle against the usual V(0,1) multigrid, each at
its tuned parameter, at the BASELINE sizes.  time/digit = (ms per V-cycle) /
(-log10 rho-bar), rho-bar by the GPU power iteration at that size.  One JSON
document.

    python tools/compare_bench.py > profiles/r2_compare.json
"""
import json
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402
from paper_math_9907190_b200 import workloads as W  # noqa: E402
from paper_math_9907190_b200.mg import Solver  # noqa: E402


def cycle_ms(s, f, cycles):
    u = s.alloc()
    s.vcycle(u, f, 5)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    ev0.record()
    s.vcycle(u, f, cycles)
    ev1.record()
    torch.cuda.synchronize()
    return ev0.elapsed_time(ev1) / cycles


def one(dim, n, order, p, conventional, cycles, iters):
    s = Solver(dim, n, order=order, p=p, dtype=torch.float64, conventional=conventional)
    f = s.alloc(W.random_field(dim, n, seed=5))
    ms = cycle_ms(s, f, cycles)
    e = s.alloc(W.random_field(dim, n, seed=3))
    rho, _ = s.convergence_factor(e, iters)
    prof = s.profile(s.alloc(), f, 3)
    alg = sum(r["alg_bytes"] for r in prof)
    N = (n - 2) ** dim
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] \
        if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6650.0
    out = dict(scheme="usual" if conventional else "diagonal", dim=dim, n=n, order=order,
               p=list(p) if isinstance(p, tuple) else [p], ms_per_cycle=ms, rho=rho,
               ms_per_digit=ms / -math.log10(rho), alg_bytes_per_cycle=alg,
               alg_bytes_per_digit_per_dof=alg / N / -math.log10(rho), launches_per_cycle=s.launches_per_cycle,
               # how close each implementation runs to the copy roofline on its own algorithmic bytes: the
               # time-per-digit ratio mixes the methods' cost with the two implementations' efficiency
               roofline_frac=alg / (ms * 1e-3) / 1e9 / peak)
    del s
    torch.cuda.empty_cache()
    return out


def main():
    runs = []
    for dim, n, order, pd, pu in [(2, 8193, 2, 1.052, 1.121), (2, 8193, 4, 1.20, 1.216),
                                  (3, 513, 2, (1.11, 1.42, 1.08, 0.99), 1.30),
                                  (3, 257, 4, (0.91, 0.80, 0.70, 1.77), 1.70)]:
        d = one(dim, n, order, pd, False, 50 if dim == 2 else 20, 100)
        u = one(dim, n, order, pu, True, 50 if dim == 2 else 20, 100)
        runs.append(dict(diagonal=d, usual=u, speedup_time_per_digit=u["ms_per_digit"] / d["ms_per_digit"],
                         # the implementation-independent part: bytes per digit (= the time-per-digit ratio if
                         # both ran at the same fraction of the roofline)
                         speedup_at_equal_roofline_frac=u["alg_bytes_per_digit_per_dof"] /
                         d["alg_bytes_per_digit_per_dof"]))
    print(json.dumps({"device": torch.cuda.get_device_name(0), "runs": runs}, indent=1))


if __name__ == "__main__":
    main()
