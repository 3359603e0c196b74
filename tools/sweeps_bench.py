#!/usr/bin/env python
"""SURVEY 8(f) NEXT-4 measurement: the paper's open question -- "the effect
of extra Jacobi iterations at each level of the diagonal grid" --
on one B200.  For 2D 8193^2 (order 2 and 4) and nu = 1, 2, 3 two-colour steps
per level: p tuned by Nelder-Mead at 1025^2 (GPU power iterations), rho-bar
at 8193^2, ms per cycle (all nu on the same plain kernels; nu = 1 also on the
production path), time per digit.  One JSON document.

    python tools/sweeps_bench.py > profiles/r1_sweeps.json
"""
import json
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402
from paper_math_9907190_b200 import rates  # noqa: E402
from paper_math_9907190_b200 import workloads as W  # noqa: E402
from paper_math_9907190_b200.mg import Solver  # noqa: E402


def cycle_ms(s, f, cycles=20):
    u = s.alloc()
    s.vcycle(u, f, 3)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    s.vcycle(u, f, cycles)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / cycles


def main():
    out = {"device": torch.cuda.get_device_name(0), "runs": []}
    n = 8193
    for order in (2, 4):
        for nu in (1, 2, 3):
            t = rates.tune(2, 1025, order, [1.0], iters=100, dtype=torch.float64, sweeps=nu)
            p = t["p"][0]
            if nu == 1:
                os.environ["MG_FORCE_REF"] = "1"   # nu = 1 on the same plain kernels
            s = Solver(2, n, order=order, p=p, dtype=torch.float64, sweeps=nu)
            os.environ.pop("MG_FORCE_REF", None)
            f = s.alloc(W.random_field(2, n, seed=5))
            ms = cycle_ms(s, f)
            e = s.alloc(W.random_field(2, n, seed=3))
            rho, _ = s.convergence_factor(e, 80)
            run = dict(order=order, sweeps=nu, p_tuned_1025=p, rho_1025=t["rho"], rho_8193=rho,
                       ms_per_cycle_plain=ms, ms_per_digit_plain=ms / -math.log10(rho))
            if nu == 1:
                sf = Solver(2, n, order=order, p=p, dtype=torch.float64)
                msf = cycle_ms(sf, sf.alloc(W.random_field(2, n, seed=5)))
                run.update(ms_per_cycle_production=msf, ms_per_digit_production=msf / -math.log10(rho))
                del sf
            out["runs"].append(run)
            del s
            torch.cuda.empty_cache()
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
