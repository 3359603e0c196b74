#!/usr/bin/env python
"""SURVEY 8(f) NEXT-2 measurement: time to a fourth-order accurate solution on
the GPU, two-stage (order-2 cycles, then order-4 cycles) against
order-4 cycles alone, on u* = prod sin(pi x) at the BASELINE sizes; the
oracle timed on the same schedule at a small size.  One JSON document.

    python tools/twostage_bench.py > profiles/r1_twostage.json
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
from paper_math_9907190_b200 import workloads as W  # noqa: E402
from paper_math_9907190_b200.twostage import P_DEFAULT, TwoStage  # noqa: E402


def err(ts, u, ustar_t):
    return float((ts.view(u) - ustar_t).abs().max())


def study(dim, n):
    ts = TwoStage(dim, n, dtype=torch.float64)
    f = ts.alloc(W.smooth_rhs(dim, n))
    ustar_t = torch.as_tensor(W.manufactured_u(dim, n), device="cuda")
    u = ts.alloc()
    ts.solve(u, f, 10, 25)
    e_disc = err(ts, u, ustar_t)
    target = 1.01 * e_disc

    def n4_needed(n2):
        for n4 in range(0, 60):
            u.zero_()
            ts.solve(u, f, n2, n4)
            if err(ts, u, ustar_t) <= target:
                return n4
        return None
    best = None
    for n2 in range(0, 16):
        n4 = n4_needed(n2)
        if n4 is None:
            continue
        cand = (n2, n4)
        if best is None or cand[1] < best[1] or (cand[1] == best[1] and cand[0] < best[0]):
            best = cand
        if n4 <= 2:
            break
    alone = n4_needed(0)

    def timed(n2, n4, reps=5):
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        u.zero_()
        ts.solve(u, f, n2, n4)   # graphs captured
        ts_ = []
        for _ in range(reps):
            u.zero_()
            torch.cuda.synchronize()
            ev0.record()
            ts.solve(u, f, n2, n4)
            ev1.record()
            torch.cuda.synchronize()
            ts_.append(ev0.elapsed_time(ev1))
        return float(np.median(ts_))
    t_two = timed(*best)
    t_alone = timed(0, alone)
    t2 = timed(20, 0) / 20
    t4 = timed(0, 20) / 20
    return dict(dim=dim, n=n, e_disc=e_disc, target=target, two_stage=dict(n2=best[0], n4=best[1], ms=t_two),
                order4_alone=dict(n4=alone, ms=t_alone), ms_per_cycle_order2=t2, ms_per_cycle_order4=t4,
                p2=P_DEFAULT[(dim, 2)], p4=P_DEFAULT[(dim, 4)])


def oracle_time(dim, n, n2, n4):
    f = W.smooth_rhs(dim, n)
    u = np.zeros_like(f)
    t = time.perf_counter()
    oracle.vcycle(u, f, P_DEFAULT[(dim, 2)], n2, order=2)
    oracle.vcycle(u, f, P_DEFAULT[(dim, 4)], n4, order=4)
    return time.perf_counter() - t


def main():
    out = {"device": torch.cuda.get_device_name(0), "runs": []}
    for dim, n in [(2, 1025), (2, 8193), (3, 129), (3, 513)]:
        r = study(dim, n)
        if (dim == 2 and n == 1025) or (dim == 3 and n == 129):
            r["oracle_s_same_schedule"] = oracle_time(dim, n, r["two_stage"]["n2"], r["two_stage"]["n4"])
            r["oracle_cores"] = 1
        out["runs"].append(r)
        torch.cuda.empty_cache()
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
