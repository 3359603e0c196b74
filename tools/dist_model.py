#!/usr/bin/env python
"""Multi-GPU efficiency model from one-GPU measurements.

On one B200 the slab solvers run their P ranks as virtual ranks (loopback):
every rank's kernels run one after another on the whole GPU, each on its own
slab -- exactly the work a rank does on its own GPU.  So, per V-cycle,

    T_loop(P) = P * T_dist(P) + T_shared + T_copies(P)

where T_shared is the redundant coarse part (levels >= the agglomeration
octave, run once in loopback, on every rank with NCCL), measured separately
from the single-GPU per-step profile.  The per-rank time on P GPUs is then

    T_rank(P) = T_dist(P) + T_shared + T_comm(P)

with T_comm modelled from the exchanges the schedule makes (stated latency
and bandwidth assumptions: no multi-GPU hardware is available to this
build), and the efficiency is T_1 / (P * T_rank(P)).

    python tools/dist_model.py [--out profiles/r2_dist_model.json]
"""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

LAT_P2P_US = 8.0      # assumed: one grouped NCCL send/recv round on NVLink 5 inside a CUDA graph
LAT_COLL_US = 12.0    # assumed: one small NCCL all-gather / all-reduce over 8 GPUs
BW_GBS = 770.0        # measured peer copy per direction (B200_PROFILING.md)


def time_cycles(s, u, f, cycles, reps=3):
    import torch
    s.vcycle(u, f, cycles)
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        s.vcycle(u, f, cycles)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) / cycles)
    return float(np.median(ts))


def agglom_octave(dim, n, P, ag=1 << 18):
    k = int(np.log2(n - 1))
    for o in range(1, k):
        M = (n - 1) >> o
        if (M - 1) ** dim < ag or M // P < 4:
            return o
    return k - 1


def main():
    import torch
    from paper_math_9907190_b200 import workloads as W
    from paper_math_9907190_b200.mg import Solver
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r2_dist_model.json"))
    ap.add_argument("--cycles", type=int, default=20)
    args = ap.parse_args()
    res = {"assumptions": {"p2p_round_us": LAT_P2P_US, "collective_us": LAT_COLL_US, "link_gbs": BW_GBS},
           "gpu": torch.cuda.get_device_name(0), "workloads": {}}
    for name in ("2d_8193", "3d_513"):
        w = W.WORKLOADS[name]
        f = W.workload_rhs(name)
        s1 = Solver(w.dim, w.n, order=w.order, p=w.p)
        u1, f1 = s1.alloc(), s1.alloc(f)
        t1 = time_cycles(s1, u1, f1, args.cycles)
        prof = s1.profile(u1, f1, 5)
        out = {"T1_ms": t1, "per_P": {}}
        for P in (2, 4, 8):
            oa = agglom_octave(w.dim, w.n, P)
            first_shared = 2 * oa if w.dim == 2 else 3 * oa
            t_shared = sum(r["ms"] for r in prof if r["level"] >= first_shared)
            sP = Solver(w.dim, w.n, order=w.order, p=w.p, nranks=P, loopback=True)
            uP, fP = sP.alloc(), sP.alloc(f)
            t_loop = time_cycles(sP, uP, fP, args.cycles)
            del sP, uP, fP
            torch.cuda.empty_cache()
            t_dist = max(t_loop - t_shared, 0.0) / P
            esz = 8
            row_b = w.n * esz if w.dim == 2 else w.n * w.n * esz
            R = (w.n - 1) // P
            if w.dim == 2:
                from paper_math_9907190_b200.mg import mg_slab_schedule
                gu = mg_slab_schedule(2, w.n, P)[1]
                rounds = 1                                   # one u exchange per cycle
                xbytes = gu * row_b * 2                      # both neighbours (concurrent)
                ag_bytes = (((w.n - 1) >> oa) + 1) * (((w.n - 1) >> oa) + 1) * esz
                sched = f"communication-avoiding: 1 u exchange of {gu} rows + 1 all-gather per cycle"
            else:
                gu = 2
                # dist3.cu: u (2 planes), f; per octave rest_gr (o >= 1), rest_rm, rest_mg on the way down,
                # v_G(2s) (below oa), v_M B, v_M C, v_R faces, v_R C, v_G (o >= 1) on the way up
                rounds = 2 + 3 * oa - 1 + 6 * oa - 2
                xbytes = 3 * row_b * 2 + (rounds - 2) * (row_b / 8) * 2   # finest planes + coarser-level halos
                ag_bytes = (((w.n - 1) >> oa) + 1) ** 3 * esz
                sched = f"per-level z-slab halos ({rounds} rounds) + 1 all-gather per cycle"
            t_comm = (rounds * LAT_P2P_US + LAT_COLL_US) * 1e-3 + (xbytes / 2 + ag_bytes) / (BW_GBS * 1e9) * 1e3
            t_rank = t_dist + t_shared + t_comm
            out["per_P"][P] = {"agglom_octave": oa, "rows_per_rank": R, "T_loop_ms": t_loop, "T_shared_ms": t_shared,
                               "T_dist_ms": t_dist, "T_comm_model_ms": t_comm, "T_rank_ms": t_rank,
                               "efficiency": t1 / (P * t_rank), "schedule": sched,
                               "efficiency_if_shared_free": t1 / (P * (t_dist + t_comm))}
            print(name, P, json.dumps(out["per_P"][P]), flush=True)
        res["workloads"][name] = out
        del s1, u1, f1
        torch.cuda.empty_cache()
    with open(args.out, "w") as fh:
        json.dump(res, fh, indent=1)


if __name__ == "__main__":
    main()
