#!/usr/bin/env python
"""Interleaved sweep of library environment switches (one bench.py process per
arm and round; median ms per V-cycle per arm).

    python tools/sweep.py --workload 3d_513 "X=1" "MG_TAIL_GRID3=64" "MG_TAIL_GRID3=32"
"""
import argparse
import statistics

from ab import run


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("arms", nargs="+")
    ap.add_argument("--workload", default="3d_513")
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--rounds", type=int, default=3)
    ap.add_argument("--dtype", default="f64")
    args = ap.parse_args()
    res = {a: [] for a in args.arms}
    for _ in range(args.rounds):
        for arm in args.arms:
            ms, mhz = run(arm, args.workload, args.steps, args.dtype)
            res[arm].append(ms)
            print(f"[{arm}] {ms:.4f} ms  {mhz} MHz", flush=True)
    for arm, v in res.items():
        print(f"median [{arm}] {statistics.median(v):.4f} ms")


if __name__ == "__main__":
    main()
