#!/usr/bin/env python
"""Interleaved A/B timing of two library configurations on the GPU box.

    python tools/ab.py "MG_K3_FUSE=1" "X=1" --workload 3d_513 --steps 100 --rounds 4

Each round runs bench.py once per arm (the library reads its switches from the
environment once per process, so every run is a fresh process) and prints
ms_per_step and the median SM clock of the timed region; the summary line
gives the median per arm.  Interleaving the arms cancels most of the drift of
a power-capped B200 (about +-1.5 % run to run on the 3D workload).
"""
import argparse
import json
import os
import statistics
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def run(env_kv, workload, steps, dtype):
    env = dict(os.environ)
    for kv in env_kv.split():
        k, v = kv.split("=", 1)
        env[k] = v
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--workload", workload, "--steps",
                          str(steps), "--warmup", "5", "--no-cpu", "--no-e2e", "--no-sub", "--dtype", dtype], env=env, capture_output=True,
                         text=True, timeout=900)
    d = json.loads(out.stdout.strip().splitlines()[-1])
    return d["ms_per_step"], d["clocks"]["sm_mhz"]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("a")
    ap.add_argument("b")
    ap.add_argument("--workload", default="3d_513")
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--rounds", type=int, default=4)
    ap.add_argument("--dtype", default="f64")
    args = ap.parse_args()
    res = {args.a: [], args.b: []}
    for _ in range(args.rounds):
        for arm in (args.a, args.b):
            ms, mhz = run(arm, args.workload, args.steps, args.dtype)
            res[arm].append(ms)
            print(f"[{arm}] {ms:.4f} ms  {mhz} MHz", flush=True)
    for arm, v in res.items():
        print(f"median [{arm}] {statistics.median(v):.4f} ms")


if __name__ == "__main__":
    main()
