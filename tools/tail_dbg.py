import os, sys
sys.path.insert(0, "/root/repo")
import torch
from paper_math_9907190_b200.mg import Solver
from paper_math_9907190_b200 import workloads as W
n = int(sys.argv[1]) if len(sys.argv) > 1 else 513
s = Solver(3, n, order=2, p=W.P3)
u = s.alloc(); f = s.alloc(W.random_field(3, n, seed=1))
s.vcycle(u, f, 3)
for r in s.profile(u, f, 3):
    print(r["name"], r["level"], round(r["ms"] * 1e3, 1))
