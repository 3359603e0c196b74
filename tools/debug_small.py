import sys, os, numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_math_9907190_b200.mg import Solver
from paper_math_9907190_b200 import workloads as W
n = int(sys.argv[1]) if len(sys.argv) > 1 else 5
s = Solver(2, n, order=2, p=1.052, dtype=torch.float64)
f = W.random_field(2, n, seed=1)
u, ft = s.alloc(), s.alloc(f)
try:
    print(s.profile(u, ft, 1))
except Exception as e:
    print("EXC", e)
