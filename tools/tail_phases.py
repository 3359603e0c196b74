#!/usr/bin/env python
"""Per-phase times of the 3D cooperative tail (MG_TAIL_DEBUG=1; the un-graphed
per-step profile path prints CTA 0's globaltimer stamps)."""
import os
import sys

import numpy as np
import torch

os.environ["MG_TAIL_DEBUG"] = "1"
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_math_9907190_b200 import workloads as W  # noqa: E402
from paper_math_9907190_b200.mg import Solver  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 513
s = Solver(3, n, order=2, dtype=torch.float64)
u, f = s.alloc(), s.alloc(W.random_field(3, n, seed=1))
for _ in range(3):
    s.profile(u, f, 1)
torch.cuda.synchronize()
