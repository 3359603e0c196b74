"""compute-sanitizer over every kernel family of libmg (race and
memory checking of the hand-written async pipelines).

Opt-in: set MG_SANITIZE to ONE tool (memcheck, racecheck, synccheck or
initcheck).  The B200 profiling recipe allows one sanitizer tool per GPU
session (several tools in one session have left a B200 unusable), so the
default `pytest -m gpu` run skips this file.  On the pool this repository is
built on, compute-sanitizer is closed altogether (its first run answered
"closed on this pool": profiles/r2_sanitizer_closed.txt); the bounds checks of
our own (MG_POISON guard bands, tests/test_gpu_paths.py) and the bit-exact
oracle comparisons stand in for it there.

The child program runs small cases of every path: the 2D TMA tile pipelines
(desc, rest_dad, jac_ad, single-CTA coarse), the cross-cycle fused
warp-streaming pass (fp64 pair and fp32 quad strips) and the plain ascent,
the 3D plane pipelines (k3p, k3s) and the cooperative tail, the order-4
kernels (k3f), the reference kernels, the conventional multigrid, the
extra-sweeps variant, the loopback slab solvers and the staging of pitch = n
caller arrays.
"""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
TOOL = os.environ.get("MG_SANITIZE", "")

CHILD = r"""
import sys
sys.path.insert(0, {root!r})
import numpy as np
import torch
from paper_math_9907190_b200 import workloads as W
from paper_math_9907190_b200 import mg
from paper_math_9907190_b200.mg import Solver
P3 = (1.11, 1.42, 1.08, 0.99)
def run(dim, n, order=2, dtype=torch.float64, cycles=3, hist=True, **kw):
    p = ((1.052 if order == 2 else 1.20),) if dim == 2 else P3
    s = Solver(dim, n, order=order, p=p, dtype=dtype, **kw)
    npdt = np.float64 if dtype == torch.float64 else np.float32
    u = s.alloc((0.1 * W.random_field(dim, n, seed=2)).astype(npdt))
    f = s.alloc(W.random_field(dim, n, seed=1).astype(npdt))
    s.vcycle(u, f, cycles, hist=hist)
    s.vcycle(u, f, 1)
    s.residual(u, f)
    torch.cuda.synchronize()
for dt in (torch.float64, torch.float32):
    run(2, 129, dtype=dt)
    run(2, 129, dtype=dt, hist=False)
    run(2, 65, order=4, dtype=dt)
    run(3, 65, dtype=dt)
    run(3, 33, order=4, dtype=dt)
run(2, 33, conventional=True)
run(3, 17, conventional=True)
run(2, 33, sweeps=2)
run(2, 65, nranks=2, loopback=True)
run(3, 33, nranks=2, loopback=True)
h = mg.mg_create(2, 65, 2, 1.052)
u = torch.zeros((65, 65), dtype=torch.float64, device="cuda")
f = torch.from_numpy(W.random_field(2, 65, seed=3)).cuda()
mg.mg_vcycle(h, u.data_ptr(), f.data_ptr(), 3, True)
mg.mg_destroy(h)
torch.cuda.synchronize()
print("SANITIZE-CHILD-OK")
"""


@pytest.mark.skipif(TOOL not in ("memcheck", "racecheck", "synccheck", "initcheck"),
                    reason="opt-in: MG_SANITIZE=<one compute-sanitizer tool>")
def test_compute_sanitizer_clean():
    exe = "/usr/local/cuda/bin/compute-sanitizer"
    code = CHILD.format(root=ROOT)
    cmd = [exe, "--tool", TOOL, "--error-exitcode", "99", "--print-limit", "50"]
    if TOOL == "racecheck":
        cmd += ["--racecheck-report", "all"]
    out = subprocess.run(cmd + [sys.executable, "-c", code], capture_output=True, text=True, timeout=3000)
    log = out.stdout + out.stderr
    dest = os.environ.get("MG_SANITIZE_LOG")
    if dest:
        with open(dest, "w") as fh:
            fh.write(log)
    assert "SANITIZE-CHILD-OK" in log, log[-4000:]
    assert out.returncode == 0, log[-4000:]
    assert "ERROR SUMMARY: 0 errors" in log, log[-4000:]
