"""The kernel-launch count the bench reports (`gpu_launches`) is what runs.

`mg_launches_per_cycle` is the steady-state count of one V-cycle; a call of
K cycles launches K times that, plus the finest descent of its first cycle
when the 2D cycles are fused.  Counted here with the CUDA
profiler (CUPTI sees the kernels of replayed CUDA graphs).
"""
import numpy as np
import pytest
import torch

from paper_math_9907190_b200 import workloads as W
from paper_math_9907190_b200.mg import Solver

pytestmark = pytest.mark.gpu


def _count(dim, n, dtype, cycles):
    p = (1.052,) if dim == 2 else (1.11, 1.42, 1.08, 0.99)
    npdt = np.float64 if dtype == torch.float64 else np.float32
    s = Solver(dim, n, order=2, p=p, dtype=dtype)
    u = s.alloc((W.random_field(dim, n, seed=8) * 0.1).astype(npdt))
    f = s.alloc(W.random_field(dim, n, seed=7).astype(npdt))
    s.vcycle(u, f, cycles)   # capture the graphs outside the profiled region
    torch.cuda.synchronize()
    with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
        s.vcycle(u, f, cycles)
        torch.cuda.synchronize()
    names = [e.name for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
    kernels = [x for x in names if "emcpy" not in x and "emset" not in x]
    return len(kernels), s.launches_per_cycle, kernels


@pytest.mark.parametrize("dim,n,dtype", [(2, 1025, torch.float64), (2, 2049, torch.float32), (3, 129, torch.float64)])
def test_launch_count_matches_claim(dim, n, dtype):
    cycles = 4
    got, lpc, kernels = _count(dim, n, dtype, cycles)
    fused = dim == 2
    want = cycles * lpc + (1 if fused else 0)
    assert got == want, (got, want, sorted(set(kernels)))
