"""Two-stage fourth-order solve.

"Fourth order accurate solutions to Poisson's equation are most quickly
obtained by initially using the diagonal multigrid method applied to the
second order accurate computation of residuals.  Then use a few multigrid
iterations based upon the fourth order residuals to refine the numerical
solution" (3D: P:753-756).

Stage 1: V-cycles with the 2nd-order residual (5-/7-point, a1 / a9) from
u = 0; stage 2: V-cycles with the 4th-order residual (Efos2 / Efos4, a1'),
on the same u and f.  Orchestration only: each stage is one mg_vcycle call
of a solver built for that order (the two solvers share the array layout);
no arithmetic of the method lives here.  Default relaxation parameters are
the paper's tuned values (Tables 1 and 3).
"""
from __future__ import annotations

import numpy as np

from .mg import Solver

P_DEFAULT = {(2, 2): 1.052, (2, 4): 1.20, (3, 2): (1.11, 1.42, 1.08, 0.99), (3, 4): (0.91, 0.80, 0.70, 1.77)}


class TwoStage:
    """A pair of solvers (order 2 and order 4) on one grid."""

    def __init__(self, dim: int, n: int, p2=None, p4=None, dtype=None):
        import torch
        dtype = dtype or torch.float64
        self.s2 = Solver(dim, n, order=2, p=p2 if p2 is not None else P_DEFAULT[(dim, 2)], dtype=dtype)
        self.s4 = Solver(dim, n, order=4, p=p4 if p4 is not None else P_DEFAULT[(dim, 4)], dtype=dtype)
        assert self.s2.shape == self.s4.shape

    def alloc(self, like=None):
        return self.s2.alloc(like)

    def view(self, t):
        return self.s2.view(t)

    def solve(self, u, f, n2: int, n4: int, hist: bool = False):
        """n2 order-2 cycles then n4 order-4 cycles, in place on u.  With hist:
        (order-2 residual history, order-4 residual history), L-inf norms
        before every cycle and after the last."""
        h2 = self.s2.vcycle(u, f, n2, hist=hist) if n2 > 0 else None
        h4 = self.s4.vcycle(u, f, n4, hist=hist) if n4 > 0 else None
        return (h2, h4) if hist else None


def two_stage(dim: int, n: int, f: np.ndarray, n2: int, n4: int, p2=None, p4=None, dtype=None):
    """Solve nabla^2 u = f (host array f, every node) by the two-stage scheme;
    returns (u as a host array, (h2, h4) residual histories)."""
    ts = TwoStage(dim, n, p2, p4, dtype)
    u = ts.alloc()
    ft = ts.alloc(f)
    h = ts.solve(u, ft, n2, n4, hist=True)
    return ts.view(u).cpu().numpy(), h
