"""Convergence-rate measurement and relaxation tuning on the GPU (SURVEY 8(f)
NEXT-1).

The paper measures each scheme by rho-bar, "the largest eigenvalue" of the
V-cycle iteration operator (Tables 1-3 at P:276-304, P:695-717,
P:770-798), and tunes the over-relaxation parameters for it (P:345-348,
P:800-811: "a 33^3 search was infeasible within one day").  Here rho-bar is
the power iteration of ``mg_convergence_factor`` (every step in the library's
kernels), and the tuning is a host-side Nelder-Mead over p (2D) or
(p_m, p_r1, p_r2, p_g) (3D) whose every function value is one GPU power
iteration.  Orchestration only: no arithmetic of the method lives here.
"""
from __future__ import annotations

import numpy as np

from . import workloads as W
from .mg import Solver


def convergence_factor(dim: int, n: int, p, order: int = 2, iters: int = 200, dtype=None, seed: int = 3,
                       solver: Solver | None = None, sweeps: int = 1):
    """rho-bar of the V-cycle with parameters p (and `sweeps` Jacobi steps
    per level, NEXT-4), from a seeded random start error; returns (rho, ratios)."""
    import torch
    dtype = dtype or torch.float64
    s = solver or Solver(dim, n, order=order, p=p, dtype=dtype, sweeps=sweeps)
    e = s.alloc(W.random_field(dim, n, seed=seed))
    return s.convergence_factor(e, iters)


def tune(dim: int, n: int, order: int = 2, p0=None, iters: int = 120, dtype=None, xatol: float = 2e-3,
         maxfev: int = 200, sweeps: int = 1):
    """Nelder-Mead over the relaxation parameters minimising rho-bar (P:345-348,
    P:800-811).  Returns dict(p=..., rho=..., nfev=...)."""
    from scipy.optimize import minimize

    if p0 is None:
        p0 = [1.0] if dim == 2 else [1.0, 1.0, 1.0, 1.0]
    cache = {}

    def f(x):
        x = np.clip(np.asarray(x, dtype=np.float64), 0.05, 3.0)
        key = tuple(np.round(x, 12))
        if key not in cache:
            p = float(x[0]) if dim == 2 else tuple(float(v) for v in x)
            cache[key] = convergence_factor(dim, n, p, order, iters, dtype, sweeps=sweeps)[0]
        return cache[key]

    simplex = None
    x0 = np.asarray(p0, dtype=np.float64)
    if dim == 2:
        simplex = np.array([x0, x0 + 0.1])
    res = minimize(f, x0, method="Nelder-Mead",
                   options=dict(xatol=xatol, fatol=1e-5, maxfev=maxfev, initial_simplex=simplex))
    x = np.clip(res.x, 0.05, 3.0)
    return dict(p=[float(v) for v in x], rho=float(res.fun), nfev=int(res.nfev))
