"""Seeded synthetic right-hand sides (BASELINE.json ``configs``).

Pure numpy input generation shared by the tests, the bench and users.  It
holds none of the V-cycle's arithmetic: only the problem data of
``nabla^2 u = f`` on the unit square / cube with homogeneous
Dirichlet data (reading A1).  Every array is generated in float64 with
``numpy.random.default_rng(seed)`` (PCG64) in the draw order stated below and
cast once to the requested dtype, so the oracle and the GPU path receive
bit-identical inputs.

Layout: C order, 2D ``(n, n)`` indexed ``[j, i]``, 3D ``(n, n, n)`` indexed
``[k, j, i]``; x = i h is the fastest index, h = 1/(n-1).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass(frozen=True)
class Workload:
    name: str
    dim: int
    n: int
    order: int
    p: tuple
    cycles: int
    seed: int
    kind: str  # "manufactured" | "uniform" | "bumps"
    note: str


P2 = (1.052,)                      # Table 1 optimum, order 2
P2_ORDER4 = (1.20,)                # order 4
P3 = (1.11, 1.42, 1.08, 0.99)      # Table 3

WORKLOADS = {
    # BASELINE.json configs[0..4]
    "2d_65": Workload("2d_65", 2, 65, 2, P2, 10, 1, "manufactured",
                      "f = L5 u* + 1e-3 U[-1,1], u* = sin(pi x) sin(pi y)"),
    "2d_1025": Workload("2d_1025", 2, 1025, 2, P2, 20, 2, "uniform", "f ~ U[-1,1] interior"),
    "2d_1025_o4": Workload("2d_1025_o4", 2, 1025, 4, P2_ORDER4, 20, 2, "uniform",
                           "f ~ U[-1,1] interior, Mehrstellen residual"),
    "2d_8193": Workload("2d_8193", 2, 8193, 2, P2, 10, 3, "bumps", "16 seeded Gaussian bumps"),
    "3d_65": Workload("3d_65", 3, 65, 2, P3, 10, 4, "manufactured",
                      "f = L7 u* + 1e-3 U[-1,1], u* = sin(pi x) sin(pi y) sin(pi z)"),
    "3d_513": Workload("3d_513", 3, 513, 2, P3, 10, 5, "uniform", "f ~ U[-1,1] interior"),
    # beyond BASELINE.json: the next size up of configs[2] / configs[4] (same recipes), to show how the
    # cycle's small-level latency share falls with the problem size
    "2d_16385": Workload("2d_16385", 2, 16385, 2, P2, 10, 6, "bumps", "16 seeded Gaussian bumps"),
    "3d_1025": Workload("3d_1025", 3, 1025, 2, P3, 10, 7, "uniform", "f ~ U[-1,1] interior"),
}


def _interior(dim):
    return (slice(1, -1),) * dim


def _coords(dim, n):
    x = np.linspace(0.0, 1.0, n)
    return x


def manufactured_u(dim: int, n: int) -> np.ndarray:
    """u* = prod_d sin(pi x_d) at every node (0 on the boundary up to rounding; forced to 0)."""
    s = np.sin(np.pi * _coords(dim, n))
    s[0] = 0.0
    s[-1] = 0.0
    if dim == 2:
        return np.multiply.outer(s, s)
    return np.multiply.outer(np.multiply.outer(s, s), s)


def discrete_laplacian(u: np.ndarray) -> np.ndarray:
    """Problem data only: the 5-/7-point Laplacian of a given u* at interior nodes,
    used to manufacture f = L_h u* (BASELINE configs[0], configs[3])."""
    dim, n = u.ndim, u.shape[0]
    inv_h2 = float((n - 1) ** 2)
    out = np.zeros_like(u)
    c = _interior(dim)
    acc = -2.0 * dim * u[c]
    for ax in range(dim):
        lo = list(c)
        hi = list(c)
        lo[ax] = slice(0, -2)
        hi[ax] = slice(2, None)
        acc = acc + u[tuple(lo)] + u[tuple(hi)]
    out[c] = acc * inv_h2
    return out


def smooth_rhs(dim: int, n: int) -> np.ndarray:
    """Problem data for accuracy studies: f = continuous Laplacian of
    u* = prod sin(pi x_d), i.e. -dim pi^2 u*, at every node (0 on the boundary)."""
    return -dim * np.pi ** 2 * manufactured_u(dim, n)


def make_rhs(dim: int, n: int, kind: str, seed: int, noise: float = 1e-3) -> np.ndarray:
    """Right-hand side f (float64)."""
    rng = np.random.default_rng(seed)
    f = np.zeros((n,) * dim, dtype=np.float64)
    c = _interior(dim)
    if kind == "manufactured":
        f = discrete_laplacian(manufactured_u(dim, n))
        f[c] += noise * rng.uniform(-1.0, 1.0, size=(n - 2,) * dim)
    elif kind == "uniform":
        f[c] = rng.uniform(-1.0, 1.0, size=(n - 2,) * dim)
    elif kind == "bumps":
        if dim != 2:
            raise ValueError("bumps are a 2D workload")
        centres = rng.uniform(0.1, 0.9, size=(16, 2))
        widths = rng.uniform(0.01, 0.1, size=16)
        amps = rng.normal(0.0, 1.0, size=16)
        x = _coords(dim, n)
        for (cx, cy), w, a in zip(centres, widths, amps):
            ex = np.exp(-((x - cx) ** 2) / (2 * w * w))
            ey = np.exp(-((x - cy) ** 2) / (2 * w * w))
            f += a * np.multiply.outer(ey, ex)   # row j (y), column i (x)
    elif kind == "zero":
        pass
    else:
        raise ValueError(kind)
    return f


def workload_rhs(name: str, dtype=np.float64) -> np.ndarray:
    w = WORKLOADS[name]
    return make_rhs(w.dim, w.n, w.kind, w.seed).astype(dtype)


def random_field(dim: int, n: int, seed: int, dtype=np.float64, boundary_zero: bool = True) -> np.ndarray:
    rng = np.random.default_rng(seed)
    a = rng.uniform(-1.0, 1.0, size=(n,) * dim)
    if boundary_zero:
        b = np.zeros_like(a)
        b[_interior(dim)] = a[_interior(dim)]
        a = b
    return a.astype(dtype)
