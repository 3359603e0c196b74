"""Independent exact references for pinning the oracle (test infrastructure).

Nothing here calls the oracle.  The discrete Dirichlet operators of the paper
are diagonalised by the DST-I (a library routine, ``scipy.fft.dstn``); their
eigenvalues are the textbook symbols of the stencils:

* 5-point / 7-point Laplacian: (sum_d 2 cos t_d - 2 d) / h^2
* Mehrstellen 9-point, Efos2:
      (1/(6h^2)) (-20 + 4 (2cx + 2cy) + 4 cx cy),   f-weight (8 + 2cx + 2cy)/12
* 19-point, Efos4:
      (1/(6h^2)) (-24 + 2 (2cx+2cy+2cz) + 4 (cx cy + cy cz + cx cz)),
      f-weight (6 + 2cx + 2cy + 2cz)/12
with t_j = pi j h, j = 1..n-2.
"""
from __future__ import annotations

import numpy as np
import scipy.fft as sfft


def _cos(n):
    j = np.arange(1, n - 1)
    return np.cos(np.pi * j / (n - 1))


def symbols(dim: int, n: int, order: int):
    """(lambda, mu): operator and f-weight symbols on the DST-I grid."""
    h2 = 1.0 / (n - 1) ** 2
    c = _cos(n)
    cs = np.meshgrid(*([c] * dim), indexing="ij")  # axis 0 = slowest (k or j)
    if order == 2:
        lam = (sum(2 * ci for ci in cs) - 2 * dim) / h2
        mu = np.ones_like(lam)
    elif dim == 2:
        cy, cx = cs
        lam = (-20 + 4 * (2 * cx + 2 * cy) + 4 * cx * cy) / (6 * h2)
        mu = (8 + 2 * cx + 2 * cy) / 12
    else:
        cz, cy, cx = cs
        lam = (-24 + 2 * (2 * cx + 2 * cy + 2 * cz) + 4 * (cx * cy + cy * cz + cx * cz)) / (6 * h2)
        mu = (6 + 2 * cx + 2 * cy + 2 * cz) / 12
    return lam, mu


def exact_solution(f: np.ndarray, order: int = 2) -> np.ndarray:
    """Exact discrete solution of L u = f (order 2) or L u = f~ (order 4)
    with homogeneous Dirichlet data; ``f`` must vanish on the boundary."""
    dim, n = f.ndim, f.shape[0]
    inner = (slice(1, -1),) * dim
    lam, mu = symbols(dim, n, order)
    fh = sfft.dstn(f[inner].astype(np.float64), type=1, norm="ortho")
    u = np.zeros(f.shape, dtype=np.float64)
    u[inner] = sfft.idstn(fh * mu / lam, type=1, norm="ortho")
    return u


def apply_operator(u: np.ndarray, order: int = 2) -> np.ndarray:
    """L u (order 2) or L u for the Mehrstellen operator, spectrally (u = 0 on boundary)."""
    dim, n = u.ndim, u.shape[0]
    inner = (slice(1, -1),) * dim
    lam, _ = symbols(dim, n, order)
    out = np.zeros(u.shape)
    out[inner] = sfft.idstn(sfft.dstn(u[inner], type=1, norm="ortho") * lam, type=1, norm="ortho")
    return out


def dense_laplacian(dim: int, n: int) -> np.ndarray:
    """Textbook Kronecker-sum 5-/7-point Dirichlet Laplacian on the (n-2)^dim interior."""
    m = n - 2
    T = (np.diag(-2.0 * np.ones(m)) + np.diag(np.ones(m - 1), 1) + np.diag(np.ones(m - 1), -1)) * (n - 1) ** 2
    I = np.eye(m)
    if dim == 2:
        return np.kron(I, T) + np.kron(T, I)
    return np.kron(np.kron(I, I), T) + np.kron(np.kron(I, T), I) + np.kron(np.kron(T, I), I)


def grid(dim: int, n: int):
    x = np.linspace(0.0, 1.0, n)
    return np.meshgrid(*([x] * dim), indexing="ij")[::-1]  # returns (x, y[, z]) with x fastest
