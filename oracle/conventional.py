"""Oracle of the "usual" multigrid the paper compares against (SURVEY 8(f)
NEXT-3, SPEC module `baseline`): TEST INFRASTRUCTURE ONLY (same import rules
as the package: tests/, smoke() and bench.py's reference leg).

V(0,1) cycle on the standard hierarchy (factor-2 coarsening, n_l = (n-1)/2^l
+ 1 down to 3 nodes per side):
  descent  r_0 = f - L u (oracle.residual, order 2 or 4); r_{l+1} = full
           weighting of r_l: 9-point (1/16)(4c + 2 sum axis + sum diag)
           ("conventional nine point restriction operator", P:187-190;
           11 flops), 27-point (1/64)(8c + 4 faces + 2 edges + corners) in 3D
           (P:534-538);
  coarsest one Jacobi step from zero: v = (1/4)(-p H^2 r) (2D), (1/6)(...) (3D)
           (reading A4);
  ascent   v_l = bi/trilinear interpolation of v_{l+1} ("the simplest
           (bilinear) conventional interpolation direct", P:240-247;
           trilinear P:674-680), then one two-colour Jacobi sweep (nu1 = 0,
           nu2 = 1; reading A18): v = (1/4)(-p h_l^2 r_l + sum of the 4 axis
           neighbours) (2D), (1/6)(... 6 ...) (3D), colour 1 (i+j[+k] odd)
           from the interpolated field, colour 2 from colour 1 --
           over-relaxation on the residual term only, as in Eq. (7);
  finest   the same with r_0 recomputed, then u <- u + v_0.
Plain numpy in the field's precision; every sum is evaluated left to right in
the order written (the CUDA kernels follow the same order).
"""
from __future__ import annotations

import numpy as np

from . import residual as _residual


def _t(a, x):
    return a.dtype.type(x)


def restrict_fw(r: np.ndarray) -> np.ndarray:
    """Full weighting onto the next coarser level (interior coarse nodes)."""
    dim, n = r.ndim, r.shape[0]
    nc = (n - 1) // 2 + 1
    rc = np.zeros((nc,) * dim, dtype=r.dtype)
    if nc < 3:
        return rc
    m = nc - 2

    def s(*off):   # fine values at (2X+ox, 2Y+oy[, 2Z+oz]) for interior coarse X, Y[, Z]
        sl = tuple(slice(2 + o, 2 + o + 2 * m - 1, 2) for o in off[::-1])
        return r[sl]
    if dim == 2:
        c = s(0, 0)
        ax = s(-1, 0) + s(1, 0)
        ax = ax + s(0, -1)
        ax = ax + s(0, 1)
        dg = s(-1, -1) + s(1, -1)
        dg = dg + s(1, 1)
        dg = dg + s(-1, 1)
        t = _t(r, 4) * c
        t = t + _t(r, 2) * ax
        t = t + dg
        rc[1:-1, 1:-1] = t * _t(r, 0.0625)
    else:
        faces = [(-1, 0, 0), (1, 0, 0), (0, -1, 0), (0, 1, 0), (0, 0, -1), (0, 0, 1)]
        edges = [(-1, -1, 0), (1, -1, 0), (1, 1, 0), (-1, 1, 0), (-1, 0, -1), (1, 0, -1), (1, 0, 1), (-1, 0, 1),
                 (0, -1, -1), (0, 1, -1), (0, 1, 1), (0, -1, 1)]
        corners = [(-1, -1, -1), (1, -1, -1), (1, 1, -1), (-1, 1, -1), (-1, -1, 1), (1, -1, 1), (1, 1, 1),
                   (-1, 1, 1)]

        def acc(offs):
            a = s(*offs[0])
            for o in offs[1:]:
                a = a + s(*o)
            return a
        t = _t(r, 8) * s(0, 0, 0)
        t = t + _t(r, 4) * acc(faces)
        t = t + _t(r, 2) * acc(edges)
        t = t + acc(corners)
        rc[1:-1, 1:-1, 1:-1] = t * _t(r, 1.0 / 64.0)
    return rc


def interpolate(vc: np.ndarray, n: int) -> np.ndarray:
    """Bi/trilinear interpolation of a coarse level onto the fine level of n
    nodes per side: coincident nodes copy, edge midpoints average 2, face
    centres 4, cell centres 8 (summed in increasing x, then y, then z)."""
    dim = vc.ndim
    v = np.zeros((n,) * dim, dtype=vc.dtype)
    half = _t(vc, 0.5)
    quarter = _t(vc, 0.25)
    eighth = _t(vc, 0.125)
    if dim == 2:
        a = vc[:-1, :-1]   # (Y, X)
        b = vc[:-1, 1:]    # (Y, X+1)
        c = vc[1:, :-1]    # (Y+1, X)
        d = vc[1:, 1:]
        v[0::2, 0::2] = vc
        v[0::2, 1::2] = (vc[:, :-1] + vc[:, 1:]) * half
        v[1::2, 0::2] = (vc[:-1, :] + vc[1:, :]) * half
        t = a + b
        t = t + c
        t = t + d
        v[1::2, 1::2] = t * quarter
    else:
        v[0::2, 0::2, 0::2] = vc
        v[0::2, 0::2, 1::2] = (vc[:, :, :-1] + vc[:, :, 1:]) * half
        v[0::2, 1::2, 0::2] = (vc[:, :-1, :] + vc[:, 1:, :]) * half
        v[1::2, 0::2, 0::2] = (vc[:-1, :, :] + vc[1:, :, :]) * half
        # face centres: (x, y odd, z even), (x odd, z odd, y even), (y odd, z odd, x even)
        t = vc[:, :-1, :-1] + vc[:, :-1, 1:]
        t = t + vc[:, 1:, :-1]
        t = t + vc[:, 1:, 1:]
        v[0::2, 1::2, 1::2] = t * quarter
        t = vc[:-1, :, :-1] + vc[:-1, :, 1:]
        t = t + vc[1:, :, :-1]
        t = t + vc[1:, :, 1:]
        v[1::2, 0::2, 1::2] = t * quarter
        t = vc[:-1, :-1, :] + vc[:-1, 1:, :]
        t = t + vc[1:, :-1, :]
        t = t + vc[1:, 1:, :]
        v[1::2, 1::2, 0::2] = t * quarter
        t = vc[:-1, :-1, :-1] + vc[:-1, :-1, 1:]
        t = t + vc[:-1, 1:, :-1]
        t = t + vc[:-1, 1:, 1:]
        t = t + vc[1:, :-1, :-1]
        t = t + vc[1:, :-1, 1:]
        t = t + vc[1:, 1:, :-1]
        t = t + vc[1:, 1:, 1:]
        v[1::2, 1::2, 1::2] = t * eighth
    return v


def _sweep(src: np.ndarray, r: np.ndarray, c) -> np.ndarray:
    """Jacobi values on the interior from the field src:
    (-(c r) + w + s + e + n [+ down + up]) / (2 dim), c = p h_l^2
    (neighbour order x-1, y-1, x+1, y+1[, z-1, z+1] as jac4 / jac6)."""
    dim = src.ndim
    w = np.zeros_like(src)
    c = _t(src, c)
    if dim == 2:
        i = (slice(1, -1), slice(1, -1))
        t = -(c * r[i])
        t = t + src[1:-1, :-2]
        t = t + src[:-2, 1:-1]
        t = t + src[1:-1, 2:]
        t = t + src[2:, 1:-1]
        w[i] = t * _t(src, 0.25)
    else:
        i = (slice(1, -1),) * 3
        t = -(c * r[i])
        t = t + src[1:-1, 1:-1, :-2]
        t = t + src[1:-1, :-2, 1:-1]
        t = t + src[1:-1, 1:-1, 2:]
        t = t + src[1:-1, 2:, 1:-1]
        t = t + src[:-2, 1:-1, 1:-1]
        t = t + src[2:, 1:-1, 1:-1]
        w[i] = t * _t(src, 1.0 / 6.0)
    return w


def jacobi(vi: np.ndarray, r: np.ndarray, c) -> np.ndarray:
    """One two-colour (red-black) Jacobi sweep on the interior (reading A18 of
    DESIGN.md): colour 1, the nodes with i+j[+k] odd (none of them on the
    coarser grid), from the interpolated field vi; colour 2, i+j[+k] even,
    from colour 1's new values.  The same two-colour form as the diagonal
    scheme's Jacobi prolongation.  (A one-colour sweep leaves the
    (pi, pi) mode undamped, rho = |1 - 2p|, and cannot give the paper's
    0.340.)"""
    dim = vi.ndim
    par = np.indices(vi.shape).sum(axis=0) & 1
    inner = np.zeros(vi.shape, dtype=bool)
    inner[(slice(1, -1),) * dim] = True
    v = vi.copy()
    w = _sweep(v, r, c)
    m1 = inner & (par == 1)
    v[m1] = w[m1]
    w = _sweep(v, r, c)
    m2 = inner & (par == 0)
    v[m2] = w[m2]
    v[~inner] = 0
    return v


def vcycle(u: np.ndarray, f: np.ndarray, p: float, ncycles: int, order: int = 2, hist: bool = False):
    """ncycles V(0,1) cycles in place on u; with hist the L-inf residual norms
    before every cycle and after the last (as oracle.vcycle)."""
    dim, n = u.ndim, u.shape[0]
    p = float(p)
    hs = []
    for _ in range(ncycles):
        rs = [_residual(u, f, order)]
        hs.append(float(np.max(np.abs(rs[0]))))
        while rs[-1].shape[0] > 3:
            rs.append(restrict_fw(rs[-1]))
        L = len(rs) - 1
        ncoarse = rs[L].shape[0]
        H = 1.0 / (ncoarse - 1)
        v = np.zeros_like(rs[L])
        cc = _t(u, p * H * H)
        if dim == 2:
            v[1, 1] = (-(cc * rs[L][1, 1])) * _t(u, 0.25)
        else:
            v[1, 1, 1] = (-(cc * rs[L][1, 1, 1])) * _t(u, 1.0 / 6.0)
        for lev in range(L - 1, -1, -1):
            nl = rs[lev].shape[0]
            h = 1.0 / (nl - 1)
            v = jacobi(interpolate(v, nl), rs[lev], p * h * h)
        u += v
    if hist:
        hs.append(float(np.max(np.abs(_residual(u, f, order)))))
        return np.array(hs)
    return None


def convergence_factor(e: np.ndarray, p: float, iters: int, order: int = 2):
    """Power iteration as oracle.convergence_factor, on this scheme."""
    f = np.zeros_like(e)
    nrm = float(np.sqrt(np.sum(e.astype(np.float64) ** 2)))
    e[...] = e * e.dtype.type(1.0 / nrm)
    ratios = np.empty(iters)
    for k in range(iters):
        vcycle(e, f, p, 1, order=order)
        nrm = float(np.sqrt(np.sum(e.astype(np.float64) ** 2)))
        ratios[k] = nrm
        e[...] = e * e.dtype.type(1.0 / nrm)
    tail = ratios[iters // 2:]
    return float(np.exp(np.mean(np.log(tail)))), ratios
