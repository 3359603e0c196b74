"""CPU oracle for Roberts' diagonal multigrid V-cycle (arXiv math/9907190).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` leg may import this
package.  The product path (``paper_math_9907190_b200``) never imports it and
shares no code with it.

The arithmetic lives in ``oracle/oracle.c`` (plain single-threaded C, built
with ``-O2 -ffp-contract=off``, once per precision).  This module is ctypes
marshalling only.  Arrays are numpy C-order: 2D ``(n, n)`` indexed ``[j, i]``,
3D ``(n, n, n)`` indexed ``[k, j, i]`` (x fastest).  Levels are stored on the
lattice of their octave: shape ``(m+1,)*dim`` with
``m = lattice(dim, n, lev)``.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_FLAGS = ["-O2", "-std=c11", "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-shared"]


def _lib_path(tag: str) -> str:
    return os.path.join(_HERE, f"liboracle_{tag}.so")


def build(force: bool = False) -> None:
    """Compile the oracle for f64 and f32 (gcc)."""
    for tag, real in (("f64", "double"), ("f32", "float")):
        out = _lib_path(tag)
        if not force and os.path.exists(out) and os.path.getmtime(out) >= os.path.getmtime(_SRC):
            continue
        subprocess.check_call(["gcc", *_FLAGS, f"-DREAL={real}", _SRC, "-o", out, "-lm"])


_LIBS: dict = {}


def _lib(dtype):
    dtype = np.dtype(dtype)
    tag = {np.dtype(np.float64): "f64", np.dtype(np.float32): "f32"}[dtype]
    if tag not in _LIBS:
        build()
        lib = ctypes.CDLL(_lib_path(tag))
        P = ctypes.c_void_p
        L = ctypes.c_long
        I = ctypes.c_int
        D = ctypes.POINTER(ctypes.c_double)
        for name, res, args in [
            ("orc_levels", I, [I, L]),
            ("orc_lattice", L, [I, L, I]),
            ("orc_count", L, [I, L, I]),
            ("orc_ftilde", I, [I, L, P, P]),
            ("orc_residual", I, [I, L, I, P, P, P]),
            ("orc_restrict", I, [I, L, I, P, P]),
            ("orc_jacobi", I, [I, L, I, D, P, P, P]),
            ("orc_coarsest", I, [I, L, D, P, P]),
            ("orc_norm_inf", ctypes.c_double, [I, L, P]),
            ("orc_vcycle", I, [I, L, I, D, P, P, I, D]),
            ("orc_vcycle_sweeps", I, [I, L, I, D, P, P, I, D, I]),
            ("orc_real_size", I, []),
        ]:
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        assert lib.orc_real_size() == dtype.itemsize
        _LIBS[tag] = lib
    return _LIBS[tag]


def _ptr(a: np.ndarray):
    assert a.flags.c_contiguous
    return a.ctypes.data_as(ctypes.c_void_p)


def _params(dim: int, p) -> ctypes.Array:
    if dim == 2:
        vals = [float(p if np.isscalar(p) else p[0])] + [0.0] * 3
    else:
        vals = [float(x) for x in (p if not np.isscalar(p) else (p, p, p, p))]
        assert len(vals) == 4
    return (ctypes.c_double * 4)(*vals)


def levels(dim: int, n: int) -> int:
    return _lib(np.float64).orc_levels(dim, n)


def lattice(dim: int, n: int, lev: int) -> int:
    return _lib(np.float64).orc_lattice(dim, n, lev)


def count(dim: int, n: int, lev: int) -> int:
    return _lib(np.float64).orc_count(dim, n, lev)


def level_shape(dim: int, n: int, lev: int):
    m = lattice(dim, n, lev)
    return (m + 1,) * dim


def ftilde(f: np.ndarray) -> np.ndarray:
    dim, n = f.ndim, f.shape[0]
    out = np.zeros_like(f)
    assert _lib(f.dtype).orc_ftilde(dim, n, _ptr(f), _ptr(out)) == 0
    return out


def residual(u: np.ndarray, f: np.ndarray, order: int = 2) -> np.ndarray:
    dim, n = u.ndim, u.shape[0]
    assert u.dtype == f.dtype and u.shape == f.shape
    r = np.zeros_like(u)
    assert _lib(u.dtype).orc_residual(dim, n, order, _ptr(u), _ptr(f), _ptr(r)) == 0
    return r


def restrict(dim: int, n: int, lev: int, rin: np.ndarray) -> np.ndarray:
    rin = np.ascontiguousarray(rin)
    assert rin.shape == level_shape(dim, n, lev)
    out = np.zeros(level_shape(dim, n, lev + 1), dtype=rin.dtype)
    assert _lib(rin.dtype).orc_restrict(dim, n, lev, _ptr(rin), _ptr(out)) == 0
    return out


def jacobi(dim: int, n: int, lev: int, p, vc: np.ndarray, r: np.ndarray) -> np.ndarray:
    vc = np.ascontiguousarray(vc)
    r = np.ascontiguousarray(r)
    assert vc.shape == level_shape(dim, n, lev + 1) and r.shape == level_shape(dim, n, lev)
    v = np.zeros_like(r)
    pp = _params(dim, p)
    assert _lib(r.dtype).orc_jacobi(dim, n, lev, pp, _ptr(vc), _ptr(r), _ptr(v)) == 0
    return v


def coarsest(dim: int, n: int, p, r: np.ndarray) -> np.ndarray:
    r = np.ascontiguousarray(r)
    v = np.zeros_like(r)
    assert _lib(r.dtype).orc_coarsest(dim, n, _params(dim, p), _ptr(r), _ptr(v)) == 0
    return v


def norm_inf(x: np.ndarray) -> float:
    return _lib(x.dtype).orc_norm_inf(x.ndim, x.shape[0], _ptr(np.ascontiguousarray(x)))


def vcycle(u: np.ndarray, f: np.ndarray, p, ncycles: int, order: int = 2, hist: bool = False, sweeps: int = 1):
    """Run ``ncycles`` V-cycles in place on ``u``; return the L-inf residual
    history (ncycles+1 values) if ``hist``.  ``sweeps`` > 1 (2D): that many
    two-colour Jacobi steps on every level (reading A19
    of DESIGN.md)."""
    dim, n = u.ndim, u.shape[0]
    assert u.dtype == f.dtype and u.shape == f.shape and u.flags.c_contiguous
    f = np.ascontiguousarray(f)
    h = (ctypes.c_double * (ncycles + 1))() if hist else None
    rc = _lib(u.dtype).orc_vcycle_sweeps(dim, n, order, _params(dim, p), _ptr(u), _ptr(f), ncycles,
                                         h if hist else None, sweeps)
    if rc != 0:
        raise RuntimeError(f"orc_vcycle failed rc={rc}")
    return np.array(list(h)) if hist else None


def convergence_factor(e: np.ndarray, p, iters: int, order: int = 2, sweeps: int = 1):
    """The paper's convergence factor rho-bar, "the largest eigenvalue" of the
    V-cycle iteration operator (reading A12: spectral radius), by
    power iteration on the error equation (f = 0): normalise e (L2 over all
    nodes; the boundary is zero), then ``iters`` times: one V-cycle of e with
    f = 0, ratio_k = ||e||_2, e <- e * (1 / ratio_k) (the factor formed in
    fp64, the product in e's precision).  Returns (rho, ratios), rho = the
    geometric mean of the ratios of the second half.  In place on e."""
    f = np.zeros_like(e)
    nrm = float(np.sqrt(np.sum(e.astype(np.float64) ** 2)))
    e[...] = e * e.dtype.type(1.0 / nrm)
    ratios = np.empty(iters)
    for k in range(iters):
        vcycle(e, f, p, 1, order=order, sweeps=sweeps)
        nrm = float(np.sqrt(np.sum(e.astype(np.float64) ** 2)))
        ratios[k] = nrm
        e[...] = e * e.dtype.type(1.0 / nrm)
    tail = ratios[iters // 2:]
    return float(np.exp(np.mean(np.log(tail)))), ratios
