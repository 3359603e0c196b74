"""Pins of the conventional-multigrid oracle (oracle/conventional.py, SURVEY
8(f) NEXT-3): textbook properties of full weighting, bi/trilinear
interpolation and the Jacobi sweep, and the paper's convergence factors of
its "usual" scheme (Tables 1-3)."""
import os

import numpy as np
import pytest

from oracle import conventional as C
from paper_math_9907190_b200 import workloads as W

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _rows():
    out = []
    for line in open(os.path.join(ROOT, "tests", "golden", "paper_tables_usual.txt")):
        line = line.split("#")[0].split()
        if line:
            out.append(line)
    return out


@pytest.mark.parametrize("dim", [2, 3])
def test_full_weighting_preserves_constants(dim):
    n = 17 if dim == 2 else 9
    r = np.full((n,) * dim, 3.25)
    rc = C.restrict_fw(r)
    inner = (slice(1, -1),) * dim
    assert np.all(rc[inner] == 3.25)


def test_full_weighting_delta_2d():
    """SPEC baseline examples: a delta at a coarse-coincident node gives 1/4
    there; at a fine-only axis node 1/8 at its two coarse neighbours; at a
    cell centre 1/16 at its four."""
    n = 17
    r = np.zeros((n, n))
    r[8, 8] = 1.0
    rc = C.restrict_fw(r)
    assert rc[4, 4] == 0.25 and np.count_nonzero(rc) == 1
    r[:] = 0
    r[8, 9] = 1.0
    rc = C.restrict_fw(r)
    assert rc[4, 4] == 0.125 and rc[4, 5] == 0.125 and np.count_nonzero(rc) == 2
    r[:] = 0
    r[9, 9] = 1.0
    rc = C.restrict_fw(r)
    assert np.count_nonzero(rc) == 4 and np.all(rc[4:6, 4:6] == 0.0625)


def test_full_weighting_delta_3d():
    n = 9
    for off, w, cnt in [((0, 0, 0), 1 / 8, 1), ((0, 0, 1), 1 / 16, 2), ((0, 1, 1), 1 / 32, 4), ((1, 1, 1), 1 / 64, 8)]:
        r = np.zeros((n, n, n))
        r[4 + off[0], 4 + off[1], 4 + off[2]] = 1.0
        rc = C.restrict_fw(r)
        assert np.count_nonzero(rc) == cnt and np.all(rc[rc != 0] == w)


@pytest.mark.parametrize("dim", [2, 3])
def test_interpolation_hat_and_constants(dim):
    nc = 5
    vc = np.zeros((nc,) * dim)
    vc[(2,) * dim] = 1.0
    v = C.interpolate(vc, 2 * nc - 1)
    c = (4,) * dim
    assert v[c] == 1.0
    e = list(c)
    e[-1] += 1
    assert v[tuple(e)] == 0.5
    d = tuple(x + 1 for x in c)
    assert v[d] == 0.5 ** dim
    assert np.all(C.interpolate(np.full((nc,) * dim, 2.0), 2 * nc - 1) == 2.0)


@pytest.mark.parametrize("dim", [2, 3])
def test_jacobi_fixed_point_on_quadratics(dim):
    """The 5/7-point Laplacian is exact on quadratics: with r = L v* for
    v* = sum x^2 on the interior and v* as the start field on a domain whose
    boundary carries v*, one two-colour sweep at p = 1 returns v*."""
    n = 9
    x = np.linspace(0, 1, n)
    G = np.meshgrid(*([x] * dim), indexing="ij")
    v = np.sum([g ** 2 for g in G], axis=0)
    r = np.full_like(v, 2.0 * dim)
    h = 1.0 / (n - 1)
    out = C.jacobi(v, r, h * h)
    inner = (slice(1, -1),) * dim
    np.testing.assert_allclose(out[inner], v[inner], rtol=1e-13)


def test_cycle_is_linear():
    n = 33
    a, b = W.random_field(2, n, seed=1), W.random_field(2, n, seed=2)
    f = np.zeros_like(a)
    ua, ub, uab = a.copy(), b.copy(), (2 * a + 3 * b)
    for u in (ua, ub, uab):
        C.vcycle(u, f, 1.121, 1)
    np.testing.assert_allclose(uab, 2 * ua + 3 * ub, atol=1e-12)


def test_one_colour_jacobi_cannot_reach_the_paper():
    """Reading A18: with a one-colour sweep the (pi, pi) mode e maps to
    (1 - 2p) e every cycle (full weighting annihilates its residual), so rho
    >= |1 - 2p| = 1 at p = 1 against the paper's 0.340; the two-colour sweep
    turns it into a smooth mode that the next cycles remove."""
    n = 17
    e = np.zeros((n, n))
    i = np.indices((n, n)).sum(axis=0)
    e[1:-1, 1:-1] = np.where(i[1:-1, 1:-1] % 2 == 0, 1.0, -1.0)
    u = e.copy()
    C.vcycle(u, np.zeros_like(e), 1.0, 4)
    assert np.max(np.abs(u)) < 0.05
    # one-colour sweep: every interior value from the interpolated field
    h = 1.0 / (n - 1)
    r = -(np.roll(e, 1, 0) + np.roll(e, -1, 0) + np.roll(e, 1, 1) + np.roll(e, -1, 1) - 4 * e) / h ** 2
    rc = C.restrict_fw(r)
    assert np.max(np.abs(rc[2:-2, 2:-2])) == 0.0            # invisible to the coarse grids
    v1 = C._sweep(np.zeros_like(e), r, h * h)               # interpolated correction ~ 0 away from the boundary
    np.testing.assert_allclose((e + v1)[4:-4, 4:-4], -e[4:-4, 4:-4])   # (1 - 2p) e at p = 1


@pytest.mark.parametrize("row", _rows(), ids=lambda r: "-".join(r[:4]))
def test_usual_convergence_factor_matches_paper(row):
    dim, n, order, p = int(row[0]), int(row[1]), int(row[2]), float(row[3])
    want, tol = float(row[4]), float(row[5])
    rho, _ = C.convergence_factor(W.random_field(dim, n, seed=3), p, 200, order)
    assert rho == pytest.approx(want, abs=tol)
