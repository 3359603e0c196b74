"""SURVEY 8(f) NEXT-3 on the GPU: the paper's "usual" V(0,1) multigrid
(MG_FLAG_CONVENTIONAL, conv.cu) bit-identical to oracle/conventional.py, and
its convergence factors against the "usual" rows of Tables 1-3."""
import os

import numpy as np
import pytest

from oracle import conventional as C
from paper_math_9907190_b200 import workloads as W

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _solver(dim, n, order, p, dtype):
    import torch
    from paper_math_9907190_b200.mg import Solver
    return Solver(dim, n, order=order, p=p, dtype=torch.float64 if dtype == np.float64 else torch.float32,
                  conventional=True)


@pytest.mark.parametrize("dtype", [np.float64, np.float32], ids=["f64", "f32"])
@pytest.mark.parametrize("dim,n,order,p", [(2, 17, 2, 1.0), (2, 65, 2, 1.121), (2, 257, 4, 1.216), (2, 129, 2, 1.0),
                                           (3, 9, 2, 1.0), (3, 33, 2, 1.30), (3, 33, 4, 1.70), (3, 65, 2, 1.30)])
def test_conventional_bit_identical_to_oracle(dim, n, order, p, dtype):
    f = W.random_field(dim, n, seed=n).astype(dtype)
    u0 = (W.random_field(dim, n, seed=n + 1) * 0.1).astype(dtype)
    s = _solver(dim, n, order, p, dtype)
    u = s.alloc(u0)
    ft = s.alloc(f)
    h = s.vcycle(u, ft, 3, hist=True)
    ug = s.view(u).cpu().numpy()
    uo = u0.copy()
    ho = C.vcycle(uo, f, p, 3, order=order, hist=True)
    assert np.array_equal(ug, uo), float(np.max(np.abs(ug.astype(np.float64) - uo)))
    np.testing.assert_array_equal(h, ho)


def _rows():
    out = []
    for line in open(os.path.join(ROOT, "tests", "golden", "paper_tables_usual.txt")):
        line = line.split("#")[0].split()
        if line:
            out.append(line)
    return out


@pytest.mark.parametrize("row", _rows(), ids=lambda r: "-".join(r[:4]))
def test_conventional_rate_matches_oracle_and_paper(row):
    dim, n, order, p = int(row[0]), int(row[1]), int(row[2]), float(row[3])
    want, tol = float(row[4]), float(row[5])
    s = _solver(dim, n, order, p, np.float64)
    e = s.alloc(W.random_field(dim, n, seed=3))
    rho, ratios = s.convergence_factor(e, 200)
    rho_o, ratios_o = C.convergence_factor(W.random_field(dim, n, seed=3), p, 200, order)
    np.testing.assert_allclose(ratios, ratios_o, rtol=1e-9)
    assert rho == pytest.approx(want, abs=tol)


def test_conventional_solves_the_manufactured_problem():
    """Fifteen cycles reach the order-2 discrete solution of u* (the same
    fixed point as the diagonal scheme: both solve L_h u = f)."""
    import torch
    from paper_math_9907190_b200.mg import Solver
    dim, n = 2, 257
    f = W.smooth_rhs(dim, n)
    sc = _solver(dim, n, 2, 1.121, np.float64)
    sd = Solver(dim, n, order=2, p=1.052, dtype=torch.float64)
    uc, ud = sc.alloc(), sd.alloc()
    sc.vcycle(uc, sc.alloc(f), 40)
    sd.vcycle(ud, sd.alloc(f), 15)
    np.testing.assert_allclose(sc.view(uc).cpu().numpy(), sd.view(ud).cpu().numpy(), atol=1e-12)
