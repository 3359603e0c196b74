"""SURVEY 8(f) NEXT-1 on the GPU: the convergence factor rho-bar by power
iteration (mg_convergence_factor) against the oracle's power iteration (same
start vector, same iteration; only the order of the L2 sums differs) and the
paper's Tables 1-3, and Nelder-Mead tuning of p against the paper's optimum."""
import os

import numpy as np
import pytest

import oracle
from paper_math_9907190_b200 import workloads as W

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _rows():
    out = []
    for line in open(os.path.join(ROOT, "tests", "golden", "paper_tables.txt")):
        line = line.split("#")[0].split()
        if line:
            out.append(line)
    return out


def _p(dim, txt):
    v = [float(t) for t in txt.split(",")]
    return v[0] if dim == 2 else tuple(v)


@pytest.mark.parametrize("row", _rows(), ids=lambda r: "-".join(r[:4]))
def test_rate_matches_oracle_and_paper(row):
    import torch
    from paper_math_9907190_b200 import rates
    dim, n, order = int(row[0]), int(row[1]), int(row[2])
    p, want, tol = _p(dim, row[3]), float(row[4]), float(row[5])
    iters = 200
    rho, ratios = rates.convergence_factor(dim, n, p, order, iters, torch.float64, seed=3)
    e = W.random_field(dim, n, seed=3)
    rho_o, ratios_o = oracle.convergence_factor(e, p, iters, order=order)
    np.testing.assert_allclose(ratios, ratios_o, rtol=1e-9)
    assert rho == pytest.approx(rho_o, rel=1e-9)
    assert rho == pytest.approx(want, abs=tol)


def test_rate_fp32_close_to_fp64():
    import torch
    from paper_math_9907190_b200 import rates
    r64, _ = rates.convergence_factor(2, 129, 1.052, 2, 150, torch.float64)
    r32, _ = rates.convergence_factor(2, 129, 1.052, 2, 150, torch.float32)
    assert r32 == pytest.approx(r64, rel=0.02)


def test_rate_is_grid_independent():
    """The paper's premise: rho-bar of the tuned 2D scheme does not grow with
    n (Table 1 is at 65^2; here up to 1025^2)."""
    import torch
    from paper_math_9907190_b200 import rates
    r = [rates.convergence_factor(2, n, 1.052, 2, 150, torch.float64)[0] for n in (65, 257, 1025)]
    assert max(r) < 0.06, r


def test_tuning_finds_the_papers_optimum():
    """Nelder-Mead from p = 1 on 2D 65^2 order 2 lands on the paper's
    p = 1.052 with rho-bar = 0.052 (Table 1)."""
    import torch
    from paper_math_9907190_b200 import rates
    res = rates.tune(2, 65, 2, [1.0], iters=120, dtype=torch.float64)
    assert res["p"][0] == pytest.approx(1.052, abs=0.01)
    assert res["rho"] == pytest.approx(0.052, abs=0.003)


def test_rate_rejects_bad_arguments():
    import torch
    from paper_math_9907190_b200.mg import MGError, Solver
    s = Solver(2, 33, dtype=torch.float64)
    e = s.alloc(W.random_field(2, 33, seed=1))
    with pytest.raises(MGError):
        s.convergence_factor(e, 1)
