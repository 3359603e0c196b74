"""SURVEY 8(f) NEXT-4 on the GPU: extra two-colour Jacobi steps at every level
(the paper's open question; reading A19), bit-identical to the
oracle's variant, and what they do to the convergence factor."""
import numpy as np
import pytest

import oracle
from paper_math_9907190_b200 import workloads as W

pytestmark = pytest.mark.gpu


def _solver(n, order, p, dtype, sweeps):
    import torch
    from paper_math_9907190_b200.mg import Solver
    return Solver(2, n, order=order, p=p, dtype=torch.float64 if dtype == np.float64 else torch.float32,
                  sweeps=sweeps)


@pytest.mark.parametrize("dtype", [np.float64, np.float32], ids=["f64", "f32"])
@pytest.mark.parametrize("n,order,sweeps", [(17, 2, 2), (65, 2, 3), (257, 2, 2), (129, 4, 2), (65, 4, 3)])
def test_sweeps_bit_identical_to_oracle(n, order, sweeps, dtype):
    p = 1.052 if order == 2 else 1.20
    f = W.random_field(2, n, seed=n).astype(dtype)
    u0 = (W.random_field(2, n, seed=n + 1) * 0.1).astype(dtype)
    s = _solver(n, order, p, dtype, sweeps)
    u = s.alloc(u0)
    ft = s.alloc(f)
    h = s.vcycle(u, ft, 3, hist=True)
    uo = u0.copy()
    ho = oracle.vcycle(uo, f, p, 3, order=order, hist=True, sweeps=sweeps)
    assert np.array_equal(s.view(u).cpu().numpy(), uo)
    np.testing.assert_array_equal(h, ho)


def test_extra_sweeps_lower_the_rate_at_p1():
    """At p = 1 a second sweep per level cuts rho-bar from 0.099 to ~0.047
    (2D 65^2); GPU and oracle power iterations agree."""
    rates = []
    for sweeps in (1, 2):
        s = _solver(65, 2, 1.0, np.float64, sweeps)
        e = s.alloc(W.random_field(2, 65, seed=3))
        rho, ratios = s.convergence_factor(e, 150)
        rho_o, ratios_o = oracle.convergence_factor(W.random_field(2, 65, seed=3), 1.0, 150, sweeps=sweeps)
        np.testing.assert_allclose(ratios, ratios_o, rtol=1e-9)
        rates.append(rho)
    assert rates[0] == pytest.approx(0.099, abs=0.003)
    assert rates[1] < 0.6 * rates[0]


def test_sweeps_rejected_in_3d():
    import torch
    from paper_math_9907190_b200.mg import MGError, Solver
    with pytest.raises(MGError):
        Solver(3, 17, p=1.0, dtype=torch.float64, sweeps=2)
