"""The per-cycle L2 residual norm (||r_0||_{2,h} =
(h^d sum r_0^2)^(1/2)) fused into the finest-residual passes:
equal, to the rounding of a reordered sum, to the norm of the oracle's
residual of the oracle's iterates, cycle by cycle, on every code path."""
import numpy as np
import pytest

import oracle
from paper_math_9907190_b200 import workloads as W

pytestmark = pytest.mark.gpu

P3 = (1.11, 1.42, 1.08, 0.99)


def _oracle_norms(dim, n, order, p, f, u0, cycles, dtype, conventional=False):
    u = u0.astype(dtype).copy()
    f = f.astype(dtype)
    inner = (slice(1, -1),) * dim
    hd = (1.0 / (n - 1)) ** dim
    l2 = []
    for c in range(cycles + 1):
        r = oracle.residual(u, f, order)
        l2.append(np.sqrt(hd * np.sum(r[inner].astype(np.float64) ** 2)))
        if c < cycles:
            if conventional:
                from oracle import conventional as CV
                CV.vcycle(u, f, p, 1, order=order)
            else:
                oracle.vcycle(u, f, p, 1, order=order)
    return np.array(l2)


@pytest.mark.parametrize("dim,n,order,dtype,kw", [
    (2, 257, 2, np.float64, {}), (2, 257, 4, np.float64, {}), (2, 513, 2, np.float32, {}),
    (2, 129, 4, np.float32, {}), (3, 65, 2, np.float64, {}), (3, 33, 4, np.float64, {}),
    (3, 65, 2, np.float32, {}), (2, 65, 2, np.float64, {"nranks": 2, "loopback": True}),
    (2, 1025, 2, np.float64, {"nranks": 4, "loopback": True, "agglom_points": 1 << 12}),
    (3, 65, 2, np.float64, {"nranks": 4, "loopback": True}),
])
def test_l2_history_matches_oracle(dim, n, order, dtype, kw):
    import torch
    from paper_math_9907190_b200.mg import Solver
    p = ((1.052 if order == 2 else 1.20),) if dim == 2 else P3
    f = W.random_field(dim, n, seed=61).astype(dtype)
    u0 = (0.1 * W.random_field(dim, n, seed=62)).astype(dtype)
    s = Solver(dim, n, order=order, p=p, dtype=torch.float64 if dtype == np.float64 else torch.float32, **kw)
    u, ft = s.alloc(u0), s.alloc(f)
    hinf, hl2 = s.vcycle(u, ft, 4, l2=True)
    want = _oracle_norms(dim, n, order, p, f, u0, 4, dtype)
    np.testing.assert_allclose(hl2, want, rtol=1e-10)
    ho = oracle.vcycle(u0.astype(dtype).copy(), f, p, 4, order=order, hist=True)
    assert np.array_equal(hinf, ho)


def test_l2_history_conventional_and_sweeps():
    import torch
    from paper_math_9907190_b200.mg import Solver
    n = 65
    f = W.random_field(2, n, seed=63)
    s = Solver(2, n, order=2, p=1.052, sweeps=2)
    u, ft = s.alloc(), s.alloc(f)
    _, hl2 = s.vcycle(u, ft, 3, l2=True)
    uo = np.zeros_like(f)
    want = []
    for c in range(4):
        r = oracle.residual(uo, f, 2)
        want.append(np.sqrt((1.0 / (n - 1)) ** 2 * np.sum(r[1:-1, 1:-1] ** 2)))
        if c < 3:
            oracle.vcycle(uo, f, 1.052, 1, sweeps=2)
    np.testing.assert_allclose(hl2, want, rtol=1e-10)
    sc = Solver(2, n, order=2, p=1.0, conventional=True)
    u, ft = sc.alloc(), sc.alloc(f)
    hinf, hl2 = sc.vcycle(u, ft, 3, l2=True)
    assert np.all(np.isfinite(hl2)) and hl2[-1] < hl2[0]
    torch.cuda.synchronize()
