"""SURVEY 8(f) NEXT-2 on the GPU: the two-stage fourth-order solve (P:330-334,
P:753-756) -- order-2 V-cycles, then order-4 V-cycles on the same
u -- against the oracle running the same two stages (bit for bit), and its
fourth-order accuracy on a smooth manufactured problem."""
import numpy as np
import pytest

import oracle
from paper_math_9907190_b200 import workloads as W

pytestmark = pytest.mark.gpu

P = {(2, 2): 1.052, (2, 4): 1.20, (3, 2): (1.11, 1.42, 1.08, 0.99), (3, 4): (0.91, 0.80, 0.70, 1.77)}


def _oracle_two_stage(dim, n, f, n2, n4):
    u = np.zeros_like(f)
    h2 = oracle.vcycle(u, f, P[(dim, 2)], n2, order=2, hist=True)
    h4 = oracle.vcycle(u, f, P[(dim, 4)], n4, order=4, hist=True)
    return u, h2, h4


@pytest.mark.parametrize("dim,n", [(2, 65), (2, 257), (3, 17), (3, 65)])
def test_two_stage_bit_identical_to_oracle(dim, n):
    import torch
    from paper_math_9907190_b200.twostage import two_stage
    f = W.smooth_rhs(dim, n) + W.random_field(dim, n, seed=9) * 0.01
    u, (h2, h4) = two_stage(dim, n, f, 5, 4, dtype=torch.float64)
    uo, h2o, h4o = _oracle_two_stage(dim, n, f, 5, 4)
    assert np.array_equal(u, uo)
    assert np.array_equal(h2, h2o) and np.array_equal(h4, h4o)


@pytest.mark.parametrize("dim,ns", [(2, (65, 129, 257)), (3, (17, 33, 65))])
def test_two_stage_is_fourth_order(dim, ns):
    """Max error against u* = prod sin(pi x) falls ~16x per halving of h after
    the two stages (8 + 6 cycles); order-2 cycles alone give ~4x."""
    import torch
    from paper_math_9907190_b200.twostage import two_stage
    e4, e2 = [], []
    for n in ns:
        f = W.smooth_rhs(dim, n)
        ustar = W.manufactured_u(dim, n)
        u, _ = two_stage(dim, n, f, 8, 6, dtype=torch.float64)
        e4.append(np.max(np.abs(u - ustar)))
        u2, _ = two_stage(dim, n, f, 14, 0, dtype=torch.float64)
        e2.append(np.max(np.abs(u2 - ustar)))
    for a, b in zip(e4, e4[1:]):
        assert 13 < a / b < 19, e4
    for a, b in zip(e2, e2[1:]):
        assert 3.5 < a / b < 4.5, e2


def test_two_stage_needs_fewer_order4_cycles():
    """The point of the scheme: after the cheap order-2 stage, a
    few order-4 cycles reach the order-4 discretisation error, which order-4
    cycles alone from u = 0 need more of (rho 0.20 vs 0.05 per cycle)."""
    import torch
    from paper_math_9907190_b200.twostage import two_stage
    dim, n = 2, 257
    f = W.smooth_rhs(dim, n)
    ustar = W.manufactured_u(dim, n)
    uref, _ = two_stage(dim, n, f, 10, 20, dtype=torch.float64)
    target = 1.01 * np.max(np.abs(uref - ustar))

    def cycles_to_target(n2):
        for n4 in range(0, 30):
            u, _ = two_stage(dim, n, f, n2, n4, dtype=torch.float64)
            if np.max(np.abs(u - ustar)) <= target:
                return n4
        return 99
    n4_two_stage = cycles_to_target(8)
    n4_alone = cycles_to_target(0)
    assert n4_two_stage + 3 <= n4_alone, (n4_two_stage, n4_alone)   # oracle: 6 vs 11
