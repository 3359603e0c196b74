"""Parity at sizes beyond BASELINE.json's configs: the largest grids of each
dimension that one B200 and the test host hold comfortably (2D 16385^2 fp64:
2.1 GB per field; 3D 1025^3 fp32: 4.3 GB per field, 1.08e9 nodes, so every
element offset and plane stride exceeds what 32-bit arithmetic would carry
once multiplied by the element size).  Both compared with the oracle bit for
bit, residual histories included.
"""
import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu


def _field(dim, n, seed, dtype):
    """U[-1, 1) on the interior, zero boundary, generated directly in `dtype`
    (the fp64 generator of workloads.random_field would need 8.6 GB at 1025^3)."""
    rng = np.random.default_rng(seed)
    a = rng.random((n,) * dim, dtype=dtype)
    a *= 2
    a -= 1
    for ax in range(dim):
        idx = [slice(None)] * dim
        idx[ax] = 0
        a[tuple(idx)] = 0
        idx[ax] = n - 1
        a[tuple(idx)] = 0
    return a


def _run(dim, n, p, dtype, cycles):
    import torch
    from paper_math_9907190_b200.mg import Solver
    f = _field(dim, n, 51 + dim, dtype)
    uo = np.zeros_like(f)
    ho = oracle.vcycle(uo, f, p, cycles, order=2, hist=True)
    s = Solver(dim, n, order=2, p=p, dtype=torch.float64 if dtype == np.float64 else torch.float32)
    u = s.alloc()
    ft = s.alloc(f)
    del f
    hg = s.vcycle(u, ft, cycles, hist=True)
    ug = s.view(u).cpu().numpy()
    return ug, hg, uo, ho


def test_parity_2d_16385_f64():
    ug, hg, uo, ho = _run(2, 16385, (1.052,), np.float64, 2)
    assert np.array_equal(ug, uo)
    assert np.array_equal(hg, ho)
    assert ho[-1] < 0.2 * ho[0]


def test_parity_3d_1025_f32():
    ug, hg, uo, ho = _run(3, 1025, (1.11, 1.42, 1.08, 0.99), np.float32, 1)
    assert np.array_equal(ug, uo)
    assert np.array_equal(hg, ho)
    assert ho[-1] < 0.2 * ho[0]


def test_parity_3d_1025_f64():
    """8.6 GB per field: byte offsets beyond 2^33."""
    ug, hg, uo, ho = _run(3, 1025, (1.11, 1.42, 1.08, 0.99), np.float64, 1)
    assert np.array_equal(ug, uo)
    assert np.array_equal(hg, ho)
    assert ho[-1] < 0.2 * ho[0]
