"""Parity of the CUDA path (through the C ABI) with the CPU oracle.

Both sides evaluate every formula in the canonical order of DESIGN.md without
FMA contraction, so the iterates are expected to be bit-identical; the
tolerances written below are the north-star bars (fp64 relative L-inf
<= 1e-11 after 10 cycles; fp32 <= 1e-5) and the bitwise check is asserted
separately.
"""
import numpy as np
import pytest

import oracle
from paper_math_9907190_b200 import workloads as W

pytestmark = pytest.mark.gpu

P2 = 1.052
P2_4 = 1.20
P3 = (1.11, 1.42, 1.08, 0.99)


def _solver(dim, n, order, p, dtype, pitch=None):
    import torch
    from paper_math_9907190_b200.mg import Solver
    tdt = torch.float64 if dtype == np.float64 else torch.float32
    return Solver(dim, n, order=order, p=p, dtype=tdt, pitch=pitch)


def _gpu_run(dim, n, order, p, f, u0, cycles, dtype, pitch=None, hist=True):
    s = _solver(dim, n, order, p, dtype, pitch)
    u = s.alloc(u0)
    ft = s.alloc(f)
    h = s.vcycle(u, ft, cycles, hist=hist)
    out = s.view(u).cpu().numpy().copy()
    return out, h


def _oracle_run(dim, n, order, p, f, u0, cycles, dtype):
    u = u0.astype(dtype).copy()
    h = oracle.vcycle(u, f.astype(dtype), p, cycles, order=order, hist=True)
    return u, h


def _rel(a, b):
    return float(np.max(np.abs(a.astype(np.float64) - b.astype(np.float64))) / max(np.max(np.abs(b)), 1e-300))


CASES_2D = [(n, o) for n in (5, 9, 17, 33, 65, 129, 257) for o in (2, 4)]
CASES_3D = [(n, o) for n in (5, 9, 17, 33, 129, 257) for o in (2, 4)]


@pytest.mark.parametrize("dtype", [np.float64, np.float32], ids=["f64", "f32"])
@pytest.mark.parametrize("n,order", CASES_2D)
def test_parity_2d_small(n, order, dtype):
    p = P2 if order == 2 else P2_4
    f = W.random_field(2, n, seed=n)
    u0 = W.random_field(2, n, seed=n + 1) * 0.1
    ug, hg = _gpu_run(2, n, order, p, f.astype(dtype), u0.astype(dtype), 4, dtype)
    uo, ho = _oracle_run(2, n, order, p, f, u0, 4, dtype)
    tol = 1e-11 if dtype == np.float64 else 1e-5
    assert _rel(ug, uo) <= tol
    assert np.array_equal(ug, uo), f"not bitwise: rel {_rel(ug, uo):.3e}"
    assert np.array_equal(hg, ho)


@pytest.mark.parametrize("dtype", [np.float64, np.float32], ids=["f64", "f32"])
@pytest.mark.parametrize("n,order", CASES_3D)
def test_parity_3d_small(n, order, dtype):
    p = P3
    f = W.random_field(3, n, seed=n)
    u0 = W.random_field(3, n, seed=n + 1) * 0.1
    ug, hg = _gpu_run(3, n, order, p, f.astype(dtype), u0.astype(dtype), 3, dtype)
    uo, ho = _oracle_run(3, n, order, p, f, u0, 3, dtype)
    tol = 1e-11 if dtype == np.float64 else 1e-5
    assert _rel(ug, uo) <= tol
    assert np.array_equal(ug, uo), f"not bitwise: rel {_rel(ug, uo):.3e}"
    assert np.array_equal(hg, ho)


@pytest.mark.parametrize("name", ["2d_65", "2d_1025", "2d_1025_o4", "3d_65"])
@pytest.mark.parametrize("dtype", [np.float64, np.float32], ids=["f64", "f32"])
def test_parity_workloads(name, dtype):
    """BASELINE.json configs[0], [1] (both orders) and [3], at their cycle counts."""
    w = W.WORKLOADS[name]
    f = W.workload_rhs(name, dtype)
    u0 = np.zeros_like(f)
    ug, hg = _gpu_run(w.dim, w.n, w.order, w.p, f, u0, w.cycles, dtype)
    uo, ho = _oracle_run(w.dim, w.n, w.order, w.p, f, u0, w.cycles, dtype)
    tol = 1e-11 if dtype == np.float64 else 1e-5
    assert _rel(ug, uo) <= tol
    assert np.array_equal(ug, uo)
    assert np.array_equal(hg, ho)


@pytest.mark.slow
@pytest.mark.parametrize("dtype", [np.float64, np.float32], ids=["f64", "f32"])
def test_parity_2d_8193_full_size(dtype):
    """BASELINE configs[2] at full size and the north star's 10 V-cycles,
    compared element by element: once with the residual history (every
    cycle's last pass is the cross-cycle fused asc_desc) and once without
    (the bench's exact call: the last cycle ends with the plain asc_fine pass,
    many tiles per CTA)."""
    f = W.workload_rhs("2d_8193").astype(dtype)
    u0 = np.zeros_like(f)
    uo, ho = _oracle_run(2, 8193, 2, P2, f, u0, 10, dtype)
    tol = 1e-11 if dtype == np.float64 else 1e-5
    for hist in (True, False):
        ug, hg = _gpu_run(2, 8193, 2, P2, f, u0, 10, dtype, hist=hist)
        assert _rel(ug, uo) <= tol
        assert np.array_equal(ug, uo), (hist, _rel(ug, uo))
        if hist:
            assert np.array_equal(hg, ho)


@pytest.mark.parametrize("dtype", [np.float64, np.float32], ids=["f64", "f32"])
@pytest.mark.parametrize("order", [2, 4])
def test_cycle_fusion_call_patterns(order, dtype):
    """Cross-cycle fusion: 1, 2 and 5 cycles per call, with and
    without the residual history, and a run split over several calls all
    equal the oracle bit for bit."""
    import torch
    n, p = 513, (P2 if order == 2 else P2_4)
    f = W.random_field(2, n, seed=31).astype(dtype)
    u0 = (W.random_field(2, n, seed=32) * 0.1).astype(dtype)
    for cycles in (1, 2, 5):
        uo, ho = _oracle_run(2, n, order, p, f, u0, cycles, dtype)
        for hist in (False, True):
            ug, hg = _gpu_run(2, n, order, p, f, u0, cycles, dtype, hist=hist)
            assert np.array_equal(ug, uo), (cycles, hist, _rel(ug, uo))
            if hist:
                assert np.array_equal(hg, ho), cycles
    s = _solver(2, n, order, p, dtype)
    u = s.alloc(u0)
    ft = s.alloc(f)
    for c in (2, 1, 3):
        s.vcycle(u, ft, c)
    torch.cuda.synchronize()
    uo, _ = _oracle_run(2, n, order, p, f, u0, 6, dtype)
    assert np.array_equal(s.view(u).cpu().numpy(), uo)


@pytest.mark.slow
@pytest.mark.parametrize("dtype", [np.float64, np.float32], ids=["f64", "f32"])
def test_parity_3d_513_full_size(dtype):
    """BASELINE configs[4] at full size and the north star's 10 V-cycles,
    compared element by element, with and without the residual history; fp32
    as well (the fp32 sublattice passes of round 2, k3s.cu)."""
    f = W.workload_rhs("3d_513").astype(dtype)
    u0 = np.zeros_like(f)
    uo, ho = _oracle_run(3, 513, 2, P3, f, u0, 10, dtype)
    for hist in (True, False):
        ug, hg = _gpu_run(3, 513, 2, P3, f, u0, 10, dtype, hist=hist)
        assert _rel(ug, uo) <= (1e-11 if dtype == np.float64 else 1e-5)
        assert np.array_equal(ug, uo), (hist, _rel(ug, uo))
        if hist:
            assert np.array_equal(hg, ho)


@pytest.mark.parametrize("dim,n,dtype", [(2, 65, np.float64), (3, 17, np.float64), (2, 257, np.float64),
                                         (2, 257, np.float32), (3, 33, np.float32)])
def test_unaligned_pitch(dim, n, dtype):
    """Caller arrays with pitch = n (rows not 16-byte aligned) and a wide pitch: staged through the work layout
    by the re-pitch kernel (n = 257: two full 128-element chunks and a one-element tail per row)."""
    p = P2 if dim == 2 else P3
    f = W.random_field(dim, n, seed=2).astype(dtype)
    uo, _ = _oracle_run(dim, n, 2, p, f, np.zeros_like(f), 3, dtype)
    for pitch in (n, n + 7, 2 * n + 3):
        ug, _ = _gpu_run(dim, n, 2, p, f, np.zeros_like(f), 3, dtype, pitch=pitch)
        assert np.array_equal(ug, uo), pitch


@pytest.mark.parametrize("dim,n,order", [(2, 65, 2), (2, 65, 4), (3, 33, 2), (3, 33, 4)])
def test_residual_and_norm(dim, n, order):
    import torch
    p = P2 if dim == 2 else P3
    f = W.random_field(dim, n, seed=4)
    u = W.random_field(dim, n, seed=5)
    s = _solver(dim, n, order, p, np.float64)
    ut, ftt = s.alloc(u), s.alloc(f)
    r = s.view(s.residual(ut, ftt)).cpu().numpy()
    ro = oracle.residual(u, f, order)
    assert np.array_equal(r, ro)
    rt = s.alloc(ro)
    assert s.norm(rt, "inf") == oracle.norm_inf(ro)
    l2 = np.sqrt((1.0 / (n - 1)) ** dim * np.sum(ro[(slice(1, -1),) * dim] ** 2))
    assert s.norm(rt, "l2") == pytest.approx(l2, rel=1e-12)
    torch.cuda.synchronize()


def test_zero_cycles_and_hist():
    n = 33
    f = W.random_field(2, n, seed=1)
    s = _solver(2, n, 2, P2, np.float64)
    u, ft = s.alloc(), s.alloc(f)
    assert s.vcycle(u, ft, 0) is None
    h = s.vcycle(u, ft, 0, hist=True)
    assert h.shape == (1,) and h[0] == oracle.norm_inf(f)
    assert float(s.view(u).abs().max()) == 0.0


def test_diverged_reports_status():
    """A NaN in f makes the residual norm non-finite: MG_EDIVERGED."""
    from paper_math_9907190_b200.mg import MGError, MG_EDIVERGED
    n = 17
    f = W.random_field(2, n, seed=1)
    f[5, 5] = np.nan
    s = _solver(2, n, 2, P2, np.float64)
    with pytest.raises(MGError) as ei:
        s.vcycle(s.alloc(), s.alloc(f), 2, hist=True)
    assert ei.value.status == MG_EDIVERGED


@pytest.mark.parametrize("dim,n", [(2, 1025), (3, 65)])
def test_green_only_mode_oracle_free(dim, n):
    """SURVEY P17 on the GPU, no oracle: an error on the green-only nodes is
    mapped by one order-2 cycle to (1 - p) e (p_g in 3D) up to rounding."""
    rng = np.random.default_rng(3)
    idx = np.indices((n,) * dim).sum(0)
    inner = np.zeros((n,) * dim, bool)
    inner[(slice(1, -1),) * dim] = True
    green = (idx % 2 == 1) & inner
    w = np.where(green, rng.uniform(-1, 1, (n,) * dim), 0.0)
    p = 1.3
    pp = p if dim == 2 else (1.11, 1.42, 1.08, p)
    ug, _ = _gpu_run(dim, n, 2, pp, np.zeros_like(w), w, 1, np.float64)
    want = np.where(green, w - p * w, 0.0)
    assert np.max(np.abs(ug - want)) < 64 * np.finfo(np.float64).eps


def test_fp32_convergence_factor_within_2pct():
    """North star: the fp32 variant's convergence factor is within 2% of fp64
    (power iteration on f = 0, 2D 1025^2)."""
    n = 1025
    f = np.zeros((n, n))
    rng = np.random.default_rng(0)
    u0 = np.zeros((n, n))
    u0[1:-1, 1:-1] = rng.uniform(-1, 1, (n - 2, n - 2))
    rates = {}
    for dtype in (np.float64, np.float32):
        s = _solver(2, n, 2, P2, dtype)
        u = s.alloc(u0.astype(dtype))
        ft = s.alloc(f.astype(dtype))
        norms = []
        for _ in range(8):
            s.vcycle(u, ft, 1)
            norms.append(float(s.view(u).abs().max()))
        rates[dtype] = (norms[-1] / norms[-4]) ** (1 / 3)
    assert rates[np.float32] == pytest.approx(rates[np.float64], rel=0.02)
    assert 0.05 <= rates[np.float64] <= 0.09


@pytest.mark.parametrize("dim,n", [(2, 129), (3, 33)])
def test_multi_cycle_graphs(dim, n):
    """Runs of cycles are replayed as CUDA graphs of MG_GRAPH_CYCLES (8) cycles,
    the remainder one cycle per graph: cycle counts around the graph size, with
    and without the residual history, and alternating call lengths on one
    solver (cached graphs of every size reused) equal the oracle bit for bit."""
    import torch
    p = P2 if dim == 2 else P3
    f = W.random_field(dim, n, seed=41)
    u0 = W.random_field(dim, n, seed=42) * 0.1
    for cycles in (8, 9, 10, 17, 18):
        uo, ho = _oracle_run(dim, n, 2, p, f, u0, cycles, np.float64)
        for hist in (False, True):
            ug, hg = _gpu_run(dim, n, 2, p, f, u0, cycles, np.float64, hist=hist)
            assert np.array_equal(ug, uo), (cycles, hist, _rel(ug, uo))
            if hist:
                assert np.array_equal(hg, ho), cycles
    s = _solver(dim, n, 2, p, np.float64)
    u = s.alloc(u0)
    ft = s.alloc(f)
    total = 0
    for c in (10, 3, 17, 1, 9):
        s.vcycle(u, ft, c)
        total += c
    torch.cuda.synchronize()
    uo, _ = _oracle_run(dim, n, 2, p, f, u0, total, np.float64)
    assert np.array_equal(s.view(u).cpu().numpy(), uo)
