"""Multi-GPU slab decomposition on one GPU: P virtual ranks
(MG_FLAG_LOOPBACK) run the same halo / agglomeration schedule as the NCCL
ranks; the iterate must equal the single-GPU solver's bit for bit."""
import numpy as np
import pytest

from paper_math_9907190_b200 import workloads as W

pytestmark = pytest.mark.gpu


def _run(n, order, dtype, cycles, nranks=1, loopback=False, agglom=0, seed=3, dim=2):
    import torch
    from paper_math_9907190_b200.mg import Solver
    tdt = torch.float64 if dtype == np.float64 else torch.float32
    p = (1.052 if order == 2 else 1.20) if dim == 2 else (1.11, 1.42, 1.08, 0.99)
    s = Solver(dim, n, order=order, p=p, dtype=tdt, nranks=nranks, loopback=loopback, agglom_points=agglom)
    f = W.random_field(dim, n, seed=seed).astype(dtype)
    u0 = (0.1 * W.random_field(dim, n, seed=seed + 1)).astype(dtype)
    u, ft = s.alloc(u0), s.alloc(f)
    h = s.vcycle(u, ft, cycles, hist=True)
    return s.view(u).cpu().numpy(), h


@pytest.mark.parametrize("dtype", [np.float64, np.float32], ids=["f64", "f32"])
@pytest.mark.parametrize("n,P", [(65, 2), (65, 4), (257, 2), (257, 8), (1025, 4), (1025, 8)])
def test_loopback_equals_single_gpu(n, P, dtype):
    ref, href = _run(n, 2, dtype, 3)
    for agglom in (0, 16):   # default threshold, and a deep decomposition
        got, h = _run(n, 2, dtype, 3, nranks=P, loopback=True, agglom=agglom)
        assert np.array_equal(got, ref), (P, agglom, float(np.max(np.abs(got - ref))))
        assert np.array_equal(h, href)


@pytest.mark.parametrize("n,P", [(129, 4), (1025, 2)])
def test_loopback_order4_and_odd_cycles(n, P):
    for cycles in (1, 2, 5):
        ref, href = _run(n, 4, np.float64, cycles)
        got, h = _run(n, 4, np.float64, cycles, nranks=P, loopback=True, agglom=16)
        assert np.array_equal(got, ref)
        assert np.array_equal(h, href)


def test_multi_rank_rejects_bad_splits():
    from paper_math_9907190_b200.mg import MGError, MG_EUNSUPPORTED
    with pytest.raises(MGError) as e:
        _run(17, 2, np.float64, 1, nranks=8, loopback=True)   # (n-1)/P < 4
    assert e.value.status == MG_EUNSUPPORTED
    with pytest.raises(MGError) as e:
        _run(65, 2, np.float64, 1, nranks=3, loopback=True)   # not a power of two
    assert e.value.status == MG_EUNSUPPORTED


# ------------------------------------------------------------ 3D z-slabs

@pytest.mark.parametrize("dtype", [np.float64, np.float32], ids=["f64", "f32"])
@pytest.mark.parametrize("n,P", [(33, 2), (65, 2), (65, 4), (129, 8)])
def test_loopback_3d_equals_single_gpu(n, P, dtype):
    ref, href = _run(n, 2, dtype, 3, dim=3)
    for agglom in (0, 16):   # default threshold (2^18), and a deep decomposition
        got, h = _run(n, 2, dtype, 3, nranks=P, loopback=True, agglom=agglom, dim=3)
        assert np.array_equal(got, ref), (P, agglom, float(np.max(np.abs(got - ref))))
        assert np.array_equal(h, href)


@pytest.mark.parametrize("n,P", [(65, 4), (129, 2)])
def test_loopback_3d_order4_and_odd_cycles(n, P):
    for cycles in (1, 2):
        ref, href = _run(n, 4, np.float64, cycles, dim=3)
        got, h = _run(n, 4, np.float64, cycles, nranks=P, loopback=True, agglom=16, dim=3)
        assert np.array_equal(got, ref)
        assert np.array_equal(h, href)


@pytest.mark.slow
def test_loopback_3d_513_p8():
    """BASELINE configs[4]'s decomposition: 513^3 over 8 z-slabs (64 planes
    each), agglomeration at G(8) (250,047 points < 2^18), one cycle."""
    ref, href = _run(513, 2, np.float64, 1, dim=3)
    got, h = _run(513, 2, np.float64, 1, nranks=8, loopback=True, dim=3)
    assert np.array_equal(got, ref)
    assert np.array_equal(h, href)


def test_residual_and_norm_on_loopback_3d():
    import torch
    from paper_math_9907190_b200.mg import Solver
    n = 33
    s1 = Solver(3, n, order=4, p=(1.11, 1.42, 1.08, 0.99))
    s4 = Solver(3, n, order=4, p=(1.11, 1.42, 1.08, 0.99), nranks=4, loopback=True)
    u = W.random_field(3, n, seed=8)
    f = W.random_field(3, n, seed=9)
    r1 = s1.view(s1.residual(s1.alloc(u), s1.alloc(f))).cpu().numpy()
    r4 = s4.view(s4.residual(s4.alloc(u), s4.alloc(f))).cpu().numpy()
    assert np.array_equal(r1, r4)
    torch.cuda.synchronize()


# ------------------------------------- 2D communication-avoiding schedule

@pytest.mark.parametrize("dtype", [np.float64, np.float32], ids=["f64", "f32"])
@pytest.mark.parametrize("n,P,agglom", [(1025, 2, 1 << 14), (1025, 4, 1 << 12), (2049, 4, 1 << 14),
                                        (2049, 8, 1 << 10), (513, 2, 0)])
def test_loopback_deep_halo_equals_single_gpu(n, P, agglom, dtype):
    """The one-exchange-per-cycle schedule (Dist2CA: deep ghost bands computed
    redundantly) with the octave-pair passes on bands (default)
    or the level passes (MG_DIST_NOFUSE=1), and the per-level schedule
    (MG_DIST_PERLEVEL=1) all equal the single-GPU iterate and residual history
    bit for bit, with agglomeration thresholds that distribute 1 to 6 octaves."""
    import os
    ref, href = _run(n, 2, dtype, 4)
    for env in ({}, {"MG_DIST_NOFUSE": "1"}, {"MG_DIST_PERLEVEL": "1"}):
        os.environ.update(env)
        try:
            got, h = _run(n, 2, dtype, 4, nranks=P, loopback=True, agglom=agglom)
        finally:
            for key in env:
                os.environ.pop(key, None)
        assert np.array_equal(got, ref), (env, float(np.max(np.abs(got - ref))))
        assert np.array_equal(h, href)


@pytest.mark.parametrize("n,P", [(1025, 4), (513, 2)])
def test_loopback_deep_halo_order4(n, P):
    for cycles in (1, 3):
        ref, href = _run(n, 4, np.float64, cycles)
        got, h = _run(n, 4, np.float64, cycles, nranks=P, loopback=True, agglom=1 << 12)
        assert np.array_equal(got, ref)
        assert np.array_equal(h, href)
