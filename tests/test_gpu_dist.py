"""Multi-GPU slab decomposition on one GPU: P virtual ranks
(MG_FLAG_LOOPBACK) run the same halo / agglomeration schedule as the NCCL
ranks; the iterate must equal the single-GPU solver's bit for bit."""
import numpy as np
import pytest

from paper_math_9907190_b200 import workloads as W

pytestmark = pytest.mark.gpu


def _run(n, order, dtype, cycles, nranks=1, loopback=False, agglom=0, seed=3):
    import torch
    from paper_math_9907190_b200.mg import Solver
    tdt = torch.float64 if dtype == np.float64 else torch.float32
    p = 1.052 if order == 2 else 1.20
    s = Solver(2, n, order=order, p=p, dtype=tdt, nranks=nranks, loopback=loopback, agglom_points=agglom)
    f = W.random_field(2, n, seed=seed).astype(dtype)
    u0 = (0.1 * W.random_field(2, n, seed=seed + 1)).astype(dtype)
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
