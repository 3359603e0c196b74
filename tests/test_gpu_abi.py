"""The C ABI as a plain C caller uses it: mg_create with the
default pitch = n (never 16-byte rows for n = 2^k+1), offset base pointers,
host arrays, and the residual-history limit.  Every case runs the sm_100a
TMA kernels (checked by kernel name with the CUDA profiler) and equals the
CPU oracle bit for bit.
"""
import ctypes

import numpy as np
import pytest
import torch

import oracle
from paper_math_9907190_b200 import mg
from paper_math_9907190_b200.mg import Solver
from paper_math_9907190_b200 import workloads as W

pytestmark = pytest.mark.gpu

P2 = 1.052
P3 = (1.11, 1.42, 1.08, 0.99)


def _create_default(dim, n, order, omega):
    """mg_create: fp64, pitch = n, legacy default stream, p[*] = omega."""
    return mg.mg_create(dim, n, order, omega)


def _kernels(fn):
    torch.cuda.synchronize()
    with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
        fn()
        torch.cuda.synchronize()
    return {e.name for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA}


@pytest.mark.parametrize("order", [2, 4])
def test_mg_create_pitch_n_runs_tma_kernels_2d(order):
    n, cycles = 1025, 10
    p = P2 if order == 2 else 1.20
    h = _create_default(2, n, order, p)
    try:
        f = W.random_field(2, n, seed=41)
        u0 = W.random_field(2, n, seed=42) * 0.1
        ft = torch.from_numpy(f).cuda()            # (n, n): pitch = n
        for hist in (False, True):
            ut = torch.from_numpy(u0).cuda()
            got = {}
            names = _kernels(lambda: got.setdefault("h", mg.mg_vcycle(h, ut.data_ptr(), ft.data_ptr(), cycles, hist)))
            assert any("tile_pipeline" in k for k in names), sorted(names)
            assert any("asc_desc_stream" in k for k in names), sorted(names)
            assert any("k_repitch" in k for k in names), sorted(names)   # staged by the library's own copy kernel
            uo = u0.copy()
            ho = oracle.vcycle(uo, f, p, cycles, order=order, hist=True)
            assert np.array_equal(ut.cpu().numpy(), uo)
            if hist:
                assert np.array_equal(got["h"], ho)
    finally:
        mg.mg_destroy(h)


def test_mg_create_pitch_n_runs_tma_kernels_3d():
    n, cycles = 65, 10
    h = mg.mg_create(3, n, 2, 1.0)
    try:
        f = W.random_field(3, n, seed=43)
        ut = torch.zeros((n, n, n), dtype=torch.float64, device="cuda")
        ft = torch.from_numpy(f).cuda()
        names = _kernels(lambda: mg.mg_vcycle(h, ut.data_ptr(), ft.data_ptr(), cycles))
        assert any("zpipe" in k for k in names), sorted(names)
        uo = np.zeros_like(f)
        oracle.vcycle(uo, f, (1.0,) * 4, cycles)
        assert np.array_equal(ut.cpu().numpy(), uo)
    finally:
        mg.mg_destroy(h)


@pytest.mark.parametrize("dim,n", [(2, 257), (3, 33)])
def test_offset_base_pointers(dim, n):
    """u and f 8 bytes past a 16-byte boundary, pitch a multiple of 16 bytes:
    staged into the work layout (the TMA encode used to reject them)."""
    from paper_math_9907190_b200.mg import Solver
    p = P2 if dim == 2 else P3
    s = Solver(dim, n, order=2, p=p)
    f = W.random_field(dim, n, seed=44)
    u0 = W.random_field(dim, n, seed=45) * 0.1
    shape = s.shape
    numel = int(np.prod(shape))
    buf_u = torch.zeros(numel + 1, dtype=torch.float64, device="cuda")
    buf_f = torch.zeros(numel + 1, dtype=torch.float64, device="cuda")
    u = buf_u[1:].view(shape)
    ft = buf_f[1:].view(shape)
    s.view(u).copy_(torch.from_numpy(u0))
    s.view(ft).copy_(torch.from_numpy(f))
    assert u.data_ptr() % 16 == 8
    hg = mg.mg_vcycle(s.h, u.data_ptr(), ft.data_ptr(), 5, True)
    uo = u0.copy()
    ho = oracle.vcycle(uo, f, p, 5, hist=True)
    assert np.array_equal(s.view(u).cpu().numpy(), uo)
    assert np.array_equal(hg, ho)


@pytest.mark.parametrize("order", [2, 4])
def test_vcycle_host_pitch_n(order):
    n = 513
    p = P2 if order == 2 else 1.20
    h = mg.mg_create(2, n, order, p)
    try:
        f = W.random_field(2, n, seed=46)
        uh = torch.zeros((n, n), dtype=torch.float64).pin_memory()
        fh = torch.from_numpy(f).pin_memory()
        hg = mg.mg_vcycle_host(h, uh.data_ptr(), fh.data_ptr(), 6, True)
        uo = np.zeros_like(f)
        ho = oracle.vcycle(uo, f, p, 6, order=order, hist=True)
        assert np.array_equal(uh.numpy(), uo)
        assert np.array_equal(hg, ho)
    finally:
        mg.mg_destroy(h)


@pytest.mark.parametrize("dim,n,order,dt", [(2, 513, 2, "f64"), (2, 257, 4, "f64"), (2, 513, 2, "f32"),
                                            (3, 65, 2, "f64"), (3, 65, 4, "f32")])
def test_solve_host_from_zero(dim, n, order, dt):
    """mg_solve_host: f in, u out, u starts at 0 on the device whatever u_host holds."""
    npdt = np.float64 if dt == "f64" else np.float32
    p = (P2 if order == 2 else 1.20) if dim == 2 else (1.11, 1.42, 1.08, 0.99)
    tdt = torch.float64 if dt == "f64" else torch.float32
    s = Solver(dim, n, order=order, p=p, dtype=tdt)
    f = W.random_field(dim, n, seed=49).astype(npdt)
    fh = torch.zeros(s.shape, dtype=tdt).pin_memory()
    s.view(fh).copy_(torch.from_numpy(f))
    uh = torch.full(s.shape, 7.0, dtype=tdt).pin_memory()   # garbage: an output-only array
    hg = s.solve_host(uh, fh, 5, True)
    uo = np.zeros_like(f)
    ho = oracle.vcycle(uo, f, p, 5, order=order, hist=True)
    assert np.array_equal(s.view(uh).numpy(), uo)
    assert np.array_equal(hg, ho)


@pytest.mark.parametrize("dim,n,order,dt,count", [(2, 513, 2, "f64", 5), (2, 257, 4, "f64", 3), (2, 513, 2, "f32", 4),
                                                  (3, 65, 2, "f64", 3), (3, 65, 4, "f32", 2), (2, 129, 2, "f64", 1),
                                                  (2, 129, 2, "f64", 0)])
def test_solve_host_batch(dim, n, order, dt, count):
    """mg_solve_host_batch: every problem of the overlapped batch equals its own
    oracle solve from u = 0 (distinct right-hand sides, garbage in the outputs)."""
    npdt = np.float64 if dt == "f64" else np.float32
    p = (P2 if order == 2 else 1.20) if dim == 2 else (1.11, 1.42, 1.08, 0.99)
    tdt = torch.float64 if dt == "f64" else torch.float32
    s = Solver(dim, n, order=order, p=p, dtype=tdt)
    fs = [W.random_field(dim, n, seed=60 + i).astype(npdt) for i in range(count)]
    fh = []
    for f in fs:
        t = torch.zeros(s.shape, dtype=tdt).pin_memory()
        s.view(t).copy_(torch.from_numpy(f))
        fh.append(t)
    uh = [torch.full(s.shape, -3.0, dtype=tdt).pin_memory() for _ in range(count)]
    s.solve_host_batch(uh, fh, 4)
    for f, u in zip(fs, uh):
        uo = np.zeros_like(f)
        oracle.vcycle(uo, f, p, 4, order=order)
        assert np.array_equal(s.view(u).numpy(), uo)


@pytest.mark.parametrize("dim,n,order", [(2, 129, 2), (2, 129, 4), (3, 33, 2), (3, 33, 4)])
def test_residual_and_norm_pitch_n(dim, n, order):
    h = mg.mg_create(dim, n, order, 1.0)
    try:
        f = W.random_field(dim, n, seed=47)
        u = W.random_field(dim, n, seed=48)
        ut, ftt = torch.from_numpy(u).cuda(), torch.from_numpy(f).cuda()
        rt = torch.empty_like(ut)
        mg.mg_residual(h, ut.data_ptr(), ftt.data_ptr(), rt.data_ptr())
        torch.cuda.synchronize()
        ro = oracle.residual(u, f, order)
        assert np.array_equal(rt.cpu().numpy(), ro)
        assert mg.mg_norm(h, rt.data_ptr(), mg.MG_NORM_INF) == oracle.norm_inf(ro)
    finally:
        mg.mg_destroy(h)


def test_convergence_factor_pitch_n_equals_padded():
    from paper_math_9907190_b200.mg import Solver
    n = 129
    e0 = W.random_field(2, n, seed=49)
    h = mg.mg_create(2, n, 2, P2)
    try:
        et = torch.from_numpy(e0.copy()).cuda()
        rho_a, ra = mg.mg_convergence_factor(h, et.data_ptr(), 40)
    finally:
        mg.mg_destroy(h)
    s = Solver(2, n, order=2, p=P2)
    e = s.alloc(e0)
    rho_b, rb = s.convergence_factor(e, 40)
    # the L2 sums are reduced in a layout-dependent order: equal to rounding
    assert rho_a == pytest.approx(rho_b, rel=1e-12)
    np.testing.assert_allclose(ra, rb, rtol=1e-12)
    np.testing.assert_allclose(et.cpu().numpy(), s.view(e).cpu().numpy(), rtol=0, atol=1e-12)


def test_history_limit():
    """res_hist holds ncycles+1 norms; more than the device history (4096)
    is refused instead of silently merging cycles."""
    n = 17
    h = mg.mg_create(2, n, 2, P2)
    try:
        ut = torch.zeros((n, n), dtype=torch.float64, device="cuda")
        ft = torch.from_numpy(W.random_field(2, n, seed=1)).cuda()
        buf = (ctypes.c_double * 5000)()
        rc = mg.load().mg_vcycle(h, ut.data_ptr(), ft.data_ptr(), 4096, buf)
        assert rc == mg.MG_EINVAL
        hist = mg.mg_vcycle(h, ut.data_ptr(), ft.data_ptr(), 4095, True)
        assert len(hist) == 4096 and hist[-1] <= hist[0]
    finally:
        mg.mg_destroy(h)
