"""The C-ABI library builds, loads and exports every symbol include/mg.h
declares; argument validation needs no GPU (no compute calls here)."""
import ctypes
import os
import re

import pytest

from paper_math_9907190_b200 import build as B
from paper_math_9907190_b200 import mg

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "mg.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(mg_[a-z_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def lib():
    B.build()
    return mg.load()


def test_header_declares_the_boundary():
    names = _declared()
    for want in ("mg_create", "mg_create_ex", "mg_residual", "mg_vcycle", "mg_norm", "mg_destroy",
                 "mg_local_extent", "mg_strerror", "mg_last_error", "mg_vcycle_host", "mg_solve_host",
                 "mg_solve_host_batch"):
        assert want in names


def test_every_declared_symbol_is_exported(lib):
    for name in _declared():
        assert hasattr(lib, name), name
        assert name in mg.EXPORTS, f"binding lacks {name}"


def test_shared_object_is_sm100a():
    B.build()
    out = os.popen(f"/usr/local/cuda/bin/cuobjdump --list-elf {B.LIB} 2>&1").read()
    assert "sm_100a" in out, out


def test_strerror(lib):
    assert mg.mg_strerror(0) == "ok"
    assert "invalid" in mg.mg_strerror(mg.MG_EINVAL)
    assert mg.mg_strerror(-99) == "unknown status"


@pytest.mark.parametrize("dim,n,order,omega", [
    (2, 6, 2, 1.0), (2, 3, 2, 1.0), (4, 17, 2, 1.0), (2, 17, 3, 1.0), (2, 17, 2, 0.0),
    (2, 17, 2, -1.0), (3, 17, 2, 3.5), (2, 0, 2, 1.0)])
def test_create_rejects_bad_arguments(lib, dim, n, order, omega):
    h = ctypes.c_void_p()
    assert lib.mg_create(dim, n, order, omega, ctypes.byref(h)) == mg.MG_EINVAL
    assert not h.value


def test_create_ex_rejects_bad_pitch(lib):
    cfg = mg.mg_config()
    cfg.dim, cfg.n, cfg.order, cfg.dtype = 2, 17, 2, mg.MG_F64
    cfg.p = (ctypes.c_double * 4)(1.0, 1.0, 1.0, 1.0)
    cfg.pitch = 16
    cfg.device, cfg.nranks = -1, 1
    h = ctypes.c_void_p()
    assert lib.mg_create_ex(ctypes.byref(cfg), ctypes.byref(h)) == mg.MG_EINVAL


def test_null_handle_calls(lib):
    assert lib.mg_vcycle(None, None, None, 1, None) == mg.MG_EINVAL
    assert lib.mg_destroy(None) == mg.MG_OK
    assert lib.mg_num_levels(None) == mg.MG_EINVAL


def test_no_cpu_fallback_without_gpu(lib):
    """Without a CUDA device the library refuses (MG_ENODEV): no CPU path."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    h = ctypes.c_void_p()
    assert lib.mg_create(2, 17, 2, 1.0, ctypes.byref(h)) == mg.MG_ENODEV


def test_convergence_factor_rejects_null_handle(lib):
    rho = ctypes.c_double()
    assert lib.mg_convergence_factor(None, None, 10, ctypes.byref(rho), None) == mg.MG_EINVAL
