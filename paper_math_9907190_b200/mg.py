"""Thin Python binding of libmg (include/mg.h): argument marshalling only.

Every step of the V-cycle runs in libmg's sm_100a kernels; this module only
passes pointers, sizes and the CUDA stream.  PyTorch supplies device memory
and streams.  There is no CPU fallback: if libmg.so cannot be loaded or no
CUDA device is present the calls raise.

The functions mirror the C ABI one to one (``mg_create``, ``mg_create_ex``,
``mg_destroy``, ``mg_local_extent``, ``mg_residual``, ``mg_vcycle``, ``mg_vcycle_norms``,
``mg_vcycle_host``, ``mg_solve_host``, ``mg_solve_host_batch``, ``mg_norm``, ``mg_num_levels``, ``mg_level_points``,
``mg_launches_per_cycle``, ``mg_strerror``, ``mg_last_error``);
:class:`Solver` wraps a handle for torch tensors.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libmg.so")

MG_OK, MG_EINVAL, MG_ENOMEM, MG_ECUDA, MG_ENCCL, MG_EUNSUPPORTED, MG_EDIVERGED, MG_ENODEV = 0, -1, -2, -3, -4, -5, -6, -7
MG_F64, MG_F32 = 0, 1
MG_NORM_INF, MG_NORM_L2 = 0, 1
MG_FLAG_LOOPBACK = 1
MG_FLAG_CONVENTIONAL = 2
MG_FLAG_SLABS = 4


class MGError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"libmg status {status} ({mg_strerror(status)}): {msg}")
        self.status = status


class mg_config(ctypes.Structure):
    _fields_ = [
        ("dim", ctypes.c_int),
        ("n", ctypes.c_int64),
        ("order", ctypes.c_int),
        ("dtype", ctypes.c_int),
        ("p", ctypes.c_double * 4),
        ("pitch", ctypes.c_int64),
        ("stream", ctypes.c_void_p),
        ("device", ctypes.c_int),
        ("nranks", ctypes.c_int),
        ("rank", ctypes.c_int),
        ("nccl_id", ctypes.c_void_p),
        ("agglom_points", ctypes.c_int64),
        ("flags", ctypes.c_int),
        ("sweeps", ctypes.c_int),
    ]


class mg_step_stat(ctypes.Structure):
    _fields_ = [("name", ctypes.c_char * 40), ("level", ctypes.c_int), ("launches", ctypes.c_int),
                ("ms", ctypes.c_double), ("alg_bytes", ctypes.c_double)]


EXPORTS = {
    "mg_create": (ctypes.c_int, [ctypes.c_int, ctypes.c_int64, ctypes.c_int, ctypes.c_double, ctypes.c_void_p]),
    "mg_create_ex": (ctypes.c_int, [ctypes.POINTER(mg_config), ctypes.c_void_p]),
    "mg_destroy": (ctypes.c_int, [ctypes.c_void_p]),
    "mg_local_extent": (ctypes.c_int, [ctypes.c_void_p, ctypes.POINTER(ctypes.c_int64),
                                       ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(ctypes.c_int64)]),
    "mg_residual": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]),
    "mg_vcycle": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int,
                                 ctypes.POINTER(ctypes.c_double)]),
    "mg_vcycle_norms": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int,
                                       ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_double)]),
    "mg_vcycle_host": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int,
                                      ctypes.POINTER(ctypes.c_double)]),
    "mg_solve_host": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int,
                                     ctypes.POINTER(ctypes.c_double)]),
    "mg_solve_host_batch": (ctypes.c_int, [ctypes.c_void_p, ctypes.POINTER(ctypes.c_void_p),
                                           ctypes.POINTER(ctypes.c_void_p), ctypes.c_int, ctypes.c_int]),
    "mg_norm": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int, ctypes.POINTER(ctypes.c_double)]),
    "mg_num_levels": (ctypes.c_int, [ctypes.c_void_p]),
    "mg_level_points": (ctypes.c_int64, [ctypes.c_void_p, ctypes.c_int]),
    "mg_launches_per_cycle": (ctypes.c_int, [ctypes.c_void_p]),
    "mg_profile": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int,
                                  ctypes.POINTER(mg_step_stat), ctypes.c_int]),
    "mg_convergence_factor": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int,
                                             ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_double)]),
    "mg_slab_plan": (ctypes.c_int, [ctypes.c_int, ctypes.c_int64, ctypes.c_int, ctypes.c_int, ctypes.c_int64,
                                    ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(ctypes.c_int64),
                                    ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(ctypes.c_int)]),
    "mg_slab_schedule": (ctypes.c_int, [ctypes.c_int, ctypes.c_int64, ctypes.c_int, ctypes.c_int64,
                                        ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_int64)]),
    "mg_nccl_unique_id": (ctypes.c_int, [ctypes.c_void_p]),
    "mg_strerror": (ctypes.c_char_p, [ctypes.c_int]),
    "mg_last_error": (ctypes.c_char_p, [ctypes.c_void_p]),
}

_lib = None


def load(path: str = LIB_PATH):
    """Load libmg.so (raises if it is missing: there is no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(path):
            raise ImportError(f"{path} not built; run __graft_entry__.build() "
                              "(python -m paper_math_9907190_b200.build)")
        lib = ctypes.CDLL(path)
        for name, (res, args) in EXPORTS.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib


def _check(rc: int, handle=None, what: str = ""):
    if rc != MG_OK:
        msg = what
        if handle is not None:
            msg += ": " + (load().mg_last_error(handle) or b"").decode()
        raise MGError(rc, msg)


# ------------------------------------------------------------ raw ABI mirror

def mg_strerror(status: int) -> str:
    return load().mg_strerror(status).decode()


def mg_create(dim: int, n: int, order: int, omega: float):
    h = ctypes.c_void_p()
    _check(load().mg_create(dim, n, order, omega, ctypes.byref(h)), None, "mg_create")
    return h


def mg_create_ex(cfg: mg_config):
    h = ctypes.c_void_p()
    _check(load().mg_create_ex(ctypes.byref(cfg), ctypes.byref(h)), None, "mg_create_ex")
    return h


def mg_destroy(h) -> int:
    return load().mg_destroy(h)


def mg_local_extent(h):
    lo, hi, g = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
    _check(load().mg_local_extent(h, ctypes.byref(lo), ctypes.byref(hi), ctypes.byref(g)), h, "mg_local_extent")
    return lo.value, hi.value, g.value


def mg_residual(h, u_ptr: int, f_ptr: int, r_ptr: int) -> None:
    _check(load().mg_residual(h, u_ptr, f_ptr, r_ptr), h, "mg_residual")


def mg_vcycle(h, u_ptr: int, f_ptr: int, ncycles: int, hist: bool = False):
    buf = (ctypes.c_double * (ncycles + 1))() if hist else None
    _check(load().mg_vcycle(h, u_ptr, f_ptr, ncycles, buf), h, "mg_vcycle")
    return np.array(list(buf)) if hist else None


def mg_vcycle_norms(h, u_ptr: int, f_ptr: int, ncycles: int):
    """(L-inf history, L2 history), ncycles + 1 entries each."""
    inf = (ctypes.c_double * (ncycles + 1))()
    l2 = (ctypes.c_double * (ncycles + 1))()
    _check(load().mg_vcycle_norms(h, u_ptr, f_ptr, ncycles, inf, l2), h, "mg_vcycle_norms")
    return np.array(list(inf)), np.array(list(l2))


def mg_vcycle_host(h, u_ptr: int, f_ptr: int, ncycles: int, hist: bool = False):
    buf = (ctypes.c_double * (ncycles + 1))() if hist else None
    _check(load().mg_vcycle_host(h, u_ptr, f_ptr, ncycles, buf), h, "mg_vcycle_host")
    return np.array(list(buf)) if hist else None


def mg_solve_host(h, u_ptr: int, f_ptr: int, ncycles: int, hist: bool = False):
    buf = (ctypes.c_double * (ncycles + 1))() if hist else None
    _check(load().mg_solve_host(h, u_ptr, f_ptr, ncycles, buf), h, "mg_solve_host")
    return np.array(list(buf)) if hist else None


def mg_solve_host_batch(h, u_ptrs, f_ptrs, ncycles: int) -> None:
    n = len(u_ptrs)
    assert len(f_ptrs) == n
    ua = (ctypes.c_void_p * max(n, 1))(*u_ptrs)
    fa = (ctypes.c_void_p * max(n, 1))(*f_ptrs)
    _check(load().mg_solve_host_batch(h, ua, fa, n, ncycles), h, "mg_solve_host_batch")


def mg_norm(h, x_ptr: int, kind: int = MG_NORM_INF) -> float:
    out = ctypes.c_double()
    _check(load().mg_norm(h, x_ptr, kind, ctypes.byref(out)), h, "mg_norm")
    return out.value


def mg_num_levels(h) -> int:
    return load().mg_num_levels(h)


def mg_level_points(h, lev: int) -> int:
    return load().mg_level_points(h, lev)


def mg_launches_per_cycle(h) -> int:
    return load().mg_launches_per_cycle(h)


def mg_profile(h, u_ptr: int, f_ptr: int, ncycles: int, cap: int = 256):
    """Per-step mean durations (CUDA events) and algorithmic bytes of one cycle."""
    buf = (mg_step_stat * cap)()
    rc = load().mg_profile(h, u_ptr, f_ptr, ncycles, buf, cap)
    if rc < 0:
        _check(rc, h, "mg_profile")
    return [dict(name=b.name.decode(), level=b.level, launches=b.launches, ms=b.ms, alg_bytes=b.alg_bytes)
            for b in buf[: min(rc, cap)]]


def mg_convergence_factor(h, e_ptr: int, iters: int):
    """Power iteration of the V-cycle on the error equation (include/mg.h):
    returns (rho, per-iteration ratios)."""
    rho = ctypes.c_double()
    buf = (ctypes.c_double * iters)()
    _check(load().mg_convergence_factor(h, e_ptr, iters, ctypes.byref(rho), buf), h, "mg_convergence_factor")
    return rho.value, np.array(list(buf))


def mg_slab_plan(dim: int, n: int, nranks: int, rank: int, agglom_points: int = 0):
    """Host-only slab plan: (lo, hi, ghost, agglomeration octave)."""
    lo, hi, g, oa = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int()
    _check(load().mg_slab_plan(dim, n, nranks, rank, agglom_points, ctypes.byref(lo), ctypes.byref(hi),
                               ctypes.byref(g), ctypes.byref(oa)), None, "mg_slab_plan")
    return lo.value, hi.value, g.value, oa.value


def mg_slab_schedule(dim: int, n: int, nranks: int, agglom_points: int = 0):
    """Host-only: (schedule, halo rows) -- 1 = communication-avoiding 2D slabs, 0 = per-level halos."""
    sch, gu = ctypes.c_int(), ctypes.c_int64()
    _check(load().mg_slab_schedule(dim, n, nranks, agglom_points, ctypes.byref(sch), ctypes.byref(gu)), None,
           "mg_slab_schedule")
    return sch.value, gu.value


def mg_nccl_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    _check(load().mg_nccl_unique_id(buf), None, "mg_nccl_unique_id")
    return buf.raw


def broadcast_nccl_id(group=None) -> bytes:
    """Rank 0 of the torch.distributed group makes the NCCL id; every rank gets it."""
    import torch
    import torch.distributed as dist
    rank = dist.get_rank(group)
    t = torch.zeros(128, dtype=torch.uint8)
    if rank == 0:
        t.copy_(torch.frombuffer(bytearray(mg_nccl_unique_id()), dtype=torch.uint8))
    backend = dist.get_backend(group)
    if backend == "nccl":
        t = t.cuda()
    dist.broadcast(t, src=dist.get_global_rank(group, 0) if group is not None else 0, group=group)
    return bytes(t.cpu().numpy().tobytes())


def split_rows(full, lo: int, hi: int, ghost: int):
    """The slab a rank passes in multi-GPU mode: rows (2D) or planes (3D)
    [lo - ghost, hi + ghost) of a full array (those outside the grid are zero)."""
    import numpy as _np
    n = full.shape[0]
    out = _np.zeros((hi - lo + 2 * ghost,) + tuple(full.shape[1:]), dtype=full.dtype)
    a, b = max(lo - ghost, 0), min(hi + ghost, n)
    out[a - (lo - ghost): b - (lo - ghost)] = full[a:b]
    return out


def mg_last_error(h) -> str:
    return (load().mg_last_error(h) or b"").decode()


# ------------------------------------------------------------ torch wrapper

def _round_pitch(n: int, itemsize: int) -> int:
    q = 128 // itemsize
    return (n + q - 1) // q * q


class Solver:
    """One libmg handle bound to torch tensors on one CUDA device.

    ``Solver(dim, n, order=2, p=1.052 | (p_m, p_r1, p_r2, p_g), dtype=torch.float64)``;
    ``conventional=True`` selects the paper's "usual" V(0,1) multigrid (p: one
    value, 3D uses p_g).
    Fields are tensors of shape ``(n, pitch)`` (2D) or ``(n, n, pitch)`` (3D)
    whose first ``n`` columns are the grid; :meth:`alloc` makes them and
    :meth:`view` strips the padding.
    """

    def __init__(self, dim: int, n: int, order: int = 2, p=None, dtype=None, device=None,
                 pitch: int | None = None, stream=None, nranks: int = 1, rank: int = 0, group=None,
                 loopback: bool = False, agglom_points: int = 0, conventional: bool = False, sweeps: int = 1,
                 slabs: bool = False):
        import torch
        if not torch.cuda.is_available():
            raise MGError(MG_ENODEV, "no CUDA device (libmg has no CPU path)")
        self.torch = torch
        self.dim, self.n, self.order = dim, n, order
        self.dtype = dtype or torch.float64
        if p is None:
            p = (1.052,) if dim == 2 else (1.11, 1.42, 1.08, 0.99)
        if np.isscalar(p):
            p = (float(p),) * (1 if dim == 2 else 4)
        p = tuple(float(x) for x in p)
        self.p = p
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        itemsize = torch.empty((), dtype=self.dtype).element_size()
        self.pitch = pitch if pitch is not None else _round_pitch(n, itemsize)
        self.stream = stream or torch.cuda.current_stream(self.device)
        cfg = mg_config()
        cfg.dim, cfg.n, cfg.order = dim, n, order
        cfg.dtype = MG_F64 if self.dtype == torch.float64 else MG_F32
        pp = list(p) + [0.0] * (4 - len(p)) if dim == 2 else list(p)
        cfg.p = (ctypes.c_double * 4)(*pp)
        cfg.pitch = self.pitch
        cfg.stream = self.stream.cuda_stream
        cfg.device = self.device.index
        if group is not None:
            import torch.distributed as dist
            nranks, rank = dist.get_world_size(group), dist.get_rank(group)
        cfg.nranks, cfg.rank = nranks, rank
        cfg.agglom_points = agglom_points
        cfg.sweeps = sweeps
        self._id = None
        if conventional:
            cfg.flags = MG_FLAG_CONVENTIONAL   # the paper's "usual" V(0,1) multigrid (NEXT-3)
        if loopback:
            cfg.flags = MG_FLAG_LOOPBACK
        elif nranks > 1:
            self._id = ctypes.create_string_buffer(broadcast_nccl_id(group), 128)
            cfg.nccl_id = ctypes.cast(self._id, ctypes.c_void_p)
        elif slabs:   # the slab solver over a one-rank NCCL communicator (tests the transport on one GPU)
            self._id = ctypes.create_string_buffer(mg_nccl_unique_id(), 128)
            cfg.nccl_id = ctypes.cast(self._id, ctypes.c_void_p)
        if slabs:
            cfg.flags |= MG_FLAG_SLABS
        self.nranks, self.rank, self.loopback = nranks, rank, loopback
        self.slabs = (nranks > 1 or slabs) and not loopback
        self.h = mg_create_ex(cfg)
        lo, hi, g = mg_local_extent(self.h)
        self.lo, self.hi, self.ghost = lo, hi, g

    def __del__(self):
        h = getattr(self, "h", None)
        if h is not None and _lib is not None:
            mg_destroy(h)
            self.h = None

    # -- layout helpers
    @property
    def shape(self):
        """Shape of a field as this rank passes it (the slab with ghost rows in multi-GPU mode)."""
        if self.slabs:
            rows = self.hi - self.lo + 2 * self.ghost
            return (rows, self.pitch) if self.dim == 2 else (rows, self.n, self.pitch)
        return (self.n, self.pitch) if self.dim == 2 else (self.n, self.n, self.pitch)

    def alloc(self, like=None):
        t = self.torch.zeros(self.shape, dtype=self.dtype, device=self.device)
        if like is not None:
            self.view(t).copy_(self.torch.as_tensor(np.asarray(like), dtype=self.dtype))
        return t

    def view(self, t):
        return t[..., : self.n]

    def _chk(self, t):
        assert t.shape == self.shape and t.dtype == self.dtype and t.device == self.device and t.is_contiguous(), \
            (t.shape, self.shape, t.dtype, self.dtype)
        return t.data_ptr()

    # -- calls
    def vcycle(self, u, f, ncycles: int, hist: bool = False, l2: bool = False):
        """ncycles V-cycles in place on u; hist: the L-inf residual history;
        l2: (L-inf history, L2 history)."""
        if l2:
            return mg_vcycle_norms(self.h, self._chk(u), self._chk(f), ncycles)
        return mg_vcycle(self.h, self._chk(u), self._chk(f), ncycles, hist)

    def residual(self, u, f, r=None):
        r = r if r is not None else self.alloc()
        mg_residual(self.h, self._chk(u), self._chk(f), self._chk(r))
        return r

    def norm(self, x, kind: str = "inf") -> float:
        return mg_norm(self.h, self._chk(x), MG_NORM_INF if kind == "inf" else MG_NORM_L2)

    def vcycle_host(self, u_host, f_host, ncycles: int, hist: bool = False):
        """u_host / f_host: CPU tensors (ideally pinned) of ``self.shape``."""
        assert u_host.shape == self.shape and f_host.shape == self.shape and not u_host.is_cuda
        return mg_vcycle_host(self.h, u_host.data_ptr(), f_host.data_ptr(), ncycles, hist)

    def solve_host(self, u_host, f_host, ncycles: int, hist: bool = False):
        """ncycles V-cycles from u = 0 on HOST tensors: f_host in, u_host out."""
        assert u_host.shape == self.shape and f_host.shape == self.shape and not u_host.is_cuda
        return mg_solve_host(self.h, u_host.data_ptr(), f_host.data_ptr(), ncycles, hist)

    def solve_host_batch(self, u_hosts, f_hosts, ncycles: int):
        """Independent solves from u = 0: f_hosts[i] in, u_hosts[i] out (HOST tensors of
        ``self.shape``), uploads and downloads overlapping the cycles (include/mg.h)."""
        for t in list(u_hosts) + list(f_hosts):
            assert t.shape == self.shape and not t.is_cuda
        mg_solve_host_batch(self.h, [t.data_ptr() for t in u_hosts], [t.data_ptr() for t in f_hosts], ncycles)

    def profile(self, u, f, ncycles: int = 5):
        return mg_profile(self.h, self._chk(u), self._chk(f), ncycles)

    def convergence_factor(self, e, iters: int = 100):
        """rho-bar of the V-cycle by power iteration from the start error e
        (a device tensor of ``self.shape``, overwritten by the slowest mode)."""
        return mg_convergence_factor(self.h, self._chk(e), iters)

    @property
    def levels(self) -> int:
        return mg_num_levels(self.h)

    def level_points(self, lev: int) -> int:
        return mg_level_points(self.h, lev)

    @property
    def launches_per_cycle(self) -> int:
        return mg_launches_per_cycle(self.h)
