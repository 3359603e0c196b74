"""The multi-GPU slab solvers over real NCCL: the iterate and the residual
history equal the single-GPU solver's bit for bit.

* several ranks (one process per GPU): whenever at least two CUDA devices are
  visible (the one-GPU boxes of this pool skip it);
* one rank on one GPU (MG_FLAG_SLABS): the slab solver's whole NCCL path runs
  with a one-rank communicator -- on every box.
The multi-rank schedule is also covered by the loopback transport
(tests/test_gpu_dist.py) and the host side by the gloo tests
(tests/test_dist_cpu.py)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
NGPU = torch.cuda.device_count() if torch.cuda.is_available() else 0


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, case, q):
    import sys
    sys.path.insert(0, ROOT)
    import torch.distributed as dist
    from paper_math_9907190_b200 import workloads as W
    from paper_math_9907190_b200.mg import Solver, split_rows
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", rank))
    try:
        dim, n, order, dtype, cycles, agglom = case
        tdt = torch.float64 if dtype == "f64" else torch.float32
        npdt = np.float64 if dtype == "f64" else np.float32
        p = ((1.052 if order == 2 else 1.20),) if dim == 2 else (1.11, 1.42, 1.08, 0.99)
        f = W.random_field(dim, n, seed=5).astype(npdt)
        u0 = (0.1 * W.random_field(dim, n, seed=6)).astype(npdt)
        s = Solver(dim, n, order=order, p=p, dtype=tdt, group=dist.group.WORLD, agglom_points=agglom)
        u = s.alloc(split_rows(u0, s.lo, s.hi, s.ghost))
        ft = s.alloc(split_rows(f, s.lo, s.hi, s.ghost))
        h = s.vcycle(u, ft, cycles, hist=True)
        own = s.view(u)[s.ghost:s.ghost + s.hi - s.lo].contiguous()
        parts = [torch.zeros_like(own) for _ in range(world)]
        dist.all_gather(parts, own)
        if rank == 0:
            glued = torch.cat(parts).cpu().numpy()
            ref = Solver(dim, n, order=order, p=p, dtype=tdt)
            ur, fr = ref.alloc(u0), ref.alloc(f)
            hr = ref.vcycle(ur, fr, cycles, hist=True)
            want = ref.view(ur).cpu().numpy()[: glued.shape[0]]
            q.put((bool(np.array_equal(glued, want)), bool(np.array_equal(h, hr))))
    except Exception as e:  # pragma: no cover - reported to the parent
        if rank == 0:
            q.put(repr(e))
        raise
    finally:
        dist.destroy_process_group()


CASES = [(2, 257, 2, "f64", 3, 0), (2, 257, 2, "f32", 3, 16), (2, 129, 4, "f64", 2, 16),
         (3, 65, 2, "f64", 2, 0), (3, 65, 2, "f64", 2, 16)]


@pytest.mark.skipif(NGPU < 2, reason="needs >= 2 CUDA devices")
@pytest.mark.parametrize("case", CASES, ids=lambda c: f"{c[0]}d{c[1]}o{c[2]}{c[3]}ag{c[5]}")
def test_nccl_slabs_equal_single_gpu(case):
    world = 2 if NGPU < 4 else 4
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, case, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = q.get(timeout=600)
    for p in procs:
        p.join(timeout=120)
    assert res == (True, True), res


@pytest.mark.parametrize("dim,n,order,dtype,env", [
    (2, 257, 2, "f64", {}), (2, 257, 4, "f64", {}), (2, 513, 2, "f32", {}),
    (2, 257, 2, "f64", {"MG_DIST_PERLEVEL": "1"}), (2, 1025, 2, "f64", {"MG_DIST_NOFUSE": "1"}),
    (3, 65, 2, "f64", {}), (3, 65, 4, "f64", {})])
def test_nccl_transport_single_rank(dim, n, order, dtype, env):
    """The NCCL transport on one GPU (MG_FLAG_SLABS, a one-rank communicator):
    the slab solver runs its whole NCCL path -- unique id, communicator, the
    grouped send/recv rounds (empty: no neighbours), the in-place all-gather,
    the norm all-reduces, all captured in CUDA graphs, and the asynchronous
    error poll -- and must equal the single-GPU solver bit for bit."""
    import os
    from paper_math_9907190_b200 import workloads as W
    from paper_math_9907190_b200.mg import Solver, split_rows
    tdt = torch.float64 if dtype == "f64" else torch.float32
    npdt = np.float64 if dtype == "f64" else np.float32
    p = ((1.052 if order == 2 else 1.20),) if dim == 2 else (1.11, 1.42, 1.08, 0.99)
    f = W.random_field(dim, n, seed=11).astype(npdt)
    u0 = (0.1 * W.random_field(dim, n, seed=12)).astype(npdt)
    ref = Solver(dim, n, order=order, p=p, dtype=tdt)
    ur, fr = ref.alloc(u0), ref.alloc(f)
    href, l2ref = ref.vcycle(ur, fr, 4, l2=True)
    want = ref.view(ur).cpu().numpy()
    os.environ.update(env)
    try:
        s = Solver(dim, n, order=order, p=p, dtype=tdt, slabs=True)
    finally:
        for key in env:
            os.environ.pop(key, None)
    assert (s.lo, s.hi, s.ghost) == (0, n - 1, 2)
    u = s.alloc(split_rows(u0, s.lo, s.hi, s.ghost))
    ft = s.alloc(split_rows(f, s.lo, s.hi, s.ghost))
    h, l2 = s.vcycle(u, ft, 4, l2=True)
    got = s.view(u)[s.ghost:s.ghost + n - 1].cpu().numpy()
    assert np.array_equal(got, want[: n - 1])
    assert np.array_equal(h, href)
    np.testing.assert_allclose(l2, l2ref, rtol=1e-12)
    s.vcycle(u, ft, 2)   # graph replay of the captured NCCL cycle
    ref.vcycle(ur, fr, 2)
    torch.cuda.synchronize()
    assert np.array_equal(s.view(u)[s.ghost:s.ghost + n - 1].cpu().numpy(), ref.view(ur).cpu().numpy()[: n - 1])
