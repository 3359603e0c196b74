"""Host side of the multi-GPU path, on CPU with torch.distributed (gloo,
world_size 2): the slab plan every rank computes independently must tile the
grid consistently, the NCCL id must reach every rank unchanged, and the slab
layout (owned rows + 2 ghost rows) must reassemble the global field."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, fn_name, q):
    import sys
    sys.path.insert(0, ROOT)
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        q.put((rank, globals()[fn_name](rank, world)))
    except Exception as e:  # pragma: no cover - reported to the parent
        q.put((rank, repr(e)))
    finally:
        dist.destroy_process_group()


def _spawn(fn_name, world=2):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, fn_name, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    return out


# ------------------------------------------------------------- rank bodies

def _plan_body(rank, world):
    import torch
    import torch.distributed as dist
    from paper_math_9907190_b200 import build, mg
    build.build()
    res = []
    for dim, sizes in ((2, (65, 129, 1025, 8193)), (3, (33, 65, 513))):
        for n in sizes:
            for ag in (0, 16, 1 << 30):
                lo, hi, g, oa = mg.mg_slab_plan(dim, n, world, rank, ag)
                t = torch.tensor([lo, hi, g, oa], dtype=torch.int64)
                allt = [torch.zeros(4, dtype=torch.int64) for _ in range(world)]
                dist.all_gather(allt, t)
                res.append((dim, n, ag, [x.tolist() for x in allt]))
    return res


def _id_body(rank, world):
    from paper_math_9907190_b200 import build, mg
    build.build()
    return mg.broadcast_nccl_id(None)


def _slab_body(rank, world):
    import torch
    import torch.distributed as dist
    from paper_math_9907190_b200 import build, mg
    from paper_math_9907190_b200 import workloads as W
    build.build()
    n = 129
    full = W.random_field(2, n, seed=7)          # same seeded field on every rank
    lo, hi, g, _ = mg.mg_slab_plan(2, n, world, rank)
    slab = mg.split_rows(full, lo, hi, g)
    own = torch.from_numpy(np.ascontiguousarray(slab[g:g + hi - lo]))
    parts = [torch.zeros_like(own) for _ in range(world)]
    dist.all_gather(parts, own)
    glued = torch.cat(parts).numpy()
    # the ghost rows a rank carries are exactly its neighbours' owned rows
    below = slab[:g]
    above = slab[g + hi - lo:]
    ok_below = np.array_equal(below, full[lo - g:lo]) if lo - g >= 0 else np.all(below[: g - lo] == 0)
    ok_above = np.array_equal(above[: max(0, min(g, n - hi))], full[hi:hi + g][: max(0, min(g, n - hi))])
    return bool(np.array_equal(glued, full[:world * (hi - lo)])), bool(ok_below), bool(ok_above)


def _schedule_body(rank, world):
    import torch
    import torch.distributed as dist
    from paper_math_9907190_b200 import build, mg
    build.build()
    out = []
    for dim, n, P, ag in ((2, 8193, 8, 0), (2, 8193, 2, 0), (2, 257, 8, 0), (2, 257, 8, 16), (2, 1025, 4, 1 << 12),
                          (3, 513, 8, 0), (2, 65, 2, 0)):
        sch, gu = mg.mg_slab_schedule(dim, n, P, ag)
        t = torch.tensor([sch, gu], dtype=torch.int64)
        allt = [torch.zeros(2, dtype=torch.int64) for _ in range(world)]
        dist.all_gather(allt, t)
        out.append(((dim, n, P, ag), [x.tolist() for x in allt]))
    return out


# ------------------------------------------------------------------ tests

def test_slab_plan_is_consistent_across_ranks():
    out = _spawn("_plan_body")
    assert not isinstance(out[0], str), out
    for (dim, n, ag, rows), (_, _, _, rows1) in zip(out[0], out[1]):
        assert rows == rows1
        (lo0, hi0, g0, oa0), (lo1, hi1, g1, oa1) = rows
        assert lo0 == 0 and hi0 == lo1 and hi1 == n - 1          # the slabs tile rows/planes [0, n-1)
        assert hi0 - lo0 == hi1 - lo1 >= 4 and g0 == g1 == 2      # ghosts owned by the neighbour
        assert oa0 == oa1 >= 1                                    # same agglomeration octave
        k = int(np.log2(n - 1))
        agp = ag if ag > 0 else 1 << 18
        # oa is the first octave whose level is below the threshold or too thin to split
        first = next(o for o in range(1, k) if (((n - 1) >> o) - 1) ** dim < agp or ((n - 1) >> o) // 2 < 4) \
            if any((((n - 1) >> o) - 1) ** dim < agp or ((n - 1) >> o) // 2 < 4 for o in range(1, k)) else k - 1
        assert oa0 == first, (dim, n, ag, oa0, first)


def test_nccl_id_reaches_every_rank():
    out = _spawn("_id_body")
    assert isinstance(out[0], bytes) and len(out[0]) == 128
    assert out[0] == out[1]


def test_slabs_reassemble_the_field():
    out = _spawn("_slab_body")
    for r in (0, 1):
        assert out[r] == (True, True, True), out


def test_slab_schedule_is_consistent_and_pinned():
    """Every rank picks the same multi-GPU schedule: the 2D
    communication-avoiding one with the band the stencils' reach gives (hand
    derivation for one distributed octave: the finest ascent reads v_D(1)
    within 2 rows, D(1) colour 1 r_D(1) within 3, the finest descent's band
    rounds to 4 half-row-aligned rows, u within 4 + 2 = 6; at 8193^2 / 8 ranks
    with agglomeration at A(16), 108 rows), the per-level one when the band
    exceeds a slab and always in 3D."""
    out = _spawn("_schedule_body")
    assert not isinstance(out[0], str), out
    want = {(2, 8193, 8, 0): [1, 108], (2, 8193, 2, 0): [1, 108], (2, 257, 8, 0): [1, 6], (2, 257, 8, 16): [0, 2],
            (2, 1025, 4, 1 << 12): [1, 108], (3, 513, 8, 0): [0, 2], (2, 65, 2, 0): [1, 6]}
    for (key, rows), (key1, rows1) in zip(out[0], out[1]):
        assert key == key1 and rows == rows1
        assert rows[0] == rows[1] == want[tuple(key)], (key, rows)
