"""Every alternative code path of the library is bit-identical to the oracle.

The library chooses between kernel variants once per process from environment
switches (fused vs separate level passes, cooperative tail on/off, first- vs
second-generation 3D kernels, the reference kernels).  Each case below runs a
small problem in a fresh subprocess with one switch set and asserts the
iterates and the residual history equal the CPU oracle's bit for bit.
"""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r"""
import json, sys
import numpy as np
sys.path.insert(0, {root!r})
import oracle
from paper_math_9907190_b200 import workloads as W
from paper_math_9907190_b200.mg import Solver
import torch
dim, n, order, dtype = {dim}, {n}, {order}, np.{dtype}
p = (1.052,) if dim == 2 else (1.11, 1.42, 1.08, 0.99)
if order == 4 and dim == 2:
    p = (1.20,)
f = W.random_field(dim, n, seed=7).astype(dtype)
u0 = (W.random_field(dim, n, seed=8) * 0.1).astype(dtype)
s = Solver(dim, n, order=order, p=p, dtype=torch.float64 if dtype == np.float64 else torch.float32)
u = s.alloc(u0)
ft = s.alloc(f)
h = s.vcycle(u, ft, 3, hist=True)
ug = s.view(u).cpu().numpy()
uo = u0.copy()
ho = oracle.vcycle(uo, f, p, 3, order=order, hist=True)
from paper_math_9907190_b200 import mg as MG
rc = MG.load().mg_destroy(s.h)   # MG_POISON: nonzero if a guard band was overwritten
s.h = None
print(json.dumps({{"bitwise": bool(np.array_equal(ug, uo)), "hist": bool(np.array_equal(h, ho)),
                  "rel": float(np.max(np.abs(ug.astype(np.float64) - uo)) / np.max(np.abs(uo))),
                  "destroy_rc": int(rc)}}))
"""

CASES = [
    # (env, dim, n, order, dtype)
    ({}, 3, 129, 2, "float64"),
    ({"MG_K3_FUSE": "1"}, 3, 129, 2, "float64"),
    ({"MG_K3_FUSE": "1"}, 3, 257, 2, "float64"),
    ({"MG_TAIL_M3": "0"}, 3, 129, 2, "float64"),
    ({"MG_TAIL_M3": "128"}, 3, 129, 2, "float64"),
    ({"MG_TAIL_M3": "64"}, 3, 257, 2, "float64"),   # round 2 session 3 default
    ({"MG_K3_GEN1": "1"}, 3, 65, 2, "float64"),
    ({"MG_K3_GEN1": "1"}, 3, 65, 4, "float64"),
    ({"MG_K3_GEN1": "1"}, 3, 129, 4, "float32"),
    ({}, 3, 129, 4, "float64"),
    ({}, 3, 129, 4, "float32"),
    ({"MG_K3S_NOF32": "1"}, 3, 129, 2, "float32"),   # round 1's fp32 sublattice kernels (k3l.cu)
    # levels with M <= 128 on the k3l.cu kernels is the default; 0 keeps every octave on the plane pipelines
    ({"MG_K3_GEN1_M": "0"}, 3, 129, 2, "float64"),
    ({"MG_K3_GEN1_M": "0"}, 3, 129, 4, "float64"),
    ({"MG_K3_GEN1_M": "0", "MG_POISON": "1"}, 3, 257, 2, "float32"),
    ({"MG_K3_GEN1_MD": "256"}, 3, 257, 2, "float64"),   # octave 1's restrictions on k3l.cu as well
    ({"MG_K3L_PDL": "1"}, 3, 257, 2, "float64"),   # k3l.cu level kernels launched programmatically
    ({"MG_K3_GEN1_MD": "256"}, 3, 257, 2, "float32"),
    ({"MG_K3_GEN1_M": "256", "MG_TAIL_M3": "0"}, 3, 257, 4, "float64"),
    ({"MG_AD_NOQUAD": "1"}, 2, 513, 2, "float32"),   # two-column fp32 jac_ad
    ({"MG_DA_NOQUAD": "1"}, 2, 513, 2, "float32"),   # two-column fp32 rest_dad
    ({"MG_DA_NOQUAD": "1", "MG_AD_NOQUAD": "1"}, 2, 1025, 4, "float32"),
    ({"MG_AD_NOQUAD": "1"}, 2, 257, 4, "float32"),
    ({"MG_K3_FUSE_MR": "1", "MG_K3_FUSE_RMG": "2"}, 3, 129, 2, "float64"),
    ({"MG_K3_FUSE_MR": "2"}, 3, 257, 2, "float64"),
    ({"MG_K3R_NW": "8", "MG_K3S_NW": "16"}, 3, 129, 2, "float32"),
    ({"MG_POISON": "1"}, 3, 129, 2, "float32"),
    ({"MG_FORCE_REF": "1"}, 3, 33, 2, "float64"),
    ({"MG_COARSE_GLOBAL": "1", "MG_TAIL_M3": "0"}, 3, 65, 2, "float64"),
    ({"MG_TAIL_M2": "128"}, 2, 513, 2, "float64"),
    ({"MG_STAGES": "3"}, 2, 513, 2, "float64"),
    ({"MG_COARSE_GLOBAL": "1", "MG_COARSE_NOCT": "1"}, 2, 257, 2, "float64"),
    ({"MG_COARSE_NOCT": "1"}, 2, 513, 2, "float64"),
    ({"MG_COARSE_NOCT": "1"}, 2, 257, 4, "float32"),
    ({"MG_FORCE_REF": "1"}, 2, 129, 4, "float64"),
    ({"MG_PDL": "1"}, 2, 257, 2, "float64"),
    ({"MG_PDL": "1"}, 3, 65, 2, "float64"),
    ({"MG_2D_NOSERP": "1"}, 2, 513, 2, "float64"),
    ({"MG_PDL_SMALL": "0"}, 2, 513, 2, "float64"),
    ({"MG_2D_NOXFUSE": "1"}, 2, 513, 2, "float64"),
    ({"MG_2D_NOXFUSE": "1"}, 2, 257, 4, "float32"),
    ({"MG_XF_PAIRS": "1"}, 2, 513, 2, "float32"),
    ({"MG_2D_NOADFUSE": "1"}, 2, 513, 2, "float64"),
    ({"MG_2D_NOADFUSE": "1"}, 2, 257, 4, "float32"),
    ({"MG_AD_MINO": "2"}, 2, 513, 2, "float64"),
    ({"MG_AD_TY": "32", "MG_AD_NT": "256"}, 2, 1025, 4, "float32"),
    ({"MG_AD_TY": "8"}, 2, 513, 2, "float64"),
    ({"MG_AD_NT": "576"}, 2, 513, 2, "float32"),
    ({"MG_2D_XRD": "1"}, 2, 513, 2, "float64"),
    ({"MG_2D_XRD": "1"}, 2, 1025, 2, "float32"),
    ({"MG_2D_XRD": "1"}, 2, 257, 4, "float32"),
    ({"MG_2D_XRD": "1", "MG_POISON": "1"}, 2, 257, 2, "float64"),
    ({"MG_2D_NODAFUSE": "1"}, 2, 513, 2, "float64"),
    ({"MG_2D_NODAFUSE": "1"}, 2, 257, 4, "float32"),
    ({"MG_DA_MINO": "1"}, 2, 513, 2, "float32"),
    ({"MG_DA_NT": "576"}, 2, 513, 2, "float32"),
    ({"MG_DA_NT": "256"}, 2, 513, 4, "float64"),
    ({"MG_DA_MINO": "2", "MG_AD_MINO": "3"}, 2, 1025, 2, "float64"),
    ({"MG_3D_NOSERP": "1"}, 3, 129, 2, "float64"),
    ({"MG_K3_NW": "8"}, 3, 129, 2, "float64"),
    ({"MG_K3_NW": "8", "MG_K3_NWL": "8"}, 3, 257, 2, "float64"),
    ({"MG_K3_NW": "8"}, 3, 65, 2, "float32"),
    ({"MG_K3_NW": "16"}, 3, 129, 2, "float64"),
    ({"MG_K3S_NW": "16"}, 3, 129, 2, "float64"),
    ({"MG_K3S_NW": "8"}, 3, 257, 2, "float64"),
    ({"MG_K3R_NW": "8"}, 3, 129, 2, "float64"),
    ({"MG_K3R_NW": "8", "MG_K3_NWL": "8"}, 3, 257, 2, "float64"),
    # bounds checks of our own (compute-sanitizer is closed on the B200 pool): level arrays with
    # poisoned (NaN) guard rows and pitch padding; a stray read makes the iterate NaN, a stray
    # write trips the guard check in mg_destroy
    ({"MG_POISON": "1"}, 2, 257, 2, "float64"),
    ({"MG_POISON": "1"}, 2, 257, 4, "float64"),
    ({"MG_POISON": "1"}, 2, 513, 2, "float32"),
    ({"MG_POISON": "1"}, 2, 129, 4, "float32"),
    ({"MG_POISON": "1"}, 3, 129, 2, "float64"),
    ({"MG_POISON": "1"}, 3, 65, 4, "float64"),
    ({"MG_POISON": "1"}, 3, 65, 2, "float32"),
    ({"MG_POISON": "1", "MG_FORCE_REF": "1"}, 2, 65, 2, "float64"),
    ({"MG_POISON": "1", "MG_FORCE_REF": "1"}, 3, 33, 2, "float64"),
    ({"MG_POISON": "1", "MG_K3_FUSE": "1"}, 3, 129, 2, "float64"),
    ({"MG_POISON": "1", "MG_2D_NOXFUSE": "1", "MG_2D_NOADFUSE": "1", "MG_2D_NODAFUSE": "1"}, 2, 257, 2, "float64"),
]


# switches of the plane-pipeline small-level passes: tested with every octave on the pipelines
_PIPE_KEYS = ("MG_K3_FUSE", "MG_K3_FUSE_MR", "MG_K3_FUSE_RMG", "MG_K3S_NW", "MG_K3R_NW", "MG_K3_NWL")
CASES = [({**e, "MG_K3_GEN1_M": "0"} if d == 3 and any(k in e for k in _PIPE_KEYS) else e, d, n, o, t)
         for e, d, n, o, t in CASES]


@pytest.mark.parametrize("env,dim,n,order,dtype", CASES,
                         ids=[f"{'+'.join(f'{k}={v}' for k, v in e.items()) or 'default'}-{d}d{n}o{o}"
                              for e, d, n, o, _ in CASES])
def test_path_is_bit_identical(env, dim, n, order, dtype):
    code = CHILD.format(root=ROOT, dim=dim, n=n, order=order, dtype=dtype)
    full_env = dict(os.environ)
    full_env.update(env)
    out = subprocess.run([sys.executable, "-c", code], env=full_env, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    res = json.loads(out.stdout.strip().splitlines()[-1])
    assert res["bitwise"], res
    assert res["hist"], res
    assert res["destroy_rc"] == 0, res


def test_poison_guard_check_has_teeth():
    """MG_POISON_SELFTEST plants one stray byte in the pitch padding of the
    first level array: mg_destroy must report it (the guard check is live)."""
    code = CHILD.format(root=ROOT, dim=2, n=65, order=2, dtype="float64")
    env = dict(os.environ, MG_POISON="1", MG_POISON_SELFTEST="1")
    out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    res = json.loads(out.stdout.strip().splitlines()[-1])
    assert res["bitwise"] and res["destroy_rc"] != 0, res
    assert "guard bytes" in out.stderr
