"""Pins of the CPU oracle against what the paper and mathematics fix (CPU only).

Each test names the passage it pins and the kind of pin (closed form,
invariant, special case, library routine, paper value, hand-derived worked
example).  None of them re-types the oracle's formula.
"""
import itertools
import os
from fractions import Fraction

import numpy as np
import pytest

import oracle
from paper_math_9907190_b200 import workloads as W
from tests import _exact

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
DTYPES = [np.float64, np.float32]


def _load(name):
    rows = []
    with open(os.path.join(GOLDEN, name)) as fh:
        for line in fh:
            line = line.strip()
            if line and not line.startswith("#"):
                rows.append(line.split())
    return rows


# ------------------------------------------------------------------ levels

@pytest.mark.parametrize("dim,n,expected", [
    (2, 5, 3), (2, 17, 7), (2, 65, 11), (2, 1025, 19), (2, 8193, 25),
    (3, 5, 4), (3, 17, 10), (3, 65, 16), (3, 513, 25)])
def test_level_count(dim, n, expected):
    """2k-1 levels in 2D (spacing h 2^(l/2)); 3k-2 in 3D
    (G,R,M per octave); coarsest has one interior node."""
    assert oracle.levels(dim, n) == expected
    assert oracle.count(dim, n, expected - 1) == 1


def test_invalid_sizes():
    for n in (4, 6, 3, 1, 0, 100):
        assert oracle.levels(2, n) == -1
    assert oracle.levels(4, 17) == -1


@pytest.mark.parametrize("dim,n", [(2, 5), (2, 17), (2, 65), (3, 5), (3, 17), (3, 33)])
def test_node_counts_closed_form(dim, n):
    """Interior node counts of every level by the closed-form counting rule
    (A(s): m^2, D(s): (m^2+1)/2, G: m^3, R: e^3+3e o^2, M: e^3+o^3 with
    m=(n-1)/s-1, o=(m+1)/2, e=(m-1)/2); node sets from P:117-125, 422-425,
    454-458, 504-505.  Nodes halve per level."""
    for lev in range(oracle.levels(dim, n)):
        s_m = oracle.lattice(dim, n, lev)
        m = s_m - 1
        o, e = (m + 1) // 2, (m - 1) // 2
        cls = lev % 2 if dim == 2 else lev % 3
        if dim == 2:
            want = m * m if cls == 0 else (m * m + 1) // 2
        else:
            want = [m ** 3, e ** 3 + 3 * e * o * o, e ** 3 + o ** 3][cls]
        assert oracle.count(dim, n, lev) == want


# ------------------------------------------------------------- restriction

def _delta(shape, idx, dtype=np.float64):
    a = np.zeros(shape, dtype=dtype)
    a[idx] = 1.0
    return a


@pytest.mark.parametrize("dtype", DTYPES)
def test_restriction_preserves_constants(dtype):
    """Every restriction is a weighted average: weights sum to 1
    (Fig. 2).  A constant is reproduced at every node
    whose stencil is interior."""
    for dim, n in ((2, 33), (3, 17)):
        for lev in range(oracle.levels(dim, n) - 1):
            shp = oracle.level_shape(dim, n, lev)
            m = shp[0] - 1
            rin = np.zeros(shp, dtype=dtype)
            # constant on all nodes of the level (masking is the oracle's job:
            # the input carries the constant everywhere, only level nodes are read)
            rin[(slice(1, -1),) * dim] = 3.0
            out = oracle.restrict(dim, n, lev, rin)
            mo = out.shape[0] - 1
            inner = (slice(2, mo - 1),) * dim if mo >= 4 else None
            if inner is None:
                continue
            vals = out[inner]
            cls = lev % 2 if dim == 2 else lev % 3
            # nodes of the target level inside `inner`
            idx = np.argwhere(np.ones(vals.shape, bool)) + 2
            for I in idx:
                I = tuple(int(t) for t in I)
                on = True
                if dim == 2 and cls == 0:
                    on = sum(I) % 2 == 0
                if dim == 3 and cls == 0:
                    on = sum(I) % 2 == 0
                if dim == 3 and cls == 1:
                    on = len({t % 2 for t in I}) == 1
                if on:
                    assert out[I[::-1]] == pytest.approx(3.0, rel=1e-6), (dim, lev, I)


def test_restriction_delta_2d():
    """delta at an axis-only node -> 1/8 at its 4 diagonal-
    level axis neighbours; delta at a diagonal node -> 1/2 there (Erest2r,
    P:166-170); delta at a diagonal-only node -> 1/8 at its 4 coarse
    diagonal neighbours (Erest2b)."""
    n = 17
    # level 0 (A(1)) -> level 1 (D(1))
    out = oracle.restrict(2, n, 0, _delta((n, n), (6, 5)))  # node (i=5, j=6): i+j odd -> axis-only
    nz = {(int(j), int(i)): out[j, i] for j, i in np.argwhere(out != 0)}
    assert nz == {(6, 4): 0.125, (6, 6): 0.125, (5, 5): 0.125, (7, 5): 0.125}
    out = oracle.restrict(2, n, 0, _delta((n, n), (6, 6)))
    nz = {(int(j), int(i)): out[j, i] for j, i in np.argwhere(out != 0)}
    assert nz == {(6, 6): 0.5}
    # level 1 (D(1)) -> level 2 (A(2)): diagonal-only node (5,7) (both odd)
    out = oracle.restrict(2, n, 1, _delta((n, n), (7, 5)))
    nz = {(int(j), int(i)): out[j, i] for j, i in np.argwhere(out != 0)}
    # coarse neighbours at fine (4,6),(6,6),(4,8),(6,8) -> coarse (2,3),(3,3),(2,4),(3,4)
    assert nz == {(3, 2): 0.125, (3, 3): 0.125, (4, 2): 0.125, (4, 3): 0.125}


def test_restriction_delta_3d():
    """Erred delta at a green-only node gives
    1/12 at its red neighbours, 1/2 at a red node; Ermagc/Ermagm
    delta at a face centre gives 1/24 at adjacent corners and 1/6 at the two
    adjacent centres; Erblu delta at a centre gives 1/16 at its 8
    corners."""
    n = 17
    sh = (n, n, n)
    out = oracle.restrict(3, n, 0, _delta(sh, (4, 4, 5)))  # (i=5,j=4,k=4): odd sum, green-only
    nz = {tuple(int(t) for t in x[::-1]): out[tuple(x)] for x in np.argwhere(out != 0)}
    assert nz == {(4, 4, 4): 1 / 12, (6, 4, 4): 1 / 12, (5, 5, 4): 1 / 12, (5, 3, 4): 1 / 12,
                  (5, 4, 5): 1 / 12, (5, 4, 3): 1 / 12}
    out = oracle.restrict(3, n, 0, _delta(sh, (4, 4, 4)))
    assert out[4, 4, 4] == 0.5 and np.count_nonzero(out) == 1
    # red face centre (i=5,j=5,k=4) (normal z) -> magenta
    out = oracle.restrict(3, n, 1, _delta(sh, (4, 5, 5)))
    nz = {tuple(int(t) for t in x[::-1]): out[tuple(x)] for x in np.argwhere(out != 0)}
    corners = {(4, 4, 4), (6, 4, 4), (4, 6, 4), (6, 6, 4)}
    centres = {(5, 5, 3), (5, 5, 5)}
    assert set(nz) == corners | centres
    for c in corners:
        assert nz[c] == pytest.approx(1 / 24, rel=1e-15)
    for c in centres:
        assert nz[c] == pytest.approx(1 / 6, rel=1e-15)
    # magenta centre (5,5,5) -> blue (G(2)) corners
    out = oracle.restrict(3, n, 2, _delta(sh, (5, 5, 5)))
    nz = {tuple(int(t) for t in x[::-1]): out[tuple(x)] for x in np.argwhere(out != 0)}
    assert set(nz) == {(a, b, c) for a in (2, 3) for b in (2, 3) for c in (2, 3)}
    assert all(v == 1 / 16 for v in nz.values())


def _composite_weights(dim):
    rows = [r for r in _load("composite_stencils.txt") if int(r[0]) == dim]
    return {tuple(int(t) for t in r[1].split(",")): Fraction(int(r[2]), int(r[3])) for r in rows}, \
        {tuple(int(t) for t in r[1].split(",")): int(r[4]) for r in rows}


@pytest.mark.parametrize("dim", [2, 3])
def test_composite_restriction(dim):
    """The restriction from one axis/green grid to the next coarser one, via the
    intermediate diagonal grids, is the 17-point (2D) / 123-point
    (3D) composite stencil derived in SURVEY 8(c).5 P2/P3 (golden file)."""
    n = 17 if dim == 2 else 17
    steps = 2 if dim == 2 else 3
    R = 3 if dim == 3 else 2
    weights, counts = _composite_weights(dim)
    centre = (8,) * dim                     # a node of the coarser axis grid, fine index
    coarse = tuple(c // 2 for c in centre)
    seen = {}
    for off in itertools.product(range(-R, R + 1), repeat=dim):
        src = tuple(c + o for c, o in zip(centre, off))
        r = _delta((n,) * dim, src[::-1])
        for lev in range(steps):
            r = oracle.restrict(dim, n, lev, r)
        w = Fraction(float(r[coarse[::-1]])).limit_denominator(1 << 20)
        if w != 0:
            cls = tuple(sorted(abs(o) for o in off))
            seen.setdefault(cls, []).append(w)
    assert set(seen) == set(weights)
    for cls, ws in seen.items():
        assert len(ws) == counts[cls]
        assert all(w == weights[cls] for w in ws)
    total = sum(weights[c] * counts[c] for c in weights)
    assert total == 1
    assert sum(counts.values()) == (17 if dim == 2 else 123)


# ------------------------------------------------------------------ Jacobi

def _quadratic(rng, dim):
    a = rng.integers(-3, 4, size=(dim, dim)).astype(float)
    a = (a + a.T) / 2
    b = rng.integers(-3, 4, size=dim).astype(float)
    c = float(rng.integers(-3, 4))
    return a, b, c


def _qval(q, X):
    a, b, c = q
    return np.einsum("...i,ij,...j->...", X, a, X) + X @ b + c


@pytest.mark.parametrize("dim", [2, 3])
def test_jacobi_exact_on_quadratics(dim):
    """Every Jacobi formula is exact on quadratics: with the
    coarser values and the same-level neighbours sampled from a quadratic q
    and r = Lap q, each update returns q.  Pins the coefficients -kappa p h^2
    (2h^2 on diagonal grids; h^2 on axis grids; 4,2,4,1 h^2 in 3D,
    P:556-661) and weights, at p = 1; with p != 1 the update moves by exactly
    -(p-1) kappa h^2 Lap q / W.  Checked at nodes away from the boundary."""
    rng = np.random.default_rng(7)
    n = 17
    for lev in range(oracle.levels(dim, n) - 1):
        m = oracle.lattice(dim, n, lev)
        s = (n - 1) // m
        h = 1.0 / (n - 1)
        q = _quadratic(rng, dim)
        lap = 2 * np.trace(q[0])
        sh = (m + 1,) * dim
        grid = np.stack(np.meshgrid(*([np.arange(m + 1) * s * h] * dim), indexing="ij")[::-1], -1)
        qv = _qval(q, grid)                       # q at every lattice node, [k,j,i]
        mc = oracle.lattice(dim, n, lev + 1)
        sc = (n - 1) // mc
        gc = np.stack(np.meshgrid(*([np.arange(mc + 1) * sc * h] * dim), indexing="ij")[::-1], -1)
        vc = _qval(q, gc)
        inner = (slice(1, -1),) * dim
        r = np.zeros(sh)
        r[inner] = lap
        vcz = np.zeros_like(vc)
        vcz[(slice(1, -1),) * dim] = vc[(slice(1, -1),) * dim]
        # nodes whose whole dependency cone stays interior: 3 lattice points from the boundary
        core = (slice(3, m - 2),) * dim
        if m < 8:
            continue
        for p in (1.0, 1.3):
            pp = p if dim == 2 else (p, p, p, p)
            v = oracle.jacobi(dim, n, lev, pp, vc, r)
            # only nodes of the level are written
            want = qv[core]
            got = v[core]
            mask = got != 0
            assert mask.any()
            if p == 1.0:
                assert np.allclose(got[mask], want[mask], rtol=0, atol=1e-12), (dim, lev)
            else:
                # the change from p=1 is linear in (p-1) and nonzero wherever a node was updated
                v1 = oracle.jacobi(dim, n, lev, 1.0 if dim == 2 else (1.0,) * 4, vc, r)
                assert np.all(np.abs(v[core] - v1[core])[mask] > 0)


def test_jacobi_delta_responses():
    """SPEC S:170 / S:260 / S:270 / S:280: coarse delta, r = 0.
    2D diagonal grid: 1/4 at the 4 new nodes, then 1/4 back at the coarse
    node (Ejacr/Ejacb).  3D magenta: 1/8 at the 8 centres, then
    1/8 at the corner.  3D red: 1/4 at each face centre whose
    normal pair contains the magenta centre."""
    n = 17
    vc = np.zeros((9, 9))
    vc[4, 4] = 1.0                       # A(2) node -> fine (8,8)
    v = oracle.jacobi(2, n, 1, 1.0, vc, np.zeros((n, n)))
    for dj, di in itertools.product((-1, 1), repeat=2):
        assert v[8 + dj, 8 + di] == 0.25
    assert v[8, 8] == 0.25
    # 3D magenta from G(2)
    vc = np.zeros((9, 9, 9))
    vc[4, 4, 4] = 1.0
    v = oracle.jacobi(3, n, 2, (1, 1, 1, 1), vc, np.zeros((n,) * 3))
    for d in itertools.product((-1, 1), repeat=3):
        assert v[8 + d[2], 8 + d[1], 8 + d[0]] == 0.125
    assert v[8, 8, 8] == 0.125
    # 3D red from magenta: delta at the magenta centre (9,9,9)
    vm = np.zeros((n,) * 3)
    vm[9, 9, 9] = 1.0
    v = oracle.jacobi(3, n, 1, (1, 1, 1, 1), vm, np.zeros((n,) * 3))
    for ax in range(3):
        for sgn in (-1, 1):
            idx = [9, 9, 9]
            idx[ax] += sgn
            assert v[idx[2], idx[1], idx[0]] == 0.25
    # magenta centres are not red nodes and are not updated
    assert v[9, 9, 9] == 0.0


@pytest.mark.parametrize("dim", [2, 3])
def test_coarsest_exact_at_p1(dim):
    """A single interior unknown: one Jacobi step from zero is the exact solve
    of the coarsest green/axis grid equation Lap_H v = r at p = 1 (SPEC S:99,
    reading A4)."""
    for n in (5, 17):
        L = oracle.levels(dim, n)
        r = np.zeros((3,) * dim)
        r[(1,) * dim] = 0.7
        v = oracle.coarsest(dim, n, 1.0 if dim == 2 else (1,) * 4, r)
        H = 1.0 / 2
        # exact: (0 * nbrs - 2d v)/H^2 = r
        assert v[(1,) * dim] == pytest.approx(-0.7 * H * H / (2 * dim), rel=1e-15)
        assert L >= 3


# ---------------------------------------------------------- worked examples

@pytest.mark.parametrize("dtype", DTYPES)
def test_worked_examples_n5(dtype):
    """Hand-derived exact rationals after one cycle at n=5 (SURVEY 8(c).6,
    golden/worked_n5.txt).  The 2D values are dyadic, so bit-exact in fp32
    and fp64; the 3D ones carry factors of 3 (weights 1/6, 1/12, 1/24) and are
    matched to the precision's rounding."""
    rows = _load("worked_n5.txt")
    for dim in (2, 3):
        n = 5
        u = np.zeros((n,) * dim, dtype=dtype)
        f = np.zeros((n,) * dim, dtype=dtype)
        f[(2,) * dim] = 1.0
        oracle.vcycle(u, f, 1.0 if dim == 2 else (1, 1, 1, 1), 1)
        for r in rows:
            if int(r[0]) != dim:
                continue
            pt = tuple(int(t) for t in r[1:1 + dim])
            num, den = int(r[1 + dim]), int(r[2 + dim])
            if dim == 2:
                assert Fraction(float(u[pt[::-1]])) == Fraction(num, den), (dim, pt)
            else:
                eps = np.finfo(dtype).eps
                assert float(u[pt[::-1]]) == pytest.approx(num / den, rel=16 * eps), (dim, pt)


def test_error_mode_contracts_by_3_64():
    """at n=5 the D4-symmetric error mode
    (centre 1, edges 1, corners 1/2) contracts by exactly 3/64 per cycle (p=1).
    Checked through the exact discrete solution: e_{k+1} = (3/64) e_k."""
    n = 5
    f = np.zeros((n, n))
    f[2, 2] = 1.0
    uex = _exact.exact_solution(f)
    u = np.zeros((n, n))
    errs = []
    for _ in range(4):
        oracle.vcycle(u, f, 1.0, 1)
        errs.append(u - uex)
    for a, b in zip(errs, errs[1:]):
        assert np.allclose(b, a * 3 / 64, rtol=0, atol=1e-15)


# --------------------------------------------------------- fixed point/exact

@pytest.mark.parametrize("dim,n,order", [(2, 65, 2), (2, 65, 4), (3, 17, 2), (3, 17, 4), (2, 17, 2), (3, 9, 2)])
def test_residual_matches_dst_operator(dim, n, order):
    """The finest residual is f - L u (Evpois P:62-67; Efos2 P:311-321; Efos4
    P:724-745): for u = the exact DST-I solution of L u = f (library routine),
    r vanishes; for arbitrary u, r = f~ - L u with L applied spectrally."""
    f = W.random_field(dim, n, seed=11)
    uex = _exact.exact_solution(f, order)
    r = oracle.residual(uex, f, order)
    assert np.max(np.abs(r)) < 1e-9 * np.max(np.abs(f)) * (n - 1) ** 0.5
    u = W.random_field(dim, n, seed=12)
    r = oracle.residual(u, f, order)
    ft = _exact.apply_operator(_exact.exact_solution(f, order), order)  # = f~ on the interior
    want = ft - _exact.apply_operator(u, order)
    assert np.max(np.abs(r - want)) < 1e-9 * np.max(np.abs(want))


@pytest.mark.parametrize("dim,n", [(2, 9), (2, 17), (3, 9)])
def test_dense_solve_fixed_point(dim, n):
    """Exact discrete solution by a dense direct solve of the textbook
    Kronecker-sum Laplacian (BASELINE north_star): it is a fixed
    point of the V-cycle, and 12 cycles from 0 reach it to ~1e-12."""
    f = W.random_field(dim, n, seed=3)
    A = _exact.dense_laplacian(dim, n)
    inner = (slice(1, -1),) * dim
    uex = np.zeros_like(f)
    uex[inner] = np.linalg.solve(A, f[inner].ravel()).reshape((n - 2,) * dim)
    p = 1.052 if dim == 2 else (1.11, 1.42, 1.08, 0.99)
    u = uex.copy()
    oracle.vcycle(u, f, p, 1)
    assert np.max(np.abs(u - uex)) < 1e-13 * np.max(np.abs(uex))
    u = np.zeros_like(f)
    oracle.vcycle(u, f, p, 12)
    assert np.max(np.abs(u - uex)) < 1e-11 * np.max(np.abs(uex))


@pytest.mark.parametrize("name", ["2d_65", "3d_65"])
def test_manufactured_recovery(name):
    """BASELINE configs[0]/[3] without noise: f = L_h u* gives the discrete
    solution exactly u* (closed form); 10 cycles recover it to rho^10."""
    w = W.WORKLOADS[name]
    ustar = W.manufactured_u(w.dim, w.n)
    f = W.discrete_laplacian(ustar)
    u = np.zeros_like(f)
    hist = oracle.vcycle(u, f, w.p, 10, hist=True)
    assert np.max(np.abs(u - ustar)) < 1e-10
    assert hist[-1] < 1e-8 * hist[0]


@pytest.mark.parametrize("name", ["2d_65", "3d_65"])
def test_config_converges_to_dst_solution(name):
    """BASELINE configs[0]/[3] with noise: after 10 cycles the iterate equals
    the exact discrete solution (DST-I) to <= ~rho^10."""
    w = W.WORKLOADS[name]
    f = W.workload_rhs(name)
    uex = _exact.exact_solution(f)
    u = np.zeros_like(f)
    oracle.vcycle(u, f, w.p, w.cycles)
    assert np.max(np.abs(u - uex)) / np.max(np.abs(uex)) < 1e-11


# ----------------------------------------------------------------- rates

def _rho(dim, n, p, order):
    from scipy.sparse.linalg import LinearOperator, eigs
    N = (n - 2) ** dim
    inner = (slice(1, -1),) * dim
    f = np.zeros((n,) * dim)

    def mv(x):
        u = np.zeros((n,) * dim)
        u[inner] = x.reshape((n - 2,) * dim)
        oracle.vcycle(u, f, p, 1, order=order)
        return u[inner].ravel()

    A = LinearOperator((N, N), matvec=mv, dtype=np.float64)
    w = eigs(A, k=2, which="LM", return_eigenvectors=False, tol=1e-8)
    return float(max(abs(w)))


@pytest.mark.parametrize("row", _load("paper_tables.txt"), ids=lambda r: "-".join(r[:4]))
def test_convergence_factor_matches_paper(row):
    """Largest eigenvalue of the V-cycle iteration operator, by a sparse
    eigen-solver as in the paper (MATLAB's sparse eigenvalue
    routine), against Tables 1-3."""
    dim, n, order = int(row[0]), int(row[1]), int(row[2])
    p = [float(t) for t in row[3].split(",")]
    p = p[0] if dim == 2 else tuple(p)
    want, tol = float(row[4]), float(row[5])
    assert _rho(dim, n, p, order) == pytest.approx(want, abs=tol)


@pytest.mark.parametrize("row", _load("paper_tables.txt"), ids=lambda r: "-".join(r[:4]))
def test_power_iteration_matches_paper(row):
    """The oracle's power iteration (oracle.convergence_factor, the reference
    of the GPU's mg_convergence_factor) reproduces Tables 1-3 (P:292-298,
    709-712, 786-792) within the same windows as the ARPACK eigenvalue."""
    dim, n, order = int(row[0]), int(row[1]), int(row[2])
    p = [float(t) for t in row[3].split(",")]
    p = p[0] if dim == 2 else tuple(p)
    want, tol = float(row[4]), float(row[5])
    rho, ratios = oracle.convergence_factor(W.random_field(dim, n, seed=3), p, 200, order=order)
    assert rho == pytest.approx(want, abs=tol)
    assert len(ratios) == 200 and np.all(ratios > 0)


def test_power_iteration_agrees_with_arpack():
    """Where the dominant eigenvalue is real and separated, the power-iteration
    ratio converges to ARPACK's spectral radius (an independent route)."""
    for dim, n, p, order in [(2, 33, 1.0, 2), (3, 9, (1.0, 1.0, 1.0, 1.0), 2)]:
        rho, _ = oracle.convergence_factor(W.random_field(dim, n, seed=4), p, 300, order=order)
        assert rho == pytest.approx(_rho(dim, n, p, order), rel=5e-3)


def test_extra_sweeps_variant():
    """NEXT-4 oracle variant (reading A19): sweeps = 1 is the V-cycle itself;
    more sweeps keep the cycle linear, leave the exact discrete solution a
    fixed point, and at p = 1 lower rho-bar (0.099 -> ~0.047, 2D 65^2)."""
    n = 33
    f = W.random_field(2, n, seed=4)
    u1, u2 = np.zeros_like(f), np.zeros_like(f)
    oracle.vcycle(u1, f, 1.052, 3)
    oracle.vcycle(u2, f, 1.052, 3, sweeps=1)
    assert np.array_equal(u1, u2)
    a, b = W.random_field(2, n, seed=1), W.random_field(2, n, seed=2)
    z = np.zeros_like(a)
    ua, ub, uab = a.copy(), b.copy(), 2 * a + 3 * b
    for u in (ua, ub, uab):
        oracle.vcycle(u, z, 1.0, 1, sweeps=3)
    np.testing.assert_allclose(uab, 2 * ua + 3 * ub, atol=1e-12)
    ustar = _exact.exact_solution(f)
    u = ustar.copy()
    oracle.vcycle(u, f, 1.0, 1, sweeps=2)
    np.testing.assert_allclose(u, ustar, atol=1e-12 * np.max(np.abs(ustar)))
    r1, _ = oracle.convergence_factor(W.random_field(2, 65, seed=3), 1.0, 150, sweeps=1)
    r2, _ = oracle.convergence_factor(W.random_field(2, 65, seed=3), 1.0, 150, sweeps=2)
    assert r1 == pytest.approx(0.099, abs=0.003) and r2 < 0.6 * r1
    with pytest.raises(RuntimeError):
        oracle.vcycle(np.zeros((9, 9, 9)), np.zeros((9, 9, 9)), (1.0,) * 4, 1, sweeps=2)


def test_optimal_p_is_linear_in_p():
    """the correction is exactly p times the p = 1 correction
    (every v is created by one -c r injection), so the error operator is
    I - p B A and p* = 2/(2 - rho0) reproduces the paper's optimum
    (1.052 / 0.052)."""
    n = 33
    f = W.random_field(2, n, seed=5)
    u0 = W.random_field(2, n, seed=6)
    corr = {}
    for p in (1.0, 1.052, 1.5):
        u = u0.copy()
        oracle.vcycle(u, f, p, 1)
        corr[p] = u - u0
    for p in (1.052, 1.5):
        assert np.allclose(corr[p], p * corr[1.0], rtol=1e-12, atol=1e-14 * np.abs(corr[1.0]).max())
    rho0 = 0.099
    assert 2 / (2 - rho0) == pytest.approx(1.052, abs=5e-4)


@pytest.mark.parametrize("dtype", DTYPES)
@pytest.mark.parametrize("dim,n", [(2, 33), (3, 17)])
def test_green_only_error_contracts_by_1_minus_p(dtype, dim, n):
    """an error supported on the green-only nodes
    (2D A(1) minus D(1); 3D G(1) minus R(1)) is mapped by one order-2 cycle to
    (1 - p) e (2D) or (1 - p_g) e (3D), size-independently.  Catches any
    wrong sign, index or dropped term in the residual, the first restriction
    and both colours of the finest Jacobi step."""
    rng = np.random.default_rng(9)
    idx = np.indices((n,) * dim).sum(0)
    green = (idx % 2 == 1)
    inner = np.zeros((n,) * dim, bool)
    inner[(slice(1, -1),) * dim] = True
    w = np.where(green & inner, rng.uniform(-1, 1, (n,) * dim), 0.0).astype(dtype)
    for p in (1.0, 1.052, 1.3):
        pp = p if dim == 2 else (1.11, 1.42, 1.08, p)
        u = w.copy()
        oracle.vcycle(u, np.zeros_like(w), pp, 1)
        want = np.where(green & inner, w - p * w, 0.0)
        eps = np.finfo(dtype).eps
        assert np.max(np.abs(u - want)) < 64 * eps


# -------------------------------------------------------------- invariants

def _d4(a):
    """The 8 elements of the square's symmetry group applied to an (n,n) array."""
    out = []
    for k in range(4):
        b = np.rot90(a, k)
        out += [b, b.T]
    return out


def test_d4_equivariance_2d():
    """All 2D stencils are D4-symmetric (Fig. 2), so the V-cycle
    commutes with the square's symmetries, up to rounding."""
    n = 33
    f = W.random_field(2, n, seed=1)
    u0 = W.random_field(2, n, seed=2)
    u = u0.copy()
    oracle.vcycle(u, f, 1.052, 2)
    for uf, ff, ut in zip(_d4(u0), _d4(f), _d4(u)):
        v = np.array(uf, order="C", copy=True)
        oracle.vcycle(v, np.ascontiguousarray(ff), 1.052, 2)
        assert np.max(np.abs(v - ut)) < 1e-12 * np.max(np.abs(ut))


def test_octahedral_equivariance_3d():
    """3D stencils commute with axis permutations and reflections;
    in particular Erprolr's face orientation (reading A8)."""
    n = 17
    f = W.random_field(3, n, seed=1)
    u0 = W.random_field(3, n, seed=2)
    p = (1.11, 1.42, 1.08, 0.99)
    u = u0.copy()
    oracle.vcycle(u, f, p, 2)
    for perm in itertools.permutations(range(3)):
        for flip in ((), (0,), (1, 2)):
            def g(a):
                b = np.transpose(a, perm)
                return np.array(np.flip(b, flip) if flip else b, order="C", copy=True)
            v = g(u0)
            oracle.vcycle(v, g(f), p, 2)
            assert np.max(np.abs(v - g(u))) < 1e-12 * np.max(np.abs(u))


def test_linearity():
    """The V-cycle is affine in (u, f): V(a u1 + b u2, a f1 + b f2) =
    a V(u1,f1) + b V(u2,f2), up to rounding."""
    for dim, n, p in ((2, 33, 1.052), (3, 17, (1.11, 1.42, 1.08, 0.99))):
        u1, u2 = W.random_field(dim, n, 1), W.random_field(dim, n, 2)
        f1, f2 = W.random_field(dim, n, 3), W.random_field(dim, n, 4)
        a, b = 0.75, -1.5
        x, y, z = u1.copy(), u2.copy(), a * u1 + b * u2
        oracle.vcycle(x, f1, p, 1)
        oracle.vcycle(y, f2, p, 1)
        oracle.vcycle(z, a * f1 + b * f2, p, 1)
        assert np.max(np.abs(z - (a * x + b * y))) < 1e-12 * np.max(np.abs(z))


@pytest.mark.parametrize("dim,n", [(2, 33), (3, 17)])
def test_fp32_tracks_fp64(dim, n):
    """The fp32 build is the same algorithm: it tracks the fp64 build to fp32
    rounding over a few cycles."""
    p = 1.052 if dim == 2 else (1.11, 1.42, 1.08, 0.99)
    f = W.random_field(dim, n, seed=8)
    u64 = np.zeros_like(f)
    u32 = np.zeros(f.shape, np.float32)
    oracle.vcycle(u64, f, p, 4)
    oracle.vcycle(u32, f.astype(np.float32), p, 4)
    assert np.max(np.abs(u32 - u64)) < 1e-4 * np.max(np.abs(u64))


@pytest.mark.parametrize("dim", [2, 3])
def test_order4_residual_is_fourth_order(dim):
    """Efos2/Efos4 are fourth-order accurate: for a
    smooth u and f = its continuous Laplacian, max|r| falls ~16x per halving
    of h; the second-order residual falls ~4x."""
    def trunc(n, order):
        xs = np.linspace(0, 1, n)
        G = np.meshgrid(*([xs] * dim), indexing="ij")
        u = np.prod([np.sin(np.pi * g) for g in G], axis=0)
        f = -dim * np.pi ** 2 * u
        return np.max(np.abs(oracle.residual(u, f, order)))
    ns = (17, 33) if dim == 3 else (33, 65)
    r4 = trunc(ns[0], 4) / trunc(ns[1], 4)
    r2 = trunc(ns[0], 2) / trunc(ns[1], 2)
    assert 14 < r4 < 18
    assert 3.5 < r2 < 4.5


# ------------------------------------------- order 4: the f~ right-hand side

@pytest.mark.parametrize("dim,n", [(2, 33), (3, 17)])
def test_ftilde_matches_dst_weight(dim, n):
    """The order-4 right-hand-side combination f~ = ((8 or 6) f + sum of the
    axis neighbours of f) / 12 (Efos2 P:311-321, Efos4 P:724-745; reading A11:
    f's boundary values as stored, here zero): applied spectrally it is the
    f-weight symbol mu of tests/_exact.py (a library DST-I), not a re-typed
    stencil."""
    import scipy.fft as sfft
    f = W.random_field(dim, n, seed=21)
    inner = (slice(1, -1),) * dim
    _, mu = _exact.symbols(dim, n, 4)
    want = sfft.idstn(sfft.dstn(f[inner], type=1, norm="ortho") * mu, type=1, norm="ortho")
    got = oracle.ftilde(f)
    assert np.max(np.abs(got[inner] - want)) < 1e-13 * np.max(np.abs(want))


@pytest.mark.parametrize("dim,n,p,cycles", [(2, 33, 1.20, 30), (2, 65, 1.20, 30),
                                            (3, 17, (0.91, 0.80, 0.70, 1.77), 45)])
def test_order4_vcycle_fixed_point_is_mehrstellen_solution(dim, n, p, cycles):
    """The order-4 V-cycle (P:324-334 / P:753-756: the second-order cycle on
    the compact fourth-order residual r = f~ - L9 u, resp. f~ - L19 u) leaves
    the exact discrete solution of the Mehrstellen system L u = f~ (DST-I,
    library routine) fixed, and converges to it from u = 0.  An oracle that
    fed the raw f (not f~) to its order-4 cycles converges to L u = f instead
    and fails this by O(h^2) relative."""
    f = W.random_field(dim, n, seed=22)
    uex = _exact.exact_solution(f, 4)
    u = uex.copy()
    oracle.vcycle(u, f, p, 1, order=4)
    assert np.max(np.abs(u - uex)) < 1e-13 * np.max(np.abs(uex))
    u = np.zeros_like(f)
    hist = oracle.vcycle(u, f, p, cycles, order=4, hist=True)
    assert np.max(np.abs(u - uex)) < 1e-11 * np.max(np.abs(uex))
    assert hist[-1] < 1e-9 * hist[0]
    # the raw-f system's solution (L u = f) is measurably different: the pin has teeth
    raw = np.zeros_like(f)
    lam4, _ = _exact.symbols(dim, n, 4)
    import scipy.fft as sfft
    inner = (slice(1, -1),) * dim
    raw[inner] = sfft.idstn(sfft.dstn(f[inner], type=1, norm="ortho") / lam4, type=1, norm="ortho")
    assert np.max(np.abs(raw - uex)) > 1e-4 * np.max(np.abs(uex))


# ------------------------------------------- 3D "mean factor"

@pytest.mark.parametrize("p,want,tol", [((1.0, 1.0, 1.0, 1.0), 0.140, 0.012),
                                        ((1.11, 1.42, 1.08, 0.99), 0.043, 0.004)])
@pytest.mark.parametrize("seed", [0, 1, 2, 3])
def test_3d_mean_factor_matches_paper(p, want, tol, seed):
    """The 3D text quotes a "mean factor of convergence rho-bar ~ 0.140"
    (Table 2 P:709-712 at p = 1, Table 3 P:786-787 0.043 tuned).
    Reading A12b: the geometric mean of the per-cycle L-inf
    residual ratios over cycles 7-12 of the error equation (f = 0) from a
    random start at 17^3.  This is tighter than the spectral-radius window
    (+-0.05), which the unstated boundary treatment moves to 0.157."""
    u = W.random_field(3, 17, seed=seed)
    hist = oracle.vcycle(u, np.zeros_like(u), p, 12, hist=True)
    ratios = hist[1:] / hist[:-1]
    mean = float(np.exp(np.mean(np.log(ratios[6:12]))))
    assert mean == pytest.approx(want, abs=tol)
