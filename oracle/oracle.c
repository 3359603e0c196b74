/*
 * oracle.c -- CPU ORACLE for Roberts' diagonally oriented multigrid V-cycle
 *             (arXiv math/9907190, /root/reference/PAPER.md).
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in the product path (the CUDA library
 * under paper_math_9907190_b200/) may include, link or call this file.  Only
 * tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
 * reference leg load it.  It shares no code, header, table or constant
 * generator with the CUDA path.
 *
 * Plain, slow, single-threaded C.  Compiled twice: -DREAL=double (f64) and
 * -DREAL=float (f32), always with -O2 -ffp-contract=off (no FMA contraction,
 * no -ffast-math), so that every formula below is evaluated left to right in
 * exactly the order it is written (the canonical order of DESIGN.md
 * "Canonical arithmetic").
 *
 * Storage (the paper's own convention, "we index variables using
 * subscripts appropriate to the fine green grid"): every level lives on the
 * lattice of its octave s = 2^o, i.e. an array of (m+1)^d entries with
 * m = (n-1)/s, indexed by lattice coordinates I = i/s (x fastest).  A level is
 * that lattice plus a node mask:
 *   2D  axis  A(s):  all lattice points
 *       diag  D(s):  I+J even                                 (Fig. 1)
 *   3D  green G(s):  all lattice points
 *       red   R(s):  I+J+K even (cube corners + face centres)
 *       mag.  M(s):  I = J = K (mod 2) (corners + centres)
 * Level order (finest first): 2D A(1),D(1),A(2),D(2),...,A(2^(k-1));
 * 3D G(1),R(1),M(1),G(2),...,G(2^(k-1)), n = 2^k+1.  Boundary nodes (I=0 or
 * I=m in any coordinate) hold 0 in every r and v array (reading A1/A3 of
 * homogeneous Dirichlet, zero extension, no renormalisation).
 *
 * Parity pins: see DESIGN.md "Oracle pins" and tests/test_oracle_*.py.
 * Parity unpinned: the exact per-cycle factors at sizes other than 65^2/17^3
 * (only the paper's windows), the coarsest-level reading A4 when p != 1
 * (corroborated, not pinned), the boundary reading A1/A3 beyond the paper's
 * table tolerances.
 */
#include <math.h>
#include <stdlib.h>
#include <string.h>

#ifndef REAL
#error "compile with -DREAL=double or -DREAL=float"
#endif

typedef REAL real;

/* ---------------------------------------------------------------- levels */

static int log2_exact(long v) {
  int k = 0;
  if (v < 1) return -1;
  while ((1L << k) < v) k++;
  return ((1L << k) == v) ? k : -1;
}

/* k with n = 2^k + 1, k >= 2; -1 otherwise (SPEC S:63 precondition). */
static int grid_k(long n) {
  int k = log2_exact(n - 1);
  return (k >= 2) ? k : -1;
}

int orc_levels(int dim, long n) {
  int k = grid_k(n);
  if (k < 0) return -1;
  if (dim == 2) return 2 * k - 1;   /* A(1) .. A(2^(k-1)) */
  if (dim == 3) return 3 * k - 2;   /* G(1) .. G(2^(k-1)) */
  return -1;
}

static int lev_octave(int dim, int lev) { return (dim == 2) ? lev / 2 : lev / 3; }
static int lev_class(int dim, int lev) { return (dim == 2) ? lev % 2 : lev % 3; }

/* m = (n-1)/s: lattice points per side are 0..m. */
long orc_lattice(int dim, long n, int lev) {
  int k = grid_k(n);
  if (k < 0 || lev < 0 || lev >= orc_levels(dim, n)) return -1;
  return (n - 1) >> lev_octave(dim, lev);
}

/* Interior node count of a level (SURVEY Appendix A counting rule). */
long orc_count(int dim, long n, int lev) {
  long m = orc_lattice(dim, n, lev), c = 0;
  if (m < 0) return -1;
  int cls = lev_class(dim, lev);
  if (dim == 2) {
    for (long J = 1; J < m; J++)
      for (long I = 1; I < m; I++)
        if (cls == 0 || ((I + J) % 2 == 0)) c++;
  } else {
    for (long K = 1; K < m; K++)
      for (long J = 1; J < m; J++)
        for (long I = 1; I < m; I++) {
          if (cls == 0) c++;
          else if (cls == 1 && (I + J + K) % 2 == 0) c++;
          else if (cls == 2 && (I % 2 == J % 2) && (J % 2 == K % 2)) c++;
        }
  }
  return c;
}

#define AT2(a, m, I, J) (a)[(long)(J) * ((m) + 1) + (I)]
#define AT3(a, m, I, J, K) (a)[((long)(K) * ((m) + 1) + (J)) * ((m) + 1) + (I)]

/* --------------------------------------------------------- coefficients
 * Every constant is formed in double and rounded once to `real`
 * (DESIGN.md "Canonical arithmetic").  (s h)^2 = (s/(n-1))^2 is a power of
 * two, so kappa*p*(s h)^2 is exact in double. */
static double hs2(long n, int octave) {
  double hs = (double)(1L << octave) / (double)(n - 1);
  return hs * hs;
}

/* ------------------------------------------------------------ residuals */

/* r = f - Lap5 u at every interior node of A(1); order 2.
 * 5-point Laplacian, centre first then the neighbours in the order of
 * Erest2r: (i-1,j),(i,j-1),(i+1,j),(i,j+1).  7 flops. */
static real res2d_o2(long m, const real *u, const real *f, long I, long J, real invh2) {
  real lap = -((real)4 * AT2(u, m, I, J));
  lap = lap + AT2(u, m, I - 1, J);
  lap = lap + AT2(u, m, I, J - 1);
  lap = lap + AT2(u, m, I + 1, J);
  lap = lap + AT2(u, m, I, J + 1);
  lap = lap * invh2;
  return AT2(f, m, I, J) - lap;
}

/* The f-combination of Efos2: (1/12)(8f + f_{i+1,j} + f_{i,j+1}
 * + f_{i-1,j} + f_{i,j-1}), terms in printed order. */
static real ft2d(long m, const real *f, long I, long J) {
  real t = (real)8 * AT2(f, m, I, J);
  t = t + AT2(f, m, I + 1, J);
  t = t + AT2(f, m, I, J + 1);
  t = t + AT2(f, m, I - 1, J);
  t = t + AT2(f, m, I, J - 1);
  return t * (real)(1.0 / 12.0);
}

/* Efos2: r = ft - (1/(6h^2)) [ -20u + 4(u_{i,j-1}+u_{i,j+1}+
 * u_{i-1,j}+u_{i+1,j}) + u_{i+1,j+1}+u_{i-1,j+1}+u_{i-1,j-1}+u_{i+1,j-1} ]. */
static real res2d_o4(long m, const real *u, real ft, long I, long J, real c6) {
  real ax = AT2(u, m, I, J - 1);
  ax = ax + AT2(u, m, I, J + 1);
  ax = ax + AT2(u, m, I - 1, J);
  ax = ax + AT2(u, m, I + 1, J);
  real b = -((real)20 * AT2(u, m, I, J));
  b = b + (real)4 * ax;
  b = b + AT2(u, m, I + 1, J + 1);
  b = b + AT2(u, m, I - 1, J + 1);
  b = b + AT2(u, m, I - 1, J - 1);
  b = b + AT2(u, m, I + 1, J - 1);
  return ft - b * c6;
}

/* 7-point Laplacian residual (P:686-687, 9 flops), centre first then the
 * neighbours in the order of Erred: i+1,i-1,j+1,j-1,k+1,k-1. */
static real res3d_o2(long m, const real *u, const real *f, long I, long J, long K, real invh2) {
  real lap = -((real)6 * AT3(u, m, I, J, K));
  lap = lap + AT3(u, m, I + 1, J, K);
  lap = lap + AT3(u, m, I - 1, J, K);
  lap = lap + AT3(u, m, I, J + 1, K);
  lap = lap + AT3(u, m, I, J - 1, K);
  lap = lap + AT3(u, m, I, J, K + 1);
  lap = lap + AT3(u, m, I, J, K - 1);
  lap = lap * invh2;
  return AT3(f, m, I, J, K) - lap;
}

/* f-combination of Efos4: (1/12)(6f + f_{i+1} + f_{j+1} +
 * f_{i-1} + f_{j-1} + f_{k+1} + f_{k-1}), printed order. */
static real ft3d(long m, const real *f, long I, long J, long K) {
  real t = (real)6 * AT3(f, m, I, J, K);
  t = t + AT3(f, m, I + 1, J, K);
  t = t + AT3(f, m, I, J + 1, K);
  t = t + AT3(f, m, I - 1, J, K);
  t = t + AT3(f, m, I, J - 1, K);
  t = t + AT3(f, m, I, J, K + 1);
  t = t + AT3(f, m, I, J, K - 1);
  return t * (real)(1.0 / 12.0);
}

/* Efos4, bracket terms in printed order. */
static real res3d_o4(long m, const real *u, real ft, long I, long J, long K, real c6) {
  real ax = AT3(u, m, I, J - 1, K);
  ax = ax + AT3(u, m, I, J + 1, K);
  ax = ax + AT3(u, m, I - 1, J, K);
  ax = ax + AT3(u, m, I + 1, J, K);
  ax = ax + AT3(u, m, I, J, K + 1);
  ax = ax + AT3(u, m, I, J, K - 1);
  real b = -((real)24 * AT3(u, m, I, J, K));
  b = b + (real)2 * ax;
  b = b + AT3(u, m, I + 1, J + 1, K);
  b = b + AT3(u, m, I - 1, J + 1, K);
  b = b + AT3(u, m, I - 1, J - 1, K);
  b = b + AT3(u, m, I + 1, J - 1, K);
  b = b + AT3(u, m, I, J + 1, K + 1);
  b = b + AT3(u, m, I, J + 1, K - 1);
  b = b + AT3(u, m, I, J - 1, K - 1);
  b = b + AT3(u, m, I, J - 1, K + 1);
  b = b + AT3(u, m, I + 1, J, K + 1);
  b = b + AT3(u, m, I - 1, J, K + 1);
  b = b + AT3(u, m, I - 1, J, K - 1);
  b = b + AT3(u, m, I + 1, J, K - 1);
  return ft - b * c6;
}

/* f~ of Efos2/Efos4 at every interior node (0 on the boundary).  The paper
 * notes it "need not be computed each iteration". */
int orc_ftilde(int dim, long n, const real *f, real *ft) {
  long m = n - 1;
  if (grid_k(n) < 0) return -1;
  if (dim == 2) {
    memset(ft, 0, sizeof(real) * (size_t)(n * n));
    for (long J = 1; J < m; J++)
      for (long I = 1; I < m; I++) AT2(ft, m, I, J) = ft2d(m, f, I, J);
  } else if (dim == 3) {
    memset(ft, 0, sizeof(real) * (size_t)(n * n * n));
    for (long K = 1; K < m; K++)
      for (long J = 1; J < m; J++)
        for (long I = 1; I < m; I++) AT3(ft, m, I, J, K) = ft3d(m, f, I, J, K);
  } else {
    return -1;
  }
  return 0;
}

/* r = f - L u on the finest grid (Evpois), order 2 or 4.  For
 * order 4, `f` is the raw right-hand side; f~ is formed pointwise (the same
 * value a precomputed f~ holds).  r = 0 on the boundary. */
int orc_residual(int dim, long n, int order, const real *u, const real *f, real *r) {
  long m = n - 1;
  if (grid_k(n) < 0 || (order != 2 && order != 4)) return -1;
  real invh2 = (real)((double)(n - 1) * (double)(n - 1));
  real c6 = (real)((double)(n - 1) * (double)(n - 1) / 6.0);
  if (dim == 2) {
    memset(r, 0, sizeof(real) * (size_t)(n * n));
    for (long J = 1; J < m; J++)
      for (long I = 1; I < m; I++)
        AT2(r, m, I, J) = (order == 2) ? res2d_o2(m, u, f, I, J, invh2)
                                       : res2d_o4(m, u, ft2d(m, f, I, J), I, J, c6);
  } else if (dim == 3) {
    memset(r, 0, sizeof(real) * (size_t)(n * n * n));
    for (long K = 1; K < m; K++)
      for (long J = 1; J < m; J++)
        for (long I = 1; I < m; I++)
          AT3(r, m, I, J, K) = (order == 2) ? res3d_o2(m, u, f, I, J, K, invh2)
                                            : res3d_o4(m, u, ft3d(m, f, I, J, K), I, J, K, c6);
  } else {
    return -1;
  }
  return 0;
}

/* residual with a precomputed f~ (order 4) -- used inside the V-cycle. */
static void residual_ft(int dim, long n, int order, const real *u, const real *f_or_ft, real *r) {
  long m = n - 1;
  real invh2 = (real)((double)(n - 1) * (double)(n - 1));
  real c6 = (real)((double)(n - 1) * (double)(n - 1) / 6.0);
  if (dim == 2) {
    for (long J = 1; J < m; J++)
      for (long I = 1; I < m; I++)
        AT2(r, m, I, J) = (order == 2) ? res2d_o2(m, u, f_or_ft, I, J, invh2)
                                       : res2d_o4(m, u, AT2(f_or_ft, m, I, J), I, J, c6);
  } else {
    for (long K = 1; K < m; K++)
      for (long J = 1; J < m; J++)
        for (long I = 1; I < m; I++)
          AT3(r, m, I, J, K) = (order == 2) ? res3d_o2(m, u, f_or_ft, I, J, K, invh2)
                                            : res3d_o4(m, u, AT3(f_or_ft, m, I, J, K), I, J, K, c6);
  }
}

/* ----------------------------------------------------------- restriction
 * orc_restrict(lev): r on level lev (lattice m) -> r on level lev+1.
 * Only the interior nodes of level lev+1 are written; all other entries of
 * rout are set to 0. */

/* 2D, axis A(s) -> diagonal D(s), Erest2r:
 * r' = (1/8)(4r + r_{i-1,j} + r_{i,j-1} + r_{i+1,j} + r_{i,j+1}). */
static void rest_2d_axis_diag(long m, const real *a, real *d) {
  for (long J = 1; J < m; J++)
    for (long I = 1; I < m; I++) {
      if ((I + J) % 2 != 0) continue;
      real t = (real)4 * AT2(a, m, I, J);
      t = t + AT2(a, m, I - 1, J);
      t = t + AT2(a, m, I, J - 1);
      t = t + AT2(a, m, I + 1, J);
      t = t + AT2(a, m, I, J + 1);
      AT2(d, m, I, J) = t * (real)(1.0 / 8.0);
    }
}

/* 2D, diagonal D(s) -> axis A(2s), Erest2b:
 * r' = (1/8)(4r + r_{i-1,j-1} + r_{i+1,j-1} + r_{i+1,j+1} + r_{i-1,j+1}).
 * Target lattice mc = m/2; target node (I,J) is source node (2I,2J). */
static void rest_2d_diag_axis(long m, const real *d, real *a) {
  long mc = m / 2;
  for (long J = 1; J < mc; J++)
    for (long I = 1; I < mc; I++) {
      long X = 2 * I, Y = 2 * J;
      real t = (real)4 * AT2(d, m, X, Y);
      t = t + AT2(d, m, X - 1, Y - 1);
      t = t + AT2(d, m, X + 1, Y - 1);
      t = t + AT2(d, m, X + 1, Y + 1);
      t = t + AT2(d, m, X - 1, Y + 1);
      AT2(a, mc, I, J) = t * (real)(1.0 / 8.0);
    }
}

/* 3D, green G(s) -> red R(s), Erred:
 * r' = (1/12)(6r + r_{i+1} + r_{i-1} + r_{j+1} + r_{j-1} + r_{k+1} + r_{k-1}). */
static void rest_3d_green_red(long m, const real *g, real *rr) {
  for (long K = 1; K < m; K++)
    for (long J = 1; J < m; J++)
      for (long I = 1; I < m; I++) {
        if ((I + J + K) % 2 != 0) continue;
        real t = (real)6 * AT3(g, m, I, J, K);
        t = t + AT3(g, m, I + 1, J, K);
        t = t + AT3(g, m, I - 1, J, K);
        t = t + AT3(g, m, I, J + 1, K);
        t = t + AT3(g, m, I, J - 1, K);
        t = t + AT3(g, m, I, J, K + 1);
        t = t + AT3(g, m, I, J, K - 1);
        AT3(rr, m, I, J, K) = t * (real)(1.0 / 12.0);
      }
}

/* The 12 face-diagonal offsets in the printed order of Ermagc
 * and Erprolm -- identical in both equations. */
static const int FD12[12][3] = {
  {+1, +1, 0}, {+1, -1, 0}, {-1, -1, 0}, {-1, +1, 0},
  {+1, 0, +1}, {+1, 0, -1}, {-1, 0, -1}, {-1, 0, +1},
  {0, +1, +1}, {0, +1, -1}, {0, -1, -1}, {0, -1, +1}};

/* The 8 body-diagonal offsets in the printed order of Erblu and
 * Emprolm/Emprolb. */
static const int BD8[8][3] = {
  {+1, +1, +1}, {+1, +1, -1}, {+1, -1, +1}, {+1, -1, -1},
  {-1, +1, +1}, {-1, +1, -1}, {-1, -1, +1}, {-1, -1, -1}};

/* The 6 axis offsets in the printed order of Erred/Ermagm/Egprolg/Egprolr. */
static const int AX6[6][3] = {
  {+1, 0, 0}, {-1, 0, 0}, {0, +1, 0}, {0, -1, 0}, {0, 0, +1}, {0, 0, -1}};

/* 3D, red R(s) -> magenta M(s).
 * corners (I,J,K all even), Ermagc: (1/24)(12 r + sum_12 face-diag)
 * centres (all odd, not red nodes), Ermagm: (1/6)(sum_6 axis),
 * zero self-weight. */
static void rest_3d_red_mag(long m, const real *rr, real *mg) {
  for (long K = 1; K < m; K++)
    for (long J = 1; J < m; J++)
      for (long I = 1; I < m; I++) {
        int pi = I % 2, pj = J % 2, pk = K % 2;
        if (!(pi == pj && pj == pk)) continue;
        real t;
        if (pi == 0) {
          t = (real)12 * AT3(rr, m, I, J, K);
          for (int q = 0; q < 12; q++)
            t = t + AT3(rr, m, I + FD12[q][0], J + FD12[q][1], K + FD12[q][2]);
          t = t * (real)(1.0 / 24.0);
        } else {
          t = AT3(rr, m, I + AX6[0][0], J + AX6[0][1], K + AX6[0][2]);
          for (int q = 1; q < 6; q++)
            t = t + AT3(rr, m, I + AX6[q][0], J + AX6[q][1], K + AX6[q][2]);
          t = t * (real)(1.0 / 6.0);
        }
        AT3(mg, m, I, J, K) = t;
      }
}

/* 3D, magenta M(s) -> blue/green G(2s), Erblu:
 * r' = (1/16)(8r + sum_8 body-diagonal). */
static void rest_3d_mag_blue(long m, const real *mg, real *g2) {
  long mc = m / 2;
  for (long K = 1; K < mc; K++)
    for (long J = 1; J < mc; J++)
      for (long I = 1; I < mc; I++) {
        long X = 2 * I, Y = 2 * J, Z = 2 * K;
        real t = (real)8 * AT3(mg, m, X, Y, Z);
        for (int q = 0; q < 8; q++) t = t + AT3(mg, m, X + BD8[q][0], Y + BD8[q][1], Z + BD8[q][2]);
        AT3(g2, mc, I, J, K) = t * (real)(1.0 / 16.0);
      }
}

int orc_restrict(int dim, long n, int lev, const real *rin, real *rout) {
  int L = orc_levels(dim, n);
  if (L < 0 || lev < 0 || lev + 1 >= L) return -1;
  long m = orc_lattice(dim, n, lev), mo = orc_lattice(dim, n, lev + 1);
  size_t cnt = (size_t)((dim == 2) ? (mo + 1) * (mo + 1) : (mo + 1) * (mo + 1) * (mo + 1));
  memset(rout, 0, sizeof(real) * cnt);
  int cls = lev_class(dim, lev);
  if (dim == 2) {
    if (cls == 0) rest_2d_axis_diag(m, rin, rout);
    else rest_2d_diag_axis(m, rin, rout);
  } else {
    if (cls == 0) rest_3d_green_red(m, rin, rout);
    else if (cls == 1) rest_3d_red_mag(m, rin, rout);
    else rest_3d_mag_blue(m, rin, rout);
  }
  return 0;
}

/* --------------------------------------------------- Jacobi prolongation
 * orc_jacobi(lev): v on level lev from v on level lev+1 (vc) and r on level
 * lev, by the paper's two-colour ("red-black") Jacobi step.  Only interior
 * nodes of level lev are written; all other entries of v are set to 0.
 * p: 2D p[0] = p (Eajacr/Eajacb, and "similarly for a green
 * grid"); 3D p = {p_m, p_r1, p_r2, p_g}. */

/* 2D diagonal level D(s) from A(2s) (Eajacr then Eajacb):
 *   colour 1, nodes of D(s) not on A(2s) (I, J odd):
 *     v = (1/4)(-2p(sh)^2 r + v^{l-1}_{i-1,j-1} + v^{l-1}_{i+1,j-1}
 *               + v^{l-1}_{i+1,j+1} + v^{l-1}_{i-1,j+1})
 *   colour 2, nodes of A(2s) (I, J even): same formula on the new values.
 * The coarse value at the coincident node is discarded (it is replaced). */
static void jac_2d_diag(long m, double p, double hsq, const real *vc, const real *r, real *v) {
  long mc = m / 2;
  real c = (real)(2.0 * p * hsq);
  for (long J = 1; J < m; J += 2)
    for (long I = 1; I < m; I += 2) {
      real t = -(c * AT2(r, m, I, J));
      t = t + AT2(vc, mc, (I - 1) / 2, (J - 1) / 2);
      t = t + AT2(vc, mc, (I + 1) / 2, (J - 1) / 2);
      t = t + AT2(vc, mc, (I + 1) / 2, (J + 1) / 2);
      t = t + AT2(vc, mc, (I - 1) / 2, (J + 1) / 2);
      AT2(v, m, I, J) = t * (real)(1.0 / 4.0);
    }
  for (long J = 2; J < m; J += 2)
    for (long I = 2; I < m; I += 2) {
      real t = -(c * AT2(r, m, I, J));
      t = t + AT2(v, m, I - 1, J - 1);
      t = t + AT2(v, m, I + 1, J - 1);
      t = t + AT2(v, m, I + 1, J + 1);
      t = t + AT2(v, m, I - 1, J + 1);
      AT2(v, m, I, J) = t * (real)(1.0 / 4.0);
    }
}

/* 2D axis level A(s) from D(s) ("similarly for a green grid", P:228-230,
 * P:360; reading A5):  colour 1 on the green-only nodes (I+J odd), then
 * colour 2 on the D(s) nodes (I+J even) with the new values:
 *   v = (1/4)(-p(sh)^2 r + v_{i-1,j} + v_{i,j-1} + v_{i+1,j} + v_{i,j+1}). */
static void jac_2d_axis(long m, double p, double hsq, const real *vd, const real *r, real *v) {
  real c = (real)(p * hsq);
  for (int colour = 1; colour <= 2; colour++) {
    const real *src = (colour == 1) ? vd : v;
    for (long J = 1; J < m; J++)
      for (long I = 1; I < m; I++) {
        int odd = (int)((I + J) % 2);
        if ((colour == 1) != (odd == 1)) continue;
        real t = -(c * AT2(r, m, I, J));
        t = t + AT2(src, m, I - 1, J);
        t = t + AT2(src, m, I, J - 1);
        t = t + AT2(src, m, I + 1, J);
        t = t + AT2(src, m, I, J + 1);
        AT2(v, m, I, J) = t * (real)(1.0 / 4.0);
      }
  }
}

/* 3D magenta level M(s) from G(2s) (Emprolm then Emprolb):
 *   centres (all odd): v = (1/8)(-4 p_m (sh)^2 r + sum_8 body-diag v^{l-1})
 *   corners (all even, = G(2s) nodes): same formula on the new centre values. */
static void jac_3d_mag(long m, double pm, double hsq, const real *vc, const real *r, real *v) {
  long mc = m / 2;
  real c = (real)(4.0 * pm * hsq);
  for (long K = 1; K < m; K += 2)
    for (long J = 1; J < m; J += 2)
      for (long I = 1; I < m; I += 2) {
        real t = -(c * AT3(r, m, I, J, K));
        for (int q = 0; q < 8; q++)
          t = t + AT3(vc, mc, (I + BD8[q][0]) / 2, (J + BD8[q][1]) / 2, (K + BD8[q][2]) / 2);
        AT3(v, m, I, J, K) = t * (real)(1.0 / 8.0);
      }
  for (long K = 2; K < m; K += 2)
    for (long J = 2; J < m; J += 2)
      for (long I = 2; I < m; I += 2) {
        real t = -(c * AT3(r, m, I, J, K));
        for (int q = 0; q < 8; q++) t = t + AT3(v, m, I + BD8[q][0], J + BD8[q][1], K + BD8[q][2]);
        AT3(v, m, I, J, K) = t * (real)(1.0 / 8.0);
      }
}

/* Erprolr offsets for a face centre whose normal is the z axis,
 * printed order: the normal pair (weight 2), then the 4 in-plane corners.
 * Other faces: "cyclically permute the role of the indices",
 * reading A8: an offset (a,b,c) of the z-face formula becomes (c,a,b) for
 * the x-face and (b,c,a) for the y-face. */
static void erprolr_offsets(int normal, int off[6][3]) {
  static const int Z[6][3] = {{0, 0, +1}, {0, 0, -1}, {+1, +1, 0}, {+1, -1, 0}, {-1, -1, 0}, {-1, +1, 0}};
  for (int q = 0; q < 6; q++) {
    int a = Z[q][0], b = Z[q][1], c = Z[q][2];
    if (normal == 2) { off[q][0] = a; off[q][1] = b; off[q][2] = c; }
    else if (normal == 0) { off[q][0] = c; off[q][1] = a; off[q][2] = b; }
    else { off[q][0] = b; off[q][1] = c; off[q][2] = a; }
  }
}

/* 3D red level R(s) from M(s) (Erprolr then Erprolm):
 *   face centres (exactly one of I,J,K even = the face normal, reading A8):
 *     v = (1/8)(-2 p_r1 (sh)^2 r + 2[v_{+n} + v_{-n}] + sum_4 in-plane v^{l-1})
 *   corners (all even): v = (1/12)(-4 p_r2 (sh)^2 r + sum_12 face-diag v^l)
 *   magenta centres are not red nodes and are not updated. */
static void jac_3d_red(long m, double pr1, double pr2, double hsq, const real *vm, const real *r, real *v) {
  real c1 = (real)(2.0 * pr1 * hsq), c2 = (real)(4.0 * pr2 * hsq);
  int off[3][6][3];
  for (int a = 0; a < 3; a++) erprolr_offsets(a, off[a]);
  for (long K = 1; K < m; K++)
    for (long J = 1; J < m; J++)
      for (long I = 1; I < m; I++) {
        if ((I + J + K) % 2 != 0) continue;
        int ne = (I % 2 == 0) + (J % 2 == 0) + (K % 2 == 0);
        if (ne != 1) continue;   /* face centres only */
        int a = (I % 2 == 0) ? 0 : ((J % 2 == 0) ? 1 : 2);
        real nrm = AT3(vm, m, I + off[a][0][0], J + off[a][0][1], K + off[a][0][2]);
        nrm = nrm + AT3(vm, m, I + off[a][1][0], J + off[a][1][1], K + off[a][1][2]);
        real t = -(c1 * AT3(r, m, I, J, K));
        t = t + (real)2 * nrm;
        for (int q = 2; q < 6; q++) t = t + AT3(vm, m, I + off[a][q][0], J + off[a][q][1], K + off[a][q][2]);
        AT3(v, m, I, J, K) = t * (real)(1.0 / 8.0);
      }
  for (long K = 2; K < m; K += 2)
    for (long J = 2; J < m; J += 2)
      for (long I = 2; I < m; I += 2) {
        real t = -(c2 * AT3(r, m, I, J, K));
        for (int q = 0; q < 12; q++) t = t + AT3(v, m, I + FD12[q][0], J + FD12[q][1], K + FD12[q][2]);
        AT3(v, m, I, J, K) = t * (real)(1.0 / 12.0);
      }
}

/* 3D green level G(s) from R(s) (Egprolg then Egprolr):
 *   green-only nodes (I+J+K odd), then red nodes with the new values:
 *   v = (1/6)(-p_g (sh)^2 r + v_{i+1} + v_{i-1} + v_{j+1} + v_{j-1} + v_{k+1} + v_{k-1}). */
static void jac_3d_green(long m, double pg, double hsq, const real *vr, const real *r, real *v) {
  real c = (real)(pg * hsq);
  for (int colour = 1; colour <= 2; colour++) {
    const real *src = (colour == 1) ? vr : v;
    for (long K = 1; K < m; K++)
      for (long J = 1; J < m; J++)
        for (long I = 1; I < m; I++) {
          int odd = (int)((I + J + K) % 2);
          if ((colour == 1) != (odd == 1)) continue;
          real t = -(c * AT3(r, m, I, J, K));
          for (int q = 0; q < 6; q++) t = t + AT3(src, m, I + AX6[q][0], J + AX6[q][1], K + AX6[q][2]);
          AT3(v, m, I, J, K) = t * (real)(1.0 / 6.0);
        }
  }
}

int orc_jacobi(int dim, long n, int lev, const double *p, const real *vc, const real *r, real *v) {
  int L = orc_levels(dim, n);
  if (L < 0 || lev < 0 || lev + 1 >= L) return -1;
  long m = orc_lattice(dim, n, lev);
  int oct = lev_octave(dim, lev), cls = lev_class(dim, lev);
  double hsq = hs2(n, oct);
  size_t cnt = (size_t)((dim == 2) ? (m + 1) * (m + 1) : (m + 1) * (m + 1) * (m + 1));
  memset(v, 0, sizeof(real) * cnt);
  if (dim == 2) {
    if (cls == 1) jac_2d_diag(m, p[0], hsq, vc, r, v);
    else jac_2d_axis(m, p[0], hsq, vc, r, v);
  } else {
    if (cls == 2) jac_3d_mag(m, p[0], hsq, vc, r, v);
    else if (cls == 1) jac_3d_red(m, p[1], p[2], hsq, vc, r, v);
    else jac_3d_green(m, p[3], hsq, vc, r, v);
  }
  return 0;
}

/* Coarsest level (one interior node; reading A4): one Jacobi iteration of
 * the green-grid formula from v = 0, with that level's parameter:
 * 2D v = (1/4)(-p H^2 r), 3D v = (1/6)(-p_g H^2 r), H = 2^(k-1) h. */
int orc_coarsest(int dim, long n, const double *p, const real *r, real *v) {
  int L = orc_levels(dim, n);
  if (L < 0) return -1;
  int lev = L - 1;
  long m = orc_lattice(dim, n, lev);   /* == 2 */
  double hsq = hs2(n, lev_octave(dim, lev));
  if (dim == 2) {
    memset(v, 0, sizeof(real) * 9);
    real c = (real)(p[0] * hsq);
    AT2(v, m, 1, 1) = -(c * AT2(r, m, 1, 1)) * (real)(1.0 / 4.0);
  } else {
    memset(v, 0, sizeof(real) * 27);
    real c = (real)(p[3] * hsq);
    AT3(v, m, 1, 1, 1) = -(c * AT3(r, m, 1, 1, 1)) * (real)(1.0 / 6.0);
  }
  return 0;
}

/* -------------------------------------------------------------- norms */

/* max |x| over interior nodes of the finest grid. */
double orc_norm_inf(int dim, long n, const real *x) {
  long m = n - 1;
  double mx = 0.0;
  if (dim == 2) {
    for (long J = 1; J < m; J++)
      for (long I = 1; I < m; I++) {
        double a = fabs((double)AT2(x, m, I, J));
        if (a > mx || a != a) mx = a;
      }
  } else {
    for (long K = 1; K < m; K++)
      for (long J = 1; J < m; J++)
        for (long I = 1; I < m; I++) {
          double a = fabs((double)AT3(x, m, I, J, K));
          if (a > mx || a != a) mx = a;
        }
  }
  return mx;
}

/* ------------------------------------------------- extra Jacobi sweeps
 * SURVEY 8(f) NEXT-4, the paper's open question "the effect of extra Jacobi
 * iterations at each level of the diagonal grid".  Reading A19:
 * an extra sweep on a 2D level repeats that level's two-colour step with
 * the level's own values in place of the coarser level's -- on D(s) colour 1
 * takes its four diagonal neighbours from the A(2s)-coincident (E) nodes of
 * v_{D(s)}; on A(s) the green nodes take their four axis neighbours from the
 * D(s) nodes of v_{A(s)} -- then colour 2 as before; on every level,
 * the finest included (u <- u + v_0 after its last sweep).  Only 2D: in 3D
 * the red level's first colour reads magenta B nodes, which the red level
 * does not hold. */
static void jac_2d_again(long m, int cls, double p, double hsq, real *v, const real *r, real *src) {
  if (cls == 1) {   /* D(s): the E nodes as a coarse (m/2+1)^2 grid */
    long mc = m / 2;
    for (long Y = 0; Y <= mc; Y++)
      for (long X = 0; X <= mc; X++) AT2(src, mc, X, Y) = AT2(v, m, 2 * X, 2 * Y);
    jac_2d_diag(m, p, hsq, src, r, v);
  } else {          /* A(s): colour 1 from v's own D nodes */
    for (long J = 0; J <= m; J++)
      for (long I = 0; I <= m; I++) AT2(src, m, I, J) = AT2(v, m, I, J);
    jac_2d_axis(m, p, hsq, src, r, v);
  }
}

/* ------------------------------------------------------------- V-cycle */

static size_t lev_size(int dim, long n, int lev) {
  long m = orc_lattice(dim, n, lev);
  return (size_t)((dim == 2) ? (m + 1) * (m + 1) : (m + 1) * (m + 1) * (m + 1));
}

/* ncycles V-cycles u <- u + v:
 *   r_0 = f - L u (order 2, or Efos2/Efos4 with precomputed f~);
 *   descent: r_{l+1} = R_l r_l for every level;
 *   coarsest: one Jacobi from zero (A4);
 *   ascent: v_l = two-colour Jacobi(v_{l+1}, r_l);
 *   u <- u + v_0 at the interior.
 * hist (may be NULL): ncycles+1 values, ||f - L u||_inf before each cycle
 * and after the last one.  Returns 0, -1 bad arguments, -2 out of memory. */
int orc_vcycle_sweeps(int dim, long n, int order, const double *p, real *u, const real *f, int ncycles, double *hist,
                      int sweeps);
int orc_vcycle(int dim, long n, int order, const double *p, real *u, const real *f, int ncycles, double *hist) {
  return orc_vcycle_sweeps(dim, n, order, p, u, f, ncycles, hist, 1);
}

/* The same with `sweeps` two-colour Jacobi steps on every level (reading
 * A19; 2D only for sweeps > 1). */
int orc_vcycle_sweeps(int dim, long n, int order, const double *p, real *u, const real *f, int ncycles, double *hist,
                      int sweeps) {
  int L = orc_levels(dim, n);
  if (L < 0 || (order != 2 && order != 4) || ncycles < 0 || sweeps < 1 || (dim == 3 && sweeps > 1)) return -1;
  real *tmp = NULL;
  real **r = (real **)calloc((size_t)L, sizeof(real *));
  real **v = (real **)calloc((size_t)L, sizeof(real *));
  real *ft = NULL;
  int rc = 0;
  if (!r || !v) { rc = -2; goto done; }
  for (int l = 0; l < L; l++) {
    r[l] = (real *)calloc(lev_size(dim, n, l), sizeof(real));
    if (l > 0) v[l] = (real *)calloc(lev_size(dim, n, l), sizeof(real));
    if (!r[l] || (l > 0 && !v[l])) { rc = -2; goto done; }
  }
  v[0] = (real *)calloc(lev_size(dim, n, 0), sizeof(real));
  if (!v[0]) { rc = -2; goto done; }
  const real *rhs = f;
  if (order == 4) {
    ft = (real *)calloc(lev_size(dim, n, 0), sizeof(real));
    if (!ft) { rc = -2; goto done; }
    orc_ftilde(dim, n, f, ft);
    rhs = ft;
  }
  long m0 = n - 1;
  for (int cyc = 0; cyc <= ncycles; cyc++) {
    residual_ft(dim, n, order, u, rhs, r[0]);
    if (hist) hist[cyc] = orc_norm_inf(dim, n, r[0]);
    if (cyc == ncycles) break;
    for (int l = 0; l + 1 < L; l++) orc_restrict(dim, n, l, r[l], r[l + 1]);
    orc_coarsest(dim, n, p, r[L - 1], v[L - 1]);
    for (int l = L - 2; l >= 0; l--) {
      orc_jacobi(dim, n, l, p, v[l + 1], r[l], v[l]);
      if (sweeps > 1) {
        if (!tmp && !(tmp = (real *)calloc(lev_size(dim, n, 0), sizeof(real)))) { rc = -2; goto done; }
        long m = orc_lattice(dim, n, l);
        for (int sw = 1; sw < sweeps; sw++)
          jac_2d_again(m, lev_class(dim, l), p[0], hs2(n, lev_octave(dim, l)), v[l], r[l], tmp);
      }
    }
    if (dim == 2) {
      for (long J = 1; J < m0; J++)
        for (long I = 1; I < m0; I++) AT2(u, m0, I, J) = AT2(u, m0, I, J) + AT2(v[0], m0, I, J);
    } else {
      for (long K = 1; K < m0; K++)
        for (long J = 1; J < m0; J++)
          for (long I = 1; I < m0; I++) AT3(u, m0, I, J, K) = AT3(u, m0, I, J, K) + AT3(v[0], m0, I, J, K);
    }
  }
done:
  free(tmp);
  if (r) for (int l = 0; l < L; l++) free(r[l]);
  if (v) for (int l = 0; l < L; l++) free(v[l]);
  free(r);
  free(v);
  free(ft);
  return rc;
}

/* Size in bytes of `real` -- lets the Python side check which build it has. */
int orc_real_size(void) { return (int)sizeof(real); }
