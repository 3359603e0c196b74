// ops2.cuh -- the 2D per-node formulas of the V-cycle, shared by the
// reference kernels (k2d.cu), the TMA tile kernels (k2f.cu) and the coarse
// persistent kernel.  Canonical evaluation order: terms left to
// right as printed in the paper, constants rounded once from double; the
// library is compiled with --fmad=false.
#pragma once
#include "common.cuh"

namespace mg {

// ------------------------------------------------------------ residual
// r = f - L u at an interior node (Evpois).
//  order 2: 5-point Laplacian, centre first then (i-1,j),(i,j-1),(i+1,j),(i,j+1)
//           (the neighbour order of Erest2r); 7 flops.
//  order 4: Efos2 with f~ precomputed: bracket
//           -20u + 4(u_{i,j-1}+u_{i,j+1}+u_{i-1,j}+u_{i+1,j}) + u_{i+1,j+1}
//           + u_{i-1,j+1} + u_{i-1,j-1} + u_{i+1,j-1}, times 1/(6h^2).
// The 9 values around a node: centre, axis (w=(i-1,j), s=(i,j-1), e=(i+1,j),
// n=(i,j+1)) and diagonals; order 2 uses only the first five.
template <class T>
struct Nb9 {
  T c, w, s, e, n, ne, nw, sw, se;
};

template <class T, int ORDER>
__device__ __forceinline__ T res2v(const Nb9<T> &q, T f, const Coef<T> &k) {
  if (ORDER == 2) {
    T lap = -((T)4 * q.c);
    lap = lap + q.w;
    lap = lap + q.s;
    lap = lap + q.e;
    lap = lap + q.n;
    lap = lap * k.invh2;
    return f - lap;
  } else {
    T ax = q.s;          // u_{i,j-1}
    ax = ax + q.n;       // u_{i,j+1}
    ax = ax + q.w;       // u_{i-1,j}
    ax = ax + q.e;       // u_{i+1,j}
    T b = -((T)20 * q.c);
    b = b + (T)4 * ax;
    b = b + q.ne;        // u_{i+1,j+1}
    b = b + q.nw;        // u_{i-1,j+1}
    b = b + q.sw;        // u_{i-1,j-1}
    b = b + q.se;        // u_{i+1,j-1}
    return f - b * k.c6;
  }
}

template <class T, int ORDER, class UA>
__device__ __forceinline__ Nb9<T> gather9(const UA &u, int x, int y) {
  Nb9<T> q;
  q.c = u(x, y);
  q.w = u(x - 1, y);
  q.s = u(x, y - 1);
  q.e = u(x + 1, y);
  q.n = u(x, y + 1);
  if (ORDER == 4) {
    q.ne = u(x + 1, y + 1);
    q.nw = u(x - 1, y + 1);
    q.sw = u(x - 1, y - 1);
    q.se = u(x + 1, y - 1);
  } else {
    q.ne = q.nw = q.sw = q.se = (T)0;
  }
  return q;
}

template <class T, int ORDER, class UA, class FA>
__device__ __forceinline__ T res2(const UA &u, const FA &f, int x, int y, const Coef<T> &k) {
  return res2v<T, ORDER>(gather9<T, ORDER>(u, x, y), f(x, y), k);
}

// r at any lattice node of the finest grid: 0 on the boundary (reading A1).
template <class T, int ORDER, class UA, class FA>
__device__ __forceinline__ T res2z(const UA &u, const FA &f, int x, int y, int M, const Coef<T> &k) {
  if (x <= 0 || y <= 0 || x >= M || y >= M) return (T)0;
  return res2<T, ORDER>(u, f, x, y, k);
}

// Erest2r: (1/8)(4r + r_{i-1,j} + r_{i,j-1} + r_{i+1,j} + r_{i,j+1}).
template <class T>
__device__ __forceinline__ T erest2r(T c, T w, T s, T e, T n) {
  T t = (T)4 * c;
  t = t + w;
  t = t + s;
  t = t + e;
  t = t + n;
  return t * (T)0.125;
}

// Erest2b: (1/8)(4r + r_{i-1,j-1} + r_{i+1,j-1} + r_{i+1,j+1} + r_{i-1,j+1}).
template <class T>
__device__ __forceinline__ T erest2b(T c, T sw, T se, T ne, T nw) {
  T t = (T)4 * c;
  t = t + sw;
  t = t + se;
  t = t + ne;
  t = t + nw;
  return t * (T)0.125;
}

// Jacobi (Eajacr/Eajacb P:350-359, green "similarly" P:360):
// (1/4)(-c r + v1 + v2 + v3 + v4), c = kappa p (sh)^2.
template <class T>
__device__ __forceinline__ T jac4(T c, T r, T v1, T v2, T v3, T v4) {
  T t = -(c * r);
  t = t + v1;
  t = t + v2;
  t = t + v3;
  t = t + v4;
  return t * (T)0.25;
}

// ------------------------------------------------ per-node step bodies
// Shared by the reference grid kernels (one thread per index t) and the
// single-CTA coarse kernel (block-stride loop over t).

// a2: Erest2r from the dense A(s) residual onto D(s); t over (M/2+1)^2,
// writes E(a,b) = node (2a,2b) and O(a,b) = node (2a+1,2b+1) when interior.
template <class T, class I>
__device__ __forceinline__ void node_rest_ad(const D2<const T> &r, const S2<T> &d, int M, I t) {
  int H = M / 2 + 1;
  int a = (int)(t % H), b = (int)(t / H);
  int x = 2 * a, y = 2 * b;
  if (x >= 2 && y >= 2 && x <= M - 2 && y <= M - 2)
    d.e[(int64_t)b * d.pitch + a] = erest2r(r(x, y), r(x - 1, y), r(x, y - 1), r(x + 1, y), r(x, y + 1));
  x += 1;
  y += 1;
  if (x <= M - 1 && y <= M - 1)
    d.o[(int64_t)b * d.pitch + a] = erest2r(r(x, y), r(x - 1, y), r(x, y - 1), r(x + 1, y), r(x, y + 1));
}

// a3: Erest2b from D(s) onto A(2s); coarse node (X,Y) is lattice node
// (2X,2Y); t over (Mc-1)^2.
template <class T, class I>
__device__ __forceinline__ void node_rest_da(const S2<const T> &d, const D2<T> &r, int Mc, I t) {
  int W = Mc - 1;
  int X = (int)(t % W) + 1, Y = (int)(t / W) + 1;
  int x = 2 * X, y = 2 * Y;
  r(X, Y) = erest2b(d.get(x, y), d.get(x - 1, y - 1), d.get(x + 1, y - 1), d.get(x + 1, y + 1), d.get(x - 1, y + 1));
}

// a4: coarsest level, one interior node (reading A4): v = (1/4)(-p H^2 r).
template <class T>
__device__ __forceinline__ void node_coarsest(const D2<const T> &r, const D2<T> &v, T c, int *counter) {
  v(1, 1) = (-(c * r(1, 1))) * (T)0.25;
  if (counter) *counter += 1;   // this cycle's norm slot is complete
}

// a5: colour 1 on O (nodes of D(s) not on A(2s)): Eajacr from
// the coarse A(2s) values at the 4 diagonal neighbours; t over (M/2)^2.
template <class T, class I>
__device__ __forceinline__ void node_jac_d1(const D2<const T> &vc, const S2<const T> &r, const S2<T> &v, int M, T c,
                                            I t) {
  int W = M / 2;
  int a = (int)(t % W), b = (int)(t / W);
  int x = 2 * a + 1, y = 2 * b + 1;
  v.o[(int64_t)b * v.pitch + a] = jac4(c, r.o[(int64_t)b * r.pitch + a], vc((x - 1) / 2, (y - 1) / 2),
                                       vc((x + 1) / 2, (y - 1) / 2), vc((x + 1) / 2, (y + 1) / 2),
                                       vc((x - 1) / 2, (y + 1) / 2));
}

// a6: colour 2 on E (= A(2s) positions): Eajacb from the new O
// values; uses the D(s) residual at that node (reading A10); t over (M/2-1)^2.
template <class T, class I>
__device__ __forceinline__ void node_jac_d2(const S2<const T> &r, const S2<T> &v, int M, T c, I t) {
  int W = M / 2 - 1;
  int a = (int)(t % W) + 1, b = (int)(t / W) + 1;
  int x = 2 * a, y = 2 * b;
  v.e[(int64_t)b * v.pitch + a] = jac4(c, r.e[(int64_t)b * r.pitch + a], v.get(x - 1, y - 1), v.get(x + 1, y - 1),
                                       v.get(x + 1, y + 1), v.get(x - 1, y + 1));
}

// a7 (s > 1): colour 1 on the green-only nodes (x+y odd) from D(s), colour 2
// on the D(s) nodes from the new green values ("similarly for a green grid",
// P:228-230; reading A5), c = p (sh)^2; t over (M-1)^2.
template <class T, class I>
__device__ __forceinline__ void node_jac_a1(const S2<const T> &vd, const D2<const T> &r, const D2<T> &v, int M, T c,
                                            I t) {
  int W = M - 1;
  int x = (int)(t % W) + 1, y = (int)(t / W) + 1;
  if (((x + y) & 1) == 0) return;
  v(x, y) = jac4(c, r(x, y), vd.get(x - 1, y), vd.get(x, y - 1), vd.get(x + 1, y), vd.get(x, y + 1));
}

template <class T, class I>
__device__ __forceinline__ void node_jac_a2(const D2<const T> &r, const D2<T> &v, int M, T c, I t) {
  int W = M - 1;
  int x = (int)(t % W) + 1, y = (int)(t / W) + 1;
  if (((x + y) & 1) == 1) return;
  v(x, y) = jac4(c, r(x, y), v(x - 1, y), v(x, y - 1), v(x + 1, y), v(x, y + 1));
}

}  // namespace mg
