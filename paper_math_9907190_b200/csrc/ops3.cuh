// ops3.cuh -- the 3D per-node formulas of the V-cycle, shared by the
// reference kernels (k3d.cu) and the TMA plane kernels (k3f.cu).  Canonical
// evaluation order; the library is compiled with --fmad=false.
#pragma once
#include "common.cuh"

namespace mg {

// Axis offsets in the printed order of Erred / Ermagm / Egprolg / Egprolr.
static __constant__ int c_ax6[6][3] = {{1, 0, 0}, {-1, 0, 0}, {0, 1, 0}, {0, -1, 0}, {0, 0, 1}, {0, 0, -1}};
// Face diagonals in the printed order of Ermagc = Erprolm.
static __constant__ int c_fd12[12][3] = {{1, 1, 0},  {1, -1, 0},  {-1, -1, 0}, {-1, 1, 0}, {1, 0, 1},  {1, 0, -1},
                                  {-1, 0, -1}, {-1, 0, 1}, {0, 1, 1},   {0, 1, -1}, {0, -1, -1}, {0, -1, 1}};
// Body diagonals in the printed order of Erblu = Emprolm/b.
static __constant__ int c_bd8[8][3] = {{1, 1, 1},  {1, 1, -1},  {1, -1, 1},  {1, -1, -1},
                                {-1, 1, 1}, {-1, 1, -1}, {-1, -1, 1}, {-1, -1, -1}};
// Erprolr for normal axis x, y, z: the normal pair (weight 2)
// then the 4 in-plane corners; the z table is printed, x and y follow by the
// cyclic permutation (a,b,c) -> (c,a,b) / (b,c,a) (reading A8).
static __constant__ int c_erp[3][6][3] = {
    {{1, 0, 0}, {-1, 0, 0}, {0, 1, 1}, {0, 1, -1}, {0, -1, -1}, {0, -1, 1}},
    {{0, 1, 0}, {0, -1, 0}, {1, 0, 1}, {-1, 0, 1}, {-1, 0, -1}, {1, 0, -1}},
    {{0, 0, 1}, {0, 0, -1}, {1, 1, 0}, {1, -1, 0}, {-1, -1, 0}, {-1, 1, 0}}};

// ------------------------------------------------------------- residual
// order 2: 7-point, centre first then i+1,i-1,j+1,j-1,k+1,k-1.
// order 4: Efos4, f~ precomputed; bracket in printed order.
// The 19 values around a node: centre, 6 axis and 12 face-diagonal
// neighbours (order 2 uses the first seven).
template <class T>
struct Nb19 {
  T c, xp, xm, yp, ym, zp, zm;
  T xpyp, xmyp, xmym, xpym, ypzp, ypzm, ymzm, ymzp, xpzp, xmzp, xmzm, xpzm;
};

template <class T, int ORDER>
__device__ __forceinline__ T res3v(const Nb19<T> &q, T f, const Coef<T> &k) {
  if (ORDER == 2) {
    T lap = -((T)6 * q.c);
    lap = lap + q.xp;
    lap = lap + q.xm;
    lap = lap + q.yp;
    lap = lap + q.ym;
    lap = lap + q.zp;
    lap = lap + q.zm;
    lap = lap * k.invh2;
    return f - lap;
  } else {
    T ax = q.ym;
    ax = ax + q.yp;
    ax = ax + q.xm;
    ax = ax + q.xp;
    ax = ax + q.zp;
    ax = ax + q.zm;
    T b = -((T)24 * q.c);
    b = b + (T)2 * ax;
    b = b + q.xpyp;
    b = b + q.xmyp;
    b = b + q.xmym;
    b = b + q.xpym;
    b = b + q.ypzp;
    b = b + q.ypzm;
    b = b + q.ymzm;
    b = b + q.ymzp;
    b = b + q.xpzp;
    b = b + q.xmzp;
    b = b + q.xmzm;
    b = b + q.xpzm;
    return f - b * k.c6;
  }
}

template <class T, int ORDER, class UA>
__device__ __forceinline__ Nb19<T> gather19(const UA &u, int x, int y, int z) {
  Nb19<T> q;
  q.c = u(x, y, z);
  q.xp = u(x + 1, y, z);
  q.xm = u(x - 1, y, z);
  q.yp = u(x, y + 1, z);
  q.ym = u(x, y - 1, z);
  q.zp = u(x, y, z + 1);
  q.zm = u(x, y, z - 1);
  if (ORDER == 4) {
    q.xpyp = u(x + 1, y + 1, z);
    q.xmyp = u(x - 1, y + 1, z);
    q.xmym = u(x - 1, y - 1, z);
    q.xpym = u(x + 1, y - 1, z);
    q.ypzp = u(x, y + 1, z + 1);
    q.ypzm = u(x, y + 1, z - 1);
    q.ymzm = u(x, y - 1, z - 1);
    q.ymzp = u(x, y - 1, z + 1);
    q.xpzp = u(x + 1, y, z + 1);
    q.xmzp = u(x - 1, y, z + 1);
    q.xmzm = u(x - 1, y, z - 1);
    q.xpzm = u(x + 1, y, z - 1);
  }
  return q;
}

template <class T, int ORDER, class UA, class FA>
__device__ __forceinline__ T res3(const UA &u, const FA &f, int x, int y, int z, const Coef<T> &k) {
  return res3v<T, ORDER>(gather19<T, ORDER>(u, x, y, z), f(x, y, z), k);
}

template <class T, int ORDER, class UA, class FA>
__device__ __forceinline__ T res3z(const UA &u, const FA &f, int x, int y, int z, int M, const Coef<T> &k) {
  if (x <= 0 || y <= 0 || z <= 0 || x >= M || y >= M || z >= M) return (T)0;
  return res3<T, ORDER>(u, f, x, y, z, k);
}

__device__ __forceinline__ bool inner3(int x, int y, int z, int M) {
  return x >= 1 && y >= 1 && z >= 1 && x <= M - 1 && y <= M - 1 && z <= M - 1;
}

// Erred: (1/12)(6r + r_{i+1} + r_{i-1} + r_{j+1} + r_{j-1} + r_{k+1} + r_{k-1}).
template <class T>
__device__ __forceinline__ T erred(T c, const T nb[6]) {
  T t = (T)6 * c;
#pragma unroll
  for (int q = 0; q < 6; q++) t = t + nb[q];
  return t * (T)(1.0 / 12.0);
}

}  // namespace mg
