// k3l.cu -- 3D level kernels on the packed parity sublattices (sm_100a).
//
// Every 3D step of the octave (Erred for s > 1, Ermagc/Ermagm, Erblu,
// Emprolm/b, Erprolr/m, Egprolg/r) is written here in half-index form: the
// sublattice arrays C, Fx, Fy, Fz (red), C, B (magenta) are dense H^3 arrays
// (H = M/2 + 1) and every stencil becomes a box stencil with offsets in
// {-1, 0, 1}.  One thread per half-index (a, b, c), a fastest (coalesced),
// block (32, 8) over (a, b), grid.z over c; no parity tests at run time.
// The neighbour order of every sum is the paper's printed order (DESIGN.md
// canonical arithmetic), so the results are bit-identical to the reference
// kernels.
#include <cooperative_groups.h>
#include <cstdio>
#include <cstdlib>
#include <initializer_list>

#include "kernels.h"
#include "tma.cuh"
#include "ops3.cuh"

namespace mg {

namespace l3 {

// sublattice slots of S3: (x&1) | (y&1)<<1 | (z&1)<<2
constexpr int C = 0, FX = 6, FY = 5, FZ = 3, B = 7;

template <class T>
struct Sub {   // one sublattice array of a split level
  T *p;
  int64_t pitch, plane;
  __device__ __forceinline__ T &operator()(int a, int b, int c) const {
    return p[(int64_t)c * plane + (int64_t)b * pitch + a];
  }
};
template <class T>
__device__ __forceinline__ Sub<T> sub(const S3<T> &s, int k) {
  return Sub<T>{s.s[k], s.pitch, s.plane};
}

template <class T>
__device__ __forceinline__ T sum6(T v0, T v1, T v2, T v3, T v4, T v5) {
  T t = v0;
  t = t + v1;
  t = t + v2;
  t = t + v3;
  t = t + v4;
  t = t + v5;
  return t;
}

}  // namespace l3

using namespace l3;

#define IDX3                                                                                    \
  pdl_trigger();                                                                                \
  pdl_wait();                                                                                   \
  const int a = blockIdx.x * 32 + threadIdx.x, b = blockIdx.y * 8 + threadIdx.y, c = blockIdx.z + c0; \
  if (a >= H || b >= H) return;

// --------------------------------------------------------- G(s) -> R(s)
// Erred from the dense G(s) residual; the 2x2x2 block (a,b,c)
// holds C (0,0,0), Fx (0,1,1), Fy (1,0,1), Fz (1,1,0).
template <class T>
__device__ __forceinline__ void b3_rest_gr(D3<const T> r, S3<T> out, int M, int H, int a, int b, int c) {
  const int x = 2 * a, y = 2 * b, z = 2 * c;
  auto er = [&](int X, int Y, int Z) {
    T nb[6] = {r(X + 1, Y, Z), r(X - 1, Y, Z), r(X, Y + 1, Z), r(X, Y - 1, Z), r(X, Y, Z + 1), r(X, Y, Z - 1)};
    return erred(r(X, Y, Z), nb);
  };
  const bool in_a = x >= 2 && x <= M - 2, in_b = y >= 2 && y <= M - 2, in_c = z >= 2 && z <= M - 2;
  const bool od_a = x + 1 <= M - 1, od_b = y + 1 <= M - 1, od_c = z + 1 <= M - 1;
  if (in_a && in_b && in_c) sub(out, C)(a, b, c) = er(x, y, z);
  if (in_a && od_b && od_c) sub(out, FX)(a, b, c) = er(x, y + 1, z + 1);
  if (od_a && in_b && od_c) sub(out, FY)(a, b, c) = er(x + 1, y, z + 1);
  if (od_a && od_b && in_c) sub(out, FZ)(a, b, c) = er(x + 1, y + 1, z);
}

template <class T>
__global__ void __launch_bounds__(256) k3l_rest_gr(D3<const T> r, S3<T> out, int M, int H, int c0) {
  IDX3
  b3_rest_gr(r, out, M, H, a, b, c);
}

// --------------------------------------------------------- R(s) -> M(s)
// corners: Ermagc (1/24)(12 r + 12 face diagonals, printed order);
// centres: Ermagm (1/6)(6 axis neighbours), zero self weight.
template <class T>
__device__ __forceinline__ void b3_rest_rm(S3<const T> rr, S3<T> rm, int H, int a, int b, int c) {
  Sub<const T> Cr{rr.s[C], rr.pitch, rr.plane}, Fx{rr.s[FX], rr.pitch, rr.plane}, Fy{rr.s[FY], rr.pitch, rr.plane},
      Fz{rr.s[FZ], rr.pitch, rr.plane};
  if (a >= 1 && b >= 1 && c >= 1 && a <= H - 2 && b <= H - 2 && c <= H - 2) {
    T t = (T)12 * Cr(a, b, c);
    t = t + Fz(a, b, c);              // (+1,+1, 0)
    t = t + Fz(a, b - 1, c);          // (+1,-1, 0)
    t = t + Fz(a - 1, b - 1, c);      // (-1,-1, 0)
    t = t + Fz(a - 1, b, c);          // (-1,+1, 0)
    t = t + Fy(a, b, c);              // (+1, 0,+1)
    t = t + Fy(a, b, c - 1);          // (+1, 0,-1)
    t = t + Fy(a - 1, b, c - 1);      // (-1, 0,-1)
    t = t + Fy(a - 1, b, c);          // (-1, 0,+1)
    t = t + Fx(a, b, c);              // ( 0,+1,+1)
    t = t + Fx(a, b, c - 1);          // ( 0,+1,-1)
    t = t + Fx(a, b - 1, c - 1);      // ( 0,-1,-1)
    t = t + Fx(a, b - 1, c);          // ( 0,-1,+1)
    sub(rm, C)(a, b, c) = t * (T)(1.0 / 24.0);
  }
  if (a <= H - 2 && b <= H - 2 && c <= H - 2) {
    // centre (2a+1, 2b+1, 2c+1): i+1, i-1, j+1, j-1, k+1, k-1
    T t = sum6(Fx(a + 1, b, c), Fx(a, b, c), Fy(a, b + 1, c), Fy(a, b, c), Fz(a, b, c + 1), Fz(a, b, c));
    sub(rm, B)(a, b, c) = t * (T)(1.0 / 6.0);
  }
}

template <class T>
__global__ void __launch_bounds__(256) k3l_rest_rm(S3<const T> rr, S3<T> rm, int H, int c0) {
  IDX3
  b3_rest_rm(rr, rm, H, a, b, c);
}

// ------------------------------------------------------- M(s) -> G(2s)
// Erblu: (1/16)(8 r + 8 body diagonals, printed order).
template <class T>
__device__ __forceinline__ void b3_rest_mg(S3<const T> rm, D3<T> g2, int Mc, int a, int b, int c) {
  if (a < 1 || b < 1 || c < 1 || a > Mc - 1 || b > Mc - 1 || c > Mc - 1) return;
  Sub<const T> Cm{rm.s[C], rm.pitch, rm.plane}, Bm{rm.s[B], rm.pitch, rm.plane};
  T t = (T)8 * Cm(a, b, c);
  t = t + Bm(a, b, c);               // (+,+,+)
  t = t + Bm(a, b, c - 1);           // (+,+,-)
  t = t + Bm(a, b - 1, c);           // (+,-,+)
  t = t + Bm(a, b - 1, c - 1);       // (+,-,-)
  t = t + Bm(a - 1, b, c);           // (-,+,+)
  t = t + Bm(a - 1, b, c - 1);       // (-,+,-)
  t = t + Bm(a - 1, b - 1, c);       // (-,-,+)
  t = t + Bm(a - 1, b - 1, c - 1);   // (-,-,-)
  g2(a, b, c) = t * (T)(1.0 / 16.0);
}

template <class T>
__global__ void __launch_bounds__(256) k3l_rest_mg(S3<const T> rm, D3<T> g2, int Mc, int c0) {
  const int H = Mc + 1;
  IDX3
  b3_rest_mg(rm, g2, Mc, a, b, c);
}

// ----------------------------------------------- M(s) from G(2s): a13
// Emprolm on the centres, then (second kernel) Emprolb
// on the corners from the new centres; c = 4 p_m (sh)^2.
template <class T>
__device__ __forceinline__ void b3_jac_m1(D3<const T> vc, S3<const T> r, S3<T> v, int H, T cc, int a, int b, int c) {
  if (a > H - 2 || b > H - 2 || c > H - 2) return;
  T t = -(cc * r.s[B][(int64_t)c * r.plane + (int64_t)b * r.pitch + a]);
  t = t + vc(a + 1, b + 1, c + 1);   // (+,+,+)
  t = t + vc(a + 1, b + 1, c);       // (+,+,-)
  t = t + vc(a + 1, b, c + 1);       // (+,-,+)
  t = t + vc(a + 1, b, c);           // (+,-,-)
  t = t + vc(a, b + 1, c + 1);       // (-,+,+)
  t = t + vc(a, b + 1, c);           // (-,+,-)
  t = t + vc(a, b, c + 1);           // (-,-,+)
  t = t + vc(a, b, c);               // (-,-,-)
  sub(v, B)(a, b, c) = t * (T)0.125;
}

template <class T>
__global__ void __launch_bounds__(256) k3l_jac_m1(D3<const T> vc, S3<const T> r, S3<T> v, int H, T cc, int c0) {
  IDX3
  b3_jac_m1(vc, r, v, H, cc, a, b, c);
}

template <class T>
__device__ __forceinline__ void b3_jac_m2(S3<const T> r, S3<T> v, int H, T cc, int a, int b, int c) {
  if (a < 1 || b < 1 || c < 1 || a > H - 2 || b > H - 2 || c > H - 2) return;
  Sub<T> Bv = sub(v, B);
  T t = -(cc * r.s[C][(int64_t)c * r.plane + (int64_t)b * r.pitch + a]);
  t = t + Bv(a, b, c);
  t = t + Bv(a, b, c - 1);
  t = t + Bv(a, b - 1, c);
  t = t + Bv(a, b - 1, c - 1);
  t = t + Bv(a - 1, b, c);
  t = t + Bv(a - 1, b, c - 1);
  t = t + Bv(a - 1, b - 1, c);
  t = t + Bv(a - 1, b - 1, c - 1);
  sub(v, C)(a, b, c) = t * (T)0.125;
}

template <class T>
__global__ void __launch_bounds__(256) k3l_jac_m2(S3<const T> r, S3<T> v, int H, T cc, int c0) {
  IDX3
  b3_jac_m2(r, v, H, cc, a, b, c);
}

// ------------------------------------------------- R(s) from M(s): a14
// Erprolr on the face centres (normal axis = the even
// coordinate, reading A8; the x- and y-face sums are the cyclic permutations
// of the printed z-face sum), c1 = 2 p_r1 (sh)^2; then Erprolm on
// the corners from the new faces, c2 = 4 p_r2 (sh)^2.
template <class T>
__device__ __forceinline__ void b3_jac_r1(S3<const T> vm, S3<const T> r, S3<T> v, int H, T c1, int a, int b, int c) {
  Sub<const T> Cm{vm.s[C], vm.pitch, vm.plane}, Bm{vm.s[B], vm.pitch, vm.plane};
  const int64_t o = (int64_t)c * r.plane + (int64_t)b * r.pitch + a;
  const bool lo_a = a <= H - 2, lo_b = b <= H - 2, lo_c = c <= H - 2;
  // Fx (2a, 2b+1, 2c+1): normal x; in-plane (0,+1,+1),(0,+1,-1),(0,-1,-1),(0,-1,+1)
  if (a >= 1 && lo_a && lo_b && lo_c) {
    T nrm = Bm(a, b, c);
    nrm = nrm + Bm(a - 1, b, c);
    T t = -(c1 * r.s[FX][o]);
    t = t + (T)2 * nrm;
    t = t + Cm(a, b + 1, c + 1);
    t = t + Cm(a, b + 1, c);
    t = t + Cm(a, b, c);
    t = t + Cm(a, b, c + 1);
    sub(v, FX)(a, b, c) = t * (T)0.125;
  }
  // Fy (2a+1, 2b, 2c+1): normal y; in-plane (+1,0,+1),(-1,0,+1),(-1,0,-1),(+1,0,-1)
  if (b >= 1 && lo_a && lo_b && lo_c) {
    T nrm = Bm(a, b, c);
    nrm = nrm + Bm(a, b - 1, c);
    T t = -(c1 * r.s[FY][o]);
    t = t + (T)2 * nrm;
    t = t + Cm(a + 1, b, c + 1);
    t = t + Cm(a, b, c + 1);
    t = t + Cm(a, b, c);
    t = t + Cm(a + 1, b, c);
    sub(v, FY)(a, b, c) = t * (T)0.125;
  }
  // Fz (2a+1, 2b+1, 2c): normal z; in-plane (+1,+1,0),(+1,-1,0),(-1,-1,0),(-1,+1,0)
  if (c >= 1 && lo_a && lo_b && lo_c) {
    T nrm = Bm(a, b, c);
    nrm = nrm + Bm(a, b, c - 1);
    T t = -(c1 * r.s[FZ][o]);
    t = t + (T)2 * nrm;
    t = t + Cm(a + 1, b + 1, c);
    t = t + Cm(a + 1, b, c);
    t = t + Cm(a, b, c);
    t = t + Cm(a, b + 1, c);
    sub(v, FZ)(a, b, c) = t * (T)0.125;
  }
}

template <class T>
__global__ void __launch_bounds__(256) k3l_jac_r1(S3<const T> vm, S3<const T> r, S3<T> v, int H, T c1, int c0) {
  IDX3
  b3_jac_r1(vm, r, v, H, c1, a, b, c);
}

template <class T>
__device__ __forceinline__ void b3_jac_r2(S3<const T> r, S3<T> v, int H, T c2, int a, int b, int c) {
  if (a < 1 || b < 1 || c < 1 || a > H - 2 || b > H - 2 || c > H - 2) return;
  Sub<T> Fx = sub(v, FX), Fy = sub(v, FY), Fz = sub(v, FZ);
  T t = -(c2 * r.s[C][(int64_t)c * r.plane + (int64_t)b * r.pitch + a]);
  t = t + Fz(a, b, c);              // (+1,+1, 0)
  t = t + Fz(a, b - 1, c);          // (+1,-1, 0)
  t = t + Fz(a - 1, b - 1, c);      // (-1,-1, 0)
  t = t + Fz(a - 1, b, c);          // (-1,+1, 0)
  t = t + Fy(a, b, c);              // (+1, 0,+1)
  t = t + Fy(a, b, c - 1);          // (+1, 0,-1)
  t = t + Fy(a - 1, b, c - 1);      // (-1, 0,-1)
  t = t + Fy(a - 1, b, c);          // (-1, 0,+1)
  t = t + Fx(a, b, c);              // ( 0,+1,+1)
  t = t + Fx(a, b, c - 1);          // ( 0,+1,-1)
  t = t + Fx(a, b - 1, c - 1);      // ( 0,-1,-1)
  t = t + Fx(a, b - 1, c);          // ( 0,-1,+1)
  sub(v, C)(a, b, c) = t * (T)(1.0 / 12.0);
}

template <class T>
__global__ void __launch_bounds__(256) k3l_jac_r2(S3<const T> r, S3<T> v, int H, T c2, int c0) {
  IDX3
  b3_jac_r2(r, v, H, c2, a, b, c);
}

// ------------------------------------------------- G(s) from R(s): a15
// Egprolg on the green-only nodes of the block (a,b,c):
// (1,0,0), (0,1,0), (0,0,1), (1,1,1); neighbours i+1, i-1, j+1, j-1, k+1, k-1.
// FINE: r recomputed from (u_old, f) and the green v kept in `g`.
template <class T, int ORDER, bool FINE>
__device__ __forceinline__ void b3_jac_g1(S3<const T> vr, D3<const T> rin, D3<const T> u, D3<const T> f,
                                                  D3<T> g, int M, int H, T cc, Coef<T> k, int a, int b, int c) {
  Sub<const T> Cr{vr.s[C], vr.pitch, vr.plane}, Fx{vr.s[FX], vr.pitch, vr.plane}, Fy{vr.s[FY], vr.pitch, vr.plane},
      Fz{vr.s[FZ], vr.pitch, vr.plane};
  const int x = 2 * a, y = 2 * b, z = 2 * c;
  auto rr = [&](int X, int Y, int Z) -> T {
    if (FINE) return res3<T, ORDER>(u, f, X, Y, Z, k);
    return rin(X, Y, Z);
  };
  auto jac6 = [&](T r, T v0, T v1, T v2, T v3, T v4, T v5) {
    T t = -(cc * r);
    t = t + v0;
    t = t + v1;
    t = t + v2;
    t = t + v3;
    t = t + v4;
    t = t + v5;
    return t * (T)(1.0 / 6.0);
  };
  const bool in_a = x >= 2 && x <= M - 2, in_b = y >= 2 && y <= M - 2, in_c = z >= 2 && z <= M - 2;
  const bool od_a = x + 1 <= M - 1, od_b = y + 1 <= M - 1, od_c = z + 1 <= M - 1;
  if (od_a && in_b && in_c)   // (2a+1, 2b, 2c)
    g(x + 1, y, z) = jac6(rr(x + 1, y, z), Cr(a + 1, b, c), Cr(a, b, c), Fz(a, b, c), Fz(a, b - 1, c), Fy(a, b, c),
                          Fy(a, b, c - 1));
  if (in_a && od_b && in_c)   // (2a, 2b+1, 2c)
    g(x, y + 1, z) = jac6(rr(x, y + 1, z), Fz(a, b, c), Fz(a - 1, b, c), Cr(a, b + 1, c), Cr(a, b, c), Fx(a, b, c),
                          Fx(a, b, c - 1));
  if (in_a && in_b && od_c)   // (2a, 2b, 2c+1)
    g(x, y, z + 1) = jac6(rr(x, y, z + 1), Fy(a, b, c), Fy(a - 1, b, c), Fx(a, b, c), Fx(a, b - 1, c), Cr(a, b, c + 1),
                          Cr(a, b, c));
  if (od_a && od_b && od_c)   // (2a+1, 2b+1, 2c+1)
    g(x + 1, y + 1, z + 1) = jac6(rr(x + 1, y + 1, z + 1), Fx(a + 1, b, c), Fx(a, b, c), Fy(a, b + 1, c), Fy(a, b, c),
                                  Fz(a, b, c + 1), Fz(a, b, c));
}

template <class T, int ORDER, bool FINE>
__global__ void __launch_bounds__(256) k3l_jac_g1(S3<const T> vr, D3<const T> rin, D3<const T> u, D3<const T> f,
                                                  D3<T> g, int M, int H, T cc, Coef<T> k, int c0) {
  IDX3
  b3_jac_g1<T, ORDER, FINE>(vr, rin, u, f, g, M, H, cc, k, a, b, c);
}

// Egprolr on the red nodes of the block from the new green
// values in `g`; FINE: out = u_old + v at all 8 nodes of the block;
// otherwise out = v_G(s) at the red nodes (the green ones are already in g = out).
template <class T, int ORDER, bool FINE>
__device__ __forceinline__ void b3_jac_g2(D3<const T> rin, D3<const T> u, D3<const T> f, D3<const T> g,
                                                  D3<T> out, int M, int H, T cc, Coef<T> k, int a, int b, int c) {
  const int x = 2 * a, y = 2 * b, z = 2 * c;
  auto rr = [&](int X, int Y, int Z) -> T {
    if (FINE) return res3<T, ORDER>(u, f, X, Y, Z, k);
    return rin(X, Y, Z);
  };
  auto red = [&](int X, int Y, int Z) {
    T t = -(cc * rr(X, Y, Z));
    t = t + g(X + 1, Y, Z);
    t = t + g(X - 1, Y, Z);
    t = t + g(X, Y + 1, Z);
    t = t + g(X, Y - 1, Z);
    t = t + g(X, Y, Z + 1);
    t = t + g(X, Y, Z - 1);
    return t * (T)(1.0 / 6.0);
  };
  const bool in_a = x >= 2 && x <= M - 2, in_b = y >= 2 && y <= M - 2, in_c = z >= 2 && z <= M - 2;
  const bool od_a = x + 1 <= M - 1, od_b = y + 1 <= M - 1, od_c = z + 1 <= M - 1;
  T vC = (in_a && in_b && in_c) ? red(x, y, z) : (T)0;
  T vFx = (in_a && od_b && od_c) ? red(x, y + 1, z + 1) : (T)0;
  T vFy = (od_a && in_b && od_c) ? red(x + 1, y, z + 1) : (T)0;
  T vFz = (od_a && od_b && in_c) ? red(x + 1, y + 1, z) : (T)0;
  if (FINE) {
    // u_new = u_old + v on the whole block (green v from g)
    if (in_a && in_b && in_c) out(x, y, z) = u(x, y, z) + vC;
    if (in_a && od_b && od_c) out(x, y + 1, z + 1) = u(x, y + 1, z + 1) + vFx;
    if (od_a && in_b && od_c) out(x + 1, y, z + 1) = u(x + 1, y, z + 1) + vFy;
    if (od_a && od_b && in_c) out(x + 1, y + 1, z) = u(x + 1, y + 1, z) + vFz;
    if (od_a && in_b && in_c) out(x + 1, y, z) = u(x + 1, y, z) + g(x + 1, y, z);
    if (in_a && od_b && in_c) out(x, y + 1, z) = u(x, y + 1, z) + g(x, y + 1, z);
    if (in_a && in_b && od_c) out(x, y, z + 1) = u(x, y, z + 1) + g(x, y, z + 1);
    if (od_a && od_b && od_c) out(x + 1, y + 1, z + 1) = u(x + 1, y + 1, z + 1) + g(x + 1, y + 1, z + 1);
  } else {
    if (in_a && in_b && in_c) out(x, y, z) = vC;
    if (in_a && od_b && od_c) out(x, y + 1, z + 1) = vFx;
    if (od_a && in_b && od_c) out(x + 1, y, z + 1) = vFy;
    if (od_a && od_b && in_c) out(x + 1, y + 1, z) = vFz;
  }
}

template <class T, int ORDER, bool FINE>
__global__ void __launch_bounds__(256) k3l_jac_g2(D3<const T> rin, D3<const T> u, D3<const T> f, D3<const T> g,
                                                  D3<T> out, int M, int H, T cc, Coef<T> k, int c0) {
  IDX3
  b3_jac_g2<T, ORDER, FINE>(rin, u, f, g, out, M, H, cc, k, a, b, c);
}

#undef IDX3

// ------------------------------------------------------ coarse octaves
// One CTA runs every octave o >= oc (oc >= 1): the same step bodies in a
// block-stride loop, __syncthreads between steps (arrays are L1/L2 resident).
template <class T>
__global__ void __launch_bounds__(1024) k3l_coarse(const Lev3<T> *lv, int oc, int k, int *counter) {
  pdl_trigger();
  pdl_wait();
  const int tid = threadIdx.x, bs = blockDim.x;
  D3<const T> none{nullptr, 0, 0};
  Coef<T> k0{};
  auto cd = [](const D3<T> &a) { return D3<const T>{a.p, a.pitch, a.plane}; };
  auto cs = [](const S3<T> &a) {
    S3<const T> o;
    for (int i = 0; i < 8; i++) o.s[i] = a.s[i];
    o.pitch = a.pitch;
    o.plane = a.plane;
    return o;
  };
#define LOOP3(HH, BODY)                                            \
  {                                                                \
    const int H_ = (HH);                                           \
    const int n_ = H_ * H_ * H_;                                   \
    for (int t = tid; t < n_; t += bs) {                           \
      const int a = t % H_, b = (t / H_) % H_, c = t / (H_ * H_); \
      BODY;                                                        \
    }                                                              \
    __syncthreads();                                               \
  }
  for (int o = oc; o + 1 < k; o++) {
    const Lev3<T> L = lv[o], Lc = lv[o + 1];
    const int H = L.M / 2 + 1;
    LOOP3(H, b3_rest_gr(cd(L.rG), L.rR, L.M, H, a, b, c));
    LOOP3(H, b3_rest_rm(cs(L.rR), L.rM, H, a, b, c));
    LOOP3(Lc.M + 1, b3_rest_mg(cs(L.rM), Lc.rG, Lc.M, a, b, c));
  }
  if (tid == 0) {
    const Lev3<T> L = lv[k - 1];
    L.vG(1, 1, 1) = (-(L.cG * L.rG(1, 1, 1))) * (T)(1.0 / 6.0);   // reading A4
    if (counter) *counter += 1;
  }
  __syncthreads();
  for (int o = k - 2; o >= oc; o--) {
    const Lev3<T> L = lv[o], Lc = lv[o + 1];
    const int H = L.M / 2 + 1;
    LOOP3(H, b3_jac_m1(cd(Lc.vG), cs(L.rM), L.vM, H, L.cMg, a, b, c));
    LOOP3(H, b3_jac_m2(cs(L.rM), L.vM, H, L.cMg, a, b, c));
    LOOP3(H, b3_jac_r1(cs(L.vM), cs(L.rR), L.vR, H, L.cR1, a, b, c));
    LOOP3(H, b3_jac_r2(cs(L.rR), L.vR, H, L.cR2, a, b, c));
    LOOP3(H, (b3_jac_g1<T, 2, false>(cs(L.vR), cd(L.rG), none, none, L.vG, L.M, H, L.cG, k0, a, b, c)));
    LOOP3(H, (b3_jac_g2<T, 2, false>(cd(L.rG), none, none, cd(L.vG), L.vG, L.M, H, L.cG, k0, a, b, c)));
  }
#undef LOOP3
}

// Shared-memory variant: every level below octave oc lives in shared memory
// (zero-filled per launch; boundary entries stay zero), only r_G(oc) is read
// from and v_G(oc) written to global memory.  Same node bodies and order as
// k3l_coarse, so the results are identical; the steps cost shared-memory
// instead of L2 latency.
template <class T>
static __host__ __device__ size_t coarse3_smem_elems(const int *Ms, int oc, int k) {
  size_t e = 0;
  for (int o = oc; o + 1 < k; o++) {
    const size_t H = Ms[o] / 2 + 1;
    e += 14 * H * H * H;   // r_R, v_R (4), r_M, v_M (2), r_G(2s), v_G(2s) (1 each)
  }
  return e;
}

template <class T>
__global__ void __launch_bounds__(1024) k3l_coarse_smem(const Lev3<T> *lvg, int oc, int k, int *counter, size_t elems) {
  pdl_trigger();
  extern __shared__ __align__(16) unsigned char dsm[];
  T *arena = (T *)dsm;
  __shared__ Lev3<T> lv[32];
  const int tid = threadIdx.x, bs = blockDim.x;
  for (size_t t = tid; t < elems; t += bs) arena[t] = (T)0;
  if (tid == 0) {
    T *p = arena;
    for (int o = oc; o < k; o++) lv[o] = lvg[o];
    for (int o = oc; o + 1 < k; o++) {
      const int H = lv[o].M / 2 + 1;
      const int64_t n3 = (int64_t)H * H * H;
      auto split = [&](S3<T> &a, std::initializer_list<int> subs) {
        for (int q = 0; q < 8; q++) a.s[q] = nullptr;
        for (int q : subs) {
          a.s[q] = p;
          p += n3;
        }
        a.pitch = H;
        a.plane = (int64_t)H * H;
      };
      split(lv[o].rR, {0, 3, 5, 6});
      split(lv[o].vR, {0, 3, 5, 6});
      split(lv[o].rM, {0, 7});
      split(lv[o].vM, {0, 7});
      lv[o + 1].rG = D3<T>{p, H, (int64_t)H * H};
      p += n3;
      lv[o + 1].vG = D3<T>{p, H, (int64_t)H * H};
      p += n3;
    }
  }
  __syncthreads();
  pdl_wait();
  D3<const T> none{nullptr, 0, 0};
  Coef<T> k0{};
  auto cd = [](const D3<T> &a) { return D3<const T>{a.p, a.pitch, a.plane}; };
  auto cs = [](const S3<T> &a) {
    S3<const T> o;
    for (int i = 0; i < 8; i++) o.s[i] = a.s[i];
    o.pitch = a.pitch;
    o.plane = a.plane;
    return o;
  };
#define LOOP3(HH, BODY)                                            \
  {                                                                \
    const int H_ = (HH);                                           \
    const int n_ = H_ * H_ * H_;                                   \
    for (int t = tid; t < n_; t += bs) {                           \
      const int a = t % H_, b = (t / H_) % H_, c = t / (H_ * H_); \
      BODY;                                                        \
    }                                                              \
    __syncthreads();                                               \
  }
  for (int o = oc; o + 1 < k; o++) {
    const Lev3<T> L = lv[o], Lc = lv[o + 1];
    const int H = L.M / 2 + 1;
    LOOP3(H, b3_rest_gr(cd(L.rG), L.rR, L.M, H, a, b, c));
    LOOP3(H, b3_rest_rm(cs(L.rR), L.rM, H, a, b, c));
    LOOP3(Lc.M + 1, b3_rest_mg(cs(L.rM), Lc.rG, Lc.M, a, b, c));
  }
  if (tid == 0) {
    const Lev3<T> L = lv[k - 1];
    L.vG(1, 1, 1) = (-(L.cG * L.rG(1, 1, 1))) * (T)(1.0 / 6.0);   // reading A4
    if (counter) *counter += 1;
  }
  __syncthreads();
  for (int o = k - 2; o >= oc; o--) {
    const Lev3<T> L = lv[o], Lc = lv[o + 1];
    const int H = L.M / 2 + 1;
    LOOP3(H, b3_jac_m1(cd(Lc.vG), cs(L.rM), L.vM, H, L.cMg, a, b, c));
    LOOP3(H, b3_jac_m2(cs(L.rM), L.vM, H, L.cMg, a, b, c));
    LOOP3(H, b3_jac_r1(cs(L.vM), cs(L.rR), L.vR, H, L.cR1, a, b, c));
    LOOP3(H, b3_jac_r2(cs(L.rR), L.vR, H, L.cR2, a, b, c));
    LOOP3(H, (b3_jac_g1<T, 2, false>(cs(L.vR), cd(L.rG), none, none, L.vG, L.M, H, L.cG, k0, a, b, c)));
    LOOP3(H, (b3_jac_g2<T, 2, false>(cd(L.rG), none, none, cd(L.vG), L.vG, L.M, H, L.cG, k0, a, b, c)));
  }
#undef LOOP3
}

// ------------------------------------------------------ cooperative tail
// One cooperative launch for every octave o >= om: the octaves om .. oc-1 run
// grid-wide (each step a grid-stride loop over its blocks, one grid barrier
// between steps; the level arrays are L2 resident), the octaves >= oc run in
// CTA 0's shared memory with __syncthreads between steps (the other CTAs wait
// at the next grid barrier).  Same node bodies, same order as the per-level
// kernels, so the results are identical.  Level descriptors come in the
// kernel parameter block (uniform, constant-cached).
template <class T>
struct Tail3 {
  Lev3<T> lv[20];
  int om, oc, k;
  int *counter;
  unsigned long long *dbg;   // MG_TAIL_DEBUG: globaltimer stamps of CTA 0's phases (else null)
};
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

namespace cc3 {
__host__ __device__ constexpr int ilog2(int v) { return v <= 1 ? 0 : 1 + ilog2(v / 2); }
}
// coarse octaves in shared memory: level arrays at fixed offsets of one arena.
// MC > 0: M(oc) = MC known at compile time (the octave sizes, strides and
// offsets become constants; the node bodies fold their bounds); MC = 0: read
// from the descriptors.  Same steps, same order.
template <class T, int MC>
__device__ __forceinline__ void coarse3_block(const Tail3<T> &P, T *arena) {
  const int tid = threadIdx.x, bs = blockDim.x, oc = P.oc, k = MC ? P.oc + cc3::ilog2(MC) : P.k;
  auto Mof = [&](int o) { return MC ? (MC >> (o - oc)) : P.lv[o].M; };
  // octave o's arrays: 14 consecutive H^3 arrays starting at off(o)
  auto off = [&](int o) {
    size_t e = 0;
    for (int q = oc; q < o; q++) {
      const size_t H = Mof(q) / 2 + 1;
      e += 14 * H * H * H;
    }
    return arena + e;
  };
  auto sub = [&](T *base, int H, std::initializer_list<int> subs, std::initializer_list<int> idx) {
    S3<T> a;
    for (int q = 0; q < 8; q++) a.s[q] = nullptr;
    const int64_t n3 = (int64_t)H * H * H;
    auto it = idx.begin();
    for (int q : subs) a.s[q] = base + (*it++) * n3;
    a.pitch = H;
    a.plane = (int64_t)H * H;
    return a;
  };
  auto cs = [](const S3<T> &a) {
    S3<const T> o;
    for (int i = 0; i < 8; i++) o.s[i] = a.s[i];
    o.pitch = a.pitch;
    o.plane = a.plane;
    return o;
  };
  auto cd = [](const D3<T> &a) { return D3<const T>{a.p, a.pitch, a.plane}; };
  // G(oc) (r and v, dense W^3) staged in shared memory after the arena: r_G(oc)
  // is read from global memory once, with every load of a thread in flight at
  // once, and v_G(oc) written back at the end (not one L2 round trip per
  // stencil access)
  const int W = Mof(oc) + 1, W3 = W * W * W;
  T *g0 = off(k - 1);
  // G(s) of octave o: the staged copy at o = oc, else the G(2s) arrays of octave o-1
  auto gr = [&](int o, int which) -> D3<T> {
    if (o == oc) return D3<T>{g0 + (int64_t)which * W3, W, (int64_t)W * W};
    const int H = Mof(o - 1) / 2 + 1;
    return D3<T>{off(o - 1) + (int64_t)(12 + which) * H * H * H, H, (int64_t)H * H};
  };
  D3<const T> none{nullptr, 0, 0};
  Coef<T> k0{};
  for (size_t t = tid, n = g0 - arena + 2 * (size_t)W3; t < n; t += bs) arena[t] = (T)0;
  {
    const D3<T> &rg = P.lv[oc].rG;
    for (int b0 = tid; b0 < W3; b0 += 8 * bs) {
      T v[8];
#pragma unroll
      for (int i = 0; i < 8; i++) {
        const int t = b0 + i * bs;
        v[i] = t < W3 ? rg.p[(int64_t)(t / (W * W)) * rg.plane + (int64_t)((t / W) % W) * rg.pitch + t % W] : (T)0;
      }
#pragma unroll
      for (int i = 0; i < 8; i++)
        if (b0 + i * bs < W3) g0[b0 + i * bs] = v[i];
    }
  }
  __syncthreads();
#define LOOPB(HH, BODY)                                            \
  {                                                                \
    const int H_ = (HH);                                           \
    const int n_ = H_ * H_ * H_;                                   \
    for (int t = tid; t < n_; t += bs) {                           \
      const int a = t % H_, b = (t / H_) % H_, c = t / (H_ * H_); \
      BODY;                                                        \
    }                                                              \
    __syncthreads();                                               \
    if (P.dbg && tid == 0) P.dbg[1 + (nph++)] = gtimer();          \
  }
  int nph = 0;
  if (P.dbg && tid == 0) P.dbg[0] = gtimer();
#pragma unroll
  for (int o = oc; o + 1 < k; o++) {
    const int M = Mof(o), H = M / 2 + 1;
    T *base = off(o);
    const S3<T> rR = sub(base, H, {0, 3, 5, 6}, {0, 1, 2, 3}), rM = sub(base, H, {0, 7}, {8, 9});
    const D3<T> rG = gr(o, 0), rG2 = gr(o + 1, 0);
    LOOPB(H, b3_rest_gr(cd(rG), rR, M, H, a, b, c));
    LOOPB(H, b3_rest_rm(cs(rR), rM, H, a, b, c));
    LOOPB(M / 2 + 1, b3_rest_mg(cs(rM), rG2, M / 2, a, b, c));
  }
  if (tid == 0) {
    const D3<T> rG = gr(k - 1, 0), vG = gr(k - 1, 1);
    vG(1, 1, 1) = (-(P.lv[k - 1].cG * rG(1, 1, 1))) * (T)(1.0 / 6.0);   // reading A4
    if (P.counter) *P.counter += 1;
  }
  __syncthreads();
#pragma unroll
  for (int o = k - 2; o >= oc; o--) {
    const Lev3<T> &L = P.lv[o];
    const int M = Mof(o), H = M / 2 + 1;
    T *base = off(o);
    const S3<T> rR = sub(base, H, {0, 3, 5, 6}, {0, 1, 2, 3}), vR = sub(base, H, {0, 3, 5, 6}, {4, 5, 6, 7});
    const S3<T> rM = sub(base, H, {0, 7}, {8, 9}), vM = sub(base, H, {0, 7}, {10, 11});
    const D3<T> rG = gr(o, 0), vG = gr(o, 1), vG2 = gr(o + 1, 1);
    LOOPB(H, b3_jac_m1(cd(vG2), cs(rM), vM, H, L.cMg, a, b, c));
    LOOPB(H, b3_jac_m2(cs(rM), vM, H, L.cMg, a, b, c));
    LOOPB(H, b3_jac_r1(cs(vM), cs(rR), vR, H, L.cR1, a, b, c));
    LOOPB(H, b3_jac_r2(cs(rR), vR, H, L.cR2, a, b, c));
    LOOPB(H, (b3_jac_g1<T, 2, false>(cs(vR), cd(rG), none, none, vG, M, H, L.cG, k0, a, b, c)));
    LOOPB(H, (b3_jac_g2<T, 2, false>(cd(rG), none, none, cd(vG), vG, M, H, L.cG, k0, a, b, c)));
  }
#undef LOOPB
  {   // v_G(oc) to global memory (interior nodes; the boundary is never written)
    const D3<T> &vg = P.lv[oc].vG;
    const T *src = g0 + W3;
    for (int t = tid; t < W3; t += bs) {
      const int x = t % W, y = (t / W) % W, z = t / (W * W);
      if (x >= 1 && y >= 1 && z >= 1 && x <= W - 2 && y <= W - 2 && z <= W - 2)
        vg.p[(int64_t)z * vg.plane + (int64_t)y * vg.pitch + x] = src[t];
    }
  }
}

// The tail: the grid-wide octaves om .. oc-1 around CTA 0's coarse octaves
// (MG = 0: sizes from the descriptors).
template <class T, int MG>
__device__ __forceinline__ void tail_run(const Tail3<T> &P, unsigned char *dsm) {
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  const int gt = blockIdx.x * blockDim.x + threadIdx.x, gs = gridDim.x * blockDim.x;
  const int om = P.om, oc = MG ? P.om + cc3::ilog2(MG) - cc3::ilog2(16) : P.oc;
  auto Mof = [&](int o) { return MG ? (MG >> (o - om)) : P.lv[o].M; };
  auto cd = [](const D3<T> &a) { return D3<const T>{a.p, a.pitch, a.plane}; };
  auto cs = [](const S3<T> &a) {
    S3<const T> o;
    for (int i = 0; i < 8; i++) o.s[i] = a.s[i];
    o.pitch = a.pitch;
    o.plane = a.plane;
    return o;
  };
  int ngp = 0;
  const bool gdbg = P.dbg && blockIdx.x == 0 && threadIdx.x == 0;
  if (gdbg) P.dbg[128] = gtimer();
#define LOOPG(HH, BODY)                                            \
  {                                                                \
    const int H_ = (HH);                                           \
    const int n_ = H_ * H_ * H_;                                   \
    for (int t = gt; t < n_; t += gs) {                            \
      const int a = t % H_, b = (t / H_) % H_, c = t / (H_ * H_); \
      BODY;                                                        \
    }                                                              \
    grid.sync();                                                   \
    if (gdbg) P.dbg[129 + (ngp++)] = gtimer();                     \
  }
#pragma unroll
  for (int o = om; o < oc; o++) {
    const Lev3<T> &L = P.lv[o], &Lc = P.lv[o + 1];
    const int M = Mof(o), H = M / 2 + 1, Mc = M / 2;
    LOOPG(H, b3_rest_gr(cd(L.rG), L.rR, M, H, a, b, c));
    LOOPG(H, b3_rest_rm(cs(L.rR), L.rM, H, a, b, c));
    LOOPG(Mc + 1, b3_rest_mg(cs(L.rM), Lc.rG, Mc, a, b, c));
  }
  if (blockIdx.x == 0) {
    switch (P.lv[P.oc].M) {   // the usual M(oc) <= 16 at compile time (the tail's coarse threshold)
      case 16: coarse3_block<T, 16>(P, (T *)dsm); break;
      case 8: coarse3_block<T, 8>(P, (T *)dsm); break;
      case 4: coarse3_block<T, 4>(P, (T *)dsm); break;
      default: coarse3_block<T, 0>(P, (T *)dsm); break;
    }
  }
  grid.sync();
  if (gdbg) P.dbg[129 + (ngp++)] = gtimer();
  D3<const T> none{nullptr, 0, 0};
  Coef<T> k0{};
#pragma unroll
  for (int o = oc - 1; o >= om; o--) {
    const Lev3<T> &L = P.lv[o], &Lc = P.lv[o + 1];
    const int M = Mof(o), H = M / 2 + 1;
    LOOPG(H, b3_jac_m1(cd(Lc.vG), cs(L.rM), L.vM, H, L.cMg, a, b, c));
    LOOPG(H, b3_jac_m2(cs(L.rM), L.vM, H, L.cMg, a, b, c));
    LOOPG(H, b3_jac_r1(cs(L.vM), cs(L.rR), L.vR, H, L.cR1, a, b, c));
    LOOPG(H, b3_jac_r2(cs(L.rR), L.vR, H, L.cR2, a, b, c));
    LOOPG(H, (b3_jac_g1<T, 2, false>(cs(L.vR), cd(L.rG), none, none, L.vG, M, H, L.cG, k0, a, b, c)));
    LOOPG(H, (b3_jac_g2<T, 2, false>(cd(L.rG), none, none, cd(L.vG), L.vG, M, H, L.cG, k0, a, b, c)));
  }
#undef LOOPG
}

template <class T>
__global__ void __launch_bounds__(512, 1) k3l_tail(const __grid_constant__ Tail3<T> P) {
  extern __shared__ __align__(16) unsigned char dsm[];
  tail_run<T, 0>(P, dsm);   // (compile-time grid sizes measured no faster: the steps are barrier-bound)
}

// ================================================================ launchers
// grid.z covers the half-index planes [c0, c1) (c1 = -1: all H).
// The level kernels start with pdl_trigger(); pdl_wait(), so they may be launched programmatically, each
// one's launch overlapping its predecessor's drain (MG_K3L_PDL=1).  Measured neutral at 513^3 (2.1265 vs
// 2.1285 ms per cycle, 3 x 100 interleaved): off by default.
static bool k3l_pdl() {
  static const bool on = env_flag("MG_K3L_PDL");
  return on;
}
static inline dim3 grid3(int H, int nz) { return dim3((H + 31) / 32, (H + 7) / 8, nz); }
static const dim3 kBlk(32, 8);
static inline int zcount(int H, int c0, int &c1) {
  if (c1 < 0 || c1 > H) c1 = H;
  return c1 - c0;
}

template <class T>
static D3<const T> cd3(const D3<T> &a) {
  return D3<const T>{a.p, a.pitch, a.plane};
}
template <class T>
static S3<const T> cs3(const S3<T> &a) {
  S3<const T> o;
  for (int i = 0; i < 8; i++) o.s[i] = a.s[i];
  o.pitch = a.pitch;
  o.plane = a.plane;
  return o;
}

template <class T>
void lv3_rest_gr(const D3<T> &r, const S3<T> &rr, int M, cudaStream_t st, int c0, int c1) {
  int H = M / 2 + 1, nz = zcount(H, c0, c1);
  if (nz > 0) note_launch(launch_pdl_if(k3l_pdl(), k3l_rest_gr<T>, grid3(H, nz), kBlk, 0, st, cd3(r), rr, M, H, c0));
}
template <class T>
void lv3_rest_rm(const S3<T> &rr, const S3<T> &rm, int M, cudaStream_t st, int c0, int c1) {
  int H = M / 2 + 1, nz = zcount(H, c0, c1);
  if (nz > 0) note_launch(launch_pdl_if(k3l_pdl(), k3l_rest_rm<T>, grid3(H, nz), kBlk, 0, st, cs3(rr), rm, H, c0));
}
template <class T>
void lv3_rest_mg(const S3<T> &rm, const D3<T> &g2, int Mc, cudaStream_t st, int c0, int c1) {
  int nz = zcount(Mc + 1, c0, c1);
  if (nz > 0) note_launch(launch_pdl_if(k3l_pdl(), k3l_rest_mg<T>, grid3(Mc + 1, nz), kBlk, 0, st, cs3(rm), g2, Mc, c0));
}
template <class T>
void lv3_jac_m(const D3<T> &vc, const S3<T> &r, const S3<T> &v, int M, T c, cudaStream_t st, int c0, int c1,
               int phase) {
  int H = M / 2 + 1, nz = zcount(H, c0, c1);
  if (nz <= 0) return;
  if (phase != 2) note_launch(launch_pdl_if(k3l_pdl(), k3l_jac_m1<T>, grid3(H, nz), kBlk, 0, st, cd3(vc), cs3(r), v, H, c, c0));
  if (phase != 1) note_launch(launch_pdl_if(k3l_pdl(), k3l_jac_m2<T>, grid3(H, nz), kBlk, 0, st, cs3(r), v, H, c, c0));
}
template <class T>
void lv3_jac_r(const S3<T> &vm, const S3<T> &r, const S3<T> &v, int M, T c1, T c2, cudaStream_t st, int cz0, int cz1,
               int phase) {
  int H = M / 2 + 1, nz = zcount(H, cz0, cz1);
  if (nz <= 0) return;
  if (phase != 2) note_launch(launch_pdl_if(k3l_pdl(), k3l_jac_r1<T>, grid3(H, nz), kBlk, 0, st, cs3(vm), cs3(r), v, H, c1, cz0));
  if (phase != 1) note_launch(launch_pdl_if(k3l_pdl(), k3l_jac_r2<T>, grid3(H, nz), kBlk, 0, st, cs3(r), v, H, c2, cz0));
}
template <class T>
void lv3_jac_g(const S3<T> &vr, const D3<T> &r, const D3<T> &v, int M, T c, cudaStream_t st, int c0, int c1,
               int phase) {
  int H = M / 2 + 1, nz = zcount(H, c0, c1);
  if (nz <= 0) return;
  Coef<T> k{};
  D3<const T> none{nullptr, 0, 0};
  if (phase != 2)
    note_launch(launch_pdl_if(k3l_pdl(), k3l_jac_g1<T, 2, false>, grid3(H, nz), kBlk, 0, st, cs3(vr), cd3(r), none, none, v, M, H, c, k, c0));
  if (phase != 1)
    note_launch(launch_pdl_if(k3l_pdl(), k3l_jac_g2<T, 2, false>, grid3(H, nz), kBlk, 0, st, cd3(r), none, none, cd3(v), v, M, H, c, k, c0));
}
template <class T>
void lv3_asc_fine(const S3<T> &vr, const D3<T> &u_old, const D3<const T> &f, const D3<T> &g, const D3<T> &u_new, int M,
                  int order, T c, const Coef<T> &k, cudaStream_t st) {
  int H = M / 2 + 1;
  D3<const T> none{nullptr, 0, 0};
  if (order == 2) {
    k3l_jac_g1<T, 2, true><<<grid3(H, H), kBlk, 0, st>>>(cs3(vr), none, cd3(u_old), f, g, M, H, c, k, 0);
    k3l_jac_g2<T, 2, true><<<grid3(H, H), kBlk, 0, st>>>(none, cd3(u_old), f, cd3(g), u_new, M, H, c, k, 0);
  } else {
    k3l_jac_g1<T, 4, true><<<grid3(H, H), kBlk, 0, st>>>(cs3(vr), none, cd3(u_old), f, g, M, H, c, k, 0);
    k3l_jac_g2<T, 4, true><<<grid3(H, H), kBlk, 0, st>>>(none, cd3(u_old), f, cd3(g), u_new, M, H, c, k, 0);
  }
}

template <class T>
void lv3_coarse(const Lev3<T> *d_lev, int oc, int k, int *counter, cudaStream_t st) {
  static const bool global = env_flag("MG_COARSE_GLOBAL");
  if (!global && oc >= 1 && k <= 32) {
    int Ms[32];
    for (int o = 0; o < k; o++) Ms[o] = 1 << (k - o);   // M of octave o for n = 2^k + 1
    const size_t elems = coarse3_smem_elems<T>(Ms, oc, k), bytes = elems * sizeof(T);
    if (bytes <= 200 * 1024) {
      cudaFuncSetAttribute(k3l_coarse_smem<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
      launch_pdl(k3l_coarse_smem<T>, dim3(1), dim3(1024), bytes, st, d_lev, oc, k, counter, elems);
      return;
    }
  }
  launch_pdl(k3l_coarse<T>, dim3(1), dim3(1024), 0, st, d_lev, oc, k, counter);
}

#define INSTL(T)                                                                                                   \
  template void lv3_coarse<T>(const Lev3<T> *, int, int, int *, cudaStream_t);                                     \
  template void lv3_rest_gr<T>(const D3<T> &, const S3<T> &, int, cudaStream_t, int, int);                         \
  template void lv3_rest_rm<T>(const S3<T> &, const S3<T> &, int, cudaStream_t, int, int);                         \
  template void lv3_rest_mg<T>(const S3<T> &, const D3<T> &, int, cudaStream_t, int, int);                         \
  template void lv3_jac_m<T>(const D3<T> &, const S3<T> &, const S3<T> &, int, T, cudaStream_t, int, int, int);    \
  template void lv3_jac_r<T>(const S3<T> &, const S3<T> &, const S3<T> &, int, T, T, cudaStream_t, int, int, int); \
  template void lv3_jac_g<T>(const S3<T> &, const D3<T> &, const D3<T> &, int, T, cudaStream_t, int, int, int);    \
  template void lv3_asc_fine<T>(const S3<T> &, const D3<T> &, const D3<const T> &, const D3<T> &, const D3<T> &,   \
                                int, int, T, const Coef<T> &, cudaStream_t);

INSTL(float)
INSTL(double)


// Octaves om .. k-1 in one cooperative launch (om <= oc; oc >= 1).  Returns
// false (nothing launched) when the tail does not fit.
template <class T>
bool lv3_tail(const Lev3<T> *h_lev, int om, int oc, int k, int *counter, cudaStream_t st) {
  if (k > 20 || om < 1 || om > oc || oc >= k) return false;
  Tail3<T> P;
  for (int o = 0; o < k; o++) P.lv[o] = h_lev[o];
  P.om = om;
  P.oc = oc;
  P.k = k;
  P.counter = counter;
  static unsigned long long *dbg = nullptr;
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  cudaStreamIsCapturing(st, &cap);
  const bool debug = env_flag("MG_TAIL_DEBUG") && cap == cudaStreamCaptureStatusNone;
  if (debug && !dbg) cudaMalloc(&dbg, 256 * sizeof(unsigned long long));
  if (debug) cudaMemsetAsync(dbg, 0, 256 * sizeof(unsigned long long), st);
  P.dbg = debug ? dbg : nullptr;
  size_t elems = 0;
  for (int o = oc; o + 1 < k; o++) {
    const size_t H = h_lev[o].M / 2 + 1;
    elems += 14 * H * H * H;
  }
  {
    const size_t W = h_lev[oc].M + 1;   // the staged r_G(oc), v_G(oc)
    elems += 2 * W * W * W;
  }
  const size_t bytes = elems * sizeof(T);
  if (bytes > 200 * 1024) return false;
  if (cudaFuncSetAttribute(k3l_tail<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes) != cudaSuccess)
    return false;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  // a cooperative launch that cannot be co-resident (MPS / green-context SM
  // limits) would be rejected -- inside a stream capture that invalidates the
  // capture, so decide on the host first and let the caller run per-level kernels
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k3l_tail<T>, 512, bytes) != cudaSuccess ||
      per_sm < 1) {
    cudaGetLastError();
    return false;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(sms);
  cfg.blockDim = dim3(512);
  cfg.dynamicSmemBytes = bytes;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeCooperative;
  at[0].val.cooperative = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  const bool ok = cudaLaunchKernelEx(&cfg, k3l_tail<T>, P) == cudaSuccess;
  if (debug && ok) {
    unsigned long long h[256] = {};
    cudaMemcpyAsync(h, dbg, sizeof h, cudaMemcpyDeviceToHost, st);
    cudaStreamSynchronize(st);
    fprintf(stderr, "[tail] CTA0 coarse phases (us):");
    for (int i = 1; i < 64 && h[i] > h[0] && h[i] - h[0] < 1000000000ull; i++)
      fprintf(stderr, " %.2f", (h[i] - h[i - 1]) * 1e-3);
    fprintf(stderr, "\n[tail] CTA0 grid phases (us):");
    for (int i = 129; i < 256 && h[i] > h[128] && h[i] - h[128] < 1000000000ull; i++)
      fprintf(stderr, " %.2f", (h[i] - h[i - 1]) * 1e-3);
    fprintf(stderr, "\n");
  }
  return ok;
}
template bool lv3_tail<float>(const Lev3<float> *, int, int, int, int *, cudaStream_t);
template bool lv3_tail<double>(const Lev3<double> *, int, int, int, int *, cudaStream_t);

}  // namespace mg
