// k2d.cu -- 2D kernels of the diagonal-multigrid V-cycle (sm_100a).
//
// Every formula is evaluated in the canonical order of DESIGN.md (terms left
// to right as printed in the paper, constants rounded once from double) and
// the file is compiled with --fmad=false, so the results are bit-identical to
// any other evaluation in the same order.
//
// Level kernels in this file work on lattice coordinates of one octave
// s = 2^o (x = i/s, y = j/s), M = (n-1)/s.
#include "kernels.h"

namespace mg {

constexpr int NT = 256;

static inline unsigned blocks_for(int64_t n, int nt = NT) { return (unsigned)((n + nt - 1) / nt); }

// ------------------------------------------------------------ residual
// r = f - L u at an interior node (Evpois).
//  order 2: 5-point Laplacian, centre first then (i-1,j),(i,j-1),(i+1,j),(i,j+1)
//           (the neighbour order of Erest2r); 7 flops.
//  order 4: Efos2 with f~ precomputed: bracket
//           -20u + 4(u_{i,j-1}+u_{i,j+1}+u_{i-1,j}+u_{i+1,j}) + u_{i+1,j+1}
//           + u_{i-1,j+1} + u_{i-1,j-1} + u_{i+1,j-1}, times 1/(6h^2).
template <class T, int ORDER>
__device__ __forceinline__ T res2(const D2<const T> &u, const D2<const T> &f, int x, int y, const Coef<T> &k) {
  if (ORDER == 2) {
    T lap = -((T)4 * u(x, y));
    lap = lap + u(x - 1, y);
    lap = lap + u(x, y - 1);
    lap = lap + u(x + 1, y);
    lap = lap + u(x, y + 1);
    lap = lap * k.invh2;
    return f(x, y) - lap;
  } else {
    T ax = u(x, y - 1);
    ax = ax + u(x, y + 1);
    ax = ax + u(x - 1, y);
    ax = ax + u(x + 1, y);
    T b = -((T)20 * u(x, y));
    b = b + (T)4 * ax;
    b = b + u(x + 1, y + 1);
    b = b + u(x - 1, y + 1);
    b = b + u(x - 1, y - 1);
    b = b + u(x + 1, y - 1);
    return f(x, y) - b * k.c6;
  }
}

// r at any lattice node of the finest grid: 0 on the boundary (reading A1).
template <class T, int ORDER>
__device__ __forceinline__ T res2z(const D2<const T> &u, const D2<const T> &f, int x, int y, int M, const Coef<T> &k) {
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

// ------------------------------------------------- descent, finest level
// Fused a1+a2: residual on A(1) recomputed on the fly, Erest2r onto D(1).
// Thread (a, b) owns the 2x2 block of fine nodes (2a..2a+1, 2b..2b+1): it
// writes E(a,b) = node (2a,2b) and O(a,b) = node (2a+1,2b+1) and reports
// max|r| over the block's interior nodes.
template <class T, int ORDER>
__global__ void __launch_bounds__(NT) k2_desc_fine_ref(D2<const T> u, D2<const T> f, S2<T> d, int M, Coef<T> k,
                                                       NormSink ns) {
  int H = M / 2 + 1;
  int64_t t = (int64_t)blockIdx.x * NT + threadIdx.x;
  double mx = 0.0;
  if (t < (int64_t)H * H) {
    int a = (int)(t % H), b = (int)(t / H);
    int x = 2 * a, y = 2 * b;
    T rc = res2z<T, ORDER>(u, f, x, y, M, k);
    T rE = res2z<T, ORDER>(u, f, x + 1, y, M, k);
    T rN = res2z<T, ORDER>(u, f, x, y + 1, M, k);
    if (x >= 1 && y >= 1 && x <= M - 1 && y <= M - 1) {
      T rW = res2z<T, ORDER>(u, f, x - 1, y, M, k);
      T rS = res2z<T, ORDER>(u, f, x, y - 1, M, k);
      d.e[(int64_t)b * d.pitch + a] = erest2r(rc, rW, rS, rE, rN);
    }
    mx = nmax(mx, absd(rc));
    mx = nmax(mx, absd(rE));
    mx = nmax(mx, absd(rN));
    if (x + 1 <= M - 1 && y + 1 <= M - 1) {
      T ro = res2z<T, ORDER>(u, f, x + 1, y + 1, M, k);
      T oW = rN;                                            // (x, y+1)
      T oS = rE;                                            // (x+1, y)
      T oE = res2z<T, ORDER>(u, f, x + 2, y + 1, M, k);
      T oN = res2z<T, ORDER>(u, f, x + 1, y + 2, M, k);
      d.o[(int64_t)b * d.pitch + a] = erest2r(ro, oW, oS, oE, oN);
      mx = nmax(mx, absd(ro));
    }
  }
  block_norm_push<NT>(ns, mx);
}

// ------------------------------------------------- descent, level kernels
// a2 for s > 1: Erest2r from the dense A(s) residual onto D(s).
template <class T>
__global__ void __launch_bounds__(NT) k2_rest_ad_ref(D2<const T> r, S2<T> d, int M) {
  int H = M / 2 + 1;
  int64_t t = (int64_t)blockIdx.x * NT + threadIdx.x;
  if (t >= (int64_t)H * H) return;
  int a = (int)(t % H), b = (int)(t / H);
  int x = 2 * a, y = 2 * b;
  if (x >= 2 && y >= 2 && x <= M - 2 && y <= M - 2)
    d.e[(int64_t)b * d.pitch + a] = erest2r(r(x, y), r(x - 1, y), r(x, y - 1), r(x + 1, y), r(x, y + 1));
  x += 1;
  y += 1;
  if (x <= M - 1 && y <= M - 1)
    d.o[(int64_t)b * d.pitch + a] = erest2r(r(x, y), r(x - 1, y), r(x, y - 1), r(x + 1, y), r(x, y + 1));
}

// a3: Erest2b from D(s) onto A(2s); coarse node (X,Y) is lattice node (2X,2Y).
template <class T>
__global__ void __launch_bounds__(NT) k2_rest_da_ref(S2<const T> d, D2<T> r, int Mc) {
  int64_t t = (int64_t)blockIdx.x * NT + threadIdx.x;
  int W = Mc - 1;
  if (t >= (int64_t)W * W) return;
  int X = (int)(t % W) + 1, Y = (int)(t / W) + 1;
  int x = 2 * X, y = 2 * Y;
  r(X, Y) = erest2b(d.get(x, y), d.get(x - 1, y - 1), d.get(x + 1, y - 1), d.get(x + 1, y + 1), d.get(x - 1, y + 1));
}

// a4: coarsest level, one interior node (reading A4): v = (1/4)(-p H^2 r).
template <class T>
__global__ void k2_coarsest(D2<const T> r, D2<T> v, T c, int *counter) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    v(1, 1) = (-(c * r(1, 1))) * (T)0.25;
    if (counter) *counter += 1;   // this cycle's norm slot is complete
  }
}

// ------------------------------------------------ ascent, diagonal level
// a5: colour 1 on O (nodes of D(s) not on A(2s)): Eajacr from
// the coarse A(2s) values at the 4 diagonal neighbours.
template <class T>
__global__ void __launch_bounds__(NT) k2_jac_d1_ref(D2<const T> vc, S2<const T> r, S2<T> v, int M, T c) {
  int W = M / 2;
  int64_t t = (int64_t)blockIdx.x * NT + threadIdx.x;
  if (t >= (int64_t)W * W) return;
  int a = (int)(t % W), b = (int)(t / W);
  int x = 2 * a + 1, y = 2 * b + 1;
  v.o[(int64_t)b * v.pitch + a] = jac4(c, r.o[(int64_t)b * r.pitch + a], vc((x - 1) / 2, (y - 1) / 2),
                                       vc((x + 1) / 2, (y - 1) / 2), vc((x + 1) / 2, (y + 1) / 2),
                                       vc((x - 1) / 2, (y + 1) / 2));
}

// a6: colour 2 on E (= A(2s) positions): Eajacb from the new O
// values; uses the D(s) residual at that node (reading A10).
template <class T>
__global__ void __launch_bounds__(NT) k2_jac_d2_ref(S2<const T> r, S2<T> v, int M, T c) {
  int W = M / 2 - 1;
  int64_t t = (int64_t)blockIdx.x * NT + threadIdx.x;
  if (t >= (int64_t)W * W) return;
  int a = (int)(t % W) + 1, b = (int)(t / W) + 1;
  int x = 2 * a, y = 2 * b;
  v.e[(int64_t)b * v.pitch + a] = jac4(c, r.e[(int64_t)b * r.pitch + a], v.get(x - 1, y - 1), v.get(x + 1, y - 1),
                                       v.get(x + 1, y + 1), v.get(x - 1, y + 1));
}

// ---------------------------------------------------- ascent, axis level
// a7 (s > 1): colour 1 on the green-only nodes (x+y odd) from D(s), colour 2
// on the D(s) nodes from the new green values ("similarly for a green grid",
// P:228-230; reading A5), c = p (sh)^2.
template <class T>
__global__ void __launch_bounds__(NT) k2_jac_a1_ref(S2<const T> vd, D2<const T> r, D2<T> v, int M, T c) {
  int W = M - 1;
  int64_t t = (int64_t)blockIdx.x * NT + threadIdx.x;
  if (t >= (int64_t)W * W) return;
  int x = (int)(t % W) + 1, y = (int)(t / W) + 1;
  if (((x + y) & 1) == 0) return;
  v(x, y) = jac4(c, r(x, y), vd.get(x - 1, y), vd.get(x, y - 1), vd.get(x + 1, y), vd.get(x, y + 1));
}

template <class T>
__global__ void __launch_bounds__(NT) k2_jac_a2_ref(D2<const T> r, D2<T> v, int M, T c) {
  int W = M - 1;
  int64_t t = (int64_t)blockIdx.x * NT + threadIdx.x;
  if (t >= (int64_t)W * W) return;
  int x = (int)(t % W) + 1, y = (int)(t / W) + 1;
  if (((x + y) & 1) == 1) return;
  v(x, y) = jac4(c, r(x, y), v(x - 1, y), v(x, y - 1), v(x + 1, y), v(x, y + 1));
}

// ---------------------------------------------------- ascent, finest level
// a8: a7 at s = 1 with r recomputed from u, f; v kept in a dense scratch.
template <class T, int ORDER>
__global__ void __launch_bounds__(NT) k2_asc_fine1_ref(S2<const T> vd, D2<const T> u, D2<const T> f, D2<T> v, int M,
                                                       T c, Coef<T> k) {
  int W = M - 1;
  int64_t t = (int64_t)blockIdx.x * NT + threadIdx.x;
  if (t >= (int64_t)W * W) return;
  int x = (int)(t % W) + 1, y = (int)(t / W) + 1;
  if (((x + y) & 1) == 0) return;
  T r = res2<T, ORDER>(u, f, x, y, k);
  v(x, y) = jac4(c, r, vd.get(x - 1, y), vd.get(x, y - 1), vd.get(x + 1, y), vd.get(x, y + 1));
}

template <class T, int ORDER>
__global__ void __launch_bounds__(NT) k2_asc_fine2_ref(D2<const T> u, D2<const T> f, D2<T> v, int M, T c, Coef<T> k) {
  int W = M - 1;
  int64_t t = (int64_t)blockIdx.x * NT + threadIdx.x;
  if (t >= (int64_t)W * W) return;
  int x = (int)(t % W) + 1, y = (int)(t / W) + 1;
  if (((x + y) & 1) == 1) return;
  T r = res2<T, ORDER>(u, f, x, y, k);
  v(x, y) = jac4(c, r, v(x - 1, y), v(x, y - 1), v(x + 1, y), v(x, y + 1));
}

// u <- u + v at the interior.
template <class T>
__global__ void __launch_bounds__(NT) k2_update_ref(D2<T> u, D2<const T> v, int M) {
  int W = M - 1;
  int64_t t = (int64_t)blockIdx.x * NT + threadIdx.x;
  if (t >= (int64_t)W * W) return;
  int x = (int)(t % W) + 1, y = (int)(t / W) + 1;
  u(x, y) = u(x, y) + v(x, y);
}

// --------------------------------------------------- standalone residual
template <class T, int ORDER>
__global__ void __launch_bounds__(NT) k2_residual(D2<const T> u, D2<const T> f, D2<T> r, int M, Coef<T> k) {
  int64_t t = (int64_t)blockIdx.x * NT + threadIdx.x;
  int Wd = M + 1;
  if (t >= (int64_t)Wd * Wd) return;
  int x = (int)(t % Wd), y = (int)(t / Wd);
  r(x, y) = res2z<T, ORDER>(u, f, x, y, M, k);
}

// f~ of Efos2: (1/12)(8f + f_{i+1,j} + f_{i,j+1} + f_{i-1,j} + f_{i,j-1}).
template <class T>
__global__ void __launch_bounds__(NT) k2_ftilde(D2<const T> f, D2<T> ft, int M) {
  int W = M - 1;
  int64_t t = (int64_t)blockIdx.x * NT + threadIdx.x;
  if (t >= (int64_t)W * W) return;
  int x = (int)(t % W) + 1, y = (int)(t / W) + 1;
  T s = (T)8 * f(x, y);
  s = s + f(x + 1, y);
  s = s + f(x, y + 1);
  s = s + f(x - 1, y);
  s = s + f(x, y - 1);
  ft(x, y) = s * (T)(1.0 / 12.0);
}

// Norms of a finest-grid array over interior nodes: max |x| and sum x^2.
template <class T>
__global__ void __launch_bounds__(NT) k2_norm(D2<const T> a, int M, unsigned long long *mx_out, double *ss_out) {
  int W = M - 1;
  double mx = 0.0, ss = 0.0;
  for (int64_t t = (int64_t)blockIdx.x * NT + threadIdx.x; t < (int64_t)W * W; t += (int64_t)gridDim.x * NT) {
    int x = (int)(t % W) + 1, y = (int)(t / W) + 1;
    double v = (double)a(x, y);
    mx = nmax(mx, fabs(v));
    ss += v * v;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    ss += __shfl_xor_sync(0xffffffffu, ss, o);
    mx = nmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  }
  __shared__ double rs[NT / 32], rm[NT / 32];
  int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (lane == 0) {
    rs[wid] = ss;
    rm[wid] = mx;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double s2 = 0.0, m2 = 0.0;
    for (int i = 0; i < NT / 32; i++) {
      s2 += rs[i];
      m2 = nmax(m2, rm[i]);
    }
    atomicAdd(ss_out, s2);
    atomicMax(mx_out, (unsigned long long)__double_as_longlong(m2));
  }
}

// ================================================================ launchers

template <class T>
static D2<const T> cd(const D2<T> &a) {
  return D2<const T>{a.p, a.pitch};
}
template <class T>
static S2<const T> cs(const S2<T> &a) {
  return S2<const T>{a.e, a.o, a.pitch};
}

template <class T>
void launch2_desc_fine(const D2<const T> &u, const D2<const T> &f, const S2<T> &d, int M, int order, const Coef<T> &k,
                       const NormSink &ns, cudaStream_t st) {
  int64_t H = M / 2 + 1;
  if (order == 2)
    k2_desc_fine_ref<T, 2><<<blocks_for(H * H), NT, 0, st>>>(u, f, d, M, k, ns);
  else
    k2_desc_fine_ref<T, 4><<<blocks_for(H * H), NT, 0, st>>>(u, f, d, M, k, ns);
}

template <class T>
void launch2_rest_ad(const D2<T> &r, const S2<T> &d, int M, cudaStream_t st) {
  int64_t H = M / 2 + 1;
  k2_rest_ad_ref<T><<<blocks_for(H * H), NT, 0, st>>>(cd(r), d, M);
}

template <class T>
void launch2_rest_da(const S2<T> &d, const D2<T> &r, int Mc, cudaStream_t st) {
  int64_t W = Mc - 1;
  k2_rest_da_ref<T><<<blocks_for(W * W), NT, 0, st>>>(cs(d), r, Mc);
}

template <class T>
void launch2_coarsest(const D2<T> &r, const D2<T> &v, T c, int *counter, cudaStream_t st) {
  k2_coarsest<T><<<1, 32, 0, st>>>(cd(r), v, c, counter);
}

template <class T>
void launch2_jac_d(const D2<T> &vc, const S2<T> &r, const S2<T> &v, int M, T c, cudaStream_t st) {
  int64_t W = M / 2;
  k2_jac_d1_ref<T><<<blocks_for(W * W), NT, 0, st>>>(cd(vc), cs(r), v, M, c);
  if (M / 2 - 1 > 0) k2_jac_d2_ref<T><<<blocks_for((W - 1) * (W - 1)), NT, 0, st>>>(cs(r), v, M, c);
}

template <class T>
void launch2_jac_a(const S2<T> &vd, const D2<T> &r, const D2<T> &v, int M, T c, cudaStream_t st) {
  int64_t W = M - 1;
  k2_jac_a1_ref<T><<<blocks_for(W * W), NT, 0, st>>>(cs(vd), cd(r), v, M, c);
  k2_jac_a2_ref<T><<<blocks_for(W * W), NT, 0, st>>>(cd(r), v, M, c);
}

template <class T>
void launch2_asc_fine(const S2<T> &vd, const D2<T> &u, const D2<const T> &f, const D2<T> &scratch, int M, int order,
                      T c, const Coef<T> &k, cudaStream_t st) {
  int64_t W = M - 1;
  if (order == 2) {
    k2_asc_fine1_ref<T, 2><<<blocks_for(W * W), NT, 0, st>>>(cs(vd), cd(u), f, scratch, M, c, k);
    k2_asc_fine2_ref<T, 2><<<blocks_for(W * W), NT, 0, st>>>(cd(u), f, scratch, M, c, k);
  } else {
    k2_asc_fine1_ref<T, 4><<<blocks_for(W * W), NT, 0, st>>>(cs(vd), cd(u), f, scratch, M, c, k);
    k2_asc_fine2_ref<T, 4><<<blocks_for(W * W), NT, 0, st>>>(cd(u), f, scratch, M, c, k);
  }
  k2_update_ref<T><<<blocks_for(W * W), NT, 0, st>>>(u, cd(scratch), M);
}

template <class T>
void launch2_residual(const D2<const T> &u, const D2<const T> &f, const D2<T> &r, int M, int order, const Coef<T> &k,
                      cudaStream_t st) {
  int64_t W = M + 1;
  if (order == 2)
    k2_residual<T, 2><<<blocks_for(W * W), NT, 0, st>>>(u, f, r, M, k);
  else
    k2_residual<T, 4><<<blocks_for(W * W), NT, 0, st>>>(u, f, r, M, k);
}

template <class T>
void launch2_ftilde(const D2<const T> &f, const D2<T> &ft, int M, cudaStream_t st) {
  int64_t W = M - 1;
  k2_ftilde<T><<<blocks_for(W * W), NT, 0, st>>>(f, ft, M);
}

template <class T>
void launch2_norm(const D2<const T> &a, int M, unsigned long long *mx, double *ss, cudaStream_t st) {
  k2_norm<T><<<148 * 4, NT, 0, st>>>(a, M, mx, ss);
}

#define INST(T)                                                                                                     \
  template void launch2_desc_fine<T>(const D2<const T> &, const D2<const T> &, const S2<T> &, int, int,            \
                                     const Coef<T> &, const NormSink &, cudaStream_t);                             \
  template void launch2_rest_ad<T>(const D2<T> &, const S2<T> &, int, cudaStream_t);                               \
  template void launch2_rest_da<T>(const S2<T> &, const D2<T> &, int, cudaStream_t);                               \
  template void launch2_coarsest<T>(const D2<T> &, const D2<T> &, T, int *, cudaStream_t);                         \
  template void launch2_jac_d<T>(const D2<T> &, const S2<T> &, const S2<T> &, int, T, cudaStream_t);               \
  template void launch2_jac_a<T>(const S2<T> &, const D2<T> &, const D2<T> &, int, T, cudaStream_t);               \
  template void launch2_asc_fine<T>(const S2<T> &, const D2<T> &, const D2<const T> &, const D2<T> &, int, int, T, \
                                    const Coef<T> &, cudaStream_t);                                                \
  template void launch2_residual<T>(const D2<const T> &, const D2<const T> &, const D2<T> &, int, int,             \
                                    const Coef<T> &, cudaStream_t);                                                \
  template void launch2_ftilde<T>(const D2<const T> &, const D2<T> &, int, cudaStream_t);                          \
  template void launch2_norm<T>(const D2<const T> &, int, unsigned long long *, double *, cudaStream_t);

INST(float)
INST(double)

}  // namespace mg
