// k2d.cu -- 2D kernels of the diagonal-multigrid V-cycle (sm_100a).
//
// Every formula is evaluated in the canonical order of DESIGN.md (terms left
// to right as printed in the paper, constants rounded once from double) and
// the file is compiled with --fmad=false, so the results are bit-identical to
// any other evaluation in the same order.
//
// Level kernels in this file work on lattice coordinates of one octave
// s = 2^o (x = i/s, y = j/s), M = (n-1)/s.
#include <cooperative_groups.h>
#include <cstdlib>

#include "kernels.h"
#include "tma.cuh"
#include "ops2.cuh"

namespace mg {

constexpr int NT = 256;

static inline unsigned blocks_for(int64_t n, int nt = NT) { return (unsigned)((n + nt - 1) / nt); }

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
  double mx = 0.0, ss = 0.0;
  if (t < (int64_t)H * H) {
    int a = (int)(t % H), b = (int)(t / H);
    int x = 2 * a, y = 2 * b;
    T rc = res2z<T, ORDER>(u, f, x, y, M, k);
    T rE = res2z<T, ORDER>(u, f, x + 1, y, M, k);
    T rN = res2z<T, ORDER>(u, f, x, y + 1, M, k);
    if (ns.sums(y)) ss += sq((double)rc) + sq((double)rE);
    if (ns.sums(y + 1)) ss += sq((double)rN);
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
      if (ns.sums(y + 1)) ss += sq((double)ro);
    }
  }
  block_norm_push<NT>(ns, mx, ss);
}

// ------------------------------------------------- descent, level kernels
template <class T>
__global__ void __launch_bounds__(NT) k2_rest_ad_ref(D2<const T> r, S2<T> d, int M) {
  int64_t t = (int64_t)blockIdx.x * NT + threadIdx.x;
  if (t < (int64_t)(M / 2 + 1) * (M / 2 + 1)) node_rest_ad(r, d, M, t);
}

template <class T>
__global__ void __launch_bounds__(NT) k2_rest_da_ref(S2<const T> d, D2<T> r, int Mc) {
  int64_t t = (int64_t)blockIdx.x * NT + threadIdx.x;
  if (t < (int64_t)(Mc - 1) * (Mc - 1)) node_rest_da(d, r, Mc, t);
}

template <class T>
__global__ void k2_coarsest(D2<const T> r, D2<T> v, T c, int *counter) {
  if (threadIdx.x == 0 && blockIdx.x == 0) node_coarsest(r, v, c, counter);
}

// ------------------------------------------------ ascent, diagonal level
template <class T>
__global__ void __launch_bounds__(NT) k2_jac_d1_ref(D2<const T> vc, S2<const T> r, S2<T> v, int M, T c) {
  int64_t t = (int64_t)blockIdx.x * NT + threadIdx.x;
  if (t < (int64_t)(M / 2) * (M / 2)) node_jac_d1(vc, r, v, M, c, t);
}

template <class T>
__global__ void __launch_bounds__(NT) k2_jac_d2_ref(S2<const T> r, S2<T> v, int M, T c) {
  int64_t t = (int64_t)blockIdx.x * NT + threadIdx.x;
  if (t < (int64_t)(M / 2 - 1) * (M / 2 - 1)) node_jac_d2(r, v, M, c, t);
}

// ---------------------------------------------------- ascent, axis level
template <class T>
__global__ void __launch_bounds__(NT) k2_jac_a1_ref(S2<const T> vd, D2<const T> r, D2<T> v, int M, T c) {
  int64_t t = (int64_t)blockIdx.x * NT + threadIdx.x;
  if (t < (int64_t)(M - 1) * (M - 1)) node_jac_a1(vd, r, v, M, c, t);
}

template <class T>
__global__ void __launch_bounds__(NT) k2_jac_a2_ref(D2<const T> r, D2<T> v, int M, T c) {
  int64_t t = (int64_t)blockIdx.x * NT + threadIdx.x;
  if (t < (int64_t)(M - 1) * (M - 1)) node_jac_a2(r, v, M, c, t);
}

// ------------------------------------------------------ coarse levels
// One CTA runs every octave o >= oc: the level arrays are tiny (L2/L1
// resident), so the cost is latency; __syncthreads orders the steps.
template <class T>
__global__ void __launch_bounds__(1024) k2_coarse(const Lev2<T> *lv, int oc, int k, int *counter) {
  pdl_trigger();
  pdl_wait();
  const int tid = threadIdx.x, bs = blockDim.x;
  for (int o = oc; o + 1 < k; o++) {
    const Lev2<T> L = lv[o];
    const Lev2<T> Lc = lv[o + 1];
    int64_t n = (int64_t)(L.M / 2 + 1) * (L.M / 2 + 1);
    for (int t = tid; t < (int)n; t += bs) node_rest_ad(D2<const T>{L.rA.p, L.rA.pitch}, L.rD, L.M, t);
    __syncthreads();
    n = (int64_t)(Lc.M - 1) * (Lc.M - 1);
    for (int t = tid; t < (int)n; t += bs) node_rest_da(S2<const T>{L.rD.e, L.rD.o, L.rD.pitch}, Lc.rA, Lc.M, t);
    __syncthreads();
  }
  if (tid == 0) {
    const Lev2<T> L = lv[k - 1];
    node_coarsest(D2<const T>{L.rA.p, L.rA.pitch}, L.vA, L.cA, counter);
  }
  __syncthreads();
  for (int o = k - 2; o >= oc; o--) {
    const Lev2<T> L = lv[o];
    const Lev2<T> Lc = lv[o + 1];
    const int M = L.M;
    S2<const T> rD{L.rD.e, L.rD.o, L.rD.pitch};
    int64_t n = (int64_t)(M / 2) * (M / 2);
    for (int t = tid; t < (int)n; t += bs) node_jac_d1(D2<const T>{Lc.vA.p, Lc.vA.pitch}, rD, L.vD, M, L.cD, t);
    __syncthreads();
    n = (int64_t)(M / 2 - 1) * (M / 2 - 1);
    for (int t = tid; t < (int)n; t += bs) node_jac_d2(rD, L.vD, M, L.cD, t);
    __syncthreads();
    n = (int64_t)(M - 1) * (M - 1);
    S2<const T> vD{L.vD.e, L.vD.o, L.vD.pitch};
    D2<const T> rA{L.rA.p, L.rA.pitch};
    for (int t = tid; t < (int)n; t += bs) node_jac_a1(vD, rA, L.vA, M, L.cA, t);
    __syncthreads();
    for (int t = tid; t < (int)n; t += bs) node_jac_a2(rA, L.vA, M, L.cA, t);
    __syncthreads();
  }
}

// Shared-memory variant of k2_coarse: the levels below octave oc live in
// shared memory (zero-filled per launch), only r_A(oc) is read from and
// v_A(oc) written to global memory; same node bodies and order.
template <class T>
__global__ void __launch_bounds__(1024) k2_coarse_smem(const Lev2<T> *lvg, int oc, int k, int *counter, int elems) {
  pdl_trigger();
  extern __shared__ __align__(16) unsigned char dsm[];
  T *arena = (T *)dsm;
  __shared__ Lev2<T> lv[32];
  const int tid = threadIdx.x, bs = blockDim.x;
  for (int t = tid; t < elems; t += bs) arena[t] = (T)0;
  if (tid == 0) {
    T *p = arena;
    for (int o = oc; o < k; o++) lv[o] = lvg[o];
    for (int o = oc; o + 1 < k; o++) {
      const int W = lv[o].M / 2 + 1, n2 = W * W;
      lv[o].rD = S2<T>{p, p + n2, W};
      p += 2 * n2;
      lv[o].vD = S2<T>{p, p + n2, W};
      p += 2 * n2;
      lv[o + 1].rA = D2<T>{p, W};
      p += n2;
      lv[o + 1].vA = D2<T>{p, W};
      p += n2;
    }
  }
  __syncthreads();
  pdl_wait();
  for (int o = oc; o + 1 < k; o++) {
    const Lev2<T> L = lv[o];
    const Lev2<T> Lc = lv[o + 1];
    int64_t n = (int64_t)(L.M / 2 + 1) * (L.M / 2 + 1);
    for (int t = tid; t < (int)n; t += bs) node_rest_ad(D2<const T>{L.rA.p, L.rA.pitch}, L.rD, L.M, t);
    __syncthreads();
    n = (int64_t)(Lc.M - 1) * (Lc.M - 1);
    for (int t = tid; t < (int)n; t += bs) node_rest_da(S2<const T>{L.rD.e, L.rD.o, L.rD.pitch}, Lc.rA, Lc.M, t);
    __syncthreads();
  }
  if (tid == 0) {
    const Lev2<T> L = lv[k - 1];
    node_coarsest(D2<const T>{L.rA.p, L.rA.pitch}, L.vA, L.cA, counter);
  }
  __syncthreads();
  for (int o = k - 2; o >= oc; o--) {
    const Lev2<T> L = lv[o];
    const Lev2<T> Lc = lv[o + 1];
    const int M = L.M;
    S2<const T> rD{L.rD.e, L.rD.o, L.rD.pitch};
    int64_t n = (int64_t)(M / 2) * (M / 2);
    for (int t = tid; t < (int)n; t += bs) node_jac_d1(D2<const T>{Lc.vA.p, Lc.vA.pitch}, rD, L.vD, M, L.cD, t);
    __syncthreads();
    n = (int64_t)(M / 2 - 1) * (M / 2 - 1);
    for (int t = tid; t < (int)n; t += bs) node_jac_d2(rD, L.vD, M, L.cD, t);
    __syncthreads();
    n = (int64_t)(M - 1) * (M - 1);
    S2<const T> vD{L.vD.e, L.vD.o, L.vD.pitch};
    D2<const T> rA{L.rA.p, L.rA.pitch};
    for (int t = tid; t < (int)n; t += bs) node_jac_a1(vD, rA, L.vA, M, L.cA, t);
    __syncthreads();
    for (int t = tid; t < (int)n; t += bs) node_jac_a2(rA, L.vA, M, L.cA, t);
    __syncthreads();
  }
}

// Compile-time coarse solver (the default): the octaves from M = MC (<= 64,
// a power of two) down to the single interior node, every level in shared
// memory at compile-time offsets, every step a loop of compile-time trip
// count over the nodes it writes (no per-node division by a run-time size,
// no masked-off iterations: the colour-1 step of an A level walks the green
// nodes only).  Same node formulas and operand order as node_* (ops2.cuh), so
// the iterate is unchanged bit for bit.  Measured on B200 at 8193^2 (MC = 64):
// see DESIGN.md 6.4.
namespace cc2 {
__host__ __device__ constexpr int ilog2(int v) { return v <= 1 ? 0 : 1 + ilog2(v / 2); }
// elements of octave j's arrays (M = MC >> j): rD, vD (E and O, (M/2+1)^2
// each) and rA, vA of the next octave ((M/2+1)^2 each) -- 6 arrays of side M/2+1
template <int MC>
__host__ __device__ constexpr int off(int j) {
  int e = 0;
  for (int q = 0; q < j; q++) {
    const int W = (MC >> q) / 2 + 1;
    e += 6 * W * W;
  }
  return e;
}
}  // namespace cc2

template <class T>
struct CC2P {
  D2<const T> rA0;   // r_A(oc), global
  D2<T> vA0;         // v_A(oc), global
  T cD[6], cA[6];    // Jacobi constants of octaves oc, oc + 1, ..
  int *counter;
};

template <class T, int MC, int NTH>
__global__ void __launch_bounds__(NTH) k2_coarse_ct(const __grid_constant__ CC2P<T> P) {
  const D2<const T> &rA0 = P.rA0;
  const D2<T> &vA0 = P.vA0;
  const T *cDs = P.cD, *cAs = P.cA;
  int *counter = P.counter;
  constexpr int K = cc2::ilog2(MC);   // octaves j = 0 .. K-1 (M = MC .. 2); j < K-1 have a D level
  extern __shared__ __align__(16) unsigned char dsm2[];
  T *ar = (T *)dsm2;
  const int tid = threadIdx.x;
  pdl_trigger();
  // zero the arena (boundary entries stay zero), then r_A(oc) into a dense
  // (MC+1)^2 array after the arena
  constexpr int NA = cc2::off<MC>(K - 1);
  constexpr int W0 = MC + 1;
  T *a0r = ar + NA, *a0v = a0r + W0 * W0;
  for (int t = tid; t < NA + 2 * W0 * W0; t += NTH) ar[t] = (T)0;
  __syncthreads();
  pdl_wait();
  {   // all loads of the thread in flight at once (one L2 round trip, not one per element)
    constexpr int NL = (W0 * W0 + NTH - 1) / NTH;
    T v[NL];
#pragma unroll
    for (int i = 0; i < NL; i++) {
      const int t = tid + i * NTH;
      v[i] = t < W0 * W0 ? rA0.p[(int64_t)(t / W0) * rA0.pitch + t % W0] : (T)0;
    }
#pragma unroll
    for (int i = 0; i < NL; i++)
      if (tid + i * NTH < W0 * W0) a0r[tid + i * NTH] = v[i];
  }
  __syncthreads();
  // A level of octave j: dense, side (M_j + 1); j = 0 is a0, else the "next A"
  // arrays of octave j - 1
  auto Ar = [&](int j) -> T * { return j == 0 ? a0r : ar + cc2::off<MC>(j - 1) + 4 * ((MC >> (j - 1)) / 2 + 1) * ((MC >> (j - 1)) / 2 + 1); };
  auto Av = [&](int j) -> T * { return j == 0 ? a0v : Ar(j) + ((MC >> (j - 1)) / 2 + 1) * ((MC >> (j - 1)) / 2 + 1); };
#define CC2_DESC(J)                                                                                        \
  if constexpr ((J) < K - 1) {                                                                             \
    constexpr int M = MC >> (J), H = M / 2 + 1, WA = M + 1, Mc = M / 2;                                    \
    const T *A = Ar(J);                                                                                    \
    T *E = ar + cc2::off<MC>(J), *O = E + H * H;                                                           \
    for (int t = tid; t < H * H; t += NTH) { /* a2, Erest2r (node_rest_ad) */                             \
      const int a = t % H, b = t / H, x = 2 * a, y = 2 * b;                                                \
      if (x >= 2 && y >= 2 && x <= M - 2 && y <= M - 2)                                                    \
        E[t] = erest2r(A[y * WA + x], A[y * WA + x - 1], A[(y - 1) * WA + x], A[y * WA + x + 1],           \
                       A[(y + 1) * WA + x]);                                                               \
      if (x + 1 <= M - 1 && y + 1 <= M - 1) {                                                              \
        const int c = (y + 1) * WA + x + 1;                                                                \
        O[t] = erest2r(A[c], A[c - 1], A[c - WA], A[c + 1], A[c + WA]);                                    \
      }                                                                                                    \
    }                                                                                                      \
    __syncthreads();                                                                                       \
    T *Ac = Ar((J) + 1);                                                                                   \
    for (int t = tid; t < (Mc - 1) * (Mc - 1); t += NTH) { /* a3, Erest2b (node_rest_da) */               \
      const int X = t % (Mc - 1) + 1, Y = t / (Mc - 1) + 1;                                                \
      Ac[Y * (Mc + 1) + X] = erest2b(E[Y * H + X], O[(Y - 1) * H + X - 1], O[(Y - 1) * H + X], O[Y * H + X], \
                                     O[Y * H + X - 1]);                                                    \
    }                                                                                                      \
    __syncthreads();                                                                                       \
  }
  CC2_DESC(0) CC2_DESC(1) CC2_DESC(2) CC2_DESC(3) CC2_DESC(4)
#undef CC2_DESC
  if (tid == 0) {   // a4: the single interior node of M = 2 (reading A4)
    const T *A = Ar(K - 1);
    Av(K - 1)[1 * 3 + 1] = (-(cAs[K - 1] * A[1 * 3 + 1])) * (T)0.25;
    if (counter) *counter += 1;   // this cycle's norm slot is complete
  }
  __syncthreads();
#define CC2_ASC(J)                                                                                           \
  if constexpr ((J) < K - 1) {                                                                               \
    constexpr int M = MC >> (J), H = M / 2 + 1, WA = M + 1, WC = M / 2 + 1, Wd = M / 2;                      \
    const T *vc = Av((J) + 1), *rE = ar + cc2::off<MC>(J), *rO = rE + H * H;                                 \
    T *vE = ar + cc2::off<MC>(J) + 2 * H * H, *vO = vE + H * H;                                              \
    const T cD = cDs[J], cA = cAs[J];                                                                        \
    for (int t = tid; t < Wd * Wd; t += NTH) { /* a5, Eajacr on O (node_jac_d1) */                          \
      const int a = t % Wd, b = t / Wd;                                                                      \
      vO[b * H + a] = jac4(cD, rO[b * H + a], vc[b * WC + a], vc[b * WC + a + 1], vc[(b + 1) * WC + a + 1],  \
                           vc[(b + 1) * WC + a]);                                                            \
    }                                                                                                        \
    __syncthreads();                                                                                         \
    for (int t = tid; t < (Wd - 1) * (Wd - 1); t += NTH) { /* a6, Eajacb on E (node_jac_d2) */              \
      const int a = t % (Wd - 1) + 1, b = t / (Wd - 1) + 1;                                                  \
      vE[b * H + a] = jac4(cD, rE[b * H + a], vO[(b - 1) * H + a - 1], vO[(b - 1) * H + a], vO[b * H + a],   \
                           vO[b * H + a - 1]);                                                               \
    }                                                                                                        \
    __syncthreads();                                                                                         \
    const T *rA = Ar(J);                                                                                     \
    T *vA = Av(J);                                                                                           \
    /* v_D(s) at node (x, y), x + y even: E (both even) or O (both odd) */                                 \
    auto vd = [&](int x, int y) -> T { return (y & 1) ? vO[(y >> 1) * H + (x >> 1)] : vE[(y >> 1) * H + (x >> 1)]; }; \
    for (int t = tid; t < (M - 1) * Wd; t += NTH) { /* a7 colour 1: the green node of pair t (node_jac_a1) */ \
      const int y = t / Wd + 1, x = 2 * (t % Wd) + 1 + (y & 1);                                              \
      if (x <= M - 1)                                                                                        \
        vA[y * WA + x] = jac4(cA, rA[y * WA + x], vd(x - 1, y), vd(x, y - 1), vd(x + 1, y), vd(x, y + 1));    \
    }                                                                                                        \
    __syncthreads();                                                                                         \
    for (int t = tid; t < (M - 1) * Wd; t += NTH) { /* a7 colour 2: the D node of pair t (node_jac_a2) */   \
      const int y = t / Wd + 1, x = 2 * (t % Wd) + 2 - (y & 1);                                              \
      if (x <= M - 1) {                                                                                      \
        const int c = y * WA + x;                                                                            \
        vA[c] = jac4(cA, rA[c], vA[c - 1], vA[c - WA], vA[c + 1], vA[c + WA]);                               \
      }                                                                                                      \
    }                                                                                                        \
    __syncthreads();                                                                                         \
  }
  CC2_ASC(4) CC2_ASC(3) CC2_ASC(2) CC2_ASC(1) CC2_ASC(0)
#undef CC2_ASC
  for (int t = tid; t < W0 * W0; t += NTH) {
    const int x = t % W0, y = t / W0;
    if (x >= 1 && y >= 1 && x <= MC - 1 && y <= MC - 1) vA0.p[(int64_t)y * vA0.pitch + x] = a0v[t];
  }
}

template <class T, int MC>
static size_t cc2_bytes() {
  constexpr int K = cc2::ilog2(MC);
  return sizeof(T) * (cc2::off<MC>(K - 1) + 2 * (MC + 1) * (MC + 1));
}

// Cooperative tail (as k3l_tail): octaves om .. oc-1 grid-wide with a grid
// barrier between steps, octaves >= oc in CTA 0's shared memory; one launch.
template <class T>
struct Tail2 {
  Lev2<T> lv[40];
  int om, oc, k;
  int *counter;
};

template <class T>
__device__ __forceinline__ void coarse2_block(const Tail2<T> &P, T *arena) {
  const int tid = threadIdx.x, bs = blockDim.x, oc = P.oc, k = P.k;
  // octave o's arrays: r_E, r_O, v_E, v_O of D(s), r, v of A(2s) -- 6 consecutive W^2 arrays
  auto off = [&](int o) {
    size_t e = 0;
    for (int q = oc; q < o; q++) {
      const size_t W = P.lv[q].M / 2 + 1;
      e += 6 * W * W;
    }
    return arena + e;
  };
  auto aa = [&](int o, int which) -> D2<T> {   // A(s) of octave o (global at oc)
    if (o == oc) return which ? P.lv[o].vA : P.lv[o].rA;
    const int W = P.lv[o - 1].M / 2 + 1;
    return D2<T>{off(o - 1) + (int64_t)(4 + which) * W * W, W};
  };
  for (size_t t = tid, n = off(k - 1) - arena; t < n; t += bs) arena[t] = (T)0;
  __syncthreads();
  for (int o = oc; o + 1 < k; o++) {
    const int M = P.lv[o].M, W = M / 2 + 1, n2 = W * W;
    T *b = off(o);
    const S2<T> rD{b, b + n2, W};
    const D2<T> rA = aa(o, 0), rA2 = aa(o + 1, 0);
    for (int t = tid; t < (int)n2; t += bs) node_rest_ad(D2<const T>{rA.p, rA.pitch}, rD, M, t);
    __syncthreads();
    const int64_t n = (int64_t)(M / 2 - 1) * (M / 2 - 1);
    for (int t = tid; t < (int)n; t += bs) node_rest_da(S2<const T>{rD.e, rD.o, rD.pitch}, rA2, M / 2, t);
    __syncthreads();
  }
  if (tid == 0) {
    const D2<T> rA = aa(k - 1, 0), vA = aa(k - 1, 1);
    node_coarsest(D2<const T>{rA.p, rA.pitch}, vA, P.lv[k - 1].cA, P.counter);
  }
  __syncthreads();
  for (int o = k - 2; o >= oc; o--) {
    const Lev2<T> &L = P.lv[o];
    const int M = L.M, W = M / 2 + 1, n2 = W * W;
    T *b = off(o);
    const S2<const T> rD{b, b + n2, W};
    const S2<T> vD{b + 2 * n2, b + 3 * n2, W};
    const D2<T> rA = aa(o, 0), vA = aa(o, 1), vA2 = aa(o + 1, 1);
    int64_t n = (int64_t)(M / 2) * (M / 2);
    for (int t = tid; t < (int)n; t += bs) node_jac_d1(D2<const T>{vA2.p, vA2.pitch}, rD, vD, M, L.cD, t);
    __syncthreads();
    n = (int64_t)(M / 2 - 1) * (M / 2 - 1);
    for (int t = tid; t < (int)n; t += bs) node_jac_d2(rD, vD, M, L.cD, t);
    __syncthreads();
    n = (int64_t)(M - 1) * (M - 1);
    const S2<const T> vDc{vD.e, vD.o, vD.pitch};
    const D2<const T> rAc{rA.p, rA.pitch};
    for (int t = tid; t < (int)n; t += bs) node_jac_a1(vDc, rAc, vA, M, L.cA, t);
    __syncthreads();
    for (int t = tid; t < (int)n; t += bs) node_jac_a2(rAc, vA, M, L.cA, t);
    __syncthreads();
  }
}

template <class T>
__global__ void __launch_bounds__(512, 1) k2_tail(const __grid_constant__ Tail2<T> P) {
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  extern __shared__ __align__(16) unsigned char dsm[];
  const int64_t gt = (int64_t)blockIdx.x * blockDim.x + threadIdx.x, gs = (int64_t)gridDim.x * blockDim.x;
  for (int o = P.om; o < P.oc; o++) {
    const Lev2<T> &L = P.lv[o], &Lc = P.lv[o + 1];
    int64_t n = (int64_t)(L.M / 2 + 1) * (L.M / 2 + 1);
    for (int t = gt; t < (int)n; t += gs) node_rest_ad(D2<const T>{L.rA.p, L.rA.pitch}, L.rD, L.M, t);
    grid.sync();
    n = (int64_t)(Lc.M - 1) * (Lc.M - 1);
    for (int t = gt; t < (int)n; t += gs) node_rest_da(S2<const T>{L.rD.e, L.rD.o, L.rD.pitch}, Lc.rA, Lc.M, t);
    grid.sync();
  }
  if (blockIdx.x == 0) coarse2_block(P, (T *)dsm);
  grid.sync();
  for (int o = P.oc - 1; o >= P.om; o--) {
    const Lev2<T> &L = P.lv[o], &Lc = P.lv[o + 1];
    const int M = L.M;
    const S2<const T> rD{L.rD.e, L.rD.o, L.rD.pitch};
    int64_t n = (int64_t)(M / 2) * (M / 2);
    for (int t = gt; t < (int)n; t += gs) node_jac_d1(D2<const T>{Lc.vA.p, Lc.vA.pitch}, rD, L.vD, M, L.cD, t);
    grid.sync();
    n = (int64_t)(M / 2 - 1) * (M / 2 - 1);
    for (int t = gt; t < (int)n; t += gs) node_jac_d2(rD, L.vD, M, L.cD, t);
    grid.sync();
    n = (int64_t)(M - 1) * (M - 1);
    const S2<const T> vD{L.vD.e, L.vD.o, L.vD.pitch};
    const D2<const T> rA{L.rA.p, L.rA.pitch};
    for (int t = gt; t < (int)n; t += gs) node_jac_a1(vD, rA, L.vA, M, L.cA, t);
    grid.sync();
    for (int t = gt; t < (int)n; t += gs) node_jac_a2(rA, L.vA, M, L.cA, t);
    grid.sync();
  }
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

// u_new <- u_old + v at the interior (u_new may alias u_old).
template <class T>
__global__ void __launch_bounds__(NT) k2_update_ref(D2<const T> uo, D2<const T> v, D2<T> un, int M) {
  int W = M - 1;
  int64_t t = (int64_t)blockIdx.x * NT + threadIdx.x;
  if (t >= (int64_t)W * W) return;
  int x = (int)(t % W) + 1, y = (int)(t / W) + 1;
  un(x, y) = uo(x, y) + v(x, y);
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

// Row-ranged variants for slabs (multi-GPU): rows [ylo, yhi) only.
template <class T>
__global__ void __launch_bounds__(NT) k2_ftilde_rows(D2<const T> f, D2<T> ft, int M, int ylo, int yhi) {
  int W = M - 1;
  int64_t t = (int64_t)blockIdx.x * NT + threadIdx.x;
  if (t >= (int64_t)W * (yhi - ylo)) return;
  int x = (int)(t % W) + 1, y = (int)(t / W) + ylo;
  if (y < 1 || y > M - 1) return;
  T s = (T)8 * f(x, y);
  s = s + f(x + 1, y);
  s = s + f(x, y + 1);
  s = s + f(x - 1, y);
  s = s + f(x, y - 1);
  ft(x, y) = s * (T)(1.0 / 12.0);
}

template <class T, int ORDER>
__global__ void __launch_bounds__(NT) k2_residual_rows(D2<const T> u, D2<const T> f, D2<T> r, int M, Coef<T> k, int ylo,
                                                       int yhi) {
  int64_t t = (int64_t)blockIdx.x * NT + threadIdx.x;
  int Wd = M + 1;
  if (t >= (int64_t)Wd * (yhi - ylo)) return;
  int x = (int)(t % Wd), y = (int)(t / Wd) + ylo;
  r(x, y) = res2z<T, ORDER>(u, f, x, y, M, k);
}

template <class T>
__global__ void __launch_bounds__(NT) k2_norm_rows(D2<const T> a, int M, int ylo, int yhi, unsigned long long *mx_out,
                                                   double *ss_out) {
  int W = M - 1;
  double mx = 0.0, ss = 0.0;
  for (int64_t t = (int64_t)blockIdx.x * NT + threadIdx.x; t < (int64_t)W * (yhi - ylo); t += (int64_t)gridDim.x * NT) {
    int x = (int)(t % W) + 1, y = (int)(t / W) + ylo;
    if (y < 1 || y > M - 1) continue;
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
void launch2_ftilde_rows(const D2<const T> &f, const D2<T> &ft, int M, int ylo, int yhi, cudaStream_t st) {
  int64_t W = M - 1;
  if (yhi > ylo) k2_ftilde_rows<T><<<blocks_for(W * (yhi - ylo)), NT, 0, st>>>(f, ft, M, ylo, yhi);
}
template <class T>
void launch2_residual_rows(const D2<const T> &u, const D2<const T> &f, const D2<T> &r, int M, int order,
                           const Coef<T> &k, int ylo, int yhi, cudaStream_t st) {
  int64_t W = M + 1;
  if (yhi <= ylo) return;
  if (order == 2)
    k2_residual_rows<T, 2><<<blocks_for(W * (yhi - ylo)), NT, 0, st>>>(u, f, r, M, k, ylo, yhi);
  else
    k2_residual_rows<T, 4><<<blocks_for(W * (yhi - ylo)), NT, 0, st>>>(u, f, r, M, k, ylo, yhi);
}
template <class T>
void launch2_norm_rows(const D2<const T> &a, int M, int ylo, int yhi, unsigned long long *mx, double *ss,
                       cudaStream_t st) {
  k2_norm_rows<T><<<148 * 4, NT, 0, st>>>(a, M, ylo, yhi, mx, ss);
}

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
void launch2_asc_fine(const S2<T> &vd, const D2<T> &u, const D2<const T> &f, const D2<T> &scratch, const D2<T> &un,
                      int M, int order, T c, const Coef<T> &k, cudaStream_t st) {
  int64_t W = M - 1;
  if (order == 2) {
    k2_asc_fine1_ref<T, 2><<<blocks_for(W * W), NT, 0, st>>>(cs(vd), cd(u), f, scratch, M, c, k);
    k2_asc_fine2_ref<T, 2><<<blocks_for(W * W), NT, 0, st>>>(cd(u), f, scratch, M, c, k);
  } else {
    k2_asc_fine1_ref<T, 4><<<blocks_for(W * W), NT, 0, st>>>(cs(vd), cd(u), f, scratch, M, c, k);
    k2_asc_fine2_ref<T, 4><<<blocks_for(W * W), NT, 0, st>>>(cd(u), f, scratch, M, c, k);
  }
  k2_update_ref<T><<<blocks_for(W * W), NT, 0, st>>>(cd(u), cd(scratch), un, M);
}

// D(s) nodes of a dense A(s) field into split E/O arrays (extra sweeps,
// reading A19): E(a,b) = v(2a, 2b), O(a,b) = v(2a+1, 2b+1).
template <class T>
__global__ void __launch_bounds__(NT) k2_gather_d(D2<const T> v, S2<T> d, int M) {
  const int H = M / 2 + 1;
  int64_t t = (int64_t)blockIdx.x * NT + threadIdx.x;
  if (t >= (int64_t)H * H) return;
  const int a = (int)(t % H), b = (int)(t / H);
  d.e[(int64_t)b * d.pitch + a] = v(2 * a, 2 * b);
  d.o[(int64_t)b * d.pitch + a] = (2 * a + 1 <= M && 2 * b + 1 <= M) ? v(2 * a + 1, 2 * b + 1) : (T)0;
}

template <class T>
void launch2_gather_d(const D2<T> &v, const S2<T> &d, int M, cudaStream_t st) {
  const int64_t H = M / 2 + 1;
  k2_gather_d<T><<<blocks_for(H * H), NT, 0, st>>>(cd(v), d, M);
}

// finest ascent with `sweeps` two-colour steps: the first from v_D(1), the
// others from the D nodes of v itself (gathered into tmp), then u_new = u + v
template <class T>
void launch2_asc_fine_sweeps(const S2<T> &vd, const D2<T> &u, const D2<const T> &f, const D2<T> &scratch,
                             const D2<T> &un, int M, int order, T c, const Coef<T> &k, int sweeps, const S2<T> &tmp,
                             cudaStream_t st) {
  int64_t W = M - 1;
  for (int sw = 0; sw < sweeps; sw++) {
    const S2<T> &src = sw == 0 ? vd : tmp;
    if (sw > 0) launch2_gather_d<T>(scratch, tmp, M, st);
    if (order == 2) {
      k2_asc_fine1_ref<T, 2><<<blocks_for(W * W), NT, 0, st>>>(cs(src), cd(u), f, scratch, M, c, k);
      k2_asc_fine2_ref<T, 2><<<blocks_for(W * W), NT, 0, st>>>(cd(u), f, scratch, M, c, k);
    } else {
      k2_asc_fine1_ref<T, 4><<<blocks_for(W * W), NT, 0, st>>>(cs(src), cd(u), f, scratch, M, c, k);
      k2_asc_fine2_ref<T, 4><<<blocks_for(W * W), NT, 0, st>>>(cd(u), f, scratch, M, c, k);
    }
  }
  k2_update_ref<T><<<blocks_for(W * W), NT, 0, st>>>(cd(u), cd(scratch), un, M);
}

// The compile-time coarse solver for M(oc) = MC (host descriptors h_lev).
template <class T, int MC>
static bool coarse_ct(const Lev2<T> *h_lev, int oc, int *counter, cudaStream_t st) {
  static_assert(MC >= 2 && MC <= 64, "");
  constexpr int NTH = MC >= 32 ? 512 : 256;
  constexpr int K = cc2::ilog2(MC);
  CC2P<T> P{};
  P.rA0 = D2<const T>{h_lev[oc].rA.p, h_lev[oc].rA.pitch};
  P.vA0 = h_lev[oc].vA;
  for (int j = 0; j < K; j++) {
    P.cD[j] = h_lev[oc + j].cD;
    P.cA[j] = h_lev[oc + j].cA;
  }
  P.counter = counter;
  const size_t bytes = cc2_bytes<T, MC>();
  if (cudaFuncSetAttribute(k2_coarse_ct<T, MC, NTH>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes))
    return false;
  note_launch(launch_pdl(k2_coarse_ct<T, MC, NTH>, dim3(1), dim3(NTH), bytes, st, P));
  return true;
}

template <class T>
void launch2_coarse(const Lev2<T> *d_lev, int oc, int k, int *counter, cudaStream_t st, const Lev2<T> *h_lev) {
  static const bool ct = !env_flag("MG_COARSE_NOCT");
  if (ct && h_lev && oc >= 1 && k - oc <= 6) {
    bool done = false;
    switch (k - oc) {   // M(oc) = 2^(k - oc)
      case 1: done = coarse_ct<T, 2>(h_lev, oc, counter, st); break;
      case 2: done = coarse_ct<T, 4>(h_lev, oc, counter, st); break;
      case 3: done = coarse_ct<T, 8>(h_lev, oc, counter, st); break;
      case 4: done = coarse_ct<T, 16>(h_lev, oc, counter, st); break;
      case 5: done = coarse_ct<T, 32>(h_lev, oc, counter, st); break;
      case 6: done = coarse_ct<T, 64>(h_lev, oc, counter, st); break;
    }
    if (done) return;
  }
  static const bool global = env_flag("MG_COARSE_GLOBAL");
  if (!global && oc >= 1 && k <= 32) {
    size_t elems = 0;
    for (int o = oc; o + 1 < k; o++) {
      const size_t W = (size_t(1) << (k - o - 1)) + 1;   // M_o / 2 + 1 for n = 2^k + 1
      elems += 6 * W * W;
    }
    const size_t bytes = elems * sizeof(T);
    if (bytes <= 200 * 1024) {
      cudaFuncSetAttribute(k2_coarse_smem<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
      launch_pdl(k2_coarse_smem<T>, dim3(1), dim3(1024), bytes, st, d_lev, oc, k, counter, (int)elems);
      return;
    }
  }
  launch_pdl(k2_coarse<T>, dim3(1), dim3(1024), 0, st, d_lev, oc, k, counter);
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
  template void launch2_ftilde_rows<T>(const D2<const T> &, const D2<T> &, int, int, int, cudaStream_t);           \
  template void launch2_residual_rows<T>(const D2<const T> &, const D2<const T> &, const D2<T> &, int, int,        \
                                         const Coef<T> &, int, int, cudaStream_t);                                 \
  template void launch2_norm_rows<T>(const D2<const T> &, int, int, int, unsigned long long *, double *,           \
                                     cudaStream_t);                                                                \
  template void launch2_desc_fine<T>(const D2<const T> &, const D2<const T> &, const S2<T> &, int, int,            \
                                     const Coef<T> &, const NormSink &, cudaStream_t);                             \
  template void launch2_rest_ad<T>(const D2<T> &, const S2<T> &, int, cudaStream_t);                               \
  template void launch2_rest_da<T>(const S2<T> &, const D2<T> &, int, cudaStream_t);                               \
  template void launch2_coarsest<T>(const D2<T> &, const D2<T> &, T, int *, cudaStream_t);                         \
  template void launch2_jac_d<T>(const D2<T> &, const S2<T> &, const S2<T> &, int, T, cudaStream_t);               \
  template void launch2_jac_a<T>(const S2<T> &, const D2<T> &, const D2<T> &, int, T, cudaStream_t);               \
  template void launch2_asc_fine<T>(const S2<T> &, const D2<T> &, const D2<const T> &, const D2<T> &, const D2<T> &, \
                                    int, int, T,                                                                   \
                                    const Coef<T> &, cudaStream_t);                                                \
  template void launch2_coarse<T>(const Lev2<T> *, int, int, int *, cudaStream_t, const Lev2<T> *);                                \
  template void launch2_gather_d<T>(const D2<T> &, const S2<T> &, int, cudaStream_t);                              \
  template void launch2_asc_fine_sweeps<T>(const S2<T> &, const D2<T> &, const D2<const T> &, const D2<T> &,        \
                                           const D2<T> &, int, int, T, const Coef<T> &, int, const S2<T> &,        \
                                           cudaStream_t);                                                           \
  template void launch2_residual<T>(const D2<const T> &, const D2<const T> &, const D2<T> &, int, int,             \
                                    const Coef<T> &, cudaStream_t);                                                \
  template void launch2_ftilde<T>(const D2<const T> &, const D2<T> &, int, cudaStream_t);                          \
  template void launch2_norm<T>(const D2<const T> &, int, unsigned long long *, double *, cudaStream_t);

INST(float)
INST(double)


template <class T>
bool launch2_tail(const Lev2<T> *h_lev, int om, int oc, int k, int *counter, cudaStream_t st) {
  if (k > 40 || om < 1 || om > oc || oc >= k) return false;
  Tail2<T> P;
  for (int o = 0; o < k; o++) P.lv[o] = h_lev[o];
  P.om = om;
  P.oc = oc;
  P.k = k;
  P.counter = counter;
  size_t elems = 0;
  for (int o = oc; o + 1 < k; o++) {
    const size_t W = h_lev[o].M / 2 + 1;
    elems += 6 * W * W;
  }
  const size_t bytes = elems * sizeof(T);
  if (bytes > 200 * 1024) return false;
  if (cudaFuncSetAttribute(k2_tail<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes) != cudaSuccess)
    return false;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  // a cooperative launch that cannot be co-resident (MPS / green-context SM
  // limits) would be rejected -- inside a stream capture that invalidates the
  // capture, so decide on the host first and let the caller run per-level kernels
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k2_tail<T>, 512, bytes) != cudaSuccess ||
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
  return cudaLaunchKernelEx(&cfg, k2_tail<T>, P) == cudaSuccess;
}
template bool launch2_tail<float>(const Lev2<float> *, int, int, int, int *, cudaStream_t);
template bool launch2_tail<double>(const Lev2<double> *, int, int, int, int *, cudaStream_t);

}  // namespace mg
