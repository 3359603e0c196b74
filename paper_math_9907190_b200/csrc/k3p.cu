// k3p.cu -- 3D finest-octave kernels, second generation (sm_100a, order 2).
//
// The two passes that carry 60 % of the 3D bytes (SURVEY 8(a) a9+a10 and
// a15 at s = 1) as register-streaming TMA plane pipelines:
//
//   * one persistent CTA per SM (512 threads, 16 warps) walks a balanced
//     list of work items, each an xy tile of TX x TY = 60 x 30 fine nodes
//     times a z range; full-height items for the first floor(T/G)*G tiles,
//     the remaining tiles split into z segments so every CTA gets the same
//     number of planes (the xy halo of concurrently streamed neighbours is
//     re-read from L2, not HBM);
//   * lane l of warp w owns the four nodes (x0-2+2l + {0,1}, y0-1+2w + {0,1})
//     of every plane: the z neighbours of a node are the thread's own
//     registers, the x/y neighbours of u come from the TMA-staged plane in
//     shared memory, and the only values exchanged through shared memory are
//     the green ones of the current plane (one 34x34 plane ring);
//   * load L_j = {u(j), f(j-1)[, v_R(j)]}; step j uses L_j and L_{j-1}, so a
//     ring of NS slots keeps NS-2 planes of TMA loads in flight.
//
// Node formulas and their evaluation order are the canonical ones of
// ops3.cuh, so the results are bit-identical to the oracle.
// Order 4 (Efos4) keeps the first-generation kernels of k3f.cu: its face
// diagonals reach the neighbours of the z +- 1 planes.
#include "kernels.h"
#include "ops3.cuh"
#include "tma.cuh"

namespace mg {

namespace zp {

constexpr int TX = 60, TY = 30, NT = 512;
constexpr int GS = 34;                       // green-plane ring: 34 x 34 (rows/lanes -1 .. 32)
constexpr int al128(int n) { return (n + 127) / 128 * 128; }

template <class T>
struct Geo {
  static constexpr int AL = 16 / (int)sizeof(T);       // TMA x alignment (elements)
  static constexpr int UXO = (AL == 2) ? 4 : 6;         // u box starts at x0 - UXO (>= 3, aligned)
  static constexpr int UW = (UXO + 63 + AL - 1) / AL * AL, UH = TY + 4;
  static constexpr int FW = 64, FH = TY + 2;            // f box: x0-2 .., y0-1 ..
  static constexpr int VW = (34 + AL - 1 + AL - 1) / AL * AL, VH = TY / 2 + 2;
  static constexpr int U_BYTES = UW * UH * (int)sizeof(T), F_BYTES = FW * FH * (int)sizeof(T);
  static constexpr int V_BYTES = VW * VH * (int)sizeof(T);
  static constexpr int GPL = al128(GS * GS * (int)sizeof(T));
};

template <class T>
struct V2t;
template <>
struct V2t<double> {
  using t = double2;
};
template <>
struct V2t<float> {
  using t = float2;
};
template <class T>
__device__ __forceinline__ void ld2(const T *p, T &a, T &b) {
  auto v = *reinterpret_cast<const typename V2t<T>::t *>(p);
  a = v.x;
  b = v.y;
}
template <class T>
__device__ __forceinline__ void st2(T *p, T a, T b) {
  typename V2t<T>::t v;
  v.x = a;
  v.y = b;
  *reinterpret_cast<typename V2t<T>::t *>(p) = v;
}

// r = f - (-(6c) + xp + xm + yp + ym + zp + zm) * (n-1)^2   (res3v, order 2)
template <class T>
__device__ __forceinline__ T res7(T c, T xp, T xm, T yp, T ym, T zp, T zm, T f, T invh2) {
  T lap = -((T)6 * c);
  lap = lap + xp;
  lap = lap + xm;
  lap = lap + yp;
  lap = lap + ym;
  lap = lap + zp;
  lap = lap + zm;
  lap = lap * invh2;
  return f - lap;
}

// Balanced work list: items k < W are whole tiles b + k*G over [zlo, zhi);
// item W (when R = T mod G > 0) is one z segment of tail tile W*G + b mod R.
struct Item {
  int x0, y0, zs, ze;
};
struct Sched {
  int T, ntx, zlo, zhi;
  __device__ __forceinline__ int count(int G) const { return T / G + (T % G ? 1 : 0); }
  __device__ __forceinline__ Item get(int k, int b, int G) const {
    const int W = T / G, R = T % G;
    int t, zs = zlo, ze = zhi;
    if (k < W) {
      t = b + k * G;
    } else {
      const int r = b % R, nseg = G / R + (r < G % R ? 1 : 0), sg = b / R;
      const long long Z = zhi - zlo;
      t = W * G + r;
      zs = zlo + (int)(Z * sg / nseg);
      ze = zlo + (int)(Z * (sg + 1) / nseg);
    }
    Item it;
    it.x0 = (t % ntx) * TX - 2;
    it.y0 = (t / ntx) * TY;
    it.zs = zs;
    it.ze = ze;
    return it;
  }
};

}  // namespace zp

using namespace zp;

// ------------------------------------------------------------ pipeline
// Op: NS (slots), SLOT (bytes), SMEM, Params (with .sc, .nunits unused),
// issue(P, it, j, slot, bar), State, begin(State&, it), step(P, State&, it, j,
// Lc, Lp, gring) -- step must not touch Lp / the ring after its barrier.
template <class Op>
__global__ void __launch_bounds__(NT, 1) zpipe(const __grid_constant__ typename Op::Params P) {
  constexpr int NS = Op::NS, D = NS - 2;
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ __align__(8) uint64_t bar[NS];
  const int G = gridDim.x, b = blockIdx.x;
  const int nit = P.sc.count(G);
  if (threadIdx.x == 0) {
    for (int s = 0; s < NS; s++) mbar_init(&bar[s], 1);
    fence_mbar_init();
    Op::prefetch(P);
  }
  __syncthreads();
  unsigned char *gring = smem + NS * Op::SLOT;

  // producer cursor (thread 0): item pk, plane pj, slot ps
  int pk = 0, pj = 0, ps = 0;
  Item pit{};
  bool pmore = false;
  auto pseek = [&](int k) {   // first non-empty item >= k
    for (; k < nit; k++) {
      Item it = P.sc.get(k, b, G);
      if (it.ze > it.zs) {
        pk = k;
        pit = it;
        pj = it.zs - 2;
        pmore = true;
        return;
      }
    }
    pmore = false;
  };
  auto produce = [&]() {
    if (!pmore) return;
    Op::issue(P, pit, pj, smem + ps * Op::SLOT, &bar[ps]);
    ps = (ps + 1 == NS) ? 0 : ps + 1;
    if (++pj > pit.ze + 1) pseek(pk + 1);
  };
  if (threadIdx.x == 0) {
    pseek(0);
    for (int d = 0; d < D; d++) produce();
  }

  typename Op::State S;
  Op::init(S);
  int cs = 0, cprev = NS - 1;
  uint32_t phase = 0;
  for (int k = 0; k < nit; k++) {
    const Item it = P.sc.get(k, b, G);
    if (it.ze <= it.zs) continue;
    for (int j = it.zs - 2; j <= it.ze + 1; j++) {
      if (threadIdx.x == 0) produce();
      mbar_wait(&bar[cs], phase);
      Op::step(P, S, it, j, smem + cs * Op::SLOT, smem + cprev * Op::SLOT, gring);
      __syncthreads();
      cprev = cs;
      if (++cs == NS) {
        cs = 0;
        phase ^= 1;
      }
    }
  }
  Op::finish(P, S);
}

template <class T>
__device__ __forceinline__ T *gptr(unsigned char *gring, int z, int row, int lane) {
  // green value of ring plane z (z >= -2) at own row index row (-1..32), lane (-1..32)
  return (T *)(gring + ((z + 3) % 3) * Geo<T>::GPL) + (row + 1) * GS + (lane + 1);
}

// =================================================== finest descent a9 + a10
// Step j: r(j-1) at the thread's 4 nodes (registers, greens also to the
// ring); then Erred at the red nodes of plane q = j-2.
template <class T>
struct OpDesc3P {
  using Gm = Geo<T>;
  static constexpr int NS = sizeof(T) == 8 ? 5 : 8;
  static constexpr int U_OFF = 0, F_OFF = al128(Gm::U_BYTES), SLOT = al128(F_OFF + Gm::F_BYTES);
  static constexpr int SMEM = NS * SLOT + 3 * Gm::GPL;
  struct Params {
    CUtensorMap tu, tf;
    S3<T> out;
    Sched sc;
    int M, fz0;
    T invh2;
    NormSink ns;
  };
  struct State {
    T um[2][2], uc[2][2];   // own u(j-2), u(j-1): [row A/B][col 0/1]
    T r0[2][2], r1[2][2];   // own r(j-3), r(j-2)
    double mx;
  };
  static __device__ void prefetch(const Params &P) {
    tma_prefetch_desc(&P.tu);
    tma_prefetch_desc(&P.tf);
  }
  static __device__ void init(State &S) { S.mx = 0.0; }
  static __device__ void issue(const Params &P, const Item &it, int j, unsigned char *slot, uint64_t *bar) {
    const bool wf = j >= it.zs;
    mbar_expect_tx(bar, Gm::U_BYTES + (wf ? Gm::F_BYTES : 0));
    tma_load_3d(slot + U_OFF, &P.tu, it.x0 - Gm::UXO, it.y0 - 2, j - P.fz0, bar);
    if (wf) tma_load_3d(slot + F_OFF, &P.tf, it.x0 - 2, it.y0 - 1, j - 1 - P.fz0, bar);
  }
  static __device__ __forceinline__ void step(const Params &P, State &S, const Item &it, int j, unsigned char *Lc,
                                              unsigned char *Lp, unsigned char *gring) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, M = P.M;
    const int xl = it.x0 - 2 + 2 * lane, yA = it.y0 - 1 + 2 * w;
    const int uo = (2 * w + 1) * Gm::UW + 2 * lane - 2 + Gm::UXO;   // u box offset of (xl, yA)
    const int fo = 2 * w * Gm::FW + 2 * lane;                         // f box offset of (xl, yA)
    T un[2][2];
    {
      const T *U = (const T *)(Lc + U_OFF);
      ld2(U + uo, un[0][0], un[0][1]);
      ld2(U + uo + Gm::UW, un[1][0], un[1][1]);
    }
    if (j >= it.zs) {
      // ---- r(j-1) at the own nodes
      const T *U = (const T *)(Lp + U_OFF) + uo;   // u(j-1) at (xl, yA)
      const T *F = (const T *)(Lc + F_OFF) + fo;   // f(j-1)
      T ymA0, ymA1, ypB0, ypB1, t, lA, rA, lB, rB, fA0, fA1, fB0, fB1;
      ld2(U - Gm::UW, ymA0, ymA1);
      ld2(U + 2 * Gm::UW, ypB0, ypB1);
      ld2(U - 2, t, lA);
      ld2(U + 2, rA, t);
      ld2(U + Gm::UW - 2, t, lB);
      ld2(U + Gm::UW + 2, rB, t);
      ld2(F, fA0, fA1);
      ld2(F + Gm::FW, fB0, fB1);
      const T h = P.invh2;
      T rn[2][2];
      // i+1, i-1, j+1, j-1, k+1, k-1
      rn[0][0] = res7(S.uc[0][0], S.uc[0][1], lA, S.uc[1][0], ymA0, un[0][0], S.um[0][0], fA0, h);
      rn[0][1] = res7(S.uc[0][1], rA, S.uc[0][0], S.uc[1][1], ymA1, un[0][1], S.um[0][1], fA1, h);
      rn[1][0] = res7(S.uc[1][0], S.uc[1][1], lB, ypB0, S.uc[0][0], un[1][0], S.um[1][0], fB0, h);
      rn[1][1] = res7(S.uc[1][1], rB, S.uc[1][0], ypB1, S.uc[0][1], un[1][1], S.um[1][1], fB1, h);
      const int z = j - 1;
      const bool zin = z >= 1 && z <= M - 1;
      const bool c0 = xl >= 1 && xl <= M - 1, c1 = xl + 1 >= 1 && xl + 1 <= M - 1;
      const bool a = zin && yA >= 1 && yA <= M - 1, bb = zin && yA + 1 >= 1 && yA + 1 <= M - 1;
      rn[0][0] = (a && c0) ? rn[0][0] : (T)0;
      rn[0][1] = (a && c1) ? rn[0][1] : (T)0;
      rn[1][0] = (bb && c0) ? rn[1][0] : (T)0;
      rn[1][1] = (bb && c1) ? rn[1][1] : (T)0;
      // every computed r is a true residual (or 0): max over all of them
      S.mx = nmax(S.mx, nmax(nmax(absd(rn[0][0]), absd(rn[0][1])), nmax(absd(rn[1][0]), absd(rn[1][1]))));
      // green (x+y+z odd) values to the ring; red column offset of row A = (yA + z) & 1
      const int pA = (yA + z) & 1;
      *gptr<T>(gring, z, 2 * w, lane) = pA ? rn[0][0] : rn[0][1];
      *gptr<T>(gring, z, 2 * w + 1, lane) = pA ? rn[1][1] : rn[1][0];
      // ---- Erred at the red nodes of q = j-2: r(q-1) = S.r0, r(q) = S.r1, r(q+1) = rn
      const int q = j - 2;
      if (q >= it.zs && q >= 1 && q <= M - 1 && lane >= 1 && lane <= TX / 2) {
        const int qA = (yA + q) & 1;   // red column of row A (row B: 1 - qA)
        const T *g = gptr<T>(gring, q, 2 * w, lane);
        T sA, sB;
        if (qA == 0) {
          // row A red at col 0: i+1 own col 1, i-1 lane-1; row B red at col 1: i+1 lane+1, i-1 own col 0
          const T xmA = g[-1], xpB = g[GS + 1], ymA = g[-GS], ypB = g[2 * GS];
          T t1 = (T)6 * S.r1[0][0];
          t1 = t1 + S.r1[0][1];
          t1 = t1 + xmA;
          t1 = t1 + S.r1[1][0];
          t1 = t1 + ymA;
          t1 = t1 + rn[0][0];
          t1 = t1 + S.r0[0][0];
          sA = t1 * (T)(1.0 / 12.0);
          T t2 = (T)6 * S.r1[1][1];
          t2 = t2 + xpB;
          t2 = t2 + S.r1[1][0];
          t2 = t2 + ypB;
          t2 = t2 + S.r1[0][1];
          t2 = t2 + rn[1][1];
          t2 = t2 + S.r0[1][1];
          sB = t2 * (T)(1.0 / 12.0);
        } else {
          // row A red at col 1: i+1 lane+1, i-1 own col 0; row B red at col 0: i+1 own col 1, i-1 lane-1
          const T xpA = g[1], xmB = g[GS - 1], ymA = g[-GS], ypB = g[2 * GS];
          T t1 = (T)6 * S.r1[0][1];
          t1 = t1 + xpA;
          t1 = t1 + S.r1[0][0];
          t1 = t1 + S.r1[1][1];
          t1 = t1 + ymA;
          t1 = t1 + rn[0][1];
          t1 = t1 + S.r0[0][1];
          sA = t1 * (T)(1.0 / 12.0);
          T t2 = (T)6 * S.r1[1][0];
          t2 = t2 + S.r1[1][1];
          t2 = t2 + xmB;
          t2 = t2 + ypB;
          t2 = t2 + S.r1[0][0];
          t2 = t2 + rn[1][0];
          t2 = t2 + S.r0[1][0];
          sB = t2 * (T)(1.0 / 12.0);
        }
        const int hx = xl >> 1;
        const int64_t zoff = (int64_t)(q >> 1) * P.out.plane;
        // row A: x = xl + qA; row B: x = xl + 1 - qA
        if (w >= 1 && yA <= M - 1 && yA >= 1 && xl + qA <= M - 1 && xl + qA >= 1) {
          const int sl = qA | ((yA & 1) << 1) | ((q & 1) << 2);
          P.out.s[sl][zoff + (int64_t)(yA >> 1) * P.out.pitch + hx] = sA;
        }
        const int yB = yA + 1, xb = xl + 1 - qA;
        if (w <= 14 && yB <= M - 1 && yB >= 1 && xb <= M - 1 && xb >= 1) {
          const int sl = (1 - qA) | ((yB & 1) << 1) | ((q & 1) << 2);
          P.out.s[sl][zoff + (int64_t)(yB >> 1) * P.out.pitch + hx] = sB;
        }
      }
#pragma unroll
      for (int r = 0; r < 2; r++)
#pragma unroll
        for (int c = 0; c < 2; c++) {
          S.r0[r][c] = S.r1[r][c];
          S.r1[r][c] = rn[r][c];
        }
    }
#pragma unroll
    for (int r = 0; r < 2; r++)
#pragma unroll
      for (int c = 0; c < 2; c++) {
        S.um[r][c] = S.uc[r][c];
        S.uc[r][c] = un[r][c];
      }
  }
  static __device__ void finish(const Params &P, State &S) { block_norm_push<NT>(P.ns, S.mx); }
};

// ================================================== finest ascent a15 (s = 1)
// Step j: r(j-1) at the 4 own nodes; Egprolg at the green node of
// each own row of plane j-1 (red neighbours from v_R(j-1) in shared memory,
// v_R(j), v_R(j-2) own); then Egprolr at the red nodes of plane
// q = j-2 from the green values, and u_new = u_old + v there.
template <class T>
struct OpAsc3P {
  using Gm = Geo<T>;
  static constexpr int NS = sizeof(T) == 8 ? 4 : 7;
  static constexpr int U_OFF = 0, F_OFF = al128(Gm::U_BYTES), V0_OFF = F_OFF + al128(Gm::F_BYTES),
                       V1_OFF = V0_OFF + al128(Gm::V_BYTES), SLOT = al128(V1_OFF + Gm::V_BYTES);
  static constexpr int SMEM = NS * SLOT + 3 * Gm::GPL;
  struct Params {
    CUtensorMap tu, tf, tv[4];   // red sublattices C, Fx, Fy, Fz of v_R(1)
    D3<T> out;
    Sched sc;
    int M, fz0, hz0;
    T c, invh2;
  };
  struct State {
    T um[2][2], uc[2][2];   // own u(j-2), u(j-1)
    T r1[2][2];             // own r(j-2)
    T g0[2], g1[2];         // own green v of planes j-3, j-2 (one per row)
    T vr0[2], vr1[2];       // own v_R of planes j-2, j-1 (at the green column of the plane below)
  };
  static __device__ void prefetch(const Params &P) {
    tma_prefetch_desc(&P.tu);
    tma_prefetch_desc(&P.tf);
    for (int i = 0; i < 4; i++) tma_prefetch_desc(&P.tv[i]);
  }
  static __device__ void init(State &) {}
  static __device__ __forceinline__ int vx0(int x0) { return (x0 / 2 - 2) & ~(Gm::AL - 1); }
  static __device__ void issue(const Params &P, const Item &it, int j, unsigned char *slot, uint64_t *bar) {
    const bool wf = j >= it.zs;
    mbar_expect_tx(bar, Gm::U_BYTES + 2 * Gm::V_BYTES + (wf ? Gm::F_BYTES : 0));
    tma_load_3d(slot + U_OFF, &P.tu, it.x0 - Gm::UXO, it.y0 - 2, j - P.fz0, bar);
    if (wf) tma_load_3d(slot + F_OFF, &P.tf, it.x0 - 2, it.y0 - 1, j - 1 - P.fz0, bar);
    // red nodes of fine plane j: even j -> C (even x), Fz (odd x); odd j -> Fx (even x), Fy (odd x)
    const int hz = j >> 1;
    const CUtensorMap *m0 = (j & 1) ? &P.tv[1] : &P.tv[0];
    const CUtensorMap *m1 = (j & 1) ? &P.tv[2] : &P.tv[3];
    tma_load_3d(slot + V0_OFF, m0, vx0(it.x0), it.y0 / 2 - 1, hz - P.hz0, bar);
    tma_load_3d(slot + V1_OFF, m1, vx0(it.x0), it.y0 / 2 - 1, hz - P.hz0, bar);
  }
  static __device__ __forceinline__ T jac6(T c, T r, T v0, T v1, T v2, T v3, T v4, T v5) {
    T t = -(c * r);
    t = t + v0;
    t = t + v1;
    t = t + v2;
    t = t + v3;
    t = t + v4;
    t = t + v5;
    return t * (T)(1.0 / 6.0);
  }
  static __device__ __forceinline__ void step(const Params &P, State &S, const Item &it, int j, unsigned char *Lc,
                                              unsigned char *Lp, unsigned char *gring) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, M = P.M;
    const int xl = it.x0 - 2 + 2 * lane, yA = it.y0 - 1 + 2 * w;
    const int uo = (2 * w + 1) * Gm::UW + 2 * lane - 2 + Gm::UXO;
    const int fo = 2 * w * Gm::FW + 2 * lane;
    const int vxo = vx0(it.x0), vyo = it.y0 / 2 - 1;
    const int z = j - 1;
    // green column of plane z in row A (row B: the other one); red column = 1 - that
    const int gA = 1 - ((yA + z) & 1);
    T un[2][2];
    {
      const T *U = (const T *)(Lc + U_OFF);
      ld2(U + uo, un[0][0], un[0][1]);
      ld2(U + uo + Gm::UW, un[1][0], un[1][1]);
    }
    // own v_R(j) at the green column of plane j-1 (x = xl + gA / xl + 1 - gA; half index xl/2)
    T vrn[2];
    {
      const int ho = (yA >> 1) - vyo, hb = ((yA + 1) >> 1) - vyo, hx = (xl >> 1) - vxo;
      const T *V0 = (const T *)(Lc + V0_OFF), *V1 = (const T *)(Lc + V1_OFF);
      vrn[0] = (gA ? V1 : V0)[ho * Gm::VW + hx];
      vrn[1] = (gA ? V0 : V1)[hb * Gm::VW + hx];
    }
    if (j >= it.zs) {
      const T *U = (const T *)(Lp + U_OFF) + uo;
      const T *F = (const T *)(Lc + F_OFF) + fo;
      T ymA0, ymA1, ypB0, ypB1, t, lA, rA, lB, rB, fA0, fA1, fB0, fB1;
      ld2(U - Gm::UW, ymA0, ymA1);
      ld2(U + 2 * Gm::UW, ypB0, ypB1);
      ld2(U - 2, t, lA);
      ld2(U + 2, rA, t);
      ld2(U + Gm::UW - 2, t, lB);
      ld2(U + Gm::UW + 2, rB, t);
      ld2(F, fA0, fA1);
      ld2(F + Gm::FW, fB0, fB1);
      const T h = P.invh2;
      T rn[2][2];
      rn[0][0] = res7(S.uc[0][0], S.uc[0][1], lA, S.uc[1][0], ymA0, un[0][0], S.um[0][0], fA0, h);
      rn[0][1] = res7(S.uc[0][1], rA, S.uc[0][0], S.uc[1][1], ymA1, un[0][1], S.um[0][1], fA1, h);
      rn[1][0] = res7(S.uc[1][0], S.uc[1][1], lB, ypB0, S.uc[0][0], un[1][0], S.um[1][0], fB0, h);
      rn[1][1] = res7(S.uc[1][1], rB, S.uc[1][0], ypB1, S.uc[0][1], un[1][1], S.um[1][1], fB1, h);
      // ---- Egprolg at the green node of rows A, B of plane z
      const bool zin = z >= 1 && z <= M - 1;
      T gn[2];
      {
        const T *V0 = (const T *)(Lp + V0_OFF), *V1 = (const T *)(Lp + V1_OFF);   // v_R(z)
        const int hx = (xl >> 1) - vxo;
#pragma unroll
        for (int R = 0; R < 2; R++) {
          const int y = yA + R, gc = R ? 1 - gA : gA, xg = xl + gc;
          const int hy = (y >> 1) - vyo;
          // x neighbours xg +- 1 have parity 1 - gc; y neighbours parity gc
          const T *VX = gc ? V0 : V1, *VY = gc ? V1 : V0;
          T xp, xm;
          if (gc) {   // xg odd: xg+1 -> half hx+1, xg-1 -> hx
            xp = VX[hy * Gm::VW + hx + 1];
            xm = VX[hy * Gm::VW + hx];
          } else {    // xg even: xg+1 -> hx, xg-1 -> hx-1
            xp = VX[hy * Gm::VW + hx];
            xm = VX[hy * Gm::VW + hx - 1];
          }
          const T yp = VY[(((y + 1) >> 1) - vyo) * Gm::VW + hx];
          const T ym = VY[(((y - 1) >> 1) - vyo) * Gm::VW + hx];
          const T r = gc ? rn[R][1] : rn[R][0];
          const bool in = zin && y >= 1 && y <= M - 1 && xg >= 1 && xg <= M - 1;
          gn[R] = in ? jac6(P.c, r, xp, xm, yp, ym, vrn[R], S.vr0[R]) : (T)0;
        }
      }
      *gptr<T>(gring, z, 2 * w, lane) = gn[0];
      *gptr<T>(gring, z, 2 * w + 1, lane) = gn[1];
      // ---- Egprolr at the red nodes of q = j-2, then u_new = u_old + v
      const int q = j - 2;
      if (q >= it.zs && q >= 1 && q <= M - 1 && lane >= 1 && lane <= TX / 2) {
        // red column of row A at plane q = green column of row A at plane z = gA
        const T *g = gptr<T>(gring, q, 2 * w, lane);
        const T ymA = g[-GS], ypB = g[2 * GS];
        T vA, vB;
        if (gA == 0) {
          // row A red col 0: i+1 own green (col 1), i-1 lane-1; row B red col 1: i+1 lane+1, i-1 own green
          vA = jac6(P.c, S.r1[0][0], S.g1[0], g[-1], S.g1[1], ymA, gn[0], S.g0[0]);
          vB = jac6(P.c, S.r1[1][1], g[GS + 1], S.g1[1], ypB, S.g1[0], gn[1], S.g0[1]);
        } else {
          vA = jac6(P.c, S.r1[0][1], g[1], S.g1[0], S.g1[1], ymA, gn[0], S.g0[0]);
          vB = jac6(P.c, S.r1[1][0], S.g1[1], g[GS - 1], ypB, S.g1[0], gn[1], S.g0[1]);
        }
        // u_new = u(q) + v: u(q) = S.um; row A: red col gA, green col 1-gA
        const T a0 = S.um[0][0] + (gA ? S.g1[0] : vA), a1 = S.um[0][1] + (gA ? vA : S.g1[0]);
        const T b0 = S.um[1][0] + (gA ? vB : S.g1[1]), b1 = S.um[1][1] + (gA ? S.g1[1] : vB);
        const bool k0 = xl >= 1 && xl <= M - 1, k1 = xl + 1 >= 1 && xl + 1 <= M - 1;
        T *dst = &P.out(xl, yA, q);
        if (w >= 1 && yA >= 1 && yA <= M - 1) {
          if (k0 && k1) st2(dst, a0, a1);
          else {
            if (k0) dst[0] = a0;
            if (k1) dst[1] = a1;
          }
        }
        dst += P.out.pitch;
        if (w <= 14 && yA + 1 >= 1 && yA + 1 <= M - 1) {
          if (k0 && k1) st2(dst, b0, b1);
          else {
            if (k0) dst[0] = b0;
            if (k1) dst[1] = b1;
          }
        }
      }
#pragma unroll
      for (int R = 0; R < 2; R++) {
        S.g0[R] = S.g1[R];
        S.g1[R] = gn[R];
#pragma unroll
        for (int c = 0; c < 2; c++) S.r1[R][c] = rn[R][c];
      }
    }
#pragma unroll
    for (int R = 0; R < 2; R++) {
      S.vr0[R] = S.vr1[R];
      S.vr1[R] = vrn[R];
#pragma unroll
      for (int c = 0; c < 2; c++) {
        S.um[R][c] = S.uc[R][c];
        S.uc[R][c] = un[R][c];
      }
    }
  }
  static __device__ void finish(const Params &, State &) {}
};

// ================================================================= launch
template <class Op>
static cudaError_t run_zpipe(typename Op::Params &P, int M, int zlo, int zhi, cudaStream_t st) {
  if (zhi <= zlo) return cudaSuccess;
  cudaError_t e = cudaFuncSetAttribute(zpipe<Op>, cudaFuncAttributeMaxDynamicSharedMemorySize, Op::SMEM);
  if (e != cudaSuccess) return e;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  P.sc.ntx = (M + 1) / TX + 1;   // tiles start at x0 = 60 t - 2; outputs x = 1 .. M-1
  const int nty = (M + TY - 1) / TY;
  P.sc.T = P.sc.ntx * nty;
  P.sc.zlo = zlo;
  P.sc.zhi = zhi;
  const int Z = zhi - zlo;
  int grid = sms;
  if ((long long)P.sc.T * Z < grid) grid = (int)((long long)P.sc.T * Z);
  zpipe<Op><<<grid, NT, Op::SMEM, st>>>(P);
  return cudaGetLastError();
}

template <class T>
static bool tmap3(CUtensorMap *tm, const T *p, int64_t nx, int64_t ny, int64_t nz, int64_t pitch, int64_t plane, int bx,
                  int by) {
  uint64_t dims[3] = {(uint64_t)nx, (uint64_t)ny, (uint64_t)nz};
  uint32_t box[3] = {(uint32_t)bx, (uint32_t)by, 1};
  return encode_tmap(tm, p, sizeof(T), 3, dims, (uint64_t)pitch, (uint64_t)plane, box);
}

template <class T>
cudaError_t fast3p_desc_fine(const T *u, const T *f, int64_t pitch, const S3<T> &rr, int M, const Coef<T> &k,
                             const NormSink &ns, cudaStream_t st, const ZRange3 &pz) {
  using Op = OpDesc3P<T>;
  using Gm = Geo<T>;
  typename Op::Params P{};
  const int64_t n = M + 1, plane = pitch * n, nz = pz.fplanes < 0 ? n : pz.fplanes;
  if (!tmap3<T>(&P.tu, u + (int64_t)pz.fz0 * plane, n, n, nz, pitch, plane, Gm::UW, Gm::UH) ||
      !tmap3<T>(&P.tf, f + (int64_t)pz.fz0 * plane, n, n, nz, pitch, plane, Gm::FW, Gm::FH))
    return cudaErrorInvalidValue;
  P.out = rr;
  P.M = M;
  P.fz0 = pz.fz0;
  P.invh2 = k.invh2;
  P.ns = ns;
  return run_zpipe<Op>(P, M, pz.zlo, pz.zhi < 0 ? M : pz.zhi, st);
}

template <class T>
cudaError_t fast3p_asc_fine(const S3<T> &vr, const T *u_old, const T *f, int64_t pitch, T *u_new, int M, T c,
                            const Coef<T> &k, cudaStream_t st, const ZRange3 &pz) {
  using Op = OpAsc3P<T>;
  using Gm = Geo<T>;
  typename Op::Params P{};
  const int64_t n = M + 1, plane = pitch * n, nz = pz.fplanes < 0 ? n : pz.fplanes;
  if (!tmap3<T>(&P.tu, u_old + (int64_t)pz.fz0 * plane, n, n, nz, pitch, plane, Gm::UW, Gm::UH) ||
      !tmap3<T>(&P.tf, f + (int64_t)pz.fz0 * plane, n, n, nz, pitch, plane, Gm::FW, Gm::FH))
    return cudaErrorInvalidValue;
  const int sub[4] = {0, 6, 5, 3};   // C, Fx, Fy, Fz
  const int64_t H = M / 2 + 1, hpl = pz.hplanes < 0 ? H : pz.hplanes;
  for (int i = 0; i < 4; i++)
    if (!tmap3<T>(&P.tv[i], vr.s[sub[i]] + (int64_t)pz.hz0 * vr.plane, H, H, hpl, vr.pitch, vr.plane, Gm::VW, Gm::VH))
      return cudaErrorInvalidValue;
  P.out = D3<T>{u_new, pitch, plane};
  P.M = M;
  P.fz0 = pz.fz0;
  P.hz0 = pz.hz0;
  P.c = c;
  P.invh2 = k.invh2;
  return run_zpipe<Op>(P, M, pz.zlo, pz.zhi < 0 ? M : pz.zhi, st);
}

template cudaError_t fast3p_desc_fine<double>(const double *, const double *, int64_t, const S3<double> &, int,
                                              const Coef<double> &, const NormSink &, cudaStream_t, const ZRange3 &);
template cudaError_t fast3p_desc_fine<float>(const float *, const float *, int64_t, const S3<float> &, int,
                                             const Coef<float> &, const NormSink &, cudaStream_t, const ZRange3 &);
template cudaError_t fast3p_asc_fine<double>(const S3<double> &, const double *, const double *, int64_t, double *, int,
                                             double, const Coef<double> &, cudaStream_t, const ZRange3 &);
template cudaError_t fast3p_asc_fine<float>(const S3<float> &, const float *, const float *, int64_t, float *, int,
                                            float, const Coef<float> &, cudaStream_t, const ZRange3 &);

}  // namespace mg
