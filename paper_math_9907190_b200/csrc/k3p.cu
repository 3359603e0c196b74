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
#include "ops3.cuh"
#include "zpipe.cuh"

namespace mg {

// own-node interior masks of an item (x: columns xl, xl+1; y: rows yA, yA+1)
struct Masks {
  bool full;             // every own node of every thread is interior in x and y
  bool c0, c1, rA, rB;   // this thread's columns / rows interior
};
template <int NW>
__device__ __forceinline__ Masks item_masks(const Item &it, int M, int xl, int yA) {
  Masks m;
  m.full = it.x0 - 2 >= 1 && it.x0 + 61 <= M - 1 && it.y0 - 1 >= 1 && it.y0 + 2 * NW - 2 <= M - 1;
  m.c0 = xl >= 1 && xl <= M - 1;
  m.c1 = xl + 1 >= 1 && xl + 1 <= M - 1;
  m.rA = yA >= 1 && yA <= M - 1;
  m.rB = yA + 1 >= 1 && yA + 1 <= M - 1;
  return m;
}

// exact max of |r| as the bit pattern of a non-negative double (NaN-safe:
// NaN patterns sort above +inf, so a diverged residual is never lost)
template <class T>
__device__ __forceinline__ unsigned long long absbits(T v) {
  return (unsigned long long)__double_as_longlong((double)v) & 0x7fffffffffffffffull;
}
__device__ __forceinline__ unsigned long long umax64(unsigned long long a, unsigned long long b) { return a > b ? a : b; }

template <class T>
__device__ __forceinline__ void sel0(T &v, bool keep) {
  v = keep ? v : (T)0;
}

// Efos4 at the thread's 4 nodes (rows yA, yA+1 x columns xl,
// xl+1) of plane z from the u boxes of planes z-1 (Uq), z (Up), z+1 (Uc),
// each offset to (xl, yA); F: f~ at the 4 nodes.  Operand order of res3v
// (ops3.cuh), so bit-identical to the oracle's res3d_o4.
template <class T, int UW>
__device__ __forceinline__ void res19_block(const T *Uq, const T *Up, const T *Uc, const T (&F)[2][2],
                                            const Coef<T> &k, T (&rn)[2][2]) {
  T P[4][4], Zp[4][4], Zm[4][4], t;   // [row yA-1 .. yA+2][col xl-1 .. xl+2]
#pragma unroll
  for (int r = 0; r < 4; r++) {
    const T *q = Up + (r - 1) * UW;
    ld2(q - 2, t, P[r][0]);
    ld2(q, P[r][1], P[r][2]);
    ld2(q + 2, P[r][3], t);
  }
#pragma unroll
  for (int r = 0; r < 4; r++) {
    const T *c = Uc + (r - 1) * UW, *m = Uq + (r - 1) * UW;
    ld2(c, Zp[r][1], Zp[r][2]);
    ld2(m, Zm[r][1], Zm[r][2]);
    if (r == 1 || r == 2) {
      ld2(c - 2, t, Zp[r][0]);
      ld2(c + 2, Zp[r][3], t);
      ld2(m - 2, t, Zm[r][0]);
      ld2(m + 2, Zm[r][3], t);
    }
  }
#pragma unroll
  for (int R = 0; R < 2; R++)
#pragma unroll
    for (int C = 0; C < 2; C++) {
      const int a = R + 1, b = C + 1;
      Nb19<T> q;
      q.c = P[a][b];
      q.xp = P[a][b + 1];
      q.xm = P[a][b - 1];
      q.yp = P[a + 1][b];
      q.ym = P[a - 1][b];
      q.zp = Zp[a][b];
      q.zm = Zm[a][b];
      q.xpyp = P[a + 1][b + 1];
      q.xmyp = P[a + 1][b - 1];
      q.xmym = P[a - 1][b - 1];
      q.xpym = P[a - 1][b + 1];
      q.ypzp = Zp[a + 1][b];
      q.ypzm = Zm[a + 1][b];
      q.ymzm = Zm[a - 1][b];
      q.ymzp = Zp[a - 1][b];
      q.xpzp = Zp[a][b + 1];
      q.xmzp = Zp[a][b - 1];
      q.xmzm = Zm[a][b - 1];
      q.xpzm = Zm[a][b + 1];
      rn[R][C] = res3v<T, 4>(q, F[R][C], k);
    }
}

// =================================================== finest descent a9 + a10
// Step j: r(j-1) at the thread's 4 nodes (registers; the green ones also to
// the ring); then Erred at the red nodes of plane q = j-2.
// Parities (yA odd, xl even): the red column of row A at plane z is (z+1) & 1,
// i.e. PH at z = j-1 and Q = 1-PH at q = j-2; row B the other way round.
// FINE = false: the same pass one octave down (G(s) -> R(s), s > 1): r is
// read from the dense level array (the "f" box) instead of computed, no norm.
// ORDER = 4 (FINE only): Efos4 with f~; the u boxes of three planes are read
// (KEEP = 3 ring slots), everything else is the order-2 pass.
template <class T, bool FINE = true, int NW_ = 16, int NSO = 0, bool UNIF = true, int ORDER = 2>
struct OpDesc3P {
  using Gm = Geo<T, NW_>;
  static_assert(ORDER == 2 || FINE, "order 4 on the finest level only");
  static constexpr int NW = NW_, NTH = Gm::NTH, MINB = NW <= 8 ? 2 : 1, KEEP = ORDER == 4 ? 3 : 2;
  static constexpr int NS = NSO ? NSO : FINE ? (sizeof(T) == 8 ? 5 : 8) : 8, GPL = Gm::GPL, PRO = FINE ? 2 : 0, EPI = 2;
  static constexpr int U_OFF = 0, F_OFF = FINE ? al128(Gm::U_BYTES) : 0, SLOT = al128(F_OFF + Gm::F_BYTES);
  static constexpr int SMEM = NS * SLOT + 3 * Gm::GPL;
  struct Params {
    CUtensorMap tu, tf;
    S3<T> out;
    Sched sc;
    int M, fz0;
    T invh2;
    NormSink ns;
    Coef<T> k;   // order 4: c6
  };
  struct State {
    T u[2][2][2];   // [z & 1][row A/B][col 0/1]: own u of the two latest planes
    T r[2][2][2];   // own r of the two latest planes
    unsigned long long mx;
    double ss;      // sum r^2 over the tile's core nodes (a16 L2 norm)
  };
  struct Ctx {
    Masks m;
    bool oA[2], oB[2];   // Erred output at row A / B, by PH
    bool sA, sB;         // row A / B of this lane lies in the tile's core (counted once in the L2 sum)
    int64_t bA, bB;      // sublattice offsets (y >> 1) * pitch + (xl >> 1) of rows A, B
  };
  static __device__ void prefetch(const Params &P) {
    if (FINE) tma_prefetch_desc(&P.tu);
    tma_prefetch_desc(&P.tf);
  }
  static __device__ void init(State &S) {
    S.mx = 0ull;
    S.ss = 0.0;
  }
  static __device__ void begin(const Params &P, Ctx &C, const Item &it) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int xl = it.x0 - 2 + 2 * lane, yA = it.y0 - 1 + 2 * w;
    C.m = item_masks<NW>(it, P.M, xl, yA);
    const bool lk = lane >= 1 && lane <= TX / 2;
    // PH = 0: row A red at col 1, row B at col 0; PH = 1: the other way round
    C.oA[0] = lk && w >= 1 && C.m.rA && C.m.c1;
    C.oA[1] = lk && w >= 1 && C.m.rA && C.m.c0;
    C.oB[0] = lk && w <= NW - 2 && C.m.rB && C.m.c0;
    C.oB[1] = lk && w <= NW - 2 && C.m.rB && C.m.c1;
    C.sA = lk && w >= 1;
    C.sB = lk && w <= NW - 2;
    C.bA = (int64_t)(yA >> 1) * P.out.pitch + (xl >> 1);
    C.bB = (int64_t)((yA + 1) >> 1) * P.out.pitch + (xl >> 1);
  }
  static __device__ void issue(const Params &P, const Item &it, int j, unsigned char *slot, uint64_t *bar) {
    const bool wf = j >= it.zs;
    mbar_expect_tx(bar, (FINE ? Gm::U_BYTES : 0) + (wf ? Gm::F_BYTES : 0));
    if (FINE) tma_load_3d(slot + U_OFF, &P.tu, it.x0 - Gm::UXO, it.y0 - 2, j - P.fz0, bar);
    if (wf) tma_load_3d(slot + F_OFF, &P.tf, it.x0 - 2, it.y0 - 1, j - 1 - P.fz0, bar);
  }
  template <int PH>
  static __device__ __forceinline__ void step(const Params &P, State &S, const Ctx &C, const Item &it, int j,
                                              unsigned char *Lc, unsigned char *Lp, unsigned char *gz,
                                              unsigned char *gq, unsigned char *gr) {
    step_o<PH>(P, S, C, it, j, Lc, Lp, nullptr, gz, gq, gr);
  }
  template <int PH>
  static __device__ __forceinline__ void step(const Params &P, State &S, const Ctx &C, const Item &it, int j,
                                              unsigned char *Lc, unsigned char *Lp, unsigned char *Lq,
                                              unsigned char *gz, unsigned char *gq, unsigned char *gr) {
    step_o<PH>(P, S, C, it, j, Lc, Lp, Lq, gz, gq, gr);
  }
  template <int PH>
  static __device__ __forceinline__ void step_o(const Params &P, State &S, const Ctx &C, const Item &it, int j,
                                                unsigned char *Lc, unsigned char *Lp, unsigned char *Lq,
                                                unsigned char *gz, unsigned char *gq, unsigned char *) {
    constexpr int Q = PH ^ 1;   // slot of planes j-1, j-3
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, M = P.M;
    const int uo = (2 * w + 1) * Gm::UW + 2 * lane - 2 + Gm::UXO;   // u box offset of (xl, yA)
    const int fo = 2 * w * Gm::FW + 2 * lane;                         // f box offset of (xl, yA)
    T un[2][2];
    if (FINE) {
      const T *U = (const T *)(Lc + U_OFF);
      ld2(U + uo, un[0][0], un[0][1]);
      ld2(U + uo + Gm::UW, un[1][0], un[1][1]);
    }
    if (j >= it.zs) {
      T rn[2][2];
      const int z = j - 1;
      if constexpr (!FINE) {
        const T *F = (const T *)(Lc + F_OFF) + fo;   // r(z) from the level array (zero outside the interior)
        ld2(F, rn[0][0], rn[0][1]);
        ld2(F + Gm::FW, rn[1][0], rn[1][1]);
      } else {
      // ---- r(z), z = j-1: centre u(j-1) = S.u[Q], z-1 = S.u[PH] (u(j-2)), z+1 = un
      const T(&uc)[2][2] = S.u[Q];
      const T(&um)[2][2] = S.u[PH];
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
      if constexpr (ORDER == 4) {   // Efos4 from the u boxes of planes z-1, z, z+1
        const T Fv[2][2] = {{fA0, fA1}, {fB0, fB1}};
        res19_block<T, Gm::UW>((const T *)(Lq + U_OFF) + uo, U, (const T *)(Lc + U_OFF) + uo, Fv, P.k, rn);
      } else {
      const T h = P.invh2;
      // i+1, i-1, j+1, j-1, k+1, k-1
      rn[0][0] = res7(uc[0][0], uc[0][1], lA, uc[1][0], ymA0, un[0][0], um[0][0], fA0, h);
      rn[0][1] = res7(uc[0][1], rA, uc[0][0], uc[1][1], ymA1, un[0][1], um[0][1], fA1, h);
      rn[1][0] = res7(uc[1][0], uc[1][1], lB, ypB0, uc[0][0], un[1][0], um[1][0], fB0, h);
      rn[1][1] = res7(uc[1][1], rB, uc[1][0], ypB1, uc[0][1], un[1][1], um[1][1], fB1, h);
      }
      const bool zin = z >= 1 && z <= M - 1;
      if (!(C.m.full && zin)) {
        sel0(rn[0][0], zin && C.m.rA && C.m.c0);
        sel0(rn[0][1], zin && C.m.rA && C.m.c1);
        sel0(rn[1][0], zin && C.m.rB && C.m.c0);
        sel0(rn[1][1], zin && C.m.rB && C.m.c1);
      }
      // every computed r is a true residual (or 0): max over all of them (only
      // when a residual history is wanted: the pass is instruction-bound)
      if (P.ns.slots)
        S.mx = umax64(S.mx, umax64(umax64(absbits(rn[0][0]), absbits(rn[0][1])),
                                   umax64(absbits(rn[1][0]), absbits(rn[1][1]))));
      if (z >= it.zs && z < it.ze && P.ns.sums(z)) {   // the sum counts the core nodes once
        if (C.sA) S.ss += sq((double)rn[0][0]) + sq((double)rn[0][1]);
        if (C.sB) S.ss += sq((double)rn[1][0]) + sq((double)rn[1][1]);
      }
      }
      // greens of plane z to the ring: red column of row A at z is PH, so its
      // green is column Q; row B (even y) the other way round
      {
        T *g = (T *)gz + (2 * w + 1) * GS + (lane + 1);
        g[0] = rn[0][Q];
        g[GS] = rn[1][PH];
      }
      // ---- Erred at the red nodes of q = j-2: r(q-1) = S.r[Q], r(q) = S.r[PH], r(q+1) = rn.
      // Red column of row A at q is Q, of row B is PH.
      const int q = j - 2;
      // warp-uniform condition only: the lanes without an output compute too and
      // skip the stores (a lane-dependent branch here cost a divergence region per step)
      if (q >= it.zs && q >= 1 && q <= M - 1 && (UNIF || C.oA[PH] || C.oB[PH])) {
        const T(&R1)[2][2] = S.r[PH];
        const T(&R0)[2][2] = S.r[Q];
        const T *g = (const T *)gq + (2 * w + 1) * GS + (lane + 1);
        const T ymA = g[-GS], ypB = g[2 * GS];
        T sA, sB;
        if (Q == 0) {
          // row A red at col 0: i+1 own col 1, i-1 lane-1; row B red at col 1: i+1 lane+1, i-1 own col 0
          T t1 = (T)6 * R1[0][0];
          t1 = t1 + R1[0][1];
          t1 = t1 + g[-1];
          t1 = t1 + R1[1][0];
          t1 = t1 + ymA;
          t1 = t1 + rn[0][0];
          t1 = t1 + R0[0][0];
          sA = t1 * (T)(1.0 / 12.0);
          T t2 = (T)6 * R1[1][1];
          t2 = t2 + g[GS + 1];
          t2 = t2 + R1[1][0];
          t2 = t2 + ypB;
          t2 = t2 + R1[0][1];
          t2 = t2 + rn[1][1];
          t2 = t2 + R0[1][1];
          sB = t2 * (T)(1.0 / 12.0);
        } else {
          // row A red at col 1: i+1 lane+1, i-1 own col 0; row B red at col 0: i+1 own col 1, i-1 lane-1
          T t1 = (T)6 * R1[0][1];
          t1 = t1 + g[1];
          t1 = t1 + R1[0][0];
          t1 = t1 + R1[1][1];
          t1 = t1 + ymA;
          t1 = t1 + rn[0][1];
          t1 = t1 + R0[0][1];
          sA = t1 * (T)(1.0 / 12.0);
          T t2 = (T)6 * R1[1][0];
          t2 = t2 + R1[1][1];
          t2 = t2 + g[GS - 1];
          t2 = t2 + ypB;
          t2 = t2 + R1[0][0];
          t2 = t2 + rn[1][0];
          t2 = t2 + R0[1][0];
          sB = t2 * (T)(1.0 / 12.0);
        }
        // sublattice (x&1 | (y&1)<<1 | (q&1)<<2): row A (odd y) x&1 = Q; row B (even y) x&1 = PH
        const int64_t zoff = (int64_t)(q >> 1) * P.out.plane;
        // streaming stores: r_R(1) is not re-read in this pass, keep L2 for the halos
        if (C.oA[PH]) __stcs(&P.out.s[Q | 2 | (PH << 2)][zoff + C.bA], sA);
        if (C.oB[PH]) __stcs(&P.out.s[PH | (PH << 2)][zoff + C.bB], sB);
      }
#pragma unroll
      for (int r = 0; r < 2; r++)
#pragma unroll
        for (int c = 0; c < 2; c++) S.r[Q][r][c] = rn[r][c];
    }
    if (FINE) {
#pragma unroll
      for (int r = 0; r < 2; r++)
#pragma unroll
        for (int c = 0; c < 2; c++) S.u[PH][r][c] = un[r][c];
    }
  }
  static __device__ void finish(const Params &P, State &S) {
    if (FINE) block_norm_push<NTH>(P.ns, __longlong_as_double((long long)S.mx), S.ss);
  }
};

// ================================================== finest ascent a15 (s = 1)
// Step j: r(j-1) at the 4 own nodes; Egprolg at the green node of
// each own row of plane z = j-1 (red neighbours from v_R(z) in shared memory,
// v_R(z+1), v_R(z-1) own); then Egprolr at the red nodes of plane
// q = j-2 from the green values, and u_new = u_old + v there.
// Green column of row A at plane z = j-1 is Q = 1-PH (row B: PH); the red
// column of row A at plane q = j-2 is Q as well.
// FINE = false: Egprolg/Egprolr one octave down (G(s) from R(s), s > 1): r is
// read from the dense level array (the "f" box) and v_G(s) is written.
template <class T, bool FINE = true, int NW_ = 16, int NSO = 0, bool UNIF = true, int ORDER = 2>
struct OpAsc3P {
  using Gm = Geo<T, NW_>;
  static_assert(ORDER == 2 || FINE, "order 4 on the finest level only");
  static constexpr int NW = NW_, NTH = Gm::NTH, MINB = NW <= 8 ? 2 : 1, KEEP = ORDER == 4 ? 3 : 2;
  static constexpr int NS = NSO ? NSO : FINE ? (sizeof(T) == 8 ? 4 : 7) : (sizeof(T) == 8 ? 7 : 10), GPL = Gm::GPL,
                       PRO = 2, EPI = 2;
  static constexpr int U_OFF = 0, F_OFF = FINE ? al128(Gm::U_BYTES) : 0, V0_OFF = F_OFF + al128(Gm::F_BYTES),
                       V1_OFF = V0_OFF + al128(Gm::V_BYTES), SLOT = al128(V1_OFF + Gm::V_BYTES);
  static constexpr int SMEM = NS * SLOT + 3 * Gm::GPL;
  struct Params {
    CUtensorMap tu, tf, tv[4];   // red sublattices C, Fx, Fy, Fz of v_R(1)
    D3<T> out;
    Sched sc;
    int M, fz0, hz0;
    T c, invh2;
    Coef<T> k;   // order 4: c6
  };
  struct State {
    T u[2][2][2];   // [z & 1][row][col] own u
    T rq[2];        // own r(j-2) at the red node of rows A, B
    T g[2][2];      // [z & 1][row] own green v
    T vr[2][2];     // [z & 1][row] own v_R(z) at the green column of plane z-1
  };
  struct Ctx {
    Masks m;
    bool oA, oB;   // u_new rows written (lane, warp, y interior)
    int hx;        // half-index column of xl in the V boxes
  };
  static __device__ void prefetch(const Params &P) {
    if (FINE) tma_prefetch_desc(&P.tu);
    tma_prefetch_desc(&P.tf);
    for (int i = 0; i < 4; i++) tma_prefetch_desc(&P.tv[i]);
  }
  static __device__ void init(State &) {}
  static __device__ __forceinline__ int vx0(int x0) { return (x0 / 2 - 2) & ~(Gm::AL - 1); }
  static __device__ void begin(const Params &P, Ctx &C, const Item &it) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int xl = it.x0 - 2 + 2 * lane, yA = it.y0 - 1 + 2 * w;
    C.m = item_masks<NW>(it, P.M, xl, yA);
    const bool lk = lane >= 1 && lane <= TX / 2;
    C.oA = lk && w >= 1 && C.m.rA;
    C.oB = lk && w <= NW - 2 && C.m.rB;
    C.hx = (xl >> 1) - vx0(it.x0);
  }
  static __device__ void issue(const Params &P, const Item &it, int j, unsigned char *slot, uint64_t *bar) {
    const bool wf = j >= it.zs;
    mbar_expect_tx(bar, (FINE ? Gm::U_BYTES : 0) + 2 * Gm::V_BYTES + (wf ? Gm::F_BYTES : 0));
    if (FINE) tma_load_3d(slot + U_OFF, &P.tu, it.x0 - Gm::UXO, it.y0 - 2, j - P.fz0, bar);
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
  template <int PH>
  static __device__ __forceinline__ void step(const Params &P, State &S, const Ctx &C, const Item &it, int j,
                                              unsigned char *Lc, unsigned char *Lp, unsigned char *gz,
                                              unsigned char *gq, unsigned char *gr) {
    step_o<PH>(P, S, C, it, j, Lc, Lp, nullptr, gz, gq, gr);
  }
  template <int PH>
  static __device__ __forceinline__ void step(const Params &P, State &S, const Ctx &C, const Item &it, int j,
                                              unsigned char *Lc, unsigned char *Lp, unsigned char *Lq,
                                              unsigned char *gz, unsigned char *gq, unsigned char *gr) {
    step_o<PH>(P, S, C, it, j, Lc, Lp, Lq, gz, gq, gr);
  }
  template <int PH>
  static __device__ __forceinline__ void step_o(const Params &P, State &S, const Ctx &C, const Item &it, int j,
                                                unsigned char *Lc, unsigned char *Lp, unsigned char *Lq,
                                                unsigned char *gz, unsigned char *gq, unsigned char *) {
    constexpr int Q = PH ^ 1;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, M = P.M;
    const int uo = (2 * w + 1) * Gm::UW + 2 * lane - 2 + Gm::UXO;
    const int fo = 2 * w * Gm::FW + 2 * lane;
    T un[2][2];
    if (FINE) {
      const T *U = (const T *)(Lc + U_OFF);
      ld2(U + uo, un[0][0], un[0][1]);
      ld2(U + uo + Gm::UW, un[1][0], un[1][1]);
    }
    // own v_R(j) at the green column of plane j-1: row A col Q (parity Q -> V box Q), row B col PH
    // (V rows: half row of yA is w, of yA+1 is w+1 in the box)
    T vrn[2];
    {
      const T *VA = (const T *)(Lc + (Q ? V1_OFF : V0_OFF)), *VB = (const T *)(Lc + (PH ? V1_OFF : V0_OFF));
      vrn[0] = VA[w * Gm::VW + C.hx];
      vrn[1] = VB[(w + 1) * Gm::VW + C.hx];
    }
    if (j >= it.zs) {
      T rn[2][2];
      if constexpr (!FINE) {
        const T *F = (const T *)(Lc + F_OFF) + fo;   // r(j-1) from the level array
        ld2(F, rn[0][0], rn[0][1]);
        ld2(F + Gm::FW, rn[1][0], rn[1][1]);
      } else {
      const T(&uc)[2][2] = S.u[Q];
      const T(&um)[2][2] = S.u[PH];
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
      if constexpr (ORDER == 4) {
        const T Fv[2][2] = {{fA0, fA1}, {fB0, fB1}};
        res19_block<T, Gm::UW>((const T *)(Lq + U_OFF) + uo, U, (const T *)(Lc + U_OFF) + uo, Fv, P.k, rn);
      } else {
      const T h = P.invh2;
      rn[0][0] = res7(uc[0][0], uc[0][1], lA, uc[1][0], ymA0, un[0][0], um[0][0], fA0, h);
      rn[0][1] = res7(uc[0][1], rA, uc[0][0], uc[1][1], ymA1, un[0][1], um[0][1], fA1, h);
      rn[1][0] = res7(uc[1][0], uc[1][1], lB, ypB0, uc[0][0], un[1][0], um[1][0], fB0, h);
      rn[1][1] = res7(uc[1][1], rB, uc[1][0], ypB1, uc[0][1], un[1][1], um[1][1], fB1, h);
      }
      }
      // ---- Egprolg at the green nodes (row A col Q, row B col PH) of plane z = j-1
      const int z = j - 1;
      const bool zin = z >= 1 && z <= M - 1;
      T gn[2];
      {
        const T *V0 = (const T *)(Lp + V0_OFF), *V1 = (const T *)(Lp + V1_OFF);   // v_R(z)
        const int hx = C.hx;
        // row A (half row w): green col Q; x neighbours have parity PH, y neighbours parity Q
        const T *XA = PH ? V1 : V0, *YA = Q ? V1 : V0;
        // row B (half row w+1): green col PH; x neighbours parity Q, y neighbours parity PH
        const T *XB = Q ? V1 : V0, *YB = PH ? V1 : V0;
        T xpA, xmA, xpB, xmB;
        if (Q) {   // row A green at odd x: xg+1 -> hx+1, xg-1 -> hx; row B green at even x
          xpA = XA[w * Gm::VW + hx + 1];
          xmA = XA[w * Gm::VW + hx];
          xpB = XB[(w + 1) * Gm::VW + hx];
          xmB = XB[(w + 1) * Gm::VW + hx - 1];
        } else {
          xpA = XA[w * Gm::VW + hx];
          xmA = XA[w * Gm::VW + hx - 1];
          xpB = XB[(w + 1) * Gm::VW + hx + 1];
          xmB = XB[(w + 1) * Gm::VW + hx];
        }
        // y neighbours: row A (yA odd): yA+1 -> half row w+1, yA-1 -> w; row B (even): yB+1 -> w+1, yB-1 -> w
        const T ypA = YA[(w + 1) * Gm::VW + hx], ymA = YA[w * Gm::VW + hx];
        const T ypB2 = YB[(w + 1) * Gm::VW + hx], ymB2 = YB[w * Gm::VW + hx];
        gn[0] = jac6(P.c, rn[0][Q], xpA, xmA, ypA, ymA, vrn[0], S.vr[PH][0]);
        gn[1] = jac6(P.c, rn[1][PH], xpB, xmB, ypB2, ymB2, vrn[1], S.vr[PH][1]);
        if (!(C.m.full && zin)) {
          sel0(gn[0], zin && C.m.rA && (Q ? C.m.c1 : C.m.c0));
          sel0(gn[1], zin && C.m.rB && (PH ? C.m.c1 : C.m.c0));
        }
      }
      {
        T *g = (T *)gz + (2 * w + 1) * GS + (lane + 1);
        g[0] = gn[0];
        g[GS] = gn[1];
      }
      // ---- Egprolr at the red nodes of q = j-2 (row A col Q, row B col PH), then u_new
      const int q = j - 2;
      if (q >= it.zs && q >= 1 && q <= M - 1 && (UNIF || C.oA || C.oB)) {   // warp-uniform (see OpDesc3P)
        const T *g = (const T *)gq + (2 * w + 1) * GS + (lane + 1);
        const T ymA = g[-GS], ypB = g[2 * GS];
        const T(&g1)[2] = S.g[PH];   // greens of plane q
        const T(&g0)[2] = S.g[Q];    // greens of plane q-1
        T vA, vB, a0, a1, b0, b1;
        if (Q == 0) {
          // row A red col 0: i+1 own green, i-1 lane-1; row B red col 1: i+1 lane+1, i-1 own green
          vA = jac6(P.c, S.rq[0], g1[0], g[-1], g1[1], ymA, gn[0], g0[0]);
          vB = jac6(P.c, S.rq[1], g[GS + 1], g1[1], ypB, g1[0], gn[1], g0[1]);
          a0 = vA;
          a1 = g1[0];
          b0 = g1[1];
          b1 = vB;
        } else {
          // row A red col 1: i+1 lane+1, i-1 own green; row B red col 0: i+1 own green, i-1 lane-1
          vA = jac6(P.c, S.rq[0], g[1], g1[0], g1[1], ymA, gn[0], g0[0]);
          vB = jac6(P.c, S.rq[1], g1[1], g[GS - 1], ypB, g1[0], gn[1], g0[1]);
          a0 = g1[0];
          a1 = vA;
          b0 = vB;
          b1 = g1[1];
        }
        if (FINE) {   // u_new = u_old + v
          a0 = S.u[PH][0][0] + a0;
          a1 = S.u[PH][0][1] + a1;
          b0 = S.u[PH][1][0] + b0;
          b1 = S.u[PH][1][1] + b1;
        }
        const int xl = it.x0 - 2 + 2 * lane, yA = it.y0 - 1 + 2 * w;
        T *dst = &P.out(xl, yA, q);
        if (C.m.c0 && C.m.c1) {
          if (C.oA) st2(dst, a0, a1);
          if (C.oB) st2(dst + P.out.pitch, b0, b1);
        } else {
          if (C.oA && C.m.c0) __stcs(dst, a0);
          if (C.oA && C.m.c1) __stcs(dst + 1, a1);
          if (C.oB && C.m.c0) __stcs(dst + P.out.pitch, b0);
          if (C.oB && C.m.c1) __stcs(dst + P.out.pitch + 1, b1);
        }
      }
      // red r of plane z for the next step (row A red col PH, row B col Q)
      S.rq[0] = rn[0][PH];
      S.rq[1] = rn[1][Q];
      S.g[Q][0] = gn[0];
      S.g[Q][1] = gn[1];
    }
#pragma unroll
    for (int R = 0; R < 2; R++) {
      S.vr[PH][R] = vrn[R];
      if (FINE)
#pragma unroll
        for (int c = 0; c < 2; c++) S.u[PH][R][c] = un[R][c];
    }
  }
  static __device__ void finish(const Params &, State &) {}
};

// ================================================================= launch
template <class Op>
static cudaError_t run_zpipe(typename Op::Params &P, int M, int zlo, int zhi, cudaStream_t st) {
  // tiles start at x0 = 60 t - 2 (outputs x = 1 .. M-1), y0 = (2NW-2) t
  constexpr int ty = Op::Gm::TYW;
  return launch_zpipe<Op>(P, TX, ty, -2, 0, (M + 1) / TX + 1, (M + ty - 1) / ty, zlo, zhi, st);
}

// warps per CTA of the finest passes (MG_K3_NW: 8 = two 256-thread CTAs per SM,
// the default: measured on B200 at 513^3 fp64, desc 505 -> 468 us, asc 700 -> 655
// us, cycle -1.6 %; 16 = one 512-thread CTA per SM)
static int k3p_nw() {
  static const int nw = getenv("MG_K3_NW") ? atoi(getenv("MG_K3_NW")) : 8;
  return nw == 8 ? 8 : 16;
}

template <class T, int NW, int NSO = 0, bool UNIF = true, int ORDER = 2>
static cudaError_t desc_fine_nw(const T *u, const T *f, int64_t pitch, const S3<T> &rr, int M, const Coef<T> &k,
                                const NormSink &ns, cudaStream_t st, const ZRange3 &pz) {
  using Op = OpDesc3P<T, true, NW, NSO, UNIF, ORDER>;
  using Gm = typename Op::Gm;
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
  P.k = k;
  return run_zpipe<Op>(P, M, pz.zlo, pz.zhi < 0 ? M : pz.zhi, st);
}

template <class T>
cudaError_t fast3p_desc_fine(const T *u, const T *f, int64_t pitch, const S3<T> &rr, int M, int order,
                             const Coef<T> &k, const NormSink &ns, cudaStream_t st, const ZRange3 &pz) {
  if (order == 4) return desc_fine_nw<T, 8, 0, true, 4>(u, f, pitch, rr, M, k, ns, st, pz);
  static const bool div = env_flag("MG_K3_DIV");   // A/B: round 1's lane-dependent output branch
  if (k3p_nw() == 8 && div) return desc_fine_nw<T, 8, 0, false>(u, f, pitch, rr, M, k, ns, st, pz);
  if (k3p_nw() == 8) return desc_fine_nw<T, 8>(u, f, pitch, rr, M, k, ns, st, pz);
  return desc_fine_nw<T, 16>(u, f, pitch, rr, M, k, ns, st, pz);
}

template <class T, int NW, int NSO = 0, bool UNIF = true, int ORDER = 2>
static cudaError_t asc_fine_nw(const S3<T> &vr, const T *u_old, const T *f, int64_t pitch, T *u_new, int M, T c,
                               const Coef<T> &k, cudaStream_t st, const ZRange3 &pz) {
  using Op = OpAsc3P<T, true, NW, NSO, UNIF, ORDER>;
  using Gm = typename Op::Gm;
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
  P.k = k;
  return run_zpipe<Op>(P, M, pz.zlo, pz.zhi < 0 ? M : pz.zhi, st);
}

template <class T>
cudaError_t fast3p_asc_fine(const S3<T> &vr, const T *u_old, const T *f, int64_t pitch, T *u_new, int M, int order,
                            T c, const Coef<T> &k, cudaStream_t st, const ZRange3 &pz) {
  if (order == 4) return asc_fine_nw<T, 8, 0, true, 4>(vr, u_old, f, pitch, u_new, M, c, k, st, pz);
  static const bool div = env_flag("MG_K3_DIV");
  if (k3p_nw() == 8 && div) return asc_fine_nw<T, 8, 0, false>(vr, u_old, f, pitch, u_new, M, c, k, st, pz);
  if (k3p_nw() == 8) return asc_fine_nw<T, 8>(vr, u_old, f, pitch, u_new, M, c, k, st, pz);
  return asc_fine_nw<T, 16>(vr, u_old, f, pitch, u_new, M, c, k, st, pz);
}

// the G(s) level passes (s > 1): MG_K3_NWL warps (default 16)
static int k3p_nwl() {
  static const int nw = getenv("MG_K3_NWL") ? atoi(getenv("MG_K3_NWL")) : 16;
  return nw == 8 ? 8 : 16;
}

template <class T, int NW>
static cudaError_t rest_gr_nw(const D3<T> &r, const S3<T> &rr, int M, cudaStream_t st) {
  using Op = OpDesc3P<T, false, NW>;
  using Gm = typename Op::Gm;
  typename Op::Params P{};
  const int64_t n = M + 1;
  if (!tmap3<T>(&P.tf, r.p, n, n, n, r.pitch, r.plane, Gm::FW, Gm::FH)) return cudaErrorInvalidValue;
  P.out = rr;
  P.M = M;
  return run_zpipe<Op>(P, M, 0, M, st);
}
template <class T>
cudaError_t fast3p_rest_gr(const D3<T> &r, const S3<T> &rr, int M, cudaStream_t st) {
  if (k3p_nwl() == 8) return rest_gr_nw<T, 8>(r, rr, M, st);
  return rest_gr_nw<T, 16>(r, rr, M, st);
}

template <class T, int NW>
static cudaError_t jac_g_nw(const S3<T> &vr, const D3<T> &r, const D3<T> &v, int M, T c, cudaStream_t st) {
  using Op = OpAsc3P<T, false, NW>;
  using Gm = typename Op::Gm;
  typename Op::Params P{};
  const int64_t n = M + 1, H = M / 2 + 1;
  if (!tmap3<T>(&P.tf, r.p, n, n, n, r.pitch, r.plane, Gm::FW, Gm::FH)) return cudaErrorInvalidValue;
  const int sub[4] = {0, 6, 5, 3};   // C, Fx, Fy, Fz
  for (int i = 0; i < 4; i++)
    if (!tmap3<T>(&P.tv[i], vr.s[sub[i]], H, H, H, vr.pitch, vr.plane, Gm::VW, Gm::VH)) return cudaErrorInvalidValue;
  P.out = v;
  P.M = M;
  P.c = c;
  return run_zpipe<Op>(P, M, 0, M, st);
}
template <class T>
cudaError_t fast3p_jac_g(const S3<T> &vr, const D3<T> &r, const D3<T> &v, int M, T c, cudaStream_t st) {
  if (k3p_nwl() == 8) return jac_g_nw<T, 8>(vr, r, v, M, c, st);
  return jac_g_nw<T, 16>(vr, r, v, M, c, st);
}

template cudaError_t fast3p_rest_gr<double>(const D3<double> &, const S3<double> &, int, cudaStream_t);
template cudaError_t fast3p_rest_gr<float>(const D3<float> &, const S3<float> &, int, cudaStream_t);
template cudaError_t fast3p_jac_g<double>(const S3<double> &, const D3<double> &, const D3<double> &, int, double,
                                          cudaStream_t);
template cudaError_t fast3p_jac_g<float>(const S3<float> &, const D3<float> &, const D3<float> &, int, float,
                                         cudaStream_t);
template cudaError_t fast3p_desc_fine<double>(const double *, const double *, int64_t, const S3<double> &, int, int,
                                              const Coef<double> &, const NormSink &, cudaStream_t, const ZRange3 &);
template cudaError_t fast3p_desc_fine<float>(const float *, const float *, int64_t, const S3<float> &, int, int,
                                             const Coef<float> &, const NormSink &, cudaStream_t, const ZRange3 &);
template cudaError_t fast3p_asc_fine<double>(const S3<double> &, const double *, const double *, int64_t, double *, int,
                                             int, double, const Coef<double> &, cudaStream_t, const ZRange3 &);
template cudaError_t fast3p_asc_fine<float>(const S3<float> &, const float *, const float *, int64_t, float *, int,
                                            int, float, const Coef<float> &, cudaStream_t, const ZRange3 &);

}  // namespace mg
