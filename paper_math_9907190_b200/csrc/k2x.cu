// k2x.cu -- cross-cycle fusion in 2D: the finest ascent of
// one V-cycle and the finest descent of the next in one pass over the grid.
//
//   ascent  (OpJac2A<FINE>): greens of A(1) from r(u_old) and v_D(1), then the
//            D(1) nodes from the greens, u_new = u_old + v_A(1)  (P:57-60,
//            Eajacr/Eajacb P:350-360);
//   descent (OpDesc2Fine):   r = f - L u_new, Erest2r onto D(1),
//            max|r| for the residual history.
//
// Separately the two passes read u and f twice per cycle (10 N words in all
// per cycle); fused they read them once (8 N).  The tile
// kernels of k2f.cu would need a 4-node halo for this (r_new needs u_new on
// ring 1, u_new needs greens on ring 2, greens need u_old on ring 4), and
// their shared-memory phases turned out instruction-bound.  This kernel is a
// register pipeline instead: one warp streams down a strip of 56 output
// columns (lane l owns the column pair x = x0 - 4 + 2l, the 4-column halo on
// both sides is the outer lanes), one row per step, x neighbours by warp
// shuffles, no barriers.  At input row j a step computes
//     r_old(j-1) -> green(j-1) -> D node(j-2) -> u_new(j-2) -> r_new(j-3)
// and, every second row, the Erest2r pair of rows (j-5, j-4).  Input rows
// (u, f pairs and the v_D value of each lane) arrive 2 (fp64) / 3 (fp32) steps ahead
// through per-lane cp.async copies into an 8-slot shared-memory ring (each
// lane reads back only its own bytes); f stays in the ring for the two steps
// that read it instead of in registers (register prefetch instead stalled on
// the zero-masking of the loads and cost 40 registers; a 7-row lookahead with
// f in registers was 17 % slower: with a short ring the halo columns and rows
// that neighbouring strips share are re-read while still in L2).  A strip is
// cut into row segments (8 rows of warm-up each) so that the grid fills every
// SM exactly once; blocks of steps whose rows all lie inside run a mask-free
// instance of the step.  fp32 order 2 uses a four-columns-per-lane variant of
// the same pipeline (StripQ, below).  Same node formulas, same evaluation
// order: bit-identical to the two separate passes.
#include <type_traits>

#include "kernels.h"
#include "ops2.cuh"

namespace mg {
namespace xf {

// rows issued ahead (cp.async ring of 8 slots, LA + 4 <= 8: f of a row stays 3 more steps); measured on
// B200 (2D 8193^2, ms per fused pass): fp64 LA = 1 / 2 / 3 / 4: 0.477 / 0.361 / 0.379 / 0.409; fp32 LA = 2 / 3 / 4:
// 0.234 / 0.223 / 0.236
template <class T>
__host__ __device__ constexpr int lookahead() {
  return sizeof(T) == 8 ? 2 : 3;
}
constexpr int SW = 56;    // output columns per strip: 32 lanes x 2 minus 2 x 4 halo

template <class T>
struct V2;
template <>
struct V2<double> {
  using t = double2;
};
template <>
struct V2<float> {
  using t = float2;
};

template <class T>
__device__ __forceinline__ T shup(T v) {   // value of lane - 1
  return __shfl_up_sync(0xffffffffu, v, 1);
}
template <class T>
__device__ __forceinline__ T shdn(T v) {   // value of lane + 1
  return __shfl_down_sync(0xffffffffu, v, 1);
}

// per-lane asynchronous global -> shared copies (cp.async, sm_80+): the lane
// later reads back only what it copied itself, so no barrier is involved
template <int BYTES>
__device__ __forceinline__ void cpa(void *s, const void *g) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(s);
  if (BYTES == 16)
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(g) : "memory");
  else
    asm volatile("cp.async.ca.shared.global [%0], [%1], %2;\n" ::"r"(sa), "l"(g), "n"(BYTES) : "memory");
}
__device__ __forceinline__ void cpa_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cpa_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

// one grid row at the lane's pair: a = (x, y), b = (x+1, y), w = (x-1, y), e = (x+2, y)
template <class T>
struct Row {
  T a, b, w, e;
};
template <class T>
__device__ __forceinline__ Row<T> mkrow(T a, T b) {
  return Row<T>{a, b, shup(b), shdn(a)};
}

template <class T>
struct Pair {
  T a, b;
};

template <class T>
struct XParams {
  const T *u, *f;     // u_old, f (row pitch `pitch`)
  const T *ve, *vo;   // v_D(1), E and O (row pitch vp)
  T *un;              // u_new (pitch)
  T *re, *ro;         // the next cycle's r_D(1), E and O (pitch rp)
  int64_t pitch, vp, rp;
  int M, nstrips, seg;
  T c;
  Coef<T> k;
  NormSink ns;
  // octave pair fused in (RD strips): r_A(2) (pitch rap) and
  // r_D(2) E/O (pitch r2p) of the next cycle's descent; Mc = M / 2
  T *ra, *r2e, *r2o;
  int64_t rap, r2p;
  int Mc;
};

// prefetched inputs of one row
template <class T>
struct In {
  T ua, ub, fa, fb, d;
};

// One warp's strip segment.  Pipeline state lives in 4-slot arrays indexed
// by row & 3 (statically, the step body is unrolled 4 times), so nothing is
// shifted between steps.  Loads are unconditional from clamped addresses:
// rows outside [0, M] and columns outside [0, M] only feed nodes that are
// not interior, whose results are all selected away (inside() is false).
template <class T, int ORDER, int DEPTH, bool RD = false>   // DEPTH: ring slots per lane (power of 2)
struct Strip {
  static constexpr int LA = lookahead<T>();
  static constexpr int H = RD ? 8 : 4;   // halo columns per side
  static constexpr int SWK = 64 - 2 * H;  // output columns per strip
  const T *pu, *pf, *pve, *pvo;
  T *pun, *pre, *pro;
  int64_t pitch, vp, rp;
  Coef<T> k;
  T c;
  int x, xc, M, ys, ye;
  bool ca, cb, outl;   // (x, y) / (x+1, y) interior columns; lane writes output
  unsigned char *ring;  // this warp's DEPTH-slot input ring in shared memory, offset to the lane
  Row<T> U[4];         // u_old
  T Dv[4];             // v_D at the row's D node
  Pair<T> RO[4];       // r(u_old)
  T G[4];              // green value of the row
  Row<T> N[4];         // u_new
  Pair<T> R[4];        // r(u_new)
  T Os[2], A[2];       // RD: r_D(1) O and r_A(2) of the last two row pairs, by (row pair & 1)
  unsigned long long mx;   // max |r| as the bit pattern of a non-negative double (NaN sorts above inf)
  double ss;               // sum r^2 over the lane's output nodes (a16 L2 norm; single GPU: all rows)
  bool l2on, hist;         // L2 sum / any residual norm wanted
  // interior warps address by increments: next load row offset, next E / O
  // v_D load pointers, u_new store pointer of row j-2, next Erest2r offset
  int64_t lo, rso;
  const T *ldE, *ldO;
  T *stp;

  __device__ __forceinline__ Strip(const XParams<T> &P, int x_, int ys_, int ye_, unsigned char *ring_) {
    ring = ring_;
    pu = P.u;
    pf = P.f;
    pve = P.ve;
    pvo = P.vo;
    pun = P.un;
    pre = P.re;
    pro = P.ro;
    pitch = P.pitch;
    vp = P.vp;
    rp = P.rp;
    k = P.k;
    c = P.c;
    M = P.M;
    x = x_;
    ys = ys_;
    ye = ye_;
    xc = min(max(x, 0), M);
    ca = x >= 1 && x <= M - 1;
    cb = x + 1 >= 1 && x + 1 <= M - 1;
    const int lane = threadIdx.x & 31;
    outl = lane >= H / 2 && lane < 32 - H / 2;
#pragma unroll
    for (int i = 0; i < 4; i++) {
      U[i] = N[i] = Row<T>{0, 0, 0, 0};
      RO[i] = R[i] = Pair<T>{0, 0};
      Dv[i] = G[i] = (T)0;
    }
    Os[0] = Os[1] = A[0] = A[1] = (T)0;
    mx = 0ull;
    ss = 0.0;
    l2on = P.ns.l2 != nullptr;
    hist = P.ns.slots != nullptr;
  }
  // incremental addressing from step j0 on (row-interior blocks only)
  __device__ __forceinline__ void start(int j0) {
    const int r = j0 + LA;   // the first row issued inside the loop
    lo = (int64_t)r * pitch + xc;
    ldE = pve + (int64_t)((r + 1) >> 1) * vp + (xc >> 1);   // first even row >= r
    ldO = pvo + (int64_t)(r >> 1) * vp + (xc >> 1);         // first odd row >= r
    stp = pun + (int64_t)(j0 - 2) * pitch + x;
    rso = (int64_t)((j0 - 4) >> 1) * rp + (x >> 1);
  }
  static __device__ __forceinline__ unsigned long long absbits(T v) {
    return (unsigned long long)__double_as_longlong((double)v) & 0x7fffffffffffffffull;
  }
  __device__ __forceinline__ bool rin(int y) const { return (unsigned)(y - 1) < (unsigned)(M - 1); }

  // slot layout: 32 u pairs, 32 f pairs, 32 v_D values (lane l at pair /
  // value l); `ring` already points at the lane's u pair of slot 0
  static constexpr int SLOT = 32 * 5 * sizeof(T), FO = 32 * 2 * sizeof(T), DO = 32 * 4 * sizeof(T);
  // start the copies of row y into slot y % DEPTH (one commit group per row)
  __device__ __forceinline__ void issue(int y) const {
    const int yc = min(max(y, 0), M);
    const int64_t o = (int64_t)yc * pitch + xc;
    unsigned char *q = ring + (y & (DEPTH - 1)) * SLOT;
    cpa<2 * sizeof(T)>(q, pu + o);
    cpa<2 * sizeof(T)>(q + FO, pf + o);
    // the D(1) node of row y in the pair: (x, y) on even rows (E), (x+1, y) on odd rows (O)
    cpa<sizeof(T)>(q + DO - (threadIdx.x & 31) * sizeof(T),
                   ((y & 1) ? pvo : pve) + (int64_t)(yc >> 1) * vp + (xc >> 1));
    cpa_commit();
  }
  // the same for an interior warp (row y in [0, M], parity YP = y & 1)
  template <int YP>
  __device__ __forceinline__ void issue_inc(int y) {
    unsigned char *q = ring + (y & (DEPTH - 1)) * SLOT;
    cpa<2 * sizeof(T)>(q, pu + lo);
    cpa<2 * sizeof(T)>(q + FO, pf + lo);
    lo += pitch;
    if (YP) {
      cpa<sizeof(T)>(q + DO - (threadIdx.x & 31) * sizeof(T), ldO);
      ldO += vp;
    } else {
      cpa<sizeof(T)>(q + DO - (threadIdx.x & 31) * sizeof(T), ldE);
      ldE += vp;
    }
    cpa_commit();
  }
  __device__ __forceinline__ Pair<T> fpair(int y) const {   // f at the lane's pair of row y (in the ring)
    const auto f = *reinterpret_cast<const typename V2<T>::t *>(ring + (y & (DEPTH - 1)) * SLOT + FO);
    return Pair<T>{f.x, f.y};
  }
  __device__ __forceinline__ In<T> fetch(int y) const {
    const unsigned char *q = ring + (y & (DEPTH - 1)) * SLOT;
    const auto u = *reinterpret_cast<const typename V2<T>::t *>(q);
    const auto f = *reinterpret_cast<const typename V2<T>::t *>(q + FO);
    const T d = *reinterpret_cast<const T *>(q + DO - (threadIdx.x & 31) * sizeof(T));
    return In<T>{u.x, u.y, f.x, f.y, d};
  }

  // r = f - L u at the pair of row y (inside-masked)
  // r at the pair of row y; ry, ka, kb: row y / column x / column x+1
  // interior (compile-time true away from the boundary)
  __device__ __forceinline__ Pair<T> res(const Row<T> &dn, const Row<T> &cr, const Row<T> &up, const Pair<T> &f,
                                         bool ry, bool ka, bool kb) const {
    Nb9<T> q0, q1;
    q0.c = cr.a;
    q0.w = cr.w;
    q0.s = dn.a;
    q0.e = cr.b;
    q0.n = up.a;
    q1.c = cr.b;
    q1.w = cr.a;
    q1.s = dn.b;
    q1.e = cr.e;
    q1.n = up.b;
    if (ORDER == 4) {
      q0.ne = up.b;
      q0.nw = up.w;
      q0.sw = dn.w;
      q0.se = dn.b;
      q1.ne = up.e;
      q1.nw = up.a;
      q1.sw = dn.a;
      q1.se = dn.e;
    } else {
      q0.ne = q0.nw = q0.sw = q0.se = q1.ne = q1.nw = q1.sw = q1.se = (T)0;
    }
    Pair<T> r;
    r.a = (ry && ka) ? res2v<T, ORDER>(q0, f.a, k) : (T)0;
    r.b = (ry && kb) ? res2v<T, ORDER>(q1, f.b, k) : (T)0;
    return r;
  }

  // one step at input row j, j & 3 == K (j - ys is a multiple of 4 at K = 0)
  // RE: a row of this step (computed, restricted or loaded) may lie outside
  // the interior (masks and clamped loads); CE: the same for the warp's columns
  template <int K, bool RE, bool CE>
  __device__ __forceinline__ void step(int j, const XParams<T> &P) {
    constexpr int PAR = K & 1;
    constexpr int s0 = K, s1 = (K + 3) & 3, s2 = (K + 2) & 3, s3 = (K + 1) & 3;   // rows j, j-1, j-2, j-3 (j-4: s0)
    // row j: wait for its copies (the LA - 1 younger groups may stay in flight),
    // then issue row j + LA into the slot of row j + LA - DEPTH, whose f was
    // last read at step j - 1 (f of row r is read at steps r+1 and r+3, from
    // the ring: it is not kept in registers)
    cpa_wait<LA - 1>();
    const In<T> in = fetch(j);
    if (RE)
      issue(j + LA);
    else
      issue_inc<(K + LA) & 1>(j + LA);
    U[s0] = mkrow(in.ua, in.ub);
    Dv[s0] = in.d;
    const bool r1 = !RE || rin(j - 1), r2 = !RE || rin(j - 2), r3 = !RE || rin(j - 3);
    const bool ka = !CE || ca, kb = !CE || cb;
    // r_old at row j-1
    RO[s1] = res(U[s2], U[s1], U[s0], fpair(j - 1), r1, ka, kb);
    // green at row j-1: (x+1) on even rows, x on odd rows
    if (PAR == 1) {   // j-1 even: W = (x, y), S = (x+1, y-1), E = (x+2, y), N = (x+1, y+1)
      const T dE = shdn(Dv[s1]);
      G[s1] = (r1 && kb) ? jac4(c, RO[s1].b, Dv[s1], Dv[s2], dE, Dv[s0]) : (T)0;
    } else {          // j-1 odd: W = (x-1, y), S = (x, y-1), E = (x+1, y), N = (x, y+1)
      const T dW = shup(Dv[s1]);
      G[s1] = (r1 && ka) ? jac4(c, RO[s1].a, dW, Dv[s2], Dv[s1], Dv[s0]) : (T)0;
    }
    // D node at row j-2 from the greens; u_new = u_old + v there
    {
      const int y = j - 2;
      T va, vb;
      if (PAR == 0) {   // y even: D node x; W = (x-1, y), S = (x, y-1), E = (x+1, y), N = (x, y+1)
        const T gW = shup(G[s2]);
        va = (r2 && ka) ? jac4(c, RO[s2].a, gW, G[s3], G[s2], G[s1]) : (T)0;
        vb = G[s2];
      } else {          // y odd: D node x+1; W = (x, y), S = (x+1, y-1), E = (x+2, y), N = (x+1, y+1)
        const T gE = shdn(G[s2]);
        va = G[s2];
        vb = (r2 && kb) ? jac4(c, RO[s2].b, G[s2], G[s3], gE, G[s1]) : (T)0;
      }
      const bool i0 = r2 && ka, i1 = r2 && kb;
      const T na = i0 ? U[s2].a + va : U[s2].a, nb = i1 ? U[s2].b + vb : U[s2].b;
      N[s2] = mkrow(na, nb);
      if (outl && y >= ys && y < ye) {
        T *p = RE ? pun + (int64_t)y * pitch + x : stp;
        if (i0 && i1) {
          typename V2<T>::t v;
          v.x = na;
          v.y = nb;
          *reinterpret_cast<typename V2<T>::t *>(p) = v;
        } else if (i1) {   // x = 0
          p[1] = nb;
        }
      }
    }
    // r_new at row j-3 (rows j-4, j-3, j-2 of u_new)
    R[s3] = res(N[s0], N[s3], N[s2], fpair(j - 3), r3, ka, kb);
    if (hist && outl && j - 3 >= ys && j - 3 < ye) {
      const unsigned long long a = absbits(R[s3].a), b = absbits(R[s3].b), m = a > b ? a : b;
      mx = m > mx ? m : mx;
      if (l2on) ss += sq((double)R[s3].a) + sq((double)R[s3].b);
    }
    // Erest2r of the row pair (y, y+1) = (j-5, j-4) when y is even
    if (PAR == 1) {
      const int y = j - 5;
      const Pair<T> R6 = R[s2], R5 = R[s1], R4 = R[s0], R3 = R[s3];
      const T rW = shup(R5.b), rE = shdn(R4.a);
      // interior D(1) nodes E = (x, y), O = (x+1, y+1) (the lower bounds only matter for halo lanes)
      const bool inE = (!CE || (x >= 2 && x <= M - 2)) && (!RE || (y >= 2 && y <= M - 2));
      const bool inO = (!CE || (x + 1 >= 1 && x + 1 <= M - 1)) && (!RE || (y + 1 >= 1 && y + 1 <= M - 1));
      const T ev = erest2r(R5.a, rW, R6.a, R5.b, R4.a), ov = erest2r(R4.b, R4.a, R5.b, rE, R3.b);
      if (outl && y >= ys && y < ye) {
        const int64_t o = RE ? (int64_t)(y >> 1) * rp + (x >> 1) : rso;
        if (inE) pre[o] = ev;
        if (inO) pro[o] = ov;
      }
      if (!RE) rso += rp;
      if constexpr (RD) restrict_pair<K, RE, CE>(y, inE ? ev : (T)0, inO ? ov : (T)0, P);
    }
    if (!RE) stp += pitch;
  }
  // RD: the next cycle's octave pair D(1) -> A(2) -> D(2) (OpRest2DAD's node
  // formulas and operand order) from the row pair (y, y+1) of r_D(1) just
  // formed: Erest2b at the A(2) node (X, Y) = (x/2, y/2) of the lane,
  // then Erest2r at the D(2) node of A(2) row Y-1 (E on even rows at
  // even X, O on odd rows at odd X).  e, o: E(X, Y), O(X, Y) of D(1), zero outside.
  template <int K, bool RE, bool CE>
  __device__ __forceinline__ void restrict_pair(int y, T e, T o, const XParams<T> &P) {
    constexpr int h = K >> 1;   // K = 1: h = 0, K = 3: h = 1 (row pairs alternate)
    const int X = x >> 1, Y = y >> 1, Mc = P.Mc;
    const T oW = shup(o), opW = shup(Os[h ^ 1]);   // O(X-1, Y), O(X-1, Y-1)
    T ra = erest2b(e, opW, Os[h ^ 1], o, oW);
    const bool inA = (!CE || (X >= 1 && X <= Mc - 1)) && (!RE || (Y >= 1 && Y <= Mc - 1));
    ra = inA ? ra : (T)0;
    const bool seg = outl && y >= ys && y < ye;
    if (seg && inA) P.ra[(int64_t)Y * P.rap + X] = ra;
    // r_A(2) rows Y-2 (A[h]), Y-1 (A[h^1]), Y (ra) -> D(2) at row Yd = Y - 1
    const T c = A[h ^ 1], w = shup(c), ea = shdn(c);
    const T d2 = erest2r(c, w, A[h], ea, ra);
    const int Yd = Y - 1, yd = 2 * Yd;
    if (outl && yd >= ys && yd < ye) {
      const int64_t od = (int64_t)(Yd >> 1) * P.r2p + (X >> 1);
      if (K == 3) {   // Yd even: E at even X
        if (!(X & 1) && (!CE || (X >= 2 && X <= Mc - 2)) && (!RE || (Yd >= 2 && Yd <= Mc - 2))) P.r2e[od] = d2;
      } else {        // Yd odd: O at odd X
        if ((X & 1) && (!CE || X <= Mc - 1) && (!RE || Yd <= Mc - 1)) P.r2o[od] = d2;
      }
    }
    A[h] = ra;
    Os[h] = o;
  }
  template <bool RE, bool CE>
  __device__ __forceinline__ void steps(int j, const XParams<T> &P) {
    step<0, RE, CE>(j, P);
    step<1, RE, CE>(j + 1, P);
    step<2, RE, CE>(j + 2, P);
    step<3, RE, CE>(j + 3, P);
  }
};

template <class T, int ORDER, int DEPTH, int MINB, bool RD = false>
__global__ void __launch_bounds__(32, MINB) asc_desc_stream(const __grid_constant__ XParams<T> P) {
  using St = Strip<T, ORDER, DEPTH, RD>;
  constexpr int H = St::H, SWK = St::SWK;
  const int lane = threadIdx.x & 31;
  const int item = blockIdx.x;
  const int nseg = (P.M + P.seg - 1) / P.seg;
  unsigned long long mx = 0ull;
  double ss = 0.0;
  (void)SWK;
  if (item < P.nstrips * nseg) {   // warp-uniform
    const int strip = item % P.nstrips, sg = item / P.nstrips;
    const int ys = sg * P.seg, ye = min(ys + P.seg, P.M);
    extern __shared__ __align__(16) unsigned char xsm[];
    St S(P, strip * SWK - H + 2 * lane, ys, ye, xsm + lane * (2 * sizeof(T)));
    // steps j0 .. jend: ye - ys + 8 (RD: + 16) of them, a multiple of 4; RD
    // also needs r_D(1) three rows above and below the segment
    const int j0 = ys - (RD ? 8 : 4), jend = ye + (RD ? 7 : 3);
#pragma unroll
    constexpr int LA = lookahead<T>();
    for (int i = 0; i < LA; i++) S.issue(j0 + i);
    // A block of 4 steps j..j+3 is row-interior when every row it computes,
    // restricts or loads lies inside: j >= 8 (RD: 12) and j + 3 + LA <= M.
    // Column-interior warps: lanes' columns x0-H .. x0-H+63 inside [1, M-1].
    const int x0 = strip * SWK;
    const bool ce = x0 - H < 1 || x0 - H + 63 > P.M - 1;
    auto rowin = [&](int j) { return j >= (RD ? 12 : 8) && j + 3 + LA <= P.M; };
    int j = j0;
    for (; j <= jend && !rowin(j); j += 4) S.template steps<true, true>(j, P);
    if (j <= jend) {
      S.start(j);
      if (ce) {
        for (; j <= jend && rowin(j); j += 4) S.template steps<false, true>(j, P);
      } else {
        for (; j <= jend && rowin(j); j += 4) S.template steps<false, false>(j, P);
      }
    }
    for (; j <= jend; j += 4) S.template steps<true, true>(j, P);
    mx = S.mx;
    ss = S.ss;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long w = __shfl_xor_sync(0xffffffffu, mx, o);
    mx = w > mx ? w : mx;
  }
  if (lane == 0 && item < P.nstrips * nseg) norm_push(P.ns, __longlong_as_double((long long)mx));
  if (item < P.nstrips * nseg) warp_l2_push(P.ns, ss);   // warp-uniform
}


// ---------------------------------------------------------------- fp32
// Four columns per lane (fp32, order 2): lane l owns x = x0 - 4 + 4l .. x+3,
// so a warp streams a strip of 120 output columns; a row of u or f is one
// 16-byte vector per lane, the x neighbours of the quad are the neighbouring
// lanes' outer values (two shuffles per row instead of four), and the halo
// costs 8 of 128 columns instead of 8 of 64.  The nodes, their formulas and
// their order are those of the pair strip above (node by node), so the results
// are bit-identical to it and to the two separate passes.
constexpr int SWQ = 120;

struct Q4 {
  float a, b, c, d;   // x, x+1, x+2, x+3
};
struct RowQ {
  Q4 q;
  float w, e;   // x-1, x+4
};
__device__ __forceinline__ RowQ mkrowq(const Q4 &q) { return RowQ{q, shup(q.d), shdn(q.a)}; }

struct XParamsQ {
  const float *u, *f, *ve, *vo;
  float *un, *re, *ro;
  int64_t pitch, vp, rp;
  int M, nstrips, seg;
  float c;
  Coef<float> k;
  NormSink ns;
};

template <int DEPTH, int LA>
struct StripQ {
  const float *pu, *pf, *pve, *pvo;
  float *pun, *pre, *pro;
  int64_t pitch, vp, rp;
  Coef<float> kk;
  float c;
  int x, xc, M, ys, ye;
  bool k0, k1, k2, k3, outl;   // interior columns x..x+3; lane writes output
  unsigned char *ring;
  RowQ U[4];
  Q4 N4[4];                    // u_new (quad only; w/e shuffled when a row becomes the centre)
  float Nw[4], Ne[4];
  float D0[4], D1[4];          // v_D at the two D nodes of the row (x, x+2 even rows; x+1, x+3 odd rows)
  Q4 RO[4];
  float G0[4], G1[4];          // the two greens of the row (x+1, x+3 even rows; x, x+2 odd rows)
  Q4 R[4];
  unsigned long long mx;
  double ss;   // sum r^2 (a16 L2 norm)
  bool l2on, hist;
  static constexpr int SLOT = 32 * 40, FO = 32 * 16, DO = 32 * 32;

  __device__ __forceinline__ StripQ(const XParamsQ &P, int x_, int ys_, int ye_, unsigned char *ring_) {
    pu = P.u; pf = P.f; pve = P.ve; pvo = P.vo; pun = P.un; pre = P.re; pro = P.ro;
    pitch = P.pitch; vp = P.vp; rp = P.rp; kk = P.k; c = P.c; M = P.M;
    x = x_; ys = ys_; ye = ye_; ring = ring_;
    xc = min(max(x, 0), M);
    k0 = x >= 1 && x <= M - 1;
    k1 = x + 1 >= 1 && x + 1 <= M - 1;
    k2 = x + 2 >= 1 && x + 2 <= M - 1;
    k3 = x + 3 >= 1 && x + 3 <= M - 1;
    const int lane = threadIdx.x & 31;
    outl = lane >= 1 && lane < 31;
#pragma unroll
    for (int i = 0; i < 4; i++) {
      U[i] = RowQ{{0, 0, 0, 0}, 0, 0};
      N4[i] = RO[i] = R[i] = Q4{0, 0, 0, 0};
      Nw[i] = Ne[i] = D0[i] = D1[i] = G0[i] = G1[i] = 0.f;
    }
    mx = 0ull;
    ss = 0.0;
    l2on = P.ns.l2 != nullptr;
    hist = P.ns.slots != nullptr;
  }
  __device__ __forceinline__ bool rin(int y) const { return (unsigned)(y - 1) < (unsigned)(M - 1); }
  __device__ __forceinline__ void issue(int y) const {
    const int yc = min(max(y, 0), M);
    const int64_t o = (int64_t)yc * pitch + xc;
    unsigned char *q = ring + (y & (DEPTH - 1)) * SLOT;
    cpa<16>(q, pu + o);
    cpa<16>(q + FO, pf + o);
    // the two D(1) nodes of row y in the quad: E at x, x+2 (even rows), O at x+1, x+3 (odd rows)
    cpa<8>(q + DO - (threadIdx.x & 31) * 8, ((y & 1) ? pvo : pve) + (int64_t)(yc >> 1) * vp + (xc >> 1));
    cpa_commit();
  }
  __device__ __forceinline__ Q4 ld4(const unsigned char *p) const {
    const float4 v = *reinterpret_cast<const float4 *>(p);
    return Q4{v.x, v.y, v.z, v.w};
  }
  // r = f - L u at the quad of row y (gather9 roles, order 2), masked
  __device__ __forceinline__ Q4 res(const Q4 &dn, const RowQ &cr, const Q4 &up, const Q4 &f, bool ry) const {
    auto one = [&](float cc, float w, float s, float e, float n, float ff, bool k) {
      Nb9<float> q;
      q.c = cc; q.w = w; q.s = s; q.e = e; q.n = n;
      q.ne = q.nw = q.sw = q.se = 0.f;
      return (ry && k) ? res2v<float, 2>(q, ff, kk) : 0.f;
    };
    Q4 r;
    r.a = one(cr.q.a, cr.w, dn.a, cr.q.b, up.a, f.a, k0);
    r.b = one(cr.q.b, cr.q.a, dn.b, cr.q.c, up.b, f.b, k1);
    r.c = one(cr.q.c, cr.q.b, dn.c, cr.q.d, up.c, f.c, k2);
    r.d = one(cr.q.d, cr.q.c, dn.d, cr.e, up.d, f.d, k3);
    return r;
  }
  template <int K>
  __device__ __forceinline__ void step(int j) {
    constexpr int PAR = K & 1;
    constexpr int s0 = K, s1 = (K + 3) & 3, s2 = (K + 2) & 3, s3 = (K + 1) & 3;
    cpa_wait<LA - 1>();
    const unsigned char *q = ring + (j & (DEPTH - 1)) * SLOT;
    const Q4 u = ld4(q);
    const float2 dd = *reinterpret_cast<const float2 *>(q + DO - (threadIdx.x & 31) * 8);
    issue(j + LA);
    U[s0] = mkrowq(u);
    D0[s0] = dd.x;
    D1[s0] = dd.y;
    const bool r1 = rin(j - 1), r2 = rin(j - 2), r3 = rin(j - 3);
    const Q4 f1 = ld4(ring + ((j - 1) & (DEPTH - 1)) * SLOT + FO);
    RO[s1] = res(U[s2].q, U[s1], U[s0].q, f1, r1);
    // greens of row j-1
    if (PAR == 1) {   // y even: greens at x+1, x+3
      const float dE = shdn(D0[s1]);   // E at x+4
      G0[s1] = (r1 && k1) ? jac4(c, RO[s1].b, D0[s1], D0[s2], D1[s1], D0[s0]) : 0.f;
      G1[s1] = (r1 && k3) ? jac4(c, RO[s1].d, D1[s1], D1[s2], dE, D1[s0]) : 0.f;
    } else {          // y odd: greens at x, x+2
      const float dW = shup(D1[s1]);   // O at x-1
      G0[s1] = (r1 && k0) ? jac4(c, RO[s1].a, dW, D0[s2], D0[s1], D0[s0]) : 0.f;
      G1[s1] = (r1 && k2) ? jac4(c, RO[s1].c, D0[s1], D1[s2], D1[s1], D1[s0]) : 0.f;
    }
    // D nodes of row j-2 and u_new there
    {
      const int y = j - 2;
      float va, vb, vc, vd;
      if (PAR == 0) {   // y even: D at x, x+2; greens at x+1 (G0), x+3 (G1)
        const float gW = shup(G1[s2]);   // green at x-1
        va = (r2 && k0) ? jac4(c, RO[s2].a, gW, G0[s3], G0[s2], G0[s1]) : 0.f;
        vb = G0[s2];
        vc = (r2 && k2) ? jac4(c, RO[s2].c, G0[s2], G1[s3], G1[s2], G1[s1]) : 0.f;
        vd = G1[s2];
      } else {          // y odd: D at x+1, x+3; greens at x (G0), x+2 (G1)
        const float gE = shdn(G0[s2]);   // green at x+4
        va = G0[s2];
        vb = (r2 && k1) ? jac4(c, RO[s2].b, G0[s2], G0[s3], G1[s2], G0[s1]) : 0.f;
        vc = G1[s2];
        vd = (r2 && k3) ? jac4(c, RO[s2].d, G1[s2], G1[s3], gE, G1[s1]) : 0.f;
      }
      const Q4 &uo = U[s2].q;
      Q4 n;
      n.a = (r2 && k0) ? uo.a + va : uo.a;
      n.b = (r2 && k1) ? uo.b + vb : uo.b;
      n.c = (r2 && k2) ? uo.c + vc : uo.c;
      n.d = (r2 && k3) ? uo.d + vd : uo.d;
      N4[s2] = n;
      Nw[s2] = shup(n.d);
      Ne[s2] = shdn(n.a);
      if (outl && y >= ys && y < ye && r2) {
        float *p = pun + (int64_t)y * pitch + x;
        if (k0 && k1 && k2 && k3) {
          *reinterpret_cast<float4 *>(p) = make_float4(n.a, n.b, n.c, n.d);
        } else {
          if (k0) p[0] = n.a;
          if (k1) p[1] = n.b;
          if (k2) p[2] = n.c;
          if (k3) p[3] = n.d;
        }
      }
    }
    // r_new at row j-3
    {
      const Q4 f3 = ld4(ring + ((j - 3) & (DEPTH - 1)) * SLOT + FO);
      const RowQ cr{N4[s3], Nw[s3], Ne[s3]};
      R[s3] = res(N4[s0], cr, N4[s2], f3, r3);
      if (hist && outl && j - 3 >= ys && j - 3 < ye) {
        auto ab = [](float v) { return (unsigned long long)__double_as_longlong((double)v) & 0x7fffffffffffffffull; };
        unsigned long long m = ab(R[s3].a);
        m = max(m, ab(R[s3].b));
        m = max(m, ab(R[s3].c));
        m = max(m, ab(R[s3].d));
        mx = max(mx, m);
        if (l2on)
          ss += sq((double)R[s3].a) + sq((double)R[s3].b) + sq((double)R[s3].c) + sq((double)R[s3].d);
      }
    }
    // Erest2r of rows (j-5, j-4) when j-5 is even
    if (PAR == 1) {
      const int y = j - 5;
      const Q4 R6 = R[s2], R5 = R[s1], R4 = R[s0], R3 = R[s3];
      const float rW = shup(R5.d), rE = shdn(R4.a);
      if (outl && y >= ys && y < ye) {
        const int64_t o = (int64_t)(y >> 1) * rp + (x >> 1);
        const bool ye_ = y >= 2 && y <= M - 2, yo_ = y + 1 <= M - 1;
        const float e0 = erest2r(R5.a, rW, R6.a, R5.b, R4.a);
        const float e2 = erest2r(R5.c, R5.b, R6.c, R5.d, R4.c);
        const float o1 = erest2r(R4.b, R4.a, R5.b, R4.c, R3.b);
        const float o3 = erest2r(R4.d, R4.c, R5.d, rE, R3.d);
        if (ye_ && x >= 2 && x <= M - 2) pre[o] = e0;
        if (ye_ && x + 2 >= 2 && x + 2 <= M - 2) pre[o + 1] = e2;
        if (yo_ && x + 1 <= M - 1) pro[o] = o1;
        if (yo_ && x + 3 <= M - 1) pro[o + 1] = o3;
      }
    }
  }
};

template <int DEPTH, int LA>
__global__ void __launch_bounds__(32, 16) asc_desc_stream_q(const __grid_constant__ XParamsQ P) {
  const int lane = threadIdx.x & 31;
  const int item = blockIdx.x;
  const int nseg = (P.M + P.seg - 1) / P.seg;
  unsigned long long mx = 0ull;
  double ss = 0.0;
  if (item < P.nstrips * nseg) {
    const int strip = item % P.nstrips, sg = item / P.nstrips;
    const int ys = sg * P.seg, ye = min(ys + P.seg, P.M);
    extern __shared__ __align__(16) unsigned char xsm[];
    StripQ<DEPTH, LA> S(P, strip * SWQ - 4 + 4 * lane, ys, ye, xsm + lane * 16);
    const int j0 = ys - 4, jend = ye + 3;
#pragma unroll
    for (int i = 0; i < LA; i++) S.issue(j0 + i);
    // (a mask-free instance for interior blocks, as in the pair strip, measured 7 % slower here)
    for (int j = j0; j <= jend; j += 4) {
      S.template step<0>(j);
      S.template step<1>(j + 1);
      S.template step<2>(j + 2);
      S.template step<3>(j + 3);
    }
    mx = S.mx;
    ss = S.ss;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long w = __shfl_xor_sync(0xffffffffu, mx, o);
    mx = w > mx ? w : mx;
  }
  if (lane == 0 && item < P.nstrips * nseg) norm_push(P.ns, __longlong_as_double((long long)mx));
  if (item < P.nstrips * nseg) warp_l2_push(P.ns, ss);   // warp-uniform
}

}  // namespace xf

template <class T, int ORDER, int DEPTH, int MINB, bool RD = false>
static cudaError_t asc_desc_launch_w(const xf::XParams<T> &P0, cudaStream_t st) {
  constexpr int SMEM = DEPTH * 32 * 5 * sizeof(T);
  static int wres = 0, sms = 0;
  if (!wres) {
    int dev = 0, nb = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, xf::asc_desc_stream<T, ORDER, DEPTH, MINB, RD>, 32, SMEM);
    wres = nb > 0 ? nb : 1;
    if (sms <= 0) sms = 148;
  }
  xf::XParams<T> P = P0;
  P.nstrips = (P.M + xf::Strip<T, ORDER, DEPTH, RD>::SWK - 1) / xf::Strip<T, ORDER, DEPTH, RD>::SWK;
  // exactly one wave: at most sms * wres warps (a second, partial wave would
  // double the tail), a segment of >= 32 rows (multiple of 4) each
  const int S = max(1, (sms * wres) / P.nstrips);
  int seg = (P.M + S - 1) / S;
  seg = (seg + 3) / 4 * 4;
  if (seg < 32) seg = 32;
  P.seg = seg;
  const int nitems = P.nstrips * ((P.M + seg - 1) / seg);
  xf::asc_desc_stream<T, ORDER, DEPTH, MINB, RD><<<nitems, 32, SMEM, st>>>(P);
  return cudaGetLastError();
}

// fp32 order 2: the four-columns-per-lane strip (MG_XF_PAIRS=1: the pair strip)
template <int LA>
static cudaError_t asc_desc_launch_q(const xf::XParams<float> &P0, cudaStream_t st) {
  constexpr int DEPTH = 8, SMEM = DEPTH * 32 * 40;
  static int wres = 0, sms = 0;
  if (!wres) {
    int dev = 0, nb = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, xf::asc_desc_stream_q<DEPTH, LA>, 32, SMEM);
    wres = nb > 0 ? nb : 1;
    if (sms <= 0) sms = 148;
  }
  xf::XParamsQ P{};
  P.u = P0.u; P.f = P0.f; P.ve = P0.ve; P.vo = P0.vo; P.un = P0.un; P.re = P0.re; P.ro = P0.ro;
  P.pitch = P0.pitch; P.vp = P0.vp; P.rp = P0.rp; P.M = P0.M; P.c = P0.c; P.k = P0.k; P.ns = P0.ns;
  P.nstrips = (P.M + xf::SWQ - 1) / xf::SWQ;
  const int S = max(1, (sms * wres) / P.nstrips);
  int seg = (P.M + S - 1) / S;
  seg = (seg + 3) / 4 * 4;
  if (seg < 32) seg = 32;
  P.seg = seg;
  const int nitems = P.nstrips * ((P.M + seg - 1) / seg);
  xf::asc_desc_stream_q<DEPTH, LA><<<nitems, 32, SMEM, st>>>(P);
  return cudaGetLastError();
}

// One warp per block: registers are allocated per block, so 1-warp blocks
// fill an SM to the register limit (2- and 4-warp blocks left 3-4 warps per
// SM unused and ran 60 % slower).  Order 2 caps the registers at 128 (16
// warps per SM, no spills); measured alternatives: a 16-row ring (fp64 +5 %,
// fp32 +4 % time), 24 warps per SM with 80 registers (spills: fp64 +50 %,
// fp32 +2 %).
template <class T, int ORDER>
static cudaError_t asc_desc_launch(const xf::XParams<T> &P, cudaStream_t st) {
  if (P.ra) return asc_desc_launch_w<T, ORDER, 8, (ORDER == 2 ? 16 : 1), true>(P, st);
  if constexpr (std::is_same<T, float>::value && ORDER == 2) {
    static const bool pairs = env_flag("MG_XF_PAIRS");
    if (!pairs) return asc_desc_launch_q<3>(P, st);   // lookahead 2 / 3 / 4 rows: 0.459 / 0.457 / 0.461 ms
  }
  return asc_desc_launch_w<T, ORDER, 8, (ORDER == 2 ? 16 : 1)>(P, st);
}

template <class T>
cudaError_t fast2_asc_desc(const S2<T> &vd, const T *u_old, const T *f, int64_t pitch, T *u_new, const S2<T> &d,
                           int M, int order, T c, const Coef<T> &k, const NormSink &ns, cudaStream_t st, bool rev,
                           const D2<T> *ra, const S2<T> *d2) {
  (void)rev;   // the strips are walked top-down; no serpentine variant
  // vector loads of the pair (x, x+1), x even, may touch column M+1: the row
  // pitch must leave a padding word and rows must be 2-word aligned
  if (((uintptr_t)u_old | (uintptr_t)f | (uintptr_t)u_new) % (2 * sizeof(T)) || pitch % 2 || pitch < M + 2)
    return cudaErrorInvalidValue;
  xf::XParams<T> P{};
  P.u = u_old;
  P.f = f;
  P.ve = vd.e;
  P.vo = vd.o;
  P.un = u_new;
  P.re = d.e;
  P.ro = d.o;
  P.pitch = pitch;
  P.vp = vd.pitch;
  P.rp = d.pitch;
  P.M = M;
  P.nstrips = (M + xf::SW - 1) / xf::SW;
  if (ra && d2) {   // the next descent's octave pair D(1) -> A(2) -> D(2) as well
    if (M % 4) return cudaErrorInvalidValue;
    P.ra = ra->p;
    P.rap = ra->pitch;
    P.r2e = d2->e;
    P.r2o = d2->o;
    P.r2p = d2->pitch;
    P.Mc = M / 2;
  }
  P.c = c;
  P.k = k;
  P.ns = ns;
  return order == 2 ? asc_desc_launch<T, 2>(P, st) : asc_desc_launch<T, 4>(P, st);
}

template cudaError_t fast2_asc_desc<float>(const S2<float> &, const float *, const float *, int64_t, float *,
                                           const S2<float> &, int, int, float, const Coef<float> &, const NormSink &,
                                           cudaStream_t, bool, const D2<float> *, const S2<float> *);
template cudaError_t fast2_asc_desc<double>(const S2<double> &, const double *, const double *, int64_t, double *,
                                            const S2<double> &, int, int, double, const Coef<double> &,
                                            const NormSink &, cudaStream_t, bool, const D2<double> *,
                                            const S2<double> *);

}  // namespace mg
