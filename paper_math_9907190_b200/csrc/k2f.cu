// k2f.cu -- 2D TMA tile kernels (sm_100a) for the large levels.
//
// Every kernel is a persistent tile pipeline: each CTA walks the tiles
// blockIdx.x, blockIdx.x + gridDim.x, ...; one elected thread keeps
// STAGES-1 tiles of TMA loads (cp.async.bulk.tensor, out-of-bounds -> 0) in
// flight into a ring of shared-memory stages, one mbarrier per stage, while
// the whole CTA computes the current tile from shared memory.
//
// Thread layout inside a tile (TX = 64 fine columns, TY = 32 rows, 8 warps):
// lane l owns the column pair (x0 + 2l, x0 + 2l + 1), so every shared-memory
// access of the core is a conflict-free 16-byte (fp64) / 8-byte (fp32) vector
// access; warps take rows.  The one-node ring around the tile is computed by
// warps 0-3 in one extra pass.  Node formulas are the shared ones of
// ops2.cuh, so results are bit-identical to the reference kernels.
#include "kernels.h"
#include "ops2.cuh"
#include "tma.cuh"

namespace mg {

constexpr int al128(int n) { return (n + 127) / 128 * 128; }
// TMA (measured on B200): the inner box extent AND the box's starting x
// coordinate must be multiples of 16 bytes (an unaligned start raises
// "illegal instruction").  w16 rounds an extent up; hx<T>(h) is the x halo
// actually loaded for a requested halo h (rounded up to 16 bytes).
template <class T>
constexpr int w16(int n) {
  return (n * (int)sizeof(T) + 15) / 16 * 16 / (int)sizeof(T);
}
template <class T>
constexpr int hx(int h) {
  return (h * (int)sizeof(T) + 15) / 16 * 16 / (int)sizeof(T);
}

template <class T>
struct Vec2;
template <>
struct Vec2<double> {
  using t = double2;
};
template <>
struct Vec2<float> {
  using t = float2;
};
template <class T>
__device__ __forceinline__ void ld2(const T *p, T &a, T &b) {
  auto v = *reinterpret_cast<const typename Vec2<T>::t *>(p);
  a = v.x;
  b = v.y;
}
template <class T>
__device__ __forceinline__ void st2(T *p, T a, T b) {
  typename Vec2<T>::t v;
  v.x = a;
  v.y = b;
  *reinterpret_cast<typename Vec2<T>::t *>(p) = v;
}

// A writable shared-memory tile addressed by global lattice coordinates.
template <class T>
struct STile {
  T *p;
  int ld, ox, oy;
  __device__ __forceinline__ T *at(int x, int y) const { return p + (y - oy) * ld + (x - ox); }
  __device__ __forceinline__ T operator()(int x, int y) const { return *at(x, y); }
};
template <class T>
__device__ __forceinline__ STile<T> stile(unsigned char *base, int ld, int ox, int oy) {
  return STile<T>{(T *)base, ld, ox, oy};
}

// v(x, y) of a split diagonal level held as two shared-memory tiles (E, O).
template <class T>
struct SplitTile2 {
  STile<T> e, o;
  __device__ __forceinline__ T operator()(int x, int y) const { return (x & 1) ? o(x >> 1, y >> 1) : e(x >> 1, y >> 1); }
};

template <class Op>
__global__ void __launch_bounds__(Op::NT) tile_pipeline(const __grid_constant__ typename Op::Params P) {
  constexpr int S = Op::STAGES;
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ __align__(8) uint64_t bar[S];
  pdl_trigger();
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; s++) mbar_init(&bar[s], 1);
    fence_mbar_init();
    Op::prefetch(P);
  }
  __syncthreads();
  pdl_wait();
  typename Op::Acc acc;
  Op::init(acc);
  const int ntiles = P.ntiles;
  if (threadIdx.x == 0)
    for (int j = 0; j + 1 < S; j++) {
      int tj = blockIdx.x + j * gridDim.x;
      if (tj < ntiles) Op::issue(P, P.rev ? ntiles - 1 - tj : tj, smem + j * Op::STAGE, &bar[j]);
    }
  int i = 0;
  for (int t = blockIdx.x; t < ntiles; t += gridDim.x, i++) {
    const int st = i % S;
    if (threadIdx.x == 0) {
      int tn = t + (S - 1) * gridDim.x;
      if (tn < ntiles) {
        int sn = (i + S - 1) % S;   // consumed at iteration i-1 (synchronised below)
        // WAR on the slot is ordered by the __syncthreads that ended its last use
        // (no proxy fence: that would wait for the in-flight TMA loads)
        Op::issue(P, P.rev ? ntiles - 1 - tn : tn, smem + sn * Op::STAGE, &bar[sn]);
      }
    }
    mbar_wait(&bar[st], (i / S) & 1);
    Op::compute(P, P.rev ? ntiles - 1 - t : t, smem + st * Op::STAGE, smem + S * Op::STAGE, acc);
    __syncthreads();
  }
  Op::finish(P, acc);
}

struct NoAcc {};

constexpr int TX = 64, TY = 32, NT = 256, NW = NT / 32;

__device__ __forceinline__ bool inside(int x, int y, int M) { return x >= 1 && y >= 1 && x <= M - 1 && y <= M - 1; }

// ============================================= finest descent: a1 + a2 fused
// r = f - L u on the tile and its ring (shared memory), then Erest2r onto
// E/O of D(1); max|r| over the tile feeds the residual-norm history.
template <class T, int ORDER, int STG>
struct OpDesc2Fine {
  static constexpr int NT = mg::NT, STAGES = STG;
  static constexpr int HU = hx<T>(2), HF = hx<T>(1), HR = hx<T>(1);
  static constexpr int UW = w16<T>(TX + HU + 2), UH = TY + 4, FW = w16<T>(TX + HF + 1), FH = TY + 2;
  static constexpr int RW = w16<T>(TX + HR + 1), RH = TY + 2;
  static constexpr int U_BYTES = UW * UH * sizeof(T), F_BYTES = FW * FH * sizeof(T);
  static constexpr int U_OFF = 0, F_OFF = al128(U_BYTES);
  static constexpr int STAGE = al128(F_OFF + F_BYTES);
  static constexpr int SMEM = STAGES * STAGE + al128(RW * RH * sizeof(T));
  struct Params {
    CUtensorMap tu, tf;
    S2<T> out;
    int M, ntx, ntiles;
    int rev;   // 1: tiles in descending order (Rows2::rev)
    Coef<T> k;
    NormSink ns;
    int ylo, yhi, yo, yh;   // output rows [ylo, yhi); TMA y = global y - yo (full rows) / - yh (half rows)
  };
  struct Acc {
    double mx, ss;   // max |r|, sum r^2 (a16)
  };
  static __device__ void prefetch(const Params &P) {
    tma_prefetch_desc(&P.tu);
    tma_prefetch_desc(&P.tf);
  }
  static __device__ void init(Acc &a) {
    a.mx = 0.0;
    a.ss = 0.0;
  }
  static __device__ void issue(const Params &P, int t, unsigned char *st, uint64_t *bar) {
    int x0 = (t % P.ntx) * TX, y0 = P.ylo + (t / P.ntx) * TY;
    mbar_expect_tx(bar, U_BYTES + F_BYTES);
    tma_load_2d(st + U_OFF, &P.tu, x0 - HU, y0 - 2 - P.yo, bar);
    tma_load_2d(st + F_OFF, &P.tf, x0 - HF, y0 - 1 - P.yo, bar);
  }
  // residual at (xl, y) and (xl + 1, y), 0 outside the interior
  static __device__ __forceinline__ void rpair(const STile<T> &U, const STile<T> &F, int xl, int y, int M,
                                               const Coef<T> &k, T &r0, T &r1) {
    Nb9<T> q0, q1;
    ld2(U.at(xl, y), q0.c, q1.c);
    ld2(U.at(xl, y - 1), q0.s, q1.s);
    ld2(U.at(xl, y + 1), q0.n, q1.n);
    q0.w = U(xl - 1, y);
    q0.e = q1.c;
    q1.w = q0.c;
    q1.e = U(xl + 2, y);
    if (ORDER == 4) {
      q0.ne = q1.n;
      q0.nw = U(xl - 1, y + 1);
      q0.sw = U(xl - 1, y - 1);
      q0.se = q1.s;
      q1.ne = U(xl + 2, y + 1);
      q1.nw = q0.n;
      q1.sw = q0.s;
      q1.se = U(xl + 2, y - 1);
    }
    T f0, f1;
    ld2(F.at(xl, y), f0, f1);
    r0 = inside(xl, y, M) ? res2v<T, ORDER>(q0, f0, k) : (T)0;
    r1 = inside(xl + 1, y, M) ? res2v<T, ORDER>(q1, f1, k) : (T)0;
  }
  static __device__ void compute(const Params &P, int t, unsigned char *st, unsigned char *scr, Acc &acc) {
    const int x0 = (t % P.ntx) * TX, y0 = P.ylo + (t / P.ntx) * TY, M = P.M, yhi = P.yhi;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, xl = x0 + 2 * lane;
    STile<T> U = stile<T>(st + U_OFF, UW, x0 - HU, y0 - 2);
    STile<T> F = stile<T>(st + F_OFF, FW, x0 - HF, y0 - 1);
    STile<T> R = stile<T>(scr, RW, x0 - HR, y0 - 1);
    T r0, r1;
#pragma unroll
    for (int y = y0 + w; y < y0 + TY; y += NW) {
      rpair(U, F, xl, y, M, P.k, r0, r1);
      st2(R.at(xl, y), r0, r1);
      if (y < yhi && P.ns.slots) {   // the residual norm only when a history is wanted
        acc.mx = nmax(nmax(acc.mx, absd(r0)), absd(r1));
        if (P.ns.sums(y)) acc.ss += sq((double)r0) + sq((double)r1);
      }
    }
    if (w < 2) {   // ring rows
      int y = w == 0 ? y0 - 1 : y0 + TY;
      rpair(U, F, xl, y, M, P.k, r0, r1);
      st2(R.at(xl, y), r0, r1);
    } else if (w < 4) {   // ring columns
      int idx = (w - 2) * 32 + lane;
      int x = idx < 32 ? x0 - 1 : x0 + TX, y = y0 + (idx & 31);
      *R.at(x, y) = res2z<T, ORDER>(U, F, x, y, M, P.k);
    }
    __syncthreads();
    const int64_t pitch = P.out.pitch;
#pragma unroll
    for (int b = w; b < TY / 2; b += NW) {
      int y = y0 + 2 * b;
      T rc, rE, rN, ro;
      ld2(R.at(xl, y), rc, rE);
      ld2(R.at(xl, y + 1), rN, ro);
      if (y >= yhi) continue;
      int64_t o = (int64_t)(y / 2) * pitch + xl / 2;
      if (xl >= 2 && xl <= M - 2 && y >= 2 && y <= M - 2)
        P.out.e[o] = erest2r(rc, R(xl - 1, y), R(xl, y - 1), rE, rN);
      if (xl + 1 <= M - 1 && y + 1 <= M - 1) P.out.o[o] = erest2r(ro, rN, rE, R(xl + 2, y + 1), R(xl + 1, y + 2));
    }
  }
  static __device__ void finish(const Params &P, Acc &acc) { block_norm_push<NT>(P.ns, acc.mx, acc.ss); }
};

// ======================================== restriction A(s) -> D(s), s > 1
template <class T, int STG>
struct OpRest2AD {
  static constexpr int NT = mg::NT, STAGES = STG;
  static constexpr int HR = hx<T>(1);
  static constexpr int RW = w16<T>(TX + HR + 1), RH = TY + 2;
  static constexpr int R_BYTES = RW * RH * sizeof(T);
  static constexpr int STAGE = al128(R_BYTES);
  static constexpr int SMEM = STAGES * STAGE;
  struct Params {
    CUtensorMap tr;
    S2<T> out;
    int M, ntx, ntiles;
    int rev;   // 1: tiles in descending order (Rows2::rev)
    int ylo, yhi, yo, yh;
  };
  using Acc = NoAcc;
  static __device__ void prefetch(const Params &P) { tma_prefetch_desc(&P.tr); }
  static __device__ void init(Acc &) {}
  static __device__ void issue(const Params &P, int t, unsigned char *st, uint64_t *bar) {
    int x0 = (t % P.ntx) * TX, y0 = P.ylo + (t / P.ntx) * TY;
    mbar_expect_tx(bar, R_BYTES);
    tma_load_2d(st, &P.tr, x0 - HR, y0 - 1 - P.yo, bar);
  }
  static __device__ void compute(const Params &P, int t, unsigned char *st, unsigned char *, Acc &) {
    const int x0 = (t % P.ntx) * TX, y0 = P.ylo + (t / P.ntx) * TY, M = P.M, yhi = P.yhi;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, xl = x0 + 2 * lane;
    STile<T> R = stile<T>(st, RW, x0 - HR, y0 - 1);
    const int64_t pitch = P.out.pitch;
#pragma unroll
    for (int b = w; b < TY / 2; b += NW) {
      int y = y0 + 2 * b;
      T rc, rE, rN, ro;
      ld2(R.at(xl, y), rc, rE);
      ld2(R.at(xl, y + 1), rN, ro);
      if (y >= yhi) continue;
      int64_t o = (int64_t)(y / 2) * pitch + xl / 2;
      if (xl >= 2 && xl <= M - 2 && y >= 2 && y <= M - 2)
        P.out.e[o] = erest2r(rc, R(xl - 1, y), R(xl, y - 1), rE, rN);
      if (xl + 1 <= M - 1 && y + 1 <= M - 1) P.out.o[o] = erest2r(ro, rN, rE, R(xl + 2, y + 1), R(xl + 1, y + 2));
    }
  }
  static __device__ void finish(const Params &, Acc &) {}
};

// ===================================== restriction D(s) -> A(2s), Erest2b
// coarse tile [X0, X0+TX) x [Y0, Y0+TY) of A(2s)
template <class T, int STG>
struct OpRest2DA {
  static constexpr int NT = mg::NT, STAGES = STG;
  static constexpr int HO = hx<T>(1);
  static constexpr int EW = w16<T>(TX), EH = TY, OW = w16<T>(TX + HO), OH = TY + 1;
  static constexpr int E_BYTES = EW * EH * sizeof(T), O_BYTES = OW * OH * sizeof(T);
  static constexpr int E_OFF = 0, O_OFF = al128(E_BYTES);
  static constexpr int STAGE = al128(O_OFF + O_BYTES);
  static constexpr int SMEM = STAGES * STAGE;
  struct Params {
    CUtensorMap te, to;
    D2<T> out;
    int Mc, ntx, ntiles;
    int rev;   // 1: tiles in descending order (Rows2::rev)
    int ylo, yhi, yo, yh;
  };
  using Acc = NoAcc;
  static __device__ void prefetch(const Params &P) {
    tma_prefetch_desc(&P.te);
    tma_prefetch_desc(&P.to);
  }
  static __device__ void init(Acc &) {}
  static __device__ void issue(const Params &P, int t, unsigned char *st, uint64_t *bar) {
    int X0 = (t % P.ntx) * TX, Y0 = P.ylo + (t / P.ntx) * TY;
    mbar_expect_tx(bar, E_BYTES + O_BYTES);
    tma_load_2d(st + E_OFF, &P.te, X0, Y0 - P.yh, bar);
    tma_load_2d(st + O_OFF, &P.to, X0 - HO, Y0 - 1 - P.yh, bar);
  }
  static __device__ void compute(const Params &P, int t, unsigned char *st, unsigned char *, Acc &) {
    const int X0 = (t % P.ntx) * TX, Y0 = P.ylo + (t / P.ntx) * TY, Mc = P.Mc, yhi = P.yhi;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, X = X0 + 2 * lane;
    STile<T> E = stile<T>(st + E_OFF, EW, X0, Y0);
    STile<T> O = stile<T>(st + O_OFF, OW, X0 - HO, Y0 - 1);
#pragma unroll
    for (int Y = Y0 + w; Y < Y0 + TY; Y += NW) {
      if (Y < 1 || Y > Mc - 1 || Y >= yhi) continue;
      T e0, e1, s0, s1, n0, n1;
      ld2(E.at(X, Y), e0, e1);
      ld2(O.at(X, Y - 1), s0, s1);
      ld2(O.at(X, Y), n0, n1);
      // Erest2b: 4r + (i-1,j-1) + (i+1,j-1) + (i+1,j+1) + (i-1,j+1); neighbour of
      // coarse node X at O(X-1, .) and O(X, .)
      T v0 = erest2b(e0, O(X - 1, Y - 1), s0, n0, O(X - 1, Y));
      T v1 = erest2b(e1, s0, s1, n1, n0);
      bool ok0 = X >= 1 && X <= Mc - 1, ok1 = X + 1 <= Mc - 1;
      if (ok0 && ok1)
        st2(&P.out(X, Y), v0, v1);
      else {
        if (ok0) P.out(X, Y) = v0;
        if (ok1) P.out(X + 1, Y) = v1;
      }
    }
  }
  static __device__ void finish(const Params &, Acc &) {}
};

// ========== restriction D(s) -> A(s+1) -> D(s+1) in one pass (Erest2b, Erest2r)
// Tile [X0, X0+TX) x [Y0, Y0+TYA) of A(s+1): r_A(s+1) is formed (OpRest2DA's
// formula) on the tile and its one-node ring in shared memory, written for the
// tile, and restricted onto D(s+1) (OpRest2AD's formulas) from shared memory.
// QD (fp32): Erest2b takes four columns per item (16-byte vectors of E and O
// from a four-aligned origin, r_A(s+1) scratch two columns further left).
// CF (two-column form): item p of a row forms r_A(s+1) at X0-1+p and X0+32+p (not at the adjacent pair
// X0-1+2p, X0+2p), so consecutive threads read and write consecutive shared-memory words (no 2-way bank
// conflicts), and Erest2r takes its x neighbours from the adjacent lanes by shuffle; same formulas and order.
template <class T, int STG, int NTH, int TYA, bool QD = false, bool CF = false>
struct OpRest2DAD {
  static_assert(!QD || sizeof(T) == 4, "four-column items are the fp32 form");
  static_assert(!(QD && CF), "CF is the two-column form");
  static constexpr int NT = NTH, STAGES = STG, NW = NT / 32, TY = TYA;
  static constexpr int XO = QD ? 2 : 0;   // extra scratch columns on the left (r_A(s+1))
  static constexpr int H1 = hx<T>(1), H2 = hx<T>(2);
  static constexpr int EW = w16<T>(TX + 1 + H1), EH = TY + 2;   // E of r_D(s): [X0-1, X0+TX] x [Y0-1, Y0+TY]
  static constexpr int OW = w16<T>(TX + 1 + H2), OH = TY + 3;   // O of r_D(s): [X0-2, X0+TX] x [Y0-2, Y0+TY]
  static constexpr int E_BYTES = EW * EH * sizeof(T), O_BYTES = OW * OH * sizeof(T);
  static constexpr int E_OFF = 0, O_OFF = al128(E_BYTES);
  static constexpr int STAGE = al128(O_OFF + O_BYTES);
  static constexpr int RSW = TX + 4 + 2 * XO, RSH = TY + 2;     // r_A(s+1) on [X0-2-XO, X0+TX+2+XO) x [Y0-1, Y0+TY]
  static constexpr int SMEM = STAGES * STAGE + al128(RSW * RSH * sizeof(T));
  struct Params {
    CUtensorMap te, to;
    D2<T> ra;    // r_A(s+1)
    S2<T> rd;    // r_D(s+1)
    int Mc, ntx, ntiles;
    int rev;
    int ylo, yhi;   // output rows [ylo, yhi) of A(s+1) (ylo even); whole level: 0, Mc + 1
  };
  using Acc = NoAcc;
  static __device__ void prefetch(const Params &P) {
    tma_prefetch_desc(&P.te);
    tma_prefetch_desc(&P.to);
  }
  static __device__ void init(Acc &) {}
  static __device__ void issue(const Params &P, int t, unsigned char *st, uint64_t *bar) {
    const int X0 = (t % P.ntx) * TX, Y0 = P.ylo + (t / P.ntx) * TY;
    mbar_expect_tx(bar, E_BYTES + O_BYTES);
    tma_load_2d(st + E_OFF, &P.te, X0 - H1, Y0 - 1, bar);
    tma_load_2d(st + O_OFF, &P.to, X0 - H2, Y0 - 2, bar);
  }
  static __device__ void compute(const Params &P, int t, unsigned char *st, unsigned char *scr, Acc &) {
    const int X0 = (t % P.ntx) * TX, Y0 = P.ylo + (t / P.ntx) * TY, Mc = P.Mc, yhi = P.yhi;
    const T *Eb = (const T *)(st + E_OFF), *Ob = (const T *)(st + O_OFF);
    T *Rb = (T *)scr;
    if constexpr (QD) {
      // r_A(s+1) at X = X0-4 .. X0+TX+3 (four per item, X0-1 .. X0+TX needed), Y = Y0-1 .. Y0+TY
      static_assert(H1 == 4 && H2 == 4, "E and O boxes start four columns left of the tile");
      constexpr int RQ = TX / 4 + 2, RR = TY + 2;
#pragma unroll
      for (int k = 0; k < (RQ * RR + NT - 1) / NT; k++) {
        const int i = threadIdx.x + k * NT;
        if (RQ * RR % NT && i >= RQ * RR) break;
        const int p = i % RQ, r = i / RQ, Y = Y0 - 1 + r, X = X0 - 4 + 4 * p;
        // E(X, Y) at Eb[r * EW + X - X0 + H1]; O(X, Y) at Ob[(r + 1) * OW + X - X0 + H2]
        const T *e = Eb + r * EW + 4 * p, *o = Ob + (r + 1) * OW + 4 * p;
        const float4 ec = *reinterpret_cast<const float4 *>(e);
        const float4 on = *reinterpret_cast<const float4 *>(o), os = *reinterpret_cast<const float4 *>(o - OW);
        const T onm = o[-1], osm = o[-1 - OW];
        const bool oky = Y >= 1 && Y <= Mc - 1;
        auto ok = [&](int x) { return oky && x >= 1 && x <= Mc - 1; };
        // Erest2b: E(X,Y), O(X-1,Y-1), O(X,Y-1), O(X,Y), O(X-1,Y)
        float4 v;
        v.x = ok(X) ? erest2b(ec.x, osm, os.x, on.x, onm) : (T)0;
        v.y = ok(X + 1) ? erest2b(ec.y, os.x, os.y, on.y, on.x) : (T)0;
        v.z = ok(X + 2) ? erest2b(ec.z, os.y, os.z, on.z, on.y) : (T)0;
        v.w = ok(X + 3) ? erest2b(ec.w, os.z, os.w, on.w, on.z) : (T)0;
        *reinterpret_cast<float4 *>(Rb + r * RSW + 4 * p) = v;   // scratch column 0 = X0-4
      }
    } else if constexpr (CF) {
    // r_A(s+1) at (X, Y), X = X0-1 .. X0+TX, Y = Y0-1 .. Y0+TY: item p takes X0-1+p and X0-1+p+RP
    constexpr int RP = TX / 2 + 1, RR = TY + 2;
#pragma unroll
    for (int k = 0; k < (RP * RR + NT - 1) / NT; k++) {
      const int i = threadIdx.x + k * NT;
      if (RP * RR % NT && i >= RP * RR) break;
      const int p = i % RP, r = i / RP, Y = Y0 - 1 + r;
      const bool oky = Y >= 1 && Y <= Mc - 1;
#pragma unroll
      for (int q = 0; q < 2; q++) {
        const int X = X0 - 1 + p + RP * q;
        // E(X, Y) at Eb[r * EW + X - X0 + H1]; O(X, Y) at Ob[(r + 1) * OW + X - X0 + H2]
        const T *e = Eb + r * EW + X - X0 + H1, *o = Ob + (r + 1) * OW + X - X0 + H2;
        const T v = (oky && X >= 1 && X <= Mc - 1) ? erest2b(e[0], o[-1 - OW], o[-OW], o[0], o[-1]) : (T)0;
        Rb[r * RSW + X - X0 + 2] = v;
      }
    }
    } else {
    // r_A(s+1) at (X, Y), X = X0-1 .. X0+TX, Y = Y0-1 .. Y0+TY: pairs (X0-1+2p, X0+2p)
    constexpr int RP = TX / 2 + 1, RR = TY + 2;
#pragma unroll
    for (int k = 0; k < (RP * RR + NT - 1) / NT; k++) {
      const int i = threadIdx.x + k * NT;
      if (RP * RR % NT && i >= RP * RR) break;
      const int p = i % RP, r = i / RP, Y = Y0 - 1 + r;
      // E(X, Y) at Eb[r * EW + X - X0 + H1]; O(X, Y) at Ob[(r + 1) * OW + X - X0 + H2]
      const T *e = Eb + r * EW + 2 * p - 1 + H1, *o = Ob + (r + 1) * OW + 2 * p - 1 + H2;
      const bool oky = Y >= 1 && Y <= Mc - 1;
#pragma unroll
      for (int q = 0; q < 2; q++) {
        const int X = X0 - 1 + 2 * p + q;
        // Erest2b: E(X,Y), O(X-1,Y-1), O(X,Y-1), O(X,Y), O(X-1,Y)
        const T v = (oky && X >= 1 && X <= Mc - 1) ? erest2b(e[q], o[q - 1 - OW], o[q - OW], o[q], o[q - 1]) : (T)0;
        Rb[r * RSW + 2 * p + 1 + q] = v;
      }
    }
    }
    __syncthreads();
    // the tile's r_A(s+1) (aligned pairs) and Erest2r onto D(s+1): rows (y, y+1), y = Y0 + 2b
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, xl = X0 + 2 * lane;
    STile<T> R = stile<T>(scr, RSW, X0 - 2 - XO, Y0 - 1);
    const int64_t pitch = P.rd.pitch;
#pragma unroll
    for (int b = w; b < TY / 2; b += NW) {
      const int y = Y0 + 2 * b;
      T rc, rE, rN, ro;
      ld2(R.at(xl, y), rc, rE);
      ld2(R.at(xl, y + 1), rN, ro);
      T rW = (T)0, rEn = (T)0;   // CF: R(xl - 1, y) = lane - 1's rE, R(xl + 2, y + 1) = lane + 1's rN
      if constexpr (CF) {
        rW = __shfl_up_sync(0xffffffffu, rE, 1);
        rEn = __shfl_down_sync(0xffffffffu, rN, 1);
        if (lane == 0) rW = R(xl - 1, y);
        if (lane == 31) rEn = R(xl + 2, y + 1);
      }
      if (y <= Mc - 1 && y < yhi) {   // (yhi even: the pair's second row is inside too)
        const bool ok0 = xl >= 1 && xl <= Mc - 1, ok1 = xl + 1 <= Mc - 1;
        if (y >= 1) {
          if (ok0 && ok1)
            st2(&P.ra(xl, y), rc, rE);
          else {
            if (ok0) P.ra(xl, y) = rc;
            if (ok1) P.ra(xl + 1, y) = rE;
          }
        }
        if (y + 1 <= Mc - 1) {
          if (ok0 && ok1)
            st2(&P.ra(xl, y + 1), rN, ro);
          else {
            if (ok0) P.ra(xl, y + 1) = rN;
            if (ok1) P.ra(xl + 1, y + 1) = ro;
          }
        }
        const int64_t o = (int64_t)(y / 2) * pitch + xl / 2;
        if constexpr (CF) {
          if (xl >= 2 && xl <= Mc - 2 && y >= 2 && y <= Mc - 2) P.rd.e[o] = erest2r(rc, rW, R(xl, y - 1), rE, rN);
          if (xl + 1 <= Mc - 1 && y + 1 <= Mc - 1) P.rd.o[o] = erest2r(ro, rN, rE, rEn, R(xl + 1, y + 2));
        } else {
        if (xl >= 2 && xl <= Mc - 2 && y >= 2 && y <= Mc - 2)
          P.rd.e[o] = erest2r(rc, R(xl - 1, y), R(xl, y - 1), rE, rN);
        if (xl + 1 <= Mc - 1 && y + 1 <= Mc - 1) P.rd.o[o] = erest2r(ro, rN, rE, R(xl + 2, y + 1), R(xl + 1, y + 2));
        }
      }
    }
  }
  static __device__ void finish(const Params &, Acc &) {}
};

// ================================ ascent D(s) from A(2s): Eajacr then Eajacb
// tile in E/O index space [a0, a0+TX) x [b0, b0+TY); the O values are also
// computed on the one-node ring below/left that the E update needs.
template <class T, int STG>
struct OpJac2D {
  static constexpr int NT = mg::NT, STAGES = STG;
  static constexpr int HA = hx<T>(1);
  static constexpr int AW = w16<T>(TX + HA + 1), AH = TY + 2, ROW = w16<T>(TX + HA), ROH = TY + 1,
                       REW = w16<T>(TX), REH = TY;
  static constexpr int A_BYTES = AW * AH * sizeof(T), RO_BYTES = ROW * ROH * sizeof(T),
                       RE_BYTES = REW * REH * sizeof(T);
  static constexpr int A_OFF = 0, RO_OFF = al128(A_BYTES), RE_OFF = RO_OFF + al128(RO_BYTES);
  static constexpr int STAGE = al128(RE_OFF + RE_BYTES);
  static constexpr int VW = w16<T>(TX + HA), VH = TY + 1;
  static constexpr int SMEM = STAGES * STAGE + al128(VW * VH * sizeof(T));
  struct Params {
    CUtensorMap tva, tro, tre;
    S2<T> v;
    int M, ntx, ntiles;
    int rev;   // 1: tiles in descending order (Rows2::rev)
    T c;
    int ylo, yhi, yo, yh;
  };
  using Acc = NoAcc;
  static __device__ void prefetch(const Params &P) {
    tma_prefetch_desc(&P.tva);
    tma_prefetch_desc(&P.tro);
    tma_prefetch_desc(&P.tre);
  }
  static __device__ void init(Acc &) {}
  static __device__ void issue(const Params &P, int t, unsigned char *st, uint64_t *bar) {
    int a0 = (t % P.ntx) * TX, b0 = P.ylo + (t / P.ntx) * TY;
    mbar_expect_tx(bar, A_BYTES + RO_BYTES + RE_BYTES);
    tma_load_2d(st + A_OFF, &P.tva, a0 - HA, b0 - 1 - P.yh, bar);
    tma_load_2d(st + RO_OFF, &P.tro, a0 - HA, b0 - 1 - P.yh, bar);
    tma_load_2d(st + RE_OFF, &P.tre, a0, b0 - P.yh, bar);
  }
  static __device__ void compute(const Params &P, int t, unsigned char *st, unsigned char *scr, Acc &) {
    const int a0 = (t % P.ntx) * TX, b0 = P.ylo + (t / P.ntx) * TY, W = P.M / 2, yhi = P.yhi;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, a = a0 + 2 * lane;
    const T c = P.c;
    STile<T> VA = stile<T>(st + A_OFF, AW, a0 - HA, b0 - 1);
    STile<T> RO = stile<T>(st + RO_OFF, ROW, a0 - HA, b0 - 1);
    STile<T> RE = stile<T>(st + RE_OFF, REW, a0, b0);
    STile<T> V = stile<T>(scr, VW, a0 - HA, b0 - 1);
    const int64_t pitch = P.v.pitch;
    // colour 1 (Eajacr) on O nodes: rows b0-1 .. b0+TY-1, the lane's column pair
    for (int b = b0 - 1 + w; b < b0 + TY; b += NW) {
      T ro0, ro1, va0, va1, vb0, vb1;
      ld2(RO.at(a, b), ro0, ro1);
      ld2(VA.at(a, b), va0, va1);
      ld2(VA.at(a, b + 1), vb0, vb1);
      T va2 = VA(a + 2, b), vb2 = VA(a + 2, b + 1);
      bool okb = b >= 0 && b <= W - 1;
      T v0 = (okb && a <= W - 1) ? jac4(c, ro0, va0, va1, vb1, vb0) : (T)0;
      T v1 = (okb && a + 1 <= W - 1) ? jac4(c, ro1, va1, va2, vb2, vb1) : (T)0;
      st2(V.at(a, b), v0, v1);
      if (okb && b >= b0 && b < yhi) {
        if (a + 1 <= W - 1)
          st2(&P.v.o[(int64_t)b * pitch + a], v0, v1);
        else if (a <= W - 1)
          P.v.o[(int64_t)b * pitch + a] = v0;
      }
    }
    if (w == NW - 1) {   // ring column a0 - 1
      for (int b = b0 - 1 + lane; b < b0 + TY; b += 32) {
        int am = a0 - 1;
        T v = (T)0;
        if (am >= 0 && am <= W - 1 && b >= 0 && b <= W - 1)
          v = jac4(c, RO(am, b), VA(am, b), VA(am + 1, b), VA(am + 1, b + 1), VA(am, b + 1));
        *V.at(am, b) = v;
      }
    }
    __syncthreads();
    // colour 2 (Eajacb) on E nodes, from the new O values (D(s) residual, reading A10)
#pragma unroll
    for (int b = b0 + w; b < b0 + TY; b += NW) {
      if (b < 1 || b > W - 1 || b >= yhi) continue;
      T re0, re1, s0, s1, n0, n1;
      ld2(RE.at(a, b), re0, re1);
      ld2(V.at(a, b - 1), s0, s1);
      ld2(V.at(a, b), n0, n1);
      T sm = V(a - 1, b - 1), nm = V(a - 1, b);
      // Eajacb: (i-1,j-1), (i+1,j-1), (i+1,j+1), (i-1,j+1) -> O(a-1,b-1), O(a,b-1), O(a,b), O(a-1,b)
      T e0 = jac4(c, re0, sm, s0, n0, nm);
      T e1 = jac4(c, re1, s0, s1, n1, n0);
      bool ok0 = a >= 1 && a <= W - 1, ok1 = a + 1 <= W - 1;
      int64_t o = (int64_t)b * pitch + a;
      if (ok0 && ok1)
        st2(&P.v.e[o], e0, e1);
      else {
        if (ok0) P.v.e[o] = e0;
        if (ok1) P.v.e[o + 1] = e1;
      }
    }
  }
  static __device__ void finish(const Params &, Acc &) {}
};

// ===================== ascent A(s) from D(s): green-only nodes, then D nodes
// FINE = true: s = 1, r recomputed from (u_old, f) and u_new = u_old + v is
// written (out of place); FINE = false: r read from r_A(s), v_A(s) written.
template <class T, int ORDER, bool FINE, int STG>
struct OpJac2A {
  static constexpr int NT = mg::NT, STAGES = STG;
  static constexpr int HU = hx<T>(2), HF = hx<T>(1), HV = hx<T>(1), HG = hx<T>(1);
  static constexpr int UW = w16<T>(TX + HU + 2), UH = TY + 4;           // u (FINE)
  static constexpr int FW = w16<T>(TX + HF + 1), FH = TY + 2;           // f (FINE) or r_A (level)
  static constexpr int VW = w16<T>(TX / 2 + HV + 1), VH = TY / 2 + 2;   // E and O of v_D
  static constexpr int U_BYTES = FINE ? UW * UH * (int)sizeof(T) : 0;
  static constexpr int F_BYTES = FW * FH * sizeof(T), V_BYTES = VW * VH * sizeof(T);
  static constexpr int U_OFF = 0, F_OFF = al128(U_BYTES), VE_OFF = F_OFF + al128(F_BYTES),
                       VO_OFF = VE_OFF + al128(V_BYTES);
  static constexpr int STAGE = al128(VO_OFF + V_BYTES);
  // green values, one per column pair: pair p = (x0-2+2p, x0-1+2p), p = 0..TX/2+1;
  // which node of the pair is green follows from the row parity
  static constexpr int GW = TX / 2 + 2, GH = TY + 2;
  static constexpr int SMEM = STAGES * STAGE + al128(GW * GH * sizeof(T));
  struct Params {
    CUtensorMap tu, tf, tve, tvo;   // tu unused when !FINE; tf = f (FINE) or r_A
    D2<T> out;                      // u_new (FINE) or v_A
    int M, ntx, ntiles;
    int rev;   // 1: tiles in descending order (Rows2::rev)
    T c;
    Coef<T> k;
    int ylo, yhi, yo, yh;
  };
  using Acc = NoAcc;
  static __device__ void prefetch(const Params &P) {
    if (FINE) tma_prefetch_desc(&P.tu);
    tma_prefetch_desc(&P.tf);
    tma_prefetch_desc(&P.tve);
    tma_prefetch_desc(&P.tvo);
  }
  static __device__ void init(Acc &) {}
  static __device__ void issue(const Params &P, int t, unsigned char *st, uint64_t *bar) {
    int x0 = (t % P.ntx) * TX, y0 = P.ylo + (t / P.ntx) * TY;
    mbar_expect_tx(bar, U_BYTES + F_BYTES + 2 * V_BYTES);
    if (FINE) tma_load_2d(st + U_OFF, &P.tu, x0 - HU, y0 - 2 - P.yo, bar);
    tma_load_2d(st + F_OFF, &P.tf, x0 - HF, y0 - 1 - P.yo, bar);
    tma_load_2d(st + VE_OFF, &P.tve, x0 / 2 - HV, y0 / 2 - 1 - P.yh, bar);
    tma_load_2d(st + VO_OFF, &P.tvo, x0 / 2 - HV, y0 / 2 - 1 - P.yh, bar);
  }
  static __device__ __forceinline__ T rnode(const Params &P, const STile<T> &U, const STile<T> &F, int x, int y) {
    if (FINE) return res2<T, ORDER>(U, F, x, y, P.k);
    return F(x, y);
  }
  static __device__ void compute(const Params &P, int t, unsigned char *st, unsigned char *scr, Acc &) {
    const int x0 = (t % P.ntx) * TX, y0 = P.ylo + (t / P.ntx) * TY, M = P.M, yhi = P.yhi;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, xl = x0 + 2 * lane, hl = xl >> 1;
    const T c = P.c;
    STile<T> U = stile<T>(st + U_OFF, UW, x0 - HU, y0 - 2);
    STile<T> F = stile<T>(st + F_OFF, FW, x0 - HF, y0 - 1);
    STile<T> VE = stile<T>(st + VE_OFF, VW, x0 / 2 - HV, y0 / 2 - 1);
    STile<T> VO = stile<T>(st + VO_OFF, VW, x0 / 2 - HV, y0 / 2 - 1);
    STile<T> G = stile<T>(scr, GW, 0, y0 - 1);   // G(p, y): the green value of pair p in row y
    const int p = lane + 1;                       // the lane's pair
    // colour 1: the green node of the lane's pair in row y ("similarly for a
    // green grid"): y even -> xl+1, y odd -> xl
    auto green = [&](int y) {
      T g = (T)0;
      if ((y & 1) == 0) {
        int xg = xl + 1;
        if (inside(xg, y, M)) {
          int Y = y >> 1;
          g = jac4(c, rnode(P, U, F, xg, y), VE(hl, Y), VO(hl, Y - 1), VE(hl + 1, Y), VO(hl, Y));
        }
      } else {
        if (inside(xl, y, M)) {
          int Y = (y - 1) >> 1;
          g = jac4(c, rnode(P, U, F, xl, y), VO(hl - 1, Y), VE(hl, Y), VO(hl, Y), VE(hl, Y + 1));
        }
      }
      *G.at(p, y) = g;
    };
#pragma unroll
    for (int y = y0 + w; y < y0 + TY; y += NW) green(y);
    if (w < 2) {
      green(w == 0 ? y0 - 1 : y0 + TY);
    } else if (w < 4) {   // ring columns x0-1 (pair 0) and x0+TX (pair TX/2+1)
      int idx = (w - 2) * 32 + lane;
      int x = idx < 32 ? x0 - 1 : x0 + TX, y = y0 + (idx & 31);
      T g = (T)0;
      if (((x + y) & 1) && inside(x, y, M)) {
        SplitTile2<T> VD{VE, VO};
        g = jac4(c, rnode(P, U, F, x, y), VD(x - 1, y), VD(x, y - 1), VD(x + 1, y), VD(x, y + 1));
      }
      *G.at(idx < 32 ? 0 : TX / 2 + 1, y) = g;
    }
    __syncthreads();
    // colour 2: the D(s) node of the pair from the new green values
#pragma unroll
    for (int y = y0 + w; y < y0 + TY; y += NW) {
      if (y < 1 || y > M - 1 || y >= yhi) continue;
      T g = G(p, y), v0, v1;
      if ((y & 1) == 0) {   // D node at xl, green at xl+1
        v1 = g;
        v0 = inside(xl, y, M) ? jac4(c, rnode(P, U, F, xl, y), G(p - 1, y), G(p, y - 1), g, G(p, y + 1)) : (T)0;
      } else {              // D node at xl+1, green at xl
        v0 = g;
        v1 = inside(xl + 1, y, M) ? jac4(c, rnode(P, U, F, xl + 1, y), g, G(p, y - 1), G(p + 1, y), G(p, y + 1)) : (T)0;
      }
      if (FINE) {   // u <- u + v
        T u0, u1;
        ld2(U.at(xl, y), u0, u1);
        v0 = u0 + v0;
        v1 = u1 + v1;
      }
      bool ok0 = xl >= 1, ok1 = xl + 1 <= M - 1;
      if (ok0 && ok1)
        st2(&P.out(xl, y), v0, v1);
      else {
        if (ok0 && xl <= M - 1) P.out(xl, y) = v0;
        if (ok1) P.out(xl + 1, y) = v1;
      }
    }
  }
  static __device__ void finish(const Params &, Acc &) {}
};

// ============ ascent A(s) then D(s-1) in one pass: v_A(s) never reaches HBM
// The tile is [a0, a0+TX) x [b0, b0+TY) of D(s-1)'s E/O index space, which is
// A(s)'s node space.  v_A(s) is computed (OpJac2A's two colours, same node
// formulas and operand order) on the ring [a0-1, a0+TX] x [b0-1, b0+TY] that
// the O update needs, then OpJac2D's two colours run from shared memory.
// QD (fp32): the two D(s-1) colours take four columns per item (16-byte
// vectors from a four-aligned origin) instead of two: half the items and
// shared-memory instructions of the two largest phases; v_A(s) and O sit two
// columns further left so every vector is aligned.  Same node formulas and
// operand order.
// SPL (two-column form): v_A(s) in shared memory as two column-parity planes (even / odd local columns), so
// the stride-2 accesses of the A(s) colours and the O colour's scalar reads become stride-1 (no 2-way bank
// conflicts); same values, same operand order.
template <class T, int STG, int NTH, int TYA, bool QD = false, bool SPL = false>
struct OpJac2AD {
  static_assert(!QD || sizeof(T) == 4, "four-column items are the fp32 form");
  static_assert(!(QD && SPL), "the split v_A(s) layout is the two-column form");
  static constexpr int NT = NTH, STAGES = STG, NW = NT / 32, TY = TYA;
  static constexpr int XO = QD ? 2 : 0;   // extra scratch columns on the left (v_A(s), O)
  static constexpr int H2 = hx<T>(2), H1 = hx<T>(1);
  static constexpr int RAW = w16<T>(TX + 2 + H2), RAH = TY + 4;            // r_A(s): [a0-2, a0+TX+2) x [b0-2, b0+TY+2)
  static constexpr int VDW = w16<T>(TX / 2 + 2 + H2), VDH = TY / 2 + 4;    // v_D(s) E/O: the D(s) ring of those greens
  static constexpr int ROW = w16<T>(TX + H1), ROH = TY + 1, REW = w16<T>(TX), REH = TY;   // r_D(s-1) O / E
  static constexpr int RA_BYTES = RAW * RAH * sizeof(T), VD_BYTES = VDW * VDH * sizeof(T),
                       RO_BYTES = ROW * ROH * sizeof(T), RE_BYTES = REW * REH * sizeof(T);
  static constexpr int RA_OFF = 0, VE_OFF = al128(RA_BYTES), VO_OFF = VE_OFF + al128(VD_BYTES),
                       RO_OFF = VO_OFF + al128(VD_BYTES), RE_OFF = RO_OFF + al128(RO_BYTES);
  static constexpr int STAGE = al128(RE_OFF + RE_BYTES);
  // scratch: v_A(s) on [a0-2-XO, a0+TX+2+XO) x [b0-2, b0+TY+2); O of v_D(s-1) on [a0-2-XO, a0+TX) x [b0-1, b0+TY)
  static constexpr int VAW = TX + 4 + 2 * XO, VAH = TY + 4, OSW = TX + 2 + XO, OSH = TY + 1;
  static constexpr int VA_BYTES = al128(VAW * VAH * (int)sizeof(T));
  static constexpr int SMEM = STAGES * STAGE + VA_BYTES + al128(OSW * OSH * sizeof(T));
  struct Params {
    CUtensorMap tra, tve, tvo, tro, tre;
    S2<T> v;
    int M, ntx, ntiles;
    int rev;
    T ca, cd;
    int ylo, yhi;   // output rows [ylo, yhi) of D(s-1) E/O = A(s) rows (ylo even); whole level: 0, M/2 + 1
  };
  using Acc = NoAcc;
  static __device__ void prefetch(const Params &P) {
    tma_prefetch_desc(&P.tra);
    tma_prefetch_desc(&P.tve);
    tma_prefetch_desc(&P.tvo);
    tma_prefetch_desc(&P.tro);
    tma_prefetch_desc(&P.tre);
  }
  static __device__ void init(Acc &) {}
  static __device__ void issue(const Params &P, int t, unsigned char *st, uint64_t *bar) {
    const int a0 = (t % P.ntx) * TX, b0 = P.ylo + (t / P.ntx) * TY;
    mbar_expect_tx(bar, RA_BYTES + 2 * VD_BYTES + RO_BYTES + RE_BYTES);
    tma_load_2d(st + RA_OFF, &P.tra, a0 - H2, b0 - 2, bar);
    tma_load_2d(st + VE_OFF, &P.tve, a0 / 2 - H2, b0 / 2 - 2, bar);
    tma_load_2d(st + VO_OFF, &P.tvo, a0 / 2 - H2, b0 / 2 - 2, bar);
    tma_load_2d(st + RO_OFF, &P.tro, a0 - H1, b0 - 1, bar);
    tma_load_2d(st + RE_OFF, &P.tre, a0, b0, bar);
  }
  static __device__ void compute(const Params &P, int t, unsigned char *st, unsigned char *scr, Acc &) {
    const int a0 = (t % P.ntx) * TX, b0 = P.ylo + (t / P.ntx) * TY, W = P.M / 2, yhi = P.yhi;   // A(s) nodes 0 .. W
    STile<T> RA = stile<T>(st + RA_OFF, RAW, a0 - H2, b0 - 2);
    STile<T> VE = stile<T>(st + VE_OFF, VDW, a0 / 2 - H2, b0 / 2 - 2);
    STile<T> VO = stile<T>(st + VO_OFF, VDW, a0 / 2 - H2, b0 / 2 - 2);
    STile<T> RO = stile<T>(st + RO_OFF, ROW, a0 - H1, b0 - 1);
    STile<T> RE = stile<T>(st + RE_OFF, REW, a0, b0);
    STile<T> VA = stile<T>(scr, VAW, a0 - 2 - XO, b0 - 2);
    STile<T> OS = stile<T>(scr + VA_BYTES, OSW, a0 - 2 - XO, b0 - 1);
    const SplitTile2<T> VD{VE, VO};
    const T ca = P.ca, cd = P.cd;
    auto in = [&](int x, int y) { return x >= 1 && y >= 1 && x <= W - 1 && y <= W - 1; };
    // A(s) colour 1: the green node (x + y odd) of each column pair (a0-2+2p, a0-1+2p), rows
    // b0-2 .. b0+TY+1 taken two at a time (even, odd) so every E/O choice is static
    const T *Eb = (const T *)(st + VE_OFF), *Ob = (const T *)(st + VO_OFF), *Rb = (const T *)(st + RA_OFF);
    T *Vb = (T *)scr + XO;   // raw v_A(s) offsets below are relative to column a0-2
    constexpr int GP = TX / 2 + 2, GR = TY / 2 + 2, DP = TX / 2 + 1, DR = TY / 2 + 1;
    constexpr int VH2 = VAW / 2;              // SPL: columns per parity plane
    T *VAe = (T *)scr, *VAo = VAe + VH2 * VAH;   // SPL: local columns 2j and 2j+1 (column a0-2 is local 0)
    if constexpr (SPL) {
#pragma unroll
      for (int k = 0; k < (GP * GR + NT - 1) / NT; k++) {
        const int i = threadIdx.x + k * NT;
        if (GP * GR % NT && i >= GP * GR) break;
        const int p = i % GP, m = i / GP;
        {   // even row, green at the odd local column 2p+1
          const int y = b0 - 2 + 2 * m, x = a0 - 1 + 2 * p;
          const T *e = Eb + (m + 1) * VDW + p + H2, *o = Ob + m * VDW + p + H2 - 1;
          T g = (T)0;
          if (in(x, y)) g = jac4(ca, Rb[2 * m * RAW + 2 * p + 1 - 2 + H2], e[-1], o[0], e[0], o[VDW]);
          VAo[2 * m * VH2 + p] = g;
        }
        {   // odd row, green at the even local column 2p
          const int y = b0 - 1 + 2 * m, x = a0 - 2 + 2 * p;
          const T *e = Eb + (m + 1) * VDW + p - 1 + H2, *o = Ob + (m + 1) * VDW + p - 1 + H2;
          T g = (T)0;
          if (in(x, y)) g = jac4(ca, Rb[(2 * m + 1) * RAW + 2 * p - 2 + H2], o[-1], e[0], o[0], e[VDW]);
          VAe[(2 * m + 1) * VH2 + p] = g;
        }
      }
      __syncthreads();
#pragma unroll
      for (int k = 0; k < (DP * DR + NT - 1) / NT; k++) {
        const int i = threadIdx.x + k * NT;
        if (DP * DR % NT && i >= DP * DR) break;
        const int p = i % DP, m = i / DP;
        {   // odd row R = 2m+1, D node at the odd local column 2p+1: x-1, y-1, x+1, y+1
          const int y = b0 - 1 + 2 * m, x = a0 - 1 + 2 * p, R = 2 * m + 1;
          T v = (T)0;
          if (in(x, y))
            v = jac4(ca, Rb[(2 * m + 1) * RAW + 2 * p + 1 - 2 + H2], VAe[R * VH2 + p], VAo[(R - 1) * VH2 + p],
                     VAe[R * VH2 + p + 1], VAo[(R + 1) * VH2 + p]);
          VAo[R * VH2 + p] = v;
        }
        {   // even row R = 2m+2, D node at the even local column 2p+2
          const int y = b0 + 2 * m, x = a0 + 2 * p, R = 2 * m + 2;
          T v = (T)0;
          if (in(x, y))
            v = jac4(ca, Rb[(2 * m + 2) * RAW + 2 * p - 2 + H2 + 2], VAo[R * VH2 + p], VAe[(R - 1) * VH2 + p + 1],
                     VAo[R * VH2 + p + 1], VAe[(R + 1) * VH2 + p + 1]);
          VAe[R * VH2 + p + 1] = v;
        }
      }
      __syncthreads();
    } else {
#pragma unroll
    for (int k = 0; k < (GP * GR + NT - 1) / NT; k++) {
      const int i = threadIdx.x + k * NT;
      if (GP * GR % NT && i >= GP * GR) break;
      const int p = i % GP, m = i / GP;
      {   // y = b0-2+2m even: green at x = a0-1+2p; E(i-1,J), O(i-1,J-1), E(i,J), O(i-1,J) with i = x/2+1, J = y/2
        const int y = b0 - 2 + 2 * m, x = a0 - 1 + 2 * p;
        const T *e = Eb + (m + 1) * VDW + p + H2, *o = Ob + m * VDW + p + H2 - 1;
        T g = (T)0;
        if (in(x, y)) g = jac4(ca, Rb[2 * m * RAW + 2 * p + 1 - 2 + H2], e[-1], o[0], e[0], o[VDW]);
        Vb[2 * m * VAW + 2 * p + 1] = g;
      }
      {   // y = b0-1+2m odd: green at x = a0-2+2p; O(i-1,J), E(i,J), O(i,J), E(i,J+1) with i = x/2, J = y/2
        const int y = b0 - 1 + 2 * m, x = a0 - 2 + 2 * p;
        const T *e = Eb + (m + 1) * VDW + p - 1 + H2, *o = Ob + (m + 1) * VDW + p - 1 + H2;
        T g = (T)0;
        if (in(x, y)) g = jac4(ca, Rb[(2 * m + 1) * RAW + 2 * p - 2 + H2], o[-1], e[0], o[0], e[VDW]);
        Vb[(2 * m + 1) * VAW + 2 * p] = g;
      }
    }
    __syncthreads();
    // A(s) colour 2: the D(s) node (x + y even) of each pair (a0-1+2p, a0+2p), rows b0-1 .. b0+TY
#pragma unroll
    for (int k = 0; k < (DP * DR + NT - 1) / NT; k++) {
      const int i = threadIdx.x + k * NT;
      if (DP * DR % NT && i >= DP * DR) break;
      const int p = i % DP, m = i / DP;
      {   // y = b0-1+2m odd: x = a0-1+2p
        const int y = b0 - 1 + 2 * m, x = a0 - 1 + 2 * p;
        T *q = Vb + (2 * m + 1) * VAW + 2 * p + 1;
        T v = (T)0;
        if (in(x, y)) v = jac4(ca, Rb[(2 * m + 1) * RAW + 2 * p + 1 - 2 + H2], q[-1], q[-VAW], q[1], q[VAW]);
        *q = v;
      }
      {   // y = b0+2m even: x = a0+2p
        const int y = b0 + 2 * m, x = a0 + 2 * p;
        T *q = Vb + (2 * m + 2) * VAW + 2 * p + 2;
        T v = (T)0;
        if (in(x, y)) v = jac4(ca, Rb[(2 * m + 2) * RAW + 2 * p - 2 + H2 + 2], q[-1], q[-VAW], q[1], q[VAW]);
        *q = v;
      }
    }
    __syncthreads();
    }
    if constexpr (QD) {
      // D(s-1) colour 1 on O nodes, four columns a = a0-4+4g .. a+3 per item (g = 0 .. TX/4), rows b0-1 .. b0+TY-1
      constexpr int QG = TX / 4 + 1;
      const int64_t pitch = P.v.pitch;
#pragma unroll
      for (int k = 0; k < (QG * (TY + 1) + NT - 1) / NT; k++) {
        const int i = threadIdx.x + k * NT;
        if (QG * (TY + 1) % NT && i >= QG * (TY + 1)) break;
        const int b = b0 - 1 + i / QG, a = a0 - 4 + 4 * (i % QG);
        const float4 ro = *reinterpret_cast<const float4 *>(RO.at(a, b));
        const float4 va = *reinterpret_cast<const float4 *>(VA.at(a, b));
        const float4 vb = *reinterpret_cast<const float4 *>(VA.at(a, b + 1));
        const T va4 = VA(a + 4, b), vb4 = VA(a + 4, b + 1);
        const bool okb = b >= 0 && b <= W - 1;
        auto ok = [&](int x) { return okb && x >= a0 - 1 && x >= 0 && x <= W - 1; };
        float4 o;
        o.x = ok(a) ? jac4(cd, ro.x, va.x, va.y, vb.y, vb.x) : (T)0;
        o.y = ok(a + 1) ? jac4(cd, ro.y, va.y, va.z, vb.z, vb.y) : (T)0;
        o.z = ok(a + 2) ? jac4(cd, ro.z, va.z, va.w, vb.w, vb.z) : (T)0;
        o.w = ok(a + 3) ? jac4(cd, ro.w, va.w, va4, vb4, vb.w) : (T)0;
        *reinterpret_cast<float4 *>(OS.at(a, b)) = o;
        if (okb && b >= b0 && b < yhi && a >= a0) {
          T *dst = &P.v.o[(int64_t)b * pitch + a];
          if (a + 3 <= W - 1)
            *reinterpret_cast<float4 *>(dst) = o;
          else {
            if (a <= W - 1) dst[0] = o.x;
            if (a + 1 <= W - 1) dst[1] = o.y;
            if (a + 2 <= W - 1) dst[2] = o.z;
          }
        }
      }
      __syncthreads();
      // D(s-1) colour 2 on E nodes from the new O values: half-warps take rows, lanes four columns
      const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, a = a0 + 4 * (lane & 15);
#pragma unroll
      for (int b = b0 + 2 * w + (lane >> 4); b < b0 + TY; b += 2 * NW) {
        if (b < 1 || b > W - 1 || b >= yhi) continue;
        const float4 re = *reinterpret_cast<const float4 *>(RE.at(a, b));
        const float4 sv = *reinterpret_cast<const float4 *>(OS.at(a, b - 1));
        const float4 nv = *reinterpret_cast<const float4 *>(OS.at(a, b));
        const T sm = OS(a - 1, b - 1), nm = OS(a - 1, b);
        float4 e;
        e.x = jac4(cd, re.x, sm, sv.x, nv.x, nm);
        e.y = jac4(cd, re.y, sv.x, sv.y, nv.y, nv.x);
        e.z = jac4(cd, re.z, sv.y, sv.z, nv.z, nv.y);
        e.w = jac4(cd, re.w, sv.z, sv.w, nv.w, nv.z);
        T *dst = &P.v.e[(int64_t)b * pitch + a];
        if (a >= 1 && a + 3 <= W - 1)
          *reinterpret_cast<float4 *>(dst) = e;
        else {
          if (a >= 1 && a <= W - 1) dst[0] = e.x;
          if (a + 1 >= 1 && a + 1 <= W - 1) dst[1] = e.y;
          if (a + 2 >= 1 && a + 2 <= W - 1) dst[2] = e.z;
          if (a + 3 >= 1 && a + 3 <= W - 1) dst[3] = e.w;
        }
      }
    } else {
      // D(s-1) colour 1 (Eajacr) on O nodes, pairs (a, a+1) = (a0-2+2p, a0-1+2p), rows b0-1 .. b0+TY-1
      const int64_t pitch = P.v.pitch;
#pragma unroll
      for (int k = 0; k < (DP * (TY + 1) + NT - 1) / NT; k++) {
        const int i = threadIdx.x + k * NT;
        if (DP * (TY + 1) % NT && i >= DP * (TY + 1)) break;
        const int b = b0 - 1 + i / DP, a = a0 - 2 + 2 * (i % DP);
        T ro0, ro1, va0, va1, vb0, vb1, va2, vb2;
        ld2(RO.at(a, b), ro0, ro1);
        if constexpr (SPL) {   // local row b - (b0 - 2), even local column 2 (i % DP)
          const int o0 = (b - b0 + 2) * VH2 + i % DP;
          va0 = VAe[o0];
          va1 = VAo[o0];
          vb0 = VAe[o0 + VH2];
          vb1 = VAo[o0 + VH2];
          va2 = VAe[o0 + 1];
          vb2 = VAe[o0 + VH2 + 1];
        } else {
          ld2(VA.at(a, b), va0, va1);
          ld2(VA.at(a, b + 1), vb0, vb1);
          va2 = VA(a + 2, b);
          vb2 = VA(a + 2, b + 1);
        }
        const bool okb = b >= 0 && b <= W - 1;
        const bool ok0 = okb && a >= a0 - 1 && a >= 0 && a <= W - 1, ok1 = okb && a + 1 >= 0 && a + 1 <= W - 1;
        const T v0 = ok0 ? jac4(cd, ro0, va0, va1, vb1, vb0) : (T)0;
        const T v1 = ok1 ? jac4(cd, ro1, va1, va2, vb2, vb1) : (T)0;
        st2(OS.at(a, b), v0, v1);
        if (okb && b >= b0 && b < yhi && a >= a0) {
          if (ok1)
            st2(&P.v.o[(int64_t)b * pitch + a], v0, v1);
          else if (ok0)
            P.v.o[(int64_t)b * pitch + a] = v0;
        }
      }
      __syncthreads();
      // D(s-1) colour 2 (Eajacb) on E nodes, from the new O values
      const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, a = a0 + 2 * lane;
#pragma unroll
      for (int b = b0 + w; b < b0 + TY; b += NW) {
        if (b < 1 || b > W - 1 || b >= yhi) continue;
        T re0, re1, s0, s1, n0, n1;
        ld2(RE.at(a, b), re0, re1);
        ld2(OS.at(a, b - 1), s0, s1);
        ld2(OS.at(a, b), n0, n1);
        T sm, nm;
        if constexpr (SPL) {   // column a-1 is lane - 1's second column (warp-uniform loop: every lane is here)
          sm = __shfl_up_sync(0xffffffffu, s1, 1);
          nm = __shfl_up_sync(0xffffffffu, n1, 1);
          if (lane == 0) {
            sm = OS(a - 1, b - 1);
            nm = OS(a - 1, b);
          }
        } else {
          sm = OS(a - 1, b - 1);
          nm = OS(a - 1, b);
        }
        const T e0 = jac4(cd, re0, sm, s0, n0, nm);
        const T e1 = jac4(cd, re1, s0, s1, n1, n0);
        const bool ok0 = a >= 1 && a <= W - 1, ok1 = a + 1 <= W - 1;
        const int64_t o = (int64_t)b * pitch + a;
        if (ok0 && ok1)
          st2(&P.v.e[o], e0, e1);
        else {
          if (ok0) P.v.e[o] = e0;
          if (ok1) P.v.e[o + 1] = e1;
        }
      }
    }
  }
  static __device__ void finish(const Params &, Acc &) {}
};


// ================================================================= launch

static int num_sms() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

// pipeline depth (TMA stages per CTA); MG_STAGES overrides (2, 3 or 4)
static int stages_cfg() {
  static int s = 0;
  if (!s) {
    s = 2;
    if (const char *e = getenv("MG_STAGES")) s = atoi(e);
    if (s < 2 || s > 4) s = 2;
  }
  return s;
}

template <class Op>
static cudaError_t run_op(const typename Op::Params &P, cudaStream_t st) {
  cudaError_t e = cudaFuncSetAttribute(tile_pipeline<Op>, cudaFuncAttributeMaxDynamicSharedMemorySize, Op::SMEM);
  if (e != cudaSuccess) return note_launch(e);
  // persistent CTAs: never more than can be resident at once (shared memory, registers and threads)
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, tile_pipeline<Op>, Op::NT, Op::SMEM) != cudaSuccess)
    per_sm = (227 * 1024) / (Op::SMEM + 1024);
  if (per_sm < 1) per_sm = 1;
  if (per_sm > 4) per_sm = 4;
  int grid = num_sms() * per_sm;
  if (grid > P.ntiles) grid = P.ntiles;
  if (grid < 1) return cudaSuccess;
  // small levels (one tile per CTA or less): programmatic launch, so the pass's launch and prologue overlap
  // the predecessor's drain (measured -0.2 .. -0.5 % per 8193^2 cycle; MG_PDL_SMALL=0 turns it off)
  static const bool pdl_small = !getenv("MG_PDL_SMALL") || env_flag("MG_PDL_SMALL");
  const bool pdl = pdl_enabled() || (pdl_small && P.ntiles <= grid);
  return note_launch(launch_pdl_if(pdl, tile_pipeline<Op>, dim3(grid), dim3(Op::NT), Op::SMEM, st, P));
}

// run the op with the configured number of stages
template <template <int> class OpOfStages, class Params>
static cudaError_t run_staged(const Params &P, cudaStream_t st) {
  switch (stages_cfg()) {
    case 3: return run_op<OpOfStages<3>>(reinterpret_cast<const typename OpOfStages<3>::Params &>(P), st);
    case 4: return run_op<OpOfStages<4>>(reinterpret_cast<const typename OpOfStages<4>::Params &>(P), st);
    default: return run_op<OpOfStages<2>>(reinterpret_cast<const typename OpOfStages<2>::Params &>(P), st);
  }
}

template <class T>
static bool tm2(CUtensorMap *tm, const void *p, int64_t nx, int64_t ny, int64_t pitch, int bx, int by) {
  uint64_t dims[2] = {(uint64_t)nx, (uint64_t)ny};
  uint32_t box[2] = {(uint32_t)bx, (uint32_t)by};
  const bool ok = encode_tmap(tm, p, sizeof(T), 2, dims, (uint64_t)pitch, 0, box);
  if (!ok) note_launch(cudaErrorInvalidValue);
  return ok;
}

// Row ranges for slab-decomposed (multi-GPU) levels; the default is the
// whole level.  Output rows [ylo, yhi) are written; inputs are local
// allocations whose row 0 is global row fy0 (full-resolution rows) or hy0
// (half rows, E/O and coarser), with frows / hrows rows.
static inline int tiles_y(int ylo, int yhi) { return yhi > ylo ? (yhi - ylo + TY - 1) / TY : 0; }

template <class T, int ORDER>
struct DescS {
  template <int S>
  using op = OpDesc2Fine<T, ORDER, S>;
};

template <class T, int ORDER>
static cudaError_t desc_impl(const T *u, const T *f, int64_t pitch, const S2<T> &d, int M, const Coef<T> &k,
                             const NormSink &ns, cudaStream_t st, const Rows2 &rw) {
  using Op = OpDesc2Fine<T, ORDER, 2>;   // Params do not depend on the stage count
  typename Op::Params P{};
  const int yhi = rw.yhi < 0 ? M : rw.yhi, frows = rw.frows < 0 ? M + 1 : rw.frows;
  if (!tm2<T>(&P.tu, u + (int64_t)rw.fy0 * pitch, M + 1, frows, pitch, Op::UW, Op::UH) ||
      !tm2<T>(&P.tf, f + (int64_t)rw.fy0 * pitch, M + 1, frows, pitch, Op::FW, Op::FH))
    return cudaErrorInvalidValue;
  int ntx = (M + TX - 1) / TX, nty = tiles_y(rw.ylo, yhi);
  P.out = d;
  P.M = M;
  P.ntx = ntx;
  P.ntiles = ntx * nty;
  P.rev = rw.rev;
  P.k = k;
  P.ns = ns;
  P.ylo = rw.ylo;
  P.yhi = yhi;
  P.yo = rw.fy0;
  P.yh = rw.hy0;
  return run_staged<DescS<T, ORDER>::template op>(P, st);
}

template <class T>
cudaError_t fast2_desc_fine(const T *u, const T *f, int64_t pitch, const S2<T> &d, int M, int order, const Coef<T> &k,
                            const NormSink &ns, cudaStream_t st, const Rows2 &rw) {
  return order == 2 ? desc_impl<T, 2>(u, f, pitch, d, M, k, ns, st, rw)
                    : desc_impl<T, 4>(u, f, pitch, d, M, k, ns, st, rw);
}

template <class T, int ORDER, bool FINE>
struct JacAS {
  template <int S>
  using op = OpJac2A<T, ORDER, FINE, S>;
};

template <class T, int ORDER, bool FINE>
static cudaError_t jac_a_impl(const T *u, const T *f_or_r, int64_t pitch_u, int64_t pitch_f, const S2<T> &vd,
                              const D2<T> &out, int M, T c, const Coef<T> &k, cudaStream_t st, const Rows2 &rw) {
  using Op = OpJac2A<T, ORDER, FINE, 2>;
  typename Op::Params P{};
  const int H = M / 2 + 1;
  const int yhi = rw.yhi < 0 ? M : rw.yhi, frows = rw.frows < 0 ? M + 1 : rw.frows,
            hrows = rw.hrows < 0 ? H : rw.hrows;
  if (FINE && !tm2<T>(&P.tu, u + (int64_t)rw.fy0 * pitch_u, M + 1, frows, pitch_u, Op::UW, Op::UH))
    return cudaErrorInvalidValue;
  if (!tm2<T>(&P.tf, f_or_r + (int64_t)rw.fy0 * pitch_f, M + 1, frows, pitch_f, Op::FW, Op::FH) ||
      !tm2<T>(&P.tve, vd.e + (int64_t)rw.hy0 * vd.pitch, H, hrows, vd.pitch, Op::VW, Op::VH) ||
      !tm2<T>(&P.tvo, vd.o + (int64_t)rw.hy0 * vd.pitch, H, hrows, vd.pitch, Op::VW, Op::VH))
    return cudaErrorInvalidValue;
  int ntx = (M + TX - 1) / TX, nty = tiles_y(rw.ylo, yhi);
  P.out = out;
  P.M = M;
  P.ntx = ntx;
  P.ntiles = ntx * nty;
  P.rev = rw.rev;
  P.c = c;
  P.k = k;
  P.ylo = rw.ylo;
  P.yhi = yhi;
  P.yo = rw.fy0;
  P.yh = rw.hy0;
  return run_staged<JacAS<T, ORDER, FINE>::template op>(P, st);
}

template <class T>
cudaError_t fast2_asc_fine(const S2<T> &vd, const T *u_old, const T *f, int64_t pitch, T *u_new, int M, int order, T c,
                           const Coef<T> &k, cudaStream_t st, const Rows2 &rw) {
  D2<T> out{u_new, pitch};
  if (order == 2) return jac_a_impl<T, 2, true>(u_old, f, pitch, pitch, vd, out, M, c, k, st, rw);
  return jac_a_impl<T, 4, true>(u_old, f, pitch, pitch, vd, out, M, c, k, st, rw);
}

template <class T>
cudaError_t fast2_jac_a(const S2<T> &vd, const D2<T> &r, const D2<T> &v, int M, T c, cudaStream_t st, const Rows2 &rw) {
  Coef<T> k{};
  return jac_a_impl<T, 2, false>(nullptr, r.p, 0, r.pitch, vd, v, M, c, k, st, rw);
}

template <class T>
struct RestADS {
  template <int S>
  using op = OpRest2AD<T, S>;
};
template <class T>
struct RestDAS {
  template <int S>
  using op = OpRest2DA<T, S>;
};
template <class T>
struct JacDS {
  template <int S>
  using op = OpJac2D<T, S>;
};

template <class T>
cudaError_t fast2_rest_ad(const D2<T> &r, const S2<T> &d, int M, cudaStream_t st, const Rows2 &rw) {
  using Op = OpRest2AD<T, 2>;
  typename Op::Params P{};
  const int yhi = rw.yhi < 0 ? M : rw.yhi, frows = rw.frows < 0 ? M + 1 : rw.frows;
  if (!tm2<T>(&P.tr, r.p + (int64_t)rw.fy0 * r.pitch, M + 1, frows, r.pitch, Op::RW, Op::RH))
    return cudaErrorInvalidValue;
  int ntx = (M + TX - 1) / TX, nty = tiles_y(rw.ylo, yhi);
  P.out = d;
  P.M = M;
  P.ntx = ntx;
  P.ntiles = ntx * nty;
  P.rev = rw.rev;
  P.ylo = rw.ylo;
  P.yhi = yhi;
  P.yo = rw.fy0;
  P.yh = rw.hy0;
  return run_staged<RestADS<T>::template op>(P, st);
}

template <class T>
cudaError_t fast2_rest_da(const S2<T> &d, const D2<T> &r, int Mc, cudaStream_t st, const Rows2 &rw) {
  using Op = OpRest2DA<T, 2>;
  typename Op::Params P{};
  const int H = Mc + 1;   // E/O arrays of D(s) have M/2 + 1 = Mc + 1 entries per side
  const int yhi = rw.yhi < 0 ? Mc : rw.yhi, hrows = rw.hrows < 0 ? H : rw.hrows;
  if (!tm2<T>(&P.te, d.e + (int64_t)rw.hy0 * d.pitch, H, hrows, d.pitch, Op::EW, Op::EH) ||
      !tm2<T>(&P.to, d.o + (int64_t)rw.hy0 * d.pitch, H, hrows, d.pitch, Op::OW, Op::OH))
    return cudaErrorInvalidValue;
  int ntx = (Mc + TX - 1) / TX, nty = tiles_y(rw.ylo, yhi);
  P.out = r;
  P.Mc = Mc;
  P.ntx = ntx;
  P.ntiles = ntx * nty;
  P.rev = rw.rev;
  P.ylo = rw.ylo;
  P.yhi = yhi;
  P.yo = rw.fy0;
  P.yh = rw.hy0;
  return run_staged<RestDAS<T>::template op>(P, st);
}

template <class T>
cudaError_t fast2_jac_d(const D2<T> &vc, const S2<T> &r, const S2<T> &v, int M, T c, cudaStream_t st,
                        const Rows2 &rw) {
  using Op = OpJac2D<T, 2>;
  typename Op::Params P{};
  const int H = M / 2 + 1, W = M / 2;
  const int yhi = rw.yhi < 0 ? W : rw.yhi, hrows = rw.hrows < 0 ? H : rw.hrows;
  if (!tm2<T>(&P.tva, vc.p + (int64_t)rw.hy0 * vc.pitch, H, hrows, vc.pitch, Op::AW, Op::AH) ||
      !tm2<T>(&P.tro, r.o + (int64_t)rw.hy0 * r.pitch, H, hrows, r.pitch, Op::ROW, Op::ROH) ||
      !tm2<T>(&P.tre, r.e + (int64_t)rw.hy0 * r.pitch, H, hrows, r.pitch, Op::REW, Op::REH))
    return cudaErrorInvalidValue;
  int ntx = (W + TX - 1) / TX, nty = tiles_y(rw.ylo, yhi);
  P.v = v;
  P.M = M;
  P.ntx = ntx;
  P.ntiles = ntx * nty;
  P.rev = rw.rev;
  P.c = c;
  P.ylo = rw.ylo;
  P.yhi = yhi;
  P.yo = rw.fy0;
  P.yh = rw.hy0;
  return run_staged<JacDS<T>::template op>(P, st);
}

template <class T>
cudaError_t fast2_rest_dad(const S2<T> &d, const D2<T> &ra, const S2<T> &rd, int Mc, cudaStream_t st, bool rev,
                           int ylo, int yhi) {
  using Op = OpRest2DAD<T, 2, 576, 32>;
  typename Op::Params P{};
  const int H = Mc + 1;   // E/O arrays of D(s) have Mc + 1 entries per side
  if (!tm2<T>(&P.te, d.e, H, H, d.pitch, Op::EW, Op::EH) || !tm2<T>(&P.to, d.o, H, H, d.pitch, Op::OW, Op::OH))
    return cudaErrorInvalidValue;
  if (yhi < 0) yhi = Mc + 1;
  if (yhi <= ylo) return cudaSuccess;
  P.ylo = ylo;
  P.yhi = yhi;
  const int ntx = (Mc + TX - 1) / TX, nty = (yhi - ylo + Op::TY - 1) / Op::TY;
  P.ra = ra;
  P.rd = rd;
  P.Mc = Mc;
  P.ntx = ntx;
  P.ntiles = ntx * nty;
  P.rev = rev;
  // measured: fp64 576 threads (two CTAs per SM), fp32 256 (four; with 576 the fp32 pass is issue-bound)
  static const int nt = getenv("MG_DA_NT") ? atoi(getenv("MG_DA_NT")) : (sizeof(T) == 4 ? 256 : 576);
  if constexpr (sizeof(T) == 4) {   // fp32: four-column Erest2b items (MG_DA_NOQUAD=1: two-column)
    static const bool quad = !env_flag("MG_DA_NOQUAD");
    using OpQ = OpRest2DAD<T, 2, 256, 32, true>;
    if (quad && nt == 256) return run_op<OpQ>(reinterpret_cast<const typename OpQ::Params &>(P), st);
  }
  if (nt == 256)
    return run_op<OpRest2DAD<T, 2, 256, 32>>(reinterpret_cast<const typename OpRest2DAD<T, 2, 256, 32>::Params &>(P), st);
  if (!env_flag("MG_DA_NOCF")) {   // conflict-free shared-memory columns (MG_DA_NOCF=1: adjacent pairs)
    using OpC = OpRest2DAD<T, 2, 576, 32, false, true>;
    return run_op<OpC>(reinterpret_cast<const typename OpC::Params &>(P), st);
  }
  return run_op<Op>(P, st);
}

template <class T>
cudaError_t fast2_jac_ad(const S2<T> &vd, const D2<T> &ra, T ca, const S2<T> &rd, const S2<T> &v, int M, T cd,
                         cudaStream_t st, bool rev, int ylo, int yhi) {
  using Op = OpJac2AD<T, 2, 512, 32>;   // Params and tile widths do not depend on NT / TY
  typename Op::Params P{};
  const int W = M / 2, H = W + 1, Hs = W / 2 + 1;
  // measured: fp64 576 threads (two CTAs per SM), fp32 256 (four)
  static const int nt = getenv("MG_AD_NT") ? atoi(getenv("MG_AD_NT")) : (sizeof(T) == 4 ? 256 : 576);
  static const int ty = getenv("MG_AD_TY") ? atoi(getenv("MG_AD_TY")) : 16;
  const int tyv = (ty == 32 || ty == 8) ? ty : 16;   // 16 rows: two CTAs per SM (measured best)
  const int ryh = tyv + 4, vdh = tyv / 2 + 4;
  if (!tm2<T>(&P.tra, ra.p, H, H, ra.pitch, Op::RAW, ryh) ||
      !tm2<T>(&P.tve, vd.e, Hs, Hs, vd.pitch, Op::VDW, vdh) ||
      !tm2<T>(&P.tvo, vd.o, Hs, Hs, vd.pitch, Op::VDW, vdh) ||
      !tm2<T>(&P.tro, rd.o, H, H, rd.pitch, Op::ROW, tyv + 1) ||
      !tm2<T>(&P.tre, rd.e, H, H, rd.pitch, Op::REW, tyv))
    return cudaErrorInvalidValue;
  if (yhi < 0) yhi = W + 1;
  if (yhi <= ylo) return cudaSuccess;
  const int ntx = (W + TX - 1) / TX, nty = (yhi - ylo + tyv - 1) / tyv;
  P.v = v;
  P.M = M;
  P.ntx = ntx;
  P.ntiles = ntx * nty;
  P.rev = rev;
  P.ca = ca;
  P.cd = cd;
  P.ylo = ylo;
  P.yhi = yhi;
#define AD_RUN(NTV, TYV) \
  return run_op<OpJac2AD<T, 2, NTV, TYV>>(reinterpret_cast<const typename OpJac2AD<T, 2, NTV, TYV>::Params &>(P), st)
  if constexpr (sizeof(T) == 4) {   // fp32: four-column D(s-1) phases (MG_AD_NOQUAD=1: two-column)
    static const bool quad = !env_flag("MG_AD_NOQUAD");
    using OpQ = OpJac2AD<T, 2, 256, 16, true>;
    if (quad && nt == 256 && tyv == 16) return run_op<OpQ>(reinterpret_cast<const typename OpQ::Params &>(P), st);
  }
  if (tyv == 8) {
    if (nt == 512) AD_RUN(512, 8);
    AD_RUN(256, 8);
  }
  if (tyv == 16) {
    if (nt == 256) AD_RUN(256, 16);
    if (nt == 512) AD_RUN(512, 16);
    if (!env_flag("MG_AD_NOSPLIT"))   // v_A(s) in column-parity planes (MG_AD_NOSPLIT=1: interleaved)
      return run_op<OpJac2AD<T, 2, 576, 16, false, true>>(
          reinterpret_cast<const typename OpJac2AD<T, 2, 576, 16, false, true>::Params &>(P), st);
    AD_RUN(576, 16);   // 18 warps: the O colour (33 x 17 pairs) in one round
  }
  if (nt == 256) AD_RUN(256, 32);
  AD_RUN(512, 32);
#undef AD_RUN
}


#define INSTF(T)                                                                                                   \
  template cudaError_t fast2_desc_fine<T>(const T *, const T *, int64_t, const S2<T> &, int, int, const Coef<T> &, \
                                          const NormSink &, cudaStream_t, const Rows2 &);                          \
  template cudaError_t fast2_asc_fine<T>(const S2<T> &, const T *, const T *, int64_t, T *, int, int, T,           \
                                         const Coef<T> &, cudaStream_t, const Rows2 &);                            \
  template cudaError_t fast2_jac_a<T>(const S2<T> &, const D2<T> &, const D2<T> &, int, T, cudaStream_t,           \
                                      const Rows2 &);                                                              \
  template cudaError_t fast2_rest_ad<T>(const D2<T> &, const S2<T> &, int, cudaStream_t, const Rows2 &);           \
  template cudaError_t fast2_rest_da<T>(const S2<T> &, const D2<T> &, int, cudaStream_t, const Rows2 &);           \
  template cudaError_t fast2_jac_d<T>(const D2<T> &, const S2<T> &, const S2<T> &, int, T, cudaStream_t,           \
                                      const Rows2 &);                                                              \
  template cudaError_t fast2_rest_dad<T>(const S2<T> &, const D2<T> &, const S2<T> &, int, cudaStream_t, bool, int, \
                                        int);                                                                      \
  template cudaError_t fast2_jac_ad<T>(const S2<T> &, const D2<T> &, T, const S2<T> &, const S2<T> &, int, T,      \
                                       cudaStream_t, bool, int, int);

INSTF(float)
INSTF(double)

}  // namespace mg
