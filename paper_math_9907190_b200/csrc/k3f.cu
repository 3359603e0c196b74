// k3f.cu -- 3D TMA plane-streaming kernels (sm_100a) for the finest octave.
//
// A work unit is an xy tile (TX x TY fine nodes) times a z chunk.  The CTA
// streams the unit plane by plane: one elected thread keeps the next planes'
// TMA loads (2D boxes of 3D tensors, out-of-bounds -> 0) in flight into a
// ring of NS shared-memory slots, one mbarrier per slot; the CTA computes
// plane p from the slots of the last few planes (2.5D blocking: only the xy
// halo is re-read, from L2).  Node formulas are the shared ones of
// ops3.cuh, so results are bit-identical to the reference kernels.
#include <cstdlib>

#include "kernels.h"
#include "ops3.cuh"
#include "tma.cuh"

namespace mg {

namespace p3 {

constexpr int al128(int n) { return (n + 127) / 128 * 128; }
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

template <class T>
struct STile {
  T *p;
  int ld, ox, oy;
  __device__ __forceinline__ T *at(int x, int y) const { return p + (y - oy) * ld + (x - ox); }
  __device__ __forceinline__ T operator()(int x, int y) const { return *at(x, y); }
};

// Three consecutive planes (z = zb-1, zb, zb+1) of a field as a 3D accessor.
template <class T>
struct Planes3 {
  STile<T> m, c, p;
  int zb;
  __device__ __forceinline__ T operator()(int x, int y, int z) const {
    return z < zb ? m(x, y) : (z == zb ? c(x, y) : p(x, y));
  }
};
template <class T>
struct Plane1 {
  STile<T> c;
  __device__ __forceinline__ T operator()(int x, int y, int) const { return c(x, y); }
};

}  // namespace p3

using namespace p3;

// --------------------------------------------------------------- pipeline
// Op provides: Unit decode(P, u) with fields pb, pe (plane range of the unit),
// issue(P, unit, p, slot, bar), step(P, unit, p, slots[3] = {L_p, L_{p-1},
// L_{p-2}}, scratch, acc).  Slot indices and mbarrier phases are tracked
// incrementally (no division in the loop).
template <class Op>
__global__ void __launch_bounds__(Op::NT, 1) plane_pipeline(const __grid_constant__ typename Op::Params P) {
  constexpr int NS = Op::NS, D = Op::D;
  static_assert(NS >= D + 2 + Op::LAFTER, "ring too small for the prefetch distance");
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ __align__(8) uint64_t bar[NS];
  pdl_trigger();
  if (threadIdx.x == 0) {
    for (int s = 0; s < NS; s++) mbar_init(&bar[s], 1);
    fence_mbar_init();
    Op::prefetch(P);
  }
  __syncthreads();
  pdl_wait();
  typename Op::Acc acc;
  Op::init(acc);
  const int nunits = P.nunits;
  // producer cursor (used by thread 0 only)
  int pu = blockIdx.x, pp = 0, ps = 0;
  typename Op::Unit pun{};
  auto produce = [&]() {
    Op::issue(P, pun, pp, smem + ps * Op::SLOT, &bar[ps]);
    ps = (ps + 1 == NS) ? 0 : ps + 1;
    if (++pp >= pun.pe) {
      pu += gridDim.x;
      if (pu < nunits) {
        pun = Op::decode(P, pu);
        pp = pun.pb;
      }
    }
  };
  if (threadIdx.x == 0 && pu < nunits) {
    pun = Op::decode(P, pu);
    pp = pun.pb;
    for (int j = 0; j <= D && pu < nunits; j++) produce();
  }
  constexpr int NB = Op::LAFTER + 1;     // slots of loads g, g-1, ..., g-LAFTER
  int sidx[NB];
#pragma unroll
  for (int j = 0; j < NB; j++) sidx[j] = (NS - j) % NS;
  uint32_t phase = 0;
  for (int u = blockIdx.x; u < nunits; u += gridDim.x) {
    const typename Op::Unit un = Op::decode(P, u);
    for (int p = un.pb; p < un.pe; p++) {
      if (threadIdx.x == 0 && pu < nunits) produce();
      mbar_wait(&bar[sidx[0]], phase);
      unsigned char *sl[NB];
#pragma unroll
      for (int j = 0; j < NB; j++) sl[j] = smem + sidx[j] * Op::SLOT;
      Op::step(P, un, p, sl, smem + NS * Op::SLOT, acc);
      __syncthreads();
#pragma unroll
      for (int j = NB - 1; j > 0; j--) sidx[j] = sidx[j - 1];
      if (++sidx[0] == NS) {
        sidx[0] = 0;
        phase ^= 1;
      }
    }
  }
  Op::finish(P, acc);
}

__device__ __forceinline__ bool inside3(int x, int y, int z, int M) {
  return x >= 1 && y >= 1 && z >= 1 && x <= M - 1 && y <= M - 1 && z <= M - 1;
}

// Balanced plane geometry: lane l owns the column pair (x0-2+2l, x0-1+2l), so
// the 32 lanes cover r on [x0-2, x0+62) and the output tile is the TX3 = 60
// columns [x0, x0+60); warp w computes r on row y0-1+w (TY3 + 2 = 16 rows,
// one per warp) and writes the outputs of row y0+w (w < TY3).  Every warp
// does the same work; no separate ring pass.
constexpr int TX3 = 60, TY3 = 14, NT3F = 512, NW3 = NT3F / 32, ZC = 64;
static_assert(TY3 + 2 == NW3, "one r row per warp");

struct Unit3 {
  int x0, y0, zs, ze, pb, pe;
};

// ============================================== finest descent a9 + a10
// r = f - L u (7-point or Efos4) on the tile plus its ring, plane by plane,
// kept in a 4-plane ring; Erred onto the four red sublattices of R(1).
// Load L_p holds u(p+1) and f(p); step p computes r(p) (needs L_{p-2..p})
// and writes the red nodes of plane p-2 (from r(p-3..p-1), computed by
// earlier steps: one barrier per step).
template <class T, int ORDER>
struct OpDesc3Fine {
  static constexpr int NT = NT3F, NS = 7, D = 3, LAFTER = 2;
  static constexpr int HX = hx<T>(3);   // u and f boxes start at x0 - HX (16-byte aligned)
  static constexpr int UW = w16<T>(64 + HX), UH = TY3 + 4, FW = w16<T>(64 + HX), FH = TY3 + 2;
  // r planes de-interleaved: per row [even columns x0-2+2l | odd columns x0-1+2l], l = 0..31
  static constexpr int RH2 = 32, RW = 2 * RH2, RH = TY3 + 2;
  static constexpr int U_BYTES = UW * UH * sizeof(T), F_BYTES = FW * FH * sizeof(T);
  static constexpr int U_OFF = 0, F_OFF = al128(U_BYTES);
  static constexpr int SLOT = al128(F_OFF + F_BYTES);
  static constexpr int RPL = al128(RW * RH * sizeof(T));
  static constexpr int NR = 4;   // r planes p-3 .. p
  static constexpr int SMEM = NS * SLOT + NR * RPL;
  struct Params {
    CUtensorMap tu, tf;
    S3<T> out;
    int M, ntx, nty, nunits;
    int zlo, zhi, fz0;   // output planes [zlo, zhi); global plane of the u/f maps' plane 0
    Coef<T> k;
    NormSink ns;
  };
  using Unit = Unit3;
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
  static __device__ __forceinline__ Unit decode(const Params &P, int u) {
    int tx = u % P.ntx, r = u / P.ntx, ty = r % P.nty, zc = r / P.nty;
    Unit un;
    un.x0 = tx * TX3;
    un.y0 = ty * TY3;
    un.zs = P.zlo + zc * ZC;
    un.ze = min(un.zs + ZC, P.zhi);
    un.pb = un.zs - 3;
    un.pe = un.ze + 2;
    return un;
  }
  static __device__ void issue(const Params &P, const Unit &un, int p, unsigned char *slot, uint64_t *bar) {
    mbar_expect_tx(bar, U_BYTES + F_BYTES);
    tma_load_3d(slot + U_OFF, &P.tu, un.x0 - HX, un.y0 - 2, p + 1 - P.fz0, bar);
    tma_load_3d(slot + F_OFF, &P.tf, un.x0 - HX, un.y0 - 1, p - P.fz0, bar);
  }
  // residuals at (xl, y, z) and (xl+1, y, z); um/uc/up point at u(xl, y) of
  // planes z-1, z, z+1 in their slots, ff at f(xl, y).
  static __device__ __forceinline__ void rpair(const T *um, const T *uc, const T *up, const T *ff, bool in0, bool in1,
                                               const Coef<T> &k, T &r0, T &r1) {
    Nb19<T> a, b;
    ld2(uc, a.c, b.c);
    ld2(uc + UW, a.yp, b.yp);
    ld2(uc - UW, a.ym, b.ym);
    ld2(up, a.zp, b.zp);
    ld2(um, a.zm, b.zm);
    a.xp = b.c;
    a.xm = uc[-1];
    b.xp = uc[2];
    b.xm = a.c;
    if (ORDER == 4) {
      a.xpyp = b.yp;
      a.xmyp = uc[UW - 1];
      a.xmym = uc[-UW - 1];
      a.xpym = b.ym;
      b.xpyp = uc[UW + 2];
      b.xmyp = a.yp;
      b.xmym = a.ym;
      b.xpym = uc[-UW + 2];
      ld2(up + UW, a.ypzp, b.ypzp);
      ld2(um + UW, a.ypzm, b.ypzm);
      ld2(um - UW, a.ymzm, b.ymzm);
      ld2(up - UW, a.ymzp, b.ymzp);
      a.xpzp = b.zp;
      a.xmzp = up[-1];
      a.xmzm = um[-1];
      a.xpzm = b.zm;
      b.xpzp = up[2];
      b.xmzp = a.zp;
      b.xmzm = a.zm;
      b.xpzm = um[2];
    }
    T f0, f1;
    ld2(ff, f0, f1);
    r0 = in0 ? res3v<T, ORDER>(a, f0, k) : (T)0;
    r1 = in1 ? res3v<T, ORDER>(b, f1, k) : (T)0;
  }
  static __device__ void step(const Params &P, const Unit &un, int p, unsigned char *const *sl, unsigned char *scr,
                              Acc &acc) {
    const int M = P.M, lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int x0 = un.x0, y0 = un.y0, xl = x0 - 2 + 2 * lane;
    auto rbase = [&](int z) { return (T *)(scr + (z & (NR - 1)) * RPL); };   // z >= -3: (z & 3) is the slot
    if (p >= un.zs - 1 && p <= un.ze) {
      const int y = y0 - 1 + w;
      const int uoff = (y - (y0 - 2)) * UW + (xl - (x0 - HX)), foff = (y - (y0 - 1)) * FW + (xl - (x0 - HX));
      const T *Up = (const T *)(sl[0] + U_OFF) + uoff, *Uc = (const T *)(sl[1] + U_OFF) + uoff,
              *Um = (const T *)(sl[2] + U_OFF) + uoff;
      const T *F = (const T *)(sl[0] + F_OFF) + foff;
      const bool yin = p >= 1 && p <= M - 1 && y >= 1 && y <= M - 1;
      T r0, r1;
      rpair(Um, Uc, Up, F, yin && xl >= 1 && xl <= M - 1, yin && xl >= 0 && xl + 1 <= M - 1, P.k, r0, r1);
      T *R = rbase(p + 4) + w * RW + lane;
      R[0] = r0;
      R[RH2] = r1;
      // norm: every interior node once -- the tile core on the unit's own planes
      if (P.ns.slots && p >= un.zs && p < un.ze && w >= 1 && w <= TY3 && lane >= 1 && lane <= TX3 / 2) {
        acc.mx = nmax(nmax(acc.mx, absd(r0)), absd(r1));
        if (P.ns.sums(p)) acc.ss += sq((double)r0) + sq((double)r1);
      }
    }
    const int q = p - 2;   // r(q-1), r(q), r(q+1) were completed in earlier steps
    if (w < TY3 && q >= un.zs && q < un.ze && q >= 1 && q <= M - 1) {
      const int y = y0 + w, par = (y + q) & 1, x = xl + par;
      if (lane >= 1 && lane <= TX3 / 2 && x >= 1 && x <= M - 1 && y >= 1 && y <= M - 1) {
        const int row = (w + 1) * RW;   // r row of y
        const T *Rm = rbase(q + 3) + row, *Rc = rbase(q + 4) + row, *Rp = rbase(q + 5) + row;
        const int o = par * RH2 + lane, oo = (1 - par) * RH2 + lane + par;
        // Erred: i+1, i-1, j+1, j-1, k+1, k-1
        T nb[6] = {Rc[oo], Rc[oo - 1], Rc[o + RW], Rc[o - RW], Rp[o], Rm[o]};
        P.out.ref(x, y, q) = erred(Rc[o], nb);
      }
    }
  }
  static __device__ void finish(const Params &P, Acc &acc) { block_norm_push<NT>(P.ns, acc.mx, acc.ss); }
};

// ============================================== finest ascent a15 (s = 1)
// Egprolg on the green-only nodes, Egprolr on the red
// nodes, both with r = f - L u recomputed from u_old, then u_new = u_old + v
// (P:57-60), in one pass.  Load L_p holds u(p+1), f(p) and the two red
// sublattices of fine plane p+1; step p computes the green values G(p) (a
// 4-plane ring) and finishes plane q = p-2 (red values from G(q-1..q+1),
// u_new of every node).  One barrier per step.
template <class T, int ORDER>
struct OpAsc3Fine {
  static constexpr int NT = NT3F, NS = 8, D = 2, LAFTER = 4;
  static constexpr int AL = 16 / (int)sizeof(T);   // TMA x alignment in elements
  static constexpr int HX = hx<T>(3);
  static constexpr int UW = w16<T>(64 + HX), UH = TY3 + 4, FW = w16<T>(64 + HX), FH = TY3 + 2;
  static constexpr int VW = w16<T>(34 + AL - 1), VH = TY3 / 2 + 2;
  static constexpr int U_BYTES = UW * UH * sizeof(T), F_BYTES = FW * FH * sizeof(T), V_BYTES = VW * VH * sizeof(T);
  static constexpr int U_OFF = 0, F_OFF = al128(U_BYTES), V0_OFF = F_OFF + al128(F_BYTES),
                       V1_OFF = V0_OFF + al128(V_BYTES);
  static constexpr int SLOT = al128(V1_OFF + V_BYTES);
  static constexpr int GH2 = 32, GW = 2 * GH2, GR = TY3 + 2;
  static constexpr int GPL = al128(GW * GR * sizeof(T));
  static constexpr int NR = 4;
  static constexpr int SMEM = NS * SLOT + NR * GPL;
  struct Params {
    CUtensorMap tu, tf, tv[4];   // tv: red sublattices C, Fx, Fy, Fz of v_R(1)
    D3<T> out;
    int M, ntx, nty, nunits;
    int zlo, zhi, fz0, hz0;   // output planes [zlo, zhi); global (half-)plane of the maps' plane 0
    T c;
    Coef<T> k;
  };
  using Unit = Unit3;
  struct Acc {};
  static __device__ void prefetch(const Params &P) {
    tma_prefetch_desc(&P.tu);
    tma_prefetch_desc(&P.tf);
    for (int i = 0; i < 4; i++) tma_prefetch_desc(&P.tv[i]);
  }
  static __device__ void init(Acc &) {}
  static __device__ __forceinline__ Unit decode(const Params &P, int u) {
    int tx = u % P.ntx, r = u / P.ntx, ty = r % P.nty, zc = r / P.nty;
    Unit un;
    un.x0 = tx * TX3;
    un.y0 = ty * TY3;
    un.zs = P.zlo + zc * ZC;
    un.ze = min(un.zs + ZC, P.zhi);
    un.pb = un.zs - 3;
    un.pe = un.ze + 2;
    return un;
  }
  static __device__ __forceinline__ int vx0(int x0) { return (x0 / 2 - 2) & ~(AL - 1); }   // V box x origin
  static __device__ void issue(const Params &P, const Unit &un, int p, unsigned char *slot, uint64_t *bar) {
    mbar_expect_tx(bar, U_BYTES + F_BYTES + 2 * V_BYTES);
    tma_load_3d(slot + U_OFF, &P.tu, un.x0 - HX, un.y0 - 2, p + 1 - P.fz0, bar);
    tma_load_3d(slot + F_OFF, &P.tf, un.x0 - HX, un.y0 - 1, p - P.fz0, bar);
    // fine plane z = p+1: even z -> C (even x) and Fz (odd x) at half plane z/2;
    // odd z -> Fx (even x) and Fy (odd x) at half plane (z-1)/2
    const int z = p + 1, hz = z >> 1;
    const CUtensorMap *m0 = (z & 1) ? &P.tv[1] : &P.tv[0];
    const CUtensorMap *m1 = (z & 1) ? &P.tv[2] : &P.tv[3];
    tma_load_3d(slot + V0_OFF, m0, vx0(un.x0), un.y0 / 2 - 1, hz - P.hz0, bar);
    tma_load_3d(slot + V1_OFF, m1, vx0(un.x0), un.y0 / 2 - 1, hz - P.hz0, bar);
  }
  static __device__ void step(const Params &P, const Unit &un, int p, unsigned char *const *sl, unsigned char *scr,
                              Acc &) {
    const int M = P.M, lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int x0 = un.x0, y0 = un.y0, xl = x0 - 2 + 2 * lane, vx = vx0(x0), vy = y0 / 2 - 1;
    const T c = P.c;
    auto gbase = [&](int z) { return (T *)(scr + (z & (NR - 1)) * GPL); };
    // element offset of (x, y) in the u / f boxes, of half-index (a, b) in a V box
    auto uo = [&](int x, int y) { return (y - (y0 - 2)) * UW + (x - (x0 - HX)); };
    auto fo = [&](int x, int y) { return (y - (y0 - 1)) * FW + (x - (x0 - HX)); };
    auto vo = [&](int a, int b) { return (b - vy) * VW + (a - vx); };
    auto vr = [&](unsigned char *slot, int x, int y) {   // v_R at the red node (x, y) of the slot's plane
      return ((const T *)(slot + ((x & 1) ? V1_OFF : V0_OFF)))[vo(x >> 1, y >> 1)];
    };
    auto resid = [&](const T *um, const T *uc, const T *up, T f) {   // pointers at u(x, y) of planes z-1, z, z+1
      Nb19<T> q;
      q.c = uc[0];
      q.xp = uc[1];
      q.xm = uc[-1];
      q.yp = uc[UW];
      q.ym = uc[-UW];
      q.zp = up[0];
      q.zm = um[0];
      if (ORDER == 4) {
        q.xpyp = uc[UW + 1];
        q.xmyp = uc[UW - 1];
        q.xmym = uc[-UW - 1];
        q.xpym = uc[-UW + 1];
        q.ypzp = up[UW];
        q.ypzm = um[UW];
        q.ymzm = um[-UW];
        q.ymzp = up[-UW];
        q.xpzp = up[1];
        q.xmzp = up[-1];
        q.xmzm = um[-1];
        q.xpzm = um[1];
      }
      return res3v<T, ORDER>(q, f, P.k);
    };
    auto jac6 = [&](T r, T v0, T v1, T v2, T v3, T v4, T v5) {
      T t = -(c * r);
      t = t + v0;
      t = t + v1;
      t = t + v2;
      t = t + v3;
      t = t + v4;
      t = t + v5;
      return t * (T)(1.0 / 6.0);
    };
    // ---- colour 1: green values of plane p on rows y0-1 .. y0+TY3
    if (p >= un.zs - 1 && p <= un.ze) {
      const int y = y0 - 1 + w, xg = xl + ((y + p + 1) & 1);
      T g = (T)0;
      if (p >= 1 && p <= M - 1 && y >= 1 && y <= M - 1 && xg >= 1 && xg <= M - 1) {
        const int o = uo(xg, y);
        const T r = resid((const T *)(sl[2] + U_OFF) + o, (const T *)(sl[1] + U_OFF) + o,
                          (const T *)(sl[0] + U_OFF) + o, ((const T *)(sl[0] + F_OFF))[fo(xg, y)]);
        // i+1, i-1, j+1, j-1, k+1, k-1: red neighbours; v_R(p) in L_{p-1}, v_R(p+1) in L_p, v_R(p-1) in L_{p-2}
        g = jac6(r, vr(sl[1], xg + 1, y), vr(sl[1], xg - 1, y), vr(sl[1], xg, y + 1), vr(sl[1], xg, y - 1),
                 vr(sl[0], xg, y), vr(sl[2], xg, y));
      }
      gbase(p + 4)[(xg & 1) * GH2 + w * GW + lane] = g;
    }
    // ---- colour 2 + update on plane q = p-2
    const int q = p - 2;
    if (w < TY3 && lane >= 1 && lane <= TX3 / 2 && q >= un.zs && q < un.ze && q >= 1 && q <= M - 1) {
      const int y = y0 + w;
      if (y >= 1 && y <= M - 1) {
        const int par = (y + q) & 1, xr = xl + par;   // red node of the pair
        const int row = (w + 1) * GW;
        const T *Gm = gbase(q + 3) + row, *Gc = gbase(q + 4) + row, *Gp = gbase(q + 5) + row;
        const int o = par * GH2 + lane, oo = (1 - par) * GH2 + lane + par;
        const T vg = Gc[oo - par];   // the pair's green node (x = xl + 1 - par): index lane in block 1-par
        T vrd = (T)0;
        if (xr >= 1 && xr <= M - 1) {
          const int uoff = uo(xr, y);
          const T r = resid((const T *)(sl[4] + U_OFF) + uoff, (const T *)(sl[3] + U_OFF) + uoff,
                            (const T *)(sl[2] + U_OFF) + uoff, ((const T *)(sl[2] + F_OFF))[fo(xr, y)]);
          vrd = jac6(r, Gc[oo], Gc[oo - 1], Gc[o + GW], Gc[o - GW], Gp[o], Gm[o]);
        }
        T u0, u1;
        ld2((const T *)(sl[3] + U_OFF) + uo(xl, y), u0, u1);
        const T v0 = par ? vg : vrd, v1 = par ? vrd : vg;
        const bool ok0 = xl >= 1, ok1 = xl + 1 <= M - 1;
        T *dst = &P.out(xl, y, q);
        if (ok0 && ok1)
          st2(dst, u0 + v0, u1 + v1);
        else {
          if (ok0 && xl <= M - 1) dst[0] = u0 + v0;
          if (ok1) dst[1] = u1 + v1;
        }
      }
    }
  }
  static __device__ void finish(const Params &, Acc &) {}
};

// ================================================================= launch
template <class Op>
static cudaError_t run_plane(const typename Op::Params &P, cudaStream_t st) {
  cudaError_t e = cudaFuncSetAttribute(plane_pipeline<Op>, cudaFuncAttributeMaxDynamicSharedMemorySize, Op::SMEM);
  if (e != cudaSuccess) return note_launch(e);
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  int per_sm = (227 * 1024) / (Op::SMEM + 1024);
  if (per_sm < 1) per_sm = 1;
  int grid = sms * per_sm;
  if (grid > P.nunits) grid = P.nunits;
  if (grid < 1) return cudaSuccess;
  return note_launch(launch_pdl(plane_pipeline<Op>, dim3(grid), dim3(Op::NT), Op::SMEM, st, P));
}

// map of planes [z0, z0 + nz) of an n x n x (any) field given by its
// virtual plane-0 pointer p (nz = -1: all n planes)
template <class T>
static bool tm3(CUtensorMap *tm, const T *p, int64_t n, int64_t pitch, int64_t plane, int bx, int by, int z0 = 0,
                int nz = -1) {
  if (nz < 0) nz = (int)n;
  p += (int64_t)z0 * plane;
  uint64_t dims[3] = {(uint64_t)n, (uint64_t)n, (uint64_t)nz};
  uint32_t box[3] = {(uint32_t)bx, (uint32_t)by, 1};
  const bool ok = encode_tmap(tm, p, sizeof(T), 3, dims, (uint64_t)pitch, (uint64_t)plane, box);
  if (!ok) note_launch(cudaErrorInvalidValue);
  return ok;
}

static inline void zrange(const ZRange3 &pz, int M, int &zlo, int &zhi) {
  zlo = pz.zlo;
  zhi = pz.zhi < 0 ? M : pz.zhi;
}

template <class T, int ORDER>
static cudaError_t desc3_impl(const T *u, const T *f, int64_t pitch, const S3<T> &rr, int M, const Coef<T> &k,
                              const NormSink &ns, cudaStream_t st, const ZRange3 &pz) {
  using Op = OpDesc3Fine<T, ORDER>;
  typename Op::Params P{};
  int64_t n = M + 1, plane = pitch * n;
  if (!tm3<T>(&P.tu, u, n, pitch, plane, Op::UW, Op::UH, pz.fz0, pz.fplanes) ||
      !tm3<T>(&P.tf, f, n, pitch, plane, Op::FW, Op::FH, pz.fz0, pz.fplanes))
    return cudaErrorInvalidValue;
  P.out = rr;
  P.M = M;
  zrange(pz, M, P.zlo, P.zhi);
  P.fz0 = pz.fz0;
  if (P.zhi <= P.zlo) return cudaSuccess;
  P.ntx = (M + TX3 - 1) / TX3;
  P.nty = (M + TY3 - 1) / TY3;
  P.nunits = P.ntx * P.nty * ((P.zhi - P.zlo + ZC - 1) / ZC);
  P.k = k;
  P.ns = ns;
  return run_plane<Op>(P, st);
}

template <class T>
cudaError_t fast3_desc_fine(const T *u, const T *f, int64_t pitch, const S3<T> &rr, int M, int order, const Coef<T> &k,
                            const NormSink &ns, cudaStream_t st, const ZRange3 &pz) {
  static const bool gen1 = env_flag("MG_K3_GEN1");   // A/B switch to the first-generation kernel
  if (!gen1) return fast3p_desc_fine<T>(u, f, pitch, rr, M, order, k, ns, st, pz);
  return order == 2 ? desc3_impl<T, 2>(u, f, pitch, rr, M, k, ns, st, pz)
                    : desc3_impl<T, 4>(u, f, pitch, rr, M, k, ns, st, pz);
}

template <class T, int ORDER>
static cudaError_t asc3_impl(const S3<T> &vr, const T *u_old, const T *f, int64_t pitch, T *u_new, int M, T c,
                             const Coef<T> &k, cudaStream_t st, const ZRange3 &pz) {
  using Op = OpAsc3Fine<T, ORDER>;
  typename Op::Params P{};
  int64_t n = M + 1, plane = pitch * n;
  if (!tm3<T>(&P.tu, u_old, n, pitch, plane, Op::UW, Op::UH, pz.fz0, pz.fplanes) ||
      !tm3<T>(&P.tf, f, n, pitch, plane, Op::FW, Op::FH, pz.fz0, pz.fplanes))
    return cudaErrorInvalidValue;
  const int sub[4] = {0, 6, 5, 3};   // C, Fx, Fy, Fz
  int64_t H = M / 2 + 1;
  const int hpl = pz.hplanes < 0 ? (int)H : pz.hplanes;
  for (int i = 0; i < 4; i++) {
    uint64_t dims[3] = {(uint64_t)H, (uint64_t)H, (uint64_t)hpl};
    uint32_t box[3] = {(uint32_t)Op::VW, (uint32_t)Op::VH, 1};
    if (!encode_tmap(&P.tv[i], vr.s[sub[i]] + (int64_t)pz.hz0 * vr.plane, sizeof(T), 3, dims, (uint64_t)vr.pitch,
                     (uint64_t)vr.plane, box))
      return cudaErrorInvalidValue;
  }
  P.out = D3<T>{u_new, pitch, plane};
  P.M = M;
  zrange(pz, M, P.zlo, P.zhi);
  P.fz0 = pz.fz0;
  P.hz0 = pz.hz0;
  if (P.zhi <= P.zlo) return cudaSuccess;
  P.ntx = (M + TX3 - 1) / TX3;
  P.nty = (M + TY3 - 1) / TY3;
  P.nunits = P.ntx * P.nty * ((P.zhi - P.zlo + ZC - 1) / ZC);
  P.c = c;
  P.k = k;
  return run_plane<Op>(P, st);
}

template <class T>
cudaError_t fast3_asc_fine(const S3<T> &vr, const T *u_old, const T *f, int64_t pitch, T *u_new, int M, int order, T c,
                           const Coef<T> &k, cudaStream_t st, const ZRange3 &pz) {
  static const bool gen1 = env_flag("MG_K3_GEN1");
  if (!gen1) return fast3p_asc_fine<T>(vr, u_old, f, pitch, u_new, M, order, c, k, st, pz);
  return order == 2 ? asc3_impl<T, 2>(vr, u_old, f, pitch, u_new, M, c, k, st, pz)
                    : asc3_impl<T, 4>(vr, u_old, f, pitch, u_new, M, c, k, st, pz);
}

template cudaError_t fast3_asc_fine<float>(const S3<float> &, const float *, const float *, int64_t, float *, int, int,
                                           float, const Coef<float> &, cudaStream_t, const ZRange3 &);
template cudaError_t fast3_asc_fine<double>(const S3<double> &, const double *, const double *, int64_t, double *, int,
                                            int, double, const Coef<double> &, cudaStream_t, const ZRange3 &);
template cudaError_t fast3_desc_fine<float>(const float *, const float *, int64_t, const S3<float> &, int, int,
                                            const Coef<float> &, const NormSink &, cudaStream_t, const ZRange3 &);
template cudaError_t fast3_desc_fine<double>(const double *, const double *, int64_t, const S3<double> &, int, int,
                                             const Coef<double> &, const NormSink &, cudaStream_t, const ZRange3 &);

}  // namespace mg
