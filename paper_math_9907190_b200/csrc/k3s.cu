// k3s.cu -- the 3D sublattice level passes as TMA plane pipelines (sm_100a,
// fp64): R(s) -> M(s) (Ermagc/Ermagm), M(s) -> G(2s) (Erblu), G(2s) -> M(s)
// (Emprolm then Emprolb, one pass) and M(s) -> R(s) (Erprolr then Erprolm,
// one pass).
//
// Everything is in half-index form (DESIGN.md data layout): the level's
// nodes live in dense parity sublattices C, Fx, Fy, Fz (R), C, B (M) of
// H^3 entries (H = M/2 + 1), and every stencil is a box stencil with offsets
// in {-1, 0, 1}.  Thread (lane l, warp w) owns one half-index column
// (a, b) of the tile and streams it in c (zpipe.cuh): lane -> a, warp -> b.
// The two-colour Jacobi passes compute colour 1 on the tile plus a one-wide
// low ring (the colour-2 stencils only reach a-1, b-1), keep it in a 3-plane
// shared-memory ring and in registers, and finish colour 2 one plane later;
// colour 1 is never written to and re-read from HBM before colour 2.
//
// Every sum keeps the paper's printed order (the b3_* bodies of k3l.cu),
// so the results are bit-identical to the oracle.
#include "zpipe.cuh"

namespace mg {

namespace hs {

// sublattice slots of S3: (x&1) | (y&1)<<1 | (z&1)<<2
constexpr int C = 0, FX = 6, FY = 5, FZ = 3, B = 7;
using T = double;                                      // the fused passes below are fp64 only
constexpr int RW = 32, RH = 16;                        // one value per thread
constexpr int RBOX = RW * RH * 8;                      // 4096 B
constexpr int BOX34 = al128(34 * 17 * 8), BOX36 = al128(36 * 17 * 8);

// TMA x alignment for element type E: box origins must be 16-byte aligned.
// Every origin these passes use is even, i.e. 0 or 2 mod A; an origin X is
// loaded from bx(X) and read back at offset X - bx(X) (<= XP), so a box that
// must hold w columns from X is W(w) wide.  fp64: A = 2, XP = 0 (nothing
// changes); fp32: A = 4, XP = 2.
template <class E>
struct XA {
  static constexpr int A = 16 / (int)sizeof(E), XP = A - 2;
  static constexpr int W(int w) { return (w + XP + A - 1) / A * A; }
  static __device__ __forceinline__ int bx(int x) { return x & ~(A - 1); }
  static __device__ __forceinline__ int ox(int x) { return XP ? (x & (A - 1)) : 0; }
};

struct Sub {
  T *p;
  int64_t pitch, plane;
  __device__ __forceinline__ T &operator()(int a, int b, int c) const {
    return p[(int64_t)c * plane + (int64_t)b * pitch + a];
  }
};
__device__ __forceinline__ Sub sub(const S3<T> &s, int k) { return Sub{s.s[k], s.pitch, s.plane}; }

// half-index interior tests (H = M/2 + 1): 0 <= v <= H-2 and 1 <= v <= H-2
struct HM {
  int H;
  __device__ __forceinline__ bool z0(int v) const { return v >= 0 && v <= H - 2; }
  __device__ __forceinline__ bool z1(int v) const { return v >= 1 && v <= H - 2; }
};

}  // namespace hs

using namespace hs;

// ===================================================== M(s) -> R(s): a14
// Thread column (a, b) = (a0-2+l, b0-1+w); core a in [a0, a0+30) (l >= 2),
// b in [b0, b0+15) (w >= 1); the ring a0-1 / b0-1 is colour 1 only.
// L_j = {C_M(j), B_M(j), r_Fx/Fy/Fz(j-1), r_C(j-2)}.  Step j: faces of plane
// j-1 (Erprolr), corners of plane j-2 (Erprolm).
// E = double or float (E = float: boxes from 16-byte aligned origins, XA).
template <class E, int NW_ = 16>
struct OpJacR3T {
  using T = E;
  using X = XA<E>;
  // NW warps: thread rows b0-1+w cover NW rows, NW-1 of them output rows
  static constexpr int NW = NW_, NTH = 32 * NW, MINB = NW <= 8 ? 2 : 1;
  static constexpr int BW = X::W(34), RWB = X::W(RW);   // C / B box and r box row strides (elements)
  static constexpr int RBE = RWB * NW, RB = RBE * (int)sizeof(T), BX = al128(BW * (NW + 1) * (int)sizeof(T));
  static constexpr int RG = RW * NW;                   // one face array of a ring plane (elements)
  static constexpr int NS = 6, PRO = 2, EPI = 2;
  static constexpr int OC = 0, OB = BX, OR = 2 * BX;   // C box, B box, 4 r boxes (Fx, Fy, Fz, C)
  static constexpr int SLOT = OR + 4 * RB;
  static constexpr int GPL = 3 * RG * (int)sizeof(T);  // face ring plane: Fx | Fy | Fz
  static constexpr int SMEM = NS * SLOT + 3 * GPL;
  struct Params {
    CUtensorMap tc, tb, tr[4];   // C_M, B_M; r_R Fx, Fy, Fz, C
    S3<T> v;                     // v_R(s) out
    Sched sc;
    int H;
    T c1, c2;
  };
  struct State {
    T bo[2];           // own B_M by plane parity
    T fx[2], fy[2], fz[2];   // own faces by plane parity
  };
  struct Ctx {
    bool a0k, a1k, b0k, b1k, core;   // a in [0,H-2] / [1,H-2], b likewise, core column
    int ox;                          // box column offset of the item (X)
    int64_t o0;                      // (a, b) in a plane of the sublattice arrays
  };
  static __device__ void prefetch(const Params &P) {
    tma_prefetch_desc(&P.tc);
    tma_prefetch_desc(&P.tb);
    for (int i = 0; i < 4; i++) tma_prefetch_desc(&P.tr[i]);
  }
  static __device__ void init(State &) {}
  static __device__ void begin(const Params &P, Ctx &C, const Item &it) {
    const int l = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int a = it.x0 - 2 + l, b = it.y0 - 1 + w;
    const HM m{P.H};
    C.a0k = m.z0(a);
    C.a1k = m.z1(a);
    C.b0k = m.z0(b);
    C.b1k = m.z1(b);
    C.core = l >= 2 && w >= 1;
    C.ox = X::ox(it.x0 - 2);
    C.o0 = (int64_t)b * P.v.pitch + a;
  }
  static __device__ void issue(const Params &P, const Item &it, int j, unsigned char *slot, uint64_t *bar) {
    const bool wf = j >= it.zs, wc = j >= it.zs + 2;
    const int x2 = X::bx(it.x0 - 2);
    mbar_expect_tx(bar, 2 * BW * (NW + 1) * (int)sizeof(T) + (wf ? 3 * RB : 0) + (wc ? RB : 0));
    tma_load_3d(slot + OC, &P.tc, x2, it.y0 - 1, j, bar);
    tma_load_3d(slot + OB, &P.tb, X::bx(it.x0 - 4), it.y0 - 2, j, bar);
    if (wf)
      for (int i = 0; i < 3; i++) tma_load_3d(slot + OR + i * RB, &P.tr[i], x2, it.y0 - 1, j - 1, bar);
    if (wc) tma_load_3d(slot + OR + 3 * RB, &P.tr[3], x2, it.y0 - 1, j - 2, bar);
  }
  template <int PH>
  static __device__ __forceinline__ void step(const Params &P, State &S, const Ctx &Cx, const Item &it, int j,
                                              unsigned char *Lc, unsigned char *Lp, unsigned char *gz,
                                              unsigned char *gq, unsigned char *gr) {
    constexpr int Q = PH ^ 1;
    const int l = threadIdx.x & 31, w = threadIdx.x >> 5;
    // C and r boxes start at bx(x0 - 2) (offset ox), the B box at bx(x0 - 4) (offset XP - ox)
    const int oc = w * BW + l + Cx.ox, ob = (w + 1) * BW + l + 2 + X::XP - Cx.ox, orb = w * RWB + l + Cx.ox,
              orr = w * RW + l;
    const HM m{P.H};
    const T bj = ((const T *)(Lc + OB))[ob];   // own B_M(j)
    if (j >= it.zs) {
      const int c = j - 1;
      const T *Cc = (const T *)(Lp + OC) + oc, *Cn = (const T *)(Lc + OC) + oc, *Bc = (const T *)(Lp + OB) + ob;
      const T *R = (const T *)(Lc + OR) + orb;
      const T bc = S.bo[Q], bm = S.bo[PH];   // B(a,b,c), B(a,b,c-1)
      const bool cz0 = m.z0(c), cz1 = m.z1(c);
      T fx, fy, fz;
      {   // Fx (2a, 2b+1, 2c+1): normal x; in-plane (0,+1,+1),(0,+1,-1),(0,-1,-1),(0,-1,+1)
        T nrm = bc;
        nrm = nrm + Bc[-1];
        T t = -(P.c1 * R[0]);
        t = t + (T)2 * nrm;
        t = t + Cn[BW];
        t = t + Cc[BW];
        t = t + Cc[0];
        t = t + Cn[0];
        fx = (Cx.a1k && Cx.b0k && cz0) ? t * (T)0.125 : (T)0;
      }
      {   // Fy (2a+1, 2b, 2c+1): normal y; in-plane (+1,0,+1),(-1,0,+1),(-1,0,-1),(+1,0,-1)
        T nrm = bc;
        nrm = nrm + Bc[-BW];
        T t = -(P.c1 * R[RBE]);
        t = t + (T)2 * nrm;
        t = t + Cn[1];
        t = t + Cn[0];
        t = t + Cc[0];
        t = t + Cc[1];
        fy = (Cx.a0k && Cx.b1k && cz0) ? t * (T)0.125 : (T)0;
      }
      {   // Fz (2a+1, 2b+1, 2c): normal z; in-plane (+1,+1,0),(+1,-1,0),(-1,-1,0),(-1,+1,0)
        T nrm = bc;
        nrm = nrm + bm;
        T t = -(P.c1 * R[2 * RBE]);
        t = t + (T)2 * nrm;
        t = t + Cc[BW + 1];
        t = t + Cc[1];
        t = t + Cc[0];
        t = t + Cc[BW];
        fz = (Cx.a0k && Cx.b0k && cz1) ? t * (T)0.125 : (T)0;
      }
      {
        T *g = (T *)gz + orr;
        g[0] = fx;
        g[RG] = fy;
        g[2 * RG] = fz;
      }
      if (Cx.core && c >= it.zs && c < it.ze) {
        const int64_t o = (int64_t)c * P.v.plane + Cx.o0;
        if (Cx.a1k && Cx.b0k && cz0) __stcs(P.v.s[FX] + o, fx);
        if (Cx.a0k && Cx.b1k && cz0) __stcs(P.v.s[FY] + o, fy);
        if (Cx.a0k && Cx.b0k && cz1) __stcs(P.v.s[FZ] + o, fz);
      }
      // ---- corners of plane q = j-2 from the faces of planes q (own: slot PH, ring gq) and q-1 (slot Q, gr)
      const int q = j - 2;
      if (q >= it.zs && Cx.core && Cx.a1k && Cx.b1k && m.z1(q)) {
        const T *Gx = (const T *)gq + orr, *Gy = Gx + RG, *Gz = Gx + 2 * RG;
        const T *Hx = (const T *)gr + orr, *Hy = Hx + RG;
        T t = -(P.c2 * R[3 * RBE]);
        t = t + S.fz[PH];      // (+1,+1, 0)
        t = t + Gz[-RW];       // (+1,-1, 0)
        t = t + Gz[-RW - 1];   // (-1,-1, 0)
        t = t + Gz[-1];        // (-1,+1, 0)
        t = t + S.fy[PH];      // (+1, 0,+1)
        t = t + S.fy[Q];       // (+1, 0,-1)
        t = t + Hy[-1];        // (-1, 0,-1)
        t = t + Gy[-1];        // (-1, 0,+1)
        t = t + S.fx[PH];      // ( 0,+1,+1)
        t = t + S.fx[Q];       // ( 0,+1,-1)
        t = t + Hx[-RW];       // ( 0,-1,-1)
        t = t + Gx[-RW];       // ( 0,-1,+1)
        __stcs(P.v.s[C] + (int64_t)q * P.v.plane + Cx.o0, t * (T)(1.0 / 12.0));
      }
      S.fx[Q] = fx;
      S.fy[Q] = fy;
      S.fz[Q] = fz;
    }
    S.bo[PH] = bj;
  }
  static __device__ void finish(const Params &, State &) {}
};

// Two half-index rows per thread for the single-colour-ring passes below:
// warp w owns rows b = b0 + 2w (+ ring offset) and the next one.
constexpr int RH2 = 32, RBOX2 = RW * RH2 * 8;                  // 8192 B
constexpr int BOX34x33 = al128(34 * 33 * 8), BOX36x33 = al128(36 * 33 * 8);

// ===================================================== G(2s) -> M(s): a13
// Thread columns (a0-2+l, b0-1+2w+R), R = 0, 1: core a in [a0, a0+30)
// (l >= 2), b in [b0, b0+31) (not the first row of warp 0).
// L_j = {v_G(2s)(j), r_B(j-1), r_C(j-2)}.  Step j: centres of plane j-1
// (Emprolm), corners of plane j-2 from the new centres
// (Emprolb).
template <class E, int NW_ = 16>
struct OpJacM3T {
  using T = E;
  using X = XA<E>;
  // NW warps: thread rows b0-1+2w+R cover 2NW rows, 2NW-1 of them output rows
  static constexpr int NW = NW_, NTH = 32 * NW, MINB = NW <= 8 ? 2 : 1;
  static constexpr int BW = X::W(34), RWB = X::W(RW);   // v_G box and r box row strides (elements)
  static constexpr int GROWS = 2 * NW + 1, RBE2 = RWB * 2 * NW, RB2 = RBE2 * (int)sizeof(T);
  static constexpr int NS = 5, PRO = 1, EPI = 2;
  static constexpr int OG = 0, OR = al128(BW * GROWS * (int)sizeof(T));   // v_G box, r boxes (B, C)
  static constexpr int SLOT = OR + 2 * RB2;
  static constexpr int GPL = RW * 2 * NW * (int)sizeof(T);   // centre ring plane
  static constexpr int SMEM = NS * SLOT + 3 * GPL;
  struct Params {
    CUtensorMap tg, tr[2];   // v_G(2s); r_M B, C
    S3<T> v;                 // v_M(s) out
    Sched sc;
    int H;
    T cc;
  };
  struct State {
    T bo[2][2];   // [plane parity][row] own new centre values
  };
  struct Ctx {
    bool b0k[2], b1k[2], core[2];   // per row: (a, b) in [0,H-2]^2 / [1,H-2]^2, core node
    int ox;                         // box column offset of the item (X)
    T *pb[2], *pc[2];               // per row: v_M B / C at (a, b) of plane 0 (+ c * plane per step)
  };
  static __device__ void prefetch(const Params &P) {
    tma_prefetch_desc(&P.tg);
    tma_prefetch_desc(&P.tr[0]);
    tma_prefetch_desc(&P.tr[1]);
  }
  static __device__ void init(State &) {}
  static __device__ void begin(const Params &P, Ctx &C, const Item &it) {
    const int l = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int a = it.x0 - 2 + l;
    const HM m{P.H};
    C.ox = X::ox(it.x0 - 2);
#pragma unroll
    for (int R = 0; R < 2; R++) {
      const int b = it.y0 - 1 + 2 * w + R;
      C.b0k[R] = m.z0(a) && m.z0(b);
      C.b1k[R] = m.z1(a) && m.z1(b);
      C.core[R] = l >= 2 && (w >= 1 || R == 1);
      const int64_t o = (int64_t)b * P.v.pitch + a;
      C.pb[R] = P.v.s[hs::B] + o;
      C.pc[R] = P.v.s[hs::C] + o;
    }
  }
  static __device__ void issue(const Params &P, const Item &it, int j, unsigned char *slot, uint64_t *bar) {
    const bool wf = j >= it.zs, wc = j >= it.zs + 2;
    const int x2 = X::bx(it.x0 - 2);
    mbar_expect_tx(bar, BW * GROWS * (int)sizeof(T) + (wf ? RB2 : 0) + (wc ? RB2 : 0));
    tma_load_3d(slot + OG, &P.tg, x2, it.y0 - 1, j, bar);
    if (wf) tma_load_3d(slot + OR, &P.tr[0], x2, it.y0 - 1, j - 1, bar);
    if (wc) tma_load_3d(slot + OR + RB2, &P.tr[1], x2, it.y0 - 1, j - 2, bar);
  }
  template <int PH>
  static __device__ __forceinline__ void step(const Params &P, State &S, const Ctx &Cx, const Item &it, int j,
                                              unsigned char *Lc, unsigned char *Lp, unsigned char *gz,
                                              unsigned char *gq, unsigned char *gr) {
    constexpr int Q = PH ^ 1;
    if (j < it.zs) return;
    const int l = threadIdx.x & 31, w = threadIdx.x >> 5;
    const HM m{P.H};
    const int c = j - 1, q = j - 2;
    const bool czin = m.z0(c), cout = c >= it.zs && c < it.ze, qok = q >= it.zs && m.z1(q);
    T bn[2];
#pragma unroll
    for (int R = 0; R < 2; R++) {
      const int og = (2 * w + R) * BW + l + Cx.ox, orb = (2 * w + R) * RWB + l + Cx.ox, orr = (2 * w + R) * RW + l;
      const T *Gc = (const T *)(Lp + OG) + og, *Gn = (const T *)(Lc + OG) + og;   // v_G planes c, c+1
      const T *Rb = (const T *)(Lc + OR) + orb;
      T t = -(P.cc * Rb[0]);
      t = t + Gn[BW + 1];   // (+,+,+)
      t = t + Gc[BW + 1];   // (+,+,-)
      t = t + Gn[1];        // (+,-,+)
      t = t + Gc[1];        // (+,-,-)
      t = t + Gn[BW];       // (-,+,+)
      t = t + Gc[BW];       // (-,+,-)
      t = t + Gn[0];        // (-,-,+)
      t = t + Gc[0];        // (-,-,-)
      const bool ok = Cx.b0k[R] && czin;
      bn[R] = ok ? t * (T)0.125 : (T)0;
      ((T *)gz)[orr] = bn[R];
      if (ok && Cx.core[R] && cout) __stcs(Cx.pb[R] + (int64_t)c * P.v.plane, bn[R]);
      if (qok && Cx.core[R] && Cx.b1k[R]) {
        const T *G0 = (const T *)gq + orr, *G1 = (const T *)gr + orr;   // centres of planes q, q-1
        T u = -(P.cc * Rb[RBE2]);
        u = u + S.bo[PH][R];     // (a, b, c)
        u = u + S.bo[Q][R];      // (a, b, c-1)
        u = u + G0[-RW];         // (a, b-1, c)
        u = u + G1[-RW];         // (a, b-1, c-1)
        u = u + G0[-1];          // (a-1, b, c)
        u = u + G1[-1];          // (a-1, b, c-1)
        u = u + G0[-RW - 1];     // (a-1, b-1, c)
        u = u + G1[-RW - 1];     // (a-1, b-1, c-1)
        __stcs(Cx.pc[R] + (int64_t)q * P.v.plane, u * (T)0.125);
      }
    }
    S.bo[Q][0] = bn[0];
    S.bo[Q][1] = bn[1];
  }
  static __device__ void finish(const Params &, State &) {}
};

// ===================================================== R(s) -> M(s): a11
// Thread columns (a0+l, b0+2w+R), tiles 32 x 32, no ring.
// L_j = {Fx(j), Fy(j), Fz(j+1), C_R(j)}; step j: corners (Ermagc)
// and centres (Ermagm) of plane j.  a0 is a multiple of 32, so
// the halo boxes (origin a0-2) sit at offset XP after their aligned origin.
template <class E>
struct OpRestRM3 {
  using T = E;
  using X = XA<E>;
  static constexpr int NS = 4, PRO = 1, EPI = 0;   // 2 planes ahead: measured 0.133 vs 0.143 ms (4 ahead)
  static constexpr int WX = X::W(36), WY = X::W(34);   // Fx box, Fy / Fz box row strides (elements)
  static constexpr int BXB = al128(WX * 33 * (int)sizeof(T)), BYB = al128(WY * 33 * (int)sizeof(T));
  static constexpr int RBB = RW * RH2 * (int)sizeof(T);
  static constexpr int OX = 0, OY = BXB, OZ = BXB + BYB, OCR = BXB + 2 * BYB;
  static constexpr int SLOT = OCR + RBB;
  static constexpr int GPL = 0;
  static constexpr int SMEM = NS * SLOT + 128;
  struct Params {
    CUtensorMap tx, ty, tz, tc;   // r_R Fx, Fy, Fz, C
    S3<T> out;                    // r_M(s): C, B
    Sched sc;
    int H;
  };
  struct State {};
  struct Ctx {
    bool k0[2], k1[2];   // per row: (a, b) in [0,H-2]^2 / [1,H-2]^2
  };
  static __device__ void prefetch(const Params &P) {
    tma_prefetch_desc(&P.tx);
    tma_prefetch_desc(&P.ty);
    tma_prefetch_desc(&P.tz);
    tma_prefetch_desc(&P.tc);
  }
  static __device__ void init(State &) {}
  static __device__ void begin(const Params &P, Ctx &C, const Item &it) {
    const int l = threadIdx.x & 31, w = threadIdx.x >> 5;
    const HM m{P.H};
#pragma unroll
    for (int R = 0; R < 2; R++) {
      C.k0[R] = m.z0(it.x0 + l) && m.z0(it.y0 + 2 * w + R);
      C.k1[R] = m.z1(it.x0 + l) && m.z1(it.y0 + 2 * w + R);
    }
  }
  static __device__ void issue(const Params &P, const Item &it, int j, unsigned char *slot, uint64_t *bar) {
    const bool wc = j >= it.zs;
    const int x2 = it.x0 - 2 - X::XP;
    mbar_expect_tx(bar, (WX + 2 * WY) * 33 * (int)sizeof(T) + (wc ? RBB : 0));
    tma_load_3d(slot + OX, &P.tx, x2, it.y0 - 1, j, bar);
    tma_load_3d(slot + OY, &P.ty, x2, it.y0, j, bar);
    tma_load_3d(slot + OZ, &P.tz, x2, it.y0 - 1, j + 1, bar);
    if (wc) tma_load_3d(slot + OCR, &P.tc, it.x0, it.y0, j, bar);
  }
  template <int PH>
  static __device__ __forceinline__ void step(const Params &P, State &, const Ctx &Cx, const Item &it, int j,
                                              unsigned char *Lc, unsigned char *Lp, unsigned char *,
                                              unsigned char *, unsigned char *) {
    if (j < it.zs) return;
    const int l = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int a = it.x0 + l, c = j;
    const HM m{P.H};
    const bool c0 = m.z0(c), c1 = m.z1(c);
#pragma unroll
    for (int R = 0; R < 2; R++) {
      const int b = it.y0 + 2 * w + R, rr = 2 * w + R;
      const int ox = (rr + 1) * WX + l + 2 + X::XP, oy = rr * WY + l + 2 + X::XP, oz = (rr + 1) * WY + l + 2 + X::XP;
      const T *Xc = (const T *)(Lc + OX) + ox, *Xp = (const T *)(Lp + OX) + ox;   // Fx planes c, c-1
      const T *Yc = (const T *)(Lc + OY) + oy, *Yp = (const T *)(Lp + OY) + oy;   // Fy planes c, c-1
      const T *Zn = (const T *)(Lc + OZ) + oz, *Zc = (const T *)(Lp + OZ) + oz;   // Fz planes c+1, c
      const int64_t o = (int64_t)c * P.out.plane + (int64_t)b * P.out.pitch + a;
      if (Cx.k1[R] && c1) {
        T t = (T)12 * ((const T *)(Lc + OCR))[rr * RW + l];
        t = t + Zc[0];          // (+1,+1, 0)
        t = t + Zc[-WY];        // (+1,-1, 0)
        t = t + Zc[-WY - 1];    // (-1,-1, 0)
        t = t + Zc[-1];         // (-1,+1, 0)
        t = t + Yc[0];          // (+1, 0,+1)
        t = t + Yp[0];          // (+1, 0,-1)
        t = t + Yp[-1];         // (-1, 0,-1)
        t = t + Yc[-1];         // (-1, 0,+1)
        t = t + Xc[0];          // ( 0,+1,+1)
        t = t + Xp[0];          // ( 0,+1,-1)
        t = t + Xp[-WX];        // ( 0,-1,-1)
        t = t + Xc[-WX];        // ( 0,-1,+1)
        __stcs(P.out.s[C] + o, t * (T)(1.0 / 24.0));
      }
      if (Cx.k0[R] && c0) {
        // centre (2a+1, 2b+1, 2c+1): i+1, i-1, j+1, j-1, k+1, k-1
        T t = Xc[1];
        t = t + Xc[0];
        t = t + Yc[WY];
        t = t + Yc[0];
        t = t + Zn[0];
        t = t + Zc[0];
        __stcs(P.out.s[B] + o, t * (T)(1.0 / 6.0));
      }
    }
  }
  static __device__ void finish(const Params &, State &) {}
};

// ===================================================== M(s) -> G(2s): a12
// Erblu.  Tiles 32 x 32, two rows per thread.
// L_j = {C_M(j), B_M(j)}; step j: plane j.
template <class E>
struct OpRestMG3 {
  using T = E;
  using X = XA<E>;
  static constexpr int NS = 6, PRO = 1, EPI = 0;   // 4 planes ahead: measured 0.0737 vs 0.0761 ms (10 ahead)
  static constexpr int WB = X::W(34);              // B box row stride (elements)
  static constexpr int RBB = RW * RH2 * (int)sizeof(T);
  static constexpr int OB = 0, OCM = al128(WB * 33 * (int)sizeof(T));
  static constexpr int SLOT = OCM + RBB;
  static constexpr int GPL = 0;
  static constexpr int SMEM = NS * SLOT + 128;
  struct Params {
    CUtensorMap tb, tc;   // r_M B, C
    D3<T> out;            // r_G(2s)
    Sched sc;
    int H;
  };
  struct State {};
  struct Ctx {
    bool k1[2];
  };
  static __device__ void prefetch(const Params &P) {
    tma_prefetch_desc(&P.tb);
    tma_prefetch_desc(&P.tc);
  }
  static __device__ void init(State &) {}
  static __device__ void begin(const Params &P, Ctx &C, const Item &it) {
    const int l = threadIdx.x & 31, w = threadIdx.x >> 5;
    const HM m{P.H};
    C.k1[0] = m.z1(it.x0 + l) && m.z1(it.y0 + 2 * w);
    C.k1[1] = m.z1(it.x0 + l) && m.z1(it.y0 + 2 * w + 1);
  }
  static __device__ void issue(const Params &P, const Item &it, int j, unsigned char *slot, uint64_t *bar) {
    const bool wc = j >= it.zs;
    mbar_expect_tx(bar, WB * 33 * (int)sizeof(T) + (wc ? RBB : 0));
    tma_load_3d(slot + OB, &P.tb, it.x0 - 2 - X::XP, it.y0 - 1, j, bar);
    if (wc) tma_load_3d(slot + OCM, &P.tc, it.x0, it.y0, j, bar);
  }
  template <int PH>
  static __device__ __forceinline__ void step(const Params &P, State &, const Ctx &Cx, const Item &it, int j,
                                              unsigned char *Lc, unsigned char *Lp, unsigned char *,
                                              unsigned char *, unsigned char *) {
    if (j < it.zs) return;
    const int l = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int a = it.x0 + l, c = j;
    const HM m{P.H};
    if (!m.z1(c)) return;
#pragma unroll
    for (int R = 0; R < 2; R++) {
      if (!Cx.k1[R]) continue;
      const int b = it.y0 + 2 * w + R, rr = 2 * w + R;
      const int ob = (rr + 1) * WB + l + 2 + X::XP;
      const T *Bc = (const T *)(Lc + OB) + ob, *Bp = (const T *)(Lp + OB) + ob;   // B planes c, c-1
      T t = (T)8 * ((const T *)(Lc + OCM))[rr * RW + l];
      t = t + Bc[0];          // (+,+,+)
      t = t + Bp[0];          // (+,+,-)
      t = t + Bc[-WB];        // (+,-,+)
      t = t + Bp[-WB];        // (+,-,-)
      t = t + Bc[-1];         // (-,+,+)
      t = t + Bp[-1];         // (-,+,-)
      t = t + Bc[-WB - 1];    // (-,-,+)
      t = t + Bp[-WB - 1];    // (-,-,-)
      __stcs(&P.out(a, b, c), t * (T)(1.0 / 16.0));
    }
  }
  static __device__ void finish(const Params &, State &) {}
};

// ================================= G(2s) -> M(s) -> R(s): a13 + a14 fused
// Emprolm, Emprolb, Erprolr, Erprolm in one pass:
// v_M(s) never goes to HBM.  Thread (l, w) owns the half-index column
// (a0-2+l, b0-2+w); the stages need ever smaller regions (centres B on all
// 32 x 16 columns, corners C_M on a >= a0-1, b >= b0-1, faces on
// [a0-1, a0+28] x [b0-1, b0+12], corners C_R on the 29 x 13 core), each
// stage lagging the previous one by the planes its stencil needs:
//   step j: B(j-1), C_M(j-2), faces(j-4), C_R(j-5).
// In-plane neighbours come from shared-memory plane rings (B: 4 planes,
// C_M: 3, faces: 3 x 3), own values of earlier planes from registers.
// Box loads of L_j: v_G(2s)(j), r_B(j-1), r_CM(j-2), r_Fx/Fy/Fz(j-4), r_CR(j-5);
// the box origin is a0-2 rounded down to 16 bytes (the tile stride 29 is odd).
struct OpJacMR3 {
  static constexpr int TA = 29, TB = 13;
  static constexpr int NS = 5, PRO = 2, EPI = 5;
  static constexpr int BW = 34, BH = 16, GH = 17;               // box extents (elements)
  static constexpr int RB_BYTES = BW * BH * 8, VG_BYTES = BW * GH * 8;
  static constexpr int RBA = al128(RB_BYTES);                   // r box stride in the slot
  static constexpr int OG = 0, OR0 = al128(VG_BYTES);           // v_G box, then 6 r boxes
  static constexpr int SLOT = OR0 + 6 * RBA;
  static constexpr int PL = 32 * 16 * 8;                        // one ring plane (one value per thread)
  static constexpr int RING_B = 0, RING_C = 4 * PL, RING_F = 7 * PL;   // B: 4, C_M: 3, faces: 3 x 3
  static constexpr int GPL = 0;
  static constexpr int SMEM = NS * SLOT + 16 * PL;
  // r boxes in the slot: rB, rCM, rFx, rFy, rFz, rCR
  static constexpr int R_B = 0, R_CM = 1, R_FX = 2, R_FY = 3, R_FZ = 4, R_CR = 5;
  struct Params {
    CUtensorMap tg, tr[6];   // v_G(2s); r_M B, r_M C, r_R Fx, Fy, Fz, C
    S3<T> v;                 // v_R(s) out
    Sched sc;
    int H;
    T cm, c1, c2;            // 4 p_m (sh)^2, 2 p_r1 (sh)^2, 4 p_r2 (sh)^2
  };
  struct State {
    T bo[5];                 // own B of planes j-1 .. j-5
    T co[3];                 // own C_M of planes j-2 .. j-4
    T fx[3], fy[3], fz[3];   // own faces of planes j-4 .. j-6
  };
  struct Ctx {
    int ox;                  // a0-2 minus the (aligned) box origin: 0 or 1
    bool a0k, a1k, b0k, b1k; // this column's a, b in [0,H-2] / [1,H-2]
    bool core, fpos;         // C_R core column; face column
  };
  static __device__ void prefetch(const Params &P) {
    tma_prefetch_desc(&P.tg);
    for (int i = 0; i < 6; i++) tma_prefetch_desc(&P.tr[i]);
  }
  static __device__ void init(State &S) {
    for (int i = 0; i < 5; i++) S.bo[i] = (T)0;
    for (int i = 0; i < 3; i++) S.co[i] = S.fx[i] = S.fy[i] = S.fz[i] = (T)0;
  }
  static __device__ __forceinline__ int bx0(const Item &it) { return (it.x0 - 2) & ~1; }
  static __device__ void begin(const Params &P, Ctx &C, const Item &it) {
    const int l = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int a = it.x0 - 2 + l, b = it.y0 - 2 + w;
    const HM m{P.H};
    C.ox = (it.x0 - 2) - bx0(it);
    C.a0k = m.z0(a);
    C.a1k = m.z1(a);
    C.b0k = m.z0(b);
    C.b1k = m.z1(b);
    C.core = l >= 2 && l <= 30 && w >= 2 && w <= 14;
    C.fpos = l >= 1 && l <= 30 && w >= 1 && w <= 14;
  }
  static __device__ void issue(const Params &P, const Item &it, int j, unsigned char *slot, uint64_t *bar) {
    const int x = bx0(it), y = it.y0 - 2;
    const bool wB = j >= it.zs - 1, wC = j >= it.zs + 1, wF = j >= it.zs + 3, wR = j >= it.zs + 5;
    mbar_expect_tx(bar, VG_BYTES + (wB + wC + 3 * wF + wR) * RB_BYTES);
    tma_load_3d(slot + OG, &P.tg, x, y, j, bar);
    if (wB) tma_load_3d(slot + OR0 + R_B * RBA, &P.tr[R_B], x, y, j - 1, bar);
    if (wC) tma_load_3d(slot + OR0 + R_CM * RBA, &P.tr[R_CM], x, y, j - 2, bar);
    if (wF)
      for (int i = R_FX; i <= R_FZ; i++) tma_load_3d(slot + OR0 + i * RBA, &P.tr[i], x, y, j - 4, bar);
    if (wR) tma_load_3d(slot + OR0 + R_CR * RBA, &P.tr[R_CR], x, y, j - 5, bar);
  }
  template <int PH>
  static __device__ __forceinline__ void step(const Params &P, State &S, const Ctx &Cx, const Item &it, int j,
                                              unsigned char *Lc, unsigned char *Lp, unsigned char *ring,
                                              unsigned char *, unsigned char *) {
    const int l = threadIdx.x & 31, w = threadIdx.x >> 5, tid = threadIdx.x;
    const int a = it.x0 - 2 + l, b = it.y0 - 2 + w;
    const HM m{P.H};
    const int ob = w * BW + l + Cx.ox;   // box offset of the own column
    auto rbox = [&](int i) { return (const T *)(Lc + OR0 + i * RBA) + ob; };
    auto bring = [&](int p) { return (T *)(ring + RING_B) + ((p & 3) * 512); };
    auto cring = [&](int p) { return (T *)(ring + RING_C) + ((((p % 3) + 3) % 3) * 512); };
    auto fring = [&](int p, int f) { return (T *)(ring + RING_F) + (((((p % 3) + 3) % 3) * 3 + f) * 512); };
    // ---- B(cb), cb = j-1: Emprolm from v_G(2s) planes cb, cb+1
    T bn = (T)0;
    const int cb = j - 1;
    if (j >= it.zs - 1) {
      const T *Gc = (const T *)(Lp + OG) + ob, *Gn = (const T *)(Lc + OG) + ob;
      T t = -(P.cm * rbox(R_B)[0]);
      t = t + Gn[BW + 1];   // (+,+,+)
      t = t + Gc[BW + 1];   // (+,+,-)
      t = t + Gn[1];        // (+,-,+)
      t = t + Gc[1];        // (+,-,-)
      t = t + Gn[BW];       // (-,+,+)
      t = t + Gc[BW];       // (-,+,-)
      t = t + Gn[0];        // (-,-,+)
      t = t + Gc[0];        // (-,-,-)
      bn = (Cx.a0k && Cx.b0k && m.z0(cb)) ? t * (T)0.125 : (T)0;
      bring(cb)[tid] = bn;
    }
    // ---- C_M(cc), cc = j-2: Emprolb from B(cc), B(cc-1) at (a-1..a, b-1..b)
    T cn = (T)0;
    const int cc = j - 2;
    if (j >= it.zs + 1 && l >= 1 && w >= 1) {
      const T *B0 = bring(cc) + tid, *B1 = bring(cc - 1) + tid;
      T u = -(P.cm * rbox(R_CM)[0]);
      u = u + S.bo[0];   // (a, b, c)    own B(j-2)
      u = u + S.bo[1];   // (a, b, c-1)  own B(j-3)
      u = u + B0[-32];   // (a, b-1, c)
      u = u + B1[-32];   // (a, b-1, c-1)
      u = u + B0[-1];    // (a-1, b, c)
      u = u + B1[-1];    // (a-1, b, c-1)
      u = u + B0[-33];   // (a-1, b-1, c)
      u = u + B1[-33];   // (a-1, b-1, c-1)
      cn = (Cx.a1k && Cx.b1k && m.z1(cc)) ? u * (T)0.125 : (T)0;
    }
    if (j >= it.zs + 1) cring(cc)[tid] = cn;
    // ---- faces(cf), cf = j-4: Erprolr from B(cf) (own + a-1 / b-1), B(cf-1) own, C_M(cf), C_M(cf+1)
    T fxn = (T)0, fyn = (T)0, fzn = (T)0;
    const int cf = j - 4;
    if (j >= it.zs + 3 && Cx.fpos) {
      const T *Bf = bring(cf) + tid;
      const T *Cf = cring(cf) + tid, *Cn = cring(cf + 1) + tid;
      const T bc = S.bo[2], bm = S.bo[3];   // own B(cf), B(cf-1)
      const T cmc = S.co[1], cmn = S.co[0]; // own C_M(cf), C_M(cf+1)
      const bool cz0 = m.z0(cf), cz1 = m.z1(cf);
      {   // Fx (2a, 2b+1, 2c+1): (0,+1,+1),(0,+1,-1),(0,-1,-1),(0,-1,+1) -> C(a,b+1,c+1), C(a,b+1,c), C(a,b,c), C(a,b,c+1)
        T nrm = bc;
        nrm = nrm + Bf[-1];
        T t = -(P.c1 * rbox(R_FX)[0]);
        t = t + (T)2 * nrm;
        t = t + Cn[32];
        t = t + Cf[32];
        t = t + cmc;
        t = t + cmn;
        fxn = (Cx.a1k && Cx.b0k && cz0) ? t * (T)0.125 : (T)0;
      }
      {   // Fy (2a+1, 2b, 2c+1): C(a+1,b,c+1), C(a,b,c+1), C(a,b,c), C(a+1,b,c)
        T nrm = bc;
        nrm = nrm + Bf[-32];
        T t = -(P.c1 * rbox(R_FY)[0]);
        t = t + (T)2 * nrm;
        t = t + Cn[1];
        t = t + cmn;
        t = t + cmc;
        t = t + Cf[1];
        fyn = (Cx.a0k && Cx.b1k && cz0) ? t * (T)0.125 : (T)0;
      }
      {   // Fz (2a+1, 2b+1, 2c): C(a+1,b+1,c), C(a+1,b,c), C(a,b,c), C(a,b+1,c)
        T nrm = bc;
        nrm = nrm + bm;
        T t = -(P.c1 * rbox(R_FZ)[0]);
        t = t + (T)2 * nrm;
        t = t + Cf[33];
        t = t + Cf[1];
        t = t + cmc;
        t = t + Cf[32];
        fzn = (Cx.a0k && Cx.b0k && cz1) ? t * (T)0.125 : (T)0;
      }
      if (Cx.core && cf >= it.zs && cf < it.ze) {
        const int64_t o = (int64_t)cf * P.v.plane + (int64_t)b * P.v.pitch + a;
        if (Cx.a1k && Cx.b0k && cz0) __stcs(P.v.s[FX] + o, fxn);
        if (Cx.a0k && Cx.b1k && cz0) __stcs(P.v.s[FY] + o, fyn);
        if (Cx.a0k && Cx.b0k && cz1) __stcs(P.v.s[FZ] + o, fzn);
      }
    }
    if (j >= it.zs + 3) {
      fring(cf, 0)[tid] = fxn;
      fring(cf, 1)[tid] = fyn;
      fring(cf, 2)[tid] = fzn;
    }
    // ---- C_R(cr), cr = j-5: Erprolm from the faces of planes cr (own S.f*[1], ring) and cr-1 (own S.f*[2], ring)
    const int cr = j - 5;
    if (j >= it.zs + 5 && Cx.core && Cx.a1k && Cx.b1k && m.z1(cr) && cr < it.ze) {
      const T *Gx = fring(cr, 0) + tid, *Gy = fring(cr, 1) + tid, *Gz = fring(cr, 2) + tid;
      const T *Hx = fring(cr - 1, 0) + tid, *Hy = fring(cr - 1, 1) + tid;
      T t = -(P.c2 * rbox(R_CR)[0]);
      t = t + S.fz[0];   // (+1,+1, 0)
      t = t + Gz[-32];   // (+1,-1, 0)
      t = t + Gz[-33];   // (-1,-1, 0)
      t = t + Gz[-1];    // (-1,+1, 0)
      t = t + S.fy[0];   // (+1, 0,+1)
      t = t + S.fy[1];   // (+1, 0,-1)
      t = t + Hy[-1];    // (-1, 0,-1)
      t = t + Gy[-1];    // (-1, 0,+1)
      t = t + S.fx[0];   // ( 0,+1,+1)
      t = t + S.fx[1];   // ( 0,+1,-1)
      t = t + Hx[-32];   // ( 0,-1,-1)
      t = t + Gx[-32];   // ( 0,-1,+1)
      __stcs(P.v.s[C] + (int64_t)cr * P.v.plane + (int64_t)b * P.v.pitch + a, t * (T)(1.0 / 12.0));
    }
    // ---- shift the own-value registers by one plane
    if (j >= it.zs + 3) {
      S.fx[2] = S.fx[1]; S.fx[1] = S.fx[0]; S.fx[0] = fxn;
      S.fy[2] = S.fy[1]; S.fy[1] = S.fy[0]; S.fy[0] = fyn;
      S.fz[2] = S.fz[1]; S.fz[1] = S.fz[0]; S.fz[0] = fzn;
    }
    if (j >= it.zs + 1) {
      S.co[2] = S.co[1]; S.co[1] = S.co[0]; S.co[0] = cn;
    }
    S.bo[4] = S.bo[3]; S.bo[3] = S.bo[2]; S.bo[2] = S.bo[1]; S.bo[1] = S.bo[0]; S.bo[0] = bn;
  }
  static __device__ void finish(const Params &, State &) {}
};

// ================================= R(s) -> M(s) -> G(2s): a11 + a12 fused
// Ermagc, Ermagm then Erblu in one pass: r_M(s) is
// written for the ascent but not read back.  Thread (l, w) owns the columns
// (a0-1+l, b0-1+2w+R), R = 0, 1: centres B_M on all of them (Erblu reaches
// a-1, b-1), corners C_M and r_G(2s) on the 31 x 31 core.  Step j: C_M(j),
// B_M(j) (L_j = {Fx(j), Fy(j), Fz(j+1), C_R(j)}), then Erblu at plane j-1
// from the centre ring (3 planes).  The face boxes share the origin
// ((a0-2) rounded down to 16 bytes, b0-2).
struct OpRestRMG3 {
  static constexpr int TA = 31, TB = 31;
  static constexpr int NS = 5, PRO = 2, EPI = 1;
  static constexpr int BW = 36, BH = 34;
  static constexpr int BOXB = al128(BW * BH * 8);
  static constexpr int OX = 0, OY = BOXB, OZ = 2 * BOXB, OCR = 3 * BOXB, SLOT = 4 * BOXB;
  static constexpr int PL = 1024 * 8;   // one ring plane: one centre per thread-row
  static constexpr int GPL = 0;
  static constexpr int SMEM = NS * SLOT + 3 * PL;
  struct Params {
    CUtensorMap tx, ty, tz, tc;   // r_R Fx, Fy, Fz, C
    S3<T> rm;                     // r_M(s) out: C, B
    D3<T> g2;                     // r_G(2s) out
    Sched sc;
    int H;
  };
  struct State {
    T cm;   // own C_M of the previous plane (row 0 and 1 packed below)
    T cm1;
  };
  struct Ctx {
    int ox;               // (a0-2) minus the box origin: 0 or 1
    bool k0[2], k1[2];    // per row: (a, b) in [0,H-2]^2 / [1,H-2]^2
    bool core[2];
  };
  static __device__ void prefetch(const Params &P) {
    tma_prefetch_desc(&P.tx);
    tma_prefetch_desc(&P.ty);
    tma_prefetch_desc(&P.tz);
    tma_prefetch_desc(&P.tc);
  }
  static __device__ void init(State &S) { S.cm = S.cm1 = (T)0; }
  static __device__ __forceinline__ int bx0(const Item &it) { return (it.x0 - 2) & ~1; }
  static __device__ void begin(const Params &P, Ctx &C, const Item &it) {
    const int l = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int a = it.x0 - 1 + l;
    const HM m{P.H};
    C.ox = (it.x0 - 2) - bx0(it);
#pragma unroll
    for (int R = 0; R < 2; R++) {
      const int b = it.y0 - 1 + 2 * w + R;
      C.k0[R] = m.z0(a) && m.z0(b);
      C.k1[R] = m.z1(a) && m.z1(b);
      C.core[R] = l >= 1 && (w >= 1 || R == 1);
    }
  }
  static __device__ void issue(const Params &P, const Item &it, int j, unsigned char *slot, uint64_t *bar) {
    const int x = bx0(it), y = it.y0 - 2;
    const bool wc = j >= it.zs && j < it.ze;
    mbar_expect_tx(bar, 3 * BW * BH * 8 + (wc ? BW * BH * 8 : 0));
    tma_load_3d(slot + OX, &P.tx, x, y, j, bar);
    tma_load_3d(slot + OY, &P.ty, x, y, j, bar);
    tma_load_3d(slot + OZ, &P.tz, x, y, j + 1, bar);
    if (wc) tma_load_3d(slot + OCR, &P.tc, x, y, j, bar);
  }
  template <int PH>
  static __device__ __forceinline__ void step(const Params &P, State &S, const Ctx &Cx, const Item &it, int j,
                                              unsigned char *Lc, unsigned char *Lp, unsigned char *ring,
                                              unsigned char *, unsigned char *) {
    if (j < it.zs - 1) return;
    const int l = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int a = it.x0 - 1 + l, c = j;
    const HM m{P.H};
    auto bring = [&](int p) { return (T *)(ring) + ((((p % 3) + 3) % 3) * 1024); };
    const bool c0 = m.z0(c), c1 = m.z1(c), cout = c >= it.zs && c < it.ze;
    T cmn[2] = {(T)0, (T)0};
#pragma unroll
    for (int R = 0; R < 2; R++) {
      const int rr = 2 * w + R, b = it.y0 - 1 + rr;
      const int o = (rr + 1) * BW + l + 1 + Cx.ox;   // box offset of (a, b)
      const T *Xc = (const T *)(Lc + OX) + o, *Xp = (const T *)(Lp + OX) + o;   // Fx planes c, c-1
      const T *Yc = (const T *)(Lc + OY) + o, *Yp = (const T *)(Lp + OY) + o;   // Fy planes c, c-1
      const T *Zn = (const T *)(Lc + OZ) + o, *Zc = (const T *)(Lp + OZ) + o;   // Fz planes c+1, c
      const int64_t og = (int64_t)c * P.rm.plane + (int64_t)b * P.rm.pitch + a;
      if (Cx.core[R] && cout && Cx.k1[R] && c1) {
        T t = (T)12 * ((const T *)(Lc + OCR))[o];
        t = t + Zc[0];         // (+1,+1, 0)
        t = t + Zc[-BW];       // (+1,-1, 0)
        t = t + Zc[-BW - 1];   // (-1,-1, 0)
        t = t + Zc[-1];        // (-1,+1, 0)
        t = t + Yc[0];         // (+1, 0,+1)
        t = t + Yp[0];         // (+1, 0,-1)
        t = t + Yp[-1];        // (-1, 0,-1)
        t = t + Yc[-1];        // (-1, 0,+1)
        t = t + Xc[0];         // ( 0,+1,+1)
        t = t + Xp[0];         // ( 0,+1,-1)
        t = t + Xp[-BW];       // ( 0,-1,-1)
        t = t + Xc[-BW];       // ( 0,-1,+1)
        cmn[R] = t * (T)(1.0 / 24.0);
        __stcs(P.rm.s[C] + og, cmn[R]);
      }
      // centre (2a+1, 2b+1, 2c+1): i+1, i-1, j+1, j-1, k+1, k-1
      T bm = (T)0;
      if (Cx.k0[R] && c0) {
        T t = Xc[1];
        t = t + Xc[0];
        t = t + Yc[BW];
        t = t + Yc[0];
        t = t + Zn[0];
        t = t + Zc[0];
        bm = t * (T)(1.0 / 6.0);
        if (Cx.core[R] && cout) __stcs(P.rm.s[B] + og, bm);
      }
      bring(c)[rr * 32 + l] = bm;
    }
    // ---- Erblu at plane q = c-1 from C_M(q) (own, previous step) and the centres of planes q, q-1
    const int q = c - 1;
    if (q >= it.zs && q < it.ze && m.z1(q)) {
#pragma unroll
      for (int R = 0; R < 2; R++) {
        if (!(Cx.core[R] && Cx.k1[R])) continue;
        const int rr = 2 * w + R, b = it.y0 - 1 + rr;
        const T *Bc = bring(q) + rr * 32 + l, *Bp = bring(q - 1) + rr * 32 + l;
        T t = (T)8 * (R ? S.cm1 : S.cm);
        t = t + Bc[0];     // (+,+,+)
        t = t + Bp[0];     // (+,+,-)
        t = t + Bc[-32];   // (+,-,+)
        t = t + Bp[-32];   // (+,-,-)
        t = t + Bc[-1];    // (-,+,+)
        t = t + Bp[-1];    // (-,+,-)
        t = t + Bc[-33];   // (-,-,+)
        t = t + Bp[-33];   // (-,-,-)
        __stcs(&P.g2(a, b, q), t * (T)(1.0 / 16.0));
      }
    }
    S.cm = cmn[0];
    S.cm1 = cmn[1];
  }
  static __device__ void finish(const Params &, State &) {}
};

// ================================================================= launch
template <class E>
static bool tsub(CUtensorMap *tm, const S3<E> &s, int k, int H, int bx, int by) {
  return tmap3<E>(tm, s.s[k], H, H, H, s.pitch, s.plane, bx, by);
}
static inline int cdiv(int a, int b) { return (a + b - 1) / b; }

template <class E, int NW>
static cudaError_t jac_r_nw(const S3<E> &vm, const S3<E> &r, const S3<E> &v, int M, E c1, E c2, cudaStream_t st) {
  using Op = OpJacR3T<E, NW>;
  typename Op::Params P{};
  const int H = M / 2 + 1;
  if (!tsub(&P.tc, vm, C, H, Op::BW, NW + 1) || !tsub(&P.tb, vm, B, H, Op::BW, NW + 1) ||
      !tsub(&P.tr[0], r, FX, H, Op::RWB, NW) || !tsub(&P.tr[1], r, FY, H, Op::RWB, NW) ||
      !tsub(&P.tr[2], r, FZ, H, Op::RWB, NW) || !tsub(&P.tr[3], r, C, H, Op::RWB, NW))
    return cudaErrorInvalidValue;
  P.v = v;
  P.H = H;
  P.c1 = c1;
  P.c2 = c2;
  return launch_zpipe<Op>(P, 30, NW - 1, 0, 0, cdiv(H - 1, 30), cdiv(H - 1, NW - 1), 0, H - 1, st);
}

// warps per CTA of the red Jacobi pass (MG_K3R_NW: 16 = one 512-thread CTA per
// SM, 8 = two 256-thread CTAs per SM)
template <class E>
cudaError_t fast3s_jac_r(const S3<E> &vm, const S3<E> &r, const S3<E> &v, int M, E c1, E c2, cudaStream_t st) {
  static const int nw = getenv("MG_K3R_NW") ? atoi(getenv("MG_K3R_NW")) : 16;
  if (nw == 8) return jac_r_nw<E, 8>(vm, r, v, M, c1, c2, st);
  return jac_r_nw<E, 16>(vm, r, v, M, c1, c2, st);
}

template <class E, int NW>
static cudaError_t jac_m_nw(const D3<E> &vc, const S3<E> &r, const S3<E> &v, int M, E cc, cudaStream_t st) {
  using Op = OpJacM3T<E, NW>;
  typename Op::Params P{};
  const int H = M / 2 + 1;
  if (!tmap3<E>(&P.tg, vc.p, H, H, H, vc.pitch, vc.plane, Op::BW, Op::GROWS) ||
      !tsub(&P.tr[0], r, B, H, Op::RWB, 2 * NW) || !tsub(&P.tr[1], r, C, H, Op::RWB, 2 * NW))
    return cudaErrorInvalidValue;
  P.v = v;
  P.H = H;
  P.cc = cc;
  constexpr int tb = 2 * NW - 1;
  return launch_zpipe<Op>(P, 30, tb, 0, 0, cdiv(H - 1, 30), cdiv(H - 1, tb), 0, H - 1, st);
}

// warps per CTA of the magenta Jacobi pass (MG_K3S_NW: 8 = two 256-thread CTAs
// per SM, the default -- measured on B200 at 513^3 fp64: jac_m(1) 142 -> 134 us,
// cycle -0.7 %; 16 = one 512-thread CTA per SM)
template <class E>
cudaError_t fast3s_jac_m(const D3<E> &vc, const S3<E> &r, const S3<E> &v, int M, E cc, cudaStream_t st) {
  static const int nw = getenv("MG_K3S_NW") ? atoi(getenv("MG_K3S_NW")) : 8;
  if (nw == 8) return jac_m_nw<E, 8>(vc, r, v, M, cc, st);
  return jac_m_nw<E, 16>(vc, r, v, M, cc, st);
}

template <class E>
cudaError_t fast3s_rest_rm(const S3<E> &rr, const S3<E> &rm, int M, cudaStream_t st) {
  using Op = OpRestRM3<E>;
  typename Op::Params P{};
  const int H = M / 2 + 1;
  if (!tsub(&P.tx, rr, FX, H, Op::WX, 33) || !tsub(&P.ty, rr, FY, H, Op::WY, 33) ||
      !tsub(&P.tz, rr, FZ, H, Op::WY, 33) || !tsub(&P.tc, rr, C, H, RW, RH2))
    return cudaErrorInvalidValue;
  P.out = rm;
  P.H = H;
  return launch_zpipe<Op>(P, 32, 32, 0, 0, cdiv(H - 1, 32), cdiv(H - 1, 32), 0, H - 1, st);
}

template <class E>
cudaError_t fast3s_rest_mg(const S3<E> &rm, const D3<E> &g2, int Mc, cudaStream_t st) {
  using Op = OpRestMG3<E>;
  typename Op::Params P{};
  const int H = Mc + 1;
  if (!tsub(&P.tb, rm, B, H, Op::WB, 33) || !tsub(&P.tc, rm, C, H, RW, RH2)) return cudaErrorInvalidValue;
  P.out = g2;
  P.H = H;
  return launch_zpipe<Op>(P, 32, 32, 0, 0, cdiv(H - 1, 32), cdiv(H - 1, 32), 1, H - 1, st);
}

#define INST3S(E)                                                                                               \
  template cudaError_t fast3s_jac_r<E>(const S3<E> &, const S3<E> &, const S3<E> &, int, E, E, cudaStream_t); \
  template cudaError_t fast3s_jac_m<E>(const D3<E> &, const S3<E> &, const S3<E> &, int, E, cudaStream_t);    \
  template cudaError_t fast3s_rest_rm<E>(const S3<E> &, const S3<E> &, int, cudaStream_t);                     \
  template cudaError_t fast3s_rest_mg<E>(const S3<E> &, const D3<E> &, int, cudaStream_t);
INST3S(double)
INST3S(float)
#undef INST3S

cudaError_t fast3s_jac_mr(const D3<double> &vc, const S3<double> &rm, const S3<double> &rr, const S3<double> &v, int M,
                          double cm, double c1, double c2, cudaStream_t st) {
  using Op = OpJacMR3;
  Op::Params P{};
  const int H = M / 2 + 1;
  if (!tmap3<T>(&P.tg, vc.p, H, H, H, vc.pitch, vc.plane, Op::BW, Op::GH) ||
      !tsub(&P.tr[Op::R_B], rm, B, H, Op::BW, Op::BH) || !tsub(&P.tr[Op::R_CM], rm, C, H, Op::BW, Op::BH) ||
      !tsub(&P.tr[Op::R_FX], rr, FX, H, Op::BW, Op::BH) || !tsub(&P.tr[Op::R_FY], rr, FY, H, Op::BW, Op::BH) ||
      !tsub(&P.tr[Op::R_FZ], rr, FZ, H, Op::BW, Op::BH) || !tsub(&P.tr[Op::R_CR], rr, C, H, Op::BW, Op::BH))
    return cudaErrorInvalidValue;
  P.v = v;
  P.H = H;
  P.cm = cm;
  P.c1 = c1;
  P.c2 = c2;
  return launch_zpipe<Op>(P, Op::TA, Op::TB, 0, 0, cdiv(H - 1, Op::TA), cdiv(H - 1, Op::TB), 0, H - 1, st);
}


cudaError_t fast3s_rest_rmg(const S3<double> &rr, const S3<double> &rm, const D3<double> &g2, int M, cudaStream_t st) {
  using Op = OpRestRMG3;
  Op::Params P{};
  const int H = M / 2 + 1;
  if (!tsub(&P.tx, rr, FX, H, Op::BW, Op::BH) || !tsub(&P.ty, rr, FY, H, Op::BW, Op::BH) ||
      !tsub(&P.tz, rr, FZ, H, Op::BW, Op::BH) || !tsub(&P.tc, rr, C, H, Op::BW, Op::BH))
    return cudaErrorInvalidValue;
  P.rm = rm;
  P.g2 = g2;
  P.H = H;
  return launch_zpipe<Op>(P, Op::TA, Op::TB, 0, 0, cdiv(H - 1, Op::TA), cdiv(H - 1, Op::TB), 0, H - 1, st);
}

}  // namespace mg
