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
using T = double;
constexpr int RW = 32, RH = 16;                        // one value per thread
constexpr int RBOX = RW * RH * 8;                      // 4096 B
constexpr int BOX34 = al128(34 * 17 * 8), BOX36 = al128(36 * 17 * 8);

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
struct OpJacR3 {
  static constexpr int NS = 6, PRO = 2, EPI = 2;
  static constexpr int OC = 0, OB = BOX34, OR = 2 * BOX34;   // C box, B box, 4 r boxes (Fx, Fy, Fz, C)
  static constexpr int SLOT = OR + 4 * RBOX;
  static constexpr int GPL = 3 * RBOX;                       // face ring plane: Fx | Fy | Fz
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
  }
  static __device__ void issue(const Params &P, const Item &it, int j, unsigned char *slot, uint64_t *bar) {
    const bool wf = j >= it.zs, wc = j >= it.zs + 2;
    mbar_expect_tx(bar, 2 * 34 * 17 * 8 + (wf ? 3 * RBOX : 0) + (wc ? RBOX : 0));
    tma_load_3d(slot + OC, &P.tc, it.x0 - 2, it.y0 - 1, j, bar);
    tma_load_3d(slot + OB, &P.tb, it.x0 - 4, it.y0 - 2, j, bar);
    if (wf)
      for (int i = 0; i < 3; i++) tma_load_3d(slot + OR + i * RBOX, &P.tr[i], it.x0 - 2, it.y0 - 1, j - 1, bar);
    if (wc) tma_load_3d(slot + OR + 3 * RBOX, &P.tr[3], it.x0 - 2, it.y0 - 1, j - 2, bar);
  }
  template <int PH>
  static __device__ __forceinline__ void step(const Params &P, State &S, const Ctx &Cx, const Item &it, int j,
                                              unsigned char *Lc, unsigned char *Lp, unsigned char *gz,
                                              unsigned char *gq, unsigned char *gr) {
    constexpr int Q = PH ^ 1;
    const int l = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int a = it.x0 - 2 + l, b = it.y0 - 1 + w;
    const int oc = w * 34 + l, ob = (w + 1) * 34 + l + 2, orr = w * RW + l;
    const HM m{P.H};
    const T bj = ((const T *)(Lc + OB))[ob];   // own B_M(j)
    if (j >= it.zs) {
      const int c = j - 1;
      const T *Cc = (const T *)(Lp + OC) + oc, *Cn = (const T *)(Lc + OC) + oc, *Bc = (const T *)(Lp + OB) + ob;
      const T *R = (const T *)(Lc + OR) + orr;
      const T bc = S.bo[Q], bm = S.bo[PH];   // B(a,b,c), B(a,b,c-1)
      const bool cz0 = m.z0(c), cz1 = m.z1(c);
      T fx, fy, fz;
      {   // Fx (2a, 2b+1, 2c+1): normal x; in-plane (0,+1,+1),(0,+1,-1),(0,-1,-1),(0,-1,+1)
        T nrm = bc;
        nrm = nrm + Bc[-1];
        T t = -(P.c1 * R[0]);
        t = t + (T)2 * nrm;
        t = t + Cn[34];
        t = t + Cc[34];
        t = t + Cc[0];
        t = t + Cn[0];
        fx = (Cx.a1k && Cx.b0k && cz0) ? t * (T)0.125 : (T)0;
      }
      {   // Fy (2a+1, 2b, 2c+1): normal y; in-plane (+1,0,+1),(-1,0,+1),(-1,0,-1),(+1,0,-1)
        T nrm = bc;
        nrm = nrm + Bc[-34];
        T t = -(P.c1 * R[RBOX / 8]);
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
        T t = -(P.c1 * R[2 * RBOX / 8]);
        t = t + (T)2 * nrm;
        t = t + Cc[35];
        t = t + Cc[1];
        t = t + Cc[0];
        t = t + Cc[34];
        fz = (Cx.a0k && Cx.b0k && cz1) ? t * (T)0.125 : (T)0;
      }
      {
        T *g = (T *)gz + orr;
        g[0] = fx;
        g[RBOX / 8] = fy;
        g[2 * RBOX / 8] = fz;
      }
      if (Cx.core && c >= it.zs && c < it.ze) {
        const int64_t o = (int64_t)c * P.v.plane + (int64_t)b * P.v.pitch + a;
        if (Cx.a1k && Cx.b0k && cz0) __stcs(P.v.s[FX] + o, fx);
        if (Cx.a0k && Cx.b1k && cz0) __stcs(P.v.s[FY] + o, fy);
        if (Cx.a0k && Cx.b0k && cz1) __stcs(P.v.s[FZ] + o, fz);
      }
      // ---- corners of plane q = j-2 from the faces of planes q (own: slot PH, ring gq) and q-1 (slot Q, gr)
      const int q = j - 2;
      if (q >= it.zs && Cx.core && Cx.a1k && Cx.b1k && m.z1(q)) {
        const T *Gx = (const T *)gq + orr, *Gy = Gx + RBOX / 8, *Gz = Gx + 2 * RBOX / 8;
        const T *Hx = (const T *)gr + orr, *Hy = Hx + RBOX / 8;
        T t = -(P.c2 * R[3 * RBOX / 8]);
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
        __stcs(P.v.s[C] + (int64_t)q * P.v.plane + (int64_t)b * P.v.pitch + a, t * (T)(1.0 / 12.0));
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
struct OpJacM3 {
  static constexpr int NS = 7, PRO = 1, EPI = 2;
  static constexpr int OG = 0, OR = BOX34x33;   // v_G box, r boxes (B, C)
  static constexpr int SLOT = OR + 2 * RBOX2;
  static constexpr int GPL = RBOX2;             // centre ring plane
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
#pragma unroll
    for (int R = 0; R < 2; R++) {
      const int b = it.y0 - 1 + 2 * w + R;
      C.b0k[R] = m.z0(a) && m.z0(b);
      C.b1k[R] = m.z1(a) && m.z1(b);
      C.core[R] = l >= 2 && (w >= 1 || R == 1);
    }
  }
  static __device__ void issue(const Params &P, const Item &it, int j, unsigned char *slot, uint64_t *bar) {
    const bool wf = j >= it.zs, wc = j >= it.zs + 2;
    mbar_expect_tx(bar, 34 * 33 * 8 + (wf ? RBOX2 : 0) + (wc ? RBOX2 : 0));
    tma_load_3d(slot + OG, &P.tg, it.x0 - 2, it.y0 - 1, j, bar);
    if (wf) tma_load_3d(slot + OR, &P.tr[0], it.x0 - 2, it.y0 - 1, j - 1, bar);
    if (wc) tma_load_3d(slot + OR + RBOX2, &P.tr[1], it.x0 - 2, it.y0 - 1, j - 2, bar);
  }
  template <int PH>
  static __device__ __forceinline__ void step(const Params &P, State &S, const Ctx &Cx, const Item &it, int j,
                                              unsigned char *Lc, unsigned char *Lp, unsigned char *gz,
                                              unsigned char *gq, unsigned char *gr) {
    constexpr int Q = PH ^ 1;
    if (j < it.zs) return;
    const int l = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int a = it.x0 - 2 + l;
    const HM m{P.H};
    const int c = j - 1, q = j - 2;
    const bool czin = m.z0(c), cout = c >= it.zs && c < it.ze, qok = q >= it.zs && m.z1(q);
    T bn[2];
#pragma unroll
    for (int R = 0; R < 2; R++) {
      const int og = (2 * w + R) * 34 + l, orr = (2 * w + R) * RW + l;
      const T *Gc = (const T *)(Lp + OG) + og, *Gn = (const T *)(Lc + OG) + og;   // v_G planes c, c+1
      const T *Rb = (const T *)(Lc + OR) + orr;
      T t = -(P.cc * Rb[0]);
      t = t + Gn[35];   // (+,+,+)
      t = t + Gc[35];   // (+,+,-)
      t = t + Gn[1];    // (+,-,+)
      t = t + Gc[1];    // (+,-,-)
      t = t + Gn[34];   // (-,+,+)
      t = t + Gc[34];   // (-,+,-)
      t = t + Gn[0];    // (-,-,+)
      t = t + Gc[0];    // (-,-,-)
      const bool ok = Cx.b0k[R] && czin;
      bn[R] = ok ? t * (T)0.125 : (T)0;
      ((T *)gz)[orr] = bn[R];
      const int b = it.y0 - 1 + 2 * w + R;
      if (ok && Cx.core[R] && cout) __stcs(P.v.s[B] + (int64_t)c * P.v.plane + (int64_t)b * P.v.pitch + a, bn[R]);
      if (qok && Cx.core[R] && Cx.b1k[R]) {
        const T *G0 = (const T *)gq + orr, *G1 = (const T *)gr + orr;   // centres of planes q, q-1
        T u = -(P.cc * Rb[RBOX2 / 8]);
        u = u + S.bo[PH][R];     // (a, b, c)
        u = u + S.bo[Q][R];      // (a, b, c-1)
        u = u + G0[-RW];         // (a, b-1, c)
        u = u + G1[-RW];         // (a, b-1, c-1)
        u = u + G0[-1];          // (a-1, b, c)
        u = u + G1[-1];          // (a-1, b, c-1)
        u = u + G0[-RW - 1];     // (a-1, b-1, c)
        u = u + G1[-RW - 1];     // (a-1, b-1, c-1)
        __stcs(P.v.s[C] + (int64_t)q * P.v.plane + (int64_t)b * P.v.pitch + a, u * (T)0.125);
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
// and centres (Ermagm) of plane j.
struct OpRestRM3 {
  static constexpr int NS = 6, PRO = 1, EPI = 0;
  static constexpr int OX = 0, OY = BOX36x33, OZ = BOX36x33 + BOX34x33, OCR = BOX36x33 + 2 * BOX34x33;
  static constexpr int SLOT = OCR + RBOX2;
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
    mbar_expect_tx(bar, 36 * 33 * 8 + 2 * 34 * 33 * 8 + (wc ? RBOX2 : 0));
    tma_load_3d(slot + OX, &P.tx, it.x0 - 2, it.y0 - 1, j, bar);
    tma_load_3d(slot + OY, &P.ty, it.x0 - 2, it.y0, j, bar);
    tma_load_3d(slot + OZ, &P.tz, it.x0 - 2, it.y0 - 1, j + 1, bar);
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
      const int ox = (rr + 1) * 36 + l + 2, oy = rr * 34 + l + 2, oz = (rr + 1) * 34 + l + 2;
      const T *Xc = (const T *)(Lc + OX) + ox, *Xp = (const T *)(Lp + OX) + ox;   // Fx planes c, c-1
      const T *Yc = (const T *)(Lc + OY) + oy, *Yp = (const T *)(Lp + OY) + oy;   // Fy planes c, c-1
      const T *Zn = (const T *)(Lc + OZ) + oz, *Zc = (const T *)(Lp + OZ) + oz;   // Fz planes c+1, c
      const int64_t o = (int64_t)c * P.out.plane + (int64_t)b * P.out.pitch + a;
      if (Cx.k1[R] && c1) {
        T t = (T)12 * ((const T *)(Lc + OCR))[rr * RW + l];
        t = t + Zc[0];         // (+1,+1, 0)
        t = t + Zc[-34];       // (+1,-1, 0)
        t = t + Zc[-35];       // (-1,-1, 0)
        t = t + Zc[-1];        // (-1,+1, 0)
        t = t + Yc[0];         // (+1, 0,+1)
        t = t + Yp[0];         // (+1, 0,-1)
        t = t + Yp[-1];        // (-1, 0,-1)
        t = t + Yc[-1];        // (-1, 0,+1)
        t = t + Xc[0];         // ( 0,+1,+1)
        t = t + Xp[0];         // ( 0,+1,-1)
        t = t + Xp[-36];       // ( 0,-1,-1)
        t = t + Xc[-36];       // ( 0,-1,+1)
        __stcs(P.out.s[C] + o, t * (T)(1.0 / 24.0));
      }
      if (Cx.k0[R] && c0) {
        // centre (2a+1, 2b+1, 2c+1): i+1, i-1, j+1, j-1, k+1, k-1
        T t = Xc[1];
        t = t + Xc[0];
        t = t + Yc[34];
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
struct OpRestMG3 {
  static constexpr int NS = 12, PRO = 1, EPI = 0;
  static constexpr int OB = 0, OCM = BOX34x33;
  static constexpr int SLOT = OCM + RBOX2;
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
    mbar_expect_tx(bar, 34 * 33 * 8 + (wc ? RBOX2 : 0));
    tma_load_3d(slot + OB, &P.tb, it.x0 - 2, it.y0 - 1, j, bar);
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
      const int ob = (rr + 1) * 34 + l + 2;
      const T *Bc = (const T *)(Lc + OB) + ob, *Bp = (const T *)(Lp + OB) + ob;   // B planes c, c-1
      T t = (T)8 * ((const T *)(Lc + OCM))[rr * RW + l];
      t = t + Bc[0];         // (+,+,+)
      t = t + Bp[0];         // (+,+,-)
      t = t + Bc[-34];       // (+,-,+)
      t = t + Bp[-34];       // (+,-,-)
      t = t + Bc[-1];        // (-,+,+)
      t = t + Bp[-1];        // (-,+,-)
      t = t + Bc[-35];       // (-,-,+)
      t = t + Bp[-35];       // (-,-,-)
      __stcs(&P.out(a, b, c), t * (T)(1.0 / 16.0));
    }
  }
  static __device__ void finish(const Params &, State &) {}
};

// ================================================================= launch
static bool tsub(CUtensorMap *tm, const S3<T> &s, int k, int H, int bx, int by) {
  return tmap3<T>(tm, s.s[k], H, H, H, s.pitch, s.plane, bx, by);
}
static inline int cdiv(int a, int b) { return (a + b - 1) / b; }

cudaError_t fast3s_jac_r(const S3<double> &vm, const S3<double> &r, const S3<double> &v, int M, double c1, double c2,
                         cudaStream_t st) {
  using Op = OpJacR3;
  Op::Params P{};
  const int H = M / 2 + 1;
  if (!tsub(&P.tc, vm, C, H, 34, 17) || !tsub(&P.tb, vm, B, H, 34, 17) || !tsub(&P.tr[0], r, FX, H, RW, RH) ||
      !tsub(&P.tr[1], r, FY, H, RW, RH) || !tsub(&P.tr[2], r, FZ, H, RW, RH) || !tsub(&P.tr[3], r, C, H, RW, RH))
    return cudaErrorInvalidValue;
  P.v = v;
  P.H = H;
  P.c1 = c1;
  P.c2 = c2;
  return launch_zpipe<Op>(P, 30, 15, 0, 0, cdiv(H - 1, 30), cdiv(H - 1, 15), 0, H - 1, st);
}

cudaError_t fast3s_jac_m(const D3<double> &vc, const S3<double> &r, const S3<double> &v, int M, double cc,
                         cudaStream_t st) {
  using Op = OpJacM3;
  Op::Params P{};
  const int H = M / 2 + 1;
  if (!tmap3<T>(&P.tg, vc.p, H, H, H, vc.pitch, vc.plane, 34, 33) || !tsub(&P.tr[0], r, B, H, RW, RH2) ||
      !tsub(&P.tr[1], r, C, H, RW, RH2))
    return cudaErrorInvalidValue;
  P.v = v;
  P.H = H;
  P.cc = cc;
  return launch_zpipe<Op>(P, 30, 31, 0, 0, cdiv(H - 1, 30), cdiv(H - 1, 31), 0, H - 1, st);
}

cudaError_t fast3s_rest_rm(const S3<double> &rr, const S3<double> &rm, int M, cudaStream_t st) {
  using Op = OpRestRM3;
  Op::Params P{};
  const int H = M / 2 + 1;
  if (!tsub(&P.tx, rr, FX, H, 36, 33) || !tsub(&P.ty, rr, FY, H, 34, 33) || !tsub(&P.tz, rr, FZ, H, 34, 33) ||
      !tsub(&P.tc, rr, C, H, RW, RH2))
    return cudaErrorInvalidValue;
  P.out = rm;
  P.H = H;
  return launch_zpipe<Op>(P, 32, 32, 0, 0, cdiv(H - 1, 32), cdiv(H - 1, 32), 0, H - 1, st);
}

cudaError_t fast3s_rest_mg(const S3<double> &rm, const D3<double> &g2, int Mc, cudaStream_t st) {
  using Op = OpRestMG3;
  Op::Params P{};
  const int H = Mc + 1;
  if (!tsub(&P.tb, rm, B, H, 34, 33) || !tsub(&P.tc, rm, C, H, RW, RH2)) return cudaErrorInvalidValue;
  P.out = g2;
  P.H = H;
  return launch_zpipe<Op>(P, 32, 32, 0, 0, cdiv(H - 1, 32), cdiv(H - 1, 32), 1, H - 1, st);
}

}  // namespace mg
