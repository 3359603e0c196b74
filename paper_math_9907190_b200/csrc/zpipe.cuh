// zpipe.cuh -- the persistent TMA plane pipeline shared by the 3D stencil
// passes (k3p.cu: fine-resolution passes; k3s.cu: sublattice level passes).
//
// One CTA per SM walks a balanced list of work items (an xy tile times a z
// range); one thread keeps NS-2 planes of TMA loads in flight in a ring of NS
// shared-memory slots (one mbarrier each); step j of an item consumes load
// L_j (and the older slots the Op declares), then one __syncthreads.
#pragma once
#include <cooperative_groups.h>

#include <type_traits>

#include "kernels.h"
#include "tma.cuh"

namespace mg {

namespace zp {

constexpr int TX = 60, TY = 30, NT = 512;
constexpr int GS = 34;                       // green-plane ring: 34 x 34 (rows/lanes -1 .. 32)
constexpr int al128(int n) { return (n + 127) / 128 * 128; }

// Tile geometry of the fine-resolution passes (k3p.cu) for NW warps of 32
// lanes: lane l owns columns x0-2+2l, +1 and warp w rows y0-1+2w, +1, so a
// CTA owns 64 x 2NW nodes per plane and outputs the inner 60 x (2NW-2).
template <class T, int NW_ = 16>
struct Geo {
  static constexpr int NW = NW_, NTH = 32 * NW;
  static constexpr int TYW = 2 * NW - 2;                 // output rows per tile
  static constexpr int GR = 2 * NW + 2;                  // green-ring rows (rows -1 .. 2NW)
  static constexpr int AL = 16 / (int)sizeof(T);       // TMA x alignment (elements)
  static constexpr int UXO = (AL == 2) ? 4 : 6;         // u box starts at x0 - UXO (>= 3, aligned)
  static constexpr int UW = (UXO + 63 + AL - 1) / AL * AL, UH = TYW + 4;
  static constexpr int FW = 64, FH = TYW + 2;           // f box: x0-2 .., y0-1 ..
  static constexpr int VW = (34 + AL - 1 + AL - 1) / AL * AL, VH = TYW / 2 + 2;
  static constexpr int U_BYTES = UW * UH * (int)sizeof(T), F_BYTES = FW * FH * (int)sizeof(T);
  static constexpr int V_BYTES = VW * VH * (int)sizeof(T);
  static constexpr int GPL = al128(GS * GR * (int)sizeof(T));
};

// Threads per CTA and resident CTAs per SM of a pipeline Op: Op::NTH /
// Op::MINB when it declares them, else one 512-thread CTA per SM.
template <class Op, class = void>
struct OpNT {
  static constexpr int nt = NT, minb = 1;
};
template <class Op>
struct OpNT<Op, std::void_t<decltype(Op::NTH), decltype(Op::MINB)>> {
  static constexpr int nt = Op::NTH, minb = Op::MINB;
};

// Ring slots an Op reads at step j: 2 (L_j, L_{j-1}: the default) or 3 (also
// L_{j-2}, passed as Lq; Op::KEEP = 3) -- the loads in flight are NS - KEEP.
template <class Op, class = void>
struct OpKeep {
  static constexpr int v = 2;
};
template <class Op>
struct OpKeep<Op, std::void_t<decltype(Op::KEEP)>> {
  static constexpr int v = Op::KEEP;
};

// Element size of a pipeline Op (Op::T, else its Geo's TMA alignment; the fp64-only fused Ops: 8).
template <class Op, class = void>
struct OpEsz {
  static constexpr int v = 8;
};
template <class Op>
struct OpEsz<Op, std::void_t<typename Op::T>> {
  static constexpr int v = (int)sizeof(typename Op::T);
};
template <class Op>
struct OpEsz<Op, std::void_t<typename Op::Gm>> {
  static constexpr int v = 16 / Op::Gm::AL;
};

// Sublattice (half-index) passes of k3s.cu declare Op::T; the fine-resolution passes of k3p.cu do not.
template <class Op, class = void>
struct OpHalf {
  static constexpr bool v = false;
};
template <class Op>
struct OpHalf<Op, std::void_t<typename Op::T>> {
  static constexpr bool v = true;
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
__device__ __forceinline__ void st2(T *p, T a, T b) {   // streaming (evict-first) vector store
  typename V2t<T>::t v;
  v.x = a;
  v.y = b;
  __stcs(reinterpret_cast<typename V2t<T>::t *>(p), v);
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

// Balanced work list.  Each of the T tiles is cut into S z pieces (S = 1
// unless T < G) giving U = T*S units; units k*G + b (k < W = U / G) are
// whole; the R = U mod G remaining units are each split into ~G/R z segments,
// one per CTA, so every CTA streams the same number of planes and tiles that
// are neighbours in xy are streamed concurrently (their halos hit in L2).
struct Item {
  int x0, y0, zs, ze;
};
struct Sched {
  int T, ntx, zlo, zhi, S;
  int tx, ty, xoff, yoff;   // tile extents and origin offsets: x0 = tx * (t % ntx) + xoff
  int rev;                  // 1: every CTA walks its items in reverse order (serpentine across passes)
  int wsync;                // 1: grid-wide barrier after every whole wave of G units (cooperative launch)
  __device__ __forceinline__ int count(int G) const { return (T * S) / G + ((T * S) % G ? 1 : 0); }
  __device__ __forceinline__ Item get(int k, int b, int G) const {
    const int U = T * S, W = U / G, R = U % G;
    if (rev) k = count(G) - 1 - k;
    const long long Z = zhi - zlo;
    int u, sg = 0, nseg = 1;
    if (k < W) {
      u = b + k * G;
    } else {
      const int r = b % R;
      u = W * G + r;
      nseg = G / R + (r < G % R ? 1 : 0);
      sg = b / R;
    }
    const int t = u % T, p = u / T;
    const int z0 = zlo + (int)(Z * p / S), z1 = zlo + (int)(Z * (p + 1) / S);
    Item it;
    it.x0 = (t % ntx) * tx + xoff;
    it.y0 = (t / ntx) * ty + yoff;
    it.zs = z0 + (int)((long long)(z1 - z0) * sg / nseg);
    it.ze = z0 + (int)((long long)(z1 - z0) * (sg + 1) / nseg);
    return it;
  }
};

}  // namespace zp

using namespace zp;

// ------------------------------------------------------------ pipeline
// Op: NS (slots), SLOT (bytes), SMEM, GPL (bytes of one ring plane), PRO /
// EPI (steps before zs / after ze-1), Params (with .sc), issue(P, it, j,
// slot, bar), State, Ctx, begin(P, Ctx&, it), step<PH>(P, State&, Ctx&, it,
// j, Lc, Lp, [Lq,] gz, gq, gr): item steps run j = zs-PRO .. ze-1+EPI.  PH = j & 1: every parity the step needs (tile origins
// y0 and x0 are even) is a compile-time function of PH, and the register
// state is double-buffered by PH, so no selects or register moves remain.
// A 3-plane ring after the slots is addressed by gz (plane j-1), gq (plane
// j-2) and gr (plane j-3).
template <class Op>
__global__ void __launch_bounds__(OpNT<Op>::nt, OpNT<Op>::minb) zpipe(const __grid_constant__ typename Op::Params P) {
  constexpr int KEEP = OpKeep<Op>::v, NS = Op::NS, D = NS - KEEP;
  static_assert(D >= 1, "at least one load in flight");
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ __align__(8) uint64_t bar[NS];
  const int G = gridDim.x, b = blockIdx.x;
  const int nit = P.sc.count(G);
  pdl_trigger();
  if (threadIdx.x == 0) {
    for (int s = 0; s < NS; s++) mbar_init(&bar[s], 1);
    fence_mbar_init();
    Op::prefetch(P);
  }
  __syncthreads();
  pdl_wait();   // the predecessor's outputs (and its reads of what this pass writes) are done
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
        pj = it.zs - Op::PRO;
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
    if (++pj > pit.ze - 1 + Op::EPI) pseek(pk + 1);
  };
  if (threadIdx.x == 0) {
    pseek(0);
    for (int d = 0; d < D; d++) produce();
  }

  typename Op::State S;
  Op::init(S);
  int cs = 0, cprev = NS - 1, cpp = NS - 2;
  uint32_t phase = 0;
  const int W = (P.sc.T * P.sc.S) / G;   // whole waves
  for (int k = 0; k < nit; k++) {
    // neighbouring tiles of one wave stream side by side and re-read each other's halo rows from L2;
    // without a barrier the CTAs drift apart over several waves and the halos come back from HBM
    if (P.sc.wsync && k >= 1 && k <= W) cooperative_groups::this_grid().sync();
    const Item it = P.sc.get(k, b, G);
    if (it.ze <= it.zs) continue;
    typename Op::Ctx C;
    Op::begin(P, C, it);
    // ring planes rotate by one per step; greens are written and read within one item
    int gz = 0, gq = 0;
    auto one = [&](auto ph, int j) {
      constexpr int PH = decltype(ph)::value;
      gq = gz;
      gz = (gz == 2 * Op::GPL) ? 0 : gz + Op::GPL;
      if (threadIdx.x == 0) produce();
      mbar_wait(&bar[cs], phase);
      const int gr = (gz == 2 * Op::GPL) ? 0 : gz + Op::GPL;   // plane j-3
      if constexpr (KEEP >= 3)
        Op::template step<PH>(P, S, C, it, j, smem + cs * Op::SLOT, smem + cprev * Op::SLOT, smem + cpp * Op::SLOT,
                              gring + gz, gring + gq, gring + gr);
      else
        Op::template step<PH>(P, S, C, it, j, smem + cs * Op::SLOT, smem + cprev * Op::SLOT, gring + gz, gring + gq,
                              gring + gr);
      __syncthreads();
      cpp = cprev;
      cprev = cs;
      if (++cs == NS) {
        cs = 0;
        phase ^= 1;
      }
    };
    // unrolled by two so the PH-indexed register state never moves
    const int jb = it.zs - Op::PRO, je = it.ze - 1 + Op::EPI;
    int j = jb;
    if (j & 1) one(std::integral_constant<int, 1>(), j++);
    for (; j + 1 <= je; j += 2) {
      one(std::integral_constant<int, 0>(), j);
      one(std::integral_constant<int, 1>(), j + 1);
    }
    if (j <= je) one(std::integral_constant<int, 0>(), j);
  }
  Op::finish(P, S);
}

// Launch one persistent CTA per SM (fewer for tiny problems) over ntx x nty
// tiles of tx x ty nodes (x0 = tx * i + xoff, y0 = ty * j + yoff) and the
// z range [zlo, zhi).
template <class Op>
static cudaError_t launch_zpipe(typename Op::Params &P, int tx, int ty, int xoff, int yoff, int ntx, int nty, int zlo,
                                int zhi, cudaStream_t st) {
  if (zhi <= zlo) return cudaSuccess;
  cudaError_t e = cudaFuncSetAttribute(zpipe<Op>, cudaFuncAttributeMaxDynamicSharedMemorySize, Op::SMEM);
  if (e != cudaSuccess) return note_launch(e);
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  P.sc.tx = tx;
  P.sc.ty = ty;
  P.sc.xoff = xoff;
  P.sc.yoff = yoff;
  P.sc.ntx = ntx;
  P.sc.T = ntx * nty;
  P.sc.zlo = zlo;
  P.sc.zhi = zhi;
  P.sc.rev = zp_next_rev();
  zp_next_rev() = 0;
  const int slots = sms * OpNT<Op>::minb;   // resident CTAs
  P.sc.S = P.sc.T >= slots ? 1 : (slots + P.sc.T - 1) / P.sc.T;
  // at most MG_K3_ZPIECE planes per work unit (default 384 in fp64, whole tiles in fp32, where it measured
  // 0.5-0.8 % slower at 513^3 and 1025^3; 0: whole tiles).  Shorter units with a
  // barrier between waves keep neighbouring tiles within a few planes of each other (halo rows hit in L2):
  // measured on B200: 1025^3 fp64 cycle 18.79 -> 15.94 ms (asc_fine HBM reads 30.8 -> 22.6 GB), 513^3
  // 2.153 -> 2.142 ms (256: 15.95 / 2.145 ms; 128 and 192 slower)
  static const int zpiece_env = getenv("MG_K3_ZPIECE") ? atoi(getenv("MG_K3_ZPIECE")) : -1;
  static const int zpiece_h = getenv("MG_K3_ZPIECE_H") ? atoi(getenv("MG_K3_ZPIECE_H")) : -1;
  int zpiece = zpiece_env >= 0 ? zpiece_env : (OpEsz<Op>::v == 8 ? 384 : 0);
  if (OpHalf<Op>::v && zpiece_h >= 0) zpiece = zpiece_h;
  if (zpiece > 0 && (zhi - zlo + zpiece - 1) / zpiece > P.sc.S) P.sc.S = (zhi - zlo + zpiece - 1) / zpiece;
  if (P.sc.S > zhi - zlo) P.sc.S = zhi - zlo;
  const long long work = (long long)P.sc.T * (zhi - zlo);
  const int grid = work < slots ? (int)work : slots;
  // small levels (at most one work unit per CTA): programmatic launch (MG_PDL_SMALL3=1)
  static const bool pdl_small = env_flag("MG_PDL_SMALL3");
  const bool pdl = pdl_enabled() || (pdl_small && (long long)P.sc.T * P.sc.S <= grid);
  // two or more whole waves: barrier between them (MG_K3_WSYNC=0 turns it off), cooperative launch so
  // that every CTA is resident (checked: a grid the occupancy cannot hold runs without the barriers)
  static const bool wsync_on = !getenv("MG_K3_WSYNC") || env_flag("MG_K3_WSYNC");
  P.sc.wsync = 0;
  if (wsync_on && !pdl && grid == slots && (long long)P.sc.T * P.sc.S / grid >= 2) {
    int per_sm = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, zpipe<Op>, OpNT<Op>::nt, Op::SMEM) == cudaSuccess &&
        per_sm >= OpNT<Op>::minb)
      P.sc.wsync = 1;
  }
  if (P.sc.wsync) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(OpNT<Op>::nt);
    cfg.dynamicSmemBytes = Op::SMEM;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeCooperative;
    at[0].val.cooperative = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    return note_launch(cudaLaunchKernelEx(&cfg, zpipe<Op>, P));
  }
  return note_launch(launch_pdl_if(pdl, zpipe<Op>, dim3(grid), dim3(OpNT<Op>::nt), Op::SMEM, st, P));
}

// 3D tensor map over nx x ny x nz elements (row pitch, plane stride in
// elements), box bx x by x 1; out-of-bounds reads return zeros.
template <class T>
static bool tmap3(CUtensorMap *tm, const T *p, int64_t nx, int64_t ny, int64_t nz, int64_t pitch, int64_t plane, int bx,
                  int by) {
  uint64_t dims[3] = {(uint64_t)nx, (uint64_t)ny, (uint64_t)nz};
  uint32_t box[3] = {(uint32_t)bx, (uint32_t)by, 1};
  const bool ok = encode_tmap(tm, p, sizeof(T), 3, dims, (uint64_t)pitch, (uint64_t)plane, box);
  if (!ok) note_launch(cudaErrorInvalidValue);
  return ok;
}

}  // namespace mg
