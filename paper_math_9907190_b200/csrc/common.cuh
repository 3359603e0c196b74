// common.cuh -- shared device-side types of libmg (sm_100a).
//
// Data layout in HBM:
//   * dense level  (2D axis A(s), 3D green G(s)): one array over the lattice
//     of the octave, (M+1)^d points with the boundary, rows padded to a
//     128-byte multiple;  M = (n-1)/s.
//   * split level  (2D diagonal D(s), 3D red R(s) / magenta M(s)): the
//     level's nodes are stored packed per parity sublattice -- lattice point
//     (x, y[, z]) lives in sublattice (x&1, y&1[, z&1]) at index
//     (x>>1, y>>1[, z>>1]).  D(s) uses E=(0,0) and O=(1,1); R(s) uses
//     C=(0,0,0), Fx=(0,1,1), Fy=(1,0,1), Fz=(1,1,0); M(s) uses C and B=(1,1,1).
//     Every sublattice array has (M/2+1)^d entries with a 128-byte row pitch.
// Boundary entries are zero and are never written by any kernel.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace mg {

// Dense 2D lattice array; p addresses global lattice point (0, 0).
template <class T>
struct D2 {
  T *p;
  int64_t pitch;
  __device__ __forceinline__ T &operator()(int x, int y) const { return p[(int64_t)y * pitch + x]; }
};

// Split diagonal level: E = (even, even), O = (odd, odd) sublattices.
template <class T>
struct S2 {
  T *e, *o;
  int64_t pitch;
  __device__ __forceinline__ T get(int x, int y) const {
    return ((x & 1) ? o : e)[(int64_t)(y >> 1) * pitch + (x >> 1)];
  }
  __device__ __forceinline__ T &ref(int x, int y) const {
    return ((x & 1) ? o : e)[(int64_t)(y >> 1) * pitch + (x >> 1)];
  }
};

// A shared-memory tile addressed by global lattice coordinates:
// element (x, y) at p[(y - oy) * ld + (x - ox)].
template <class T>
struct Tile2 {
  const T *p;
  int ld, ox, oy;
  __device__ __forceinline__ T operator()(int x, int y) const { return p[(y - oy) * ld + (x - ox)]; }
};

// Dense 3D lattice array.
template <class T>
struct D3 {
  T *p;
  int64_t pitch, plane;
  __device__ __forceinline__ T &operator()(int x, int y, int z) const {
    return p[(int64_t)z * plane + (int64_t)y * pitch + x];
  }
};

// Split 3D level: s[(x&1) | (y&1)<<1 | (z&1)<<2] holds that parity sublattice.
template <class T>
struct S3 {
  T *s[8];
  int64_t pitch, plane;
  __device__ __forceinline__ T &ref(int x, int y, int z) const {
    return s[(x & 1) | ((y & 1) << 1) | ((z & 1) << 2)][(int64_t)(z >> 1) * plane + (int64_t)(y >> 1) * pitch + (x >> 1)];
  }
  __device__ __forceinline__ T get(int x, int y, int z) const { return ref(x, y, z); }
};

// Constants, each formed in double on the host and rounded once to T
// (DESIGN.md "Canonical arithmetic").
template <class T>
struct Coef {
  T invh2;   // (n-1)^2
  T c6;      // (n-1)^2 / 6
};

// Residual-norm sink: max |r| as the bit pattern of a non-negative double
// (monotone in the value; NaN sorts above +inf so it is never lost).
// Sum of squares (the L2 norm: ||r||_{2,h} = (h^d sum r^2)^(1/2))
// into l2[slot] when l2 is set: every node is counted once, by the pass that
// owns it, and only on rows (3D: planes) [nlo, nhi) of the fine grid (a slab
// solver's own rows; the ghost bands it also computes are another rank's).
struct NormSink {
  unsigned long long *slots;   // per-cycle maxima
  int *counter;                // which slot the current cycle writes
  int cap;
  double *l2 = nullptr;        // per-cycle sums of r^2 (or null)
  int nlo = 0, nhi = 1 << 30;  // fine rows / planes whose r^2 this launch adds
  __device__ __forceinline__ bool sums(int y) const { return l2 != nullptr && y >= nlo && y < nhi; }
};

__device__ __forceinline__ void norm_push(const NormSink &ns, double v) {
  if (ns.slots == nullptr) return;
  int slot = *ns.counter;
  if (slot >= ns.cap) slot = ns.cap - 1;
  atomicMax(ns.slots + slot, (unsigned long long)__double_as_longlong(v));
}
__device__ __forceinline__ void norm_push_l2(const NormSink &ns, double ss) {
  if (ns.l2 == nullptr || ns.slots == nullptr) return;
  int slot = *ns.counter;
  if (slot >= ns.cap) slot = ns.cap - 1;
  atomicAdd(ns.l2 + slot, ss);
}
__device__ __forceinline__ double sq(double v) { return v * v; }

// max that propagates NaN (a diverged residual must not be hidden).
__device__ __forceinline__ double nmax(double a, double b) { return (b > a || b != b) ? b : a; }

template <class T>
__device__ __forceinline__ double absd(T v) {
  return fabs((double)v);
}

// Warp-wide sum of squares, one atomic per warp (lane 0).
__device__ __forceinline__ void warp_l2_push(const NormSink &ns, double ss) {
  if (ns.l2 == nullptr) return;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
  if ((threadIdx.x & 31) == 0) norm_push_l2(ns, ss);
}

// Block-wide max reduction then one atomic per block (and the sum of squares,
// one atomic per warp, when ns.l2 is set).
template <int NT>
__device__ __forceinline__ void block_norm_push(const NormSink &ns, double v, double ss = 0.0) {
  if (ns.slots == nullptr) return;
  warp_l2_push(ns, ss);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    double w = __shfl_xor_sync(0xffffffffu, v, o);
    v = (w > v || w != w) ? w : v;
  }
  __shared__ double red[NT / 32];
  int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (lane == 0) red[wid] = v;
  __syncthreads();
  if (wid == 0) {
    v = (lane < NT / 32) ? red[lane] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      double w = __shfl_xor_sync(0xffffffffu, v, o);
      v = (w > v || w != w) ? w : v;
    }
    if (lane == 0) norm_push(ns, v);
  }
}

}  // namespace mg
