// conv.cu -- the paper's "usual" multigrid, the baseline
// of its "twice as fast" claim (
// Tables 1-3, "usual" rows).
//
// V(0,1) cycle on the standard hierarchy (factor-2 coarsening, M_l = (n-1)/2^l
// down to M = 2, one interior node):
//   descent  r_0 = f - L u (the library's residual kernels, order 2 or 4);
//            r_{l+1} = full weighting of r_l: 9-point (1/16)(4c + 2 axis +
//            diag) in 2D, 27-point (1/64)(8c + 4 faces + 2 edges + corners)
//            in 3D; max |r_0| to the residual history;
//   coarsest v = -(p H^2 r) / 4 (2D) or / 6 (3D) (reading A4);
//   ascent   bi/trilinear interpolation of v_{l+1}, then one two-colour
//            Jacobi sweep (reading A18): colour 1 (i+j[+k] odd) from the
//            interpolated field -- interpolated on the fly from v_{l+1}, never
//            stored -- colour 2 (even) from colour 1;
//   finest   the same on r_0, colour 1 also adds its v to u, colour 2 adds
//            its own: u <- u + v, in place (colour 2 reads only
//            r_0 and colour-1 v, never u).
// Every sum in the order of oracle/conventional.py; the library is compiled
// with --fmad=false, so the iterates are bit-identical to that oracle.
// Plain grid-stride node kernels (one thread per node, 32 x 8 blocks): this
// is the comparison baseline, not a tuned path.
#include <vector>

#include "kernels.h"
#include "ops2.cuh"
#include "solver.h"

namespace mg {
namespace cv {

constexpr int BX = 32, BY = 8;

// ------------------------------------------------------------------- 2D
template <class T>
__global__ void k_fw2(D2<const T> rf, D2<T> rc, int Mc) {
  const int X = blockIdx.x * BX + threadIdx.x, Y = blockIdx.y * BY + threadIdx.y;
  if (X < 1 || Y < 1 || X > Mc - 1 || Y > Mc - 1) return;
  const int x = 2 * X, y = 2 * Y;
  T ax = rf(x - 1, y) + rf(x + 1, y);
  ax = ax + rf(x, y - 1);
  ax = ax + rf(x, y + 1);
  T dg = rf(x - 1, y - 1) + rf(x + 1, y - 1);
  dg = dg + rf(x + 1, y + 1);
  dg = dg + rf(x - 1, y + 1);
  T t = (T)4 * rf(x, y);
  t = t + (T)2 * ax;
  t = t + dg;
  rc(X, Y) = t * (T)0.0625;
}

// bilinear interpolation of the coarse field at fine node (x, y)
template <class T>
__device__ __forceinline__ T vint2(const D2<const T> &vc, int x, int y) {
  const int X = x >> 1, Y = y >> 1;
  if (!(x & 1) && !(y & 1)) return vc(X, Y);
  if (!(y & 1)) return (vc(X, Y) + vc(X + 1, Y)) * (T)0.5;
  if (!(x & 1)) return (vc(X, Y) + vc(X, Y + 1)) * (T)0.5;
  T t = vc(X, Y) + vc(X + 1, Y);
  t = t + vc(X, Y + 1);
  t = t + vc(X + 1, Y + 1);
  return t * (T)0.25;
}

// colour 1 (x+y odd) from the interpolated field; u != null: finest level, u += v
template <class T>
__global__ void k_c1_2(D2<const T> vc, D2<const T> r, D2<T> v, int M, T c, T *u, int64_t up) {
  const int x = blockIdx.x * BX + threadIdx.x, y = blockIdx.y * BY + threadIdx.y;
  if (x < 1 || y < 1 || x > M - 1 || y > M - 1 || !((x + y) & 1)) return;
  const T w = jac4(c, r(x, y), vint2(vc, x - 1, y), vint2(vc, x, y - 1), vint2(vc, x + 1, y), vint2(vc, x, y + 1));
  v(x, y) = w;
  if (u) {
    T *p = u + (int64_t)y * up + x;
    *p = *p + w;
  }
}

// colour 2 (x+y even) from colour 1
template <class T>
__global__ void k_c2_2(D2<const T> r, D2<T> v, int M, T c, T *u, int64_t up) {
  const int x = blockIdx.x * BX + threadIdx.x, y = blockIdx.y * BY + threadIdx.y;
  if (x < 1 || y < 1 || x > M - 1 || y > M - 1 || ((x + y) & 1)) return;
  const T w = jac4(c, r(x, y), (T)v(x - 1, y), (T)v(x, y - 1), (T)v(x + 1, y), (T)v(x, y + 1));
  if (u) {
    T *p = u + (int64_t)y * up + x;
    *p = *p + w;
  } else {
    v(x, y) = w;
  }
}

// ------------------------------------------------------------------- 3D
template <class T>
__global__ void k_fw3(D3<const T> rf, D3<T> rc, int Mc) {
  const int X = blockIdx.x * BX + threadIdx.x, Y = blockIdx.y * BY + threadIdx.y, Z = blockIdx.z;
  if (X < 1 || Y < 1 || Z < 1 || X > Mc - 1 || Y > Mc - 1 || Z > Mc - 1) return;
  const int x = 2 * X, y = 2 * Y, z = 2 * Z;
  auto R = [&](int a, int b, int d) { return rf(x + a, y + b, z + d); };
  T fa = R(-1, 0, 0) + R(1, 0, 0);
  fa = fa + R(0, -1, 0);
  fa = fa + R(0, 1, 0);
  fa = fa + R(0, 0, -1);
  fa = fa + R(0, 0, 1);
  T ed = R(-1, -1, 0) + R(1, -1, 0);
  ed = ed + R(1, 1, 0);
  ed = ed + R(-1, 1, 0);
  ed = ed + R(-1, 0, -1);
  ed = ed + R(1, 0, -1);
  ed = ed + R(1, 0, 1);
  ed = ed + R(-1, 0, 1);
  ed = ed + R(0, -1, -1);
  ed = ed + R(0, 1, -1);
  ed = ed + R(0, 1, 1);
  ed = ed + R(0, -1, 1);
  T co = R(-1, -1, -1) + R(1, -1, -1);
  co = co + R(1, 1, -1);
  co = co + R(-1, 1, -1);
  co = co + R(-1, -1, 1);
  co = co + R(1, -1, 1);
  co = co + R(1, 1, 1);
  co = co + R(-1, 1, 1);
  T t = (T)8 * R(0, 0, 0);
  t = t + (T)4 * fa;
  t = t + (T)2 * ed;
  t = t + co;
  rc(X, Y, Z) = t * (T)(1.0 / 64.0);
}

// trilinear interpolation at fine node (x, y, z)
template <class T>
__device__ __forceinline__ T vint3(const D3<const T> &vc, int x, int y, int z) {
  const int X = x >> 1, Y = y >> 1, Z = z >> 1, ox = x & 1, oy = y & 1, oz = z & 1;
  const int k = ox + oy + oz;
  if (k == 0) return vc(X, Y, Z);
  if (k == 1) {
    if (ox) return (vc(X, Y, Z) + vc(X + 1, Y, Z)) * (T)0.5;
    if (oy) return (vc(X, Y, Z) + vc(X, Y + 1, Z)) * (T)0.5;
    return (vc(X, Y, Z) + vc(X, Y, Z + 1)) * (T)0.5;
  }
  if (k == 2) {
    T t;
    if (!oz) {   // x, y odd
      t = vc(X, Y, Z) + vc(X + 1, Y, Z);
      t = t + vc(X, Y + 1, Z);
      t = t + vc(X + 1, Y + 1, Z);
    } else if (!oy) {   // x, z odd
      t = vc(X, Y, Z) + vc(X + 1, Y, Z);
      t = t + vc(X, Y, Z + 1);
      t = t + vc(X + 1, Y, Z + 1);
    } else {   // y, z odd
      t = vc(X, Y, Z) + vc(X, Y + 1, Z);
      t = t + vc(X, Y, Z + 1);
      t = t + vc(X, Y + 1, Z + 1);
    }
    return t * (T)0.25;
  }
  T t = vc(X, Y, Z) + vc(X + 1, Y, Z);
  t = t + vc(X, Y + 1, Z);
  t = t + vc(X + 1, Y + 1, Z);
  t = t + vc(X, Y, Z + 1);
  t = t + vc(X + 1, Y, Z + 1);
  t = t + vc(X, Y + 1, Z + 1);
  t = t + vc(X + 1, Y + 1, Z + 1);
  return t * (T)0.125;
}

template <class T>
__device__ __forceinline__ T jac6c(T c, T r, T v0, T v1, T v2, T v3, T v4, T v5) {
  T t = -(c * r);
  t = t + v0;
  t = t + v1;
  t = t + v2;
  t = t + v3;
  t = t + v4;
  t = t + v5;
  return t * (T)(1.0 / 6.0);
}

template <class T>
__global__ void k_c1_3(D3<const T> vc, D3<const T> r, D3<T> v, int M, T c, T *u, int64_t up, int64_t upl) {
  const int x = blockIdx.x * BX + threadIdx.x, y = blockIdx.y * BY + threadIdx.y, z = blockIdx.z;
  if (x < 1 || y < 1 || z < 1 || x > M - 1 || y > M - 1 || z > M - 1 || !((x + y + z) & 1)) return;
  const T w = jac6c(c, r(x, y, z), vint3(vc, x - 1, y, z), vint3(vc, x, y - 1, z), vint3(vc, x + 1, y, z),
                    vint3(vc, x, y + 1, z), vint3(vc, x, y, z - 1), vint3(vc, x, y, z + 1));
  v(x, y, z) = w;
  if (u) {
    T *p = u + (int64_t)z * upl + (int64_t)y * up + x;
    *p = *p + w;
  }
}

template <class T>
__global__ void k_c2_3(D3<const T> r, D3<T> v, int M, T c, T *u, int64_t up, int64_t upl) {
  const int x = blockIdx.x * BX + threadIdx.x, y = blockIdx.y * BY + threadIdx.y, z = blockIdx.z;
  if (x < 1 || y < 1 || z < 1 || x > M - 1 || y > M - 1 || z > M - 1 || ((x + y + z) & 1)) return;
  const T w = jac6c(c, r(x, y, z), (T)v(x - 1, y, z), (T)v(x, y - 1, z), (T)v(x + 1, y, z), (T)v(x, y + 1, z),
                    (T)v(x, y, z - 1), (T)v(x, y, z + 1));
  if (u) {
    T *p = u + (int64_t)z * upl + (int64_t)y * up + x;
    *p = *p + w;
  } else {
    v(x, y, z) = w;
  }
}

// ------------------------------------------------------------- shared
template <class T>
__global__ void k_coarsest(T *v, const T *r, int64_t off, T c, T inv, int *counter) {
  v[off] = (-(c * r[off])) * inv;   // the one interior node; reading A4
  if (counter) *counter += 1;        // this cycle's norm slot is complete
}

// max |r| over the interior to this cycle's residual-history slot
template <class T, int DIM>
__global__ void k_norm_push(const T *r, int64_t pitch, int64_t plane, int M, NormSink ns) {
  double mx = 0.0, ss = 0.0;
  const int64_t W = M - 1, cnt = DIM == 2 ? W * W : W * W * W;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < cnt; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t x = t % W + 1, y = (t / W) % W + 1, z = DIM == 2 ? 0 : t / (W * W) + 1;
    const T v = r[z * plane + y * pitch + x];
    mx = nmax(mx, absd(v));
    if (ns.sums(DIM == 2 ? (int)y : (int)z)) ss += sq((double)v);
  }
  block_norm_push<256>(ns, mx, ss);
}

template <class T, int DIM>
struct ImplConv : ImplBase {
  const mg_solver *s;
  int k, L;
  int64_t n, pitch;
  std::vector<int> M;           // M_l = (n-1) >> l, l = 0 .. L (M_L = 2)
  std::vector<T *> r, v;        // level arrays (l = 0: r_0 and the colour-1 scratch of the finest level)
  std::vector<int64_t> lp;      // row pitch per level
  std::vector<T> c;             // p h_l^2
  T cL = 0;
  Coef<T> coef{};
  double p;
  explicit ImplConv(const mg_solver *sv) : s(sv), k(sv->k), n(sv->cfg.n), pitch(sv->pitch) {
    p = DIM == 2 ? sv->cfg.p[0] : sv->cfg.p[3];
  }
  int64_t pitch_for(int64_t cnt) const { return (cnt + 128 / (int64_t)sizeof(T) - 1) / (128 / (int64_t)sizeof(T)) * (128 / (int64_t)sizeof(T)); }
  size_t plane_of(int l) const { return (size_t)lp[l] * (M[l] + 1); }
  cudaError_t alloc() override {
    L = k - 1;
    M.resize(L + 1);
    r.resize(L + 1);
    v.resize(L + 1);
    lp.resize(L + 1);
    c.resize(L + 1);
    for (int l = 0; l <= L; l++) {
      M[l] = (int)((n - 1) >> l);
      lp[l] = l == 0 ? pitch : pitch_for(M[l] + 1);
      const size_t elems = (DIM == 2 ? 1 : (size_t)(M[l] + 1)) * plane_of(l);
      for (auto *a : {&r[l], &v[l]}) {
        void *q;
        cudaError_t e = dalloc(&q, sizeof(T) * elems);
        if (e) return e;
        *a = (T *)q;
      }
      const double h = 1.0 / (double)M[l];
      c[l] = (T)(p * h * h);
    }
    coef.invh2 = (T)((double)(n - 1) * (double)(n - 1));
    coef.c6 = (T)((double)(n - 1) * (double)(n - 1) / 6.0);
    return cudaSuccess;
  }
  NormSink sink() const {
    return NormSink{hist_on(s) ? s->d_hist : nullptr, s->d_counter, kHistCap, s->sum_l2 ? s->d_l2 : nullptr};
  }
  dim3 grid(int cnt, int nz = 1) const { return dim3((cnt + BX - 1) / BX, (cnt + BY - 1) / BY, nz); }

  template <class U>
  D2<U> d2(U *p, int l) const { return D2<U>{p, lp[l]}; }
  template <class U>
  D3<U> d3(U *p, int l) const { return D3<U>{p, lp[l], (int64_t)plane_of(l)}; }

  void residual0(const void *u, const void *f_eff, cudaStream_t st) {
    if (DIM == 2)
      launch2_residual<T>(D2<const T>{(const T *)u, pitch}, D2<const T>{(const T *)f_eff, pitch}, d2(r[0], 0), M[0],
                          s->cfg.order, coef, st);
    else
      launch3_residual<T>(D3<const T>{(const T *)u, pitch, pitch * n}, D3<const T>{(const T *)f_eff, pitch, pitch * n},
                          d3(r[0], 0), M[0], s->cfg.order, coef, st);
  }
  void push_norm(cudaStream_t st) {
    k_norm_push<T, DIM><<<148 * 4, 256, 0, st>>>(r[0], lp[0], DIM == 2 ? 0 : (int64_t)plane_of(0), M[0], sink());
  }
  void enqueue_cycle(const void *u_in, void *u_out, const void *f_eff, cudaStream_t st, Prof *prof) override {
    (void)u_out;   // in place (fast() is false)
    T *u = (T *)const_cast<void *>(u_in);
    const double w = sizeof(T);
    auto N = [&](int l) { return DIM == 2 ? (double)(M[l] - 1) * (M[l] - 1) : std::pow((double)(M[l] - 1), 3.0); };
    STEP("residual", 0, 2, w * (3 * N(0)));
    residual0(u, f_eff, st);
    push_norm(st);
    for (int l = 0; l < L; l++) {
      STEP("restrict", l, 1, w * (N(l) + N(l + 1)));
      if (DIM == 2)
        k_fw2<T><<<grid(M[l + 1] + 1), dim3(BX, BY), 0, st>>>(d2<const T>(r[l], l), d2(r[l + 1], l + 1), M[l + 1]);
      else
        k_fw3<T><<<grid(M[l + 1] + 1, M[l + 1] + 1), dim3(BX, BY), 0, st>>>(d3<const T>(r[l], l),
                                                                            d3(r[l + 1], l + 1), M[l + 1]);
    }
    STEP("coarsest", L, 1, w * 2);
    {
      const int64_t off = DIM == 2 ? lp[L] + 1 : (int64_t)plane_of(L) + lp[L] + 1;
      k_coarsest<T><<<1, 1, 0, st>>>(v[L], r[L], off, c[L], DIM == 2 ? (T)0.25 : (T)(1.0 / 6.0), s->d_counter);
    }
    for (int l = L - 1; l >= 0; l--) {
      T *uu = l == 0 ? u : nullptr;
      STEP("jacobi", l, 2, w * (N(l + 1) + 2 * N(l) + (l == 0 ? 2 * N(0) : 0)));
      if (DIM == 2) {
        k_c1_2<T><<<grid(M[l] + 1), dim3(BX, BY), 0, st>>>(d2<const T>(v[l + 1], l + 1), d2<const T>(r[l], l),
                                                          d2(v[l], l), M[l], c[l], uu, pitch);
        k_c2_2<T><<<grid(M[l] + 1), dim3(BX, BY), 0, st>>>(d2<const T>(r[l], l), d2(v[l], l), M[l], c[l], uu, pitch);
      } else {
        k_c1_3<T><<<grid(M[l] + 1, M[l] + 1), dim3(BX, BY), 0, st>>>(d3<const T>(v[l + 1], l + 1),
                                                                    d3<const T>(r[l], l), d3(v[l], l), M[l], c[l],
                                                                    uu, pitch, pitch * n);
        k_c2_3<T><<<grid(M[l] + 1, M[l] + 1), dim3(BX, BY), 0, st>>>(d3<const T>(r[l], l), d3(v[l], l), M[l], c[l],
                                                                    uu, pitch, pitch * n);
      }
    }
  }
  void enqueue_final_norm(void *u, const void *f_eff, cudaStream_t st) override {
    residual0(u, f_eff, st);
    push_norm(st);
  }
  void enqueue_residual(const void *u, const void *f, void *rr, cudaStream_t st, int64_t) override {
    if (DIM == 2)
      launch2_residual<T>(D2<const T>{(const T *)u, pitch}, D2<const T>{(const T *)f, pitch}, D2<T>{(T *)rr, pitch},
                          M[0], s->cfg.order, coef, st);
    else
      launch3_residual<T>(D3<const T>{(const T *)u, pitch, pitch * n}, D3<const T>{(const T *)f, pitch, pitch * n},
                          D3<T>{(T *)rr, pitch, pitch * n}, M[0], s->cfg.order, coef, st);
  }
  void enqueue_ftilde(const void *f, void *ft, cudaStream_t st, int64_t) override {
    if (DIM == 2)
      launch2_ftilde<T>(D2<const T>{(const T *)f, pitch}, D2<T>{(T *)ft, pitch}, M[0], st);
    else
      launch3_ftilde<T>(D3<const T>{(const T *)f, pitch, pitch * n}, D3<T>{(T *)ft, pitch, pitch * n}, M[0], st);
  }
  void enqueue_norm(const void *x, unsigned long long *mx, double *ss, cudaStream_t st, int64_t) override {
    if (DIM == 2)
      launch2_norm<T>(D2<const T>{(const T *)x, pitch}, M[0], mx, ss, st);
    else
      launch3_norm<T>(D3<const T>{(const T *)x, pitch, pitch * n}, M[0], mx, ss, st);
  }
  int launches_per_cycle() const override { return 2 + L + 1 + 2 * L; }
};

}  // namespace cv

ImplBase *make_conv(const mg_solver *s) {
  if (s->cfg.dim == 2) {
    if (s->cfg.dtype == MG_F64) return new cv::ImplConv<double, 2>(s);
    return new cv::ImplConv<float, 2>(s);
  }
  if (s->cfg.dtype == MG_F64) return new cv::ImplConv<double, 3>(s);
  return new cv::ImplConv<float, 3>(s);
}

}  // namespace mg
