// k3d.cu -- 3D kernels of the diagonal-multigrid V-cycle (sm_100a).
//
// Hierarchy per octave s: green G(s) (simple cubic) -> red R(s)
// (FCC: I+J+K even) -> magenta M(s) (BCC: I=J=K mod 2) -> G(2s).
// Canonical evaluation order and --fmad=false as in k2d.cu.
#include "kernels.h"
#include "ops3.cuh"

namespace mg {

constexpr int NT3 = 256;

static inline unsigned blocks3(int64_t n) { return (unsigned)((n + NT3 - 1) / NT3); }

// -------------------------------------------------- descent, finest level
// Fused a9+a10: residual recomputed, Erred onto R(1).  Thread (a,b,c) owns
// the 2x2x2 block at (2a,2b,2c); it writes the four red sublattices
// C (0,0,0), Fx (0,1,1), Fy (1,0,1), Fz (1,1,0) and reports max|r| of the block.
template <class T, int ORDER>
__global__ void __launch_bounds__(NT3) k3_desc_fine_ref(D3<const T> u, D3<const T> f, S3<T> rr, int M, Coef<T> k,
                                                        NormSink ns) {
  int H = M / 2 + 1;
  int64_t t = (int64_t)blockIdx.x * NT3 + threadIdx.x;
  double mx = 0.0, ss = 0.0;
  if (t < (int64_t)H * H * H) {
    int a = (int)(t % H), b = (int)((t / H) % H), c = (int)(t / ((int64_t)H * H));
    for (int par = 0; par < 8; par++) {
      int x = 2 * a + (par & 1), y = 2 * b + ((par >> 1) & 1), z = 2 * c + ((par >> 2) & 1);
      T rc = res3z<T, ORDER>(u, f, x, y, z, M, k);
      mx = nmax(mx, absd(rc));
      if (ns.sums(z)) ss += sq((double)rc);
      bool red = (((par & 1) + ((par >> 1) & 1) + ((par >> 2) & 1)) & 1) == 0;
      if (!red || !inner3(x, y, z, M)) continue;
      T nb[6];
#pragma unroll
      for (int q = 0; q < 6; q++) nb[q] = res3z<T, ORDER>(u, f, x + c_ax6[q][0], y + c_ax6[q][1], z + c_ax6[q][2], M, k);
      rr.ref(x, y, z) = erred(rc, nb);
    }
  }
  block_norm_push<NT3>(ns, mx, ss);
}

// ------------------------------------------------- descent, level kernels
// a10 for s > 1: Erred from the dense G(s) residual onto R(s).
template <class T>
__global__ void __launch_bounds__(NT3) k3_rest_gr_ref(D3<const T> r, S3<T> rr, int M) {
  int64_t W = M - 1;
  int64_t t = (int64_t)blockIdx.x * NT3 + threadIdx.x;
  if (t >= W * W * W) return;
  int x = (int)(t % W) + 1, y = (int)((t / W) % W) + 1, z = (int)(t / (W * W)) + 1;
  if ((x + y + z) & 1) return;
  T nb[6];
#pragma unroll
  for (int q = 0; q < 6; q++) nb[q] = r(x + c_ax6[q][0], y + c_ax6[q][1], z + c_ax6[q][2]);
  rr.ref(x, y, z) = erred(r(x, y, z), nb);
}

// a11: corners (all even) by Ermagc, centres (all odd) by
// Ermagm (zero self-weight).
template <class T>
__global__ void __launch_bounds__(NT3) k3_rest_rm_ref(S3<const T> rr, S3<T> rm, int M) {
  int64_t W = M - 1;
  int64_t t = (int64_t)blockIdx.x * NT3 + threadIdx.x;
  if (t >= W * W * W) return;
  int x = (int)(t % W) + 1, y = (int)((t / W) % W) + 1, z = (int)(t / (W * W)) + 1;
  int px = x & 1, py = y & 1, pz = z & 1;
  if (px != py || py != pz) return;
  T v;
  if (px == 0) {
    v = (T)12 * rr.get(x, y, z);
#pragma unroll
    for (int q = 0; q < 12; q++) v = v + rr.get(x + c_fd12[q][0], y + c_fd12[q][1], z + c_fd12[q][2]);
    v = v * (T)(1.0 / 24.0);
  } else {
    v = rr.get(x + c_ax6[0][0], y + c_ax6[0][1], z + c_ax6[0][2]);
#pragma unroll
    for (int q = 1; q < 6; q++) v = v + rr.get(x + c_ax6[q][0], y + c_ax6[q][1], z + c_ax6[q][2]);
    v = v * (T)(1.0 / 6.0);
  }
  rm.ref(x, y, z) = v;
}

// a12: Erblu onto G(2s): (1/16)(8r + sum of the 8 centres).
template <class T>
__global__ void __launch_bounds__(NT3) k3_rest_mg_ref(S3<const T> rm, D3<T> rg, int Mc) {
  int64_t W = Mc - 1;
  int64_t t = (int64_t)blockIdx.x * NT3 + threadIdx.x;
  if (t >= W * W * W) return;
  int X = (int)(t % W) + 1, Y = (int)((t / W) % W) + 1, Z = (int)(t / (W * W)) + 1;
  int x = 2 * X, y = 2 * Y, z = 2 * Z;
  T v = (T)8 * rm.get(x, y, z);
#pragma unroll
  for (int q = 0; q < 8; q++) v = v + rm.get(x + c_bd8[q][0], y + c_bd8[q][1], z + c_bd8[q][2]);
  rg(X, Y, Z) = v * (T)(1.0 / 16.0);
}

// Coarsest (reading A4): v = (1/6)(-p_g H^2 r) at the one interior node.
template <class T>
__global__ void k3_coarsest(D3<const T> r, D3<T> v, T c, int *counter) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    v(1, 1, 1) = (-(c * r(1, 1, 1))) * (T)(1.0 / 6.0);
    if (counter) *counter += 1;
  }
}

// ------------------------------------------------------ ascent, magenta
// a13: Emprolm on the centres from G(2s), then Emprolb
// on the corners from the new centres; c = 4 p_m (sh)^2.
template <class T>
__global__ void __launch_bounds__(NT3) k3_jac_m1_ref(D3<const T> vc, S3<const T> r, S3<T> v, int M, T c) {
  int64_t W = M / 2;
  int64_t t = (int64_t)blockIdx.x * NT3 + threadIdx.x;
  if (t >= W * W * W) return;
  int x = 2 * (int)(t % W) + 1, y = 2 * (int)((t / W) % W) + 1, z = 2 * (int)(t / (W * W)) + 1;
  T s = -(c * r.get(x, y, z));
#pragma unroll
  for (int q = 0; q < 8; q++) s = s + vc((x + c_bd8[q][0]) / 2, (y + c_bd8[q][1]) / 2, (z + c_bd8[q][2]) / 2);
  v.ref(x, y, z) = s * (T)0.125;
}

template <class T>
__global__ void __launch_bounds__(NT3) k3_jac_m2_ref(S3<const T> r, S3<T> v, int M, T c) {
  int64_t W = M / 2 - 1;
  int64_t t = (int64_t)blockIdx.x * NT3 + threadIdx.x;
  if (t >= W * W * W) return;
  int x = 2 * ((int)(t % W) + 1), y = 2 * ((int)((t / W) % W) + 1), z = 2 * ((int)(t / (W * W)) + 1);
  T s = -(c * r.get(x, y, z));
#pragma unroll
  for (int q = 0; q < 8; q++) s = s + v.get(x + c_bd8[q][0], y + c_bd8[q][1], z + c_bd8[q][2]);
  v.ref(x, y, z) = s * (T)0.125;
}

// ---------------------------------------------------------- ascent, red
// a14: Erprolr on the face centres from M(s), c1 = 2 p_r1 (sh)^2,
// then Erprolm on the corners from the new face values,
// c2 = 4 p_r2 (sh)^2.  Magenta centres are not red nodes.
template <class T>
__global__ void __launch_bounds__(NT3) k3_jac_r1_ref(S3<const T> vm, S3<const T> r, S3<T> v, int M, T c1) {
  int64_t W = M - 1;
  int64_t t = (int64_t)blockIdx.x * NT3 + threadIdx.x;
  if (t >= W * W * W) return;
  int x = (int)(t % W) + 1, y = (int)((t / W) % W) + 1, z = (int)(t / (W * W)) + 1;
  if ((x + y + z) & 1) return;
  int ne = ((x & 1) == 0) + ((y & 1) == 0) + ((z & 1) == 0);
  if (ne != 1) return;
  int a = ((x & 1) == 0) ? 0 : (((y & 1) == 0) ? 1 : 2);
  T nrm = vm.get(x + c_erp[a][0][0], y + c_erp[a][0][1], z + c_erp[a][0][2]);
  nrm = nrm + vm.get(x + c_erp[a][1][0], y + c_erp[a][1][1], z + c_erp[a][1][2]);
  T s = -(c1 * r.get(x, y, z));
  s = s + (T)2 * nrm;
#pragma unroll
  for (int q = 2; q < 6; q++) s = s + vm.get(x + c_erp[a][q][0], y + c_erp[a][q][1], z + c_erp[a][q][2]);
  v.ref(x, y, z) = s * (T)0.125;
}

template <class T>
__global__ void __launch_bounds__(NT3) k3_jac_r2_ref(S3<const T> r, S3<T> v, int M, T c2) {
  int64_t W = M / 2 - 1;
  int64_t t = (int64_t)blockIdx.x * NT3 + threadIdx.x;
  if (t >= W * W * W) return;
  int x = 2 * ((int)(t % W) + 1), y = 2 * ((int)((t / W) % W) + 1), z = 2 * ((int)(t / (W * W)) + 1);
  T s = -(c2 * r.get(x, y, z));
#pragma unroll
  for (int q = 0; q < 12; q++) s = s + v.get(x + c_fd12[q][0], y + c_fd12[q][1], z + c_fd12[q][2]);
  v.ref(x, y, z) = s * (T)(1.0 / 12.0);
}

// -------------------------------------------------------- ascent, green
// a15 (s > 1): Egprolg on green-only nodes (odd sum) from R(s),
// then Egprolr on the red nodes; c = p_g (sh)^2.
template <class T>
__global__ void __launch_bounds__(NT3) k3_jac_g1_ref(S3<const T> vr, D3<const T> r, D3<T> v, int M, T c) {
  int64_t W = M - 1;
  int64_t t = (int64_t)blockIdx.x * NT3 + threadIdx.x;
  if (t >= W * W * W) return;
  int x = (int)(t % W) + 1, y = (int)((t / W) % W) + 1, z = (int)(t / (W * W)) + 1;
  if (((x + y + z) & 1) == 0) return;
  T s = -(c * r(x, y, z));
#pragma unroll
  for (int q = 0; q < 6; q++) s = s + vr.get(x + c_ax6[q][0], y + c_ax6[q][1], z + c_ax6[q][2]);
  v(x, y, z) = s * (T)(1.0 / 6.0);
}

template <class T>
__global__ void __launch_bounds__(NT3) k3_jac_g2_ref(D3<const T> r, D3<T> v, int M, T c) {
  int64_t W = M - 1;
  int64_t t = (int64_t)blockIdx.x * NT3 + threadIdx.x;
  if (t >= W * W * W) return;
  int x = (int)(t % W) + 1, y = (int)((t / W) % W) + 1, z = (int)(t / (W * W)) + 1;
  if ((x + y + z) & 1) return;
  T s = -(c * r(x, y, z));
#pragma unroll
  for (int q = 0; q < 6; q++) s = s + v(x + c_ax6[q][0], y + c_ax6[q][1], z + c_ax6[q][2]);
  v(x, y, z) = s * (T)(1.0 / 6.0);
}

// a15 at s = 1 with the residual recomputed from u, f into a dense scratch,
// then u <- u + v.
template <class T, int ORDER>
__global__ void __launch_bounds__(NT3) k3_asc_fine1_ref(S3<const T> vr, D3<const T> u, D3<const T> f, D3<T> v, int M,
                                                        T c, Coef<T> k) {
  int64_t W = M - 1;
  int64_t t = (int64_t)blockIdx.x * NT3 + threadIdx.x;
  if (t >= W * W * W) return;
  int x = (int)(t % W) + 1, y = (int)((t / W) % W) + 1, z = (int)(t / (W * W)) + 1;
  if (((x + y + z) & 1) == 0) return;
  T s = -(c * res3<T, ORDER>(u, f, x, y, z, k));
#pragma unroll
  for (int q = 0; q < 6; q++) s = s + vr.get(x + c_ax6[q][0], y + c_ax6[q][1], z + c_ax6[q][2]);
  v(x, y, z) = s * (T)(1.0 / 6.0);
}

template <class T, int ORDER>
__global__ void __launch_bounds__(NT3) k3_asc_fine2_ref(D3<const T> u, D3<const T> f, D3<T> v, int M, T c, Coef<T> k) {
  int64_t W = M - 1;
  int64_t t = (int64_t)blockIdx.x * NT3 + threadIdx.x;
  if (t >= W * W * W) return;
  int x = (int)(t % W) + 1, y = (int)((t / W) % W) + 1, z = (int)(t / (W * W)) + 1;
  if ((x + y + z) & 1) return;
  T s = -(c * res3<T, ORDER>(u, f, x, y, z, k));
#pragma unroll
  for (int q = 0; q < 6; q++) s = s + v(x + c_ax6[q][0], y + c_ax6[q][1], z + c_ax6[q][2]);
  v(x, y, z) = s * (T)(1.0 / 6.0);
}

template <class T>
__global__ void __launch_bounds__(NT3) k3_update_ref(D3<const T> uo, D3<const T> v, D3<T> un, int M) {
  int64_t W = M - 1;
  int64_t t = (int64_t)blockIdx.x * NT3 + threadIdx.x;
  if (t >= W * W * W) return;
  int x = (int)(t % W) + 1, y = (int)((t / W) % W) + 1, z = (int)(t / (W * W)) + 1;
  un(x, y, z) = uo(x, y, z) + v(x, y, z);
}

// planes [z0, z0 + nz) (multi-GPU slabs; the whole grid by default)
template <class T, int ORDER>
__global__ void __launch_bounds__(NT3) k3_residual(D3<const T> u, D3<const T> f, D3<T> r, int M, Coef<T> k, int z0,
                                                   int nz) {
  int64_t W = M + 1;
  int64_t t = (int64_t)blockIdx.x * NT3 + threadIdx.x;
  if (t >= W * W * nz) return;
  int x = (int)(t % W), y = (int)((t / W) % W), z = (int)(t / (W * W)) + z0;
  r(x, y, z) = res3z<T, ORDER>(u, f, x, y, z, M, k);
}

// f~ of Efos4: (1/12)(6f + f_{i+1} + f_{j+1} + f_{i-1} + f_{j-1} + f_{k+1} + f_{k-1}).
template <class T>
__global__ void __launch_bounds__(NT3) k3_ftilde(D3<const T> f, D3<T> ft, int M, int z0, int nz) {
  int64_t W = M - 1;
  int64_t t = (int64_t)blockIdx.x * NT3 + threadIdx.x;
  if (t >= W * W * nz) return;
  int x = (int)(t % W) + 1, y = (int)((t / W) % W) + 1, z = (int)(t / (W * W)) + z0;
  T s = (T)6 * f(x, y, z);
  s = s + f(x + 1, y, z);
  s = s + f(x, y + 1, z);
  s = s + f(x - 1, y, z);
  s = s + f(x, y - 1, z);
  s = s + f(x, y, z + 1);
  s = s + f(x, y, z - 1);
  ft(x, y, z) = s * (T)(1.0 / 12.0);
}

template <class T>
__global__ void __launch_bounds__(NT3) k3_norm(D3<const T> a, int M, unsigned long long *mx_out, double *ss_out, int z0,
                                               int nz) {
  int64_t W = M - 1;
  double mx = 0.0, ss = 0.0;
  for (int64_t t = (int64_t)blockIdx.x * NT3 + threadIdx.x; t < W * W * nz; t += (int64_t)gridDim.x * NT3) {
    int x = (int)(t % W) + 1, y = (int)((t / W) % W) + 1, z = (int)(t / (W * W)) + z0;
    double v = (double)a(x, y, z);
    mx = nmax(mx, fabs(v));
    ss += v * v;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    ss += __shfl_xor_sync(0xffffffffu, ss, o);
    mx = nmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  }
  __shared__ double rs[NT3 / 32], rm[NT3 / 32];
  int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (lane == 0) {
    rs[wid] = ss;
    rm[wid] = mx;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double s2 = 0.0, m2 = 0.0;
    for (int i = 0; i < NT3 / 32; i++) {
      s2 += rs[i];
      m2 = nmax(m2, rm[i]);
    }
    atomicAdd(ss_out, s2);
    atomicMax(mx_out, (unsigned long long)__double_as_longlong(m2));
  }
}

// ================================================================ launchers

template <class T>
static D3<const T> cd3(const D3<T> &a) {
  return D3<const T>{a.p, a.pitch, a.plane};
}
template <class T>
static S3<const T> cs3(const S3<T> &a) {
  S3<const T> o;
  for (int i = 0; i < 8; i++) o.s[i] = a.s[i];
  o.pitch = a.pitch;
  o.plane = a.plane;
  return o;
}

template <class T>
void launch3_desc_fine(const D3<const T> &u, const D3<const T> &f, const S3<T> &rr, int M, int order,
                       const Coef<T> &k, const NormSink &ns, cudaStream_t st) {
  int64_t H = M / 2 + 1;
  if (order == 2)
    k3_desc_fine_ref<T, 2><<<blocks3(H * H * H), NT3, 0, st>>>(u, f, rr, M, k, ns);
  else
    k3_desc_fine_ref<T, 4><<<blocks3(H * H * H), NT3, 0, st>>>(u, f, rr, M, k, ns);
}

template <class T>
void launch3_rest_gr(const D3<T> &r, const S3<T> &rr, int M, cudaStream_t st) {
  int64_t W = M - 1;
  k3_rest_gr_ref<T><<<blocks3(W * W * W), NT3, 0, st>>>(cd3(r), rr, M);
}

template <class T>
void launch3_rest_rm(const S3<T> &rr, const S3<T> &rm, int M, cudaStream_t st) {
  int64_t W = M - 1;
  k3_rest_rm_ref<T><<<blocks3(W * W * W), NT3, 0, st>>>(cs3(rr), rm, M);
}

template <class T>
void launch3_rest_mg(const S3<T> &rm, const D3<T> &rg, int Mc, cudaStream_t st) {
  int64_t W = Mc - 1;
  k3_rest_mg_ref<T><<<blocks3(W * W * W), NT3, 0, st>>>(cs3(rm), rg, Mc);
}

template <class T>
void launch3_coarsest(const D3<T> &r, const D3<T> &v, T c, int *counter, cudaStream_t st) {
  k3_coarsest<T><<<1, 32, 0, st>>>(cd3(r), v, c, counter);
}

template <class T>
void launch3_jac_m(const D3<T> &vc, const S3<T> &r, const S3<T> &v, int M, T c, cudaStream_t st) {
  int64_t W = M / 2;
  k3_jac_m1_ref<T><<<blocks3(W * W * W), NT3, 0, st>>>(cd3(vc), cs3(r), v, M, c);
  if (W - 1 > 0) k3_jac_m2_ref<T><<<blocks3((W - 1) * (W - 1) * (W - 1)), NT3, 0, st>>>(cs3(r), v, M, c);
}

template <class T>
void launch3_jac_r(const S3<T> &vm, const S3<T> &r, const S3<T> &v, int M, T c1, T c2, cudaStream_t st) {
  int64_t W = M - 1;
  k3_jac_r1_ref<T><<<blocks3(W * W * W), NT3, 0, st>>>(cs3(vm), cs3(r), v, M, c1);
  int64_t W2 = M / 2 - 1;
  if (W2 > 0) k3_jac_r2_ref<T><<<blocks3(W2 * W2 * W2), NT3, 0, st>>>(cs3(r), v, M, c2);
}

template <class T>
void launch3_jac_g(const S3<T> &vr, const D3<T> &r, const D3<T> &v, int M, T c, cudaStream_t st) {
  int64_t W = M - 1;
  k3_jac_g1_ref<T><<<blocks3(W * W * W), NT3, 0, st>>>(cs3(vr), cd3(r), v, M, c);
  k3_jac_g2_ref<T><<<blocks3(W * W * W), NT3, 0, st>>>(cd3(r), v, M, c);
}

template <class T>
void launch3_asc_fine(const S3<T> &vr, const D3<T> &u, const D3<const T> &f, const D3<T> &scratch, const D3<T> &un,
                      int M, int order, T c, const Coef<T> &k, cudaStream_t st) {
  int64_t W = M - 1;
  unsigned g = blocks3(W * W * W);
  if (order == 2) {
    k3_asc_fine1_ref<T, 2><<<g, NT3, 0, st>>>(cs3(vr), cd3(u), f, scratch, M, c, k);
    k3_asc_fine2_ref<T, 2><<<g, NT3, 0, st>>>(cd3(u), f, scratch, M, c, k);
  } else {
    k3_asc_fine1_ref<T, 4><<<g, NT3, 0, st>>>(cs3(vr), cd3(u), f, scratch, M, c, k);
    k3_asc_fine2_ref<T, 4><<<g, NT3, 0, st>>>(cd3(u), f, scratch, M, c, k);
  }
  k3_update_ref<T><<<g, NT3, 0, st>>>(cd3(u), cd3(scratch), un, M);
}

// [zlo, zhi) clipped to the planes the kernel covers (residual: 0..M, the
// others: the interior 1..M-1)
template <class T>
void launch3_residual(const D3<const T> &u, const D3<const T> &f, const D3<T> &r, int M, int order, const Coef<T> &k,
                      cudaStream_t st, int zlo, int zhi) {
  int64_t W = M + 1;
  if (zhi < 0 || zhi > M + 1) zhi = M + 1;
  if (zlo < 0) zlo = 0;
  const int nz = zhi - zlo;
  if (nz <= 0) return;
  if (order == 2)
    k3_residual<T, 2><<<blocks3(W * W * nz), NT3, 0, st>>>(u, f, r, M, k, zlo, nz);
  else
    k3_residual<T, 4><<<blocks3(W * W * nz), NT3, 0, st>>>(u, f, r, M, k, zlo, nz);
}

template <class T>
void launch3_ftilde(const D3<const T> &f, const D3<T> &ft, int M, cudaStream_t st, int zlo, int zhi) {
  int64_t W = M - 1;
  if (zhi < 0 || zhi > M) zhi = M;
  if (zlo < 1) zlo = 1;
  const int nz = zhi - zlo;
  if (nz > 0) k3_ftilde<T><<<blocks3(W * W * nz), NT3, 0, st>>>(f, ft, M, zlo, nz);
}

template <class T>
void launch3_norm(const D3<const T> &a, int M, unsigned long long *mx, double *ss, cudaStream_t st, int zlo, int zhi) {
  if (zhi < 0 || zhi > M) zhi = M;
  if (zlo < 1) zlo = 1;
  const int nz = zhi - zlo;
  if (nz > 0) k3_norm<T><<<148 * 4, NT3, 0, st>>>(a, M, mx, ss, zlo, nz);
}

#define INST3(T)                                                                                                    \
  template void launch3_desc_fine<T>(const D3<const T> &, const D3<const T> &, const S3<T> &, int, int,            \
                                     const Coef<T> &, const NormSink &, cudaStream_t);                             \
  template void launch3_rest_gr<T>(const D3<T> &, const S3<T> &, int, cudaStream_t);                               \
  template void launch3_rest_rm<T>(const S3<T> &, const S3<T> &, int, cudaStream_t);                               \
  template void launch3_rest_mg<T>(const S3<T> &, const D3<T> &, int, cudaStream_t);                               \
  template void launch3_coarsest<T>(const D3<T> &, const D3<T> &, T, int *, cudaStream_t);                         \
  template void launch3_jac_m<T>(const D3<T> &, const S3<T> &, const S3<T> &, int, T, cudaStream_t);               \
  template void launch3_jac_r<T>(const S3<T> &, const S3<T> &, const S3<T> &, int, T, T, cudaStream_t);            \
  template void launch3_jac_g<T>(const S3<T> &, const D3<T> &, const D3<T> &, int, T, cudaStream_t);               \
  template void launch3_asc_fine<T>(const S3<T> &, const D3<T> &, const D3<const T> &, const D3<T> &, const D3<T> &, \
                                    int, int, T,                                                                   \
                                    const Coef<T> &, cudaStream_t);                                                \
  template void launch3_residual<T>(const D3<const T> &, const D3<const T> &, const D3<T> &, int, int,             \
                                    const Coef<T> &, cudaStream_t, int, int);                                      \
  template void launch3_ftilde<T>(const D3<const T> &, const D3<T> &, int, cudaStream_t, int, int);                \
  template void launch3_norm<T>(const D3<const T> &, int, unsigned long long *, double *, cudaStream_t, int, int);

INST3(float)
INST3(double)

}  // namespace mg
