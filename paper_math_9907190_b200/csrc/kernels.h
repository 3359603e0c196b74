// kernels.h -- internal launcher interface between the host plan (mg_api.cpp)
// and the sm_100a kernels (k2d.cu, k3d.cu).  Not part of the public ABI.
#pragma once
#include <cstdlib>

#include "common.cuh"

namespace mg {

// A boolean environment switch: set and not "0".
inline bool env_flag(const char *name) {
  const char *e = std::getenv(name);
  return e && *e && !(e[0] == '0' && e[1] == 0);
}

// ----------------------------------------------------------------- 2D
template <class T>
void launch2_desc_fine(const D2<const T> &u, const D2<const T> &f, const S2<T> &d, int M, int order, const Coef<T> &k,
                       const NormSink &ns, cudaStream_t st);
template <class T>
void launch2_rest_ad(const D2<T> &r, const S2<T> &d, int M, cudaStream_t st);
template <class T>
void launch2_rest_da(const S2<T> &d, const D2<T> &r, int Mc, cudaStream_t st);
template <class T>
void launch2_coarsest(const D2<T> &r, const D2<T> &v, T c, int *counter, cudaStream_t st);
template <class T>
void launch2_jac_d(const D2<T> &vc, const S2<T> &r, const S2<T> &v, int M, T c, cudaStream_t st);
template <class T>
void launch2_jac_a(const S2<T> &vd, const D2<T> &r, const D2<T> &v, int M, T c, cudaStream_t st);
template <class T>
void launch2_asc_fine(const S2<T> &vd, const D2<T> &u, const D2<const T> &f, const D2<T> &scratch, const D2<T> &un,
                      int M, int order, T c, const Coef<T> &k, cudaStream_t st);

// Per-octave level descriptors for the single-CTA coarse kernel.
template <class T>
struct Lev2 {
  S2<T> rD, vD;   // D(s)
  D2<T> rA, vA;   // A(s)
  int M;
  T cD, cA;
};
// All octaves o >= oc (oc >= 1) in one CTA: restrictions from r_A(oc) down,
// the coarsest step, the Jacobi steps back up to v_A(oc).
// h_lev: the host copy of the descriptors (enables the compile-time solver
// k2_coarse_ct for M(oc) <= 64), or null.
template <class T>
void launch2_coarse(const Lev2<T> *d_lev, int oc, int k, int *counter, cudaStream_t st,
                    const Lev2<T> *h_lev = nullptr);
// Octaves om .. oc-1 grid-wide and oc .. k-1 in one CTA's shared memory, one
// cooperative launch (h_lev: host copy of the descriptors).  false: not launched.
template <class T>
bool launch2_tail(const Lev2<T> *h_lev, int om, int oc, int k, int *counter, cudaStream_t st);

// TMA tile kernels (k2f.cu); every pointer/pitch must be 16-byte aligned.
// Rows2: the output rows a launch writes and the local allocations of its
// inputs (multi-GPU slabs); the default (all -1 / 0) is the whole level.
// First configuration failure of a kernel launch on this host thread (a
// rejected dynamic shared-memory size, an unencodable tensor map, a launch
// error): the generic launchers record it here, and the ABI checks and clears
// it after enqueueing a cycle, so a pass that could not be launched is an
// MG_ECUDA error, never a silently skipped pass.
inline cudaError_t &sticky_launch_error() {
  static thread_local cudaError_t e = cudaSuccess;
  return e;
}
inline cudaError_t note_launch(cudaError_t e) {
  if (e != cudaSuccess && sticky_launch_error() == cudaSuccess) sticky_launch_error() = e;
  return e;
}
inline cudaError_t take_launch_error() {
  cudaError_t e = sticky_launch_error();
  sticky_launch_error() = cudaSuccess;
  return e;
}

// Direction of the next 3D plane-pipeline launch on this host thread
// (zpipe Sched::rev, items walked in reverse): the 3D V-cycle alternates it
// so that every pass first reads what its producer wrote last (still in L2).
// launch_zpipe resets it to 0.
inline int &zp_next_rev() {
  static thread_local int r = 0;
  return r;
}

struct Rows2 {
  bool rev = false;         // walk the tiles in descending order (reuse the L2-resident tail of the producer's output)
  int ylo = 0, yhi = -1;    // output rows [ylo, yhi) in the output array's row units (-1: all)
  int fy0 = 0, frows = -1;  // full-resolution inputs: global row of local row 0, local rows (-1: all)
  int hy0 = 0, hrows = -1;  // half-resolution inputs (E/O of D(s), A(2s))
};
template <class T>
cudaError_t fast2_desc_fine(const T *u, const T *f, int64_t pitch, const S2<T> &d, int M, int order, const Coef<T> &k,
                            const NormSink &ns, cudaStream_t st, const Rows2 &rw = Rows2());
template <class T>
cudaError_t fast2_asc_fine(const S2<T> &vd, const T *u_old, const T *f, int64_t pitch, T *u_new, int M, int order, T c,
                           const Coef<T> &k, cudaStream_t st, const Rows2 &rw = Rows2());
template <class T>
cudaError_t fast2_jac_a(const S2<T> &vd, const D2<T> &r, const D2<T> &v, int M, T c, cudaStream_t st,
                        const Rows2 &rw = Rows2());
template <class T>
cudaError_t fast2_rest_ad(const D2<T> &r, const S2<T> &d, int M, cudaStream_t st, const Rows2 &rw = Rows2());
template <class T>
cudaError_t fast2_rest_da(const S2<T> &d, const D2<T> &r, int Mc, cudaStream_t st, const Rows2 &rw = Rows2());
// Finest ascent of one cycle fused with the finest descent of the next
// (u_new = u_old + v_A(1); r = f - L u_new -> Erest2r onto d; max|r| -> ns);
// whole domain only (single GPU).  ra, d2 non-null: the next descent's octave
// pair as well (r_A(2) -> ra, r_D(2) -> d2, fast2_rest_dad's results).
template <class T>
cudaError_t fast2_asc_desc(const S2<T> &vd, const T *u_old, const T *f, int64_t pitch, T *u_new, const S2<T> &d,
                           int M, int order, T c, const Coef<T> &k, const NormSink &ns, cudaStream_t st, bool rev,
                           const D2<T> *ra = nullptr, const S2<T> *d2 = nullptr);
template <class T>
cudaError_t fast2_jac_d(const D2<T> &vc, const S2<T> &r, const S2<T> &v, int M, T c, cudaStream_t st,
                        const Rows2 &rw = Rows2());
// rest_da of D(s) (r_A(s+1), written) fused with rest_ad of A(s+1) (r_D(s+1));
// Mc = the size of A(s+1).
// Rows [ylo, yhi) of A(s+1) (ylo even) only -- the slab solvers' bands; yhi < 0: the whole level.
template <class T>
cudaError_t fast2_rest_dad(const S2<T> &d, const D2<T> &ra, const S2<T> &rd, int Mc, cudaStream_t st, bool rev,
                           int ylo = 0, int yhi = -1);
// jac_a on A(s) (v_A(s) from v_D(s), r_A(s); M = the fine size of D(s-1))
// fused with jac_d on D(s-1) (v_D(s-1) from v_A(s), r_D(s-1)): v_A(s) stays in
// shared memory.
// Rows [ylo, yhi) of D(s-1)'s E/O arrays (= A(s) rows; ylo even) only; yhi < 0: the whole level.
template <class T>
cudaError_t fast2_jac_ad(const S2<T> &vd, const D2<T> &ra, T ca, const S2<T> &rd, const S2<T> &v, int M, T cd,
                         cudaStream_t st, bool rev, int ylo = 0, int yhi = -1);
template <class T>
void launch2_gather_d(const D2<T> &v, const S2<T> &d, int M, cudaStream_t st);
template <class T>
void launch2_asc_fine_sweeps(const S2<T> &vd, const D2<T> &u, const D2<const T> &f, const D2<T> &scratch,
                             const D2<T> &un, int M, int order, T c, const Coef<T> &k, int sweeps, const S2<T> &tmp,
                             cudaStream_t st);
template <class T>
void launch2_residual(const D2<const T> &u, const D2<const T> &f, const D2<T> &r, int M, int order, const Coef<T> &k,
                      cudaStream_t st);
template <class T>
void launch2_ftilde(const D2<const T> &f, const D2<T> &ft, int M, cudaStream_t st);
template <class T>
void launch2_norm(const D2<const T> &a, int M, unsigned long long *mx, double *ss, cudaStream_t st);

template <class T>
void launch2_ftilde_rows(const D2<const T> &f, const D2<T> &ft, int M, int ylo, int yhi, cudaStream_t st);
template <class T>
void launch2_residual_rows(const D2<const T> &u, const D2<const T> &f, const D2<T> &r, int M, int order,
                           const Coef<T> &k, int ylo, int yhi, cudaStream_t st);
template <class T>
void launch2_norm_rows(const D2<const T> &a, int M, int ylo, int yhi, unsigned long long *mx, double *ss,
                       cudaStream_t st);

// ----------------------------------------------------------------- 3D
template <class T>
void launch3_desc_fine(const D3<const T> &u, const D3<const T> &f, const S3<T> &rr, int M, int order,
                       const Coef<T> &k, const NormSink &ns, cudaStream_t st);
template <class T>
void launch3_rest_gr(const D3<T> &r, const S3<T> &rr, int M, cudaStream_t st);
template <class T>
void launch3_rest_rm(const S3<T> &rr, const S3<T> &rm, int M, cudaStream_t st);
template <class T>
void launch3_rest_mg(const S3<T> &rm, const D3<T> &rg, int Mc, cudaStream_t st);
template <class T>
void launch3_coarsest(const D3<T> &r, const D3<T> &v, T c, int *counter, cudaStream_t st);
template <class T>
void launch3_jac_m(const D3<T> &vc, const S3<T> &r, const S3<T> &v, int M, T c, cudaStream_t st);
template <class T>
void launch3_jac_r(const S3<T> &vm, const S3<T> &r, const S3<T> &v, int M, T c1, T c2, cudaStream_t st);
template <class T>
void launch3_jac_g(const S3<T> &vr, const D3<T> &r, const D3<T> &v, int M, T c, cudaStream_t st);
template <class T>
void launch3_asc_fine(const S3<T> &vr, const D3<T> &u, const D3<const T> &f, const D3<T> &scratch, const D3<T> &un,
                      int M, int order, T c, const Coef<T> &k, cudaStream_t st);
// z ranges [zlo, zhi) of global planes (multi-GPU z-slabs); zhi = -1: all.
template <class T>
void launch3_residual(const D3<const T> &u, const D3<const T> &f, const D3<T> &r, int M, int order, const Coef<T> &k,
                      cudaStream_t st, int zlo = 0, int zhi = -1);
template <class T>
void launch3_ftilde(const D3<const T> &f, const D3<T> &ft, int M, cudaStream_t st, int zlo = 0, int zhi = -1);
// TMA plane-streaming kernels (k3f.cu); 16-byte aligned pointers and pitches.
// ZRange3: the fine planes a launch writes and the local allocations of its
// inputs (multi-GPU slabs); the default is the whole grid.
struct ZRange3 {
  int zlo = 0, zhi = -1;      // output fine planes [zlo, zhi) (-1: all)
  int fz0 = 0, fplanes = -1;  // fine inputs (u, f): global plane of local plane 0, local planes (-1: all)
  int hz0 = 0, hplanes = -1;  // half-resolution sublattice inputs (v_R(1))
};
template <class T>
cudaError_t fast3_desc_fine(const T *u, const T *f, int64_t pitch, const S3<T> &rr, int M, int order, const Coef<T> &k,
                            const NormSink &ns, cudaStream_t st, const ZRange3 &pz = ZRange3());
template <class T>
cudaError_t fast3_asc_fine(const S3<T> &vr, const T *u_old, const T *f, int64_t pitch, T *u_new, int M, int order, T c,
                           const Coef<T> &k, cudaStream_t st, const ZRange3 &pz = ZRange3());

// Second-generation register-streaming plane pipelines (k3p.cu), orders 2 and
// 4 (Efos4 reads the u boxes of three planes); fast3_desc_fine /
// fast3_asc_fine dispatch to them unless MG_K3_GEN1=1.
template <class T>
cudaError_t fast3p_desc_fine(const T *u, const T *f, int64_t pitch, const S3<T> &rr, int M, int order,
                             const Coef<T> &k, const NormSink &ns, cudaStream_t st, const ZRange3 &pz);
template <class T>
cudaError_t fast3p_asc_fine(const S3<T> &vr, const T *u_old, const T *f, int64_t pitch, T *u_new, int M, int order,
                            T c, const Coef<T> &k, cudaStream_t st, const ZRange3 &pz);

// The same pipelines one octave down (s > 1, single GPU): G(s) -> R(s)
// (Erred from the dense r_G(s)) and G(s) from R(s) (Egprolg + Egprolr, both
// colours in one pass).
template <class T>
cudaError_t fast3p_rest_gr(const D3<T> &r, const S3<T> &rr, int M, cudaStream_t st);
template <class T>
cudaError_t fast3p_jac_g(const S3<T> &vr, const D3<T> &r, const D3<T> &v, int M, T c, cudaStream_t st);

// Sublattice level passes as plane pipelines (k3s.cu, fp64 and fp32, single
// GPU): R(s) -> M(s), M(s) -> G(2s), G(2s) -> M(s) and M(s) -> R(s) (both
// colours of each Jacobi level in one pass).
template <class T>
cudaError_t fast3s_rest_rm(const S3<T> &rr, const S3<T> &rm, int M, cudaStream_t st);
template <class T>
cudaError_t fast3s_rest_mg(const S3<T> &rm, const D3<T> &g2, int Mc, cudaStream_t st);
template <class T>
cudaError_t fast3s_jac_m(const D3<T> &vc, const S3<T> &r, const S3<T> &v, int M, T cc, cudaStream_t st);
template <class T>
cudaError_t fast3s_jac_r(const S3<T> &vm, const S3<T> &r, const S3<T> &v, int M, T c1, T c2, cudaStream_t st);
// R(s) -> M(s) -> G(2s) in one pass (r_M written, not re-read): rest_rm and rest_mg fused (fp64).
cudaError_t fast3s_rest_rmg(const S3<double> &rr, const S3<double> &rm, const D3<double> &g2, int M, cudaStream_t st);
// G(2s) -> M(s) -> R(s) in one pass (v_M(s) stays on chip): jac_m and jac_r fused.
cudaError_t fast3s_jac_mr(const D3<double> &vc, const S3<double> &rm, const S3<double> &rr, const S3<double> &v, int M,
                          double cm, double c1, double c2, cudaStream_t st);

// Per-octave level descriptors for the 3D single-CTA coarse kernel.
template <class T>
struct Lev3 {
  S3<T> rR, vR, rM, vM;   // R(s), M(s)
  D3<T> rG, vG;           // G(s)
  int M;
  T cMg, cR1, cR2, cG;
};
template <class T>
void lv3_coarse(const Lev3<T> *d_lev, int oc, int k, int *counter, cudaStream_t st);
// Octaves om .. oc-1 grid-wide and oc .. k-1 in one CTA's shared memory, one
// cooperative launch (h_lev: host copy of the descriptors).  false: not launched.
template <class T>
bool lv3_tail(const Lev3<T> *h_lev, int om, int oc, int k, int *counter, cudaStream_t st);

// Sublattice level kernels (k3l.cu).  [c0, c1): the half-index planes
// (2x2x2 blocks; for rest_mg the G(2s) planes) a launch writes; c1 = -1: all.
// jac_m, jac_r, jac_g run two kernels (the paper's two colours); phase 1 or 2
// launches only that one (multi-GPU: a halo exchange goes in between), 0 both.
template <class T>
void lv3_rest_gr(const D3<T> &r, const S3<T> &rr, int M, cudaStream_t st, int c0 = 0, int c1 = -1);
template <class T>
void lv3_rest_rm(const S3<T> &rr, const S3<T> &rm, int M, cudaStream_t st, int c0 = 0, int c1 = -1);
template <class T>
void lv3_rest_mg(const S3<T> &rm, const D3<T> &g2, int Mc, cudaStream_t st, int c0 = 0, int c1 = -1);
template <class T>
void lv3_jac_m(const D3<T> &vc, const S3<T> &r, const S3<T> &v, int M, T c, cudaStream_t st, int c0 = 0, int c1 = -1,
               int phase = 0);
template <class T>
void lv3_jac_r(const S3<T> &vm, const S3<T> &r, const S3<T> &v, int M, T c1, T c2, cudaStream_t st, int cz0 = 0,
               int cz1 = -1, int phase = 0);
template <class T>
void lv3_jac_g(const S3<T> &vr, const D3<T> &r, const D3<T> &v, int M, T c, cudaStream_t st, int c0 = 0, int c1 = -1,
               int phase = 0);
template <class T>
void lv3_asc_fine(const S3<T> &vr, const D3<T> &u_old, const D3<const T> &f, const D3<T> &g, const D3<T> &u_new, int M,
                  int order, T c, const Coef<T> &k, cudaStream_t st);
template <class T>
void launch3_norm(const D3<const T> &a, int M, unsigned long long *mx, double *ss, cudaStream_t st, int zlo = 0,
                  int zhi = -1);

}  // namespace mg
