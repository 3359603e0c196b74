// mg_api.cu -- the C ABI of include/mg.h: argument checking, the level plan
// (buffers in HBM), the per-cycle launch schedule captured in a CUDA graph,
// norms, staging.  Host code only; the kernels live in k2d.cu / k3d.cu.
#include "comm.h"
#include "solver.h"

ImplBase *make_dist2(mg_solver *s, bool loopback, std::string *err);
ImplBase *make_dist3(mg_solver *s, bool loopback, std::string *err);

// ------------------------------------------------------------------ 2D
template <class T>
struct Impl2 : ImplBase {
  const mg_solver *s;
  int k;
  int64_t n, pitch;   // pitch: the work layout of u, f~ in the cycle (mg_solver::wpitch)
  int64_t cpitch;     // the caller's layout (mg_residual / mg_norm operands)
  // per octave o: D level (o = 0..k-2), A level (o = 1..k-1)
  std::vector<S2<T>> rD, vD;
  std::vector<D2<T>> rA, vA;
  std::vector<int> M;   // lattice extent per octave
  D2<T> scratch{};
  Coef<T> coef{};
  std::vector<T> cD, cA;   // Jacobi coefficients per octave
  bool use_fast = false;   // TMA tile kernels for the large levels
  int oc = 1;              // first octave handled by the single-CTA coarse kernel
  int om = 1;              // first octave of the cooperative tail kernel (om <= oc)
  bool use_tail = false;
  bool serp = !env_flag("MG_2D_NOSERP");   // serpentine tile order across passes
  int sweeps = 1;          // two-colour steps per level (> 1: NEXT-4, plain kernels)
  D2<T> tmpA{};            // sweeps > 1: E nodes of v_D(s) as a dense A(2s)-shaped array
  S2<T> tmpD{};            //             D nodes of v_A(s) as split E/O arrays
  bool xfuse = !env_flag("MG_2D_NOXFUSE");   // cross-cycle fusion of the finest ascent and descent
  // ... which also runs the next descent's octave pair D(1) -> A(2) -> D(2) (r_D(1) not re-read): opt-in
  // (MG_2D_XRD=1), measured slower on B200 at 8193^2: fp64 0.7575 vs 0.7453 ms, fp32 0.480 vs 0.452
  bool xrd = env_flag("MG_2D_XRD");
  bool adfuse = !env_flag("MG_2D_NOADFUSE");  // jac_a(s) fused with jac_d(s-1): v_A(s) stays on chip
  // ... for octaves s >= ad_min (MG_AD_MINO, default 1): 16-row tiles, two 90 KB CTAs of 512 threads per SM
  bool dafuse = !env_flag("MG_2D_NODAFUSE");  // rest_da(s) fused with rest_ad(s+1): r_A(s+1) not re-read
  // ... for octaves s >= da_min (MG_DA_MINO, default 0); measured on B200 at 8193^2 fp64 s = 0: 0.089 vs
  // 0.066 + 0.033 ms; fp32 (256-thread CTAs) 0.052 vs 0.034 + 0.021 ms
  int da_min = getenv("MG_DA_MINO") ? atoi(getenv("MG_DA_MINO")) : 0;
  int ad_min = getenv("MG_AD_MINO") && atoi(getenv("MG_AD_MINO")) >= 1 ? atoi(getenv("MG_AD_MINO")) : 1;
  Lev2<T> *d_lev = nullptr;
  std::vector<Lev2<T>> h_lev;   // host copy of the level descriptors (tail kernel parameters)
  explicit Impl2(const mg_solver *sv) : s(sv), k(sv->k), n(sv->cfg.n), pitch(sv->wpitch), cpitch(sv->pitch) {}
  bool fast() const override { return use_fast; }

  int64_t pitch_for(int64_t cnt) const { return round_up(cnt, 128 / (int64_t)sizeof(T)); }

  cudaError_t alloc() override {
    const double p = s->cfg.p[0];
    M.resize(k);
    rD.resize(k - 1);
    vD.resize(k - 1);
    rA.resize(k);
    vA.resize(k);
    cD.resize(k);
    cA.resize(k);
    for (int o = 0; o < k; o++) {
      M[o] = (int)((n - 1) >> o);
      double hs = std::ldexp(1.0, o) / (double)(n - 1);
      cD[o] = (T)(2.0 * p * hs * hs);
      cA[o] = (T)(p * hs * hs);
    }
    for (int o = 0; o + 1 < k; o++) {
      int64_t H = M[o] / 2 + 1, ph = pitch_for(H);
      for (auto *lv : {&rD, &vD}) {
        void *e, *oo;
        cudaError_t st = dalloc2d(&e, sizeof(T), H, ph, H);
        if (st) return st;
        st = dalloc2d(&oo, sizeof(T), H, ph, H);
        if (st) return st;
        (*lv)[o] = S2<T>{(T *)e, (T *)oo, ph};
      }
    }
    for (int o = 1; o < k; o++) {
      int64_t W = M[o] + 1, pa = pitch_for(W);
      for (auto *lv : {&rA, &vA}) {
        void *q;
        cudaError_t st = dalloc2d(&q, sizeof(T), W, pa, W);
        if (st) return st;
        (*lv)[o] = D2<T>{(T *)q, pa};
      }
    }
    coef.invh2 = (T)((double)(n - 1) * (double)(n - 1));
    coef.c6 = (T)((double)(n - 1) * (double)(n - 1) / 6.0);
    // TMA needs 16-byte row strides on the caller's arrays (and on ours)
    sweeps = s->cfg.sweeps > 1 ? s->cfg.sweeps : 1;
    use_fast = ((pitch * (int64_t)sizeof(T)) % 16 == 0) && !env_flag("MG_FORCE_REF") && sweeps == 1;
    if (sweeps > 1) {
      const int64_t H = M[0] / 2 + 1, ph = pitch_for(H);
      void *a, *e, *o;
      cudaError_t st = dalloc(&a, sizeof(T) * H * ph);
      if (!st) st = dalloc(&e, sizeof(T) * H * ph);
      if (!st) st = dalloc(&o, sizeof(T) * H * ph);
      if (st) return st;
      tmpA = D2<T>{(T *)a, ph};
      tmpD = S2<T>{(T *)e, (T *)o, ph};
    }
    if (!use_fast) {
      int64_t ps = pitch_for(n);
      void *q;
      cudaError_t st = dalloc(&q, sizeof(T) * n * ps);
      if (st) return st;
      scratch = D2<T>{(T *)q, ps};
    }
    int thresh = 64;
    if (const char *e = getenv("MG_COARSE_M")) thresh = atoi(e);
    oc = k - 1;
    for (int o = 1; o < k; o++)
      if (M[o] <= thresh) {
        oc = o;
        break;
      }
    std::vector<Lev2<T>> lv(k);
    for (int o = 0; o < k; o++) {
      lv[o].M = M[o];
      lv[o].cD = cD[o];
      lv[o].cA = cA[o];
      if (o + 1 < k) {
        lv[o].rD = rD[o];
        lv[o].vD = vD[o];
      }
      if (o >= 1) {
        lv[o].rA = rA[o];
        lv[o].vA = vA[o];
      }
    }
    void *q;
    cudaError_t st = dalloc(&q, sizeof(Lev2<T>) * k);
    if (st) return st;
    d_lev = (Lev2<T> *)q;
    h_lev = lv;
    // cooperative tail: octaves with M <= MG_TAIL_M2 in one launch; off by
    // default in 2D (measured on B200: no gain over the per-level kernels)
    int tm = 0;
    if (const char *e = getenv("MG_TAIL_M2")) tm = atoi(e);
    om = oc;
    for (int o = 1; o < oc; o++)
      if (M[o] <= tm) {
        om = o;
        break;
      }
    use_tail = use_fast && tm > 0 && k <= 40;
    return cudaMemcpy(d_lev, lv.data(), sizeof(Lev2<T>) * k, cudaMemcpyHostToDevice);
  }

  NormSink sink() const {
    return NormSink{hist_on(s) ? s->d_hist : nullptr, s->d_counter, kHistCap, s->sum_l2 ? s->d_l2 : nullptr};
  }

  bool fuses_cycles() const override { return use_fast && xfuse; }
  // the fused pass also ran rest_dad(0) (decided once per solver: producer and consumer cycles agree)
  bool xrd_on() const { return fuses_cycles() && xrd && dafuse && da_min == 0 && 1 < (use_tail ? om : oc) && M[0] % 4 == 0; }
  void enqueue_cycle_mode(const void *u_in, void *u_out, const void *f_eff, cudaStream_t st, Prof *prof,
                          int mode) override {
    if (use_fast) return enqueue_fast(u_in, u_out, f_eff, st, prof, mode);
    enqueue_cycle(u_in, u_out, f_eff, st, prof);
  }
  void enqueue_cycle(const void *u_in, void *u_out, const void *f_eff, cudaStream_t st, Prof *prof) override {
    if (use_fast) return enqueue_fast(u_in, u_out, f_eff, st, prof);
    D2<const T> uc{(const T *)u_in, pitch}, fc{(const T *)f_eff, pitch};
    D2<T> uu{(T *)u_in, pitch}, uo{(T *)u_out, pitch};
    const double w = sizeof(T);
    const int L = 2 * k - 1;
    STEP("desc_fine", 0, 1, w * (2 * Nl[0] + Nl[1]));
    launch2_desc_fine<T>(uc, fc, rD[0], M[0], s->cfg.order, coef, sink(), st);
    for (int o = 0; o + 1 < k; o++) {
      if (o >= 1) {
        STEP("rest_ad", 2 * o, 1, w * (Nl[2 * o] + Nl[2 * o + 1]));
        launch2_rest_ad<T>(rA[o], rD[o], M[o], st);
      }
      STEP("rest_da", 2 * o + 1, 1, w * (Nl[2 * o + 1] + Nl[2 * o + 2]));
      launch2_rest_da<T>(rD[o], rA[o + 1], M[o + 1], st);
    }
    STEP("coarsest", L - 1, 1, w * 2);
    launch2_coarsest<T>(rA[k - 1], vA[k - 1], cA[k - 1], s->d_counter, st);
    for (int o = k - 2; o >= 0; o--) {
      STEP("jac_d", 2 * o + 1, 2, w * (Nl[2 * o + 2] + 2 * Nl[2 * o + 1]));
      launch2_jac_d<T>(vA[o + 1], rD[o], vD[o], M[o], cD[o], st);
      for (int sw = 1; sw < sweeps; sw++) {   // again, from the E nodes of v_D itself (reading A19)
        const int64_t H = M[o] / 2 + 1;
        cudaMemcpy2DAsync(tmpA.p, tmpA.pitch * sizeof(T), vD[o].e, vD[o].pitch * sizeof(T), H * sizeof(T), H,
                          cudaMemcpyDeviceToDevice, st);
        launch2_jac_d<T>(tmpA, rD[o], vD[o], M[o], cD[o], st);
      }
      if (o >= 1) {
        STEP("jac_a", 2 * o, 2, w * (Nl[2 * o + 1] + 2 * Nl[2 * o]));
        launch2_jac_a<T>(vD[o], rA[o], vA[o], M[o], cA[o], st);
        for (int sw = 1; sw < sweeps; sw++) {   // again, from the D nodes of v_A itself
          const S2<T> td{tmpD.e, tmpD.o, tmpD.pitch};
          launch2_gather_d<T>(vA[o], td, M[o], st);
          launch2_jac_a<T>(td, rA[o], vA[o], M[o], cA[o], st);
        }
      } else if (sweeps > 1) {
        STEP("asc_fine", 0, 3 * sweeps, w * (Nl[1] + 3 * Nl[0]));
        launch2_asc_fine_sweeps<T>(vD[0], uu, fc, scratch, uo, M[0], s->cfg.order, cA[0], coef, sweeps, tmpD, st);
      } else {
        STEP("asc_fine", 0, 3, w * (Nl[1] + 3 * Nl[0]));
        launch2_asc_fine<T>(vD[0], uu, fc, scratch, uo, M[0], s->cfg.order, cA[0], coef, st);
      }
    }
  }

  // The B200 path: TMA tile kernels on octaves < oc, one CTA below.
  void enqueue_fast(const void *u_in, void *u_out, const void *f_eff, cudaStream_t st, Prof *prof, int mode = 0) {
    const double w = sizeof(T);
    const int L = 2 * k - 1;
    const T *uin = (const T *)u_in, *fe = (const T *)f_eff;
    // Serpentine tile order: each pass starts where its producer finished,
    // so the last ~100 MB the producer wrote are still in L2.
    // The finest descent runs forwards; the fused ascent+descent backwards,
    // and the restrictions follow whichever produced r_D(1).
    Rows2 fwd, bwd;
    bwd.rev = serp;
    const bool skip = mode & kSkipDesc;
    Rows2 dA = skip ? bwd : fwd, dD = skip ? fwd : bwd;   // rest_ad, rest_da
    if (!skip) {
      STEP("desc_fine", 0, 1, w * (2 * Nl[0] + Nl[1]));
      fast2_desc_fine<T>(uin, fe, pitch, rD[0], M[0], s->cfg.order, coef, sink(), st, fwd);
    }
    const int od = use_tail ? om : oc;   // first octave not run by per-level kernels
    bool a_done = false;                 // rest_ad(o) already ran inside the fused pass of octave o - 1
    auto descent = [&](int o) {
      if (o >= 1 && !a_done) {
        STEP("rest_ad", 2 * o, 1, w * (Nl[2 * o] + Nl[2 * o + 1]));
        fast2_rest_ad<T>(rA[o], rD[o], M[o], st, dA);
      }
      a_done = false;
      if (dafuse && o >= da_min && o + 1 < od) {
        STEP("rest_dad", 2 * o + 1, 1, w * (Nl[2 * o + 1] + Nl[2 * o + 2] + Nl[2 * o + 3]));
        // serpentine: consecutive octave-pair passes walk in opposite directions
        fast2_rest_dad<T>(rD[o], rA[o + 1], rD[o + 1], M[o + 1], st, dD.rev ^ (serp && (o & 1)));
        a_done = true;
        return;
      }
      STEP("rest_da", 2 * o + 1, 1, w * (Nl[2 * o + 1] + Nl[2 * o + 2]));
      fast2_rest_da<T>(rD[o], rA[o + 1], M[o + 1], st, dD);
    };
    bool d_done = false;   // jac_d(o) already ran inside the fused pass of octave o + 1
    auto ascent = [&](int o) {
      if (!d_done) {
        STEP("jac_d", 2 * o + 1, 1, w * (Nl[2 * o + 2] + 2 * Nl[2 * o + 1]));
        fast2_jac_d<T>(vA[o + 1], rD[o], vD[o], M[o], cD[o], st, fwd);
      }
      d_done = false;
      if (o >= 1 && adfuse && o >= ad_min) {
        STEP("jac_ad", 2 * o, 1, w * (Nl[2 * o + 1] + Nl[2 * o] + 2 * Nl[2 * o - 1]));
        fast2_jac_ad<T>(vD[o], rA[o], cA[o], rD[o - 1], vD[o - 1], M[o - 1], cD[o - 1], st,
                        serp && !((o - 1) & 1));   // alternating, backwards at s = 1
        d_done = true;
      } else if (o >= 1) {
        STEP("jac_a", 2 * o, 1, w * (Nl[2 * o + 1] + 2 * Nl[2 * o]));
        fast2_jac_a<T>(vD[o], rA[o], vA[o], M[o], cA[o], st, bwd);
      } else if (mode & kFuseNext) {
        if (xrd_on()) {
          STEP("asc_desc", 0, 1, w * (2 * Nl[1] + 3 * Nl[0] + Nl[2] + Nl[3]));
          fast2_asc_desc<T>(vD[0], uin, fe, pitch, (T *)u_out, rD[0], M[0], s->cfg.order, cA[0], coef, sink(), st,
                            serp, &rA[1], &rD[1]);
        } else {
          STEP("asc_desc", 0, 1, w * (2 * Nl[1] + 3 * Nl[0]));
          fast2_asc_desc<T>(vD[0], uin, fe, pitch, (T *)u_out, rD[0], M[0], s->cfg.order, cA[0], coef, sink(), st,
                            serp);
        }
      } else {
        STEP("asc_fine", 0, 1, w * (Nl[1] + 3 * Nl[0]));
        fast2_asc_fine<T>(vD[0], uin, fe, pitch, (T *)u_out, M[0], s->cfg.order, cA[0], coef, st, bwd);
      }
    };
    for (int o = 0; o < od; o++) {
      if (o == 0 && skip && xrd_on()) {   // the previous cycle's fused pass ran rest_dad(0)
        a_done = true;
        continue;
      }
      descent(o);
    }
    bool tail_done = false;
    if (use_tail) {
      double b = 0;
      for (int l = 2 * om; l < L; l++) b += 5 * Nl[l];
      b -= Nl[L - 1] + 2 * Nl[2 * om];
      STEP("tail", 2 * om, 1, w * b);
      tail_done = launch2_tail<T>(h_lev.data(), om, oc, k, s->d_counter, st);
      if (!tail_done) {
        static bool warned = false;
        if (!warned) fprintf(stderr, "[mg] cooperative tail kernel not launched; per-level kernels instead\n");
        warned = true;
      }
    }
    if (!tail_done) {
      for (int o = od; o < oc; o++) descent(o);
      double b = 0;
      for (int l = 2 * oc; l < L; l++) b += 5 * Nl[l];
      b -= Nl[L - 1] + 2 * Nl[2 * oc];   // coarsest: 4 touches; r_A(oc): read twice, written outside
      STEP("coarse", 2 * oc, 1, w * b);
      launch2_coarse<T>(d_lev, oc, k, s->d_counter, st, h_lev.data());
      for (int o = oc - 1; o >= od; o--) ascent(o);
    }
    for (int o = od - 1; o >= 0; o--) ascent(o);
  }
  void enqueue_pre_descent(void *u, const void *f_eff, cudaStream_t st) override {
    enqueue_final_norm(u, f_eff, st);
    if (xrd_on()) fast2_rest_dad<T>(rD[0], rA[1], rD[1], M[1], st, false);
  }
  void enqueue_final_norm(void *u, const void *f_eff, cudaStream_t st) override {
    if (use_fast) {
      fast2_desc_fine<T>((const T *)u, (const T *)f_eff, pitch, rD[0], M[0], s->cfg.order, coef, sink(), st);
      return;
    }
    D2<const T> uc{(const T *)u, pitch}, fc{(const T *)f_eff, pitch};
    launch2_desc_fine<T>(uc, fc, rD[0], M[0], s->cfg.order, coef, sink(), st);
  }
  void enqueue_residual(const void *u, const void *f, void *r, cudaStream_t st, int64_t fp) override {
    launch2_residual<T>(D2<const T>{(const T *)u, cpitch}, D2<const T>{(const T *)f, fp}, D2<T>{(T *)r, cpitch},
                        M[0], s->cfg.order, coef, st);
  }
  void enqueue_ftilde(const void *f, void *ft, cudaStream_t st, int64_t ftp) override {
    launch2_ftilde<T>(D2<const T>{(const T *)f, cpitch}, D2<T>{(T *)ft, ftp}, M[0], st);
  }
  void enqueue_norm(const void *x, unsigned long long *mx, double *ss, cudaStream_t st, int64_t xp) override {
    launch2_norm<T>(D2<const T>{(const T *)x, xp}, M[0], mx, ss, st);
  }
  int launches_per_cycle() const override {
    if (use_fast) {
      const int od = use_tail ? om : oc;
      // desc_fine, rest_ad (o >= 1) + rest_da per descent octave, tail or coarse, jac_d + jac_a/asc per ascent
      // octave; with cross-cycle fusion a steady-state cycle has no desc_fine (the previous cycle's asc_desc ran it)
      // jac_a(o) and jac_d(o - 1) share one pass for o >= 1
      return 1 + (od - 1) + od + 1 + 2 * od + (use_tail ? 0 : 3 * (oc - od)) - (fuses_cycles() ? 1 : 0) -
             (adfuse && od > ad_min ? od - ad_min : 0) -
             (dafuse && od - 1 > da_min ? od - 1 - da_min : 0) - (xrd_on() ? 1 : 0);
    }
    int c = 1;                               // desc fine
    for (int o = 0; o + 1 < k; o++) c += (o >= 1) + 1;
    c += 1;                                  // coarsest
    for (int o = k - 2; o >= 0; o--) c += 2 + ((o >= 1) ? 2 : 3);
    return c;
  }
};

// ------------------------------------------------------------------ 3D
// sublattice pipelines (k3s.cu, fp64 and fp32); the fused octave passes are
// fp64 only (their fp32 overloads are never reached: fuse_rmg / fuse_mr need fp64).
template <class T>
static void sub3_rest_rm(const S3<T> &rr, const S3<T> &rm, int M, cudaStream_t st) {
  fast3s_rest_rm<T>(rr, rm, M, st);
}
template <class T>
static void sub3_rest_mg(const S3<T> &rm, const D3<T> &g2, int Mc, cudaStream_t st) {
  fast3s_rest_mg<T>(rm, g2, Mc, st);
}
template <class T>
static void sub3_jac_m(const D3<T> &vc, const S3<T> &r, const S3<T> &v, int M, T c, cudaStream_t st) {
  fast3s_jac_m<T>(vc, r, v, M, c, st);
}
template <class T>
static void sub3_jac_r(const S3<T> &vm, const S3<T> &r, const S3<T> &v, int M, T c1, T c2, cudaStream_t st) {
  fast3s_jac_r<T>(vm, r, v, M, c1, c2, st);
}
static void sub3_jac_mr(const D3<double> &vc, const S3<double> &rm, const S3<double> &rr, const S3<double> &v, int M,
                        double cm, double c1, double c2, cudaStream_t st) {
  fast3s_jac_mr(vc, rm, rr, v, M, cm, c1, c2, st);
}
static void sub3_jac_mr(const D3<float> &, const S3<float> &, const S3<float> &, const S3<float> &, int, float, float,
                        float, cudaStream_t) {}
static void sub3_rest_rmg(const S3<double> &rr, const S3<double> &rm, const D3<double> &g2, int M, cudaStream_t st) {
  fast3s_rest_rmg(rr, rm, g2, M, st);
}
static void sub3_rest_rmg(const S3<float> &, const S3<float> &, const D3<float> &, int, cudaStream_t) {}

// First octave of the fused fp64 octave passes (k3s.cu): G(2s) -> M(s) -> R(s)
// (jac_mr) and R(s) -> M(s) -> G(2s) (rest_rmg); 1000 = never.  MG_K3_FUSE=1
// fuses both everywhere they exist (jac_mr from octave 1, rest_rmg from 0);
// MG_K3_FUSE_MR / MG_K3_FUSE_RMG = o set the first octave of each.
static int k3_fuse_min(bool mr) {
  const char *e = getenv(mr ? "MG_K3_FUSE_MR" : "MG_K3_FUSE_RMG");
  if (e && *e) return atoi(e) < 0 ? 1000 : (mr ? std::max(1, atoi(e)) : atoi(e));
  return env_flag("MG_K3_FUSE") ? (mr ? 1 : 0) : 1000;
}
// Octaves with M(o) <= this run their level steps on the one-thread-per-node k3l.cu kernels instead of
// the plane pipelines (MG_K3_GEN1_M; 0 = never): small levels sit in L2, where a pipeline's prologue and
// epilogue per z-split work item cost more than the massively parallel kernels' extra launches.
static int k3_gen1_m() {
  static const int m = [] {
    const char *e = getenv("MG_K3_GEN1_M");
    return e && *e ? atoi(e) : 128;
  }();
  return m;
}
// The same for the descent's restriction steps alone (MG_K3_GEN1_MD; default: MG_K3_GEN1_M).
static int k3_gen1_md() {
  static const int m = [] {
    const char *e = getenv("MG_K3_GEN1_MD");
    return e && *e ? atoi(e) : k3_gen1_m();
  }();
  return m;
}

template <class T>
struct Impl3 : ImplBase {
  const mg_solver *s;
  int k;
  int64_t n, pitch;   // the work layout (mg_solver::wpitch)
  int64_t cpitch;     // the caller's layout (mg_residual / mg_norm operands)
  std::vector<S3<T>> rR, vR, rM, vM;   // octave 0..k-2
  std::vector<D3<T>> rG, vG;           // octave 1..k-1
  std::vector<int> M;
  D3<T> scratch{};
  Coef<T> coef{};
  std::vector<T> cMg, cR1, cR2, cG;
  bool use_fast = false;   // TMA plane kernels for the finest octave
  int oc = 1;              // first octave run by the single-CTA coarse kernel
  int om = 1;              // first octave of the cooperative tail kernel (om <= oc)
  bool use_tail = false;
  Lev3<T> *d_lev = nullptr;
  std::vector<Lev3<T>> h_lev;   // host copy of the level descriptors (tail kernel parameters)
  explicit Impl3(const mg_solver *sv) : s(sv), k(sv->k), n(sv->cfg.n), pitch(sv->wpitch), cpitch(sv->pitch) {}
  bool fast() const override { return use_fast; }
  int64_t pitch_for(int64_t cnt) const { return round_up(cnt, 128 / (int64_t)sizeof(T)); }

  cudaError_t split(S3<T> &out, int64_t H, std::initializer_list<int> parities) {
    int64_t ph = pitch_for(H);
    out = S3<T>{};
    out.pitch = ph;
    out.plane = ph * H;
    for (int par : parities) {
      void *q;
      cudaError_t st = dalloc2d(&q, sizeof(T), H, ph, H * H);
      if (st) return st;
      out.s[par] = (T *)q;
    }
    return cudaSuccess;
  }

  cudaError_t alloc() override {
    const double pm = s->cfg.p[0], pr1 = s->cfg.p[1], pr2 = s->cfg.p[2], pg = s->cfg.p[3];
    M.resize(k);
    rR.resize(k - 1);
    vR.resize(k - 1);
    rM.resize(k - 1);
    vM.resize(k - 1);
    rG.resize(k);
    vG.resize(k);
    cMg.resize(k);
    cR1.resize(k);
    cR2.resize(k);
    cG.resize(k);
    for (int o = 0; o < k; o++) {
      M[o] = (int)((n - 1) >> o);
      double hs = std::ldexp(1.0, o) / (double)(n - 1);
      double h2 = hs * hs;
      cMg[o] = (T)(4.0 * pm * h2);
      cR1[o] = (T)(2.0 * pr1 * h2);
      cR2[o] = (T)(4.0 * pr2 * h2);
      cG[o] = (T)(pg * h2);
    }
    // parity index = (x&1) | (y&1)<<1 | (z&1)<<2 ; C=0, Fx=(0,1,1)=6, Fy=(1,0,1)=5, Fz=(1,1,0)=3, B=7
    for (int o = 0; o + 1 < k; o++) {
      int64_t H = M[o] / 2 + 1;
      cudaError_t st;
      if ((st = split(rR[o], H, {0, 6, 5, 3}))) return st;
      if ((st = split(vR[o], H, {0, 6, 5, 3}))) return st;
      if ((st = split(rM[o], H, {0, 7}))) return st;
      if ((st = split(vM[o], H, {0, 7}))) return st;
    }
    for (int o = 1; o < k; o++) {
      int64_t W = M[o] + 1, pa = pitch_for(W);
      for (auto *lv : {&rG, &vG}) {
        void *q;
        cudaError_t st = dalloc2d(&q, sizeof(T), W, pa, W * W);
        if (st) return st;
        (*lv)[o] = D3<T>{(T *)q, pa, pa * W};
      }
    }
    {
      int64_t ps = pitch_for(n);
      void *q;
      cudaError_t st = dalloc(&q, sizeof(T) * n * n * ps);
      if (st) return st;
      scratch = D3<T>{(T *)q, ps, ps * n};
    }
    coef.invh2 = (T)((double)(n - 1) * (double)(n - 1));
    coef.c6 = (T)((double)(n - 1) * (double)(n - 1) / 6.0);
    use_fast = ((pitch * (int64_t)sizeof(T)) % 16 == 0) && !env_flag("MG_FORCE_REF");
    int thresh = 16;
    if (const char *e = getenv("MG_COARSE_M3")) thresh = atoi(e);
    oc = k - 1;
    for (int o = 1; o < k; o++)
      if (M[o] <= thresh) {
        oc = o;
        break;
      }
    std::vector<Lev3<T>> lv(k);
    for (int o = 0; o < k; o++) {
      lv[o].M = M[o];
      lv[o].cMg = cMg[o];
      lv[o].cR1 = cR1[o];
      lv[o].cR2 = cR2[o];
      lv[o].cG = cG[o];
      if (o + 1 < k) {
        lv[o].rR = rR[o];
        lv[o].vR = vR[o];
        lv[o].rM = rM[o];
        lv[o].vM = vM[o];
      }
      if (o >= 1) {
        lv[o].rG = rG[o];
        lv[o].vG = vG[o];
      }
    }
    void *q;
    cudaError_t st = dalloc(&q, sizeof(Lev3<T>) * k);
    if (st) return st;
    d_lev = (Lev3<T> *)q;
    h_lev = lv;
    // cooperative tail: octaves with M <= MG_TAIL_M3 (default 32; 64 until the M <= 128 octaves moved to the
    // k3l.cu level kernels, after which the M = 64 octave is cheaper there: 2.1174 vs 2.1258 ms at 513^3)
    int tm = 32;
    if (const char *e = getenv("MG_TAIL_M3")) tm = atoi(e);
    om = oc;
    for (int o = 1; o < oc; o++)
      if (M[o] <= tm) {
        om = o;
        break;
      }
    use_tail = use_fast && tm > 0 && k <= 20;
    return cudaMemcpy(d_lev, lv.data(), sizeof(Lev3<T>) * k, cudaMemcpyHostToDevice);
  }

  NormSink sink() const {
    return NormSink{hist_on(s) ? s->d_hist : nullptr, s->d_counter, kHistCap, s->sum_l2 ? s->d_l2 : nullptr};
  }
  void desc_fine(const void *u, const void *f_eff, cudaStream_t st) {
    if (use_fast && ((uintptr_t)u & 15) == 0 && ((uintptr_t)f_eff & 15) == 0)
      fast3_desc_fine<T>((const T *)u, (const T *)f_eff, pitch, rR[0], M[0], s->cfg.order, coef, sink(), st);
    else
      launch3_desc_fine<T>(cfield(u), cfield(f_eff), rR[0], M[0], s->cfg.order, coef, sink(), st);
  }
  D3<const T> cfield(const void *a) const { return D3<const T>{(const T *)a, pitch, pitch * n}; }
  D3<T> field(void *a) const { return D3<T>{(T *)a, pitch, pitch * n}; }

  void enqueue_cycle(const void *u_in, void *u_out, const void *f_eff, cudaStream_t st, Prof *prof) override {
    if (use_fast) return enqueue_fast(u_in, u_out, f_eff, st, prof);
    const double w = sizeof(T);
    const int L = 3 * k - 2;
    void *u = const_cast<void *>(u_in);
    STEP("desc_fine", 0, 1, w * (2 * Nl[0] + Nl[1]));
    desc_fine(u, f_eff, st);
    for (int o = 0; o + 1 < k; o++) {
      int g = 3 * o;
      if (o >= 1) {
        STEP("rest_gr", g, 1, w * (Nl[g] + Nl[g + 1]));
        if (use_fast) lv3_rest_gr<T>(rG[o], rR[o], M[o], st);
        else launch3_rest_gr<T>(rG[o], rR[o], M[o], st);
      }
      STEP("rest_rm", g + 1, 1, w * (Nl[g + 1] + Nl[g + 2]));
      if (use_fast) lv3_rest_rm<T>(rR[o], rM[o], M[o], st);
      else launch3_rest_rm<T>(rR[o], rM[o], M[o], st);
      STEP("rest_mg", g + 2, 1, w * (Nl[g + 2] + Nl[g + 3]));
      if (use_fast) lv3_rest_mg<T>(rM[o], rG[o + 1], M[o + 1], st);
      else launch3_rest_mg<T>(rM[o], rG[o + 1], M[o + 1], st);
    }
    STEP("coarsest", L - 1, 1, w * 2);
    launch3_coarsest<T>(rG[k - 1], vG[k - 1], cG[k - 1], s->d_counter, st);
    for (int o = k - 2; o >= 0; o--) {
      int g = 3 * o;
      STEP("jac_m", g + 2, 2, w * (Nl[g + 3] + 2 * Nl[g + 2]));
      if (use_fast) lv3_jac_m<T>(vG[o + 1], rM[o], vM[o], M[o], cMg[o], st);
      else launch3_jac_m<T>(vG[o + 1], rM[o], vM[o], M[o], cMg[o], st);
      STEP("jac_r", g + 1, 2, w * (Nl[g + 2] + 2 * Nl[g + 1]));
      if (use_fast) lv3_jac_r<T>(vM[o], rR[o], vR[o], M[o], cR1[o], cR2[o], st);
      else launch3_jac_r<T>(vM[o], rR[o], vR[o], M[o], cR1[o], cR2[o], st);
      if (o >= 1) {
        STEP("jac_g", g, 2, w * (Nl[g + 1] + 2 * Nl[g]));
        if (use_fast) lv3_jac_g<T>(vR[o], rG[o], vG[o], M[o], cG[o], st);
        else launch3_jac_g<T>(vR[o], rG[o], vG[o], M[o], cG[o], st);
      } else if (use_fast) {
        STEP("asc_fine", 0, 2, w * (Nl[1] + 3 * Nl[0]));
        lv3_asc_fine<T>(vR[0], field(u), cfield(f_eff), scratch, field(u_out), M[0], s->cfg.order, cG[0], coef, st);
      } else {
        STEP("asc_fine", 0, 3, w * (Nl[1] + 3 * Nl[0]));
        launch3_asc_fine<T>(vR[0], field(u), cfield(f_eff), scratch, field(u_out), M[0], s->cfg.order, cG[0], coef,
                            st);
      }
    }
  }
  // The B200 path: TMA plane kernel for the finest descent, sublattice
  // kernels for the octaves below oc, one CTA for the rest.
  void enqueue_fast(const void *u_in, void *u_out, const void *f_eff, cudaStream_t st, Prof *prof) {
    const double w = sizeof(T);
    const int L = 3 * k - 2;
    static const bool gen2 = !env_flag("MG_K3_GEN1");   // plane pipelines for the G(s) levels
    static const bool s32 = !env_flag("MG_K3S_NOF32");   // fp32 sublattice pipelines (round 2)
    const bool gen2s = gen2 && (sizeof(T) == 8 || s32);   // and for the sublattice levels
    void *u = const_cast<void *>(u_in);
    // fused octave passes: bit-identical, but no measurable gain in graph replay on B200 (A/B in
    // DESIGN.md), so opt-in (MG_K3_FUSE=1, or per octave MG_K3_FUSE_RMG / MG_K3_FUSE_MR)
    static const int rmg_min = k3_fuse_min(false);
    const int g1m = k3_gen1_m(), g1md = k3_gen1_md();
    auto pipe = [&](int o) { return gen2 && M[o] > g1m; };     // G(s) level steps on plane pipelines
    auto pipes = [&](int o) { return gen2s && M[o] > g1m; };   // sublattice steps on plane pipelines
    auto piped = [&](int o) { return gen2 && M[o] > g1md; };   // restriction steps (descent)
    auto pipeds = [&](int o) { return gen2s && M[o] > g1md; };
    // Serpentine item order (zpipe Sched::rev): descent pass d (desc_fine = 0,
    // then rest_rm, rest_mg, rest_gr, ...) runs reversed when d is odd; ascent
    // passes alternate backwards from asc_fine (reversed), so the next
    // cycle's desc_fine (forward) starts where asc_fine ended.
    static const bool serp = !env_flag("MG_3D_NOSERP");
    auto dir = [&](int pass) { zp_next_rev() = serp ? (pass & 1) : 0; };
    STEP("desc_fine", 0, 1, w * (2 * Nl[0] + Nl[1]));
    dir(0);
    desc_fine(u, f_eff, st);
    auto descent = [&](int o) {
      int g = 3 * o;
      if (o >= 1) {
        STEP("rest_gr", g, 1, w * (Nl[g] + Nl[g + 1]));
        dir(3 * o);
        if (piped(o)) fast3p_rest_gr<T>(rG[o], rR[o], M[o], st);
        else lv3_rest_gr<T>(rG[o], rR[o], M[o], st);
      }
      if (pipeds(o) && sizeof(T) == 8 && o >= rmg_min) {   // R(s) -> M(s) -> G(2s) in one pass (r_M written, not re-read)
        STEP("rest_rmg", g + 1, 1, w * (Nl[g + 1] + Nl[g + 2] + Nl[g + 3]));
        sub3_rest_rmg(rR[o], rM[o], rG[o + 1], M[o], st);
        return;
      }
      STEP("rest_rm", g + 1, 1, w * (Nl[g + 1] + Nl[g + 2]));
      dir(3 * o + 1);
      if (pipeds(o)) sub3_rest_rm(rR[o], rM[o], M[o], st);
      else lv3_rest_rm<T>(rR[o], rM[o], M[o], st);
      STEP("rest_mg", g + 2, 1, w * (Nl[g + 2] + Nl[g + 3]));
      dir(3 * o + 2);
      if (pipeds(o)) sub3_rest_mg(rM[o], rG[o + 1], M[o + 1], st);
      else lv3_rest_mg<T>(rM[o], rG[o + 1], M[o + 1], st);
    };
    // G(2s) -> M(s) -> R(s): one fused pass (v_M(s) stays on chip) or the two level kernels.
    // Measured on B200: the fused pass wins on the octaves o >= 1 (2 launches -> 1) but loses at
    // o = 0 (0.41 vs 0.39 ms: its 29 x 13 core tile recomputes 26 % ring and is issue-bound there).
    static const int mr_min = k3_fuse_min(true);
    auto jac_mr = [&](int o) {
      int g = 3 * o;
      if (pipes(o) && sizeof(T) == 8 && o >= mr_min) {
        STEP("jac_mr", g + 1, 1, w * (Nl[g + 3] + Nl[g + 2] + 2 * Nl[g + 1]));
        sub3_jac_mr(vG[o + 1], rM[o], rR[o], vR[o], M[o], cMg[o], cR1[o], cR2[o], st);
        return;
      }
      STEP("jac_m", g + 2, pipes(o) ? 1 : 2, w * (Nl[g + 3] + 2 * Nl[g + 2]));
      dir(3 * o + 3);
      if (pipes(o)) sub3_jac_m(vG[o + 1], rM[o], vM[o], M[o], cMg[o], st);
      else lv3_jac_m<T>(vG[o + 1], rM[o], vM[o], M[o], cMg[o], st);
      STEP("jac_r", g + 1, pipes(o) ? 1 : 2, w * (Nl[g + 2] + 2 * Nl[g + 1]));
      dir(3 * o + 2);
      if (pipes(o)) sub3_jac_r(vM[o], rR[o], vR[o], M[o], cR1[o], cR2[o], st);
      else lv3_jac_r<T>(vM[o], rR[o], vR[o], M[o], cR1[o], cR2[o], st);
    };
    auto ascent = [&](int o) {   // o >= 1
      int g = 3 * o;
      jac_mr(o);
      if (pipe(o)) {
        STEP("jac_g", g, 1, w * (Nl[g + 1] + 2 * Nl[g]));
        dir(3 * o + 1);
        fast3p_jac_g<T>(vR[o], rG[o], vG[o], M[o], cG[o], st);
      } else {
        STEP("jac_g", g, 2, w * (Nl[g + 1] + 2 * Nl[g]));
        lv3_jac_g<T>(vR[o], rG[o], vG[o], M[o], cG[o], st);
      }
    };
    const int od = use_tail ? om : oc;   // first octave not run by per-level kernels
    for (int o = 0; o < od; o++) descent(o);
    bool tail_done = false;
    if (use_tail) {
      double b = 0;
      for (int l = 3 * om; l < L; l++) b += 5 * Nl[l];
      b -= Nl[L - 1] + 2 * Nl[3 * om];
      STEP("tail", 3 * om, 1, w * b);
      tail_done = lv3_tail<T>(h_lev.data(), om, oc, k, s->d_counter, st);
      if (!tail_done) {
        static bool warned = false;
        if (!warned) fprintf(stderr, "[mg] cooperative tail kernel not launched; per-level kernels instead\n");
        warned = true;
      }
    }
    if (!tail_done) {
      for (int o = od; o < oc; o++) descent(o);
      double b = 0;
      for (int l = 3 * oc; l < L; l++) b += 5 * Nl[l];
      b -= Nl[L - 1] + 2 * Nl[3 * oc];
      STEP("coarse", 3 * oc, 1, w * b);
      lv3_coarse<T>(d_lev, oc, k, s->d_counter, st);
      for (int o = oc - 1; o >= od && o >= 1; o--) ascent(o);
    }
    for (int o = od - 1; o >= 0; o--) {
      if (o >= 1) {
        ascent(o);
        continue;
      }
      int g = 3 * o;
      jac_mr(o);
      if (!env_flag("MG_ASC3_DIRECT") && ((uintptr_t)u & 15) == 0 && ((uintptr_t)f_eff & 15) == 0 &&
                 ((uintptr_t)u_out & 15) == 0) {
        STEP("asc_fine", 0, 1, w * (Nl[1] + 3 * Nl[0]));
        dir(1);
        fast3_asc_fine<T>(vR[0], (const T *)u, (const T *)f_eff, pitch, (T *)u_out, M[0], s->cfg.order, cG[0], coef,
                          st);
      } else {
        STEP("asc_fine", 0, 2, w * (Nl[1] + 3 * Nl[0]));
        lv3_asc_fine<T>(vR[0], field(u), cfield(f_eff), scratch, field(u_out), M[0], s->cfg.order, cG[0], coef, st);
      }
    }
    zp_next_rev() = 0;
  }
  void enqueue_final_norm(void *u, const void *f_eff, cudaStream_t st) override { desc_fine(u, f_eff, st); }
  void enqueue_residual(const void *u, const void *f, void *r, cudaStream_t st, int64_t fp) override {
    launch3_residual<T>(D3<const T>{(const T *)u, cpitch, cpitch * n}, D3<const T>{(const T *)f, fp, fp * n},
                        D3<T>{(T *)r, cpitch, cpitch * n}, M[0], s->cfg.order, coef, st);
  }
  void enqueue_ftilde(const void *f, void *ft, cudaStream_t st, int64_t ftp) override {
    launch3_ftilde<T>(D3<const T>{(const T *)f, cpitch, cpitch * n}, D3<T>{(T *)ft, ftp, ftp * n}, M[0], st);
  }
  void enqueue_norm(const void *x, unsigned long long *mx, double *ss, cudaStream_t st, int64_t xp) override {
    launch3_norm<T>(D3<const T>{(const T *)x, xp, xp * n}, M[0], mx, ss, st);
  }
  int launches_per_cycle() const override {
    int c = 1;
    for (int o = 0; o + 1 < k; o++) c += (o >= 1) + 2;
    c += 1;
    if (use_fast) {
      c = 1;
      for (int o = 0; o < oc; o++) c += (o >= 1) + 2;
      c += 1;
      const bool gen2 = !env_flag("MG_K3_GEN1"), gen2s = gen2 && (sizeof(T) == 8 || !env_flag("MG_K3S_NOF32"));
      const bool f64 = gen2s && sizeof(T) == 8;
      const int mr_min = k3_fuse_min(true), rmg_min = k3_fuse_min(false);
      const int g1m = k3_gen1_m(), g1md = k3_gen1_md();
      auto p1 = [&](int o) { return gen2 && M[o] > g1m; };
      auto ps = [&](int o) { return gen2s && M[o] > g1m; };
      auto per_mr_o = [&](int o) { return ps(o) ? (f64 && o >= mr_min ? 1 : 2) : 4; };
      const int od = use_tail ? om : oc;
      c = 1;
      for (int o = 0; o < od; o++) c += (o >= 1) + (gen2s && M[o] > g1md && f64 && o >= rmg_min ? 1 : 2);
      c += 1;   // tail or coarse
      if (!use_tail)
        for (int o = oc - 1; o >= od; o--) c += per_mr_o(o) + (p1(o) ? 1 : 2);
      for (int o = od - 1; o >= 0; o--) c += per_mr_o(o) + (o >= 1 ? (p1(o) ? 1 : 2) : 1);
      return c;
    }
    for (int o = k - 2; o >= 0; o--) c += 2 + 2 + ((o >= 1) ? 2 : 3);
    return c;
  }
};

// ------------------------------------------------------------ helpers

static void drop_graphs(mg_solver *s) {
  for (auto &g : s->graphs) cudaGraphExecDestroy(g.exec);
  s->graphs.clear();
}

// Launch `count` V-cycles of one mode, the first u_in -> u_out, each further
// one reading the previous one's output (u alternates between the two arrays
// when they differ): replay the CUDA graph captured for these pointers
// (captured on first use; a few are cached).  Several cycles per graph: a
// graph launch waits for the previous graph to drain completely, ~4-6 us
// between the last pass of one cycle and the first of the next (CUPTI
// timeline), which inside one graph the passes do not pay.
static int run_cycles(mg_solver *s, const void *u_in, void *u_out, const void *f_eff, int mode, int count) {
  cudaGraphExec_t ex = nullptr;
  for (auto &g : s->graphs)
    if (g.uin == u_in && g.uout == u_out && g.f == f_eff && g.mode == mode && g.count == count &&
        g.l2 == s->sum_l2 && g.hist == hist_on(s))
      ex = g.exec;
  if (!ex) {
    if (s->graphs.size() >= 48) drop_graphs(s);
    cudaGraph_t g = nullptr;
    CKS(s, cudaStreamBeginCapture(s->st, cudaStreamCaptureModeThreadLocal));
    take_launch_error();
    const void *a = u_in;
    void *b = u_out;
    for (int i = 0; i < count; i++) {
      s->impl->enqueue_cycle_mode(a, b, f_eff, s->st, nullptr, mode);
      if (a != b) {
        void *t = const_cast<void *>(a);
        a = b;
        b = t;
      }
    }
    cudaError_t le = cudaGetLastError();
    if (le == cudaSuccess) le = take_launch_error();
    std::string tmsg;
    const int tc = s->impl->take_status(&tmsg);   // a failed transport step (multi-GPU)
    cudaError_t e = cudaStreamEndCapture(s->st, &g);
    if (tc != MG_OK) {   // never instantiate a half-enqueued cycle
      if (g) cudaGraphDestroy(g);
      return fail(s, tc, "V-cycle capture: " + tmsg);
    }
    if (le != cudaSuccess) {
      if (g) cudaGraphDestroy(g);
      return fail(s, MG_ECUDA, std::string("kernel launch during capture: ") + cudaGetErrorString(le));
    }
    CKS(s, e);
    e = cudaGraphInstantiate(&ex, g, 0);
    cudaGraphDestroy(g);
    CKS(s, e);
    s->graphs.push_back({ex, u_in, u_out, f_eff, mode, count, s->sum_l2, hist_on(s)});
  }
  CKS(s, cudaGraphLaunch(ex, s->st));
  return MG_OK;
}
static int run_cycle(mg_solver *s, const void *u_in, void *u_out, const void *f_eff, int mode) {
  return run_cycles(s, u_in, u_out, f_eff, mode, 1);
}

// V-cycles per CUDA graph in a run of cycles of one mode (MG_GRAPH_CYCLES, default 8; 1 = one graph per cycle)
static int graph_cycles() {
  static const int k = [] {
    const char *e = getenv("MG_GRAPH_CYCLES");
    const int v = e ? atoi(e) : 8;
    return v < 1 ? 1 : (v > 64 ? 64 : v);
  }();
  return k;
}

static bool aligned16(const void *p) { return ((uintptr_t)p & 15) == 0; }

static int begin(mg_solver *s) {
  CKS(s, cudaEventRecord(s->ev_in, s->user));
  CKS(s, cudaStreamWaitEvent(s->st, s->ev_in, 0));
  return MG_OK;
}
static int end(mg_solver *s) {
  CKS(s, cudaGetLastError());
  CKS(s, take_launch_error());   // a pass whose launch was rejected (kernels.h)
  std::string tmsg;
  const int tc = s->impl ? s->impl->take_status(&tmsg) : MG_OK;   // transport (NCCL) failures
  if (tc != MG_OK) {
    drop_graphs(s);
    return fail(s, tc, tmsg);
  }
  CKS(s, cudaEventRecord(s->ev_out, s->st));
  CKS(s, cudaStreamWaitEvent(s->user, s->ev_out, 0));
  return MG_OK;
}

static int check_config(const mg_config *c, int *k_out) {
  if (!c) return MG_EINVAL;
  if (c->dim != 2 && c->dim != 3) return MG_EINVAL;
  if (c->order != 2 && c->order != 4) return MG_EINVAL;
  if (c->dtype != MG_F64 && c->dtype != MG_F32) return MG_EINVAL;
  int k = log2_exact(c->n - 1);
  if (k < 2) return MG_EINVAL;
  if (c->dim == 3 && c->n > 2049) return MG_EUNSUPPORTED;
  if (c->n > (int64_t(1) << 30)) return MG_EUNSUPPORTED;
  int np = (c->dim == 2) ? 1 : 4;
  for (int i = 0; i < np; i++)
    if (!(c->p[i] > 0.0 && c->p[i] <= 3.0)) return MG_EINVAL;
  if (c->pitch != 0 && c->pitch < c->n) return MG_EINVAL;
  if (c->sweeps < 0 || c->sweeps > 8) return MG_EINVAL;
  if (c->sweeps > 1 && (c->dim != 2 || c->nranks > 1 || (c->flags & MG_FLAG_CONVENTIONAL))) return MG_EUNSUPPORTED;
  if (c->nranks < 0 || (c->nranks > 1 && (c->rank < 0 || c->rank >= c->nranks))) return MG_EINVAL;
  if (c->nranks > 1 || (c->flags & MG_FLAG_SLABS)) {
    // y-slabs (2D, dist2.cu) / z-slabs (3D, dist3.cu) of the hierarchy
    if (log2_exact(c->nranks) < 0 || ((c->n - 1) / c->nranks) < 4) return MG_EUNSUPPORTED;
    int64_t pt = c->pitch ? c->pitch : c->n;
    if ((pt * (c->dtype == MG_F64 ? 8 : 4)) % 16 != 0) return MG_EUNSUPPORTED;
    if (!(c->flags & MG_FLAG_LOOPBACK) && !c->nccl_id) return MG_EINVAL;
  }
  *k_out = k;
  return MG_OK;
}

// =================================================================== ABI
__global__ void k_rate_norm(const double *ss, double *ratios, int k, double *prev, double *inv) {
  const double nrm = sqrt(*ss);
  ratios[k] = nrm / *prev;
  *inv = nrm > 0.0 ? 1.0 / nrm : 0.0;
  *prev = 1.0;
}
template <class T>
__global__ void k_rate_scale(const T *src, T *dst, size_t n, const double *inv) {
  const T f = (T)*inv;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    dst[i] = src[i] * f;
}

// Device-to-device re-pitch (staging of pitch = n callers): each warp copies
// 128-element chunks of a row, four coalesced element loads in flight per lane.
// cudaMemcpy2DAsync moves such rows (n * esz bytes, never a multiple of 16)
// at about a third of the copy rate.
template <typename E>
__global__ void __launch_bounds__(256) k_repitch(E *__restrict__ dst, int64_t dp, const E *__restrict__ src,
                                                 int64_t sp, int n, unsigned chunks, unsigned units) {
  const unsigned lane = threadIdx.x & 31, nw = gridDim.x * (blockDim.x >> 5);
  for (unsigned w = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); w < units; w += nw) {
    const unsigned r = w / chunks, c0 = (w - r * chunks) * 128 + lane;
    const E *sr = src + (int64_t)r * sp;
    E *dr = dst + (int64_t)r * dp;
    E v[4];
#pragma unroll
    for (int k = 0; k < 4; k++)
      if (c0 + 32 * k < (unsigned)n) v[k] = sr[c0 + 32 * k];
#pragma unroll
    for (int k = 0; k < 4; k++)
      if (c0 + 32 * k < (unsigned)n) dr[c0 + 32 * k] = v[k];
  }
}

extern "C" {

int mg_create_ex(const mg_config *cfg, mg_solver **out) {
  if (!out) return MG_EINVAL;
  *out = nullptr;
  int k = 0;
  int rc = check_config(cfg, &k);
  if (rc != MG_OK) return rc;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
    cudaGetLastError();
    return MG_ENODEV;
  }
  auto s = std::make_unique<mg_solver>();
  s->cfg = *cfg;
  s->k = k;
  s->L = (cfg->dim == 2) ? 2 * k - 1 : 3 * k - 2;
  s->esz = (cfg->dtype == MG_F64) ? 8 : 4;
  s->pitch = cfg->pitch ? cfg->pitch : cfg->n;
  s->cfg.pitch = s->pitch;
  {
    // the work layout: the caller's when its rows are 16-byte multiples, else
    // n rounded up to 128 bytes for the solvers that run the TMA kernels
    // (single GPU, diagonal scheme, one sweep); the others read any pitch
    const bool tma = cfg->nranks <= 1 && !(cfg->flags & (MG_FLAG_CONVENTIONAL | MG_FLAG_SLABS)) && cfg->sweeps <= 1 &&
                     !env_flag("MG_FORCE_REF");
    const int64_t q = 128 / s->esz;
    s->wpitch = ((s->pitch * s->esz) % 16 == 0 || !tma) ? s->pitch : round_up(cfg->n, q);
  }
  if (cfg->nranks == 0) s->cfg.nranks = 1;
  if (cfg->device >= 0) {
    if (cfg->device >= ndev) return MG_EINVAL;
    s->device = cfg->device;
  } else {
    cudaGetDevice(&s->device);
  }
  DeviceGuard g(s->device);
  s->user = (cudaStream_t)cfg->stream;
  mg_solver *sp = s.get();
  CKS(sp, cudaStreamCreateWithFlags(&s->st, cudaStreamNonBlocking));
  CKS(sp, cudaEventCreateWithFlags(&s->ev_in, cudaEventDisableTiming));
  CKS(sp, cudaEventCreateWithFlags(&s->ev_out, cudaEventDisableTiming));
  CKS(sp, cudaMalloc(&s->d_hist, sizeof(unsigned long long) * kHistCap));
  CKS(sp, cudaMalloc(&s->d_counter, sizeof(int)));
  CKS(sp, cudaMalloc(&s->d_mx, sizeof(unsigned long long)));
  CKS(sp, cudaMalloc(&s->d_ss, sizeof(double)));
  CKS(sp, cudaMemset(s->d_hist, 0, sizeof(unsigned long long) * kHistCap));
  CKS(sp, cudaMemset(s->d_counter, 0, sizeof(int)));
  CKS(sp, cudaMallocHost(&s->h_hist, sizeof(unsigned long long) * kHistCap));
  CKS(sp, cudaMalloc(&s->d_l2, sizeof(double) * kHistCap));
  CKS(sp, cudaMemset(s->d_l2, 0, sizeof(double) * kHistCap));
  CKS(sp, cudaMallocHost(&s->h_l2, sizeof(double) * kHistCap));
  if (cfg->flags & MG_FLAG_CONVENTIONAL) {
    if (cfg->nranks > 1 || (cfg->flags & MG_FLAG_SLABS)) {
      mg_destroy(s.release());
      return MG_EUNSUPPORTED;
    }
    s->impl.reset(make_conv(sp));
  } else if (cfg->nranks > 1 || (cfg->flags & MG_FLAG_SLABS)) {
    std::string why;
    const bool lb = (cfg->flags & MG_FLAG_LOOPBACK) != 0;
    ImplBase *d = cfg->dim == 2 ? make_dist2(sp, lb, &why) : make_dist3(sp, lb, &why);
    if (!d) {
      fprintf(stderr, "[libmg] multi-GPU init failed: %s\n", why.c_str());
      mg_destroy(s.release());
      return MG_ENCCL;
    }
    s->impl.reset(d);
  } else if (cfg->dim == 2) {
    if (cfg->dtype == MG_F64) s->impl.reset(new Impl2<double>(sp));
    else s->impl.reset(new Impl2<float>(sp));
  } else {
    if (cfg->dtype == MG_F64) s->impl.reset(new Impl3<double>(sp));
    else s->impl.reset(new Impl3<float>(sp));
  }
  cudaError_t e = s->impl->alloc();
  if (e != cudaSuccess) {
    int code = (e == cudaErrorMemoryAllocation) ? MG_ENOMEM : MG_ECUDA;
    mg_destroy(s.release());
    return code;
  }
  for (int l = 0; l < s->L; l++) s->impl->Nl.push_back((double)mg_level_points(sp, l));
  if (cfg->order == 4) {
    CKS(sp, cudaMalloc(&s->d_ft, s->work_elems() * s->esz));
    CKS(sp, cudaMemset(s->d_ft, 0, s->work_elems() * s->esz));
  }
  CKS(sp, cudaDeviceSynchronize());
  *out = s.release();
  return MG_OK;
}

int mg_create(int dim, int64_t n, int order, double omega, mg_solver **out) {
  mg_config c{};
  c.dim = dim;
  c.n = n;
  c.order = order;
  c.dtype = MG_F64;
  for (int i = 0; i < 4; i++) c.p[i] = omega;
  c.pitch = 0;
  c.stream = nullptr;
  c.device = -1;
  c.nranks = 1;
  c.rank = 0;
  return mg_create_ex(&c, out);
}

int mg_destroy(mg_solver *s) {
  if (!s) return MG_OK;
  DeviceGuard g(s->device);
  if (s->st) cudaStreamSynchronize(s->st);
  drop_graphs(s);
  int rc = MG_OK;
  if (s->impl && ImplBase::poison()) {
    const int bad = s->impl->check_guards();
    if (bad) {
      fprintf(stderr, "[libmg] MG_POISON: guard bytes of %d level arrays overwritten\n", bad);
      rc = MG_ECUDA;
    }
  }
  cudaFree(s->d_ualt);
  if (s->impl) s->impl->free_all();
  cudaFree(s->d_hist);
  cudaFree(s->d_counter);
  cudaFree(s->d_mx);
  if (s->d_zero) cudaFree(s->d_zero);
  cudaFree(s->d_ss);
  cudaFree(s->d_ft);
  cudaFree(s->d_u_stage);
  cudaFree(s->d_f_stage);
  cudaFree(s->d_u_stage2);
  cudaFree(s->d_f_stage2);
  for (int i = 0; i < 2; i++) {
    if (s->ev_h2d[i]) cudaEventDestroy(s->ev_h2d[i]);
    if (s->ev_comp[i]) cudaEventDestroy(s->ev_comp[i]);
    if (s->ev_d2h[i]) cudaEventDestroy(s->ev_d2h[i]);
  }
  if (s->st_h2d) cudaStreamDestroy(s->st_h2d);
  if (s->st_d2h) cudaStreamDestroy(s->st_d2h);
  if (s->h_hist) cudaFreeHost(s->h_hist);
  cudaFree(s->d_l2);
  if (s->h_l2) cudaFreeHost(s->h_l2);
  if (s->ev_in) cudaEventDestroy(s->ev_in);
  if (s->ev_out) cudaEventDestroy(s->ev_out);
  if (s->st) cudaStreamDestroy(s->st);
  delete s;
  return rc;
}

int mg_local_extent(const mg_solver *s, int64_t *lo, int64_t *hi, int64_t *ghost) {
  if (!s) return MG_EINVAL;
  int64_t l, h, g;
  if (s->impl && s->impl->extent(&l, &h, &g)) {
    if (lo) *lo = l;
    if (hi) *hi = h;
    if (ghost) *ghost = g;
    return MG_OK;
  }
  if (lo) *lo = 0;
  if (hi) *hi = s->cfg.n;
  if (ghost) *ghost = 0;
  return MG_OK;
}

int mg_num_levels(const mg_solver *s) { return s ? s->L : MG_EINVAL; }

int64_t mg_level_points(const mg_solver *s, int lev) {
  if (!s || lev < 0 || lev >= s->L) return MG_EINVAL;
  int dim = s->cfg.dim;
  int o = (dim == 2) ? lev / 2 : lev / 3, cls = (dim == 2) ? lev % 2 : lev % 3;
  int64_t m = ((s->cfg.n - 1) >> o) - 1;
  int64_t od = (m + 1) / 2, ev = (m - 1) / 2;
  if (dim == 2) return cls == 0 ? m * m : (m * m + 1) / 2;
  if (cls == 0) return m * m * m;
  if (cls == 1) return ev * ev * ev + 3 * ev * od * od;
  return ev * ev * ev + od * od * od;
}

int mg_launches_per_cycle(const mg_solver *s) { return s ? s->impl->launches_per_cycle() : MG_EINVAL; }

// ---------------------------------------------------------- staging
// The cycle kernels read u and f (or f~) in the work layout: row pitch
// s->wpitch (16-byte rows), 16-byte aligned base.  A caller whose layout is
// that already is read in place; otherwise (pitch = n with n = 2^k+1 never
// gives 16-byte rows; an offset base pointer) each call copies u and f into
// the library's work arrays (one 2D copy each), runs the cycles there and
// copies u back -- the TMA kernels run either way.
static bool work_layout(const mg_solver *s, const void *a) { return s->wpitch == s->pitch && aligned16(a); }

static int ensure_stage(mg_solver *s) {
  if (s->d_u_stage) return MG_OK;
  const size_t bytes = s->work_elems() * s->esz;
  CKS(s, cudaMalloc(&s->d_u_stage, bytes));
  CKS(s, cudaMalloc(&s->d_f_stage, bytes));
  CKS(s, cudaMemsetAsync(s->d_u_stage, 0, bytes, s->st));   // padding columns stay zero
  CKS(s, cudaMemsetAsync(s->d_f_stage, 0, bytes, s->st));
  return MG_OK;
}

// rows x n elements between two layouts (pitches in elements); one contiguous
// copy when the layouts agree (a pitched host<->device copy of 64 KB rows is
// slower than one linear DMA transfer)
static cudaError_t copy_field_st(mg_solver *s, void *dst, int64_t dp, const void *src, int64_t sp,
                                 cudaMemcpyKind kind, cudaStream_t st) {
  if (dp == sp) return cudaMemcpyAsync(dst, src, (size_t)s->rows() * sp * s->esz, kind, st);
  static const bool own = !env_flag("MG_STAGE_MEMCPY2D");
  const int64_t chunks = (s->cfg.n + 127) / 128, units = (int64_t)s->rows() * chunks;
  if (own && kind == cudaMemcpyDeviceToDevice && units > 0 && units < (int64_t)1 << 31 &&
      (((uintptr_t)dst | (uintptr_t)src) & (s->esz - 1)) == 0) {
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, s->device);
    const unsigned grid = (unsigned)std::min<int64_t>((units + 7) / 8, (int64_t)sms * 8);
    if (s->esz == 8)
      k_repitch<unsigned long long><<<grid, 256, 0, st>>>((unsigned long long *)dst, dp, (const unsigned long long *)src,
                                                          sp, s->cfg.n, (unsigned)chunks, (unsigned)units);
    else
      k_repitch<unsigned><<<grid, 256, 0, st>>>((unsigned *)dst, dp, (const unsigned *)src, sp, s->cfg.n,
                                                (unsigned)chunks, (unsigned)units);
    return cudaGetLastError();
  }
  return cudaMemcpy2DAsync(dst, dp * s->esz, src, sp * s->esz, s->cfg.n * s->esz, s->rows(), kind, st);
}
static cudaError_t copy_field(mg_solver *s, void *dst, int64_t dp, const void *src, int64_t sp, cudaMemcpyKind kind) {
  return copy_field_st(s, dst, dp, src, sp, kind, s->st);
}

int mg_residual(mg_solver *s, const void *u, const void *f, void *r) {
  if (!s || !u || !f || !r) return fail(s, MG_EINVAL, "mg_residual: NULL argument");
  DeviceGuard g(s->device);
  int rc = begin(s);
  if (rc) return rc;
  if (s->cfg.order == 4) {
    // r uses f~ formed from f (Efos2/Efos4), in the f~ buffer (work layout)
    s->impl->enqueue_ftilde(f, s->d_ft, s->st, s->wpitch);
    s->impl->enqueue_residual(u, s->d_ft, r, s->st, s->wpitch);
  } else {
    s->impl->enqueue_residual(u, f, r, s->st, s->pitch);
  }
  return end(s);
}

// ncycles V-cycles on u_w (work layout, aligned) with the right-hand side
// f_eff (work layout: f, or f~ for order 4).
static int cycles_work(mg_solver *s, void *u, const void *fe, int ncycles, double *res_hist) {
  const int nslots = ncycles + 1;   // <= kHistCap (checked by the callers)
  CKS(s, clear_hist(s, nslots, s->st));
  CKS(s, cudaMemsetAsync(s->d_counter, 0, sizeof(int), s->st));
  // TMA path: u alternates between u and an internal partner (the ascent
  // reads the old u in a 2-node halo, so it cannot update in place); an odd
  // cycle count ends with one copy back.
  const bool alt = s->impl->fast();
  if (alt && !s->d_ualt) {
    size_t bytes = s->work_elems() * s->esz;
    CKS(s, cudaMalloc(&s->d_ualt, bytes));
    CKS(s, cudaMemsetAsync(s->d_ualt, 0, bytes, s->st));
  }
  // Cross-cycle fusion: every cycle but the first skips its finest descent,
  // which the previous cycle's last pass computed (and the final residual
  // norm comes from the last cycle's when it is wanted).
  const bool xf = alt && s->impl->fuses_cycles();
  void *cur = u;
  auto mode_of = [&](int c) {
    int mode = 0;
    if (xf && c > 0) mode |= ImplBase::kSkipDesc;
    if (xf && (c + 1 < ncycles || res_hist)) mode |= ImplBase::kFuseNext;
    return mode;
  };
  for (int c = 0; c < ncycles;) {
    void *dst = alt ? (cur == u ? s->d_ualt : u) : u;
    const int mode = mode_of(c);
    // graph_cycles() cycles of this mode per graph while the run has that many left, then one per graph:
    // only two graph sizes per mode, so a call never captures a graph a shorter earlier call did not
    int run = 1;
    while (c + run < ncycles && run < graph_cycles() && mode_of(c + run) == mode) run++;
    const int cnt = run == graph_cycles() ? run : 1;
    int rc = run_cycles(s, cur, dst, fe, mode, cnt);
    if (rc) return rc;
    if (cnt & 1) cur = dst;
    c += cnt;
  }
  if (cur != u) CKS(s, cudaMemcpyAsync(u, cur, s->work_elems() * s->esz, cudaMemcpyDeviceToDevice, s->st));
  if (res_hist) {
    if (!xf || ncycles == 0) s->impl->enqueue_final_norm(u, fe, s->st);
    CKS(s, s->impl->reduce_hist(s->d_hist, nslots, s->st));
    return read_hist(s, ncycles, res_hist, s->st);
  }
  return MG_OK;
}

// f_eff in the work layout from the caller's f (device, caller layout)
static int rhs_work(mg_solver *s, const void *f, const void **fe) {
  if (s->cfg.order == 4) {
    s->impl->enqueue_ftilde(f, s->d_ft, s->st, s->wpitch);   // reads f in the caller's layout
    *fe = s->d_ft;
    return MG_OK;
  }
  if (work_layout(s, f)) {
    *fe = f;
    return MG_OK;
  }
  int rc = ensure_stage(s);
  if (rc) return rc;
  CKS(s, copy_field(s, s->d_f_stage, s->wpitch, f, s->pitch, cudaMemcpyDeviceToDevice));
  *fe = s->d_f_stage;
  return MG_OK;
}

static int vcycle_dev(mg_solver *s, void *u, const void *f, int ncycles, double *res_hist) {
  const void *fe = nullptr;
  int rc = rhs_work(s, f, &fe);
  if (rc) return rc;
  if (work_layout(s, u)) return cycles_work(s, u, fe, ncycles, res_hist);
  rc = ensure_stage(s);
  if (rc) return rc;
  CKS(s, copy_field(s, s->d_u_stage, s->wpitch, u, s->pitch, cudaMemcpyDeviceToDevice));
  rc = cycles_work(s, s->d_u_stage, fe, ncycles, res_hist);
  if (rc) return rc;
  CKS(s, copy_field(s, u, s->pitch, s->d_u_stage, s->wpitch, cudaMemcpyDeviceToDevice));
  return MG_OK;
}

int mg_vcycle_norms(mg_solver *s, void *u, const void *f, int ncycles, double *res_inf, double *res_l2) {
  if (!s) return MG_EINVAL;
  if (!u || !f) return fail(s, MG_EINVAL, "mg_vcycle: NULL u or f");
  if (ncycles < 0) return fail(s, MG_EINVAL, "mg_vcycle: ncycles < 0");
  if (res_l2 && !res_inf) return fail(s, MG_EINVAL, "mg_vcycle_norms: res_l2 needs res_inf");
  if (res_inf && ncycles + 1 > kHistCap) return fail(s, MG_EINVAL, "mg_vcycle: res_hist needs ncycles < 4096");
  if (ncycles == 0 && !res_inf) return MG_OK;
  DeviceGuard g(s->device);
  int rc = begin(s);
  if (rc) return rc;
  s->l2_out = res_l2;
  s->sum_l2 = res_l2 != nullptr;
  s->want_hist = res_inf != nullptr;
  rc = s->impl->vcycle_all(s, u, f, ncycles, res_inf);
  if (rc == 1) rc = vcycle_dev(s, u, f, ncycles, res_inf);
  s->l2_out = nullptr;
  s->sum_l2 = false;
  s->want_hist = false;
  int rc2 = end(s);
  return rc ? rc : rc2;
}

int mg_vcycle(mg_solver *s, void *u, const void *f, int ncycles, double *res_hist) {
  return mg_vcycle_norms(s, u, f, ncycles, res_hist, nullptr);
}

// Host arrays (caller layout) are copied straight into the work layout.
// mg_vcycle_host / mg_solve_host: host arrays in and out, the work layout in
// between; zero_start: u starts from 0 on the device (a memset, no upload).
static int host_cycles(mg_solver *s, void *u_host, const void *f_host, int ncycles, double *res_hist, bool zero_start,
                       const char *who) {
  if (!s) return MG_EINVAL;
  if (!u_host || !f_host) return fail(s, MG_EINVAL, std::string(who) + ": NULL u or f");
  if (ncycles < 0) return fail(s, MG_EINVAL, std::string(who) + ": ncycles < 0");
  if (res_hist && ncycles + 1 > kHistCap) return fail(s, MG_EINVAL, std::string(who) + ": res_hist needs ncycles < 4096");
  DeviceGuard g(s->device);
  int rc = begin(s);
  if (rc) return rc;
  rc = ensure_stage(s);
  if (!rc) rc = [&]() -> int {
    if (zero_start) CKS(s, cudaMemsetAsync(s->d_u_stage, 0, s->work_elems() * s->esz, s->st));
    else CKS(s, copy_field(s, s->d_u_stage, s->wpitch, u_host, s->pitch, cudaMemcpyHostToDevice));
    const void *fe = s->d_f_stage;
    if (s->cfg.order == 4) {
      // f~ is formed on the device from f in the caller's layout (d_f_stage is large enough)
      CKS(s, cudaMemcpyAsync(s->d_f_stage, f_host, s->field_elems() * s->esz, cudaMemcpyHostToDevice, s->st));
      s->impl->enqueue_ftilde(s->d_f_stage, s->d_ft, s->st, s->wpitch);
      fe = s->d_ft;
    } else {
      CKS(s, copy_field(s, s->d_f_stage, s->wpitch, f_host, s->pitch, cudaMemcpyHostToDevice));
    }
    // (loopback slabs take the raw f: one layout there, so d_f_stage holds it as given)
    s->want_hist = res_hist != nullptr;
    int r = s->impl->vcycle_all(s, s->d_u_stage, s->d_f_stage, ncycles, res_hist);
    if (r == 1) r = cycles_work(s, s->d_u_stage, fe, ncycles, res_hist);
    s->want_hist = false;
    if (r) return r;
    CKS(s, copy_field(s, u_host, s->pitch, s->d_u_stage, s->wpitch, cudaMemcpyDeviceToHost));
    CKS(s, cudaStreamSynchronize(s->st));
    return MG_OK;
  }();
  int rc2 = end(s);   // joins the caller's stream on every path
  return rc ? rc : rc2;
}

int mg_vcycle_host(mg_solver *s, void *u_host, const void *f_host, int ncycles, double *res_hist) {
  return host_cycles(s, u_host, f_host, ncycles, res_hist, false, "mg_vcycle_host");
}

int mg_solve_host(mg_solver *s, void *u_host, const void *f_host, int ncycles, double *res_hist) {
  return host_cycles(s, u_host, f_host, ncycles, res_hist, true, "mg_solve_host");
}

// Independent solves from u = 0 of `count` right-hand sides: problem i's f
// upload (stream st_h2d), cycles (the solver stream) and u download (st_d2h)
// run on three streams over two device staging slots, so the download of
// problem i-1 and the upload of problem i+1 overlap the cycles of problem i
// (PCIe is full duplex).  Slot reuse is ordered by events: the upload into a
// slot waits for the cycles that last read its f, the cycles wait for the
// download that last read its u.
int mg_solve_host_batch(mg_solver *s, void *const *u_hosts, const void *const *f_hosts, int count, int ncycles) {
  if (!s) return MG_EINVAL;
  if (count < 0 || ncycles < 0 || (count > 0 && (!u_hosts || !f_hosts)))
    return fail(s, MG_EINVAL, "mg_solve_host_batch: bad argument");
  for (int i = 0; i < count; i++)
    if (!u_hosts[i] || !f_hosts[i]) return fail(s, MG_EINVAL, "mg_solve_host_batch: NULL u or f");
  if (s->cfg.nranks > 1 || (s->cfg.flags & MG_FLAG_SLABS)) {   // slab solvers: one problem at a time
    for (int i = 0; i < count; i++) {
      int rc = host_cycles(s, u_hosts[i], f_hosts[i], ncycles, nullptr, true, "mg_solve_host_batch");
      if (rc) return rc;
    }
    return MG_OK;
  }
  DeviceGuard g(s->device);
  int rc = begin(s);
  if (rc) return rc;
  rc = ensure_stage(s);
  if (!rc) rc = [&]() -> int {
    const size_t bytes = s->work_elems() * s->esz;
    if (!s->d_u_stage2) {
      CKS(s, cudaMalloc(&s->d_u_stage2, bytes));
      CKS(s, cudaMalloc(&s->d_f_stage2, bytes));
      CKS(s, cudaMemsetAsync(s->d_u_stage2, 0, bytes, s->st));
      CKS(s, cudaMemsetAsync(s->d_f_stage2, 0, bytes, s->st));
    }
    if (!s->st_h2d) {
      CKS(s, cudaStreamCreateWithFlags(&s->st_h2d, cudaStreamNonBlocking));
      CKS(s, cudaStreamCreateWithFlags(&s->st_d2h, cudaStreamNonBlocking));
      for (int i = 0; i < 2; i++) {
        CKS(s, cudaEventCreateWithFlags(&s->ev_h2d[i], cudaEventDisableTiming));
        CKS(s, cudaEventCreateWithFlags(&s->ev_comp[i], cudaEventDisableTiming));
        CKS(s, cudaEventCreateWithFlags(&s->ev_d2h[i], cudaEventDisableTiming));
      }
    }
    void *us[2] = {s->d_u_stage, s->d_u_stage2}, *fs[2] = {s->d_f_stage, s->d_f_stage2};
    // the copy streams start after everything queued so far on the solver stream (and so the caller's)
    CKS(s, cudaEventRecord(s->ev_comp[0], s->st));
    CKS(s, cudaStreamWaitEvent(s->st_h2d, s->ev_comp[0], 0));
    CKS(s, cudaStreamWaitEvent(s->st_d2h, s->ev_comp[0], 0));
    for (int i = 0; i < count; i++) {
      const int k = i & 1;
      if (i >= 2) CKS(s, cudaStreamWaitEvent(s->st_h2d, s->ev_comp[k], 0));   // f[k] free
      if (s->cfg.order == 4)
        CKS(s, cudaMemcpyAsync(fs[k], f_hosts[i], s->field_elems() * s->esz, cudaMemcpyHostToDevice, s->st_h2d));
      else
        CKS(s, copy_field_st(s, fs[k], s->wpitch, f_hosts[i], s->pitch, cudaMemcpyHostToDevice, s->st_h2d));
      CKS(s, cudaEventRecord(s->ev_h2d[k], s->st_h2d));
      CKS(s, cudaStreamWaitEvent(s->st, s->ev_h2d[k], 0));
      if (i >= 2) CKS(s, cudaStreamWaitEvent(s->st, s->ev_d2h[k], 0));          // u[k] downloaded
      CKS(s, cudaMemsetAsync(us[k], 0, bytes, s->st));
      const void *fe = fs[k];
      if (s->cfg.order == 4) {
        s->impl->enqueue_ftilde(fs[k], s->d_ft, s->st, s->wpitch);
        fe = s->d_ft;
      }
      int r = cycles_work(s, us[k], fe, ncycles, nullptr);
      if (r) return r;
      CKS(s, cudaEventRecord(s->ev_comp[k], s->st));
      CKS(s, cudaStreamWaitEvent(s->st_d2h, s->ev_comp[k], 0));
      CKS(s, copy_field_st(s, u_hosts[i], s->pitch, us[k], s->wpitch, cudaMemcpyDeviceToHost, s->st_d2h));
      CKS(s, cudaEventRecord(s->ev_d2h[k], s->st_d2h));
    }
    // the solver stream (and through end() the caller's) ends after the last download
    CKS(s, cudaEventRecord(s->ev_d2h[0], s->st_d2h));
    CKS(s, cudaStreamWaitEvent(s->st, s->ev_d2h[0], 0));
    CKS(s, cudaStreamSynchronize(s->st));
    return MG_OK;
  }();
  int rc2 = end(s);
  return rc ? rc : rc2;
}

// ---------------------------------------------------- convergence factor
// power iteration on the error equation (f = 0), every
// step on the device.  One iteration: one V-cycle e -> e' (no cross-cycle
// fusion: e is rescaled between cycles), ss = sum e'^2 over the interior
// (the norm kernel), then k_rate_scale: ratio_k = sqrt(ss) / prev, e = e' /
// sqrt(ss), prev = 1.
int mg_convergence_factor(mg_solver *s, void *e_user, int iters, double *rho, double *ratios) {
  if (!s) return MG_EINVAL;
  if (!e_user || iters < 2 || !rho) return fail(s, MG_EINVAL, "mg_convergence_factor: bad argument");
  if (s->cfg.nranks > 1 || (s->cfg.flags & MG_FLAG_SLABS))
    return fail(s, MG_EUNSUPPORTED, "mg_convergence_factor: single GPU only");
  DeviceGuard g(s->device);
  int rc = begin(s);
  if (rc) return rc;
  double *d_rate = nullptr;   // [0] prev, [1] 1/norm, [2 ..] ratios
  std::vector<double> h(iters + 1);
  rc = [&]() -> int {
    // the iteration runs on e in the work layout (staged when the caller's is another)
    void *e = e_user;
    const bool staged = !work_layout(s, e_user);
    if (staged) {
      int r = ensure_stage(s);
      if (r) return r;
      e = s->d_u_stage;
      CKS(s, copy_field(s, e, s->wpitch, e_user, s->pitch, cudaMemcpyDeviceToDevice));
    }
    const size_t ne = s->work_elems(), bytes = ne * s->esz;
    if (!s->d_zero) {
      CKS(s, cudaMalloc(&s->d_zero, bytes));
      CKS(s, cudaMemsetAsync(s->d_zero, 0, bytes, s->st));
    }
    const bool alt = s->impl->fast();
    if (alt && !s->d_ualt) {
      CKS(s, cudaMalloc(&s->d_ualt, bytes));
      CKS(s, cudaMemsetAsync(s->d_ualt, 0, bytes, s->st));
    }
    CKS(s, cudaMalloc(&d_rate, sizeof(double) * (iters + 3)));
    const double one = 1.0;
    // normalise the start vector first (ratio 0 of the history is its norm)
    CKS(s, cudaMemcpyAsync(d_rate, &one, sizeof one, cudaMemcpyHostToDevice, s->st));
    CKS(s, cudaMemsetAsync(s->d_mx, 0, sizeof(unsigned long long), s->st));
    CKS(s, cudaMemsetAsync(s->d_ss, 0, sizeof(double), s->st));
    s->impl->enqueue_norm(e, s->d_mx, s->d_ss, s->st, s->wpitch);
    k_rate_norm<<<1, 1, 0, s->st>>>(s->d_ss, d_rate + 2, 0, d_rate, d_rate + 1);
    const int nb = 148 * 8;
    if (s->esz == 8)
      k_rate_scale<double><<<nb, 256, 0, s->st>>>((const double *)e, (double *)e, ne, d_rate + 1);
    else
      k_rate_scale<float><<<nb, 256, 0, s->st>>>((const float *)e, (float *)e, ne, d_rate + 1);
    CKS(s, cudaMemsetAsync(s->d_counter, 0, sizeof(int), s->st));
    for (int it = 1; it <= iters; it++) {
      void *dst = alt ? s->d_ualt : e;
      int r = run_cycle(s, e, dst, s->d_zero, 0);
      if (r) return r;
      CKS(s, cudaMemsetAsync(s->d_mx, 0, sizeof(unsigned long long), s->st));
      CKS(s, cudaMemsetAsync(s->d_ss, 0, sizeof(double), s->st));
      s->impl->enqueue_norm(dst, s->d_mx, s->d_ss, s->st, s->wpitch);
      k_rate_norm<<<1, 1, 0, s->st>>>(s->d_ss, d_rate + 2, it, d_rate, d_rate + 1);
      if (s->esz == 8)
        k_rate_scale<double><<<nb, 256, 0, s->st>>>((const double *)dst, (double *)e, ne, d_rate + 1);
      else
        k_rate_scale<float><<<nb, 256, 0, s->st>>>((const float *)dst, (float *)e, ne, d_rate + 1);
    }
    if (staged) CKS(s, copy_field(s, e_user, s->pitch, e, s->wpitch, cudaMemcpyDeviceToDevice));
    CKS(s, cudaMemcpyAsync(h.data(), d_rate + 2, sizeof(double) * (iters + 1), cudaMemcpyDeviceToHost, s->st));
    CKS(s, cudaStreamSynchronize(s->st));
    return MG_OK;
  }();
  if (d_rate) cudaFree(d_rate);
  int rc2 = end(s);
  if (rc || rc2) return rc ? rc : rc2;
  // geometric mean of the ratios of the second half of the iterations
  double lg = 0.0;
  int m = 0;
  for (int it = iters / 2 + 1; it <= iters; it++, m++) lg += std::log(h[it]);
  *rho = std::exp(lg / m);
  if (ratios)
    for (int it = 0; it < iters; it++) ratios[it] = h[it + 1];
  if (!std::isfinite(*rho)) return fail(s, MG_EDIVERGED, "mg_convergence_factor: non-finite ratio");
  return MG_OK;
}

int mg_norm(mg_solver *s, const void *x, int kind, double *out) {
  if (!s || !x || !out) return fail(s, MG_EINVAL, "mg_norm: NULL argument");
  if (kind != MG_NORM_INF && kind != MG_NORM_L2) return fail(s, MG_EINVAL, "mg_norm: bad kind");
  DeviceGuard g(s->device);
  int rc = begin(s);
  if (rc) return rc;
  unsigned long long mx = 0;
  double ss = 0;
  rc = [&]() -> int {
    CKS(s, cudaMemsetAsync(s->d_mx, 0, sizeof(unsigned long long), s->st));
    CKS(s, cudaMemsetAsync(s->d_ss, 0, sizeof(double), s->st));
    s->impl->enqueue_norm(x, s->d_mx, s->d_ss, s->st, s->pitch);
    CKS(s, cudaMemcpyAsync(&mx, s->d_mx, sizeof mx, cudaMemcpyDeviceToHost, s->st));
    CKS(s, cudaMemcpyAsync(&ss, s->d_ss, sizeof ss, cudaMemcpyDeviceToHost, s->st));
    CKS(s, cudaStreamSynchronize(s->st));
    return MG_OK;
  }();
  int rc2 = end(s);
  if (rc || rc2) return rc ? rc : rc2;
  if (kind == MG_NORM_INF) {
    std::memcpy(out, &mx, sizeof(double));
  } else {
    double h = 1.0 / (double)(s->cfg.n - 1);
    *out = std::sqrt(std::pow(h, s->cfg.dim) * ss);
  }
  if (!std::isfinite(*out)) return fail(s, MG_EDIVERGED, "non-finite norm");
  return MG_OK;
}

int mg_profile(mg_solver *s, void *u_user, const void *f, int ncycles, mg_step_stat *out, int cap) {
  if (!s) return MG_EINVAL;
  if (!u_user || !f || ncycles < 1 || cap < 0 || (cap > 0 && !out)) return fail(s, MG_EINVAL, "mg_profile: bad argument");
  DeviceGuard g(s->device);
  int rc = begin(s);
  if (rc) return rc;
  Prof prof;
  prof.st = s->st;
  std::vector<double> acc;
  rc = [&]() -> int {
    const void *fe = nullptr;
    int r = rhs_work(s, f, &fe);
    if (r) return r;
    void *u = u_user;
    const bool staged = !work_layout(s, u_user);
    if (staged) {
      r = ensure_stage(s);
      if (r) return r;
      u = s->d_u_stage;
      CKS(s, copy_field(s, u, s->wpitch, u_user, s->pitch, cudaMemcpyDeviceToDevice));
    }
    CKS(s, cudaMemsetAsync(s->d_counter, 0, sizeof(int), s->st));
    const bool alt = s->impl->fast();
    if (alt && !s->d_ualt) {
      size_t bytes = s->work_elems() * s->esz;
      CKS(s, cudaMalloc(&s->d_ualt, bytes));
      CKS(s, cudaMemsetAsync(s->d_ualt, 0, bytes, s->st));
    }
    // with cross-cycle fusion every profiled cycle is a steady-state one: the
    // descent of the first runs unprofiled before the loop
    const bool xf = alt && s->impl->fuses_cycles();
    const int mode = xf ? ImplBase::kSkipDesc | ImplBase::kFuseNext : 0;
    if (xf) s->impl->enqueue_pre_descent(u, fe, s->st);
    void *cur = u;
    for (int c = 0; c < ncycles; c++) {
      void *dst = alt ? (cur == u ? s->d_ualt : u) : u;
      s->impl->enqueue_cycle_mode(cur, dst, fe, s->st, &prof, mode);
      prof.end_cycle();
      cur = dst;
    }
    if (cur != u) CKS(s, cudaMemcpyAsync(u, cur, s->work_elems() * s->esz, cudaMemcpyDeviceToDevice, s->st));
    if (staged) CKS(s, copy_field(s, u_user, s->pitch, u, s->wpitch, cudaMemcpyDeviceToDevice));
    CKS(s, cudaGetLastError());
    CKS(s, take_launch_error());
    CKS(s, cudaStreamSynchronize(s->st));
    size_t ns = prof.steps.size();
    acc.assign(ns, 0.0);
    for (int c = 0; c < ncycles; c++)
      for (size_t i = 0; i < ns; i++) {
        float ms = 0;
        CKS(s, cudaEventElapsedTime(&ms, prof.evs[c * (ns + 1) + i], prof.evs[c * (ns + 1) + i + 1]));
        acc[i] += ms;
      }
    return MG_OK;
  }();
  int rc2 = end(s);
  if (rc || rc2) return rc ? rc : rc2;
  const size_t ns = acc.size();
  for (size_t i = 0; i < ns && (int)i < cap; i++) {
    std::memset(out[i].name, 0, sizeof out[i].name);
    std::strncpy(out[i].name, prof.steps[i].name.c_str(), sizeof out[i].name - 1);
    out[i].level = prof.steps[i].level;
    out[i].launches = prof.steps[i].launches;
    out[i].ms = acc[i] / ncycles;
    out[i].alg_bytes = prof.steps[i].bytes;
  }
  return (int)ns;
}

int mg_slab_plan(int dim, int64_t n, int nranks, int rank, int64_t agglom_points, int64_t *lo, int64_t *hi,
                 int64_t *ghost, int *agglom_octave) {
  int k = log2_exact(n - 1);
  if (k < 2 || nranks < 1 || rank < 0 || rank >= nranks) return MG_EINVAL;
  if (dim != 2 && dim != 3) return MG_EINVAL;
  if (nranks == 1) {
    if (lo) *lo = 0;
    if (hi) *hi = n;
    if (ghost) *ghost = 0;
    if (agglom_octave) *agglom_octave = 0;
    return MG_OK;
  }
  if (log2_exact(nranks) < 0 || (n - 1) / nranks < 4) return MG_EUNSUPPORTED;
  int64_t R = (n - 1) / nranks;
  if (lo) *lo = rank * R;
  if (hi) *hi = (rank + 1) * R;
  if (ghost) *ghost = 2;
  if (agglom_octave)
    *agglom_octave =
        slab_agglom_octave(n, k, nranks, agglom_points > 0 ? agglom_points : (int64_t(1) << 18), dim);
  return MG_OK;
}

int mg_slab_schedule(int dim, int64_t n, int nranks, int64_t agglom_points, int *schedule, int64_t *halo_rows) {
  int k = log2_exact(n - 1);
  if (k < 2 || nranks < 1 || (dim != 2 && dim != 3)) return MG_EINVAL;
  if (nranks > 1 && (log2_exact(nranks) < 0 || (n - 1) / nranks < 4)) return MG_EUNSUPPORTED;
  int sch = 0;
  int64_t gu = 0;
  if (nranks > 1) {
    const int oa = slab_agglom_octave(n, k, nranks, agglom_points > 0 ? agglom_points : (int64_t(1) << 18), dim);
    gu = 2;
    if (dim == 2) {
      std::vector<int> WD, WA, waD, waA;
      const int g = slab_bands_2d(oa, WD, WA, waD, waA);
      if (oa >= 1 && g <= (n - 1) / nranks) {   // as Dist2CA::alloc (without the MG_DIST_PERLEVEL override)
        sch = 1;
        gu = g;
      }
    }
  }
  if (schedule) *schedule = sch;
  if (halo_rows) *halo_rows = gu;
  return MG_OK;
}

int mg_nccl_unique_id(void *out) {
  if (!out) return MG_EINVAL;
  std::string err;
  int rc = nccl_unique_id(out, &err);
  if (rc) fprintf(stderr, "[libmg] %s\n", err.c_str());
  return rc;
}

const char *mg_strerror(int status) {
  switch (status) {
    case MG_OK: return "ok";
    case MG_EINVAL: return "invalid argument";
    case MG_ENOMEM: return "out of memory";
    case MG_ECUDA: return "CUDA error";
    case MG_ENCCL: return "NCCL error";
    case MG_EUNSUPPORTED: return "unsupported configuration";
    case MG_EDIVERGED: return "diverged (non-finite norm)";
    case MG_ENODEV: return "no CUDA device";
    default: return "unknown status";
  }
}

const char *mg_last_error(const mg_solver *s) { return s ? s->err.c_str() : "NULL handle"; }

}  // extern "C"
