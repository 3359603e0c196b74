// dist2.cu -- the 2D V-cycle on y-slabs over several ranks.
//
// Rank q owns the lattice rows [q M_s/P, (q+1) M_s/P) of every level of
// octave s while M_s/P >= 4 and the level has at least agglom_points
// interior nodes; each slab array carries 2 ghost rows on each side (global
// row indices are kept: the device descriptors point at the virtual global
// row 0).  Before a kernel, the ghost rows it reads are refreshed by a halo
// exchange (1 or 2 rows); at the first agglomerated octave oa the level's
// residual is all-gathered into full arrays and every rank runs the coarse
// octaves redundantly (bit-identical), so the ascent needs no gather back.
// The per-cycle residual-norm maxima are max-reduced over ranks.
//
// Two transports (comm.cu) implement the same schedule: NCCL, one process per
// GPU; and loopback (MG_FLAG_LOOPBACK), P virtual ranks in one process on one
// GPU whose kernels never wait on one another -- it tests the decomposition
// bit for bit against the single-GPU solver.
#include "comm.h"
#include "solver.h"

// ================================================================ Dist2
template <class T>
struct Dist2 : ImplBase {
  mg_solver *s;
  int k, P, nloc;   // nloc = local (virtual) ranks: P in loopback, 1 with NCCL
  bool loop;
  int64_t n, pitch;
  std::unique_ptr<Comm2> comm;
  int oa = 1, oc = 1;
  std::vector<int> M;
  std::vector<T> cD, cA;
  Coef<T> coef{};
  struct Rk {
    int q;
    std::vector<S2<T>> rD, vD;   // octaves o < oa
    std::vector<D2<T>> rA, vA;   // 1 <= o < oa
    D2<T> u[2], f;               // loopback: internal slabs of u (pair) and f / f~
  };
  std::vector<Rk> rk;
  std::vector<S2<T>> rDf, vDf;   // full arrays, octaves o >= oa
  std::vector<D2<T>> rAf, vAf;
  D2<T> uf_scratch{};            // loopback: full f~ (order 4)
  Lev2<T> *d_lev = nullptr;
  std::vector<Lev2<T>> h_lev;   // host copy of the descriptors (coarse solver parameters)

  Dist2(mg_solver *sv, bool loopback) : s(sv), k(sv->k), P(sv->cfg.nranks), loop(loopback), n(sv->cfg.n),
                                        pitch(sv->pitch) {
    nloc = loop ? P : 1;
  }
  bool fast() const override { return true; }
  int64_t pitch_for(int64_t cnt) const { return round_up(cnt, 128 / (int64_t)sizeof(T)); }
  int R(int o) const { return M[o] / P; }                 // A(s) rows per rank at octave o
  int lo(int o, int q) const { return q * R(o); }
  int hi(int o, int q) const { return (q + 1) * R(o); }

  // slab of rows [lo-2, hi+2): virtual global-row-0 pointer
  cudaError_t slab(D2<T> &out, int64_t cols, int lo_, int hi_) {
    int64_t pt = pitch_for(cols);
    void *q;
    cudaError_t e = dalloc(&q, sizeof(T) * pt * (hi_ - lo_ + 4));
    if (e) return e;
    out = D2<T>{(T *)q - (int64_t)(lo_ - 2) * pt, pt};
    return cudaSuccess;
  }
  cudaError_t slab_s(S2<T> &out, int64_t cols, int lo_, int hi_) {
    D2<T> e, o;
    cudaError_t r = slab(e, cols, lo_, hi_);
    if (r) return r;
    r = slab(o, cols, lo_, hi_);
    if (r) return r;
    out = S2<T>{e.p, o.p, e.pitch};
    return cudaSuccess;
  }
  // full array of rows [0, rows) with 2 zero rows of padding on each side
  cudaError_t full(D2<T> &out, int64_t cols, int rows) { return slab(out, cols, 0, rows); }
  cudaError_t full_s(S2<T> &out, int64_t cols, int rows) { return slab_s(out, cols, 0, rows); }

  cudaError_t alloc() override {
    const double p = s->cfg.p[0];
    M.resize(k);
    cD.resize(k);
    cA.resize(k);
    for (int o = 0; o < k; o++) {
      M[o] = (int)((n - 1) >> o);
      double hs = std::ldexp(1.0, o) / (double)(n - 1);
      cD[o] = (T)(2.0 * p * hs * hs);
      cA[o] = (T)(p * hs * hs);
    }
    coef.invh2 = (T)((double)(n - 1) * (double)(n - 1));
    coef.c6 = (T)((double)(n - 1) * (double)(n - 1) / 6.0);
    int64_t ag = s->cfg.agglom_points > 0 ? s->cfg.agglom_points : (int64_t(1) << 18);
    oa = slab_agglom_octave(n, k, P, ag);
    int thresh = 64;
    if (const char *e = getenv("MG_COARSE_M")) thresh = atoi(e);
    oc = k - 1;
    for (int o = oa; o < k; o++)
      if (M[o] <= thresh || o == k - 1) {
        oc = o;
        break;
      }
    if (oc < 1) oc = 1;
    rk.resize(nloc);
    for (int i = 0; i < nloc; i++) {
      Rk &r = rk[i];
      r.q = loop ? i : s->cfg.rank;
      r.rD.resize(oa);
      r.vD.resize(oa);
      r.rA.resize(oa);
      r.vA.resize(oa);
      for (int o = 0; o < oa; o++) {
        int H = M[o] / 2 + 1, l = lo(o, r.q) / 2, h = hi(o, r.q) / 2;
        cudaError_t e;
        if ((e = slab_s(r.rD[o], H, l, h)) || (e = slab_s(r.vD[o], H, l, h))) return e;
        if (o >= 1 && ((e = slab(r.rA[o], M[o] + 1, lo(o, r.q), hi(o, r.q))) ||
                       (e = slab(r.vA[o], M[o] + 1, lo(o, r.q), hi(o, r.q)))))
          return e;
      }
      if (loop) {
        cudaError_t e;
        if ((e = slab(r.u[0], n, lo(0, r.q), hi(0, r.q))) || (e = slab(r.u[1], n, lo(0, r.q), hi(0, r.q))) ||
            (e = slab(r.f, n, lo(0, r.q), hi(0, r.q))))
          return e;
      }
    }
    rDf.resize(k);
    vDf.resize(k);
    rAf.resize(k);
    vAf.resize(k);
    for (int o = oa; o < k; o++) {
      cudaError_t e;
      if ((e = full(rAf[o], M[o] + 1, M[o] + 1)) || (e = full(vAf[o], M[o] + 1, M[o] + 1))) return e;
      if (o + 1 < k && ((e = full_s(rDf[o], M[o] / 2 + 1, M[o] / 2 + 1)) || (e = full_s(vDf[o], M[o] / 2 + 1, M[o] / 2 + 1))))
        return e;
    }
    if (loop && s->cfg.order == 4) {
      cudaError_t e = full(uf_scratch, n, n);
      if (e) return e;
    }
    std::vector<Lev2<T>> lv(k);
    for (int o = oa; o < k; o++) {
      lv[o].M = M[o];
      lv[o].cD = cD[o];
      lv[o].cA = cA[o];
      lv[o].rA = rAf[o];
      lv[o].vA = vAf[o];
      if (o + 1 < k) {
        lv[o].rD = rDf[o];
        lv[o].vD = vDf[o];
      }
    }
    void *q;
    cudaError_t e = dalloc(&q, sizeof(Lev2<T>) * k);
    if (e) return e;
    d_lev = (Lev2<T> *)q;
    h_lev = lv;
    return cudaMemcpy(d_lev, lv.data(), sizeof(Lev2<T>) * k, cudaMemcpyHostToDevice);
  }

  NormSink sink() const {
    return NormSink{hist_on(s) ? s->d_hist : nullptr, s->d_counter, kHistCap, s->sum_l2 ? s->d_l2 : nullptr};
  }
  size_t local_elems() const override { return loop ? 0 : (size_t)(R(0) + 4) * pitch; }
  bool extent(int64_t *l, int64_t *h, int64_t *g) const override {
    if (loop) return false;
    *l = lo(0, s->cfg.rank);
    *h = hi(0, s->cfg.rank);
    *g = 2;
    return true;
  }

  // ---- exchanges of an array family over the local ranks
  template <class GetPtr>
  cudaError_t xchg(int o, bool half, int g, cudaStream_t st, GetPtr get, int64_t pt) {
    std::vector<char *> p(nloc);
    std::vector<int> l(nloc), h(nloc);
    for (int i = 0; i < nloc; i++) {
      p[i] = (char *)get(i);
      l[i] = half ? lo(o, rk[i].q) / 2 : lo(o, rk[i].q);
      h[i] = half ? hi(o, rk[i].q) / 2 : hi(o, rk[i].q);
    }
    return comm->exchange(p, (size_t)pt * sizeof(T), l, h, g, st);
  }

  Rows2 rows_full(int o, int q) const {   // kernels whose output rows are A(s) rows of octave o
    Rows2 r;
    r.ylo = lo(o, q);
    r.yhi = hi(o, q);
    r.fy0 = lo(o, q) - 2;
    r.frows = R(o) + 4;
    r.hy0 = lo(o, q) / 2 - 2;
    r.hrows = R(o) / 2 + 4;
    return r;
  }
  Rows2 rows_half(int o, int q) const {   // kernels whose output rows are E/O (= A(2s)) rows of octave o
    Rows2 r;
    r.ylo = lo(o, q) / 2;
    r.yhi = hi(o, q) / 2;
    r.hy0 = lo(o, q) / 2 - 2;
    r.hrows = R(o) / 2 + 4;
    return r;
  }

  // Octaves >= oa on the full arrays (every NCCL rank; once in loopback), once
  // r_A(oa) is complete on every rank: the single-GPU pass sequence, octave
  // pairs fused (rest_dad, jac_ad) where both levels are full; ends with
  // v_A(oa) (the distributed ascent starts with jac_d of octave oa - 1).
  cudaError_t coarse_part(cudaStream_t st, Prof *prof) {
    const double w = sizeof(T);
    cudaError_t e;
    bool a_done = false;
    for (int o = oa; o < oc; o++) {
      if (!a_done) {
        STEP("rest_ad", 2 * o, 1, w * (Nl[2 * o] + Nl[2 * o + 1]));
        if ((e = fast2_rest_ad<T>(rAf[o], rDf[o], M[o], st))) return e;
      }
      a_done = o + 1 < oc;
      if (a_done) {
        STEP("rest_dad", 2 * o + 1, 1, w * (Nl[2 * o + 1] + Nl[2 * o + 2] + Nl[2 * o + 3]));
        if ((e = fast2_rest_dad<T>(rDf[o], rAf[o + 1], rDf[o + 1], M[o + 1], st, false))) return e;
      } else {
        STEP("rest_da", 2 * o + 1, 1, w * (Nl[2 * o + 1] + Nl[2 * o + 2]));
        if ((e = fast2_rest_da<T>(rDf[o], rAf[o + 1], M[o + 1], st))) return e;
      }
    }
    STEP("coarse", 2 * oc, 1, 0);
    launch2_coarse<T>(d_lev, oc, k, s->d_counter, st, h_lev.data());
    bool d_done = false;
    for (int o = oc - 1; o >= oa; o--) {
      if (!d_done) {
        STEP("jac_d", 2 * o + 1, 1, w * (Nl[2 * o + 2] + 2 * Nl[2 * o + 1]));
        if ((e = fast2_jac_d<T>(vAf[o + 1], rDf[o], vDf[o], M[o], cD[o], st))) return e;
      }
      d_done = o > oa;
      if (d_done) {
        STEP("jac_ad", 2 * o, 1, w * (Nl[2 * o + 1] + Nl[2 * o] + 2 * Nl[2 * o - 1]));
        if ((e = fast2_jac_ad<T>(vDf[o], rAf[o], cA[o], rDf[o - 1], vDf[o - 1], M[o - 1], cD[o - 1], st, false)))
          return e;
      } else {
        STEP("jac_a", 2 * o, 1, w * (Nl[2 * o + 1] + 2 * Nl[2 * o]));
        if ((e = fast2_jac_a<T>(vDf[o], rAf[o], vAf[o], M[o], cA[o], st))) return e;
      }
    }
    return cudaSuccess;
  }
  int coarse_launches() const {
    int c = 0;
    for (int o = oa; o < oc; o++) c += (o == oa) + 1;
    c += 1;
    for (int o = oc - 1; o >= oa; o--) c += (o == oc - 1) + 1;
    return c;
  }

  cudaError_t cycle(const std::vector<const T *> &uin, const std::vector<T *> &uout, const std::vector<const T *> &fe,
                    cudaStream_t st, Prof *prof) {
    const double w = sizeof(T);
    cudaError_t e;
    STEP("halo_u_f", 0, 0, 0);
    if ((e = xchg(0, false, 2, st, [&](int i) { return uin[i]; }, pitch))) return e;
    if ((e = xchg(0, false, 1, st, [&](int i) { return fe[i]; }, pitch))) return e;
    STEP("desc_fine", 0, nloc, w * (2 * Nl[0] + Nl[1]));
    for (int i = 0; i < nloc; i++)
      if ((e = fast2_desc_fine<T>(uin[i], fe[i], pitch, rk[i].rD[0], M[0], s->cfg.order, coef, sink(), st,
                                  rows_full(0, rk[i].q))))
        return e;
    for (int o = 0; o < oa; o++) {
      if (o >= 1) {
        STEP("rest_ad", 2 * o, nloc, w * (Nl[2 * o] + Nl[2 * o + 1]));
        if ((e = xchg(o, false, 1, st, [&](int i) { return rk[i].rA[o].p; }, rk[0].rA[o].pitch))) return e;
        for (int i = 0; i < nloc; i++)
          if ((e = fast2_rest_ad<T>(rk[i].rA[o], rk[i].rD[o], M[o], st, rows_full(o, rk[i].q)))) return e;
      }
      STEP("rest_da", 2 * o + 1, nloc, w * (Nl[2 * o + 1] + Nl[2 * o + 2]));
      if ((e = xchg(o, true, 1, st, [&](int i) { return rk[i].rD[o].o; }, rk[0].rD[o].pitch))) return e;
      for (int i = 0; i < nloc; i++) {
        const D2<T> &out = (o + 1 < oa) ? rk[i].rA[o + 1] : rAf[oa];
        if ((e = fast2_rest_da<T>(rk[i].rD[o], out, M[o + 1], st, rows_half(o, rk[i].q)))) return e;
      }
    }
    STEP("agglomerate", 2 * oa, 0, 0);
    if ((e = comm->allgather((char *)rAf[oa].p, rAf[oa].pitch * sizeof(T), lo(oa, rk[0].q), R(oa), sizeof(T), st)))
      return e;
    if ((e = coarse_part(st, prof))) return e;
    // ---- distributed ascent
    for (int o = oa - 1; o >= 0; o--) {
      STEP("jac_d", 2 * o + 1, nloc, w * (Nl[2 * o + 2] + 2 * Nl[2 * o + 1]));
      if (o + 1 < oa && (e = xchg(o + 1, false, 1, st, [&](int i) { return rk[i].vA[o + 1].p; }, rk[0].vA[o + 1].pitch)))
        return e;
      for (int i = 0; i < nloc; i++) {
        const D2<T> &vc = (o + 1 < oa) ? rk[i].vA[o + 1] : vAf[oa];
        if ((e = fast2_jac_d<T>(vc, rk[i].rD[o], rk[i].vD[o], M[o], cD[o], st, rows_half(o, rk[i].q)))) return e;
      }
      if ((e = xchg(o, true, 1, st, [&](int i) { return rk[i].vD[o].e; }, rk[0].vD[o].pitch)) ||
          (e = xchg(o, true, 1, st, [&](int i) { return rk[i].vD[o].o; }, rk[0].vD[o].pitch)))
        return e;
      if (o >= 1) {
        STEP("jac_a", 2 * o, nloc, w * (Nl[2 * o + 1] + 2 * Nl[2 * o]));
        for (int i = 0; i < nloc; i++)
          if ((e = fast2_jac_a<T>(rk[i].vD[o], rk[i].rA[o], rk[i].vA[o], M[o], cA[o], st, rows_full(o, rk[i].q))))
            return e;
      } else {
        STEP("asc_fine", 0, nloc, w * (Nl[1] + 3 * Nl[0]));
        for (int i = 0; i < nloc; i++)
          if ((e = fast2_asc_fine<T>(rk[i].vD[0], uin[i], fe[i], pitch, uout[i], M[0], s->cfg.order, cA[0], coef, st,
                                     rows_full(0, rk[i].q))))
            return e;
      }
    }
    return cudaSuccess;
  }

  // virtual global-row-0 pointer of a caller slab (NCCL mode)
  template <class P_>
  P_ *vg(P_ *ptr) const {
    return ptr - (int64_t)(lo(0, s->cfg.rank) - 2) * pitch;
  }

  void enqueue_cycle(const void *u_in, void *u_out, const void *f_eff, cudaStream_t st, Prof *prof) override {
    // NCCL mode: one local rank; the caller's arrays are slabs
    std::vector<const T *> ui{vg((const T *)u_in)}, fe{vg((const T *)f_eff)};
    std::vector<T *> uo{vg((T *)u_out)};
    status.note(cycle(ui, uo, fe, st, prof), comm.get(), "V-cycle");
  }
  int take_status(std::string *m) override { return status.take(m, comm.get()); }
  TransportStatus status;

  void enqueue_final_norm(void *u, const void *f_eff, cudaStream_t st) override {
    const T *ui = vg((const T *)u), *fe = vg((const T *)f_eff);
    status.note(xchg(0, false, 2, st, [&](int) { return ui; }, pitch), comm.get(), "halo exchange");
    status.note(xchg(0, false, 1, st, [&](int) { return fe; }, pitch), comm.get(), "halo exchange");
    fast2_desc_fine<T>(ui, fe, pitch, rk[0].rD[0], M[0], s->cfg.order, coef, sink(), st, rows_full(0, rk[0].q));
  }
  cudaError_t reduce_hist(unsigned long long *d, int nslots, cudaStream_t st) override {
    cudaError_t e = comm->allreduce_max_u64(d, nslots, st);
    return e ? e : comm->allreduce_sum_f64(s->d_l2, nslots, st);
  }
  // f~ (order 4) on the slab: f's ghost row first, then the own rows
  void enqueue_ftilde(const void *f, void *ft, cudaStream_t st, int64_t) override {
    if (loop) {
      launch2_ftilde<T>(D2<const T>{(const T *)f, pitch}, D2<T>{(T *)ft, pitch}, M[0], st);
      return;
    }
    const T *fv = vg((const T *)f);
    status.note(xchg(0, false, 1, st, [&](int) { return fv; }, pitch), comm.get(), "halo exchange");
    launch2_ftilde_rows<T>(D2<const T>{fv, pitch}, D2<T>{vg((T *)ft), pitch}, M[0], lo(0, rk[0].q), hi(0, rk[0].q), st);
  }
  void enqueue_residual(const void *u, const void *f, void *r, cudaStream_t st, int64_t) override {
    if (loop) {
      launch2_residual<T>(D2<const T>{(const T *)u, pitch}, D2<const T>{(const T *)f, pitch}, D2<T>{(T *)r, pitch},
                          M[0], s->cfg.order, coef, st);
      return;
    }
    const T *uv = vg((const T *)u), *fv = vg((const T *)f);
    status.note(xchg(0, false, 1, st, [&](int) { return uv; }, pitch), comm.get(), "halo exchange");
    launch2_residual_rows<T>(D2<const T>{uv, pitch}, D2<const T>{fv, pitch}, D2<T>{vg((T *)r), pitch}, M[0],
                             s->cfg.order, coef, lo(0, rk[0].q), hi(0, rk[0].q), st);
  }
  void enqueue_norm(const void *x, unsigned long long *mx, double *ss, cudaStream_t st, int64_t) override {
    if (loop) {
      launch2_norm<T>(D2<const T>{(const T *)x, pitch}, M[0], mx, ss, st);
      return;
    }
    launch2_norm_rows<T>(D2<const T>{vg((const T *)x), pitch}, M[0], lo(0, rk[0].q), hi(0, rk[0].q), mx, ss, st);
    status.note(comm->allreduce_max_u64(mx, 1, st), comm.get(), "norm all-reduce");
    status.note(comm->allreduce_sum_f64(ss, 1, st), comm.get(), "norm all-reduce");
  }
  int launches_per_cycle() const override {
    int c = nloc;   // desc
    for (int o = 0; o < oa; o++) c += ((o >= 1) + 1) * nloc;
    c += coarse_launches();
    for (int o = oa - 1; o >= 0; o--) c += 2 * nloc;
    return c;
  }

  // ---- loopback: the whole mg_vcycle on full caller arrays
  int vcycle_all(mg_solver *sv, void *u, const void *f, int ncycles, double *res_hist) override {
    if (!loop) return 1;
    cudaStream_t st = sv->st;
    const size_t pb = pitch * sizeof(T);
    const T *fsrc = (const T *)f;
    if (s->cfg.order == 4) {
      launch2_ftilde<T>(D2<const T>{(const T *)f, pitch}, uf_scratch, M[0], st);
      fsrc = uf_scratch.p;
    }
    // scatter: rows [lo-2, hi+2) clipped to the grid
    for (int i = 0; i < nloc; i++) {
      int a = std::max(lo(0, i) - 2, 0), b = std::min(hi(0, i) + 2, (int)n);
      for (int j = 0; j < 2; j++) cudaMemsetAsync(rk[i].u[j].p + (int64_t)(lo(0, i) - 2) * pitch, 0, (R(0) + 4) * pb, st);
      cudaMemsetAsync(rk[i].f.p + (int64_t)(lo(0, i) - 2) * pitch, 0, (R(0) + 4) * pb, st);
      cudaMemcpyAsync(rk[i].u[0].p + (int64_t)a * pitch, (const T *)u + (int64_t)a * pitch, (b - a) * pb,
                      cudaMemcpyDeviceToDevice, st);
      cudaMemcpyAsync(rk[i].f.p + (int64_t)a * pitch, fsrc + (int64_t)a * pitch, (b - a) * pb, cudaMemcpyDeviceToDevice,
                      st);
    }
    int nslots = ncycles + 1 < kHistCap ? ncycles + 1 : kHistCap;
    clear_hist(sv, nslots, st);
    cudaMemsetAsync(sv->d_counter, 0, sizeof(int), st);
    std::vector<const T *> fe(nloc);
    for (int i = 0; i < nloc; i++) fe[i] = rk[i].f.p;
    int cur = 0;
    for (int c = 0; c < ncycles; c++) {
      std::vector<const T *> ui(nloc);
      std::vector<T *> uo(nloc);
      for (int i = 0; i < nloc; i++) {
        ui[i] = rk[i].u[cur].p;
        uo[i] = rk[i].u[cur ^ 1].p;
      }
      cudaError_t e = cycle(ui, uo, fe, st, nullptr);
      if (e) return fail(sv, MG_ECUDA, std::string("loopback cycle: ") + cudaGetErrorString(e));
      cur ^= 1;
    }
    if (res_hist) {
      std::vector<const T *> ui(nloc);
      for (int i = 0; i < nloc; i++) ui[i] = rk[i].u[cur].p;
      xchg(0, false, 2, st, [&](int i) { return ui[i]; }, pitch);
      xchg(0, false, 1, st, [&](int i) { return fe[i]; }, pitch);
      for (int i = 0; i < nloc; i++)
        fast2_desc_fine<T>(ui[i], fe[i], pitch, rk[i].rD[0], M[0], s->cfg.order, coef, sink(), st, rows_full(0, i));
    }
    // gather own rows back
    for (int i = 0; i < nloc; i++)
      cudaMemcpyAsync((T *)u + (int64_t)lo(0, i) * pitch, rk[i].u[cur].p + (int64_t)lo(0, i) * pitch, R(0) * pb,
                      cudaMemcpyDeviceToDevice, st);
    CKS(sv, cudaGetLastError());
    if (res_hist) return read_hist(sv, ncycles, res_hist, st);
    return MG_OK;
  }
};

// ============================================================== Dist2CA
// Communication-avoiding variant ("one u-exchange per cycle"):
// every rank keeps full-size level arrays and computes each distributed level
// on its own rows plus a level-dependent band of ghost rows, redundantly, so
// that a V-cycle needs ONE halo exchange of u (Gu rows per side) and the
// all-gather of the agglomeration level r_A(oa), instead of one exchange per
// level and colour.  The bands follow from the stencils' reach (derived in
// DESIGN.md 8): the ascent's A(1) output is the own rows; a D(s) level output
// band w needs v_A(2s) on w + 2s and r_D(s) on w + s; an A(s) band w needs
// v_D(s) on w + 2s and r_A(s) on w + s; the descent's bands cover both the
// ascent's r needs and the next restriction's reach (+s per step).  At 8193^2
// over 8 ranks (agglomeration at A(16)) Gu = 108 fine rows (1024 owned).  The node formulas are those of
// the single-GPU kernels (the same kernels, on row windows), so the iterate is
// bit-identical to the single-GPU solver (tests/test_gpu_dist.py).
// Used when Gu fits in one neighbour's slab (Gu <= rows per rank); otherwise
// (thin slabs, deep agglomeration) the per-level schedule of Dist2 runs.
template <class T>
struct Dist2CA : Dist2<T> {
  using B = Dist2<T>;
  using B::comm;
  using B::k;
  using B::loop;
  using B::M;
  using B::n;
  using B::nloc;
  using B::oa;
  using B::pitch;
  using B::rk;
  using B::s;
  bool ca = false;
  bool fused = !env_flag("MG_DIST_NOFUSE");   // octave-pair passes on the bands (MG_DIST_NOFUSE=1: level passes)
  int Gu = 0;
  std::vector<int> WD, WA, waD, waA;   // bands (fine rows): descent r_D / r_A, ascent v_D / v_A
  struct Full {
    D2<T> u[2], f, ft;
    std::vector<S2<T>> rD, vD;   // octaves o < oa
    std::vector<D2<T>> rA, vA;   // 1 <= o < oa
  };
  std::vector<Full> fl;   // per local rank
  cudaGraphExec_t gexec[2][4] = {};   // the cycle u[p] -> u[p^1], [p][L2 sums on | history on]

  Dist2CA(mg_solver *sv, bool loopback) : B(sv, loopback) {}
  ~Dist2CA() override {
    for (auto &gp : gexec)
      for (auto &g : gp)
        if (g) cudaGraphExecDestroy(g);
  }

  static int up(int v, int m) { return (v + m - 1) / m * m; }
  void plan() { Gu = slab_bands_2d(oa, WD, WA, waD, waA); }

  cudaError_t alloc() override {
    cudaError_t e = B::alloc();
    if (e) return e;
    plan();
    ca = !env_flag("MG_DIST_PERLEVEL") && oa >= 1 && Gu <= B::R(0);
    if (!ca) return cudaSuccess;
    fl.resize(nloc);
    const int64_t nn = n;
    for (int i = 0; i < nloc; i++) {
      Full &F = fl[i];
      void *q;
      for (D2<T> *d : {&F.u[0], &F.u[1], &F.f}) {
        if ((e = B::dalloc(&q, sizeof(T) * nn * pitch))) return e;
        *d = D2<T>{(T *)q, pitch};
      }
      if (s->cfg.order == 4) {
        if ((e = B::dalloc(&q, sizeof(T) * nn * pitch))) return e;
        F.ft = D2<T>{(T *)q, pitch};
      }
      F.rD.resize(oa);
      F.vD.resize(oa);
      F.rA.resize(oa);
      F.vA.resize(oa);
      for (int o = 0; o < oa; o++) {
        const int64_t H = M[o] / 2 + 1, ph = B::pitch_for(H);
        for (S2<T> *d : {&F.rD[o], &F.vD[o]}) {
          void *ee, *oo;
          if ((e = B::dalloc(&ee, sizeof(T) * H * ph)) || (e = B::dalloc(&oo, sizeof(T) * H * ph))) return e;
          *d = S2<T>{(T *)ee, (T *)oo, ph};
        }
        if (o >= 1) {
          const int64_t Wd = M[o] + 1, pa = B::pitch_for(Wd);
          for (D2<T> *d : {&F.rA[o], &F.vA[o]}) {
            if ((e = B::dalloc(&q, sizeof(T) * Wd * pa))) return e;
            *d = D2<T>{(T *)q, pa};
          }
        }
      }
    }
    return cudaSuccess;
  }

  // row window of a level: fine rows [lo - W, hi + W) of rank q in units of u
  // fine rows, clipped to [0, top)
  Rows2 win(int q, int W, int unit, int top) const {
    Rows2 r;
    r.ylo = std::max(0, (B::lo(0, q) - W) / unit);
    r.yhi = std::min(top, (B::hi(0, q) + W) / unit);
    return r;
  }
  const T *fe(int i) const { return s->cfg.order == 4 ? fl[i].ft.p : fl[i].f.p; }
  // the residual-norm sink of rank q: the L2 sum counts its own rows only (the
  // ghost bands' residuals are the neighbours' own rows)
  NormSink own_sink(int q) const {
    NormSink ns = B::sink();
    ns.nlo = B::lo(0, q);
    ns.nhi = B::hi(0, q);
    return ns;
  }

  // one V-cycle on the internal arrays, u[cur] -> u[cur ^ 1]
  cudaError_t cycle_ca(int cur, cudaStream_t st, Prof *prof) {
    const double w = sizeof(T);
    auto &Nl = B::Nl;
    const auto &cD = B::cD;
    const auto &cA = B::cA;
    const auto &coef = B::coef;
    cudaError_t e;
    STEP("halo_u", 0, 0, 0);
    if ((e = B::xchg(0, false, Gu, st, [&](int i) { return fl[i].u[cur].p; }, pitch))) return e;
    STEP("desc_fine", 0, nloc, w * (2 * Nl[0] + Nl[1]));
    for (int i = 0; i < nloc; i++)
      if ((e = fast2_desc_fine<T>(fl[i].u[cur].p, fe(i), pitch, fl[i].rD[0], M[0], s->cfg.order, coef,
                                  own_sink(rk[i].q), st, win(rk[i].q, WD[0], 1, M[0]))))
        return e;
    // the octave-pair passes of the single-GPU cycle on row bands:
    // rest_dad = rest_da(o) + rest_ad(o+1) on A(o+1)'s band, jac_ad = jac_a(o) +
    // jac_d(o-1) on D(o-1)'s band (rounded out to an even first row; the extra
    // rows are never read)
    bool a_done = false;
    for (int o = 0; o < oa; o++) {
      const int s_ = 1 << o;
      if (o >= 1 && !a_done) {
        STEP("rest_ad", 2 * o, nloc, w * (Nl[2 * o] + Nl[2 * o + 1]));
        for (int i = 0; i < nloc; i++)
          if ((e = fast2_rest_ad<T>(fl[i].rA[o], fl[i].rD[o], M[o], st, win(rk[i].q, WD[o], s_, M[o])))) return e;
      }
      a_done = false;
      if (o + 1 < oa && fused) {
        STEP("rest_dad", 2 * o + 1, nloc, w * (Nl[2 * o + 1] + Nl[2 * o + 2] + Nl[2 * o + 3]));
        const int band = std::max(WA[o + 1], WD[o + 1]);
        for (int i = 0; i < nloc; i++) {
          const Rows2 r = win(rk[i].q, band, 2 * s_, M[o + 1] + 1);
          if ((e = fast2_rest_dad<T>(fl[i].rD[o], fl[i].rA[o + 1], fl[i].rD[o + 1], M[o + 1], st, false, r.ylo,
                                     r.yhi)))
            return e;
        }
        a_done = true;
        continue;
      }
      STEP("rest_da", 2 * o + 1, nloc, w * (Nl[2 * o + 1] + Nl[2 * o + 2]));
      for (int i = 0; i < nloc; i++) {
        const D2<T> &out = (o + 1 < oa) ? fl[i].rA[o + 1] : B::rAf[oa];
        if ((e = fast2_rest_da<T>(fl[i].rD[o], out, M[o + 1], st, win(rk[i].q, WA[o + 1], 2 * s_, M[o + 1]))))
          return e;
      }
    }
    STEP("agglomerate", 2 * oa, 0, 0);
    if ((e = comm->allgather((char *)B::rAf[oa].p, B::rAf[oa].pitch * sizeof(T), B::lo(oa, rk[0].q), B::R(oa),
                             sizeof(T), st)))
      return e;
    if ((e = B::coarse_part(st, prof))) return e;
    bool d_done = false;
    for (int o = oa - 1; o >= 0; o--) {
      const int s_ = 1 << o;
      if (!d_done) {
        STEP("jac_d", 2 * o + 1, nloc, w * (Nl[2 * o + 2] + 2 * Nl[2 * o + 1]));
        for (int i = 0; i < nloc; i++) {
          const D2<T> &vc = (o + 1 < oa) ? fl[i].vA[o + 1] : B::vAf[oa];
          if ((e = fast2_jac_d<T>(vc, fl[i].rD[o], fl[i].vD[o], M[o], cD[o], st,
                                  win(rk[i].q, waD[o], 2 * s_, M[o] / 2))))
            return e;
        }
      }
      d_done = false;
      if (o >= 1 && fused) {
        STEP("jac_ad", 2 * o, nloc, w * (Nl[2 * o + 1] + Nl[2 * o] + 2 * Nl[2 * o - 1]));
        for (int i = 0; i < nloc; i++) {
          const Rows2 r = win(rk[i].q, up(waD[o - 1], 2 * s_), s_, M[o - 1] / 2 + 1);
          if ((e = fast2_jac_ad<T>(fl[i].vD[o], fl[i].rA[o], cA[o], fl[i].rD[o - 1], fl[i].vD[o - 1], M[o - 1],
                                   cD[o - 1], st, false, r.ylo, r.yhi)))
            return e;
        }
        d_done = true;
      } else if (o >= 1) {
        STEP("jac_a", 2 * o, nloc, w * (Nl[2 * o + 1] + 2 * Nl[2 * o]));
        for (int i = 0; i < nloc; i++)
          if ((e = fast2_jac_a<T>(fl[i].vD[o], fl[i].rA[o], fl[i].vA[o], M[o], cA[o], st,
                                  win(rk[i].q, waA[o], s_, M[o]))))
            return e;
      } else {
        STEP("asc_fine", 0, nloc, w * (Nl[1] + 3 * Nl[0]));
        for (int i = 0; i < nloc; i++)
          if ((e = fast2_asc_fine<T>(fl[i].vD[0], fl[i].u[cur].p, fe(i), pitch, fl[i].u[cur ^ 1].p, M[0],
                                     s->cfg.order, cA[0], coef, st, win(rk[i].q, 0, 1, M[0]))))
            return e;
      }
    }
    return cudaSuccess;
  }

  int launches_per_cycle() const override {
    if (!ca) return B::launches_per_cycle();
    int c = nloc;   // desc_fine
    if (fused)      // rest_dad for o < oa-1, rest_da at oa-1; jac_d at oa-1, jac_ad for o >= 1, asc_fine
      c += oa * nloc + B::coarse_launches() + (1 + (oa - 1) + 1) * nloc;
    else
      c += (2 * oa - 1) * nloc + B::coarse_launches() + 2 * oa * nloc;
    return c;
  }

  // the caller's rows [lo, hi) of rank i: full arrays (loopback) or the slab (row 2 = lo)
  T *caller_row0(void *a, int i) const {
    return loop ? (T *)a : (T *)a - (int64_t)(B::lo(0, rk[i].q) - 2) * pitch;
  }

  // one cycle, captured once per parity into a CUDA graph (NCCL calls and the
  // loopback copies are capturable) and replayed
  int run_graph(mg_solver *sv, int cur) {
    cudaStream_t st = sv->st;
    cudaGraphExec_t &gx = gexec[cur][(s->sum_l2 ? 1 : 0) | (s->want_hist ? 2 : 0)];
    if (!gx) {
      cudaGraph_t g = nullptr;
      CKS(sv, cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
      cudaError_t e = cycle_ca(cur, st, nullptr);
      cudaError_t e2 = cudaStreamEndCapture(st, &g);
      if (e || e2) {
        if (g) cudaGraphDestroy(g);
        TransportStatus ts;
        ts.note(e ? e : e2, comm.get(), "slab cycle capture");
        std::string m;
        const int code = ts.take(&m, nullptr);
        return fail(sv, code, m);
      }
      e = cudaGraphInstantiate(&gx, g, 0);
      cudaGraphDestroy(g);
      CKS(sv, e);
    }
    CKS(sv, cudaGraphLaunch(gx, st));
    return MG_OK;
  }

  int vcycle_all(mg_solver *sv, void *u, const void *f, int ncycles, double *res_hist) override {
    if (!ca) return B::vcycle_all(sv, u, f, ncycles, res_hist);
    cudaStream_t st = sv->st;
    const size_t pb = pitch * sizeof(T);
    // caller rows in, then the deep halos of u and f (once per call)
    for (int i = 0; i < nloc; i++) {
      const int l = B::lo(0, rk[i].q), h = B::hi(0, rk[i].q);
      CKS(sv, cudaMemcpyAsync(fl[i].u[0].p + (int64_t)l * pitch, caller_row0(u, i) + (int64_t)l * pitch, (h - l) * pb,
                              cudaMemcpyDeviceToDevice, st));
      CKS(sv, cudaMemcpyAsync(fl[i].f.p + (int64_t)l * pitch, caller_row0(const_cast<void *>(f), i) + (int64_t)l * pitch,
                              (h - l) * pb, cudaMemcpyDeviceToDevice, st));
    }
    {
      TransportStatus ts;
      ts.note(B::xchg(0, false, Gu, st, [&](int i) { return fl[i].f.p; }, pitch), comm.get(), "halo exchange of f");
      std::string m;
      if (int code = ts.take(&m, nullptr)) return fail(sv, code, m);
    }
    if (s->cfg.order == 4)
      for (int i = 0; i < nloc; i++)   // f~ on the band the finest descent reads (f known on Gu rows)
        launch2_ftilde_rows<T>(D2<const T>{fl[i].f.p, pitch}, fl[i].ft, M[0],
                               std::max(1, B::lo(0, rk[i].q) - Gu + 1), std::min(M[0], B::hi(0, rk[i].q) + Gu - 1), st);
    const int nslots = ncycles + 1;
    CKS(sv, clear_hist(sv, nslots, st));
    CKS(sv, cudaMemsetAsync(sv->d_counter, 0, sizeof(int), st));
    int cur = 0;
    for (int c = 0; c < ncycles; c++) {
      int rc = run_graph(sv, cur);
      if (rc) return rc;
      cur ^= 1;
    }
    if (res_hist) {   // ||f - L u||_inf after the last cycle: the finest descent on the own rows
      TransportStatus ts;
      ts.note(B::xchg(0, false, 2, st, [&](int i) { return fl[i].u[cur].p; }, pitch), comm.get(), "halo exchange");
      for (int i = 0; i < nloc; i++)
        ts.note(fast2_desc_fine<T>(fl[i].u[cur].p, fe(i), pitch, fl[i].rD[0], M[0], s->cfg.order, B::coef,
                                   own_sink(rk[i].q), st, win(rk[i].q, 0, 1, M[0])),
                nullptr, "final residual");
      ts.note(B::reduce_hist(sv->d_hist, nslots, st), comm.get(), "norm all-reduce");
      std::string m;
      if (int code = ts.take(&m, nullptr)) return fail(sv, code, m);
    }
    for (int i = 0; i < nloc; i++) {
      const int l = B::lo(0, rk[i].q), h = B::hi(0, rk[i].q);
      CKS(sv, cudaMemcpyAsync(caller_row0(u, i) + (int64_t)l * pitch, fl[i].u[cur].p + (int64_t)l * pitch, (h - l) * pb,
                              cudaMemcpyDeviceToDevice, st));
    }
    CKS(sv, cudaGetLastError());
    if (res_hist) return read_hist(sv, ncycles, res_hist, st);
    return MG_OK;
  }
};

// factory used by mg_create_ex
ImplBase *make_dist2(mg_solver *s, bool loopback, std::string *err) {
  Comm2 *c = loopback ? make_loop_comm(s->cfg.nranks)
                      : make_nccl_comm(s->cfg.nranks, s->cfg.rank, s->cfg.nccl_id, s->esz, err);
  if (!c) return nullptr;
  if (s->cfg.dtype == MG_F64) {
    auto *d = new Dist2CA<double>(s, loopback);
    d->comm.reset(c);
    return d;
  }
  auto *d = new Dist2CA<float>(s, loopback);
  d->comm.reset(c);
  return d;
}
