// dist3.cu -- the 3D V-cycle on z-slabs over several ranks.
//
// Rank q owns the G(s) planes [q M_s/P, (q+1) M_s/P) of octave s, and with
// them the half-index planes [lo/2, hi/2) of that octave's parity
// sublattices (R(s): C, Fx, Fy, Fz; M(s): C, B), while M_s/P >= 4 and G(s)
// has at least agglom_points interior nodes.  Every slab array carries 2
// ghost planes on each side and is addressed through a virtual global-plane-0
// pointer, so the kernels of k3f.cu / k3l.cu run unchanged on a plane range.
// Before each kernel the ghost planes it reads are refreshed (1 half-plane of
// a sublattice, or 1-2 fine planes; the reach of every stencil is listed at
// the exchange).  At the first agglomerated octave oa, r_G(2^oa) is
// all-gathered and every rank runs the coarse octaves redundantly, so the
// ascent needs no gather back.  Transports: comm.cu (NCCL or loopback).
#include "comm.h"
#include "solver.h"

template <class T>
struct Dist3 : ImplBase {
  mg_solver *s;
  int k, P, nloc;   // nloc = local (virtual) ranks: P in loopback, 1 with NCCL
  bool loop;
  int64_t n, pitch;
  std::unique_ptr<Comm2> comm;
  int oa = 1, oc = 1;
  std::vector<int> M;
  std::vector<T> cMg, cR1, cR2, cG;
  Coef<T> coef{};
  struct Rk {
    int q;
    std::vector<S3<T>> rR, vR, rM, vM;   // octaves o < oa
    std::vector<D3<T>> rG, vG;           // 1 <= o < oa
    D3<T> u[2], f;                       // loopback: internal slabs of u (pair) and f / f~
  };
  std::vector<Rk> rk;
  std::vector<S3<T>> rRf, vRf, rMf, vMf;   // full arrays, octaves o >= oa
  std::vector<D3<T>> rGf, vGf;
  D3<T> ft_full{};                         // loopback: full f~ (order 4)
  Lev3<T> *d_lev = nullptr;

  Dist3(mg_solver *sv, bool loopback) : s(sv), k(sv->k), P(sv->cfg.nranks), loop(loopback), n(sv->cfg.n),
                                        pitch(sv->pitch) {
    nloc = loop ? P : 1;
  }
  bool fast() const override { return true; }
  int64_t pitch_for(int64_t cnt) const { return round_up(cnt, 128 / (int64_t)sizeof(T)); }
  int R(int o) const { return M[o] / P; }   // G(s) planes per rank at octave o
  int lo(int o, int q) const { return q * R(o); }
  int hi(int o, int q) const { return (q + 1) * R(o); }
  int64_t fplane() const { return pitch * n; }

  // dense slab of planes [lo-2, hi+2), W x W per plane: virtual plane-0 pointer
  cudaError_t slab(D3<T> &out, int64_t W, int lo_, int hi_) {
    int64_t pt = pitch_for(W), pl = pt * W;
    void *q;
    cudaError_t e = dalloc(&q, sizeof(T) * pl * (hi_ - lo_ + 4));
    if (e) return e;
    out = D3<T>{(T *)q - (int64_t)(lo_ - 2) * pl, pt, pl};
    return cudaSuccess;
  }
  // sublattice slab (H x H per half-plane) of the listed parities
  cudaError_t slab_s(S3<T> &out, int64_t H, int lo_, int hi_, std::initializer_list<int> parities) {
    int64_t ph = pitch_for(H), pl = ph * H;
    out = S3<T>{};
    out.pitch = ph;
    out.plane = pl;
    for (int par : parities) {
      void *q;
      cudaError_t e = dalloc(&q, sizeof(T) * pl * (hi_ - lo_ + 4));
      if (e) return e;
      out.s[par] = (T *)q - (int64_t)(lo_ - 2) * pl;
    }
    return cudaSuccess;
  }

  cudaError_t alloc() override {
    const double pm = s->cfg.p[0], pr1 = s->cfg.p[1], pr2 = s->cfg.p[2], pg = s->cfg.p[3];
    M.resize(k);
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
    coef.invh2 = (T)((double)(n - 1) * (double)(n - 1));
    coef.c6 = (T)((double)(n - 1) * (double)(n - 1) / 6.0);
    int64_t ag = s->cfg.agglom_points > 0 ? s->cfg.agglom_points : (int64_t(1) << 18);
    oa = slab_agglom_octave(n, k, P, ag, 3);
    int thresh = 16;
    if (const char *e = getenv("MG_COARSE_M3")) thresh = atoi(e);
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
      r.rR.resize(oa);
      r.vR.resize(oa);
      r.rM.resize(oa);
      r.vM.resize(oa);
      r.rG.resize(oa);
      r.vG.resize(oa);
      for (int o = 0; o < oa; o++) {
        int H = M[o] / 2 + 1, l = lo(o, r.q) / 2, h = hi(o, r.q) / 2;
        cudaError_t e;
        if ((e = slab_s(r.rR[o], H, l, h, {0, 6, 5, 3})) || (e = slab_s(r.vR[o], H, l, h, {0, 6, 5, 3})) ||
            (e = slab_s(r.rM[o], H, l, h, {0, 7})) || (e = slab_s(r.vM[o], H, l, h, {0, 7})))
          return e;
        if (o >= 1 && ((e = slab(r.rG[o], M[o] + 1, lo(o, r.q), hi(o, r.q))) ||
                       (e = slab(r.vG[o], M[o] + 1, lo(o, r.q), hi(o, r.q)))))
          return e;
      }
      if (loop) {
        // caller-shaped slabs: n x pitch rows per plane
        for (D3<T> *d : {&r.u[0], &r.u[1], &r.f}) {
          void *q;
          cudaError_t e = dalloc(&q, sizeof(T) * fplane() * (R(0) + 4));
          if (e) return e;
          *d = D3<T>{(T *)q - (int64_t)(lo(0, r.q) - 2) * fplane(), pitch, fplane()};
        }
      }
    }
    rRf.resize(k);
    vRf.resize(k);
    rMf.resize(k);
    vMf.resize(k);
    rGf.resize(k);
    vGf.resize(k);
    for (int o = oa; o < k; o++) {
      cudaError_t e;
      if ((e = slab(rGf[o], M[o] + 1, 0, M[o] + 1)) || (e = slab(vGf[o], M[o] + 1, 0, M[o] + 1))) return e;
      if (o + 1 < k) {
        int H = M[o] / 2 + 1;
        if ((e = slab_s(rRf[o], H, 0, H, {0, 6, 5, 3})) || (e = slab_s(vRf[o], H, 0, H, {0, 6, 5, 3})) ||
            (e = slab_s(rMf[o], H, 0, H, {0, 7})) || (e = slab_s(vMf[o], H, 0, H, {0, 7})))
          return e;
      }
    }
    if (loop && s->cfg.order == 4) {
      void *q;
      cudaError_t e = dalloc(&q, sizeof(T) * fplane() * n);
      if (e) return e;
      ft_full = D3<T>{(T *)q, pitch, fplane()};
    }
    std::vector<Lev3<T>> lv(k);
    for (int o = oa; o < k; o++) {
      lv[o].M = M[o];
      lv[o].cMg = cMg[o];
      lv[o].cR1 = cR1[o];
      lv[o].cR2 = cR2[o];
      lv[o].cG = cG[o];
      lv[o].rG = rGf[o];
      lv[o].vG = vGf[o];
      if (o + 1 < k) {
        lv[o].rR = rRf[o];
        lv[o].vR = vRf[o];
        lv[o].rM = rMf[o];
        lv[o].vM = vMf[o];
      }
    }
    void *q;
    cudaError_t e = dalloc(&q, sizeof(Lev3<T>) * k);
    if (e) return e;
    d_lev = (Lev3<T> *)q;
    return cudaMemcpy(d_lev, lv.data(), sizeof(Lev3<T>) * k, cudaMemcpyHostToDevice);
  }

  NormSink sink() const {
    return NormSink{hist_on(s) ? s->d_hist : nullptr, s->d_counter, kHistCap, s->sum_l2 ? s->d_l2 : nullptr};
  }
  size_t local_elems() const override { return loop ? 0 : (size_t)(R(0) + 4) * fplane(); }
  bool extent(int64_t *l, int64_t *h, int64_t *g) const override {
    if (loop) return false;
    *l = lo(0, s->cfg.rank);
    *h = hi(0, s->cfg.rank);
    *g = 2;
    return true;
  }

  // ---- exchanges: one array (a plane family) over the local ranks
  template <class GetPtr>
  cudaError_t xchg(int o, bool half, int g, cudaStream_t st, GetPtr get, int64_t plane_elems) {
    std::vector<char *> p(nloc);
    std::vector<int> l(nloc), h(nloc);
    for (int i = 0; i < nloc; i++) {
      p[i] = (char *)get(i);
      l[i] = half ? lo(o, rk[i].q) / 2 : lo(o, rk[i].q);
      h[i] = half ? hi(o, rk[i].q) / 2 : hi(o, rk[i].q);
    }
    return comm->exchange(p, (size_t)plane_elems * sizeof(T), l, h, g, st);
  }
  // the listed parity arrays of a sublattice family, 1 half-plane
  cudaError_t xchg_s(int o, cudaStream_t st, std::vector<S3<T>> Rk::*fam, std::initializer_list<int> pars) {
    for (int par : pars) {
      cudaError_t e = xchg(o, true, 1, st, [&](int i) { return (rk[i].*fam)[o].s[par]; }, (rk[0].*fam)[o].plane);
      if (e) return e;
    }
    return cudaSuccess;
  }
  cudaError_t xchg_g(int o, cudaStream_t st, std::vector<D3<T>> Rk::*fam) {
    return xchg(o, false, 1, st, [&](int i) { return (rk[i].*fam)[o].p; }, (rk[0].*fam)[o].plane);
  }
  ZRange3 zr_fine(int q) const {
    ZRange3 z;
    z.zlo = lo(0, q);
    z.zhi = hi(0, q);
    z.fz0 = lo(0, q) - 2;
    z.fplanes = R(0) + 4;
    z.hz0 = lo(0, q) / 2 - 2;
    z.hplanes = R(0) / 2 + 4;
    return z;
  }
  int c0(int o, int q) const { return lo(o, q) / 2; }
  int c1(int o, int q) const { return hi(o, q) / 2; }

  cudaError_t cycle(const std::vector<const T *> &uin, const std::vector<T *> &uout, const std::vector<const T *> &fe,
                    cudaStream_t st, Prof *prof) {
    const double w = sizeof(T);
    const int L = 3 * k - 2;
    cudaError_t e;
    // ---- finest descent: r0 from u (2-plane reach) and f (1 plane)
    STEP("halo_u_f", 0, 0, 0);
    if ((e = xchg(0, false, 2, st, [&](int i) { return uin[i]; }, fplane()))) return e;
    if ((e = xchg(0, false, 1, st, [&](int i) { return fe[i]; }, fplane()))) return e;
    STEP("desc_fine", 0, nloc, w * (2 * Nl[0] + Nl[1]));
    for (int i = 0; i < nloc; i++)
      if ((e = fast3_desc_fine<T>(uin[i], fe[i], pitch, rk[i].rR[0], M[0], s->cfg.order, coef, sink(), st,
                                  zr_fine(rk[i].q))))
        return e;
    for (int o = 0; o < oa; o++) {
      const int g = 3 * o;
      if (o >= 1) {   // Erred reads r_G(s) at z +- 1
        STEP("rest_gr", g, nloc, w * (Nl[g] + Nl[g + 1]));
        if ((e = xchg_g(o, st, &Rk::rG))) return e;
        for (int i = 0; i < nloc; i++) lv3_rest_gr<T>(rk[i].rG[o], rk[i].rR[o], M[o], st, c0(o, rk[i].q), c1(o, rk[i].q));
      }
      // Ermagc reads Fx, Fy at c-1; Ermagm reads Fz at c+1
      STEP("rest_rm", g + 1, nloc, w * (Nl[g + 1] + Nl[g + 2]));
      if ((e = xchg_s(o, st, &Rk::rR, {6, 5, 3}))) return e;
      for (int i = 0; i < nloc; i++) lv3_rest_rm<T>(rk[i].rR[o], rk[i].rM[o], M[o], st, c0(o, rk[i].q), c1(o, rk[i].q));
      // Erblu reads B at c-1
      STEP("rest_mg", g + 2, nloc, w * (Nl[g + 2] + Nl[g + 3]));
      if ((e = xchg_s(o, st, &Rk::rM, {7}))) return e;
      for (int i = 0; i < nloc; i++) {
        const D3<T> &out = (o + 1 < oa) ? rk[i].rG[o + 1] : rGf[oa];
        lv3_rest_mg<T>(rk[i].rM[o], out, M[o + 1], st, c0(o, rk[i].q), c1(o, rk[i].q));
      }
    }
    STEP("agglomerate", 3 * oa, 0, 0);
    if ((e = comm->allgather((char *)rGf[oa].p, rGf[oa].plane * sizeof(T), lo(oa, rk[0].q), R(oa), sizeof(T), st)))
      return e;
    // ---- coarse octaves on full arrays (every NCCL rank; once in loopback)
    for (int o = oa; o < oc; o++) {
      const int g = 3 * o;
      STEP("rest_gr", g, 1, w * (Nl[g] + Nl[g + 1]));
      lv3_rest_gr<T>(rGf[o], rRf[o], M[o], st);
      STEP("rest_rm", g + 1, 1, w * (Nl[g + 1] + Nl[g + 2]));
      lv3_rest_rm<T>(rRf[o], rMf[o], M[o], st);
      STEP("rest_mg", g + 2, 1, w * (Nl[g + 2] + Nl[g + 3]));
      lv3_rest_mg<T>(rMf[o], rGf[o + 1], M[o + 1], st);
    }
    {
      double b = 0;
      for (int l = 3 * oc; l < L; l++) b += 5 * Nl[l];
      b -= Nl[L - 1] + 2 * Nl[3 * oc];
      STEP("coarse", 3 * oc, 1, w * b);
    }
    lv3_coarse<T>(d_lev, oc, k, s->d_counter, st);
    for (int o = oc - 1; o >= oa; o--) {
      const int g = 3 * o;
      STEP("jac_m", g + 2, 2, w * (Nl[g + 3] + 2 * Nl[g + 2]));
      lv3_jac_m<T>(vGf[o + 1], rMf[o], vMf[o], M[o], cMg[o], st);
      STEP("jac_r", g + 1, 2, w * (Nl[g + 2] + 2 * Nl[g + 1]));
      lv3_jac_r<T>(vMf[o], rRf[o], vRf[o], M[o], cR1[o], cR2[o], st);
      STEP("jac_g", g, 2, w * (Nl[g + 1] + 2 * Nl[g]));
      lv3_jac_g<T>(vRf[o], rGf[o], vGf[o], M[o], cG[o], st);
    }
    // ---- distributed ascent
    for (int o = oa - 1; o >= 0; o--) {
      const int g = 3 * o;
      // Emprolm reads v_G(2s) at c+1; Emprolb reads B at c-1
      STEP("jac_m", g + 2, 2 * nloc, w * (Nl[g + 3] + 2 * Nl[g + 2]));
      if (o + 1 < oa && (e = xchg_g(o + 1, st, &Rk::vG))) return e;
      for (int i = 0; i < nloc; i++) {
        const D3<T> &vc = (o + 1 < oa) ? rk[i].vG[o + 1] : vGf[oa];
        lv3_jac_m<T>(vc, rk[i].rM[o], rk[i].vM[o], M[o], cMg[o], st, c0(o, rk[i].q), c1(o, rk[i].q), 1);
      }
      if ((e = xchg_s(o, st, &Rk::vM, {7}))) return e;
      for (int i = 0; i < nloc; i++)
        lv3_jac_m<T>(vGf[oa], rk[i].rM[o], rk[i].vM[o], M[o], cMg[o], st, c0(o, rk[i].q), c1(o, rk[i].q), 2);
      // Erprolr reads B at c-1 and C at c+1; Erprolm reads Fx, Fy at c-1
      STEP("jac_r", g + 1, 2 * nloc, w * (Nl[g + 2] + 2 * Nl[g + 1]));
      if ((e = xchg_s(o, st, &Rk::vM, {0}))) return e;
      for (int i = 0; i < nloc; i++)
        lv3_jac_r<T>(rk[i].vM[o], rk[i].rR[o], rk[i].vR[o], M[o], cR1[o], cR2[o], st, c0(o, rk[i].q), c1(o, rk[i].q),
                     1);
      if ((e = xchg_s(o, st, &Rk::vR, {6, 5, 3}))) return e;
      for (int i = 0; i < nloc; i++)
        lv3_jac_r<T>(rk[i].vM[o], rk[i].rR[o], rk[i].vR[o], M[o], cR1[o], cR2[o], st, c0(o, rk[i].q), c1(o, rk[i].q),
                     2);
      // Egprolg reads C, Fz at c+1 and Fx, Fy at c-1 (the fine ascent the same)
      if ((e = xchg_s(o, st, &Rk::vR, {0}))) return e;
      if (o >= 1) {
        STEP("jac_g", g, 2 * nloc, w * (Nl[g + 1] + 2 * Nl[g]));
        for (int i = 0; i < nloc; i++)
          lv3_jac_g<T>(rk[i].vR[o], rk[i].rG[o], rk[i].vG[o], M[o], cG[o], st, c0(o, rk[i].q), c1(o, rk[i].q), 1);
        // Egprolr reads the green v at z +- 1
        if ((e = xchg_g(o, st, &Rk::vG))) return e;
        for (int i = 0; i < nloc; i++)
          lv3_jac_g<T>(rk[i].vR[o], rk[i].rG[o], rk[i].vG[o], M[o], cG[o], st, c0(o, rk[i].q), c1(o, rk[i].q), 2);
      } else {
        STEP("asc_fine", 0, nloc, w * (Nl[1] + 3 * Nl[0]));
        for (int i = 0; i < nloc; i++)
          if ((e = fast3_asc_fine<T>(rk[i].vR[0], uin[i], fe[i], pitch, uout[i], M[0], s->cfg.order, cG[0], coef, st,
                                     zr_fine(rk[i].q))))
            return e;
      }
    }
    return cudaSuccess;
  }

  // virtual global-plane-0 pointer of a caller slab (NCCL mode)
  template <class P_>
  P_ *vg(P_ *ptr) const {
    return ptr - (int64_t)(lo(0, s->cfg.rank) - 2) * fplane();
  }
  D3<const T> cfv(const void *p) const { return D3<const T>{vg((const T *)p), pitch, fplane()}; }
  D3<T> fv(void *p) const { return D3<T>{vg((T *)p), pitch, fplane()}; }

  TransportStatus status;
  void enqueue_cycle(const void *u_in, void *u_out, const void *f_eff, cudaStream_t st, Prof *prof) override {
    std::vector<const T *> ui{vg((const T *)u_in)}, fe{vg((const T *)f_eff)};
    std::vector<T *> uo{vg((T *)u_out)};
    status.note(cycle(ui, uo, fe, st, prof), comm.get(), "V-cycle");
  }
  int take_status(std::string *m) override { return status.take(m, comm.get()); }
  void enqueue_final_norm(void *u, const void *f_eff, cudaStream_t st) override {
    const T *ui = vg((const T *)u), *fe = vg((const T *)f_eff);
    status.note(xchg(0, false, 2, st, [&](int) { return ui; }, fplane()), comm.get(), "halo exchange");
    status.note(xchg(0, false, 1, st, [&](int) { return fe; }, fplane()), comm.get(), "halo exchange");
    fast3_desc_fine<T>(ui, fe, pitch, rk[0].rR[0], M[0], s->cfg.order, coef, sink(), st, zr_fine(rk[0].q));
  }
  cudaError_t reduce_hist(unsigned long long *d, int nslots, cudaStream_t st) override {
    cudaError_t e = comm->allreduce_max_u64(d, nslots, st);
    return e ? e : comm->allreduce_sum_f64(s->d_l2, nslots, st);
  }
  void enqueue_ftilde(const void *f, void *ft, cudaStream_t st, int64_t) override {
    if (loop) {
      launch3_ftilde<T>(D3<const T>{(const T *)f, pitch, fplane()}, D3<T>{(T *)ft, pitch, fplane()}, M[0], st);
      return;
    }
    const T *fvp = vg((const T *)f);
    status.note(xchg(0, false, 1, st, [&](int) { return fvp; }, fplane()), comm.get(), "halo exchange");
    launch3_ftilde<T>(cfv(f), fv(ft), M[0], st, lo(0, rk[0].q), hi(0, rk[0].q));
  }
  void enqueue_residual(const void *u, const void *f, void *r, cudaStream_t st, int64_t) override {
    if (loop) {
      launch3_residual<T>(D3<const T>{(const T *)u, pitch, fplane()}, D3<const T>{(const T *)f, pitch, fplane()},
                          D3<T>{(T *)r, pitch, fplane()}, M[0], s->cfg.order, coef, st);
      return;
    }
    const T *uvp = vg((const T *)u);
    status.note(xchg(0, false, 1, st, [&](int) { return uvp; }, fplane()), comm.get(), "halo exchange");
    launch3_residual<T>(cfv(u), cfv(f), fv(r), M[0], s->cfg.order, coef, st, lo(0, rk[0].q), hi(0, rk[0].q));
  }
  void enqueue_norm(const void *x, unsigned long long *mx, double *ss, cudaStream_t st, int64_t) override {
    if (loop) {
      launch3_norm<T>(D3<const T>{(const T *)x, pitch, fplane()}, M[0], mx, ss, st);
      return;
    }
    launch3_norm<T>(cfv(x), M[0], mx, ss, st, lo(0, rk[0].q), hi(0, rk[0].q));
    status.note(comm->allreduce_max_u64(mx, 1, st), comm.get(), "norm all-reduce");
    status.note(comm->allreduce_sum_f64(ss, 1, st), comm.get(), "norm all-reduce");
  }
  int launches_per_cycle() const override {
    int c = nloc;   // desc
    for (int o = 0; o < oa; o++) c += ((o >= 1) + 2) * nloc;
    c += 3 * (oc - oa) + 1;
    c += 6 * (oc - oa);
    for (int o = oa - 1; o >= 0; o--) c += (o >= 1 ? 6 : 5) * nloc;
    return c;
  }

  // ---- loopback: the whole mg_vcycle on full caller arrays
  int vcycle_all(mg_solver *sv, void *u, const void *f, int ncycles, double *res_hist) override {
    if (!loop) return 1;
    cudaStream_t st = sv->st;
    const size_t pb = fplane() * sizeof(T);
    const T *fsrc = (const T *)f;
    if (s->cfg.order == 4) {
      launch3_ftilde<T>(D3<const T>{(const T *)f, pitch, fplane()}, ft_full, M[0], st);
      fsrc = ft_full.p;
    }
    // scatter: planes [lo-2, hi+2) clipped to the grid
    for (int i = 0; i < nloc; i++) {
      const int a = std::max(lo(0, i) - 2, 0), b = std::min(hi(0, i) + 2, (int)n);
      const int64_t z0 = lo(0, i) - 2;
      for (int j = 0; j < 2; j++) cudaMemsetAsync(rk[i].u[j].p + z0 * fplane(), 0, (R(0) + 4) * pb, st);
      cudaMemsetAsync(rk[i].f.p + z0 * fplane(), 0, (R(0) + 4) * pb, st);
      cudaMemcpyAsync(rk[i].u[0].p + (int64_t)a * fplane(), (const T *)u + (int64_t)a * fplane(), (b - a) * pb,
                      cudaMemcpyDeviceToDevice, st);
      cudaMemcpyAsync(rk[i].f.p + (int64_t)a * fplane(), fsrc + (int64_t)a * fplane(), (b - a) * pb,
                      cudaMemcpyDeviceToDevice, st);
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
      xchg(0, false, 2, st, [&](int i) { return ui[i]; }, fplane());
      xchg(0, false, 1, st, [&](int i) { return fe[i]; }, fplane());
      for (int i = 0; i < nloc; i++)
        fast3_desc_fine<T>(ui[i], fe[i], pitch, rk[i].rR[0], M[0], s->cfg.order, coef, sink(), st, zr_fine(i));
    }
    // gather the owned planes back
    for (int i = 0; i < nloc; i++)
      cudaMemcpyAsync((T *)u + (int64_t)lo(0, i) * fplane(), rk[i].u[cur].p + (int64_t)lo(0, i) * fplane(), R(0) * pb,
                      cudaMemcpyDeviceToDevice, st);
    CKS(sv, cudaGetLastError());
    if (res_hist) return read_hist(sv, ncycles, res_hist, st);
    return MG_OK;
  }
};

// factory used by mg_create_ex
ImplBase *make_dist3(mg_solver *s, bool loopback, std::string *err) {
  Comm2 *c = loopback ? make_loop_comm(s->cfg.nranks)
                      : make_nccl_comm(s->cfg.nranks, s->cfg.rank, s->cfg.nccl_id, s->esz, err);
  if (!c) return nullptr;
  if (s->cfg.dtype == MG_F64) {
    auto *d = new Dist3<double>(s, loopback);
    d->comm.reset(c);
    return d;
  }
  auto *d = new Dist3<float>(s, loopback);
  d->comm.reset(c);
  return d;
}
