// api.cu — the extern "C" boundary (include/seaice.h) and the Newton driver.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstring>
#include <vector>

#include "ctx.cuh"
#include "stencil.cuh"

using namespace seaice;

struct seaice_ctx {
  Ctx c;
};

#define API_BEGIN(ctx)                                   \
  if (!(ctx)) return SEAICE_EINVAL;                      \
  Ctx& c = (ctx)->c;                                     \
  try {
#define API_END                                          \
  }                                                      \
  catch (const Error& e) {                               \
    c.err = e.what();                                    \
    if (e.code == SEAICE_ECUDA) cudaGetLastError();      \
    return e.code;                                       \
  }                                                      \
  catch (const std::exception& e) {                      \
    c.err = e.what();                                    \
    return SEAICE_ECUDA;                                 \
  }

namespace {

// Reading G12b: |DeltaPhi| <= kLsEta * sum|terms| is fp64 roundoff.
constexpr double kLsEta = 1e-12;

struct EvTimer {
  Ctx& c;
  explicit EvTimer(Ctx& cc) : c(cc) { SI_CUDA(cudaEventRecord(c.ev0, c.s)); }
  double ms() {
    SI_CUDA(cudaEventRecord(c.ev1, c.s));
    SI_CUDA(cudaEventSynchronize(c.ev1));
    float t = 0.f;
    SI_CUDA(cudaEventElapsedTime(&t, c.ev0, c.ev1));
    return (double)t;
  }
};

void validate(const seaice_params* p) {
  SI_CHECK(p, SEAICE_EINVAL, "NULL params");
  SI_CHECK(p->n >= 2, SEAICE_EINVAL, "n must be >= 2");
  SI_CHECK(p->L > 0 && std::isfinite(p->L), SEAICE_EINVAL, "L must be positive");
  const double pos[] = {p->rho_i, p->rho_a, p->rho_o, p->C_a, p->C_o, p->e, p->delta_min};
  for (double v : pos) SI_CHECK(v > 0 && std::isfinite(v), SEAICE_EINVAL, "physical constants must be positive");
  SI_CHECK(p->P_star >= 0 && p->C >= 0 && std::isfinite(p->f_c), SEAICE_EINVAL, "P*, C must be >= 0");
  const long long Nn = (long long)(p->n + 1) * (p->n + 1);
  SI_CHECK(36LL * Nn < (1LL << 31), SEAICE_EINVAL, "mesh too large for int32 CSR indices");
  SI_CHECK(p->restart >= 1 && p->restart <= 60, SEAICE_EINVAL, "restart must be in [1, 60]");
  SI_CHECK(p->krylov_maxit >= 1 && p->newton_maxit >= 0, SEAICE_EINVAL, "bad iteration caps");
  SI_CHECK(p->ls_max_halvings >= 0 && p->ls_max_halvings <= 60, SEAICE_EINVAL, "ls_max_halvings in [0,60]");
  SI_CHECK(p->jacobian >= 0 && p->jacobian <= 2, SEAICE_EINVAL, "bad jacobian kind");
  SI_CHECK(p->precond >= 0 && p->precond <= 2, SEAICE_EINVAL, "bad preconditioner kind");
  SI_CHECK(p->cheb_degree >= 1 && p->cheb_degree <= 16, SEAICE_EINVAL, "cheb_degree in [1,16]");
  SI_CHECK(p->max_levels >= 1 && p->max_levels <= 40, SEAICE_EINVAL, "max_levels in [1,40]");
  SI_CHECK(p->coarse_max_dof >= 3 && p->coarse_max_dof <= 8192, SEAICE_EINVAL, "coarse_max_dof in [3,8192]");
  SI_CHECK(p->agg_dist0 >= 1 && p->agg_dist0 <= 3 && p->agg_dist >= 1 && p->agg_dist <= 3, SEAICE_EINVAL,
           "agg_dist0/agg_dist must be 1, 2 or 3");
  SI_CHECK(p->cheb_fused >= 0 && p->cheb_fused <= 2, SEAICE_EINVAL, "cheb_fused must be 0, 1 or 2");
  SI_CHECK(p->cheb_degree0 >= 0 && p->cheb_degree0 <= 16, SEAICE_EINVAL, "cheb_degree0 in [0,16]");
  SI_CHECK(p->matfree == 0 || p->matfree == 1, SEAICE_EINVAL, "matfree must be 0 or 1");
  SI_CHECK(p->krylov_forcing == 0 || p->krylov_forcing == 1, SEAICE_EINVAL, "krylov_forcing must be 0 or 1");
  SI_CHECK(p->nullspace_dim == 3 || p->nullspace_dim == 4, SEAICE_EINVAL, "nullspace_dim must be 3 or 4");
  SI_CHECK(p->krylov_method == 0 || p->krylov_method == 1, SEAICE_EINVAL, "krylov_method must be 0 or 1");
  SI_CHECK(p->spgemm_path >= 0 && p->spgemm_path <= 6, SEAICE_EINVAL, "spgemm_path must be in 0..6");
  SI_CHECK(p->amg_lag >= 0, SEAICE_EINVAL, "amg_lag must be >= 0");
  SI_CHECK(p->amg_reuse == 0 || p->amg_reuse == 1, SEAICE_EINVAL, "amg_reuse must be 0 or 1");
  SI_CHECK(p->vcycle_tail == 0 || p->vcycle_tail == 1, SEAICE_EINVAL, "vcycle_tail must be 0 or 1");
}

int newton_step_impl(Ctx& c, double* v, double* pi_inout, seaice_newton_stats* out) {
  seaice_newton_stats st;
  std::memset(&st, 0, sizeof(st));
  double* pi = pi_inout ? pi_inout : c.pi.get();
  SI_CHECK(v, SEAICE_EINVAL, "NULL velocity");
  // a-2 / a-3: fused residual + Jacobian
  {
    EvTimer t(c);
    double nr = 0.0;
    assemble_impl(c, v, pi, true, nullptr, &nr);
    st.t_assemble = t.ms();
    SI_CHECK(std::isfinite(nr), SEAICE_ENONFINITE, "non-finite residual norm");
    if (!c.have_r0) {
      c.r0 = nr;
      c.have_r0 = true;
    }
    st.res_norm = nr;
    st.res_norm0 = c.r0;
    if (c.r0 < 1e-14 || nr <= c.p.newton_rtol * c.r0) {
      st.converged_on_entry = 1;
      if (out) *out = st;
      return SEAICE_OK;
    }
  }
  // a-4: AMG setup
  if (c.p.precond == SEAICE_PC_AMG) {
    EvTimer t(c);
    // reading G31: keep the coarse levels while the previous solve stayed cheap
    const bool lag = c.p.amg_lag > 0 && c.lag_ok && c.nlev > 1 && c.last_krylov_its <= c.p.amg_lag &&
                     amg_lag_allowed(c);
    if (lag) amg_refresh_finest(c);
    else amg_setup_impl(c);
    c.lag_ok = true;
    st.amg_rebuilt = lag ? 0 : 1;
    st.amg_reused = (!lag && c.last_setup_reused) ? 1 : 0;
    st.t_amg = t.ms();
    st.amg_levels = c.nlev;
    st.amg_op_complexity = c.op_complexity;
  }
  // a-5: J vt = R (to krylov_rtol, or to the Eisenstat-Walker forcing term, reading G29)
  c.vt.ensure(c.al, c.N);
  int kst;
  {
    EvTimer t(c);
    const double rtol_fixed = c.p.krylov_rtol;
    if (c.p.krylov_forcing == 1) {
      double eta = 0.1;
      if (c.ew_prev_res > 0.0) {
        const double ratio = st.res_norm / c.ew_prev_res;
        eta = 0.9 * ratio * ratio;
        const double sg = 0.9 * c.ew_prev_eta * c.ew_prev_eta;
        if (sg > 0.1) eta = std::max(eta, sg);
      }
      eta = std::max(eta, 0.5 * c.p.newton_rtol * c.r0 / st.res_norm);
      eta = std::min(std::max(eta, rtol_fixed), 0.1);
      // safeguard: after a line search that found no energy decrease the inexact direction was
      // not a descent direction; solve the next system to the floor tolerance
      if (c.ew_ls_failed) eta = rtol_fixed;
      c.ew_prev_res = st.res_norm;
      c.ew_prev_eta = eta;
      c.p.krylov_rtol = eta;
    }
    try {
      kst = fgmres_impl(c, c.R.get(), c.vt.get(), &st.krylov);
      c.last_krylov_its = st.krylov.iters;
    } catch (...) {
      c.p.krylov_rtol = rtol_fixed;
      throw;
    }
    c.p.krylov_rtol = rtol_fixed;
    st.t_krylov = t.ms();
  }
  // a-6: backtracking on Phi, difference form
  {
    EvTimer t(c);
    const int K = c.p.ls_max_halvings + 1;
    std::vector<double> al(K), dphi(K), sab(K);
    for (int k = 0; k < K; ++k) al[k] = std::ldexp(1.0, -k);
    int acc = -1;
    const double nr0 = st.res_norm;
    // alpha = 1 alone first (accepted by almost every Newton iteration; the kernel's fp64 work
    // grows with the number of step lengths: 2.1 ms for 8 against 0.7 ms for 1 at config 4), then
    // batches of 8.  Each step length is summed on its own, so the values do not depend on the batching.
    for (int k0 = 0, cnt = 1; k0 < K && acc < 0; k0 += cnt, cnt = std::min(8, K - k0)) {
      delta_energy_impl(c, v, c.vt.get(), al.data() + k0, cnt, dphi.data() + k0, sab.data() + k0);
      for (int k = k0; k < k0 + cnt; ++k) {
        if (dphi[k] < -kLsEta * sab[k]) {
          acc = k;
          break;
        }
        if (dphi[k] <= kLsEta * sab[k]) {
          // energy change below fp64 roundoff: accept iff ||R|| decreases (reading G12b)
          c.w.ensure(c.al, c.N);
          copy(c, c.w.get(), v, c.N);
          axpy(c, al[k], c.vt.get(), c.w.get(), c.N);
          double nr1 = 0.0;
          assemble_impl(c, c.w.get(), nullptr, false, nullptr, &nr1);
          if (nr1 < nr0) {
            acc = k;
            break;
          }
        }
      }
    }
    c.ew_ls_failed = acc < 0;  // EW safeguard for the next solve (reading G29)
    if (acc < 0) {
      st.ls_stagnated = 1;
      acc = K - 1;
    }
    st.alpha = al[acc];
    st.dphi = dphi[acc];
    st.halvings = acc;
    // a-7: pi += alpha pi~ (uses v_l), then v += alpha vt
    if (c.p.jacobian == SEAICE_JAC_SV) pi_tilde_impl(c, v, pi, c.vt.get(), pi, st.alpha, true);
    axpy(c, st.alpha, c.vt.get(), v, c.N);
    st.t_ls = t.ms();
  }
  if (out) *out = st;
  return kst == SEAICE_NOT_CONVERGED ? SEAICE_NOT_CONVERGED : SEAICE_OK;
}

int solve_step_impl(Ctx& c, double dt, double t_new, const double* h, const double* A, const double* v_prev,
                    const double* v_air, const double* v_ocean, double* v_out, seaice_step_stats* out) {
  seaice_step_stats st;
  std::memset(&st, 0, sizeof(st));
  auto t0 = std::chrono::steady_clock::now();
  {
    EvTimer t(c);
    set_step_impl(c, dt, t_new, h, A, v_prev, v_air, v_ocean, nullptr);
    st.t_setup = t.ms();
  }
  copy(c, v_out, c.vprev.get(), c.N);
  int status = SEAICE_NOT_CONVERGED;
  for (int l = 0; l <= c.p.newton_maxit; ++l) {
    seaice_newton_stats ns;
    newton_step_impl(c, v_out, nullptr, &ns);
    if (l == 0) st.res_norm0 = ns.res_norm0;
    st.res_norm_final = ns.res_norm;
    st.t_assemble += ns.t_assemble;
    if (ns.converged_on_entry) {
      status = SEAICE_OK;
      st.converged = 1;
      break;
    }
    st.newton_iters++;
    st.krylov_iters_total += ns.krylov.iters;
    st.krylov_solves++;
    if (!ns.krylov.converged) st.krylov_capped++;
    st.krylov_max_iters = std::max(st.krylov_max_iters, ns.krylov.iters);
    st.amg_setups += ns.amg_rebuilt;
    st.amg_reuses += ns.amg_reused;
    st.t_amg += ns.t_amg;
    st.t_krylov += ns.t_krylov;
    st.t_ls += ns.t_ls;
  }
  SI_CUDA(cudaStreamSynchronize(c.s));
  st.seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  if (out) *out = st;
  return status;
}

}  // namespace

extern "C" {

void seaice_default_params(seaice_params* p, int32_t n) {
  if (!p) return;
  std::memset(p, 0, sizeof(*p));
  p->n = n;
  p->L = 512.0e3;
  p->rho_i = 900.0;
  p->rho_a = 1.3;
  p->rho_o = 1026.0;
  p->C_a = 1.2e-3;
  p->C_o = 5.5e-3;
  p->P_star = 27500.0;
  p->C = 20.0;
  p->e = 2.0;
  p->delta_min = 2.0e-9;
  p->f_c = 1.46e-4;
  p->jacobian = SEAICE_JAC_SV;
  p->newton_rtol = 1e-8;
  p->newton_maxit = 200;
  p->ls_max_halvings = 20;
  p->krylov_rtol = 1e-8;
  p->restart = 60;  // reading G13 (config 4: 2.88 -> 2.61 s per step against restart 30; the late solves need 100-160 iterations)
  p->krylov_maxit = 300;
  p->precond = SEAICE_PC_AMG;
  p->amg_theta = 0.04;
  p->cheb_degree = 3;
  p->coarse_max_dof = 400;
  p->max_levels = 25;
  p->cheb_lower = 0.03;
  p->cheb_upper = 1.1;
  p->power_iters = 20;
  p->project_pi = 0;
  p->amg_seed = 0;
  p->agg_dist0 = 2;
  p->agg_dist = 3;  // MIS(3) on coarse levels (config 4: 3.98 -> 3.61 s per step)
  p->cheb_fused = 2;  // TMA-streamed (config 4: 190 us per smoothing vs 322 + 166 us tile + residual)
  p->cheb_degree0 = 0;  // measured no gain on B200 (grid barriers ~ launch gaps in the graph)
  p->matfree = 0;       // the assembled 19-value stencil SpMV is ~4x cheaper than the matrix-free apply
  p->krylov_forcing = 1;  // Eisenstat-Walker forcing, floor krylov_rtol (reading G29)
  p->nullspace_dim = 4;  // rigid-body modes + the linearisation point (reading G30)
  p->krylov_method = 0;
  p->spgemm_path = 0;
  p->amg_lag = 10;  // lagged hierarchy after cheap solves (config 4: 3.35 -> 3.05 s; Problem II 1.4-2.5x, DESIGN G31)
  p->amg_reuse = 0;
  p->vcycle_tail = 0;  // measured on B200 (config 4): 136 us instead of 184 us of kernels, but the captured V-cycle 2442 -> 2499 us
}

int seaice_create(const seaice_params* p, const seaice_runtime* rt, seaice_ctx** out) {
  if (!out) return SEAICE_EINVAL;
  *out = nullptr;
  seaice_ctx* h = new seaice_ctx();
  Ctx& c = h->c;
  try {
    validate(p);
    c.p = *p;
    if (rt) c.al.rt = *rt;
    c.s = rt ? (cudaStream_t)rt->stream : nullptr;
    c.al.s = c.s;
    c.n = p->n;
    c.Nn = (p->n + 1) * (p->n + 1);
    c.N = 2 * c.Nn;
    c.Nc = p->n * p->n;
    c.dx = p->L / p->n;
    c.ph = Phys{p->rho_i, p->rho_a, p->rho_o, p->C_a, p->C_o, p->P_star, p->C, p->e, p->delta_min, p->f_c,
                c.dx, 0.0, p->n};
    c.use_graphs = getenv("SEAICE_NO_GRAPHS") == nullptr;
    {
      int dev = 0, sms = 0;
      SI_CUDA(cudaGetDevice(&dev));
      SI_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
      if (sms > 0) c.sms = sms;
    }
    SI_CUDA(cudaMallocHost(&c.hbuf, 256 * sizeof(double)));
    SI_CUDA(cudaEventCreate(&c.ev0));
    SI_CUDA(cudaEventCreate(&c.ev1));
    c.P.ensure(c.al, c.Nc);
    c.rhoh.ensure(c.al, c.Nc);
    c.F.ensure(c.al, c.N);
    c.vprev.ensure(c.al, c.N);
    c.vair.ensure(c.al, c.N);
    c.vocean.ensure(c.al, c.N);
    c.pi.ensure(c.al, 12LL * c.Nc);
    c.flag.ensure(c.al, 16);
    c.Jst.ensure(c.al, (long long)kJS * c.Nn);
    c.R.ensure(c.al, c.N);
    c.scal.ensure(c.al, 256);
    c.part.ensure(c.al, 4096);
    SI_CUDA(cudaStreamSynchronize(c.s));
  } catch (const Error& e) {
    int code = e.code;
    seaice_destroy(h);
    return code;
  }
  *out = h;
  return SEAICE_OK;
}

int seaice_destroy(seaice_ctx* h) {
  if (!h) return SEAICE_OK;
  Ctx& c = h->c;
  cudaStreamSynchronize(c.s);
  amg_free(c);
  DBuf<double>* dbs[] = {&c.P, &c.rhoh, &c.F, &c.vprev, &c.vair, &c.vocean, &c.pi, &c.vwork, &c.load, &c.Jst, &c.Jsm, &c.mf_v, &c.mf_pi, &c.lin_v,
                         &c.R, &c.csr_val, &c.part, &c.scal, &c.vt, &c.pit, &c.V, &c.Z, &c.w, &c.xk, &c.rk,
                         &c.cinv, &c.dwork, &c.cg_p, &c.cg_q, &c.cg_s};
  for (auto* b : dbs) b->free_();
  c.flag.free_();
  c.csr_rp.free_();
  c.csr_ci.free_();
  c.iwork.free_();
  c.lwork.free_();
  for (auto* b : {&c.st_h, &c.st_A, &c.st_vp, &c.st_va, &c.st_vo, &c.st_v}) b->free_();
  prof_harvest(c, true);
  for (auto e : c.prof.free_ev) cudaEventDestroy(e);
  if (c.hbuf) cudaFreeHost(c.hbuf);
  if (c.cap_stream) cudaStreamDestroy(c.cap_stream);
  if (c.ev0) cudaEventDestroy(c.ev0);
  if (c.ev1) cudaEventDestroy(c.ev1);
  for (auto e : c.arn_ev)
    if (e) cudaEventDestroy(e);
  cudaStreamSynchronize(c.s);
  delete h;
  return SEAICE_OK;
}

const char* seaice_last_error(const seaice_ctx* h) { return h ? h->c.err.c_str() : "NULL context"; }

int seaice_set_step(seaice_ctx* h, double dt, double t_new, const double* hh, const double* A, const double* v_prev,
                    const double* v_air, const double* v_ocean, const double* extra_load) {
  API_BEGIN(h)
  set_step_impl(c, dt, t_new, hh, A, v_prev, v_air, v_ocean, extra_load);
  return SEAICE_OK;
  API_END
}

int seaice_residual(seaice_ctx* h, const double* v, double* r_out, double* norm2_host) {
  API_BEGIN(h)
  double nr = 0.0;
  assemble_impl(c, v, nullptr, false, r_out, &nr);
  if (norm2_host) *norm2_host = nr;
  SI_CHECK(std::isfinite(nr), SEAICE_ENONFINITE, "non-finite residual norm");
  return SEAICE_OK;
  API_END
}

int seaice_assemble_jacobian(seaice_ctx* h, const double* v, const double* pi, seaice_csr* view) {
  API_BEGIN(h)
  assemble_impl(c, v, pi, true, nullptr, nullptr);
  if (view) build_csr_view(c, view);
  SI_CUDA(cudaStreamSynchronize(c.s));
  return SEAICE_OK;
  API_END
}

int seaice_spmv(seaice_ctx* h, const double* x, double* y) {
  API_BEGIN(h)
  SI_CHECK(c.assembled, SEAICE_ESTATE, "spmv before assemble_jacobian");
  stencil_spmv(c, x, y);
  return SEAICE_OK;
  API_END
}

int seaice_transport(seaice_ctx* h, double dt, const double* v, const double* A, const double* H, double A_in,
                     double H_in, double* A_out, double* H_out, double* cfl_host, int32_t* substeps_host) {
  API_BEGIN(h)
  int m = 1;
  transport_impl(c, dt, v, A, H, A_in, H_in, A_out, H_out, cfl_host, &m);
  if (substeps_host) *substeps_host = m;
  return SEAICE_OK;
  API_END
}

int seaice_jv_matfree(seaice_ctx* h, const double* v, const double* pi, const double* x, double* y) {
  API_BEGIN(h)
  jv_matfree_impl(c, v, pi, x, y);
  return SEAICE_OK;
  API_END
}

int seaice_amg_setup(seaice_ctx* h, int32_t* levels_out, double* oc_out) {
  API_BEGIN(h)
  SI_CHECK(c.assembled, SEAICE_ESTATE, "amg_setup before assemble_jacobian");
  amg_setup_impl(c);
  if (levels_out) *levels_out = (int32_t)c.nlev;
  if (oc_out) *oc_out = c.op_complexity;
  return SEAICE_OK;
  API_END
}

int seaice_amg_level(seaice_ctx* h, int32_t level, seaice_bsr* A_out, seaice_bsr* P_out, int32_t* agg_host) {
  API_BEGIN(h)
  SI_CHECK(c.amg_ready, SEAICE_ESTATE, "no AMG hierarchy");
  SI_CHECK(level >= 0 && level < c.nlev, SEAICE_EINVAL, "level out of range");
  const Level& L = c.lv[level];
  if (A_out) *A_out = seaice_bsr{L.nb, L.nb, L.b, L.b, L.nnzb, L.rp.get(), L.ci.get(), L.val.get()};
  const bool last = level + 1 == c.nlev;
  if (P_out) {
    if (last)
      std::memset(P_out, 0, sizeof(*P_out));
    else
      *P_out = seaice_bsr{L.nb, L.nbc, L.b, c.lv[level + 1].b, L.Pnnzb, L.Prp.get(), L.Pci.get(), L.Pval.get()};
  }
  if (agg_host && !last) {
    SI_CUDA(cudaMemcpyAsync(agg_host, L.agg.get(), sizeof(int) * L.nb, cudaMemcpyDeviceToHost, c.s));
  }
  SI_CUDA(cudaStreamSynchronize(c.s));
  return SEAICE_OK;
  API_END
}

int seaice_precond_apply(seaice_ctx* h, const double* r, double* z) {
  API_BEGIN(h)
  SI_CHECK(c.assembled, SEAICE_ESTATE, "precond before assemble_jacobian");
  precond_apply(c, r, z);
  SI_CUDA(cudaStreamSynchronize(c.s));
  return SEAICE_OK;
  API_END
}

int seaice_fgmres_solve(seaice_ctx* h, const double* b, double* x, seaice_krylov_stats* st) {
  API_BEGIN(h)
  return fgmres_impl(c, b, x, st);
  API_END
}

int seaice_delta_energy(seaice_ctx* h, const double* v, const double* vt, const double* alphas, int32_t count,
                        double* out) {
  API_BEGIN(h)
  SI_CHECK(alphas && out && v && vt, SEAICE_EINVAL, "NULL argument");
  delta_energy_impl(c, v, vt, alphas, count, out);
  return SEAICE_OK;
  API_END
}

int seaice_pi_tilde(seaice_ctx* h, const double* v, const double* pi, const double* vt, double* pi_out) {
  API_BEGIN(h)
  SI_CHECK(v && vt && pi_out, SEAICE_EINVAL, "NULL argument");
  pi_tilde_impl(c, v, pi ? pi : c.pi.get(), vt, pi_out, 0.0, false);
  SI_CUDA(cudaStreamSynchronize(c.s));
  return SEAICE_OK;
  API_END
}

int seaice_get_pi(seaice_ctx* h, double* pi_out) {
  API_BEGIN(h)
  copy(c, pi_out, c.pi.get(), 12LL * c.Nc);
  SI_CUDA(cudaStreamSynchronize(c.s));
  return SEAICE_OK;
  API_END
}

int seaice_set_pi(seaice_ctx* h, const double* pi_in) {
  API_BEGIN(h)
  copy(c, c.pi.get(), pi_in, 12LL * c.Nc);
  SI_CUDA(cudaStreamSynchronize(c.s));
  return SEAICE_OK;
  API_END
}

int seaice_newton_step(seaice_ctx* h, double* v, double* pi, seaice_newton_stats* st) {
  API_BEGIN(h)
  return newton_step_impl(c, v, pi, st);
  API_END
}

int seaice_solve_step(seaice_ctx* h, double dt, double t_new, const double* hh, const double* A,
                      const double* v_prev, const double* v_air, const double* v_ocean, double* v_out,
                      seaice_step_stats* st) {
  API_BEGIN(h)
  SI_CHECK(v_out, SEAICE_EINVAL, "NULL v_out");
  return solve_step_impl(c, dt, t_new, hh, A, v_prev, v_air, v_ocean, v_out, st);
  API_END
}

int seaice_solve_step_host(seaice_ctx* h, double dt, double t_new, const double* h_host, const double* A_host,
                           const double* vp_host, const double* va_host, const double* vo_host, double* vout_host,
                           seaice_step_stats* st) {
  API_BEGIN(h)
  SI_CHECK(h_host && A_host && vp_host && va_host && vo_host && vout_host, SEAICE_EINVAL, "NULL host buffer");
  c.st_h.ensure(c.al, c.Nc);
  c.st_A.ensure(c.al, c.Nc);
  c.st_vp.ensure(c.al, c.N);
  c.st_va.ensure(c.al, c.N);
  c.st_vo.ensure(c.al, c.N);
  c.st_v.ensure(c.al, c.N);
  SI_CUDA(cudaMemcpyAsync(c.st_h.get(), h_host, sizeof(double) * c.Nc, cudaMemcpyHostToDevice, c.s));
  SI_CUDA(cudaMemcpyAsync(c.st_A.get(), A_host, sizeof(double) * c.Nc, cudaMemcpyHostToDevice, c.s));
  SI_CUDA(cudaMemcpyAsync(c.st_vp.get(), vp_host, sizeof(double) * c.N, cudaMemcpyHostToDevice, c.s));
  SI_CUDA(cudaMemcpyAsync(c.st_va.get(), va_host, sizeof(double) * c.N, cudaMemcpyHostToDevice, c.s));
  SI_CUDA(cudaMemcpyAsync(c.st_vo.get(), vo_host, sizeof(double) * c.N, cudaMemcpyHostToDevice, c.s));
  int rc = solve_step_impl(c, dt, t_new, c.st_h.get(), c.st_A.get(), c.st_vp.get(), c.st_va.get(), c.st_vo.get(),
                           c.st_v.get(), st);
  SI_CUDA(cudaMemcpyAsync(vout_host, c.st_v.get(), sizeof(double) * c.N, cudaMemcpyDeviceToHost, c.s));
  SI_CUDA(cudaStreamSynchronize(c.s));
  return rc;
  API_END
}

int64_t seaice_launch_count(const seaice_ctx* h) { return h ? (int64_t)h->c.launches : 0; }

int seaice_profile_enable(seaice_ctx* h, int32_t on) {
  API_BEGIN(h)
  SI_CUDA(cudaStreamSynchronize(c.s));
  prof_harvest(c, true);
  for (int k = 0; k < PC_NCLASS; ++k) {
    c.prof.ms[k] = 0.0;
    c.prof.cnt[k] = 0;
    c.prof.bytes[k] = 0.0;
  }
  c.prof.on = on != 0;
  return SEAICE_OK;
  API_END
}

int seaice_profile_read(seaice_ctx* h, double* ms, int64_t* cnt, double* bytes) {
  API_BEGIN(h)
  SI_CUDA(cudaStreamSynchronize(c.s));
  prof_harvest(c, true);
  for (int k = 0; k < SEAICE_PROF_CLASSES; ++k) {
    if (ms) ms[k] = k < PC_NCLASS ? c.prof.ms[k] : 0.0;
    if (cnt) cnt[k] = k < PC_NCLASS ? c.prof.cnt[k] : 0;
    if (bytes) bytes[k] = k < PC_NCLASS ? c.prof.bytes[k] : 0.0;
  }
  return SEAICE_OK;
  API_END
}

int seaice_spgemm_path_hits(const seaice_ctx* h, int64_t* hits, int32_t n) {
  if (!h || !hits || n < 0) return SEAICE_EINVAL;
  for (int k = 0; k < n && k < SEAICE_SPGEMM_PATHS; ++k) hits[k] = (int64_t)h->c.sg_hits[k];
  return SEAICE_OK;
}

int seaice_memory(const seaice_ctx* h, int64_t* live, int64_t* peak) {
  if (!h) return SEAICE_EINVAL;
  if (live) *live = (int64_t)h->c.al.live_bytes;
  if (peak) *peak = (int64_t)h->c.al.peak_bytes;
  return SEAICE_OK;
}

}  // extern "C"
