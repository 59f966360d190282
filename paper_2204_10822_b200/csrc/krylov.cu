// krylov.cu — right-preconditioned FGMRES(m) driven from the host.
// Definition shared with oracle/krylov.py (as a definition, not code): x0 = 0,
// classical Gram-Schmidt in one pass, Givens rotations, the inner loop stops when the
// estimate |g_{j+1}| <= rtol ||b||; convergence is declared only when the explicit residual
// computed at the end of the cycle satisfies ||b - A x|| <= rtol ||b|| (else restart).
#include <cmath>
#include <vector>

#include "ctx.cuh"
#include "stencil.cuh"

namespace seaice {

// FGMRES operator: the assembled stencil J, or (matfree = 1) J(v, pi) applied
// matrix-free at the linearisation point saved by the last assembly
static void apply_A(Ctx& c, const double* x, double* y) {
  if (c.p.matfree) jv_matfree_impl(c, c.mf_v.get(), c.mf_pi.get(), x, y);
  else stencil_spmv(c, x, y);
}

__global__ void k_point_jacobi(int Nn, const double* __restrict__ J, const double* __restrict__ r,
                               double* __restrict__ z) {
  const int node = blockIdx.x * blockDim.x + threadIdx.x;
  if (node >= Nn) return;
  // diagonal entries of the node's own block
  z[2 * node] = r[2 * node] / J[(long long)kJDxx * Nn + node];
  z[2 * node + 1] = r[2 * node + 1] / J[(long long)kJDyy * Nn + node];
}

void precond_apply(Ctx& c, const double* r, double* z) {
  switch (c.p.precond) {
    case SEAICE_PC_NONE:
      copy(c, z, r, c.N);
      break;
    case SEAICE_PC_JACOBI:
      k_point_jacobi<<<grid_for(c.Nn), kThreads, 0, c.s>>>(c.Nn, c.Jst.get(), r, z);
      SI_LAUNCHED(c);
      break;
    default:
      SI_CHECK(c.amg_ready, SEAICE_ESTATE, "AMG preconditioner requested before seaice_amg_setup");
      amg_vcycle(c, r, z);
  }
}

// ------------------------------------------------------------------ PCG (krylov_method = 1)
// Textbook preconditioned conjugate gradients (oracle/krylov.py pcg, same definition): x0 = 0,
// r = b, z = M r, p = z; alpha = (r.z)/(p.Ap); x += alpha p; r -= alpha Ap; stop when
// ||r|| <= rtol ||b||; beta = (r.z)_new/(r.z)_old; p = z + beta p.  J is SPD (eq:modification,
// P:534-539) and the V-cycle is symmetric (same Chebyshev polynomial pre and post, R = P^T).
// The scalars live on the device (s[0] = r.z, s[1] = beta, s[2] = alpha, s[3] = ||r||^2): one
// host synchronisation per iteration, for the stopping test.  Convergence is declared only when
// the explicit residual ||b - A x|| also meets the tolerance (else CG restarts from it).
enum { kCgRZ = 0, kCgBeta = 1, kCgAlpha = 2, kCgRR = 3, kCgPQ = 4 };

__global__ void k_cg_rz(const double* __restrict__ part, int nparts, double* __restrict__ s, int first) {
  __shared__ double sh[32];
  double v = 0.0;
  for (int i = threadIdx.x; i < nparts; i += blockDim.x) v += part[i];
  v = block_sum(v, sh);
  if (threadIdx.x == 0) {
    s[kCgBeta] = first ? 0.0 : v / s[kCgRZ];
    s[kCgRZ] = v;
  }
}
__global__ void k_cg_alpha(const double* __restrict__ part, int nparts, double* __restrict__ s) {
  __shared__ double sh[32];
  double v = 0.0;
  for (int i = threadIdx.x; i < nparts; i += blockDim.x) v += part[i];
  v = block_sum(v, sh);
  if (threadIdx.x == 0) {
    s[kCgPQ] = v;
    s[kCgAlpha] = s[kCgRZ] / v;
  }
}
__global__ void k_cg_sum(const double* __restrict__ part, int nparts, double* __restrict__ out) {
  __shared__ double sh[32];
  double v = 0.0;
  for (int i = threadIdx.x; i < nparts; i += blockDim.x) v += part[i];
  v = block_sum(v, sh);
  if (threadIdx.x == 0) *out = v;
}
// partial r.z
__global__ void k_cg_dot(long long n, const double* __restrict__ a, const double* __restrict__ b,
                         double* __restrict__ part) {
  __shared__ double sh[32];
  double v = 0.0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    v += a[i] * b[i];
  v = block_sum(v, sh);
  if (threadIdx.x == 0) part[blockIdx.x] = v;
}
// p = z + beta p
__global__ void k_cg_p(long long n, const double* __restrict__ z, const double* __restrict__ s,
                       double* __restrict__ p) {
  const double beta = s[kCgBeta];
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    p[i] = (beta == 0.0) ? z[i] : z[i] + beta * p[i];  // first step: p may hold stale data
}
// x += alpha p; r -= alpha q; partial ||r||^2
__global__ void k_cg_update(long long n, const double* __restrict__ p, const double* __restrict__ q,
                            const double* __restrict__ s, double* __restrict__ x, double* __restrict__ r,
                            double* __restrict__ part) {
  __shared__ double sh[32];
  const double alpha = s[kCgAlpha];
  double v = 0.0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    x[i] += alpha * p[i];
    const double ri = r[i] - alpha * q[i];
    r[i] = ri;
    v += ri * ri;
  }
  v = block_sum(v, sh);
  if (threadIdx.x == 0) part[blockIdx.x] = v;
}

static int pcg_impl(Ctx& c, const double* b, double* x, seaice_krylov_stats* st) {
  const long long N = c.N;
  c.cg_p.ensure(c.al, N);
  c.cg_q.ensure(c.al, N);
  c.cg_s.ensure(c.al, 8);
  c.w.ensure(c.al, N);
  c.rk.ensure(c.al, N);
  double *p = c.cg_p.get(), *q = c.cg_q.get(), *s = c.cg_s.get(), *z = c.w.get(), *r = c.rk.get();
  const int g = red_grid(N);
  c.part.ensure(c.al, (size_t)g + 64);
  double* part = c.part.get();
  fill(c, x, 0.0, N);
  const double bnorm = norm2(c, b, N);
  seaice_krylov_stats S{0, 0, 1, 0.0, 0.0};
  if (bnorm == 0.0) {
    if (st) *st = S;
    return SEAICE_OK;
  }
  SI_CHECK(std::isfinite(bnorm), SEAICE_ENONFINITE, "pcg: non-finite right-hand side");
  const double tol = c.p.krylov_rtol * bnorm;
  copy(c, r, b, N);
  int its = 0;
  bool converged = false;
  double rn = bnorm;
  while (true) {
    bool first = true;
    while (its < c.p.krylov_maxit) {
      precond_apply(c, r, z);
      k_cg_dot<<<g, kThreads, 0, c.s>>>(N, r, z, part);
      k_cg_rz<<<1, 1024, 0, c.s>>>(part, g, s, first ? 1 : 0);
      k_cg_p<<<g, kThreads, 0, c.s>>>(N, z, s, p);
      SI_LAUNCHED(c);
      c.launches += 2;
      apply_A(c, p, q);
      k_cg_dot<<<g, kThreads, 0, c.s>>>(N, p, q, part);
      k_cg_alpha<<<1, 1024, 0, c.s>>>(part, g, s);
      k_cg_update<<<g, kThreads, 0, c.s>>>(N, p, q, s, x, r, part);
      k_cg_sum<<<1, 1024, 0, c.s>>>(part, g, s + kCgRR);
      SI_LAUNCHED(c);
      c.launches += 3;
      SI_CUDA(cudaMemcpyAsync(c.hbuf, s, sizeof(double) * 8, cudaMemcpyDeviceToHost, c.s));
      SI_CUDA(cudaStreamSynchronize(c.s));
      ++its;
      first = false;
      rn = std::sqrt(c.hbuf[kCgRR]);
      SI_CHECK(std::isfinite(rn) && std::isfinite(c.hbuf[kCgAlpha]), SEAICE_ENONFINITE, "pcg: non-finite iterate");
      SI_CHECK(c.hbuf[kCgPQ] > 0.0, SEAICE_ENONFINITE, "pcg: operator not positive definite (p.Ap <= 0)");
      if (rn <= tol) break;
    }
    S.relres_est = rn / bnorm;
    // explicit residual r = b - A x
    apply_A(c, x, r);
    xpby(c, b, -1.0, r, N);
    rn = norm2(c, r, N);
    if (rn <= tol) {
      converged = true;
      break;
    }
    if (its >= c.p.krylov_maxit) break;
    S.restarts++;
  }
  S.iters = its;
  S.relres_true = rn / bnorm;
  S.converged = converged ? 1 : 0;
  if (st) *st = S;
  return converged ? SEAICE_OK : SEAICE_NOT_CONVERGED;
}

int fgmres_impl(Ctx& c, const double* b, double* x, seaice_krylov_stats* st) {
  SI_CHECK(c.assembled, SEAICE_ESTATE, "fgmres before assemble_jacobian");
  if (c.p.krylov_method == 1) return pcg_impl(c, b, x, st);
  const int m = c.p.restart;
  const long long N = c.N;
  c.V.ensure(c.al, (size_t)(m + 1) * N);
  c.Z.ensure(c.al, (size_t)m * N);
  c.w.ensure(c.al, N);
  c.rk.ensure(c.al, N);
  double* V = c.V.get();
  double* Z = c.Z.get();
  double* w = c.w.get();
  for (auto& e : c.arn_ev)
    if (!e) SI_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  fill(c, x, 0.0, N);
  const double bnorm = norm2(c, b, N);
  seaice_krylov_stats S{0, 0, 1, 0.0, 0.0};
  if (bnorm == 0.0) {
    if (st) *st = S;
    return SEAICE_OK;
  }
  SI_CHECK(std::isfinite(bnorm), SEAICE_ENONFINITE, "fgmres: non-finite right-hand side");
  const double tol = c.p.krylov_rtol * bnorm;
  std::vector<double> H((m + 1) * m), cs(m), sn(m), g(m + 1), h(m + 2), y(m);
  double beta = bnorm;
  const double* r = b;
  int its = 0;
  double est = bnorm;
  bool converged = false;
  while (true) {
    std::fill(H.begin(), H.end(), 0.0);
    std::fill(g.begin(), g.end(), 0.0);
    g[0] = beta;
    scal_copy(c, 1.0 / beta, r, V, N);
    int jd = 0;
    // Arnoldi steps are enqueued one ahead: step j + 1 (V-cycle, SpMV, orthogonalisation; all on
    // the device, v_{j+1} normalised there) is queued before the host waits for step j's scalars,
    // so the GPU does not idle during the host's Givens update.  A step queued past convergence
    // is discarded (it only writes Z_{j+1}, w, V_{j+2} and its own scalar slot).
    auto enqueue = [&](int j) {
      double* vj = V + (long long)j * N;
      double* zj = Z + (long long)j * N;
      precond_apply(c, vj, zj);
      apply_A(c, zj, w);
      arnoldi_enqueue(c, V, N, j + 1, w, N, V + (long long)(j + 1) * N, j & 1);
      SI_CUDA(cudaEventRecord(c.arn_ev[j & 1], c.s));
    };
    enqueue(0);
    for (int j = 0; j < m; ++j) {
      if (j + 1 < m && its + 1 < c.p.krylov_maxit) enqueue(j + 1);
      SI_CUDA(cudaEventSynchronize(c.arn_ev[j & 1]));
      const double* hh = c.hbuf + 64 * (j & 1);
      for (int i = 0; i <= j; ++i) h[i] = hh[i];
      const double hn = std::sqrt(hh[63]);
      SI_CHECK(std::isfinite(hn), SEAICE_ENONFINITE, "fgmres: non-finite Arnoldi vector");
      for (int i = 0; i <= j; ++i) H[i * m + j] = h[i];
      H[(j + 1) * m + j] = hn;
      for (int i = 0; i < j; ++i) {
        const double t = cs[i] * H[i * m + j] + sn[i] * H[(i + 1) * m + j];
        H[(i + 1) * m + j] = -sn[i] * H[i * m + j] + cs[i] * H[(i + 1) * m + j];
        H[i * m + j] = t;
      }
      const double den = std::hypot(H[j * m + j], H[(j + 1) * m + j]);
      cs[j] = H[j * m + j] / den;
      sn[j] = H[(j + 1) * m + j] / den;
      H[j * m + j] = den;
      H[(j + 1) * m + j] = 0.0;
      g[j + 1] = -sn[j] * g[j];
      g[j] = cs[j] * g[j];
      ++its;
      jd = j + 1;
      est = std::fabs(g[j + 1]);
      if (est <= tol || hn == 0.0 || its >= c.p.krylov_maxit) break;
    }
    // y = H^-1 g (upper triangular), x += Z y
    for (int i = jd - 1; i >= 0; --i) {
      double t = g[i];
      for (int k = i + 1; k < jd; ++k) t -= H[i * m + k] * y[k];
      y[i] = t / H[i * m + i];
    }
    multi_axpy(c, Z, N, jd, y.data(), x, N);
    // explicit residual r = b - A x
    apply_A(c, x, c.rk.get());
    xpby(c, b, -1.0, c.rk.get(), N);
    beta = norm2(c, c.rk.get(), N);
    r = c.rk.get();
    S.relres_est = est / bnorm;
    if (beta <= tol) {
      converged = true;
      break;
    }
    if (its >= c.p.krylov_maxit) break;
    S.restarts++;
  }
  S.iters = its;
  S.relres_true = beta / bnorm;
  S.converged = converged ? 1 : 0;
  if (st) *st = S;
  return converged ? SEAICE_OK : SEAICE_NOT_CONVERGED;
}

}  // namespace seaice
