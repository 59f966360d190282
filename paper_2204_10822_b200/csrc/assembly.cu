// assembly.cu — per-step setup (K2, K22), fused residual + Jacobian assembly (K1),
// line-search energy differences (K11) and the dual update (K12).
//
// All kernels are atomics-free gathers: one thread per node recomputes the
// quadrature-point quantities of its (up to) four cells, so every matrix value
// and residual entry is written exactly once by one thread (bitwise deterministic).
#include <cmath>
#include <vector>

#include "ctx.cuh"
#include "stencil.cuh"

namespace seaice {

// ------------------------------------------------------------------ K2 / K22
// P = P* h exp(-C (1-A)) (eq:ice-strength); rho_i h; range checks.
__global__ void k_cell_setup(int Nc, Phys ph, const double* __restrict__ h, const double* __restrict__ A,
                             double* __restrict__ P, double* __restrict__ rhoh, int* __restrict__ flag) {
  int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= Nc) return;
  double hc = h[c], Ac = A[c];
  bool bad = !(isfinite(hc) && isfinite(Ac) && hc >= 0.0 && Ac >= 0.0 && Ac <= 1.0);
  if (bad) atomicOr(flag, 1);
  P[c] = ph.P_star * hc * exp(-ph.C * (1.0 - Ac));
  rhoh[c] = ph.rho_i * hc;
}

__global__ void k_check_finite(long long n, const double* __restrict__ x, int* __restrict__ flag, int bit) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i < n && !isfinite(x[i])) atomicOr(flag, bit);
}

// Load the 4 nodal 2-vectors of cell (ci,cj).
__device__ __forceinline__ void load_cell_vec(const double* __restrict__ x, int n, int ci, int cj, double u[4][2]) {
  const int s = n + 1;
  const int n0 = cj * s + ci;
  const int ids[4] = {n0, n0 + 1, n0 + s + 1, n0 + s};
#pragma unroll
  for (int b = 0; b < 4; ++b) {
    double2 t = __ldg(reinterpret_cast<const double2*>(x) + ids[b]);
    u[b][0] = t.x;
    u[b][1] = t.y;
  }
}

// F(phi_{a,k}) contributions of one cell to local node AL (eq:F):
//   sum_q w N_a [rho h v^n - dt rho h f_c e_r x (v^n - v_o) + dt tau_atm(v_a)]_k
template <int AL>
__device__ __forceinline__ void force_cell(const Phys& ph, int ci, int cj, const double* __restrict__ vn,
                                           const double* __restrict__ vo, const double* __restrict__ va,
                                           const double* __restrict__ rhoh, double& f0, double& f1) {
  double un[4][2], uo[4][2], ua[4][2];
  load_cell_vec(vn, ph.n, ci, cj, un);
  load_cell_vec(vo, ph.n, ci, cj, uo);
  load_cell_vec(va, ph.n, ci, cj, ua);
  const double rh = rhoh[cj * ph.n + ci];
  const double w = 0.25 * ph.dx * ph.dx;
  const double ca = ph.C_a * ph.rho_a;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    double vnx = 0, vny = 0, vox = 0, voy = 0, vax = 0, vay = 0;
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const double N = Nq(q, b);
      vnx += N * un[b][0]; vny += N * un[b][1];
      vox += N * uo[b][0]; voy += N * uo[b][1];
      vax += N * ua[b][0]; vay += N * ua[b][1];
    }
    const double sa = ca * sqrt(vax * vax + vay * vay);
    const double dux = vnx - vox, duy = vny - voy;
    // e_r x u = (-u_y, u_x)
    const double gxv = rh * vnx - ph.dt * rh * ph.f_c * (-duy) + ph.dt * sa * vax;
    const double gyv = rh * vny - ph.dt * rh * ph.f_c * (dux) + ph.dt * sa * vay;
    const double wn = w * Nq(q, AL);
    f0 += wn * gxv;
    f1 += wn * gyv;
  }
}

__global__ void k_force(Phys ph, int Nn, const double* __restrict__ vn, const double* __restrict__ vo,
                        const double* __restrict__ va, const double* __restrict__ rhoh,
                        const double* __restrict__ load, double* __restrict__ F) {
  int node = blockIdx.x * blockDim.x + threadIdx.x;
  if (node >= Nn) return;
  const int s = ph.n + 1;
  const int i = node % s, j = node / s;
  double f0 = 0.0, f1 = 0.0;
  if (i > 0 && i < ph.n && j > 0 && j < ph.n) {
    force_cell<2>(ph, i - 1, j - 1, vn, vo, va, rhoh, f0, f1);
    force_cell<3>(ph, i, j - 1, vn, vo, va, rhoh, f0, f1);
    force_cell<1>(ph, i - 1, j, vn, vo, va, rhoh, f0, f1);
    force_cell<0>(ph, i, j, vn, vo, va, rhoh, f0, f1);
    if (load) {
      f0 += load[2 * node];
      f1 += load[2 * node + 1];
    }
  }
  F[2 * node] = f0;
  F[2 * node + 1] = f1;
}

// Velocity gradient of a Q1 field at Gauss point q (physical, 1/dx applied).
template <int Q>
__device__ __forceinline__ void grad_at(const double u[4][2], double inv_dx, double& L00, double& L01, double& L10,
                                        double& L11) {
  L00 = L01 = L10 = L11 = 0.0;
#pragma unroll
  for (int b = 0; b < 4; ++b) {
    L00 += u[b][0] * Gx(Q, b);
    L01 += u[b][0] * Gy(Q, b);
    L10 += u[b][1] * Gx(Q, b);
    L11 += u[b][1] * Gy(Q, b);
  }
  L00 *= inv_dx; L01 *= inv_dx; L10 *= inv_dx; L11 *= inv_dx;
}

// pi = tau(v^n)/Delta(v^n) at every Gauss point (eq:pi; reading G4).
__global__ void k_pi_init(Phys ph, int Nc, const double* __restrict__ v, double* __restrict__ pi) {
  int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= Nc) return;
  const int ci = c % ph.n, cj = c / ph.n;
  double u[4][2];
  load_cell_vec(v, ph.n, ci, cj, u);
  const double inv_dx = 1.0 / ph.dx, inv_e = 1.0 / ph.e;
  double L00, L01, L10, L11;
#define PI_Q(Q)                                                                  \
  {                                                                              \
    grad_at<Q>(u, inv_dx, L00, L01, L10, L11);                                   \
    V3 t = tau_hat_grad(L00, L01, L10, L11, inv_e);                              \
    const double D = sqrt(ph.delta_min * ph.delta_min + 2.0 * dot3(t, t));      \
    V3 p{t.x / D, t.y / D, t.z / D};                                             \
    double p11, p12, p22;                                                        \
    from_hat(p, p11, p12, p22);                                                  \
    pi[(0 * 4 + Q) * (long long)Nc + c] = p11;                                   \
    pi[(1 * 4 + Q) * (long long)Nc + c] = p12;                                   \
    pi[(2 * 4 + Q) * (long long)Nc + c] = p22;                                   \
  }
  PI_Q(0) PI_Q(1) PI_Q(2) PI_Q(3)
#undef PI_Q
}

// ------------------------------------------------------------------ K1 (residual only)
// Contribution of one cell to the two residual rows of its local node AL (eq:A + eq:sigma):
//   R_k  -= sum_q w [rho h v_k N_a + dt (P/Delta) tau^(v).tau^(N_a e_k) - dt (P/2) dN_a/dx_k
//                    - dt C_o rho_o |w| w_k N_a]
template <int AL>
__device__ __forceinline__ void residual_cell(const Phys& ph, int ci, int cj, const double* __restrict__ v,
                                              const double* __restrict__ P, const double* __restrict__ rhoh,
                                              const double* __restrict__ vo, double& r0, double& r1) {
  const int n = ph.n;
  const int cell = cj * n + ci;
  double u[4][2], uo[4][2];
  load_cell_vec(v, n, ci, cj, u);
  load_cell_vec(vo, n, ci, cj, uo);
  const double Pc = P[cell], rh = rhoh[cell];
  const double inv_dx = 1.0 / ph.dx, inv_e = 1.0 / ph.e;
  const double w = 0.25 * ph.dx * ph.dx;
  const double co = ph.C_o * ph.rho_o;
  const double dt = ph.dt;
  const double dmin2 = ph.delta_min * ph.delta_min;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    double vx = 0, vy = 0, ox_ = 0, oy_ = 0;
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      vx += Nq(q, b) * u[b][0];
      vy += Nq(q, b) * u[b][1];
      ox_ += Nq(q, b) * uo[b][0];
      oy_ += Nq(q, b) * uo[b][1];
    }
    double L00 = 0, L01 = 0, L10 = 0, L11 = 0;
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      L00 += u[b][0] * Gx(q, b);
      L01 += u[b][0] * Gy(q, b);
      L10 += u[b][1] * Gx(q, b);
      L11 += u[b][1] * Gy(q, b);
    }
    L00 *= inv_dx; L01 *= inv_dx; L10 *= inv_dx; L11 *= inv_dx;
    const V3 t = tau_hat_grad(L00, L01, L10, L11, inv_e);
    const double D = sqrt(dmin2 + 2.0 * dot3(t, t));
    const double c0 = Pc / D;
    const double wx = ox_ - vx, wy = oy_ - vy;
    const double nw = sqrt(wx * wx + wy * wy);
    const double gxa = Gx(q, AL) * inv_dx, gya = Gy(q, AL) * inv_dx;
    const V3 ta0 = tau_hat_ex(gxa, gya, inv_e);
    const V3 ta1 = tau_hat_ey(gxa, gya, inv_e);
    const double Na = Nq(q, AL);
    r0 -= w * (rh * vx * Na + dt * c0 * dot3(t, ta0) - dt * 0.5 * Pc * gxa - dt * co * nw * wx * Na);
    r1 -= w * (rh * vy * Na + dt * c0 * dot3(t, ta1) - dt * 0.5 * Pc * gya - dt * co * nw * wy * Na);
  }
}

__global__ void __launch_bounds__(128) k_residual(Phys ph, int Nn, const double* __restrict__ v,
                                                  const double* __restrict__ P, const double* __restrict__ rhoh,
                                                  const double* __restrict__ vo, const double* __restrict__ F,
                                                  double* __restrict__ R, double* __restrict__ part) {
  __shared__ double sh[32];
  const int node = blockIdx.x * blockDim.x + threadIdx.x;
  double nrm = 0.0;
  if (node < Nn) {
    const int s = ph.n + 1;
    const int i = node % s, j = node / s;
    const bool interior = (i > 0 && i < ph.n && j > 0 && j < ph.n);
    if (!interior) {
      R[2 * node] = 0.0;
      R[2 * node + 1] = 0.0;
    } else {
      double r0 = F[2 * node], r1 = F[2 * node + 1];
      residual_cell<2>(ph, i - 1, j - 1, v, P, rhoh, vo, r0, r1);
      residual_cell<3>(ph, i, j - 1, v, P, rhoh, vo, r0, r1);
      residual_cell<1>(ph, i - 1, j, v, P, rhoh, vo, r0, r1);
      residual_cell<0>(ph, i, j, v, P, rhoh, vo, r0, r1);
      R[2 * node] = r0;
      R[2 * node + 1] = r1;
      nrm = r0 * r0 + r1 * r1;
    }
  }
  double bs = block_sum(nrm, sh);
  if (threadIdx.x == 0) part[blockIdx.x] = bs;
}

// ------------------------------------------------------------------ K11
// Phi(v + a vt) - Phi(v) per alpha, difference form (reading G12; eq:energy P:261-268).
constexpr int kMaxAlpha = 8;
__global__ void __launch_bounds__(128) k_delta_energy(Phys ph, int Nc, const double* __restrict__ v,
                                                      const double* __restrict__ vt, const double* __restrict__ vn,
                                                      const double* __restrict__ vo, const double* __restrict__ va,
                                                      const double* __restrict__ P, const double* __restrict__ rhoh,
                                                      const double* __restrict__ alphas_d, int count,
                                                      double* __restrict__ part) {
  __shared__ double sh[32];
  double acc[kMaxAlpha], sab[kMaxAlpha];
  double al[kMaxAlpha];
#pragma unroll
  for (int k = 0; k < kMaxAlpha; ++k) {
    acc[k] = 0.0;
    sab[k] = 0.0;
    al[k] = (k < count) ? alphas_d[k] : 0.0;
  }
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c < Nc) {
    const int n = ph.n, ci = c % n, cj = c / n;
    double u[4][2], ut[4][2], un[4][2], uo[4][2], ua[4][2];
    load_cell_vec(v, n, ci, cj, u);
    load_cell_vec(vt, n, ci, cj, ut);
    load_cell_vec(vn, n, ci, cj, un);
    load_cell_vec(vo, n, ci, cj, uo);
    load_cell_vec(va, n, ci, cj, ua);
    const double Pc = P[c], rh = rhoh[c];
    const double inv_dx = 1.0 / ph.dx, inv_e = 1.0 / ph.e;
    const double w = 0.25 * ph.dx * ph.dx, dt = ph.dt;
    const double co3 = ph.C_o * ph.rho_o / 3.0, ca = ph.C_a * ph.rho_a;
    const double dmin2 = ph.delta_min * ph.delta_min;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      double x0 = 0, y0 = 0, xt = 0, yt = 0, xn = 0, yn = 0, xo = 0, yo = 0, xa = 0, ya = 0, xd = 0, yd = 0;
      double A00 = 0, A01 = 0, A10 = 0, A11 = 0, B00 = 0, B01 = 0, B10 = 0, B11 = 0;
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        const double N = Nq(q, b);
        x0 += N * u[b][0]; y0 += N * u[b][1];
        xt += N * ut[b][0]; yt += N * ut[b][1];
        xn += N * un[b][0]; yn += N * un[b][1];
        xd += N * (u[b][0] - un[b][0]); yd += N * (u[b][1] - un[b][1]);  // v - v^n from nodal differences
        xo += N * uo[b][0]; yo += N * uo[b][1];
        xa += N * ua[b][0]; ya += N * ua[b][1];
        A00 += u[b][0] * Gx(q, b); A01 += u[b][0] * Gy(q, b); A10 += u[b][1] * Gx(q, b); A11 += u[b][1] * Gy(q, b);
        B00 += ut[b][0] * Gx(q, b); B01 += ut[b][0] * Gy(q, b); B10 += ut[b][1] * Gx(q, b); B11 += ut[b][1] * Gy(q, b);
      }
      const V3 t0 = tau_hat_grad(A00 * inv_dx, A01 * inv_dx, A10 * inv_dx, A11 * inv_dx, inv_e);
      const V3 tt = tau_hat_grad(B00 * inv_dx, B01 * inv_dx, B10 * inv_dx, B11 * inv_dx, inv_e);
      const double trt = (B00 + B11) * inv_dx;
      const double D0 = sqrt(dmin2 + 2.0 * dot3(t0, t0));
      const double w0x = xo - x0, w0y = yo - y0;
      const double n0 = sqrt(w0x * w0x + w0y * w0y);
      const double sa = ca * sqrt(xa * xa + ya * ya);
      // linear terms: rho h f_c (e_r x (v^n - v_o)).vt - tau_atm.vt
      const double dux = xn - xo, duy = yn - yo;
      const double lin = rh * ph.f_c * (-duy * xt + dux * yt) - sa * (xa * xt + ya * yt);
      const double vtd = xt * xd + yt * yd, vtvt = xt * xt + yt * yt;
      const double tt_t0 = dot3(tt, t0), tt_tt = dot3(tt, tt);
      const double vt_w0 = xt * w0x + yt * w0y;
#pragma unroll
      for (int k = 0; k < kMaxAlpha; ++k) {
        if (k < count) {
          const double a = al[k];
          // 1/2 rho h (|v + a vt|^2 - |v|^2) - rho h v^n.(a vt) = rho h a vt.(v - v^n) + 1/2 rho h a^2 |vt|^2
          const double tmass = rh * a * vtd + 0.5 * rh * a * a * vtvt;
          const V3 t1{t0.x + a * tt.x, t0.y + a * tt.y, t0.z + a * tt.z};
          const double D1 = sqrt(dmin2 + 2.0 * dot3(t1, t1));
          const double dD = 2.0 * a * (2.0 * tt_t0 + a * tt_tt) / (D1 + D0);
          const double tpl = 0.5 * Pc * (dD - a * trt);
          const double w1x = w0x - a * xt, w1y = w0y - a * yt;
          const double n1 = sqrt(w1x * w1x + w1y * w1y);
          const double den = n1 + n0;
          // |w1| - |w0| = (w1 - w0).(w1 + w0)/(|w1| + |w0|), w1 - w0 = -a vt taken exactly
          const double dn = den > 0.0 ? (-a) * (2.0 * vt_w0 - a * vtvt) / den : 0.0;
          const double toc = co3 * dn * (n1 * n1 + n1 * n0 + n0 * n0);
          acc[k] += w * (tmass + dt * (tpl + toc + a * lin));
          sab[k] += w * (fabs(tmass) + dt * (fabs(tpl) + fabs(toc) + fabs(a * lin)));
        }
      }
    }
  }
#pragma unroll
  for (int k = 0; k < kMaxAlpha; ++k) {
    if (k < count) {
      const double bs = block_sum(acc[k], sh);
      if (threadIdx.x == 0) part[(long long)k * gridDim.x + blockIdx.x] = bs;
      const double bsa = block_sum(sab[k], sh);
      if (threadIdx.x == 0) part[(long long)(kMaxAlpha + k) * gridDim.x + blockIdx.x] = bsa;
    }
  }
}

// ------------------------------------------------------------------ K12
// pi~ = -pi + tau/Delta + tau(vt)/Delta - [(tau.tau(vt)) pi + (pi.tau(vt)) tau]/(s Delta^2)
// (eq:tautilde P:504-511 with eq:modification).  mode 0: out = pi~;
// mode 1: out = pi + alpha pi~ (in place allowed), optionally projected (reading G5 flag).
__global__ void k_pi_tilde(Phys ph, int Nc, const double* __restrict__ v, const double* pi,
                           const double* __restrict__ vt, double* out, double alpha, int mode, int project) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= Nc) return;
  const int n = ph.n, ci = c % n, cj = c / n;
  double u[4][2], ut[4][2];
  load_cell_vec(v, n, ci, cj, u);
  load_cell_vec(vt, n, ci, cj, ut);
  const double inv_dx = 1.0 / ph.dx, inv_e = 1.0 / ph.e;
  const double dmin2 = ph.delta_min * ph.delta_min;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    double A00 = 0, A01 = 0, A10 = 0, A11 = 0, B00 = 0, B01 = 0, B10 = 0, B11 = 0;
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      A00 += u[b][0] * Gx(q, b); A01 += u[b][0] * Gy(q, b); A10 += u[b][1] * Gx(q, b); A11 += u[b][1] * Gy(q, b);
      B00 += ut[b][0] * Gx(q, b); B01 += ut[b][0] * Gy(q, b); B10 += ut[b][1] * Gx(q, b); B11 += ut[b][1] * Gy(q, b);
    }
    const V3 t = tau_hat_grad(A00 * inv_dx, A01 * inv_dx, A10 * inv_dx, A11 * inv_dx, inv_e);
    const V3 tt = tau_hat_grad(B00 * inv_dx, B01 * inv_dx, B10 * inv_dx, B11 * inv_dx, inv_e);
    const double D = sqrt(dmin2 + 2.0 * dot3(t, t));
    const long long i0 = (0 * 4 + q) * (long long)Nc + c, i1 = (1 * 4 + q) * (long long)Nc + c,
                    i2 = (2 * 4 + q) * (long long)Nc + c;
    const V3 p = pi_hat(pi[i0], pi[i1], pi[i2]);
    const double s = fmax(1.0, kR2 * sqrt(dot3(p, p)));
    const double iD = 1.0 / D;
    const double k1 = dot3(t, tt) / (s * D * D), k2 = dot3(p, tt) / (s * D * D);
    V3 pt{-p.x + (t.x + tt.x) * iD - (k1 * p.x + k2 * t.x), -p.y + (t.y + tt.y) * iD - (k1 * p.y + k2 * t.y),
          -p.z + (t.z + tt.z) * iD - (k1 * p.z + k2 * t.z)};
    V3 r = pt;
    if (mode == 1) {
      r = V3{p.x + alpha * pt.x, p.y + alpha * pt.y, p.z + alpha * pt.z};
      if (project) {
        const double sc = fmax(1.0, kR2 * sqrt(dot3(r, r)));
        r.x /= sc; r.y /= sc; r.z /= sc;
      }
    }
    double p11, p12, p22;
    from_hat(r, p11, p12, p22);
    out[i0] = p11;
    out[i1] = p12;
    out[i2] = p22;
  }
}

// ------------------------------------------------------------------ CSR view
__global__ void k_csr_values(int n, int Nn, const double* __restrict__ Jst, const int* __restrict__ rp,
                             double* __restrict__ val) {
  const int node = blockIdx.x * blockDim.x + threadIdx.x;
  if (node >= Nn) return;
  const int s = n + 1, i = node % s, j = node / s;
  const bool interior = (i > 0 && i < n && j > 0 && j < n);
  for (int k = 0; k < 2; ++k) {
    const int row = 2 * node + k;
    long long o = rp[row];
    if (!interior) {
      val[o] = 1.0;
      continue;
    }
    double Jr[36];
    stencil_row(Jst, Nn, s, node, Jr);
    for (int sl = 0; sl < 9; ++sl)
      for (int m = 0; m < 2; ++m) val[o++] = Jr[sl * 4 + k * 2 + m];
  }
}

// ------------------------------------------------------------------ host side
static double finish_sum(Ctx& c, const double* part, int nparts);

void set_step_impl(Ctx& c, double dt, double t_new, const double* h, const double* A, const double* v_prev,
                   const double* v_air, const double* v_ocean, const double* load) {
  SI_CHECK(h && A && v_prev && v_air && v_ocean, SEAICE_EINVAL, "set_step: NULL input pointer");
  SI_CHECK(dt > 0.0 && std::isfinite(dt), SEAICE_EINVAL, "set_step: dt must be positive");
  c.dt = dt;
  c.t_new = t_new;
  c.ph.dt = dt;
  cudaStream_t s = c.s;
  SI_CUDA(cudaMemsetAsync(c.flag.get(), 0, sizeof(int) * 4, s));
  SI_CUDA(cudaMemcpyAsync(c.vprev.get(), v_prev, sizeof(double) * c.N, cudaMemcpyDeviceToDevice, s));
  SI_CUDA(cudaMemcpyAsync(c.vair.get(), v_air, sizeof(double) * c.N, cudaMemcpyDeviceToDevice, s));
  SI_CUDA(cudaMemcpyAsync(c.vocean.get(), v_ocean, sizeof(double) * c.N, cudaMemcpyDeviceToDevice, s));
  k_cell_setup<<<grid_for(c.Nc), kThreads, 0, s>>>(c.Nc, c.ph, h, A, c.P.get(), c.rhoh.get(), c.flag.get());
  SI_LAUNCHED(c);
  for (int k = 0; k < 3; ++k) {
    const double* x = k == 0 ? c.vprev.get() : k == 1 ? c.vair.get() : c.vocean.get();
    k_check_finite<<<grid_for(c.N), kThreads, 0, s>>>(c.N, x, c.flag.get(), 2);
    SI_LAUNCHED(c);
  }
  c.have_load = load != nullptr;
  if (load) {
    c.load.ensure(c.al, c.N);
    SI_CUDA(cudaMemcpyAsync(c.load.get(), load, sizeof(double) * c.N, cudaMemcpyDeviceToDevice, s));
    k_check_finite<<<grid_for(c.N), kThreads, 0, s>>>(c.N, c.load.get(), c.flag.get(), 2);
    SI_LAUNCHED(c);
  }
  k_force<<<grid_for(c.Nn), kThreads, 0, s>>>(c.ph, c.Nn, c.vprev.get(), c.vocean.get(), c.vair.get(), c.rhoh.get(),
                                               c.have_load ? c.load.get() : nullptr, c.F.get());
  SI_LAUNCHED(c);
  k_pi_init<<<grid_for(c.Nc), kThreads, 0, s>>>(c.ph, c.Nc, c.vprev.get(), c.pi.get());
  SI_LAUNCHED(c);
  int flag = 0;
  SI_CUDA(cudaMemcpyAsync(c.hbuf, c.flag.get(), sizeof(int), cudaMemcpyDeviceToHost, s));
  SI_CUDA(cudaStreamSynchronize(s));
  std::memcpy(&flag, c.hbuf, sizeof(int));
  c.step_set = false;
  SI_CHECK(!(flag & 1), SEAICE_EINVAL, "set_step: A outside [0,1], h < 0 or non-finite cell field");
  SI_CHECK(!(flag & 2), SEAICE_EINVAL, "set_step: non-finite nodal input");
  c.step_set = true;
  c.assembled = false;
  c.amg_ready = false;
  c.have_r0 = false;
  c.lag_ok = false;  // a new time step starts with a full AMG setup (reading G31)
  c.reuse_ok = false;  // ... and builds its own aggregates (reading G32)
  c.ew_prev_res = 0.0;
  c.ew_prev_eta = 0.0;
  c.ew_ls_failed = false;
}

// ------------------------------------------------------------------ K1, fused residual + Jacobian
// Two-phase, atomics-free: a CTA owns a TX x TY tile of nodes.  Phase 1: one thread per cell of
// the (TX+1) x (TY+1) cells touching the tile computes the packed 8x8 element matrix (upper
// triangle, 36 values) and the 8 element residual terms into shared memory (SoA, bank-conflict
// free).  Phase 2: one thread per node gathers its residual pair and the 19 values of its
// symmetric stencil row (stencil.cuh) from the four adjacent cells and writes them coalesced.
// Each cell's quadrature-point algebra is done once per tile (1.13x recompute for the halo at
// 15 x 16) instead of once per node (4x); every value is written once by one thread.
//
// Per-cell algebra: exact identities of the uniform Q1 cell (Walsh-Hadamard structure):
//  * Phi = [phi_a] (rows phi_a = (1, xi_a, eta_a, xi_a eta_a)) is a signed Hadamard matrix, so a
//    nodal field f has modal coefficients F^ = Phi^T f (one 8-add butterfly) and
//      f(q) = (F0 + xi_q F1 + eta_q F2 + xi_q eta_q F3)/4,  df/dx = (F1 + eta F3)/(2dx),
//      df/dy = (F2 + xi F3)/(2dx):  tau^(v)(q) is affine in (xi_q, eta_q) with 7 coefficients.
//  * tau^(N_a e_k)(q) = W_{q,k} mode_a/(2dx), mode_a = (xi_a, eta_a, xi_a eta_a), with the columns
//    of W in span{p1, p2, p3}: p1 = (al, be, 0), p2 = (0, 0, be), p3 = (al, -be, 0)
//    (al = 1/sqrt2, be = 1/(sqrt2 e)), so the viscous element stiffness
//    sum_q w dt tau^_a . C_q tau^_b (eq:linearSVNewton + eq:modification) is mode_a^T S^km mode_b
//    with S built from the six Q_ij = p_i^T C_q p_j = c0 p_i.p_j - c1 (a_i b_j + a_j b_i),
//    a_i = p_i.pi^, b_i = p_i.tau^.
//  * The per-Gauss-point Q_ij and drag values are parked (9 per q) and reduced to their four
//    q-moments (sum, xi-, eta-, xi*eta-weighted) by the same butterfly.
//  * Each 4x4 component block of the element matrix is E^km = Phi M^km Phi^T with
//      M^km = (1/16) sum_q E_km(q) m_q m_q^T  (mass + ocean drag, m_q = (1, xi_q, eta_q, xi_q eta_q))
//             + [0, 0; 0, S^km]                (viscous stiffness),
//    i.e. one 2-D 4x4 Walsh-Hadamard transform per block.
//  * The element residual stays in per-Gauss-point nodal form (it decides Newton convergence at
//    1e-8: a moment form raised the rounding floor), with -w, dt, 1/dx folded into 5 per-q
//    coefficients.
constexpr int kKE = 36;
__host__ __device__ constexpr int ke_idx(int p, int q) { return p * 8 - p * (p - 1) / 2 + (q - p); }  // p <= q
__host__ __device__ constexpr int lidx(int x, int y) { return y ? (x ? 2 : 3) : (x ? 1 : 0); }

struct ElemH {
  double ka, kb;              // al/(2dx), be/(2dx): tau^ coefficients from unscaled modal gradients
  double al, be;              // 1/sqrt2, 1/(sqrt2 e)
  double ka1, ka2, ka3;       // a_i = p_i . pi^ in terms of (p11, p12, p22)
  double sc;                  // w dt / (2dx)^2
  double pp11, pp13, pp22;    // p_i . p_j
  double mwdtdx;              // -w dt / dx
  double hwdtdx;              // w dt / (2 dx)
  double wdtco;               // w dt C_o rho_o
  double kd;                  // w dt C_o rho_o / 16 (drag block of M^)
  double mass16;              // 4 w / 16 (times rho_i h: consistent mass in M^00)
  double w, dmin2;
};
static ElemH make_elemh(const Phys& ph) {
  ElemH k;
  const double inv_dx = 1.0 / ph.dx;
  k.al = kR2I;
  k.be = kR2I / ph.e;
  k.ka = 0.5 * inv_dx * k.al;
  k.kb = 0.5 * inv_dx * k.be;
  k.ka1 = (k.al + k.be) * kR2I;
  k.ka3 = (k.al - k.be) * kR2I;
  k.ka2 = kR2 * k.be;
  k.w = 0.25 * ph.dx * ph.dx;
  const double wdt = k.w * ph.dt;
  k.sc = wdt * 0.25 * inv_dx * inv_dx;
  k.pp11 = k.al * k.al + k.be * k.be;
  k.pp13 = k.al * k.al - k.be * k.be;
  k.pp22 = k.be * k.be;
  k.mwdtdx = -wdt * inv_dx;
  k.hwdtdx = 0.5 * wdt * inv_dx;
  k.wdtco = wdt * ph.C_o * ph.rho_o;
  k.kd = k.wdtco / 16.0;
  k.mass16 = 4.0 * k.w / 16.0;
  k.dmin2 = ph.delta_min * ph.delta_min;
  return k;
}

// Per-Gauss-point constants (q order (-g,-g), (g,-g), (g,g), (-g,g)); uniform across a warp.
struct QC {
  double xq, eq, x4, e4, xe4;   // xi_q, eta_q, xi_q/4, eta_q/4, xi_q eta_q/4
  double N[4], Gx[4], Gy[4];    // N_a(q), dx * dN_a/dx(q), dx * dN_a/dy(q)
};
__constant__ QC cQ[4];
static void upload_qc() {
  static bool done = false;
  if (done) return;
  QC h[4];
  for (int q = 0; q < 4; ++q) {
    h[q].xq = xi_q(q);
    h[q].eq = eta_q(q);
    h[q].x4 = 0.25 * xi_q(q);
    h[q].e4 = 0.25 * eta_q(q);
    h[q].xe4 = 0.25 * xi_q(q) * eta_q(q);
    for (int a = 0; a < 4; ++a) {
      h[q].N[a] = Nq(q, a);
      h[q].Gx[a] = Gx(q, a);
      h[q].Gy[a] = Gy(q, a);
    }
  }
  SI_CUDA(cudaMemcpyToSymbol(cQ, h, sizeof(h)));
  done = true;
}

// F^ = Phi^T f: (f0+f1+f2+f3, -f0+f1+f2-f3, -f0-f1+f2+f3, f0-f1+f2-f3)
__device__ __forceinline__ void had_t(double f0, double f1, double f2, double f3, double F[4]) {
  const double s02 = f0 + f2, d02 = f2 - f0, s13 = f1 + f3, d13 = f1 - f3;
  F[0] = s02 + s13;
  F[1] = d02 + d13;
  F[2] = d02 - d13;
  F[3] = s02 - s13;
}
// y_a = phi_a . r for a = 0..3 (phi_0 = (1,-1,-1,1), phi_1 = (1,1,-1,-1), phi_2 = 1, phi_3 = (1,-1,1,-1))
__device__ __forceinline__ void had_n(double r0, double r1, double r2, double r3, double y[4]) {
  const double s03 = r0 + r3, d03 = r0 - r3, s12 = r1 + r2, d12 = r1 - r2;
  y[0] = s03 - s12;
  y[1] = d03 + d12;
  y[2] = s03 + s12;
  y[3] = d03 - d12;
}
// E = Phi M Phi^T for a 4x4 M (row-major); SYM: M symmetric, only a <= b of E is used.
template <bool SYM>
__device__ __forceinline__ void had2(const double M[16], double E[16]) {
  double T[16];  // T[i][b] = (M phi_b)_i
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    double y[4];
    had_n(M[4 * i], M[4 * i + 1], M[4 * i + 2], M[4 * i + 3], y);
#pragma unroll
    for (int b = 0; b < 4; ++b) T[4 * i + b] = y[b];
  }
#pragma unroll
  for (int b = 0; b < 4; ++b) {
    double y[4];
    had_n(T[b], T[4 + b], T[8 + b], T[12 + b], y);
#pragma unroll
    for (int a = 0; a < 4; ++a) E[4 * a + b] = y[a];  // dead (a > b) entries are removed for SYM
  }
}

__device__ __forceinline__ void cp_async8(unsigned saddr, const double* g) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(saddr), "l"(g) : "memory");
}

template <int KIND, int TC, bool RES = true>
__device__ __forceinline__ void element_had(const ElemH& K, int n, int ci, int cj, const double* __restrict__ v,
                                            const double* __restrict__ vo, const double* __restrict__ pi,
                                            const double* __restrict__ P, const double* __restrict__ rhoh,
                                            double* __restrict__ Ks, double* __restrict__ Rs, int t) {
  const int s = n + 1;
  const long long Nc = (long long)n * n;
  const int cell = cj * n + ci;
  // All per-cell inputs are requested up front (one memory latency instead of one per Gauss
  // point): pi(q, c) is staged asynchronously in this thread's Ks slot 24 + 3q + c (slot 9q + j
  // is only written after pi(q) has been read), P and rho_i h in its Rs slots 0 and 1.
  {
    const unsigned ks = (unsigned)__cvta_generic_to_shared(Ks + t);
    const unsigned rs = (unsigned)__cvta_generic_to_shared(Rs + t);
    if (KIND == SEAICE_JAC_SV) {
#pragma unroll
      for (int q = 0; q < 4; ++q)
#pragma unroll
        for (int c = 0; c < 3; ++c) cp_async8(ks + (24 + 3 * q + c) * TC * 8, pi + (c * 4 + q) * Nc + cell);
    }
    cp_async8(rs, P + cell);
    cp_async8(rs + TC * 8, rhoh + cell);
    asm volatile("cp.async.commit_group;" ::: "memory");
  }
  double X[4], Y[4], WX[4], WY[4];  // modal coefficients of v_x, v_y and of w = v_o - v
  {
    const int nd0 = cj * s + ci;
    double ux[4], uy[4], wx[4], wy[4];
    const int ids[4] = {nd0, nd0 + 1, nd0 + s + 1, nd0 + s};
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const double2 a1 = __ldg(reinterpret_cast<const double2*>(v) + ids[b]);
      const double2 a2 = __ldg(reinterpret_cast<const double2*>(vo) + ids[b]);
      ux[b] = a1.x; uy[b] = a1.y;
      wx[b] = a2.x - a1.x; wy[b] = a2.y - a1.y;
    }
    had_t(ux[0], ux[1], ux[2], ux[3], X);
    had_t(uy[0], uy[1], uy[2], uy[3], Y);
    had_t(wx[0], wx[1], wx[2], wx[3], WX);
    had_t(wy[0], wy[1], wy[2], wy[3], WY);
  }
  asm volatile("cp.async.wait_all;" ::: "memory");
  const double Pc = Rs[t], rh = Rs[TC + t];
  // tau^(v)(q) = (A0 + eta A1 + xi A2, B0 + eta B1 - xi B2, C0 + xi B1 + eta B2)
  const double A0 = K.ka * (X[1] + Y[2]), A1 = K.ka * X[3], A2 = K.ka * Y[3];
  const double B0 = K.kb * (X[1] - Y[2]), B1 = K.kb * X[3], B2 = K.kb * Y[3];
  const double C0 = K.kb * (X[2] + Y[1]);
  X[0] *= 0.25; Y[0] *= 0.25; WX[0] *= 0.25; WY[0] *= 0.25;
  const double scP = K.sc * Pc, mP = K.mwdtdx * Pc, hpw = K.hwdtdx * Pc, wrh = -K.w * rh;
  double Ra[8];
#pragma unroll
  for (int p = 0; p < 8; ++p) Ra[p] = 0.0;
#pragma unroll 1
  for (int q = 0; q < 4; ++q) {
    double p11 = 0.0, p12 = 0.0, p22 = 0.0;
    if (KIND == SEAICE_JAC_SV) {
      const double* ps = Ks + (24 + 3 * q) * TC + t;
      p11 = ps[0]; p12 = ps[TC]; p22 = ps[2 * TC];
    }
    const double xq = cQ[q].xq, eq = cQ[q].eq, x4 = cQ[q].x4, e4 = cQ[q].e4, xe4 = cQ[q].xe4;
    const double vx = fma(x4, X[1], fma(e4, X[2], fma(xe4, X[3], X[0])));
    const double vy = fma(x4, Y[1], fma(e4, Y[2], fma(xe4, Y[3], Y[0])));
    const double wx = fma(x4, WX[1], fma(e4, WX[2], fma(xe4, WX[3], WX[0])));
    const double wy = fma(x4, WY[1], fma(e4, WY[2], fma(xe4, WY[3], WY[0])));
    const double tx = fma(xq, A2, fma(eq, A1, A0));
    const double ty = fma(-xq, B2, fma(eq, B1, B0));
    const double tz = fma(eq, B2, fma(xq, B1, C0));
    const double X2 = fma(2.0, fma(tx, tx, fma(ty, ty, tz * tz)), K.dmin2);  // Delta^2 >= Delta_min^2 > 0
    const double rD = rsqrt(X2);                                              // 1/Delta
    const double alt = K.al * tx;
    const double b1 = fma(K.be, ty, alt), b3 = fma(-K.be, ty, alt), b2 = K.be * tz;
    const double cs = scP * rD;  // sc P/Delta
    double Q11 = cs * K.pp11, Q13 = cs * K.pp13, Q22 = cs * K.pp22, Q33 = Q11, Q12 = 0.0, Q23 = 0.0;
    if (KIND == SEAICE_JAC_SV) {
      const double a1 = fma(K.ka1, p11, K.ka3 * p22), a3 = fma(K.ka3, p11, K.ka1 * p22), a2 = K.ka2 * p12;
      const double pq = 2.0 * fma(p11, p11, fma(p22, p22, 2.0 * p12 * p12));  // 2 |pi^|^2
      const double isf = pq > 1.0 ? rsqrt(pq) : 1.0;                            // 1/max(1, sqrt2 |pi^|)
      const double mc1 = -(cs * rD * isf);                                       // -sc P/(Delta^2 s)
      Q11 = fma(2.0 * mc1, a1 * b1, Q11);
      Q22 = fma(2.0 * mc1, a2 * b2, Q22);
      Q33 = fma(2.0 * mc1, a3 * b3, Q33);
      Q12 = mc1 * fma(a1, b2, a2 * b1);
      Q13 = fma(mc1, fma(a1, b3, a3 * b1), Q13);
      Q23 = mc1 * fma(a2, b3, a3 * b2);
    } else if (KIND == SEAICE_JAC_STD) {
      const double mc1 = -2.0 * cs * (rD * rD);  // -sc 2P/Delta^3
      Q11 = fma(mc1, b1 * b1, Q11);
      Q22 = fma(mc1, b2 * b2, Q22);
      Q33 = fma(mc1, b3 * b3, Q33);
      Q12 = mc1 * (b1 * b2);
      Q13 = fma(mc1, b1 * b3, Q13);
      Q23 = mc1 * (b2 * b3);
    }
    double* slot = Ks + (9 * q) * TC + t;
    slot[0 * TC] = Q11; slot[1 * TC] = Q12; slot[2 * TC] = Q13;
    slot[3 * TC] = Q22; slot[4 * TC] = Q23; slot[5 * TC] = Q33;
    // ocean drag linearisation C_o rho_o (|w| I + w w^T/|w|), w = v_o - v (eq:A), times w dt/16
    const double n2 = fma(wx, wx, wy * wy);
    double nw, r = 0.0;
    if (n2 >= 1e-24) {  // |w| >= 1e-12
      r = rsqrt(n2);
      nw = n2 * r;
    } else {
      nw = sqrt(n2);
    }
    const double wxr = wx * r, wyr = wy * r;
    slot[6 * TC] = K.kd * fma(wxr, wx, nw);
    slot[7 * TC] = K.kd * fma(wyr, wy, nw);
    slot[8 * TC] = K.kd * (wxr * wy);
    // element residual -A(v, phi_{a,k}) (eq:A) = sum_a N_a MX + dN_a/dx CX + dN_a/dy CZ (x row)
    if (!RES) continue;
    const double wdcn = K.wdtco * nw;
    const double MX = fma(wdcn, wx, wrh * vx), MY = fma(wdcn, wy, wrh * vy);
    const double m = mP * rD;  // -w dt P/(Delta dx)
    const double CX = fma(m, b1, hpw), CY = fma(m, b3, hpw), CZ = m * b2;
#pragma unroll
    for (int a = 0; a < 4; ++a) {
      const double Na = cQ[q].N[a], gx = cQ[q].Gx[a], gy = cQ[q].Gy[a];
      Ra[2 * a] = fma(Na, MX, fma(gx, CX, fma(gy, CZ, Ra[2 * a])));
      Ra[2 * a + 1] = fma(Na, MY, fma(gy, CY, fma(gx, CZ, Ra[2 * a + 1])));
    }
  }
  if (RES) {
#pragma unroll
    for (int p = 0; p < 8; ++p) Rs[p * TC + t] = Ra[p];
  }
  // q-moments of the parked values: mom[0] = sum, [1] = sum xi_q/g, [2] = sum eta_q/g, [3] = sum xi_q eta_q * 3
  auto moments = [&](int j, double mom[4]) {
    const double* sl = Ks + j * TC + t;
    had_t(sl[0], sl[9 * TC], sl[18 * TC], sl[27 * TC], mom);
  };
  constexpr double g = kG, g2 = 1.0 / 3.0;
  double S[15];  // s00 s01 s02 s11 s12 s22 s04 s05 s14 s15 s24 s25 s44 s45 s55
  {
    double q11[4], q12[4], q13[4], q22[4], q23[4], q33[4];
    moments(0, q11); moments(1, q12); moments(2, q13); moments(3, q22); moments(4, q23); moments(5, q33);
    S[0] = q11[0];
    S[1] = q12[0];
    S[2] = g * (q11[2] + q12[1]);
    S[3] = q22[0];
    S[4] = g * (q12[2] + q22[1]);
    S[5] = g2 * ((q11[0] + q22[0]) + 2.0 * q12[3]);
    S[6] = q13[0];
    S[7] = g * (q12[2] + q13[1]);
    S[8] = q23[0];
    S[9] = g * (q22[2] + q23[1]);
    S[10] = g * (q13[2] + q23[1]);
    S[11] = g2 * ((q12[0] + q23[0]) + (q13[3] + q22[3]));
    S[12] = q33[0];
    S[13] = g * (q23[2] + q33[1]);
    S[14] = g2 * ((q22[0] + q33[0]) + 2.0 * q23[3]);
  }
  // drag (+ mass) moment matrices (1/16 folded into kd, mass16): mu = (sum, sum xi, sum eta, sum xi eta)
  auto md = [&](const double mu[4], double M[16]) {
    const double m0 = mu[0], mx = g * mu[1], my = g * mu[2], mxy = g2 * mu[3];
    M[0] = m0;       M[1] = mx;        M[2] = my;        M[3] = mxy;
    M[4] = mx;       M[5] = g2 * m0;   M[6] = mxy;       M[7] = g2 * my;
    M[8] = my;       M[9] = mxy;       M[10] = g2 * m0;  M[11] = g2 * mx;
    M[12] = mxy;     M[13] = g2 * my;  M[14] = g2 * mx;  M[15] = (g2 * g2) * m0;
  };
  // S^xx = [s00 s01 s02; s01 s11 s12; s02 s12 s22], S^yy = [s11 s14 s15; s14 s44 s45; s15 s45 s55],
  // S^xy = [s01 s04 s05; s11 s14 s15; s12 s24 s25]   (rows: x modes of a, cols: y modes of b)
  const int sxx[9] = {0, 1, 2, 1, 3, 4, 2, 4, 5};
  const int syy[9] = {3, 8, 9, 8, 12, 13, 9, 13, 14};
  const int sxy[9] = {1, 6, 7, 3, 8, 9, 4, 10, 11};
  const double mass = K.mass16 * rh;
  double mus[3][4];  // all parked values are read before the element matrix overwrites them
  moments(6, mus[0]);  // d00
  moments(7, mus[1]);  // d11
  moments(8, mus[2]);  // d01
  mus[0][0] += mass;
  mus[1][0] += mass;
#pragma unroll
  for (int blk = 0; blk < 3; ++blk) {  // 0: xx, 1: yy, 2: xy
    double M[16], E[16];
    md(mus[blk], M);
#pragma unroll
    for (int r = 0; r < 3; ++r)
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        const int si = blk == 0 ? sxx[3 * r + c] : blk == 1 ? syy[3 * r + c] : sxy[3 * r + c];
        M[4 * (r + 1) + (c + 1)] += S[si];
      }
    if (blk < 2) had2<true>(M, E);
    else had2<false>(M, E);
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        if (blk == 0 && a <= b) Ks[ke_idx(2 * a, 2 * b) * TC + t] = E[4 * a + b];
        if (blk == 1 && a <= b) Ks[ke_idx(2 * a + 1, 2 * b + 1) * TC + t] = E[4 * a + b];
        if (blk == 2) {
          if (a <= b) Ks[ke_idx(2 * a, 2 * b + 1) * TC + t] = E[4 * a + b];  // K_(a,x),(b,y)
          else Ks[ke_idx(2 * b + 1, 2 * a) * TC + t] = E[4 * a + b];        // K_(b,y),(a,x)
        }
      }
  }
}

// Phase 2 of the tiled kernels: the two rows of node (i, j) gathered from its four cells.
template <int TX, int TC>
__device__ __forceinline__ double gather_node_rows(int n, int Nn, int i0, int j0, int i, int j,
                                                   const double* __restrict__ Ks, const double* __restrict__ Rs,
                                                   const double* __restrict__ F, double* __restrict__ Jst,
                                                   double* __restrict__ R) {
  const int s = n + 1;
  const int node = j * s + i;
  if (!(i > 0 && i < n && j > 0 && j < n)) {  // Dirichlet row: identity
#pragma unroll
    for (int e = 0; e < kJS; ++e) Jst[(long long)e * Nn + node] = (e == kJDxx || e == kJDyy) ? 1.0 : 0.0;
    R[2 * node] = 0.0;
    R[2 * node + 1] = 0.0;
    return 0.0;
  }
  // cell cc at offset (cc&1, cc>>1) from (i-1, j-1); the node is its local corner (1-ox, 1-oy)
  const int lc0 = (i - i0) + (j - j0) * (TX + 1);
  double r0 = F[2 * node], r1 = F[2 * node + 1];
#pragma unroll
  for (int cc = 0; cc < 4; ++cc) {
    const int a = lidx(1 - (cc & 1), 1 - (cc >> 1));
    const int lc = lc0 + (cc & 1) + (cc >> 1) * (TX + 1);
    r0 += Rs[(2 * a) * TC + lc];
    r1 += Rs[(2 * a + 1) * TC + lc];
  }
  R[2 * node] = r0;
  R[2 * node + 1] = r1;
  // stencil slots 4 (own block: xx, xy, yy) and 5..8 (E, NW, N, NE: full 2x2 blocks)
#pragma unroll
  for (int sl = 4; sl < 9; ++sl) {
    const int dxs = sl % 3 - 1, dys = sl / 3 - 1;
    const bool bnd = (i + dxs == 0 || i + dxs == n || j + dys == 0 || j + dys == n);  // symmetric elimination
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      if (sl == 4 && e == 2) continue;  // J_yx = J_xy
      const int k = e >> 1, m = e & 1;
      double acc = 0.0;
      bool first = true;
#pragma unroll
      for (int cc = 0; cc < 4; ++cc) {
        const int ax = 1 - (cc & 1), ay = 1 - (cc >> 1);
        const int bx = ax + dxs, by = ay + dys;
        if (bx < 0 || bx > 1 || by < 0 || by > 1) continue;
        const int p = 2 * lidx(ax, ay) + k, q = 2 * lidx(bx, by) + m;
        const int lc = lc0 + (cc & 1) + (cc >> 1) * (TX + 1);
        const double val = Ks[(p <= q ? ke_idx(p, q) : ke_idx(q, p)) * TC + lc];
        acc = first ? val : acc + val;  // no 0.0 + x (not foldable under IEEE signed zeros)
        first = false;
      }
      const int dst = sl == 4 ? kJDxx + (e == 3 ? 2 : e) : (sl - 5) * 4 + e;
      Jst[(long long)dst * Nn + node] = bnd ? 0.0 : acc;
    }
  }
  return r0 * r0 + r1 * r1;
}

// One CTA per tile (persistent CTAs with an L2 prefetch of the next tile measured no faster and
// spilled registers).
template <int TX, int TY>
struct HadTile {
  static constexpr int TC = (TX + 1) * (TY + 1), NT = TC, SMEM = (kKE + 8) * TC * 8;
};

template <int KIND, int TX, int TY>
__global__ void __launch_bounds__(HadTile<TX, TY>::NT, (HadTile<TX, TY>::NT <= 160 ? 4 : 2))
    k_assemble_had(Phys ph, ElemH K, int Nn, int tiles_x, const double* __restrict__ v,
                   const double* __restrict__ pi, const double* __restrict__ P, const double* __restrict__ rhoh,
                   const double* __restrict__ vo, const double* __restrict__ F, double* __restrict__ Jst,
                   double* __restrict__ R, double* __restrict__ part) {
  constexpr int TC = HadTile<TX, TY>::TC;
  extern __shared__ double smem[];
  double* Ks = smem;             // [36][TC]
  double* Rs = smem + kKE * TC;  // [8][TC]
  __shared__ double sh[32];
  const int n = ph.n;
  const int t = threadIdx.x;
  const int i0 = (blockIdx.x % tiles_x) * TX, j0 = (blockIdx.x / tiles_x) * TY;
  {
    const int ci = i0 - 1 + t % (TX + 1), cj = j0 - 1 + t / (TX + 1);
    if (ci >= 0 && ci < n && cj >= 0 && cj < n) element_had<KIND, TC>(K, n, ci, cj, v, vo, pi, P, rhoh, Ks, Rs, t);
  }
  __syncthreads();
  double nrm = 0.0;
  if (t < TX * TY) {
    const int i = i0 + t % TX, j = j0 + t / TX;
    if (i <= n && j <= n) nrm = gather_node_rows<TX, TC>(n, Nn, i0, j0, i, j, Ks, Rs, F, Jst, R);
  }
  const double bs = block_sum(nrm, sh);
  if (threadIdx.x == 0) part[blockIdx.x] = bs;
}

template <int KIND, int TX, int TY>
static int launch_assemble_had_t(Ctx& c, const double* v, const double* pi, double* R) {
  using HT = HadTile<TX, TY>;
  static bool attr = false;
  if (!attr) {
    SI_CUDA(cudaFuncSetAttribute(k_assemble_had<KIND, TX, TY>, cudaFuncAttributeMaxDynamicSharedMemorySize, HT::SMEM));
    attr = true;
  }
  upload_qc();
  const int tx = (c.n + 1 + TX - 1) / TX, ty = (c.n + 1 + TY - 1) / TY;
  const int g = tx * ty;
  c.part.ensure(c.al, g + 64);
  prof_begin(c);
  k_assemble_had<KIND, TX, TY><<<g, HT::NT, HT::SMEM, c.s>>>(c.ph, make_elemh(c.ph), c.Nn, tx, v, pi, c.P.get(),
                                                             c.rhoh.get(), c.vocean.get(), c.F.get(), c.Jst.get(), R,
                                                             c.part.get());
  SI_LAUNCHED(c);
  prof_end(c, PC_ASSEMBLE, kAsmBytesNode * c.Nn + 112.0 * c.Nc);
  return g;
}

// ------------------------------------------------------------------ NEXT-4: matrix-free J x
// Phase 2 of the matrix-free apply: (J x)_node from the element matrices of its four cells and x
// at its 3 x 3 node neighbourhood; Dirichlet columns are eliminated (x_b taken as 0) and Dirichlet
// rows return x, exactly as in the assembled stencil.
template <int TX, int TC>
__device__ __forceinline__ void gather_node_apply(int n, int i0, int j0, int i, int j, const double* __restrict__ Ks,
                                                  const double2* __restrict__ x, double2* __restrict__ y) {
  const int s = n + 1;
  const int node = j * s + i;
  if (!(i > 0 && i < n && j > 0 && j < n)) {
    y[node] = x[node];
    return;
  }
  double2 xn[9];
#pragma unroll
  for (int sl = 0; sl < 9; ++sl) {
    const int ii = i + sl % 3 - 1, jj = j + sl / 3 - 1;
    const bool bnd = (ii == 0 || ii == n || jj == 0 || jj == n);
    xn[sl] = bnd ? make_double2(0.0, 0.0) : __ldg(x + jj * s + ii);
  }
  const int lc0 = (i - i0) + (j - j0) * (TX + 1);
  double y0 = 0.0, y1 = 0.0;
#pragma unroll
  for (int cc = 0; cc < 4; ++cc) {
    const int ax = 1 - (cc & 1), ay = 1 - (cc >> 1);
    const int lc = lc0 + (cc & 1) + (cc >> 1) * (TX + 1);
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const int bx = ox(b), by = oy(b);
      const double2 xv = xn[(by - ay + 1) * 3 + (bx - ax + 1)];
#pragma unroll
      for (int k = 0; k < 2; ++k)
#pragma unroll
        for (int m = 0; m < 2; ++m) {
          const int p = 2 * lidx(ax, ay) + k, q = 2 * b + m;
          const double e = Ks[(p <= q ? ke_idx(p, q) : ke_idx(q, p)) * TC + lc];
          const double xm = m ? xv.y : xv.x;
          if (k == 0) y0 = fma(e, xm, y0);
          else y1 = fma(e, xm, y1);
        }
    }
  }
  y[node] = make_double2(y0, y1);
}

template <int KIND, int TX, int TY>
__global__ void __launch_bounds__(HadTile<TX, TY>::NT, (HadTile<TX, TY>::NT <= 160 ? 4 : 2))
    k_jv_matfree(Phys ph, ElemH K, int tiles_x, const double* __restrict__ v, const double* __restrict__ pi,
                 const double* __restrict__ P, const double* __restrict__ rhoh, const double* __restrict__ vo,
                 const double2* __restrict__ x, double2* __restrict__ y) {
  constexpr int TC = HadTile<TX, TY>::TC;
  extern __shared__ double smem[];
  double* Ks = smem;             // [36][TC]
  double* Rs = smem + kKE * TC;  // [8][TC] (input staging only)
  const int n = ph.n;
  const int t = threadIdx.x;
  const int i0 = (blockIdx.x % tiles_x) * TX, j0 = (blockIdx.x / tiles_x) * TY;
  {
    const int ci = i0 - 1 + t % (TX + 1), cj = j0 - 1 + t / (TX + 1);
    if (ci >= 0 && ci < n && cj >= 0 && cj < n)
      element_had<KIND, TC, false>(K, n, ci, cj, v, vo, pi, P, rhoh, Ks, Rs, t);
  }
  __syncthreads();
  if (t < TX * TY) {
    const int i = i0 + t % TX, j = j0 + t / TX;
    if (i <= n && j <= n) gather_node_apply<TX, TC>(n, i0, j0, i, j, Ks, x, y);
  }
}

template <int KIND>
static void launch_jv_matfree(Ctx& c, const double* v, const double* pi, const double* x, double* y) {
  constexpr int TX = 15, TY = 16;
  using HT = HadTile<TX, TY>;
  static bool attr = false;
  if (!attr) {
    SI_CUDA(cudaFuncSetAttribute(k_jv_matfree<KIND, TX, TY>, cudaFuncAttributeMaxDynamicSharedMemorySize, HT::SMEM));
    attr = true;
  }
  upload_qc();
  const int tx = (c.n + 1 + TX - 1) / TX, ty = (c.n + 1 + TY - 1) / TY;
  prof_begin(c);
  k_jv_matfree<KIND, TX, TY><<<tx * ty, HT::NT, HT::SMEM, c.s>>>(c.ph, make_elemh(c.ph), tx, v, pi, c.P.get(), c.rhoh.get(),
                                                                 c.vocean.get(), reinterpret_cast<const double2*>(x),
                                                                 reinterpret_cast<double2*>(y));
  SI_LAUNCHED(c);
  // algorithmic bytes: v, v_o, x read, y written per node; pi, P, rho_i h per cell
  prof_end(c, PC_MATFREE, 64.0 * c.Nn + 112.0 * c.Nc);
}

void jv_matfree_impl(Ctx& c, const double* v, const double* pi, const double* x, double* y) {
  SI_CHECK(c.step_set, SEAICE_ESTATE, "jv_matfree before set_step");
  SI_CHECK(v && x && y, SEAICE_EINVAL, "jv_matfree: NULL vector");
  SI_CHECK(x != y, SEAICE_EINVAL, "jv_matfree: y must not alias x");
  const double* pp = pi ? pi : c.pi.get();
  if (c.p.jacobian == SEAICE_JAC_SV) launch_jv_matfree<SEAICE_JAC_SV>(c, v, pp, x, y);
  else if (c.p.jacobian == SEAICE_JAC_STD) launch_jv_matfree<SEAICE_JAC_STD>(c, v, pp, x, y);
  else launch_jv_matfree<SEAICE_JAC_PICARD>(c, v, pp, x, y);
}

template <int KIND>
static int launch_assemble_had(Ctx& c, const double* v, const double* pi, double* R) {
  // 15 x 16 node tiles (16 x 17 cells: 1.13x element recompute, 2 CTAs/SM) measured fastest on B200
  // (config 5: 2.18 ms vs 2.23 ms for 31 x 8, 2.27 ms for 31 x 4, 2.47 ms for 15 x 8 at 4 CTAs/SM)
  static const int variant = getenv("SEAICE_ASM_TILE") ? atoi(getenv("SEAICE_ASM_TILE")) : 1;  // tuning aid
  if (variant == 0) return launch_assemble_had_t<KIND, 31, 8>(c, v, pi, R);
  if (variant == 2) return launch_assemble_had_t<KIND, 15, 8>(c, v, pi, R);
  if (variant == 3) return launch_assemble_had_t<KIND, 31, 4>(c, v, pi, R);
  return launch_assemble_had_t<KIND, 15, 16>(c, v, pi, R);
}

static void launch_residual(Ctx& c, const double* v, double* R) {
  const int g = grid_for(c.Nn, 128);
  c.part.ensure(c.al, g + 64);
  prof_begin(c);
  k_residual<<<g, 128, 0, c.s>>>(c.ph, c.Nn, v, c.P.get(), c.rhoh.get(), c.vocean.get(), c.F.get(), R, c.part.get());
  SI_LAUNCHED(c);
  prof_end(c, PC_ASSEMBLE, 64.0 * c.Nn + 16.0 * c.Nc);
}

void assemble_impl(Ctx& c, const double* v, const double* pi, bool jac, double* r_out, double* norm_host) {
  SI_CHECK(c.step_set, SEAICE_ESTATE, "assemble/residual called before set_step");
  SI_CHECK(v, SEAICE_EINVAL, "NULL velocity");
  const double* pp = pi ? pi : c.pi.get();
  double* R = c.R.get();
  const int kind = c.p.jacobian;
  int nparts = grid_for(c.Nn, 128);
  if (!jac) {
    launch_residual(c, v, R);  // residual only: per-node gather
  } else if (kind == SEAICE_JAC_SV) {
    nparts = launch_assemble_had<SEAICE_JAC_SV>(c, v, pp, R);
  } else if (kind == SEAICE_JAC_STD) {
    nparts = launch_assemble_had<SEAICE_JAC_STD>(c, v, pp, R);
  } else {
    nparts = launch_assemble_had<SEAICE_JAC_PICARD>(c, v, pp, R);
  }
  if (r_out) {
    SI_CUDA(cudaMemcpyAsync(r_out, R, sizeof(double) * c.N, cudaMemcpyDeviceToDevice, c.s));
  }
  const double n2 = finish_sum(c, c.part.get(), nparts);
  c.last_res_norm = std::sqrt(n2);
  if (norm_host) *norm_host = c.last_res_norm;
  if (jac) {
    c.assembled = true;
    c.amg_ready = false;
    if (c.p.nullspace_dim == 4) {  // AMG near-nullspace column v_l (reading G30)
      c.lin_v.ensure(c.al, c.N);
      SI_CUDA(cudaMemcpyAsync(c.lin_v.get(), v, sizeof(double) * c.N, cudaMemcpyDeviceToDevice, c.s));
    }
    if (c.p.matfree) {  // the matrix-free FGMRES operator needs the linearisation point
      c.mf_v.ensure(c.al, c.N);
      c.mf_pi.ensure(c.al, 12LL * c.Nc);
      SI_CUDA(cudaMemcpyAsync(c.mf_v.get(), v, sizeof(double) * c.N, cudaMemcpyDeviceToDevice, c.s));
      SI_CUDA(cudaMemcpyAsync(c.mf_pi.get(), pp, sizeof(double) * 12 * c.Nc, cudaMemcpyDeviceToDevice, c.s));
    }
  }
}

// sum of partials -> host (one block, fixed order)
__global__ void k_sum_partials(const double* __restrict__ part, int nparts, int ncols, long long stride,
                               double* __restrict__ out) {
  __shared__ double sh[32];
  for (int col = 0; col < ncols; ++col) {
    double s = 0.0;
    for (int i = threadIdx.x; i < nparts; i += blockDim.x) s += part[col * stride + i];
    s = block_sum(s, sh);
    if (threadIdx.x == 0) out[col] = s;
    __syncthreads();
  }
}

static double finish_sum(Ctx& c, const double* part, int nparts) {
  k_sum_partials<<<1, 1024, 0, c.s>>>(part, nparts, 1, 0, c.scal.get());
  SI_LAUNCHED(c);
  SI_CUDA(cudaMemcpyAsync(c.hbuf, c.scal.get(), sizeof(double), cudaMemcpyDeviceToHost, c.s));
  SI_CUDA(cudaStreamSynchronize(c.s));
  return c.hbuf[0];
}

void delta_energy_impl(Ctx& c, const double* v, const double* vt, const double* alphas, int count, double* out,
                       double* sabs) {
  SI_CHECK(c.step_set, SEAICE_ESTATE, "delta_energy before set_step");
  SI_CHECK(count >= 1 && count <= 32, SEAICE_EINVAL, "delta_energy: 1 <= count <= 32");
  const int g = grid_for(c.Nc, 128);
  c.part.ensure(c.al, (size_t)g * 2 * kMaxAlpha + 64);
  for (int k0 = 0; k0 < count; k0 += kMaxAlpha) {
    const int cnt = std::min(kMaxAlpha, count - k0);
    std::memcpy(c.hbuf, alphas + k0, sizeof(double) * cnt);
    SI_CUDA(cudaMemcpyAsync(c.scal.get() + 32, c.hbuf, sizeof(double) * cnt, cudaMemcpyHostToDevice, c.s));
    prof_begin(c);
    k_delta_energy<<<g, 128, 0, c.s>>>(c.ph, c.Nc, v, vt, c.vprev.get(), c.vocean.get(), c.vair.get(), c.P.get(),
                                        c.rhoh.get(), c.scal.get() + 32, cnt, c.part.get());
    SI_LAUNCHED(c);
    prof_end(c, PC_DENERGY, 80.0 * c.Nn + 16.0 * c.Nc);
    k_sum_partials<<<1, 1024, 0, c.s>>>(c.part.get(), g, 2 * kMaxAlpha, g, c.scal.get());
    SI_LAUNCHED(c);
    SI_CUDA(cudaMemcpyAsync(c.hbuf, c.scal.get(), sizeof(double) * 2 * kMaxAlpha, cudaMemcpyDeviceToHost, c.s));
    SI_CUDA(cudaStreamSynchronize(c.s));
    for (int k = 0; k < cnt; ++k) {
      out[k0 + k] = c.hbuf[k];
      if (sabs) sabs[k0 + k] = c.hbuf[kMaxAlpha + k];
    }
  }
  if (c.have_load) {
    const double lv = dot(c, c.load.get(), vt, c.N);
    for (int k = 0; k < count; ++k) {
      out[k] -= alphas[k] * lv;
      if (sabs) sabs[k] += std::fabs(alphas[k] * lv);
    }
  }
}

void pi_tilde_impl(Ctx& c, const double* v, const double* pi, const double* vt, double* out, double alpha,
                   bool update) {
  SI_CHECK(c.step_set, SEAICE_ESTATE, "pi_tilde before set_step");
  prof_begin(c);
  k_pi_tilde<<<grid_for(c.Nc), kThreads, 0, c.s>>>(c.ph, c.Nc, v, pi, vt, out, alpha, update ? 1 : 0,
                                                    c.p.project_pi);
  SI_LAUNCHED(c);
  prof_end(c, PC_PIUPD, 32.0 * c.Nn + 192.0 * c.Nc);
}

void build_csr_view(Ctx& c, seaice_csr* out) {
  if (!c.csr_pattern) {
    const int n = c.n, s = n + 1;
    std::vector<int> rp(c.N + 1), ci;
    long long nnz = 0;
    for (int node = 0; node < c.Nn; ++node) {
      const int i = node % s, j = node / s;
      const bool interior = (i > 0 && i < n && j > 0 && j < n);
      for (int k = 0; k < 2; ++k) {
        rp[2 * node + k] = (int)nnz;
        nnz += interior ? 18 : 1;
      }
    }
    rp[c.N] = (int)nnz;
    ci.resize(nnz);
    for (int node = 0; node < c.Nn; ++node) {
      const int i = node % s, j = node / s;
      const bool interior = (i > 0 && i < n && j > 0 && j < n);
      for (int k = 0; k < 2; ++k) {
        long long o = rp[2 * node + k];
        if (!interior) {
          ci[o] = 2 * node + k;
          continue;
        }
        for (int sl = 0; sl < 9; ++sl) {
          const int nb = (j + sl / 3 - 1) * s + (i + sl % 3 - 1);
          for (int m = 0; m < 2; ++m) ci[o++] = 2 * nb + m;
        }
      }
    }
    c.csr_rp.ensure(c.al, c.N + 1);
    c.csr_ci.ensure(c.al, nnz);
    c.csr_val.ensure(c.al, nnz);
    SI_CUDA(cudaMemcpyAsync(c.csr_rp.get(), rp.data(), sizeof(int) * (c.N + 1), cudaMemcpyHostToDevice, c.s));
    SI_CUDA(cudaMemcpyAsync(c.csr_ci.get(), ci.data(), sizeof(int) * nnz, cudaMemcpyHostToDevice, c.s));
    SI_CUDA(cudaStreamSynchronize(c.s));
    c.csr_nnz = nnz;
    c.csr_pattern = true;
  }
  k_csr_values<<<grid_for(c.Nn), kThreads, 0, c.s>>>(c.n, c.Nn, c.Jst.get(), c.csr_rp.get(), c.csr_val.get());
  SI_LAUNCHED(c);
  out->nrows = c.N;
  out->ncols = c.N;
  out->nnz = c.csr_nnz;
  out->row_ptr = c.csr_rp.get();
  out->col_idx = c.csr_ci.get();
  out->val = c.csr_val.get();
}

}  // namespace seaice
