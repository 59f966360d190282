// fem.cuh — per-quadrature-point algebra of the sv Newton step in the orthonormal
// basis of symmetric 2x2 tensors (device side).
//
// Basis E1 = I/sqrt2, E2 = diag(1,-1)/sqrt2, E3 = (e1 e2^T + e2 e1^T)/sqrt2, so for a
// symmetric T: T^ = ((T11+T22)/sqrt2, (T11-T22)/sqrt2, sqrt2 T12) and T:S = T^.S^.
//   tau^(v) = ((e11+e22)/sqrt2, (e11-e22)/(e sqrt2), sqrt2 e12/e)   (tau of P:388-391)
//   Delta   = sqrt(Delta_min^2 + 2 |tau^|^2)
//   sv:   C = (P/Delta) I - (P/(Delta^2 s)) (pi^ tau^T + tau^ pi^T),  s = max(1, sqrt2 |pi^|)
//         (eq:linearSVNewton P:512-525 with eq:modification P:534-539)
//   std:  C = (P/Delta) I - (2P/Delta^3) tau^ tau^T                   (eq:standardNewton P:416-427)
//   picard: C = (P/Delta) I
// Q1 on cell [0,dx]^2, local nodes CCW (0,0),(1,0),(1,1),(0,1); 2x2 Gauss points
// (-g,-g),(g,-g),(g,g),(-g,g), physical weight dx^2/4.  This file is independent of
// oracle/ (which works with 2x2 matrices); only the definitions are shared.
#pragma once
#include <math.h>

namespace seaice {

constexpr double kG = 0.57735026918962576451;       // 1/sqrt(3)
constexpr double kR2I = 0.70710678118654752440;     // 1/sqrt(2)
constexpr double kR2 = 1.41421356237309504880;      // sqrt(2)

__host__ __device__ constexpr double xi_a(int a) { return (a == 1 || a == 2) ? 1.0 : -1.0; }
__host__ __device__ constexpr double eta_a(int a) { return (a >= 2) ? 1.0 : -1.0; }
__host__ __device__ constexpr double xi_q(int q) { return (q == 1 || q == 2) ? kG : -kG; }
__host__ __device__ constexpr double eta_q(int q) { return (q >= 2) ? kG : -kG; }
// N_a at Gauss point q
__host__ __device__ constexpr double Nq(int q, int a) {
  return 0.25 * (1.0 + xi_a(a) * xi_q(q)) * (1.0 + eta_a(a) * eta_q(q));
}
// reference-gradient * 2: physical gradient = value * (1/dx)
__host__ __device__ constexpr double Gx(int q, int a) { return 0.5 * xi_a(a) * (1.0 + eta_a(a) * eta_q(q)); }
__host__ __device__ constexpr double Gy(int q, int a) { return 0.5 * eta_a(a) * (1.0 + xi_a(a) * xi_q(q)); }
// local node offsets
__host__ __device__ constexpr int ox(int a) { return (a == 1 || a == 2) ? 1 : 0; }
__host__ __device__ constexpr int oy(int a) { return (a >= 2) ? 1 : 0; }
// stencil slot of neighbour b seen from node a (both local nodes of one cell)
__host__ __device__ constexpr int slot_ab(int a, int b) { return (oy(b) - oy(a) + 1) * 3 + (ox(b) - ox(a) + 1); }

struct Phys {
  double rho_i, rho_a, rho_o, C_a, C_o, P_star, C, e, delta_min, f_c;
  double dx, dt;
  int n;
};

struct V3 {
  double x, y, z;
};
__device__ __forceinline__ double dot3(const V3& a, const V3& b) { return a.x * b.x + a.y * b.y + a.z * b.z; }

// tau^ of phi = N e_x and N e_y given physical gradient (gx, gy) of N.
__device__ __forceinline__ V3 tau_hat_ex(double gx, double gy, double inv_e) {
  return V3{gx * kR2I, gx * kR2I * inv_e, gy * kR2I * inv_e};
}
__device__ __forceinline__ V3 tau_hat_ey(double gx, double gy, double inv_e) {
  return V3{gy * kR2I, -gy * kR2I * inv_e, gx * kR2I * inv_e};
}
// tau^ from the velocity gradient L[k][m] = d v_k / d x_m
__device__ __forceinline__ V3 tau_hat_grad(double L00, double L01, double L10, double L11, double inv_e) {
  const double e11 = L00, e22 = L11, e12 = 0.5 * (L01 + L10);
  return V3{(e11 + e22) * kR2I, (e11 - e22) * kR2I * inv_e, kR2 * e12 * inv_e};
}
__device__ __forceinline__ V3 pi_hat(double p11, double p12, double p22) {
  return V3{(p11 + p22) * kR2I, (p11 - p22) * kR2I, kR2 * p12};
}
// back from hat coordinates to (T11, T12, T22)
__device__ __forceinline__ void from_hat(const V3& h, double& t11, double& t12, double& t22) {
  t11 = (h.x + h.y) * kR2I;
  t22 = (h.x - h.y) * kR2I;
  t12 = h.z * kR2I;
}

}  // namespace seaice
