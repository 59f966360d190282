// transport.cu — explicit transport of the ice concentration A and mean thickness h between
// implicit momentum steps (eq:model:A / eq:model:H; "an explicit time
// step (e.g., an explicit Euler step)").  Reading G28: first-order upwind finite
// volumes on the Q0 cells, face-normal velocity = mean of the face's two Q1 nodal velocities,
// explicit Euler, A clamped to [0, 1] and h to [0, inf) (A in [0,1]).  One thread per
// cell; both fields in one pass (the face velocities are shared); out of place.  HBM-bound:
// 32 B per cell read (A, h) + 16 B per node (v) + 32 B per cell written, neighbour values and
// node velocities are L1/L2 hits.
#include "ctx.cuh"

namespace seaice {

__global__ void k_transport(int n, double dt_dx, const double2* __restrict__ v, const double* __restrict__ A,
                            const double* __restrict__ H, double A_in, double H_in, double* __restrict__ Ao,
                            double* __restrict__ Ho) {
  const int cell = blockIdx.x * blockDim.x + threadIdx.x;
  if (cell >= n * n) return;
  const int i = cell % n, j = cell / n, s = n + 1;
  const int nd = j * s + i;
  const double2 v00 = __ldg(v + nd), v10 = __ldg(v + nd + 1), v01 = __ldg(v + nd + s), v11 = __ldg(v + nd + s + 1);
  const double uw = 0.5 * (v00.x + v01.x), ue = 0.5 * (v10.x + v11.x);  // x-normal faces
  const double us = 0.5 * (v00.y + v10.y), un = 0.5 * (v01.y + v11.y);  // y-normal faces
  const double a = A[cell], h = H[cell];
  const double aw = i > 0 ? __ldg(A + cell - 1) : A_in, hw = i > 0 ? __ldg(H + cell - 1) : H_in;
  const double ae = i + 1 < n ? __ldg(A + cell + 1) : A_in, he = i + 1 < n ? __ldg(H + cell + 1) : H_in;
  const double as = j > 0 ? __ldg(A + cell - n) : A_in, hs = j > 0 ? __ldg(H + cell - n) : H_in;
  const double an = j + 1 < n ? __ldg(A + cell + n) : A_in, hn = j + 1 < n ? __ldg(H + cell + n) : H_in;
  // net outflow sum_f u_f q_upwind (outward normals: -x, +x, -y, +y)
  const double fa = -uw * (uw > 0.0 ? aw : a) + ue * (ue > 0.0 ? a : ae) - us * (us > 0.0 ? as : a) +
                    un * (un > 0.0 ? a : an);
  const double fh = -uw * (uw > 0.0 ? hw : h) + ue * (ue > 0.0 ? h : he) - us * (us > 0.0 ? hs : h) +
                    un * (un > 0.0 ? h : hn);
  Ao[cell] = fmin(fmax(a - dt_dx * fa, 0.0), 1.0);
  Ho[cell] = fmax(h - dt_dx * fh, 0.0);
}

void transport_impl(Ctx& c, double dt, const double* v, const double* A, const double* H, double A_in, double H_in,
                    double* Ao, double* Ho) {
  SI_CHECK(v && A && H && Ao && Ho, SEAICE_EINVAL, "transport: NULL field");
  SI_CHECK(Ao != A && Ho != H && Ao != H && Ho != A, SEAICE_EINVAL, "transport: outputs must not alias inputs");
  SI_CHECK(std::isfinite(dt) && dt >= 0.0, SEAICE_EINVAL, "transport: dt must be finite and >= 0");
  const double dx = c.ph.dx;
  prof_begin(c);
  k_transport<<<grid_for((long long)c.n * c.n), kThreads, 0, c.s>>>(c.n, dt / dx, reinterpret_cast<const double2*>(v), A,
                                                                   H, A_in, H_in, Ao, Ho);
  SI_LAUNCHED(c);
  prof_end(c, PC_TRANSPORT, 64.0 * c.Nc + 16.0 * c.Nn);
}

}  // namespace seaice
