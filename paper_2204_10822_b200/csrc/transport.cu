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

// Courant number of the upwind update per cell: dt/dx * (sum of outflow face velocities); the
// update a' = a (1 - dt/dx out) + dt/dx sum_in u a_nb is monotone (and A stays in [0,1] without
// the clamp) iff it is <= 1.  Max over cells: order-independent, so the integer atomicMax on the
// bit pattern of a non-negative double is deterministic.
__global__ void k_transport_cfl(int n, double dt_dx, const double2* __restrict__ v,
                                unsigned long long* __restrict__ out) {
  __shared__ double sh[32];
  double m = 0.0;
  for (int cell = blockIdx.x * blockDim.x + threadIdx.x; cell < n * n; cell += gridDim.x * blockDim.x) {
    const int i = cell % n, j = cell / n, s = n + 1;
    const int nd = j * s + i;
    const double2 v00 = __ldg(v + nd), v10 = __ldg(v + nd + 1), v01 = __ldg(v + nd + s), v11 = __ldg(v + nd + s + 1);
    const double uw = 0.5 * (v00.x + v01.x), ue = 0.5 * (v10.x + v11.x);
    const double us = 0.5 * (v00.y + v10.y), un = 0.5 * (v01.y + v11.y);
    const double out_sum = fmax(-uw, 0.0) + fmax(ue, 0.0) + fmax(-us, 0.0) + fmax(un, 0.0);
    m = fmax(m, dt_dx * out_sum);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_down_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) m = fmax(m, sh[w]);
    atomicMax(out, (unsigned long long)__double_as_longlong(m));
  }
}

void transport_impl(Ctx& c, double dt, const double* v, const double* A, const double* H, double A_in, double H_in,
                    double* Ao, double* Ho, double* cfl_out, int* substeps_out) {
  SI_CHECK(v && A && H && Ao && Ho, SEAICE_EINVAL, "transport: NULL field");
  SI_CHECK(Ao != A && Ho != H && Ao != H && Ho != A, SEAICE_EINVAL, "transport: outputs must not alias inputs");
  SI_CHECK(std::isfinite(dt) && dt >= 0.0, SEAICE_EINVAL, "transport: dt must be finite and >= 0");
  const double dx = c.ph.dx;
  const long long Nc = (long long)c.n * c.n;
  // CFL guard (reading G28): m = ceil(CFL) explicit sub-steps of dt/m when CFL > 1
  c.lwork.ensure(c.al, 1);
  SI_CUDA(cudaMemsetAsync(c.lwork.get(), 0, sizeof(long long), c.s));
  k_transport_cfl<<<red_grid(Nc), kThreads, 0, c.s>>>(c.n, dt / dx, reinterpret_cast<const double2*>(v),
                                                      reinterpret_cast<unsigned long long*>(c.lwork.get()));
  SI_LAUNCHED(c);
  SI_CUDA(cudaMemcpyAsync(c.hbuf + 128, c.lwork.get(), sizeof(double), cudaMemcpyDeviceToHost, c.s));
  SI_CUDA(cudaStreamSynchronize(c.s));
  const double cfl = c.hbuf[128];
  SI_CHECK(std::isfinite(cfl), SEAICE_ENONFINITE, "transport: non-finite velocity");
  const int m = cfl > 1.0 ? (int)std::ceil(cfl) : 1;
  SI_CHECK(m <= 100000, SEAICE_EINVAL, "transport: CFL number above 1e5");
  if (cfl_out) *cfl_out = cfl;
  if (substeps_out) *substeps_out = m;
  const double* a_in = A;
  const double* h_in = H;
  if (m > 1) c.dwork.ensure(c.al, 2 * Nc);
  for (int k = 0; k < m; ++k) {
    // ping-pong so that the last sub-step writes (Ao, Ho); scratch = dwork
    const bool to_out = ((m - 1 - k) % 2) == 0;
    double* a_o = to_out ? Ao : c.dwork.get();
    double* h_o = to_out ? Ho : c.dwork.get() + Nc;
    prof_begin(c);
    k_transport<<<grid_for(Nc), kThreads, 0, c.s>>>(c.n, dt / m / dx, reinterpret_cast<const double2*>(v), a_in, h_in,
                                                    A_in, H_in, a_o, h_o);
    SI_LAUNCHED(c);
    prof_end(c, PC_TRANSPORT, 64.0 * c.Nc + 16.0 * c.Nn);
    a_in = a_o;
    h_in = h_o;
  }
}

}  // namespace seaice
