// linalg.cu — finest-level stencil SpMV (K3), block-CSR SpMV, vector kernels and the
// fused Krylov multi-dot / multi-axpy kernels (K7/K8/K10, K21).  fp64, HBM-bound.
// Reductions are two-stage with a fixed grid: results are bitwise reproducible.
#include <algorithm>
#include <cstring>

#include "ctx.cuh"
#include "stencil.cuh"

namespace seaice {

// ------------------------------------------------------------------ stencil SpMV
// y = J x with J in the symmetric 19-value slot-major SoA storage of stencil.cuh: every load of
// J is coalesced and no index is read.  x is read as double2 per neighbour node; the 3 node
// lines a warp touches stay in L1/L2, and the lower-neighbour blocks (one node line below) are
// L2 hits, so J crosses HBM once (152 B per node).
__global__ void __launch_bounds__(256) k_stencil_spmv(int n, int Nn, const double* __restrict__ J,
                                                      const double2* __restrict__ x, double2* __restrict__ y) {
  const int node = blockIdx.x * blockDim.x + threadIdx.x;
  if (node >= Nn) return;
  const int s = n + 1, i = node % s, j = node / s;
  if (i > 0 && i < n && j > 0 && j < n) {
    y[node] = stencil_apply(J, Nn, s, node, x);
  } else {
    const double2 xv = x[node];
    const double4 D = stencil_diag(J, Nn, node);
    y[node] = make_double2(D.x * xv.x + D.y * xv.y, D.z * xv.x + D.w * xv.y);
  }
}

void stencil_spmv(Ctx& c, const double* x, double* y) {
  prof_begin(c);
  k_stencil_spmv<<<grid_for(c.Nn), 256, 0, c.s>>>(c.n, c.Nn, c.Jst.get(), reinterpret_cast<const double2*>(x),
                                                  reinterpret_cast<double2*>(y));
  SI_LAUNCHED(c);
  prof_end(c, PC_SPMV0, kSpmvBytesNode * c.Nn);
}

// ------------------------------------------------------------------ BSR SpMV
template <int BR, int BC>
__global__ void k_bsr_spmv(int nb, const int* __restrict__ rp, const int* __restrict__ ci,
                           const double* __restrict__ val, const double* __restrict__ x, double* __restrict__ y) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= nb) return;
  double acc[BR];
#pragma unroll
  for (int a = 0; a < BR; ++a) acc[a] = 0.0;
  const int e1 = rp[r + 1];
  for (int e = rp[r]; e < e1; ++e) {
    const int col = ci[e];
    double xv[BC];
#pragma unroll
    for (int b = 0; b < BC; ++b) xv[b] = __ldg(x + (long long)col * BC + b);
    const double* v = val + (long long)e * BR * BC;
#pragma unroll
    for (int a = 0; a < BR; ++a)
#pragma unroll
      for (int b = 0; b < BC; ++b) acc[a] += __ldg(v + a * BC + b) * xv[b];
  }
#pragma unroll
  for (int a = 0; a < BR; ++a) y[(long long)r * BR + a] = acc[a];
}

template <int BR, int BC>
static void launch_bsr(Ctx& c, int nb, const int* rp, const int* ci, const double* val, const double* x, double* y) {
  k_bsr_spmv<BR, BC><<<grid_for(nb), kThreads, 0, c.s>>>(nb, rp, ci, val, x, y);
  SI_LAUNCHED(c);
}

void bsr_apply(Ctx& c, int nb, int br, int bc, const int* rp, const int* ci, const double* val, const double* x,
               double* y) {
  if (br == 2 && bc == 2) launch_bsr<2, 2>(c, nb, rp, ci, val, x, y);
  else if (br == 3 && bc == 3) launch_bsr<3, 3>(c, nb, rp, ci, val, x, y);
  else if (br == 2 && bc == 3) launch_bsr<2, 3>(c, nb, rp, ci, val, x, y);
  else if (br == 3 && bc == 2) launch_bsr<3, 2>(c, nb, rp, ci, val, x, y);
  else if (br == 4 && bc == 4) launch_bsr<4, 4>(c, nb, rp, ci, val, x, y);
  else if (br == 2 && bc == 4) launch_bsr<2, 4>(c, nb, rp, ci, val, x, y);
  else if (br == 4 && bc == 2) launch_bsr<4, 2>(c, nb, rp, ci, val, x, y);
  else throw Error(SEAICE_EINVAL, "bsr_apply: unsupported block shape");
}

void bsr_spmv(Ctx& c, const Level& L, const double* x, double* y) {
  bsr_apply(c, L.nb, L.b, L.b, L.rp.get(), L.ci.get(), L.val.get(), x, y);
}

// ------------------------------------------------------------------ vectors
__global__ void k_axpy(long long n, double a, const double* __restrict__ x, double* __restrict__ y) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    y[i] += a * x[i];
}
__global__ void k_scal_copy(long long n, double a, const double* __restrict__ x, double* __restrict__ y) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    y[i] = a * x[i];
}
__global__ void k_xpby(long long n, const double* __restrict__ x, double b, double* __restrict__ y) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    y[i] = x[i] + b * y[i];
}
__global__ void k_fill(long long n, double v, double* __restrict__ y) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    y[i] = v;
}

static int vgrid(long long n) { return (int)std::min<long long>((n + kThreads - 1) / kThreads, 148LL * 16); }

void axpy(Ctx& c, double a, const double* x, double* y, long long n) {
  k_axpy<<<vgrid(n), kThreads, 0, c.s>>>(n, a, x, y);
  SI_LAUNCHED(c);
}
void scal_copy(Ctx& c, double a, const double* x, double* y, long long n) {
  k_scal_copy<<<vgrid(n), kThreads, 0, c.s>>>(n, a, x, y);
  SI_LAUNCHED(c);
}
void xpby(Ctx& c, const double* x, double b, double* y, long long n) {
  k_xpby<<<vgrid(n), kThreads, 0, c.s>>>(n, x, b, y);
  SI_LAUNCHED(c);
}
void fill(Ctx& c, double* y, double v, long long n) {
  k_fill<<<vgrid(n), kThreads, 0, c.s>>>(n, v, y);
  SI_LAUNCHED(c);
}
void copy(Ctx& c, double* dst, const double* src, long long n) {
  SI_CUDA(cudaMemcpyAsync(dst, src, sizeof(double) * n, cudaMemcpyDeviceToDevice, c.s));
}

// ------------------------------------------------------------------ reductions
__global__ void k_dot_part(long long n, const double* __restrict__ a, const double* __restrict__ b,
                           double* __restrict__ part) {
  __shared__ double sh[32];
  double s = 0.0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    s += a[i] * b[i];
  s = block_sum(s, sh);
  if (threadIdx.x == 0) part[blockIdx.x] = s;
}

__global__ void k_sum_cols(const double* __restrict__ part, int nparts, int ncols, double* __restrict__ out) {
  __shared__ double sh[32];
  for (int col = 0; col < ncols; ++col) {
    double s = 0.0;
    for (int i = threadIdx.x; i < nparts; i += blockDim.x) s += part[(long long)col * nparts + i];
    s = block_sum(s, sh);
    if (threadIdx.x == 0) out[col] = s;
    __syncthreads();
  }
}

static void finish_cols(Ctx& c, int g, int ncols, double* host) {
  k_sum_cols<<<1, 1024, 0, c.s>>>(c.part.get(), g, ncols, c.scal.get());
  SI_LAUNCHED(c);
  SI_CUDA(cudaMemcpyAsync(c.hbuf, c.scal.get(), sizeof(double) * ncols, cudaMemcpyDeviceToHost, c.s));
  SI_CUDA(cudaStreamSynchronize(c.s));
  std::memcpy(host, c.hbuf, sizeof(double) * ncols);
}

double dot(Ctx& c, const double* a, const double* b, long long n) {
  const int g = red_grid(n);
  c.part.ensure(c.al, (size_t)g * 40);
  k_dot_part<<<g, kThreads, 0, c.s>>>(n, a, b, c.part.get());
  SI_LAUNCHED(c);
  double r;
  finish_cols(c, g, 1, &r);
  return r;
}
double norm2(Ctx& c, const double* a, long long n) { return std::sqrt(dot(c, a, a, n)); }

// h[i] = V_i . w for i < k (classical Gram-Schmidt projections).  One launch: block row y owns
// vectors [8y, 8y + 8) (8 accumulators per thread keep the occupancy high), each thread 2
// consecutive entries (16-byte loads); partial sums combined warp-wise, then across the block's
// warps in a fixed order (deterministic).
constexpr int kMDT = 256, kMDC = 8;
__global__ void __launch_bounds__(kMDT) k_multidot(long long n2, const double2* __restrict__ V, long long ld2, int k,
                                                   const double2* __restrict__ w, double* __restrict__ part) {
  __shared__ double sh[kMDT / 32][kMDC];
  const int k0 = blockIdx.y * kMDC;
  double acc[kMDC];
#pragma unroll
  for (int t = 0; t < kMDC; ++t) acc[t] = 0.0;
  for (long long i = blockIdx.x * (long long)kMDT + threadIdx.x; i < n2; i += (long long)gridDim.x * kMDT) {
    // ptxas keeps two of the eight column loads in flight (SASS: LDG, LDG, DFMA, LDG, DFMA ...);
    // the thread's eight 16-byte pieces are requested up front as L1 prefetches
#pragma unroll
    for (int t = 0; t < kMDC; ++t)
      if (k0 + t < k) asm volatile("prefetch.global.L1 [%0];" ::"l"(V + (k0 + t) * ld2 + i));
    const double2 wi = w[i];
#pragma unroll
    for (int t = 0; t < kMDC; ++t)
      if (k0 + t < k) {
        const double2 v = __ldg(V + (k0 + t) * ld2 + i);
        acc[t] += v.x * wi.x + v.y * wi.y;
      }
  }
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
  for (int t = 0; t < kMDC; ++t) {
    const double v = warp_sum(acc[t]);
    if (lane == 0) sh[wid][t] = v;
  }
  __syncthreads();
  if (threadIdx.x < kMDC && k0 + threadIdx.x < k) {
    double s = 0.0;
#pragma unroll
    for (int q = 0; q < kMDT / 32; ++q) s += sh[q][threadIdx.x];
    part[(long long)(k0 + threadIdx.x) * gridDim.x + blockIdx.x] = s;
  }
}

// w -= sum_i h_i V_i, then partial ||w||^2 (2 entries per thread, 16-byte loads).
__global__ void __launch_bounds__(256) k_multi_axpy_norm(long long n2, const double2* __restrict__ V, long long ld2,
                                                         int k, const double* __restrict__ h,
                                                         double2* __restrict__ w, double* __restrict__ part) {
  __shared__ double sh[32];
  __shared__ double hs[64];
  if (threadIdx.x < k) hs[threadIdx.x] = h[threadIdx.x];
  __syncthreads();
  double s = 0.0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n2; i += (long long)gridDim.x * blockDim.x) {
    double2 wi = w[i];
    int t = 0;
    for (; t + 4 <= k; t += 4) {
      const double2 a0 = __ldg(V + t * ld2 + i), a1 = __ldg(V + (t + 1) * ld2 + i);
      const double2 a2 = __ldg(V + (t + 2) * ld2 + i), a3 = __ldg(V + (t + 3) * ld2 + i);
      wi.x -= hs[t] * a0.x; wi.y -= hs[t] * a0.y;
      wi.x -= hs[t + 1] * a1.x; wi.y -= hs[t + 1] * a1.y;
      wi.x -= hs[t + 2] * a2.x; wi.y -= hs[t + 2] * a2.y;
      wi.x -= hs[t + 3] * a3.x; wi.y -= hs[t + 3] * a3.y;
    }
    for (; t < k; ++t) {
      const double2 a0 = __ldg(V + t * ld2 + i);
      wi.x -= hs[t] * a0.x; wi.y -= hs[t] * a0.y;
    }
    w[i] = wi;
    s += wi.x * wi.x + wi.y * wi.y;
  }
  s = block_sum(s, sh);
  if (threadIdx.x == 0) part[blockIdx.x] = s;
}

// One Arnoldi orthogonalisation step with a single host synchronisation: h = V^T w (device),
// w -= V h, ||w|| (device), v_{k} = w / ||w|| (device), then h and ||w||^2 are copied to the host
// together.  (The previous form round-tripped h through the host before the update.)
__global__ void k_normalize(long long n, const double* __restrict__ w, const double* __restrict__ nrm2,
                            double* __restrict__ out) {
  const double s2 = *nrm2;
  const double a = s2 > 0.0 ? 1.0 / sqrt(s2) : 0.0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    out[i] = a * w[i];
}

void arnoldi_enqueue(Ctx& c, const double* V, long long ld, int k, double* w, long long n, double* vnext, int slot) {
  SI_CHECK(n % 2 == 0 && ld % 2 == 0, SEAICE_EINVAL, "arnoldi: odd length");
  SI_CHECK(k <= 63, SEAICE_EINVAL, "arnoldi: k > 63");
  const int g = red_grid(n / 2);
  c.part.ensure(c.al, (size_t)g * (k + 8));
  double* hd = c.scal.get() + 64 + 96 * slot;  // h (k values), then ||w||^2 at +64
  double* n2d = hd + 64;
  const double2* V2 = reinterpret_cast<const double2*>(V);
  const double2* w2 = reinterpret_cast<const double2*>(w);
  prof_begin(c);
  k_multidot<<<dim3(g, (k + kMDC - 1) / kMDC), kMDT, 0, c.s>>>(n / 2, V2, ld / 2, k, w2, c.part.get());
  SI_LAUNCHED(c);
  prof_end(c, PC_MDOT, 8.0 * (k + 1) * n);
  k_sum_cols<<<1, 1024, 0, c.s>>>(c.part.get(), g, k, hd);
  SI_LAUNCHED(c);
  prof_begin(c);
  k_multi_axpy_norm<<<g, 256, 0, c.s>>>(n / 2, V2, ld / 2, k, hd, reinterpret_cast<double2*>(w), c.part.get());
  SI_LAUNCHED(c);
  prof_end(c, PC_MAXPY_NORM, 8.0 * (k + 2) * n);
  k_sum_cols<<<1, 1024, 0, c.s>>>(c.part.get(), g, 1, n2d);
  k_normalize<<<vgrid(n), kThreads, 0, c.s>>>(n, w, n2d, vnext);
  SI_LAUNCHED(c);
  double* hh = c.hbuf + 64 * slot;
  SI_CUDA(cudaMemcpyAsync(hh, hd, sizeof(double) * k, cudaMemcpyDeviceToHost, c.s));
  SI_CUDA(cudaMemcpyAsync(hh + 63, n2d, sizeof(double), cudaMemcpyDeviceToHost, c.s));
}

// One Arnoldi orthogonalisation step with a single host synchronisation (kept for callers that
// do not pipeline): h = V^T w, w -= V h, vnext = w / ||w||; returns ||w||.
double arnoldi_step(Ctx& c, const double* V, long long ld, int k, double* w, long long n, double* vnext,
                    double* h_host) {
  arnoldi_enqueue(c, V, ld, k, w, n, vnext, 0);
  SI_CUDA(cudaStreamSynchronize(c.s));
  std::memcpy(h_host, c.hbuf, sizeof(double) * k);
  return std::sqrt(c.hbuf[63]);
}

// x += sum_i y_i Z_i
__global__ void __launch_bounds__(256) k_multi_axpy(long long n, const double* __restrict__ Z, long long ld, int k,
                                                    const double* __restrict__ y, double* __restrict__ x) {
  __shared__ double ys[64];
  if (threadIdx.x < k) ys[threadIdx.x] = y[threadIdx.x];
  __syncthreads();
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    double xi = x[i];
    for (int t = 0; t < k; ++t) xi += ys[t] * Z[(long long)t * ld + i];
    x[i] = xi;
  }
}

void multi_axpy(Ctx& c, const double* Z, long long ld, int k, const double* y_host, double* x, long long n) {
  SI_CHECK(k <= 64, SEAICE_EINVAL, "multi_axpy: k > 64");
  SI_CUDA(cudaMemcpyAsync(c.scal.get() + 128, y_host, sizeof(double) * k, cudaMemcpyHostToDevice, c.s));
  prof_begin(c);
  k_multi_axpy<<<vgrid(n), 256, 0, c.s>>>(n, Z, ld, k, c.scal.get() + 128, x);
  SI_LAUNCHED(c);
  prof_end(c, PC_MAXPY, 8.0 * (k + 2) * n);
}

}  // namespace seaice
