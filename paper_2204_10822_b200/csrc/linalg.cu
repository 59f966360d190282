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

// h[i] = V_i . w for i < k (classical Gram-Schmidt projections), chunks of 8 vectors.
template <int CH>
__global__ void __launch_bounds__(256) k_multidot(long long n, const double* __restrict__ V, long long ld, int k0,
                                                  int k, const double* __restrict__ w, double* __restrict__ part) {
  __shared__ double sh[32];
  double acc[CH];
#pragma unroll
  for (int t = 0; t < CH; ++t) acc[t] = 0.0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const double wi = w[i];
#pragma unroll
    for (int t = 0; t < CH; ++t)
      if (k0 + t < k) acc[t] += V[(long long)(k0 + t) * ld + i] * wi;
  }
#pragma unroll
  for (int t = 0; t < CH; ++t) {
    if (k0 + t < k) {
      const double s = block_sum(acc[t], sh);
      if (threadIdx.x == 0) part[(long long)(k0 + t) * gridDim.x + blockIdx.x] = s;
    }
  }
}

void multidot(Ctx& c, const double* V, long long ld, int k, const double* w, long long n, double* h_host) {
  const int g = red_grid(n);
  c.part.ensure(c.al, (size_t)g * (k + 8));
  prof_begin(c);
  for (int k0 = 0; k0 < k; k0 += 8) {
    k_multidot<8><<<g, 256, 0, c.s>>>(n, V, ld, k0, k, w, c.part.get());
    SI_LAUNCHED(c);
  }
  prof_end(c, PC_MDOT, 8.0 * (k + 1) * n);
  finish_cols(c, g, k, h_host);
}

// w -= sum_i h_i V_i, then partial ||w||^2.
__global__ void __launch_bounds__(256) k_multi_axpy_norm(long long n, const double* __restrict__ V, long long ld, int k,
                                                         const double* __restrict__ h, double* __restrict__ w,
                                                         double* __restrict__ part) {
  __shared__ double sh[32];
  __shared__ double hs[64];
  if (threadIdx.x < k) hs[threadIdx.x] = h[threadIdx.x];
  __syncthreads();
  double s = 0.0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    double wi = w[i];
    for (int t = 0; t < k; ++t) wi -= hs[t] * V[(long long)t * ld + i];
    w[i] = wi;
    s += wi * wi;
  }
  s = block_sum(s, sh);
  if (threadIdx.x == 0) part[blockIdx.x] = s;
}

double multi_axpy_norm(Ctx& c, const double* V, long long ld, int k, const double* h_host, double* w, long long n) {
  SI_CHECK(k <= 64, SEAICE_EINVAL, "multi_axpy: k > 64");
  const int g = red_grid(n);
  c.part.ensure(c.al, (size_t)g * 40);
  // pageable source: the runtime stages it before returning, so h_host may be reused at once
  SI_CUDA(cudaMemcpyAsync(c.scal.get() + 64, h_host, sizeof(double) * k, cudaMemcpyHostToDevice, c.s));
  prof_begin(c);
  k_multi_axpy_norm<<<g, 256, 0, c.s>>>(n, V, ld, k, c.scal.get() + 64, w, c.part.get());
  SI_LAUNCHED(c);
  prof_end(c, PC_MAXPY_NORM, 8.0 * (k + 2) * n);
  double r;
  finish_cols(c, g, 1, &r);
  return std::sqrt(r);
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
