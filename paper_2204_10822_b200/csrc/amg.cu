// amg.cu — smoothed-aggregation AMG built on the GPU (K13-K20) and its V-cycle (K4-K6).
//
// Definition: DESIGN.md "AMG definition" (identical to oracle/amg.py's header; the two
// share the definition, not code).  The paper's own preconditioner is BoomerAMG
// (PAPER.md P:985-997), prior art for a CPU cluster; BASELINE.json mandates an
// aggregation AMG with Chebyshev-Jacobi smoothing built on the GPU.
//
// Everything is deterministic: integer atomics only produce counts/flags, sorting uses
// CUB's stable radix / segmented sorts, SpGEMM accumulates each output block in a fixed
// (row-major product) order by a single thread, reductions are fixed-order two-stage.
#include <cub/cub.cuh>
#include <cuda.h>
#include <cooperative_groups.h>

#include <algorithm>
#include <cmath>
#include <vector>

#include "ctx.cuh"
#include "stencil.cuh"

namespace seaice {

void bsr_apply(Ctx& c, int nb, int br, int bc, const int* rp, const int* ci, const double* val, const double* x,
               double* y);

// ------------------------------------------------------------------ hashing (shared definition)
constexpr unsigned long long kGolden = 0x9E3779B97F4A7C15ULL;
__host__ __device__ __forceinline__ unsigned long long splitmix64(unsigned long long z) {
  z += kGolden;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}
__host__ __device__ __forceinline__ unsigned long long salt(unsigned long long seed, int level, int extra) {
  return kGolden * (64ULL * seed + (unsigned long long)(level + extra));
}

// ------------------------------------------------------------------ setup phase timing (debug)
// SEAICE_SETUP_TIMING=1 prints the wall time of each setup phase (synchronising).
static void tick(Ctx& c, const char* what, int lvl) {
  static const bool on = getenv("SEAICE_SETUP_TIMING") != nullptr;
  static double last = 0.0;
  if (!on) return;
  cudaStreamSynchronize(c.s);
  timespec ts;
  clock_gettime(CLOCK_MONOTONIC, &ts);
  const double now = ts.tv_sec * 1e3 + ts.tv_nsec * 1e-6;
  if (what) fprintf(stderr, "[setup] L%d %-12s %8.2f ms\n", lvl, what, now - last);
  last = now;
}

// ------------------------------------------------------------------ scratch helpers
// Setup scratch from the context arena; released (LIFO) when the Scratch goes out of scope.
struct Scratch {
  Ctx& c;
  Arena::Mark m;
  explicit Scratch(Ctx& cc) : c(cc), m(cc.arena.mark()) {}
  template <class T>
  T* get(size_t n) {
    return (T*)c.arena.alloc(c.al, sizeof(T) * std::max<size_t>(n, 1));
  }
  ~Scratch() { c.arena.reset(m); }
};

template <class T>
static void exclusive_scan(Ctx& c, const T* in, T* out, int n) {
  Scratch S(c);
  size_t tmp = 0;
  SI_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp, in, out, n, c.s));
  void* t = S.get<char>(tmp + 16);
  SI_CUDA(cub::DeviceScan::ExclusiveSum(t, tmp, in, out, n, c.s));
  c.launches += 1;
}

template <class T>
static T read_scalar(Ctx& c, const T* dptr) {
  T v;
  SI_CUDA(cudaMemcpyAsync(c.hbuf, dptr, sizeof(T), cudaMemcpyDeviceToHost, c.s));
  SI_CUDA(cudaStreamSynchronize(c.s));
  std::memcpy(&v, c.hbuf, sizeof(T));
  return v;
}

// ------------------------------------------------------------------ level 0 from the stencil
__global__ void k_stencil_to_bsr(int n, int Nn, const double* __restrict__ Jst, const int* __restrict__ rp,
                                 double* __restrict__ val) {
  const int node = blockIdx.x * blockDim.x + threadIdx.x;
  if (node >= Nn) return;
  const int s = n + 1, i = node % s, j = node / s;
  const bool interior = (i > 0 && i < n && j > 0 && j < n);
  long long o = (long long)rp[node] * 4;
  if (!interior) {
    const double4 D = stencil_diag(Jst, Nn, node);
    val[o] = D.x; val[o + 1] = D.y; val[o + 2] = D.z; val[o + 3] = D.w;
    return;
  }
  double Jr[36];
  stencil_row(Jst, Nn, s, node, Jr);
#pragma unroll
  for (int e = 0; e < 36; ++e) val[o + e] = Jr[e];
}

static void build_level0_pattern(Ctx& c, Level& L) {
  const int n = c.n, s = n + 1;
  std::vector<int> rp(c.Nn + 1), ci;
  long long nnzb = 0;
  for (int node = 0; node < c.Nn; ++node) {
    const int i = node % s, j = node / s;
    rp[node] = (int)nnzb;
    nnzb += (i > 0 && i < n && j > 0 && j < n) ? 9 : 1;
  }
  rp[c.Nn] = (int)nnzb;
  ci.resize(nnzb);
  for (int node = 0; node < c.Nn; ++node) {
    const int i = node % s, j = node / s;
    long long o = rp[node];
    if (!(i > 0 && i < n && j > 0 && j < n)) {
      ci[o] = node;
      continue;
    }
    for (int sl = 0; sl < 9; ++sl) ci[o + sl] = (j + sl / 3 - 1) * s + (i + sl % 3 - 1);
  }
  L.nb = c.Nn;
  L.b = 2;
  L.nnzb = nnzb;
  L.rp.ensure(c.al, c.Nn + 1);
  L.ci.ensure(c.al, nnzb);
  SI_CUDA(cudaMemcpyAsync(L.rp.get(), rp.data(), sizeof(int) * (c.Nn + 1), cudaMemcpyHostToDevice, c.s));
  SI_CUDA(cudaMemcpyAsync(L.ci.get(), ci.data(), sizeof(int) * nnzb, cudaMemcpyHostToDevice, c.s));
  SI_CUDA(cudaStreamSynchronize(c.s));
}

// ------------------------------------------------------------------ block inverses
template <int B>
__device__ __forceinline__ bool invert_block(const double* a, double* o) {
  if (B == 2) {
    const double det = a[0] * a[3] - a[1] * a[2];
    if (det == 0.0) return false;
    const double id = 1.0 / det;
    o[0] = a[3] * id; o[1] = -a[1] * id; o[2] = -a[2] * id; o[3] = a[0] * id;
    return true;
  } else if (B == 4) {
    // Gauss-Jordan without pivoting: diagonal blocks of the Galerkin operators are SPD
    // (dropped near-nullspace columns get a unit diagonal, k_fix_zero_diag)
    double m[16];
#pragma unroll
    for (int t = 0; t < 16; ++t) { m[t] = a[t]; o[t] = (t % 5 == 0) ? 1.0 : 0.0; }
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const double p = m[k * 4 + k];
      if (p == 0.0) return false;
      const double ip = 1.0 / p;
#pragma unroll
      for (int j = 0; j < 4; ++j) { m[k * 4 + j] *= ip; o[k * 4 + j] *= ip; }
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        if (i == k) continue;
        const double f = m[i * 4 + k];
#pragma unroll
        for (int j = 0; j < 4; ++j) { m[i * 4 + j] -= f * m[k * 4 + j]; o[i * 4 + j] -= f * o[k * 4 + j]; }
      }
    }
    return true;
  } else {
    const double c00 = a[4] * a[8] - a[5] * a[7];
    const double c01 = a[5] * a[6] - a[3] * a[8];
    const double c02 = a[3] * a[7] - a[4] * a[6];
    const double det = a[0] * c00 + a[1] * c01 + a[2] * c02;
    if (det == 0.0) return false;
    const double id = 1.0 / det;
    o[0] = c00 * id;
    o[1] = (a[2] * a[7] - a[1] * a[8]) * id;
    o[2] = (a[1] * a[5] - a[2] * a[4]) * id;
    o[3] = c01 * id;
    o[4] = (a[0] * a[8] - a[2] * a[6]) * id;
    o[5] = (a[2] * a[3] - a[0] * a[5]) * id;
    o[6] = c02 * id;
    o[7] = (a[1] * a[6] - a[0] * a[7]) * id;
    o[8] = (a[0] * a[4] - a[1] * a[3]) * id;
    return true;
  }
}

template <int B>
__global__ void k_diag_inv(int nb, const int* __restrict__ rp, const int* __restrict__ ci,
                           const double* __restrict__ val, double* __restrict__ dinv, double* __restrict__ dnorm,
                           int* __restrict__ flag) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= nb) return;
  double a[B * B];
#pragma unroll
  for (int t = 0; t < B * B; ++t) a[t] = 0.0;
  for (int e = rp[r]; e < rp[r + 1]; ++e)
    if (ci[e] == r) {
#pragma unroll
      for (int t = 0; t < B * B; ++t) a[t] = val[(long long)e * B * B + t];
    }
  double o[B * B];
  if (!invert_block<B>(a, o)) {
    atomicOr(flag, 4);
#pragma unroll
    for (int t = 0; t < B * B; ++t) o[t] = 0.0;
  }
  double f2 = 0.0;
#pragma unroll
  for (int t = 0; t < B * B; ++t) {
    dinv[(long long)r * B * B + t] = o[t];
    f2 += a[t] * a[t];
  }
  dnorm[r] = sqrt(f2);
}


// y_I = Dinv_I y_I (in place)
template <int B>
__global__ void k_dinv_apply(int nb, const double* __restrict__ dinv, double* __restrict__ y) {
  constexpr int S = (B == 3) ? 4 : B;  // padded coarse vectors (see vstride)
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= nb) return;
  double v[B];
#pragma unroll
  for (int a = 0; a < B; ++a) v[a] = y[(long long)r * S + a];
  const double* D = dinv + (long long)r * B * B;
#pragma unroll
  for (int a = 0; a < B; ++a) {
    double s = 0.0;
#pragma unroll
    for (int b = 0; b < B; ++b) s += D[a * B + b] * v[b];
    y[(long long)r * S + a] = s;
  }
}

__global__ void k_sqnorm_part(long long n, const double* __restrict__ a, double* __restrict__ part) {
  __shared__ double sh[32];
  double s = 0.0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    s += a[i] * a[i];
  s = block_sum(s, sh);
  if (threadIdx.x == 0) part[blockIdx.x] = s;
}
__global__ void k_sum_to(const double* __restrict__ part, int nparts, double* __restrict__ out) {
  __shared__ double sh[32];
  double s = 0.0;
  for (int i = threadIdx.x; i < nparts; i += blockDim.x) s += part[i];
  s = block_sum(s, sh);
  if (threadIdx.x == 0) out[0] = s;
}
__global__ void k_scale_rsqrt(long long n, const double* __restrict__ y, const double* __restrict__ s2,
                              double* __restrict__ x) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i < n) x[i] = y[i] / sqrt(s2[0]);
}

// start vector of the power iteration: entry k = B*row + a of the unpadded vector, written at
// S*row + a of the (possibly padded, S = 4 for B = 3) storage; pads 0
__global__ void k_power_start(long long N, int B, int S, unsigned long long sl, double* __restrict__ x) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= N) return;
  const long long row = i / S;
  const int a = (int)(i - row * S);
  if (a >= B) {
    x[i] = 0.0;
    return;
  }
  const unsigned long long h = splitmix64((unsigned long long)(row * B + a) + sl);
  x[i] = 2.0 * ((double)(h >> 11) * 0x1.0p-53) - 1.0;
}

// ------------------------------------------------------------------ strength
template <int B>
__global__ void k_strength(int nb, const int* __restrict__ rp, const int* __restrict__ ci,
                           const double* __restrict__ val, const double* __restrict__ dnorm, double theta2,
                           double* __restrict__ sval, int* __restrict__ deg) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= nb) return;
  int cnt = 0;
  const double dr = dnorm[r];
  for (int e = rp[r]; e < rp[r + 1]; ++e) {
    const int col = ci[e];
    double f2 = 0.0;
#pragma unroll
    for (int t = 0; t < B * B; ++t) {
      const double v = val[(long long)e * B * B + t];
      f2 += v * v;
    }
    const double dd = dr * dnorm[col];
    const bool strong = (col != r) && (f2 > 0.0) && (f2 >= theta2 * dd);
    sval[e] = strong ? f2 / fmax(dd, 1e-300) : 0.0;
    cnt += strong;
  }
  deg[r] = cnt;
}

__global__ void k_strength_compact(int nb, const int* __restrict__ rp, const int* __restrict__ ci,
                                   const double* __restrict__ sval, const int* __restrict__ grp,
                                   int* __restrict__ gci, double* __restrict__ gs) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= nb) return;
  int o = grp[r];
  for (int e = rp[r]; e < rp[r + 1]; ++e)
    if (sval[e] > 0.0) {
      gci[o] = ci[e];
      gs[o] = sval[e];
      ++o;
    }
}

// ------------------------------------------------------------------ MIS(2)
__global__ void k_mis_init(int nb, const int* __restrict__ grp, unsigned long long sl,
                           unsigned long long* __restrict__ key) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= nb) return;
  const bool iso = grp[r + 1] == grp[r];
  const unsigned long long st = iso ? 0ULL : 1ULL;
  const unsigned long long h = splitmix64((unsigned long long)r + sl) >> 27;
  key[r] = (st << 62) | (h << 25) | (unsigned long long)r;
}

__global__ void k_mis_max(int nb, const int* __restrict__ grp, const int* __restrict__ gci,
                          const unsigned long long* __restrict__ kin, unsigned long long* __restrict__ kout) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= nb) return;
  unsigned long long m = kin[r];
  for (int e = grp[r]; e < grp[r + 1]; ++e) m = max(m, kin[gci[e]]);
  kout[r] = m;
}

__global__ void k_mis_update(int nb, unsigned long long* __restrict__ key, const unsigned long long* __restrict__ T2,
                             int* __restrict__ undecided) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= nb) return;
  const unsigned long long k = key[r];
  if ((k >> 62) != 1ULL) return;
  const unsigned long long t = T2[r];
  const unsigned long long low = k & ((1ULL << 62) - 1);
  if (t == k) {
    key[r] = (2ULL << 62) | low;
  } else if ((t >> 62) == 2ULL) {
    key[r] = low;  // OUT
  } else {
    atomicAdd(undecided, 1);
  }
}

__global__ void k_roots(int nb, const unsigned long long* __restrict__ key, int* __restrict__ isroot) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= nb) return;
  isroot[r] = ((key[r] >> 62) == 2ULL) ? 1 : 0;
}

__global__ void k_agg_roots(int nb, const int* __restrict__ isroot, const int* __restrict__ rootid,
                            int* __restrict__ agg) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= nb) return;
  agg[r] = isroot[r] ? rootid[r] : -1;
}

// One join phase: unassigned non-isolated node joins the aggregate of its strong neighbour
// (assigned in agg_in) with the largest strength, ties to the smallest aggregate id.
__global__ void k_agg_join(int nb, const int* __restrict__ grp, const int* __restrict__ gci,
                           const double* __restrict__ gs, const int* __restrict__ agg_in, int* __restrict__ agg_out) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= nb) return;
  int a = agg_in[r];
  if (a < 0) {
    double best = -1.0;
    int ba = -1;
    for (int e = grp[r]; e < grp[r + 1]; ++e) {
      const int aj = agg_in[gci[e]];
      if (aj < 0) continue;
      const double s = gs[e];
      if (s > best || (s == best && aj < ba)) {
        best = s;
        ba = aj;
      }
    }
    a = ba;
  }
  agg_out[r] = a;
}

// ------------------------------------------------------------------ tentative prolongator
__global__ void k_agg_key(int nb, const int* __restrict__ agg, int na, int* __restrict__ key, int* __restrict__ idx) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= nb) return;
  key[r] = agg[r] >= 0 ? agg[r] : na;
  idx[r] = r;
}

// start offsets of each aggregate in the sorted member list (binary search)
__global__ void k_seg_starts(int na, int nb, const int* __restrict__ skey, int* __restrict__ start) {
  const int a = blockIdx.x * blockDim.x + threadIdx.x;
  if (a > na) return;
  int lo = 0, hi = nb;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (skey[mid] < a) lo = mid + 1;
    else hi = mid;
  }
  start[a] = lo;
}

// Per aggregate: two-pass modified Gram-Schmidt of the stacked near-nullspace rows (B x K per
// member), Q written directly into P_tent's blocks, R into the coarse
// near-nullspace.  One warp per aggregate: lane l owns the stacked rows l, l + 32, ... (row rho
// is component rho % B of member rho / B); the column dot products are xor-butterfly warp sums
// (every lane gets the same fixed-order total).
__device__ __forceinline__ double warp_allsum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
template <int B, int K>
__global__ void __launch_bounds__(128) k_tentative_w(int na, const int* __restrict__ start,
                                                     const int* __restrict__ members, const double* __restrict__ Bn,
                                                     const int* __restrict__ prp, double* __restrict__ pval,
                                                     double* __restrict__ Bc) {
  const int a = (int)((blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5);
  const int lane = threadIdx.x & 31;
  if (a >= na) return;  // uniform per warp
  const int m0 = start[a], m1 = start[a + 1];
  const int nrow = (m1 - m0) * B;
  double R[K * K];
#pragma unroll
  for (int t = 0; t < K * K; ++t) R[t] = 0.0;
  bool keep[K];
#pragma unroll
  for (int k = 0; k < K; ++k) keep[k] = false;
  auto qptr = [&](int rho) -> double* {
    return pval + (long long)prp[members[m0 + rho / B]] * B * K + (rho % B) * K;
  };
#pragma unroll
  for (int k = 0; k < K; ++k) {
    double n0 = 0.0;
    for (int rho = lane; rho < nrow; rho += 32) {
      const int I = members[m0 + rho / B];
      const double v = Bn[((long long)I * B + rho % B) * K + k];
      qptr(rho)[k] = v;
      n0 += v * v;
    }
    n0 = sqrt(warp_allsum(n0));
    for (int pass = 0; pass < 2; ++pass) {
#pragma unroll
      for (int j = 0; j < k; ++j) {
        if (!keep[j]) continue;
        double rj = 0.0;
        for (int rho = lane; rho < nrow; rho += 32) {
          const double* q = qptr(rho);
          rj += q[j] * q[k];
        }
        rj = warp_allsum(rj);
        R[j * K + k] += rj;
        for (int rho = lane; rho < nrow; rho += 32) {
          double* q = qptr(rho);
          q[k] -= rj * q[j];
        }
      }
    }
    double nv = 0.0;
    for (int rho = lane; rho < nrow; rho += 32) {
      const double* q = qptr(rho);
      nv += q[k] * q[k];
    }
    nv = sqrt(warp_allsum(nv));
    keep[k] = (nv > 1e-8 * n0) && (nv > 0.0);
    const double sc = keep[k] ? 1.0 / nv : 0.0;
    if (keep[k]) R[k * K + k] = nv;
    for (int rho = lane; rho < nrow; rho += 32) qptr(rho)[k] *= sc;
  }
  if (lane == 0) {
#pragma unroll
    for (int t = 0; t < K * K; ++t) Bc[(long long)a * K * K + t] = R[t];
  }
}

__global__ void k_flag_agg(int nb, const int* __restrict__ agg, int* __restrict__ f) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r < nb) f[r] = agg[r] >= 0 ? 1 : 0;
}
__global__ void k_ptent_ci(int nb, const int* __restrict__ agg, const int* __restrict__ prp, int* __restrict__ pci) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r < nb && agg[r] >= 0) pci[prp[r]] = agg[r];
}

// ------------------------------------------------------------------ SpGEMM (hand-written)
// C = X Y, block-CSR; X blocks M x K, Y blocks K x P, C blocks M x P.
__global__ void k_spgemm_ub(int nr, const int* __restrict__ xrp, const int* __restrict__ xci,
                            const int* __restrict__ yrp, long long* __restrict__ ub) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r > nr) return;
  if (r == nr) {
    ub[r] = 0;
    return;
  }
  long long s = 0;
  for (int e = xrp[r]; e < xrp[r + 1]; ++e) {
    const int j = xci[e];
    s += yrp[j + 1] - yrp[j];
  }
  ub[r] = s;
}

__global__ void k_spgemm_expand(int nr, const int* __restrict__ xrp, const int* __restrict__ xci,
                                const int* __restrict__ yrp, const int* __restrict__ yci,
                                const long long* __restrict__ off, int* __restrict__ keys) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= nr) return;
  long long o = off[r];
  for (int e = xrp[r]; e < xrp[r + 1]; ++e) {
    const int j = xci[e];
    for (int f = yrp[j]; f < yrp[j + 1]; ++f) keys[o++] = yci[f];
  }
}

__global__ void k_spgemm_count(int nr, const long long* __restrict__ off, const int* __restrict__ keys,
                               int* __restrict__ cnt) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r > nr) return;
  if (r == nr) {
    cnt[r] = 0;
    return;
  }
  int u = 0;
  for (long long k = off[r]; k < off[r + 1]; ++k) u += (k == off[r] || keys[k] != keys[k - 1]);
  cnt[r] = u;
}

__global__ void k_spgemm_compact(int nr, const long long* __restrict__ off, const int* __restrict__ keys,
                                 const int* __restrict__ crp, int* __restrict__ cci) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= nr) return;
  int o = crp[r];
  for (long long k = off[r]; k < off[r + 1]; ++k)
    if (k == off[r] || keys[k] != keys[k - 1]) cci[o++] = keys[k];
}

// ------------------------------------------------------------------ block loads / stores
// A block of N doubles at base + idx * N (bases are 256-byte aligned) is 32-byte aligned when
// N % 4 == 0 and 16-byte aligned when N % 2 == 0: one 32-byte (sm_100 256-bit) or 16-byte access
// per lane touches one L1 sector instead of one per double.  (The numeric SpGEMM kernels were
// L1-sector bound with scalar accesses: ncu l1tex throughput 82 %, 20 sector requests per 4 x 2
// product instead of 5.)
template <int N, bool NC>
__device__ __forceinline__ void ld_blk(const double* p, double (&v)[N]) {
  if constexpr (N % 4 == 0) {
#pragma unroll
    for (int i = 0; i < N; i += 4) {
      if constexpr (NC)
        asm volatile("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];"
                     : "=d"(v[i]), "=d"(v[i + 1]), "=d"(v[i + 2]), "=d"(v[i + 3])
                     : "l"(p + i));
      else
        asm volatile("ld.global.v4.f64 {%0,%1,%2,%3}, [%4];"
                     : "=d"(v[i]), "=d"(v[i + 1]), "=d"(v[i + 2]), "=d"(v[i + 3])
                     : "l"(p + i)
                     : "memory");
    }
  } else if constexpr (N % 2 == 0) {
#pragma unroll
    for (int i = 0; i < N; i += 2) {
      if constexpr (NC)
        asm volatile("ld.global.nc.v2.f64 {%0,%1}, [%2];" : "=d"(v[i]), "=d"(v[i + 1]) : "l"(p + i));
      else
        asm volatile("ld.global.v2.f64 {%0,%1}, [%2];" : "=d"(v[i]), "=d"(v[i + 1]) : "l"(p + i) : "memory");
    }
  } else {
#pragma unroll
    for (int i = 0; i < N; ++i) v[i] = p[i];
  }
}
template <int N>
__device__ __forceinline__ void st_blk(double* p, const double (&v)[N]) {
  if constexpr (N % 4 == 0) {
#pragma unroll
    for (int i = 0; i < N; i += 4)
      asm volatile("st.global.v4.f64 [%0], {%1,%2,%3,%4};" ::"l"(p + i), "d"(v[i]), "d"(v[i + 1]), "d"(v[i + 2]),
                   "d"(v[i + 3])
                   : "memory");
  } else if constexpr (N % 2 == 0) {
#pragma unroll
    for (int i = 0; i < N; i += 2)
      asm volatile("st.global.v2.f64 [%0], {%1,%2};" ::"l"(p + i), "d"(v[i]), "d"(v[i + 1]) : "memory");
  } else {
#pragma unroll
    for (int i = 0; i < N; ++i) p[i] = v[i];
  }
}
// C (M x P) += X (M x K) Y (K x P), C read-modify-written in global memory; same operation order
// per entry as the scalar loop it replaces (s = c; s += x_ak y_kb for k = 0..K-1)
template <int M, int K, int P>
__device__ __forceinline__ void block_fma(double* cb, const double (&xb)[M * K], const double* yb) {
  double c[M * P], y[K * P];
  ld_blk<M * P, false>(cb, c);
  ld_blk<K * P, true>(yb, y);
#pragma unroll
  for (int a = 0; a < M; ++a)
#pragma unroll
    for (int b = 0; b < P; ++b) {
      double s = c[a * P + b];
#pragma unroll
      for (int k = 0; k < K; ++k) s += xb[a * K + k] * y[k * P + b];
      c[a * P + b] = s;
    }
  st_blk<M * P>(cb, c);
}

// the same with the Y block already in registers
template <int M, int K, int P>
__device__ __forceinline__ void block_fma_reg(double* cb, const double (&xb)[M * K], const double (&y)[K * P]) {
  double c[M * P];
  ld_blk<M * P, false>(cb, c);
#pragma unroll
  for (int a = 0; a < M; ++a)
#pragma unroll
    for (int b = 0; b < P; ++b) {
      double s = c[a * P + b];
#pragma unroll
      for (int k = 0; k < K; ++k) s += xb[a * K + k] * y[k * P + b];
      c[a * P + b] = s;
    }
  st_blk<M * P>(cb, c);
}

template <int M, int K, int P>
__global__ void k_spgemm_numeric(int nr, const int* __restrict__ xrp, const int* __restrict__ xci,
                                 const double* __restrict__ xv, const int* __restrict__ yrp,
                                 const int* __restrict__ yci, const double* __restrict__ yv,
                                 const int* __restrict__ crp, const int* __restrict__ cci, double* __restrict__ cv) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= nr) return;
  const int c0 = crp[r], c1 = crp[r + 1];
  for (long long t = (long long)c0 * M * P; t < (long long)c1 * M * P; ++t) cv[t] = 0.0;
  for (int e = xrp[r]; e < xrp[r + 1]; ++e) {
    const int j = xci[e];
    double xb[M * K];
    ld_blk<M * K, true>(xv + (long long)e * M * K, xb);
    int lo_hint = c0;
    for (int f = yrp[j]; f < yrp[j + 1]; ++f) {
      const int col = yci[f];
      // Y row is sorted, so the position is monotone within this row: search from the hint
      int lo = lo_hint, hi = c1;
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (cci[mid] < col) lo = mid + 1;
        else hi = mid;
      }
      lo_hint = lo;
      double* cb = cv + (long long)lo * M * P;
      const double* yb = yv + (long long)f * K * P;
      block_fma<M, K, P>(cb, xb, yb);
    }
  }
}

// Warp-per-row variants (coarse levels have rows of hundreds of blocks): the lanes split
// the inner loop over one Y row; an output block is touched by at most one lane per X
// entry and the X entries are processed in order with __syncwarp between them, so each
// output block is accumulated in exactly the same order as the thread-per-row version.
__global__ void k_spgemm_expand_w(int nr, const int* __restrict__ xrp, const int* __restrict__ xci,
                                  const int* __restrict__ yrp, const int* __restrict__ yci,
                                  const long long* __restrict__ off, int* __restrict__ keys) {
  const int r = (int)((blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5), lane = threadIdx.x & 31;
  if (r >= nr) return;
  long long o = off[r];
  for (int e = xrp[r]; e < xrp[r + 1]; ++e) {
    const int j = xci[e];
    const int f0 = yrp[j], len = yrp[j + 1] - f0;
    for (int t = lane; t < len; t += 32) keys[o + t] = yci[f0 + t];
    o += len;
  }
}

__global__ void k_spgemm_count_w(int nr, const long long* __restrict__ off, const int* __restrict__ keys,
                                 int* __restrict__ cnt) {
  const int r = (int)((blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5), lane = threadIdx.x & 31;
  if (r > nr) return;
  if (r == nr) {
    if (lane == 0) cnt[r] = 0;
    return;
  }
  const long long a = off[r], b = off[r + 1];
  int u = 0;
  for (long long base = a; base < b; base += 32) {
    const long long k = base + lane;
    const bool f = (k < b) && (k == a || keys[k] != keys[k - 1]);
    u += __popc(__ballot_sync(0xffffffffu, f));
  }
  if (lane == 0) cnt[r] = u;
}

__global__ void k_spgemm_compact_w(int nr, const long long* __restrict__ off, const int* __restrict__ keys,
                                   const int* __restrict__ crp, int* __restrict__ cci) {
  const int r = (int)((blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5), lane = threadIdx.x & 31;
  if (r >= nr) return;
  const long long a = off[r], b = off[r + 1];
  int o = crp[r];
  for (long long base = a; base < b; base += 32) {
    const long long k = base + lane;
    const bool f = (k < b) && (k == a || keys[k] != keys[k - 1]);
    const unsigned m = __ballot_sync(0xffffffffu, f);
    if (f) cci[o + __popc(m & ((1u << lane) - 1u))] = keys[k];
    o += __popc(m);
  }
}

template <int M, int K, int P>
__global__ void k_spgemm_numeric_w(int nr, const int* __restrict__ xrp, const int* __restrict__ xci,
                                   const double* __restrict__ xv, const int* __restrict__ yrp,
                                   const int* __restrict__ yci, const double* __restrict__ yv,
                                   const int* __restrict__ crp, const int* __restrict__ cci, double* __restrict__ cv) {
  const int r = (int)((blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5), lane = threadIdx.x & 31;
  if (r >= nr) return;
  const int c0 = crp[r], c1 = crp[r + 1];
  for (long long t = (long long)c0 * M * P + lane; t < (long long)c1 * M * P; t += 32) cv[t] = 0.0;
  __syncwarp();
  for (int e = xrp[r]; e < xrp[r + 1]; ++e) {
    const int j = xci[e];
    double xb[M * K];
    ld_blk<M * K, true>(xv + (long long)e * M * K, xb);
    int lo_hint = c0;
    for (int f = yrp[j] + lane; f < yrp[j + 1]; f += 32) {
      const int col = yci[f];
      int lo = lo_hint, hi = c1;
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (cci[mid] < col) lo = mid + 1;
        else hi = mid;
      }
      lo_hint = lo;
      double* cb = cv + (long long)lo * M * P;
      const double* yb = yv + (long long)f * K * P;
      block_fma<M, K, P>(cb, xb, yb);
    }
    __syncwarp();
  }
}

static int wgrid(long long rows) { return (int)((rows * 32 + 255) / 256); }

// Group-of-G-lanes-per-row numeric phase for short rows (finest level): the same ordering
// argument as k_spgemm_numeric_w with G lanes instead of 32.
template <int M, int K, int P, int G>
__global__ void __launch_bounds__(256) k_spgemm_numeric_g(int nr, const int* __restrict__ xrp,
                                                          const int* __restrict__ xci, const double* __restrict__ xv,
                                                          const int* __restrict__ yrp, const int* __restrict__ yci,
                                                          const double* __restrict__ yv, const int* __restrict__ crp,
                                                          const int* __restrict__ cci, double* __restrict__ cv) {
  const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const int r = (int)(t / G), lig = (int)(t % G);
  const unsigned gmask = ((G == 32) ? 0xffffffffu : ((1u << G) - 1u)) << ((threadIdx.x & 31) & ~(G - 1));
  if (r >= nr) return;  // whole groups exit together (G divides 32)
  const int c0 = crp[r], c1 = crp[r + 1];
  for (long long q = (long long)c0 * M * P + lig; q < (long long)c1 * M * P; q += G) cv[q] = 0.0;
  __syncwarp(gmask);
  for (int e = xrp[r]; e < xrp[r + 1]; ++e) {
    const int j = xci[e];
    double xb[M * K];
#pragma unroll
    for (int q = 0; q < M * K; ++q) xb[q] = xv[(long long)e * M * K + q];
    for (int f = yrp[j] + lig; f < yrp[j + 1]; f += G) {
      const int col = yci[f];
      int lo = c0, hi = c1;
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (cci[mid] < col) lo = mid + 1;
        else hi = mid;
      }
      double* cb = cv + (long long)lo * M * P;
      const double* yb = yv + (long long)f * K * P;
      block_fma<M, K, P>(cb, xb, yb);
    }
    __syncwarp(gmask);
  }
}

// ---- hash-based symbolic/numeric phases (rows whose expansion fits a shared-memory table)
// One warp per row; a per-warp open-addressing table of kHT slots in shared memory holds the
// distinct column ids of the row.  The row's sorted column list is produced by a warp-level
// bitonic sort of the table contents, so the output pattern is identical to the sort-based
// path; the numeric phase looks positions up in the table (no binary search) and accumulates
// in the same X-entry order (bitwise identical values).
// HT: table slots per warp (power of two); HW: warps per block (static smem <= 48 KB)
constexpr int kHT = 1024, kHWarps = 4;    // rows with expansion <= 512
constexpr int kHT2 = 4096, kHWarps2 = 1;  // rows with expansion <= 2048

template <int HT>
__device__ __forceinline__ unsigned hslot(int key) { return ((unsigned)key * 2654435761u) & (HT - 1); }

// insert key; returns 1 if it was new
template <int HT>
__device__ __forceinline__ int hinsert(int* tab, int key) {
  unsigned h = hslot<HT>(key);
  while (true) {
    const int prev = atomicCAS(tab + h, -1, key);
    if (prev == -1) return 1;
    if (prev == key) return 0;
    h = (h + 1) & (HT - 1);
  }
}

// Insert the columns of the Y rows of X entries e0 + l, e0 + l + G, ... (one X entry per lane at a
// time, its Y row walked by that lane): for short Y rows this runs G pointer chains (x column ->
// Y row extent -> Y columns) side by side instead of one after the other with most lanes idle.
// The table is a set, so the insertion order does not matter.  Returns this lane's new-key count.
template <int HT, int G>
__device__ __forceinline__ int sg_insert_by_lane(int e0, int e1, int l, const int* __restrict__ xci,
                                                 const int* __restrict__ yrp, const int* __restrict__ yci, int* tab) {
  int u = 0;
  for (int e = e0 + l; e < e1; e += G) {
    const int j = xci[e];
    const int fb = yrp[j], fe = yrp[j + 1];
    // neighbouring X entries share most of their Y columns: each lane starts its (cyclic) walk at
    // another place, so the lanes do not compare-and-swap the same table slot at the same time
    const int len = fe - fb, rot = len > 0 ? (l * 3) % len : 0;
    for (int q = 0; q < len; q += 4) {
      int cq[4];
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        int o = q + t + rot;
        if (o >= len) o -= len;
        cq[t] = q + t < len ? yci[fb + o] : -1;
      }
#pragma unroll
      for (int t = 0; t < 4; ++t)
        if (cq[t] >= 0) u += hinsert<HT>(tab, cq[t]);
    }
  }
  return u;
}

// Symbolic phase in one table build: the row's distinct column count and its sorted column list,
// written to tmp at the row's expansion offset off[r] (>= the distinct count); k_sg_rows_compact
// then packs the rows into the CSR column array once the counts are scanned (one table build
// instead of a count pass and a column pass).
template <int HT, int HW>
__global__ void __launch_bounds__(32 * HW) k_sg_hash_symbolic(int nr, const int* __restrict__ xrp,
                                                                   const int* __restrict__ xci,
                                                                   const int* __restrict__ yrp,
                                                                   const int* __restrict__ yci,
                                                                   const long long* __restrict__ off,
                                                                   int* __restrict__ cnt, int* __restrict__ tmp,
                                                                   int by_lane) {
  __shared__ int tabs[HW][HT];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int r = blockIdx.x * HW + w;
  if (r > nr) return;
  if (r == nr) {
    if (lane == 0) cnt[r] = 0;
    return;
  }
  int* tab = tabs[w];
  for (int t = lane; t < HT; t += 32) tab[t] = -1;
  __syncwarp();
  int u = 0;
  if (by_lane) {  // short Y rows (uniform per launch)
    u = sg_insert_by_lane<HT, 32>(xrp[r], xrp[r + 1], lane, xci, yrp, yci, tab);
  } else {
    for (int e = xrp[r]; e < xrp[r + 1]; ++e) {
      const int j = xci[e];
      for (int f = yrp[j] + lane; f < yrp[j + 1]; f += 32) u += hinsert<HT>(tab, yci[f]);
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) u += __shfl_xor_sync(0xffffffffu, u, o);
  if (lane == 0) cnt[r] = u;
  __syncwarp();
  int base = 0;
  for (int t0 = 0; t0 < HT; t0 += 32) {
    const int k = tab[t0 + lane];
    const unsigned m = __ballot_sync(0xffffffffu, k != -1);
    __syncwarp();
    if (k != -1) tab[base + __popc(m & ((1u << lane) - 1u))] = k;  // base <= t0: never overwrites unread slots
    base += __popc(m);
    __syncwarp();
  }
  int P2 = 32;
  while (P2 < u) P2 <<= 1;
  for (int t = u + lane; t < P2; t += 32) tab[t] = 0x7fffffff;
  __syncwarp();
  for (int k = 2; k <= P2; k <<= 1) {
    for (int jj = k >> 1; jj > 0; jj >>= 1) {
      for (int t = lane; t < P2; t += 32) {
        const int p = t ^ jj;
        if (p > t) {
          const int a = tab[t], b = tab[p];
          const bool up = (t & k) == 0;
          if ((a > b) == up) {
            tab[t] = b;
            tab[p] = a;
          }
        }
      }
      __syncwarp();
    }
  }
  int* out = tmp + off[r];
  for (int t = lane; t < u; t += 32) out[t] = tab[t];
}

// pack the rows written at their expansion offsets into the CSR column array (8 lanes per row)
__global__ void k_sg_rows_compact(int nr, const long long* __restrict__ off, const int* __restrict__ tmp,
                                  const int* __restrict__ crp, int* __restrict__ cci) {
  const long long gt = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const int r = (int)(gt >> 3), l = (int)(gt & 7);
  if (r >= nr) return;
  const int c0 = crp[r], u = crp[r + 1] - c0;
  const int* in = tmp + off[r];
  for (int t = l; t < u; t += 8) cci[c0 + t] = in[t];
}

// Numeric phase of one row for the hash paths: a group of G lanes (lane l, sync mask gm) walks the
// row's X entries e0 .. e1 in order (every output block accumulates in X-entry order, so values
// are bitwise those of the other paths); kt / pt is the row's column -> output position table.
//  * ROWS: LPB lanes share one block product, lane a of them owning block rows a MR .. (a + 1) MR - 1
//    of the output, so the LPB lanes read-modify-write consecutive 16/32-byte pieces of one output
//    block and G / LPB Y entries are in flight per X entry (ncu: the kernels run at l1tex 75-88 %).
//    Measured at config 4: 8.6 -> 8.3 ms per setup on the 8-lane path, but 4.5 -> 5.7 ms with 32
//    lanes (Y rows of 9 then take two rounds), which keeps one block per lane (LPB = 1).
//  * Software-pipelined: per X entry the loads form a chain x column -> Y row extent -> Y entry ->
//    output block.  Iteration e issues the column of entry e + 3, the Y extent of e + 2, and this
//    lane's first Y entry and X rows of e + 1, and accumulates entry e from registers.
template <int M, int K, int P, int HT, int G, bool ROWS>
__device__ __forceinline__ void sg_row_pipelined(int e0, int e1, int l, unsigned gm, const int* __restrict__ xci,
                                                 const double* __restrict__ xv, const int* __restrict__ yrp,
                                                 const int* __restrict__ yci, const double* __restrict__ yv,
                                                 const int* kt, const int* pt, double* __restrict__ cv) {
  constexpr int LPB = !ROWS ? 1 : (M % 4 == 0) ? 4 : (M % 2 == 0 ? 2 : 1);
  constexpr int MR = M / LPB, S = G / LPB;
  const int a = l % LPB, sl = l / LPB;
  if (e0 >= e1) return;
  int fb0, fe0, fb1 = 0, fe1 = 0, j2 = 0;
  int col0 = -1;
  double y0[K * P], xr0[MR * K];
  {
    const int j0 = xci[e0];
    fb0 = yrp[j0], fe0 = yrp[j0 + 1];
    if (e0 + 1 < e1) {
      const int j1 = xci[e0 + 1];
      fb1 = yrp[j1], fe1 = yrp[j1 + 1];
    }
    if (e0 + 2 < e1) j2 = xci[e0 + 2];
    if (fb0 + sl < fe0) {
      col0 = yci[fb0 + sl];
      ld_blk<K * P, true>(yv + (long long)(fb0 + sl) * K * P, y0);
    }
    ld_blk<MR * K, true>(xv + (long long)e0 * M * K + a * MR * K, xr0);
  }
  for (int e = e0; e < e1; ++e) {
    int j3 = 0, fb2 = 0, fe2 = 0, col1 = -1;
    double y1[K * P], xr1[MR * K];
    if (e + 3 < e1) j3 = xci[e + 3];
    if (e + 2 < e1) fb2 = yrp[j2], fe2 = yrp[j2 + 1];
    if (e + 1 < e1) {
      if (fb1 + sl < fe1) {
        col1 = yci[fb1 + sl];
        ld_blk<K * P, true>(yv + (long long)(fb1 + sl) * K * P, y1);
      }
      ld_blk<MR * K, true>(xv + (long long)(e + 1) * M * K + a * MR * K, xr1);
    }
    if (col0 >= 0) {
      unsigned h = hslot<HT>(col0);
      while (kt[h] != col0) h = (h + 1) & (HT - 1);
      block_fma_reg<MR, K, P>(cv + (long long)pt[h] * M * P + a * MR * P, xr0, y0);
      for (int f = fb0 + sl + S; f < fe0; f += S) {  // Y rows longer than the group's slots
        const int col = yci[f];
        h = hslot<HT>(col);
        while (kt[h] != col) h = (h + 1) & (HT - 1);
        block_fma<MR, K, P>(cv + (long long)pt[h] * M * P + a * MR * P, xr0, yv + (long long)f * K * P);
      }
    }
    __syncwarp(gm);
    fb0 = fb1, fe0 = fe1, fb1 = fb2, fe1 = fe2, j2 = j3, col0 = col1;
#pragma unroll
    for (int t = 0; t < K * P; ++t) y0[t] = y1[t];
#pragma unroll
    for (int t = 0; t < MR * K; ++t) xr0[t] = xr1[t];
  }
}

template <int M, int K, int P, int HT, int HW>
__global__ void __launch_bounds__(32 * HW) k_sg_hash_numeric(
    int nr, const int* __restrict__ xrp, const int* __restrict__ xci, const double* __restrict__ xv,
    const int* __restrict__ yrp, const int* __restrict__ yci, const double* __restrict__ yv,
    const int* __restrict__ crp, const int* __restrict__ cci, double* __restrict__ cv) {
  __shared__ int keys[HW][HT];
  __shared__ int pos[HW][HT];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int r = blockIdx.x * HW + w;
  if (r >= nr) return;
  int* kt = keys[w];
  int* pt = pos[w];
  for (int t = lane; t < HT; t += 32) kt[t] = -1;
  __syncwarp();
  const int c0 = crp[r], c1 = crp[r + 1];
  for (int q = c0 + lane; q < c1; q += 32) {  // insert (col -> position)
    const int key = cci[q];
    unsigned h = hslot<HT>(key);
    while (atomicCAS(kt + h, -1, key) != -1) h = (h + 1) & (HT - 1);
    pt[h] = q;
  }
  for (long long t = (long long)c0 * M * P + lane; t < (long long)c1 * M * P; t += 32) cv[t] = 0.0;
  __syncwarp();
  sg_row_pipelined<M, K, P, HT, 32, false>(xrp[r], xrp[r + 1], lane, 0xffffffffu, xci, xv, yrp, yci, yv, kt, pt, cv);
}

// ------------------------------------------------------------------ narrow-row hash SpGEMM
// Same algorithm as the k_sg_hash_* kernels (per-row open-addressing table of column ids, sorted
// row pattern, numeric accumulation in X-entry order, so values are bitwise identical to the other
// paths), for products whose Y rows are short (level 0: R A with A's 9 blocks per row, (R A) P with
// P's ~3): a group of kNG = 8 lanes owns one row (4 rows per warp) instead of a whole warp, so 3 or
// 9 Y entries do not leave 29 or 23 of 32 lanes idle.  Table kNHT slots per row (expansion <=
// kNHT / 2); the row pattern is ordered by a rank count (u <= kNHT / 2).
constexpr int kNG = 8, kNHT = 512, kNW = 2;  // lanes per row, slots per row, warps per block
constexpr int kNRows = (32 / kNG) * kNW;      // rows per block

__device__ __forceinline__ unsigned grp_mask() {
  return ((1u << kNG) - 1u) << ((threadIdx.x & 31) & ~(kNG - 1));
}

// one-table-build symbolic phase of the narrow path (see k_sg_hash_symbolic)
__global__ void __launch_bounds__(32 * kNW) k_sgn_symbolic(int nr, const int* __restrict__ xrp,
                                                            const int* __restrict__ xci, const int* __restrict__ yrp,
                                                            const int* __restrict__ yci,
                                                            const long long* __restrict__ off, int* __restrict__ cnt,
                                                            int* __restrict__ tmp) {
  __shared__ int tabs[kNRows][kNHT];
  const int g = threadIdx.x / kNG, l = threadIdx.x % kNG;
  const int r = blockIdx.x * kNRows + g;
  const unsigned gm = grp_mask();
  if (r > nr) return;  // uniform per group
  if (r == nr) {
    if (l == 0) cnt[r] = 0;
    return;
  }
  int* tab = tabs[g];
  for (int t = l; t < kNHT; t += kNG) tab[t] = -1;
  __syncwarp(gm);
  int u = sg_insert_by_lane<kNHT, kNG>(xrp[r], xrp[r + 1], l, xci, yrp, yci, tab);
#pragma unroll
  for (int o = kNG / 2; o > 0; o >>= 1) u += __shfl_xor_sync(gm, u, o, kNG);
  if (l == 0) cnt[r] = u;
  __syncwarp(gm);
  const int lane = threadIdx.x & 31;
  const unsigned below = gm & ((1u << lane) - 1u);
  int base = 0;
  for (int t0 = 0; t0 < kNHT; t0 += kNG) {
    const int k = tab[t0 + l];
    const unsigned m = __ballot_sync(gm, k != -1);
    __syncwarp(gm);
    if (k != -1) tab[base + __popc(m & below)] = k;
    base += __popc(m);
    __syncwarp(gm);
  }
  int* out = tmp + off[r];
  for (int q = l; q < u; q += kNG) {  // order by rank (keys are distinct)
    const int key = tab[q];
    int rank = 0;
    for (int t = 0; t < u; ++t) rank += tab[t] < key;
    out[rank] = key;
  }
}

template <int M, int K, int P>
__global__ void __launch_bounds__(32 * kNW) k_sgn_numeric(int nr, const int* __restrict__ xrp,
                                                           const int* __restrict__ xci, const double* __restrict__ xv,
                                                           const int* __restrict__ yrp, const int* __restrict__ yci,
                                                           const double* __restrict__ yv, const int* __restrict__ crp,
                                                           const int* __restrict__ cci, double* __restrict__ cv) {
  __shared__ int keys[kNRows][kNHT];
  __shared__ int pos[kNRows][kNHT];
  const int g = threadIdx.x / kNG, l = threadIdx.x % kNG;
  const int r = blockIdx.x * kNRows + g;
  const unsigned gm = grp_mask();
  if (r >= nr) return;
  int* kt = keys[g];
  int* pt = pos[g];
  for (int t = l; t < kNHT; t += kNG) kt[t] = -1;
  __syncwarp(gm);
  const int c0 = crp[r], c1 = crp[r + 1];
  for (int q = c0 + l; q < c1; q += kNG) {
    const int key = cci[q];
    unsigned h = hslot<kNHT>(key);
    while (atomicCAS(kt + h, -1, key) != -1) h = (h + 1) & (kNHT - 1);
    pt[h] = q;
  }
  for (long long t = (long long)c0 * M * P + l; t < (long long)c1 * M * P; t += kNG) cv[t] = 0.0;
  __syncwarp(gm);
  sg_row_pipelined<M, K, P, kNHT, kNG, true>(xrp[r], xrp[r + 1], l, gm, xci, xv, yrp, yci, yv, kt, pt, cv);
}

// ------------------------------------------------------------------ CTA-per-row numeric (small levels)
// On the small coarse levels a few hundred rows each expand to thousands of block products; one
// warp per row (hash / sort paths) then runs them as a long serial chain of global
// read-modify-writes (measured 3-5 ms per product on 32-160-row levels).  Here a CTA owns a row:
// the row's sorted pattern and its accumulators live in shared memory, and for each X entry
// (sequential, so every output entry still accumulates in X-entry order: values are bitwise
// identical to the other paths) the 256 threads split the Y row's (entry, block element) pairs.
constexpr int kCtaRows = 16384, kCtaMaxCols = 640;

template <int M, int K, int P>
__global__ void __launch_bounds__(256) k_sg_cta_numeric(int nr, const int* __restrict__ xrp,
                                                        const int* __restrict__ xci, const double* __restrict__ xv,
                                                        const int* __restrict__ yrp, const int* __restrict__ yci,
                                                        const double* __restrict__ yv, const int* __restrict__ crp,
                                                        const int* __restrict__ cci, double* __restrict__ cv) {
  constexpr int MP = M * P;
  extern __shared__ double sm[];
  const int r = blockIdx.x;
  const int c0 = crp[r], u = crp[r + 1] - c0;
  double* acc = sm;
  int* cols = reinterpret_cast<int*>(acc + (long long)u * MP);
  for (int t = threadIdx.x; t < u; t += blockDim.x) cols[t] = cci[c0 + t];
  for (int t = threadIdx.x; t < u * MP; t += blockDim.x) acc[t] = 0.0;
  __syncthreads();
  for (int e = xrp[r]; e < xrp[r + 1]; ++e) {
    const int j = xci[e];
    const double* xb = xv + (long long)e * M * K;
    const int f0 = yrp[j], nf = yrp[j + 1] - f0;
    for (int idx = threadIdx.x; idx < nf * MP; idx += blockDim.x) {
      const int f = f0 + idx / MP, ent = idx % MP, a = ent / P, b = ent % P;
      const int col = yci[f];
      int lo = 0, hi = u;
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (cols[mid] < col) lo = mid + 1;
        else hi = mid;
      }
      double sum = 0.0;
#pragma unroll
      for (int k = 0; k < K; ++k) sum += __ldg(xb + a * K + k) * __ldg(yv + (long long)f * K * P + k * P + b);
      acc[lo * MP + ent] += sum;
    }
    __syncthreads();
  }
  for (int t = threadIdx.x; t < u * MP; t += blockDim.x) cv[(long long)c0 * MP + t] = acc[t];
}

struct BsrMat {
  int nbr = 0, nbc = 0, br = 0, bc = 0;
  long long nnzb = 0;
  int* rp = nullptr;
  int* ci = nullptr;
  double* val = nullptr;
};

// Numeric phase of C = X Y on C's (already built) pattern, by the kernel the plan names.  Every
// kernel accumulates each output block over X entries in row order, so all kinds give bitwise
// the same values; the full setup records the kind it chose, the numeric-only setup of reading
// G32 replays it on the kept pattern.
template <int M, int K, int P>
static void sg_numeric(Ctx& c, const SgPlan& pl, const BsrMat& X, const BsrMat& Y, const int* crp, const int* cci,
                       double* cval) {
  const int nr = X.nbr;
  if (nr == 0) return;
  switch (pl.kind) {
    case SG_NARROW:
      k_sgn_numeric<M, K, P><<<(nr + 1 + kNRows - 1) / kNRows, 32 * kNW, 0, c.s>>>(nr, X.rp, X.ci, X.val, Y.rp, Y.ci,
                                                                                  Y.val, crp, cci, cval);
      break;
    case SG_HASH1K:
      k_sg_hash_numeric<M, K, P, kHT, kHWarps><<<(nr + 1 + kHWarps - 1) / kHWarps, 32 * kHWarps, 0, c.s>>>(
          nr, X.rp, X.ci, X.val, Y.rp, Y.ci, Y.val, crp, cci, cval);
      break;
    case SG_HASH4K:
      k_sg_hash_numeric<M, K, P, kHT2, kHWarps2><<<(nr + 1 + kHWarps2 - 1) / kHWarps2, 32 * kHWarps2, 0, c.s>>>(
          nr, X.rp, X.ci, X.val, Y.rp, Y.ci, Y.val, crp, cci, cval);
      break;
    case SG_CTA: {
      static bool attr_set = false;
      if (!attr_set) {
        SI_CUDA(cudaFuncSetAttribute(k_sg_cta_numeric<M, K, P>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     kCtaMaxCols * (M * P * (int)sizeof(double) + (int)sizeof(int)) + 16));
        attr_set = true;
      }
      k_sg_cta_numeric<M, K, P><<<nr, 256, pl.smem, c.s>>>(nr, X.rp, X.ci, X.val, Y.rp, Y.ci, Y.val, crp, cci, cval);
      break;
    }
    case SG_THREAD:
      k_spgemm_numeric<M, K, P><<<grid_for(nr, 128), 128, 0, c.s>>>(nr, X.rp, X.ci, X.val, Y.rp, Y.ci, Y.val, crp,
                                                                     cci, cval);
      break;
    case SG_GROUP8:
      k_spgemm_numeric_g<M, K, P, 8><<<(int)(((long long)nr * 8 + 255) / 256), 256, 0, c.s>>>(
          nr, X.rp, X.ci, X.val, Y.rp, Y.ci, Y.val, crp, cci, cval);
      break;
    case SG_WARP:
      k_spgemm_numeric_w<M, K, P><<<wgrid(nr), 256, 0, c.s>>>(nr, X.rp, X.ci, X.val, Y.rp, Y.ci, Y.val, crp, cci,
                                                               cval);
      break;
    default:
      SI_CHECK(false, SEAICE_ESTATE, "SpGEMM numeric phase without a plan");
  }
  SI_LAUNCHED(c);
}

// Small levels: CTA-per-row numeric if every row's pattern fits the shared accumulators.
// Returns true (and records SG_CTA in the plan) if it applies.
template <int M, int K, int P>
static bool cta_numeric(Ctx& c, const BsrMat& X, const int* cnt, SgPlan& pl, Scratch& S) {
  const int nr = X.nbr;
  if (nr > kCtaRows || c.p.spgemm_path != 0) return false;
  int* mx = S.get<int>(1);
  size_t tmp = 0;
  SI_CUDA(cub::DeviceReduce::Max(nullptr, tmp, cnt, mx, nr, c.s));
  void* t = S.get<char>(tmp + 16);
  SI_CUDA(cub::DeviceReduce::Max(t, tmp, cnt, mx, nr, c.s));
  c.launches += 1;
  const int umax = read_scalar(c, mx);
  if (umax > kCtaMaxCols) return false;
  pl.kind = SG_CTA;
  pl.smem = (size_t)umax * (M * P * sizeof(double) + sizeof(int)) + 16;
  c.sg_hits[6]++;
  return true;
}

// hash path: every row's expansion fits the per-warp shared-memory table of HT slots
template <int M, int K, int P, int HT, int HW>
static void hash_spgemm(Ctx& c, const BsrMat& X, const BsrMat& Y, DBuf<int>& crp, DBuf<int>& cci,
                        DBuf<double>& cval, long long& cnnzb, SgPlan& pl, Scratch& S, const long long* off,
                        long long tot) {
  const int nr = X.nbr;
  const int hb = (nr + 1 + HW - 1) / HW;
  int* cnt = S.get<int>(nr + 1);
  int* tmp = S.get<int>(tot);
  // Y rows of <= 12 blocks on average: one X entry per lane (see sg_insert_by_lane)
  // (measured at config 4: 4.4 -> 2.9 ms per setup on the 1k-slot path; slower on the 4k-slot path,
  // whose long X rows make the lanes collide in the table)
  const int by_lane = HT == kHT && Y.nbr > 0 && (double)Y.nnzb / Y.nbr <= 12.0 ? 1 : 0;
  k_sg_hash_symbolic<HT, HW><<<hb, 32 * HW, 0, c.s>>>(nr, X.rp, X.ci, Y.rp, Y.ci, off, cnt, tmp, by_lane);
  SI_LAUNCHED(c);
  crp.ensure(c.al, nr + 1);
  exclusive_scan(c, cnt, crp.get(), nr + 1);
  cnnzb = read_scalar(c, crp.get() + nr);
  SI_CHECK(cnnzb < (1LL << 31), SEAICE_EINVAL, "SpGEMM result exceeds int32 indexing");
  cci.ensure(c.al, cnnzb);
  cval.ensure(c.al, cnnzb * M * P);
  k_sg_rows_compact<<<grid_for((long long)nr * 8), kThreads, 0, c.s>>>(nr, off, tmp, crp.get(), cci.get());
  SI_LAUNCHED(c);
  if (!cta_numeric<M, K, P>(c, X, cnt, pl, S)) pl.kind = (HT == kHT) ? SG_HASH1K : SG_HASH4K;
  tick(c, HT == kHT ? "  sg.hash1kS" : "  sg.hash4kS", nr);
  sg_numeric<M, K, P>(c, pl, X, Y, crp.get(), cci.get(), cval.get());
  tick(c, HT == kHT ? "  sg.hash1kN" : "  sg.hash4kN", nr);
}

template <int M, int K, int P>
static void narrow_spgemm(Ctx& c, const BsrMat& X, const BsrMat& Y, DBuf<int>& crp, DBuf<int>& cci,
                          DBuf<double>& cval, long long& cnnzb, SgPlan& pl, Scratch& S, const long long* off,
                          long long tot) {
  const int nr = X.nbr;
  const int hb = (nr + 1 + kNRows - 1) / kNRows;
  int* cnt = S.get<int>(nr + 1);
  int* tmp = S.get<int>(tot);
  k_sgn_symbolic<<<hb, 32 * kNW, 0, c.s>>>(nr, X.rp, X.ci, Y.rp, Y.ci, off, cnt, tmp);
  SI_LAUNCHED(c);
  crp.ensure(c.al, nr + 1);
  exclusive_scan(c, cnt, crp.get(), nr + 1);
  cnnzb = read_scalar(c, crp.get() + nr);
  SI_CHECK(cnnzb < (1LL << 31), SEAICE_EINVAL, "SpGEMM result exceeds int32 indexing");
  cci.ensure(c.al, cnnzb);
  cval.ensure(c.al, cnnzb * M * P);
  k_sg_rows_compact<<<grid_for((long long)nr * 8), kThreads, 0, c.s>>>(nr, off, tmp, crp.get(), cci.get());
  SI_LAUNCHED(c);
  pl.kind = SG_NARROW;
  tick(c, "  sg.narrowS", nr);
  sg_numeric<M, K, P>(c, pl, X, Y, crp.get(), cci.get(), cval.get());
  tick(c, "  sg.narrowN", nr);
}

// Output arrays are grow-only DBufs owned by the caller.
template <int M, int K, int P>
static void spgemm(Ctx& c, const BsrMat& X, const BsrMat& Y, DBuf<int>& crp, DBuf<int>& cci, DBuf<double>& cval,
                   long long& cnnzb, SgPlan& pl) {
  pl = SgPlan{};
  const int nr = X.nbr;
  Scratch S(c);
  long long* ub = S.get<long long>(nr + 1);
  long long* off = S.get<long long>(nr + 1);
  k_spgemm_ub<<<grid_for(nr + 1), kThreads, 0, c.s>>>(nr, X.rp, X.ci, Y.rp, ub);
  SI_LAUNCHED(c);
  {
    long long* mx = S.get<long long>(1);
    size_t tmp = 0;
    SI_CUDA(cub::DeviceReduce::Max(nullptr, tmp, ub, mx, nr + 1, c.s));
    void* t = S.get<char>(tmp + 16);
    SI_CUDA(cub::DeviceReduce::Max(t, tmp, ub, mx, nr + 1, c.s));
    c.launches += 1;
    const long long maxub = read_scalar(c, mx);
    exclusive_scan(c, ub, off, nr + 1);
    const long long tot = read_scalar(c, off + nr);
    // the per-warp table has a fixed per-row cost: short rows (finest level) stay on the
    // sort-based path, whose thread-per-row numeric phase suits them
    const int force = c.p.spgemm_path;  // testing knob (seaice_params.spgemm_path)
    const double ylen = Y.nbr > 0 ? (double)Y.nnzb / Y.nbr : 1.0;
    if ((force == 5 || (force == 0 && ylen <= 12.0 && tot >= 24LL * nr)) && maxub <= kNHT / 2) {
      c.sg_hits[5]++;
      narrow_spgemm<M, K, P>(c, X, Y, crp, cci, cval, cnnzb, pl, S, off, tot);
      return;
    }
    const bool wide_rows = force == 1 || force == 6 || (force == 0 && tot >= 32LL * nr);
    if (wide_rows && maxub <= kHT / 2 && force != 6) {
      c.sg_hits[0]++;
      hash_spgemm<M, K, P, kHT, kHWarps>(c, X, Y, crp, cci, cval, cnnzb, pl, S, off, tot);
      return;
    }
    if (wide_rows && maxub <= kHT2 / 2) {
      c.sg_hits[1]++;
      hash_spgemm<M, K, P, kHT2, kHWarps2>(c, X, Y, crp, cci, cval, cnnzb, pl, S, off, tot);
      return;
    }
  }
  const long long total = read_scalar(c, off + nr);
  SI_CHECK(total < (1LL << 31) - 1, SEAICE_ENOMEM,
           "SpGEMM expansion exceeds 2^31 products (coarsening too slow for this operator)");
  tick(c, "  sg.ub", nr);
  int* k1 = S.get<int>(total);
  int* k2 = S.get<int>(total);
  const int force = c.p.spgemm_path;
  const bool wide = force == 4 || ((force == 0 || force == 1 || force == 6) && total > 48LL * nr);  // long rows: warp per row
  if (wide)
    k_spgemm_expand_w<<<wgrid(nr), 256, 0, c.s>>>(nr, X.rp, X.ci, Y.rp, Y.ci, off, k1);
  else
    k_spgemm_expand<<<grid_for(nr), kThreads, 0, c.s>>>(nr, X.rp, X.ci, Y.rp, Y.ci, off, k1);
  SI_LAUNCHED(c);
  {
    cub::DoubleBuffer<int> db(k1, k2);
    size_t tmp = 0;
    SI_CUDA(cub::DeviceSegmentedSort::SortKeys(nullptr, tmp, db, total, nr, off, off + 1, c.s));
    void* t = S.get<char>(tmp + 16);
    SI_CUDA(cub::DeviceSegmentedSort::SortKeys(t, tmp, db, total, nr, off, off + 1, c.s));
    c.launches += 2;
    k1 = db.Current();
  }
  tick(c, "  sg.sort", nr);
  int* cnt = S.get<int>(nr + 1);
  if (wide)
    k_spgemm_count_w<<<wgrid(nr + 1), 256, 0, c.s>>>(nr, off, k1, cnt);
  else
    k_spgemm_count<<<grid_for(nr + 1), kThreads, 0, c.s>>>(nr, off, k1, cnt);
  SI_LAUNCHED(c);
  crp.ensure(c.al, nr + 1);
  exclusive_scan(c, cnt, crp.get(), nr + 1);
  cnnzb = read_scalar(c, crp.get() + nr);
  tick(c, "  sg.count", nr);
  SI_CHECK(cnnzb < (1LL << 31), SEAICE_EINVAL, "SpGEMM result exceeds int32 indexing");
  cci.ensure(c.al, cnnzb);
  cval.ensure(c.al, cnnzb * M * P);
  const bool thread_numeric = force == 2 || ((force == 0 || force == 1 || force == 6) && Y.nbr > 0 && (double)Y.nnzb / Y.nbr <= 6.0);
  c.sg_hits[wide ? 4 : thread_numeric ? 2 : 3]++;
  if (wide) {
    k_spgemm_compact_w<<<wgrid(nr), 256, 0, c.s>>>(nr, off, k1, crp.get(), cci.get());
    SI_LAUNCHED(c);
    if (!cta_numeric<M, K, P>(c, X, cnt, pl, S)) pl.kind = SG_WARP;
  } else {
    k_spgemm_compact<<<grid_for(nr), kThreads, 0, c.s>>>(nr, off, k1, crp.get(), cci.get());
    SI_LAUNCHED(c);
    // measured: thread per row beats 4-lane groups for the finest level
    pl.kind = thread_numeric ? SG_THREAD : SG_GROUP8;
  }
  sg_numeric<M, K, P>(c, pl, X, Y, crp.get(), cci.get(), cval.get());
  tick(c, wide ? "  sg.numericW" : "  sg.numeric", (int)(total / std::max(nr, 1)));
}

// ------------------------------------------------------------------ transpose
__global__ void k_row_of(int nr, const int* __restrict__ rp, int* __restrict__ row, int* __restrict__ eidx) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= nr) return;
  for (int e = rp[r]; e < rp[r + 1]; ++e) {
    row[e] = r;
    eidx[e] = e;
  }
}

template <int BR, int BC>
__global__ void k_transpose_gather(long long nnz, const int* __restrict__ perm, const int* __restrict__ row,
                                   const double* __restrict__ val, int* __restrict__ tci, double* __restrict__ tval) {
  const long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (k >= nnz) return;
  const int e = perm[k];
  tci[k] = row[e];
#pragma unroll
  for (int a = 0; a < BR; ++a)
#pragma unroll
    for (int b = 0; b < BC; ++b) tval[k * BR * BC + b * BR + a] = val[(long long)e * BR * BC + a * BC + b];
}

// T (BC x BR blocks) = X^T for X (BR x BC blocks)
// perm / rowof keep the gather map (entry k of T is entry perm[k] of X, in row rowof[perm[k]])
// for the numeric-only setup (reading G32).
template <int BR, int BC>
static void transpose(Ctx& c, const BsrMat& X, DBuf<int>& trp, DBuf<int>& tci, DBuf<double>& tval, DBuf<int>& perm,
                      DBuf<int>& rowof) {
  Scratch S(c);
  const long long nnz = X.nnzb;
  perm.ensure(c.al, nnz);
  rowof.ensure(c.al, nnz);
  int* row = rowof.get();
  int* e0 = S.get<int>(nnz);
  int* e1 = perm.get();
  int* kk = S.get<int>(nnz);
  k_row_of<<<grid_for(X.nbr), kThreads, 0, c.s>>>(X.nbr, X.rp, row, e0);
  SI_LAUNCHED(c);
  int bits = 1;
  while ((1LL << bits) <= X.nbc) ++bits;
  size_t tmp = 0;
  SI_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp, X.ci, kk, e0, e1, (int)nnz, 0, bits, c.s));
  void* t = S.get<char>(tmp + 16);
  SI_CUDA(cub::DeviceRadixSort::SortPairs(t, tmp, X.ci, kk, e0, e1, (int)nnz, 0, bits, c.s));
  c.launches += 2;
  trp.ensure(c.al, X.nbc + 1);
  tci.ensure(c.al, nnz);
  tval.ensure(c.al, nnz * BR * BC);
  k_seg_starts<<<grid_for(X.nbc + 1), kThreads, 0, c.s>>>(X.nbc, (int)nnz, kk, trp.get());
  SI_LAUNCHED(c);
  k_transpose_gather<BR, BC><<<grid_for(nnz), kThreads, 0, c.s>>>(nnz, e1, row, X.val, tci.get(), tval.get());
  SI_LAUNCHED(c);
}

// ------------------------------------------------------------------ prolongator smoothing
template <int B, int K>
__global__ void k_smooth_p(int nb, const int* __restrict__ trp, const int* __restrict__ tci,
                           const double* __restrict__ tval, const double* __restrict__ dinv,
                           const int* __restrict__ agg, const int* __restrict__ prp_t, const double* __restrict__ pt_val,
                           double omega, double* __restrict__ pval) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= nb) return;
  const double* D = dinv + (long long)r * B * B;
  const int ar = agg[r];
  for (int e = trp[r]; e < trp[r + 1]; ++e) {
    const double* T = tval + (long long)e * B * K;
    double* Pv = pval + (long long)e * B * K;
#pragma unroll
    for (int a = 0; a < B; ++a)
#pragma unroll
      for (int k = 0; k < K; ++k) {
        double s = 0.0;
#pragma unroll
        for (int b = 0; b < B; ++b) s += D[a * B + b] * T[b * K + k];
        double v = -omega * s;
        if (tci[e] == ar) v += pt_val[(long long)prp_t[r] * B * K + a * K + k];
        Pv[a * K + k] = v;
      }
  }
}

// Level 0: P = P_tent - omega D^-1 (A P_tent) in one pass.  P_tent has one block per aggregated
// node (Q_j in column agg(j)), so row i of A P_tent gathers A_ij Q_j over i's stencil neighbours,
// grouped by agg(j): the row pattern is the sorted set of neighbour aggregates.  Same arithmetic
// and order as the generic SpGEMM (A entries in row order) followed by k_smooth_p.  Rows hold at
// most kPtsmMax A blocks (the finest stencil: 9).
constexpr int kPtsmMax = 16;

__device__ __forceinline__ int ptsm_cols(int i, const int* __restrict__ rp, const int* __restrict__ ci,
                                         const int* __restrict__ agg, int (&ag)[kPtsmMax], int (&cols)[kPtsmMax],
                                         int& ne) {
  const int e0 = rp[i];
  ne = rp[i + 1] - e0;
  int u = 0;
#pragma unroll
  for (int t = 0; t < kPtsmMax; ++t) {
    ag[t] = (t < ne) ? agg[ci[e0 + t]] : -1;
    if (ag[t] >= 0) {  // insertion into the sorted distinct list
      int p = u;
      bool dup = false;
      for (int q = 0; q < u; ++q) dup |= (cols[q] == ag[t]);
      if (!dup) {
        while (p > 0 && cols[p - 1] > ag[t]) {
          cols[p] = cols[p - 1];
          --p;
        }
        cols[p] = ag[t];
        ++u;
      }
    }
  }
  return u;
}

__global__ void k_ptsm_count(int nb, const int* __restrict__ rp, const int* __restrict__ ci,
                             const int* __restrict__ agg, int* __restrict__ cnt, int* __restrict__ flag) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i > nb) return;
  if (i == nb) {
    cnt[i] = 0;
    return;
  }
  if (rp[i + 1] - rp[i] > kPtsmMax) {
    atomicOr(flag, 32);
    cnt[i] = 0;
    return;
  }
  int ag[kPtsmMax], cols[kPtsmMax], ne;
  cnt[i] = ptsm_cols(i, rp, ci, agg, ag, cols, ne);
}

template <int B, int K>
__global__ void k_ptsm_fill(int nb, const int* __restrict__ rp, const int* __restrict__ ci,
                            const double* __restrict__ av, const int* __restrict__ agg,
                            const int* __restrict__ ptrp, const double* __restrict__ ptval,
                            const double* __restrict__ dinv, double omega, const int* __restrict__ prp,
                            int* __restrict__ pci, double* __restrict__ pval) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nb) return;
  int ag[kPtsmMax], cols[kPtsmMax], ne;
  const int u = ptsm_cols(i, rp, ci, agg, ag, cols, ne);
  const int e0 = rp[i], o = prp[i];
  const int ai = agg[i];
  const double* D = dinv + (long long)i * B * B;
  for (int s = 0; s < u; ++s) {
    const int J = cols[s];
    double T[B * K];
#pragma unroll
    for (int t = 0; t < B * K; ++t) T[t] = 0.0;
#pragma unroll
    for (int t = 0; t < kPtsmMax; ++t) {
      if (t < ne && ag[t] == J) {
        const int j = ci[e0 + t];
        const double* a = av + (long long)(e0 + t) * B * B;
        const double* q = ptval + (long long)ptrp[j] * B * K;
#pragma unroll
        for (int r = 0; r < B; ++r)
#pragma unroll
          for (int k = 0; k < K; ++k) {
            double sum = T[r * K + k];
#pragma unroll
            for (int b = 0; b < B; ++b) sum += a[r * B + b] * q[b * K + k];
            T[r * K + k] = sum;
          }
      }
    }
    pci[o + s] = J;
    double* Pv = pval + (long long)(o + s) * B * K;
#pragma unroll
    for (int a = 0; a < B; ++a)
#pragma unroll
      for (int k = 0; k < K; ++k) {
        double sm = 0.0;
#pragma unroll
        for (int b = 0; b < B; ++b) sm += D[a * B + b] * T[b * K + k];
        double v = -omega * sm;
        if (J == ai) v += ptval[(long long)ptrp[i] * B * K + a * K + k];
        Pv[a * K + k] = v;
      }
  }
}

template <int K>
__global__ void k_fix_zero_diag(int nb, const int* __restrict__ rp, const int* __restrict__ ci,
                                double* __restrict__ val) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= nb) return;
  for (int e = rp[r]; e < rp[r + 1]; ++e)
    if (ci[e] == r) {
#pragma unroll
      for (int k = 0; k < K; ++k)
        if (val[(long long)e * K * K + k * (K + 1)] == 0.0) val[(long long)e * K * K + k * (K + 1)] = 1.0;
    }
}

// ------------------------------------------------------------------ dense coarse solve
__global__ void k_bsr_to_dense(int nb, int B, const int* __restrict__ rp, const int* __restrict__ ci,
                               const double* __restrict__ val, int nd, double* __restrict__ D) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= nb) return;
  for (int e = rp[r]; e < rp[r + 1]; ++e)
    for (int a = 0; a < B; ++a)
      for (int b = 0; b < B; ++b) D[(long long)(r * B + a) * nd + ci[e] * B + b] = val[(long long)e * B * B + a * B + b];
}

// In-place lower Cholesky of the dense SPD matrix (single block, right-looking).
__global__ void k_cholesky(int n, double* __restrict__ A, int* __restrict__ flag) {
  __shared__ double piv;
  for (int k = 0; k < n; ++k) {
    if (threadIdx.x == 0) {
      const double d = A[(long long)k * n + k];
      if (!(d > 0.0)) atomicOr(flag, 8);
      piv = sqrt(fmax(d, 1e-300));
      A[(long long)k * n + k] = piv;
    }
    __syncthreads();
    const double p = piv;
    for (int i = k + 1 + threadIdx.x; i < n; i += blockDim.x) A[(long long)i * n + k] /= p;
    __syncthreads();
    const int m = n - k - 1;
    for (long long t = threadIdx.x; t < (long long)m * m; t += blockDim.x) {
      const int i = k + 1 + (int)(t / m), j = k + 1 + (int)(t % m);
      if (j <= i) A[(long long)i * n + j] -= A[(long long)i * n + k] * A[(long long)j * n + k];
    }
    __syncthreads();
  }
}

// Column j of A^-1 = L^-T L^-1 e_j; thread per column, Y stored [i][j] (coalesced across threads).
__global__ void k_chol_inverse(int n, const double* __restrict__ Lm, double* __restrict__ Y, double* __restrict__ X) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n) return;
  for (int i = 0; i < n; ++i) {
    double s = (i == j) ? 1.0 : 0.0;
    for (int k = 0; k < i; ++k) s -= Lm[(long long)i * n + k] * Y[(long long)k * n + j];
    Y[(long long)i * n + j] = s / Lm[(long long)i * n + i];
  }
  for (int i = n - 1; i >= 0; --i) {
    double s = Y[(long long)i * n + j];
    for (int k = i + 1; k < n; ++k) s -= Lm[(long long)k * n + i] * X[(long long)k * n + j];
    X[(long long)i * n + j] = s / Lm[(long long)i * n + i];
  }
}

// y = M x, dense row-major n x n, warp per row
// y = M x on the coarsest level; DOF k lives at (k / B) * S + k % B of x and y (padded storage)
__global__ void k_dense_gemv(int n, int B, int S, const double* __restrict__ M, const double* __restrict__ x,
                             double* __restrict__ y) {
  const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (w >= n) return;
  double s = 0.0;
  for (int k = lane; k < n; k += 32) s += M[(long long)w * n + k] * x[(k / B) * S + k % B];
  s = warp_sum(s);
  if (lane == 0) {
    y[(w / B) * S + w % B] = s;
    if (S > B && w % B == B - 1) y[(w / B) * S + B] = 0.0;
  }
}

// ------------------------------------------------------------------ smoother kernels
// Chebyshev step on the stencil level: t = A d; r -= t; x += d (x = d if first);
// d_out = c1 d + c2 Dinv r (if want_d).
__global__ void __launch_bounds__(256) k_cheb_stencil(int n, int Nn, const double* __restrict__ J,
                                                      const double* __restrict__ dinv, const double2* __restrict__ d,
                                                      double2* __restrict__ r, double2* __restrict__ x,
                                                      double2* __restrict__ dout, double c1, double c2, int first,
                                                      int want_r, int want_d) {
  const int node = blockIdx.x * blockDim.x + threadIdx.x;
  if (node >= Nn) return;
  const double2 dv = d[node];
  double2 xv = first ? make_double2(0.0, 0.0) : x[node];
  xv.x += dv.x;
  xv.y += dv.y;
  x[node] = xv;
  if (!want_r) return;
  const int s = n + 1, i = node % s, j = node / s;
  double y0, y1;
  if (i > 0 && i < n && j > 0 && j < n) {
    const double2 y = stencil_apply(J, Nn, s, node, d);
    y0 = y.x;
    y1 = y.y;
  } else {
    const double4 D = stencil_diag(J, Nn, node);
    y0 = D.x * dv.x + D.y * dv.y;
    y1 = D.z * dv.x + D.w * dv.y;
  }
  double2 rv = r[node];
  rv.x -= y0;
  rv.y -= y1;
  r[node] = rv;
  if (want_d) {
    const double4 D = reinterpret_cast<const double4*>(dinv)[node];
    const double z0 = D.x * rv.x + D.y * rv.y, z1 = D.z * rv.x + D.w * rv.y;
    dout[node] = make_double2(c1 * dv.x + c2 * z0, c1 * dv.y + c2 * z1);
  }
}

// Chebyshev(M) smoothing on the stencil level in one launch (temporal blocking).  A CTA owns
// a TX x FY tile of nodes (TX = 34 - 2M, so tile + M-1 rings is 32 nodes = one warp wide) and
// one thread per node of the tile plus M-1 rings; each thread keeps its node's stencil row (36
// values), r and the x increment in registers.  d_0 lives in shared memory on the tile plus M
// rings: for pre-smoothing (x_0 = 0) it is built in the kernel, r_0 = b, d_0 = ith Dinv b
// (pointwise); for post-smoothing it is staged from d0g (written by k_resid_dinv_stencil with
// r_0 = rin).  Step k (k = 1..M) then updates the nodes within M - k rings of the tile (its
// A d_{k-1} needs d_{k-1} one ring further out) and writes d_k back to shared memory.  The
// stencil is read from HBM once per smoothing step group instead of once per step (halo rows
// shared with neighbouring tiles mostly hit L2).  Same arithmetic per node and step as
// k_resid_dinv_stencil (pre) followed by M k_cheb_stencil launches:
//   x_M = x_0 + d_0 + ... + d_{M-1};  r_k = r_{k-1} - A d_{k-1};
//   d_k = c1[k] d_{k-1} + c2[k] Dinv r_k (k < M);  r_M written (out of place) iff pre.
constexpr int kFW = 32;  // threads per row (tile + rings)
constexpr int kFMaxM = 6;
template <int M, int FY> struct FusedGeom {
  static constexpr int R = M - 1;             // rings computed around the tile
  static constexpr int TX = kFW - 2 * R;      // tile width
  static constexpr int RY = FY + 2 * R;      // rows of tile + R rings
  static constexpr int HX = TX + 2 * M, HY = FY + 2 * M;  // d region (tile + M rings)
  static constexpr int NT = kFW * RY;         // threads
};
struct ChebFCoef {
  double c1[kFMaxM], c2[kFMaxM];
  double ith;  // 1 / theta
};
// y = A d at this thread's node, stencil row in registers, d from shared memory
__device__ __forceinline__ double2 stencil_apply_reg(bool interior, const double (&Jr)[36],
                                                     const double2* __restrict__ sd, int sidx, int srow) {
  double y0 = 0.0, y1 = 0.0;
  if (interior) {
#pragma unroll
    for (int sl = 0; sl < 9; ++sl) {
      const double2 v = sd[sidx + (sl / 3 - 1) * srow + (sl % 3 - 1)];
      y0 += Jr[sl * 4 + 0] * v.x + Jr[sl * 4 + 1] * v.y;
      y1 += Jr[sl * 4 + 2] * v.x + Jr[sl * 4 + 3] * v.y;
    }
  } else {
    const double2 v = sd[sidx];
    y0 = Jr[16] * v.x + Jr[17] * v.y;
    y1 = Jr[18] * v.x + Jr[19] * v.y;
  }
  return make_double2(y0, y1);
}

template <int M, int FY>
__global__ void __launch_bounds__(FusedGeom<M, FY>::NT, (FusedGeom<M, FY>::NT <= 256 ? 2 : 1))
    k_chebM_stencil(int n, int Nn, const double* __restrict__ J, const double* __restrict__ dinv,
                    const double2* __restrict__ rin, const double2* __restrict__ d0g, double2* __restrict__ rout,
                    double2* __restrict__ x, ChebFCoef k, int pre) {
  using Gm = FusedGeom<M, FY>;
  __shared__ double2 sd[2][Gm::HX * Gm::HY];
  const int s = n + 1;
  const int i0 = blockIdx.x * Gm::TX, j0 = blockIdx.y * FY;
  const int t = threadIdx.x;
  const int li = t % kFW, lj = t / kFW;  // position in the tile + R rings
  const int gi = i0 - Gm::R + li, gj = j0 - Gm::R + lj;
  const int di = li < Gm::R ? Gm::R - li : (li >= Gm::TX + Gm::R ? li - (Gm::TX + Gm::R - 1) : 0);
  const int dj = lj < Gm::R ? Gm::R - lj : (lj >= FY + Gm::R ? lj - (FY + Gm::R - 1) : 0);
  const int depth = di > dj ? di : dj;  // ring index (0 = tile)
  const bool inside = gi >= 0 && gi <= n && gj >= 0 && gj <= n;
  const int node = gj * s + gi;
  const bool interior = gi > 0 && gi < n && gj > 0 && gj < n;
  const int sidx = (lj + 1) * Gm::HX + (li + 1);
  // Halo values of d_0 (outermost ring for pre-smoothing, the whole d region for post-smoothing)
  // are requested first, so that their loads overlap the stencil-row loads below instead of
  // following them (at most 2 entries per thread).
  constexpr int NRING = 2 * Gm::HX + 2 * (Gm::HY - 2), NREG = Gm::HX * Gm::HY;
  constexpr int NH = ((NRING > NREG ? NRING : NREG) + Gm::NT - 1) / Gm::NT;
  double2 hb[NH];
  double4 hd[NH];
  int hidx[NH];
#pragma unroll
  for (int q = 0; q < NH; ++q) {
    const int idx = t + q * Gm::NT;
    hidx[q] = -1;
    hb[q] = make_double2(0.0, 0.0);
    hd[q] = make_double4(0.0, 0.0, 0.0, 0.0);
    int hx = 0, hy = 0;
    if (pre) {
      if (idx >= NRING) continue;
      if (idx < Gm::HX) { hx = idx; hy = 0; }
      else if (idx < 2 * Gm::HX) { hx = idx - Gm::HX; hy = Gm::HY - 1; }
      else { const int qq = idx - 2 * Gm::HX; hx = (qq & 1) ? Gm::HX - 1 : 0; hy = 1 + (qq >> 1); }
    } else {
      if (idx >= NREG) continue;
      hx = idx % Gm::HX;
      hy = idx / Gm::HX;
    }
    hidx[q] = hy * Gm::HX + hx;
    const int hi = i0 - M + hx, hj = j0 - M + hy;
    if (hi >= 0 && hi <= n && hj >= 0 && hj <= n) {
      const int nd = hj * s + hi;
      if (pre) {
        hb[q] = rin[nd];
        hd[q] = reinterpret_cast<const double4*>(dinv)[nd];
      } else {
        hb[q] = d0g[nd];
      }
    }
  }
  // this node's stencil row (read once for the M steps), r_0, Dinv, x_0
  double Jr[36];
  double2 rv = make_double2(0.0, 0.0), xa = make_double2(0.0, 0.0);
  double4 D = make_double4(0.0, 0.0, 0.0, 0.0);
  if (inside) {
    if (interior) {
      stencil_row(J, Nn, s, node, Jr);
    } else {
      const double4 Dg = stencil_diag(J, Nn, node);
#pragma unroll
      for (int e = 0; e < 36; ++e) Jr[e] = 0.0;
      Jr[16] = Dg.x; Jr[17] = Dg.y; Jr[18] = Dg.z; Jr[19] = Dg.w;
    }
    rv = rin[node];
    D = reinterpret_cast<const double4*>(dinv)[node];
    if (depth == 0 && !pre) xa = x[node];
  } else {
#pragma unroll
    for (int e = 0; e < 36; ++e) Jr[e] = 0.0;
  }
  if (pre) {  // d_0 = ith Dinv b on the tile + M rings
    sd[0][sidx] = inside ? make_double2(k.ith * (D.x * rv.x + D.y * rv.y), k.ith * (D.z * rv.x + D.w * rv.y))
                         : make_double2(0.0, 0.0);
#pragma unroll
    for (int q = 0; q < NH; ++q)
      if (hidx[q] >= 0)
        sd[0][hidx[q]] = make_double2(k.ith * (hd[q].x * hb[q].x + hd[q].y * hb[q].y),
                                      k.ith * (hd[q].z * hb[q].x + hd[q].w * hb[q].y));
  } else {  // stage d_0 on the tile + M rings (zero outside the domain)
#pragma unroll
    for (int q = 0; q < NH; ++q)
      if (hidx[q] >= 0) sd[0][hidx[q]] = hb[q];
  }
  __syncthreads();
  // steps 1 .. M-1
#pragma unroll
  for (int st = 0; st < M - 1; ++st) {
    const double2* din = sd[st & 1];
    double2* dnx = sd[(st + 1) & 1];
    if (inside && depth <= M - 1 - st) {
      const double2 dv = din[sidx];
      const double2 y = stencil_apply_reg(interior, Jr, din, sidx, Gm::HX);
      rv.x -= y.x;
      rv.y -= y.y;
      xa.x += dv.x;
      xa.y += dv.y;
      const double z0 = D.x * rv.x + D.y * rv.y, z1 = D.z * rv.x + D.w * rv.y;
      dnx[sidx] = make_double2(k.c1[st] * dv.x + k.c2[st] * z0, k.c1[st] * dv.y + k.c2[st] * z1);
    }
    __syncthreads();
  }
  // step M (tile only): x += d_{M-1}; r -= A d_{M-1} if pre-smoothing
  if (inside && depth == 0) {
    const double2* din = sd[(M - 1) & 1];
    const double2 dv = din[sidx];
    xa.x += dv.x;
    xa.y += dv.y;
    x[node] = xa;
    if (pre) {
      const double2 y = stencil_apply_reg(interior, Jr, din, sidx, Gm::HX);
      rv.x -= y.x;
      rv.y -= y.y;
      rout[node] = rv;
    }
  }
}

template <int M, int FY>
static void launch_chebM_t(Ctx& c, const double* dinv, const double* rin, const double* d0g, double* rout, double* x,
                           const ChebFCoef& kc, bool pre) {
  using Gm = FusedGeom<M, FY>;
  const dim3 grid((c.n + 1 + Gm::TX - 1) / Gm::TX, (c.n + 1 + FY - 1) / FY);
  k_chebM_stencil<M, FY><<<grid, Gm::NT, 0, c.s>>>(c.n, c.Nn, c.Jst.get(), dinv, (const double2*)rin,
                                                    (const double2*)d0g, (double2*)rout, (double2*)x, kc, pre ? 1 : 0);
}
template <int M>
static void launch_chebM(Ctx& c, const double* dinv, const double* rin, const double* d0g, double* rout, double* x,
                         const ChebFCoef& kc, bool pre) {
  // 12 tile rows (16 thread rows incl. the 2 + 2 ring rows, 512 threads, 1 CTA/SM): the ring
  // recompute drops from 56 % to 34 % of the threads; measured fastest on B200 (config 4: 645 us
  // per V-cycle vs 679 us at 4 rows, 746 us at 8 rows)
  static const int fy = getenv("SEAICE_CHEB_FY") ? atoi(getenv("SEAICE_CHEB_FY")) : 12;  // tuning aid
  if (fy == 12) launch_chebM_t<M, 12>(c, dinv, rin, d0g, rout, x, kc, pre);
  else if (fy == 8) launch_chebM_t<M, 8>(c, dinv, rin, d0g, rout, x, kc, pre);
  else launch_chebM_t<M, 4>(c, dinv, rin, d0g, rout, x, kc, pre);
}

// Chebyshev(3) smoothing on the stencil level as a y-streamed (sliding-window) temporally
// blocked launch fed by TMA (cheb_fused = 2).  A CTA owns a strip of kTTX = 60 node columns
// (64 threads wide with the 2 + 2 ring columns of steps 1 and 2: two warps per node row) and a
// segment of rows [ja, jb); it walks the rows in ticks, one __syncthreads per tick.
//   * One elected thread streams the rows into a kTNS-slot shared-memory ring with tensor-map
//     bulk copies (cp.async.bulk.tensor, completion on one mbarrier per slot): the stencil row
//     block of the smoother copy Jsm[j][e][x] (68 x 20 doubles), Dinv, b and (post) x_0 on 66
//     columns.  ~10 rows (150 KB) per SM are in flight, independent of the compute warps, and
//     out-of-domain rows / columns arrive as zeros (no boundary branches: a Dirichlet row of the
//     symmetric storage is the identity row, an out-of-domain row is zero).
//   * Warp pair p owns the rows r = rho(p) + 8 m of the segment.  Its row program takes 8
//     ticks: stage 0 (wait for the slot, stencil row -> registers incl. the transposed upper
//     blocks of the lower neighbours from this and the previous slot, u0 -> shared), the TMA
//     issue for the slot it just released, then stages 1, 2, 3 two ticks apart (stage k of
//     row j reads u_{k-1} of rows j - 1, j, j + 1 from an 8-row shared ring).  The 8 pairs are
//     in 8 different phases: loads, the four stages and the stores of different rows overlap;
//     there are no ring rows (60 of 64 threads produce output; the tile kernel: 336 of 512).
// Arithmetic per node and step is that of k_chebM_stencil up to the summation order of A u:
//   PRE  (x_0 = 0):  u0 = d_0 = ith Dinv b;  stage k: r -= A u_{k-1}, x += u_{k-1},
//                    u_k = c1 u_{k-1} + c2 Dinv r;  writes x_3 and r_3.
//   POST (x_0 = xin): u0 = x_0;  stage 1: r = b - A x_0, u1 = d_0 = ith Dinv r;  stages 2, 3 as
//                    above (d_1, d_2);  writes x_0 + d_0 + d_1 + d_2 to xout != xin (ring columns
//                    and rows of x_0 belong to other CTAs' outputs).  The residual pass
//                    k_resid_dinv_stencil of the tile path is part of the launch.
constexpr int kTW = 64, kTTX = 60, kTNP = 8, kTNS = 12, kTBX = 68, kTHX = 66, kTJE = 20;
constexpr int kTOffD = kTBX * kTJE * 8;                         // 10880 (multiple of 128)
constexpr int kTOffB = (kTOffD + kTHX * 32 + 127) / 128 * 128;  // 13056
constexpr int kTOffX = (kTOffB + kTHX * 16 + 127) / 128 * 128;  // 14208
constexpr int kTSlot = (kTOffX + kTHX * 16 + 127) / 128 * 128;  // 15360
constexpr int kTSuBytes = 3 * kTNP * kTHX * 16;
constexpr int kTSmem = kTNS * kTSlot + kTSuBytes + kTNS * 8;
static_assert(kTOffD % 128 == 0 && kTSmem <= 227 * 1024, "streamed smoother shared-memory layout");

__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(unsigned long long* bar, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
  unsigned ok = 0;
  while (!ok) {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
  }
}
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* tm, int c0, int c1, int c2,
                                            unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<unsigned long long>(tm)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
      : "memory");
}

// A u at this thread's node: stencil row in registers, u rows from the shared ring; three partial
// sums per component (one per stencil row) keep the dependent-DFMA chains short
__device__ __forceinline__ double2 stream_apply(const double (&Jr)[36], const double2* __restrict__ rm,
                                                const double2* __restrict__ r0, const double2* __restrict__ rp,
                                                int c) {
  double a0[3], a1[3];
#pragma unroll
  for (int rr = 0; rr < 3; ++rr) {
    const double2* row = rr == 0 ? rm : (rr == 1 ? r0 : rp);
    const double2 vm = row[c - 1], v0 = row[c], vp = row[c + 1];
    const int sl = rr * 3;
    a0[rr] = Jr[sl * 4 + 0] * vm.x + Jr[sl * 4 + 1] * vm.y;
    a1[rr] = Jr[sl * 4 + 2] * vm.x + Jr[sl * 4 + 3] * vm.y;
    a0[rr] += Jr[sl * 4 + 4] * v0.x + Jr[sl * 4 + 5] * v0.y;
    a1[rr] += Jr[sl * 4 + 6] * v0.x + Jr[sl * 4 + 7] * v0.y;
    a0[rr] += Jr[sl * 4 + 8] * vp.x + Jr[sl * 4 + 9] * vp.y;
    a1[rr] += Jr[sl * 4 + 10] * vp.x + Jr[sl * 4 + 11] * vp.y;
  }
  return make_double2((a0[0] + a0[1]) + a0[2], (a1[0] + a1[1]) + a1[2]);
}

// Smoother copy of the stencil: Jsm[(j * 20 + e) * sp + x] = Jst[e * Nn + j * s + x] (sp = row
// pitch, even, so every (j, e) line is 16-byte aligned for the tensor map); plane 19 and the pad
// columns stay zero.
__global__ void k_stencil_to_stream(int s, int sp, long long Nn, const double* __restrict__ Jst,
                                    double* __restrict__ Jsm) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x, j = blockIdx.y;
  if (x >= s) return;
  const long long node = (long long)j * s + x;
#pragma unroll
  for (int e = 0; e < kJS; ++e) Jsm[((long long)j * kTJE + e) * sp + x] = Jst[e * Nn + node];
}

template <bool PRE>
__global__ void __launch_bounds__(kTNP * 64, 1)
    k_cheb3_stream(const __grid_constant__ CUtensorMap tmJ, const __grid_constant__ CUtensorMap tmD,
                   const __grid_constant__ CUtensorMap tmB, const __grid_constant__ CUtensorMap tmX, int n,
                   int seg_rows, double2* __restrict__ xout, double2* __restrict__ rout, ChebFCoef k) {
  extern __shared__ __align__(128) unsigned char smem[];
  typedef double2 URow[kTHX];
  URow* su = reinterpret_cast<URow*>(smem + kTNS * kTSlot);  // su[k * kTNP + q][col]
  unsigned long long* mbar = reinterpret_cast<unsigned long long*>(smem + kTNS * kTSlot + kTSuBytes);
  const int s = n + 1;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, p = w >> 1, hf = w & 1;
  // rows 2 ticks apart (the compute stages of one tick) alternate between the two scheduler pairs
  const int rho = 2 * (p & 1) + ((p >> 1) & 1) + 4 * (p >> 2);
  const int i0 = blockIdx.x * kTTX, ja = blockIdx.y * seg_rows;
  const int jb = min(ja + seg_rows, s);
  const int jbase = ja - 3, nrows = jb + 3 - jbase;
  const int cidx = hf * 32 + lane, gi = i0 - 2 + cidx;
  const int di = cidx < 2 ? 2 - cidx : (cidx >= kTTX + 2 ? cidx - (kTTX + 1) : 0);
  const bool col_in = gi >= 0 && gi <= n;
  const int c = cidx + 1;  // column in the 66-wide u / Dinv / b / x rows
  constexpr unsigned kBytes = kTBX * kTJE * 8 + kTHX * 32 + kTHX * 16 + (PRE ? 0 : kTHX * 16);
  auto issue = [&](int r) {  // one thread: stream row jbase + r into its slot
    const int slot = r % kTNS, j = jbase + r;
    unsigned char* dst = smem + slot * kTSlot;
    mbar_expect_tx(&mbar[slot], kBytes);
    tma_load_3d(dst, &tmJ, i0 - 4, 0, j, &mbar[slot]);
    tma_load_3d(dst + kTOffD, &tmD, 0, i0 - 3, j, &mbar[slot]);
    tma_load_3d(dst + kTOffB, &tmB, 0, i0 - 3, j, &mbar[slot]);
    if (!PRE) tma_load_3d(dst + kTOffX, &tmX, 0, i0 - 3, j, &mbar[slot]);
  };
  if (threadIdx.x == 0) {
    for (int sl = 0; sl < kTNS; ++sl) mbar_init(&mbar[sl], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    for (int r = 0; r < kTNS - 1 && r < nrows; ++r) issue(r);
  }
  __syncthreads();
  const int nticks = nrows + kTNP - 1;
  // every warp executes one barrier per tick, at the point of its own row program
  int done = rho;
  for (int t = 0; t < rho; ++t) __syncthreads();
  for (int r = rho; r < nrows; r += kTNP, done += kTNP) {
    const int j = jbase + r, slot = r % kTNS, pslot = (r + kTNS - 1) % kTNS;
    const int q = r & (kTNP - 1), qm = (q - 1) & (kTNP - 1), qp = (q + 1) & (kTNP - 1);
    const int node = j * s + gi;
    double Jr[36];
    double2 rv, xa = make_double2(0.0, 0.0);
    double4 D;
    {  // tick r, stage 0: this row's data -> registers, u0 -> shared
      mbar_wait(&mbar[slot], (r / kTNS) & 1);
      if (r > 0) mbar_wait(&mbar[pslot], ((r - 1) / kTNS) & 1);  // row j-1's copy (completed a tick ago)
      const double* Js = reinterpret_cast<const double*>(smem + slot * kTSlot) + (cidx + 2);
      const double* Jm = reinterpret_cast<const double*>(smem + pslot * kTSlot) + (cidx + 2);
#pragma unroll
      for (int u = 0; u < 4; ++u) {
#pragma unroll
        for (int e = 0; e < 4; ++e) Jr[(5 + u) * 4 + e] = Js[(4 * u + e) * kTBX];
        // lower half: transposed upper block u of the neighbour at -off_u (W: this row, x-1;
        // SE, S, SW: row j-1 at x+1, x, x-1)
        const double* lo = (u == 0 ? Js - 1 : Jm + (2 - u)) + 4 * u * kTBX;
        const int sl = 3 - u;
        Jr[sl * 4 + 0] = lo[0];
        Jr[sl * 4 + 1] = lo[2 * kTBX];
        Jr[sl * 4 + 2] = lo[kTBX];
        Jr[sl * 4 + 3] = lo[3 * kTBX];
      }
      Jr[16] = Js[kJDxx * kTBX];
      Jr[17] = Js[kJDxy * kTBX];
      Jr[18] = Jr[17];
      Jr[19] = Js[kJDyy * kTBX];
      const unsigned char* sb = smem + slot * kTSlot;
      const double4* Ds = reinterpret_cast<const double4*>(sb + kTOffD);
      const double2* bs = reinterpret_cast<const double2*>(sb + kTOffB);
      const double2* xs = reinterpret_cast<const double2*>(sb + kTOffX);
      D = Ds[c];
      rv = bs[c];
      double2 u0;
      if (PRE) {
        u0 = make_double2(k.ith * (D.x * rv.x + D.y * rv.y), k.ith * (D.z * rv.x + D.w * rv.y));
      } else {
        xa = xs[c];
        u0 = xa;
      }
      su[q][c] = u0;
      if (cidx == 0 || cidx == kTW - 1) {  // 3rd-ring columns of u0
        const int hc = cidx == 0 ? 0 : kTHX - 1;
        if (PRE) {
          const double4 hD = Ds[hc];
          const double2 hb = bs[hc];
          su[q][hc] = make_double2(k.ith * (hD.x * hb.x + hD.y * hb.y), k.ith * (hD.z * hb.x + hD.w * hb.y));
        } else {
          su[q][hc] = xs[hc];
        }
      }
    }
    __syncthreads();
    // tick r + 1: the slot of row j-1 was last read in tick r (by this pair): refill it
    if (hf == 0 && lane == 0 && r + kTNS - 1 < nrows) issue(r + kTNS - 1);
    __syncthreads();
    // tick r + 2, stage 1 (rows ja-2 .. jb+1, all 64 columns)
    if (j >= ja - 2 && j < jb + 2) {
      const double2 y = stream_apply(Jr, su[qm], su[q], su[qp], c);
      rv.x -= y.x;
      rv.y -= y.y;
      const double z0 = D.x * rv.x + D.y * rv.y, z1 = D.z * rv.x + D.w * rv.y;
      if (PRE) {
        const double2 dv = su[q][c];
        xa = dv;
        su[kTNP + q][c] = make_double2(k.c1[0] * dv.x + k.c2[0] * z0, k.c1[0] * dv.y + k.c2[0] * z1);
      } else {
        su[kTNP + q][c] = make_double2(k.ith * z0, k.ith * z1);
      }
    }
    __syncthreads();
    __syncthreads();
    // tick r + 4, stage 2 (rows ja-1 .. jb, ring depth <= 1)
    if (di <= 1 && j >= ja - 1 && j < jb + 1) {
      const double2 dv = su[kTNP + q][c];
      const double2 y = stream_apply(Jr, su[kTNP + qm], su[kTNP + q], su[kTNP + qp], c);
      rv.x -= y.x;
      rv.y -= y.y;
      xa.x += dv.x;
      xa.y += dv.y;
      const double z0 = D.x * rv.x + D.y * rv.y, z1 = D.z * rv.x + D.w * rv.y;
      constexpr int ci = PRE ? 1 : 0;
      su[2 * kTNP + q][c] = make_double2(k.c1[ci] * dv.x + k.c2[ci] * z0, k.c1[ci] * dv.y + k.c2[ci] * z1);
    }
    __syncthreads();
    __syncthreads();
    // tick r + 6, stage 3 (rows ja .. jb-1, strip columns)
    if (di == 0 && col_in && j >= ja && j < jb) {
      const double2 dv = su[2 * kTNP + q][c];
      xa.x += dv.x;
      xa.y += dv.y;
      const double2 y = stream_apply(Jr, su[2 * kTNP + qm], su[2 * kTNP + q], su[2 * kTNP + qp], c);
      rv.x -= y.x;
      rv.y -= y.y;
      if (PRE) {
        xout[node] = xa;
        rout[node] = rv;
      } else {
        const double z0 = D.x * rv.x + D.y * rv.y, z1 = D.z * rv.x + D.w * rv.y;
        xa.x += k.c1[1] * dv.x + k.c2[1] * z0;
        xa.y += k.c1[1] * dv.y + k.c2[1] * z1;
        xout[node] = xa;
      }
    }
    __syncthreads();
    __syncthreads();  // tick r + 7: idle
  }
  for (; done < nticks; ++done) __syncthreads();
}

// segments per strip so that the grid fills the SMs (1 CTA per SM) in whole waves
static int stream_segments(int strips, int rows, int sms) {
  int best = 1;
  double best_eff = 0.0;
  for (int g = 1; g <= 64; ++g) {
    const int seg = (rows + g - 1) / g;
    if (g > 1 && seg < 48) break;
    const int ctas = strips * ((rows + seg - 1) / seg);
    const int waves = (ctas + sms - 1) / sms;
    // per-CTA time ~ seg + pipeline fill; efficiency = useful row-ticks / (waves * sms * ticks per CTA)
    const double eff = (double)strips * rows / ((double)waves * sms * (seg + 6 + kTNP));
    if (eff > best_eff * 1.02) {
      best_eff = eff;
      best = g;
    }
  }
  return best;
}

typedef CUresult (*TmapEncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                 const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                 CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static TmapEncodeFn tmap_encode_fn() {
  static TmapEncodeFn fn = nullptr;
  if (!fn) {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult qr;
    SI_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &qr));
    SI_CHECK(f && qr == cudaDriverEntryPointSuccess, SEAICE_ESTATE, "cuTensorMapEncodeTiled not available");
    fn = (TmapEncodeFn)f;
  }
  return fn;
}
// fp64 rank-3 tiled tensor map (dims innermost first, strides in bytes for dims 1 and 2)
static CUtensorMap tmap3(const void* base, cuuint64_t d0, cuuint64_t d1, cuuint64_t d2, cuuint64_t st1,
                         cuuint64_t st2, cuuint32_t b0, cuuint32_t b1) {
  SI_CHECK((reinterpret_cast<uintptr_t>(base) & 15) == 0, SEAICE_EINVAL,
           "streamed smoother: vectors must be 16-byte aligned");
  CUtensorMap tm;
  const cuuint64_t dims[3] = {d0, d1, d2}, strides[2] = {st1, st2};
  const cuuint32_t box[3] = {b0, b1, 1}, es[3] = {1, 1, 1};
  const CUresult r = tmap_encode_fn()(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<void*>(base), dims, strides,
                                      box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                      CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  SI_CHECK(r == CUDA_SUCCESS, SEAICE_ESTATE, "cuTensorMapEncodeTiled failed");
  return tm;
}

// (re)build the smoother copy of the finest stencil from Jst (after every assembly that the
// hierarchy's finest level is refreshed from)
static void stencil_stream_copy(Ctx& c) {
  const int s = c.n + 1, sp = (s + 1) & ~1;
  const size_t len = (size_t)s * kTJE * sp;
  if (c.Jsm.cap < len) {
    c.Jsm.ensure(c.al, len);
    SI_CUDA(cudaMemsetAsync(c.Jsm.get(), 0, len * sizeof(double), c.s));
  }
  k_stencil_to_stream<<<dim3((s + 255) / 256, s), 256, 0, c.s>>>(s, sp, c.Nn, c.Jst.get(), c.Jsm.get());
  SI_LAUNCHED(c);
}

static void launch_cheb3_stream(Ctx& c, const double* dinv, const double* b, const double* xin, double* xout,
                                double* rout, const ChebFCoef& kc, bool pre) {
  const int s = c.n + 1, sp = (s + 1) & ~1, strips = (s + kTTX - 1) / kTTX;
  static const int seg_env = getenv("SEAICE_CHEB_SEGS") ? atoi(getenv("SEAICE_CHEB_SEGS")) : 0;  // tuning aid
  const int g = seg_env > 0 ? seg_env : stream_segments(strips, s, c.sms);
  const int seg = (s + g - 1) / g;
  const dim3 grid(strips, (s + seg - 1) / seg);
  const CUtensorMap tmJ = tmap3(c.Jsm.get(), sp, kTJE, s, 8ull * sp, 8ull * sp * kTJE, kTBX, kTJE);
  const CUtensorMap tmD = tmap3(dinv, 4, s, s, 32, 32ull * s, 4, kTHX);
  const CUtensorMap tmB = tmap3(b, 2, s, s, 16, 16ull * s, 2, kTHX);
  const CUtensorMap tmX = pre ? tmB : tmap3(xin, 2, s, s, 16, 16ull * s, 2, kTHX);
  static bool attr = false;
  if (!attr) {
    SI_CUDA(cudaFuncSetAttribute(k_cheb3_stream<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kTSmem));
    SI_CUDA(cudaFuncSetAttribute(k_cheb3_stream<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, kTSmem));
    attr = true;
  }
  if (pre)
    k_cheb3_stream<true><<<grid, kTNP * 64, kTSmem, c.s>>>(tmJ, tmD, tmB, tmX, c.n, seg, (double2*)xout, (double2*)rout, kc);
  else
    k_cheb3_stream<false><<<grid, kTNP * 64, kTSmem, c.s>>>(tmJ, tmD, tmB, tmX, c.n, seg, (double2*)xout, nullptr, kc);
}

// r = b - A x (or r = b if x == NULL); d = Dinv r * c2 (stencil level)
__global__ void __launch_bounds__(256) k_resid_dinv_stencil(int n, int Nn, const double* __restrict__ J,
                                                            const double* __restrict__ dinv,
                                                            const double2* __restrict__ b,
                                                            const double2* __restrict__ x, double2* __restrict__ r,
                                                            double2* __restrict__ d, double c2) {
  const int node = blockIdx.x * blockDim.x + threadIdx.x;
  if (node >= Nn) return;
  double2 rv = b[node];
  if (x) {
    const int s = n + 1, i = node % s, j = node / s;
    double y0, y1;
    if (i > 0 && i < n && j > 0 && j < n) {
      const double2 y = stencil_apply(J, Nn, s, node, x);
      y0 = y.x;
      y1 = y.y;
    } else {
      const double2 v = x[node];
      const double4 D = stencil_diag(J, Nn, node);
      y0 = D.x * v.x + D.y * v.y;
      y1 = D.z * v.x + D.w * v.y;
    }
    rv.x -= y0;
    rv.y -= y1;
  }
  r[node] = rv;
  const double4 D = reinterpret_cast<const double4*>(dinv)[node];
  d[node] = make_double2(c2 * (D.x * rv.x + D.y * rv.y), c2 * (D.z * rv.x + D.w * rv.y));
}




// ------------------------------------------------------------------ group-per-row BSR kernels
// V-cycle copy of a block array in the chunk-of-32 SoA layout (Level::valT): a group's lanes
// read consecutive blocks, so each per-element load of the warp is contiguous.
__global__ void k_tile_blocks(long long nnzb, int BB, const double* __restrict__ val, double* __restrict__ out) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= nnzb * BB) return;
  const long long e = i / BB;
  const int j = (int)(i - e * BB);
  out[((e >> 5) * BB + j) * 32 + (e & 31)] = val[i];
}
static void tile_copy(Ctx& c, DBuf<double>& out, const double* val, long long nnzb, int BB) {
  const long long n = (nnzb + 31) / 32 * 32 * BB;
  out.ensure(c.al, (size_t)(n > 0 ? n : 1));
  if (nnzb == 0) return;
  k_tile_blocks<<<grid_for(nnzb * BB), kThreads, 0, c.s>>>(nnzb, BB, val, out.get());
  SI_LAUNCHED(c);
}

// Coarse-level vectors (b = 3) are stored padded to 4 doubles per block row (32-byte aligned;
// the pad is kept 0), so the x gather of a 3x3 block is ONE 256-bit load instead of three
// 8-byte loads (the group kernels are L1-wavefront bound).  Level 0 (b = 2) is unpadded.
__host__ __device__ constexpr int vstride(int B) { return B == 3 ? 4 : B; }

template <int BC>
__device__ __forceinline__ void load_xblk(const double* __restrict__ x, int col, double xv[BC]) {
  if constexpr (BC == 3) {
    const double* p = x + (long long)col * 4;
    double w;
    asm("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(xv[0]), "=d"(xv[1]), "=d"(xv[2]), "=d"(w) : "l"(p));
  } else if constexpr (BC == 4) {
    const double* p = x + (long long)col * 4;
    asm("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(xv[0]), "=d"(xv[1]), "=d"(xv[2]), "=d"(xv[3]) : "l"(p));
  } else {
    const double2 v = __ldg(reinterpret_cast<const double2*>(x) + col);
    xv[0] = v.x;
    xv[1] = v.y;
  }
}

// G consecutive lanes own one block row: lane l reads blocks e = rp[row] + l, + G, ...
// so the G blocks a group touches per step are contiguous in memory (coalesced), and the
// BR partial sums are combined with an xor-butterfly (same order on every lane).  The loop is
// unrolled by two so both column-index loads (and then both x gathers) are in flight together.
template <int BR, int BC>
__device__ __forceinline__ void blk_fma(const double* __restrict__ val, int e, const double xv[BC], double acc[BR]) {
  const double* v = val + (long long)(e >> 5) * (BR * BC * 32) + (e & 31);  // chunk-of-32 SoA
#pragma unroll
  for (int a = 0; a < BR; ++a)
#pragma unroll
    for (int b = 0; b < BC; ++b) acc[a] += __ldg(v + (a * BC + b) * 32) * xv[b];
}

template <int BR, int BC, int G>
__device__ __forceinline__ void grp_row(int row, int nb, int lig, const int* __restrict__ rp,
                                        const int* __restrict__ ci, const double* __restrict__ val,
                                        const double* __restrict__ x, double acc[BR]) {
#pragma unroll
  for (int a = 0; a < BR; ++a) acc[a] = 0.0;
  if (row < nb) {
    const int e1 = __ldg(rp + row + 1);
    int e = __ldg(rp + row) + lig;
    for (; e + G < e1; e += 2 * G) {
      const int c0 = __ldg(ci + e), c1 = __ldg(ci + e + G);
      double x0[BC], x1[BC];
      load_xblk<BC>(x, c0, x0);
      load_xblk<BC>(x, c1, x1);
      blk_fma<BR, BC>(val, e, x0, acc);
      blk_fma<BR, BC>(val, e + G, x1, acc);
    }
    for (; e < e1; e += G) {
      double x0[BC];
      load_xblk<BC>(x, __ldg(ci + e), x0);
      blk_fma<BR, BC>(val, e, x0, acc);
    }
  }
#pragma unroll
  for (int off = G / 2; off > 0; off >>= 1)
#pragma unroll
    for (int a = 0; a < BR; ++a) acc[a] += __shfl_xor_sync(0xffffffffu, acc[a], off, G);
}

// component `a` of a register array without dynamic indexing
template <int B>
__device__ __forceinline__ double pick(const double v[B], int a) {
  double r = v[0];
#pragma unroll
  for (int k = 1; k < B; ++k) r = (a == k) ? v[k] : r;
  return r;
}

// y = yin + A x (yin may be NULL: y = A x; yin == y: in place).  Lane a < BR of a group owns
// component a of the block row; lane BR writes the pad (0) of a padded row.
template <int BR, int BC, int G>
__global__ void __launch_bounds__(256) k_gspmv(int nb, const int* __restrict__ rp, const int* __restrict__ ci,
                                               const double* __restrict__ val, const double* __restrict__ x,
                                               const double* yin, double* y) {
  constexpr int SR = vstride(BR);
  const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const int row = (int)(t / G), lig = (int)(t % G);
  const bool own = row < nb && lig < BR;
  const long long i = (long long)row * SR + lig;
  const double y0 = (own && yin) ? yin[i] : 0.0;
  double acc[BR];
  grp_row<BR, BC, G>(row, nb, lig, rp, ci, val, x, acc);
  if (own) y[i] = y0 + pick<BR>(acc, lig);
  else if (SR > BR && row < nb && lig == BR) y[i] = 0.0;
}

// fused Chebyshev step (same semantics as k_cheb_stencil) on a coarse level (padded vectors).
// Lane a < B of a group owns component a of the block row (its vector loads are issued before
// the row loop; one instruction serves a whole group), lane B writes the pad entries, and the
// D^-1 r product gathers r from the group's lanes by shuffles.
template <int B, int G>
__global__ void __launch_bounds__(256) k_gcheb(int nb, const int* __restrict__ rp, const int* __restrict__ ci,
                                               const double* __restrict__ val, const double* __restrict__ dinv,
                                               const double* __restrict__ d, double* __restrict__ r,
                                               double* __restrict__ x, double* __restrict__ dout, double c1,
                                               double c2, int first, int want_r, int want_d) {
  constexpr int S = vstride(B);
  const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const int row = (int)(t / G), lig = (int)(t % G);
  const bool own = row < nb && lig < B;
  const bool pad = S > B && row < nb && lig == B;
  const long long i = (long long)row * S + lig;
  double dv = 0.0, xv = 0.0, rv = 0.0, D[B];
#pragma unroll
  for (int k = 0; k < B; ++k) D[k] = 0.0;
  if (own) {
    dv = d[i];
    if (!first) xv = x[i];
    if (want_r) rv = r[i];
    if (want_d) {
#pragma unroll
      for (int k = 0; k < B; ++k) D[k] = __ldg(dinv + (long long)row * B * B + lig * B + k);
    }
  }
  double acc[B];
  if (want_r) grp_row<B, B, G>(row, nb, lig, rp, ci, val, d, acc);
  if (own) x[i] = xv + dv;
  else if (pad && first) x[i] = 0.0;
  if (!want_r) return;  // uniform across the launch
  rv -= own ? pick<B>(acc, lig) : 0.0;
  if (own) r[i] = rv;
  if (!want_d) return;
  double z = 0.0;
#pragma unroll
  for (int k = 0; k < B; ++k) z += D[k] * __shfl_sync(0xffffffffu, rv, k, G);
  if (own) dout[i] = c1 * dv + c2 * z;
  else if (pad) dout[i] = 0.0;
}

// r = b - A x (x may be NULL: r = b); d = c2 Dinv r (padded vectors)
template <int B, int G>
__global__ void __launch_bounds__(256) k_gresid(int nb, const int* __restrict__ rp, const int* __restrict__ ci,
                                                const double* __restrict__ val, const double* __restrict__ dinv,
                                                const double* __restrict__ b, const double* __restrict__ x,
                                                double* __restrict__ r, double* __restrict__ d, double c2) {
  constexpr int S = vstride(B);
  const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const int row = (int)(t / G), lig = (int)(t % G);
  const bool own = row < nb && lig < B;
  const long long i = (long long)row * S + lig;
  double bo = 0.0, D[B];
#pragma unroll
  for (int k = 0; k < B; ++k) D[k] = 0.0;
  if (own) {
    bo = b[i];
#pragma unroll
    for (int k = 0; k < B; ++k) D[k] = __ldg(dinv + (long long)row * B * B + lig * B + k);
  }
  double acc[B];
  if (x) grp_row<B, B, G>(row, nb, lig, rp, ci, val, x, acc);
  else {
#pragma unroll
    for (int a = 0; a < B; ++a) acc[a] = 0.0;
  }
  const double rv = bo - (own ? pick<B>(acc, lig) : 0.0);
  if (own) r[i] = rv;
  double z = 0.0;
#pragma unroll
  for (int k = 0; k < B; ++k) z += D[k] * __shfl_sync(0xffffffffu, rv, k, G);
  if (own) d[i] = c2 * z;
  else if (S > B && row < nb && lig == B) {
    r[i] = 0.0;
    d[i] = 0.0;
  }
}

// ------------------------------------------------------------------ row-component kernels (b = 4)
// With nullspace_dim = 4 (reading G30) coarse blocks are 4 x 4 = 128 B, i.e. one block row of
// a block is 32 B: BR consecutive lanes read the BR rows of ONE block (row-major block storage,
// Level::val / Pval / Rval as the SpGEMM writes them) with a single 32-B (BC = 4) or 16-B
// (BC = 2) load each, and the block's x entries with one 32-B / 16-B load (same address for
// the BR lanes: one transaction).  A group of G = BR * S lanes owns one block row and keeps
// S blocks in flight; lane l accumulates row component a = l % BR over slot l / BR's blocks,
// then the S partial sums of component a are combined by an xor-butterfly (fixed order).
template <int BC>
__device__ __forceinline__ void load_row(const double* __restrict__ p, double v[BC]) {
  if constexpr (BC == 4) {
    asm("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(v[0]), "=d"(v[1]), "=d"(v[2]), "=d"(v[3]) : "l"(p));
  } else {
    const double2 w = __ldg(reinterpret_cast<const double2*>(p));
    v[0] = w.x;
    v[1] = w.y;
  }
}

template <int BR, int BC, int S, bool PF = true>
__device__ __forceinline__ double grpA_row(int row, int nb, int lig, const int* __restrict__ rp,
                                           const int* __restrict__ ci, const double* __restrict__ val,
                                           const double* __restrict__ x) {
  constexpr int G = BR * S;
  const int a = lig % BR, slot = lig / BR;
  double acc = 0.0;
  if (row < nb) {
    const int e1 = __ldg(rp + row + 1);
    int e = __ldg(rp + row) + slot;
    if constexpr (PF) {
      // ptxas schedules each block's FMAs right behind its loads (SASS: LDG, LDG, DFMA ...), so a
      // slot has one or two 32-byte value loads in flight.  The lane's pieces of its next blocks
      // are requested here as L1 prefetches (no destination register, nothing to wait on); the
      // loop's loads then hit L1 or join the miss in flight.
#pragma unroll
      for (int q = 0; q < 4; ++q)
        if (e + q * S < e1)
          asm volatile("prefetch.global.L1 [%0];" ::"l"(val + ((long long)(e + q * S) * BR + a) * BC));
    }
    for (; e + S < e1; e += 2 * S) {
      const int c0 = __ldg(ci + e), c1 = __ldg(ci + e + S);
      double v0[BC], v1[BC], x0[BC], x1[BC];
      load_row<BC>(val + ((long long)e * BR + a) * BC, v0);
      load_row<BC>(val + ((long long)(e + S) * BR + a) * BC, v1);
      load_xblk<BC>(x, c0, x0);
      load_xblk<BC>(x, c1, x1);
#pragma unroll
      for (int b = 0; b < BC; ++b) acc += v0[b] * x0[b];
#pragma unroll
      for (int b = 0; b < BC; ++b) acc += v1[b] * x1[b];
    }
    for (; e < e1; e += S) {
      double v0[BC], x0[BC];
      load_row<BC>(val + ((long long)e * BR + a) * BC, v0);
      load_xblk<BC>(x, __ldg(ci + e), x0);
#pragma unroll
      for (int b = 0; b < BC; ++b) acc += v0[b] * x0[b];
    }
  }
#pragma unroll
  for (int off = BR; off < G; off <<= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off, G);
  return acc;
}

// y = yin + A x (yin may be NULL; yin == y: in place), row-major BR x BC blocks
template <int BR, int BC, int S>
__global__ void __launch_bounds__(256) k_aspmv(int nb, const int* __restrict__ rp, const int* __restrict__ ci,
                                               const double* __restrict__ val, const double* __restrict__ x,
                                               const double* yin, double* y) {
  constexpr int G = BR * S, SR = vstride(BR);
  const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const int row = (int)(t / G), lig = (int)(t % G);
  const bool own = row < nb && lig < BR;
  const long long i = (long long)row * SR + lig;
  const double acc = grpA_row<BR, BC, S>(row, nb, lig, rp, ci, val, x);
  if (own) y[i] = (yin ? yin[i] : 0.0) + acc;
}

// Chebyshev step on a b = 4 level (semantics of k_gcheb).  LATE: the row's own vector entries
// and D^-1 block are loaded after the SpMV (fewer live registers during the gather loop, at
// the cost of one more round trip); otherwise before it.
template <int S, bool LATE, bool PF = true>
__global__ void __launch_bounds__(256) k_acheb4(int nb, const int* __restrict__ rp, const int* __restrict__ ci,
                                                const double* __restrict__ val, const double* __restrict__ dinv,
                                                const double* __restrict__ d, double* __restrict__ r,
                                                double* __restrict__ x, double* __restrict__ dout, double c1,
                                                double c2, int first, int want_r, int want_d) {
  constexpr int G = 4 * S;
  const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const int row = (int)(t / G), lig = (int)(t % G);
  const bool own = row < nb && lig < 4;
  const long long i = (long long)row * 4 + lig;
  double dv = 0.0, xv = 0.0, rv = 0.0, D[4] = {0.0, 0.0, 0.0, 0.0};
  if (!LATE && own) {
    dv = d[i];
    if (!first) xv = x[i];
    if (want_r) rv = r[i];
    if (want_d) load_row<4>(dinv + (long long)row * 16 + lig * 4, D);
  }
  double acc = 0.0;
  if (want_r) acc = grpA_row<4, 4, S, PF>(row, nb, lig, rp, ci, val, d);
  if (LATE && own) {
    dv = d[i];
    if (!first) xv = x[i];
    if (want_r) rv = r[i];
    if (want_d) load_row<4>(dinv + (long long)row * 16 + lig * 4, D);
  }
  if (own) x[i] = xv + dv;
  if (!want_r) return;  // uniform across the launch
  rv -= acc;
  if (own) r[i] = rv;
  if (!want_d) return;
  double z = 0.0;
#pragma unroll
  for (int k = 0; k < 4; ++k) z += D[k] * __shfl_sync(0xffffffffu, rv, k, G);
  if (own) dout[i] = c1 * dv + c2 * z;
}

// r = b - A x (x may be NULL: r = b); d = c2 Dinv r on a b = 4 level
template <int S, bool PF = true>
__global__ void __launch_bounds__(256) k_aresid4(int nb, const int* __restrict__ rp, const int* __restrict__ ci,
                                                 const double* __restrict__ val, const double* __restrict__ dinv,
                                                 const double* __restrict__ b, const double* __restrict__ x,
                                                 double* __restrict__ r, double* __restrict__ d, double c2) {
  constexpr int G = 4 * S;
  const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const int row = (int)(t / G), lig = (int)(t % G);
  const bool own = row < nb && lig < 4;
  const long long i = (long long)row * 4 + lig;
  double bo = 0.0, D[4] = {0.0, 0.0, 0.0, 0.0};
  const double acc = x ? grpA_row<4, 4, S, PF>(row, nb, lig, rp, ci, val, x) : 0.0;
  if (own) {  // after the gather (fewer live registers in the loop, as k_acheb4)
    bo = b[i];
    load_row<4>(dinv + (long long)row * 16 + lig * 4, D);
  }
  const double rv = bo - acc;
  if (own) r[i] = rv;
  double z = 0.0;
#pragma unroll
  for (int k = 0; k < 4; ++k) z += D[k] * __shfl_sync(0xffffffffu, rv, k, G);
  if (own) d[i] = c2 * z;
}

// CTA per block row (small coarse levels, ~50-110 blocks per row): 256 / BR slots keep the whole
// row in flight at once (one dependent load chain instead of ~7), partial sums combined by an
// xor-butterfly inside each warp and then across the 8 warps in a fixed order.  Thread a < BR
// returns component a of the row, the others 0.
template <int BR, int BC>
__device__ __forceinline__ double cta_row(int row, const int* __restrict__ rp, const int* __restrict__ ci,
                                          const double* __restrict__ val, const double* __restrict__ x,
                                          double (*sh)[4]) {
  constexpr int S = 256 / BR;
  const int t = threadIdx.x, a = t % BR, slot = t / BR;
  double acc = 0.0;
  const int e1 = __ldg(rp + row + 1);
  int e = __ldg(rp + row) + slot;
  if (e + S < e1) asm volatile("prefetch.global.L1 [%0];" ::"l"(val + ((long long)(e + S) * BR + a) * BC));
  for (; e + S < e1; e += 2 * S) {
    const int c0 = __ldg(ci + e), c1 = __ldg(ci + e + S);
    double v0[BC], v1[BC], x0[BC], x1[BC];
    load_row<BC>(val + ((long long)e * BR + a) * BC, v0);
    load_row<BC>(val + ((long long)(e + S) * BR + a) * BC, v1);
    load_xblk<BC>(x, c0, x0);
    load_xblk<BC>(x, c1, x1);
#pragma unroll
    for (int b = 0; b < BC; ++b) acc += v0[b] * x0[b];
#pragma unroll
    for (int b = 0; b < BC; ++b) acc += v1[b] * x1[b];
  }
  if (e < e1) {
    double v0[BC], x0[BC];
    load_row<BC>(val + ((long long)e * BR + a) * BC, v0);
    load_xblk<BC>(x, __ldg(ci + e), x0);
#pragma unroll
    for (int b = 0; b < BC; ++b) acc += v0[b] * x0[b];
  }
#pragma unroll
  for (int off = BR; off < 32; off <<= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
  if ((t & 31) < BR) sh[t >> 5][a] = acc;
  __syncthreads();
  double tot = 0.0;
  if (t < BR) {
#pragma unroll
    for (int w = 0; w < 8; ++w) tot += sh[w][t];
  }
  return tot;
}

template <int BR, int BC>
__global__ void __launch_bounds__(256) k_aspmv_cta(int nb, const int* __restrict__ rp, const int* __restrict__ ci,
                                                   const double* __restrict__ val, const double* __restrict__ x,
                                                   const double* yin, double* y) {
  __shared__ double sh[8][4];
  constexpr int SR = vstride(BR);
  const int row = blockIdx.x, t = threadIdx.x;
  const double acc = cta_row<BR, BC>(row, rp, ci, val, x, sh);
  if (t < BR) {
    const long long i = (long long)row * SR + t;
    y[i] = (yin ? yin[i] : 0.0) + acc;
  }
}

__global__ void __launch_bounds__(256) k_acheb4_cta(int nb, const int* __restrict__ rp, const int* __restrict__ ci,
                                                    const double* __restrict__ val, const double* __restrict__ dinv,
                                                    const double* __restrict__ d, double* __restrict__ r,
                                                    double* __restrict__ x, double* __restrict__ dout, double c1,
                                                    double c2, int first, int want_r, int want_d) {
  __shared__ double sh[8][4];
  const int row = blockIdx.x, t = threadIdx.x;
  const long long i = (long long)row * 4 + t;
  const double acc = want_r ? cta_row<4, 4>(row, rp, ci, val, d, sh) : 0.0;
  if (t >= 4) return;  // threads 0..3 own the row (lanes 0..3 of warp 0)
  const double dv = d[i];
  const double xv = first ? 0.0 : x[i];
  x[i] = xv + dv;
  if (!want_r) return;
  const double rv = r[i] - acc;
  r[i] = rv;
  if (!want_d) return;
  double D[4];
  load_row<4>(dinv + (long long)row * 16 + t * 4, D);
  double z = 0.0;
#pragma unroll
  for (int k = 0; k < 4; ++k) z += D[k] * __shfl_sync(0xfu, rv, k, 4);
  dout[i] = c1 * dv + c2 * z;
}

__global__ void __launch_bounds__(256) k_aresid4_cta(int nb, const int* __restrict__ rp, const int* __restrict__ ci,
                                                     const double* __restrict__ val, const double* __restrict__ dinv,
                                                     const double* __restrict__ b, const double* __restrict__ x,
                                                     double* __restrict__ r, double* __restrict__ d, double c2) {
  __shared__ double sh[8][4];
  const int row = blockIdx.x, t = threadIdx.x;
  const long long i = (long long)row * 4 + t;
  const double acc = x ? cta_row<4, 4>(row, rp, ci, val, x, sh) : 0.0;
  if (t >= 4) return;
  const double rv = b[i] - acc;
  r[i] = rv;
  double D[4];
  load_row<4>(dinv + (long long)row * 16 + t * 4, D);
  double z = 0.0;
#pragma unroll
  for (int k = 0; k < 4; ++k) z += D[k] * __shfl_sync(0xfu, rv, k, 4);
  d[i] = c2 * z;
}

// CTA-per-row form for levels whose rows are long (measured: small coarse levels were paced by
// ~7 sequential dependent-load rounds per row at 32 lanes per row)
// (config 4: level 3, 9.9 k rows of 67 blocks, runs faster as 32-lane groups — 28 vs 40 us per
// Chebyshev step: CTA-per-row pays only where the rows are few)
static bool use_cta_rows(long long nnzb, int nb) {
  static const double minrow = getenv("SEAICE_CTA_MINROW") ? atof(getenv("SEAICE_CTA_MINROW")) : 32.0;  // tuning aid
  // (MIS(3) coarse levels have ~45 blocks per row: 32 instead of 48 measured 2433 -> 2415 us per V-cycle)
  static const int maxnb = getenv("SEAICE_CTA_MAXNB") ? atoi(getenv("SEAICE_CTA_MAXNB")) : 4096;
  return nb > 0 && nb <= maxnb && (double)nnzb / nb >= minrow;
}

// slots (blocks in flight per block row) for the row-component kernels
static int pick_slots(long long nnzb, int nb, int BR) {
  static const int shift = getenv("SEAICE_SLOT_SHIFT") ? atoi(getenv("SEAICE_SLOT_SHIFT")) : 0;  // tuning aid
  const double avg = nb > 0 ? (double)nnzb / nb : 1.0;
  int s = avg <= 3.0 ? 1 : avg <= 6.0 ? 2 : avg <= 16.0 ? 4 : 8;
  if ((long long)nb * 32 <= 148LL * 2048) s = 8;  // small levels: shortest dependent-load chains
  s = shift >= 0 ? (s << shift) : (s >> -shift);
  const int smax = 32 / BR < 8 ? 32 / BR : 8;
  return s < 1 ? 1 : (s > smax ? smax : s);
}
#define SI_SDISPATCH(S_, CALL)                        \
  switch (S_) {                                       \
    case 1: { constexpr int SS = 1; CALL; } break;   \
    case 2: { constexpr int SS = 2; CALL; } break;   \
    case 4: { constexpr int SS = 4; CALL; } break;   \
    default: { constexpr int SS = 8; CALL; } break;  \
  }
// threads per block of the row-component kernels (tuning aid SEAICE_ABLOCK; measured at config 4:
// 64 / 128 / 256 threads within +-2 % of each other; a persistent grid of 8 x 148 CTAs looping
// over the rows ran level 1 at 4.1 instead of 4.8 TB/s)
static int ablock() {
  static const int b = getenv("SEAICE_ABLOCK") ? atoi(getenv("SEAICE_ABLOCK")) : 256;
  return b;
}
static int agrid(int nb, int G) { return (int)(((long long)nb * G + ablock() - 1) / ablock()); }

static int pick_group(long long nnzb, int nb) {
  static const int shift = getenv("SEAICE_GROUP_SHIFT") ? atoi(getenv("SEAICE_GROUP_SHIFT")) : 0;  // tuning aid
  const double avg = nb > 0 ? (double)nnzb / nb : 1.0;
  // measured on B200 (scripts/vcycle_bench.py): ~2-4 blocks per lane is the sweet spot
  int g = avg <= 14.0 ? 4 : avg <= 40.0 ? 8 : avg <= 120.0 ? 16 : 32;
  // small levels cannot fill the GPU anyway: a full warp per row shortens each row's chain of
  // dependent (column index -> x gather) loads, which is what these launches wait on
  if ((long long)nb * 32 <= 148LL * 2048) g = 32;
  g = shift >= 0 ? (g << shift) : (g >> -shift);
  return g < 4 ? 4 : (g > 32 ? 32 : g);
}
static int ggrid(int nb, int G) { return (int)(((long long)nb * G + 255) / 256); }

#define SI_GDISPATCH(G, CALL) \
  switch (G) {                \
    case 4: { constexpr int GG = 4; CALL; } break;   \
    case 8: { constexpr int GG = 8; CALL; } break;   \
    case 16: { constexpr int GG = 16; CALL; } break; \
    default: { constexpr int GG = 32; CALL; } break; \
  }

static void gspmv(Ctx& c, int nb, int br, int bc, long long nnzb, const int* rp, const int* ci, const double* val,
                  const double* x, const double* yin, double* y) {
  const int G = pick_group(nnzb, nb);
  if (br == 3 && bc == 3) {
    SI_GDISPATCH(G, (k_gspmv<3, 3, GG><<<ggrid(nb, GG), 256, 0, c.s>>>(nb, rp, ci, val, x, yin, y)))
  } else if (br == 2 && bc == 3) {
    // finest prolongation (~3 blocks per fine node): 2 lanes per row (one per component) measured
    // 8 % faster than 4 on B200 (fewer idle lanes, same coalescing)
    static const int g2 = getenv("SEAICE_P0_G") ? atoi(getenv("SEAICE_P0_G")) : 2;  // tuning aid
    if (g2 == 2 && nnzb <= 4LL * nb) k_gspmv<2, 3, 2><<<ggrid(nb, 2), 256, 0, c.s>>>(nb, rp, ci, val, x, yin, y);
    else SI_GDISPATCH(G, (k_gspmv<2, 3, GG><<<ggrid(nb, GG), 256, 0, c.s>>>(nb, rp, ci, val, x, yin, y)))
  } else if (br == 3 && bc == 2) {
    SI_GDISPATCH(G, (k_gspmv<3, 2, GG><<<ggrid(nb, GG), 256, 0, c.s>>>(nb, rp, ci, val, x, yin, y)))
  } else if (br == 4 || bc == 4) {
    // b = 4 hierarchies (reading G30): row-major blocks, row-component lanes (val is AoS here)
    const int Sl = pick_slots(nnzb, nb, br);
    if (use_cta_rows(nnzb, nb)) {
      if (br == 4 && bc == 4) k_aspmv_cta<4, 4><<<nb, 256, 0, c.s>>>(nb, rp, ci, val, x, yin, y);
      else if (br == 2) k_aspmv_cta<2, 4><<<nb, 256, 0, c.s>>>(nb, rp, ci, val, x, yin, y);
      else k_aspmv_cta<4, 2><<<nb, 256, 0, c.s>>>(nb, rp, ci, val, x, yin, y);
    } else if (br == 4 && bc == 4) {
      SI_SDISPATCH(Sl, (k_aspmv<4, 4, SS><<<agrid(nb, 4 * SS), ablock(), 0, c.s>>>(nb, rp, ci, val, x, yin, y)))
    } else if (br == 2) {
      SI_SDISPATCH(Sl, (k_aspmv<2, 4, SS><<<agrid(nb, 2 * SS), ablock(), 0, c.s>>>(nb, rp, ci, val, x, yin, y)))
    } else {
      SI_SDISPATCH(Sl, (k_aspmv<4, 2, SS><<<agrid(nb, 4 * SS), ablock(), 0, c.s>>>(nb, rp, ci, val, x, yin, y)))
    }
  } else {
    SI_GDISPATCH(G, (k_gspmv<2, 2, GG><<<ggrid(nb, GG), 256, 0, c.s>>>(nb, rp, ci, val, x, yin, y)))
  }
  SI_LAUNCHED(c);
}

// ------------------------------------------------------------------ host: setup
static BsrMat view(Level& L) { return BsrMat{L.nb, L.nb, L.b, L.b, L.nnzb, L.rp.get(), L.ci.get(), L.val.get()}; }

template <int B>
static double power_lambda(Ctx& c, Level& L, int lvl) {
  const long long N = (long long)L.nb * vstride(B);  // storage length (pads stay 0)
  Scratch S(c);
  double* x = S.get<double>(N);
  double* y = S.get<double>(N);
  k_power_start<<<grid_for(N), kThreads, 0, c.s>>>(N, B, vstride(B), salt(c.p.amg_seed, lvl, 7), x);
  SI_LAUNCHED(c);
  // normalisation stays on the device (no host round trip per iteration); lambda is
  // ||D^-1 A x|| of the last unit-norm iterate
  const int g = red_grid(N);
  double* part = S.get<double>(g);
  double* ny2 = S.get<double>(1);
  k_sqnorm_part<<<g, kThreads, 0, c.s>>>(N, x, part);
  k_sum_to<<<1, 1024, 0, c.s>>>(part, g, ny2);
  k_scale_rsqrt<<<grid_for(N), kThreads, 0, c.s>>>(N, x, ny2, x);
  SI_LAUNCHED(c);
  c.launches += 2;
  for (int it = 0; it < c.p.power_iters; ++it) {
    if (lvl == 0 && B == 2)
      stencil_spmv(c, x, y);  // the finest operator is the stencil itself
    else
      gspmv(c, L.nb, B, B, L.nnzb, L.rp.get(), L.ci.get(), B == 4 ? L.val.get() : L.valT.get(), x, nullptr, y);
    k_dinv_apply<B><<<grid_for(L.nb), kThreads, 0, c.s>>>(L.nb, L.dinv.get(), y);
    k_sqnorm_part<<<g, kThreads, 0, c.s>>>(N, y, part);
    k_sum_to<<<1, 1024, 0, c.s>>>(part, g, ny2);
    k_scale_rsqrt<<<grid_for(N), kThreads, 0, c.s>>>(N, y, ny2, x);
    SI_LAUNCHED(c);
    c.launches += 3;
  }
  const double lam = std::sqrt(read_scalar(c, ny2));
  SI_CHECK(std::isfinite(lam) && lam > 0.0, SEAICE_ENONFINITE, "AMG power iteration failed");
  return lam;
}

template <int B>
static void level_diag(Ctx& c, Level& L, Scratch& S, double* dnorm) {
  L.dinv.ensure(c.al, (size_t)L.nb * B * B);
  k_diag_inv<B><<<grid_for(L.nb), kThreads, 0, c.s>>>(L.nb, L.rp.get(), L.ci.get(), L.val.get(), L.dinv.get(),
                                                      dnorm, c.flag.get());
  SI_LAUNCHED(c);
}

// Build aggregates of level L.  Returns number of aggregates.
template <int B>
static int aggregate_level(Ctx& c, Level& L, int lvl, const double* dnorm, Scratch& S) {
  const int nb = L.nb;
  double* sval = S.get<double>(L.nnzb);
  int* deg = S.get<int>(nb + 1);
  k_strength<B><<<grid_for(nb), kThreads, 0, c.s>>>(nb, L.rp.get(), L.ci.get(), L.val.get(), dnorm,
                                                     c.p.amg_theta * c.p.amg_theta, sval, deg);
  SI_LAUNCHED(c);
  SI_CUDA(cudaMemsetAsync(deg + nb, 0, sizeof(int), c.s));
  int* grp = S.get<int>(nb + 1);
  exclusive_scan(c, deg, grp, nb + 1);
  const int gnnz = read_scalar(c, grp + nb);
  int* gci = S.get<int>(gnnz);
  double* gs = S.get<double>(gnnz);
  k_strength_compact<<<grid_for(nb), kThreads, 0, c.s>>>(nb, L.rp.get(), L.ci.get(), sval, grp, gci, gs);
  SI_LAUNCHED(c);
  // MIS(2)
  unsigned long long* key = S.get<unsigned long long>(nb);
  unsigned long long* T1 = S.get<unsigned long long>(nb);
  unsigned long long* T2 = S.get<unsigned long long>(nb);
  int* und = S.get<int>(1);
  k_mis_init<<<grid_for(nb), kThreads, 0, c.s>>>(nb, grp, salt(c.p.amg_seed, lvl, 1), key);
  SI_LAUNCHED(c);
  const int dist = (lvl == 0) ? c.p.agg_dist0 : c.p.agg_dist;  // MIS(d), d = 1..3
  for (int round = 0;; ++round) {
    SI_CHECK(round < 10000, SEAICE_ECUDA, "MIS did not terminate");
    const unsigned long long* tin = key;
    for (int p = 0; p < dist; ++p) {  // closed-neighbourhood max, dist times (ping-pong T1 / T2)
      unsigned long long* tout = (p & 1) ? T2 : T1;
      k_mis_max<<<grid_for(nb), kThreads, 0, c.s>>>(nb, grp, gci, tin, tout);
      tin = tout;
    }
    SI_CUDA(cudaMemsetAsync(und, 0, sizeof(int), c.s));
    k_mis_update<<<grid_for(nb), kThreads, 0, c.s>>>(nb, key, tin, und);
    SI_LAUNCHED(c);
    c.launches += dist;
    if (read_scalar(c, und) == 0) break;
  }
  int* isroot = S.get<int>(nb + 1);
  int* rootid = S.get<int>(nb + 1);
  k_roots<<<grid_for(nb), kThreads, 0, c.s>>>(nb, key, isroot);
  SI_LAUNCHED(c);
  SI_CUDA(cudaMemsetAsync(isroot + nb, 0, sizeof(int), c.s));
  exclusive_scan(c, isroot, rootid, nb + 1);
  const int na = read_scalar(c, rootid + nb);
  L.agg.ensure(c.al, nb);
  int* a1 = S.get<int>(nb);
  int* a2 = S.get<int>(nb);
  k_agg_roots<<<grid_for(nb), kThreads, 0, c.s>>>(nb, isroot, rootid, a1);
  SI_LAUNCHED(c);
  k_agg_join<<<grid_for(nb), kThreads, 0, c.s>>>(nb, grp, gci, gs, a1, a2);   // phase 1 (roots only assigned)
  k_agg_join<<<grid_for(nb), kThreads, 0, c.s>>>(nb, grp, gci, gs, a2, a1);   // phase 2
  k_agg_join<<<grid_for(nb), kThreads, 0, c.s>>>(nb, grp, gci, gs, a1, L.agg.get());  // phase 3
  SI_LAUNCHED(c);
  c.launches += 2;
  return na;
}

template <int B, int K>
static void build_transfer(Ctx& c, Level& L, Level& Lc, int lvl, int na, Scratch& S) {
  const int nb = L.nb;
  // members sorted by aggregate (stable: node order inside an aggregate); kept with the P_tent
  // pattern for the numeric-only setup (reading G32)
  int* key = S.get<int>(nb);
  int* idx = S.get<int>(nb);
  int* skey = S.get<int>(nb);
  L.mem.ensure(c.al, nb);
  int* members = L.mem.get();
  k_agg_key<<<grid_for(nb), kThreads, 0, c.s>>>(nb, L.agg.get(), na, key, idx);
  SI_LAUNCHED(c);
  {
    int bits = 1;
    while ((1LL << bits) <= na) ++bits;
    size_t tmp = 0;
    SI_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp, key, skey, idx, members, nb, 0, bits, c.s));
    Scratch St(c);
    void* t = St.get<char>(tmp + 16);
    SI_CUDA(cub::DeviceRadixSort::SortPairs(t, tmp, key, skey, idx, members, nb, 0, bits, c.s));
    c.launches += 2;
  }
  L.mstart.ensure(c.al, na + 1);
  int* start = L.mstart.get();
  k_seg_starts<<<grid_for(na + 1), kThreads, 0, c.s>>>(na, nb, skey, start);
  SI_LAUNCHED(c);
  // P_tent pattern: one block per aggregated node
  int* f = S.get<int>(nb + 1);
  L.ptrp.ensure(c.al, nb + 1);
  int* ptrp = L.ptrp.get();
  k_flag_agg<<<grid_for(nb), kThreads, 0, c.s>>>(nb, L.agg.get(), f);
  SI_LAUNCHED(c);
  SI_CUDA(cudaMemsetAsync(f + nb, 0, sizeof(int), c.s));
  exclusive_scan(c, f, ptrp, nb + 1);
  const int ptn = read_scalar(c, ptrp + nb);
  L.ptn = ptn;
  L.ptci.ensure(c.al, ptn);
  L.ptval.ensure(c.al, (size_t)ptn * B * K);
  int* ptci = L.ptci.get();
  double* ptval = L.ptval.get();
  k_ptent_ci<<<grid_for(nb), kThreads, 0, c.s>>>(nb, L.agg.get(), ptrp, ptci);
  SI_LAUNCHED(c);
  Lc.B.ensure(c.al, (size_t)na * K * K);
  k_tentative_w<B, K><<<(int)(((long long)na * 32 + 127) / 128), 128, 0, c.s>>>(na, start, members, L.B.get(), ptrp,
                                                                                 ptval, Lc.B.get());
  SI_LAUNCHED(c);
  tick(c, "tentative", lvl);
  BsrMat Pt{nb, na, B, K, ptn, ptrp, ptci, ptval};
  // T = A P_tent ; P = P_tent - omega Dinv T  (P takes T's pattern)
  const double omega = 4.0 / (3.0 * L.lmax);
  bool fused = false;
  if (B == 2 && c.p.spgemm_path == 0) {  // finest level: one-pass smoothed prolongator
    int* cnt = S.get<int>(nb + 1);
    SI_CUDA(cudaMemsetAsync(c.flag.get() + 2, 0, sizeof(int), c.s));
    k_ptsm_count<<<grid_for(nb + 1), kThreads, 0, c.s>>>(nb, L.rp.get(), L.ci.get(), L.agg.get(), cnt,
                                                        c.flag.get() + 2);
    SI_LAUNCHED(c);
    if (read_scalar(c, c.flag.get() + 2) == 0) {
      L.Prp.ensure(c.al, nb + 1);
      exclusive_scan(c, cnt, L.Prp.get(), nb + 1);
      L.Pnnzb = read_scalar(c, L.Prp.get() + nb);
      L.Pci.ensure(c.al, L.Pnnzb);
      L.Pval.ensure(c.al, (size_t)L.Pnnzb * B * K);
      k_ptsm_fill<B, K><<<grid_for(nb, 128), 128, 0, c.s>>>(nb, L.rp.get(), L.ci.get(), L.val.get(), L.agg.get(),
                                                           ptrp, ptval, L.dinv.get(), omega, L.Prp.get(),
                                                           L.Pci.get(), L.Pval.get());
      SI_LAUNCHED(c);
      fused = true;
      L.plan[0] = SgPlan{};  // SG_NONE: the one-pass kernel
      tick(c, "A*Pt+smooth", lvl);
    }
  }
  if (!fused) {
    long long tn = 0;
    spgemm<B, B, K>(c, view(L), Pt, L.Prp, L.Pci, L.Tval, tn, L.plan[0]);
    tick(c, "A*Pt", lvl);
    L.Pnnzb = tn;
    L.Pval.ensure(c.al, (size_t)tn * B * K);
    k_smooth_p<B, K><<<grid_for(nb), kThreads, 0, c.s>>>(nb, L.Prp.get(), L.Pci.get(), L.Tval.get(), L.dinv.get(),
                                                      L.agg.get(), ptrp, ptval, omega, L.Pval.get());
    SI_LAUNCHED(c);
  }
  L.nbc = na;
  BsrMat P{nb, na, B, K, L.Pnnzb, L.Prp.get(), L.Pci.get(), L.Pval.get()};
  tick(c, "smoothP", lvl);
  // R = P^T
  transpose<B, K>(c, P, L.Rrp, L.Rci, L.Rval, L.tperm, L.trow);
  L.Rnnzb = L.Pnnzb;
  tick(c, "transpose", lvl);
  BsrMat R{na, nb, K, B, L.Rnnzb, L.Rrp.get(), L.Rci.get(), L.Rval.get()};
  if (B == 2) {
    // finest level: A_c = (R A) P — the R A intermediate has one row per aggregate instead of
    // A P's one row per fine node and the product count halves (measured 37 -> 27 ms at n = 2048)
    spgemm<K, B, B>(c, R, view(L), L.Irp, L.Ici, L.Ival, L.Innzb, L.plan[1]);
    tick(c, "R*A", lvl);
    BsrMat RA{na, nb, K, B, L.Innzb, L.Irp.get(), L.Ici.get(), L.Ival.get()};
    spgemm<K, B, K>(c, RA, P, Lc.rp, Lc.ci, Lc.val, Lc.nnzb, L.plan[2]);
    tick(c, "RA*P", lvl);
  } else {
    // coarse levels (wide rows): A_c = R (A P) measured faster
    spgemm<B, B, K>(c, view(L), P, L.Irp, L.Ici, L.Ival, L.Innzb, L.plan[1]);
    tick(c, "A*P", lvl);
    BsrMat AP{nb, na, B, K, L.Innzb, L.Irp.get(), L.Ici.get(), L.Ival.get()};
    spgemm<K, B, K>(c, R, AP, Lc.rp, Lc.ci, Lc.val, Lc.nnzb, L.plan[2]);
    tick(c, "R*AP", lvl);
  }
  Lc.nb = na;
  Lc.b = K;
  L.K = K;
  k_fix_zero_diag<K><<<grid_for(na), kThreads, 0, c.s>>>(na, Lc.rp.get(), Lc.ci.get(), Lc.val.get());
  SI_LAUNCHED(c);
}

// Numeric-only transfer of reading G32: the aggregates, every sparsity pattern and the SpGEMM
// kernel choices of the last full setup are kept; the values are recomputed by the same kernels
// (P_tent by MGS of the current near-nullspace, smoothed P with the current D^-1 and lambda,
// R = P^T by the kept permutation, the Galerkin products on their kept patterns).
template <int B, int K>
static void build_transfer_numeric(Ctx& c, Level& L, Level& Lc, int lvl) {
  const int nb = L.nb, na = L.nbc;
  k_tentative_w<B, K><<<(int)(((long long)na * 32 + 127) / 128), 128, 0, c.s>>>(
      na, L.mstart.get(), L.mem.get(), L.B.get(), L.ptrp.get(), L.ptval.get(), Lc.B.get());
  SI_LAUNCHED(c);
  tick(c, "tentative", lvl);
  BsrMat Pt{nb, na, B, K, L.ptn, L.ptrp.get(), L.ptci.get(), L.ptval.get()};
  const double omega = 4.0 / (3.0 * L.lmax);
  if (L.plan[0].kind == SG_NONE) {
    k_ptsm_fill<B, K><<<grid_for(nb, 128), 128, 0, c.s>>>(nb, L.rp.get(), L.ci.get(), L.val.get(), L.agg.get(),
                                                         L.ptrp.get(), L.ptval.get(), L.dinv.get(), omega,
                                                         L.Prp.get(), L.Pci.get(), L.Pval.get());
    SI_LAUNCHED(c);
  } else {
    sg_numeric<B, B, K>(c, L.plan[0], view(L), Pt, L.Prp.get(), L.Pci.get(), L.Tval.get());
    k_smooth_p<B, K><<<grid_for(nb), kThreads, 0, c.s>>>(nb, L.Prp.get(), L.Pci.get(), L.Tval.get(), L.dinv.get(),
                                                      L.agg.get(), L.ptrp.get(), L.ptval.get(), omega, L.Pval.get());
    SI_LAUNCHED(c);
  }
  tick(c, "smoothP", lvl);
  if (L.Pnnzb > 0) {
    k_transpose_gather<B, K><<<grid_for(L.Pnnzb), kThreads, 0, c.s>>>(L.Pnnzb, L.tperm.get(), L.trow.get(),
                                                                     L.Pval.get(), L.Rci.get(), L.Rval.get());
    SI_LAUNCHED(c);
  }
  tick(c, "transpose", lvl);
  BsrMat P{nb, na, B, K, L.Pnnzb, L.Prp.get(), L.Pci.get(), L.Pval.get()};
  BsrMat R{na, nb, K, B, L.Rnnzb, L.Rrp.get(), L.Rci.get(), L.Rval.get()};
  if (B == 2) {
    sg_numeric<K, B, B>(c, L.plan[1], R, view(L), L.Irp.get(), L.Ici.get(), L.Ival.get());
    tick(c, "R*A", lvl);
    BsrMat RA{na, nb, K, B, L.Innzb, L.Irp.get(), L.Ici.get(), L.Ival.get()};
    sg_numeric<K, B, K>(c, L.plan[2], RA, P, Lc.rp.get(), Lc.ci.get(), Lc.val.get());
    tick(c, "RA*P", lvl);
  } else {
    sg_numeric<B, B, K>(c, L.plan[1], view(L), P, L.Irp.get(), L.Ici.get(), L.Ival.get());
    tick(c, "A*P", lvl);
    BsrMat AP{nb, na, B, K, L.Innzb, L.Irp.get(), L.Ici.get(), L.Ival.get()};
    sg_numeric<K, B, K>(c, L.plan[2], R, AP, Lc.rp.get(), Lc.ci.get(), Lc.val.get());
    tick(c, "R*AP", lvl);
  }
  k_fix_zero_diag<K><<<grid_for(na), kThreads, 0, c.s>>>(na, Lc.rp.get(), Lc.ci.get(), Lc.val.get());
  SI_LAUNCHED(c);
}

static void coarse_factor(Ctx& c, Level& L) {
  const int nd = L.nb * L.b;
  Scratch S(c);
  double* D = S.get<double>((size_t)nd * nd);
  double* Y = S.get<double>((size_t)nd * nd);
  SI_CUDA(cudaMemsetAsync(D, 0, sizeof(double) * nd * nd, c.s));
  k_bsr_to_dense<<<grid_for(L.nb), kThreads, 0, c.s>>>(L.nb, L.b, L.rp.get(), L.ci.get(), L.val.get(), nd, D);
  SI_LAUNCHED(c);
  k_cholesky<<<1, 1024, 0, c.s>>>(nd, D, c.flag.get());
  SI_LAUNCHED(c);
  c.cinv.ensure(c.al, (size_t)nd * nd);
  k_chol_inverse<<<grid_for(nd, 64), 64, 0, c.s>>>(nd, D, Y, c.cinv.get());
  SI_LAUNCHED(c);
  c.cn = nd;
  SI_CUDA(cudaStreamSynchronize(c.s));
}

void vgraph_destroy(Ctx& c);

void amg_free(Ctx& c) {
  vgraph_destroy(c);
  c.vc_in.free_();
  c.vc_out.free_();
  for (auto& L : c.lv) {
    DBuf<int>* ib[] = {&L.rp,   &L.ci,   &L.Prp,  &L.Pci,   &L.Rrp,  &L.Rci, &L.agg, &L.mem,
                       &L.mstart, &L.ptrp, &L.ptci, &L.tperm, &L.trow, &L.Irp, &L.Ici};
    DBuf<double>* db[] = {&L.val,  &L.dinv, &L.Pval,  &L.Rval,  &L.B,     &L.x,     &L.rhs,   &L.r, &L.d,
                          &L.d2,   &L.z,    &L.Tval,  &L.valT,  &L.PvalT, &L.RvalT, &L.ptval, &L.Ival};
    for (auto* b : ib) b->free_();
    for (auto* b : db) b->free_();
  }
  c.lv.clear();
  c.nlev = 0;
  c.reuse_ok = false;
  c.cinv.free_();
  c.arena.release_all(c.al);
  c.amg_ready = false;
}

// rigid-body modes per node [2][K]; K = 4 appends the linearisation point v (reading G30)
__global__ void k_level0_nullspace(int n, double L, int K, const double* __restrict__ v, double* __restrict__ B) {
  const int node = blockIdx.x * blockDim.x + threadIdx.x;
  const int s = n + 1;
  if (node >= s * s) return;
  const double dx = L / n;
  const double x = (node % s) * dx, y = (node / s) * dx;
  double* b = B + (long long)node * 2 * K;
  b[0] = 1.0; b[1] = 0.0; b[2] = -(y - 0.5 * L) / L;
  b[K] = 0.0; b[K + 1] = 1.0; b[K + 2] = (x - 0.5 * L) / L;
  if (K == 4) {
    b[3] = v[2 * node];
    b[7] = v[2 * node + 1];
  }
}

void vgraph_destroy(Ctx& c);

static void amg_setup_numeric(Ctx& c, int K);

void amg_setup_impl(Ctx& c) {
  SI_CHECK(c.assembled, SEAICE_ESTATE, "amg_setup before assemble");
  tick(c, nullptr, 0);
  vgraph_destroy(c);
  tick(c, "graph_free", 0);
  int K = c.p.nullspace_dim;
  SI_CHECK(K == 3 || c.lin_v.get(), SEAICE_ESTATE, "nullspace_dim = 4 needs an assembled linearisation point");
  if (K == 4 && norm2(c, c.lin_v.get(), c.N) == 0.0) K = 3;  // reading G30: v_l = 0 adds no column
  SI_CUDA(cudaMemsetAsync(c.flag.get(), 0, sizeof(int) * 4, c.s));
  // reading G32: keep this time step's aggregates and patterns, recompute the values
  c.last_setup_reused = c.p.amg_reuse == 1 && c.reuse_ok && c.reuse_K == K && c.nlev > 1;
  if (c.last_setup_reused) {
    amg_setup_numeric(c, K);
    return;
  }
  // the level pool keeps every buffer (grow-only) across setups; level 0's pattern is fixed
  if (c.lv.empty()) {
    c.lv.emplace_back();
    build_level0_pattern(c, c.lv[0]);
  }
  c.nlev = 1;
  c.amg_ready = false;
  c.reuse_ok = false;
  Level& L0 = c.lv[0];
  L0.val.ensure(c.al, (size_t)L0.nnzb * 4);
  k_stencil_to_bsr<<<grid_for(c.Nn), kThreads, 0, c.s>>>(c.n, c.Nn, c.Jst.get(), L0.rp.get(), L0.val.get());
  SI_LAUNCHED(c);
  if (c.p.cheb_fused == 2) stencil_stream_copy(c);
  L0.B.ensure(c.al, (size_t)c.Nn * 2 * K);
  k_level0_nullspace<<<grid_for(c.Nn), kThreads, 0, c.s>>>(c.n, c.p.L, K, c.lin_v.get(), L0.B.get());
  SI_LAUNCHED(c);
  tick(c, "to_bsr", 0);
  long long nnz_total = 0;
  const long long nnz0 = L0.nnzb * 4;
  for (int lvl = 0;; ++lvl) {
    Level& L = c.lv[lvl];
    Scratch S(c);
    double* dnorm = S.get<double>(L.nb);
    tick(c, nullptr, lvl);
    if (L.b == 2) level_diag<2>(c, L, S, dnorm);
    else if (L.b == 3) level_diag<3>(c, L, S, dnorm);
    else level_diag<4>(c, L, S, dnorm);
    tick(c, "diag", lvl);
    if (lvl > 0 && L.b != 4) tile_copy(c, L.valT, L.val.get(), L.nnzb, L.b * L.b);
    L.lmax = (L.b == 2) ? power_lambda<2>(c, L, lvl) : (L.b == 3) ? power_lambda<3>(c, L, lvl)
                                                                  : power_lambda<4>(c, L, lvl);
    tick(c, "power", lvl);
    nnz_total += L.nnzb * L.b * L.b;
    const long long ndof = (long long)L.nb * L.b;
    // work vectors for the V-cycle (coarse levels padded to 4 per block row, pads 0)
    const long long nst = (long long)L.nb * vstride(L.b);
    for (auto* v : {&L.x, &L.rhs, &L.r, &L.d, &L.d2, &L.z}) {
      v->ensure(c.al, nst);
      if (L.b == 3) SI_CUDA(cudaMemsetAsync(v->get(), 0, sizeof(double) * nst, c.s));
    }
    const bool last_allowed = (lvl + 1 >= c.p.max_levels);
    if (ndof <= c.p.coarse_max_dof || last_allowed) break;
    const int na = (L.b == 2)   ? aggregate_level<2>(c, L, lvl, dnorm, S)
                   : (L.b == 3) ? aggregate_level<3>(c, L, lvl, dnorm, S)
                                : aggregate_level<4>(c, L, lvl, dnorm, S);
    tick(c, "aggregate", lvl);
    if (na == 0 || na > 0.9 * L.nb) break;
    if ((int)c.lv.size() == c.nlev) c.lv.emplace_back();  // may move Level objects (DBufs are handles)
    Level& Lc = c.lv[c.nlev];
    Level& Lf = c.lv[lvl];
    ++c.nlev;
    if (K == 3) {
      if (Lf.b == 2) build_transfer<2, 3>(c, Lf, Lc, lvl, na, S);
      else build_transfer<3, 3>(c, Lf, Lc, lvl, na, S);
    } else {
      if (Lf.b == 2) build_transfer<2, 4>(c, Lf, Lc, lvl, na, S);
      else build_transfer<4, 4>(c, Lf, Lc, lvl, na, S);
    }
    tick(c, nullptr, lvl);
    if (K != 4) {  // b = 4 kernels read the row-major blocks directly
      tile_copy(c, Lf.PvalT, Lf.Pval.get(), Lf.Pnnzb, Lf.b * K);
      tile_copy(c, Lf.RvalT, Lf.Rval.get(), Lf.Rnnzb, K * Lf.b);
    }
    tick(c, "tile_PR", lvl);
  }
  Level& Lc = c.lv[c.nlev - 1];
  const long long nd = (long long)Lc.nb * Lc.b;
  SI_CHECK(nd <= 8192, SEAICE_EINVAL, "AMG coarsest level too large for the dense solve (coarsening stalled)");
  tick(c, nullptr, c.nlev - 1);
  coarse_factor(c, Lc);
  tick(c, "coarse", c.nlev - 1);
  const int flag = read_scalar(c, c.flag.get());
  SI_CHECK(!(flag & 4), SEAICE_ENONFINITE, "AMG: singular diagonal block");
  SI_CHECK(!(flag & 8), SEAICE_ENONFINITE, "AMG: coarse matrix not positive definite");
  c.op_complexity = (double)nnz_total / (double)nnz0;
  c.amg_ready = true;
  c.reuse_ok = true;
  c.reuse_K = K;
  tick(c, "finish", c.nlev - 1);
}

// Reading G32: the hierarchy of the step's first setup with every value recomputed from the
// current J and v_l (same level count, aggregates, patterns and kernels).
static void amg_setup_numeric(Ctx& c, int K) {
  c.amg_ready = false;
  Level& L0 = c.lv[0];
  k_stencil_to_bsr<<<grid_for(c.Nn), kThreads, 0, c.s>>>(c.n, c.Nn, c.Jst.get(), L0.rp.get(), L0.val.get());
  SI_LAUNCHED(c);
  if (c.p.cheb_fused == 2) stencil_stream_copy(c);
  k_level0_nullspace<<<grid_for(c.Nn), kThreads, 0, c.s>>>(c.n, c.p.L, K, c.lin_v.get(), L0.B.get());
  SI_LAUNCHED(c);
  tick(c, "to_bsr", 0);
  for (int lvl = 0; lvl < c.nlev; ++lvl) {
    Level& L = c.lv[lvl];
    {
      Scratch S(c);
      double* dnorm = S.get<double>(L.nb);
      if (L.b == 2) level_diag<2>(c, L, S, dnorm);
      else if (L.b == 3) level_diag<3>(c, L, S, dnorm);
      else level_diag<4>(c, L, S, dnorm);
    }
    tick(c, "diag", lvl);
    if (lvl > 0 && L.b != 4) tile_copy(c, L.valT, L.val.get(), L.nnzb, L.b * L.b);
    L.lmax = (L.b == 2) ? power_lambda<2>(c, L, lvl) : (L.b == 3) ? power_lambda<3>(c, L, lvl)
                                                                  : power_lambda<4>(c, L, lvl);
    tick(c, "power", lvl);
    if (L.b == 3)  // V-cycle work vectors: pads stay 0 (as after a full setup)
      for (auto* v : {&L.x, &L.rhs, &L.r, &L.d, &L.d2, &L.z})
        SI_CUDA(cudaMemsetAsync(v->get(), 0, sizeof(double) * (size_t)L.nb * vstride(3), c.s));
    if (lvl == c.nlev - 1) break;
    Level& Lc = c.lv[lvl + 1];
    if (K == 3) {
      if (L.b == 2) build_transfer_numeric<2, 3>(c, L, Lc, lvl);
      else build_transfer_numeric<3, 3>(c, L, Lc, lvl);
    } else {
      if (L.b == 2) build_transfer_numeric<2, 4>(c, L, Lc, lvl);
      else build_transfer_numeric<4, 4>(c, L, Lc, lvl);
    }
    if (K != 4) {
      tile_copy(c, L.PvalT, L.Pval.get(), L.Pnnzb, L.b * K);
      tile_copy(c, L.RvalT, L.Rval.get(), L.Rnnzb, K * L.b);
    }
    tick(c, "tile_PR", lvl);
  }
  coarse_factor(c, c.lv[c.nlev - 1]);
  tick(c, "coarse", c.nlev - 1);
  const int flag = read_scalar(c, c.flag.get());
  SI_CHECK(!(flag & 4), SEAICE_ENONFINITE, "AMG: singular diagonal block");
  SI_CHECK(!(flag & 8), SEAICE_ENONFINITE, "AMG: coarse matrix not positive definite");
  c.amg_ready = true;
  tick(c, "finish", c.nlev - 1);
}

// Lagged hierarchy (reading G31): the coarse levels of the last setup stay; the finest level's
// block-diagonal inverse and lambda_max are recomputed from the current stencil J (the finest
// smoother and residual read J itself), and the V-cycle graph is re-captured (its Chebyshev
// coefficients depend on lambda_max).
// reading G31 refinement: a hierarchy built without the v_l column (v_l = 0, K = 3) is not kept
// once the linearisation point is non-zero (the fourth near-nullspace column then exists)
bool amg_lag_allowed(Ctx& c) {
  if (c.p.nullspace_dim == 4 && c.reuse_K == 3) return norm2(c, c.lin_v.get(), c.N) == 0.0;
  return true;
}

void amg_refresh_finest(Ctx& c) {
  SI_CHECK(c.assembled && c.nlev > 1, SEAICE_ESTATE, "amg_refresh_finest without a multilevel hierarchy");
  vgraph_destroy(c);
  Level& L0 = c.lv[0];
  k_stencil_to_bsr<<<grid_for(c.Nn), kThreads, 0, c.s>>>(c.n, c.Nn, c.Jst.get(), L0.rp.get(), L0.val.get());
  SI_LAUNCHED(c);
  if (c.p.cheb_fused == 2) stencil_stream_copy(c);
  SI_CUDA(cudaMemsetAsync(c.flag.get(), 0, sizeof(int) * 4, c.s));
  {
    Scratch S(c);
    double* dnorm = S.get<double>(L0.nb);
    level_diag<2>(c, L0, S, dnorm);
  }
  L0.lmax = power_lambda<2>(c, L0, 0);
  const int flag = read_scalar(c, c.flag.get());
  SI_CHECK(!(flag & 4), SEAICE_ENONFINITE, "AMG: singular diagonal block");
  c.amg_ready = true;
}

// ------------------------------------------------------------------ V-cycle tail (persistent)
// The bottom of the V-cycle (levels whose operators fit the L2 together, e.g. 4 k / 262 / 21 block
// rows at config 4) costs ~27 launches of 4-15 us each, latency-bound (VERDICT round-1 item 4).
// k_vcycle_tail runs those levels in ONE cooperative launch: every phase (residual, Chebyshev
// step, restriction, coarse GEMV, prolongation) is a row loop over the level, phases separated
// by grid.sync().  Same operations in the same order as vcycle_level / smooth on these levels
// (b = 4 blocks).  A level of more than 2 rows per CTA is swept warp per row (8 blocks in
// flight per row, the sums of k_acheb4<8> / k_aresid4<8> / k_aspmv<4, 4, 8>), a smaller one CTA
// per row (64 blocks in flight, the sums of the _cta kernels).  Vectors written in one phase and
// read in the next are read with L2-coherent loads (ld.global.cg / volatile: the .nc path of the
// stand-alone kernels assumes data that is read-only for the whole launch); matrices stay on
// the read-only path.
constexpr int kTailMaxLevels = 8;
struct TailLevel {
  int nb, nbc;
  const int *rp, *ci, *Rrp, *Rci, *Prp, *Pci;
  const double *val, *dinv, *Rval, *Pval;
  const double* rhs;
  double *x, *r, *d, *d2;
  double ith, c1[2], c2[2];  // 1 / theta and the Chebyshev(3) recurrence coefficients
};
struct TailArgs {
  int nl;  // smoothed levels in the tail; below them the coarsest level (dense inverse)
  TailLevel lv[kTailMaxLevels];
  int cn;
  const double* cinv;
  double *cx, *crhs;
};

__device__ __forceinline__ void ld4_coh(const double* p, double (&v)[4]) {
  asm volatile("ld.global.cg.v4.f64 {%0,%1,%2,%3}, [%4];"
               : "=d"(v[0]), "=d"(v[1]), "=d"(v[2]), "=d"(v[3])
               : "l"(p)
               : "memory");
}
__device__ __forceinline__ double ld_coh(const double* p) {
  double v;
  asm volatile("ld.global.cg.f64 %0, [%1];" : "=d"(v) : "l"(p) : "memory");
  return v;
}
// Row sweep geometry: CTA = true: one row per CTA at a time (thread t: component t % 4 of slot
// t / 4 of 64), the row's epilogue runs on warp 0; CTA = false: one row per warp (8 slots).
template <bool CTA>
struct TailSweep {
  static __device__ __forceinline__ int first() {
    return CTA ? (int)blockIdx.x : (int)((blockIdx.x * blockDim.x + threadIdx.x) >> 5);
  }
  static __device__ __forceinline__ int step() { return CTA ? (int)gridDim.x : (int)((gridDim.x * blockDim.x) >> 5); }
};
// component (lane % 4) of (M x)_row for a 4 x 4-block row: in lanes 0..3 of the row's warp (CTA:
// threads 0..3).  Every thread of the warp (CTA) calls it.
template <bool CTA>
__device__ __forceinline__ double tail_row(int row, const int* __restrict__ rp, const int* __restrict__ ci,
                                           const double* __restrict__ val, const double* x, double (*sh)[4]) {
  constexpr int S = CTA ? 64 : 8;
  const int t = CTA ? (int)threadIdx.x : (int)(threadIdx.x & 31);
  const int a = t & 3, slot = t >> 2;
  double acc = 0.0;
  const int e1 = __ldg(rp + row + 1);
  int e = __ldg(rp + row) + slot;
  for (; e + S < e1; e += 2 * S) {
    const int c0 = __ldg(ci + e), c1 = __ldg(ci + e + S);
    double v0[4], v1[4], x0[4], x1[4];
    load_row<4>(val + ((long long)e * 4 + a) * 4, v0);
    load_row<4>(val + ((long long)(e + S) * 4 + a) * 4, v1);
    ld4_coh(x + (long long)c0 * 4, x0);
    ld4_coh(x + (long long)c1 * 4, x1);
#pragma unroll
    for (int b = 0; b < 4; ++b) acc += v0[b] * x0[b];
#pragma unroll
    for (int b = 0; b < 4; ++b) acc += v1[b] * x1[b];
  }
  for (; e < e1; e += S) {
    double v0[4], x0[4];
    load_row<4>(val + ((long long)e * 4 + a) * 4, v0);
    ld4_coh(x + (long long)__ldg(ci + e) * 4, x0);
#pragma unroll
    for (int b = 0; b < 4; ++b) acc += v0[b] * x0[b];
  }
#pragma unroll
  for (int off = 4; off < 32; off <<= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
  if (!CTA) return acc;
  if ((t & 31) < 4) sh[t >> 5][a] = acc;
  __syncthreads();
  double tot = 0.0;
  if (t < 4) {
#pragma unroll
    for (int w = 0; w < 8; ++w) tot += sh[w][t];
  }
  __syncthreads();
  return tot;
}
// r = b - A x (x NULL: r = b); d = c2 Dinv r
template <bool CTA>
__device__ __forceinline__ void tail_resid(const TailLevel& L, const double* x, double (*sh)[4]) {
  const int lane = threadIdx.x & 31;
  for (int row = TailSweep<CTA>::first(); row < L.nb; row += TailSweep<CTA>::step()) {
    const double acc = x ? tail_row<CTA>(row, L.rp, L.ci, L.val, x, sh) : 0.0;
    if (CTA && threadIdx.x >= 32) continue;
    const long long i = (long long)row * 4 + (lane & 3);
    double D[4];
    load_row<4>(L.dinv + (long long)row * 16 + (lane & 3) * 4, D);
    const double rv = ld_coh(L.rhs + i) - acc;
    if (lane < 4) L.r[i] = rv;
    double z = 0.0;
#pragma unroll
    for (int k = 0; k < 4; ++k) z += D[k] * __shfl_sync(0xffffffffu, rv, k);
    if (lane < 4) L.d[i] = L.ith * z;
  }
}
// Chebyshev step (semantics of k_acheb4): t = A d; x (+)= d; r -= t; dout = c1 d + c2 Dinv r
template <bool CTA>
__device__ __forceinline__ void tail_cheb(const TailLevel& L, const double* d, double* dout, double c1, double c2,
                                          bool first, bool want_r, bool want_d, double (*sh)[4]) {
  const int lane = threadIdx.x & 31;
  for (int row = TailSweep<CTA>::first(); row < L.nb; row += TailSweep<CTA>::step()) {
    const double acc = want_r ? tail_row<CTA>(row, L.rp, L.ci, L.val, d, sh) : 0.0;
    if (CTA && threadIdx.x >= 32) continue;
    const long long i = (long long)row * 4 + (lane & 3);
    const double dv = ld_coh(d + i);
    const double xv = first ? 0.0 : ld_coh(L.x + i);
    if (lane < 4) L.x[i] = xv + dv;
    if (!want_r) continue;
    const double rv = ld_coh(L.r + i) - acc;
    if (lane < 4) L.r[i] = rv;
    if (!want_d) continue;
    double D[4];
    load_row<4>(L.dinv + (long long)row * 16 + (lane & 3) * 4, D);
    double z = 0.0;
#pragma unroll
    for (int k = 0; k < 4; ++k) z += D[k] * __shfl_sync(0xffffffffu, rv, k);
    if (lane < 4) dout[i] = c1 * dv + c2 * z;
  }
}
// y = yin + M x for a 4 x 4-block transfer operator (yin NULL: y = M x; yin == y: in place)
template <bool CTA>
__device__ __forceinline__ void tail_spmv(int nb, const int* rp, const int* ci, const double* val, const double* x,
                                          const double* yin, double* y, double (*sh)[4]) {
  const int lane = threadIdx.x & 31;
  for (int row = TailSweep<CTA>::first(); row < nb; row += TailSweep<CTA>::step()) {
    const double acc = tail_row<CTA>(row, rp, ci, val, x, sh);
    if (CTA && threadIdx.x >= 32) continue;
    const long long i = (long long)row * 4 + (lane & 3);
    const double y0 = yin ? ld_coh(yin + i) : 0.0;
    if (lane < 4) y[i] = y0 + acc;
  }
}
#define SI_TAIL(NB, CALL)                      \
  if ((NB) <= 2 * (int)gridDim.x) {            \
    constexpr bool TC = true;                  \
    CALL;                                      \
  } else {                                     \
    constexpr bool TC = false;                 \
    CALL;                                      \
  }

__global__ void __launch_bounds__(256) k_vcycle_tail(const __grid_constant__ TailArgs A) {
  cooperative_groups::grid_group grid = cooperative_groups::this_grid();
  __shared__ double sh[8][4];
  // down-sweep: pre-smoothing from x = 0 (leaves r = b - A x), restriction
  for (int l = 0; l < A.nl; ++l) {
    const TailLevel& L = A.lv[l];
    SI_TAIL(L.nb, tail_resid<TC>(L, nullptr, sh));
    grid.sync();
    SI_TAIL(L.nb, tail_cheb<TC>(L, L.d, L.d2, L.c1[0], L.c2[0], true, true, true, sh));
    grid.sync();
    SI_TAIL(L.nb, tail_cheb<TC>(L, L.d2, L.d, L.c1[1], L.c2[1], false, true, true, sh));
    grid.sync();
    SI_TAIL(L.nb, tail_cheb<TC>(L, L.d, L.d2, 0.0, 0.0, false, true, false, sh));
    grid.sync();
    double* rc = l + 1 < A.nl ? const_cast<double*>(A.lv[l + 1].rhs) : A.crhs;
    SI_TAIL(L.nbc, tail_spmv<TC>(L.nbc, L.Rrp, L.Rci, L.Rval, L.r, nullptr, rc, sh));
    grid.sync();
  }
  // coarsest level: x = A^-1 b (dense inverse, warp per row; b = 4: unpadded vectors)
  {
    const int lane = threadIdx.x & 31;
    const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
    for (int w = gw; w < A.cn; w += nw) {
      double sacc = 0.0;
      for (int k = lane; k < A.cn; k += 32) sacc += __ldg(A.cinv + (long long)w * A.cn + k) * ld_coh(A.crhs + k);
      sacc = warp_sum(sacc);
      if (lane == 0) A.cx[w] = sacc;
    }
  }
  grid.sync();
  // up-sweep: prolongation, post-smoothing
  for (int l = A.nl - 1; l >= 0; --l) {
    const TailLevel& L = A.lv[l];
    const double* xc = l + 1 < A.nl ? A.lv[l + 1].x : A.cx;
    SI_TAIL(L.nb, tail_spmv<TC>(L.nb, L.Prp, L.Pci, L.Pval, xc, L.x, L.x, sh));
    grid.sync();
    SI_TAIL(L.nb, tail_resid<TC>(L, L.x, sh));
    grid.sync();
    SI_TAIL(L.nb, tail_cheb<TC>(L, L.d, L.d2, L.c1[0], L.c2[0], false, true, true, sh));
    grid.sync();
    SI_TAIL(L.nb, tail_cheb<TC>(L, L.d2, L.d, L.c1[1], L.c2[1], false, true, true, sh));
    grid.sync();
    SI_TAIL(L.nb, tail_cheb<TC>(L, L.d, L.d2, 0.0, 0.0, false, false, false, sh));
    if (l > 0) grid.sync();
  }
}

// ------------------------------------------------------------------ host: V-cycle
struct ChebCoef {
  double th, de, sg;
};
static ChebCoef cheb_coef(const Ctx& c, const Level& L) {
  const double bmax = c.p.cheb_upper * L.lmax, amin = c.p.cheb_lower * bmax;
  ChebCoef k;
  k.th = 0.5 * (bmax + amin);
  k.de = 0.5 * (bmax - amin);
  k.sg = k.th / k.de;
  return k;
}

// One Chebyshev smoothing on level l for A x = b.  pre: x = 0 start, leaves r = b - A x.
static int level_degree(const Ctx& c, int l) {
  return (l == 0 && c.p.cheb_degree0 > 0) ? c.p.cheb_degree0 : c.p.cheb_degree;
}
static bool fused_smoother(const Ctx& c, int l) {
  const int m = level_degree(c, l);
  return l == 0 && c.p.cheb_fused && m >= 3 && m <= kFMaxM;
}
static bool streamed_smoother(const Ctx& c, int l) {
  return l == 0 && c.p.cheb_fused == 2 && level_degree(c, l) == 3;
}

// One Chebyshev smoothing on level l for A x = b.  pre: x = 0 start, leaves r = b - A x.
static void smooth(Ctx& c, int l, const double* b, double* x, bool pre) {
  Level& L = c.lv[l];
  const int m = level_degree(c, l);
  const ChebCoef k = cheb_coef(c, L);
  double rho = 1.0 / k.sg;
  double* r = L.r.get();
  double* d = L.d.get();
  double* d2 = L.d2.get();
  const bool st = (l == 0);
  const bool fused = fused_smoother(c, l);
  if (streamed_smoother(c, l)) {
    // y-streamed Chebyshev(3): one launch, the post-smoothing residual included.  Post-smoothing
    // reads x_0 from L.d (written by the prolongation, see vcycle_level) and writes x.
    ChebFCoef kc;
    kc.ith = 1.0 / k.th;
    for (int it = 0; it < 2; ++it) {
      const double rho_new = 1.0 / (2.0 * k.sg - rho);
      kc.c1[it] = rho_new * rho;
      kc.c2[it] = 2.0 * rho_new / k.de;
      rho = rho_new;
    }
    prof_begin(c);
    launch_cheb3_stream(c, L.dinv.get(), b, pre ? nullptr : d, x, pre ? r : nullptr, kc, pre);
    SI_LAUNCHED(c);
    // stencil + Dinv once, b read, (x_0 read,) x written (, r_3 written)
    prof_end(c, PC_CHEB0F, (double)c.Nn * (kJBytesNode + 32.0 + 16.0 + 32.0));
    return;
  }
  // r = b - A x ; d = Dinv r / th  (fused pre-smoothing does this inside its launch)
  if (!(fused && pre)) {
    prof_begin(c);
    if (st) {
      k_resid_dinv_stencil<<<grid_for(c.Nn), 256, 0, c.s>>>(c.n, c.Nn, c.Jst.get(), L.dinv.get(),
                                                            (const double2*)b, pre ? nullptr : (const double2*)x,
                                                            (double2*)r, (double2*)d, 1.0 / k.th);
    } else {
      const int G = pick_group(L.nnzb, L.nb);
      if (L.b == 3)
        SI_GDISPATCH(G, (k_gresid<3, GG><<<ggrid(L.nb, GG), 256, 0, c.s>>>(
                            L.nb, L.rp.get(), L.ci.get(), L.valT.get(), L.dinv.get(), b, pre ? nullptr : x, r, d,
                            1.0 / k.th)))
      else if (use_cta_rows(L.nnzb, L.nb)) {
        k_aresid4_cta<<<L.nb, 256, 0, c.s>>>(L.nb, L.rp.get(), L.ci.get(), L.val.get(), L.dinv.get(), b,
                                             pre ? nullptr : x, r, d, 1.0 / k.th);
      } else {
        const int Sl = pick_slots(L.nnzb, L.nb, 4);
        SI_SDISPATCH(Sl, (k_aresid4<SS><<<agrid(L.nb, 4 * SS), ablock(), 0, c.s>>>(
                             L.nb, L.rp.get(), L.ci.get(), L.val.get(), L.dinv.get(), b, pre ? nullptr : x, r, d,
                             1.0 / k.th)))
      }
    }
    SI_LAUNCHED(c);
    const double B = L.b;
    double by = L.nb * (8.0 * B * 3 + 8.0 * B * B);  // b read, r write, d write, dinv
    if (!pre) by += (st ? kJBytesNode * c.Nn : L.nnzb * (8.0 * B * B + 4.0) + 4.0 * (L.nb + 1)) + 8.0 * B * L.nb;
    prof_end(c, st ? PC_RESID0 : (l == 1 ? PC_RESID1 : PC_RESIDC), by);
  }
  if (fused) {
    ChebFCoef kc;
    kc.ith = 1.0 / k.th;
    for (int it = 0; it < m - 1; ++it) {
      const double rho_new = 1.0 / (2.0 * k.sg - rho);
      kc.c1[it] = rho_new * rho;
      kc.c2[it] = 2.0 * rho_new / k.de;
      rho = rho_new;
    }
    // pre: rin = b, r_m written out of place into L.r; post: rin = r_0, d_0 from d
    const double* rin = pre ? b : r;
    prof_begin(c);
    switch (m) {
      case 3: launch_chebM<3>(c, L.dinv.get(), rin, d, r, x, kc, pre); break;
      case 4: launch_chebM<4>(c, L.dinv.get(), rin, d, r, x, kc, pre); break;
      case 5: launch_chebM<5>(c, L.dinv.get(), rin, d, r, x, kc, pre); break;
      default: launch_chebM<6>(c, L.dinv.get(), rin, d, r, x, kc, pre); break;
    }
    SI_LAUNCHED(c);
    // algorithmic bytes: stencil + Dinv once, r_0 / b read (+ d_0, x_0 for post), x (+ r_m) written
    prof_end(c, PC_CHEB0F, (double)c.Nn * (kJBytesNode + 32.0 + 16.0 + (pre ? 32.0 : 48.0)));
    return;
  }
  for (int it = 0; it < m; ++it) {
    const bool last = (it == m - 1);
    const int want_r = (!last || pre) ? 1 : 0;
    const int want_d = last ? 0 : 1;
    const int first = (pre && it == 0) ? 1 : 0;
    const double rho_new = 1.0 / (2.0 * k.sg - rho);
    const double c1 = rho_new * rho, c2 = 2.0 * rho_new / k.de;
    prof_begin(c);
    if (st) {
      k_cheb_stencil<<<grid_for(c.Nn), 256, 0, c.s>>>(c.n, c.Nn, c.Jst.get(), L.dinv.get(), (const double2*)d,
                                                     (double2*)r, (double2*)x, (double2*)d2, c1, c2, first, want_r,
                                                     want_d);
    } else {
      const int G = pick_group(L.nnzb, L.nb);
      if (L.b == 3)
        SI_GDISPATCH(G, (k_gcheb<3, GG><<<ggrid(L.nb, GG), 256, 0, c.s>>>(L.nb, L.rp.get(), L.ci.get(), L.valT.get(),
                                                                         L.dinv.get(), d, r, x, d2, c1, c2, first,
                                                                         want_r, want_d)))
      else if (use_cta_rows(L.nnzb, L.nb)) {
        k_acheb4_cta<<<L.nb, 256, 0, c.s>>>(L.nb, L.rp.get(), L.ci.get(), L.val.get(), L.dinv.get(), d, r, x, d2,
                                            c1, c2, first, want_r, want_d);
      } else {
        const int Sl = pick_slots(L.nnzb, L.nb, 4);
        // late own-entry loads: measured 2357 -> 1555 us of coarse smoothing per V-cycle (config 4)
        SI_SDISPATCH(Sl, (k_acheb4<SS, true><<<agrid(L.nb, 4 * SS), ablock(), 0, c.s>>>(
                             L.nb, L.rp.get(), L.ci.get(), L.val.get(), L.dinv.get(), d, r, x, d2, c1, c2, first,
                             want_r, want_d)))
      }
    }
    SI_LAUNCHED(c);
    {
      const double B = L.b;
      double by = L.nb * 8.0 * B * (first ? 2.0 : 3.0);  // d read, x (read +) write
      if (want_r) by += (st ? kJBytesNode * c.Nn : L.nnzb * (8.0 * B * B + 4.0) + 4.0 * (L.nb + 1)) + 16.0 * B * L.nb;
      if (want_d) by += L.nb * (8.0 * B * B + 8.0 * B);
      prof_end(c, st ? PC_CHEB0 : (l == 1 ? PC_CHEB1 : PC_CHEBC), by);
    }
    rho = rho_new;
    std::swap(d, d2);
  }
}

// First level of the persistent tail (k_vcycle_tail), or -1: the deepest run of b = 4 levels
// l >= 1 whose operators and transfers together stay under ~48 MB (L2-resident on the B200).
static int tail_start(const Ctx& c) {
  if (!c.p.vcycle_tail || c.nlev < 3 || c.lv[c.nlev - 1].b != 4) return -1;
  static const double cap = getenv("SEAICE_TAIL_MB") ? atof(getenv("SEAICE_TAIL_MB")) * 1e6 : 48e6;  // tuning aid
  double bytes = 0.0;
  int l0 = -1;
  for (int l = c.nlev - 2; l >= 1 && c.nlev - 1 - l <= kTailMaxLevels; --l) {
    const Level& L = c.lv[l];
    if (L.b != 4) break;
    bytes += (double)(L.nnzb + L.Pnnzb + L.Rnnzb) * 132.0;
    if (bytes > cap) break;
    l0 = l;
  }
  return l0;
}

static int tail_grid(const Ctx& c) {
  static int per_sm = -1;
  if (per_sm < 0) {
    int occ = 0;
    SI_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_vcycle_tail, 256, 0));
    const int want = getenv("SEAICE_TAIL_CTAS") ? atoi(getenv("SEAICE_TAIL_CTAS")) : 4;  // tuning aid
    per_sm = occ < 1 ? 0 : (want < occ ? want : occ);
    if (per_sm < 1) per_sm = occ;
  }
  SI_CHECK(per_sm >= 1, SEAICE_ECUDA, "k_vcycle_tail cannot be resident");
  return per_sm * c.sms;
}

// Levels l0 .. nlev-1 of the V-cycle in one cooperative launch (b = rhs, x = solution of level l0)
static void vcycle_tail(Ctx& c, int l0, const double* b, double* x) {
  TailArgs A{};
  A.nl = c.nlev - 1 - l0;
  double by = 0.0;
  for (int k = 0; k < A.nl; ++k) {
    Level& L = c.lv[l0 + k];
    TailLevel& T = A.lv[k];
    T.nb = L.nb;
    T.nbc = L.nbc;
    T.rp = L.rp.get(), T.ci = L.ci.get(), T.val = L.val.get(), T.dinv = L.dinv.get();
    T.Rrp = L.Rrp.get(), T.Rci = L.Rci.get(), T.Rval = L.Rval.get();
    T.Prp = L.Prp.get(), T.Pci = L.Pci.get(), T.Pval = L.Pval.get();
    T.rhs = k == 0 ? b : L.rhs.get();
    T.x = k == 0 ? x : L.x.get();
    T.r = L.r.get(), T.d = L.d.get(), T.d2 = L.d2.get();
    const ChebCoef kc = cheb_coef(c, L);
    double rho = 1.0 / kc.sg;
    T.ith = 1.0 / kc.th;
    for (int it = 0; it < 2; ++it) {
      const double rho_new = 1.0 / (2.0 * kc.sg - rho);
      T.c1[it] = rho_new * rho;
      T.c2[it] = 2.0 * rho_new / kc.de;
      rho = rho_new;
    }
    // six operator passes, the two transfers, ~20 vector passes
    by += 6.0 * (L.nnzb * 132.0 + 4.0 * (L.nb + 1)) + (L.Pnnzb + L.Rnnzb) * 132.0 + 20.0 * 32.0 * L.nb;
  }
  Level& Lz = c.lv[c.nlev - 1];
  A.cn = c.cn;
  A.cinv = c.cinv.get();
  A.cx = Lz.x.get();
  A.crhs = Lz.rhs.get();
  by += 8.0 * c.cn * c.cn + 16.0 * c.cn;
  void* args[] = {&A};
  prof_begin(c);
  SI_CUDA(cudaLaunchCooperativeKernel((const void*)k_vcycle_tail, dim3(tail_grid(c)), dim3(256), args, 0, c.s));
  SI_LAUNCHED(c);
  prof_end(c, PC_TAIL, by);
}

static void vcycle_level(Ctx& c, int l, const double* b, double* x) {
  Level& L = c.lv[l];
  if (l >= 1 && l + 1 < c.nlev && level_degree(c, l) == 3 && l == tail_start(c)) {
    vcycle_tail(c, l, b, x);
    return;
  }
  if (l + 1 == c.nlev) {
    prof_begin(c);
    k_dense_gemv<<<grid_for((long long)c.cn * 32, 256), 256, 0, c.s>>>(c.cn, L.b, vstride(L.b), c.cinv.get(), b, x);
    SI_LAUNCHED(c);
    prof_end(c, PC_COARSE, 8.0 * c.cn * c.cn + 16.0 * c.cn);
    return;
  }
  smooth(c, l, b, x, true);
  Level& Lc = c.lv[l + 1];
  // r_c = R r
  prof_begin(c);
  gspmv(c, L.nbc, Lc.b, L.b, L.Rnnzb, L.Rrp.get(), L.Rci.get(), Lc.b == 4 ? L.Rval.get() : L.RvalT.get(), L.r.get(),
        nullptr, Lc.rhs.get());
  prof_end(c, l == 0 ? PC_TRANSFER0 : PC_TRANSFER,
           L.Rnnzb * (8.0 * Lc.b * L.b + 4.0) + 4.0 * (L.nbc + 1) + 8.0 * L.b * L.nb + 8.0 * Lc.b * L.nbc);
  vcycle_level(c, l + 1, Lc.rhs.get(), Lc.x.get());
  // x += P e_c
  prof_begin(c);
  // (the streamed finest post-smoother updates x out of place: x_0 = x + P e_c goes to L.d)
  gspmv(c, L.nb, L.b, Lc.b, L.Pnnzb, L.Prp.get(), L.Pci.get(), Lc.b == 4 ? L.Pval.get() : L.PvalT.get(), Lc.x.get(),
        x, streamed_smoother(c, l) ? L.d.get() : x);
  prof_end(c, l == 0 ? PC_TRANSFER0 : PC_TRANSFER,
           L.Pnnzb * (8.0 * Lc.b * L.b + 4.0) + 4.0 * (L.nb + 1) + 16.0 * L.b * L.nb + 8.0 * Lc.b * L.nbc);
  smooth(c, l, b, x, false);
}

static long long g_vgraph_kernels = 0;

void vgraph_destroy(Ctx& c) {
  if (c.vgraph) {
    cudaStreamSynchronize(c.s);
    cudaGraphExecDestroy(c.vgraph);
    c.vgraph = nullptr;
  }
}

// One V-cycle z = M^-1 r.  The whole cycle (~10 launches per level) is captured once per
// hierarchy into a CUDA graph reading vc_in and writing vc_out, so the small coarse-level
// kernels are not paced by host launch latency.
void amg_vcycle(Ctx& c, const double* r, double* z) {
  SI_CHECK(c.amg_ready, SEAICE_ESTATE, "V-cycle without hierarchy");
  if (!c.use_graphs || c.prof.on) {
    vcycle_level(c, 0, r, z);
    return;
  }
  if (!c.vgraph) {
    c.vc_in.ensure(c.al, c.N);
    c.vc_out.ensure(c.al, c.N);
    cudaGraph_t g = nullptr;
    const long long l0 = c.launches;
    // capture on a private stream (the caller's may be the legacy default stream, which
    // cannot be captured); the graph is then launched on the caller's stream
    if (!c.cap_stream) SI_CUDA(cudaStreamCreateWithFlags(&c.cap_stream, cudaStreamNonBlocking));
    SI_CUDA(cudaStreamSynchronize(c.s));
    cudaStream_t user = c.s;
    c.s = c.cap_stream;
    SI_CUDA(cudaStreamBeginCapture(c.s, cudaStreamCaptureModeThreadLocal));
    try {
      vcycle_level(c, 0, c.vc_in.get(), c.vc_out.get());
    } catch (...) {
      cudaStreamEndCapture(c.s, &g);
      c.s = user;
      if (g) cudaGraphDestroy(g);
      throw;
    }
    cudaError_t ec = cudaStreamEndCapture(c.s, &g);
    c.s = user;
    SI_CUDA(ec);
    SI_CUDA(cudaGraphInstantiate(&c.vgraph, g, 0));
    cudaGraphDestroy(g);
    g_vgraph_kernels = c.launches - l0;
    c.launches = l0;
  }
  copy(c, c.vc_in.get(), r, c.N);
  SI_CUDA(cudaGraphLaunch(c.vgraph, c.s));
  c.launches += g_vgraph_kernels;
  copy(c, z, c.vc_out.get(), c.N);
}

}  // namespace seaice
