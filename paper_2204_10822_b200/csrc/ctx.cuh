// ctx.cuh — the library context and the host-side entry points of every kernel family.
#pragma once
#include <cmath>
#include <string>
#include <vector>

#include "common.cuh"
#include "fem.cuh"

namespace seaice {

// Which numeric SpGEMM kernel produced a product (recorded by the full setup, replayed by the
// numeric-only setup of reading G32; every path accumulates in the same order, so the choice
// does not change the values).
enum SgKind { SG_NONE = -1, SG_NARROW, SG_HASH1K, SG_HASH4K, SG_CTA, SG_THREAD, SG_GROUP8, SG_WARP };
struct SgPlan {
  int kind = SG_NONE;
  size_t smem = 0;  // SG_CTA: dynamic shared memory of the launch
};

// One level of the AMG hierarchy.  Matrices are
// block-CSR: A_l has b x b blocks (b = 2 on the finest level, 3 below), P_l has
// b x 3 blocks, R_l = P_l^T has 3 x b blocks.
struct Level {
  int nb = 0, b = 0;          // block rows, block size
  long long nnzb = 0;
  DBuf<int> rp, ci;
  DBuf<double> val;
  DBuf<double> dinv;          // inverse diagonal blocks [nb][b*b]
  double lmax = 0.0;          // power-iteration estimate of lambda_max(D^-1 A)
  // transfer to the next level
  int nbc = 0;                // coarse block rows
  long long Pnnzb = 0, Rnnzb = 0;
  DBuf<int> Prp, Pci, Rrp, Rci;
  DBuf<double> Pval, Rval;
  DBuf<int> agg;              // aggregate id per block row (-1: isolated, zero P row)
  DBuf<double> B;             // near-nullspace rows [nb*b][K], K = nullspace_dim
  // V-cycle work vectors (length nb*b)
  DBuf<double> x, rhs, r, d, d2, z;
  DBuf<double> Tval;          // A P_tent values (pattern of P), setup scratch kept for reuse
  // V-cycle copies of val / Pval / Rval in the chunk-of-32 SoA layout read by the group-per-row
  // kernels: element j of block e at ((e >> 5) * BB + j) * 32 + (e & 31)  (coalesced loads)
  DBuf<double> valT, PvalT, RvalT;
  // kept for the numeric-only setup (reading G32): aggregate members sorted by aggregate and
  // their segment starts, the P_tent pattern and values, the transpose permutation of P, the
  // Galerkin intermediate (R A on the finest level, A P below) and the numeric kernel of each
  // product (0: A P_tent, 1: the intermediate, 2: A_c)
  DBuf<int> mem, mstart, ptrp, ptci, tperm, trow, Irp, Ici;
  DBuf<double> ptval, Ival;
  int ptn = 0, K = 0;
  long long Innzb = 0;
  SgPlan plan[3];
};

// Grow-only chunked bump allocator for setup scratch (LIFO marks): avoids an allocator
// round trip (a Python callback when torch provides the memory) per temporary buffer.
struct Arena {
  struct Chunk {
    char* p;
    size_t size, used;
  };
  std::vector<Chunk> chunks;
  size_t cur = 0;  // index of the chunk being filled
  struct Mark {
    size_t chunk, used;
  };
  Mark mark() const { return chunks.empty() ? Mark{0, 0} : Mark{cur, chunks[cur].used}; }
  void reset(Mark m) {
    if (chunks.empty()) return;
    for (size_t i = m.chunk + 1; i < chunks.size(); ++i) chunks[i].used = 0;
    cur = m.chunk;
    chunks[cur].used = m.used;
  }
  void* alloc(Allocator& al, size_t bytes) {
    bytes = (bytes + 255) & ~size_t(255);
    if (bytes == 0) bytes = 256;
    while (true) {
      if (!chunks.empty() && chunks[cur].used + bytes <= chunks[cur].size) {
        void* p = chunks[cur].p + chunks[cur].used;
        chunks[cur].used += bytes;
        return p;
      }
      if (!chunks.empty() && cur + 1 < chunks.size()) {
        ++cur;
        chunks[cur].used = 0;
        continue;
      }
      size_t sz = std::max(bytes, chunks.empty() ? (size_t)64 << 20 : chunks.back().size * 2);
      chunks.push_back({(char*)al.alloc(sz), sz, 0});
      cur = chunks.size() - 1;
    }
  }
  void release_all(Allocator& al) {
    for (auto& ch : chunks) al.release(ch.p, ch.size);
    chunks.clear();
    cur = 0;
  }
};

// Per-kernel-class CUDA-event timing (seaice_profile_enable/read): event pairs are
// recorded on the context stream around the launches of one class and harvested
// at host synchronisation points.
enum ProfClass {
  PC_ASSEMBLE = 0,  // K1 fused residual + Jacobian
  PC_SPMV0 = 1,     // K3 finest stencil SpMV (FGMRES operator)
  PC_CHEB0 = 2,     // K4 Chebyshev step, finest level
  PC_CHEBC = 3,     // K4 Chebyshev step, coarse levels
  PC_RESID0 = 4,    // residual + Dinv, finest level
  PC_MDOT = 5,      // K7 multi-dot (CGS projections)
  PC_MAXPY_NORM = 6,// K8 multi-axpy + norm
  PC_MAXPY = 7,     // K10 solution update
  PC_DENERGY = 8,   // K11 line-search energy differences
  PC_TRANSFER = 9,  // K5 restriction / prolongation
  PC_COARSE = 10,   // K6 dense coarse solve
  PC_RESIDC = 11,   // residual + Dinv, coarse levels
  PC_PIUPD = 12,    // K12 dual update
  PC_CHEB0F = 13,   // K4 three Chebyshev steps fused (temporal blocking), finest level
  PC_TRANSPORT = 14,  // NEXT-3 explicit upwind transport of A, h
  PC_MATFREE = 15,  // NEXT-4 matrix-free Jacobian apply
  PC_CHEB1 = 16,    // K4 Chebyshev step on level 1 (PC_CHEBC: levels >= 2)
  PC_RESID1 = 17,   // residual + Dinv on level 1 (PC_RESIDC: levels >= 2)
  PC_TRANSFER0 = 18,  // restriction / prolongation between levels 0 and 1 (PC_TRANSFER: deeper)
  PC_TAIL = 19,       // levels of the persistent V-cycle tail (one cooperative launch)
  PC_NCLASS = 20
};
struct Prof {
  bool on = false;
  std::vector<cudaEvent_t> free_ev;
  struct Rec {
    int k;
    cudaEvent_t a, b;
    bool owned_by_graph;
  };
  std::vector<Rec> pending;
  cudaEvent_t cur_a = nullptr;
  double ms[PC_NCLASS] = {0};
  long long cnt[PC_NCLASS] = {0};
  double bytes[PC_NCLASS] = {0};  // algorithmic bytes of the launches recorded
};

struct Ctx {
  seaice_params p{};
  Prof prof;
  Allocator al;
  cudaStream_t s = nullptr;
  int n = 0, Nn = 0, N = 0, Nc = 0;
  double dx = 0.0;
  Phys ph{};
  std::string err;
  long long launches = 0;
  bool lag_ok = false;       // a hierarchy of this time step exists (amg_lag, reading G31)
  bool reuse_ok = false;     // the hierarchy's aggregates were built in this time step (amg_reuse, G32)
  int reuse_K = 0;           // its near-nullspace dimension
  bool last_setup_reused = false;
  int last_krylov_its = 0;   // Krylov iterations of the previous Newton solve
  long long sg_hits[SEAICE_SPGEMM_PATHS] = {0, 0, 0, 0, 0, 0, 0};  // SpGEMM path counters (seaice_spgemm_path_hits)

  // per-step state
  bool step_set = false, assembled = false, amg_ready = false;
  double dt = 0.0, t_new = 0.0;
  DBuf<double> P, rhoh, F, vprev, vair, vocean, pi, vwork, load;
  bool have_load = false;
  DBuf<int> flag;  // validation / misc device flags

  // finest-level Jacobian: upper half of the symmetric 3x3 node stencil of 2x2 blocks,
  // 19 values per node, slot-major SoA (layout in stencil.cuh)
  DBuf<double> Jst;
  DBuf<double> Jsm;  // smoother copy Jsm[j][20][sp] for the TMA-streamed Chebyshev (cheb_fused = 2)
  DBuf<double> mf_v, mf_pi;  // (v, pi) of the last assembly, for the matrix-free FGMRES operator
  DBuf<double> lin_v;        // v of the last assembly (AMG near-nullspace column, nullspace_dim = 4)
  DBuf<double> R;  // residual of the last assemble
  double last_res_norm = 0.0;
  // scalar CSR view (built on demand)
  DBuf<int> csr_rp, csr_ci;
  DBuf<double> csr_val;
  bool csr_pattern = false;
  long long csr_nnz = 0;

  // reductions
  DBuf<double> part, scal;
  double* hbuf = nullptr;  // pinned host scratch (64 doubles)

  // Newton
  bool have_r0 = false;
  double r0 = 0.0;
  double ew_prev_res = 0.0, ew_prev_eta = 0.0;  // Eisenstat-Walker state of the current step
  bool ew_ls_failed = false;                     // last line search found no decrease
  DBuf<double> vt, pit;

  // Krylov
  DBuf<double> V, Z, w, xk, rk;
  DBuf<double> cg_p, cg_q, cg_s;  // PCG (krylov_method = 1): direction, A p, device scalars

  // AMG (lv is a pool: levels [0, nlev) are active; buffers are reused across setups)
  std::vector<Level> lv;
  int nlev = 0;
  Arena arena;
  // the V-cycle as one CUDA graph (rebuilt after each setup): in vc_in -> out vc_out
  cudaGraphExec_t vgraph = nullptr;
  cudaStream_t cap_stream = nullptr;
  bool use_graphs = true;
  int sms = 148;      // SM count of the device (grid sizing of the streamed smoother)
  DBuf<double> vc_in, vc_out;
  DBuf<double> cinv;  // dense coarse inverse
  int cn = 0;         // coarse DOFs
  double op_complexity = 0.0;
  DBuf<int> iwork;
  DBuf<double> dwork;
  DBuf<long long> lwork;

  // staging buffers of the host-pointer entry point
  DBuf<double> st_h, st_A, st_vp, st_va, st_vo, st_v;

  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  cudaEvent_t arn_ev[2] = {nullptr, nullptr};  // FGMRES: scalars of Arnoldi step j landed in hbuf slot j & 1
};

inline void count_launch(Ctx& c, int k = 1) { c.launches += k; }

inline void prof_harvest(Ctx& c, bool wait) {
  auto& P = c.prof;
  size_t keep = 0;
  for (size_t i = 0; i < P.pending.size(); ++i) {
    auto& r = P.pending[i];
    if (wait) cudaEventSynchronize(r.b);
    if (cudaEventQuery(r.b) == cudaSuccess) {
      float t = 0.f;
      cudaEventElapsedTime(&t, r.a, r.b);
      P.ms[r.k] += t;
      P.cnt[r.k] += 1;
      if (!r.owned_by_graph) {
        P.free_ev.push_back(r.a);
        P.free_ev.push_back(r.b);
      }
    } else {
      P.pending[keep++] = r;
    }
  }
  P.pending.resize(keep);
}
inline cudaEvent_t prof_event(Ctx& c) {
  auto& P = c.prof;
  if (P.free_ev.empty()) {
    if (P.pending.size() > 4096) prof_harvest(c, true);
    if (P.free_ev.empty()) {
      cudaEvent_t e;
      cudaEventCreate(&e);
      return e;
    }
  }
  cudaEvent_t e = P.free_ev.back();
  P.free_ev.pop_back();
  return e;
}
// Per-kernel timing is eager-only: while profiling is on the V-cycle is not replayed as a
// CUDA graph (timing events cannot be taken inside graph replays).
inline void prof_begin(Ctx& c) {
  if (!c.prof.on) return;
  c.prof.cur_a = prof_event(c);
  cudaEventRecord(c.prof.cur_a, c.s);
}
inline void prof_end(Ctx& c, int k, double bytes = 0.0) {
  if (!c.prof.on) return;
  c.prof.bytes[k] += bytes;
  cudaEvent_t b = prof_event(c);
  cudaEventRecord(b, c.s);
  c.prof.pending.push_back({k, c.prof.cur_a, b, false});
}
#define SI_LAUNCHED(c) \
  do {                 \
    SI_CUDA(cudaGetLastError()); \
    (c).launches++;    \
  } while (0)

// assembly.cu
void set_step_impl(Ctx& c, double dt, double t_new, const double* h, const double* A, const double* v_prev,
                   const double* v_air, const double* v_ocean, const double* load);
void assemble_impl(Ctx& c, const double* v, const double* pi, bool jacobian, double* r_out, double* norm_host);
void jv_matfree_impl(Ctx& c, const double* v, const double* pi, const double* x, double* y);
void transport_impl(Ctx& c, double dt, const double* v, const double* A, const double* H, double A_in, double H_in,
                    double* Ao, double* Ho, double* cfl_out = nullptr, int* substeps_out = nullptr);
void build_csr_view(Ctx& c, seaice_csr* out);
void delta_energy_impl(Ctx& c, const double* v, const double* vt, const double* alphas, int count, double* out,
                       double* sabs = nullptr);
void pi_tilde_impl(Ctx& c, const double* v, const double* pi, const double* vt, double* out, double alpha,
                   bool update_in_place);

// linalg.cu
void stencil_spmv(Ctx& c, const double* x, double* y);
void bsr_spmv(Ctx& c, const Level& L, const double* x, double* y);
double dot(Ctx& c, const double* a, const double* b, long long n);
double norm2(Ctx& c, const double* a, long long n);
void axpy(Ctx& c, double a, const double* x, double* y, long long n);   // y += a x
void scal_copy(Ctx& c, double a, const double* x, double* y, long long n);  // y = a x
void xpby(Ctx& c, const double* x, double b, double* y, long long n);   // y = x + b y
void fill(Ctx& c, double* y, double v, long long n);
void copy(Ctx& c, double* dst, const double* src, long long n);
// FGMRES helpers: h[0..j] = V[0..j]^T w ; w -= V h, return ||w||
// h = V[:, :k]^T w, w -= V h, vnext = w / ||w||; returns ||w|| (one host sync)
double arnoldi_step(Ctx& c, const double* V, long long ld, int k, double* w, long long n, double* vnext, double* h_host);
// device part of one Arnoldi step; h (k values) and ||w||^2 are copied to hbuf[64 slot .. ] and
// hbuf[64 slot + 63] without synchronising
void arnoldi_enqueue(Ctx& c, const double* V, long long ld, int k, double* w, long long n, double* vnext, int slot);
void multi_axpy(Ctx& c, const double* Z, long long ld, int k, const double* y_host, double* x, long long n);

// krylov.cu
int fgmres_impl(Ctx& c, const double* b, double* x, seaice_krylov_stats* st);
void precond_apply(Ctx& c, const double* r, double* z);

// amg.cu
void amg_setup_impl(Ctx& c);
void amg_refresh_finest(Ctx& c);
bool amg_lag_allowed(Ctx& c);
void amg_vcycle(Ctx& c, const double* r, double* z);
void amg_free(Ctx& c);

}  // namespace seaice
