/* seaice.h — C-ABI of the B200-native stress-velocity (primal-dual) Newton-Krylov
 * step for the implicit viscous-plastic sea-ice momentum equation
 * (Shih, Mehlmann, Losch, Stadler, arXiv 2204.10822; "P:<line>" = PAPER.md line).
 *
 * Problem statement: given ice thickness h,
 * concentration A (per cell), the previous velocity v^n, wind v_a and ocean
 * velocity v_o (per node), the time step dt and t_{n+1}, find v^{n+1} solving
 * A(v, phi) = F(phi) for all Q1 test functions phi vanishing on the boundary.
 *
 * Conventions (all entry points):
 *  - All array arguments are DEVICE pointers to contiguous fp64 (int32 where noted),
 *    owned by the caller, unless the name ends in _host.  The library never frees them.
 *  - All work is enqueued on the CUDA stream given at create.  Calls that return
 *    host scalars or statistics synchronize that stream before returning.
 *  - Mesh: n x n uniform square cells of side dx = L/n on (0,L)^2.
 *    Cell (i,j) -> j*n+i.  Node (i,j) -> j*(n+1)+i.  DOF = 2*node + c, c = 0 (x), 1 (y).
 *    N = 2(n+1)^2 DOFs, Nc = n^2 cells.
 *  - pi (the dual variable, eq:pi P:444-448) is stored per Gauss point as
 *    double[3][4][Nc]: component (pi11, pi12, pi22) major, then Gauss point
 *    (-g,-g),(g,-g),(g,g),(-g,g) with g = 1/sqrt3, then cell.
 *  - Dirichlet v = 0 on the boundary: residual entries of boundary DOFs
 *    are 0 and the Jacobian has identity rows/columns there (symmetric elimination).
 *  - Errors: every call returns a seaice_status; on a negative status the text is
 *    available from seaice_last_error(ctx).  A context is used by one host thread.
 */
#ifndef SEAICE_H
#define SEAICE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct seaice_ctx seaice_ctx;

typedef enum {
  SEAICE_OK = 0,
  SEAICE_NOT_CONVERGED = 1, /* result valid, iteration cap hit (Krylov maxit / Newton maxit) */
  SEAICE_EINVAL = -1,       /* bad argument / parameter / out-of-range input field */
  SEAICE_ENOMEM = -2,       /* device allocation failed */
  SEAICE_ECUDA = -3,        /* CUDA runtime error (text in seaice_last_error) */
  SEAICE_ENONFINITE = -4,   /* NaN/Inf in a residual norm */
  SEAICE_ESTATE = -5        /* call order violated (e.g. residual before set_step) */
} seaice_status;

typedef enum { SEAICE_JAC_SV = 0, SEAICE_JAC_STD = 1, SEAICE_JAC_PICARD = 2 } seaice_jacobian_kind;
typedef enum { SEAICE_PC_AMG = 0, SEAICE_PC_JACOBI = 1, SEAICE_PC_NONE = 2 } seaice_precond_kind;

/* Device memory comes from these callbacks when alloc != NULL (the Python binding
 * passes the torch caching allocator); otherwise cudaMallocAsync on `stream`.
 * Internal buffers are grow-only and released by seaice_destroy. */
typedef struct {
  void* stream; /* cudaStream_t; NULL = legacy default stream */
  void* (*alloc)(size_t bytes, void* stream, void* user);
  void (*free)(void* ptr, void* stream, void* user);
  void* user;
} seaice_runtime;

typedef struct {
  int32_t n;          /* cells per side, n >= 2 */
  double L;           /* domain edge [m] (512 km) */
  /* Table 1 with BASELINE.json's P* = 27500 N/m and f_c = 1.46e-4 1/s */
  double rho_i, rho_a, rho_o, C_a, C_o, P_star, C, e, delta_min, f_c;
  int32_t jacobian;        /* seaice_jacobian_kind: SV = eq:linearSVNewton + eq:modification */
  double newton_rtol;      /* ||R(v_l)|| <= rtol ||R(v_0)|| (BASELINE.json 1e-8) */
  int32_t newton_maxit;    /* 200 */
  int32_t ls_max_halvings; /* 20: alpha = 1, 1/2, ..., 2^-20 */
  double krylov_rtol;      /* 1e-8 relative to ||b|| */
  int32_t restart;         /* FGMRES restart m (60; 1..60).  The paper does not state it (reading G13) */
  int32_t krylov_maxit;    /* 300 */
  int32_t precond;         /* seaice_precond_kind */
  double amg_theta;        /* strength threshold of the node-block measure */
  int32_t cheb_degree;     /* Chebyshev(block-Jacobi) degree per pre/post smoothing */
  int32_t coarse_max_dof;  /* dense coarse solve at or below this many DOFs */
  int32_t max_levels;
  double cheb_lower;       /* smoothing interval [cheb_lower * b, b], b = cheb_upper * lambda_max */
  double cheb_upper;
  int32_t power_iters;     /* power iterations for lambda_max(D^-1 A) */
  int32_t project_pi;      /* 0 (default): store pi unprojected (reading G5) */
  uint64_t amg_seed;
  int32_t agg_dist0;       /* aggregation root distance on the finest level: 2 = MIS(2) (default), 1 = MIS(1),
                              3 = MIS(3) (larger aggregates) */
  int32_t agg_dist;        /* same on coarse levels (default 3) */
  int32_t cheb_fused;      /* finest-level Chebyshev(3): 2 (default) one y-streamed, TMA-fed temporally
                              blocked launch per smoothing (the post-smoothing residual included; reads a
                              tensor-map copy of the stencil, vectors must be 16-byte aligned); 1: one
                              tile-blocked launch (+ a residual launch for post-smoothing); 0: one launch
                              per step.  Same arithmetic per node and step (A u summed in another order
                              for 2) */
  int32_t cheb_degree0;    /* Chebyshev degree on the finest level (0: cheb_degree) */
  int32_t matfree;         /* 0 (default): FGMRES applies the assembled stencil J; 1: FGMRES applies
                              J(v, pi) matrix-free from the (v, pi) of the
                              last assembly, the AMG hierarchy still built from the assembled J */
  int32_t krylov_forcing;  /* 0: every Newton solve to krylov_rtol (reading G13);
                              1 (default): Eisenstat-Walker choice-2 forcing (inexact Newton; the paper is
                              silent on its Krylov tolerance): eta_0 = 0.1, eta_l = 0.9 (|R_l| /
                              |R_{l-1}|)^2 with the safeguards eta_l >= 0.9 eta_{l-1}^2 (when that
                              exceeds 0.1) and eta_l >= 0.5 newton_rtol |R_0| / |R_l|, clamped to
                              [krylov_rtol, 0.1] (reading G29) */
  int32_t nullspace_dim;   /* AMG near-nullspace columns per aggregate = coarse block size:
                              3 = rigid-body modes (1,0), (0,1), rotation; 4 (default, reading G30)
                              adds the linearisation point v_l of the last seaice_assemble_jacobian,
                              a near-null vector of the plastic part of eq:modification:
                              C_q tau(v_l) = (P/Delta)(Delta_min^2/Delta^2) tau(v_l) at consistent pi */
  int32_t krylov_method;   /* 0 (default): FGMRES(restart); 1: preconditioned CG (J and the
                              symmetric V-cycle are SPD, eq:modification P:534-539; same stopping test) */
  int32_t spgemm_path;     /* 0 (default): SpGEMM code path chosen by row-expansion size; testing knob
                              to force one path for every product: 1 hash tables (1k, else 4k
                              entries, else sort), 2 sort + thread-per-row numeric, 3 sort + 8-lane
                              groups, 4 sort + warp per row, 5 8-lane hash tables (falls back when a
                              row's expansion exceeds 256), 6 hash tables of 4k entries (else sort)
                              (see seaice_spgemm_path_hits) */
  int32_t amg_lag;         /* default 10.  0: full AMG setup at every Newton iteration; T > 0 (reading G31):
                              at Newton iteration l >= 1 of a time step the hierarchy is rebuilt only
                              if the previous linear solve needed more than T Krylov iterations,
                              otherwise its coarse levels (P, R, A_l, l >= 1) are kept and only the
                              finest level (D^-1 blocks, lambda_max) is refreshed from the current J */
  int32_t amg_reuse;       /* 0: every AMG setup builds its aggregates; 1 (reading G32): the
                              first setup of a time step builds them, every later setup of the step
                              keeps the aggregates and all sparsity patterns (P_tent, P, R, Galerkin
                              products) and recomputes every value from the current J and v_l
                              (near-nullspace, P_tent, lambda_max, smoothed P, A_l, coarse factor);
                              falls back to a full setup when the near-nullspace dimension changes */
  int32_t vcycle_tail;     /* 0 (default): one launch per smoothing step / transfer on every level; 1: the bottom
                              levels of the V-cycle (4 x 4-block levels whose operators and transfers
                              together stay under ~48 MB, i.e. L2-resident) run in ONE cooperative launch,
                              phases separated by grid barriers.  Same operations in the same order (row
                              sums grouped as the per-launch kernels group them).  Measured on B200 at
                              config 4: the launch takes 136 us against 184 us for the 27 launches it
                              replaces, but inside the captured V-cycle graph the cooperative node costs
                              more than it saves (2442 -> 2499 us per V-cycle), hence off by default */
} seaice_params;

/* Compressed-sparse-row view (scalar rows). Index arrays int32, values fp64. */
typedef struct {
  int32_t nrows, ncols;
  int64_t nnz;
  const int32_t* row_ptr;
  const int32_t* col_idx;
  const double* val;
} seaice_csr;

/* Block CSR view: block rows of br x bc dense blocks, row-major inside a block,
 * blocks stored contiguously (val[e*br*bc + r*bc + c]). */
typedef struct {
  int32_t nbrows, nbcols, br, bc;
  int64_t nnzb;
  const int32_t* row_ptr;
  const int32_t* col_idx;
  const double* val;
} seaice_bsr;

typedef struct {
  int32_t iters, restarts, converged;
  double relres_est, relres_true;
} seaice_krylov_stats;

typedef struct {
  int32_t converged_on_entry; /* ||R(v)|| <= newton_rtol * r0 at entry: no step taken */
  double res_norm, res_norm0;  /* ||R(v_l)||_2 at entry, r0 = ||R(v_0)||_2 */
  double alpha, dphi;          /* accepted step and Phi(v+alpha v~) - Phi(v) */
  int32_t halvings, ls_stagnated;
  seaice_krylov_stats krylov;
  int32_t amg_levels;
  double amg_op_complexity;
  double t_assemble, t_amg, t_krylov, t_ls; /* milliseconds (CUDA events) */
  int32_t amg_rebuilt;      /* 1: full AMG setup this iteration; 0: coarse levels kept (amg_lag) */
  int32_t amg_reused;       /* 1: the setup kept the step's aggregates and patterns (amg_reuse) */
} seaice_newton_stats;

typedef struct {
  int32_t newton_iters, converged, krylov_iters_total;
  double res_norm0, res_norm_final, seconds;
  double t_assemble, t_amg, t_krylov, t_ls, t_setup; /* milliseconds */
  int32_t krylov_solves;    /* linear solves in the step (= newton_iters) */
  int32_t krylov_capped;    /* solves that stopped at krylov_maxit without reaching krylov_rtol
                               (their iterations are counted in krylov_iters_total; the Newton
                               step still used the capped iterate) */
  int32_t krylov_max_iters; /* largest iteration count of one solve */
  int32_t amg_setups;       /* full AMG setups in the step (< newton_iters with amg_lag) */
  int32_t amg_reuses;       /* of those, setups that kept the aggregates and patterns (amg_reuse) */
} seaice_step_stats;

/* Default parameters (Table 1 + BASELINE.json + DESIGN.md readings) for mesh size n. */
void seaice_default_params(seaice_params* p, int32_t n);

/* Allocate a context for the mesh in `p` (SURVEY §8(b) seaice_create <-> build_grid +
 * PhysicsParams).  EINVAL on n < 2, non-positive physical constants or
 * 36 (n+1)^2 >= 2^31 (int32 CSR indices). */
int seaice_create(const seaice_params* p, const seaice_runtime* rt, seaice_ctx** out);
int seaice_destroy(seaice_ctx* ctx);
const char* seaice_last_error(const seaice_ctx* ctx);

/* Per-step inputs (eq:F P:330-331 uses tau_atm(t_{n+1})).  h, A [Nc];
 * v_prev, v_air, v_ocean [N] interleaved nodal; extra_load [N] or NULL (a load
 * vector added to F, used by manufactured-solution tests).  Copies the inputs,
 * computes P = P* h exp(-C(1-A)), rho_i h, F, and resets the dual
 * variable pi := tau(v_prev)/Delta(v_prev) (reading G4) and the Newton state.
 * EINVAL if some A is outside [0,1], h < 0, or a value is not finite. */
int seaice_set_step(seaice_ctx* ctx, double dt, double t_new, const double* h, const double* A,
                    const double* v_prev, const double* v_air, const double* v_ocean,
                    const double* extra_load);

/* R(v) = F - A(v) with A from eq:A / eq:sigma; r_out [N]
 * (may be NULL); *norm2_host = ||R||_2 (may be NULL). */
int seaice_residual(seaice_ctx* ctx, const double* v, double* r_out, double* norm2_host);

/* Assemble the Newton Jacobian at (v, pi) (pi NULL = the context's pi):
 * SV: eq:linearSVNewton with eq:modification;
 * STD: eq:standardNewton; PICARD: viscous part (P/Delta) only.
 * Also computes R(v) into the context.  J_view (may be NULL) receives a scalar CSR
 * view (ctx-owned, valid until the next assemble or destroy); interior rows hold
 * 18 entries (explicit zeros toward boundary columns), boundary rows 1. */
int seaice_assemble_jacobian(seaice_ctx* ctx, const double* v, const double* pi, seaice_csr* J_view);

/* y = J x with the last assembled Jacobian. */
int seaice_spmv(seaice_ctx* ctx, const double* x, double* y);

/* Explicit transport of A and H between momentum steps: explicit-Euler,
 * first-order upwind finite-volume steps of eq:model:A / eq:model:H ("an explicit
 * time step (e.g., an explicit Euler step)"; scheme = DESIGN.md reading G28).
 * v: nodal velocity [2(n+1)^2] interleaved (device); A, H: cell fields [n*n] row-major
 * (device, read); A_out, H_out: [n*n] (device, written; must not alias A or H).  Face-normal
 * velocity = mean of the face's two nodal velocities; an inflow boundary face carries A_in /
 * H_in; A_out is clamped to [0,1], H_out to [0,inf).
 * CFL guard: CFL = max over cells of dt/dx * (sum of the cell's outflow face velocities), the
 * bound under which the upwind update is monotone.  If CFL > 1 the step is taken as
 * m = ceil(CFL) sub-steps of dt/m (same v).  *cfl_host and *substeps_host (each may be NULL)
 * receive CFL and m.  Synchronises the ctx stream once (to read CFL).  EINVAL on NULL /
 * aliased buffers, dt < 0 / non-finite or CFL > 1e5; ENONFINITE on a non-finite velocity. */
int seaice_transport(seaice_ctx* ctx, double dt, const double* v, const double* A, const double* H,
                     double A_in, double H_in, double* A_out, double* H_out, double* cfl_host,
                     int32_t* substeps_host);

/* Matrix-free Jacobian apply y = J(v, pi) x (eq:linearSVNewton P:512-525 with
 * eq:modification P:534-539; the JFNK discussion P:545-653): the element matrices of the ctx's
 * jacobian kind are recomputed per cell (same arithmetic as seaice_assemble_jacobian) and applied
 * to x without storing J; Dirichlet rows return x, Dirichlet columns are eliminated.  v, x, y:
 * [2(n+1)^2] interleaved (device); pi: [3][4][n*n] (device) or NULL = ctx pi.  Needs set_step.
 * Enqueued on the ctx stream.  EINVAL on NULL v / x / y or y aliasing x. */
int seaice_jv_matfree(seaice_ctx* ctx, const double* v, const double* pi, const double* x, double* y);

/* Build the AMG hierarchy of the last assembled Jacobian on the GPU: node-block
 * strength, MIS(2) aggregation, rigid-body tentative prolongator, smoothed
 * prolongator, Galerkin R A P via SpGEMM, block-Jacobi Chebyshev data, dense
 * coarse inverse.  Outputs may be NULL. */
int seaice_amg_setup(seaice_ctx* ctx, int32_t* levels_out, double* op_complexity_out);

/* Views of AMG level l (0 = finest): A_l (BSR), P_l (BSR, l < levels-1). */
int seaice_amg_level(seaice_ctx* ctx, int32_t level, seaice_bsr* A_out, seaice_bsr* P_out,
                     int32_t* aggregates_host_or_null);

/* z = M^-1 r: one application of the configured preconditioner (AMG V-cycle). */
int seaice_precond_apply(seaice_ctx* ctx, const double* r, double* z);

/* Right-preconditioned FGMRES(restart) on J x = b, x0 = 0. */
int seaice_fgmres_solve(seaice_ctx* ctx, const double* b, double* x, seaice_krylov_stats* st);

/* Phi(v + alpha_k vt) - Phi(v) (eq:energy P:261-268, difference form, reading G12)
 * for alpha_k = alphas_host[k], k < count (count <= 32); out_host[count]. */
int seaice_delta_energy(seaice_ctx* ctx, const double* v, const double* vt, const double* alphas_host,
                        int32_t count, double* out_host);

/* pi_out = pi~(v, pi, vt) (eq:tautilde P:504-511 with eq:modification). */
int seaice_pi_tilde(seaice_ctx* ctx, const double* v, const double* pi, const double* vt, double* pi_out);

/* Copy the context's pi to / from caller memory ([3][4][Nc]). */
int seaice_get_pi(seaice_ctx* ctx, double* pi_out);
int seaice_set_pi(seaice_ctx* ctx, const double* pi_in);

/* One Newton iteration of the stress-velocity method: v_{l+1} = v_l + alpha v~,
 * pi_{l+1} = pi_l + alpha pi~ with J(v_l, pi_l) v~ = R(v_l) (eq:linearSVNewton
 * P:512-527, eq:modification P:534-539) and alpha from backtracking on Phi (P:355-360,
 * P:727-732; difference form, reading G12/G12b).  The first call after set_step
 * records r0 = ||R(v)||; a call that finds ||R(v)|| <= newton_rtol*r0 (or r0 < 1e-14)
 * sets converged_on_entry = 1 and takes no step.  Otherwise: assemble, (AMG setup),
 * FGMRES, energy backtracking, v += alpha v~, pi += alpha pi~.  pi_inout may be
 * NULL (context pi).  Returns NOT_CONVERGED if the linear solve hit its cap. */
int seaice_newton_step(seaice_ctx* ctx, double* v_inout, double* pi_inout, seaice_newton_stats* st);

/* Whole implicit step: set_step + Newton loop to convergence; v_out [N] device.
 * NOT_CONVERGED if newton_maxit is reached.  Linear solves that hit krylov_maxit do not
 * change the return code (Newton tolerates inexact solves) but are counted in
 * st->krylov_capped. */
int seaice_solve_step(seaice_ctx* ctx, double dt, double t_new, const double* h, const double* A,
                      const double* v_prev, const double* v_air, const double* v_ocean, double* v_out,
                      seaice_step_stats* st);

/* Same with HOST input/output buffers: copies inputs H2D, solves, copies v_out D2H
 * (end-to-end path; host buffers should be pinned for full copy bandwidth). */
int seaice_solve_step_host(seaice_ctx* ctx, double dt, double t_new, const double* h_host,
                           const double* A_host, const double* v_prev_host, const double* v_air_host,
                           const double* v_ocean_host, double* v_out_host, seaice_step_stats* st);

/* Number of kernels the library launched since create (evidence for bench.py). */
int64_t seaice_launch_count(const seaice_ctx* ctx);

/* Per-kernel-class timing with CUDA events recorded on the context stream around
 * each launch.  Classes: 0 assembly (K1), 1 finest SpMV, 2 finest Chebyshev step,
 * 3 coarse Chebyshev step, 4 finest residual+Dinv, 5 Krylov multi-dot, 6 multi-axpy+norm,
 * 7 solution update, 8 line-search energy, 9 restriction/prolongation, 10 coarse solve,
 * 11 coarse residual+Dinv (levels >= 2), 12 dual update, 13 fused finest Chebyshev(3),
 * 14 transport, 15 matrix-free apply, 16 Chebyshev step on level 1, 17 residual+Dinv on level 1,
 * 18 restriction/prolongation between levels 0 and 1 (9: deeper levels; 3: coarse Chebyshev on
 * levels >= 2).  enable: resets the counters and turns the
 * timing on (1) or off (0).  read: synchronizes, returns total milliseconds, launch
 * counts and algorithmic bytes (DESIGN.md formulas) per class (arrays of
 * SEAICE_PROF_CLASSES; any pointer may be NULL). */
#define SEAICE_PROF_CLASSES 24
int seaice_profile_enable(seaice_ctx* ctx, int32_t on);
int seaice_profile_read(seaice_ctx* ctx, double* ms_host, int64_t* launches_host, double* alg_bytes_host);

/* Which SpGEMM code path each Galerkin / prolongator-smoothing product of seaice_amg_setup took,
 * counted since create (the numeric result is the same definition on every path;
 * the choice depends only on row-expansion sizes).  hits[0] 1k-entry hash table per row,
 * [1] 4k-entry hash table, [2] sort-based thread-per-row numeric, [3] sort-based 8-lane-group
 * numeric, [4] sort-based warp-per-row (wide rows), [5] 8-lane-per-row hash tables (short Y
 * rows: the level-0 Galerkin products), [6] numeric phase by a CTA per row with shared-memory
 * accumulators (levels of <= 16384 rows whose rows have <= 640 block columns; replaces the
 * numeric kernel of paths 0, 1 and 4 there).  n_host: entries to write (<= 7). */
#define SEAICE_SPGEMM_PATHS 7
int seaice_spgemm_path_hits(const seaice_ctx* ctx, int64_t* hits_host, int32_t n_host);

/* Bytes of device memory the context currently holds (and its peak). */
int seaice_memory(const seaice_ctx* ctx, int64_t* live_bytes, int64_t* peak_bytes);

#ifdef __cplusplus
}
#endif
#endif /* SEAICE_H */
