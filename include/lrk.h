/*
 * lrk.h — C ABI of the B200-native low-rank space-time Hessian apply.
 *
 * This is the drop-in boundary for the hot path of the reference package
 * `lrpostcov` (/root/reference/pkg/src/lrpostcov).  The reference has no FFI:
 * its "operator API" is the Python callable HessianContext.apply
 * (hessian.py:202-208) plus the module functions it is built from.  Each entry
 * point below replaces one of those functions; the Python package
 * `paper_1703_05638_b200` binds them with ctypes and keeps
 * the reference's Python names and signatures.
 *
 * Conventions
 *  - All arrays are fp64 device pointers owned by the caller, except workspace,
 *    which the context owns.  Factors are COLUMN-MAJOR: column j of W1 starts
 *    at W1 + j*ld1 (ld1 >= n_x), so every spatial column is contiguous.
 *  - `stream` is a cudaStream_t passed as void* (NULL = legacy default stream).
 *  - Every function returns an lrk_status; nothing throws across the ABI.
 *    lrk_last_error(ctx) returns the message of the last failure on ctx.
 *  - One call in flight per context (the reference's HessianContext contract,
 *    hessian.py:163-166).  Use several contexts for concurrency.
 */
#ifndef LRK_H_
#define LRK_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes; the Python shim maps them onto the reference's exceptions
 * (errors.py:4-21): SHAPE -> ValueError, CONFIG -> InvalidConfigError,
 * NUMERICAL -> NumericalError, CONVERGENCE -> ConvergenceFailure. */
typedef enum {
  LRK_OK = 0,
  LRK_ERR_SHAPE = 1,
  LRK_ERR_CONFIG = 2,
  LRK_ERR_NUMERICAL = 3,
  LRK_ERR_CONVERGENCE = 4,
  LRK_ERR_CUDA = 5,
  LRK_ERR_UNSUPPORTED = 6
} lrk_status;

typedef struct lrk_ctx lrk_ctx;

/* A low-rank space-time field Y = W1 * W2^T (lowrank.py:39-78).
 * rank r may be 0 (the zero field).  cap = allocated columns (>= r). */
typedef struct {
  double* W1;
  double* W2;
  int64_t ld1;
  int64_t ld2;
  int n_x;
  int n_t;
  int r;
  int cap;
} lrk_lr;

/* Spatial operator + time grid (discretize.py:107-127, forward.py:40-51).
 * kind: 0 = heat, 1 = convection-diffusion (physical-space sweep).
 * stencil: 0 = FD (5-point in 2-D as the reference, 7-point in 3-D),
 *          1 = Q1 bilinear FEM stiffness with lumped mass (9-point, 2-D only;
 *              L = K_Q1 / h^2).
 * The step matrix is S = m_scale * (I + tau * L). */
enum { LRK_OP_HEAT = 0, LRK_OP_CONVDIFF = 1 };
enum { LRK_STENCIL_FD = 0, LRK_STENCIL_Q1 = 1 };
enum { LRK_WIND_CONST = 0, LRK_WIND_ROTATING = 1 };
typedef struct {
  int kind;
  int dim;      /* spatial dimension; 2 or 3 */
  int n_side;   /* interior points per axis; n_x = n_side^dim */
  int n_t;      /* time steps */
  double h;     /* mesh size 1/(n_side+1) */
  double tau;   /* time step T/n_t */
  double m_scale; /* lumped mass h^dim */
  double nu;
  double wind[3];
  int stencil;  /* LRK_STENCIL_* (0 = the reference's FD operator) */
  /* convdiff wind: 0 = constant wind[] (the reference); 1 = wind[] + the
   * rotating field (2 x2 (1 - x1^2), -2 x1 (1 - x2^2), 0) of configs C3/C5,
   * upwinded per node by the sign of the local wind (discretize.py:96-104
   * applied node by node). */
  int wind_field;
} lrk_operator_desc;

/* Observation operator (hessian.py:78-156).
 * kind 0: full observation; 1: separable sensor subgrid (mask = rows2 x rows1,
 * x1 fastest); 2: arbitrary list of observed dofs (sorted ascending). */
enum { LRK_OBS_FULL = 0, LRK_OBS_SUBGRID = 1, LRK_OBS_LIST = 2 };
typedef struct {
  int kind;
  int n1, n2;              /* subgrid sizes per axis (kind 1) */
  const int32_t* idx1;     /* host pointers, x1 indices (kind 1) */
  const int32_t* idx2;     /* x2 indices (kind 1) */
  int n_list;              /* number of observed dofs (kind 2) */
  const int32_t* list;     /* host pointer, sorted dof indices (kind 2) */
} lrk_obs_desc;

/* Hessian configuration (HessianContext, hessian.py:159-187). */
enum { LRK_MODE_IC = 0, LRK_MODE_SOURCE = 1 };
typedef struct {
  int mode;
  double gamma_prior;   /* Gamma_prior = gamma * I                          */
  double obs_weight;    /* beta_noise * tau * m_scale (hessian.py:153)        */
  double eps0;          /* TruncationPolicy.eps0                             */
  int r_max;            /* TruncationPolicy.r_max, < 0 means None            */
  int compress_every;   /* sweep flush period (hessian.py:174)               */
  /* Config extensions; all-zero = reference:
   * prior_gamma > 0: Gamma_prior^{1/2} = sqrt(gamma_prior) (prior_delta I +
   *   prior_gamma L)^{-1}, applied on both sides of the misfit Hessian;
   * obs_every > 1: observe only time steps k (0-based) with (k+1) % obs_every
   *   == 0 (a row mask on the W2 time factor). */
  double prior_delta;
  double prior_gamma;
  int obs_every;
} lrk_hessian_desc;

/* ---- context ---------------------------------------------------------- */
int lrk_ctx_create(int device, lrk_ctx** out);
void lrk_ctx_destroy(lrk_ctx* ctx);
const char* lrk_last_error(const lrk_ctx* ctx);
/* Library build/version string. */
const char* lrk_version(void);

/* Install the spatial operator; replaces SpaceTimeOperator.__init__
 * (forward.py:40-51): instead of a sparse LU it precomputes the DST-I
 * diagonalisation of the step matrix. */
int lrk_set_operator(lrk_ctx* ctx, const lrk_operator_desc* op);
/* Install the observation layout (SensorLayout mask, hessian.py:78-135). */
int lrk_set_observation(lrk_ctx* ctx, const lrk_obs_desc* obs);

/* ---- factor algebra (lowrank.py) --------------------------------------- */
/* lr_truncate (lowrank.py:124-144) incl. _rank_cut (:98-111) and _svd_flip
 * (:114-121).  out must not alias in; out->cap >= min(in->r, r_max).
 * flags: bit0 = W1 columns already orthonormal, bit1 = W2 = V*diag(s) with
 * V orthonormal (skip the QRs).  On return out->r and *r_out hold the rank. */
enum { LRK_TRUNC_W1_ORTHO = 1, LRK_TRUNC_W2_ORTHOSCALED = 2 };
int lrk_truncate(lrk_ctx* ctx, const lrk_lr* in, lrk_lr* out, double eps0,
                 int r_max, int flags, int* r_out, void* stream);
/* lr_dot (lowrank.py:163-168): *out (host) = <vec(A), vec(B)>. */
int lrk_dot(lrk_ctx* ctx, const lrk_lr* a, const lrk_lr* b, double* out,
            void* stream);
/* Singular values of a field (lowrank.py:176-182): writes min(r, cap) values
 * to s_host (descending), count to *n_out. */
int lrk_singular_values(lrk_ctx* ctx, const lrk_lr* a, double* s_host,
                        int cap, int* n_out, void* stream);

/* ---- space-time operator (forward.py) ---------------------------------- */
/* SpaceTimeOperator.solve_step (forward.py:61-68): X = S^{-1} B (or S^{-T}). */
int lrk_step_solve(lrk_ctx* ctx, const double* B, int64_t ldb, int ncols,
                   int adjoint, double* X, int64_t ldx, void* stream);
/* Steady Poisson solve X = L^{-1} B (heat operator; hessian.py:248-259). */
int lrk_poisson_solve(lrk_ctx* ctx, const double* B, int64_t ldb, int ncols,
                      double* X, int64_t ldx, void* stream);
/* SpaceTimeOperator.apply / apply_adjoint (forward.py:79-95): out = K Y in
 * factor form, rank 2r (not truncated). out->cap >= 2*Y->r. */
int lrk_operator_apply(lrk_ctx* ctx, const lrk_lr* Y, int adjoint,
                       lrk_lr* out, void* stream);
/* st_solve_sweep / st_solve_adjoint_sweep (forward.py:133-201).  trace
 * (host, may be NULL) receives the pane rank after every flush plus the final
 * rank (forward.py:175, :187); *trace_len its length. */
int lrk_st_solve_sweep(lrk_ctx* ctx, const lrk_lr* rhs, int adjoint,
                       int compress_every, double eps0, int r_max,
                       lrk_lr* out, int* trace, int trace_cap, int* trace_len,
                       void* stream);

/* Fused concatenate-and-truncate (lowrank.py:147-154 then :124-144):
 * out = truncate(sum_i coef[i] * terms[i]) with ONE truncation of the whole
 * concatenation, as the reference's GMRES (forward.py:247-251) and Ritz
 * combinations do.  coef is a host array (NULL = all ones).  Widths above the
 * 160-column device core are handled exactly: through the dense n_x x n_t
 * (or n_t x n_x) product when min(n_x, n_t) <= 160, otherwise by folding
 * slices at the rounding floor (LRK_ERR_UNSUPPORTED only if the numerical rank
 * of a partial sum exceeds 160).  out->r and *r_out hold the rank. */
int lrk_add_truncate(lrk_ctx* ctx, int nterms, const lrk_lr* terms, const double* coef,
                     double eps0, int r_max, lrk_lr* out, int* r_out, void* stream);
/* Batched lr_dot of one field against many (lowrank.py:163-168):
 * basis is the column-wise concatenation of nseg fields (segment g has
 * seg_cols[g] columns, host array); out_host[g] = <w, field g>.  Two Gram
 * launches on the FP64 tensor pipe + one segmented reduction + ONE readback
 * (the per-pass inner products of CGS/MGS without per-pair host syncs). */
int lrk_lr_dots(lrk_ctx* ctx, const lrk_lr* w, const lrk_lr* basis, int nseg,
                const int* seg_cols, double* out_host, void* stream);

/* Space-time solve with a selectable backend (forward.py:133-201, :217-274). */
enum { LRK_SOLVE_SWEEP = 0, LRK_SOLVE_GMRES = 1 };
typedef struct {
  int backend;          /* LRK_SOLVE_*                                       */
  double eps0;          /* TruncationPolicy.eps0                             */
  int r_max;            /* < 0: None                                          */
  int compress_every;   /* sweep flush period                                 */
  double tol;           /* GMRES relative residual (forward.py:221)          */
  int max_iter;         /* GMRES iteration cap; <= 0: n_t + 5 (:235-236)     */
} lrk_solve_desc;
/* Filled on return, also on LRK_ERR_CONVERGENCE (ConvergenceFailure's
 * achieved_residual and iterations, errors.py:12-21, forward.py:269-274). */
typedef struct {
  double achieved_residual;
  int iterations;
  int rank;
} lrk_solve_info;
/* K vec(Y) = vec(rhs) (K^T when adjoint).  trace (host, may be NULL): sweep =
 * pane rank per flush + final (forward.py:175, :187); GMRES = rank of each
 * orthogonalised Krylov field (forward.py:252-253). */
int lrk_st_solve(lrk_ctx* ctx, const lrk_lr* rhs, int adjoint, const lrk_solve_desc* sd,
                 lrk_lr* out, lrk_solve_info* info, int* trace, int trace_cap, int* trace_len,
                 void* stream);

/* ---- Hessian apply (hessian.py:211-245) -------------------------------- */
/* misfit_apply_ic: out = H~ v for nbatch independent dense vectors (columns
 * of V, ld ldv) -> columns of OUT.  max_rank (host, nbatch entries, may be
 * NULL) receives the per-apply max intermediate rank (hessian.py:225). */
int lrk_hessian_apply_ic(lrk_ctx* ctx, const lrk_hessian_desc* hd, int nbatch,
                         const double* V, int64_t ldv, double* OUT,
                         int64_t ldo, int* max_rank, void* stream);
/* misfit_apply_st: out = truncate(H~ vec(v)) for a low-rank field. */
int lrk_hessian_apply_st(lrk_ctx* ctx, const lrk_hessian_desc* hd,
                         const lrk_lr* v, lrk_lr* out, int* max_rank,
                         void* stream);

/* ---- dense Krylov helpers for lr_arnoldi (arnoldi.py:313-354) ---------- */
/* Two-pass classical Gram-Schmidt of w (length n) against the k columns of
 * Q (ld ldq); h_host[0..k) accumulates both passes' coefficients (the
 * reference's `H[i, j] +=`, arnoldi.py:325), *norm_out = ||w|| after. */
int lrk_cgs2(lrk_ctx* ctx, const double* Q, int64_t ldq, int k, double* w,
             int n, double* h_host, double* norm_out, void* stream);
/* y = Q c (n rows, k columns; c on host) — Ritz-vector combination
 * (arnoldi.py:120-125). */
int lrk_combine(lrk_ctx* ctx, const double* Q, int64_t ldq, int k,
                const double* c_host, int n, double* y, void* stream);

/* Number of device kernels this context has launched (instrumentation). */
int64_t lrk_launch_count(const lrk_ctx* ctx);

/* Instrumentation for the roofline: when enabled, every sweep launch is
 * bracketed by CUDA events on its stream and its algorithmic bytes (DESIGN.md
 * §Roofline) are accumulated once the apply's ranks are known. */
/* Config prior on physical rows:
 * Y = (delta I + gamma L)^{-power} X (power 1 or 2), and its diagonal
 * out[n_x] = diag((delta I + gamma L)^{-power}) (posterior variance with a
 * non-scalar prior: diag(G_post) = g [diag(P^2) - sum_i l~_i (P v_i)^2]). */
int lrk_prior_apply(lrk_ctx* ctx, double delta, double gamma, int power, const double* X,
                    int64_t ldx, int ncols, double* Y, int64_t ldy, void* stream);
int lrk_prior_diag(lrk_ctx* ctx, double delta, double gamma, int power, double* out,
                   void* stream);
/* Run every subsequent sweep of this context as nshard n_x shards (the
 * multi-GPU decomposition of SURVEY §8(e): global CTA rows, partials read
 * through a per-shard table, one shared barrier) emulated as nshard groups of
 * ONE cooperative launch on this device.  Results are bit-identical to the
 * unsharded sweep when the CTA count divides evenly; used by the tests. */
/* n_x sharding across GPUs (the reference's time loop
 * forward.py:179-186 and flush truncation lowrank.py:133-135, sharded by
 * rows).  One process per GPU; every rank installs the same operator and
 * observation, then
 *   lrk_shard_setup(ctx, rank, world, handle)   -> 64-byte IPC handle of this
 *       rank's peer-shared arena (exchange slots + the two sweep panes);
 *   all-gather the handles (torch.distributed / MPI / a file);
 *   lrk_shard_connect(ctx, handles)             -> maps the peers' arenas.
 * Afterwards lrk_hessian_apply_ic runs its two sweeps on this rank's row slab
 * (streaming-flush form): every pass ends in a small rank total that the last
 * CTA stores straight into all peers' exchange slots over NVLink, followed by
 * a system-scope release flag; the rank's slab of the final pane is pushed
 * into the peers' panes the same way.  Inputs and outputs stay replicated
 * n_x vectors, all ranks return identical results.  world <= 8. */
int lrk_shard_setup(lrk_ctx* ctx, int rank, int world, void* handle_out);
int lrk_shard_connect(lrk_ctx* ctx, const void* handles);
/* Single-device emulation of the same sharded sweeps (tests): nshard row
 * slabs driven by one process, launched pass by pass. */
int lrk_set_emulated_shards(lrk_ctx* ctx, int nshard);
int lrk_profile_enable(lrk_ctx* ctx, int enable);
int lrk_profile_read(lrk_ctx* ctx, double* sweep_ms, int64_t* sweep_launches,
                     double* sweep_alg_bytes, int reset);
/* Rank traces of the last Hessian apply: forward and adjoint sweeps (pane
 * rank after every flush + final) and the observation rank. */
int lrk_last_traces(lrk_ctx* ctx, int* fwd, int* bwd, int cap, int* n_fwd,
                    int* n_bwd, int* obs_rank);

#ifdef __cplusplus
}
#endif
#endif /* LRK_H_ */
