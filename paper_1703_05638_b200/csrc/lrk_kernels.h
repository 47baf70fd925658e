// lrk_kernels.h — host-visible kernel argument blocks and launchers.
#pragma once
#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

namespace lrk {

// One low-rank sweep (forward.py:133-188) in the operator's eigenbasis.
constexpr int SHARD_MAX = 8;

struct SweepArgs {
  int64_t n_x;
  int n_t;
  int adjoint;
  int p;            // compress_every
  int r_max;        // < 0: none
  double eps0;
  double ftz;              // |y| below this is flushed to zero (0 = off)
  const double* theta;     // n_x: eigenvalues of S^{-1} M
  const double* rowscale;  // n_x or NULL: B~ = rowscale .* B
  const double* B;         // n_x x rb (rhs spatial factor, eigenbasis)
  int64_t ldb;
  int rb;
  const int* rb_dev;       // optional device rank of the rhs (rb = min(rb, *rb_dev))
  const double* W2;        // n_t x rb (rhs time factor)
  int64_t ldw2;
  double* U0; double* U1; int64_t ldu;   // ping-pong pane bases, n_x x ucap
  double* V0; double* V1; int64_t ldv;   // ping-pong time bases, n_t x ucap
  int ucap;
  double* sigma;           // ucap, output singular values
  int* info;               // [0]=final rank, [1]=which buffer, [2]=error code
  int* trace;              // nflush+1 ranks
  double* ybuf; int64_t ldy;   // n_x x p
  double* qbuf; int64_t ldq;   // n_x x p
  double* yprev;               // n_x
  double* part; int64_t pstride;  // 3 * ncta * pstride
  double* scratch; int64_t scratch_stride;  // per-CTA
  unsigned* bar;           // 2 unsigned per group
  int ncta;
  long long* dbg;          // optional per-phase cycle counters (10), CTA 0
  double* cdump;           // optional (LRK_DUMP_CORES): per flush [n, core 32x33] from CTA 0
  int nopipe;              // 1: no overlap of the next flush's phase 1 with the Jacobi (LRK_NOPIPE)
  // external-trajectory mode (physical-space solvers, e.g. convection-diffusion):
  // when yext != NULL the buffered columns are read from yext (column j = the
  // j-th step processed by this launch) instead of the spectral recurrence.
  const double* yext; int64_t ldyext;
  // n_x sharding: nshard groups (one per GPU, or emulated as
  // groups of one launch) form ONE logical sweep; global CTA = shard*ncta + cta
  // owns rows row_range(n_x, gcta, nshard*ncta); partials of shard s live at
  // spart[s] (peer memory across GPUs), all CTAs meet at the shared counter
  // gbar; sys_fence selects system-scope fences (peer GPUs).  nshard <= 1:
  // spart[0] = part, gbar = bar.
  int nshard, shard, sys_fence;
  double* spart[SHARD_MAX];
  unsigned* gbar;
  // chunked execution: flushes [flush0, flush1) of the full schedule, resuming
  // from a pane of rank r_init held in U0 / V0 / sigma (r_init < 0: the rank
  // the previous chunk left in info[0]; every chunk must contain a flush)
  int flush0, flush1, r_init;
  // shared-memory plan (offsets in doubles, computed by sweep_plan)
  int resident;            // 1: CTA row blocks of U/Y/Q~ live in shared memory
  int mp;                  // padded rows per CTA (leading dim of resident blocks)
  int tp;                  // padded time rows per CTA (resident V block)
  int off_V, off_U, off_Y, off_Q, off_yp, off_th, off_rs;
  int off_small, off_scr;  // small matrices; phase-4 scratch (stack QR / Jacobi)
  int stack_smem;          // stacked-R QR in shared memory
  int smem_doubles;
};

// Shared-memory plan for a sweep over n_x rows with ncta CTAs per group.
void sweep_plan(SweepArgs& a, int64_t n_x, int ncta, int ucap, int p, size_t smem_limit,
                int nshard = 1);

// Independent sweeps launched together, one group of ncta CTAs each (passed
// by value as a __grid_constant__ kernel parameter: no host->device copy).
constexpr int SWEEP_MAXG = 16;
struct SweepBatch {
  SweepArgs g[SWEEP_MAXG];
  int ngroups;
};

size_t sweep_smem_bytes();
int64_t sweep_scratch_stride(int ncta);
int64_t sweep_part_stride();
cudaError_t launch_sweep(const SweepBatch& batch, cudaStream_t s);

// General lr_truncate (lowrank.py:124-144) of W1 (n_x x R) W2^T (n_t x R).
struct TruncArgs {
  int64_t n_x;
  int n_t;
  int R;
  const int* R_dev;  // optional device column count (R = min(R, *R_dev))
  int flags;         // LRK_TRUNC_* bits
  int r_max;
  double eps0;
  const double* W1; int64_t ld1;
  const double* W2; int64_t ld2;
  double* Q1; int64_t ldq1;   // workspace n_x x R
  double* Q2; int64_t ldq2;   // workspace n_t x R
  double* tmpw; int64_t ldtmp;  // workspace max(n_x,n_t) x PMAX
  double* out1; int64_t ldo1; // n_x x cap
  double* out2; int64_t ldo2; // n_t x cap
  int cap;
  double* sigma;              // cap (output singular values), may be NULL
  double* sv_all;             // all R singular values (may be NULL)
  int* info;                  // [0]=rank, [2]=error
  double* part; int64_t pstride;
  double* scratch; int64_t scratch_stride;
  unsigned* bar;
  int ncta;
  int no_flip;                // skip _svd_flip
};
size_t trunc_smem_bytes();
int64_t trunc_scratch_stride(int ncta);
int64_t trunc_part_stride();
cudaError_t launch_truncate(const TruncArgs& args, cudaStream_t s);

// fp64 batched GEMM: C[b] = alpha * A[b] B[b] + beta * C[b], all row-major.
struct GemmArgs {
  int M, N, K;
  const double* A; int64_t lda; int64_t sA;
  const double* B; int64_t ldb; int64_t sB;
  double* C; int64_t ldc; int64_t sC;
  double alpha, beta;
  int batch;
  const int* batch_dev;    // optional: batch = min(batch, *batch_dev * batch_mult)
  int batch_mult;
  const int* m_dev;        // optional: M = min(M, *m_dev * m_mult)
  int m_mult;
  const double* emul;      // optional epilogue: C = alpha * (A B) .* E + beta * C, E[row*lde + col]
  int64_t lde;
};
cudaError_t launch_gemm(const GemmArgs& g, cudaStream_t s);

}  // namespace lrk
