// lrk_sflush.h — launcher interface of the streaming-flush sweep (lrk_sflush.cu).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

namespace lrk {

// Streaming-flush sweep (lrk_sflush.cu): the large-n_x form of the sweep,
// one kernel per row pass, flush width <= 4, pane rank <= 64.
constexpr int SF_CAP = 64;
constexpr int SF_P = 4;
constexpr int SF_N = SF_CAP + SF_P;
constexpr int SF_LDW = 68;

// Small per-sweep state in global memory (written by the last CTA of each
// pass and by sf_finish, read by the next pass).
struct SFState {
  int r;         // valid pane columns of U (after the last applied update)
  int rn;        // pane rank of the pending update
  int pcp;       // width of the remainder block next to U (X = [U, y])
  int pending;   // an update (Wp, Vc) is pending
  int startp;    // flush start of the pending update (time-row selection)
  int drop_all;  // the current remainder is at the rounding floor
  int pc_new;    // width of the flush being projected (Yn)
  int pad;
  double sig[SF_N];
  double C[SF_CAP * SF_P];   // C1 (+ P2) of the flush being orthogonalised, [i * SF_P + s]
  double P2[SF_CAP * SF_P];
  double M[SF_N * SF_P];     // [U, y2]^T Yn of the next flush, [k * SF_P + s]
  double Wd[SF_N * SF_P];    // -Wp C1: y1 = Yn + [U, y2] Wd, [k * SF_P + s]
  double G0[16];             // remainder Gram y2^T y2 (row-major 4x4), input of the shifted Cholesky
  double yn[SF_P];           // |Y_s|^2 of the flush being orthogonalised
  double yn_next[SF_P];      // ... of the flush being projected
  double Rc[16];             // remainder R (row-major 4x4)
  double Rinv[16];           // Q = y2 Rinv
  double Wp[SF_N * SF_LDW];  // pending spatial update (n x rn), col-major
  double Vc[SF_N * SF_LDW];  // pending time update (n x rn), col-major
};

// n_x-sharded sweeps: every pass ends in a small rank total (projection or
// Gram block) that all shards need summed.  Each shard owns one SFXBuf; the
// last CTA of a pass stores its total into slot [seq & 1][shard] of EVERY
// shard's buffer (peer-mapped over NVLink, or the same device under
// emulation) and then releases flag[seq & 1][shard] = seq at system scope; a
// one-CTA tail kernel acquires the flags of all shards and sums the slots in
// shard order, so every shard takes bit-identical decisions.
constexpr int SF_XMAXR = 8;
constexpr int SF_XLEN = 304;
struct SFXBuf {
  double data[2][SF_XMAXR][SF_XLEN];
  unsigned long long flag[2][SF_XMAXR];
};

struct SFArgs {
  int64_t n_x;           // rows of this shard
  int64_t n_x_glob;      // rows of the whole (unsharded) field
  int nshard, shard;     // n_x shards (1: unsharded) and this shard's index
  SFXBuf* xpeer[SF_XMAXR];  // exchange buffer of every shard ([shard] = own)
  int n_t, p, cap, adjoint, r_max, nflush;
  double eps0, ftz;
  double* U; int64_t ldu;
  double* V; int64_t ldv;
  double* Yg[3]; int64_t ldy;   // flush f lives in Yg[f % 3]
  double* yprev;
  const double* theta;
  const double* rowscale;
  const double* B; int64_t ldb; int rb;
  const int* rb_dev;
  const double* W2; int64_t ldw2;
  double* part;          // G * sf_part_stride() doubles
  unsigned* ticket;      // 8 counters (zero)
  SFState* st;
  int* trace; int* info; double* sigma;
  int G;                 // CTAs of the staged row passes
  int Ggen;              // CTAs of the light grid-stride passes
  int dbg_print;         // LRK_SF_DEBUG: flushes to report (diagnostics)
  int smem_pass;         // dynamic shared memory of the staged passes (bytes)
  long long* dbg;        // LRK_SF_TIMING: cycle sums of the last-CTA tails (diagnostics), else null
};
size_t sf_smem_pass();
int64_t sf_part_stride();
// aux: a second (non-blocking) stream + two events, used to run the next
// flush's column generation under the single-CTA core SVD.
struct SFAux {
  cudaStream_t stream;
  cudaEvent_t ready, done;
};
// `sh`: the nlocal shards this process drives (1 in production: one process
// per GPU; all of them under single-device emulation, launched pass by pass
// so that no kernel ever waits for a later launch).  xseq: the context's
// exchange sequence counter (advanced by the number of exchanges).
cudaError_t launch_sweep_stream(const SFArgs* sh, int nlocal, int nflush, cudaStream_t s,
                                const SFAux& aux, unsigned long long* xseq, int64_t* launches);

// Sharded sweeps: push this rank's rows [x0, x0 + rows) of its pane (the first
// min(cap, info[0]) columns) into every peer's pane, then a flag barrier.
cudaError_t sf_allgather_pane(const SFArgs& a, double* const* pane, int64_t ld, int64_t x0, int64_t rows,
                              int cap, cudaStream_t s, unsigned long long* xseq, int64_t* launches);

}  // namespace lrk
