// lrk_sflush.cu — the streaming-flush sweep for large n_x (C4/C5 sizes).
//
// Same mathematics as the persistent sweep_kernel (lrk_sweep.cu) and the
// reference's flush (forward.py:165-177 = lr_truncate(lr_add(pane, buffered
// columns)), lowrank.py:124-144): the pane U diag(s) V^T is canonical, so the
// truncation of [U, Y] is an incremental SVD,
//     QR([U, Y]) = [U, Q~] [[I, C], [0, R~]],   core = [[diag(s), C], [0, R~]],
// with C from block CGS2 against U and (Q~, R~) a QR of the remainder.  What
// differs is the organisation, built for HBM streaming when the CTA row blocks
// cannot stay resident in shared memory:
//
//   sf_update_project  U' = [U, y2] W' (the PREVIOUS flush's basis update,
//                      the remainder's transform folded into W'), V' likewise
//                      on the time rows; M = [U, y2]^T Y for the new columns
//                      (P1 = W'^T M) and |Y|^2                 -> C1
//   sf_generate        the next flush's columns y_k = theta y_{k-1} + B~ w2_k
//   sf_sub_project     y1 = Y - U C1, P2 = U^T y1              -> C = C1 + P2
//   sf_sub_gram        y2 = y1 - U P2, G0 = y2^T y2            -> shifted Cholesky R0
//   sf_cholqr (x2)     G = (y2 R^-1)^T (y2 R^-1)               -> R <- chol(G) R
//                      (shifted CholeskyQR3 of the 4-column remainder, pivoted
//                      and drop-tolerant for numerically rank-deficient
//                      remainders), then on the last pass the flush's small
//                      algebra in one CTA: the rank-revealing fix-up with the
//                      rounding-floor drop of the persistent kernel, the core
//                      SVD (register Jacobi), _rank_cut (lowrank.py:98-111)
//                      and the update matrices W' for the next launch.
//
// Each kernel streams its CTA's contiguous rows in 64-row chunks through a
// cp.async ring (16-byte copies, four stages in flight), runs the row x small
// products on the FP64 tensor pipe (DMMA m8n8k4) from shared memory, writes a
// CTA partial and the LAST CTA to finish (atomic ticket) reduces the partials
// in CTA order — deterministic, no grid barrier, no cooperative launch.  Per
// flush the pane basis U is read three times and written once (the persistent
// kernel read it four times and streamed it at ~1/3 of the HBM share).
#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include "lrk_device.cuh"
#include "lrk_kernels.h"
#include "lrk_small.cuh"

namespace lrk {

namespace {

constexpr int ST = 256;           // threads per CTA
constexpr int TR = 64;            // rows per staged chunk
constexpr int LDX = 68;           // shared leading dimension (== 4 mod 16: conflict-free fragments)
constexpr int NSTAGE = 4;         // cp.async ring depth
constexpr int PSTR = SF_N * SF_P + SF_P + 8;  // per-CTA partial stride (doubles)

__device__ __forceinline__ void cp16(void* smem, const void* gmem, bool valid) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  const int sz = valid ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(sz));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

// Stage rows [i0, i0 + TR) of `ncols` columns into shared memory (column c at
// dst + c * LDX); column c comes from src(c) (a global column pointer, 16-byte
// aligned, n_x even).  Rows >= nrows are zero-filled.
template <typename ColFn>
__device__ __forceinline__ void stage_cols(double* dst, int ncols, ColFn src, int64_t i0,
                                           int64_t nrows) {
  constexpr int PER = TR / 2;  // 16-byte pieces per column
  for (int idx = threadIdx.x; idx < ncols * PER; idx += ST) {
    const int c = idx / PER, k = idx - c * PER;
    const int64_t row = i0 + 2 * k;
    const bool ok = row < nrows;
    const double* g = src(c) + (ok ? row : 0);
    cp16(dst + c * LDX + 2 * k, g, ok);
  }
}

// Rows of this CTA: whole chunks [c0, c1) of the 64-row chunk grid.
__device__ __forceinline__ void cta_chunks(int64_t n_x, int& c0, int& c1) {
  const int nch = (int)((n_x + TR - 1) / TR);
  const int per = (nch + gridDim.x - 1) / gridDim.x;
  c0 = min(nch, (int)blockIdx.x * per);
  c1 = min(nch, c0 + per);
}

// Block-wide sum of K per-thread values into out (shared), fixed order.
template <int K>
__device__ __forceinline__ void cta_sum(double (&v)[K], double* red, double* out) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
  for (int k = 0; k < K; ++k) v[k] = warp_sum(v[k]);
  if (lane == 0)
#pragma unroll
    for (int k = 0; k < K; ++k) red[w * K + k] = v[k];
  __syncthreads();
  if (threadIdx.x < K) {
    double s = 0.0;
    for (int ww = 0; ww < ST / 32; ++ww) s += red[ww * K + threadIdx.x];
    out[threadIdx.x] = s;
  }
  __syncthreads();
}

// Last-CTA election: every CTA has written its partial; returns true in the
// CTA that arrived last (which then sees all partials).
__device__ __forceinline__ bool last_cta(unsigned* ticket, int* flag) {
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned t = atomicAdd(ticket, 1u);
    *flag = (t == gridDim.x - 1) ? 1 : 0;
  }
  __syncthreads();
  if (*flag) {
    __threadfence();
    if (threadIdx.x == 0) *ticket = 0u;  // ready for the next launch
  }
  return *flag != 0;
}

// out[e] = sum over CTAs (in order) of part[c * PSTR + e], e < len
__device__ __forceinline__ void reduce_parts(const double* part, int len, double* out) {
  for (int e = threadIdx.x; e < len; e += ST) {
    double s = 0.0;
    for (int c = 0; c < (int)gridDim.x; ++c) s += __ldcg(part + (int64_t)c * PSTR + e);
    out[e] = s;
  }
  __syncthreads();
}

// C = A B for row-major 4x4 blocks restricted to n x n (zero outside); one
// thread, fully unrolled (register resident).
__device__ __forceinline__ void mat4_mul(const double* A, const double* B, double* C, int n) {
  double T[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      double s = 0.0;
#pragma unroll
      for (int k = 0; k < 4; ++k)
        if (k < n) s = fma(A[i * 4 + k], B[k * 4 + j], s);
      T[i][j] = (i < n && j < n) ? s : 0.0;
    }
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) C[i * 4 + j] = T[i][j];
}

// Pivoted, drop-tolerant Cholesky of the n x n SPD-ish G (row-major 4x4):
// P^T G P = L L^T on the kept pivots (pivot > tol * first pivot).  Returns
// R (rows = kept directions, zero elsewhere) with G ~ R^T R and Z with
// (Q Z)^T (Q Z) ~ I on the kept columns (Z = P L^{-T}, dropped columns 0).
// Fully unrolled with compile-time indices (register resident: no dynamically
// indexed local arrays; the pivot swap is a select per entry).
__device__ __forceinline__ int pivoted_chol4(const double* G, int n, double tol, double* R,
                                             double* Z) {
  double A[4][4], L[4][4];
  int perm[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    perm[i] = i;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      A[i][j] = (i < n && j < n) ? G[i * 4 + j] : 0.0;
      L[i][j] = 0.0;
    }
  }
  int kept = 0;
  bool stop = false;
  double d0 = 0.0;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    if (k >= n || stop) continue;
    // pivot: largest remaining diagonal (first on ties)
    int piv = k;
    double best = A[k][k];
#pragma unroll
    for (int i = k + 1; i < 4; ++i)
      if (i < n && A[i][i] > best) { best = A[i][i]; piv = i; }
    // symmetric swap k <-> piv of A, rows of L, perm (selects)
#pragma unroll
    for (int i = k + 1; i < 4; ++i) {
      if (i != piv) continue;
#pragma unroll
      for (int j = 0; j < 4; ++j) { const double t = A[k][j]; A[k][j] = A[i][j]; A[i][j] = t; }
#pragma unroll
      for (int j = 0; j < 4; ++j) { const double t = A[j][k]; A[j][k] = A[j][i]; A[j][i] = t; }
#pragma unroll
      for (int j = 0; j < 4; ++j) { const double t = L[k][j]; L[k][j] = L[i][j]; L[i][j] = t; }
      const int t = perm[k]; perm[k] = perm[i]; perm[i] = t;
    }
    const double d = A[k][k];
    if (k == 0) d0 = d;
    if (!(d > tol * d0) || !(d > 0.0)) { stop = true; continue; }
    const double l = sqrt(d);
    L[k][k] = l;
#pragma unroll
    for (int i = k + 1; i < 4; ++i) L[i][k] = (i < n) ? A[i][k] / l : 0.0;
#pragma unroll
    for (int i = k + 1; i < 4; ++i)
#pragma unroll
      for (int j = k + 1; j < 4; ++j) A[i][j] -= L[i][k] * L[j][k];
    kept = k + 1;
  }
  // Li = L^{-1} on the kept block (lower triangular)
  double Li[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) Li[i][j] = 0.0;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    if (i >= kept) continue;
    Li[i][i] = 1.0 / L[i][i];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      if (j >= i) continue;
      double s = 0.0;
#pragma unroll
      for (int q = 0; q < 4; ++q)
        if (q >= j && q < i) s += L[i][q] * Li[q][j];
      Li[i][j] = -s / L[i][i];
    }
  }
  // R[a][c] = L[j][a] with perm[j] == c (j >= a); Z[c][a] = Li[a][j] with perm[j] == c
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      double rv = 0.0, zv = 0.0;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const bool hit = perm[j] == c && a < kept && j < n;
        if (hit && j >= a) rv = L[j][a];
        if (hit && j < kept && a >= j) zv = Li[a][j];
      }
      R[a * 4 + c] = rv;
      Z[c * 4 + a] = zv;
    }
  return kept;
}

}  // namespace

// --------------------------------------------------------------- update + project
// Pending update (st->pending): U'[:, :rn] = [U[:, :r], y2] Wp, V' likewise;
// then (unless final) M = [U', ...] handled as P1 = Wp^T ([U, y2]^T Y).
__global__ void __launch_bounds__(ST, 1) sf_update_project(const SFArgs a, int f, int final_only) {
  extern __shared__ double smem[];
  SFState* st = a.st;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int r = st->r;
  const bool pend = st->pending != 0;
  const int pcp = pend ? st->pcp : 0;
  const int n = r + pcp;                      // columns of X = [U, y2]
  const int rn = pend ? st->rn : r;           // columns of U'
  const int start = f * a.p;
  const int pc = final_only ? 0 : min(a.p, a.n_t - start);
  const double* Ycur = a.Yg[f & 1];
  const double* Y2 = a.Yg[(f + 1) & 1];       // the previous flush's remainder
  double* W = smem;                           // SF_N x LDX (Wp, col-major by output column)
  double* stage = W + SF_N * LDX;
  const int xcols = SF_CAP + SF_P;            // X region columns per stage
  const int scols = xcols + SF_P;             // + Y columns
  int* flag = reinterpret_cast<int*>(stage + NSTAGE * scols * LDX);
  double* red = stage;                        // reused after the main loop

  if (pend) {
    for (int idx = tid; idx < n * rn; idx += ST) {
      const int k = idx % n, c = idx / n;
      W[c * LDX + k] = st->Wp[k + c * SF_LDW];
    }
    // time rows of this CTA: V' = [V, E] Vc   (in place, via shared memory)
    const int64_t tper = ((int64_t)a.n_t + gridDim.x - 1) / gridDim.x;
    const int64_t nt64 = a.n_t;
    const int64_t t0 = min(nt64, (int64_t)blockIdx.x * tper), t1 = min(nt64, t0 + tper);
    const int nrow = (int)(t1 - t0);
    double* Vs = stage;  // nrow x r
    double* Vc = stage + nrow * SF_CAP + 8;
    for (int idx = tid; idx < n * rn; idx += ST) Vc[idx] = st->Vc[(idx % n) + (idx / n) * SF_LDW];
    for (int idx = tid; idx < nrow * r; idx += ST)
      Vs[idx] = a.V[(t0 + idx % nrow) + (int64_t)(idx / nrow) * a.ldv];
    __syncthreads();
    const int sp = st->startp;
    for (int idx = tid; idx < nrow * rn; idx += ST) {
      const int tl = idx % nrow, c = idx / nrow;
      const int64_t tt = t0 + tl;
      const int sel = a.adjoint ? (a.n_t - 1 - sp) - (int)tt : (int)tt - sp;
      double acc = (sel >= 0 && sel < pcp) ? Vc[(r + sel) + c * n] : 0.0;
      for (int k = 0; k < r; ++k) acc += Vs[tl + k * nrow] * Vc[k + c * n];
      a.V[tt + (int64_t)c * a.ldv] = acc;
    }
    __syncthreads();
  }

  int c0, c1;
  cta_chunks(a.n_x, c0, c1);
  const int nk = (n + 3) >> 2, nj = (rn + 7) >> 3;
  const double* U = a.U;
  auto issue = [&](int ch) {
    if (ch < c1) {
      double* s = stage + ((ch - c0) % NSTAGE) * scols * LDX;
      const int64_t i0 = (int64_t)ch * TR;
      stage_cols(s, n, [&](int c) { return c < r ? U + (int64_t)c * a.ldu : Y2 + (int64_t)(c - r) * a.ldy; },
                 i0, a.n_x);
      if (pc > 0) stage_cols(s + xcols * LDX, pc, [&](int c) { return Ycur + (int64_t)c * a.ldy; }, i0, a.n_x);
    }
    cp_commit();
  };
  // projection accumulators: M rows (X columns) 8*warp + g (and 64 + g on warp 0)
  double m0[2] = {0.0, 0.0}, m1[2] = {0.0, 0.0};
  double ysq = 0.0;
  const bool do_upd = pend && rn > 0 && n > 0;
  for (int s = 0; s < NSTAGE - 1; ++s) issue(c0 + s);
  for (int ch = c0; ch < c1; ++ch) {
    cp_wait<NSTAGE - 2>();
    __syncthreads();
    issue(ch + NSTAGE - 1);
    const double* X = stage + ((ch - c0) % NSTAGE) * scols * LDX;
    const double* Yt = X + xcols * LDX;
    const int64_t i0 = (int64_t)ch * TR;
    if (do_upd) {
      // U' rows of tile `warp`: acc[j] = X[8w.., :] W[:, 8j..]
      double acc[8][2];
#pragma unroll
      for (int j = 0; j < 8; ++j) acc[j][0] = acc[j][1] = 0.0;
      for (int kk = 0; kk < nk; ++kk) {
        const int k = 4 * kk + t;
        const double av = (k < n) ? X[k * LDX + 8 * warp + g] : 0.0;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          if (j >= nj) break;
          const double bv = (k < n && 8 * j + g < rn) ? W[(8 * j + g) * LDX + k] : 0.0;
          dmma884(acc[j][0], acc[j][1], av, bv);
        }
      }
      const int64_t row = i0 + 8 * warp + g;
      if (row < a.n_x) {
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          if (j >= nj) break;
          const int c = 8 * j + 2 * t;
          if (c < rn) a.U[row + (int64_t)c * a.ldu] = acc[j][0];
          if (c + 1 < rn) a.U[row + (int64_t)(c + 1) * a.ldu] = acc[j][1];
        }
      }
    }
    if (pc > 0) {
      // M += X^T Y  (rows = X columns, k = chunk rows)
      if (8 * warp < n) {
#pragma unroll 4
        for (int kk = 0; kk < TR / 4; ++kk) {
          const double av = X[(8 * warp + g) * LDX + 4 * kk + t];
          const double bv = (g < pc) ? Yt[g * LDX + 4 * kk + t] : 0.0;
          dmma884(m0[0], m0[1], av, bv);
        }
      }
      if (warp == 0 && n > 64) {
#pragma unroll 4
        for (int kk = 0; kk < TR / 4; ++kk) {
          const double av = (64 + g < n) ? X[(64 + g) * LDX + 4 * kk + t] : 0.0;
          const double bv = (g < pc) ? Yt[g * LDX + 4 * kk + t] : 0.0;
          dmma884(m1[0], m1[1], av, bv);
        }
      }
      if (tid < TR * pc) {
        const double y = Yt[(tid / TR) * LDX + (tid % TR)];
        ysq += y * y;
      }
    }
  }
  cp_wait<0>();
  __syncthreads();
  // ---- CTA partial: M (n x pc, row-major), then |Y_s|^2
  double* part = a.part + (int64_t)blockIdx.x * PSTR;
  if (pc > 0) {
    const int row = 8 * warp + g;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int c = 2 * t + h;
      if (row < n && c < pc) part[row * pc + c] = m0[h];
      if (warp == 0 && 64 + g < n && c < pc) part[(64 + g) * pc + c] = m1[h];
    }
    // ysq: thread tid covers column tid / TR
    double v[SF_P];
#pragma unroll
    for (int s = 0; s < SF_P; ++s) v[s] = (tid < TR * pc && tid / TR == s) ? ysq : 0.0;
    double* outv = red + 8 * SF_P;
    cta_sum<SF_P>(v, red, outv);
    if (tid < pc) part[n * pc + tid] = outv[tid];
  }
  if (!last_cta(a.ticket + 0, flag)) return;
  // ---- last CTA: P1 = Wp^T M (or M), pane bookkeeping
  double* tot = red + 64;
  reduce_parts(a.part, n * pc + pc, tot);
  if (pc > 0) {
    for (int idx = tid; idx < rn * pc; idx += ST) {
      const int i = idx / pc, s = idx % pc;
      double acc = 0.0;
      if (pend) {
        for (int k = 0; k < n; ++k) acc += W[i * LDX + k] * tot[k * pc + s];
      } else {
        acc = tot[i * pc + s];
      }
      st->C[i * SF_P + s] = acc;
    }
    if (tid < pc) st->yn[tid] = tot[n * pc + tid];
  }
  __syncthreads();
  if (tid == 0) {
    st->r = rn;
    st->pending = 0;
    st->pc = pc;
    if (final_only) {
      a.info[0] = rn;
      a.trace[a.nflush] = rn;
    }
  }
  if (final_only)
    for (int k = tid; k < rn; k += ST) a.sigma[k] = st->sig[k];
}

// ------------------------------------------------------------ generation
// The next flush's buffered columns (forward.py:180 in the DST eigenbasis):
// y_k = theta .* y_{k-1} + rowscale .* (B w2_k), k = the flush's steps.
__global__ void __launch_bounds__(ST) sf_generate(const SFArgs a, int f) {
  __shared__ double w2s[SF_CAP * SF_P];
  const int start = f * a.p;
  const int pc = min(a.p, a.n_t - start);
  const int rb = a.rb_dev ? min(a.rb, *a.rb_dev) : a.rb;
  for (int idx = threadIdx.x; idx < rb * pc; idx += ST) {
    const int j = idx / pc, s = idx % pc;
    const int k = a.adjoint ? (a.n_t - 1 - (start + s)) : (start + s);
    w2s[j * SF_P + s] = a.W2[k + (int64_t)j * a.ldw2];
  }
  __syncthreads();
  double* Y = a.Yg[f & 1];
  for (int64_t i = (int64_t)blockIdx.x * ST + threadIdx.x; i < a.n_x; i += (int64_t)gridDim.x * ST) {
    double acc[SF_P] = {0.0, 0.0, 0.0, 0.0};
    int j = 0;
    for (; j + 4 <= rb; j += 4) {
      double b[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) b[u] = a.B[i + (int64_t)(j + u) * a.ldb];
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int s = 0; s < SF_P; ++s) acc[s] += b[u] * w2s[(j + u) * SF_P + s];
    }
    for (; j < rb; ++j) {
      const double b = a.B[i + (int64_t)j * a.ldb];
#pragma unroll
      for (int s = 0; s < SF_P; ++s) acc[s] += b * w2s[j * SF_P + s];
    }
    const double tv = a.theta[i];
    const double rs = a.rowscale ? a.rowscale[i] : 1.0;
    double y = a.yprev[i];
#pragma unroll
    for (int s = 0; s < SF_P; ++s) {
      if (s < pc) {
        y = tv * y + rs * acc[s];
        if (fabs(y) < a.ftz) y = 0.0;
        Y[i + (int64_t)s * a.ldy] = y;
      }
    }
    a.yprev[i] = y;
  }
}

// ------------------------------------------------------- CGS subtractions
// mode 0: y1 = Y - U C1 (in place), P2 = U^T y1          -> C += P2
// mode 1: y2 = y1 - U P2 (in place), G0 = y2^T y2        -> shifted Cholesky
__global__ void __launch_bounds__(ST, 1) sf_subtract(const SFArgs a, int f, int mode) {
  extern __shared__ double smem[];
  SFState* st = a.st;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int r = st->r;
  const int pc = st->pc;
  double* Ybuf = a.Yg[f & 1];
  double* Cs = smem;                           // r x SF_P (row-major)
  double* stage = Cs + SF_CAP * SF_P + 8;
  const int scols = SF_CAP + SF_P;
  int* flag = reinterpret_cast<int*>(stage + NSTAGE * scols * LDX);
  double* red = stage;
  const double* Csrc = mode == 0 ? st->C : st->P2;
  for (int idx = tid; idx < r * SF_P; idx += ST) Cs[idx] = Csrc[idx];
  __syncthreads();
  int c0, c1;
  cta_chunks(a.n_x, c0, c1);
  const int nk = (r + 3) >> 2;
  auto issue = [&](int ch) {
    if (ch < c1) {
      double* s = stage + ((ch - c0) % NSTAGE) * scols * LDX;
      const int64_t i0 = (int64_t)ch * TR;
      stage_cols(s, r, [&](int c) { return a.U + (int64_t)c * a.ldu; }, i0, a.n_x);
      stage_cols(s + SF_CAP * LDX, pc, [&](int c) { return Ybuf + (int64_t)c * a.ldy; }, i0, a.n_x);
    }
    cp_commit();
  };
  double p2[2] = {0.0, 0.0};   // mode 0: P2 rows 8*warp + g (U columns)
  double gacc[10] = {};        // mode 1: upper triangle of y2^T y2 (thread = row)
  for (int s = 0; s < NSTAGE - 1; ++s) issue(c0 + s);
  for (int ch = c0; ch < c1; ++ch) {
    cp_wait<NSTAGE - 2>();
    __syncthreads();
    issue(ch + NSTAGE - 1);
    double* X = stage + ((ch - c0) % NSTAGE) * scols * LDX;
    double* Yt = X + SF_CAP * LDX;
    const int64_t i0 = (int64_t)ch * TR;
    // D = U_tile C  (rows 8*warp.., cols 0..pc)
    double d0 = 0.0, d1 = 0.0, e0 = 0.0, e1 = 0.0;
    for (int kk = 0; kk < nk; ++kk) {
      const int k = 4 * kk + t;
      const double av = (k < r) ? X[k * LDX + 8 * warp + g] : 0.0;
      const double bv = (k < r && g < pc) ? Cs[k * SF_P + g] : 0.0;
      if (kk & 1) dmma884(e0, e1, av, bv);
      else dmma884(d0, d1, av, bv);
    }
    d0 += e0;
    d1 += e1;
    {
      const int row = 8 * warp + g;
      const int64_t grow = i0 + row;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int c = 2 * t + h;
        if (c < pc) {
          const double y = Yt[c * LDX + row] - (h ? d1 : d0);
          Yt[c * LDX + row] = y;
          if (grow < a.n_x) Ybuf[grow + (int64_t)c * a.ldy] = y;
        }
      }
    }
    __syncthreads();
    if (mode == 0) {
      if (8 * warp < r) {
#pragma unroll 4
        for (int kk = 0; kk < TR / 4; ++kk) {
          const double av = X[(8 * warp + g) * LDX + 4 * kk + t];
          const double bv = (g < pc) ? Yt[g * LDX + 4 * kk + t] : 0.0;
          dmma884(p2[0], p2[1], av, bv);
        }
      }
    } else if (tid < TR) {
      double y[SF_P];
#pragma unroll
      for (int s = 0; s < SF_P; ++s) y[s] = s < pc ? Yt[s * LDX + tid] : 0.0;
      int q = 0;
#pragma unroll
      for (int u = 0; u < SF_P; ++u)
#pragma unroll
        for (int v = u; v < SF_P; ++v) gacc[q++] += y[u] * y[v];
    }
  }
  cp_wait<0>();
  __syncthreads();
  double* part = a.part + (int64_t)blockIdx.x * PSTR;
  int plen;
  if (mode == 0) {
    const int row = 8 * warp + g;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int c = 2 * t + h;
      if (row < r && c < pc) part[row * pc + c] = p2[h];
    }
    plen = r * pc;
  } else {
    double* outv = red + 8 * 10;
    cta_sum<10>(gacc, red, outv);
    if (tid < 10) part[tid] = outv[tid];
    plen = 10;
  }
  if (!last_cta(a.ticket + 1 + mode, flag)) return;
  double* tot = red + 256;
  reduce_parts(a.part, plen, tot);
  if (mode == 0) {
    for (int idx = tid; idx < r * pc; idx += ST) {
      const int i = idx / pc, s = idx % pc;
      st->P2[i * SF_P + s] = tot[idx];
      st->C[i * SF_P + s] += tot[idx];
    }
    return;
  }
  if (tid != 0) return;
  // shifted Cholesky of G0 (Fukaya et al. shifted CholeskyQR3, first step);
  // a remainder at the block's rounding floor 16 eps ||Y|| is dropped whole
  double G[16] = {};
  int q = 0;
  for (int u = 0; u < SF_P; ++u)
    for (int v = u; v < SF_P; ++v) {
      G[u * 4 + v] = G[v * 4 + u] = tot[q];
      ++q;
    }
  double tr = 0.0, ysq = 0.0;
  for (int s = 0; s < pc; ++s) { tr += G[s * 5]; ysq += st->yn[s]; }
  const double delta = 16.0 * DEPS * sqrt(ysq);
  st->drop_all = !(sqrt(tr) > delta);
  double R[16], Z[16];
  if (st->drop_all) {
    for (int i = 0; i < 16; ++i) { R[i] = 0.0; Z[i] = 0.0; }
  } else {
    const double shift = 11.0 * ((double)a.n_x * pc + pc * (pc + 1)) * DEPS * tr;
    for (int s = 0; s < pc; ++s) G[s * 5] += shift;
    pivoted_chol4(G, pc, 0.0, R, Z);
  }
  for (int i = 0; i < 16; ++i) { st->Rc[i] = R[i]; st->Rinv[i] = Z[i]; }
}

// ----------------------------------------------------------- CholeskyQR passes
// G = Q^T Q with Q = y2 Rinv; R <- chol(G) R, Rinv <- Rinv chol(G)^{-1}
// (pivoted, drop-tolerant).  Light streaming kernel (4 columns, L2-resident).
__global__ void __launch_bounds__(ST) sf_cholqr(const SFArgs a, int f, int pass) {
  SFState* st = a.st;
  __shared__ int flag;
  __shared__ double red[8 * 10 + 16];
  __shared__ double tot[16];
  const int tid = threadIdx.x;
  const int pc = st->pc;
  const bool skip = st->drop_all != 0;
  double gacc[10] = {};
  if (!skip) {
    double Ri[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) Ri[i] = st->Rinv[i];
    const double* Y = a.Yg[f & 1];
    for (int64_t i = (int64_t)blockIdx.x * ST + tid; i < a.n_x; i += (int64_t)gridDim.x * ST) {
      double y[SF_P], qv[SF_P];
#pragma unroll
      for (int s = 0; s < SF_P; ++s) y[s] = s < pc ? Y[i + (int64_t)s * a.ldy] : 0.0;
#pragma unroll
      for (int c = 0; c < SF_P; ++c) {
        double acc = 0.0;
#pragma unroll
        for (int s = 0; s < SF_P; ++s) acc += y[s] * Ri[s * 4 + c];
        qv[c] = acc;
      }
      int q = 0;
#pragma unroll
      for (int u = 0; u < SF_P; ++u)
#pragma unroll
        for (int v = u; v < SF_P; ++v) gacc[q++] += qv[u] * qv[v];
    }
  }
  double* outv = red + 8 * 10;
  cta_sum<10>(gacc, red, outv);
  double* part = a.part + (int64_t)blockIdx.x * PSTR;
  if (tid < 10) part[tid] = outv[tid];
  if (!last_cta(a.ticket + 3 + pass, &flag)) return;
  reduce_parts(a.part, 10, tot);
  if (tid == 0 && !skip) {
    double G[16] = {};
    int q = 0;
    for (int u = 0; u < SF_P; ++u)
      for (int v = u; v < SF_P; ++v) {
        G[u * 4 + v] = G[v * 4 + u] = tot[q];
        ++q;
      }
    double R1[16], Z1[16], Rc[16], Ri[16];
    // pivots below (1e-10)^2 of the leading one are rounding residue of a
    // numerically rank-deficient remainder: dropped (see header)
    pivoted_chol4(G, pc, 1e-20, R1, Z1);
    for (int i = 0; i < 16; ++i) { Rc[i] = st->Rc[i]; Ri[i] = st->Rinv[i]; }
    double Rn[16], Zn[16];
    mat4_mul(R1, Rc, Rn, pc);
    mat4_mul(Ri, Z1, Zn, pc);
    for (int i = 0; i < 16; ++i) { st->Rc[i] = Rn[i]; st->Rinv[i] = Zn[i]; }
  }
}

// The flush's small algebra (one CTA): rank-revealing fix-up of R, core
// assembly, core SVD, zero test and _rank_cut, update matrices for the next
// sf_update_project launch.
__global__ void __launch_bounds__(ST, 1) sf_finish(const SFArgs a, int f) {
  extern __shared__ double sm[];
  SFState* st = a.st;
  const int tid = threadIdx.x, warp = tid >> 5;
  const int r = st->r, pc = st->pc, n = r + pc;
  const int start = f * a.p;
  double* sT = sm;                // 16: y2 -> Q~ transform
  double* sR = sm + 16;           // 16: R~ (row-major 4x4)
  double* sS = sm + 32;           // SF_N singular values
  double* sScr = sS + SF_N + 4;   // 2*4*32 Jacobi exchange + scratch
  double* sCore = sScr + 512;     // 32 x 33 (n <= 32) or SF_N x SF_N (jacobi_svd)
  double* Uc = sCore + SF_N * SF_N + 8;   // n x n (ld n)
  double* Vc = Uc + SF_N * SF_N + 8;
  double* Vj = Vc + SF_N * SF_N + 8;
  int* iPerm = reinterpret_cast<int*>(Vj + SF_N * SF_N + 8);
  int* iFlag = iPerm + SF_N + 4;
  if (tid == 0) {
    double A[4][4], X[4][4];
    int pv[4];
    for (int i = 0; i < 4; ++i)
      for (int k = 0; k < 4; ++k) A[i][k] = (i < pc && k < pc) ? st->Rc[i * 4 + k] : 0.0;
    pivoted_qr_reg<4>(A, pc, X, pv);
    double ysq = 0.0;
    for (int s = 0; s < pc; ++s) ysq += st->yn[s];
    const double delta = 16.0 * DEPS * sqrt(ysq);
    for (int j = 0; j < 4; ++j)
      if (fabs(A[j][j]) <= delta || st->drop_all) {
        for (int k = 0; k < 4; ++k) { A[j][k] = 0.0; X[k][j] = 0.0; }
      }
    for (int i = 0; i < 16; ++i) sR[i] = 0.0;
    for (int j = 0; j < pc; ++j)
      for (int kk = 0; kk < pc; ++kk) sR[j * 4 + pv[kk]] = A[j][kk];
    // T = Rinv X  (q~ = y2 T)
    for (int i = 0; i < 4; ++i)
      for (int j = 0; j < 4; ++j) {
        double acc = 0.0;
        for (int k = 0; k < 4; ++k) acc += st->Rinv[i * 4 + k] * X[k][j];
        sT[i * 4 + j] = (i < pc && j < pc) ? acc : 0.0;
      }
  }
  __syncthreads();
  auto Kel = [&](int i, int j) -> double {
    if (i < r) return (j < r) ? (i == j ? st->sig[i] : 0.0) : st->C[i * SF_P + (j - r)];
    return (j >= r) ? sR[(i - r) * 4 + (j - r)] : 0.0;
  };
  const int ldc = n;
  if (n <= 32) {
    for (int idx = tid; idx < n * n; idx += ST) {
      const int i = idx % n, j = idx / n;
      sCore[j + i * 33] = Kel(i, j);  // K^T: Jacobi on the rows of the core
    }
    __syncthreads();
    if (warp < 4) {
      if (n <= 8) multi_warp_jacobi<8, 4>(sCore, 33, n, Vc, Uc, ldc, sS, iPerm, sScr);
      else if (n <= 12) multi_warp_jacobi<12, 4>(sCore, 33, n, Vc, Uc, ldc, sS, iPerm, sScr);
      else if (n <= 16) multi_warp_jacobi<16, 4>(sCore, 33, n, Vc, Uc, ldc, sS, iPerm, sScr);
      else if (n <= 20) multi_warp_jacobi<20, 4>(sCore, 33, n, Vc, Uc, ldc, sS, iPerm, sScr);
      else if (n <= 24) multi_warp_jacobi<24, 4>(sCore, 33, n, Vc, Uc, ldc, sS, iPerm, sScr);
      else multi_warp_jacobi<32, 4>(sCore, 33, n, Vc, Uc, ldc, sS, iPerm, sScr);
    }
    __syncthreads();
  } else {
    for (int idx = tid; idx < n * n; idx += ST) {
      const int i = idx % n, j = idx / n;
      sCore[i + j * n] = Kel(i, j);
    }
    __syncthreads();
    jacobi_svd(sCore, n, Vj, n, n, sS, iPerm, sScr, iFlag, sScr + SF_N + 8);
    for (int idx = tid; idx < n * n; idx += ST) {
      const int i = idx % n, k = idx / n;
      const double sv = sS[k];
      Uc[i + k * ldc] = sv > 0.0 ? sCore[i + iPerm[k] * n] / sv : 0.0;
      Vc[i + k * ldc] = Vj[i + iPerm[k] * n];
    }
    __syncthreads();
  }
  if (tid == 0) {
    double ysq = 0.0, ssq = 0.0;
    for (int s = 0; s < pc; ++s) ysq += st->yn[s];
    for (int i = 0; i < r; ++i) ssq += st->sig[i] * st->sig[i];
    const double fs = sqrt((double)r + ysq) * sqrt(ssq + (double)pc);
    int rn = (sS[0] <= NOISE_FLOOR * fs) ? 0 : rank_cut_dev(sS, n, a.eps0, a.r_max);
    if (rn > a.cap) { rn = a.cap; a.info[2] = 2; }
    iFlag[0] = rn;
  }
  __syncthreads();
  const int rn = iFlag[0];
  // W' = [Uc_top; T Uc_bot] (n x rn), Vc, singular values
  for (int idx = tid; idx < n * rn; idx += ST) {
    const int i = idx % n, c = idx / n;
    double w;
    if (i < r) {
      w = Uc[i + c * ldc];
    } else {
      w = 0.0;
      for (int q = 0; q < pc; ++q) w += sT[(i - r) * 4 + q] * Uc[r + q + c * ldc];
    }
    st->Wp[i + c * SF_LDW] = w;
    st->Vc[i + c * SF_LDW] = Vc[i + c * ldc];
  }
  for (int k = tid; k < rn; k += ST) st->sig[k] = sS[k];
  if (tid == 0) {
    st->rn = rn;
    st->pcp = pc;
    st->startp = start;
    st->pending = 1;
    a.trace[f] = rn;
  }
}

// ------------------------------------------------------------------ host side
size_t sf_smem_update() {
  return ((size_t)SF_N * LDX + (size_t)NSTAGE * (SF_CAP + 2 * SF_P) * LDX) * sizeof(double) + 64;
}
size_t sf_smem_subtract() {
  return ((size_t)SF_CAP * SF_P + 8 + (size_t)NSTAGE * (SF_CAP + SF_P) * LDX) * sizeof(double) + 64;
}
size_t sf_smem_finish() {
  return (size_t)(16 + 16 + SF_N + 4 + 512 + 4 * (SF_N * SF_N + 8) + 2 * SF_N + 16) * sizeof(double);
}
int64_t sf_part_stride() { return PSTR; }

cudaError_t sf_configure() {
  static bool done[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev >= 0 && dev < 64 && done[dev]) return cudaSuccess;
  cudaError_t e = cudaFuncSetAttribute(sf_update_project, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)sf_smem_update());
  if (e != cudaSuccess) return e;
  e = cudaFuncSetAttribute(sf_subtract, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)sf_smem_subtract());
  if (e != cudaSuccess) return e;
  e = cudaFuncSetAttribute(sf_finish, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)sf_smem_finish());
  if (e != cudaSuccess) return e;
  if (dev >= 0 && dev < 64) done[dev] = true;
  return cudaSuccess;
}

// The whole sweep: nflush x (update+project, generate, subtract, subtract,
// CholeskyQR x 2, finish) + one final update.  Returns the number of launches.
cudaError_t launch_sweep_stream(const SFArgs& a, int nflush, cudaStream_t s, int64_t* launches) {
  cudaError_t e = sf_configure();
  if (e != cudaSuccess) return e;
  const int G = a.G;
  const int Gg = a.Ggen;
  const size_t su = sf_smem_update(), ss = sf_smem_subtract(), sfin = sf_smem_finish();
  int64_t nl = 0;
  const int dbg = a.dbg_print;
  auto show = [&](const char* what, int f) {
    if (f >= dbg) return;
    SFState h;
    cudaStreamSynchronize(s);
    cudaMemcpy(&h, a.st, sizeof(h), cudaMemcpyDeviceToHost);
    std::fprintf(stderr, "[sf] f=%d %-8s r=%d rn=%d pc=%d pend=%d drop=%d err=%s | yn %.3e %.3e | C00 %.6e C01 %.6e P2_00 %.3e | sig %.6e %.6e | Rc %.4e %.4e %.4e %.4e\n",
                 f, what, h.r, h.rn, h.pc, h.pending, h.drop_all, cudaGetErrorString(cudaGetLastError()),
                 h.yn[0], h.yn[1], h.C[0], h.C[1], h.P2[0], h.sig[0], h.sig[1], h.Rc[0], h.Rc[5], h.Rc[10], h.Rc[15]);
  };
  sf_generate<<<Gg, ST, 0, s>>>(a, 0);
  ++nl;
  for (int f = 0; f < nflush; ++f) {
    sf_update_project<<<G, ST, su, s>>>(a, f, 0);
    show("update", f);
    if (f + 1 < nflush) { sf_generate<<<Gg, ST, 0, s>>>(a, f + 1); ++nl; }
    sf_subtract<<<G, ST, ss, s>>>(a, f, 0);
    show("sub1", f);
    sf_subtract<<<G, ST, ss, s>>>(a, f, 1);
    show("sub2", f);
    sf_cholqr<<<Gg, ST, 0, s>>>(a, f, 0);
    sf_cholqr<<<Gg, ST, 0, s>>>(a, f, 1);
    show("cholqr", f);
    sf_finish<<<1, ST, sfin, s>>>(a, f);
    show("finish", f);
    nl += 6;
  }
  sf_update_project<<<G, ST, su, s>>>(a, nflush, 1);
  ++nl;
  if (launches) *launches += nl;
  return cudaGetLastError();
}

}  // namespace lrk
