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
// TMA bulk-copy ring (cp.async.bulk + mbarriers, depth sized from the actual
// pane rank so ~150 KB are in flight per SM), runs the row x small
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

constexpr int ST = 256;           // threads per CTA of the light passes
constexpr int NW = 16;            // warps of the staged row passes
constexpr int SPT = 32 * NW;
constexpr int LDW = 68;           // shared leading dimension of the update matrix (== 4 mod 16)
constexpr int PSTR = SF_N * SF_P + SF_P + 8;  // per-CTA partial stride (doubles)

// ---- warp-private cp.async rings.  Every staged pass works on 8-row tiles
// and each warp only ever touches its own tiles (the update tile, its share
// of the projections and Grams), so a warp streams its rows through its own
// shared-memory ring: 16-byte cp.async per lane, cp.async.wait_group, no CTA
// barrier and no cross-warp handshake in the main loop.  The ring depth is
// chosen from the ACTUAL column count (the pane rank is only known on the
// device): deep rings at low rank, >= 2 tiles at rank 64.
__device__ __forceinline__ void cp16(void* smem, const void* gmem, bool valid) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  const int sz = valid ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(sa), "l"(gmem), "r"(sz)
               : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory"); }
__device__ __forceinline__ void cp_wait_dyn(int n) {
  switch (n) {
    case 0: cp_wait<0>(); break;
    case 1: cp_wait<1>(); break;
    case 2: cp_wait<2>(); break;
    case 3: cp_wait<3>(); break;
    case 4: cp_wait<4>(); break;
    case 5: cp_wait<5>(); break;
    case 6: cp_wait<6>(); break;
    case 7: cp_wait<7>(); break;
    case 8: cp_wait<8>(); break;
    case 9: cp_wait<9>(); break;
    case 10: cp_wait<10>(); break;
    case 11: cp_wait<11>(); break;
    case 12: cp_wait<12>(); break;
    case 13: cp_wait<13>(); break;
    default: cp_wait<14>(); break;
  }
}
constexpr int LDT = 8;        // rows per tile = leading dimension of a staged column
constexpr int MAXDEPTH = 15;  // (cp_wait_dyn covers depth - 1 <= 14)

struct WRing {
  double* base;  // this warp's region
  int slot;      // doubles per tile (ncols * LDT)
  int depth;
};

__device__ __forceinline__ WRing wring(double* region, int per_warp, int ncols) {
  WRing R;
  R.base = region + (int64_t)(threadIdx.x >> 5) * per_warp;
  R.slot = (ncols > 0 ? ncols : 1) * LDT;
  R.depth = per_warp / R.slot;
  R.depth = R.depth < 2 ? 2 : (R.depth > MAXDEPTH ? MAXDEPTH : R.depth);
  return R;
}

// Copy tile `tile` (rows tile*8 .. +8) of ncols columns into slot `sl`; every
// lane commits one group (possibly empty) so the group counts stay aligned.
template <typename ColFn>
__device__ __forceinline__ void wring_issue(const WRing& R, int sl, int64_t tile, bool valid, int ncols,
                                            ColFn src, int64_t n_x) {
  if (valid) {
    const int lane = threadIdx.x & 31;
    double* dst = R.base + (int64_t)sl * R.slot;
    const int64_t r0 = tile * LDT;
    for (int q = lane; q < ncols * 4; q += 32) {
      const int c = q >> 2, j = q & 3;
      const int64_t row = r0 + 2 * j;
      const bool ok = row < n_x;
      cp16(dst + c * LDT + 2 * j, src(c) + (ok ? row : 0), ok);
    }
  }
  cp_commit();
}

// Tiles of this CTA: a contiguous range [t0, t1) of the 8-row tile grid;
// warp w takes tiles t0 + w, t0 + w + NW, ...
__device__ __forceinline__ void cta_tiles(int64_t n_x, int64_t& t0, int64_t& t1) {
  const int64_t nt = (n_x + LDT - 1) / LDT;
  const int64_t per = (nt + gridDim.x - 1) / gridDim.x;
  t0 = min(nt, (int64_t)blockIdx.x * per);
  t1 = min(nt, t0 + per);
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
    for (int ww = 0; ww < (int)(blockDim.x / 32); ++ww) s += red[ww * K + threadIdx.x];
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

// out[e] = sum over CTAs of part[c * PSTR + e], e < len: one warp per entry,
// lanes stride over the CTAs (independent loads in flight), then a fixed
// shuffle tree — deterministic.
__device__ __forceinline__ void reduce_parts(const double* part, int len, double* out) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int e = w; e < len; e += nw) {
    double s0 = 0.0, s1 = 0.0;
    int c = lane;
    for (; c + 32 < (int)gridDim.x; c += 64) {
      s0 += __ldcg(part + (int64_t)c * PSTR + e);
      s1 += __ldcg(part + (int64_t)(c + 32) * PSTR + e);
    }
    if (c < (int)gridDim.x) s0 += __ldcg(part + (int64_t)c * PSTR + e);
    const double v = warp_sum(s0 + s1);
    if (lane == 0) out[e] = v;
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

// Tail of the second CGS pass (thread 0): the shifted Cholesky factor of
// G0 = y2^T y2 (Fukaya et al. shifted CholeskyQR3, first step); a remainder at
// the block's rounding floor 16 eps ||Y|| is dropped whole.  Out of line: keeps
// the streaming kernel's register count low.
static __device__ __noinline__ void sf_shifted_chol(const SFArgs& a, SFState* st, const double* tot,
                                                    int pc) {
  double G[16] = {};
  for (int u = 0; u < pc; ++u)
    for (int v = 0; v < pc; ++v) G[u * 4 + v] = tot[u * pc + v];
  double tr = 0.0, ysq = 0.0;
  for (int s = 0; s < pc; ++s) { tr += G[s * 5]; ysq += st->yn[s]; }
  const double delta = 16.0 * DEPS * sqrt(ysq);
  st->drop_all = !(sqrt(tr) > delta);
  double Rm[16], Zm[16];
  if (st->drop_all) {
    for (int i = 0; i < 16; ++i) { Rm[i] = 0.0; Zm[i] = 0.0; }
  } else {
    const double shift = 11.0 * ((double)a.n_x * pc + pc * (pc + 1)) * DEPS * tr;
    for (int s = 0; s < pc; ++s) G[s * 5] += shift;
    pivoted_chol4(G, pc, 0.0, Rm, Zm);
  }
  for (int i = 0; i < 16; ++i) { st->Rc[i] = Rm[i]; st->Rinv[i] = Zm[i]; }
}

// CholeskyQR pass tail (thread 0): R <- chol(G) R, Rinv <- Rinv chol(G)^{-1};
// pivots below (1e-10)^2 of the leading one are rounding residue of a
// numerically rank-deficient remainder and are dropped (see header).
static __device__ __noinline__ void sf_chol_update(SFState* st, const double* tot, int pc) {
  double G[16] = {};
  int q = 0;
  for (int u = 0; u < SF_P; ++u)
    for (int v = u; v < SF_P; ++v) {
      G[u * 4 + v] = G[v * 4 + u] = tot[q];
      ++q;
    }
  double R1[16], Z1[16], Rc[16], Ri[16], Rn[16], Zn[16];
  pivoted_chol4(G, pc, 1e-20, R1, Z1);
  for (int i = 0; i < 16; ++i) { Rc[i] = st->Rc[i]; Ri[i] = st->Rinv[i]; }
  mat4_mul(R1, Rc, Rn, pc);
  mat4_mul(Ri, Z1, Zn, pc);
  for (int i = 0; i < 16; ++i) { st->Rc[i] = Rn[i]; st->Rinv[i] = Zn[i]; }
}

// --------------------------------------------------------------- update + project
// Pending update (st->pending): U'[:, :rn] = [U[:, :r], y2] Wp, V' likewise;
// then (unless final) P1 = U'^T Y evaluated as Wp^T ([U, y2]^T Y).
// Warp w owns rows 8w..8w+7 of every 128-row chunk: the update tile and its
// share of the projection need no CTA barrier inside a chunk.
__global__ void __launch_bounds__(SPT, 1) sf_update_project(const SFArgs a, int f, int final_only) {
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
  double* W = smem;                           // Wp (n x rn), column c at W + c * LDW
  double* stage = W + SF_N * LDW;             // V update scratch, then the warp rings
  const int avail = a.smem_update / (int)sizeof(double) - SF_N * LDW - 16;
  int* flag = reinterpret_cast<int*>(stage + avail);
  double* red = stage;                        // reused after the main loop

  if (pend) {
    for (int idx = tid; idx < n * rn; idx += SPT) {
      const int k = idx % n, c = idx / n;
      W[c * LDW + k] = st->Wp[k + c * SF_LDW];
    }
    // time rows of this CTA: V' = [V, E] Vc   (in place, via shared memory)
    const int64_t tper = ((int64_t)a.n_t + gridDim.x - 1) / gridDim.x;
    const int64_t nt64 = a.n_t;
    const int64_t t0 = min(nt64, (int64_t)blockIdx.x * tper), t1 = min(nt64, t0 + tper);
    const int nrow = (int)(t1 - t0);
    double* Vs = stage;  // nrow x r
    double* Vc = stage + nrow * SF_CAP + 8;
    for (int idx = tid; idx < n * rn; idx += SPT) Vc[idx] = st->Vc[(idx % n) + (idx / n) * SF_LDW];
    for (int idx = tid; idx < nrow * r; idx += SPT)
      Vs[idx] = a.V[(t0 + idx % nrow) + (int64_t)(idx / nrow) * a.ldv];
    __syncthreads();
    const int sp = st->startp;
    for (int idx = tid; idx < nrow * rn; idx += SPT) {
      const int tl = idx % nrow, c = idx / nrow;
      const int64_t tt = t0 + tl;
      const int sel = a.adjoint ? (a.n_t - 1 - sp) - (int)tt : (int)tt - sp;
      double acc = (sel >= 0 && sel < pcp) ? Vc[(r + sel) + c * n] : 0.0;
      for (int k = 0; k < r; ++k) acc += Vs[tl + k * nrow] * Vc[k + c * n];
      a.V[tt + (int64_t)c * a.ldv] = acc;
    }
  }

  int64_t ct0, ct1;
  cta_tiles(a.n_x, ct0, ct1);
  const int nk = (n + 3) >> 2, nj = (rn + 7) >> 3, nm = (n + 7) >> 3;
  const double* U = a.U;
  const int ncol = n + pc;  // tile: X = [U, y2] columns, then Y
  __syncthreads();          // W and the V-update scratch are settled
  const WRing R = wring(stage, (avail / NW) & ~1, ncol);
  auto src = [&](int c) -> const double* {
    return c < r ? U + (int64_t)c * a.ldu
                 : (c < n ? Y2 + (int64_t)(c - r) * a.ldy : Ycur + (int64_t)(c - n) * a.ldy);
  };
  // projection M = X^T Y over this warp's rows: tile jt = X columns 8jt..8jt+7
  double m[9][2];
#pragma unroll
  for (int j = 0; j < 9; ++j) m[j][0] = m[j][1] = 0.0;
  double ysq = 0.0;
  const bool do_upd = pend && rn > 0 && n > 0;
  const int64_t first = ct0 + warp;
  for (int q = 0; q < R.depth - 1; ++q) {
    const int64_t tq = first + (int64_t)q * NW;
    wring_issue(R, q, tq, tq < ct1, ncol, src, a.n_x);
  }
  int cur = 0, nxt = R.depth - 1;
  for (int64_t tile = first; tile < ct1; tile += NW) {
    {
      const int64_t tq = tile + (int64_t)(R.depth - 1) * NW;
      wring_issue(R, nxt, tq, tq < ct1, ncol, src, a.n_x);
    }
    cp_wait_dyn(R.depth - 1);
    __syncwarp();
    const double* X = R.base + (int64_t)cur * R.slot;
    const double* Yt = X + n * LDT;
    if (do_upd) {
      double acc[8][2];
#pragma unroll
      for (int j = 0; j < 8; ++j) acc[j][0] = acc[j][1] = 0.0;
      for (int kk = 0; kk < nk; ++kk) {
        const int k = 4 * kk + t;
        const double av = (k < n) ? X[k * LDT + g] : 0.0;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          if (j >= nj) break;
          const double bv = (k < n && 8 * j + g < rn) ? W[(8 * j + g) * LDW + k] : 0.0;
          dmma884(acc[j][0], acc[j][1], av, bv);
        }
      }
      const int64_t row = tile * LDT + g;
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
#pragma unroll
      for (int kk = 0; kk < 2; ++kk) {
        const int rho = 4 * kk + t;
        const double bv = (g < pc) ? Yt[g * LDT + rho] : 0.0;
#pragma unroll
        for (int j = 0; j < 9; ++j) {
          if (j >= nm) break;
          const double av = (8 * j + g < n) ? X[(8 * j + g) * LDT + rho] : 0.0;
          dmma884(m[j][0], m[j][1], av, bv);
        }
      }
      if ((lane >> 3) < pc) {
        const double y = Yt[(lane >> 3) * LDT + (lane & 7)];
        ysq += y * y;
      }
    }
    __syncwarp();  // every lane is done with this slot before it is refilled
    cur = cur + 1 == R.depth ? 0 : cur + 1;
    nxt = nxt + 1 == R.depth ? 0 : nxt + 1;
  }
  cp_wait<0>();
  __syncthreads();
  // ---- CTA partial: M (n x pc, row-major), then |Y_s|^2; warps meet in
  // shared memory and are summed in warp order
  double* part = a.part + (int64_t)blockIdx.x * PSTR;
  const int plen = n * pc + pc;
  if (pc > 0) {
    double* wp = stage;  // NW x plen
    for (int idx = tid; idx < NW * plen; idx += SPT) wp[idx] = 0.0;
    __syncthreads();
#pragma unroll
    for (int j = 0; j < 9; ++j) {
      if (j >= nm) break;
      const int row = 8 * j + g;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int c = 2 * t + h;
        if (row < n && c < pc) wp[warp * plen + row * pc + c] = m[j][h];
      }
    }
    double yw = ysq;
    yw += __shfl_xor_sync(0xffffffffu, yw, 1);
    yw += __shfl_xor_sync(0xffffffffu, yw, 2);
    yw += __shfl_xor_sync(0xffffffffu, yw, 4);
    if ((lane & 7) == 0 && (lane >> 3) < pc) wp[warp * plen + n * pc + (lane >> 3)] = yw;
    __syncthreads();
    for (int e = tid; e < plen; e += SPT) {
      double acc = 0.0;
      for (int w = 0; w < NW; ++w) acc += wp[w * plen + e];
      part[e] = acc;
    }
  }
  if (!last_cta(a.ticket + 0, flag)) return;
  // ---- last CTA: P1 = Wp^T M (or M), pane bookkeeping
  double* tot = red + NW * (SF_N * SF_P + SF_P) + 64;
  reduce_parts(a.part, plen * (pc > 0), tot);
  if (pc > 0) {
    for (int idx = tid; idx < rn * pc; idx += SPT) {
      const int i = idx / pc, s2 = idx % pc;
      double acc = 0.0;
      if (pend) {
        for (int k = 0; k < n; ++k) acc += W[i * LDW + k] * tot[k * pc + s2];
      } else {
        acc = tot[i * pc + s2];
      }
      st->C[i * SF_P + s2] = acc;
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
    for (int k = tid; k < rn; k += SPT) a.sigma[k] = st->sig[k];
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
// Warp w owns rows 8w..8w+7 of every chunk (subtraction tile and its share of
// the projection / Gram): one CTA barrier per chunk, for the slot refill.
__global__ void __launch_bounds__(SPT, 1) sf_subtract(const SFArgs a, int f, int mode) {
  extern __shared__ double smem[];
  SFState* st = a.st;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int r = st->r;
  const int pc = st->pc;
  double* Ybuf = a.Yg[f & 1];
  double* Cs = smem;                           // r x SF_P (row-major)
  double* stage = Cs + SF_CAP * SF_P + 8;
  const int avail = a.smem_subtract / (int)sizeof(double) - SF_CAP * SF_P - 8 - 16;
  int* flag = reinterpret_cast<int*>(stage + avail);
  double* red = stage;
  const double* Csrc = mode == 0 ? st->C : st->P2;
  for (int idx = tid; idx < r * SF_P; idx += SPT) Cs[idx] = Csrc[idx];
  int64_t ct0, ct1;
  cta_tiles(a.n_x, ct0, ct1);
  const int nk = (r + 3) >> 2, nm = (r + 7) >> 3;
  const int ncol = r + pc;  // tile: U columns, then Y
  __syncthreads();          // Cs is settled
  const WRing R = wring(stage, (avail / NW) & ~1, ncol);
  auto src = [&](int c) -> const double* {
    return c < r ? a.U + (int64_t)c * a.ldu : Ybuf + (int64_t)(c - r) * a.ldy;
  };
  double p2[8][2];  // mode 0: P2 tile j = U columns 8j.. ; mode 1: p2[0] = Gram
#pragma unroll
  for (int j = 0; j < 8; ++j) p2[j][0] = p2[j][1] = 0.0;
  const int64_t first = ct0 + warp;
  for (int q = 0; q < R.depth - 1; ++q) {
    const int64_t tq = first + (int64_t)q * NW;
    wring_issue(R, q, tq, tq < ct1, ncol, src, a.n_x);
  }
  int cur = 0, nxt = R.depth - 1;
  for (int64_t tile = first; tile < ct1; tile += NW) {
    {
      const int64_t tq = tile + (int64_t)(R.depth - 1) * NW;
      wring_issue(R, nxt, tq, tq < ct1, ncol, src, a.n_x);
    }
    cp_wait_dyn(R.depth - 1);
    __syncwarp();
    double* X = R.base + (int64_t)cur * R.slot;
    double* Yt = X + r * LDT;
    // D = U_rows C  (this tile's 8 rows, columns 0..pc)
    double d0 = 0.0, d1 = 0.0, e0 = 0.0, e1 = 0.0;
    for (int kk = 0; kk < nk; ++kk) {
      const int k = 4 * kk + t;
      const double av = (k < r) ? X[k * LDT + g] : 0.0;
      const double bv = (k < r && g < pc) ? Cs[k * SF_P + g] : 0.0;
      if (kk & 1) dmma884(e0, e1, av, bv);
      else dmma884(d0, d1, av, bv);
    }
    d0 += e0;
    d1 += e1;
    {
      const int64_t grow = tile * LDT + g;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int c = 2 * t + h;
        if (c < pc) {
          const double y = Yt[c * LDT + g] - (h ? d1 : d0);
          Yt[c * LDT + g] = y;
          if (grow < a.n_x) Ybuf[grow + (int64_t)c * a.ldy] = y;
        }
      }
    }
    __syncwarp();
#pragma unroll
    for (int kk = 0; kk < 2; ++kk) {
      const int rho = 4 * kk + t;
      const double yv = (g < pc) ? Yt[g * LDT + rho] : 0.0;
      if (mode == 0) {
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          if (j >= nm) break;
          const double av = (8 * j + g < r) ? X[(8 * j + g) * LDT + rho] : 0.0;
          dmma884(p2[j][0], p2[j][1], av, yv);
        }
      } else {
        dmma884(p2[0][0], p2[0][1], yv, yv);  // G[g][2t..] += y2[rho][g] y2[rho][2t..]
      }
    }
    __syncwarp();  // every lane is done with this slot before it is refilled
    cur = cur + 1 == R.depth ? 0 : cur + 1;
    nxt = nxt + 1 == R.depth ? 0 : nxt + 1;
  }
  cp_wait<0>();
  __syncthreads();
  // ---- CTA partial (warp partials summed in warp order)
  double* part = a.part + (int64_t)blockIdx.x * PSTR;
  const int plen = mode == 0 ? r * pc : pc * pc;
  double* wp = stage;
  for (int idx = tid; idx < NW * plen; idx += SPT) wp[idx] = 0.0;
  __syncthreads();
  if (mode == 0) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      if (j >= nm) break;
      const int row = 8 * j + g;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int c = 2 * t + h;
        if (row < r && c < pc) wp[warp * plen + row * pc + c] = p2[j][h];
      }
    }
  } else {
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int c = 2 * t + h;
      if (g < pc && c < pc) wp[warp * plen + g * pc + c] = p2[0][h];
    }
  }
  __syncthreads();
  for (int e = tid; e < plen; e += SPT) {
    double acc = 0.0;
    for (int w = 0; w < NW; ++w) acc += wp[w * plen + e];
    part[e] = acc;
  }
  if (!last_cta(a.ticket + 1 + mode, flag)) return;
  double* tot = red + NW * SF_CAP * SF_P + 64;
  reduce_parts(a.part, plen, tot);
  if (mode == 0) {
    for (int idx = tid; idx < r * pc; idx += SPT) {
      const int i = idx / pc, s2 = idx % pc;
      st->P2[i * SF_P + s2] = tot[idx];
      st->C[i * SF_P + s2] += tot[idx];
    }
    return;
  }
  if (tid == 0) sf_shifted_chol(a, st, tot, pc);
}

// ----------------------------------------------------------- CholeskyQR passes
// G = Q^T Q with Q = y2 Rinv; R <- chol(G) R, Rinv <- Rinv chol(G)^{-1}
// (pivoted, drop-tolerant).  Light streaming kernel (4 columns, L2-resident).
__global__ void __launch_bounds__(ST, 4) sf_cholqr(const SFArgs a, int f, int pass) {
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
    const int64_t stride = (int64_t)gridDim.x * ST;
    for (int64_t i0 = (int64_t)blockIdx.x * ST + tid; i0 < a.n_x; i0 += 2 * stride) {
      double y[2][SF_P];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int64_t i = i0 + h * stride;
#pragma unroll
        for (int s = 0; s < SF_P; ++s) y[h][s] = (s < pc && i < a.n_x) ? Y[i + (int64_t)s * a.ldy] : 0.0;
      }
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        double qv[SF_P];
#pragma unroll
        for (int c = 0; c < SF_P; ++c) {
          double acc = 0.0;
#pragma unroll
          for (int s = 0; s < SF_P; ++s) acc += y[h][s] * Ri[s * 4 + c];
          qv[c] = acc;
        }
        int q = 0;
#pragma unroll
        for (int u = 0; u < SF_P; ++u)
#pragma unroll
          for (int v = u; v < SF_P; ++v) gacc[q++] += qv[u] * qv[v];
      }
    }
  }
  double* outv = red + 8 * 10;
  cta_sum<10>(gacc, red, outv);
  double* part = a.part + (int64_t)blockIdx.x * PSTR;
  if (tid < 10) part[tid] = outv[tid];
  if (!last_cta(a.ticket + 3 + pass, &flag)) return;
  reduce_parts(a.part, 10, tot);
  if (tid == 0 && !skip) sf_chol_update(st, tot, pc);
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
size_t sf_smem_update() { return 200 * 1024; }
size_t sf_smem_subtract() { return 200 * 1024; }
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
  const size_t su = a.smem_update, ss = a.smem_subtract, sfin = sf_smem_finish();
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
    sf_update_project<<<G, SPT, su, s>>>(a, f, 0);
    show("update", f);
    if (f + 1 < nflush) { sf_generate<<<Gg, ST, 0, s>>>(a, f + 1); ++nl; }
    sf_subtract<<<G, SPT, ss, s>>>(a, f, 0);
    show("sub1", f);
    sf_subtract<<<G, SPT, ss, s>>>(a, f, 1);
    show("sub2", f);
    sf_cholqr<<<Gg, ST, 0, s>>>(a, f, 0);
    sf_cholqr<<<Gg, ST, 0, s>>>(a, f, 1);
    show("cholqr", f);
    sf_finish<<<1, ST, sfin, s>>>(a, f);
    show("finish", f);
    nl += 6;
  }
  sf_update_project<<<G, SPT, su, s>>>(a, nflush, 1);
  ++nl;
  if (launches) *launches += nl;
  return cudaGetLastError();
}

}  // namespace lrk
