// lrk_small.cuh — latency-oriented building blocks for the persistent sweep,
// specialised at compile time on the flush width Q (columns appended per
// truncation) so no loop runs over unused padding.
//
// All row-local routines take raw pointers that the sweep resolves either to
// a CTA's shared-memory block or to global rows; loads are issued before any
// dependent store (explicit register staging) so generic-pointer aliasing
// never serialises the loops.
#pragma once
#include "lrk_device.cuh"

namespace lrk {

// Householder QR of X (m x q, col-major) by the whole CTA, one fused block
// reduction per column: sums[0] = ||x_j below diag||^2, sums[k] = x_j . x_k.
// Reflectors overwrite X below the diagonal, tau[j] saved, R (q x q
// row-major, zero padded) to Rout.  red: NWARP*Q, tmp: Q (shared).
// RB > 1 (rows streaming from HBM/L2): RB rows per thread per iteration with
// all their loads issued first; per-thread accumulation order unchanged.
template <int Q, int RB = 1>
__device__ __forceinline__ void block_qr_t(double* __restrict__ X, int64_t ldx, int m, int q,
                           double* __restrict__ tau, double* __restrict__ Rout,
                           double* __restrict__ red, double* __restrict__ tmp) {
  const int tid = threadIdx.x;
  for (int i = tid; i < q * q; i += NT) Rout[i] = 0.0;
  const int kmax = m < q ? m : q;
  for (int j = 0; j < kmax; ++j) {
    double s[Q];
#pragma unroll
    for (int k = 0; k < Q; ++k) s[k] = 0.0;
    if constexpr (RB > 1) {
      for (int i0 = j + 1 + tid; i0 < m; i0 += RB * NT) {
        double xv[RB][Q];
#pragma unroll
        for (int h = 0; h < RB; ++h) {
          const int i = i0 + h * NT;
#pragma unroll
          for (int k = 0; k < Q; ++k)
            xv[h][k] = (i < m && k >= j && k < q) ? X[i + (int64_t)k * ldx] : 0.0;
        }
#pragma unroll
        for (int h = 0; h < RB; ++h)
          if (i0 + h * NT < m) {
            double xj = 0.0;
#pragma unroll
            for (int k = 0; k < Q; ++k)
              if (k == j) xj = xv[h][k];
#pragma unroll
            for (int k = 0; k < Q; ++k)
              if (k >= j && k < q) s[k] += xj * xv[h][k];
          }
      }
    } else {
#pragma unroll 4
    for (int i = j + 1 + tid; i < m; i += NT) {
      const double xj = X[i + (int64_t)j * ldx];
#pragma unroll
      for (int k = 0; k < Q; ++k)
        if (k >= j && k < q) s[k] += xj * X[i + (int64_t)k * ldx];
    }
    }
    // s[j] = ||x_j||^2 below the diagonal, s[k>j] = x_j . x_k (below the diagonal)
    block_sum<Q>(s, red, tmp);
    double xr[Q];  // row j before the update (all threads read it)
#pragma unroll
    for (int k = 0; k < Q; ++k) xr[k] = (k > j && k < q) ? X[j + (int64_t)k * ldx] : 0.0;
    const double alpha = X[j + (int64_t)j * ldx];
    double sig = 0.0;
#pragma unroll
    for (int k = 0; k < Q; ++k)
      if (k == j) sig = s[k];
    double beta, t, scale;
    if (sig == 0.0) {
      t = 0.0; beta = alpha; scale = 0.0;
    } else {
      const double nrm = sqrt_fast(alpha * alpha + sig);
      beta = alpha >= 0.0 ? -nrm : nrm;
      t = (beta - alpha) * rcp_fast(beta);
      scale = rcp_fast(alpha - beta);
    }
    // w_k = x_jk + scale * (x_j . x_k)  for k > j  (v_i = scale x_ij, v_j = 1)
    double f[Q];
#pragma unroll
    for (int k = 0; k < Q; ++k) f[k] = (k > j && k < q) ? t * (xr[k] + scale * s[k]) : 0.0;
    __syncthreads();  // row j read by everyone before it changes
    if constexpr (RB > 1) {
      for (int i0 = j + 1 + tid; i0 < m; i0 += RB * NT) {
        double xv[RB][Q];
#pragma unroll
        for (int h = 0; h < RB; ++h) {
          const int i = i0 + h * NT;
#pragma unroll
          for (int k = 0; k < Q; ++k)
            xv[h][k] = (i < m && k >= j && k < q) ? X[i + (int64_t)k * ldx] : 0.0;
        }
#pragma unroll
        for (int h = 0; h < RB; ++h) {
          const int i = i0 + h * NT;
          if (i < m) {
            double vi = 0.0;
#pragma unroll
            for (int k = 0; k < Q; ++k)
              if (k == j) vi = xv[h][k] * scale;
            X[i + (int64_t)j * ldx] = vi;
#pragma unroll
            for (int k = 0; k < Q; ++k)
              if (k > j && k < q) X[i + (int64_t)k * ldx] = xv[h][k] - f[k] * vi;
          }
        }
      }
    } else {
#pragma unroll 4
    for (int i = j + 1 + tid; i < m; i += NT) {
      const double vi = X[i + (int64_t)j * ldx] * scale;
      double x[Q];
#pragma unroll
      for (int k = 0; k < Q; ++k) x[k] = (k > j && k < q) ? X[i + (int64_t)k * ldx] : 0.0;
      X[i + (int64_t)j * ldx] = vi;
#pragma unroll
      for (int k = 0; k < Q; ++k)
        if (k > j && k < q) X[i + (int64_t)k * ldx] = x[k] - f[k] * vi;
    }
    }
    if (tid == 0) {
      tau[j] = t;
#pragma unroll
      for (int k = 0; k < Q; ++k)
        if (k > j && k < q) {
          const double v = xr[k] - f[k];
          X[j + (int64_t)k * ldx] = v;
          Rout[j * q + k] = v;
        }
      Rout[j * q + j] = beta;
      X[j + (int64_t)j * ldx] = beta;
    }
    __syncthreads();
  }
  for (int j = kmax + tid; j < q; j += NT) tau[j] = 0.0;
  __syncthreads();
}

// Y (m x q) = H_0 ... H_{kmax-1} [G; 0]  (G q x q row-major), whole CTA.
template <int Q>
__device__ __forceinline__ void block_apply_q_t(const double* __restrict__ X, int64_t ldx, int m, int q,
                                const double* __restrict__ tau, const double* __restrict__ G,
                                double* __restrict__ Y, int64_t ldy, double* __restrict__ red,
                                double* __restrict__ tmp) {
  const int tid = threadIdx.x;
  for (int i = tid; i < m; i += NT) {
#pragma unroll
    for (int c = 0; c < Q; ++c)
      if (c < q) Y[i + (int64_t)c * ldy] = (i < q) ? G[i * q + c] : 0.0;
  }
  __syncthreads();
  const int kmax = m < q ? m : q;
  for (int j = kmax - 1; j >= 0; --j) {
    const double t = tau[j];
    if (t == 0.0) continue;  // uniform
    double w[Q];
#pragma unroll
    for (int c = 0; c < Q; ++c) w[c] = 0.0;
#pragma unroll 4
    for (int i = j + 1 + tid; i < m; i += NT) {
      const double vi = X[i + (int64_t)j * ldx];
#pragma unroll
      for (int c = 0; c < Q; ++c)
        if (c < q) w[c] += vi * Y[i + (int64_t)c * ldy];
    }
    block_sum<Q>(w, red, tmp);
    double f[Q];
#pragma unroll
    for (int c = 0; c < Q; ++c) f[c] = (c < q) ? t * (w[c] + Y[j + (int64_t)c * ldy]) : 0.0;
    __syncthreads();
#pragma unroll 4
    for (int i = j + 1 + tid; i < m; i += NT) {
      const double vi = X[i + (int64_t)j * ldx];
#pragma unroll
      for (int c = 0; c < Q; ++c)
        if (c < q) Y[i + (int64_t)c * ldy] -= f[c] * vi;
    }
    if (tid == 0) {
#pragma unroll
      for (int c = 0; c < Q; ++c)
        if (c < q) Y[j + (int64_t)c * ldy] -= f[c];
    }
    __syncthreads();
  }
}

// Y (m x q) = H_0 ... H_{q-1} [G; 0] in ONE pass over the rows via the compact
// WY form H_0...H_{q-1} = I - V T V^T (LAPACK larft, forward columnwise):
// Y = [G; 0] - V M,  M = T (V_top^T G),  V unit lower-trapezoidal (the
// reflectors left below the diagonal of X by block_qr_t).  One reduction pass
// forms V^T V; T and M are q x q on one thread.  wsm: 3*Q*Q shared doubles.
template <int Q>  // Q <= 4 (block_sum scratch: NWARP * Q(Q+1)/2 <= NWARP * PMAX)
__device__ __forceinline__ void block_apply_q_wy(const double* __restrict__ X, int64_t ldx, int m,
                                                 int q, const double* __restrict__ tau,
                                                 const double* __restrict__ G,
                                                 double* __restrict__ Y, int64_t ldy,
                                                 double* __restrict__ red, double* __restrict__ tmp,
                                                 double* __restrict__ wsm) {
  constexpr int NP = Q * (Q + 1) / 2;
  const int tid = threadIdx.x;
  // V^T V (upper triangle, packed): rows >= q only; the q x q top is added below
  double acc[NP];
#pragma unroll
  for (int k = 0; k < NP; ++k) acc[k] = 0.0;
#pragma unroll 4
  for (int i = q + tid; i < m; i += NT) {
    double v[Q];
#pragma unroll
    for (int c = 0; c < Q; ++c) v[c] = (c < q) ? X[i + (int64_t)c * ldx] : 0.0;
    int k = 0;
#pragma unroll
    for (int a = 0; a < Q; ++a)
#pragma unroll
      for (int b = a; b < Q; ++b) acc[k++] += v[a] * v[b];
  }
  block_sum<NP>(acc, red, tmp);  // tmp[0..NP) = packed V_bot^T V_bot (all threads see acc)
  double* T = wsm;
  double* M = wsm + Q * Q;
  if (tid == 0) {
    double Vt[Q][Q];  // V_top (unit lower)
#pragma unroll
    for (int i = 0; i < Q; ++i)
#pragma unroll
      for (int c = 0; c < Q; ++c)
        Vt[i][c] = (i < q && i < m && c < q) ? (i == c ? 1.0 : (i > c ? X[i + (int64_t)c * ldx] : 0.0)) : 0.0;
    double VV[Q][Q];
    {
      int k = 0;
#pragma unroll
      for (int a = 0; a < Q; ++a)
#pragma unroll
        for (int b = a; b < Q; ++b) {
          double sv = acc[k++];
#pragma unroll
          for (int i = 0; i < Q; ++i) sv += Vt[i][a] * Vt[i][b];
          VV[a][b] = sv;
          VV[b][a] = sv;
        }
    }
    double Tm[Q][Q];
#pragma unroll
    for (int i = 0; i < Q; ++i)
#pragma unroll
      for (int j = 0; j < Q; ++j) Tm[i][j] = 0.0;
#pragma unroll
    for (int j = 0; j < Q; ++j) {
      if (j >= q) break;
      const double tj = tau[j];
      Tm[j][j] = tj;
      // T[0:j, j] = -tau_j T[0:j, 0:j] (V^T v_j)[0:j]
#pragma unroll
      for (int i = 0; i < Q; ++i) {
        if (i >= j) break;
        double sv = 0.0;
#pragma unroll
        for (int l = 0; l < Q; ++l)
          if (l >= i && l < j) sv += Tm[i][l] * VV[l][j];
        Tm[i][j] = -tj * sv;
      }
    }
    // M = T (V_top^T G)
    double W[Q][Q];
#pragma unroll
    for (int a = 0; a < Q; ++a)
#pragma unroll
      for (int c = 0; c < Q; ++c) {
        double sv = 0.0;
#pragma unroll
        for (int i = 0; i < Q; ++i)
          if (i < q && c < q) sv += Vt[i][a] * G[i * q + c];
        W[a][c] = sv;
      }
#pragma unroll
    for (int a = 0; a < Q; ++a)
#pragma unroll
      for (int c = 0; c < Q; ++c) {
        double sv = 0.0;
#pragma unroll
        for (int l = 0; l < Q; ++l) sv += Tm[a][l] * W[l][c];
        M[a * Q + c] = sv;
      }
  }
  __syncthreads();
  double Mr[Q][Q];
#pragma unroll
  for (int a = 0; a < Q; ++a)
#pragma unroll
    for (int c = 0; c < Q; ++c) Mr[a][c] = M[a * Q + c];
#pragma unroll 4
  for (int i = tid; i < m; i += NT) {
    double v[Q];
#pragma unroll
    for (int c = 0; c < Q; ++c)
      v[c] = (c < q) ? (i == c ? 1.0 : (i > c ? X[i + (int64_t)c * ldx] : 0.0)) : 0.0;
#pragma unroll
    for (int c = 0; c < Q; ++c) {
      if (c >= q) break;
      double y = (i < q) ? G[i * q + c] : 0.0;
#pragma unroll
      for (int a = 0; a < Q; ++a) y -= v[a] * Mr[a][c];
      Y[i + (int64_t)c * ldy] = y;
    }
  }
  __syncthreads();
}

// X[:, 0..nx) -= A[:, 0..na) Cm, Cm na x nx row-major (shared); nx <= Q.
// RPI rows per thread iteration (independent load streams; 4 when the rows
// stream from HBM).
template <int Q, int RPI = 2>
__device__ __forceinline__ void rows_sub_t(double* __restrict__ X, int64_t ldx, int nx,
                           const double* __restrict__ A, int64_t lda, int na,
                           const double* __restrict__ Cm, int nrows) {
  for (int t = threadIdx.x; t < nrows; t += RPI * NT) {
    double acc[RPI][Q];
#pragma unroll
    for (int q = 0; q < RPI; ++q)
#pragma unroll
      for (int j = 0; j < Q; ++j) acc[q][j] = 0.0;
    if constexpr (RPI >= 4 && Q <= 4) {
      // rows from HBM: four columns of A for all RPI rows loaded before
      // their FMAs (same per-row accumulation order)
      for (int i0 = 0; i0 < na; i0 += 4) {
        double av[4][RPI];
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
          for (int q = 0; q < RPI; ++q)
            av[u][q] = (i0 + u < na && t + q * NT < nrows) ? A[t + q * NT + (int64_t)(i0 + u) * lda] : 0.0;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          if (i0 + u >= na) break;
#pragma unroll
          for (int j = 0; j < Q; ++j)
            if (j < nx) {
              const double c = Cm[(i0 + u) * nx + j];
#pragma unroll
              for (int q = 0; q < RPI; ++q) acc[q][j] += av[u][q] * c;
            }
        }
      }
    } else {
#pragma unroll 8
    for (int i = 0; i < na; ++i) {
      double a[RPI];
#pragma unroll
      for (int q = 0; q < RPI; ++q) a[q] = (t + q * NT < nrows) ? A[t + q * NT + (int64_t)i * lda] : 0.0;
#pragma unroll
      for (int j = 0; j < Q; ++j)
        if (j < nx) {
          const double c = Cm[i * nx + j];
#pragma unroll
          for (int q = 0; q < RPI; ++q) acc[q][j] += a[q] * c;
        }
    }
    }
#pragma unroll
    for (int j = 0; j < Q; ++j)
      if (j < nx) {
#pragma unroll
        for (int q = 0; q < RPI; ++q)
          if (t + q * NT < nrows) X[t + q * NT + (int64_t)j * ldx] -= acc[q][j];
      }
  }
}

// ----------------------------------------------------------- DMMA helpers
// (dmma884 lives in lrk_device.cuh)

// In-place row update on the tensor pipe: rows [0, m) of X = [A (na cols) | B
// (nb cols)] (column-major, lda/ldb) times W (n x rn, col-major ld ldw) are
// written into A's first rn columns (rn <= 8*NT8).  Each warp owns whole
// 8-row tiles, so every row is read (into fragments) before the warp writes
// it.  Called by all threads of the CTA.
template <int NT8, int TPI = 2>
__device__ __forceinline__ void update_rows_dmma(double* __restrict__ A, int64_t lda, int na,
                                                 const double* __restrict__ B, int64_t ldb, int nb,
                                                 const double* __restrict__ W, int ldw, int rn,
                                                 int m) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int n = na + nb;  // <= 32: every operand of a row tile is loaded up front
  const int ntile = (m + 7) >> 3;
  // TPI row tiles per warp iteration: 8*TPI independent loads in flight per
  // lane (TPI 4 when the rows stream from HBM)
  for (int tile0 = warp * TPI; tile0 < ntile; tile0 += NWARP * TPI) {
    double av[TPI][8];
#pragma unroll
    for (int h = 0; h < TPI; ++h) {
      const int row = (tile0 + h) * 8 + g;
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) {
        const int k = kk * 4 + t;
        av[h][kk] = 0.0;
        if (row < m && k < n) av[h][kk] = (k < na) ? A[row + (int64_t)k * lda] : B[row + (int64_t)(k - na) * ldb];
      }
    }
    // all row tiles advance together: TPI*NT8 independent DMMA chains
    double acc[TPI][NT8][2];
#pragma unroll
    for (int h = 0; h < TPI; ++h)
#pragma unroll
      for (int j = 0; j < NT8; ++j) acc[h][j][0] = acc[h][j][1] = 0.0;
#pragma unroll
    for (int kk = 0; kk < 8; ++kk) {
      if (kk * 4 >= n) break;
      const int k = kk * 4 + t;
#pragma unroll
      for (int j = 0; j < NT8; ++j) {
        const int col = j * 8 + g;
        const double b = (k < n && col < rn) ? W[k + col * ldw] : 0.0;
#pragma unroll
        for (int h = 0; h < TPI; ++h) dmma884(acc[h][j][0], acc[h][j][1], av[h][kk], b);
      }
    }
    __syncwarp();
#pragma unroll
    for (int h = 0; h < TPI; ++h) {
      const int row = (tile0 + h) * 8 + g;
#pragma unroll
      for (int j = 0; j < NT8; ++j) {
        const int c0 = j * 8 + 2 * t;
        if (row < m) {
          if (c0 < rn) A[row + (int64_t)c0 * lda] = acc[h][j][0];
          if (c0 + 1 < rn) A[row + (int64_t)(c0 + 1) * lda] = acc[h][j][1];
        }
      }
    }
  }
}

// Wide-core variant (n = na + nb <= 64, rn <= 64): the same in-place row-tile
// update with 16 k-steps and 8 output column tiles; W is read through L1
// (global per-CTA scratch, n x rn <= 32 KB) and amortised over TPI row tiles.
template <int TPI>
__device__ __forceinline__ void update_rows_dmma_wide(double* __restrict__ A, int64_t lda, int na,
                                                      const double* __restrict__ B, int64_t ldb,
                                                      int nb, const double* __restrict__ W,
                                                      int ldw, int rn, int m) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int n = na + nb;
  const int ntile = (m + 7) >> 3;
  const int nk = (n + 3) >> 2, nj = (rn + 7) >> 3;
  for (int tile0 = warp * TPI; tile0 < ntile; tile0 += NWARP * TPI) {
    double av[TPI][16];
#pragma unroll
    for (int h = 0; h < TPI; ++h) {
      const int row = (tile0 + h) * 8 + g;
#pragma unroll
      for (int kk = 0; kk < 16; ++kk) {
        const int k = kk * 4 + t;
        av[h][kk] = 0.0;
        if (row < m && k < n) av[h][kk] = (k < na) ? A[row + (int64_t)k * lda] : B[row + (int64_t)(k - na) * ldb];
      }
    }
    double acc[TPI][8][2];
#pragma unroll
    for (int h = 0; h < TPI; ++h)
#pragma unroll
      for (int j = 0; j < 8; ++j) acc[h][j][0] = acc[h][j][1] = 0.0;
#pragma unroll
    for (int kk = 0; kk < 16; ++kk) {
      if (kk >= nk) break;
      const int k = kk * 4 + t;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        if (j >= nj) break;
        const int col = j * 8 + g;
        const double b = (k < n && col < rn) ? W[k + col * ldw] : 0.0;
#pragma unroll
        for (int h = 0; h < TPI; ++h) dmma884(acc[h][j][0], acc[h][j][1], av[h][kk], b);
      }
    }
    __syncwarp();
#pragma unroll
    for (int h = 0; h < TPI; ++h) {
      const int row = (tile0 + h) * 8 + g;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int c0 = j * 8 + 2 * t;
        if (row < m) {
          if (c0 < rn) A[row + (int64_t)c0 * lda] = acc[h][j][0];
          if (c0 + 1 < rn) A[row + (int64_t)(c0 + 1) * lda] = acc[h][j][1];
        }
      }
    }
  }
}

// CTA partial of A^T B (na <= 8*NI, nb <= 8) on the FP64 tensor pipe:
// warp w takes a contiguous row chunk; m8n8k4 with the A-operand = rows k..k+3
// of 8 columns of A (lane (g,t) reads A[k+t, 8i+g]: fully used 32-byte
// sectors) and the B-operand = B[k+t, g]; U k-steps of loads are issued
// before their DMMAs.  Per-warp partials meet in wbuf (NWARP*na*nb shared
// doubles) and are summed in warp order into out[i*nb + j].
// Warp-group synchronisation: the whole CTA (GW == NWARP) or the GW warps
// starting at warp WOFF on named barrier 2 (barrier 1 belongs to the Jacobi).
template <int GW, int WOFF>
__device__ __forceinline__ void grp_sync() {
  if constexpr (GW == NWARP) __syncthreads();
  else asm volatile("bar.sync 2, %0;" ::"r"(GW * 32));
}

// Executed by the GW warps [WOFF, WOFF+GW) (default: the whole CTA).
template <int NI, int GW = NWARP, int WOFF = 0>
__device__ __forceinline__ void cta_tn_dmma(const double* __restrict__ A, int64_t lda, int na,
                                            const double* __restrict__ B, int64_t ldb, int nb,
                                            int nrows, double* __restrict__ out,
                                            double* __restrict__ wbuf) {
  const int lane = threadIdx.x & 31, warp = (threadIdx.x >> 5) - WOFF;
  const int g = lane >> 2, t = lane & 3;
  const int chunk = (((nrows + GW - 1) / GW) + 3) & ~3;
  const int r0 = warp * chunk;
  const int r1 = min(nrows, r0 + chunk);
  double acc[NI][2];
#pragma unroll
  for (int i = 0; i < NI; ++i) acc[i][0] = acc[i][1] = 0.0;
  constexpr int U = 8 / (NI > 4 ? 2 : 1);  // k-steps of loads in flight
  for (int k0 = r0; k0 < r1; k0 += 4 * U) {
    double av[U][NI], bv[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int k = k0 + 4 * u + t;
      const bool ok = k < r1;
#pragma unroll
      for (int i = 0; i < NI; ++i) {
        const int col = 8 * i + g;
        av[u][i] = (ok && col < na) ? A[k + (int64_t)col * lda] : 0.0;
      }
      bv[u] = (ok && g < nb) ? B[k + (int64_t)g * ldb] : 0.0;
    }
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      for (int i = 0; i < NI; ++i) dmma884(acc[i][0], acc[i][1], av[u][i], bv[u]);
  }
#pragma unroll
  for (int i = 0; i < NI; ++i)
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int ii = 8 * i + g, jj = 2 * t + h;
      if (ii < na && jj < nb) wbuf[(warp * na + ii) * nb + jj] = acc[i][h];
    }
  grp_sync<GW, WOFF>();
  for (int o = threadIdx.x - 32 * WOFF; o < na * nb; o += 32 * GW) {
    double s = 0.0;
#pragma unroll
    for (int w = 0; w < GW; ++w) s += wbuf[w * na * nb + o];
    out[o] = s;
  }
  grp_sync<GW, WOFF>();
}

// Fused first CGS pass, one sweep over the rows: Y -= U Cm (in place), then
// the CTA partial of U^T Y (na <= 8*NI, nb <= 4) on the FP64 tensor pipe.
// Lane (g,t) holds U[k+t, 8i+g]; the 8 lanes sharing t together hold row k+t,
// so the row's (U Cm)[k+t, :] is a 3-level xor-shuffle sum of their partials
// and lane (g,t) subtracts entry g from its Y[k+t, g] before that value
// becomes the DMMA B-operand.  Halves the passes over U of rows_sub_t + cta_tn_dmma.
template <int NI>
__device__ __forceinline__ void cta_subtn_dmma(const double* __restrict__ A, int64_t lda, int na,
                                               double* __restrict__ B, int64_t ldb, int nb,
                                               const double* __restrict__ Cm, int nrows,
                                               double* __restrict__ out,
                                               double* __restrict__ wbuf) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, t = lane & 3;
  const unsigned full = 0xffffffffu;
  const int chunk = (((nrows + NWARP - 1) / NWARP) + 3) & ~3;
  const int r0 = warp * chunk;
  const int r1 = min(nrows, r0 + chunk);
  // this lane's rows of Cm (rows 8i+g, nb <= 4 columns)
  double cm[NI][4];
#pragma unroll
  for (int i = 0; i < NI; ++i)
#pragma unroll
    for (int s2 = 0; s2 < 4; ++s2) {
      const int row = 8 * i + g;
      cm[i][s2] = (row < na && s2 < nb) ? Cm[row * nb + s2] : 0.0;
    }
  double acc[NI][2];
#pragma unroll
  for (int i = 0; i < NI; ++i) acc[i][0] = acc[i][1] = 0.0;
  constexpr int U = 4 / (NI > 4 ? 2 : 1);
  for (int k0 = r0; k0 < r1; k0 += 4 * U) {
    double av[U][NI], yv[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int k = k0 + 4 * u + t;
      const bool ok = k < r1;
#pragma unroll
      for (int i = 0; i < NI; ++i) {
        const int col = 8 * i + g;
        av[u][i] = (ok && col < na) ? A[k + (int64_t)col * lda] : 0.0;
      }
      yv[u] = (ok && g < nb) ? B[k + (int64_t)g * ldb] : 0.0;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      double ps[4];
#pragma unroll
      for (int s2 = 0; s2 < 4; ++s2) {
        double v = 0.0;
#pragma unroll
        for (int i = 0; i < NI; ++i) v += av[u][i] * cm[i][s2];
        ps[s2] = v;
      }
#pragma unroll
      for (int o = 4; o < 32; o <<= 1)
#pragma unroll
        for (int s2 = 0; s2 < 4; ++s2) ps[s2] += __shfl_xor_sync(full, ps[s2], o);
      const double sub = g == 0 ? ps[0] : (g == 1 ? ps[1] : (g == 2 ? ps[2] : ps[3]));
      const int k = k0 + 4 * u + t;
      double y = 0.0;
      if (k < r1 && g < nb) {
        y = yv[u] - sub;
        B[k + (int64_t)g * ldb] = y;
      }
#pragma unroll
      for (int i = 0; i < NI; ++i) dmma884(acc[i][0], acc[i][1], av[u][i], y);
    }
  }
#pragma unroll
  for (int i = 0; i < NI; ++i)
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int ii = 8 * i + g, jj = 2 * t + h;
      if (ii < na && jj < nb) wbuf[(warp * na + ii) * nb + jj] = acc[i][h];
    }
  __syncthreads();
  for (int o = threadIdx.x; o < na * nb; o += NT) {
    double s2 = 0.0;
#pragma unroll
    for (int w = 0; w < NWARP; ++w) s2 += wbuf[w * na * nb + o];
    out[o] = s2;
  }
  __syncthreads();
}

// Column-pivoted Householder QR of the q x q (q <= Q) matrix A held in
// registers by one thread (compile-time unrolled, no local memory):
// A P = X Rt.  On exit A = Rt (upper), X orthogonal, perm[k] = source column
// of Rt's column k.  Used for the rank-revealing fix-up of the TSQR's R.
template <int Q>
__device__ __forceinline__ void pivoted_qr_reg(double (&A)[Q][Q], int q, double (&X)[Q][Q],
                                               int (&perm)[Q]) {
#pragma unroll
  for (int i = 0; i < Q; ++i) {
    perm[i] = i;
#pragma unroll
    for (int k = 0; k < Q; ++k) X[i][k] = (i == k) ? 1.0 : 0.0;
  }
#pragma unroll
  for (int j = 0; j < Q; ++j) {
    if (j >= q) break;
    // pivot: largest trailing column norm (exact)
    double best = -1.0;
    int piv = j;
#pragma unroll
    for (int k = 0; k < Q; ++k) {
      if (k < j || k >= q) continue;
      double s = 0.0;
#pragma unroll
      for (int i = 0; i < Q; ++i)
        if (i >= j && i < q) s += A[i][k] * A[i][k];
      if (s > best) { best = s; piv = k; }
    }
#pragma unroll
    for (int k = 0; k < Q; ++k) {
      if (k == piv && k != j) {
#pragma unroll
        for (int i = 0; i < Q; ++i) { const double t = A[i][j]; A[i][j] = A[i][k]; A[i][k] = t; }
        const int t = perm[j]; perm[j] = perm[k]; perm[k] = t;
      }
    }
    double sig = 0.0, alpha = 0.0;
#pragma unroll
    for (int i = 0; i < Q; ++i) {
      if (i > j && i < q) sig += A[i][j] * A[i][j];
      if (i == j) alpha = A[i][j];
    }
    if (sig == 0.0) continue;
    const double nrm = sqrt_fast(alpha * alpha + sig);
    const double beta = alpha >= 0.0 ? -nrm : nrm;
    const double tau = (beta - alpha) * rcp_fast(beta);
    const double sc = rcp_fast(alpha - beta);
    double v[Q];
#pragma unroll
    for (int i = 0; i < Q; ++i) v[i] = (i == j) ? 1.0 : ((i > j && i < q) ? A[i][j] * sc : 0.0);
    // A <- H A on columns >= j
#pragma unroll
    for (int k = 0; k < Q; ++k) {
      if (k < j || k >= q) continue;
      double w = 0.0;
#pragma unroll
      for (int i = 0; i < Q; ++i) w += v[i] * A[i][k];
      w *= tau;
#pragma unroll
      for (int i = 0; i < Q; ++i) A[i][k] -= w * v[i];
    }
    // X <- X H
#pragma unroll
    for (int i = 0; i < Q; ++i) {
      double w = 0.0;
#pragma unroll
      for (int l = 0; l < Q; ++l) w += X[i][l] * v[l];
      w *= tau;
#pragma unroll
      for (int l = 0; l < Q; ++l) X[i][l] -= w * v[l];
    }
#pragma unroll
    for (int i = 0; i < Q; ++i)
      if (i > j) A[i][j] = 0.0;
  }
}

// Warp form of the stacked-R fix-up (pivoted_qr_reg + rounding-floor drop +
// G = Qs X), lane c holding column c of the pc x pc R (pc <= Q <= 4): the
// column norms, the pivot argmax (xor-shuffle, first index on ties like the
// serial scan), the swap and the reflector broadcast are shuffles; every lane
// forms the reflectors redundantly.  Writes R (row j in the ORIGINAL column
// order) back to Rp and G (row-major) — the same outputs as the one-thread
// form, to rounding.  All 32 lanes of one warp call it.
template <int Q>
__device__ __forceinline__ void warp_pivqr_fixup(double* __restrict__ Rp,
                                                 const double* __restrict__ Qs,
                                                 double* __restrict__ G,
                                                 const double* __restrict__ Yn, int pc) {
  const int lane = threadIdx.x & 31;
  const unsigned full = 0xffffffffu;
  const bool own = lane < pc;
  double a[Q];
#pragma unroll
  for (int i = 0; i < Q; ++i) a[i] = (own && i < pc) ? Rp[i * pc + lane] : 0.0;
  double ysq = 0.0;
  for (int s2 = 0; s2 < pc; ++s2) ysq += Yn[s2];
  const double delta = 16.0 * DEPS * sqrt(ysq);
  int perm = lane;
  double vs[Q][Q], taus[Q];
#pragma unroll
  for (int j = 0; j < Q; ++j) {
    taus[j] = 0.0;
#pragma unroll
    for (int i = 0; i < Q; ++i) vs[j][i] = 0.0;
    if (j >= pc) continue;  // uniform
    double sn = -1.0;
    if (own && lane >= j) {
      sn = 0.0;
#pragma unroll
      for (int i = 0; i < Q; ++i)
        if (i >= j && i < pc) sn += a[i] * a[i];
    }
    double bs = sn;
    int bi = lane;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const double os = __shfl_xor_sync(full, bs, o);
      const int oi = __shfl_xor_sync(full, bi, o);
      if (os > bs || (os == bs && oi < bi)) { bs = os; bi = oi; }
    }
    const int piv = bi;
    const int src = (lane == j) ? piv : ((lane == piv) ? j : lane);
#pragma unroll
    for (int i = 0; i < Q; ++i) a[i] = __shfl_sync(full, a[i], src);
    perm = __shfl_sync(full, perm, src);
    double cj[Q];
#pragma unroll
    for (int i = 0; i < Q; ++i) cj[i] = __shfl_sync(full, a[i], j);
    double sig = 0.0;
#pragma unroll
    for (int i = 0; i < Q; ++i)
      if (i > j && i < pc) sig += cj[i] * cj[i];
    const double alpha = cj[j];
    if (sig == 0.0) continue;  // uniform (same values in every lane)
    const double nrm = sqrt_fast(alpha * alpha + sig);
    const double beta = alpha >= 0.0 ? -nrm : nrm;
    const double tau = (beta - alpha) * rcp_fast(beta);
    const double sc = rcp_fast(alpha - beta);
    double v[Q];
#pragma unroll
    for (int i = 0; i < Q; ++i) v[i] = (i == j) ? 1.0 : ((i > j && i < pc) ? cj[i] * sc : 0.0);
    if (own && lane >= j) {
      double w = 0.0;
#pragma unroll
      for (int i = 0; i < Q; ++i) w += v[i] * a[i];
      w *= tau;
#pragma unroll
      for (int i = 0; i < Q; ++i) a[i] -= w * v[i];
    }
    if (lane == j) {
#pragma unroll
      for (int i = 0; i < Q; ++i)
        if (i > j) a[i] = 0.0;
    }
#pragma unroll
    for (int i = 0; i < Q; ++i) vs[j][i] = v[i];
    taus[j] = tau;
  }
  // column `lane` of X = H_0 ... H_{pc-1}: the reflectors applied to e_lane, last first
  double x[Q];
#pragma unroll
  for (int i = 0; i < Q; ++i) x[i] = (i == lane) ? 1.0 : 0.0;
#pragma unroll
  for (int j = Q - 1; j >= 0; --j) {
    if (taus[j] == 0.0) continue;
    double w = 0.0;
#pragma unroll
    for (int i = 0; i < Q; ++i) w += vs[j][i] * x[i];
    w *= taus[j];
#pragma unroll
    for (int i = 0; i < Q; ++i) x[i] -= w * vs[j][i];
  }
  // rows of R at the block's rounding floor are dropped (with their X column)
#pragma unroll
  for (int j = 0; j < Q; ++j) {
    const double dj = __shfl_sync(full, a[j], j);
    if (j < pc && fabs(dj) <= delta) {
      a[j] = 0.0;
      if (lane == j) {
#pragma unroll
        for (int i = 0; i < Q; ++i) x[i] = 0.0;
      }
    }
  }
  __syncwarp();
  if (own) {
#pragma unroll
    for (int j = 0; j < Q; ++j)
      if (j < pc) Rp[j * pc + perm] = a[j];
#pragma unroll
    for (int i = 0; i < Q; ++i) {
      if (i >= pc) continue;
      double acc = 0.0;
#pragma unroll
      for (int k = 0; k < Q; ++k)
        if (k < pc) acc += Qs[i * pc + k] * x[k];
      G[i * pc + lane] = acc;
    }
  }
  __syncwarp();
}

// ---------------------------------------------------------------------------
// Register-resident warp Householder QR of a tall chunk: lane l holds rows
// l + 32k (k < ROWS) of an (32*ROWS) x q matrix (q <= Q, zero rows padded).
// Same reflector convention as block_qr_t (beta = -sign(alpha) ||x||); on exit
// rows i > j of column j hold v_i (unit v_j implicit), rows <= j of columns
// >= j hold R (lanes < q, k = 0), tau[j] in every lane.
template <int Q, int ROWS>
__device__ __forceinline__ void warp_hh_regs(double (&x)[ROWS][Q], int q, double (&tau)[Q]) {
  const int lane = threadIdx.x & 31;
  const unsigned full = 0xffffffffu;
#pragma unroll
  for (int j = 0; j < Q; ++j) {
    tau[j] = 0.0;
    if (j >= q) continue;  // uniform
    double s[Q];
#pragma unroll
    for (int c = 0; c < Q; ++c) s[c] = 0.0;
#pragma unroll
    for (int k = 0; k < ROWS; ++k) {
      const bool below = (lane + 32 * k) > j;
#pragma unroll
      for (int c = j; c < Q; ++c)
        if (below) s[c] += x[k][j] * x[k][c];
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1)
#pragma unroll
      for (int c = j; c < Q; ++c) s[c] += __shfl_xor_sync(full, s[c], o);
    double xr[Q];
#pragma unroll
    for (int c = j; c < Q; ++c) xr[c] = __shfl_sync(full, x[0][c], j);
    const double alpha = xr[j], sig = s[j];
    double beta = alpha, t = 0.0, scale = 0.0;
    if (sig != 0.0) {
      const double nrm = sqrt_fast(alpha * alpha + sig);
      beta = alpha >= 0.0 ? -nrm : nrm;
      t = (beta - alpha) * rcp_fast(beta);
      scale = rcp_fast(alpha - beta);
    }
    double f[Q];
#pragma unroll
    for (int c = j + 1; c < Q; ++c) f[c] = (c < q) ? t * (xr[c] + scale * s[c]) : 0.0;
#pragma unroll
    for (int k = 0; k < ROWS; ++k) {
      const int i = lane + 32 * k;
      if (i > j) {
        const double v = x[k][j] * scale;
        x[k][j] = v;
#pragma unroll
        for (int c = j + 1; c < Q; ++c) x[k][c] -= f[c] * v;
      } else if (i == j) {
#pragma unroll
        for (int c = j + 1; c < Q; ++c) x[k][c] = xr[c] - f[c];
        x[k][j] = beta;
      }
    }
    tau[j] = t;
  }
}

// y <- H_0 ... H_{q-1} y for the reflectors left in x by warp_hh_regs.
template <int Q, int ROWS>
__device__ __forceinline__ void warp_apply_hh_regs(const double (&x)[ROWS][Q], int q,
                                                   const double (&tau)[Q], double (&y)[ROWS][Q]) {
  const int lane = threadIdx.x & 31;
  const unsigned full = 0xffffffffu;
#pragma unroll
  for (int j = Q - 1; j >= 0; --j) {
    if (j >= q || tau[j] == 0.0) continue;  // uniform
    double w[Q];
#pragma unroll
    for (int c = 0; c < Q; ++c) w[c] = 0.0;
#pragma unroll
    for (int k = 0; k < ROWS; ++k) {
      const int i = lane + 32 * k;
#pragma unroll
      for (int c = 0; c < Q; ++c) {
        if (i > j) w[c] += x[k][j] * y[k][c];
        else if (i == j) w[c] += y[k][c];
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1)
#pragma unroll
      for (int c = 0; c < Q; ++c) w[c] += __shfl_xor_sync(full, w[c], o);
#pragma unroll
    for (int k = 0; k < ROWS; ++k) {
      const int i = lane + 32 * k;
      const double v = (i > j) ? x[k][j] : ((i == j) ? 1.0 : 0.0);
#pragma unroll
      for (int c = 0; c < Q; ++c) y[k][c] -= tau[j] * w[c] * v;
    }
  }
}

// Stacked TSQR of the per-CTA R blocks of a flush (ncta blocks of pc x pc,
// block o row-major at part[o*pstride]), two levels, all in registers:
// warp w factors blocks [w*cpw, (w+1)*cpw) (lane = stacked row, loaded
// straight from L2), publishes its R_w in sRw (NWARP*Q*Q doubles, shared);
// after the CTA barrier the warp that owns block `me` factors the NWARP
// stacked R_w's (<= 32 rows) into Rout and forms rows me*pc.. of the stacked
// Q (= Q_w * (rows of Q_top)) into Qout (both pc x pc row-major, shared).
// Returns the owner warp.  Requires cpw*Q <= 32*ROWS and NWARP*Q <= 32.
template <int Q, int ROWS>
__device__ __forceinline__ int warp_stack_tsqr(const PartTab& tab, int ncta, int pc, int me,
                                               double* __restrict__ sRw,
                                               double* __restrict__ Rout,
                                               double* __restrict__ Qout) {
  static_assert(NWARP * Q <= 32, "top level must fit one warp");
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int cpw = (ncta + NWARP - 1) / NWARP;
  const int wo = me / cpw;
  const int b0 = w * cpw;
  int nb = ncta - b0;
  nb = nb < 0 ? 0 : (nb > cpw ? cpw : nb);
  const int rows = nb * pc;
  double x[ROWS][Q];
#pragma unroll
  for (int k = 0; k < ROWS; ++k) {
    const int i = lane + 32 * k;
    const int o = i / pc, lr = i - o * pc;
    const double* src = (i < rows) ? tab.at(2, b0 + o) + lr * pc : nullptr;
#pragma unroll
    for (int c = 0; c < Q; ++c) x[k][c] = (i < rows && c < pc) ? __ldcg(src + c) : 0.0;
  }
  double tau[Q];
  warp_hh_regs<Q, ROWS>(x, pc, tau);
  if (lane < Q) {
#pragma unroll
    for (int c = 0; c < Q; ++c) sRw[(w * Q + lane) * Q + c] = (c >= lane && lane < pc) ? x[0][c] : 0.0;
  }
  __syncthreads();
  if (w == wo) {
    // top level: row l = (warp l/Q, row l%Q) of the stacked R_w (pc-strided)
    double xt[1][Q];
#pragma unroll
    for (int c = 0; c < Q; ++c) xt[0][c] = sRw[lane * Q + c];
    // compact the rows so that the live ones are contiguous (row index tw*pc+tl)
    double xc[1][Q];
    {
      // destination row d = lane takes source row (d/pc)*Q + d%pc
      const int sw = lane / pc, sl = lane - sw * pc;
      const int sidx = (sw < NWARP) ? (sw * Q + sl) : 31;
#pragma unroll
      for (int c = 0; c < Q; ++c) {
        const double v = __shfl_sync(0xffffffffu, xt[0][c], sidx & 31);
        xc[0][c] = (sw < NWARP) ? v : 0.0;
      }
    }
    double tt[Q];
    warp_hh_regs<Q, 1>(xc, pc, tt);
    if (lane < pc) {
#pragma unroll
      for (int c = 0; c < Q; ++c)
        if (c < pc) Rout[lane * pc + c] = (c >= lane) ? xc[0][c] : 0.0;
    }
    // rows wo*pc .. wo*pc+pc-1 of Q_top = H..[I; 0]
    double e[1][Q];
#pragma unroll
    for (int c = 0; c < Q; ++c) e[0][c] = (lane == c && c < pc) ? 1.0 : 0.0;
    warp_apply_hh_regs<Q, 1>(xc, pc, tt, e);
    double y[ROWS][Q];
#pragma unroll
    for (int c = 0; c < Q; ++c) {
      const double tv = __shfl_sync(0xffffffffu, e[0][c], (wo * pc + lane) & 31);
      y[0][c] = (lane < pc) ? tv : 0.0;
    }
#pragma unroll
    for (int k = 1; k < ROWS; ++k)
#pragma unroll
      for (int c = 0; c < Q; ++c) y[k][c] = 0.0;
    warp_apply_hh_regs<Q, ROWS>(x, pc, tau, y);
    const int base = (me - b0) * pc;
#pragma unroll
    for (int k = 0; k < ROWS; ++k) {
      const int i = lane + 32 * k - base;
      if (i >= 0 && i < pc) {
#pragma unroll
        for (int c = 0; c < Q; ++c)
          if (c < pc) Qout[i * pc + c] = y[k][c];
      }
    }
    __syncwarp();
  }
  return wo;
}

// Same algorithm as warp_jacobi_reg, executed by JW warps (threads
// [0, 32*JW)): lane j still owns column j, warp w holds rows
// [w*NR, (w+1)*NR) of every column (NR = NJ/JW).  Per round each warp forms
// its partial of the column dot product from its rows; the partials meet in
// shared memory behind a named barrier (bar 1) and are summed in a fixed
// order, so every warp derives bit-identical rotations.  gbuf: 2*JW*32
// doubles (double-buffered by round parity).
template <int NJ, int JW>
__device__ __forceinline__ int multi_warp_jacobi(const double* __restrict__ Ain, int lda, int n,
                                                 double* __restrict__ Uo, double* __restrict__ Vo,
                                                 int ldo, double* __restrict__ s_sorted,
                                                 int* __restrict__ perm, double* __restrict__ gbuf) {
  constexpr int NR = NJ / JW;
  static_assert(NR * JW == NJ, "NJ must be a multiple of JW");
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const unsigned full = 0xffffffffu;
  const bool own = lane < n;
  const int row0 = w * NR;
  double a[NR], v[NR];
#pragma unroll
  for (int k = 0; k < NR; ++k) {
    const int i = row0 + k;
    a[k] = (own && i < n) ? Ain[i + lane * lda] : 0.0;
    v[k] = (i == lane) ? 1.0 : 0.0;
  }
  int buf = 0;
  auto xsum = [&](double part) {  // sum a per-lane value over the JW warps
    gbuf[(buf * JW + w) * 32 + lane] = part;
    asm volatile("bar.sync 1, %0;" ::"r"(JW * 32));
    double s = 0.0;
#pragma unroll
    for (int ww = 0; ww < JW; ++ww) s += gbuf[(buf * JW + ww) * 32 + lane];
    buf ^= 1;
    return s;
  };
  auto colnorm_part = [&]() {
    double s0 = 0.0, s1 = 0.0;
#pragma unroll
    for (int k = 0; k < NR; ++k) {
      if (k & 1) s1 += a[k] * a[k];
      else s0 += a[k] * a[k];
    }
    return s0 + s1;
  };
  double nrm = xsum(colnorm_part());
  const double tiny = warp_sum(nrm) * 1e-32;
  const double tol = 2.0 * DEPS * (double)(n > 8 ? n : 8);
  const double tol2 = tol * tol;
  const int ne = n + (n & 1);
  const int m1 = ne - 1;
  int nsweep = 0;
  for (int sweep = 0; sweep < 40 && n > 1; ++sweep) {
    nrm = xsum(colnorm_part());
    bool big = false, rotated = false;
    int pf = (lane < m1) ? (m1 - lane) % m1 : 0;
    for (int rnd = 0; rnd < m1; ++rnd) {
      int p = pf;
      if (lane == m1) p = rnd;
      else if (lane == rnd) p = m1;
      if (lane >= ne) p = lane;
      pf += 2;
      if (pf >= m1) pf -= m1;
      const bool act = own && p < n;
      const bool lo = lane < p;
      const double np = __shfl_sync(full, nrm, p & 31);
      double ap[NR];
      double g0 = 0.0, g1 = 0.0;
#pragma unroll
      for (int k = 0; k < NR; ++k) {
        ap[k] = __shfl_sync(full, a[k], p & 31);
        if (k & 1) g1 += a[k] * ap[k];
        else g0 += a[k] * ap[k];
      }
      // partial products are symmetric in (lane, p): both lanes of a pair
      // reduce identical values in the same order
      const double g = xsum(g0 + g1);
      const double al = lo ? nrm : np, be = lo ? np : nrm;
      // rotation parameters computed without branches (selects only): the
      // tangent in fp32 after an exact power-of-two rescale (only its
      // convergence effect depends on its accuracy), c in fp64 so that
      // c^2 + s^2 = 1 to working precision; t = 0 gives c = 1, s = 0 exactly
      const double g2 = g * g, ab = al * be;
      const bool ok = act && al > tiny && be > tiny;
      big = big || (ok && g2 > 1e-16 * ab);
      const bool rot = ok && g2 > tol2 * ab;
      const double d = be - al;
      int e = ilog2_normal(fmax(fmax(fabs(d), fabs(g)), 1e-300));
      e = e > 1000 ? 1000 : e;
      const double scl = pow2i(-e);
      const float df = (float)(d * scl), gf = (float)(g * scl);
      const float hyp = df * df + 4.0f * gf * gf;
      const float tb = __fdividef(2.0f * gf, fabsf(df) + hyp * rsqrtf(hyp));
      const float tf = (fabsf(gf) < 1e-4f * fabsf(df)) ? __fdividef(gf, df) : (df < 0.0f ? -tb : tb);
      const double t = rot ? (double)tf : 0.0;
      const double t2 = t * t;
      const double cser = 1.0 - t2 * (0.5 - 0.375 * t2);
      const double c = (t2 < 1e-8) ? cser : rsqrt_u(1.0 + t2);
      const double sl = lo ? -c * t : c * t;
      // unconditional update (c = 1, sl = 0 leaves a column bit-identical):
      // shuffles outside data-dependent branches compile to plain SHFL
#pragma unroll
      for (int k = 0; k < NR; ++k) {
        a[k] = c * a[k] + sl * ap[k];
        const double vp = __shfl_sync(full, v[k], p & 31);
        v[k] = c * v[k] + sl * vp;
      }
      const double nn = lo ? (al - t * g) : (be + t * g);
      nrm = rot ? nn : nrm;
      rotated = rotated || rot;
    }
    ++nsweep;
    if (!__any_sync(full, rotated) || !__any_sync(full, big)) break;
  }
  const double nfin = xsum(colnorm_part());  // every lane takes part in the barrier
  const double sv = own ? sqrt_fast(nfin) : 0.0;
  int rk = 0;
  for (int j = 0; j < n; ++j) {
    const double sj = __shfl_sync(full, sv, j);
    if (sj > sv || (sj == sv && j < lane)) ++rk;
  }
  if (own) {
    if (w == 0) {
      perm[rk] = lane;
      s_sorted[rk] = sv;
    }
    const double inv = sv > 0.0 ? rcp_fast(sv) : 0.0;
#pragma unroll
    for (int k = 0; k < NR; ++k) {
      const int i = row0 + k;
      if (i < n) {
        Uo[i + rk * ldo] = a[k] * inv;
        Vo[i + rk * ldo] = v[k];
      }
    }
  }
  asm volatile("bar.sync 1, %0;" ::"r"(JW * 32));
  return nsweep;
}

}  // namespace lrk
