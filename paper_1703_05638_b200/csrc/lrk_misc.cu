// lrk_misc.cu — streaming kernels around the persistent sweep/truncation:
// matrix-free stencil SpMM, sign canonicalisation, low-rank inner products,
// dense CGS2 for the IC-mode Arnoldi, row gathers/scatters, column scalings.
#include "lrk_device.cuh"
#include "lrk_misc.h"

namespace lrk {

// ---------------------------------------------------------------- stencil
// K.apply / apply_adjoint spatial part (forward.py:79-95):
// (S x) = m_scale (x + tau L x) for the constant-coefficient box stencils of
// discretize.py:90-127 (5-point FD) and their config extensions (Q1-lumped
// 9-point, 3-D 7-point), generated on the fly (no CSR), zero Dirichlet data.
// One thread per output entry, coalesced along x1; neighbours come through L1.
// Local wind at interior node (i1, i2, i3): w0 + (2 x2 (1 - x1^2), -2 x1 (1 - x2^2), 0).
__device__ __forceinline__ double wind_at(const StencilArgs& a, int ax, int i1, int i2) {
  const double x1 = a.h * (i1 + 1), x2 = a.h * (i2 + 1);
  if (ax == 0) return a.w0[0] + 2.0 * x2 * (1.0 - x1 * x1);
  if (ax == 1) return a.w0[1] - 2.0 * x1 * (1.0 - x2 * x2);
  return a.w0[2];
}

// Per-node first-order upwind (row i of W, or of W^T for the adjoint):
// row q: diag += |w_a(q)|/h; entry (q, q - e_a) = -w_a(q)/h if w_a(q) > 0,
// entry (q, q + e_a) = +w_a(q)/h if w_a(q) < 0.
__device__ __forceinline__ double var_upwind(const StencilArgs& a, const double* x, int64_t i,
                                             int i1, int i2, int i3, int64_t plane) {
  const int n = a.n;
  const double ih = 1.0 / a.h;
  double acc = 0.0;
  const int idx[3] = {i1, i2, i3};
  const int64_t stride[3] = {1, n, plane};
  for (int ax = 0; ax < a.dim; ++ax) {
    const double w = wind_at(a, ax, i1, i2);
    acc += fabs(w) * ih * x[i];
    if (!a.adjoint) {
      if (w > 0.0 && idx[ax] > 0) acc -= w * ih * x[i - stride[ax]];
      if (w < 0.0 && idx[ax] < n - 1) acc += w * ih * x[i + stride[ax]];
    } else {
      // column i of W: rows i + e_a (their lower neighbour is i) and i - e_a
      if (idx[ax] < n - 1) {
        const double wp = wind_at(a, ax, i1 + (ax == 0), i2 + (ax == 1));
        if (wp > 0.0) acc -= wp * ih * x[i + stride[ax]];
      }
      if (idx[ax] > 0) {
        const double wm = wind_at(a, ax, i1 - (ax == 0), i2 - (ax == 1));
        if (wm < 0.0) acc += wm * ih * x[i - stride[ax]];
      }
    }
  }
  return acc;
}

__global__ void stencil_kernel(StencilArgs a) {
  const int c = blockIdx.y;
  const int n = a.n;
  const int64_t plane = (int64_t)n * n;
  const int64_t n_x = a.dim == 3 ? plane * n : plane;
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n_x || c >= a.ncols) return;
  const double* x = a.X + (int64_t)c * a.ldx;
  const int i1 = (int)(i % n), i2 = (int)((i / n) % n), i3 = (int)(i / plane);
  const double xc = x[i];
  double lx = 0.0;
  const int d3lo = a.dim == 3 ? -1 : 0, d3hi = a.dim == 3 ? 1 : 0;
  for (int d3 = d3lo; d3 <= d3hi; ++d3) {
    if (i3 + d3 < 0 || i3 + d3 >= (a.dim == 3 ? n : 1)) continue;
#pragma unroll
    for (int d2 = -1; d2 <= 1; ++d2) {
      if (i2 + d2 < 0 || i2 + d2 >= n) continue;
#pragma unroll
      for (int d1 = -1; d1 <= 1; ++d1) {
        const double cf = a.coef[(d3 + 1) * 9 + (d2 + 1) * 3 + (d1 + 1)];
        if (cf == 0.0 || i1 + d1 < 0 || i1 + d1 >= n) continue;
        lx += cf * x[i + d1 + (int64_t)d2 * n + (int64_t)d3 * plane];
      }
    }
  }
  if (a.wind_field) lx += var_upwind(a, x, i, i1, i2, i3, plane);
  const double sx = a.m_scale * (xc + a.tau * lx);
  a.Y[i + (int64_t)c * a.ldy] = a.Bres ? a.Bres[i + (int64_t)c * a.ldbres] - sx : sx;
}

// out2[:, c] = shift(W2[:, c]) (forward: down one row; adjoint: up one row)
__global__ void shift_kernel(const double* W2, int64_t ld2, int n_t, int ncols, int adjoint,
                             double* out, int64_t ldo, const double* W1, int64_t ld1,
                             int64_t n_x, double neg_m, double* out1, int64_t ldo1) {
  const int c = blockIdx.y;
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= ncols) return;
  if (i < n_t) {
    double v;
    if (adjoint) v = (i + 1 < n_t) ? W2[(i + 1) + (int64_t)c * ld2] : 0.0;
    else v = (i > 0) ? W2[(i - 1) + (int64_t)c * ld2] : 0.0;
    out[i + (int64_t)c * ldo] = v;
  }
  if (i < n_x) out1[i + (int64_t)c * ldo1] = neg_m * W1[i + (int64_t)c * ld1];
}

// ---------------------------------------------------------- utilities
// Y[:, c] = alpha * X[:, c] / (delta + gamma * lam): the spectral image of the
// config prior (delta I + gamma L)^{-1}.
__global__ void prior_scale_kernel(const double* X, int64_t ldx, const double* lam, int64_t n,
                                   int ncols, const int* ncols_dev, double alpha, double delta,
                                   double gamma, double* Y, int64_t ldy) {
  const int c = blockIdx.y;
  const int nc = ncols_dev ? min(ncols, *ncols_dev) : ncols;
  if (c >= nc) return;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    Y[i + (int64_t)c * ldy] = alpha * X[i + (int64_t)c * ldx] / (delta + gamma * lam[i]);
}

// y += B w, B n x rb (ld ldb), w strided by ldw (one row of a time factor):
// the rhs term B~ w2_k of a physical-space sweep step.
__global__ void rank_axpy_kernel(const double* B, int64_t ldb, int rb, const double* w,
                                 int64_t ldw, double* y, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    double acc = y[i];
    for (int j = 0; j < rb; ++j) acc += B[i + (int64_t)j * ldb] * w[(int64_t)j * ldw];
    y[i] = acc;
  }
}

// flag |= (||r||^2 > tol2 ||b||^2): device-side convergence check of an
// iterative step solve (grid-wide; the last block to finish reduces the
// per-block partials in a fixed order and re-arms the counter).
__global__ void resid_flag_kernel(const double* r, const double* b, int64_t n, double tol2,
                                  double* part, unsigned* counter, int* flag) {
  __shared__ double srr[NWARP], sbb[NWARP];
  __shared__ bool last;
  double rr = 0.0, bb = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    rr += r[i] * r[i];
    bb += b[i] * b[i];
  }
  rr = warp_sum(rr);
  bb = warp_sum(bb);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (lane == 0) { srr[w] = rr; sbb[w] = bb; }
  __syncthreads();
  if (threadIdx.x == 0) {
    double a = 0.0, c = 0.0;
    for (int k = 0; k < (int)(blockDim.x >> 5); ++k) { a += srr[k]; c += sbb[k]; }
    part[2 * blockIdx.x] = a;
    part[2 * blockIdx.x + 1] = c;
    __threadfence();
    last = atomicAdd(counter, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (last && threadIdx.x == 0) {
    __threadfence();
    double a = 0.0, c = 0.0;
    for (unsigned k = 0; k < gridDim.x; ++k) { a += __ldcg(part + 2 * k); c += __ldcg(part + 2 * k + 1); }
    if (a > tol2 * c) *flag = 1;
    *counter = 0;
  }
}

// out = a x + b y (y may be NULL when b == 0)
__global__ void axpby_kernel(const double* x, double a, const double* y, double b, double* out,
                             int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = a * x[i] + (b != 0.0 ? b * y[i] : 0.0);
}

// Zero the rows k of a time factor with (k+1) % every != 0 (time-subsampled
// sensors).
__global__ void mask_time_rows_kernel(double* W2, int64_t ld2, int n_t, int ncols, int every) {
  const int c = blockIdx.y;
  if (c >= ncols) return;
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n_t; k += gridDim.x * blockDim.x)
    if ((k + 1) % every != 0) W2[k + (int64_t)c * ld2] = 0.0;
}

__global__ void scale_rows_kernel(const double* X, int64_t ldx, const double* s, int64_t n,
                                  int ncols, const int* ncols_dev, double alpha, double* Y,
                                  int64_t ldy) {
  const int c = blockIdx.y;
  const int nc = ncols_dev ? min(ncols, *ncols_dev) : ncols;
  if (c >= nc) return;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double f = s ? s[i] * alpha : alpha;
    Y[i + (int64_t)c * ldy] = f * X[i + (int64_t)c * ldx];
  }
}

// Y[:, c] = X[:, c] * (alpha * colscale[c]) for c < ncols (device count)
__global__ void scale_cols_kernel(const double* X, int64_t ldx, int64_t n, const double* colscale,
                                  const int* ncols_dev, int ncols, double alpha, double* Y,
                                  int64_t ldy) {
  const int c = blockIdx.y;
  const int nc = ncols_dev ? min(ncols, *ncols_dev) : ncols;
  if (c >= nc) return;
  const double f = alpha * (colscale ? colscale[c] : 1.0);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    Y[i + (int64_t)c * ldy] = f * X[i + (int64_t)c * ldx];
}

// y = U * (sigma .* V[row, :]) over r (device) columns: the IC extract
// M * Q.column(0) (forward.py:111-112) before the inverse transform.
__global__ void column_eval_kernel(const double* U, int64_t ldu, int64_t n, const double* sigma,
                                   const double* V, int64_t ldv, int row, const int* r_dev,
                                   double* y) {
  const int r = *r_dev;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    double acc = 0.0;
    for (int c = 0; c < r; ++c) acc += U[i + (int64_t)c * ldu] * (sigma[c] * V[row + (int64_t)c * ldv]);
    y[i] = acc;
  }
}

__global__ void gather_rows_kernel(const double* X, int64_t ldx, const int32_t* idx, int nidx,
                                   const int* ncols_dev, int ncols, double* Y, int64_t ldy) {
  const int c = blockIdx.y;
  const int nc = ncols_dev ? min(ncols, *ncols_dev) : ncols;
  if (c >= nc) return;
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < nidx; k += gridDim.x * blockDim.x)
    Y[k + (int64_t)c * ldy] = X[idx[k] + (int64_t)c * ldx];
}

__global__ void scatter_rows_kernel(const double* X, int64_t ldx, const int32_t* idx, int nidx,
                                    const int* ncols_dev, int ncols, double* Y, int64_t ldy) {
  const int c = blockIdx.y;
  const int nc = ncols_dev ? min(ncols, *ncols_dev) : ncols;
  if (c >= nc) return;
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < nidx; k += gridDim.x * blockDim.x)
    Y[idx[k] + (int64_t)c * ldy] = X[k + (int64_t)c * ldx];
}

__global__ void fill_kernel(double* X, int64_t ldx, int64_t n, int ncols, double v) {
  const int c = blockIdx.y;
  if (c >= ncols) return;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    X[i + (int64_t)c * ldx] = v;
}

// --------------------------------------------------------- _svd_flip
// Per-block partial argmax |U[:, c]| (first index on ties), then finalize
// + apply: largest-|entry| of each column positive (lowrank.py:114-121).
__global__ void __launch_bounds__(256) flip_partial_kernel(const double* U, int64_t ldu,
                                                           int64_t n, const int* r_dev, int rcap,
                                                           double* part) {
  const int c = blockIdx.y;
  const int r = r_dev ? min(rcap, *r_dev) : rcap;
  if (c >= r) return;
  __shared__ double sb[8], sv[8];
  __shared__ long long si[8];
  double best = -1.0, bval = 0.0;
  long long bidx = 0;
  const int64_t per = (n + gridDim.x - 1) / gridDim.x;
  const int64_t lo = per * blockIdx.x, hi = min(n, lo + per);
  for (int64_t i = lo + threadIdx.x; i < hi; i += blockDim.x) {
    const double x = U[i + (int64_t)c * ldu];
    if (fabs(x) > best) { best = fabs(x); bidx = i; bval = x; }
  }
  for (int o = 16; o > 0; o >>= 1) {
    const double ob = __shfl_xor_sync(0xffffffffu, best, o);
    const long long oi = __shfl_xor_sync(0xffffffffu, bidx, o);
    const double ov = __shfl_xor_sync(0xffffffffu, bval, o);
    if (ob > best || (ob == best && oi < bidx)) { best = ob; bidx = oi; bval = ov; }
  }
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) { sb[w] = best; si[w] = bidx; sv[w] = bval; }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int k = 1; k < (int)(blockDim.x >> 5); ++k)
      if (sb[k] > best || (sb[k] == best && si[k] < bidx)) { best = sb[k]; bidx = si[k]; bval = sv[k]; }
    double* q = part + ((int64_t)c * gridDim.x + blockIdx.x) * 3;
    q[0] = best; q[1] = (double)bidx; q[2] = bval;
  }
}

__global__ void flip_apply_kernel(double* U, int64_t ldu, int64_t n_x, double* V, int64_t ldv,
                                  int n_t, const int* r_dev, int rcap, const double* part,
                                  int nparts) {
  const int c = blockIdx.y;
  const int r = r_dev ? min(rcap, *r_dev) : rcap;
  if (c >= r) return;
  __shared__ double sgn;
  if (threadIdx.x == 0) {
    double best = -1.0, bval = 0.0, bidx = 0.0;
    for (int k = 0; k < nparts; ++k) {
      const double* q = part + ((int64_t)c * nparts + k) * 3;
      if (q[0] > best || (q[0] == best && q[1] < bidx)) { best = q[0]; bidx = q[1]; bval = q[2]; }
    }
    sgn = (bval < 0.0) ? -1.0 : 1.0;
  }
  __syncthreads();
  if (sgn > 0.0) return;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n_x;
       i += (int64_t)gridDim.x * blockDim.x)
    U[i + (int64_t)c * ldu] = -U[i + (int64_t)c * ldu];
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n_t;
       i += (int64_t)gridDim.x * blockDim.x)
    V[i + (int64_t)c * ldv] = -V[i + (int64_t)c * ldv];
}

// ---------------------------------------------------- Gram partials
// part[blk][i*nb + j] = sum over the block's rows of A[:, i] B[:, j]
__global__ void __launch_bounds__(NT) gram_partial_kernel(const double* A, int64_t lda, int na,
                                                          const double* B, int64_t ldb, int nb,
                                                          int64_t n, double* part) {
  __shared__ double out[NMAX * 4 > NT ? NMAX * 4 : NT];
  __shared__ double scr[NT];
  const int64_t per = (n + gridDim.x - 1) / gridDim.x;
  const int64_t lo = per * blockIdx.x, hi = min(n, lo + per);
  const int nout = na * nb;
  // chunk the output so the shared buffer suffices
  for (int i0 = 0; i0 < na; ) {
    int ni = na - i0;
    if (ni * nb > NT) ni = NT / nb > 0 ? NT / nb : 1;
    cta_tn(A + lo + (int64_t)i0 * lda, lda, ni, B + lo, ldb, nb, (int)(hi - lo), out, scr);
    for (int o = threadIdx.x; o < ni * nb; o += NT)
      part[(int64_t)blockIdx.x * nout + i0 * nb + o] = out[o];
    __syncthreads();
    i0 += ni;
  }
}

// dot = sum_{ij} G1[ij] * G2[ij] with G1, G2 the reduced partials.
__global__ void dot_finalize_kernel(const double* p1, int n1, const double* p2, int n2, int nout,
                                    double* out) {
  __shared__ double red[32];
  double acc = 0.0;
  for (int o = threadIdx.x; o < nout; o += blockDim.x) {
    double g1 = 0.0, g2 = 0.0;
    for (int k = 0; k < n1; ++k) g1 += p1[(int64_t)k * nout + o];
    for (int k = 0; k < n2; ++k) g2 += p2[(int64_t)k * nout + o];
    acc += g1 * g2;
  }
  acc = warp_sum(acc);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += red[w];
    *out = s;
  }
}

// reduce partials (nparts x nout) into out (nout), optionally accumulate
__global__ void reduce_parts_kernel(const double* p, int nparts, int nout, double* out,
                                    double* acc_out) {
  for (int o = blockIdx.x * blockDim.x + threadIdx.x; o < nout; o += gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int k = 0; k < nparts; ++k) s += p[(int64_t)k * nout + o];
    out[o] = s;
    if (acc_out) acc_out[o] += s;
  }
}

// w -= Q h  (n rows, k columns)
__global__ void sub_qh_kernel(const double* Q, int64_t ldq, int k, const double* h, double* w,
                              int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    double acc = 0.0;
    for (int c = 0; c < k; ++c) acc += Q[i + (int64_t)c * ldq] * h[c];
    w[i] -= acc;
  }
}

// y = Q c
__global__ void combine_kernel(const double* Q, int64_t ldq, int k, const double* cf, double* y,
                               int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    double acc = 0.0;
    for (int c = 0; c < k; ++c) acc += Q[i + (int64_t)c * ldq] * cf[c];
    y[i] = acc;
  }
}

}  // namespace lrk
