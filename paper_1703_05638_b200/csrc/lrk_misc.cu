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
  if (a.Ycopy) a.Ycopy[i + (int64_t)c * a.ldycopy] = a.copy_scale * xc;
}

// Upwind terms from the six axis neighbours (xm[a] = x_{i - e_a}, xp[a] =
// x_{i + e_a}, zero outside the domain: the Dirichlet data), same arithmetic
// as var_upwind.
__device__ __forceinline__ double upwind_nb(const StencilArgs& a, int i1, int i2, double xc,
                                            const double (&xm)[3], const double (&xp)[3]) {
  const double ih = 1.0 / a.h;
  double acc = 0.0;
#pragma unroll
  for (int ax = 0; ax < 3; ++ax) {
    if (ax >= a.dim) break;
    const double w = wind_at(a, ax, i1, i2);
    acc += fabs(w) * ih * xc;
    if (!a.adjoint) {
      if (w > 0.0) acc -= w * ih * xm[ax];
      if (w < 0.0) acc += w * ih * xp[ax];
    } else {
      const double wp = wind_at(a, ax, i1 + (ax == 0), i2 + (ax == 1));
      if (wp > 0.0) acc -= wp * ih * xp[ax];
      const double wm = wind_at(a, ax, i1 - (ax == 0), i2 - (ax == 1));
      if (wm < 0.0) acc += wm * ih * xm[ax];
    }
  }
  return acc;
}

// 2-D box stencil (5- or 9-point, optional upwind wind) on a shared-memory
// tile: CTA = 32 x 8 threads, 32 x 32 outputs (4 rows per thread); the tile
// with its one-node halo is staged once (coalesced rows, zero padding = the
// Dirichlet data), so every input is read from HBM once; 16 B per output.
constexpr int ST2 = 32;
__global__ void __launch_bounds__(256) stencil2d_kernel(StencilArgs a) {
  __shared__ double tile[ST2 + 2][ST2 + 3];
  const int c = blockIdx.z;
  const int n = a.n;
  const int x0 = blockIdx.x * ST2, y0 = blockIdx.y * ST2;
  const int tx = threadIdx.x, ty = threadIdx.y, tid = ty * 32 + tx;
  const double* x = a.X + (int64_t)c * a.ldx;
  for (int idx = tid; idx < (ST2 + 2) * (ST2 + 2); idx += 256) {
    const int ly = idx / (ST2 + 2), lx = idx - ly * (ST2 + 2);
    const int gx = x0 + lx - 1, gy = y0 + ly - 1;
    tile[ly][lx] = (gx >= 0 && gx < n && gy >= 0 && gy < n) ? x[(int64_t)gy * n + gx] : 0.0;
  }
  __syncthreads();
  double cf[9];
#pragma unroll
  for (int q = 0; q < 9; ++q) cf[q] = a.coef[9 + q];
  const int gx = x0 + tx;
#pragma unroll
  for (int rr = 0; rr < ST2 / 8; ++rr) {
    const int ly = ty + 8 * rr, gy = y0 + ly;
    if (gx >= n || gy >= n) continue;
    double lx = 0.0;
#pragma unroll
    for (int d2 = 0; d2 < 3; ++d2)
#pragma unroll
      for (int d1 = 0; d1 < 3; ++d1) lx += cf[d2 * 3 + d1] * tile[ly + d2][tx + d1];
    const double xc = tile[ly + 1][tx + 1];
    if (a.wind_field) {
      const double xm[3] = {tile[ly + 1][tx], tile[ly][tx + 1], 0.0};
      const double xp[3] = {tile[ly + 1][tx + 2], tile[ly + 2][tx + 1], 0.0};
      lx += upwind_nb(a, gx, gy, xc, xm, xp);
    }
    const double sx = a.m_scale * (xc + a.tau * lx);
    const int64_t i = (int64_t)gy * n + gx;
    a.Y[i + (int64_t)c * a.ldy] = a.Bres ? a.Bres[i + (int64_t)c * a.ldbres] - sx : sx;
    if (a.Ycopy) a.Ycopy[i + (int64_t)c * a.ldycopy] = a.copy_scale * xc;
  }
}

// 3-D 7-point stencil (optional upwind wind): CTA = 32 x 8 threads over an
// (x1, x2) tile, marching ST3Z planes along x3 with the x3 neighbours in
// registers and the current plane (+ halo) in shared memory; 16 B per output.
constexpr int ST3Z = 16;
__global__ void __launch_bounds__(256) stencil3d7_kernel(StencilArgs a, int nzb) {
  __shared__ double tile[8 + 2][32 + 3];
  const int zb = blockIdx.z % nzb, c = blockIdx.z / nzb;
  const int n = a.n;
  const int64_t plane = (int64_t)n * n;
  const int x0 = blockIdx.x * 32, y0 = blockIdx.y * 8;
  const int tx = threadIdx.x, ty = threadIdx.y, tid = ty * 32 + tx;
  const int gx = x0 + tx, gy = y0 + ty;
  const bool in = gx < n && gy < n;
  const double* x = a.X + (int64_t)c * a.ldx;
  const int z0 = zb * ST3Z, z1 = min(n, z0 + ST3Z);
  const double cxm = a.coef[12], cxp = a.coef[14], cym = a.coef[10], cyp = a.coef[16];
  const double czm = a.coef[4], czp = a.coef[22], cc = a.coef[13];
  const int64_t col = (int64_t)gy * n + gx;
  // x3 neighbours in a register queue, loads issued two planes ahead (and
  // the halo one plane ahead) so each thread keeps several loads in flight
  auto ld = [&](int z) { return (in && z >= 0 && z < n) ? x[(int64_t)z * plane + col] : 0.0; };
  double below = ld(z0 - 1), cur = ld(z0), a1 = ld(z0 + 1);
  // halo slot of this thread (84 of the 340 tile entries; threads < 84)
  const bool hh = tid < 2 * 34 + 2 * 8;
  int hy = 0, hx = 0;
  if (tid < 34) { hy = 0; hx = tid; }
  else if (tid < 68) { hy = 9; hx = tid - 34; }
  else if (tid < 76) { hy = tid - 68 + 1; hx = 0; }
  else if (hh) { hy = tid - 76 + 1; hx = 33; }
  const int hgx = x0 + hx - 1, hgy = y0 + hy - 1;
  const bool hin = hh && hgx >= 0 && hgx < n && hgy >= 0 && hgy < n;
  const int64_t hcol = (int64_t)hgy * n + hgx;
  double hv = hin ? x[(int64_t)z0 * plane + hcol] : 0.0;
  for (int z = z0; z < z1; ++z) {
    const double a2 = ld(z + 2);
    const double hvn = (hin && z + 1 < z1) ? x[(int64_t)(z + 1) * plane + hcol] : 0.0;
    __syncthreads();  // the previous plane's tile is consumed
    tile[ty + 1][tx + 1] = cur;
    if (hh) tile[hy][hx] = hv;
    __syncthreads();
    if (in) {
      const double xl = tile[ty + 1][tx], xr = tile[ty + 1][tx + 2];
      const double xd = tile[ty][tx + 1], xu = tile[ty + 2][tx + 1];
      double lx = cc * cur + cxm * xl + cxp * xr + cym * xd + cyp * xu + czm * below + czp * a1;
      if (a.wind_field) {
        const double xm[3] = {xl, xd, below};
        const double xp[3] = {xr, xu, a1};
        lx += upwind_nb(a, gx, gy, cur, xm, xp);
      }
      const double sx = a.m_scale * (cur + a.tau * lx);
      const int64_t i = (int64_t)z * plane + col;
      a.Y[i + (int64_t)c * a.ldy] = a.Bres ? a.Bres[i + (int64_t)c * a.ldbres] - sx : sx;
      if (a.Ycopy) a.Ycopy[i + (int64_t)c * a.ldycopy] = a.copy_scale * cur;
    }
    below = cur;
    cur = a1;
    a1 = a2;
    hv = hvn;
  }
}

// Launch the tiled kernel that fits the operator (2-D box; 3-D 7-point),
// the generic one otherwise.  a.ncols columns.
void launch_stencil(const StencilArgs& a, cudaStream_t s) {
  const int n = a.n;
  if (a.dim == 2) {
    dim3 grid((n + ST2 - 1) / ST2, (n + ST2 - 1) / ST2, a.ncols);
    stencil2d_kernel<<<grid, dim3(32, 8), 0, s>>>(a);
    return;
  }
  bool seven = true;
  for (int q = 0; q < 27; ++q) {
    const int d3 = q / 9, d2 = (q / 3) % 3, d1 = q % 3;
    const int nnz_axes = (d3 != 1) + (d2 != 1) + (d1 != 1);
    if (nnz_axes > 1 && a.coef[q] != 0.0) seven = false;
  }
  if (seven) {
    const int nzb = (n + ST3Z - 1) / ST3Z;
    dim3 grid((n + 31) / 32, (n + 7) / 8, nzb * a.ncols);
    stencil3d7_kernel<<<grid, dim3(32, 8), 0, s>>>(a, nzb);
    return;
  }
  const int64_t nx = (int64_t)n * n * n;
  stencil_kernel<<<dim3((unsigned)((nx + 255) / 256), a.ncols), 256, 0, s>>>(a);
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

// ---------------------------------------------- Gram partials (DMMA)
// part[blockIdx.x * pstride + i*ldo + j] = sum over the CTA's rows of
// A[:, i] B[:, j]  (i < na <= 8*TA, j < nb <= 8*TB).  Every warp streams its
// own contiguous slice of the CTA's rows — each row of A and B is read once
// from HBM, in 4-row k-steps with U steps of loads in flight — and
// accumulates ALL TA x TB output tiles with m8n8k4 DMMA (lane (g,t) loads
// A[k+t, 8i+g] and B[k+t, 8j+g]: every 32-byte sector fully used).  The
// warp partials meet in shared memory in warp order (deterministic).
// Bound: HBM for r <~ 40, the FP64 tensor pipe beyond (2 n r_a r_b flops
// per 8 n (r_a + r_b) bytes).
template <int TA, int TB>
__global__ void __launch_bounds__(NT, 1)
    gram_dmma_kernel(const double* __restrict__ A, int64_t lda, int na,
                     const double* __restrict__ B, int64_t ldb, int nb, int64_t n,
                     double* __restrict__ part, int ldo, int64_t pstride) {
  // the 64-tile case splits the B tiles over two warp halves (64 accumulators
  // per thread instead of 128: no spills); the halves read the same rows of A
  // at the same time (L1 hits)
  constexpr int WB = (TA * TB >= 64) ? 2 : 1;
  constexpr int TBW = TB / WB;
  constexpr int NS = NWARP / WB;  // row slices
  __shared__ double buf[64 * 64];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int half = warp % WB, slice = warp / WB;
  const int64_t per = (n + gridDim.x - 1) / gridDim.x;
  const int64_t lo = per * blockIdx.x, hi = min(n, lo + per);
  const int64_t cnt = hi > lo ? hi - lo : 0;
  const int64_t wchunk = (((cnt + NS - 1) / NS) + 3) & ~int64_t(3);
  const int64_t w0 = lo + slice * wchunk, w1 = min(hi, w0 + wchunk);
  // column 8i+g of A is Ab + i*la8 (one base pointer per operand)
  const double* Ab = A + (int64_t)g * lda;
  const double* Bb = B + (int64_t)(8 * TBW * half + g) * ldb;
  const int64_t la8 = 8 * lda, lb8 = 8 * ldb;
  const int jb0 = 8 * TBW * half;
  double acc[TA][TBW][2];
#pragma unroll
  for (int i = 0; i < TA; ++i)
#pragma unroll
    for (int j = 0; j < TBW; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  constexpr int U = (TA * TBW >= 32) ? 1 : (TA * TBW >= 8 ? 2 : 4);
  // software pipeline: the fragments of the next U k-steps are loaded while
  // the DMMAs of the current ones issue
  double av[U][TA], bv[U][TBW];
  auto load = [&](int64_t kb, double (&xa)[U][TA], double (&xb)[U][TBW]) {
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t k = kb + 4 * u + t;
      const bool ok = k < w1;
#pragma unroll
      for (int i = 0; i < TA; ++i) xa[u][i] = (ok && 8 * i + g < na) ? __ldg(Ab + i * la8 + k) : 0.0;
#pragma unroll
      for (int j = 0; j < TBW; ++j)
        xb[u][j] = (ok && jb0 + 8 * j + g < nb) ? __ldg(Bb + j * lb8 + k) : 0.0;
    }
  };
  if (w0 < w1) load(w0, av, bv);
  for (int64_t k0 = w0; k0 < w1; k0 += 4 * U) {
    double an[U][TA], bn[U][TBW];
    load(k0 + 4 * U, an, bn);  // predicated off past w1
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      for (int i = 0; i < TA; ++i)
#pragma unroll
        for (int j = 0; j < TBW; ++j) dmma884(acc[i][j][0], acc[i][j][1], av[u][i], bv[u][j]);
#pragma unroll
    for (int u = 0; u < U; ++u) {
#pragma unroll
      for (int i = 0; i < TA; ++i) av[u][i] = an[u][i];
#pragma unroll
      for (int j = 0; j < TBW; ++j) bv[u][j] = bn[u][j];
    }
  }
  // warp partials in slice order (each output element has exactly NS adds)
  for (int sl = 0; sl < NS; ++sl) {
    if (slice == sl) {
#pragma unroll
      for (int i = 0; i < TA; ++i)
#pragma unroll
        for (int j = 0; j < TBW; ++j)
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int ii = 8 * i + g, jj = jb0 + 8 * j + 2 * t + h;
            if (ii < na && jj < nb) {
              const double v = acc[i][j][h];
              buf[ii * nb + jj] = (sl == 0) ? v : buf[ii * nb + jj] + v;
            }
          }
    }
    __syncthreads();
  }
  for (int o = threadIdx.x; o < na * nb; o += NT)
    part[(int64_t)blockIdx.x * pstride + (int64_t)(o / nb) * ldo + (o % nb)] = buf[o];
}

template <int TA>
static void gram_tb(int tb, const double* A, int64_t lda, int na, const double* B, int64_t ldb,
                    int nb, int64_t n, double* part, int ldo, int64_t pstride, int nparts,
                    cudaStream_t s) {
  if (tb <= 1) gram_dmma_kernel<TA, 1><<<nparts, NT, 0, s>>>(A, lda, na, B, ldb, nb, n, part, ldo, pstride);
  else if (tb <= 2) gram_dmma_kernel<TA, 2><<<nparts, NT, 0, s>>>(A, lda, na, B, ldb, nb, n, part, ldo, pstride);
  else if (tb <= 4) gram_dmma_kernel<TA, 4><<<nparts, NT, 0, s>>>(A, lda, na, B, ldb, nb, n, part, ldo, pstride);
  else gram_dmma_kernel<TA, 8><<<nparts, NT, 0, s>>>(A, lda, na, B, ldb, nb, n, part, ldo, pstride);
}

// nparts x (na*nb) partials of A^T B over n rows (row-major i*nb + j per
// part); column blocks of 64 beyond the kernel's tile bound.
void launch_gram(const double* A, int64_t lda, int na, const double* B, int64_t ldb, int nb,
                 int64_t n, double* part, int nparts, cudaStream_t s) {
  const int64_t pstride = (int64_t)na * nb;
  for (int a0 = 0; a0 < na; a0 += 64)
    for (int b0 = 0; b0 < nb; b0 += 64) {
      const int ca = na - a0 < 64 ? na - a0 : 64, cb = nb - b0 < 64 ? nb - b0 : 64;
      const int ta = (ca + 7) / 8, tb = (cb + 7) / 8;
      const double* Ab = A + (int64_t)a0 * lda;
      const double* Bb = B + (int64_t)b0 * ldb;
      double* pb = part + (int64_t)a0 * nb + b0;
      if (ta <= 1) gram_tb<1>(tb, Ab, lda, ca, Bb, ldb, cb, n, pb, nb, pstride, nparts, s);
      else if (ta <= 2) gram_tb<2>(tb, Ab, lda, ca, Bb, ldb, cb, n, pb, nb, pstride, nparts, s);
      else if (ta <= 4) gram_tb<4>(tb, Ab, lda, ca, Bb, ldb, cb, n, pb, nb, pstride, nparts, s);
      else gram_tb<8>(tb, Ab, lda, ca, Bb, ldb, cb, n, pb, nb, pstride, nparts, s);
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

// lr_dot tail: G1 = sum of the n1 partials, G2 = sum of the n2 partials,
// per-CTA partial of sum(G1 .* G2) (block order, deterministic) -> part;
// dot_finalize_kernel(part, 1, ...) is not needed: dot_sum_kernel adds them.
__global__ void __launch_bounds__(256) dot_parts_kernel(const double* __restrict__ p1, int n1,
                                                        const double* __restrict__ p2, int n2,
                                                        int nout, double* __restrict__ part) {
  __shared__ double red[8];
  const int o = blockIdx.x * 256 + threadIdx.x;
  double prod = 0.0;
  if (o < nout) {
    double g1 = 0.0, g2 = 0.0;
#pragma unroll 8
    for (int k = 0; k < n1; ++k) g1 += p1[(int64_t)k * nout + o];
#pragma unroll 8
    for (int k = 0; k < n2; ++k) g2 += p2[(int64_t)k * nout + o];
    prod = g1 * g2;
  }
  prod = warp_sum(prod);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = prod;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int w = 0; w < 8; ++w) s += red[w];
    part[blockIdx.x] = s;
  }
}
__global__ void dot_sum_kernel(const double* __restrict__ part, int n, double* __restrict__ out) {
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int k = 0; k < n; ++k) s += part[k];
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
