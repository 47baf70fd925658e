// lrk_misc.cu — streaming kernels around the persistent sweep/truncation:
// matrix-free stencil SpMM, sign canonicalisation, low-rank inner products,
// dense CGS2 for the IC-mode Arnoldi, row gathers/scatters, column scalings.
#include "lrk_device.cuh"
#include "lrk_misc.h"
#include "lrk_stencil.cuh"

namespace lrk {

// ---------------------------------------------------------------- stencil
// K.apply / apply_adjoint spatial part (forward.py:79-95):
// (S x) = m_scale (x + tau L x) for the constant-coefficient box stencils of
// discretize.py:90-127 (5-point FD) and their config extensions (Q1-lumped
// 9-point, 3-D 7-point), generated on the fly (no CSR), zero Dirichlet data.
// One thread per output entry, coalesced along x1; neighbours come through L1.
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
  const double lx = stencil_lx(a, x, i, i1, i2, i3, [](const double* q) { return *q; });
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

// Marching box stencils with a cp.async plane pipeline.  A CTA owns a TX x TY
// in-plane tile and marches MZ planes along the slowest axis (x3 in 3-D, x2 in
// 2-D, where a "plane" is a TX-wide row segment); planes (+ one-node halo,
// zero-filled outside the domain = the Dirichlet data) stream into an NS-slot
// shared-memory ring with 8-byte cp.async, NA planes ahead of the one being
// computed, so each thread keeps several loads in flight without registers
// and every input is read from HBM once (16 B per output + the z halo, which
// L2 serves).  One __syncthreads per plane: the slot refilled at step z held
// plane z - 2, read during step z - 1.
//   D = 3: TX = 32, TY = 16, 7-point (+ optional upwind), 2 rows per thread, MZ = 32.
//   D = 2: TX = 256, TY = 1, 3 x 3 box (5- or 9-point, + optional upwind), MZ = 16.
template <int D> struct MarchShape;
template <> struct MarchShape<3> { static constexpr int TX = 32, TY = 16; };
template <> struct MarchShape<2> { static constexpr int TX = 256, TY = 1; };
constexpr int MARCH_NA = 3;                 // planes in flight beyond z + 1
constexpr int MARCH_NS = MARCH_NA + 3;      // ring slots: z-1, z, z+1, NA in flight

__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory"); }

template <int D, bool WIND, int MZ>
__global__ void __launch_bounds__(256, WIND ? 3 : 4) stencil_march_kernel(StencilArgs a, int nzb) {
  constexpr int TX = MarchShape<D>::TX, TY = MarchShape<D>::TY;
  constexpr int PW = TX + 2, PH = D == 3 ? TY + 2 : 1, PS = PW * PH;  // plane slot (doubles)
  constexpr int RPT = TY * TX / 256;                       // rows per thread
  constexpr int NS = MARCH_NS, NA = MARCH_NA;
  __shared__ __align__(16) double ring[NS * PS];
  const int zb = blockIdx.z % nzb, c = blockIdx.z / nzb;
  const int n = a.n;
  const int64_t pstride = D == 3 ? (int64_t)n * n : n;    // march-axis stride
  const int tid = threadIdx.x;
  const int x0 = blockIdx.x * TX, y0 = blockIdx.y * TY;
  const double* x = a.X + (int64_t)c * a.ldx;
  const int z0 = zb * MZ, z1 = min(n, z0 + MZ);
  // this thread's slot elements (the same for every plane): in-plane
  // offset, in-domain flag and shared-memory address, computed once
  constexpr int NE = (PS + 255) / 256;
  int64_t eoff[NE];
  bool eok[NE];
  unsigned edst[NE];
#pragma unroll
  for (int m = 0; m < NE; ++m) {
    const int e = tid + 256 * m;
    const int ly = e / PW, lx = e - ly * PW;
    const int gx = x0 + lx - 1, gy = y0 + ly - 1;
    eok[m] = e < PS && gx >= 0 && gx < n && (D == 2 || (gy >= 0 && gy < n));
    eoff[m] = eok[m] ? (D == 3 ? (int64_t)gy * n : 0) + gx : 0;
    edst[m] = (unsigned)__cvta_generic_to_shared(ring + (e < PS ? e : 0));
  }
  // load index q = 0, 1, ... is plane z0 - 1 + q, slot q % NS
  auto issue = [&](int q) {
    const int pz = z0 - 1 + q;
    if (pz <= z1) {
      const unsigned soff = (unsigned)((q % NS) * PS * sizeof(double));
      const bool zin = pz >= 0 && pz < n;
      const double* xp = x + (zin ? (int64_t)pz * pstride : 0);
#pragma unroll
      for (int m = 0; m < NE; ++m) {
        if (tid + 256 * m < PS) {
          const bool ok = zin && eok[m];
          const int sz = ok ? 8 : 0;  // 0: zero-fill, nothing read
          asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(edst[m] + soff),
                       "l"(xp + eoff[m]), "r"(sz)
                       : "memory");
        }
      }
    }
    cp_async_commit();  // one group per load index, empty past the end
  };
#pragma unroll
  for (int q = 0; q < NA + 2; ++q) issue(q);
  const int gx = x0 + (tid % TX);
  const int lx = tid % TX + 1;
  double cf[9];
  if (D == 2) {
#pragma unroll
    for (int q = 0; q < 9; ++q) cf[q] = a.coef[9 + q];
  } else {
    cf[0] = a.coef[12]; cf[1] = a.coef[14]; cf[2] = a.coef[10]; cf[3] = a.coef[16];
    cf[4] = a.coef[4]; cf[5] = a.coef[22]; cf[6] = a.coef[13];
  }
  for (int z = z0; z < z1; ++z) {
    const int q = z - z0 + 1;           // load index of plane z
    cp_async_wait<NA - 1>();            // own copies of plane z + 1 landed
    __syncthreads();                    // everyone's, and plane z - 2 is consumed
    issue(q + NA + 1);                  // plane z + NA + 1 into the slot of z - 2
    const double* pm = ring + ((q - 1) % NS) * PS;
    const double* p0 = ring + (q % NS) * PS;
    const double* pp = ring + ((q + 1) % NS) * PS;
#pragma unroll
    for (int rr = 0; rr < RPT; ++rr) {
      const int ly = D == 3 ? tid / TX + rr * (256 / TX) + 1 : 0;
      const int gy = D == 3 ? y0 + ly - 1 : z;
      if (gx >= n || gy >= n) continue;
      const int k = ly * PW + lx;
      const double cur = p0[k];
      double lx_acc;
      double xm[3], xp[3];
      if (D == 3) {
        xm[0] = p0[k - 1]; xp[0] = p0[k + 1];
        xm[1] = p0[k - PW]; xp[1] = p0[k + PW];
        xm[2] = pm[k]; xp[2] = pp[k];
        lx_acc = cf[6] * cur + cf[0] * xm[0] + cf[1] * xp[0] + cf[2] * xm[1] + cf[3] * xp[1] +
                 cf[4] * xm[2] + cf[5] * xp[2];
      } else {
        lx_acc = cf[0] * pm[k - 1] + cf[1] * pm[k] + cf[2] * pm[k + 1] +
                 cf[3] * p0[k - 1] + cf[4] * cur + cf[5] * p0[k + 1] +
                 cf[6] * pp[k - 1] + cf[7] * pp[k] + cf[8] * pp[k + 1];
        xm[0] = p0[k - 1]; xp[0] = p0[k + 1];
        xm[1] = pm[k]; xp[1] = pp[k];
        xm[2] = 0.0; xp[2] = 0.0;
        if (WIND && a.galerkin) {
          const double v[9] = {pm[k - 1], pm[k], pm[k + 1], p0[k - 1], cur, p0[k + 1],
                               pp[k - 1], pp[k], pp[k + 1]};
          lx_acc += galerkin_nb(a, gx, gy, v);
        }
      }
      if (WIND && a.wind_field) lx_acc += upwind_nb(a, gx, gy, cur, xm, xp);
      const double sx = a.m_scale * (cur + a.tau * lx_acc);
      const int64_t i = D == 3 ? (int64_t)z * pstride + (int64_t)gy * n + gx
                               : (int64_t)gy * n + gx;
      a.Y[i + (int64_t)c * a.ldy] = a.Bres ? a.Bres[i + (int64_t)c * a.ldbres] - sx : sx;
      if (a.Ycopy) a.Ycopy[i + (int64_t)c * a.ldycopy] = a.copy_scale * cur;
    }
  }
  cp_async_wait<0>();
}

template <int D, int MZ>
static void launch_march_mz(const StencilArgs& a, cudaStream_t s) {
  constexpr int TX = MarchShape<D>::TX, TY = MarchShape<D>::TY;
  const int n = a.n;
  const int nzb = (n + MZ - 1) / MZ;
  dim3 grid((n + TX - 1) / TX, D == 3 ? (n + TY - 1) / TY : 1, nzb * a.ncols);
  if (a.wind_field || a.galerkin)
    stencil_march_kernel<D, true, MZ><<<grid, 256, 0, s>>>(a, nzb);
  else
    stencil_march_kernel<D, false, MZ><<<grid, 256, 0, s>>>(a, nzb);
}

// planes per CTA (measured at C3 / C4: 2-D 8/16/32/64 -> 80/78/82/91 us,
// 3-D 16/32/64 -> 717/710/709 us)
template <int D>
static void launch_march(const StencilArgs& a, cudaStream_t s) {
  if (D == 2) {
    // few columns (the step solves of the physical-space sweep work on ONE column):
    // a CTA's run time is its chain of dependent plane steps, so short marches on
    // more CTAs (512^2 x 1 column: 64 CTAs x 19 steps -> 256 CTAs x 7 steps)
    const int64_t ctas16 = (int64_t)((a.n + 255) / 256) * ((a.n + 15) / 16) * a.ncols;
    if (ctas16 < 2 * 148) {
      launch_march_mz<D, 4>(a, s);
      return;
    }
  }
  launch_march_mz<D, D == 2 ? 16 : 32>(a, s);
}

// Launch the marching kernel that fits the operator (2-D box; 3-D 7-point),
// the generic one otherwise.  a.ncols columns.
void launch_stencil(const StencilArgs& a, cudaStream_t s) {
  const int n = a.n;
  if (a.dim == 2) {
    launch_march<2>(a, s);
    return;
  }
  bool seven = true;
  for (int q = 0; q < 27; ++q) {
    const int d3 = q / 9, d2 = (q / 3) % 3, d1 = q % 3;
    const int nnz_axes = (d3 != 1) + (d2 != 1) + (d1 != 1);
    if (nnz_axes > 1 && a.coef[q] != 0.0) seven = false;
  }
  if (seven) {
    launch_march<3>(a, s);
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

// Y = alpha * X^T for a rows x cols column-major X (Y is cols x rows, ld ldy):
// the row-major views the DMMA GEMM needs for the wide truncation path.
__global__ void transpose_kernel(const double* X, int64_t ldx, int64_t rows, int cols, double alpha,
                                 double* Y, int64_t ldy) {
  __shared__ double t[32][33];
  const int64_t i0 = (int64_t)blockIdx.x * 32;
  const int c0 = blockIdx.y * 32;
  for (int k = threadIdx.y; k < 32; k += blockDim.y) {
    const int64_t i = i0 + threadIdx.x;
    const int c = c0 + k;
    t[k][threadIdx.x] = (i < rows && c < cols) ? X[i + (int64_t)c * ldx] : 0.0;
  }
  __syncthreads();
  for (int k = threadIdx.y; k < 32; k += blockDim.y) {
    const int c = c0 + threadIdx.x;
    const int64_t i = i0 + k;
    if (i < rows && c < cols) Y[c + i * ldy] = alpha * t[threadIdx.x][k];
  }
}

// n x n identity (ld ldx)
__global__ void eye_kernel(double* X, int64_t ldx, int n) {
  const int c = blockIdx.y;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    X[i + (int64_t)c * ldx] = (i == c) ? 1.0 : 0.0;
}

// Segmented Hadamard sums of two reduced Gram blocks (the batched lr_dot of
// one field against many, lowrank.py:163-168): out[g] = sum over rows a < na
// and columns b in [segoff[g], segoff[g+1]) of G1[a][b] * G2[a][b], where
// G1 / G2 are the sums of the n1 / n2 partials (row-major a * nb + b).
// One block per segment, fixed summation order -> deterministic.
__global__ void __launch_bounds__(256) seg_dot_kernel(const double* __restrict__ p1, int n1,
                                                      const double* __restrict__ p2, int n2,
                                                      int na, int nb, const int* __restrict__ segoff,
                                                      double* __restrict__ out) {
  __shared__ double red[8];
  const int g = blockIdx.x;
  const int b0 = segoff[g], b1 = segoff[g + 1], w = b1 - b0;
  const int nout = na * nb;
  double acc = 0.0;
  for (int e = threadIdx.x; e < na * w; e += 256) {
    const int o = (e / w) * nb + b0 + e % w;
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
    for (int k = 0; k < 8; ++k) s += red[k];
    out[g] = s;
  }
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

// Staged variant for wide Grams (both sides > 32 columns, the FP64-tensor-
// bound shape): the CTA streams chunks of GKC rows of up to 64 columns of A
// and B into a GST-stage shared-memory ring with 16-byte cp.async (GST - 1
// chunks, ~96 KB, in flight per SM: enough for HBM latency at the ridge
// point), and its 8 warps split the 64 x 64 output 16 x 32 each, reading
// their m8n8k4 fragments from shared memory (column stride GKC + 4 doubles:
// two wavefronts per fragment load, conflict-free).  Each output element is
// accumulated by one warp in row order (deterministic).  Requires lda, ldb
// even and 16-byte-aligned bases (checked by the launcher).
constexpr int GKC = 32, GST = 4, GSS = GKC + 4;
__global__ void __launch_bounds__(NT, 1)
    gram_staged_kernel(const double* __restrict__ A, int64_t lda, int na,
                       const double* __restrict__ B, int64_t ldb, int nb, int64_t n,
                       double* __restrict__ part, int ldo, int64_t pstride) {
  extern __shared__ __align__(16) double gsm[];  // [GST][128 columns][GSS]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t = lane & 3;
  // CTA row range: whole GKC chunks (the 16-byte copies stay aligned)
  const int64_t nch = (n + GKC - 1) / GKC;
  const int64_t cper = (nch + gridDim.x - 1) / gridDim.x;
  const int64_t c0 = cper * blockIdx.x, c1 = min(nch, c0 + cper);
  const int nc = c1 > c0 ? (int)(c1 - c0) : 0;
  auto issue = [&](int q) {
    if (q < nc) {
      double* st = gsm + (q % GST) * (128 * GSS);
      const int64_t r0 = (c0 + q) * GKC;
#pragma unroll
      for (int m = 0; m < 128 * (GKC / 2) / NT; ++m) {
        const int e = tid + NT * m;
        const int col = e / (GKC / 2), seg = e % (GKC / 2);
        const bool isa = col < 64;
        const int cc = isa ? col : col - 64;
        if (cc < (isa ? na : nb)) {
          const int64_t row = r0 + 2 * seg;
          const int64_t left = n - row;
          const int bytes = left >= 2 ? 16 : (left == 1 ? 8 : 0);
          const double* src = isa ? A + (int64_t)cc * lda : B + (int64_t)cc * ldb;
          src += bytes ? row : 0;
          const unsigned d = (unsigned)__cvta_generic_to_shared(st + col * GSS + 2 * seg);
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(d), "l"(src), "r"(bytes)
                       : "memory");
        }
      }
    }
    asm volatile("cp.async.commit_group;\n" ::: "memory");
  };
#pragma unroll
  for (int q = 0; q < GST - 1; ++q) issue(q);
  const int ia = 16 * (warp >> 1), jb = 64 + 32 * (warp & 1);
  double acc[2][4][2];
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  for (int q = 0; q < nc; ++q) {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(GST - 2) : "memory");
    __syncthreads();       // chunk q visible; chunk q - 1's slot is free
    issue(q + GST - 1);
    const double* st = gsm + (q % GST) * (128 * GSS);
    const double* pa = st + (ia + g) * GSS + t;
    const double* pb = st + (jb + g) * GSS + t;
#pragma unroll
    for (int k = 0; k < GKC; k += 4) {
      double af[2], bf[4];
#pragma unroll
      for (int i = 0; i < 2; ++i) af[i] = pa[8 * i * GSS + k];
#pragma unroll
      for (int j = 0; j < 4; ++j) bf[j] = pb[8 * j * GSS + k];
#pragma unroll
      for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) dmma884(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
    }
  }
  asm volatile("cp.async.wait_group 0;\n" ::: "memory");
  // a zero-filled tail contributes exact zeros; columns >= na / nb hold stale
  // shared memory and only reach the masked outputs
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int ii = ia + 8 * i + g, jj = jb - 64 + 8 * j + 2 * t + h;
        if (ii < na && jj < nb)
          part[(int64_t)blockIdx.x * pstride + (int64_t)ii * ldo + jj] = nc ? acc[i][j][h] : 0.0;
      }
}

static bool gram_staged_ok(const double* A, int64_t lda, const double* B, int64_t ldb) {
  return ((lda | ldb) & 1) == 0 && (((uintptr_t)A | (uintptr_t)B) & 15) == 0;
}

static void launch_gram_staged(const double* A, int64_t lda, int na, const double* B, int64_t ldb,
                               int nb, int64_t n, double* part, int ldo, int64_t pstride,
                               int nparts, cudaStream_t s) {
  const int smem = GST * 128 * GSS * (int)sizeof(double);
  // the opt-in shared-memory size is a per-device function attribute
  static bool attr[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64 || !attr[dev]) {
    cudaFuncSetAttribute(gram_staged_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (dev >= 0 && dev < 64) attr[dev] = true;
  }
  gram_staged_kernel<<<nparts, NT, smem, s>>>(A, lda, na, B, ldb, nb, n, part, ldo, pstride);
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
      if (ca > 32 && cb > 32 && gram_staged_ok(Ab, lda, Bb, ldb) && !getenv("LRK_GRAM_DIRECT")) {
        launch_gram_staged(Ab, lda, ca, Bb, ldb, cb, n, pb, nb, pstride, nparts, s);
        continue;
      }
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
