// lrk_misc.h — declarations of the streaming kernels in lrk_misc.cu.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace lrk {

struct StencilArgs {
  const double* X; int64_t ldx;
  double* Y; int64_t ldy;
  int n;          // n_side
  int dim;        // 2 or 3
  int ncols;
  // (L x)_i = sum over the 3^dim box of coef[(d3+1)*9 + (d2+1)*3 + (d1+1)] x_{i+d}
  // (already mirrored for the adjoint); zero entries are skipped uniformly
  double coef[27];
  double m_scale, tau;
  const double* Bres;     // optional: Y = Bres - S X (residual form)
  int64_t ldbres;
  // variable wind (wind_field = 1): per-node upwind of w = w0 + rotating field,
  // added on top of coef (which then holds the diffusion part only)
  int wind_field;
  // Galerkin Q1 convection (config C3, SUPG delta_k = 0 at
  // element Peclet < 1): N_ij = int (w . grad phi_j) phi_i with the wind taken
  // at the element centres (w0, plus the rotating field when `rotating`),
  // lumped mass; coef then holds nu K_Q1 / h^2
  int galerkin;
  int rotating;
  int adjoint;
  double w0[3];
  double h;
  // optional fused copy: Ycopy[:, c] = copy_scale * X[:, c] (K.apply's -M W1 block)
  double* Ycopy; int64_t ldycopy; double copy_scale;
};

__global__ void stencil_kernel(StencilArgs a);
// Persistent preconditioned Richardson step solve (lrk_rich.cu): x = S^{-1} b by
// x0 = P^{-1} b and `sweeps` corrections in one cooperative launch, then the
// true-residual check (flag raised when ||b - S x||^2 > tol2 ||b||^2).
// cudaErrorNotSupported: shape outside its scope (3-D, odd n, per-node upwind).
// part[] of launch_rich: two doubles per CTA (at most 2 CTAs on each of up to 148 SMs), then the
// diagnostics triple {sweeps used, ||r||^2, ||b||^2}
constexpr int RICH_PART_DIAG = 2 * 296;
constexpr int RICH_PART_LEN = RICH_PART_DIAG + 4;
cudaError_t launch_rich(const StencilArgs& st, int n, int sweeps, const double* S1, const double* D,
                        const double* b, double* x, double* r, double* T1, double* T2, unsigned* bar,
                        double* part, int* flag, double tol2, int num_sms, cudaStream_t s);
// tiled kernels (2-D box, 3-D 7-point) or the generic one; a.ncols columns
void launch_stencil(const StencilArgs& a, cudaStream_t s);
__global__ void shift_kernel(const double* W2, int64_t ld2, int n_t, int ncols, int adjoint,
                             double* out, int64_t ldo, const double* W1, int64_t ld1,
                             int64_t n_x, double neg_m, double* out1, int64_t ldo1);
__global__ void prior_scale_kernel(const double* X, int64_t ldx, const double* lam, int64_t n,
                                   int ncols, const int* ncols_dev, double alpha, double delta,
                                   double gamma, double* Y, int64_t ldy);
__global__ void rank_axpy_kernel(const double* B, int64_t ldb, int rb, const double* w,
                                 int64_t ldw, double* y, int64_t n);
__global__ void resid_flag_kernel(const double* r, const double* b, int64_t n, double tol2,
                                  double* part, unsigned* counter, int* flag);
__global__ void axpby_kernel(const double* x, double a, const double* y, double b, double* out,
                             int64_t n);
__global__ void mask_time_rows_kernel(double* W2, int64_t ld2, int n_t, int ncols, int every);
__global__ void scale_rows_kernel(const double* X, int64_t ldx, const double* s, int64_t n,
                                  int ncols, const int* ncols_dev, double alpha, double* Y,
                                  int64_t ldy);
__global__ void scale_cols_kernel(const double* X, int64_t ldx, int64_t n, const double* colscale,
                                  const int* ncols_dev, int ncols, double alpha, double* Y,
                                  int64_t ldy);
__global__ void column_eval_kernel(const double* U, int64_t ldu, int64_t n, const double* sigma,
                                   const double* V, int64_t ldv, int row, const int* r_dev,
                                   double* y);
__global__ void gather_rows_kernel(const double* X, int64_t ldx, const int32_t* idx, int nidx,
                                   const int* ncols_dev, int ncols, double* Y, int64_t ldy);
__global__ void scatter_rows_kernel(const double* X, int64_t ldx, const int32_t* idx, int nidx,
                                    const int* ncols_dev, int ncols, double* Y, int64_t ldy);
__global__ void fill_kernel(double* X, int64_t ldx, int64_t n, int ncols, double v);
__global__ void transpose_kernel(const double* X, int64_t ldx, int64_t rows, int cols, double alpha,
                                 double* Y, int64_t ldy);
__global__ void eye_kernel(double* X, int64_t ldx, int n);
__global__ void seg_dot_kernel(const double* p1, int n1, const double* p2, int n2, int na, int nb,
                               const int* segoff, double* out);
__global__ void flip_partial_kernel(const double* U, int64_t ldu, int64_t n, const int* r_dev,
                                    int rcap, double* part);
__global__ void flip_apply_kernel(double* U, int64_t ldu, int64_t n_x, double* V, int64_t ldv,
                                  int n_t, const int* r_dev, int rcap, const double* part,
                                  int nparts);
__global__ void gram_partial_kernel(const double* A, int64_t lda, int na, const double* B,
                                    int64_t ldb, int nb, int64_t n, double* part);
// nparts x (na*nb) partials of A^T B over n rows on the FP64 tensor pipe
// (row-major i*nb + j per part); launches enqueue on s.
void launch_gram(const double* A, int64_t lda, int na, const double* B, int64_t ldb, int nb,
                 int64_t n, double* part, int nparts, cudaStream_t s);
__global__ void dot_parts_kernel(const double* p1, int n1, const double* p2, int n2, int nout,
                                 double* part);
__global__ void dot_sum_kernel(const double* part, int n, double* out);
__global__ void dot_finalize_kernel(const double* p1, int n1, const double* p2, int n2, int nout,
                                    double* out);
__global__ void reduce_parts_kernel(const double* p, int nparts, int nout, double* out,
                                    double* acc_out);
__global__ void sub_qh_kernel(const double* Q, int64_t ldq, int k, const double* h, double* w,
                              int64_t n);
__global__ void combine_kernel(const double* Q, int64_t ldq, int k, const double* cf, double* y,
                               int64_t n);

}  // namespace lrk
