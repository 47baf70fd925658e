// lrk_gemm.cu — fp64 batched GEMM on the FP64 tensor pipe (DMMA).
//
// sm_100a has no tcgen05 kind for f64; the FP64 tensor path is the warp-level
// mma.sync.m8n8k4 f64 (SASS DMMA).  Used for the DST-I transforms that
// diagonalise the heat step matrix (the B200 replacement of SuperLU's
// solve, forward.py:61-68) and for the sensor-subgrid gathers.
// C[b] = alpha * A[b] * B[b] + beta * C[b]; row-major operands.
// CTA tile 64x64, K-step 16, 4 warps each owning a 32x32 sub-tile (4x4 mma).
#include "lrk_kernels.h"

namespace lrk {

namespace {
constexpr int TM = 64, TN = 64, TK = 16, GT = 128;
constexpr int SP = TM + 4;  // padded k-major stride (conflict-free fragments)

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile(
      "mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(d0), "+d"(d1)
      : "d"(a), "d"(b));
}
}  // namespace

__global__ void __launch_bounds__(GT) gemm_kernel(GemmArgs g) {
  __shared__ double As[2][TK][SP];
  __shared__ double Bs[2][TK][SP];
  int M = g.M;
  if (g.m_dev) { const int md = (*g.m_dev) * g.m_mult; if (md < M) M = md; }
  int batch = g.batch;
  if (g.batch_dev) {
    const int bd = (*g.batch_dev) * (g.batch_mult > 0 ? g.batch_mult : 1);
    if (bd < batch) batch = bd;
  }
  const int b = blockIdx.z;
  if (b >= batch) return;
  const int m0 = blockIdx.y * TM, n0 = blockIdx.x * TN;
  if (m0 >= M) return;
  const int N = g.N, K = g.K;
  const double* A = g.A + (int64_t)b * g.sA;
  const double* B = g.B + (int64_t)b * g.sB;
  double* C = g.C + (int64_t)b * g.sC;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = (warp >> 1) * 32, wn = (warp & 1) * 32;
  const int gi = lane >> 2, ti = lane & 3;

  double acc[4][4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  // global -> register staging: A tile 64x16 (8 per thread), B tile 16x64
  double ra[8], rb[8];
  auto load_tile = [&](int k0) {
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int e = tid + q * GT;        // 0..1023
      const int am = e >> 4, ak = e & 15;  // A: row am, col ak
      const int gm = m0 + am, gk = k0 + ak;
      ra[q] = (gm < M && gk < K) ? A[(int64_t)gm * g.lda + gk] : 0.0;
      const int bk = e >> 6, bn = e & 63;  // B: row bk, col bn
      const int gk2 = k0 + bk, gn = n0 + bn;
      rb[q] = (gk2 < K && gn < N) ? B[(int64_t)gk2 * g.ldb + gn] : 0.0;
    }
  };
  auto store_tile = [&](int buf) {
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int e = tid + q * GT;
      As[buf][e & 15][e >> 4] = ra[q];
      Bs[buf][e >> 6][e & 63] = rb[q];
    }
  };
  const int nk = (K + TK - 1) / TK;
  load_tile(0);
  store_tile(0);
  __syncthreads();
  for (int kt = 0; kt < nk; ++kt) {
    const int buf = kt & 1;
    if (kt + 1 < nk) load_tile((kt + 1) * TK);
#pragma unroll
    for (int kk = 0; kk < TK; kk += 4) {
      double af[4], bf[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) af[i] = As[buf][kk + ti][wm + i * 8 + gi];
#pragma unroll
      for (int j = 0; j < 4; ++j) bf[j] = Bs[buf][kk + ti][wn + j * 8 + gi];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) dmma(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
    }
    if (kt + 1 < nk) store_tile(buf ^ 1);
    __syncthreads();
  }
  // epilogue
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int row = m0 + wm + i * 8 + gi;
    if (row >= M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int col = n0 + wn + j * 8 + 2 * ti + h;
        if (col < N) {
          double* c = C + (int64_t)row * g.ldc + col;
          const double v = g.alpha * acc[i][j][h];
          *c = (g.beta == 0.0) ? v : v + g.beta * (*c);
        }
      }
    }
  }
}

cudaError_t launch_gemm(const GemmArgs& g, cudaStream_t s) {
  if (g.M <= 0 || g.N <= 0 || g.batch <= 0) return cudaSuccess;
  dim3 grid((g.N + TN - 1) / TN, (g.M + TM - 1) / TM, g.batch);
  gemm_kernel<<<grid, GT, 0, s>>>(g);
  return cudaGetLastError();
}

}  // namespace lrk
