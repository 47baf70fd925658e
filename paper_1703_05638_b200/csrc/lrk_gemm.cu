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
constexpr int GT = 128;

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(d0), "+d"(d1)
      : "d"(a), "d"(b));
}
}  // namespace

// TM x TN CTA tile (64x64 or 32x32), 4 warps each owning a (TM/2)x(TN/2)
// sub-tile of FI x FJ m8n8 fragments; K-step TK (the next K-step's global
// loads are in flight while the current one computes, so a longer step hides
// more of the load latency in the latency-bound small-grid case).
template <int TM, int TN, int TK>
__global__ void __launch_bounds__(GT) gemm_kernel(GemmArgs g) {
  constexpr int SP = TM + 4;  // padded k-major stride (conflict-free fragments)
  constexpr int SPN = TN + 4;
  constexpr int FI = TM / 16, FJ = TN / 16;
  constexpr int LA = TM * TK / GT, LB = TK * TN / GT;  // staged elements per thread
  __shared__ double As[2][TK][SP];
  __shared__ double Bs[2][TK][SPN];
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
  const int wm = (warp >> 1) * (TM / 2), wn = (warp & 1) * (TN / 2);
  const int gi = lane >> 2, ti = lane & 3;

  double acc[FI][FJ][2];
#pragma unroll
  for (int i = 0; i < FI; ++i)
#pragma unroll
    for (int j = 0; j < FJ; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  // global -> register staging: A tile TMx16, B tile 16xTN
  double ra[LA], rb[LB];
  auto load_tile = [&](int k0) {
#pragma unroll
    for (int q = 0; q < LA; ++q) {
      const int e = tid + q * GT;
      const int am = e / TK, ak = e % TK;  // A: row am, col ak
      const int gm = m0 + am, gk = k0 + ak;
      ra[q] = (gm < M && gk < K) ? A[(int64_t)gm * g.lda + gk] : 0.0;
    }
#pragma unroll
    for (int q = 0; q < LB; ++q) {
      const int e = tid + q * GT;
      const int bk = e / TN, bn = e % TN;  // B: row bk, col bn
      const int gk2 = k0 + bk, gn = n0 + bn;
      rb[q] = (gk2 < K && gn < N) ? B[(int64_t)gk2 * g.ldb + gn] : 0.0;
    }
  };
  auto store_tile = [&](int buf) {
#pragma unroll
    for (int q = 0; q < LA; ++q) {
      const int e = tid + q * GT;
      As[buf][e % TK][e / TK] = ra[q];
    }
#pragma unroll
    for (int q = 0; q < LB; ++q) {
      const int e = tid + q * GT;
      Bs[buf][e / TN][e % TN] = rb[q];
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
      double af[FI], bf[FJ];
#pragma unroll
      for (int i = 0; i < FI; ++i) af[i] = As[buf][kk + ti][wm + i * 8 + gi];
#pragma unroll
      for (int j = 0; j < FJ; ++j) bf[j] = Bs[buf][kk + ti][wn + j * 8 + gi];
#pragma unroll
      for (int i = 0; i < FI; ++i)
#pragma unroll
        for (int j = 0; j < FJ; ++j) dmma(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
    }
    if (kt + 1 < nk) store_tile(buf ^ 1);
    __syncthreads();
  }
  // epilogue
#pragma unroll
  for (int i = 0; i < FI; ++i) {
    const int row = m0 + wm + i * 8 + gi;
    if (row >= M) continue;
#pragma unroll
    for (int j = 0; j < FJ; ++j) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int col = n0 + wn + j * 8 + 2 * ti + h;
        if (col < N) {
          double* c = C + (int64_t)row * g.ldc + col;
          double v = g.alpha * acc[i][j][h];
          if (g.emul) v *= g.emul[(int64_t)row * g.lde + col];
          *c = (g.beta == 0.0) ? v : v + g.beta * (*c);
        }
      }
    }
  }
}

cudaError_t launch_gemm(const GemmArgs& g, cudaStream_t s) {
  if (g.M <= 0 || g.N <= 0 || g.batch <= 0) return cudaSuccess;
  const int64_t tiles64 = (int64_t)((g.N + 63) / 64) * ((g.M + 63) / 64) * g.batch;
  if (tiles64 >= 2 * 148) {
    dim3 grid((g.N + 63) / 64, (g.M + 63) / 64, g.batch);
    gemm_kernel<64, 64, 16><<<grid, GT, 0, s>>>(g);
  } else {  // under-filled grid (e.g. one 512^2 DST column): 4x more CTAs,
            // K-step 32 (half the latency-bound K iterations)
    dim3 grid((g.N + 31) / 32, (g.M + 31) / 32, g.batch);
    gemm_kernel<32, 32, 32><<<grid, GT, 0, s>>>(g);
  }
  return cudaGetLastError();
}

}  // namespace lrk
