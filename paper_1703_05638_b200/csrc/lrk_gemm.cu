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

// Small-grid variant (one 512^2 DST column = 64..256 CTAs: every CTA walks the
// whole K range, so the kernel is bound by the latency of its K-steps, not by
// DMMA or bandwidth): the operand tiles stream through an NSTAGE-deep shared
// ring with 8-byte cp.async (no alignment requirement on lda/ldb; zero-fill at
// the edges), NSTAGE - 1 K-steps in flight, one barrier per K-step.  A stays
// row-major in shared memory (stride TK + 4), B k-major (stride TN + 4): both
// fragment patterns are two wavefronts per 8-byte warp load.
template <int TM, int TN, int TK, int NSTAGE>
__global__ void __launch_bounds__(GT) gemm_async_kernel(GemmArgs g) {
  extern __shared__ __align__(16) double gsm[];
  constexpr int SA = TK + 4, SB = TN + 4;
  constexpr int FI = TM / 16, FJ = TN / 16;
  constexpr int LA = TM * TK / GT, LB = TK * TN / GT;
  double* As = gsm;                          // [NSTAGE][TM][SA]
  double* Bs = gsm + NSTAGE * TM * SA;       // [NSTAGE][TK][SB]
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
  auto cp8 = [](double* dst, const double* src, bool ok) {
    const unsigned sa = (unsigned)__cvta_generic_to_shared(dst);
    const int sz = ok ? 8 : 0;
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(sa), "l"(src), "r"(sz) : "memory");
  };
  const int nk = (K + TK - 1) / TK;
  auto issue = [&](int kt) {
    if (kt < nk) {
      const int st = kt % NSTAGE, k0 = kt * TK;
      double* as = As + st * TM * SA;
      double* bs = Bs + st * TK * SB;
#pragma unroll
      for (int q = 0; q < LA; ++q) {
        const int e = tid + q * GT;
        const int am = e / TK, ak = e % TK;
        const bool ok = m0 + am < M && k0 + ak < K;
        cp8(as + am * SA + ak, A + (ok ? (int64_t)(m0 + am) * g.lda + k0 + ak : 0), ok);
      }
#pragma unroll
      for (int q = 0; q < LB; ++q) {
        const int e = tid + q * GT;
        const int bk = e / TN, bn = e % TN;
        const bool ok = k0 + bk < K && n0 + bn < N;
        cp8(bs + bk * SB + bn, B + (ok ? (int64_t)(k0 + bk) * g.ldb + n0 + bn : 0), ok);
      }
    }
    asm volatile("cp.async.commit_group;\n" ::: "memory");  // one group per K-step, empty past the end
  };
  double acc[FI][FJ][2];
#pragma unroll
  for (int i = 0; i < FI; ++i)
#pragma unroll
    for (int j = 0; j < FJ; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
#pragma unroll
  for (int sidx = 0; sidx < NSTAGE - 1; ++sidx) issue(sidx);
  for (int kt = 0; kt < nk; ++kt) {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(NSTAGE - 2) : "memory");  // K-step kt landed
    __syncthreads();          // everyone's copies, and K-step kt - 1 is consumed
    issue(kt + NSTAGE - 1);   // into the slot of K-step kt - 1
    const double* as = As + (kt % NSTAGE) * TM * SA;
    const double* bs = Bs + (kt % NSTAGE) * TK * SB;
#pragma unroll
    for (int kk = 0; kk < TK; kk += 4) {
      double af[FI], bf[FJ];
#pragma unroll
      for (int i = 0; i < FI; ++i) af[i] = as[(wm + i * 8 + gi) * SA + kk + ti];
#pragma unroll
      for (int j = 0; j < FJ; ++j) bf[j] = bs[(kk + ti) * SB + wn + j * 8 + gi];
#pragma unroll
      for (int i = 0; i < FI; ++i)
#pragma unroll
        for (int j = 0; j < FJ; ++j) dmma(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
    }
  }
  asm volatile("cp.async.wait_group 0;\n" ::: "memory");
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
    constexpr int NS = 4;
    constexpr size_t smem = (size_t)NS * (32 * 36 + 32 * 36) * sizeof(double);
    static bool configured[64] = {};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev >= 0 && dev < 64 && !configured[dev]) {
      cudaError_t e = cudaFuncSetAttribute(gemm_async_kernel<32, 32, 32, NS>,
                                           cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      if (e != cudaSuccess) return e;
      configured[dev] = true;
    }
    gemm_async_kernel<32, 32, 32, NS><<<grid, GT, smem, s>>>(g);
  }
  return cudaGetLastError();
}

}  // namespace lrk
