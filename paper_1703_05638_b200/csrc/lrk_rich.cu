// lrk_rich.cu — one persistent kernel per preconditioned Richardson step solve
// (2-D physical-space sweeps: convection-diffusion, SURVEY config C3).
//
// S x = b with S = M (I + tau L) (forward.py:61-68's solve, here for the
// non-normal operators the DST does not diagonalise) is solved by
//     x_0 = P^{-1} b,   x_{k+1} = x_k + P^{-1} (b - S x_k),
// P = M (I + tau nu L_Delta) = Phi diag(.) Phi exactly (Phi = S1 (x) S1 the 2-D
// DST-I), i.e. per sweep one matrix-free residual and four n x n x n GEMMs
//     T1 = R S1,  T2 = (S1 T1) .* D,  T1 = T2 S1,  X (+)= S1 T1.
// As separate launches that is ~70 dependent small kernels per time step, each
// paying launch, ramp-up and drain (~20 us per 512^3 GEMM against ~7 us of
// work).  Here all phases of one solve run in ONE cooperative launch: every CTA
// owns 32 x 32 output tiles, streams its operand panels from L2 through a
// 3-stage cp.async ring (16-byte .cg copies: operands written by other CTAs in
// the previous phase must not be served from a stale L1), multiplies on the
// FP64 tensor pipe (DMMA m8n8k4), and the phases are separated by a grid
// barrier.  The final true-residual check (||b - S x|| <= tol ||b||) raises a
// device flag exactly like the multi-launch path, which remains the fallback
// for 3-D grids, odd n and the per-node upwind field.
#include <algorithm>

#include "lrk_device.cuh"
#include "lrk_kernels.h"
#include "lrk_stencil.cuh"

namespace lrk {

namespace {
// 8 warps per CTA: warps 0-3 and 4-7 each cover the 32 x 32 tile with 16 x 16
// sub-tiles and take one half of every k-step (split-K inside the CTA, summed
// through shared memory in the epilogue) — twice the DMMA chains in flight per
// scheduler for the same tile grid.  Measured on C3's grid (n 512, n_t 256, ms
// per apply): this form 922, four warps without split-K 933, 32 x 64 tiles with
// eight warps 1033 and with four 1373 (128 CTAs leave 20 SMs idle); ncu shows
// the DMMA pipe 40 % and the shared-memory pipe 43 % busy, barrier waits first
// among the stall reasons (profiles/ncu_rich_kernel_r02l.txt).  k-steps of 64
// with a 3-stage ring (half the CTA barriers per tile of the 32-deep 4-stage
// ring, same 2 CTAs per SM) took the full C3 apply from 2.33 to 2.25 s.
constexpr int RT = 256;
constexpr int TM = 32, TN = 32, TK = 64, NS = 3;
constexpr int FI = TM / 16, FJ = TN / 16;
constexpr int SA = TK + 4, SB = TN + 4;

__device__ __forceinline__ void cp16cg(double* dst, const double* src, bool ok) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(dst);
  const int sz = ok ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(sa), "l"(src), "r"(sz) : "memory");
}

// C tile (m0, n0) of C = (A B) .* emul + beta C; A, B, C n x n row-major (ld n).
__device__ __forceinline__ void gemm_tile(const double* __restrict__ A, const double* __restrict__ B,
                                          double* __restrict__ C, const double* __restrict__ emul,
                                          double beta, int n, int m0, int n0, double* sm) {
  double* As = sm;                     // [NS][TM][SA]
  double* Bs = sm + NS * TM * SA;      // [NS][TK][SB]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = ((warp >> 1) & 1) * (TM / 2), wn = (warp & 1) * (TN / 2);
  const int kh = (warp >> 2) * (TK / 2);   // this warp's half of each k-step
  const int gi = lane >> 2, ti = lane & 3;
  const int nk = (n + TK - 1) / TK;
  auto issue = [&](int kt) {
    if (kt < nk) {
      const int st = kt % NS, k0 = kt * TK;
      double* as = As + st * TM * SA;
      double* bs = Bs + st * TK * SB;
#pragma unroll
      for (int q = 0; q < TM * TK / 2 / RT; ++q) {   // A panel: TM rows x TK/2 pairs along k
        const int e = tid + q * RT;
        const int am = e / (TK / 2), ak = 2 * (e % (TK / 2));
        const bool ok = m0 + am < n && k0 + ak < n;
        cp16cg(as + am * SA + ak, A + (ok ? (int64_t)(m0 + am) * n + k0 + ak : 0), ok);
      }
#pragma unroll
      for (int q = 0; q < TK * TN / 2 / RT; ++q) {   // B panel: TK rows x TN/2 pairs along n
        const int e = tid + q * RT;
        const int bk = e / (TN / 2), bn = 2 * (e % (TN / 2));
        const bool ok = k0 + bk < n && n0 + bn < n;
        cp16cg(bs + bk * SB + bn, B + (ok ? (int64_t)(k0 + bk) * n + n0 + bn : 0), ok);
      }
    }
    asm volatile("cp.async.commit_group;\n" ::: "memory");
  };
  double acc[FI][FJ][2];
#pragma unroll
  for (int i = 0; i < FI; ++i)
#pragma unroll
    for (int j = 0; j < FJ; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  __syncthreads();  // the ring is free (previous tile / phase)
#pragma unroll
  for (int q = 0; q < NS - 1; ++q) issue(q);
  for (int kt = 0; kt < nk; ++kt) {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(NS - 2) : "memory");
    __syncthreads();
    issue(kt + NS - 1);
    const double* as = As + (kt % NS) * TM * SA;
    const double* bs = Bs + (kt % NS) * TK * SB;
#pragma unroll
    for (int kk = kh; kk < kh + TK / 2; kk += 4) {
      double af[FI], bf[FJ];
#pragma unroll
      for (int i = 0; i < FI; ++i) af[i] = as[(wm + i * 8 + gi) * SA + kk + ti];
#pragma unroll
      for (int j = 0; j < FJ; ++j) bf[j] = bs[(kk + ti) * SB + wn + j * 8 + gi];
#pragma unroll
      for (int i = 0; i < FI; ++i)
#pragma unroll
        for (int j = 0; j < FJ; ++j) dmma884(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
    }
  }
  asm volatile("cp.async.wait_group 0;\n" ::: "memory");
  __syncthreads();                      // every warp is done with the ring
  double* red = sm + ((warp & 3) * 32 + lane) * (FI * FJ * 2);
  if (warp >= 4) {
#pragma unroll
    for (int i = 0; i < FI; ++i)
#pragma unroll
      for (int j = 0; j < FJ; ++j)
        *reinterpret_cast<double2*>(red + (i * FJ + j) * 2) = make_double2(acc[i][j][0], acc[i][j][1]);
  }
  __syncthreads();
  if (warp >= 4) return;
#pragma unroll
  for (int i = 0; i < FI; ++i)
#pragma unroll
    for (int j = 0; j < FJ; ++j) {
      const double2 o = *reinterpret_cast<const double2*>(red + (i * FJ + j) * 2);
      acc[i][j][0] += o.x;
      acc[i][j][1] += o.y;
    }
#pragma unroll
  for (int i = 0; i < FI; ++i) {
    const int row = m0 + wm + i * 8 + gi;
    if (row >= n) continue;
#pragma unroll
    for (int j = 0; j < FJ; ++j) {
      const int col = n0 + wn + j * 8 + 2 * ti;   // n is even: the pair is in or out together
      if (col < n) {
        double2 v = make_double2(acc[i][j][0], acc[i][j][1]);
        const int64_t o = (int64_t)row * n + col;
        if (emul) {
          v.x *= emul[o];
          v.y *= emul[o + 1];
        }
        if (beta != 0.0) {
          const double2 c0 = __ldcg(reinterpret_cast<const double2*>(C + o));
          v.x += beta * c0.x;
          v.y += beta * c0.y;
        }
        *reinterpret_cast<double2*>(C + o) = v;
      }
    }
  }
}
}  // namespace

struct RichArgs {
  StencilArgs st;        // operator coefficients (X / Y / Bres unused)
  int n, sweeps, ntm, ntn;
  const double* S1;      // n x n DST-I
  const double* D;       // n^2 spectral scaling of P^{-1} (x1 fastest)
  const double* b;
  double *x, *r, *T1, *T2;
  unsigned* bar;         // grid barrier (2 words)
  double* part;          // 2 * gridDim doubles
  int* flag;
  double tol2;           // squared relative residual the solve must reach (else the flag)
  double exit2;          // squared relative residual at which the sweeps stop early
};

__global__ void __launch_bounds__(RT) rich_kernel(const RichArgs a) {
  extern __shared__ __align__(16) double rsm[];
  __shared__ double srr[RT / 32], sbb[RT / 32];
  const int n = a.n, G = (int)gridDim.x;
  const int64_t nx = (int64_t)n * n;
  auto gemm_phase = [&](const double* A, const double* B, double* C, const double* emul, double beta) {
    for (int tl = blockIdx.x; tl < a.ntm * a.ntn; tl += G)
      gemm_tile(A, B, C, emul, beta, n, (tl / a.ntn) * TM, (tl % a.ntn) * TN, rsm);
    group_barrier(a.bar, G);
  };
  // x (+)= P^{-1} v
  auto precond = [&](const double* v, double beta) {
    gemm_phase(v, a.S1, a.T1, nullptr, 0.0);
    gemm_phase(a.S1, a.T1, a.T2, a.D, 0.0);
    gemm_phase(a.T2, a.S1, a.T1, nullptr, 0.0);
    gemm_phase(a.S1, a.T1, a.x, nullptr, beta);
  };
  // r = b - S x (x was written by other CTAs of this launch: L2 loads) and, after the grid
  // barrier, ||r||^2 and ||b||^2 summed in a fixed order by every CTA (identical values
  // everywhere, so the exit decision below is uniform across the grid)
  __shared__ double stot[2];
  auto residual = [&](double& rr_tot, double& bb_tot) {
    double rr = 0.0, bb = 0.0;
    for (int64_t i = (int64_t)blockIdx.x * RT + threadIdx.x; i < nx; i += (int64_t)G * RT) {
      const int i1 = (int)(i % n), i2 = (int)(i / n);
      const double xc = __ldcg(a.x + i);
      const double lx = stencil_lx(a.st, a.x, i, i1, i2, 0, [](const double* q) { return __ldcg(q); });
      const double bi = a.b[i];
      const double ri = bi - a.st.m_scale * (xc + a.st.tau * lx);
      a.r[i] = ri;
      rr += ri * ri;
      bb += bi * bi;
    }
    rr = warp_sum(rr);
    bb = warp_sum(bb);
    if ((threadIdx.x & 31) == 0) { srr[threadIdx.x >> 5] = rr; sbb[threadIdx.x >> 5] = bb; }
    __syncthreads();
    if (threadIdx.x == 0) {
      double s0 = 0.0, s1 = 0.0;
      for (int k = 0; k < RT / 32; ++k) { s0 += srr[k]; s1 += sbb[k]; }
      a.part[2 * blockIdx.x] = s0;
      a.part[2 * blockIdx.x + 1] = s1;
    }
    group_barrier(a.bar, G);
    double s0 = 0.0, s1 = 0.0;
    for (int k = threadIdx.x; k < G; k += RT) {
      s0 += __ldcg(a.part + 2 * k);
      s1 += __ldcg(a.part + 2 * k + 1);
    }
    s0 = warp_sum(s0);
    s1 = warp_sum(s1);
    if ((threadIdx.x & 31) == 0) { srr[threadIdx.x >> 5] = s0; sbb[threadIdx.x >> 5] = s1; }
    __syncthreads();
    if (threadIdx.x == 0) {
      double t0 = 0.0, t1 = 0.0;
      for (int k = 0; k < RT / 32; ++k) { t0 += srr[k]; t1 += sbb[k]; }
      stot[0] = t0;
      stot[1] = t1;
    }
    __syncthreads();
    rr_tot = stot[0];
    bb_tot = stot[1];
  };
  // The sweep bound comes from the contraction measured once per operator; the loop leaves
  // as soon as the true residual is below exit2 (a tenth of the step tolerance) or has
  // stopped contracting below the tolerance, which at C3 is 12-13 of the 16 sweeps the bound allows.  part[] is rewritten only after the four
  // GEMM phases (and their barriers) of the next sweep, i.e. after every CTA has read it.
  precond(a.b, 0.0);
  double rr = 0.0, bb = 0.0;
  bool done = false;
  int it = 0;
  double rr_prev = 0.0;
  for (; it < a.sweeps; ++it) {
    residual(rr, bb);
    // below a tenth of the tolerance, or below the tolerance and no longer contracting (the
    // attainable residual eps * cond(S) can sit between the two: n_t 256 at C3's grid)
    if (rr <= a.exit2 * bb || (it > 0 && rr <= a.tol2 * bb && rr > 0.49 * rr_prev)) {
      done = true;
      break;
    }
    rr_prev = rr;
    precond(a.r, 1.0);
  }
  if (!done) {
    residual(rr, bb);
    if (blockIdx.x == 0 && threadIdx.x == 0 && rr > a.tol2 * bb) *a.flag = 1;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {   // diagnostics (LRK_RICH_DEBUG): past the CTA partials
    a.part[RICH_PART_DIAG] = (double)it;
    a.part[RICH_PART_DIAG + 1] = rr;
    a.part[RICH_PART_DIAG + 2] = bb;
  }
}

size_t rich_smem_bytes() { return (size_t)NS * (TM * SA + TK * SB) * sizeof(double); }

// Launches the persistent step solve; returns cudaErrorNotSupported when the
// shape is outside its scope (the caller then takes the multi-launch path).
cudaError_t launch_rich(const StencilArgs& st, int n, int sweeps, const double* S1, const double* D,
                        const double* b, double* x, double* r, double* T1, double* T2, unsigned* bar,
                        double* part, int* flag, double tol2, int num_sms, cudaStream_t s) {
  if (st.dim != 2 || (n & 1) || st.wind_field) return cudaErrorNotSupported;
  static int max_ctas[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) return cudaErrorNotSupported;
  if (max_ctas[dev] == 0) {
    cudaError_t e = cudaFuncSetAttribute(rich_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)rich_smem_bytes());
    if (e != cudaSuccess) return e;
    int per_sm = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, rich_kernel, RT, rich_smem_bytes());
    if (e != cudaSuccess) return e;
    max_ctas[dev] = std::max(1, per_sm) * num_sms;
  }
  RichArgs a{};
  a.st = st;
  a.n = n; a.sweeps = sweeps; a.ntm = (n + TM - 1) / TM; a.ntn = (n + TN - 1) / TN;
  a.S1 = S1; a.D = D; a.b = b; a.x = x; a.r = r; a.T1 = T1; a.T2 = T2;
  a.bar = bar; a.part = part; a.flag = flag; a.tol2 = tol2; a.exit2 = 0.01 * tol2;
  const int G = std::min(std::min(a.ntm * a.ntn, RICH_PART_DIAG / 2), std::min(max_ctas[dev], 2 * num_sms));
  void* params[] = {(void*)&a};
  return cudaLaunchCooperativeKernel((const void*)rich_kernel, dim3(G), dim3(RT), params,
                                     rich_smem_bytes(), s);
}

}  // namespace lrk
