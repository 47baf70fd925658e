// lrk_sweep.cu — persistent cooperative kernel for the low-rank time sweep.
//
// Replaces st_solve_sweep (forward.py:133-188) for operators whose step
// matrix S = M(I + tau L) is diagonal in a fixed orthogonal basis (DST-I for
// the Dirichlet heat operator).  In that basis the reference's per-step sparse
// solve y_k = S^{-1}(M y_{k-1}) + B w2_k (forward.py:180) is the pointwise
// recurrence  y_k = theta .* y_{k-1} + rowscale .* (B w2_k),  so every column
// of the solution pane is produced row-locally.  Every `p` steps the buffered
// columns are folded into the pane exactly like flush() (forward.py:165-177):
// truncate(pane + [Y_buf, E_buf]).  Because the pane is kept canonical
// (orthonormal U, V) and the buffered time factors are unit selectors on
// unvisited rows, that truncation is an incremental SVD:
//   QR([U, Y]) = [U, Q~] [[I, C], [0, R~]]   (block CGS2 + Householder TSQR,
//                                             pivoted fix-up of the small R)
//   QR([V S, E]) = [V, E] diag(S, I)
//   core = [[S, C], [0, R~]]  ->  one-sided Jacobi SVD  ->  _rank_cut
// with the same zero test and rank cut as lr_truncate (lowrank.py:124-144).
// Orthogonal invariance makes the singular values (hence every rank decision)
// those of the reference; the pane is returned in the eigenbasis and mapped
// back by the caller.
//
// Grid: ngroups x ncta CTAs (one group per independent sweep), NT threads,
// one CTA per SM, launched cooperatively so all CTAs are co-resident.
#include "lrk_device.cuh"
#include "lrk_kernels.h"

namespace lrk {

namespace {
struct SweepSmem {
  // offsets in doubles
  static constexpr int off_C = 0;                         // NMAX*PMAX
  static constexpr int off_Yn = off_C + NMAX * PMAX;      // PMAX
  static constexpr int off_R = off_Yn + PMAX;             // PMAX^2
  static constexpr int off_Rp = off_R + PMAX * PMAX;      // PMAX^2
  static constexpr int off_X = off_Rp + PMAX * PMAX;      // PMAX^2
  static constexpr int off_G = off_X + PMAX * PMAX;       // PMAX^2
  static constexpr int off_I = off_G + PMAX * PMAX;       // PMAX^2
  static constexpr int off_Q = off_I + PMAX * PMAX;       // PMAX^2
  static constexpr int off_Rb = off_Q + PMAX * PMAX;      // PMAX^2
  static constexpr int off_tau = off_Rb + PMAX * PMAX;    // PMAX
  static constexpr int off_taut = off_tau + PMAX;         // PMAX
  static constexpr int off_cn = off_taut + PMAX;          // PMAX
  static constexpr int off_sig = off_cn + PMAX;           // NMAX
  static constexpr int off_s = off_sig + NMAX;            // NMAX
  static constexpr int off_inv = off_s + NMAX;            // NMAX
  static constexpr int off_nrm = off_inv + NMAX;          // NMAX
  static constexpr int off_red = off_nrm + NMAX;          // NWARP*PMAX
  static constexpr int off_tmp = off_red + NWARP * PMAX;  // PMAX
  static constexpr int off_scr = off_tmp + PMAX;          // NT
  static constexpr int off_part = off_scr + NT;           // NMAX*PMAX + PMAX
  static constexpr int off_jac = off_part + NMAX * PMAX + PMAX;  // 2*JMAX^2
  static constexpr int n_double = off_jac + 2 * JMAX_SMEM * JMAX_SMEM;
  static constexpr int n_int = NMAX + PMAX + 8;
  static constexpr size_t bytes = n_double * sizeof(double) + n_int * sizeof(int);
};
}  // namespace

size_t sweep_smem_bytes() { return SweepSmem::bytes; }
int64_t sweep_scratch_stride(int ncta) {
  return 2 * (int64_t)ncta * PMAX * PMAX + 2 * (int64_t)NMAX * NMAX;
}
int64_t sweep_part_stride() { return NMAX * PMAX + PMAX + 8; }

__global__ void __launch_bounds__(NT, 1) sweep_kernel(const SweepArgs* __restrict__ all_args) {
  extern __shared__ double sm[];
  const int ncta = all_args[0].ncta;
  const SweepArgs& a = all_args[blockIdx.x / ncta];
  const int cta = blockIdx.x % ncta;
  const int tid = threadIdx.x;

  double* sC = sm + SweepSmem::off_C;
  double* sYn = sm + SweepSmem::off_Yn;
  double* sR = sm + SweepSmem::off_R;
  double* sRp = sm + SweepSmem::off_Rp;
  double* sX = sm + SweepSmem::off_X;
  double* sG = sm + SweepSmem::off_G;
  double* sI = sm + SweepSmem::off_I;
  double* sQ = sm + SweepSmem::off_Q;
  double* sRb = sm + SweepSmem::off_Rb;
  double* sTau = sm + SweepSmem::off_tau;
  double* sTauT = sm + SweepSmem::off_taut;
  double* sCn = sm + SweepSmem::off_cn;
  double* sSig = sm + SweepSmem::off_sig;
  double* sS = sm + SweepSmem::off_s;
  double* sInv = sm + SweepSmem::off_inv;
  double* sNrm = sm + SweepSmem::off_nrm;
  double* sRed = sm + SweepSmem::off_red;
  double* sTmp = sm + SweepSmem::off_tmp;
  double* sScr = sm + SweepSmem::off_scr;
  double* sPart = sm + SweepSmem::off_part;
  double* sJac = sm + SweepSmem::off_jac;
  int* iPerm = reinterpret_cast<int*>(sm + SweepSmem::n_double);
  int* iPiv = iPerm + NMAX;
  int* iFlag = iPiv + PMAX;  // [0] jacobi flag, [1] new rank, [2] error

  const int64_t n_x = a.n_x;
  const int n_t = a.n_t;
  const int p = a.p;
  const int rb = a.rb_dev ? min(a.rb, *a.rb_dev) : a.rb;
  int64_t r0, r1, t0, t1;
  row_range(n_x, cta, ncta, r0, r1);
  row_range(n_t, cta, ncta, t0, t1);
  const int m_loc = (int)(r1 - r0);

  double* Ucur = a.U0;
  double* Ualt = a.U1;
  double* Vcur = a.V0;
  double* Valt = a.V1;
  int r = 0;

  double* stack = a.scratch + (int64_t)cta * a.scratch_stride;
  double* stackY = stack + (int64_t)ncta * PMAX * PMAX;
  double* jacG = stackY + (int64_t)ncta * PMAX * PMAX;

  double* part1 = a.part;
  double* part2 = a.part + (int64_t)ncta * a.pstride;
  double* part3 = a.part + 2 * (int64_t)ncta * a.pstride;

  for (int64_t i = r0 + tid; i < r1; i += NT) a.yprev[i] = 0.0;
  for (int i = tid; i < PMAX * PMAX; i += NT) sI[i] = 0.0;
  __syncthreads();

  const int nflush = (n_t + p - 1) / p;
  for (int f = 0; f < nflush; ++f) {
    const int start = f * p;
    const int pc = (n_t - start) < p ? (n_t - start) : p;
    if (tid < pc) sI[tid * pc + tid] = 1.0;  // identity pc x pc (row-major)
    // ---------------- phase 1: generate the buffered columns (row-local)
    for (int64_t row = r0 + tid; row < r1; row += NT) {
      double acc[PMAX];
#pragma unroll
      for (int s = 0; s < PMAX; ++s) acc[s] = 0.0;
      for (int j = 0; j < rb; ++j) {
        const double b = a.B[row + (int64_t)j * a.ldb];
        const double* w2 = a.W2 + (int64_t)j * a.ldw2;
#pragma unroll
        for (int s = 0; s < PMAX; ++s) {
          if (s < pc) {
            const int k = a.adjoint ? (n_t - 1 - (start + s)) : (start + s);
            acc[s] += b * w2[k];
          }
        }
      }
      const double th = a.theta[row];
      const double rs = a.rowscale ? a.rowscale[row] : 1.0;
      double y = a.yprev[row];
#pragma unroll
      for (int s = 0; s < PMAX; ++s) {
        if (s < pc) {
          y = th * y + rs * acc[s];
          a.ybuf[row + (int64_t)s * a.ldy] = y;
        }
      }
      a.yprev[row] = y;
    }
    __syncthreads();
    double* Yl = a.ybuf + r0;
    const double* Ul = Ucur + r0;
    // partial: [U^T Y (r x pc) | ||Y_s||^2 (pc)]
    if (r > 0) cta_tn(Ul, a.ldu, r, Yl, a.ldy, pc, m_loc, sPart, sScr);
    {
      double v[PMAX];
#pragma unroll
      for (int s = 0; s < PMAX; ++s) v[s] = 0.0;
      for (int i = tid; i < m_loc; i += NT) {
#pragma unroll
        for (int s = 0; s < PMAX; ++s)
          if (s < pc) { const double y = Yl[i + (int64_t)s * a.ldy]; v[s] += y * y; }
      }
      block_sum<PMAX>(v, sRed, sTmp);
      if (tid < pc) sPart[r * pc + tid] = v[tid];
    }
    __syncthreads();
    for (int i = tid; i < r * pc + pc; i += NT) part1[(int64_t)cta * a.pstride + i] = sPart[i];
    group_barrier(a.bar, ncta);
    // ---------------- phase 2: block CGS2 against the orthonormal pane
    reduce_partials(part1, a.pstride, ncta, r * pc + pc, sPart);
    for (int i = tid; i < pc; i += NT) sYn[i] = sPart[r * pc + i];
    for (int i = tid; i < r * pc; i += NT) sC[i] = sPart[i];
    __syncthreads();
    if (r > 0) {
      rows_sub_gemm(Yl, a.ldy, pc, Ul, a.ldu, r, sC, m_loc);
      __syncthreads();
      cta_tn(Ul, a.ldu, r, Yl, a.ldy, pc, m_loc, sPart, sScr);
      for (int i = tid; i < r * pc; i += NT) part2[(int64_t)cta * a.pstride + i] = sPart[i];
      group_barrier(a.bar, ncta);
      reduce_partials(part2, a.pstride, ncta, r * pc, sPart);
      rows_sub_gemm(Yl, a.ldy, pc, Ul, a.ldu, r, sPart, m_loc);
      for (int i = tid; i < r * pc; i += NT) sC[i] += sPart[i];
      __syncthreads();
    }
    // ---------------- phase 3: local Householder QR of the remainder
    block_householder_qr(Yl, a.ldy, m_loc, pc, sTau, sR, sRed, sTmp);
    for (int i = tid; i < pc * pc; i += NT) part3[(int64_t)cta * a.pstride + i] = sR[i];
    group_barrier(a.bar, ncta);
    // ---------------- phase 4 (every CTA, redundantly): finish TSQR + SVD
    const int ms = ncta * pc;
    if (tid < 32) {
      for (int idx = tid; idx < ms * pc; idx += 32) {
        const int c = idx / ms, rr = idx % ms;
        const int owner = rr / pc, lr = rr % pc;
        stack[rr + (int64_t)c * ms] = __ldcg(part3 + (int64_t)owner * a.pstride + lr * pc + c);
      }
      __syncwarp();
      warp_householder_qr(stack, ms, ms, pc, sTauT, sRp);
      // rows of the stacked Q that belong to this CTA
      warp_householder_q_rows(stack, ms, ms, pc, sTauT, sI, stackY, ms, cta * pc, pc, sQ);
      if (tid == 0) {
        // rank-revealing fix-up: Rp P = X Rt (column pivoting)
        for (int i = 0; i < pc * pc; ++i) sRb[i] = sRp[i];
        small_pivoted_qr(sRb, pc, sX, iPiv, sCn);
        double ysq = 0.0;
        for (int s = 0; s < pc; ++s) ysq += sYn[s];
        const double delta = 16.0 * DEPS * sqrt(ysq);
        for (int j = 0; j < pc; ++j) {
          if (fabs(sRb[j * pc + j]) <= delta) {
            for (int k = 0; k < pc; ++k) { sRb[j * pc + k] = 0.0; sX[k * pc + j] = 0.0; }
          }
        }
        // Rblock (original column order) into sRp; G = Qrows * X into sG
        for (int j = 0; j < pc; ++j)
          for (int kk = 0; kk < pc; ++kk) sRp[j * pc + iPiv[kk]] = sRb[j * pc + kk];
        for (int i = 0; i < pc; ++i)
          for (int j = 0; j < pc; ++j) {
            double acc = 0.0;
            for (int k = 0; k < pc; ++k) acc += sQ[i * pc + k] * sX[k * pc + j];
            sG[i * pc + j] = acc;
          }
      }
    }
    __syncthreads();
    // explicit Q~ rows of this CTA: Q_loc * G  -> qbuf
    block_householder_apply_q(Yl, a.ldy, m_loc, pc, sTau, sG, a.qbuf + r0, a.ldq, sRed, sTmp);
    // core matrix (n x n, col-major) = [[diag(sig), C], [0, Rblock]]
    const int n = r + pc;
    if (n > NMAX) {  // uniform across the group; report and stop
      if (tid == 0 && cta == 0) a.info[2] = 1;
      return;
    }
    double* Aj = (n <= JMAX_SMEM) ? sJac : jacG;
    double* Vj = Aj + n * n;
    const int lda = n;
    for (int idx = tid; idx < n * n; idx += NT) {
      const int i = idx % n, j = idx / n;
      double v = 0.0;
      if (i < r) {
        if (j < r) v = (i == j) ? sSig[i] : 0.0;
        else v = sC[i * pc + (j - r)];
      } else if (j >= r) {
        v = sRp[(i - r) * pc + (j - r)];
      }
      Aj[i + j * lda] = v;
    }
    __syncthreads();
    jacobi_svd(Aj, lda, Vj, lda, n, sS, iPerm, sNrm, iFlag);
    if (tid == 0) {
      double ysq = 0.0, ssq = 0.0;
      for (int s = 0; s < pc; ++s) ysq += sYn[s];
      for (int i = 0; i < r; ++i) ssq += sSig[i] * sSig[i];
      const double fs = sqrt((double)r + ysq) * sqrt(ssq + (double)pc);
      int rn;
      if (n == 0 || sS[0] <= NOISE_FLOOR * fs) rn = 0;
      else rn = rank_cut_dev(sS, n, a.eps0, a.r_max);
      if (rn > a.ucap) { rn = a.ucap; if (cta == 0) a.info[2] = 2; }
      iFlag[1] = rn;
      for (int k = 0; k < rn; ++k) sInv[k] = 1.0 / sS[k];
    }
    __syncthreads();
    const int rn = iFlag[1];
    // ---------------- basis update (row-local): U' = [U, Q~] Uc[:, :rn]
    for (int c0 = 0; c0 < rn; c0 += 8) {
      const int cn = (rn - c0) < 8 ? (rn - c0) : 8;
      for (int64_t row = r0 + tid; row < r1; row += NT) {
        double acc[8];
#pragma unroll
        for (int c = 0; c < 8; ++c) acc[c] = 0.0;
        for (int i = 0; i < n; ++i) {
          const double x = (i < r) ? Ucur[row + (int64_t)i * a.ldu]
                                   : a.qbuf[row + (int64_t)(i - r) * a.ldq];
#pragma unroll
          for (int c = 0; c < 8; ++c)
            if (c < cn) acc[c] += x * Aj[i + iPerm[c0 + c] * lda];
        }
#pragma unroll
        for (int c = 0; c < 8; ++c)
          if (c < cn) Ualt[row + (int64_t)(c0 + c) * a.ldu] = acc[c] * sInv[c0 + c];
      }
      // time basis: V' = [V, E] Vc[:, :rn]
      for (int64_t t = t0 + tid; t < t1; t += NT) {
        int sel = a.adjoint ? (n_t - 1 - start) - (int)t : (int)t - start;
        if (sel < 0 || sel >= pc) sel = -1;
        double acc[8];
#pragma unroll
        for (int c = 0; c < 8; ++c) acc[c] = 0.0;
        for (int i = 0; i < r; ++i) {
          const double x = Vcur[t + (int64_t)i * a.ldv];
#pragma unroll
          for (int c = 0; c < 8; ++c)
            if (c < cn) acc[c] += x * Vj[i + iPerm[c0 + c] * lda];
        }
        if (sel >= 0) {
#pragma unroll
          for (int c = 0; c < 8; ++c)
            if (c < cn) acc[c] += Vj[(r + sel) + iPerm[c0 + c] * lda];
        }
#pragma unroll
        for (int c = 0; c < 8; ++c)
          if (c < cn) Valt[t + (int64_t)(c0 + c) * a.ldv] = acc[c];
      }
    }
    for (int k = tid; k < rn; k += NT) sSig[k] = sS[k];
    if (tid == 0 && cta == 0) a.trace[f] = rn;
    __syncthreads();
    r = rn;
    { double* t = Ucur; Ucur = Ualt; Ualt = t; }
    { double* t = Vcur; Vcur = Valt; Valt = t; }
    if (tid < pc) sI[tid * pc + tid] = 0.0;
    __syncthreads();
  }
  // leave the result in slot 0 (row-local copies, no barrier needed)
  if (Ucur != a.U0) {
    for (int c = 0; c < r; ++c) {
      for (int64_t i = r0 + tid; i < r1; i += NT) a.U0[i + (int64_t)c * a.ldu] = Ucur[i + (int64_t)c * a.ldu];
      for (int64_t t = t0 + tid; t < t1; t += NT) a.V0[t + (int64_t)c * a.ldv] = Vcur[t + (int64_t)c * a.ldv];
    }
  }
  if (cta == 0) {
    for (int k = tid; k < r; k += NT) a.sigma[k] = sSig[k];
    if (tid == 0) {
      a.info[0] = r;
      a.info[1] = 0;
      a.trace[nflush] = r;
    }
  }
}

cudaError_t launch_sweep(const SweepArgs* d_args, int ngroups, int ncta, cudaStream_t s) {
  static bool attr_set = false;
  const size_t smem = SweepSmem::bytes;
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(sweep_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  void* params[] = {(void*)&d_args};
  return cudaLaunchCooperativeKernel((const void*)sweep_kernel, dim3(ngroups * ncta), dim3(NT),
                                     params, smem, s);
}

}  // namespace lrk
