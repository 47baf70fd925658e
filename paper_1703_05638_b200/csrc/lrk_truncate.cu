// lrk_truncate.cu — persistent cooperative kernel for lr_truncate.
//
// Reference: lr_truncate (lowrank.py:124-144):
//   Q1 R1 = qr(W1); Q2 R2 = qr(W2); U s Vt = svd(R1 R2^T);
//   zero test s0 <= 1e-15 ||R1|| ||R2||; r = _rank_cut(s) (lowrank.py:98-111);
//   U = Q1 U[:, :r], V = Q2 Vt[:r].T * s[:r]; _svd_flip (lowrank.py:114-121).
// Here the two thin QRs are blocked Gram-Schmidt (two projection passes per
// block of <= PB columns) with a Householder TSQR of each block remainder and
// a column-pivoted fix-up of its small R (rank-revealing, so dependent
// columns never inject non-orthogonal directions).  The core SVD is a
// one-sided Jacobi computed redundantly by every CTA of the group.
#include "../../include/lrk.h"
#include "lrk_device.cuh"
#include "lrk_kernels.h"
#include "lrk_small.cuh"

namespace lrk {

namespace {
constexpr int PB = 8;  // QR block width

struct TruncSmem {
  static constexpr int off_C = 0;                       // NMAX*PB
  static constexpr int off_Yn = off_C + NMAX * PB;      // PB
  static constexpr int off_R = off_Yn + PB;             // PMAX^2 (local R)
  static constexpr int off_Rp = off_R + PMAX * PMAX;
  static constexpr int off_X = off_Rp + PMAX * PMAX;
  static constexpr int off_G = off_X + PMAX * PMAX;
  static constexpr int off_I = off_G + PMAX * PMAX;
  static constexpr int off_Q = off_I + PMAX * PMAX;
  static constexpr int off_Rb = off_Q + PMAX * PMAX;
  static constexpr int off_tau = off_Rb + PMAX * PMAX;  // PMAX
  static constexpr int off_taut = off_tau + PMAX;
  static constexpr int off_cn = off_taut + PMAX;
  static constexpr int off_s = off_cn + PMAX;           // NMAX
  static constexpr int off_inv = off_s + NMAX;          // NMAX
  static constexpr int off_nrm = off_inv + NMAX;        // NMAX
  static constexpr int off_misc = off_nrm + NMAX;       // 16
  static constexpr int off_red = off_misc + 16;         // NWARP*PMAX
  static constexpr int off_tmp = off_red + NWARP * PMAX;
  static constexpr int off_scr = off_tmp + PMAX;        // NT
  static constexpr int off_part = off_scr + NT;         // 3*NMAX + NMAX*PB + 8
  static constexpr int off_jac = off_part + 3 * NMAX + NMAX * PB + 8;
  static constexpr int n_double = off_jac + 2 * JMAX_SMEM * JMAX_SMEM;
  static constexpr int n_int = NMAX + PMAX + 8;
  static constexpr size_t bytes = n_double * sizeof(double) + n_int * sizeof(int);
};

struct TS {  // shared-memory pointers
  double *C, *Yn, *R, *Rp, *X, *G, *I, *Q, *Rb, *tau, *taut, *cn, *s, *inv, *nrm, *misc, *red,
      *tmp, *scr, *part, *jac;
  int *perm, *piv, *flag;
};
}  // namespace

size_t trunc_smem_bytes() { return TruncSmem::bytes; }
int64_t trunc_part_stride() { return 3 * NMAX + NMAX * PB + 8; }
int64_t trunc_scratch_stride(int ncta) {
  // stack + stackY + R1 + R2 + jacobi(2)
  return 2 * (int64_t)ncta * PMAX * PMAX + 4 * (int64_t)NMAX * NMAX;
}

// Blocked QR of X (N rows split over the group, R columns) into Q (N x R)
// and Rm (R x R row-major, per-CTA copy).  tmp: N x PMAX workspace.
__device__ void group_blocked_qr(const double* X, int64_t ldx, int64_t N, int R, double* Q,
                                 int64_t ldq, double* Rm, double* tmp, int64_t ldt,
                                 const TruncArgs& a, int cta, TS& s, double* stack,
                                 double* stackY, int& pphase) {
  const int ncta = a.ncta, tid = threadIdx.x;
  int64_t r0, r1;
  row_range(N, cta, ncta, r0, r1);
  const int m_loc = (int)(r1 - r0);
  for (int i = tid; i < R * R; i += NT) Rm[i] = 0.0;
  __syncthreads();
  auto next_part = [&]() -> double* {
    double* p = a.part + (int64_t)pphase * ncta * a.pstride;
    pphase = (pphase + 1) % 3;
    return p;
  };
  for (int b0 = 0; b0 < R; b0 += PB) {
    const int pc = (R - b0) < PB ? (R - b0) : PB;
    double* Yl = Q + r0 + (int64_t)b0 * ldq;
    for (int c = 0; c < pc; ++c)
      for (int64_t i = r0 + tid; i < r1; i += NT)
        Q[i + (int64_t)(b0 + c) * ldq] = X[i + (int64_t)(b0 + c) * ldx];
    __syncthreads();
    const double* Ql = Q + r0;
    // projections against the first b0 (orthonormal) columns + block norms
    if (b0 > 0) cta_tn(Ql, ldq, b0, Yl, ldq, pc, m_loc, s.part, s.scr);
    {
      double v[PMAX];
#pragma unroll
      for (int c = 0; c < PMAX; ++c) v[c] = 0.0;
      for (int i = tid; i < m_loc; i += NT) {
#pragma unroll
        for (int c = 0; c < PMAX; ++c)
          if (c < pc) { const double y = Yl[i + (int64_t)c * ldq]; v[c] += y * y; }
      }
      block_sum<PMAX>(v, s.red, s.tmp);
      if (tid < pc) s.part[b0 * pc + tid] = v[tid];
    }
    __syncthreads();
    double* p1 = next_part();
    for (int i = tid; i < b0 * pc + pc; i += NT) p1[(int64_t)cta * a.pstride + i] = s.part[i];
    group_barrier(a.bar, ncta);
    reduce_partials(p1, a.pstride, ncta, b0 * pc + pc, s.part);
    for (int i = tid; i < pc; i += NT) s.Yn[i] = s.part[b0 * pc + i];
    for (int i = tid; i < b0 * pc; i += NT) s.C[i] = s.part[i];
    __syncthreads();
    if (b0 > 0) {
      rows_sub_gemm(Yl, ldq, pc, Ql, ldq, b0, s.C, m_loc);
      __syncthreads();
      cta_tn(Ql, ldq, b0, Yl, ldq, pc, m_loc, s.part, s.scr);
      double* p2 = next_part();
      for (int i = tid; i < b0 * pc; i += NT) p2[(int64_t)cta * a.pstride + i] = s.part[i];
      group_barrier(a.bar, ncta);
      reduce_partials(p2, a.pstride, ncta, b0 * pc, s.part);
      rows_sub_gemm(Yl, ldq, pc, Ql, ldq, b0, s.part, m_loc);
      for (int i = tid; i < b0 * pc; i += NT) s.C[i] += s.part[i];
      __syncthreads();
    }
    // R entries above the block
    for (int idx = tid; idx < b0 * pc; idx += NT) {
      const int i = idx / pc, c = idx % pc;
      Rm[i * R + b0 + c] = s.C[idx];
    }
    // TSQR of the remainder
    block_householder_qr(Yl, ldq, m_loc, pc, s.tau, s.R, s.red, s.tmp);
    double* p3 = next_part();
    for (int i = tid; i < pc * pc; i += NT) p3[(int64_t)cta * a.pstride + i] = s.R[i];
    for (int i = tid; i < PMAX * PMAX; i += NT) s.I[i] = 0.0;
    __syncthreads();
    if (tid < pc) s.I[tid * pc + tid] = 1.0;
    group_barrier(a.bar, ncta);
    const int ms = ncta * pc;
    if (tid < 32) {
      for (int idx = tid; idx < ms * pc; idx += 32) {
        const int c = idx / ms, rr = idx % ms;
        const int owner = rr / pc, lr = rr % pc;
        stack[rr + (int64_t)c * ms] = __ldcg(p3 + (int64_t)owner * a.pstride + lr * pc + c);
      }
      __syncwarp();
      warp_householder_qr(stack, ms, ms, pc, s.taut, s.Rp);
      warp_householder_q_rows(stack, ms, ms, pc, s.taut, s.I, stackY, ms, cta * pc, pc, s.Q);
      if (tid == 0) {
        for (int i = 0; i < pc * pc; ++i) s.Rb[i] = s.Rp[i];
        small_pivoted_qr(s.Rb, pc, s.X, s.piv, s.cn);
        double ysq = 0.0;
        for (int c = 0; c < pc; ++c) ysq += s.Yn[c];
        const double delta = 16.0 * DEPS * sqrt(ysq);
        for (int j = 0; j < pc; ++j)
          if (fabs(s.Rb[j * pc + j]) <= delta)
            for (int k = 0; k < pc; ++k) { s.Rb[j * pc + k] = 0.0; s.X[k * pc + j] = 0.0; }
        for (int j = 0; j < pc; ++j)
          for (int kk = 0; kk < pc; ++kk) Rm[(b0 + j) * R + b0 + s.piv[kk]] = s.Rb[j * pc + kk];
        for (int i = 0; i < pc; ++i)
          for (int j = 0; j < pc; ++j) {
            double acc = 0.0;
            for (int k = 0; k < pc; ++k) acc += s.Q[i * pc + k] * s.X[k * pc + j];
            s.G[i * pc + j] = acc;
          }
      }
    }
    __syncthreads();
    block_householder_apply_q(Yl, ldq, m_loc, pc, s.tau, s.G, tmp + r0, ldt, s.red, s.tmp);
    for (int c = 0; c < pc; ++c)
      for (int64_t i = r0 + tid; i < r1; i += NT)
        Q[i + (int64_t)(b0 + c) * ldq] = tmp[i + (int64_t)c * ldt];
    __syncthreads();
  }
}

__global__ void __launch_bounds__(NT, 1) truncate_kernel(const __grid_constant__ TruncArgs a) {
  extern __shared__ double sm[];
  const int ncta = a.ncta, cta = blockIdx.x, tid = threadIdx.x;
  TS s;
  s.C = sm + TruncSmem::off_C; s.Yn = sm + TruncSmem::off_Yn; s.R = sm + TruncSmem::off_R;
  s.Rp = sm + TruncSmem::off_Rp; s.X = sm + TruncSmem::off_X; s.G = sm + TruncSmem::off_G;
  s.I = sm + TruncSmem::off_I; s.Q = sm + TruncSmem::off_Q; s.Rb = sm + TruncSmem::off_Rb;
  s.tau = sm + TruncSmem::off_tau; s.taut = sm + TruncSmem::off_taut; s.cn = sm + TruncSmem::off_cn;
  s.s = sm + TruncSmem::off_s; s.inv = sm + TruncSmem::off_inv; s.nrm = sm + TruncSmem::off_nrm;
  s.misc = sm + TruncSmem::off_misc; s.red = sm + TruncSmem::off_red; s.tmp = sm + TruncSmem::off_tmp;
  s.scr = sm + TruncSmem::off_scr; s.part = sm + TruncSmem::off_part; s.jac = sm + TruncSmem::off_jac;
  s.perm = reinterpret_cast<int*>(sm + TruncSmem::n_double);
  s.piv = s.perm + NMAX;
  s.flag = s.piv + PMAX;

  const int R = a.R_dev ? min(a.R, *a.R_dev) : a.R;
  double* scr = a.scratch + (int64_t)cta * a.scratch_stride;
  double* stack = scr;
  double* stackY = stack + (int64_t)ncta * PMAX * PMAX;
  double* R1 = stackY + (int64_t)ncta * PMAX * PMAX;
  double* R2 = R1 + (int64_t)NMAX * NMAX;
  double* jacG = R2 + (int64_t)NMAX * NMAX;
  int pphase = 0;

  int64_t x0, x1, t0, t1;
  row_range(a.n_x, cta, ncta, x0, x1);
  row_range(a.n_t, cta, ncta, t0, t1);

  // ---- QR of W1
  const double* Q1 = a.W1;
  int64_t ldq1 = a.ld1;
  if (!(a.flags & LRK_TRUNC_W1_ORTHO)) {
    group_blocked_qr(a.W1, a.ld1, a.n_x, R, a.Q1, a.ldq1, R1, a.tmpw, a.ldtmp,
                     a, cta, s, stack, stackY, pphase);
    Q1 = a.Q1;
    ldq1 = a.ldq1;
  } else {
    for (int i = tid; i < R * R; i += NT) R1[i] = (i / R == i % R) ? 1.0 : 0.0;
  }
  // ---- QR of W2
  const double* Q2 = a.W2;
  int64_t ldq2 = a.ld2;
  bool w2_colscaled = (a.flags & LRK_TRUNC_W2_ORTHOSCALED) != 0;
  if (!w2_colscaled) {
    group_blocked_qr(a.W2, a.ld2, a.n_t, R, a.Q2, a.ldq2, R2, a.tmpw, a.ldtmp,
                     a, cta, s, stack, stackY, pphase);
    Q2 = a.Q2;
    ldq2 = a.ldq2;
  } else {
    // column norms of W2 (R2 = diag(norms), Q2 = W2 / norms)
    for (int c = 0; c < R; ++c) {
      double v[1] = {0.0};
      for (int64_t t = t0 + tid; t < t1; t += NT) { const double x = a.W2[t + (int64_t)c * a.ld2]; v[0] += x * x; }
      block_sum<1>(v, s.red, s.tmp);
      if (tid == 0) s.part[c] = v[0];
    }
    __syncthreads();
    double* p = a.part + (int64_t)pphase * ncta * a.pstride;
    pphase = (pphase + 1) % 3;
    for (int i = tid; i < R; i += NT) p[(int64_t)cta * a.pstride + i] = s.part[i];
    group_barrier(a.bar, ncta);
    reduce_partials(p, a.pstride, ncta, R, s.part);
    for (int i = tid; i < R * R; i += NT) R2[i] = (i / R == i % R) ? sqrt(s.part[i / R]) : 0.0;
    for (int i = tid; i < R; i += NT) s.nrm[i] = s.part[i] > 0.0 ? 1.0 / sqrt(s.part[i]) : 0.0;
  }
  __syncthreads();
  // ---- core = R1 R2^T, Frobenius norms for the zero test
  const int n = R;
  double* Aj = (n <= JMAX_SMEM) ? s.jac : jacG;
  double* Vj = Aj + n * n;
  double* colscale = s.inv;  // reuse as Q2 column scaling when colscaled
  if (w2_colscaled)
    for (int i = tid; i < R; i += NT) colscale[i] = s.nrm[i];
  __syncthreads();
  for (int idx = tid; idx < n * n; idx += NT) {
    const int i = idx % n, j = idx / n;
    double acc = 0.0;
    for (int k = 0; k < R; ++k) acc += R1[i * R + k] * R2[j * R + k];
    Aj[i + j * n] = acc;
  }
  {
    double v[2] = {0.0, 0.0};
    for (int idx = tid; idx < R * R; idx += NT) { v[0] += R1[idx] * R1[idx]; v[1] += R2[idx] * R2[idx]; }
    block_sum<2>(v, s.red, s.tmp);
    if (tid == 0) s.misc[0] = sqrt(v[0]) * sqrt(v[1]);
  }
  __syncthreads();
  // core SVD: the 4-warp register Jacobi of the sweep for n <= 32 (outputs
  // normalised and sorted, U to the per-CTA global scratch), the CTA-wide
  // Jacobi beyond
  const bool reg_svd = n <= 32;
  const double* Ucol = Aj;
  if (reg_svd) {
    if (tid < 128) {
      if (n <= 8) multi_warp_jacobi<8, 4>(Aj, n, n, jacG, Vj, n, s.s, s.perm, s.scr);
      else if (n <= 16) multi_warp_jacobi<16, 4>(Aj, n, n, jacG, Vj, n, s.s, s.perm, s.scr);
      else if (n <= 24) multi_warp_jacobi<24, 4>(Aj, n, n, jacG, Vj, n, s.s, s.perm, s.scr);
      else multi_warp_jacobi<32, 4>(Aj, n, n, jacG, Vj, n, s.s, s.perm, s.scr);
    }
    Ucol = jacG;
    __syncthreads();
    for (int k = tid; k < n; k += NT) s.perm[k] = k;
    __syncthreads();
  } else {
    jacobi_svd(Aj, n, Vj, n, n, s.s, s.perm, s.nrm, s.flag, s.tmp);
  }
  if (tid == 0) {
    int rn;
    if (n == 0 || s.s[0] <= NOISE_FLOOR * s.misc[0]) rn = 0;
    else rn = rank_cut_dev(s.s, n, a.eps0, a.r_max);
    if (rn > a.cap) { rn = a.cap; if (cta == 0) a.info[2] = 2; }
    s.flag[1] = rn;
  }
  __syncthreads();
  const int rn = s.flag[1];
  if (cta == 0) {
    for (int k = tid; k < rn; k += NT) if (a.sigma) a.sigma[k] = s.s[k];
    for (int k = tid; k < n; k += NT) if (a.sv_all) a.sv_all[k] = s.s[k];
  }
  // ---- outputs: out1 = Q1 Uc, out2 = Q2 Vc diag(s)
  for (int c0 = 0; c0 < rn; c0 += 8) {
    const int cn = (rn - c0) < 8 ? (rn - c0) : 8;
    for (int64_t row = x0 + tid; row < x1; row += NT) {
      double acc[8];
#pragma unroll
      for (int c = 0; c < 8; ++c) acc[c] = 0.0;
      for (int i = 0; i < n; ++i) {
        const double x = Q1[row + (int64_t)i * ldq1];
#pragma unroll
        for (int c = 0; c < 8; ++c)
          if (c < cn) acc[c] += x * Ucol[i + s.perm[c0 + c] * n];
      }
#pragma unroll
      for (int c = 0; c < 8; ++c)
        if (c < cn) a.out1[row + (int64_t)(c0 + c) * a.ldo1] = reg_svd ? acc[c] : acc[c] / s.s[c0 + c];
    }
    for (int64_t t = t0 + tid; t < t1; t += NT) {
      double acc[8];
#pragma unroll
      for (int c = 0; c < 8; ++c) acc[c] = 0.0;
      for (int i = 0; i < n; ++i) {
        double x = Q2[t + (int64_t)i * ldq2];
        if (w2_colscaled) x *= colscale[i];
#pragma unroll
        for (int c = 0; c < 8; ++c)
          if (c < cn) acc[c] += x * Vj[i + s.perm[c0 + c] * n];
      }
#pragma unroll
      for (int c = 0; c < 8; ++c)
        if (c < cn) a.out2[t + (int64_t)(c0 + c) * a.ldo2] = acc[c] * s.s[c0 + c];
    }
  }
  __syncthreads();
  // ---- _svd_flip: largest-|entry| of each U column positive (first index on ties)
  if (!a.no_flip && rn > 0) {
    const int lane = tid & 31, w = tid >> 5;
    double* p = a.part + (int64_t)pphase * ncta * a.pstride;
    pphase = (pphase + 1) % 3;
    for (int c = w; c < rn; c += NWARP) {
      double best = -1.0, bval = 0.0;
      long long bidx = 0;
      for (int64_t row = x0 + lane; row < x1; row += 32) {
        const double x = a.out1[row + (int64_t)c * a.ldo1];
        if (fabs(x) > best) { best = fabs(x); bidx = row; bval = x; }
      }
      for (int o = 16; o > 0; o >>= 1) {
        const double ob = __shfl_xor_sync(0xffffffffu, best, o);
        const long long oi = __shfl_xor_sync(0xffffffffu, bidx, o);
        const double ov = __shfl_xor_sync(0xffffffffu, bval, o);
        if (ob > best || (ob == best && oi < bidx)) { best = ob; bidx = oi; bval = ov; }
      }
      if (lane == 0) {
        double* q = p + (int64_t)cta * a.pstride + 3 * c;
        q[0] = best; q[1] = (double)bidx; q[2] = bval;
      }
    }
    group_barrier(a.bar, ncta);
    for (int c = tid; c < rn; c += NT) {
      double best = -1.0, bval = 0.0, bidx = 0.0;
      for (int k = 0; k < ncta; ++k) {
        const double* q = p + (int64_t)k * a.pstride + 3 * c;
        const double b = __ldcg(q), ix = __ldcg(q + 1), v = __ldcg(q + 2);
        if (b > best || (b == best && ix < bidx)) { best = b; bidx = ix; bval = v; }
      }
      s.nrm[c] = (bval < 0.0) ? -1.0 : 1.0;
    }
    __syncthreads();
    for (int c = 0; c < rn; ++c) {
      const double sg = s.nrm[c];
      if (sg < 0.0) {
        for (int64_t row = x0 + tid; row < x1; row += NT) a.out1[row + (int64_t)c * a.ldo1] *= -1.0;
        for (int64_t t = t0 + tid; t < t1; t += NT) a.out2[t + (int64_t)c * a.ldo2] *= -1.0;
      }
    }
  }
  if (cta == 0 && tid == 0) a.info[0] = rn;
}

cudaError_t launch_truncate(const TruncArgs& args, cudaStream_t st) {
  // the opt-in shared-memory size is a per-device function attribute
  static bool attr_set[64] = {};
  const size_t smem = TruncSmem::bytes;
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64 || !attr_set[dev]) {
    cudaError_t e = cudaFuncSetAttribute(truncate_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess) return e;
    if (dev >= 0 && dev < 64) attr_set[dev] = true;
  }
  void* params[] = {(void*)&args};
  return cudaLaunchCooperativeKernel((const void*)truncate_kernel, dim3(args.ncta), dim3(NT), params,
                                     smem, st);
}

}  // namespace lrk
