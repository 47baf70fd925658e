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
// Latency design (the sweep is a chain of n_t/p dependent truncations):
//  * every CTA keeps its block of U, Y, Q~, the carried column and the
//    eigenvalues resident in shared memory for the whole sweep when they fit
//    (sweep_plan), so row-local passes never touch L2;
//  * three grid barriers per flush; the small algebra (stacked-R QR, pivoted
//    fix-up, core SVD, rank cut) is computed redundantly by every CTA from the
//    same reduced partials, so no broadcast barrier is needed;
//  * the core SVD is a register-resident single-warp Jacobi (no CTA barrier);
//  * all loops are specialised on the flush width Q (template) and the basis
//    update runs in place with register accumulators.
//
// Grid: ngroups x ncta CTAs (one group per independent sweep), NT threads,
// one CTA per SM, launched cooperatively so all CTAs are co-resident.
#include <algorithm>

#include "lrk_device.cuh"
#include "lrk_kernels.h"
#include "lrk_small.cuh"

namespace lrk {

namespace {
constexpr int NINT = NMAX + PMAX + 8;
__device__ __forceinline__ int lane_of(int t) { return t & 31; }

// a warp group: GW warps starting at warp WOFF
template <int GW_, int WOFF_>
struct Grp {
  static constexpr int GW = GW_, WOFF = WOFF_;
};

struct Small {  // offsets inside the small region, sized by (cap, pc)
  int C, Part, Yn, R, Rp, X, G, I, Qs, Rb, Tau, TauT, Cn, Sig, S, Red, Tmp, Scr, Uc, Vc, Core, Int,
      total;
  __host__ __device__ Small(int cap, int pc) {
    int o = 0;
    C = o; o += cap * pc;
    Part = o; o += (cap + pc + 1) * pc + 8;  // pipelined partials: [U, Q~] rows
    Yn = o; o += pc;
    R = o; o += pc * pc;
    Rp = o; o += pc * pc;
    X = o; o += pc * pc;
    G = o; o += pc * pc;
    I = o; o += pc * pc;
    Qs = o; o += pc * pc;
    Rb = o; o += pc * pc;
    Tau = o; o += pc;
    TauT = o; o += pc;
    Cn = o; o += pc;
    Sig = o; o += NMAX;
    S = o; o += NMAX;
    Red = o; o += NWARP * PMAX;
    Tmp = o; o += PMAX;
    Scr = o; o += NT;
    Uc = o; o += 32 * 32;
    Vc = o; o += 32 * 32;
    Core = o; o += 32 * 33;
    Int = o; o += (NINT + 1) / 2;
    total = o;
  }
};

// Rows i in [0, m) of X = [A (na cols), B (nb cols)] times W (n x rn, ld ldw),
// written in place into A's first rn columns (accumulators in registers;
// every read of a row happens before its write).  rn <= RA.
template <int RA>
__device__ __forceinline__ void update_rows(double* __restrict__ A, int64_t lda, int na, const double* __restrict__ B,
                            int64_t ldb, int nb, const double* __restrict__ W, int ldw, int rn, int m) {
  const int n = na + nb;
  for (int i = threadIdx.x; i < m; i += NT) {
    double acc[RA];
#pragma unroll
    for (int c = 0; c < RA; ++c) acc[c] = 0.0;
    for (int k = 0; k < n; ++k) {
      const double x = (k < na) ? A[i + (int64_t)k * lda] : B[i + (int64_t)(k - na) * ldb];
      const double* w = W + k;
#pragma unroll
      for (int c = 0; c < RA; ++c)
        if (c < rn) acc[c] += x * w[c * ldw];
    }
#pragma unroll
    for (int c = 0; c < RA; ++c)
      if (c < rn) A[i + (int64_t)c * lda] = acc[c];
  }
}

// Time rows: V'[t] = V[t, :r] W[:r, :rn] + [t visited at slot s] W[r+s, :rn]
// (V points at this CTA's first time row t0; local row index tl = t - t0.)
// One thread per output (t, c): the CTA's few time rows x rn columns run in
// parallel (a thread per row would chain rn x r dependent loads); results are
// staged in registers and written after a CTA barrier (the update is in place).
template <int RA>
__device__ __forceinline__ void update_time_rows(double* __restrict__ V, int64_t ldv, int r, const double* __restrict__ W,
                                 int ldw, int rn, int64_t t0, int64_t t1, int adjoint, int n_t,
                                 int start, int pc) {
  (void)RA;
  const int nrow = (int)(t1 - t0);
  if (rn <= 0) return;
  constexpr int PER = 2;  // outputs per thread per chunk
  const int rc = (PER * NT) / rn > 0 ? (PER * NT) / rn : 1;  // whole rows per chunk
  for (int rb = 0; rb < nrow; rb += rc) {  // uniform trip count (CTA barriers inside)
    const int nr = nrow - rb < rc ? nrow - rb : rc;
    const int total = nr * rn;
    double res[PER];
#pragma unroll
    for (int q = 0; q < PER; ++q) {
      const int o = threadIdx.x + q * NT;
      res[q] = 0.0;
      if (o < total) {
        const int tl = rb + o / rn, c = o % rn;
        const int64_t t = t0 + tl;
        const int sel = adjoint ? (n_t - 1 - start) - (int)t : (int)t - start;
        double acc = (sel >= 0 && sel < pc) ? W[(r + sel) + c * ldw] : 0.0;
        for (int k = 0; k < r; ++k) acc += V[tl + (int64_t)k * ldv] * W[k + c * ldw];
        res[q] = acc;
      }
    }
    __syncthreads();  // every read of these rows precedes the in-place writes
#pragma unroll
    for (int q = 0; q < PER; ++q) {
      const int o = threadIdx.x + q * NT;
      if (o < total) V[(rb + o / rn) + (int64_t)(o % rn) * ldv] = res[q];
    }
  }
}
}  // namespace

void sweep_plan(SweepArgs& a, int64_t n_x, int ncta, int ucap, int p, size_t smem_limit,
                int nshard) {
  const int nall = ncta * (nshard > 1 ? nshard : 1);  // CTAs of the logical sweep
  const int64_t mloc = (n_x + nall - 1) / nall;
  const int mp = (int)(mloc | 1);
  Small sm(ucap, p);
  const int stack = 2 * nall * p * p;
  const int64_t limit = (int64_t)(smem_limit / sizeof(double)) - 64;
  int scr = 0;
  int stack_smem = 0;
  if (sm.total + stack <= limit) { scr = stack; stack_smem = 1; }
  const int tp = (int)(((int64_t)a.n_t + ncta - 1) / ncta) | 1;
  const int64_t resident_rows = (int64_t)mp * (ucap + 2 * p + 3) + (int64_t)tp * ucap;
  // resident mode keeps the stacked-R QR in shared memory too
  const bool resident = stack_smem && sm.total + scr + resident_rows <= limit;
  int o = 0;
  a.resident = resident ? 1 : 0;
  a.mp = resident ? mp : 0;
  a.tp = resident ? tp : 0;
  if (resident) {
    a.off_V = o; o += tp * ucap;
    a.off_U = o; o += mp * ucap;
    a.off_Y = o; o += mp * p;
    a.off_Q = o; o += mp * p;
    a.off_yp = o; o += mp;
    a.off_th = o; o += mp;
    a.off_rs = o; o += mp;
  } else {
    a.off_U = a.off_Y = a.off_Q = a.off_yp = a.off_th = a.off_rs = 0;
  }
  a.off_small = o; o += sm.total;
  a.off_scr = o; o += scr;
  a.stack_smem = stack_smem;
  a.smem_doubles = o;
}

size_t sweep_smem_bytes() { return 227 * 1024; }
int64_t sweep_scratch_stride(int ncta) {
  return 2 * (int64_t)ncta * PMAX * PMAX + 4 * (int64_t)NMAX * NMAX;
}
int64_t sweep_part_stride() { return NMAX * PMAX + PMAX + 8; }

template <int Q, bool RES>
__global__ void __launch_bounds__(NT, 1) sweep_kernel(const __grid_constant__ SweepBatch batch) {
  extern __shared__ double sm[];
  const int ncta = batch.g[0].ncta;
  const SweepArgs& a = batch.g[blockIdx.x / ncta];
  const int cta = blockIdx.x % ncta;
  const int tid = threadIdx.x, warp = tid >> 5;
  // sharding: this CTA's place in the logical sweep (SweepArgs::nshard)
  const int nsh = a.nshard > 1 ? a.nshard : 1;
  const int gcta = (nsh > 1 ? a.shard : 0) * ncta + cta;
  const int ncta_all = nsh * ncta;
  const PartTab tab{a.spart, ncta, nsh, a.pstride};
  const bool sysf = a.sys_fence != 0;

  const int64_t n_x = a.n_x;
  const int n_t = a.n_t;
  const int p = a.p;
  const int cap = a.ucap;
  const int rb = a.rb_dev ? min(a.rb, *a.rb_dev) : a.rb;
  int64_t r0, r1, t0, t1;
  row_range(n_x, gcta, ncta_all, r0, r1);
  row_range(n_t, cta, ncta, t0, t1);  // the time factor is replicated per shard
  const int m_loc = (int)(r1 - r0);

  // ---- storage: resident shared-memory blocks or global rows.  RES is a
  // template parameter so every pointer has a single, provable address space
  // (the compiler emits LDS/STS for the resident blocks, not generic LD/ST).
  constexpr bool res = RES;
  double* Ul;
  double* Yl;
  double* Ql;
  double* Vl;
  double* yp;
  const double* th;
  const double* rsc;
  int64_t ldu, ldy, ldq, ldvl;
  if constexpr (RES) {
    Ul = sm + a.off_U; Yl = sm + a.off_Y; Ql = sm + a.off_Q; Vl = sm + a.off_V;
    yp = sm + a.off_yp; th = sm + a.off_th; rsc = sm + a.off_rs;
    ldu = ldy = ldq = a.mp;
    ldvl = a.tp;
    for (int i = tid; i < m_loc; i += NT) {
      sm[a.off_yp + i] = 0.0;
      sm[a.off_th + i] = a.theta ? a.theta[r0 + i] : 0.0;
      sm[a.off_rs + i] = a.rowscale ? a.rowscale[r0 + i] : 1.0;
    }
  } else {
    Ul = a.U0 + r0; Yl = a.ybuf + r0; Ql = a.qbuf + r0; Vl = a.V0 + t0;
    yp = a.yprev + r0; th = a.theta + r0; rsc = a.rowscale ? a.rowscale + r0 : nullptr;
    ldu = a.ldu; ldy = a.ldy; ldq = a.ldq; ldvl = a.ldv;
    for (int i = tid; i < m_loc; i += NT) yp[i] = 0.0;
  }

  Small L(cap, p);
  double* small = sm + a.off_small;
  double* sC = small + L.C;
  double* sPart = small + L.Part;
  double* sYn = small + L.Yn;
  double* sR = small + L.R;
  double* sRp = small + L.Rp;
  double* sX = small + L.X;
  double* sG = small + L.G;
  double* sI = small + L.I;
  double* sQs = small + L.Qs;
  double* sRb = small + L.Rb;
  double* sTau = small + L.Tau;
  double* sTauT = small + L.TauT;
  double* sCn = small + L.Cn;
  double* sSig = small + L.Sig;
  double* sS = small + L.S;
  double* sRed = small + L.Red;
  double* sTmp = small + L.Tmp;
  double* sScr = small + L.Scr;
  double* sCore = small + L.Core;
  int* iPerm = reinterpret_cast<int*>(small + L.Int);
  int* iPiv = iPerm + NMAX;
  int* iFlag = iPiv + PMAX;

  double* gscr = a.scratch + (int64_t)cta * a.scratch_stride;  // global per-CTA scratch
  // this CTA's own partial slots (regions 0..2 of its shard's buffer)
  double* part1 = a.spart[nsh > 1 ? a.shard : 0] + (int64_t)cta * a.pstride;
  double* part2 = part1 + (int64_t)ncta * a.pstride;
  double* part3 = part2 + (int64_t)ncta * a.pstride;
  __syncthreads();

  const bool timing = a.dbg != nullptr && cta == 0 && tid == 0;
  long long tacc[20] = {};
  long long tprev = timing ? clock64() : 0;
#define LRK_TSTAMP(k)               \
  if (timing) {                     \
    const long long t_ = clock64(); \
    tacc[k] += t_ - tprev;          \
    tprev = t_;                     \
  }

  // U^T Y projections of the CGS passes: DMMA with per-warp partials in the
  // (then idle) stack scratch; scalar fallback for very wide panes
  double* const wbuf = a.stack_smem ? sm + a.off_scr : gscr;
  const int wcap = a.stack_smem ? 2 * ncta_all * p * p : (int)a.scratch_stride;
  auto proj = [&](int rr, int pcc, double* outp) {
    if (rr <= 32 && NWARP * rr * pcc <= wcap)
      cta_tn_dmma<4>(Ul, ldu, rr, Yl, ldy, pcc, m_loc, outp, wbuf);
    else if (rr <= 64 && NWARP * rr * pcc <= wcap)
      cta_tn_dmma<8>(Ul, ldu, rr, Yl, ldy, pcc, m_loc, outp, wbuf);
    else
      cta_tn(Ul, ldu, rr, Yl, ldy, pcc, m_loc, outp, sScr);
  };
  int r = a.r_init >= 0 ? a.r_init : a.info[0];  // < 0: rank left by the previous chunk
  int jac_sweeps = 0;
  const int nflush = (n_t + p - 1) / p;
  if (r > 0) {  // resume a chunked sweep: the pane comes back from global memory
    for (int k = tid; k < r; k += NT) sSig[k] = a.sigma[k];
    if constexpr (RES)
      for (int c = 0; c < r; ++c) {
        for (int i = tid; i < m_loc; i += NT) Ul[i + (int64_t)c * ldu] = a.U0[r0 + i + (int64_t)c * a.ldu];
        for (int64_t t = t0 + tid; t < t1; t += NT)
          Vl[(t - t0) + (int64_t)c * ldvl] = a.V0[t + (int64_t)c * a.ldv];
      }
    __syncthreads();
  }
  // Phase 1 of a flush (buffered columns + projections + norms -> partial
  // slot 1).  Executed by the whole CTA, or — pipelined — by warps 4..7 for
  // the NEXT flush while warps 0..3 run the core Jacobi: the projection is
  // then taken against [U, Q~] of the current flush (rows nU + nQ), and the
  // next flush maps it to the updated pane with the core's vectors.
  auto phase1 = [&](auto grp, int fi, int nU, int nQ) {
    constexpr int GW = decltype(grp)::GW, WOFF = decltype(grp)::WOFF;
    const int gt = tid - 32 * WOFF;
    const int st = fi * p;
    const int pcn = (n_t - st) < p ? (n_t - st) : p;
    // squared column norms accumulated by the batched generation (global rows;
    // same rows per thread in the same order as the separate pass below)
    double vgen[Q];
#pragma unroll
    for (int s = 0; s < Q; ++s) vgen[s] = 0.0;
    bool have_vgen = false;
    if (a.yext) {
      const double* ye = a.yext + r0 + (int64_t)(st - a.flush0 * p) * a.ldyext;
      for (int i = gt; i < m_loc; i += 32 * GW) {
#pragma unroll
        for (int s = 0; s < Q; ++s)
          if (s < pcn) Yl[i + (int64_t)s * ldy] = ye[i + (int64_t)s * a.ldyext];
      }
    } else {
      int ks[Q];
#pragma unroll
      for (int s = 0; s < Q; ++s) ks[s] = a.adjoint ? (n_t - 1 - (st + s)) : (st + s);
      if constexpr (!RES && Q <= 8) {
        // rows from HBM: GR rows per thread with all their loads issued
        // before the recurrence (same per-row arithmetic and order)
        constexpr int GR = 4;
        const int gs = 32 * GW;
        for (int i0 = gt; i0 < m_loc; i0 += GR * gs) {
          double acc[GR][Q], tv[GR], rs[GR], y[GR];
#pragma unroll
          for (int h = 0; h < GR; ++h) {
            const int i = i0 + h * gs;
            const bool ok = i < m_loc;
            tv[h] = ok ? th[i] : 0.0;
            rs[h] = ok ? (rsc ? rsc[i] : 1.0) : 0.0;
            y[h] = ok ? yp[i] : 0.0;
#pragma unroll
            for (int s = 0; s < Q; ++s) acc[h][s] = 0.0;
          }
          for (int j0 = 0; j0 < rb; j0 += 4) {
            double bv[GR][4];
#pragma unroll
            for (int h = 0; h < GR; ++h)
#pragma unroll
              for (int u = 0; u < 4; ++u) {
                const int i = i0 + h * gs;
                bv[h][u] = (i < m_loc && j0 + u < rb) ? a.B[r0 + i + (int64_t)(j0 + u) * a.ldb] : 0.0;
              }
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              if (j0 + u >= rb) break;
              const double* w2 = a.W2 + (int64_t)(j0 + u) * a.ldw2;
#pragma unroll
              for (int s = 0; s < Q; ++s)
                if (s < pcn) {
                  const double wv = w2[ks[s]];
#pragma unroll
                  for (int h = 0; h < GR; ++h) acc[h][s] += bv[h][u] * wv;
                }
            }
          }
#pragma unroll
          for (int h = 0; h < GR; ++h) {
            const int i = i0 + h * gs;
            if (i < m_loc) {
              double yy = y[h];
#pragma unroll
              for (int s = 0; s < Q; ++s) {
                if (s < pcn) {
                  yy = tv[h] * yy + rs[h] * acc[h][s];
                  if (fabs(yy) < a.ftz) yy = 0.0;
                  Yl[i + (int64_t)s * ldy] = yy;
                  vgen[s] += yy * yy;
                }
              }
              yp[i] = yy;
            }
          }
        }
        have_vgen = true;
      } else {
      for (int i = gt; i < m_loc; i += 32 * GW) {
        double acc[Q];
#pragma unroll
        for (int s = 0; s < Q; ++s) acc[s] = 0.0;
#pragma unroll 4
        for (int j = 0; j < rb; ++j) {
          const double b = a.B[r0 + i + (int64_t)j * a.ldb];
          const double* w2 = a.W2 + (int64_t)j * a.ldw2;
#pragma unroll
          for (int s = 0; s < Q; ++s)
            if (s < pcn) acc[s] += b * w2[ks[s]];
        }
        const double tv = th[i];
        const double rs = rsc ? rsc[i] : 1.0;
        double y = yp[i];
#pragma unroll
        for (int s = 0; s < Q; ++s) {
          if (s < pcn) {
            y = tv * y + rs * acc[s];
            if (fabs(y) < a.ftz) y = 0.0;
            Yl[i + (int64_t)s * ldy] = y;
          }
        }
        yp[i] = y;
      }
      }
    }
    grp_sync<GW, WOFF>();
    // projections straight into this CTA's partial slot (rows nU of U, then
    // nQ of Q~), squared norms after them
    if (nU > 0) {
      if (nU <= 32 && GW * nU * pcn <= wcap)
        cta_tn_dmma<4, GW, WOFF>(Ul, ldu, nU, Yl, ldy, pcn, m_loc, part1, wbuf);
      else if (nU <= 64 && GW * nU * pcn <= wcap)
        cta_tn_dmma<8, GW, WOFF>(Ul, ldu, nU, Yl, ldy, pcn, m_loc, part1, wbuf);
      else if constexpr (GW == NWARP)
        cta_tn(Ul, ldu, nU, Yl, ldy, pcn, m_loc, part1, sScr);
    }
    if (nQ > 0) cta_tn_dmma<2, GW, WOFF>(Ql, ldq, nQ, Yl, ldy, pcn, m_loc, part1 + nU * pcn, wbuf);
    {
      double v[Q];
#pragma unroll
      for (int s = 0; s < Q; ++s) v[s] = vgen[s];
      if (!have_vgen)
        for (int i = gt; i < m_loc; i += 32 * GW) {
#pragma unroll
          for (int s = 0; s < Q; ++s)
            if (s < pcn) { const double y = Yl[i + (int64_t)s * ldy]; v[s] += y * y; }
        }
#pragma unroll
      for (int s = 0; s < Q; ++s) v[s] = warp_sum(v[s]);
      double* red = sRed;  // GW * Q <= NWARP * PMAX doubles (unused by the Jacobi warps)
      if ((tid & 31) == 0) {
#pragma unroll
        for (int s = 0; s < Q; ++s) red[(tid / 32 - WOFF) * Q + s] = v[s];
      }
      grp_sync<GW, WOFF>();
      if (gt < pcn) {
        double sum = 0.0;
#pragma unroll
        for (int w = 0; w < GW; ++w) sum += red[w * Q + gt];
        part1[(nU + nQ) * pcn + gt] = sum;
      }
      grp_sync<GW, WOFF>();
    }
  };
  // pipelining state: the next flush's phase 1 was done during the Jacobi
  bool have_next = false;
  int rP = 0, ldcP = 0;  // rows of its basis [U, Q~]; leading dim of the core vectors
  for (int f = a.flush0; f < a.flush1; ++f) {
    const int start = f * p;
    const int pc = (n_t - start) < p ? (n_t - start) : p;
    int rows_in = r;
    if (!have_next) {
      // ---------------- phase 1 (whole CTA) + barrier 1
      phase1(Grp<NWARP, 0>{}, f, r, 0);
      LRK_TSTAMP(0);
      group_barrier(a.gbar, ncta_all, sysf);
    } else {
      rows_in = rP;
      LRK_TSTAMP(0);
      if (tid == 0) group_wait(a.gbar, (unsigned)iFlag[3], sysf);
      __syncthreads();
    }
    LRK_TSTAMP(1);
    // ---------------- phase 2: block CGS2 against the orthonormal pane
    reduce_partials(tab, 0, ncta_all, rows_in * pc + pc, sPart);
    for (int i = tid; i < pc; i += NT) sYn[i] = sPart[rows_in * pc + i];
    if (!have_next) {
      for (int i = tid; i < r * pc; i += NT) sC[i] = sPart[i];
    } else {
      // C = W^T P: the projection onto [U_prev, Q~_prev] mapped to the pane
      // U = [U_prev, Q~_prev] W (W = the previous core's first r vectors)
      // (four lanes per entry, each summing every fourth k, then xor shuffles)
      const double* Wp = small + L.Uc;
      for (int base = 0; base < r * pc * 4; base += NT) {
        const int idx = base + tid, o = idx >> 2, sub = idx & 3;
        double acc = 0.0;
        if (o < r * pc) {
          const int i = o / pc, sI = o - i * pc;
          for (int k = sub; k < rP; k += 4) acc += Wp[k + i * ldcP] * sPart[k * pc + sI];
        }
        acc += __shfl_xor_sync(0xffffffffu, acc, 1);
        acc += __shfl_xor_sync(0xffffffffu, acc, 2);
        if (o < r * pc && sub == 0) sC[o] = acc;
      }
    }
    have_next = false;
    __syncthreads();
    LRK_TSTAMP(9);
    if (r > 0) {
      // first CGS pass: Y -= U C and the projection U^T Y in one pass over U
      // when the rows stream from HBM (C4: 1.36 -> 1.21 s per apply); with
      // resident rows the two shared-memory passes are faster (the fused
      // pass's shuffles cost more than the second read: 6k vs 10.7k cycles)
      if (!RES && Q <= 4 && r <= 32 && NWARP * r * pc <= wcap) {
        cta_subtn_dmma<4>(Ul, ldu, r, Yl, ldy, pc, sC, m_loc, sPart, wbuf);
      } else if (!RES && Q <= 4 && r <= 64 && NWARP * r * pc <= wcap) {
        cta_subtn_dmma<8>(Ul, ldu, r, Yl, ldy, pc, sC, m_loc, sPart, wbuf);
      } else {
        rows_sub_t<Q, RES ? 2 : 4>(Yl, ldy, pc, Ul, ldu, r, sC, m_loc);
        __syncthreads();
        proj(r, pc, sPart);
      }
      for (int i = tid; i < r * pc; i += NT) part2[i] = sPart[i];
      LRK_TSTAMP(10);
      group_barrier(a.gbar, ncta_all, sysf);
      LRK_TSTAMP(11);
      reduce_partials(tab, 1, ncta_all, r * pc, sPart);
      rows_sub_t<Q, RES ? 2 : 4>(Yl, ldy, pc, Ul, ldu, r, sPart, m_loc);
      for (int i = tid; i < r * pc; i += NT) sC[i] += sPart[i];
      __syncthreads();
    }
    LRK_TSTAMP(2);
    // ---------------- phase 3: local Householder QR of the remainder
    block_qr_t<Q, (!RES && Q <= 4) ? 4 : 1>(Yl, ldy, m_loc, pc, sTau, sR, sRed, sTmp);
    for (int i = tid; i < pc * pc; i += NT) part3[i] = sR[i];
    LRK_TSTAMP(3);
    group_barrier(a.gbar, ncta_all, sysf);
    LRK_TSTAMP(4);
    // ---------------- phase 4 (every CTA, redundantly): finish the TSQR
    const int ms = ncta_all * pc;
    double* stack;
    if constexpr (RES) stack = sm + a.off_scr;
    else stack = a.stack_smem ? sm + a.off_scr : gscr;
    double* stackY = stack + ms * pc;
    // register two-level TSQR when the stacked blocks fit 3 rows per lane
    const bool fast_stack = (Q <= 4) && ((ncta_all + NWARP - 1) / NWARP) * pc <= 96;
    int tail_tid = 0;
    if (fast_stack) {
      if constexpr (Q <= 4) {
        const int wo = warp_stack_tsqr<Q, 3>(tab, ncta_all, pc, gcta, sCore, sRp, sQs);
        tail_tid = wo * 32;
      }
      LRK_TSTAMP(13);
    } else {
      // all loads of the stacked R's are issued before any store
      constexpr int BATCH = 16;
      const int pp = pc * pc, tot = ms * pc;
      for (int base = 0; base < tot; base += BATCH * NT) {
        double v[BATCH];
#pragma unroll
        for (int u = 0; u < BATCH; ++u) {
          const int idx = base + u * NT + tid;
          v[u] = (idx < tot) ? __ldcg(tab.at(2, idx / pp) + idx % pp) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < BATCH; ++u) {
          const int idx = base + u * NT + tid;
          if (idx < tot) {
            const int owner = idx / pp, e = idx % pp;  // e = lr * pc + c
            stack[(owner * pc + e / pc) + (e % pc) * ms] = v[u];
          }
        }
      }
      for (int i = tid; i < pc * pc; i += NT) sI[i] = (i / pc == i % pc) ? 1.0 : 0.0;
      __syncthreads();
      LRK_TSTAMP(13);
      block_qr_t<Q>(stack, ms, ms, pc, sTauT, sRp, sRed, sTmp);
      LRK_TSTAMP(14);
      block_apply_q_t<Q>(stack, ms, ms, pc, sTauT, sI, stackY, ms, sRed, sTmp);
      for (int i = tid; i < pc * pc; i += NT) sQs[i] = stackY[(gcta * pc + i / pc) + (i % pc) * ms];
      __syncthreads();
      LRK_TSTAMP(15);
    }
    if constexpr (Q <= 4) {
      // rank-revealing fix-up Rp P = X Rt by the warp that owns this CTA's
      // rows of the stacked Q (shuffle form of the one-thread path below)
      if ((tid >> 5) == (tail_tid >> 5)) warp_pivqr_fixup<Q>(sRp, sQs, sG, sYn, pc);
    } else if (tid == tail_tid) {
      // rows of the stacked Q that belong to this CTA; rank-revealing fix-up
      // Rp P = X Rt (column pivoting); drop rows at the block's rounding floor
      double ysq = 0.0;
      for (int s = 0; s < pc; ++s) ysq += sYn[s];
      const double delta = 16.0 * DEPS * sqrt(ysq);
      if constexpr (Q <= 8) {
        double A[Q][Q], X[Q][Q], Qr[Q][Q];
        int pv[Q];
#pragma unroll
        for (int i = 0; i < Q; ++i)
#pragma unroll
          for (int k = 0; k < Q; ++k) {
            A[i][k] = (i < pc && k < pc) ? sRp[i * pc + k] : 0.0;
            Qr[i][k] = (i < pc && k < pc) ? sQs[i * pc + k] : 0.0;
          }
        pivoted_qr_reg<Q>(A, pc, X, pv);
#pragma unroll
        for (int j = 0; j < Q; ++j)
          if (fabs(A[j][j]) <= delta) {
#pragma unroll
            for (int k = 0; k < Q; ++k) { A[j][k] = 0.0; X[k][j] = 0.0; }
          }
#pragma unroll
        for (int j = 0; j < Q; ++j)
#pragma unroll
          for (int kk = 0; kk < Q; ++kk)
            if (j < pc && kk < pc) sRp[j * pc + pv[kk]] = A[j][kk];
#pragma unroll
        for (int i = 0; i < Q; ++i)
#pragma unroll
          for (int j = 0; j < Q; ++j) {
            double acc = 0.0;
#pragma unroll
            for (int k = 0; k < Q; ++k) acc += Qr[i][k] * X[k][j];
            if (i < pc && j < pc) sG[i * pc + j] = acc;
          }
      } else {
        for (int i = 0; i < pc * pc; ++i) sRb[i] = sRp[i];
        small_pivoted_qr(sRb, pc, sX, iPiv, sCn);
        for (int j = 0; j < pc; ++j)
          if (fabs(sRb[j * pc + j]) <= delta)
            for (int k = 0; k < pc; ++k) { sRb[j * pc + k] = 0.0; sX[k * pc + j] = 0.0; }
        for (int j = 0; j < pc; ++j)
          for (int kk = 0; kk < pc; ++kk) sRp[j * pc + iPiv[kk]] = sRb[j * pc + kk];
        for (int i = 0; i < pc; ++i)
          for (int j = 0; j < pc; ++j) {
            double acc = 0.0;
            for (int k = 0; k < pc; ++k) acc += sQs[i * pc + k] * sX[k * pc + j];
            sG[i * pc + j] = acc;
          }
      }
    }
    __syncthreads();
    LRK_TSTAMP(5);
    // explicit Q~ rows of this CTA: Q_loc * G
    if constexpr (Q <= 4) block_apply_q_wy<Q>(Yl, ldy, m_loc, pc, sTau, sG, Ql, ldq, sRed, sTmp, sCore);
    else block_apply_q_t<Q>(Yl, ldy, m_loc, pc, sTau, sG, Ql, ldq, sRed, sTmp);
    LRK_TSTAMP(6);
    // ---------------- core SVD: [[diag(sig), C], [0, Rblock]]
    const int n = r + pc;
    if (n > NMAX) {  // uniform across the group; report and stop
      if (tid == 0 && cta == 0) a.info[2] = 1;
      return;
    }
    double* const Ucs = small + L.Uc;  // compact singular vectors (shared, n <= 32)
    double* const Vcs = small + L.Vc;
    double* Ucg = nullptr;             // (global, wide cores)
    double* Vcg = nullptr;
    const int ldc = n;
    if (n <= 32) {
      double* Uc = Ucs;
      double* Vc = Vcs;
      for (int idx = tid; idx < n * n; idx += NT) {
        const int i = idx % n, j = idx / n;
        double v = 0.0;
        if (i < r) v = (j < r) ? (i == j ? sSig[i] : 0.0) : sC[i * pc + (j - r)];
        else if (j >= r) v = sRp[(i - r) * pc + (j - r)];
        sCore[j + i * 33] = v;  // K^T: Jacobi on the rows of the core
      }
      __syncthreads();
      if (a.cdump && cta == 0) {  // diagnostics: the cores the Jacobi sees
        double* d = a.cdump + (int64_t)f * (1 + 32 * 33);
        if (tid == 0) d[0] = n;
        for (int idx = tid; idx < 32 * 33; idx += NT) d[1 + idx] = sCore[idx];
        __syncthreads();
      }
      // the next flush's phase 1 overlaps the Jacobi when the rows are
      // resident (with global rows, C4-sized, the 4-warp row pass is longer
      // than the Jacobi: 305 -> 377 ms per apply measured) and its
      // projection fits the tensor-core path of the 4-warp group
      const bool pipe = RES && !a.nopipe && (f + 1 < a.flush1) && (n <= 32) && (pc <= 4) &&
                        (NWARP / 2) * n * p <= wcap;
      if (warp < 4) {  // 4-warp register Jacobi (named barrier 1), sScr = gbuf
        // K^T = Vk S Uk^T: the routine's left vectors are K's right ones
        // NJ (rows per warp NJ/4) tracks n closely: the padding rows cost the
        // same instructions as live ones in every rotation round
        if (n <= 8) jac_sweeps += multi_warp_jacobi<8, 4>(sCore, 33, n, Vc, Uc, ldc, sS, iPerm, sScr);
        else if (n <= 12) jac_sweeps += multi_warp_jacobi<12, 4>(sCore, 33, n, Vc, Uc, ldc, sS, iPerm, sScr);
        else if (n <= 16) jac_sweeps += multi_warp_jacobi<16, 4>(sCore, 33, n, Vc, Uc, ldc, sS, iPerm, sScr);
        else if (n <= 20) jac_sweeps += multi_warp_jacobi<20, 4>(sCore, 33, n, Vc, Uc, ldc, sS, iPerm, sScr);
        else if (n <= 24) jac_sweeps += multi_warp_jacobi<24, 4>(sCore, 33, n, Vc, Uc, ldc, sS, iPerm, sScr);
        else jac_sweeps += multi_warp_jacobi<32, 4>(sCore, 33, n, Vc, Uc, ldc, sS, iPerm, sScr);
      } else if (pipe) {
        phase1(Grp<NWARP / 2, NWARP / 2>{}, f + 1, r, pc);
        if (tid == 32 * (NWARP / 2)) iFlag[3] = (int)group_arrive(a.gbar, ncta_all, sysf);
      }
      __syncthreads();
      if (pipe) { have_next = true; rP = n; ldcP = ldc; }
    } else {
      double* Aj = gscr + 2 * (int64_t)ncta_all * PMAX * PMAX;
      double* Vj = Aj + (int64_t)NMAX * NMAX;
      for (int idx = tid; idx < n * n; idx += NT) {
        const int i = idx % n, j = idx / n;
        double v = 0.0;
        if (i < r) v = (j < r) ? (i == j ? sSig[i] : 0.0) : sC[i * pc + (j - r)];
        else if (j >= r) v = sRp[(i - r) * pc + (j - r)];
        Aj[i + j * n] = v;
      }
      __syncthreads();
      jac_sweeps += jacobi_svd(Aj, n, Vj, n, n, sS, iPerm, sScr, iFlag, sTmp);
      Ucg = Vj + (int64_t)n * n;
      Vcg = Ucg + (int64_t)n * n;
      for (int idx = tid; idx < n * n; idx += NT) {
        const int i = idx % n, k = idx / n;
        const double sv = sS[k];
        Ucg[i + k * ldc] = sv > 0.0 ? Aj[i + iPerm[k] * n] / sv : 0.0;
        Vcg[i + k * ldc] = Vj[i + iPerm[k] * n];
      }
      __syncthreads();
    }
    LRK_TSTAMP(7);
    if (n <= 32 && r <= 32 && warp == 0) {
      // zero test and _rank_cut (lowrank.py:98-144) on one warp
      const double ysq = warp_sum(lane_of(tid) < pc ? sYn[lane_of(tid)] : 0.0);
      const double sg = lane_of(tid) < r ? sSig[lane_of(tid)] : 0.0;
      const double ssq = warp_sum(sg * sg);
      const double fs = sqrt((double)r + ysq) * sqrt(ssq + (double)pc);
      int rn = rank_cut_warp(sS, n, a.eps0, a.r_max);
      if (sS[0] <= NOISE_FLOOR * fs) rn = 0;
      if (rn > cap) { rn = cap; if (cta == 0 && tid == 0) a.info[2] = 2; }
      if (tid == 0) iFlag[1] = rn;
    } else if (!(n <= 32 && r <= 32) && tid == 0) {
      double ysq = 0.0, ssq = 0.0;
      for (int s = 0; s < pc; ++s) ysq += sYn[s];
      for (int i = 0; i < r; ++i) ssq += sSig[i] * sSig[i];
      const double fs = sqrt((double)r + ysq) * sqrt(ssq + (double)pc);
      int rn;
      if (sS[0] <= NOISE_FLOOR * fs) rn = 0;
      else rn = rank_cut_dev(sS, n, a.eps0, a.r_max);
      if (rn > cap) { rn = cap; if (cta == 0) a.info[2] = 2; }
      iFlag[1] = rn;
    }
    __syncthreads();
    const int rn = iFlag[1];
    LRK_TSTAMP(12);
    // ---------------- basis update in place: U' = [U, Q~] Uc[:, :rn]
    if (n <= 32 && rn <= 16) {
      update_rows_dmma<2, RES ? 2 : 4>(Ul, ldu, r, Ql, ldq, pc, Ucs, ldc, rn, m_loc);
      LRK_TSTAMP(16);
      update_time_rows<16>(Vl, ldvl, r, Vcs, ldc, rn, t0, t1, a.adjoint, n_t, start, pc);
      LRK_TSTAMP(17);
    } else if (n <= 32) {
      update_rows_dmma<4, RES ? 2 : 4>(Ul, ldu, r, Ql, ldq, pc, Ucs, ldc, rn, m_loc);
      update_time_rows<32>(Vl, ldvl, r, Vcs, ldc, rn, t0, t1, a.adjoint, n_t, start, pc);
    } else if (n <= 64) {
      // wide core (n <= 64): U rows in place on the DMMA pipe (one pass over
      // U; the former per-column loop re-read the row block rn times); the
      // time rows out of place through the global alternate, then copied back
      update_rows_dmma_wide<RES ? 1 : 2>(Ul, ldu, r, Ql, ldq, pc, Ucg, ldc, rn, m_loc);
      const double* Vc = Vcg;
      for (int c = 0; c < rn; ++c)
        for (int64_t t = t0 + tid; t < t1; t += NT) {
          int sel = a.adjoint ? (n_t - 1 - start) - (int)t : (int)t - start;
          double acc = (sel >= 0 && sel < pc) ? Vc[(r + sel) + c * ldc] : 0.0;
          for (int k = 0; k < r; ++k) acc += Vl[(t - t0) + (int64_t)k * ldvl] * Vc[k + c * ldc];
          a.V1[t + (int64_t)c * a.ldv] = acc;
        }
      __syncthreads();
      for (int c = 0; c < rn; ++c)
        for (int64_t t = t0 + tid; t < t1; t += NT) Vl[(t - t0) + (int64_t)c * ldvl] = a.V1[t + (int64_t)c * a.ldv];
    } else {
      // widest cores (n > 64, no rank cap): out of place through the global
      // alternates, then copy back
      const double* Uc = Ucg;
      const double* Vc = Vcg;
      for (int c = 0; c < rn; ++c) {
        for (int i = tid; i < m_loc; i += NT) {
          double acc = 0.0;
          for (int k = 0; k < n; ++k)
            acc += ((k < r) ? Ul[i + (int64_t)k * ldu] : Ql[i + (int64_t)(k - r) * ldq]) * Uc[k + c * ldc];
          a.U1[r0 + i + (int64_t)c * a.ldu] = acc;
        }
        for (int64_t t = t0 + tid; t < t1; t += NT) {
          int sel = a.adjoint ? (n_t - 1 - start) - (int)t : (int)t - start;
          double acc = (sel >= 0 && sel < pc) ? Vc[(r + sel) + c * ldc] : 0.0;
          for (int k = 0; k < r; ++k) acc += Vl[(t - t0) + (int64_t)k * ldvl] * Vc[k + c * ldc];
          a.V1[t + (int64_t)c * a.ldv] = acc;
        }
      }
      __syncthreads();
      for (int c = 0; c < rn; ++c) {
        for (int i = tid; i < m_loc; i += NT) Ul[i + (int64_t)c * ldu] = a.U1[r0 + i + (int64_t)c * a.ldu];
        for (int64_t t = t0 + tid; t < t1; t += NT) Vl[(t - t0) + (int64_t)c * ldvl] = a.V1[t + (int64_t)c * a.ldv];
      }
    }
    for (int k = tid; k < rn; k += NT) sSig[k] = sS[k];
    if (tid == 0 && cta == 0) a.trace[f] = rn;
    __syncthreads();
    r = rn;
    LRK_TSTAMP(8);
  }
  if (timing)
    for (int k = 0; k < 20; ++k) a.dbg[k] = tacc[k];
#undef LRK_TSTAMP
  // the pane: resident U rows go back to global slot 0
  if (res)
    for (int c = 0; c < r; ++c) {
      for (int i = tid; i < m_loc; i += NT) a.U0[r0 + i + (int64_t)c * a.ldu] = Ul[i + (int64_t)c * ldu];
      for (int64_t t = t0 + tid; t < t1; t += NT)
        a.V0[t + (int64_t)c * a.ldv] = Vl[(t - t0) + (int64_t)c * ldvl];
    }
  if (cta == 0) {
    for (int k = tid; k < r; k += NT) a.sigma[k] = sSig[k];
    if (tid == 0) {
      a.info[0] = r;
      a.info[1] = 0;
      a.info[3] = jac_sweeps;
      if (a.flush1 == nflush) a.trace[nflush] = r;
    }
  }
}

template <int Q, bool RES>
static cudaError_t launch_q(const SweepBatch& batch, cudaStream_t s) {
  // the opt-in shared-memory size is a per-device function attribute
  static int attr_bytes[64] = {};
  const int smem = batch.g[0].smem_doubles * (int)sizeof(double);
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64 || smem > attr_bytes[dev]) {
    cudaError_t e = cudaFuncSetAttribute(sweep_kernel<Q, RES>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    if (dev >= 0 && dev < 64) attr_bytes[dev] = smem;
  }
  void* params[] = {(void*)&batch};
  return cudaLaunchCooperativeKernel((const void*)sweep_kernel<Q, RES>,
                                     dim3(batch.ngroups * batch.g[0].ncta), dim3(NT), params,
                                     (size_t)smem, s);
}

template <bool RES>
static cudaError_t launch_r(const SweepBatch& batch, cudaStream_t s) {
  const int p = batch.g[0].p;
  if (p <= 1) return launch_q<1, RES>(batch, s);
  if (p <= 2) return launch_q<2, RES>(batch, s);
  if (p <= 4) return launch_q<4, RES>(batch, s);
  if (p <= 8) return launch_q<8, RES>(batch, s);
  return launch_q<16, RES>(batch, s);
}

cudaError_t launch_sweep(const SweepBatch& batch, cudaStream_t s) {
  return batch.g[0].resident ? launch_r<true>(batch, s) : launch_r<false>(batch, s);
}

}  // namespace lrk
