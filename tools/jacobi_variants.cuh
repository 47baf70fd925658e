// jacobi_variants.cuh — core-SVD variants measured against the sweep's
// 4-warp register Jacobi and not used by the library (kept for the
// microbenchmarks in this directory): the one-warp register Jacobi, the
// one-warp (pivoted) Householder QR and the QR-preconditioned Jacobi.
#pragma once
#include "lrk_small.cuh"

namespace lrk {

// One-sided Jacobi SVD of an n x n matrix (n <= NJ <= 32) by ONE warp with
// the columns in registers: lane j holds column j of A and of V (zero padded
// to NJ, which leaves the arithmetic unchanged).  The partner column of a
// round arrives by shuffles, so there is no shared-memory traffic and no CTA
// barrier.  Rotation test: cosine above the rounding floor of an n-term dot
// product; columns under 1e-16 ||M||_F are noise (see jacobi_svd).  Stops
// after a sweep whose largest cosine was <= 1e-8: the next sweep could only
// change the result at the 1e-16 level (quadratic convergence).
// Output (lanes < n): Uo[:, k] (ld ldo) k-th left singular vector, Vo[:, k]
// right singular vector, s_sorted[k] descending, perm[k] source column.
template <int NJ, bool KEEP = (NJ <= 24)>
__device__ __forceinline__ int warp_jacobi_reg(const double* __restrict__ Ain, int lda, int n,
                               double* __restrict__ Uo, double* __restrict__ Vo, int ldo,
                               double* __restrict__ s_sorted, int* __restrict__ perm) {
  const int lane = threadIdx.x & 31;
  const unsigned full = 0xffffffffu;
  const bool own = lane < n;
  double a[NJ], v[NJ];
#pragma unroll
  for (int i = 0; i < NJ; ++i) {
    a[i] = (own && i < n) ? Ain[i + lane * lda] : 0.0;
    v[i] = (i == lane) ? 1.0 : 0.0;
  }
  auto colnorm = [&]() {
    double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
#pragma unroll
    for (int i = 0; i < NJ; i += 4) {
      s0 += a[i] * a[i];
      if (i + 1 < NJ) s1 += a[i + 1] * a[i + 1];
      if (i + 2 < NJ) s2 += a[i + 2] * a[i + 2];
      if (i + 3 < NJ) s3 += a[i + 3] * a[i + 3];
    }
    return (s0 + s1) + (s2 + s3);
  };
  double nrm = colnorm();
  const double tiny = warp_sum(nrm) * 1e-32;
  const double tol = 2.0 * DEPS * (double)(n > 8 ? n : 8);
  const double tol2 = tol * tol;
  const int ne = n + (n & 1);
  const int m1 = ne - 1;
  int nsweep = 0;
  for (int sweep = 0; sweep < 40 && n > 1; ++sweep) {
    nrm = colnorm();
    double maxcos2 = 0.0;
    bool rotated = false;
    // partner of lane for round rnd: (2 rnd - lane) mod (ne-1), kept
    // incrementally; lane ne-1 meets rnd, lane rnd meets ne-1
    int pf = (lane < m1) ? (m1 - lane) % m1 : 0;
    for (int rnd = 0; rnd < m1; ++rnd) {
      int p = pf;
      if (lane == m1) p = rnd;
      else if (lane == rnd) p = m1;
      if (lane >= ne) p = lane;
      pf += 2;
      if (pf >= m1) pf -= m1;
      const bool act = own && p < n;
      const bool lo = lane < p;
      const double np = __shfl_sync(full, nrm, p & 31);
      double g0 = 0.0, g1 = 0.0, g2 = 0.0, g3 = 0.0;
      double ap[KEEP ? NJ : 1];
#pragma unroll
      for (int i = 0; i < NJ; ++i) {
        const double x = __shfl_sync(full, a[i], p & 31);
        if (KEEP) ap[KEEP ? i : 0] = x;
        if ((i & 3) == 0) g0 += a[i] * x;
        else if ((i & 3) == 1) g1 += a[i] * x;
        else if ((i & 3) == 2) g2 += a[i] * x;
        else g3 += a[i] * x;
      }
      // identical summation order on both lanes of a pair: products commute
      const double g = (g0 + g1) + (g2 + g3);
      const double al = lo ? nrm : np, be = lo ? np : nrm;
      double c = 1.0, s = 0.0, t = 0.0;
      bool rot = false;
      if (act && al > tiny && be > tiny) {
        const double g2 = g * g, ab = al * be;
        if (g2 > 1e-16 * ab) maxcos2 = 1.0;  // a cosine above 1e-8 this sweep
        if (g2 > tol2 * ab) {
          // tangent of the rotation angle: only its convergence effect depends
          // on its accuracy, so it is formed in fp32 after an exact power-of-two
          // rescale; c (and so c^2 + s^2 = 1) is then computed in fp64.
          const double d = be - al;
          const double m = fmax(fabs(d), fabs(g));
          const int e = ((int)(__double_as_longlong(m) >> 52) & 0x7ff) - 1023;
          const double sc = __longlong_as_double((long long)(1023 - e) << 52);
          const float df = (float)(d * sc), gf = (float)(g * sc);
          float tf;
          if (fabsf(gf) < 1e-4f * fabsf(df)) tf = __fdividef(gf, df);  // t ~ g/d
          else {
            tf = __fdividef(2.0f * gf, fabsf(df) + sqrtf(df * df + 4.0f * gf * gf));
            if (df < 0.0f) tf = -tf;
          }
          t = (double)tf;
          const double t2 = t * t;
          c = (t2 < 1e-8) ? 1.0 - t2 * (0.5 - 0.375 * t2) : rsqrt_u(1.0 + t2);
          s = c * t;
          rot = true;
        }
      }
      const bool any = __any_sync(full, rot);
      if (any) {
        const double sl = lo ? -s : s;  // lo: a' = c a - s ap ; hi: a' = c a + s ap
#pragma unroll
        for (int i = 0; i < NJ; ++i) {
          // both lanes of a pair shuffle index i before either updates it
          const double xp = KEEP ? ap[KEEP ? i : 0] : __shfl_sync(full, a[i], p & 31);
          a[i] = rot ? (c * a[i] + sl * xp) : a[i];
          const double vp = __shfl_sync(full, v[i], p & 31);
          v[i] = rot ? (c * v[i] + sl * vp) : v[i];
        }
        if (rot) nrm = lo ? (al - t * g) : (be + t * g);
        rotated = true;
      }
    }
    ++nsweep;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) maxcos2 = fmax(maxcos2, __shfl_xor_sync(full, maxcos2, o));
    if (!rotated || maxcos2 <= 1e-16) break;
  }
  double sv = own ? sqrt_fast(colnorm()) : 0.0;
  int rk = 0;
  for (int j = 0; j < n; ++j) {
    const double sj = __shfl_sync(full, sv, j);
    if (sj > sv || (sj == sv && j < lane)) ++rk;
  }
  if (own) {
    perm[rk] = lane;
    s_sorted[rk] = sv;
    const double inv = sv > 0.0 ? rcp_fast(sv) : 0.0;
#pragma unroll
    for (int i = 0; i < NJ; ++i)
      if (i < n) {
        Uo[i + rk * ldo] = a[i] * inv;
        Vo[i + rk * ldo] = v[i];
      }
  }
  __syncwarp();
  return nsweep;
}

// Householder QR (optionally with column pivoting) of an n x n matrix held by
// ONE warp in registers, lane j = column j (a[i] = entry i, zero padded to
// NJ).  On exit a[] holds column `lane` of R; the reflector of step j is
// stored in Vh[i + j*ldv] (i > j, unit leading entry implicit) with tau[j];
// colid returns the original column index of the lane (pivot permutation).
template <int NJ, bool PIVOT>
__device__ __forceinline__ void warp_qr_cols(double (&a)[NJ], int n, double* __restrict__ Vh,
                                             int ldv, double* __restrict__ tau, int& colid,
                                             bool writer = true) {
  const int lane = threadIdx.x & 31;
  const unsigned full = 0xffffffffu;
  colid = lane;
  for (int j = 0; j < n - 1; ++j) {
    if (PIVOT) {
      double tn = 0.0;
#pragma unroll
      for (int i = 0; i < NJ; ++i)
        if (i >= j) tn += a[i] * a[i];
      if (lane < j || lane >= n) tn = -1.0;
      int idx = lane;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const double ot = __shfl_xor_sync(full, tn, o);
        const int oi = __shfl_xor_sync(full, idx, o);
        if (ot > tn || (ot == tn && oi < idx)) { tn = ot; idx = oi; }
      }
      // swap columns j and idx (identity shuffle when idx == j; kept
      // unconditional so it compiles to plain SHFL)
      const int src = (lane == j) ? idx : ((lane == idx) ? j : lane);
#pragma unroll
      for (int i = 0; i < NJ; ++i) a[i] = __shfl_sync(full, a[i], src);
      colid = __shfl_sync(full, colid, src);
    }
    double x[NJ];
#pragma unroll
    for (int i = 0; i < NJ; ++i) x[i] = __shfl_sync(full, a[i], j);
    double sig = 0.0, alpha = 0.0;
#pragma unroll
    for (int i = 0; i < NJ; ++i) {
      if (i > j) sig += x[i] * x[i];
      if (i == j) alpha = x[i];
    }
    double beta = alpha, t = 0.0, scale = 0.0;
    if (sig != 0.0) {
      const double nrm = sqrt_fast(alpha * alpha + sig);
      beta = alpha >= 0.0 ? -nrm : nrm;
      t = (beta - alpha) * rcp_fast(beta);
      scale = rcp_fast(alpha - beta);
    }
    // v_i = x_i * scale (i > j), v_j = 1
    if (lane > j && lane < n) {
      double w = 0.0;
#pragma unroll
      for (int i = 0; i < NJ; ++i) {
        if (i == j) w += a[i];
        else if (i > j) w += x[i] * scale * a[i];
      }
      const double f = t * w;
#pragma unroll
      for (int i = 0; i < NJ; ++i) {
        if (i == j) a[i] -= f;
        else if (i > j) a[i] -= f * x[i] * scale;
      }
    } else if (lane == j) {
#pragma unroll
      for (int i = 0; i < NJ; ++i) {
        if (i > j) {
          if (writer) Vh[i + j * ldv] = x[i] * scale;
          a[i] = 0.0;
        }
        if (i == j) a[i] = beta;
      }
      if (writer) tau[j] = t;
    }
  }
  if (lane == 0 && writer) tau[n - 1] = 0.0;
  __syncwarp();
}

// Preconditioned one-sided Jacobi SVD of the n x n core (n <= NJ <= 32):
//   M P = Q1 R1 (Householder QR with column pivoting),
//   R1^T = Q2 R2 (unpivoted QR),
//   X = R2^T,  X W = U_X diag(s)  (multi-warp Jacobi, typically ~2 sweeps
//   instead of ~6 on the raw core),
// so M = (Q1 U_X) diag(s) (P Q2 W)^T.  Executed by ALL threads of the CTA
// (no divergent call site).  Outputs as warp_jacobi_reg: Uo[:, k], Vo[:, k]
// (ld ldo), s_sorted (descending).  scr: PRECOND_SCR doubles of shared memory.
constexpr int PRECOND_SCR = 5 * 32 * 33 + 2 * 32 + 2 * NWARP * 32 + 32;
template <int NJ>
__device__ __forceinline__ int precond_svd(const double* __restrict__ core, int ldm, int n,
                                           double* __restrict__ Uo, double* __restrict__ Vo,
                                           int ldo, double* __restrict__ s_sorted,
                                           int* __restrict__ perm, double* __restrict__ scr) {
  constexpr int L = 33;
  double* V1 = scr;
  double* V2 = V1 + 32 * L;
  double* X = V2 + 32 * L;
  double* Uj = X + 32 * L;
  double* Wj = Uj + 32 * L;
  double* t1 = Wj + 32 * L;
  double* t2 = t1 + 32;
  double* gbuf = t2 + 32;
  int* P = reinterpret_cast<int*>(gbuf + 2 * NWARP * 32);
  const int tid = threadIdx.x, lane = tid & 31;
  const bool w0 = tid < 32;
  {
    // every warp runs the two register QRs redundantly (no divergent shuffle
    // paths); warp 0 publishes the reflectors, permutation and R2^T
    double a[NJ];
#pragma unroll
    for (int i = 0; i < NJ; ++i) a[i] = (lane < n && i < n) ? core[i + lane * ldm] : 0.0;
    int colid;
    warp_qr_cols<NJ, true>(a, n, V1, L, t1, colid, w0);
    if (w0 && lane < n) P[lane] = colid;
    // R1^T through shared memory: column i of R1^T = row i of R1
    if (w0) {
#pragma unroll
      for (int i = 0; i < NJ; ++i)
        if (lane < n && i < n) X[lane + i * L] = a[i];
    }
    __syncthreads();
    double b[NJ];
#pragma unroll
    for (int i = 0; i < NJ; ++i) b[i] = (lane < n && i < n) ? X[i + lane * L] : 0.0;
    __syncthreads();
    int dummy;
    warp_qr_cols<NJ, false>(b, n, V2, L, t2, dummy, w0);
    // X = R2^T
    if (w0) {
#pragma unroll
      for (int i = 0; i < NJ; ++i)
        if (lane < n && i < n) X[lane + i * L] = b[i];
    }
  }
  __syncthreads();
  int nsw = multi_warp_jacobi<NJ, NWARP>(X, L, n, Uj, Wj, L, s_sorted, perm, gbuf);
  {
    // back-transforms: U = Q1 U_X (threads [0,32)), V = P Q2 W (threads [32,64))
    const bool isU = tid < 32;
    const int k = isU ? tid : tid - 32;
    if (tid < 64 && k < n) {
      const double* src = isU ? Uj : Wj;
      const double* Vh = isU ? V1 : V2;
      const double* th = isU ? t1 : t2;
      double u[NJ];
#pragma unroll
      for (int i = 0; i < NJ; ++i) u[i] = (i < n) ? src[i + k * L] : 0.0;
      for (int j = n - 2; j >= 0; --j) {
        const double tj = th[j];
        if (tj == 0.0) continue;
        double w = 0.0;
#pragma unroll
        for (int i = 0; i < NJ; ++i) {
          if (i == j) w += u[i];
          else if (i > j && i < n) w += Vh[i + j * L] * u[i];
        }
        const double f = tj * w;
#pragma unroll
        for (int i = 0; i < NJ; ++i) {
          if (i == j) u[i] -= f;
          else if (i > j && i < n) u[i] -= f * Vh[i + j * L];
        }
      }
      if (isU) {
#pragma unroll
        for (int i = 0; i < NJ; ++i)
          if (i < n) Uo[i + k * ldo] = u[i];
      } else {
#pragma unroll
        for (int i = 0; i < NJ; ++i)
          if (i < n) Vo[P[i] + k * ldo] = u[i];
      }
    }
    __syncthreads();
  }
  return nsw;
}

}  // namespace lrk
