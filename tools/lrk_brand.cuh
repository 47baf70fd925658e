// lrk_brand.cuh — SVD of a flush core by successive column appends, each
// solved through the secular equation (Gu–Eisenstat vectors).
//
// The flush core of the sweep (lrk_sweep.cu) is
//     K = [[diag(S), C], [0, R]]        (r + pc square),
// S the pane's singular values (descending), C = U^T Y (r x pc), R the
// upper-triangular factor of the remainder (columns in pivot order).  Its SVD
// replaces the QR + SVD of lr_truncate (lowrank.py:124-144) inside flush()
// (forward.py:165-177); the singular values — hence every rank decision —
// are those of the reference's truncation in exact arithmetic.
//
// Appending column k of the new block to the SVD U_k diag(s) V_k^T of the
// leading (r+k) square block gives the bordered matrix
//     M = [[diag(s), z], [0, rho]],   z = U_k^T c,  rho = R[k, k],
// with  M M^T = diag(s_0^2, ..., s_{m-1}^2, 0) + w w^T,  w = (z, rho):
// sigma^2 are the roots of the secular equation
//     f(lam) = 1 + sum_j w_j^2 / (d_j^2 - lam)        (poles d = (s, 0)),
// left vectors u_i ~ w_j / (d_j^2 - lam_i), right vectors
// v_i ~ (s_j w_j / (d_j^2 - lam_i), -1).  As in LAPACK's divide-and-conquer
// SVD (dlasd2/dlasd3/dlasd4):
//  * deflation: |w_j| <= tol drops pole j (sigma = s_j); poles closer than
//    tol are merged by a Givens rotation; rho below tol is raised to tol;
//  * each root is kept as lam = d_o^2 + tau relative to its nearer pole, so
//    every difference d_j^2 - lam = (d_j - d_o)(d_j + d_o) - tau is formed
//    without cancellation; roots by the "middle way" rational iteration from
//    the exact two-pole initial guess, safeguarded by bisection;
//  * the weights are recomputed from the computed roots (Loewner), so the
//    vectors are orthogonal to working precision.
// Accuracy: singular values to absolute O(eps ||K||) (the reference's own
// gesdd gives the same bound), U and V orthogonal to O(eps).
//
// Execution: the secular phases run on JW = 4 warps — lane i owns pole /
// root i, warp w sums the terms j = w (mod 4) and the partial sums meet in
// shared memory behind named barrier 1 (summed in warp order, so the four
// warps take bit-identical decisions); the basis accumulations use the CTA.
// The arithmetic depth is O(pc * iterations) instead of the O(sweeps * n)
// rotation rounds of one-sided Jacobi.
#pragma once

#include "lrk_device.cuh"

namespace lrk {

namespace brand {
constexpr int JW = 4;   // warps in the secular phases
constexpr int LD = 33;  // leading dimension of the append's vector blocks
// workspace (doubles) for brand_core_svd
constexpr int OFF_UU = 0;                        // N x N left vectors (pole rows, sorted cols)
constexpr int OFF_VV = OFF_UU + 32 * LD;         // N x N right vectors
constexpr int OFF_PART = OFF_VV + 32 * LD;       // [2][JW][4][32] partial sums
constexpr int OFF_D = OFF_PART + 2 * JW * 4 * 32;  // active poles d (ascending)
constexpr int OFF_W = OFF_D + 32;                // active weights (signed)
constexpr int OFF_TAU = OFF_W + 32;              // roots: tau
constexpr int OFF_SIG = OFF_TAU + 32;            // sigma per pole lane (unsorted)
constexpr int OFF_SC = OFF_SIG + 32;             // current singular values (descending)
constexpr int OFF_Z = OFF_SC + 32;               // z partials [JW][32]
constexpr int OFF_G = OFF_Z + JW * 32;           // Givens list (rare): 32 x 4
constexpr int OFF_M = OFF_G + 4 * 32;            // merge scratch: d, w (rare path)
constexpr int OFF_DOR = OFF_M + 64;              // per root: d of its origin
constexpr int OFF_ZH = OFF_DOR + 32;             // Loewner weights
constexpr int OFF_I = OFF_ZH + 32;               // int region: 7 x 32 ints
constexpr int WK = OFF_I + 112;
}  // namespace brand

__device__ __forceinline__ void bar_jw() { asm volatile("bar.sync 1, %0;" ::"r"(brand::JW * 32)); }

// SVD of the core K = [[diag(sig0), C], [0, R]] (n = r + pc <= 32) by pc
// appends.  C: r x pc row-major (ldc = pc), R: pc x pc row-major whose column
// piv[k] is the k-th column in triangular order (rows > k zero).  Outputs (all
// threads of the CTA call it): Uo[i + c*32] (row i of the core, column c),
// Vo[j + c*32] (row j in the ORIGINAL column order of K), s_out[c] descending.
// wk: brand::WK doubles of shared memory.  Returns the total root iterations.
// Loops over poles are unrolled to the compile-time bound (T terms per warp,
// predicated), so their loads and reciprocals overlap.
__device__ __forceinline__ int brand_core_svd(const double* __restrict__ sig0, int r,
                                              const double* __restrict__ Cm,
                                              const double* __restrict__ Rm,
                                              const int* __restrict__ piv, int pc,
                                              double* __restrict__ Uo, double* __restrict__ Vo,
                                              double* __restrict__ s_out, double* __restrict__ wk,
                                              long long* __restrict__ tph = nullptr) {
  using namespace brand;
  constexpr int T = 32 / JW;  // pole terms per warp
  long long tprev = clock64();
  long long tacc[12] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
#define BR_T(k)                                 \
  if (tph && threadIdx.x == 0) {                \
    const long long t_ = clock64();             \
    tacc[k] += t_ - tprev;                      \
    tprev = t_;                                 \
  }
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const unsigned full = 0xffffffffu;
  const bool sec = w < JW;  // warps of the secular phases
  double* UU = wk + OFF_UU;
  double* VV = wk + OFF_VV;
  double* part = wk + OFF_PART;
  double* sD = wk + OFF_D;
  double* sW = wk + OFF_W;
  double* sTau = wk + OFF_TAU;
  double* sSig = wk + OFF_SIG;
  double* sc = wk + OFF_SC;
  double* zp = wk + OFF_Z;
  double* gl = wk + OFF_G;
  double* sDor = wk + OFF_DOR;
  double* sZh = wk + OFF_ZH;
  int* iCol = reinterpret_cast<int*>(wk + OFF_I);  // sorted column of each pole lane
  int* iLane = iCol + 32;  // pole lane of active index
  int* iMr = iLane + 32;   // M row of active index
  int* mm = iMr + 32;      // merge scratch (rare path): M row, v column, active flag
  int* mv = mm + 32;
  int* ma = mv + 32;
  double* md = wk + OFF_M;
  double* mw = md + 32;
  // U_acc, V_acc row-major (ld 32) in Uo / Vo during the appends
  for (int idx = tid; idx < 32 * 32; idx += NT) {
    const int i = idx >> 5, j = idx & 31;
    const double e = (i == j && i < r) ? 1.0 : 0.0;
    Uo[idx] = e;
    Vo[idx] = e;
  }
  if (tid < 32) sc[tid] = tid < r ? sig0[tid] : 0.0;
  __syncthreads();
  int its_total = 0;
  for (int k = 0; k < pc; ++k) {
    const int m = r + k, N = m + 1;
    const int col = piv[k];
    // ---------------- z = U_acc^T c (warp w sums rows j = w mod JW)
    if (sec) {
      double acc = 0.0;
#pragma unroll
      for (int t = 0; t < T; ++t) {
        const int j = w + JW * t;
        if (j < m) {
          const double cj = j < r ? Cm[j * pc + col] : Rm[(j - r) * pc + col];
          acc += Uo[j * 32 + lane] * cj;
        }
      }
      zp[w * 32 + lane] = acc;
    }
    // zero the append's vector blocks
    for (int idx = tid; idx < 32 * LD; idx += NT) { UU[idx] = 0.0; VV[idx] = 0.0; }
    __syncthreads();
    BR_T(0)
    int K = 0;          // active poles
    unsigned amask = 0;
    int merged = 0;     // Givens rotations recorded (rare path)
    double my_d = 0.0, my_w = 0.0;
    int my_midx = 0, my_vcol = 0;
    bool my_act = false;
    double scl = 1.0;  // power-of-two scale of this append's poles and weights
    if (sec) {
      // pole q (lane): q = 0 the appended row (d = 0, w = rho); q >= 1 the old
      // singular value s_{m-q} (ascending order since sc is descending)
      const int q = lane;
      if (q < N) {
        if (q == 0) {
          my_w = Rm[k * pc + col];
          my_midx = m;
        } else {
          const int j = m - q;
          my_d = sc[j];
          double z = 0.0;
#pragma unroll
          for (int ww = 0; ww < JW; ++ww) z += zp[ww * 32 + j];
          my_w = z;
          my_midx = j;
        }
      }
      my_vcol = my_midx;
      BR_T(8)
      double mx = fmax(my_d, fabs(my_w));
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(full, mx, o));
      // exact power-of-two scaling to ~1: squares stay far from under/overflow
      {
        int e = mx > 0.0 ? ilog2_normal(mx) : 0;
        e = e < -1000 ? -1000 : (e > 1000 ? 1000 : e);
        scl = pow2i(e);
        const double isc = pow2i(-e);
        my_d *= isc;
        my_w *= isc;
        mx *= isc;
      }
      const double tol = 8.0 * DEPS * mx;
      BR_T(9)
      if (q == 0 && fabs(my_w) < tol) my_w = my_w < 0.0 ? -tol : tol;
      my_act = (q < N) && (q == 0 || fabs(my_w) > tol);
      amask = __ballot_sync(full, my_act);
      // close poles: next active pole within tol
      const unsigned higher = (q < 31) ? (amask & ~((2u << q) - 1u)) : 0u;
      const int nxt = higher ? __ffs(higher) - 1 : -1;
      const double dn = __shfl_sync(full, my_d, nxt < 0 ? q : nxt);
      const bool close = my_act && nxt >= 0 && dn - my_d <= tol;
      BR_T(10)
      if (__any_sync(full, close)) {
        // rare: serial merge by lane 0 of warp 0, Givens list in gl
        if (w == 0) {
          md[q] = my_d; mw[q] = my_w; mm[q] = my_midx; mv[q] = my_vcol; ma[q] = my_act ? 1 : 0;
        }
        bar_jw();
        if (w == 0 && lane == 0) {
          int zpole = 0;  // lane holding the zero pole (d = 0, no diagonal column)
          int a = -1;
          int ng = 0;
          for (int b = 0; b < N; ++b) {
            if (!ma[b]) continue;
            if (a >= 0 && md[b] - md[a] <= tol) {
              const double rr = hypot(mw[a], mw[b]);
              const double c = mw[b] / rr, s = mw[a] / rr;  // w_a -> 0, w_b -> rr
              const int left_only = (a == zpole) ? 1 : 0;
              gl[4 * ng + 0] = (double)mm[a];
              gl[4 * ng + 1] = (double)mm[b];
              gl[4 * ng + 2] = c;
              gl[4 * ng + 3] = left_only ? -(s + 4.0) : s;  // flag in the encoding
              ++ng;
              if (!left_only) {
                md[a] = md[b];
              } else {
                md[b] = 0.0;
                mv[a] = mm[b];  // the deflated zero value takes column b's v
                zpole = b;
              }
              mw[a] = 0.0;
              mw[b] = rr;
              ma[a] = 0;
            }
            if (ma[b]) a = b;
          }
          gl[4 * 31 + 3] = (double)ng;
        }
        bar_jw();
        my_d = md[q]; my_w = mw[q]; my_vcol = mv[q]; my_act = (q < N) && ma[q];
        merged = (int)gl[4 * 31 + 3];
        amask = __ballot_sync(full, my_act);
        bar_jw();
      }
      BR_T(11)
      K = __popc(amask);
      const int pos = __popc(amask & ((1u << q) - 1u));
      if (w == 0 && my_act) {
        sD[pos] = my_d;
        sW[pos] = my_w;
        iLane[pos] = q;
        iMr[pos] = my_midx;
      }
    }
    __syncthreads();
    BR_T(1)
    // ---------------- roots (lane i = root i < K)
    if (sec) {
      const int i = lane;
      const bool live = i < K;
      const bool last = i == K - 1;
      // this warp's pole terms j = w + JW t in registers
      double rd[T], rw2[T];
#pragma unroll
      for (int t = 0; t < T; ++t) {
        const int j = w + JW * t;
        rd[t] = j < K ? sD[j] : 0.0;
        const double wj = j < K ? sW[j] : 0.0;
        rw2[t] = wj * wj;
      }
      double nz2;
      {
        const double wl = lane < K ? sW[lane] : 0.0;
        nz2 = warp_sum(wl * wl);  // identical in every warp
      }
      const int ia = last ? (K > 1 ? K - 2 : 0) : i;
      const int ib = last ? K - 1 : i + 1;
      const double di = live ? sD[i] : 0.0;
      const double dip = (live && !last) ? sD[i + 1] : di;
      const double gap = (dip - di) * (dip + di);
      // midpoint (relative to d_i): gap/2 (interior) or nz2/2 (last)
      const double tm_i = last ? 0.5 * nz2 : 0.5 * gap;
      double pf = 0.0, pab = 0.0;  // sum of all terms / of the two model poles
#pragma unroll
      for (int t = 0; t < T; ++t) {
        const int j = w + JW * t;
        if (live && j < K) {
          const double dl = (rd[t] - di) * (rd[t] + di) - tm_i;
          const double term = rw2[t] * rcp_u(dl);
          pf += term;
          if (j == ia || j == ib) pab += term;
        }
      }
      double* pp = part + w * 4 * 32;
      pp[lane] = pf;
      pp[32 + lane] = pab;
      bar_jw();
      double fm = 1.0, sab = 0.0;
#pragma unroll
      for (int ww = 0; ww < JW; ++ww) {
        fm += part[ww * 4 * 32 + lane];
        sab += part[ww * 4 * 32 + 32 + lane];
      }
      double lo = 0.0, hi = 0.0, tau = 0.0;
      int org = i;
      if (live) {
        if (K == 1) {
          org = 0;
          tau = nz2;
        } else {
          if (!last) {
            if (fm >= 0.0) { org = i; lo = 0.0; hi = 0.5 * gap; }
            else { org = i + 1; lo = -0.5 * gap; hi = 0.0; }
          } else {
            org = i;
            if (fm > 0.0) { lo = 0.0; hi = 0.5 * nz2; } else { lo = 0.5 * nz2; hi = nz2; }
          }
        }
      }
      const double dorg = live ? sD[org] : 0.0;
      // model poles relative to the origin
      const double dA = live ? sD[ia] : 0.0, dB = live ? sD[ib] : 0.0;
      const double pa = (dA - dorg) * (dA + dorg), pb = (dB - dorg) * (dB + dorg);
      if (live && K > 1) {
        // initial guess: Cc + wa/(pa - t) + wb/(pb - t) = 0, other poles frozen
        const double Cc = fm - sab;
        const double wa = sW[ia] * sW[ia], wb = sW[ib] * sW[ib];
        double t = 0.5 * (lo + hi);
        if (ia != ib) {
          const double qa = Cc;
          const double qb = -(Cc * (pa + pb) + wa + wb);
          const double qc = Cc * pa * pb + wa * pb + wb * pa;
          double c1 = t, c2 = t;
          bool ok1 = false, ok2 = false;
          if (qa != 0.0) {
            const double disc = qb * qb - 4.0 * qa * qc;
            if (disc >= 0.0) {
              const double qq = -0.5 * (qb + copysign(sqrt_u(disc), qb));
              if (qq != 0.0) { c1 = qq * rcp_u(qa); c2 = qc * rcp_u(qq); ok1 = true; ok2 = true; }
            }
          } else if (qb != 0.0) {
            c1 = -qc * rcp_u(qb); ok1 = true;
          }
          if (ok1 && c1 > lo && c1 < hi) t = c1;
          else if (ok2 && c2 > lo && c2 < hi) t = c2;
        }
        tau = t;
      }
      // poles relative to the origin; left (psi) / right (phi) split
      double base[T];
      unsigned leftm = 0;
#pragma unroll
      for (int t = 0; t < T; ++t) {
        const int j = w + JW * t;
        base[t] = (rd[t] - dorg) * (rd[t] + dorg);
        if (last ? (j < K - 1) : (j <= i)) leftm |= 1u << t;
      }
      // middle-way iterations (all JW warps, identical decisions)
      bool done = !live || K == 1;
      int it = 0;
      int buf = 1;
      for (; it < 80; ++it) {
        if (__all_sync(full, done)) break;
        double psi = 0.0, phi = 0.0, dpsi = 0.0, dphi = 0.0;
#pragma unroll
        for (int t = 0; t < T; ++t) {
          const int j = w + JW * t;
          if (!done && j < K) {
            const double rc = rcp_u(base[t] - tau);
            const double term = rw2[t] * rc;
            if (leftm & (1u << t)) { psi += term; dpsi += term * rc; }
            else { phi += term; dphi += term * rc; }
          }
        }
        double* pq = part + (buf * JW + w) * 4 * 32;
        pq[lane] = psi; pq[32 + lane] = phi; pq[64 + lane] = dpsi; pq[96 + lane] = dphi;
        bar_jw();
        psi = phi = dpsi = dphi = 0.0;
#pragma unroll
        for (int ww = 0; ww < JW; ++ww) {
          const double* pr = part + (buf * JW + ww) * 4 * 32;
          psi += pr[lane]; phi += pr[32 + lane]; dpsi += pr[64 + lane]; dphi += pr[96 + lane];
        }
        buf ^= 1;
        if (done) continue;
        const double f = 1.0 + psi + phi;
        const double err = 8.0 * DEPS * (double)K * (1.0 + fabs(psi) + fabs(phi));
        if (fabs(f) <= err) { done = true; continue; }
        if (f > 0.0) hi = fmin(hi, tau); else lo = fmax(lo, tau);
        const double da = pa - tau, db = pb - tau;
        const double c = f - da * dpsi - db * dphi;
        const double a = (da + db) * f - da * db * (dpsi + dphi);
        const double b = da * db * f;
        // the step only steers convergence (the test is on f): fast functions
        const double disc = sqrt_u(fabs(a * a - 4.0 * b * c));
        double eta;
        if (c == 0.0) eta = (a != 0.0) ? b * rcp_u(a) : 0.0;
        else if (!last) eta = (a <= 0.0) ? (a - disc) * rcp_u(2.0 * c) : 2.0 * b * rcp_u(a + disc);
        else eta = (a >= 0.0) ? (a + disc) * rcp_u(2.0 * c) : 2.0 * b * rcp_u(a - disc);
        double tn = tau + eta;
        if (!(tn > lo && tn < hi) || eta == 0.0) tn = 0.5 * (lo + hi);
        if (tn == tau) { done = true; continue; }
        tau = tn;
      }
      its_total += it;
      if (w == 0) {
        if (live) { sTau[i] = tau; sDor[i] = dorg; }
        // sigma of every pole lane: roots to the lanes of the active poles,
        // deflated poles keep d (0 for a zero-pole merge)
        const int q = lane;
        if (q < N && !my_act) sSig[q] = (my_vcol != my_midx) ? 0.0 : my_d * scl;
        if (live) sSig[iLane[i]] = sqrt_u(dorg * dorg + tau) * scl;
      }
    }
    __syncthreads();
    BR_T(2)
    // ---------------- sort: sorted column of each pole lane (descending)
    if (tid < 32) {
      const double sv = sSig[tid];
      int rk = 0;
#pragma unroll 4
      for (int e = 0; e < N; ++e) {
        const double se = sSig[e];
        rk += (se > sv) || (se == sv && e < tid);
      }
      if (tid < N) iCol[tid] = rk;
    }
    __syncthreads();
    BR_T(3)
    // ---------------- Loewner weights (lane j, factors i = w mod JW) + vectors
    if (sec) {
      {
        const int j = lane;
        const bool live = j < K;
        const double dj = live ? sD[j] : 0.0;
        double prod = 1.0;
#pragma unroll
        for (int t = 0; t < T; ++t) {
          const int i = w + JW * t;
          if (live && i < K) {
            const double dor = sDor[i];
            const double lm = sTau[i] - (dj - dor) * (dj + dor);  // lam_i - d_j^2
            const double dk = (i < j) ? sD[i] : sD[i + 1 < K ? i + 1 : i];
            prod *= (i == K - 1) ? lm : lm * rcp_u((dk - dj) * (dk + dj));
          }
        }
        part[w * 32 + lane] = prod;
        bar_jw();
        double zh = 1.0;
#pragma unroll
        for (int ww = 0; ww < JW; ++ww) zh *= part[ww * 32 + lane];
        zh = live ? copysign(sqrt_u(fmax(zh, 0.0)), sW[j]) : 0.0;
        if (w == 0) sZh[lane] = zh;
        bar_jw();
      }
      // vectors: lane i = root, warp w = entries j = w mod JW
      const int i = lane;
      const bool rl = i < K;
      const double tau_i = rl ? sTau[i] : 0.0;
      const double dor = rl ? sDor[i] : 0.0;
      double uu[T];
      double nu = 0.0, nv = 0.0;
#pragma unroll
      for (int t = 0; t < T; ++t) {
        const int jj = w + JW * t;
        double u = 0.0;
        if (rl && jj < K) {
          const double d2 = sD[jj];
          const double del = (d2 - dor) * (d2 + dor) - tau_i;  // d_j^2 - lam_i
          u = sZh[jj] * rcp_u(del);
          nu += u * u;
          nv += (d2 * u) * (d2 * u);
        }
        uu[t] = u;
      }
      part[(JW + w) * 32 + lane] = nu;
      part[(2 * JW + w) * 32 + lane] = nv;
      bar_jw();
      nu = 0.0; nv = 1.0;  // the -1 entry of v
#pragma unroll
      for (int ww = 0; ww < JW; ++ww) { nu += part[(JW + ww) * 32 + lane]; nv += part[(2 * JW + ww) * 32 + lane]; }
      if (rl) {
        const double iu = rsqrt_u(nu), iv = rsqrt_u(nv);
        const int c = iCol[iLane[i]];  // sorted column of root i's pole lane
#pragma unroll
        for (int t = 0; t < T; ++t) {
          const int jj = w + JW * t;
          if (jj < K) {
            const int mr = iMr[jj];
            UU[mr + c * LD] = uu[t] * iu;
            VV[mr + c * LD] = sD[jj] * uu[t] * iv;
          }
        }
      }
      bar_jw();
      if (rl && w == 0) VV[m + iCol[iLane[i]] * LD] = -rsqrt_u(nv);
      // deflated poles: unit vectors
      if (w == 0 && lane < N && !my_act) {
        const int c = iCol[lane];
        UU[my_midx + c * LD] = 1.0;
        VV[my_vcol + c * LD] = 1.0;
      }
    }
    __syncthreads();
    BR_T(4)
    // rare: the merge rotations, last first, as row operations
    if (merged && tid < 32) {
      const int ng = (int)gl[4 * 31 + 3];
      for (int g = ng - 1; g >= 0; --g) {
        const int a = (int)gl[4 * g], b = (int)gl[4 * g + 1];
        const double c = gl[4 * g + 2];
        double s = gl[4 * g + 3];
        const bool left_only = s < -2.0;
        if (left_only) s = -(s + 4.0);
        const int cc = tid;
        if (cc < N) {
          const double ua = UU[a + cc * LD], ub = UU[b + cc * LD];
          UU[a + cc * LD] = c * ua + s * ub;
          UU[b + cc * LD] = -s * ua + c * ub;
          if (!left_only) {
            const double va = VV[a + cc * LD], vb = VV[b + cc * LD];
            VV[a + cc * LD] = c * va + s * vb;
            VV[b + cc * LD] = -s * va + c * vb;
          }
        }
        __syncwarp();
      }
    }
    // new singular values
    if (tid < N) sc[iCol[tid]] = sSig[tid];
    __syncthreads();
    BR_T(5)
    // ---------------- accumulate: U <- blockdiag(U, 1) UU, V likewise
    const bool fin = (k == pc - 1);
    double au[4], av[4];
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      const int i = (tid >> 5) + 8 * t, c = lane;
      double su = 0.0, sv = 0.0;
      if (i < m) {
#pragma unroll 4
        for (int j = 0; j < m; ++j) {
          su += Uo[i * 32 + j] * UU[j + c * LD];
          sv += Vo[i * 32 + j] * VV[j + c * LD];
        }
      } else if (i == m) {
        su = UU[m + c * LD];
        sv = VV[m + c * LD];
      }
      au[t] = (i < N && c < N) ? su : 0.0;
      av[t] = (i < N && c < N) ? sv : 0.0;
    }
    __syncthreads();
    BR_T(6)
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      const int i = (tid >> 5) + 8 * t, c = lane;
      if (!fin) {
        Uo[i * 32 + c] = au[t];
        Vo[i * 32 + c] = av[t];
      } else {
        // final layout: column-major; V rows back to the original column order
        Uo[i + c * 32] = au[t];
        const int vi = (i < r || i >= N) ? i : r + piv[i - r];
        Vo[vi + c * 32] = av[t];
      }
    }
    __syncthreads();
    BR_T(7)
  }
  if (tid < 32) s_out[tid] = tid < r + pc ? sc[tid] : 0.0;
  __syncthreads();
  if (tph && tid == 0)
    for (int q = 0; q < 12; ++q) tph[q] += tacc[q];
  return its_total;
#undef BR_T
}

}  // namespace lrk
