// lrk_sflush.cu — the streaming-flush sweep for large n_x (C4/C5 sizes).
//
// Same mathematics as the persistent sweep_kernel (lrk_sweep.cu) and the
// reference's flush (forward.py:165-177 = lr_truncate(lr_add(pane, buffered
// columns)), lowrank.py:124-144): the pane U diag(s) V^T is canonical, so the
// truncation of [U, Y] is an incremental SVD,
//     QR([U, Y]) = [U, Q~] [[I, C], [0, R~]],   core = [[diag(s), C], [0, R~]],
// with C from block CGS2 against U and (Q~, R~) a QR of the remainder.  What
// differs is the organisation, built for HBM streaming when the CTA row blocks
// cannot stay resident in shared memory:
//
//   sf_pass<0> (A)   closes flush f-1 and opens flush f in ONE read of U:
//                      y2 = y1 - U P2 (second CGS subtraction of flush f-1),
//                      G0 = y2^T y2 -> shifted Cholesky R0, and the projection
//                      M = [U, y2]^T Y_f of the next flush's columns plus |Y_f|^2
//   sf_cholqr (x2)     G = (y2 R^-1)^T (y2 R^-1) -> R <- chol(G) R  (shifted
//                      CholeskyQR3 of the 4-column remainder, pivoted and
//                      drop-tolerant for numerically rank-deficient remainders)
//   sf_finish          one CTA: rank-revealing fix-up with the rounding-floor
//                      drop of the persistent kernel, core SVD (register
//                      Jacobi), _rank_cut (lowrank.py:98-111), the update
//                      matrices W' and, for flush f, C1 = W'^T M and
//                      Wd = -W' C1                       (runs next to sf_generate)
//   sf_pass<1> (B)   the basis update of flush f-1 and the first CGS pass of
//                      flush f in ONE read of U: U' = [U, y2] W' (in place, V'
//                      likewise on the time rows), y1 = Y_f + [U, y2] Wd
//                      (= Y_f - U' C1), Pm = [U, y2]^T y1 -> P2 = W'^T Pm
//   sf_generate        the next flush's columns y_k = theta y_{k-1} + B~ w2_k,
//                      on a second stream under sf_finish (three Y buffers)
//
// Per flush the pane basis U is read twice and written once — the compulsory
// traffic of a truncation (Gram read, update read, update write).
// Each pass streams its CTA's contiguous rows in 8-row tiles through
// warp-private cp.async rings (depth sized from the actual pane rank), runs
// the row x small products on the FP64 tensor pipe (DMMA m8n8k4) from shared
// memory, writes a CTA partial and the LAST CTA to finish (atomic ticket)
// reduces the partials in CTA order — deterministic, no grid barrier, no
// cooperative launch.
#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include "lrk_device.cuh"
#include "lrk_kernels.h"
#include "lrk_sflush.h"
#include "lrk_small.cuh"

namespace lrk {

namespace {

constexpr int ST = 256;           // threads per CTA of the light passes
constexpr int NW = 20;            // warps of the staged row passes (96 registers per thread)
constexpr int SPT = 32 * NW;
constexpr int LDW = 68;           // shared leading dimension of the update matrix (== 4 mod 16)
static_assert(LDW == SF_LDW, "pass_b_tail reads the shared and the global update matrix alike");
constexpr int PSTR = SF_N * SF_P + 16 + SF_P + 4;  // per-CTA partial stride (doubles)

// ---- warp-private cp.async rings.  Every staged pass works on 8-row tiles
// and each warp only ever touches its own tiles (the update tile, its share
// of the projections and Grams), so a warp streams its rows through its own
// shared-memory ring: 16-byte cp.async per lane, cp.async.wait_group, no CTA
// barrier and no cross-warp handshake in the main loop.  The ring depth is
// chosen from the ACTUAL column count (the pane rank is only known on the
// device): deep rings at low rank, >= 2 tiles at rank 64.
__device__ __forceinline__ void cp16(void* smem, const void* gmem, bool valid) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  const int sz = valid ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(sa), "l"(gmem), "r"(sz)
               : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory"); }
__device__ __forceinline__ void cp_wait_dyn(int n) {
  switch (n) {
    case 0: cp_wait<0>(); break;
    case 1: cp_wait<1>(); break;
    case 2: cp_wait<2>(); break;
    case 3: cp_wait<3>(); break;
    case 4: cp_wait<4>(); break;
    case 5: cp_wait<5>(); break;
    case 6: cp_wait<6>(); break;
    case 7: cp_wait<7>(); break;
    case 8: cp_wait<8>(); break;
    case 9: cp_wait<9>(); break;
    case 10: cp_wait<10>(); break;
    case 11: cp_wait<11>(); break;
    case 12: cp_wait<12>(); break;
    case 13: cp_wait<13>(); break;
    default: cp_wait<14>(); break;
  }
}
constexpr int LDT = 8;        // rows per tile = leading dimension of a staged column
// Row i of staged column c sits at c * LDT + (i ^ swz(c)): flipping bit 2 of
// the row for every other column pair makes both fragment access patterns
// (rows as the M/N index, rows as the K index) two wavefronts per 8-byte warp
// load — the minimum — without padding the 8-row tiles.
__device__ __forceinline__ int swz(int c) { return (c & 2) << 1; }
constexpr int MAXDEPTH = 15;  // (cp_wait_dyn covers depth - 1 <= 14)

// Tiles of this CTA: a contiguous range [t0, t1) of the 8-row tile grid;
// warp w takes tiles t0 + w, t0 + w + NW, ...
__device__ __forceinline__ void cta_tiles(int64_t n_x, int64_t& t0, int64_t& t1) {
  const int64_t nt = (n_x + LDT - 1) / LDT;
  const int64_t per = (nt + gridDim.x - 1) / gridDim.x;
  t0 = min(nt, (int64_t)blockIdx.x * per);
  t1 = min(nt, t0 + per);
}

// Block-wide sum of K per-thread values into out (shared), fixed order.
template <int K>
__device__ __forceinline__ void cta_sum(double (&v)[K], double* red, double* out) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
  for (int k = 0; k < K; ++k) v[k] = warp_sum(v[k]);
  if (lane == 0)
#pragma unroll
    for (int k = 0; k < K; ++k) red[w * K + k] = v[k];
  __syncthreads();
  if (threadIdx.x < K) {
    double s = 0.0;
    for (int ww = 0; ww < (int)(blockDim.x / 32); ++ww) s += red[ww * K + threadIdx.x];
    out[threadIdx.x] = s;
  }
  __syncthreads();
}

// Last-CTA election: every CTA has written its partial; returns true in the
// CTA that arrived last (which then sees all partials).
__device__ __forceinline__ bool last_cta(unsigned* ticket, int* flag) {
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned t = atomicAdd(ticket, 1u);
    *flag = (t == gridDim.x - 1) ? 1 : 0;
  }
  __syncthreads();
  if (*flag) {
    __threadfence();
    if (threadIdx.x == 0) *ticket = 0u;  // ready for the next launch
  }
  return *flag != 0;
}

// out[e] = sum over CTAs of part[c * PSTR + e], e < len.  The gather runs on
// ONE SM, whose rate of distinct sector requests is the limit (a lane-per-CTA
// layout asked for one sector per 8 bytes: 26k cycles per pass), so lanes
// take consecutive entries (coalesced) and RG thread groups split the CTAs:
// group g adds c = g, g + RG, ... in increasing order with 8 loads in flight,
// the RG group sums meet in shared memory and are added in a fixed tree —
// deterministic.  scr: RG * len doubles of shared scratch.
constexpr int RG = 8;
__device__ __forceinline__ void reduce_parts(const double* part, int len, double* out, double* scr) {
  const int G = (int)gridDim.x;
  for (int idx = threadIdx.x; idx < len * RG; idx += blockDim.x) {
    const int e = idx % len, g = idx / len;
    const double* p = part + e;
    double acc = 0.0;
    int c = g;
    for (; c + 7 * RG < G; c += 8 * RG) {
      double v[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) v[i] = __ldcg(p + (int64_t)(c + i * RG) * PSTR);
#pragma unroll
      for (int i = 0; i < 8; ++i) acc += v[i];
    }
    for (; c < G; c += RG) acc += __ldcg(p + (int64_t)c * PSTR);
    scr[g * len + e] = acc;
  }
  __syncthreads();
  for (int e = threadIdx.x; e < len; e += blockDim.x) {
    double v[RG];
#pragma unroll
    for (int g = 0; g < RG; ++g) v[g] = scr[g * len + e];
    out[e] = ((v[0] + v[1]) + (v[2] + v[3])) + ((v[4] + v[5]) + (v[6] + v[7]));
  }
  __syncthreads();
}

static_assert(PSTR <= SF_XLEN, "rank totals must fit an exchange slot");

// Sharded sweeps: store this shard's total into every shard's exchange slot,
// then release the flags (see SFXBuf).  Called by the whole last CTA.
__device__ __forceinline__ void xr_deposit(const SFArgs& a, unsigned long long seq, const double* tot,
                                           int len) {
  const int par = (int)(seq & 1ull);
  for (int q = 0; q < a.nshard; ++q) {
    double* dst = a.xpeer[q]->data[par][a.shard];
    for (int e = threadIdx.x; e < len; e += blockDim.x) dst[e] = tot[e];
  }
  __threadfence_system();
  __syncthreads();
  if ((int)threadIdx.x < a.nshard) {
    unsigned long long* fl = &a.xpeer[threadIdx.x]->flag[par][a.shard];
    asm volatile("st.release.sys.global.u64 [%0], %1;\n" ::"l"(fl), "l"(seq) : "memory");
  }
}

// Wait for every shard's deposit of exchange `seq` and sum the slots in shard
// order.  A shard that never arrives (lost peer) is reported through info[5]
// after ~4e9 cycles instead of hanging the device.
__device__ __forceinline__ void xr_collect(const SFArgs& a, unsigned long long seq, int len, double* tot) {
  const int par = (int)(seq & 1ull);
  SFXBuf* own = a.xpeer[a.shard];
  // (after one timeout every later exchange of the sweep is let through: the
  // host reports the failure once the sweep has drained)
  if ((int)threadIdx.x < a.nshard && *reinterpret_cast<volatile int*>(a.info + 5) == 0) {
    const unsigned long long* fl = &own->flag[par][threadIdx.x];
    const long long t0 = clock64();
    for (;;) {
      unsigned long long v;
      asm volatile("ld.acquire.sys.global.u64 %0, [%1];\n" : "=l"(v) : "l"(fl) : "memory");
      if (v >= seq) break;
      if (clock64() - t0 > (1ll << 32)) {
        a.info[5] = 1;
        break;
      }
    }
  }
  __syncthreads();
  for (int e = threadIdx.x; e < len; e += blockDim.x) {
    double s = 0.0;
    for (int q = 0; q < a.nshard; ++q) s += __ldcv(&own->data[par][q][e]);
    tot[e] = s;
  }
  __syncthreads();
}

// C = A B for row-major 4x4 blocks restricted to n x n (zero outside); one
// thread, fully unrolled (register resident).
__device__ __forceinline__ void mat4_mul(const double* A, const double* B, double* C, int n) {
  double T[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      double s = 0.0;
#pragma unroll
      for (int k = 0; k < 4; ++k)
        if (k < n) s = fma(A[i * 4 + k], B[k * 4 + j], s);
      T[i][j] = (i < n && j < n) ? s : 0.0;
    }
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) C[i * 4 + j] = T[i][j];
}

// Pivoted, drop-tolerant Cholesky of the n x n SPD-ish G (row-major 4x4):
// P^T G P = L L^T on the kept pivots (pivot > tol * first pivot).  Returns
// R (rows = kept directions, zero elsewhere) with G ~ R^T R and Z with
// (Q Z)^T (Q Z) ~ I on the kept columns (Z = P L^{-T}, dropped columns 0).
// Fully unrolled with compile-time indices (register resident: no dynamically
// indexed local arrays; the pivot swap is a select per entry).
__device__ __forceinline__ int pivoted_chol4(const double* G, int n, double tol, double* R,
                                             double* Z) {
  double A[4][4], L[4][4];
  int perm[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    perm[i] = i;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      A[i][j] = (i < n && j < n) ? G[i * 4 + j] : 0.0;
      L[i][j] = 0.0;
    }
  }
  int kept = 0;
  bool stop = false;
  double d0 = 0.0;
  double iL[4] = {0.0, 0.0, 0.0, 0.0};  // 1 / L[k][k]
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    if (k >= n || stop) continue;
    // pivot: largest remaining diagonal (first on ties)
    int piv = k;
    double best = A[k][k];
#pragma unroll
    for (int i = k + 1; i < 4; ++i)
      if (i < n && A[i][i] > best) { best = A[i][i]; piv = i; }
    // symmetric swap k <-> piv of A, rows of L, perm (selects)
#pragma unroll
    for (int i = k + 1; i < 4; ++i) {
      if (i != piv) continue;
#pragma unroll
      for (int j = 0; j < 4; ++j) { const double t = A[k][j]; A[k][j] = A[i][j]; A[i][j] = t; }
#pragma unroll
      for (int j = 0; j < 4; ++j) { const double t = A[j][k]; A[j][k] = A[j][i]; A[j][i] = t; }
#pragma unroll
      for (int j = 0; j < 4; ++j) { const double t = L[k][j]; L[k][j] = L[i][j]; L[i][j] = t; }
      const int t = perm[k]; perm[k] = perm[i]; perm[i] = t;
    }
    const double d = A[k][k];
    if (k == 0) d0 = d;
    if (!(d > tol * d0) || !(d > 0.0)) { stop = true; continue; }
    const double il = rsqrt_fast(d);  // Newton-refined MUFU reciprocal square root (a few ulp)
    L[k][k] = d * il;
    iL[k] = il;
#pragma unroll
    for (int i = k + 1; i < 4; ++i) L[i][k] = (i < n) ? A[i][k] * il : 0.0;
#pragma unroll
    for (int i = k + 1; i < 4; ++i)
#pragma unroll
      for (int j = k + 1; j < 4; ++j) A[i][j] -= L[i][k] * L[j][k];
    kept = k + 1;
  }
  // Li = L^{-1} on the kept block (lower triangular)
  double Li[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) Li[i][j] = 0.0;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    if (i >= kept) continue;
    Li[i][i] = iL[i];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      if (j >= i) continue;
      double s = 0.0;
#pragma unroll
      for (int q = 0; q < 4; ++q)
        if (q >= j && q < i) s += L[i][q] * Li[q][j];
      Li[i][j] = -s * iL[i];
    }
  }
  // R[a][c] = L[j][a] with perm[j] == c (j >= a); Z[c][a] = Li[a][j] with perm[j] == c
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      double rv = 0.0, zv = 0.0;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const bool hit = perm[j] == c && a < kept && j < n;
        if (hit && j >= a) rv = L[j][a];
        if (hit && j < kept && a >= j) zv = Li[a][j];
      }
      R[a * 4 + c] = rv;
      Z[c * 4 + a] = zv;
    }
  return kept;
}

}  // namespace

// Start of the first CholeskyQR pass (thread 0 of EVERY CTA, redundantly: the
// code stays hot in the instruction caches of all SMs, whereas in the tail of
// pass A — once per launch on whichever SM finished last — the same ~1,500
// instructions took 28k cycles of cold instruction fetch): the shifted
// Cholesky factor of G0 = y2^T y2 (Fukaya et al. shifted CholeskyQR3, first
// step); a remainder at the block's rounding floor 16 eps ||Y|| is dropped
// whole.  G0 row-major with stride 4.  Returns drop_all; R, Z: 16 doubles each.
static __device__ __noinline__ int sf_shifted_chol(int64_t n_x_glob, const double* G0, const double* yn,
                                                   int pc, double* R, double* Z) {
  double G[16] = {};
  for (int u = 0; u < pc; ++u)
    for (int v = 0; v < pc; ++v) G[u * 4 + v] = G0[u * 4 + v];
  double tr = 0.0, ysq = 0.0;
  for (int s = 0; s < pc; ++s) { tr += G[s * 5]; ysq += yn[s]; }
  const double delta = 16.0 * DEPS * sqrt(ysq);
  const int drop = !(sqrt(tr) > delta);
  double Rm[16], Zm[16];
  if (drop) {
    for (int i = 0; i < 16; ++i) { Rm[i] = 0.0; Zm[i] = 0.0; }
  } else {
    const double shift = 11.0 * ((double)n_x_glob * pc + pc * (pc + 1)) * DEPS * tr;
    for (int s = 0; s < pc; ++s) G[s * 5] += shift;
    pivoted_chol4(G, pc, 0.0, Rm, Zm);
  }
  for (int i = 0; i < 16; ++i) { R[i] = Rm[i]; Z[i] = Zm[i]; }
  return drop;
}

// CholeskyQR pass tail (thread 0): R <- chol(G) R, Rinv <- Rinv chol(G)^{-1};
// pivots below (1e-10)^2 of the leading one are rounding residue of a
// numerically rank-deficient remainder and are dropped (see header).
static __device__ __noinline__ void sf_chol_update(SFState* st, const double* tot, int pc) {
  double G[16] = {};
  int q = 0;
  for (int u = 0; u < SF_P; ++u)
    for (int v = u; v < SF_P; ++v) {
      G[u * 4 + v] = G[v * 4 + u] = tot[q];
      ++q;
    }
  double R1[16], Z1[16], Rc[16], Ri[16], Rn[16], Zn[16];
  pivoted_chol4(G, pc, 1e-20, R1, Z1);
  for (int i = 0; i < 16; ++i) { Rc[i] = st->Rc[i]; Ri[i] = st->Rinv[i]; }
  mat4_mul(R1, Rc, Rn, pc);
  mat4_mul(Ri, Z1, Zn, pc);
  for (int i = 0; i < 16; ++i) { st->Rc[i] = Rn[i]; st->Rinv[i] = Zn[i]; }
}

// ------------------------------------------------------------ staged row pass
// X = [U(:, :r), y] with y the pcp-column block of flush f-1 in Yg[(f-1) % 3]
// (y1 on entry to pass A, y2 afterwards); Yn = the pcn columns of flush f.
//
// MODE 0 (pass A):  y2 = y1 - U P2 = X [-P2; I]            (in place)
//                   T  = X^T [Yn | y2]: M = X^T Yn (n x 4), G0 = y2^T y2, |Yn_s|^2
//   last CTA: M, yn_next -> state; shifted Cholesky of G0.
// MODE 1 (pass B):  [U' | d] = X [Wp | Wd]: U' in place over U (rn columns),
//                   y1 = Yn + d (in place), V' = [V, E] Vc on this CTA's time rows
//                   Pm = X^T y1 (n x 4)
//   last CTA: P2 = Wp^T Pm, C = C1 + P2, pane bookkeeping (r <- rn, pcp <- pcn).
// Warp w owns tiles w, w+16, ... of the CTA's 8-row tile range: its step-1
// output tile and its share of the projections need no CTA barrier.
// Tail of pass A (whole CTA; tot = M (n x 4) | G0 (4 x 4) | |Yn_s|^2): the
// projection of the flush being opened goes to the state, the remainder of
// the flush being closed gets its shifted Cholesky factor.
__device__ __forceinline__ void pass_a_tail(const SFArgs& a, SFState* st, const double* tot, int f) {
  const int tid = threadIdx.x;
  const int r = st->r, pcp = st->pcp, n = r + pcp;
  const int pcn = f < a.nflush ? min(a.p, a.n_t - f * a.p) : 0;
  for (int idx = tid; idx < n * SF_P; idx += blockDim.x) st->M[idx] = tot[idx];
  if (tid < SF_P) st->yn_next[tid] = tot[n * SF_P + 16 + tid];
  __syncthreads();
  if (tid == 0) {
    st->pc_new = pcn;
    if (pcp > 0) {
      for (int i = 0; i < 16; ++i) st->G0[i] = tot[n * SF_P + i];  // shifted Cholesky: first CholeskyQR pass
    } else {
      // nothing to close (first flush): no sf_finish will run before pass B
      for (int s2 = 0; s2 < SF_P; ++s2) st->yn[s2] = tot[n * SF_P + 16 + s2];
      st->rn = r;
      st->pending = 0;
    }
  }
}

// Tail of pass B (whole CTA; tot = Pm (n x 4); Wp: n x rn, column stride LDW):
// P2 = Wp^T Pm, C = C1 + P2; the pane now has rn explicit columns.
__device__ __forceinline__ void pass_b_tail(const SFArgs& a, SFState* st, const double* tot,
                                            const double* Wp, int f) {
  const int tid = threadIdx.x;
  const int r = st->r, pcp = st->pcp, n = r + pcp, rn = st->rn;
  const int pcn = f < a.nflush ? min(a.p, a.n_t - f * a.p) : 0;
  for (int idx = tid; idx < rn * pcn; idx += blockDim.x) {
    const int i = idx / pcn, s2 = idx % pcn;
    double acc = 0.0;
    for (int k = 0; k < n; ++k) acc += Wp[i * LDW + k] * tot[k * SF_P + s2];
    st->P2[i * SF_P + s2] = acc;
    st->C[i * SF_P + s2] += acc;
  }
  const bool final_pass = f >= a.nflush;
  if (final_pass)
    for (int k = tid; k < rn; k += blockDim.x) a.sigma[k] = st->sig[k];
  __syncthreads();
  if (tid == 0) {
    st->r = rn;
    st->pcp = pcn;
    st->pending = 0;
    if (final_pass) {
      a.info[0] = rn;
      a.trace[a.nflush] = rn;
    }
  }
}

// Runtime sizes and pointers of one pass (uniform over the CTA).
struct PassRt {
  int r, pcp, n, pcn, rn, nwc, ncol, per_warp;
  int nwa;  // warps that stream tiles (all NW unless the rank is so high that two slots per warp need more room)
  int64_t ct0, ct1;
  double *Yab, *Ynb, *W, *ring;
  const unsigned long long* colp;  // shared: base address of every staged column
};

// The tile loop of a pass for NT 8-column fragment tiles (compile time: the
// fragment loops are branch free, every shared-memory operand is one load at
// an immediate offset from a per-lane base).  See sf_pass for the mathematics.
template <int MODE, int NT>
__device__ __forceinline__ void pass_loop(const SFArgs& a, const PassRt& P, double (&m9)[9][2],
                                          double& ysq_out) {
  constexpr int NK = NT == 9 ? 17 : 2 * NT;   // k groups of 4 (rows of W are zero past n)
  constexpr int NJ = MODE == 0 ? 1 : NT;      // column tiles of the step-1 product
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int r = P.r, n = P.n, pcp = P.pcp, pcn = P.pcn, rn = P.rn, nwc = P.nwc, ncol = P.ncol;
  const int slot = (ncol > 0 ? ncol : 1) * LDT;
  int depth = P.per_warp / slot;
  depth = depth < 2 ? 2 : (depth > MAXDEPTH ? MAXDEPTH : depth);
  double* base = P.ring + (int64_t)warp * P.per_warp;
  // cp.async: the lane copies row pair jp of columns cg, cg + 8, ...
  const int jp = lane & 3, cg = lane >> 2;
  const int dlane = cg * LDT + 2 * (jp ^ (cg & 2));
  const int nci = (ncol - cg + 7) >> 3;
  auto issue = [&](int sl, int64_t tile, bool valid) {
    if (valid) {
      const int64_t row = tile * LDT + 2 * jp;
      const bool ok = row < a.n_x;
      const int64_t roff = ok ? row : 0;
      double* dst = base + sl * slot + dlane;
      for (int i = 0; i < nci; ++i)
        cp16(dst + i * 8 * LDT, reinterpret_cast<const double*>(P.colp[cg + 8 * i]) + roff, ok);
    }
    cp_commit();
  };
  // step 1 (transposed: D = W^T X^T): X[k][row g], k = 4kk + t; W[k][col 8j + g]
  const int xo1 = t * LDT + (g ^ ((t & 2) << 1));
  const double* Wl = P.W + g * LDW + t;
  // step 2: A = X^T[col 8j + g][row 4kk + t], B = [Yn | y2][row 4kk + t][col g]
  const int sg = (g & 2) << 1;
  const int ao0 = g * LDT + (t ^ sg), ao1 = g * LDT + ((4 + t) ^ sg);
  const int cy = (MODE == 0 && g >= 4) ? r + g - 4 : n + g;
  const bool bok = (MODE == 0 && g >= 4) ? (g - 4 < pcp) : (g < pcn);
  const int bo0 = cy * LDT + (t ^ swz(cy)), bo1 = cy * LDT + ((4 + t) ^ swz(cy));
  const bool step1 = n > 0 && nwc > 0;
  const bool step2 = n > 0 && (pcn > 0 || (MODE == 0 && pcp > 0));
  double m[NT][2];
#pragma unroll
  for (int j = 0; j < NT; ++j) m[j][0] = m[j][1] = 0.0;
  double ysq = 0.0;
  const int nwa = P.nwa;
  // (warps past nwa own no tiles: their loop below is empty)
  const int64_t first = warp < nwa ? P.ct0 + warp : P.ct1;
  for (int q = 0; q < depth - 1; ++q) {
    const int64_t tq = first + (int64_t)q * nwa;
    issue(q, tq, tq < P.ct1);
  }
  int cur = 0, nxt = depth - 1;
  for (int64_t tile = first; tile < P.ct1; tile += nwa) {
    {
      const int64_t tq = tile + (int64_t)(depth - 1) * nwa;
      issue(nxt, tq, tq < P.ct1);
    }
    cp_wait_dyn(depth - 1);
    __syncwarp();
    double* X = base + cur * slot;   // element (row i, staged column c) at X[c * LDT + (i ^ swz(c))]
    const int64_t row2 = tile * LDT + 2 * t;     // the lane's row pair of step 1
    const bool rok = row2 < a.n_x;
    if (step1) {
      double acc[NJ][2];
#pragma unroll
      for (int j = 0; j < NJ; ++j) acc[j][0] = acc[j][1] = 0.0;
#pragma unroll
      for (int kk = 0; kk < NK; ++kk) {
        const double xv = X[kk * 4 * LDT + xo1];
#pragma unroll
        for (int j = 0; j < NJ; ++j) dmma884(acc[j][0], acc[j][1], Wl[j * 8 * LDW + 4 * kk], xv);
      }
      __syncwarp();  // all lanes have read X before y is overwritten in place
      if (MODE == 0) {
        if (g < pcp) {
          const double2 v = make_double2(acc[0][0], acc[0][1]);
          *reinterpret_cast<double2*>(X + (r + g) * LDT + ((2 * t) ^ swz(r + g))) = v;
          if (rok) *reinterpret_cast<double2*>(P.Yab + row2 + (int64_t)g * a.ldy) = v;
        }
      } else {
        double* pu = a.U + row2 + (int64_t)g * a.ldu;
#pragma unroll
        for (int j = 0; j < NJ; ++j) {
          const int c = 8 * j + g;
          double2 v = make_double2(acc[j][0], acc[j][1]);
          if (c < rn) {
            if (rok) *reinterpret_cast<double2*>(pu) = v;
          } else if (c < nwc) {
            const int s2 = c - rn;
            double2* ys = reinterpret_cast<double2*>(X + (n + s2) * LDT + ((2 * t) ^ swz(n + s2)));
            const double2 y0 = *ys;
            v.x += y0.x;
            v.y += y0.y;
            *ys = v;
            if (rok) *reinterpret_cast<double2*>(P.Ynb + row2 + (int64_t)s2 * a.ldy) = v;
          }
          pu += 8 * a.ldu;
        }
      }
      __syncwarp();
    }
    if (step2) {
      const double b0 = bok ? X[bo0] : 0.0, b1 = bok ? X[bo1] : 0.0;
#pragma unroll
      for (int j = 0; j < NT; ++j) dmma884(m[j][0], m[j][1], X[j * 8 * LDT + ao0], b0);
#pragma unroll
      for (int j = 0; j < NT; ++j) dmma884(m[j][0], m[j][1], X[j * 8 * LDT + ao1], b1);
    }
    if (MODE == 0 && (lane >> 3) < pcn) {
      const double y = X[(n + (lane >> 3)) * LDT + (lane & 7)];
      ysq += y * y;
    }
    __syncwarp();  // every lane is done with this slot before it is refilled
    cur = cur + 1 == depth ? 0 : cur + 1;
    nxt = nxt + 1 == depth ? 0 : nxt + 1;
  }
  cp_wait<0>();
#pragma unroll
  for (int j = 0; j < NT; ++j) { m9[j][0] = m[j][0]; m9[j][1] = m[j][1]; }
  ysq_out = ysq;
}

template <int MODE>
__global__ void __launch_bounds__(SPT, 1) sf_pass(const SFArgs a, int f, unsigned long long seq) {
  extern __shared__ __align__(16) double smem[];
  __shared__ unsigned long long colp[SF_N + SF_P + 8];
  const long long tstart = a.dbg ? clock64() : 0;
  SFState* st = a.st;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int r = st->r, pcp = st->pcp;
  const int n = r + pcp;                      // columns of X
  const int start = f * a.p;
  const int pcn = f < a.nflush ? min(a.p, a.n_t - start) : 0;
  const int rn = MODE == 1 ? st->rn : 0;
  const int nwc = MODE == 1 ? rn + pcn : pcp;   // columns of the step-1 matrix W
  double* Yab = a.Yg[(f + 2) % 3];            // flush f-1
  double* Ynb = a.Yg[f % 3];                  // flush f
  double* W = smem;                           // n x nwc, column c at W + c * LDW
  double* stage = W + (SF_N + SF_P) * LDW;    // V update scratch, then the warp rings
  const int avail = a.smem_pass / (int)sizeof(double) - (SF_N + SF_P) * LDW - 16;
  int* flag = reinterpret_cast<int*>(stage + avail);
  double* red = stage;                        // reused after the main loop

  // NT: 8-column tiles of the widest fragment loop (X columns or W columns);
  // W is zero padded to 8 NT columns and min(8 NT, 68) rows
  const int NT = max(1, max((n + 7) >> 3, (nwc + 7) >> 3));
  {
    const int nk4 = min(8 * NT, SF_N), nc8 = 8 * NT;
    for (int idx = tid; idx < nk4 * nc8; idx += SPT) {
      const int k = idx % nk4, c = idx / nk4;
      double v = 0.0;
      if (k < n && c < nwc) {
        if (MODE == 0) v = k < r ? -st->P2[k * SF_P + c] : (k - r == c ? 1.0 : 0.0);
        else v = c < rn ? st->Wp[k + c * SF_LDW] : st->Wd[k * SF_P + (c - rn)];
      }
      W[c * LDW + k] = v;
    }
  }
  if (MODE == 1) {
    if (st->pending) {
      // time rows of this CTA: V' = [V, E] Vc   (in place, via shared memory)
      const int64_t tper = ((int64_t)a.n_t + gridDim.x - 1) / gridDim.x;
      const int64_t nt64 = a.n_t;
      const int64_t t0 = min(nt64, (int64_t)blockIdx.x * tper), t1 = min(nt64, t0 + tper);
      const int nrow = (int)(t1 - t0);
      double* Vs = stage;  // nrow x r
      double* Vc = stage + nrow * SF_CAP + 8;
      for (int idx = tid; idx < n * rn; idx += SPT) Vc[idx] = st->Vc[(idx % n) + (idx / n) * SF_LDW];
      for (int idx = tid; idx < nrow * r; idx += SPT)
        Vs[idx] = a.V[(t0 + idx % nrow) + (int64_t)(idx / nrow) * a.ldv];
      __syncthreads();
      const int sp = st->startp;
      for (int idx = tid; idx < nrow * rn; idx += SPT) {
        const int tl = idx % nrow, c = idx / nrow;
        const int64_t tt = t0 + tl;
        const int sel = a.adjoint ? (a.n_t - 1 - sp) - (int)tt : (int)tt - sp;
        double acc = (sel >= 0 && sel < pcp) ? Vc[(r + sel) + c * n] : 0.0;
        for (int k = 0; k < r; ++k) acc += Vs[tl + k * nrow] * Vc[k + c * n];
        a.V[tt + (int64_t)c * a.ldv] = acc;
      }
    }
  }

  const int nm = (n + 7) >> 3;
  const int ncol = n + pcn;  // tile: X columns, then Yn
  for (int c = tid; c < ncol; c += SPT)
    colp[c] = reinterpret_cast<unsigned long long>(
        c < r ? a.U + (int64_t)c * a.ldu
              : (c < n ? Yab + (int64_t)(c - r) * a.ldy : Ynb + (int64_t)(c - n) * a.ldy));
  __syncthreads();           // the V-update scratch is free again
  // columns past ncol are read by the padded (branch-free) fragment loops and
  // multiplied by zero rows of W: they must hold finite numbers
  for (int idx = tid; idx < avail; idx += SPT) stage[idx] = 0.0;
  __syncthreads();
  PassRt P;
  P.r = r; P.pcp = pcp; P.n = n; P.pcn = pcn; P.rn = rn; P.nwc = nwc; P.ncol = ncol;
  cta_tiles(a.n_x, P.ct0, P.ct1);
  P.Yab = Yab; P.Ynb = Ynb; P.W = W; P.ring = stage; P.colp = colp;
  // two ring slots per streaming warp must fit (headroom: the padded fragment
  // loops read up to 7 columns past a slot)
  P.nwa = min(NW, max(1, (avail - 128) / (2 * (ncol > 0 ? ncol : 1) * LDT)));
  P.per_warp = ((avail - 128) / P.nwa) & ~1;
  double m[9][2];  // T tile j = X columns 8j..8j+7
#pragma unroll
  for (int j = 0; j < 9; ++j) m[j][0] = m[j][1] = 0.0;
  double ysq = 0.0;
  switch (NT) {
    case 1: pass_loop<MODE, 1>(a, P, m, ysq); break;
    case 2: pass_loop<MODE, 2>(a, P, m, ysq); break;
    case 3: pass_loop<MODE, 3>(a, P, m, ysq); break;
    case 4: pass_loop<MODE, 4>(a, P, m, ysq); break;
    case 5: pass_loop<MODE, 5>(a, P, m, ysq); break;
    case 6: pass_loop<MODE, 6>(a, P, m, ysq); break;
    case 7: pass_loop<MODE, 7>(a, P, m, ysq); break;
    case 8: pass_loop<MODE, 8>(a, P, m, ysq); break;
    default: pass_loop<MODE, 9>(a, P, m, ysq); break;
  }
  __syncthreads();
  // ---- CTA partial (warps meet in shared memory and are summed in warp order)
  // MODE 0: M (n x 4 row-major), G0 (4 x 4, stride 4), |Yn_s|^2 (4); MODE 1: Pm (n x 4)
  double* part = a.part + (int64_t)blockIdx.x * PSTR;
  const int plen = MODE == 0 ? n * SF_P + 16 + SF_P : n * SF_P;
  if (plen > 0) {
    double* wp = stage;  // NW x plen
    for (int idx = tid; idx < NW * plen; idx += SPT) wp[idx] = 0.0;
    __syncthreads();
#pragma unroll
    for (int j = 0; j < 9; ++j) {
      if (j >= nm) break;
      const int xr = 8 * j + g;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int c = 2 * t + h;
        if (xr < n && c < SF_P) wp[warp * plen + xr * SF_P + c] = m[j][h];
        if (MODE == 0 && xr >= r && xr < n && c >= SF_P)
          wp[warp * plen + n * SF_P + (xr - r) * 4 + (c - SF_P)] = m[j][h];
      }
    }
    if (MODE == 0) {
      double yw = ysq;
      yw += __shfl_xor_sync(0xffffffffu, yw, 1);
      yw += __shfl_xor_sync(0xffffffffu, yw, 2);
      yw += __shfl_xor_sync(0xffffffffu, yw, 4);
      if ((lane & 7) == 0 && (lane >> 3) < SF_P) wp[warp * plen + n * SF_P + 16 + (lane >> 3)] = yw;
    }
    __syncthreads();
    for (int e = tid; e < plen; e += SPT) {
      double acc = 0.0;
      for (int w = 0; w < NW; ++w) acc += wp[w * plen + e];
      part[e] = acc;
    }
  }
  const long long tq0 = a.dbg ? clock64() : 0;
  if (!last_cta(a.ticket + MODE, flag)) return;
  const long long tq1 = a.dbg ? clock64() : 0;
  double* tot = red + NW * PSTR + 64;
  reduce_parts(a.part, plen, tot, tot + PSTR + 8);
  const long long tq2 = a.dbg ? clock64() : 0;
  if (a.nshard > 1) {  // the tail runs in sf_tail once every shard has deposited
    xr_deposit(a, seq, tot, plen);
    return;
  }
  if (MODE == 0) pass_a_tail(a, st, tot, f);
  else pass_b_tail(a, st, tot, W, f);
  if (a.dbg && tid == 0) {  // diagnostics: cycles of the election, the reduction and the tail algebra
    long long* d = a.dbg + 8 * MODE;
    d[0] += tq1 - tq0;
    d[1] += tq2 - tq1;
    d[2] += clock64() - tq2;
    d[3] += 1;
    d[4] += tq0 - tstart;
  }
}

// One-CTA tail of a sharded pass: collect the shard totals, then the same
// small algebra the last CTA runs in an unsharded sweep.
// KIND 0: pass A, 1: pass B, 2: CholeskyQR pass.
template <int KIND>
__global__ void __launch_bounds__(ST) sf_tail(const SFArgs a, int f, unsigned long long seq) {
  __shared__ double tot[SF_XLEN];
  SFState* st = a.st;
  const int n = st->r + st->pcp;
  const int len = KIND == 0 ? n * SF_P + 16 + SF_P : (KIND == 1 ? n * SF_P : 10);
  xr_collect(a, seq, len, tot);
  if (KIND == 0) pass_a_tail(a, st, tot, f);
  else if (KIND == 1) pass_b_tail(a, st, tot, st->Wp, f);
  else if (threadIdx.x == 0 && !st->drop_all) sf_chol_update(st, tot, st->pcp);
}

// ------------------------------------------------------------ generation
// The next flush's buffered columns (forward.py:180 in the DST eigenbasis):
// y_k = theta .* y_{k-1} + rowscale .* (B w2_k), k = the flush's steps.
__global__ void __launch_bounds__(ST) sf_generate(const SFArgs a, int f) {
  __shared__ double w2s[SF_CAP * SF_P];
  __shared__ int any;
  const int start = f * a.p;
  const int pc = min(a.p, a.n_t - start);
  const int rb = a.rb_dev ? min(a.rb, *a.rb_dev) : a.rb;
  if (threadIdx.x == 0) any = 0;
  __syncthreads();
  bool nz = false;
  for (int idx = threadIdx.x; idx < rb * SF_P; idx += ST) {
    const int j = idx / SF_P, s = idx % SF_P;
    const int k = a.adjoint ? (a.n_t - 1 - (start + s)) : (start + s);
    const double v = s < pc ? a.W2[k + (int64_t)j * a.ldw2] : 0.0;
    w2s[j * SF_P + s] = v;
    nz |= v != 0.0;
  }
  if (nz) any = 1;
  __syncthreads();
  const int rbe = any ? rb : 0;  // a flush without a nonzero rhs time row skips B
  double* Y = a.Yg[f % 3];
  for (int64_t i = (int64_t)blockIdx.x * ST + threadIdx.x; i < a.n_x; i += (int64_t)gridDim.x * ST) {
    double acc[SF_P] = {0.0, 0.0, 0.0, 0.0};
    int j = 0;
    for (; j + 16 <= rbe; j += 16) {  // 16 independent loads in flight per thread
      double b[16];
#pragma unroll
      for (int u = 0; u < 16; ++u) b[u] = a.B[i + (int64_t)(j + u) * a.ldb];
#pragma unroll
      for (int u = 0; u < 16; ++u)
#pragma unroll
        for (int s = 0; s < SF_P; ++s) acc[s] += b[u] * w2s[(j + u) * SF_P + s];
    }
    for (; j + 4 <= rbe; j += 4) {
      double b[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) b[u] = a.B[i + (int64_t)(j + u) * a.ldb];
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int s = 0; s < SF_P; ++s) acc[s] += b[u] * w2s[(j + u) * SF_P + s];
    }
    for (; j < rbe; ++j) {
      const double b = a.B[i + (int64_t)j * a.ldb];
#pragma unroll
      for (int s = 0; s < SF_P; ++s) acc[s] += b * w2s[j * SF_P + s];
    }
    const double tv = a.theta[i];
    const double rs = a.rowscale ? a.rowscale[i] : 1.0;
    double y = a.yprev[i];
#pragma unroll
    for (int s = 0; s < SF_P; ++s) {
      if (s < pc) {
        y = tv * y + rs * acc[s];
        if (fabs(y) < a.ftz) y = 0.0;
        Y[i + (int64_t)s * a.ldy] = y;
      }
    }
    a.yprev[i] = y;
  }
}

// ----------------------------------------------------------- CholeskyQR passes
// G = Q^T Q with Q = y2 Rinv; R <- chol(G) R, Rinv <- Rinv chol(G)^{-1}
// (pivoted, drop-tolerant).  Light streaming kernel over the 4 columns of
// flush f (usually still in L2): 4 rows per thread and step, 16 loads in flight.
__global__ void __launch_bounds__(ST, 2) sf_cholqr(const SFArgs a, int f, int pass,
                                                     unsigned long long seq) {
  SFState* st = a.st;
  const long long tstart = a.dbg ? clock64() : 0;
  __shared__ int flag;
  __shared__ double red[8 * 10 + 16];
  __shared__ double tot[16];
  const int tid = threadIdx.x;
  const int pc = st->pcp;
  __shared__ double sRc[16], sRi[16], sG0[16], sYn[SF_P];
  __shared__ int sdrop;
  if (pass == 0) {
    if (tid < 16) sG0[tid] = st->G0[tid];
    if (tid < SF_P) sYn[tid] = st->yn[tid];
    __syncthreads();
    if (tid == 0) {
      sdrop = sf_shifted_chol(a.n_x_glob, sG0, sYn, pc, sRc, sRi);
      if (blockIdx.x == 0) {  // the state the later kernels (and this pass's tail) read
        st->drop_all = sdrop;
        for (int i = 0; i < 16; ++i) { st->Rc[i] = sRc[i]; st->Rinv[i] = sRi[i]; }
      }
    }
  } else {
    if (tid < 16) sRi[tid] = st->Rinv[tid];
    if (tid == 0) sdrop = st->drop_all;
  }
  __syncthreads();
  const bool skip = sdrop != 0;
  double gacc[10] = {};
  if (!skip) {
    double Ri[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) Ri[i] = sRi[i];
    const double* Y = a.Yg[f % 3];
    const int64_t stride = (int64_t)gridDim.x * ST;
    for (int64_t i0 = (int64_t)blockIdx.x * ST + tid; i0 < a.n_x; i0 += 4 * stride) {
      double y[4][SF_P];
#pragma unroll
      for (int h = 0; h < 4; ++h) {
        const int64_t i = i0 + h * stride;
#pragma unroll
        for (int s = 0; s < SF_P; ++s) y[h][s] = (s < pc && i < a.n_x) ? Y[i + (int64_t)s * a.ldy] : 0.0;
      }
#pragma unroll
      for (int h = 0; h < 4; ++h) {
        double qv[SF_P];
#pragma unroll
        for (int c = 0; c < SF_P; ++c) {
          double acc = 0.0;
#pragma unroll
          for (int s = 0; s < SF_P; ++s) acc += y[h][s] * Ri[s * 4 + c];
          qv[c] = acc;
        }
        int q = 0;
#pragma unroll
        for (int u = 0; u < SF_P; ++u)
#pragma unroll
          for (int v = u; v < SF_P; ++v) gacc[q++] += qv[u] * qv[v];
      }
    }
  }
  double* outv = red + 8 * 10;
  cta_sum<10>(gacc, red, outv);
  double* part = a.part + (int64_t)blockIdx.x * PSTR;
  if (tid < 10) part[tid] = outv[tid];
  const long long tq0 = a.dbg ? clock64() : 0;
  if (!last_cta(a.ticket + 3 + pass, &flag)) return;
  const long long tq1 = a.dbg ? clock64() : 0;
  reduce_parts(a.part, 10, tot, red);
  const long long tq2 = a.dbg ? clock64() : 0;
  if (a.nshard > 1) {
    xr_deposit(a, seq, tot, 10);
    return;
  }
  if (tid == 0 && !skip) sf_chol_update(st, tot, pc);
  if (a.dbg && tid == 0) {
    long long* d = a.dbg + 16;
    d[0] += tq1 - tq0;
    d[1] += tq2 - tq1;
    d[2] += clock64() - tq2;
    d[3] += 1;
    d[4] += tq0 - tstart;
  }
}

// The small algebra closing flush f (one CTA): rank-revealing fix-up of R,
// core assembly, core SVD, zero test and _rank_cut, the update matrices of the
// next pass B and the first CGS coefficients of the flush being projected.
__global__ void __launch_bounds__(ST, 1) sf_finish(const SFArgs a, int f) {
  extern __shared__ double sm[];
  SFState* st = a.st;
  const long long tf0 = a.dbg ? clock64() : 0;
  const int tid = threadIdx.x, warp = tid >> 5;
  const int r = st->r, pc = st->pcp, n = r + pc;
  const int start = f * a.p;
  double* sT = sm;                // 16: y2 -> Q~ transform
  double* sR = sm + 16;           // 16: R~ (row-major 4x4)
  double* sS = sm + 32;           // SF_N singular values
  double* sScr = sS + SF_N + 4;   // 2*4*32 Jacobi exchange + scratch
  double* sCore = sScr + 512;     // 32 x 33 (n <= 32) or SF_N x SF_N (jacobi_svd)
  double* Uc = sCore + SF_N * SF_N + 8;   // n x n (ld n)
  double* Vc = Uc + SF_N * SF_N + 8;
  double* Vj = Vc + SF_N * SF_N + 8;
  int* iPerm = reinterpret_cast<int*>(Vj + SF_N * SF_N + 8);
  int* iFlag = iPerm + SF_N + 4;
  // the small state the single-thread sections read is staged by all threads
  // first (one parallel round trip to L2 instead of a serial chain of loads)
  __shared__ double gRc[16], gRi[16], gYn[SF_P], gSig[SF_N], gM[SF_N * SF_P];
  if (tid < 16) { gRc[tid] = st->Rc[tid]; gRi[tid] = st->Rinv[tid]; }
  if (tid < SF_P) gYn[tid] = st->yn[tid];
  for (int i = tid; i < r; i += ST) gSig[i] = st->sig[i];
  for (int i = tid; i < n * SF_P; i += ST) gM[i] = st->M[i];
  __syncthreads();
  if (tid == 0) {
    double A[4][4], X[4][4];
    int pv[4];
    for (int i = 0; i < 4; ++i)
      for (int k = 0; k < 4; ++k) A[i][k] = (i < pc && k < pc) ? gRc[i * 4 + k] : 0.0;
    pivoted_qr_reg<4>(A, pc, X, pv);
    double ysq = 0.0;
    for (int s = 0; s < pc; ++s) ysq += gYn[s];
    const double delta = 16.0 * DEPS * sqrt(ysq);
    for (int j = 0; j < 4; ++j)
      if (fabs(A[j][j]) <= delta || st->drop_all) {
        for (int k = 0; k < 4; ++k) { A[j][k] = 0.0; X[k][j] = 0.0; }
      }
    for (int i = 0; i < 16; ++i) sR[i] = 0.0;
    for (int j = 0; j < pc; ++j)
      for (int kk = 0; kk < pc; ++kk) sR[j * 4 + pv[kk]] = A[j][kk];
    // T = Rinv X  (q~ = y2 T)
    for (int i = 0; i < 4; ++i)
      for (int j = 0; j < 4; ++j) {
        double acc = 0.0;
        for (int k = 0; k < 4; ++k) acc += gRi[i * 4 + k] * X[k][j];
        sT[i * 4 + j] = (i < pc && j < pc) ? acc : 0.0;
      }
  }
  __syncthreads();
  const long long tf1 = a.dbg ? clock64() : 0;
  auto Kel = [&](int i, int j) -> double {
    if (i < r) return (j < r) ? (i == j ? gSig[i] : 0.0) : st->C[i * SF_P + (j - r)];
    return (j >= r) ? sR[(i - r) * 4 + (j - r)] : 0.0;
  };
  const int ldc = n;
  if (n <= 32) {
    for (int idx = tid; idx < n * n; idx += ST) {
      const int i = idx % n, j = idx / n;
      sCore[j + i * 33] = Kel(i, j);  // K^T: Jacobi on the rows of the core
    }
    __syncthreads();
    if (warp < 4) {
      if (n <= 8) multi_warp_jacobi<8, 4>(sCore, 33, n, Vc, Uc, ldc, sS, iPerm, sScr);
      else if (n <= 12) multi_warp_jacobi<12, 4>(sCore, 33, n, Vc, Uc, ldc, sS, iPerm, sScr);
      else if (n <= 16) multi_warp_jacobi<16, 4>(sCore, 33, n, Vc, Uc, ldc, sS, iPerm, sScr);
      else if (n <= 20) multi_warp_jacobi<20, 4>(sCore, 33, n, Vc, Uc, ldc, sS, iPerm, sScr);
      else if (n <= 24) multi_warp_jacobi<24, 4>(sCore, 33, n, Vc, Uc, ldc, sS, iPerm, sScr);
      else multi_warp_jacobi<32, 4>(sCore, 33, n, Vc, Uc, ldc, sS, iPerm, sScr);
    }
    __syncthreads();
  } else {
    for (int idx = tid; idx < n * n; idx += ST) {
      const int i = idx % n, j = idx / n;
      sCore[i + j * n] = Kel(i, j);
    }
    __syncthreads();
    jacobi_svd(sCore, n, Vj, n, n, sS, iPerm, sScr, iFlag, sScr + SF_N + 8);
    for (int idx = tid; idx < n * n; idx += ST) {
      const int i = idx % n, k = idx / n;
      const double sv = sS[k];
      Uc[i + k * ldc] = sv > 0.0 ? sCore[i + iPerm[k] * n] / sv : 0.0;
      Vc[i + k * ldc] = Vj[i + iPerm[k] * n];
    }
    __syncthreads();
  }
  const long long tf2 = a.dbg ? clock64() : 0;
  if (tid == 0) {
    double ysq = 0.0, ssq = 0.0;
    for (int s = 0; s < pc; ++s) ysq += gYn[s];
    for (int i = 0; i < r; ++i) ssq += gSig[i] * gSig[i];
    const double fs = sqrt((double)r + ysq) * sqrt(ssq + (double)pc);
    int rn = (sS[0] <= NOISE_FLOOR * fs) ? 0 : rank_cut_dev(sS, n, a.eps0, a.r_max);
    if (rn > a.cap) { rn = a.cap; a.info[2] = 2; }
    iFlag[0] = rn;
  }
  __syncthreads();
  const int rn = iFlag[0];
  const long long tf3 = a.dbg ? clock64() : 0;
  // W' = [Uc_top; T Uc_bot] (n x rn), kept in shared memory (reusing the core) for C1 / Wd
  double* sW = sCore;  // n x rn, ld n
  for (int idx = tid; idx < n * rn; idx += ST) {
    const int i = idx % n, c = idx / n;
    double w;
    if (i < r) {
      w = Uc[i + c * ldc];
    } else {
      w = 0.0;
      for (int q = 0; q < pc; ++q) w += sT[(i - r) * 4 + q] * Uc[r + q + c * ldc];
    }
    sW[i + c * n] = w;
    st->Wp[i + c * SF_LDW] = w;
    st->Vc[i + c * SF_LDW] = Vc[i + c * ldc];
  }
  for (int k = tid; k < rn; k += ST) st->sig[k] = sS[k];
  __syncthreads();
  // the flush being projected: C1 = W'^T M, Wd = -W' C1
  const int pcn = st->pc_new;
  double* sC1 = Uc;  // rn x 4
  for (int idx = tid; idx < rn * SF_P; idx += ST) {
    const int i = idx / SF_P, s2 = idx % SF_P;
    double acc = 0.0;
    if (s2 < pcn)
      for (int k = 0; k < n; ++k) acc += sW[k + i * n] * gM[k * SF_P + s2];
    sC1[idx] = acc;
    st->C[idx] = acc;
  }
  __syncthreads();
  for (int idx = tid; idx < n * SF_P; idx += ST) {
    const int k = idx / SF_P, s2 = idx % SF_P;
    double acc = 0.0;
    for (int i = 0; i < rn; ++i) acc += sW[k + i * n] * sC1[i * SF_P + s2];
    st->Wd[idx] = -acc;
  }
  if (tid < SF_P) st->yn[tid] = st->yn_next[tid];
  if (tid == 0) {
    st->rn = rn;
    st->startp = start;
    st->pending = 1;
    a.trace[f] = rn;
  }
  if (a.dbg && tid == 0) {
    long long* d = a.dbg + 24;
    d[0] += tf1 - tf0;
    d[1] += tf2 - tf1;
    d[2] += tf3 - tf2;
    d[3] += 1;
    d[4] += clock64() - tf3;
  }
}

// ---------------------------------------------------- pane all-gather (sharded)
// After a sharded sweep every rank holds its own row slab of the pane basis;
// the stages that follow (observation, extraction) run replicated on the full
// basis, so each rank pushes its slab into every peer's pane over NVLink and
// all ranks meet at a flag barrier (the same exchange slots, zero payload).
struct SFPanes {
  double* p[SF_XMAXR];
};
__global__ void __launch_bounds__(ST) sf_push_rows(const SFPanes panes, int nshard, int shard, int64_t ld,
                                                   int64_t x0, int64_t rows, const int* r_dev, int cap) {
  const int col = blockIdx.y;
  const int r = r_dev ? min(cap, *r_dev) : cap;
  if (col >= r) return;
  const double* src = panes.p[shard] + x0 + (int64_t)col * ld;
  for (int64_t i = (int64_t)blockIdx.x * ST + threadIdx.x; i < rows; i += (int64_t)gridDim.x * ST) {
    const double v = src[i];
    for (int q = 0; q < nshard; ++q)
      if (q != shard) panes.p[q][x0 + i + (int64_t)col * ld] = v;
  }
}
__global__ void __launch_bounds__(32) sf_barrier(const SFArgs a, unsigned long long seq) {
  __shared__ double dummy[1];
  xr_deposit(a, seq, dummy, 0);
  xr_collect(a, seq, 0, dummy);
}

cudaError_t sf_allgather_pane(const SFArgs& a, double* const* pane, int64_t ld, int64_t x0, int64_t rows,
                              int cap, cudaStream_t s, unsigned long long* xseq, int64_t* launches) {
  SFPanes P{};
  for (int q = 0; q < a.nshard; ++q) P.p[q] = pane[q];
  int gx = (int)std::min<int64_t>((rows + ST - 1) / ST, 1184);
  if (gx < 1) gx = 1;
  sf_push_rows<<<dim3(gx, cap), ST, 0, s>>>(P, a.nshard, a.shard, ld, x0, rows, a.info, cap);
  const unsigned long long seq = ++(*xseq);
  sf_barrier<<<1, 32, 0, s>>>(a, seq);
  if (launches) *launches += 2;
  return cudaGetLastError();
}

// ------------------------------------------------------------------ host side
size_t sf_smem_pass() { return 210 * 1024; }
size_t sf_smem_finish() {
  return (size_t)(16 + 16 + SF_N + 4 + 512 + 4 * (SF_N * SF_N + 8) + 2 * SF_N + 16) * sizeof(double);
}
int64_t sf_part_stride() { return PSTR; }

cudaError_t sf_configure() {
  static bool done[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev >= 0 && dev < 64 && done[dev]) return cudaSuccess;
  cudaError_t e = cudaFuncSetAttribute(sf_pass<0>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)sf_smem_pass());
  if (e != cudaSuccess) return e;
  e = cudaFuncSetAttribute(sf_pass<1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)sf_smem_pass());
  if (e != cudaSuccess) return e;
  e = cudaFuncSetAttribute(sf_finish, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)sf_smem_finish());
  if (e != cudaSuccess) return e;
  if (dev >= 0 && dev < 64) done[dev] = true;
  return cudaSuccess;
}

// The whole sweep: for f = 0..nflush: pass A(f) [closes f-1, projects f],
// CholeskyQR x 2 + finish of flush f-1 (with the generation of flush f+1 next
// to them on the aux stream), pass B(f) [update of f-1, first CGS pass of f].
// Sharded sweeps (nshard > 1) add a one-CTA tail kernel after every pass that
// ends in a rank total.  With several local shards (single-device emulation)
// every step is launched for all shards before the next step, on one stream.
cudaError_t launch_sweep_stream(const SFArgs* sh, int nlocal, int nflush, cudaStream_t s,
                                const SFAux& aux, unsigned long long* xseq, int64_t* launches) {
  cudaError_t e = sf_configure();
  if (e != cudaSuccess) return e;
  const SFArgs& a0 = sh[0];
  const int G = a0.G;
  const int Gg = a0.Ggen;
  const int Gc = 2 * (Gg / 8 > 0 ? Gg / 8 : 1);  // CholeskyQR passes: 2 CTAs per SM
  const size_t sp = a0.smem_pass, sfin = sf_smem_finish();
  const bool sharded = a0.nshard > 1;
  const bool use_aux = nlocal == 1 && aux.stream != nullptr;
  unsigned long long seq = xseq ? *xseq : 0ull;
  int64_t nl = 0;
  const int dbg = a0.dbg_print;
  auto show = [&](const char* what, int f) {
    if (f >= dbg) return;
    SFState* h = new SFState;
    cudaStreamSynchronize(s);
    cudaMemcpy(h, a0.st, sizeof(*h), cudaMemcpyDeviceToHost);
    std::fprintf(stderr, "[sf] f=%d %-8s r=%d rn=%d pcp=%d pcn=%d pend=%d drop=%d err=%s | yn %.3e %.3e | C00 %.6e C01 %.6e P2_00 %.3e M00 %.6e | sig %.6e %.6e | Rc %.4e %.4e %.4e %.4e\n",
                 f, what, h->r, h->rn, h->pcp, h->pc_new, h->pending, h->drop_all,
                 cudaGetErrorString(cudaGetLastError()), h->yn[0], h->yn[1], h->C[0], h->C[1],
                 h->P2[0], h->M[0], h->sig[0], h->sig[1], h->Rc[0], h->Rc[5], h->Rc[10], h->Rc[15]);
    delete h;
  };
  for (int g = 0; g < nlocal; ++g) sf_generate<<<Gg, ST, 0, s>>>(sh[g], 0);
  nl += nlocal;
  for (int f = 0; f <= nflush; ++f) {
    ++seq;
    for (int g = 0; g < nlocal; ++g) sf_pass<0><<<G, SPT, sp, s>>>(sh[g], f, seq);
    if (sharded)
      for (int g = 0; g < nlocal; ++g) sf_tail<0><<<1, ST, 0, s>>>(sh[g], f, seq);
    nl += nlocal * (sharded ? 2 : 1);
    show("passA", f);
    if (f > 0) {
      for (int pass = 0; pass < 2; ++pass) {
        ++seq;
        for (int g = 0; g < nlocal; ++g) sf_cholqr<<<Gc, ST, 0, s>>>(sh[g], f - 1, pass, seq);
        if (sharded)
          for (int g = 0; g < nlocal; ++g) sf_tail<2><<<1, ST, 0, s>>>(sh[g], f - 1, seq);
        nl += nlocal * (sharded ? 2 : 1);
      }
    }
    // flush f+1's columns (buffer (f+1) % 3, last read by pass B(f-1)) are
    // generated on the aux stream, next to the single-CTA sf_finish
    const bool gen = f + 1 < nflush;
    if (gen) {
      if (use_aux) {
        if ((e = cudaEventRecord(aux.ready, s)) != cudaSuccess) return e;
        if ((e = cudaStreamWaitEvent(aux.stream, aux.ready, 0)) != cudaSuccess) return e;
        sf_generate<<<Gg, ST, 0, aux.stream>>>(sh[0], f + 1);
        if ((e = cudaEventRecord(aux.done, aux.stream)) != cudaSuccess) return e;
      } else {
        for (int g = 0; g < nlocal; ++g) sf_generate<<<Gg, ST, 0, s>>>(sh[g], f + 1);
      }
      nl += nlocal;
    }
    if (f > 0) {
      for (int g = 0; g < nlocal; ++g) sf_finish<<<1, ST, sfin, s>>>(sh[g], f - 1);
      nl += nlocal;
      show("finish", f);
    }
    ++seq;
    for (int g = 0; g < nlocal; ++g) sf_pass<1><<<G, SPT, sp, s>>>(sh[g], f, seq);
    if (sharded)
      for (int g = 0; g < nlocal; ++g) sf_tail<1><<<1, ST, 0, s>>>(sh[g], f, seq);
    nl += nlocal * (sharded ? 2 : 1);
    show("passB", f);
    if (gen && use_aux && (e = cudaStreamWaitEvent(s, aux.done, 0)) != cudaSuccess) return e;
  }
  if (a0.dbg) {
    long long h[32];
    cudaStreamSynchronize(s);
    cudaMemcpy(h, a0.dbg, sizeof(h), cudaMemcpyDeviceToHost);
    if (h[16 + 3] > 0)
      std::fprintf(stderr, "[sf timing] cholqr last CTA, mean cycles over %lld launches: main loop %lld, election %lld, reduce %lld, tail %lld\n",
                   h[19], h[20] / h[19], h[16] / h[19], h[17] / h[19], h[18] / h[19]);
    if (h[24 + 3] > 0)
      std::fprintf(stderr, "[sf timing] finish, mean cycles over %lld launches: fix-up (thread 0) %lld, core SVD %lld, rank cut (thread 0) %lld, update matrices %lld\n",
                   h[27], h[24] / h[27], h[25] / h[27], h[26] / h[27], h[28] / h[27]);
    for (int m = 0; m < 2; ++m)
      if (h[8 * m + 3] > 0)
        std::fprintf(stderr, "[sf timing] pass %c last CTA, mean cycles over %lld launches: main loop %lld, election %lld, reduce %lld, tail %lld\n",
                     m ? 'B' : 'A', h[8 * m + 3], h[8 * m + 4] / h[8 * m + 3], h[8 * m] / h[8 * m + 3],
                     h[8 * m + 1] / h[8 * m + 3], h[8 * m + 2] / h[8 * m + 3]);
  }
  if (xseq) *xseq = seq;
  if (launches) *launches += nl;
  return cudaGetLastError();
}

}  // namespace lrk
