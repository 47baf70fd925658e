// lrk_device.cuh — device building blocks shared by the persistent kernels.
//
// Everything here runs inside cooperative kernels whose CTAs form "groups":
// a group of `ncta` CTAs owns one problem (one sweep / one truncation) and
// synchronises with a software grid barrier.  Rows of every tall factor
// (n_x or n_t rows) are split into contiguous per-CTA ranges, so all
// "row-local" work needs no synchronisation; only small r x p partial sums
// cross CTAs, through L2 (ld.global.cg), reduced in a fixed order so every CTA
// of a group sees bit-identical results and takes identical control flow.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace lrk {

constexpr int NT = 256;            // threads per CTA of the persistent kernels
constexpr int NWARP = NT / 32;
constexpr int PMAX = 16;           // max columns appended per block (compress_every)
constexpr int JMAX_SMEM = 80;      // Jacobi SVD kept in SMEM up to this order
constexpr int NMAX = 160;          // absolute max order of a core matrix
constexpr double DEPS = 2.220446049250313e-16;
constexpr double NOISE_FLOOR = 1e-15;   // lowrank.py:20-22

// ------------------------------------------------------------------ barrier
// Sense-free generation barrier for the `ncta` CTAs of one group.
// bar[0] = arrival count, bar[1] = generation.  PTX memory-model form: the
// arrival is one acq_rel atomic (it releases the CTA's writes, cumulative
// through the preceding bar.sync, and acquires the earlier arrivals'), the
// last arriver resets the count and publishes the new generation with a
// release store, the others poll it with acquire loads; no separate fences.
// sys selects .sys scope (peer GPUs of a sharded sweep), else .gpu.
__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned* p, bool sys) {
  unsigned v;
  if (sys) asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  else asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned ld_relaxed_u32(const unsigned* p, bool sys) {
  unsigned v;
  if (sys) asm volatile("ld.relaxed.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  else asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned atom_add_acq_rel_u32(unsigned* p, unsigned x, bool sys) {
  unsigned v;
  if (sys) asm volatile("atom.acq_rel.sys.global.add.u32 %0, [%1], %2;" : "=r"(v) : "l"(p), "r"(x) : "memory");
  else asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], %2;" : "=r"(v) : "l"(p), "r"(x) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed_u32(unsigned* p, unsigned x, bool sys) {
  if (sys) asm volatile("st.relaxed.sys.global.u32 [%0], %1;" ::"l"(p), "r"(x) : "memory");
  else asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(x) : "memory");
}
__device__ __forceinline__ void st_release_u32(unsigned* p, unsigned x, bool sys) {
  if (sys) asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(x) : "memory");
  else asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(x) : "memory");
}

// Split form for a barrier whose arrival and wait happen at different points
// (one thread each, after the arriving threads have synced): arrive returns
// the generation to wait on.
__device__ __forceinline__ unsigned group_arrive(unsigned* bar, int ncta, bool sys) {
  const unsigned gen = ld_relaxed_u32(bar + 1, sys);
  const unsigned arrived = atom_add_acq_rel_u32(bar, 1u, sys);
  if (arrived == (unsigned)ncta - 1u) {
    st_relaxed_u32(bar, 0u, sys);
    st_release_u32(bar + 1, gen + 1u, sys);
  }
  return gen;
}
__device__ __forceinline__ void group_wait(unsigned* bar, unsigned gen, bool sys) {
  while (ld_acquire_u32(bar + 1, sys) == gen) {
  }
}

__device__ __forceinline__ void group_barrier(unsigned* bar, int ncta, bool sys = false) {
  __syncthreads();
  if (threadIdx.x == 0) group_wait(bar, group_arrive(bar, ncta, sys), sys);
  __syncthreads();
}

// Per-CTA partial buffers of a (possibly sharded) sweep: region k (0..2) of
// global CTA c lives at p[c / ncta] + (k * ncta + c % ncta) * stride.
struct PartTab {
  double* const* p;
  int ncta;        // CTAs per shard
  int nshard;
  int64_t stride;
  __device__ __forceinline__ const double* at(int k, int c) const {
    if (nshard <= 1) return p[0] + ((int64_t)k * ncta + c) * stride;
    const int s = c / ncta, l = c - s * ncta;
    return p[s] + ((int64_t)k * ncta + l) * stride;
  }
};

// ------------------------------------------------ fast fp64 special functions
// The library sqrt / rsqrt / division of fp64 cost ~75-210 cycles of
// dependent latency on sm_100a (tools/lat_bench.cu); the MUFU seeds plus
// Newton steps below cost ~40-50 and are accurate to the last bit or two in
// the normal range (no denormal / inf handling: callers keep operands normal).
// out-of-range fallbacks: one out-of-line copy each (keeps callers compact)
static __device__ __noinline__ double rcp_slow(double x) { return 1.0 / x; }
static __device__ __noinline__ double rsqrt_slow(double x) { return rsqrt(x); }
static __device__ __noinline__ double sqrt_slow(double x) { return sqrt(x); }
__device__ __forceinline__ double rcp_fast(double x) {
  const double ax = fabs(x);
  if (!(ax > 1e-300 && ax < 1e300)) return rcp_slow(x);  // denormal / huge / 0 / inf / nan
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  double e = fma(-x, r, 1.0);
  r = fma(r, e, r);
  e = fma(-x, r, 1.0);
  return fma(r, e, r);
}
__device__ __forceinline__ double rsqrt_fast(double x) {
  if (!(x > 1e-300 && x < 1e300)) return rsqrt_slow(x);
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  const double hx = 0.5 * x;
  y = y * fma(-hx * y, y, 1.5);
  y = y * fma(-hx * y, y, 1.5);
  return y;
}
// sqrt(x), x >= 0
__device__ __forceinline__ double sqrt_fast(double x) {
  if (!(x > 1e-300 && x < 1e300)) return sqrt_slow(x);
  return x * rsqrt_fast(x);
}
// Unchecked (branch-free) variants for operands known to be normal and in
// range (e.g. after an exact power-of-two rescale): no slow-path branch, so
// unrolled independent calls overlap instead of serialising at each branch.
__device__ __forceinline__ double rcp_u(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  double e = fma(-x, r, 1.0);
  r = fma(r, e, r);
  e = fma(-x, r, 1.0);
  return fma(r, e, r);
}
__device__ __forceinline__ double rsqrt_u(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  const double hx = 0.5 * x;
  y = y * fma(-hx * y, y, 1.5);
  y = y * fma(-hx * y, y, 1.5);
  return y;
}
// sqrt for x >= 0 in range or exactly 0
__device__ __forceinline__ double sqrt_u(double x) {
  const double r = x * rsqrt_u(x);
  return x > 0.0 ? r : 0.0;
}
// 2^e exactly (|e| < 1023)
__device__ __forceinline__ double pow2i(int e) { return __longlong_as_double((long long)(e + 1023) << 52); }
// floor(log2(x)) for a normal positive x
__device__ __forceinline__ int ilog2_normal(double x) {
  return (int)((__double_as_longlong(x) >> 52) & 0x7ff) - 1023;
}

// FP64 tensor-core MMA (sm_100a has no tcgen05 f64 kind; this is SASS DMMA):
// D(8x8) += A(8x4, row) * B(4x8, col).  Fragments: a = A[g][t], b = B[t][g],
// d0,d1 = D[g][2t], D[g][2t+1] with g = lane>>2, t = lane&3.  Not volatile:
// the scheduler may interleave it with the loads feeding the next step.
__device__ __forceinline__ void dmma884(double& d0, double& d1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(d0), "+d"(d1)
      : "d"(a), "d"(b));
}

// ------------------------------------------------------------- reductions
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Sum K per-thread values over the whole CTA; every thread gets the sums in
// out[0..K).  red must hold NWARP*K doubles; fixed order -> deterministic.
template <int K>
__device__ __forceinline__ void block_sum(double (&v)[K], double* red, double* out) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
  for (int i = 0; i < K; ++i) v[i] = warp_sum(v[i]);
  if (lane == 0) {
#pragma unroll
    for (int i = 0; i < K; ++i) red[w * K + i] = v[i];
  }
  __syncthreads();
  if (threadIdx.x < K) {
    double s = 0.0;
    for (int ww = 0; ww < NWARP; ++ww) s += red[ww * K + threadIdx.x];
    out[threadIdx.x] = s;
  }
  __syncthreads();
#pragma unroll
  for (int i = 0; i < K; ++i) v[i] = out[i];
  __syncthreads();
}

// Reduce per-CTA partials written by the ncta CTAs of a group:
// out[o] = sum_c part[c*stride + o], o < len.  Reads through L2 (.cg) because
// other SMs wrote the data.  Every CTA computes the same sums in the same
// order.  out is shared memory.
__device__ __forceinline__ void reduce_partials(const double* part, int64_t stride, int ncta,
                                       int len, double* out) {
  int lp = 1;
  while (lp < 32 && lp * 2 * len <= NT) lp *= 2;  // keeps lp * len <= NT
  const int tid = threadIdx.x;
  if (lp > 1) {
    const int o = tid / lp, sub = tid % lp;
    double acc = 0.0;
    if (o < len) {
      // issue a batch of independent L2 loads before summing (latency-bound)
      constexpr int B = 16;
      for (int c0 = sub; c0 < ncta; c0 += B * lp) {
        double v[B];
#pragma unroll
        for (int u = 0; u < B; ++u) {
          const int c = c0 + u * lp;
          v[u] = (c < ncta) ? __ldcg(part + (int64_t)c * stride + o) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < B; ++u) acc += v[u];
      }
    }
    for (int m = lp >> 1; m > 0; m >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, m);
    if (o < len && sub == 0) out[o] = acc;
  } else {
    for (int o = tid; o < len; o += NT) {
      double acc = 0.0;
      for (int c = 0; c < ncta; ++c) acc += __ldcg(part + (int64_t)c * stride + o);
      out[o] = acc;
    }
  }
  __syncthreads();
}

// Same reduction over the partials of every CTA of a sharded sweep (fixed
// order over global CTA ids, so every CTA of every shard gets identical sums).
__device__ __forceinline__ void reduce_partials(const PartTab& t, int k, int ncta_all, int len,
                                                double* out) {
  if (t.nshard <= 1) {
    reduce_partials(t.at(k, 0), t.stride, ncta_all, len, out);
    return;
  }
  int lp = 1;
  while (lp < 32 && lp * 2 * len <= NT) lp *= 2;
  const int tid = threadIdx.x;
  if (lp > 1) {
    const int o = tid / lp, sub = tid % lp;
    double acc = 0.0;
    if (o < len) {
      constexpr int B = 16;
      for (int c0 = sub; c0 < ncta_all; c0 += B * lp) {
        double v[B];
#pragma unroll
        for (int u = 0; u < B; ++u) {
          const int c = c0 + u * lp;
          v[u] = (c < ncta_all) ? __ldcg(t.at(k, c) + o) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < B; ++u) acc += v[u];
      }
    }
    for (int m = lp >> 1; m > 0; m >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, m);
    if (o < len && sub == 0) out[o] = acc;
  } else {
    for (int o = tid; o < len; o += NT) {
      double acc = 0.0;
      for (int c = 0; c < ncta_all; ++c) acc += __ldcg(t.at(k, c) + o);
      out[o] = acc;
    }
  }
  __syncthreads();
}

// CTA-partial of A^T B over `nrows` rows: out[i*nb + j] = sum_t A[t + i*lda] *
// B[t + j*ldb].  scratch: NT doubles of shared memory; out: shared.
__device__ __forceinline__ void cta_tn(const double* A, int64_t lda, int na, const double* B,
                              int64_t ldb, int nb, int nrows, double* out, double* scratch) {
  const int nout = na * nb;
  const int tid = threadIdx.x;
  if (nout == 0) return;
  if (nout <= NT) {
    const int nslice = NT / nout;
    const int o = tid % nout, s = tid / nout;
    double acc = 0.0;
    if (s < nslice) {
      const int i = o / nb, j = o % nb;
      const double* a = A + (int64_t)i * lda;
      const double* b = B + (int64_t)j * ldb;
      double a0 = 0, a1 = 0, a2 = 0, a3 = 0;
      int t = s;
      for (; t + 3 * nslice < nrows; t += 4 * nslice) {
        a0 += a[t] * b[t];
        a1 += a[t + nslice] * b[t + nslice];
        a2 += a[t + 2 * nslice] * b[t + 2 * nslice];
        a3 += a[t + 3 * nslice] * b[t + 3 * nslice];
      }
      for (; t < nrows; t += nslice) a0 += a[t] * b[t];
      acc = (a0 + a1) + (a2 + a3);
    }
    if (s < nslice) scratch[s * nout + o] = acc;
    __syncthreads();
    if (tid < nout) {
      double v = 0.0;
      for (int q = 0; q < nslice; ++q) v += scratch[q * nout + tid];
      out[tid] = v;
    }
    __syncthreads();
  } else {
    for (int o = tid; o < nout; o += NT) {
      const int i = o / nb, j = o % nb;
      const double* a = A + (int64_t)i * lda;
      const double* b = B + (int64_t)j * ldb;
      double acc = 0.0;
      for (int t = 0; t < nrows; ++t) acc += a[t] * b[t];
      out[o] = acc;
    }
    __syncthreads();
  }
}

// Row-local update X[:, 0..nx) -= A[:, 0..na) * Cm, Cm is na x nx row-major
// in shared memory (Cm[i*nx + j]).
__device__ inline void rows_sub_gemm(double* X, int64_t ldx, int nx, const double* A,
                                     int64_t lda, int na, const double* Cm, int nrows) {
  for (int t = threadIdx.x; t < nrows; t += NT) {
    double acc[PMAX];
#pragma unroll
    for (int j = 0; j < PMAX; ++j) acc[j] = 0.0;
    for (int i = 0; i < na; ++i) {
      const double a = A[t + (int64_t)i * lda];
#pragma unroll
      for (int j = 0; j < PMAX; ++j)
        if (j < nx) acc[j] += a * Cm[i * nx + j];
    }
#pragma unroll
    for (int j = 0; j < PMAX; ++j)
      if (j < nx) X[t + (int64_t)j * ldx] -= acc[j];
  }
}

// ------------------------------------------------- block Householder QR
// In-place Householder QR of the CTA-local block X (m x q, col-major, ldx),
// q <= PMAX.  Reflector vectors overwrite X below the diagonal (unit leading
// entry implicit), tau[j] saved; R (q x q, row-major, zero-padded when m < q)
// is written to Rout.  red: NWARP*PMAX doubles, tmp: PMAX doubles (shared).
__device__ inline void block_householder_qr(double* X, int64_t ldx, int m, int q,
                                            double* tau, double* Rout, double* red,
                                            double* tmp) {
  const int tid = threadIdx.x;
  for (int i = tid; i < q * q; i += NT) Rout[i] = 0.0;
  __syncthreads();
  const int kmax = m < q ? m : q;
  for (int j = 0; j < kmax; ++j) {
    double v1[1];
    {
      double s = 0.0;
      for (int i = j + 1 + tid; i < m; i += NT) {
        double x = X[i + (int64_t)j * ldx];
        s += x * x;
      }
      v1[0] = s;
    }
    block_sum<1>(v1, red, tmp);
    const double sig = v1[0];
    const double alpha = X[j + (int64_t)j * ldx];
    double beta, t, scale;
    if (sig == 0.0) {
      t = 0.0; beta = alpha; scale = 0.0;
    } else {
      double nrm = sqrt(alpha * alpha + sig);
      beta = alpha >= 0.0 ? -nrm : nrm;
      t = (beta - alpha) / beta;
      scale = 1.0 / (alpha - beta);
    }
    __syncthreads();  // everyone has read alpha before row j changes
    if (tid == 0) tau[j] = t;
    // v_i = X[i,j]*scale for i>j (stored in place)
    for (int i = j + 1 + tid; i < m; i += NT) X[i + (int64_t)j * ldx] *= scale;
    __syncthreads();
    // w_k = x_jk + sum_{i>j} v_i x_ik for k in (j, q)
    double w[PMAX];
#pragma unroll
    for (int k = 0; k < PMAX; ++k) w[k] = 0.0;
    for (int i = j + 1 + tid; i < m; i += NT) {
      const double vi = X[i + (int64_t)j * ldx];
#pragma unroll
      for (int k = 0; k < PMAX; ++k)
        if (k > j && k < q) w[k] += vi * X[i + (int64_t)k * ldx];
    }
    block_sum<PMAX>(w, red, tmp);
    // apply: x_ik -= tau * v_i * w_k (row j: v_j = 1)
    for (int k = j + 1; k < q; ++k) {
      const double wk = w[k] + X[j + (int64_t)k * ldx];
      const double f = t * wk;
      for (int i = j + 1 + tid; i < m; i += NT) X[i + (int64_t)k * ldx] -= f * X[i + (int64_t)j * ldx];
      __syncthreads();
      if (tid == 0) {
        X[j + (int64_t)k * ldx] -= f;
        Rout[j * q + k] = X[j + (int64_t)k * ldx];
      }
    }
    if (tid == 0) { Rout[j * q + j] = beta; X[j + (int64_t)j * ldx] = beta; }
    __syncthreads();
  }
  for (int j = kmax + tid; j < q; j += NT) tau[j] = 0.0;
  __syncthreads();
}

// Y (m x q) = H_0 H_1 ... H_{kmax-1} [G; 0], G (q x q row-major, shared),
// reflectors from block_householder_qr stored in X.  Y is written fresh.
__device__ inline void block_householder_apply_q(const double* X, int64_t ldx, int m, int q,
                                                 const double* tau, const double* G,
                                                 double* Y, int64_t ldy, double* red,
                                                 double* tmp) {
  const int tid = threadIdx.x;
  for (int c = 0; c < q; ++c)
    for (int i = tid; i < m; i += NT) Y[i + (int64_t)c * ldy] = (i < q) ? G[i * q + c] : 0.0;
  __syncthreads();
  const int kmax = m < q ? m : q;
  for (int j = kmax - 1; j >= 0; --j) {
    const double t = tau[j];
    if (t == 0.0) continue;  // uniform across the CTA
    double w[PMAX];
#pragma unroll
    for (int c = 0; c < PMAX; ++c) w[c] = 0.0;
    for (int i = j + 1 + tid; i < m; i += NT) {
      const double vi = X[i + (int64_t)j * ldx];
#pragma unroll
      for (int c = 0; c < PMAX; ++c)
        if (c < q) w[c] += vi * Y[i + (int64_t)c * ldy];
    }
    block_sum<PMAX>(w, red, tmp);
    for (int c = 0; c < q; ++c) {
      const double f = t * (w[c] + Y[j + (int64_t)c * ldy]);
      for (int i = j + 1 + tid; i < m; i += NT) Y[i + (int64_t)c * ldy] -= f * X[i + (int64_t)j * ldx];
      __syncthreads();
      if (tid == 0) Y[j + (int64_t)c * ldy] -= f;
    }
    __syncthreads();
  }
}

// ------------------------------------------------ small dense helpers
// Single-thread column-pivoted Householder QR of a q x q matrix A (row-major,
// in place): A*P = X*Rt.  Writes X (q x q row-major, orthogonal), Rt (upper,
// row-major, in A) and perm (Rt column k corresponds to A column perm[k]).
__device__ __forceinline__ void small_pivoted_qr(double* A, int q, double* X, int* perm, double* cn) {
  for (int k = 0; k < q; ++k) {
    perm[k] = k;
    double s = 0;
    for (int i = 0; i < q; ++i) s += A[i * q + k] * A[i * q + k];
    cn[k] = s;
  }
  for (int i = 0; i < q * q; ++i) X[i] = (i / q == i % q) ? 1.0 : 0.0;
  for (int j = 0; j < q; ++j) {
    // pivot: largest remaining column norm (recomputed exactly)
    int best = j; double bv = -1.0;
    for (int k = j; k < q; ++k) {
      double s = 0;
      for (int i = j; i < q; ++i) s += A[i * q + k] * A[i * q + k];
      cn[k] = s;
      if (s > bv) { bv = s; best = k; }
    }
    if (best != j) {
      for (int i = 0; i < q; ++i) { double t = A[i * q + j]; A[i * q + j] = A[i * q + best]; A[i * q + best] = t; }
      int t = perm[j]; perm[j] = perm[best]; perm[best] = t;
    }
    double sig = 0;
    for (int i = j + 1; i < q; ++i) sig += A[i * q + j] * A[i * q + j];
    if (sig == 0.0) continue;
    double alpha = A[j * q + j];
    double nrm = sqrt(alpha * alpha + sig);
    double beta = alpha >= 0 ? -nrm : nrm;
    double tau = (beta - alpha) / beta;
    double sc = 1.0 / (alpha - beta);
    double v[PMAX];
    v[j] = 1.0;
    for (int i = j + 1; i < q; ++i) v[i] = A[i * q + j] * sc;
    // A <- H A on columns j..q-1
    for (int k = j; k < q; ++k) {
      double w = 0;
      for (int i = j; i < q; ++i) w += v[i] * A[i * q + k];
      w *= tau;
      for (int i = j; i < q; ++i) A[i * q + k] -= w * v[i];
    }
    // X <- X H (accumulate Q = H_0 H_1 ...)
    for (int i = 0; i < q; ++i) {
      double w = 0;
      for (int l = j; l < q; ++l) w += X[i * q + l] * v[l];
      w *= tau;
      for (int l = j; l < q; ++l) X[i * q + l] -= w * v[l];
    }
    for (int i = j + 1; i < q; ++i) A[i * q + j] = 0.0;
  }
}

// _rank_cut (lowrank.py:98-111) on descending s[0..n); single thread.
// tail[r] = sqrt(sum_{i>=r} s_i^2) accumulated from the end (as np.cumsum on
// the reversed array); keep = smallest r with tail[r] <= eps0*tail[0].  Two
// backward passes with the same summation order (no local-memory array):
// the first gives tail[0], the second walks the suffix {r : tail[r] <= thr}.
__device__ __forceinline__ int rank_cut_dev(const double* s, int n, double eps0, int r_max) {
  if (n == 0 || !(s[0] > 0.0)) return 0;
  const double floor_v = NOISE_FLOOR * s[0];
  double acc = 0.0;
  int nnz = 0;
#pragma unroll 8
  for (int i = n - 1; i >= 0; --i) {
    const double si = s[i] < floor_v ? 0.0 : s[i];
    nnz += si != 0.0;
    acc += si * si;
  }
  const double thr = eps0 * sqrt(acc);
  int keep = 0;  // searchsorted(-tail, -thr, 'left') over indices 0..n-1
  acc = 0.0;
  // sqrt(acc) > thr decided on squares; the IEEE sqrt only inside a guard
  // band around thr^2 (keeps the exact decision, no sqrt latency per step)
  const double thr2 = thr * thr, hi2 = thr2 * (1.0 + 1e-13), lo2 = thr2 * (1.0 - 1e-13);
  for (int i = n - 1; i >= 0; --i) {
    const double si = s[i] < floor_v ? 0.0 : s[i];
    acc += si * si;
    if (acc > hi2 || (acc >= lo2 && sqrt(acc) > thr)) { keep = i + 1; break; }
  }
  if (keep > nnz) keep = nnz;
  if (r_max >= 0 && keep > r_max) keep = r_max;
  return keep;
}

// rank_cut_dev on one warp for n <= 32 (lane i holds s[i]): the total by a
// warp tree sum and the tails by a suffix scan instead of two dependent
// serial loops; the tail-vs-threshold decision keeps the guard band with an
// IEEE sqrt inside it.  (Summation order differs from the serial loop at the
// rounding level only; the reference's own numpy sums are pairwise.)
__device__ __forceinline__ int rank_cut_warp(const double* s, int n, double eps0, int r_max) {
  const int lane = threadIdx.x & 31;
  const unsigned full = 0xffffffffu;
  const double s0 = s[0];
  if (n == 0 || !(s0 > 0.0)) return 0;
  const double floor_v = NOISE_FLOOR * s0;
  const double v = lane < n ? s[lane] : 0.0;
  const double si = v < floor_v ? 0.0 : v;
  const int nnz = __popc(__ballot_sync(full, si != 0.0));
  const double sq = si * si;
  const double total = warp_sum(sq);
  const double thr = eps0 * sqrt(total);
  const double thr2 = thr * thr, hi2 = thr2 * (1.0 + 1e-13), lo2 = thr2 * (1.0 - 1e-13);
  // inclusive suffix sum: tail[i] = sum_{j >= i} sq[j]
  double tail = sq;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const double t = __shfl_down_sync(full, tail, o);
    if (lane + o < 32) tail += t;
  }
  const bool over = lane < n && (tail > hi2 || (tail >= lo2 && sqrt(tail) > thr));
  const unsigned m = __ballot_sync(full, over);
  int keep = m ? (32 - __clz(m)) : 0;  // largest i with tail_i > thr, plus one
  if (keep > nnz) keep = nnz;
  if (r_max >= 0 && keep > r_max) keep = r_max;
  return keep;
}

// --------------------------------------------------- one-sided Jacobi SVD
// SVD of the n x n matrix held in A (col-major, lda) by cyclic one-sided
// (Hestenes) Jacobi with a round-robin parallel ordering; one warp per
// column pair.  On exit: V (col-major, ldv) holds right singular vectors
// (unsorted), columns of A hold U*diag(s) (unsorted), s_sorted[k] the k-th
// largest singular value, perm[k] its column.  nrm: n doubles, flag: 1 int
// (all shared).
__device__ inline int jacobi_svd(double* A, int lda, double* V, int ldv, int n,
                                 double* s_sorted, int* perm, double* nrm, int* flag,
                                 double* fro) {
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  int nsweep = 0;
  // columns below 1e-16 ||M||_F are rounding noise (far under the 1e-15
  // noise floor of _rank_cut): rotating them never converges and cannot
  // change any retained singular triplet, so such pairs are skipped
  if (w == 0) {
    double s = 0.0;
    for (int idx = lane; idx < n * n; idx += 32) {
      const double x = A[(idx % n) + (idx / n) * lda];
      s += x * x;
    }
    s = warp_sum(s);
    if (lane == 0) *fro = s * 1e-32;
  }
  for (int idx = tid; idx < n * n; idx += NT) {
    int i = idx % n, j = idx / n;
    V[i + j * ldv] = (i == j) ? 1.0 : 0.0;
  }
  __syncthreads();
  const int ne = n + (n & 1);
  // rotate only when the cosine between two columns exceeds the rounding
  // floor of an n-term dot product (a tighter test never terminates)
  const double tol = 2.0 * DEPS * (double)(n > 8 ? n : 8);
  for (int sweep = 0; sweep < 40 && n > 1; ++sweep) {
    // exact column norms
    for (int c = w; c < n; c += NWARP) {
      double s = 0.0;
      for (int i = lane; i < n; i += 32) { double a = A[i + c * lda]; s += a * a; }
      s = warp_sum(s);
      if (lane == 0) nrm[c] = s;
    }
    if (tid == 0) *flag = 0;
    __syncthreads();
    for (int rnd = 0; rnd < ne - 1; ++rnd) {
      for (int k = w; k < ne / 2; k += NWARP) {
        int i, j;
        if (k == 0) { i = ne - 1; j = rnd; }
        else { i = (rnd + k) % (ne - 1); j = (rnd - k + ne - 1) % (ne - 1); }
        if (i >= n || j >= n) continue;
        if (i > j) { int t = i; i = j; j = t; }
        const double al = nrm[i], be = nrm[j];
        double g = 0.0;
        for (int l = lane; l < n; l += 32) g += A[l + i * lda] * A[l + j * lda];
        g = warp_sum(g);
        if (!(al > *fro) || !(be > *fro)) continue;
        if (fabs(g) <= tol * sqrt(al) * sqrt(be)) continue;
        const double zeta = (be - al) / (2.0 * g);
        double t;
        if (fabs(zeta) > 1e150) t = 0.5 / zeta;
        else t = (zeta >= 0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
        const double c = 1.0 / sqrt(1.0 + t * t), s = c * t;
        for (int l = lane; l < n; l += 32) {
          const double ai = A[l + i * lda], aj = A[l + j * lda];
          A[l + i * lda] = c * ai - s * aj;
          A[l + j * lda] = s * ai + c * aj;
          const double vi = V[l + i * ldv], vj = V[l + j * ldv];
          V[l + i * ldv] = c * vi - s * vj;
          V[l + j * ldv] = s * vi + c * vj;
        }
        if (lane == 0) {
          nrm[i] = al - t * g;
          nrm[j] = be + t * g;
          *flag = 1;
        }
      }
      __syncthreads();
    }
    ++nsweep;
    if (*flag == 0) break;
    __syncthreads();
  }
  // final exact norms -> singular values
  for (int c = w; c < n; c += NWARP) {
    double s = 0.0;
    for (int i = lane; i < n; i += 32) { double a = A[i + c * lda]; s += a * a; }
    s = warp_sum(s);
    if (lane == 0) nrm[c] = sqrt(s);
  }
  __syncthreads();
  // stable descending order (ties by index)
  for (int i = tid; i < n; i += NT) {
    const double si = nrm[i];
    int rk = 0;
    for (int j = 0; j < n; ++j) {
      const double sj = nrm[j];
      if (sj > si || (sj == si && j < i)) ++rk;
    }
    perm[rk] = i;
    s_sorted[rk] = si;
  }
  __syncthreads();
  return nsweep;
}

// ------------------------------------------- single-warp Jacobi (n <= 32)
// One-sided Jacobi executed by ONE warp with no CTA barrier: lane j owns
// column j of the matrix and of the accumulated rotations.  Columns live in
// two shared-memory ping-pong copies (A0/A1, V0/V1; leading dimension ld,
// odd so the 32 lanes hit distinct banks); each round a lane reads its own
// and its partner's column from the current copy and writes its rotated
// column to the other, so the only synchronisation is __syncwarp().
// Round-robin pairing: lanes a, b with a + b = 2*rnd (mod ne-1), lane ne-1
// paired with rnd.  On exit: Uo[:, k] (ld ldo) = k-th left singular vector,
// Vo[:, k] = right singular vector, s_sorted[k] descending, perm[k] source
// column.  A0 holds the input on entry.  Returns the number of sweeps.
__device__ inline int warp_jacobi_svd(double* A0, double* A1, double* V0, double* V1, int ld,
                                      int n, double* Uo, double* Vo, int ldo, double* s_sorted,
                                      int* perm) {
  const int lane = threadIdx.x & 31;
  const unsigned full = 0xffffffffu;
  const bool own = lane < n;
  if (own)
    for (int i = 0; i < n; ++i) V0[i + lane * ld] = (i == lane) ? 1.0 : 0.0;
  double nrm = 0.0;
  if (own)
    for (int i = 0; i < n; ++i) { const double x = A0[i + lane * ld]; nrm += x * x; }
  const double tiny = warp_sum(nrm) * 1e-32;  // (1e-16 ||M||_F)^2, see jacobi_svd
  const double tol = 2.0 * DEPS * (double)(n > 8 ? n : 8);
  const int ne = n + (n & 1);
  double *Ac = A0, *An = A1, *Vc = V0, *Vn = V1;
  int nsweep = 0;
  __syncwarp();
  for (int sweep = 0; sweep < 40 && n > 1; ++sweep) {
    bool rotated = false;
    if (own) {
      nrm = 0.0;
      for (int i = 0; i < n; ++i) { const double x = Ac[i + lane * ld]; nrm += x * x; }
    }
    for (int rnd = 0; rnd < ne - 1; ++rnd) {
      int p;
      if (lane == ne - 1) p = rnd;
      else if (lane == rnd) p = ne - 1;
      else { p = 2 * rnd - lane; p %= (ne - 1); if (p < 0) p += ne - 1; }
      const double np = __shfl_sync(full, nrm, p & 31);
      const bool act = own && p < n;
      double c = 1.0, s = 0.0, t = 0.0, g = 0.0;
      bool rot = false;
      const bool lo = lane < p;
      const double al = lo ? nrm : np, be = lo ? np : nrm;
      if (act) {
        const double* me = Ac + lane * ld;
        const double* pa = Ac + p * ld;
        for (int i = 0; i < n; ++i) g += me[i] * pa[i];
        if (al > tiny && be > tiny && fabs(g) > tol * sqrt(al * be)) {
          const double d = be - al;
          t = 2.0 * g / (fabs(d) + sqrt(d * d + 4.0 * g * g));
          if (d < 0.0) t = -t;
          c = rsqrt(1.0 + t * t);
          s = c * t;
          rot = true;
        }
      }
      if (own) {
        const double* me = Ac + lane * ld;
        const double* pa = Ac + (act ? p : lane) * ld;
        const double* vm = Vc + lane * ld;
        const double* vp = Vc + (act ? p : lane) * ld;
        double* mo = An + lane * ld;
        double* vo = Vn + lane * ld;
        if (!rot) {
          for (int i = 0; i < n; ++i) { mo[i] = me[i]; vo[i] = vm[i]; }
        } else if (lo) {  // I am column i: a_i' = c a_i - s a_j
          for (int i = 0; i < n; ++i) { mo[i] = c * me[i] - s * pa[i]; vo[i] = c * vm[i] - s * vp[i]; }
          nrm = al - t * g;
        } else {          // I am column j: a_j' = s a_i + c a_j
          for (int i = 0; i < n; ++i) { mo[i] = s * pa[i] + c * me[i]; vo[i] = s * vp[i] + c * vm[i]; }
          nrm = be + t * g;
        }
      }
      rotated |= rot;
      { double* tp = Ac; Ac = An; An = tp; }
      { double* tp = Vc; Vc = Vn; Vn = tp; }
      __syncwarp();
    }
    ++nsweep;
    if (!__any_sync(full, rotated)) break;
  }
  // singular values, stable descending order, normalised outputs
  double sv = 0.0;
  if (own) {
    for (int i = 0; i < n; ++i) { const double x = Ac[i + lane * ld]; sv += x * x; }
    sv = sqrt(sv);
  }
  int rk = 0;
  for (int j = 0; j < n; ++j) {
    const double sj = __shfl_sync(full, sv, j);
    if (sj > sv || (sj == sv && j < lane)) ++rk;
  }
  if (own) {
    perm[rk] = lane;
    s_sorted[rk] = sv;
    const double inv = sv > 0.0 ? 1.0 / sv : 0.0;
    for (int i = 0; i < n; ++i) {
      Uo[i + rk * ldo] = Ac[i + lane * ld] * inv;
      Vo[i + rk * ldo] = Vc[i + lane * ld];
    }
  }
  __syncwarp();
  return nsweep;
}

// Row range owned by CTA `cta` of `ncta` over `n` rows.
__device__ __forceinline__ void row_range(int64_t n, int cta, int ncta, int64_t& r0, int64_t& r1) {
  const int64_t per = (n + ncta - 1) / ncta;
  r0 = per * cta;
  r1 = r0 + per;
  if (r0 > n) r0 = n;
  if (r1 > n) r1 = n;
}

}  // namespace lrk

namespace lrk {

// ---------------------------------------------- warp-level Householder QR
// Same contract as block_householder_qr, executed by ONE warp (no CTA
// barriers).  Used for the small stacked-R level of the TSQR.
__device__ inline void warp_householder_qr(double* X, int64_t ldx, int m, int q,
                                           double* tau, double* Rout) {
  const int lane = threadIdx.x & 31;
  for (int i = lane; i < q * q; i += 32) Rout[i] = 0.0;
  __syncwarp();
  const int kmax = m < q ? m : q;
  for (int j = 0; j < kmax; ++j) {
    double s = 0.0;
    for (int i = j + 1 + lane; i < m; i += 32) { double x = X[i + (int64_t)j * ldx]; s += x * x; }
    const double sig = warp_sum(s);
    const double alpha = X[j + (int64_t)j * ldx];
    double beta, t, scale;
    if (sig == 0.0) { t = 0.0; beta = alpha; scale = 0.0; }
    else {
      const double nrm = sqrt(alpha * alpha + sig);
      beta = alpha >= 0.0 ? -nrm : nrm;
      t = (beta - alpha) / beta;
      scale = 1.0 / (alpha - beta);
    }
    __syncwarp();
    for (int i = j + 1 + lane; i < m; i += 32) X[i + (int64_t)j * ldx] *= scale;
    __syncwarp();
    double w[PMAX];
#pragma unroll
    for (int k = 0; k < PMAX; ++k) w[k] = 0.0;
    for (int i = j + 1 + lane; i < m; i += 32) {
      const double vi = X[i + (int64_t)j * ldx];
#pragma unroll
      for (int k = 0; k < PMAX; ++k)
        if (k > j && k < q) w[k] += vi * X[i + (int64_t)k * ldx];
    }
#pragma unroll
    for (int k = 0; k < PMAX; ++k)
      if (k > j && k < q) w[k] = warp_sum(w[k]);
    for (int k = j + 1; k < q; ++k) {
      const double f = t * (w[k] + X[j + (int64_t)k * ldx]);
      for (int i = j + 1 + lane; i < m; i += 32) X[i + (int64_t)k * ldx] -= f * X[i + (int64_t)j * ldx];
      __syncwarp();
      if (lane == 0) { X[j + (int64_t)k * ldx] -= f; Rout[j * q + k] = X[j + (int64_t)k * ldx]; }
      __syncwarp();
    }
    if (lane == 0) { Rout[j * q + j] = beta; X[j + (int64_t)j * ldx] = beta; tau[j] = t; }
    __syncwarp();
  }
  for (int j = kmax + lane; j < q; j += 32) tau[j] = 0.0;
  __syncwarp();
}

// Rows [row0, row0+nrow) of H_0 ... H_{kmax-1} [G; 0] (m x q), one warp,
// G (q x q row-major).  Y: scratch m x q col-major (ldy); result rows copied
// to out (nrow x q row-major).
__device__ inline void warp_householder_q_rows(const double* X, int64_t ldx, int m, int q,
                                               const double* tau, const double* G,
                                               double* Y, int64_t ldy, int row0, int nrow,
                                               double* out) {
  const int lane = threadIdx.x & 31;
  for (int c = 0; c < q; ++c)
    for (int i = lane; i < m; i += 32) Y[i + (int64_t)c * ldy] = (i < q) ? G[i * q + c] : 0.0;
  __syncwarp();
  const int kmax = m < q ? m : q;
  for (int j = kmax - 1; j >= 0; --j) {
    const double t = tau[j];
    if (t == 0.0) continue;
    double w[PMAX];
#pragma unroll
    for (int c = 0; c < PMAX; ++c) w[c] = 0.0;
    for (int i = j + 1 + lane; i < m; i += 32) {
      const double vi = X[i + (int64_t)j * ldx];
#pragma unroll
      for (int c = 0; c < PMAX; ++c)
        if (c < q) w[c] += vi * Y[i + (int64_t)c * ldy];
    }
#pragma unroll
    for (int c = 0; c < PMAX; ++c)
      if (c < q) w[c] = warp_sum(w[c]);
    for (int c = 0; c < q; ++c) {
      const double f = t * (w[c] + Y[j + (int64_t)c * ldy]);
      for (int i = j + 1 + lane; i < m; i += 32) Y[i + (int64_t)c * ldy] -= f * X[i + (int64_t)j * ldx];
      __syncwarp();
      if (lane == 0) Y[j + (int64_t)c * ldy] -= f;
      __syncwarp();
    }
  }
  for (int idx = lane; idx < nrow * q; idx += 32) {
    const int i = idx / q, c = idx % q;
    out[idx] = Y[(row0 + i) + (int64_t)c * ldy];
  }
  __syncwarp();
}

}  // namespace lrk
