// core_svd_bench.cu — the core-SVD routines of the sweep on REAL flush cores
// dumped by the library (LRK_DUMP_CORES=<prefix> writes <prefix>.fwd/.bwd:
// per flush [n, X (32 x 33, ld 33)] with X = K^T, the matrix the Jacobi sees).
// Reports cycles per core (clock64 on one CTA), Jacobi sweeps, and accuracy:
// reconstruction ||X - U S V^T|| / ||X||, orthogonality of U and V, and the
// largest singular-value difference against variant 0 (relative to s_0).
// Build (from tools/): nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I.
//        --expt-relaxed-constexpr -I../paper_1703_05638_b200/csrc -o core_svd_bench core_svd_bench.cu
// Usage: ./core_svd_bench <dumpfile> <variant>...
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <algorithm>

#include "lrk_small.cuh"
#include "jacobi_variants.cuh"
#include "lrk_brand.cuh"  // tools/: experimental secular-equation core SVD

using namespace lrk;

constexpr int CS = 1 + 32 * 33;

template <int VAR, int NJ>
__device__ int run_var(const double* A, int n, double* U, double* V, double* s, int* perm,
                       double* gbuf, double* scr) {
  if constexpr (VAR == 0) {
    int sw = 0;
    if (threadIdx.x < 128) sw = multi_warp_jacobi<NJ, 4>(A, 33, n, U, V, n, s, perm, gbuf);
    return sw;
  } else if constexpr (VAR == 1) {
    int sw = 0;
    if (NJ % 2 == 0 && threadIdx.x < 64) sw = multi_warp_jacobi<NJ, 2>(A, 33, n, U, V, n, s, perm, gbuf);
    return sw;
  } else if constexpr (VAR == 2) {
    int sw = 0;
    if (threadIdx.x < 32) sw = warp_jacobi_reg<NJ>(A, 33, n, U, V, n, s, perm);
    return sw;
  } else if constexpr (VAR == 3) {
    return multi_warp_jacobi<NJ, 8>(A, 33, n, U, V, n, s, perm, gbuf);
  } else if constexpr (VAR == 4) {
    return -1;  // handled in k_file (needs the pivot order)
  } else {
    return 0;
  }
}

template <int VAR>
__global__ void k_file(const double* cores, int ncore, double* Uo, double* Vo, double* So,
                       long long* cyc, int* sws, const int* pivs, long long* tph) {
  __shared__ double A[32 * 33];
  __shared__ double U[32 * 32], V[32 * 32], s[32];
  __shared__ int perm[32];
  __shared__ double gbuf[2 * 8 * 32];
  extern __shared__ double scr[];
  for (int f = 0; f < ncore; ++f) {
    const double* c = cores + (int64_t)f * CS;
    const int n = (int)c[0];
    for (int i = threadIdx.x; i < 32 * 33; i += blockDim.x) A[i] = c[1 + i];
    for (int i = threadIdx.x; i < 32 * 32; i += blockDim.x) U[i] = V[i] = 0.0;
    __syncthreads();
    if (n < 2) continue;
    if constexpr (VAR == 4) {
      // K[i][j] = A[j + i*33]; pc = 4 new columns (fewer when n < 4)
      const int pc = n < 4 ? n : 4, r = n - pc;
      double* sig0 = scr;
      double* Cm = sig0 + 32;
      double* Rm = Cm + 32 * 16;
      int* pv = reinterpret_cast<int*>(Rm + 16 * 16);
      double* Ub = reinterpret_cast<double*>(pv + 32);
      double* Vb = Ub + 1024;
      double* so = Vb + 1024;
      double* wk = so + 32;
      for (int i = threadIdx.x; i < r; i += blockDim.x) sig0[i] = A[i + i * 33];
      for (int idx = threadIdx.x; idx < r * pc; idx += blockDim.x) {
        const int i = idx / pc, j = idx % pc;
        Cm[idx] = A[(r + j) + i * 33];
      }
      for (int idx = threadIdx.x; idx < pc * pc; idx += blockDim.x) {
        const int i = idx / pc, j = idx % pc;
        Rm[idx] = A[(r + j) + (r + i) * 33];
      }
      if (threadIdx.x < pc) pv[threadIdx.x] = pivs[f * 16 + threadIdx.x];
      __syncthreads();
#ifdef WARM
      brand_core_svd(sig0, r, Cm, Rm, pv, pc, Ub, Vb, so, wk, nullptr);
      __syncthreads();
#endif
      long long t0 = clock64();
      int sw = brand_core_svd(sig0, r, Cm, Rm, pv, pc, Ub, Vb, so, wk, tph);
      __syncthreads();
      long long t1 = clock64();
      if (threadIdx.x == 0) { cyc[f] = t1 - t0; sws[f] = sw; }
      // X = K^T = Vb S Ub^T
      for (int i = threadIdx.x; i < n * n; i += blockDim.x) {
        const int a = i % n, c = i / n;
        Uo[(int64_t)f * 1024 + i] = Vb[a + c * 32];
        Vo[(int64_t)f * 1024 + i] = Ub[a + c * 32];
      }
      for (int i = threadIdx.x; i < n; i += blockDim.x) So[f * 32 + i] = so[i];
      __syncthreads();
      continue;
    }
    long long t0 = clock64();
    int sw;
    if (n <= 8) sw = run_var<VAR, 8>(A, n, U, V, s, perm, gbuf, scr);
    else if (n <= 16) sw = run_var<VAR, 16>(A, n, U, V, s, perm, gbuf, scr);
    else if (n <= 24) sw = run_var<VAR, 24>(A, n, U, V, s, perm, gbuf, scr);
    else sw = run_var<VAR, 32>(A, n, U, V, s, perm, gbuf, scr);
    __syncthreads();
    long long t1 = clock64();
    if (threadIdx.x == 0) { cyc[f] = t1 - t0; sws[f] = sw; }
    for (int i = threadIdx.x; i < n * n; i += blockDim.x) {
      Uo[(int64_t)f * 1024 + i] = U[i];
      Vo[(int64_t)f * 1024 + i] = V[i];
    }
    for (int i = threadIdx.x; i < n; i += blockDim.x) So[f * 32 + i] = s[i];
    __syncthreads();
  }
}

int main(int argc, char** argv) {
  if (argc < 3) { std::fprintf(stderr, "usage: %s dumpfile variant...\n", argv[0]); return 2; }
  FILE* fp = std::fopen(argv[1], "rb");
  if (!fp) { std::perror(argv[1]); return 2; }
  std::vector<double> h;
  double buf[CS];
  while (std::fread(buf, sizeof(double), CS, fp) == (size_t)CS) h.insert(h.end(), buf, buf + CS);
  std::fclose(fp);
  const int ncore = (int)(h.size() / CS);
  double *dC, *dU, *dV, *dS;
  long long* dc;
  int* dsw;
  cudaMalloc(&dC, h.size() * 8);
  cudaMemcpy(dC, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
  cudaMalloc(&dU, (size_t)ncore * 1024 * 8);
  cudaMalloc(&dV, (size_t)ncore * 1024 * 8);
  cudaMalloc(&dS, (size_t)ncore * 32 * 8);
  cudaMalloc(&dc, ncore * 8);
  cudaMalloc(&dsw, ncore * 4);
  // pivot order of the new block: column j's last nonzero row in R (stable)
  std::vector<int> piv(ncore * 16, 0);
  for (int f = 0; f < ncore; ++f) {
    const double* X = h.data() + (size_t)f * CS;
    const int n = (int)X[0];
    const int pc = n < 4 ? n : 4, r = n - pc;
    std::vector<std::pair<int, int>> key;
    for (int j = 0; j < pc; ++j) {
      int last = -1;
      for (int i = 0; i < pc; ++i)
        if (X[1 + (r + j) + (r + i) * 33] != 0.0) last = i;
      key.push_back({last, j});
    }
    std::stable_sort(key.begin(), key.end(), [](auto a, auto b) { return a.first < b.first; });
    for (int j = 0; j < pc; ++j) piv[f * 16 + j] = key[j].second;
  }
  int* dpiv;
  cudaMalloc(&dpiv, piv.size() * 4);
  cudaMemcpy(dpiv, piv.data(), piv.size() * 4, cudaMemcpyHostToDevice);
  long long* dtph;
  cudaMalloc(&dtph, 16 * 8);
  std::vector<double> S0;
  for (int ai = 2; ai < argc; ++ai) {
    const int var = std::atoi(argv[ai]);
    const int smem = 64 * 1024;
#define RUN(V)                                                                                    \
  case V:                                                                                         \
    cudaFuncSetAttribute(k_file<V>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);           \
    k_file<V><<<1, 256, smem>>>(dC, ncore, dU, dV, dS, dc, dsw, dpiv, dtph);                                  \
    break;
    cudaMemset(dtph, 0, 16 * 8);
    switch (var) { RUN(0) RUN(1) RUN(2) RUN(3) RUN(4) default: break; }
    cudaError_t e = cudaDeviceSynchronize();
    long long tp[16];
    cudaMemcpy(tp, dtph, 16 * 8, cudaMemcpyDeviceToHost);
    std::vector<long long> cyc(ncore);
    std::vector<int> sw(ncore);
    std::vector<double> U((size_t)ncore * 1024), V((size_t)ncore * 1024), S((size_t)ncore * 32);
    cudaMemcpy(cyc.data(), dc, ncore * 8, cudaMemcpyDeviceToHost);
    cudaMemcpy(sw.data(), dsw, ncore * 4, cudaMemcpyDeviceToHost);
    cudaMemcpy(U.data(), dU, U.size() * 8, cudaMemcpyDeviceToHost);
    cudaMemcpy(V.data(), dV, V.size() * 8, cudaMemcpyDeviceToHost);
    cudaMemcpy(S.data(), dS, S.size() * 8, cudaMemcpyDeviceToHost);
    double tc = 0, tsw = 0, rec = 0, ou = 0, ov = 0, ds = 0;
    int cnt = 0, nsum = 0;
    for (int f = 0; f < ncore; ++f) {
      const double* X = h.data() + (size_t)f * CS;
      const int n = (int)X[0];
      if (n < 2) continue;
      ++cnt; nsum += n;
      tc += cyc[f]; tsw += sw[f];
      const double* u = U.data() + (size_t)f * 1024;
      const double* v = V.data() + (size_t)f * 1024;
      const double* s = S.data() + (size_t)f * 32;
      double err = 0, nm = 0;
      for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j) {
          double x = 0;
          for (int k = 0; k < n; ++k) x += u[i + k * n] * s[k] * v[j + k * n];
          const double a = X[1 + i + j * 33];
          err += (x - a) * (x - a);
          nm += a * a;
        }
      rec = std::fmax(rec, std::sqrt(err / nm));
      for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j) {
          if (s[i] <= 1e-15 * s[0] || s[j] <= 1e-15 * s[0]) continue;
          double du = 0, dv = 0;
          for (int k = 0; k < n; ++k) { du += u[k + i * n] * u[k + j * n]; dv += v[k + i * n] * v[k + j * n]; }
          ou = std::fmax(ou, std::fabs(du - (i == j)));
          ov = std::fmax(ov, std::fabs(dv - (i == j)));
        }
      if (!S0.empty())
        for (int k = 0; k < n; ++k) ds = std::fmax(ds, std::fabs(s[k] - S0[f * 32 + k]) / S0[f * 32]);
    }
    if (S0.empty()) S0 = S;
    std::printf("var %d: %d cores (mean n %.1f): %.0f cycles/core, %.2f sweeps/core, rec %.1e, "
                "orthU %.1e, orthV %.1e, max|ds|/s0 vs var0 %.1e (%s)\n",
                var, cnt, (double)nsum / cnt, tc / cnt, tsw / cnt, rec, ou, ov, ds,
                cudaGetErrorString(e));
    if (var == 4) {
      std::printf("   phases/core:");
      for (int k = 0; k < 12; ++k) std::printf(" %lld", tp[k] / cnt);
      std::printf("\n");
    }
  }
  return 0;
}
