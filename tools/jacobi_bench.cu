// jacobi_bench.cu — cycles of the core-SVD routine in isolation, on a
// Brand-update-shaped core [[diag(s), C], [0, R]] (n = r + 4).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../paper_1703_05638_b200/csrc -o jacobi_bench jacobi_bench.cu
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>
#include "lrk_small.cuh"
#include "jacobi_variants.cuh"

using namespace lrk;

template <int NJ, int JW>
__global__ void k_jac(const double* M, int n, double* U, double* V, double* s, int* perm,
                      long long* cyc, int* sweeps, int reps) {
  __shared__ double A[32 * 33];
  __shared__ double gbuf[2 * 8 * 32];
  extern __shared__ double scr[];
  for (int i = threadIdx.x; i < n * n; i += blockDim.x) A[(i % n) + (i / n) * 33] = M[i];
  __syncthreads();
  if constexpr (JW == 9) {  // stacked TSQR of 148 4x4 blocks (M holds the part buffer)
    long long t0 = clock64();
    int wo = 0;
    for (int r = 0; r < reps; ++r) {
      __shared__ double* pp[1];
      pp[0] = const_cast<double*>(M) - 2 * 148 * 16;
      __syncthreads();
      const PartTab tab{pp, 148, 1, 16};
      wo += warp_stack_tsqr<4, 3>(tab, 148, 4, 77, A, scr, scr + 64);
      __syncthreads();
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) { cyc[0] = (t1 - t0) / reps; sweeps[0] = wo; }
    if (threadIdx.x < 16) U[threadIdx.x] = scr[threadIdx.x] + scr[64 + threadIdx.x];
  } else if constexpr (JW == 6) {  // the two preconditioning QRs only
    long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
      if (threadIdx.x < 32) {
        double a[NJ];
        const int lane = threadIdx.x;
#pragma unroll
        for (int i = 0; i < NJ; ++i) a[i] = (lane < n && i < n) ? A[i + lane * 33] : 0.0;
        int colid;
        warp_qr_cols<NJ, true>(a, n, scr, 33, scr + 2000, colid);
        warp_qr_cols<NJ, false>(a, n, scr + 3000, 33, scr + 5000, colid);
        if (lane < n) U[lane] = a[0] + colid;
      }
      __syncthreads();
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) { cyc[0] = (t1 - t0) / reps; sweeps[0] = 1; }
  } else if constexpr (JW == 8) {  // all warps, convergent call site
    long long t0 = clock64();
    int sw = 0;
    for (int r = 0; r < reps; ++r) sw += multi_warp_jacobi<NJ, 8>(A, 33, n, U, V, n, s, perm, gbuf);
    long long t1 = clock64();
    if (threadIdx.x == 0) { cyc[0] = (t1 - t0) / reps; sweeps[0] = sw / reps; }
  } else if constexpr (JW == 5) {
    long long t0 = clock64();
    int sw = 0;
    for (int r = 0; r < reps; ++r) {
      sw += precond_svd<NJ>(A, 33, n, U, V, n, s, perm, scr);
      __syncthreads();
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) { cyc[0] = (t1 - t0) / reps; sweeps[0] = sw / reps; }
  } else if (threadIdx.x < 32 * JW) {
    long long t0 = clock64();
    int sw = 0;
    for (int r = 0; r < reps; ++r) {
      if constexpr (JW == 1) sw += warp_jacobi_reg<NJ>(A, 33, n, U, V, n, s, perm);
      else sw += multi_warp_jacobi<NJ, JW>(A, 33, n, U, V, n, s, perm, gbuf);
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) { cyc[0] = (t1 - t0) / reps; sweeps[0] = sw / reps; }
  }
}

int main(int argc, char** argv) {
  const int r = argc > 1 ? atoi(argv[1]) : 15;
  const int pc = 4, n = r + pc;
  std::vector<double> M(n * n, 0.0);
  srand(1);
  auto rnd = [] { return (double)rand() / RAND_MAX - 0.5; };
  for (int i = 0; i < r; ++i) M[i + i * n] = pow(10.0, -8.0 * i / (r - 1));
  for (int j = r; j < n; ++j)
    for (int i = 0; i <= j; ++i) M[i + j * n] = (i < r ? 1e-2 : 1e-3) * rnd();
  double *dM, *dU, *dV, *ds;
  int *dp, *dsw;
  long long* dc;
  cudaMalloc(&dM, 8 * n * n); cudaMalloc(&dU, 8 * n * n); cudaMalloc(&dV, 8 * n * n);
  cudaMalloc(&ds, 8 * n); cudaMalloc(&dp, 4 * n); cudaMalloc(&dc, 8); cudaMalloc(&dsw, 4);
  cudaMemcpy(dM, M.data(), 8 * n * n, cudaMemcpyHostToDevice);
  const int jw = argc > 2 ? atoi(argv[2]) : 1;
#define LAUNCH(NJ, JW)                                                                        \
  do {                                                                                        \
    cudaFuncSetAttribute(k_jac<NJ, JW>, cudaFuncAttributeMaxDynamicSharedMemorySize,          \
                         PRECOND_SCR * 8);                                                    \
    k_jac<NJ, JW><<<1, 256, PRECOND_SCR * 8>>>(dM, n, dU, dV, ds, dp, dc, dsw, 20);           \
  } while (0)
  if (jw == 1) { if (n <= 16) LAUNCH(16, 1); else if (n <= 24) LAUNCH(24, 1); else LAUNCH(32, 1); }
  else if (jw == 4) { if (n <= 16) LAUNCH(16, 4); else if (n <= 24) LAUNCH(24, 4); else LAUNCH(32, 4); }
  else if (jw == 5) { if (n <= 16) LAUNCH(16, 5); else if (n <= 24) LAUNCH(24, 5); else LAUNCH(32, 5); }
  else if (jw == 9) {
    std::vector<double> P(148 * 16);
    for (auto& x : P) x = rnd();
    double* dP;
    cudaMalloc(&dP, 8 * P.size());
    cudaMemcpy(dP, P.data(), 8 * P.size(), cudaMemcpyHostToDevice);
    cudaFuncSetAttribute(k_jac<16, 9>, cudaFuncAttributeMaxDynamicSharedMemorySize, PRECOND_SCR * 8);
    k_jac<16, 9><<<1, 256, PRECOND_SCR * 8>>>(dP, n, dU, dV, ds, dp, dc, dsw, 20);
  }
  else if (jw == 6) { if (n <= 16) LAUNCH(16, 6); else if (n <= 24) LAUNCH(24, 6); else LAUNCH(32, 6); }
  else { if (n <= 16) LAUNCH(16, 8); else if (n <= 24) LAUNCH(24, 8); else LAUNCH(32, 8); }
  long long cyc;
  int sw;
  cudaMemcpy(&cyc, dc, 8, cudaMemcpyDeviceToHost);
  cudaMemcpy(&sw, dsw, 4, cudaMemcpyDeviceToHost);
  std::vector<double> s(n), U(n * n);
  cudaMemcpy(s.data(), ds, 8 * n, cudaMemcpyDeviceToHost);
  cudaMemcpy(U.data(), dU, 8 * n * n, cudaMemcpyDeviceToHost);
  double orth = 0.0;  // max |U^T U - I| over columns with s > 1e-15 s0
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) {
      if (s[i] <= 1e-15 * s[0] || s[j] <= 1e-15 * s[0]) continue;
      double d = 0.0;
      for (int k = 0; k < n; ++k) d += U[k + i * n] * U[k + j * n];
      orth = fmax(orth, fabs(d - (i == j ? 1.0 : 0.0)));
    }
  // reconstruction error ||M - U S V^T|| / ||M||
  std::vector<double> V(n * n);
  cudaMemcpy(V.data(), dV, 8 * n * n, cudaMemcpyDeviceToHost);
  double err = 0.0, nm = 0.0;
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) {
      double x = 0.0;
      for (int k = 0; k < n; ++k) x += U[i + k * n] * s[k] * V[j + k * n];
      err += (x - M[i + j * n]) * (x - M[i + j * n]);
      nm += M[i + j * n] * M[i + j * n];
    }
  printf("n=%d jw=%d: %lld cycles, %d sweeps, %.0f cycles/round; s0=%.3e s_last=%.3e orth=%.1e rec=%.1e (%s)\n",
         n, jw, cyc, sw, (double)cyc / (sw * (n + (n & 1) - 1)), s[0], s[n - 1], orth,
         sqrt(err / nm), cudaGetErrorString(cudaGetLastError()));
  return 0;
}
