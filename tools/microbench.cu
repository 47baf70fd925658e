// microbench.cu — measured latencies/throughputs of the primitives the
// persistent sweep is built from (single SM, clock64 in-kernel timing).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o microbench microbench.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_dfma_lat(double* out, long long* cyc, int iters) {
  double a = out[0], b = 1.0000001, c = 1e-9;
  __syncwarp();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) a = fma(a, b, c);
  long long t1 = clock64();
  out[1] = a;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

__global__ void k_dfma_tput(double* out, long long* cyc, int iters) {
  double a0 = threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5,
         a6 = a0 + 6, a7 = a0 + 7;
  const double b = 1.0000001, c = 1e-9;
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    a0 = fma(a0, b, c); a1 = fma(a1, b, c); a2 = fma(a2, b, c); a3 = fma(a3, b, c);
    a4 = fma(a4, b, c); a5 = fma(a5, b, c); a6 = fma(a6, b, c); a7 = fma(a7, b, c);
  }
  __syncthreads();
  long long t1 = clock64();
  out[threadIdx.x] = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

__global__ void k_lds_lat(double* out, long long* cyc, int iters) {
  __shared__ long long s[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) s[i] = (i * 7 + 3) % 1024;
  __syncthreads();
  long long p = threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) p = s[p];
  long long t1 = clock64();
  out[0] = (double)p;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

__global__ void k_shfl_lat(double* out, long long* cyc, int iters) {
  double v = threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) v = __shfl_xor_sync(0xffffffffu, v, 1) + 1.0;
  long long t1 = clock64();
  out[threadIdx.x] = v;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

__global__ void k_sqrt_lat(double* out, long long* cyc, int iters, int which) {
  double v = out[0] + 2.0;
  long long t0 = clock64();
  if (which == 0)
    for (int i = 0; i < iters; ++i) v = sqrt(v) + 1.5;
  else if (which == 1)
    for (int i = 0; i < iters; ++i) v = 3.0 / v + 1.5;
  else
    for (int i = 0; i < iters; ++i) v = rsqrt(v) + 1.5;
  long long t1 = clock64();
  out[1] = v;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

__global__ void k_syncthreads(long long* cyc, int iters) {
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

__global__ void k_gld_lat(const long long* __restrict__ g, double* out, long long* cyc, int iters) {
  long long p = 0;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) p = __ldcg(g + p);
  long long t1 = clock64();
  out[0] = (double)p;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

int main() {
  double* d;
  long long* c;
  long long* g;
  cudaMalloc(&d, 1 << 20);
  cudaMalloc(&c, 64);
  cudaMalloc(&g, 8 << 20);
  cudaMemset(d, 0, 1 << 20);
  {
    long long* h = new long long[1 << 20];
    for (int i = 0; i < (1 << 20); ++i) h[i] = (i * 4099LL + 977) % (1 << 20);
    cudaMemcpy(g, h, 8 << 20, cudaMemcpyHostToDevice);
    delete[] h;
  }
  long long h;
  const int it = 4096;
  auto rd = [&]() { cudaDeviceSynchronize(); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost); return (double)h; };
  k_dfma_lat<<<1, 32>>>(d, c, it);
  printf("DFMA dependent latency: %.2f cyc\n", rd() / it);
  for (int nt : {32, 128, 256, 1024}) {
    k_dfma_tput<<<1, nt>>>(d, c, it);
    printf("DFMA throughput %4d threads: %.2f DFMA/clk/SM\n", nt, 8.0 * it * nt / rd());
  }
  k_lds_lat<<<1, 32>>>(d, c, it);
  printf("LDS.64 dependent latency: %.2f cyc\n", rd() / it);
  k_shfl_lat<<<1, 32>>>(d, c, it);
  printf("SHFL(f64)+DADD dependent latency: %.2f cyc\n", rd() / it);
  const char* nm[3] = {"sqrt", "div", "rsqrt"};
  for (int w = 0; w < 3; ++w) {
    k_sqrt_lat<<<1, 32>>>(d, c, it, w);
    printf("DP %s (+DADD) dependent latency: %.2f cyc\n", nm[w], rd() / it);
  }
  for (int nt : {32, 256, 512}) {
    k_syncthreads<<<1, nt>>>(c, it);
    printf("__syncthreads (%d threads): %.2f cyc\n", nt, rd() / it);
  }
  k_gld_lat<<<1, 32>>>(g, d, c, 2048);
  printf("LDG.cg dependent latency (8 MiB, L2): %.2f cyc\n", rd() / 2048);
  int clk;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("clock rate attr: %d kHz\n", clk);
  return 0;
}
