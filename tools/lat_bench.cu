// lat_bench.cu — dependent-chain latencies of the FP64 / MUFU / SMEM / barrier
// operations the small-matrix code of the sweep is built from (one warp).
#include <cstdio>
#define REP 256
__global__ void k(double* out, long long* cyc, double x0) {
  __shared__ double sm[256];
  double x = x0 + threadIdx.x * 1e-3, y = 1.0 + x0;
  sm[threadIdx.x] = x;
  __syncthreads();
  long long t0, t1;
  int ci = 0;
#define MEAS(body)                        \
  t0 = clock64();                         \
  for (int i = 0; i < REP; ++i) { body; } \
  t1 = clock64();                         \
  if (threadIdx.x == 0) cyc[ci] = (t1 - t0) / REP; \
  ++ci;
  MEAS(x = fma(x, y, 1e-9))                       // 0 DFMA
  MEAS(x = x + y)                                 // 1 DADD
  MEAS(x = __drcp_rn(x))                          // 2 drcp_rn
  MEAS(x = 1.0 / x)                               // 3 div
  MEAS(x = sqrt(x))                               // 4 sqrt
  MEAS(x = rsqrt(x))                              // 5 rsqrt
  MEAS(x = sm[((int)x) & 255])                    // 6 LDS dependent
  MEAS(x = __shfl_sync(0xffffffff, x, (threadIdx.x + 1) & 31))  // 7 shfl
  MEAS(asm volatile("bar.sync 1, 128;"); x += 1.0)               // 8 named bar (128) + dadd
  MEAS(__syncthreads(); x += 1.0)                                // 9 syncthreads + dadd
  MEAS(x = (double)(float)x)                      // 10 F2F round trip
  MEAS(x = x * y)                                 // 11 DMUL
  out[threadIdx.x] = x;
}
int main() {
  double* o; long long* c;
  cudaMalloc(&o, 256 * 8); cudaMalloc(&c, 64 * 8);
  k<<<1, 128>>>(o, c, 0.5);
  long long h[12];
  cudaMemcpy(h, c, 12 * 8, cudaMemcpyDeviceToHost);
  const char* nm[] = {"dfma", "dadd", "drcp_rn", "ddiv", "dsqrt", "drsqrt", "lds_dep", "shfl64", "bar128+dadd", "syncthreads+dadd", "f2f_roundtrip", "dmul"};
  for (int i = 0; i < 12; ++i) printf("%-18s %lld cycles\n", nm[i], h[i]);
  return 0;
}
