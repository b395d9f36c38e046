// fp64 latency microbenchmark (diagnostics): dependent chains of DFMA, rsqrt.approx.f64, sqrt.rn,
// rcp.rn, div, shfl, smem load.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(double* out, long long* cyc, double x0, int n) {
  double x = x0 + threadIdx.x * 1e-9;
  long long t0, t1;
  __shared__ double sm[64];
  sm[threadIdx.x & 63] = x;
  __syncwarp();
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = fma(x, 0.999999, 1e-9);
  t1 = clock64(); if (threadIdx.x == 0) cyc[0] = (t1 - t0);
  t0 = clock64();
  for (int i = 0; i < n; ++i) { double r; asm volatile("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x)); x = r + 1.0; }
  t1 = clock64(); if (threadIdx.x == 0) cyc[1] = (t1 - t0);
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = sqrt(x) + 1.0;
  t1 = clock64(); if (threadIdx.x == 0) cyc[2] = (t1 - t0);
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = 1.0 / x + 1.0;
  t1 = clock64(); if (threadIdx.x == 0) cyc[3] = (t1 - t0);
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = __shfl_sync(0xffffffffu, x, (threadIdx.x + 1) & 31) * 1.0000001;
  t1 = clock64(); if (threadIdx.x == 0) cyc[4] = (t1 - t0);
  t0 = clock64();
  int idx = threadIdx.x & 63;
  for (int i = 0; i < n; ++i) { double v = sm[idx]; idx = ((int)v) & 63; x += v; }
  t1 = clock64(); if (threadIdx.x == 0) cyc[5] = (t1 - t0);
  t0 = clock64();
  for (int i = 0; i < n; ++i) { x = x * 1.0000001; __syncwarp(); }
  t1 = clock64(); if (threadIdx.x == 0) cyc[6] = (t1 - t0);
  t0 = clock64();
  for (int i = 0; i < n; ++i) { x = x * 1.0000001; __syncthreads(); }
  t1 = clock64(); if (threadIdx.x == 0) cyc[7] = (t1 - t0);
  t0 = clock64();
  for (int i = 0; i < n; ++i) { x = x * 1.0000001; }
  t1 = clock64(); if (threadIdx.x == 0) cyc[8] = (t1 - t0);
  out[threadIdx.x] = x;
}
int main() {
  double* o; long long* c; cudaMalloc(&o, 1024 * 8); cudaMalloc(&c, 64 * 8);
  const char* nm[] = {"dfma", "rsqrt.approx.f64 (+dadd)", "sqrt.rn (+dadd)", "rcp/div (+dadd)", "shfl (+dmul)", "lds (+dadd, cvt)", "syncwarp (+dmul)", "syncthreads 256t (+dmul)", "dmul"};
  for (int threads : {32, 256}) {
    k<<<1, threads>>>(o, c, 1.5, 1000);
    k<<<1, threads>>>(o, c, 1.5, 1000);
    long long h[9]; cudaMemcpy(h, c, sizeof(h), cudaMemcpyDeviceToHost);
    printf("threads %d\n", threads);
    for (int i = 0; i < 9; ++i) printf("  %-28s %6.1f cyc/iter\n", nm[i], h[i] / 1000.0);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
