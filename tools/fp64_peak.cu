// fp64 peak microbenchmark for the roofline denominators.
// DMMA: mma.sync m8n8k4 f64 back-to-back on independent accumulators; DFMA: fma.rn.f64 chains.
#include <cstdio>
#include <cuda_runtime.h>
#define ITERS 4096
__global__ void dmma_loop(double* out, double seed) {
  double a = seed + threadIdx.x * 1e-9, b = seed * 0.5;
  double c[8][2];
#pragma unroll
  for (int i = 0; i < 8; ++i) { c[i][0] = 0; c[i][1] = 0; }
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.678) out[0] = s;
}
__global__ void dmma16_loop(double* out, double seed) {
  double a0 = seed + threadIdx.x * 1e-9, a1 = seed*0.3, a2=seed*0.1, a3=seed*0.7, b0 = seed * 0.5, b1=seed*0.2;
  double c[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i) for (int j=0;j<4;++j) c[i][j] = 0;
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < 4; ++i)
      asm volatile("mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                   : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3]) : "d"(a0), "d"(a1), "d"(a2), "d"(a3), "d"(b0), "d"(b1));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 4; ++i) for (int j=0;j<4;++j) s += c[i][j];
  if (s == 12345.678) out[0] = s;
}
__global__ void dfma_loop(double* out, double seed) {
  double x[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) x[i] = seed + i + threadIdx.x;
  const double m = 0.999999, a = 1e-7;
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = fma(x[i], m, a);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += x[i];
  if (s == 12345.678) out[0] = s;
}
int main() {
  double* d; cudaMalloc(&d, 8);
  int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int warps = 4; warps <= 32; warps *= 2) {
    int blocks = nsm * 2, threads = 32 * warps / 2;
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(e0); dmma_loop<<<blocks, threads>>>(d, 1.0); cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      double fl = 2.0 * 8 * 8 * 4 * 8.0 * ITERS * (blocks * threads / 32);
      if (rep) printf("DMMA m8n8k4  warps/SM=%2d: %.2f TFLOP/s\n", warps, fl / ms / 1e9);
      cudaEventRecord(e0); dmma16_loop<<<blocks, threads>>>(d, 1.0); cudaEventRecord(e1); cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
      fl = 2.0 * 16 * 8 * 8 * 4.0 * ITERS * (blocks * threads / 32);
      if (rep) printf("DMMA m16n8k8 warps/SM=%2d: %.2f TFLOP/s\n", warps, fl / ms / 1e9);
      cudaEventRecord(e0); dfma_loop<<<blocks, threads>>>(d, 1.0); cudaEventRecord(e1); cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
      fl = 2.0 * 8.0 * ITERS * (double)(blocks * threads);
      if (rep) printf("DFMA         warps/SM=%2d: %.2f TFLOP/s\n", warps, fl / ms / 1e9);
    }
  }
  // HBM copy
  size_t n = 1ull << 30; double *a, *b; cudaMalloc(&a, n); cudaMalloc(&b, n);
  cudaMemset(a, 0, n);
  float best = 1e9;
  for (int r = 0; r < 10; ++r) { cudaEventRecord(e0); cudaMemcpy(b, a, n, cudaMemcpyDeviceToDevice); cudaEventRecord(e1); cudaEventSynchronize(e1); float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms; }
  printf("D2D memcpy 1 GiB: %.1f GB/s (read+write)\n", 2.0 * n / best / 1e6);
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
