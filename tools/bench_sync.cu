// diagnostics: cost of barrier-separated steps with 1024 threads, and fp64 sqrt/rcp chains
#include <cstdio>
__global__ void k_bar(double* out, int steps) {
  __shared__ double v[2];
  double x = threadIdx.x;
  for (int c = 0; c < steps; ++c) {
    if (threadIdx.x == 0 && threadIdx.y == 0) v[c & 1] = x + c;
    __syncthreads();
    x += v[c & 1];
  }
  if (x == -1) out[0] = x;
}
__global__ void k_chain(double* out, int steps) {
  double x = 2.0 + threadIdx.x;
  for (int c = 0; c < steps; ++c) { double l = sqrt(x); x = 1.0 / l + 3.0; }
  if (x == -1) out[0] = x;
}
int main() {
  double* d; cudaMalloc(&d, 8);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1); float ms;
  for (int thr : {32, 256, 1024}) {
    k_bar<<<1, dim3(32, thr / 32)>>>(d, 384);
    cudaEventRecord(e0); k_bar<<<1, dim3(32, thr / 32)>>>(d, 384); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1); printf("384 barriers, %4d threads: %.2f us\n", thr, ms * 1000);
  }
  k_chain<<<1, 32>>>(d, 128);
  cudaEventRecord(e0); k_chain<<<1, 32>>>(d, 128); cudaEventRecord(e1); cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms, e0, e1); printf("128 x (sqrt + rcp) chain: %.2f us\n", ms * 1000);
  return 0;
}
