#include <cstdio>
__global__ void k_empty(double* o) { extern __shared__ double sm[]; if (threadIdx.x == 1000) o[0] = sm[0]; }
__global__ void k_shfl(double* o, int reps) {
  double row[32];
  const int lane = threadIdx.x & 31;
  for (int j = 0; j < 32; ++j) row[j] = lane + j;
  for (int r = 0; r < reps; ++r) {
#pragma unroll
    for (int c = 0; c < 32; ++c) {
      double dc = __shfl_sync(0xffffffffu, row[c], c);
      const double l = sqrt(dc), il = 1.0 / l;
      if (lane > c) row[c] *= il;
#pragma unroll
      for (int j = c + 1; j < 32; ++j) {
        const double lj = __shfl_sync(0xffffffffu, row[c], j);
        if (lane >= j) row[j] -= row[c] * lj;
      }
    }
  }
  double s = 0; for (int j = 0; j < 32; ++j) s += row[j];
  if (s == 1234.5) o[0] = s;
}
int main() {
  double* d; cudaMalloc(&d, 8);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1); float ms;
  for (int kb : {0, 48, 100, 140, 200}) {
    size_t smem = kb * 1024;
    cudaFuncSetAttribute(k_empty, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    for (int i = 0; i < 3; ++i) k_empty<<<1, 256, smem>>>(d);
    cudaEventRecord(e0); for (int i = 0; i < 100; ++i) k_empty<<<1, 256, smem>>>(d); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1); printf("empty kernel smem %3d KB: %.2f us/launch\n", kb, ms * 10);
  }
  k_shfl<<<1, 32>>>(d, 1);
  cudaEventRecord(e0); k_shfl<<<1, 32>>>(d, 10); cudaEventRecord(e1); cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms, e0, e1); printf("warp 32x32 chol in regs: %.2f us each\n", ms * 100);
  return 0;
}
