// Reference point for k_symm: cuBLAS DGEMM (strided batched) on the same shapes as cfg2's a2+a3
// (64 blocks, b = 448, s = 128): U_j = M_j W_j with a FULL (not symmetric-packed) M_j.  Diagnostics
// only - not part of the library.
#include <cstdio>
#include <vector>
#include <cublas_v2.h>
#include <cuda_runtime.h>
int main() {
  const int nb = 64, b = 448, s = 128;
  double *M, *W, *U, *flush;
  cudaMalloc(&M, (size_t)nb * b * b * 8); cudaMalloc(&W, (size_t)nb * b * s * 8); cudaMalloc(&U, (size_t)nb * b * s * 8);
  cudaMalloc(&flush, 256 << 20);
  cudaMemset(M, 0, (size_t)nb * b * b * 8); cudaMemset(W, 0, (size_t)nb * b * s * 8);
  cublasHandle_t h; cublasCreate(&h);
  cudaStream_t st; cudaStreamCreate(&st); cublasSetStream(h, st);
  const double one = 1.0, zero = 0.0;
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const double flops = 2.0 * nb * b * (double)b * s;
  for (int mode = 0; mode < 2; ++mode) {
    float best = 1e9;
    for (int r = 0; r < 10; ++r) {
      cudaMemsetAsync(flush, r, 256 << 20, st);
      cudaEventRecord(e0, st);
      if (mode == 0)   // row-major U (b x s) = M (b x b) W (b x s)  <=>  col-major U^T = W^T M^T
        cublasDgemmStridedBatched(h, CUBLAS_OP_N, CUBLAS_OP_N, s, b, b, &one, W, s, (long long)b * s, M, b,
                                  (long long)b * b, &zero, U, s, (long long)b * s, nb);
      else             // symmetric M: cublasDsymm per block (no batched symm)
        for (int j = 0; j < nb; ++j)
          cublasDsymm(h, CUBLAS_SIDE_RIGHT, CUBLAS_FILL_MODE_UPPER, s, b, &one, M + (size_t)j * b * b, b,
                      W + (size_t)j * b * s, s, &zero, U + (size_t)j * b * s, s);
      cudaEventRecord(e1, st); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      if (r >= 3) best = ms < best ? ms : best;
    }
    printf("%s: %.1f us (%.2f TFLOP/s)  %s\n", mode == 0 ? "cublasDgemmStridedBatched" : "64 x cublasDsymm",
           best * 1e3, flops / (best * 1e-3) / 1e12, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
