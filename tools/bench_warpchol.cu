// warp-level 32x32 Cholesky + inverse variants (diagnostics for k_small_chol)
#include <cstdio>
#include <vector>
#include <cmath>
__device__ __forceinline__ double rsqrt_nr(double d) {
  double r;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(d));
  const double h = 0.5 * d;
  r = r * fma(-h * r, r, 1.5);
  r = r * fma(-h * r, r, 1.5);
  return r;
}
template <int V>
__global__ void k_wc(const double* A, double* Lout, double* Yout, int reps) {
  const int lane = threadIdx.x & 31;
  double row[32], y[32], ild[32];
  for (int rep = 0; rep < reps; ++rep) {
#pragma unroll 32
  for (int j = 0; j < 32; ++j) row[j] = A[lane * 32 + j];
#pragma unroll 32
  for (int c = 0; c < 32; ++c) {
    double dc = __shfl_sync(0xffffffffu, row[c], c);
    const double il = (V == 0) ? 1.0 / sqrt(dc) : rsqrt_nr(dc);
    ild[c] = il;
    if (lane > c) row[c] *= il;
    else if (lane == c) row[c] = dc * il;
#pragma unroll 32
    for (int j = c + 1; j < 32; ++j) {
      const double lj = __shfl_sync(0xffffffffu, row[c], j);
      if (lane >= j) row[j] = fma(-row[c], lj, row[j]);
    }
  }
  // right-looking inverse: lane = column j; acc[i] for all i
#pragma unroll 32
  for (int i = 0; i < 32; ++i) y[i] = (lane == i) ? 1.0 : 0.0;
#pragma unroll 32
  for (int k = 0; k < 32; ++k) {
    y[k] = (V == 0) ? y[k] / __shfl_sync(0xffffffffu, row[k], k) : y[k] * ild[k];
#pragma unroll 32
    for (int i = k + 1; i < 32; ++i) {
      const double lik = __shfl_sync(0xffffffffu, row[k], i);
      y[i] = fma(-lik, y[k], y[i]);
    }
  }
  }
#pragma unroll 32
  for (int j = 0; j < 32; ++j) Lout[lane * 32 + j] = row[j];
#pragma unroll 32
  for (int i = 0; i < 32; ++i) Yout[i * 32 + lane] = y[i];
}
int main() {
  std::vector<double> A(1024);
  for (int i = 0; i < 32; ++i) for (int j = 0; j < 32; ++j) A[i*32+j] = (i==j ? 40.0 : 0.0) + 1.0/(1+i+j);
  double *dA, *dL, *dY; cudaMalloc(&dA, 8192); cudaMalloc(&dL, 8192); cudaMalloc(&dY, 8192);
  cudaMemcpy(dA, A.data(), 8192, cudaMemcpyHostToDevice);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1); float ms;
  k_wc<0><<<1,32>>>(dA, dL, dY, 1); k_wc<1><<<1,32>>>(dA, dL, dY, 1);
  cudaEventRecord(e0); k_wc<0><<<1,32>>>(dA, dL, dY, 20); cudaEventRecord(e1); cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms, e0, e1); printf("sqrt+div: %.2f us per chol+inv\n", ms * 50);
  cudaEventRecord(e0); k_wc<1><<<1,32>>>(dA, dL, dY, 20); cudaEventRecord(e1); cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms, e0, e1); printf("rsqrt: %.2f us per chol+inv\n", ms * 50);
  std::vector<double> L(1024), Y(1024);
  cudaMemcpy(L.data(), dL, 8192, cudaMemcpyDeviceToHost); cudaMemcpy(Y.data(), dY, 8192, cudaMemcpyDeviceToHost);
  double e = 0, e2 = 0;
  for (int i = 0; i < 32; ++i) for (int j = 0; j < 32; ++j) {
    double s = 0, t = 0; for (int k = 0; k <= std::min(i,j); ++k) s += L[i*32+k]*L[j*32+k];
    for (int k = 0; k < 32; ++k) t += (k <= i ? L[i*32+k] : 0) * Y[k*32+j];
    e = std::max(e, std::abs(s - A[i*32+j])); e2 = std::max(e2, std::abs(t - (i==j)));
  }
  printf("LL^T - A %.2e  L Y - I %.2e\n", e, e2);
  return 0;
}
