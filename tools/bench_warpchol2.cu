// warp-level 32x32 Cholesky + inverse with the tile in shared memory (diagnostics)
#include <cstdio>
#include <vector>
#include <cmath>
#include <algorithm>
__device__ __forceinline__ double rsqrt_nr(double d) {
  double r;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(d));
  const double h = 0.5 * d;
  r = r * fma(-h * r, r, 1.5);
  r = r * fma(-h * r, r, 1.5);
  return r;
}
// S: 32 x LD tile (row-major) in smem, lower part = A on entry, L on exit; Y: 32 x LD, Y = L^{-1}
// (lower); ild[32]: reciprocal pivots; returns false on a non-positive pivot
__device__ bool warp_chol32(double* S, int ld, double* Y, double* ild, double* piv) {
  const int lane = threadIdx.x & 31;
  bool ok = true;
  for (int c = 0; c < 32; ++c) {
    double dc = S[c * ld + c];
    if (lane == 0) piv[c] = dc;
    if (!(dc > 0.0)) { ok = false; dc = 1.0; }
    const double il = rsqrt_nr(dc);
    double lic = 0.0;
    if (lane > c) { lic = S[lane * ld + c] * il; S[lane * ld + c] = lic; }
    if (lane == c) { S[c * ld + c] = dc * il; ild[c] = il; }
    __syncwarp();
    if (lane > c)
      for (int j = c + 1; j <= lane; ++j) S[lane * ld + j] = fma(-lic, S[j * ld + c], S[lane * ld + j]);
    __syncwarp();
  }
  // Y = L^{-1}: lane = column j, right-looking
  for (int i = 0; i < 32; ++i) Y[i * ld + lane] = (i == lane) ? 1.0 : 0.0;
  __syncwarp();
  double yk;
  for (int k = 0; k < 32; ++k) {
    yk = Y[k * ld + lane] * ild[k];
    Y[k * ld + lane] = yk;
    for (int i = k + 1; i < 32; ++i) Y[i * ld + lane] = fma(-S[i * ld + k], yk, Y[i * ld + lane]);
  }
  __syncwarp();
  return ok;
}
__global__ void k_wc2(const double* A, double* Lout, double* Yout, int reps) {
  __shared__ double S[32 * 33], Y[32 * 33], ild[32], piv[32];
  const int lane = threadIdx.x;
  for (int rep = 0; rep < reps; ++rep) {
    for (int j = 0; j < 32; ++j) S[lane * 33 + j] = A[lane * 32 + j];
    __syncwarp();
    warp_chol32(S, 33, Y, ild, piv);
  }
  for (int j = 0; j < 32; ++j) { Lout[lane * 32 + j] = j <= lane ? S[lane * 33 + j] : 0.0; Yout[lane * 32 + j] = Y[lane * 33 + j]; }
}
int main() {
  std::vector<double> A(1024);
  for (int i = 0; i < 32; ++i) for (int j = 0; j < 32; ++j) A[i*32+j] = (i==j ? 40.0 : 0.0) + 1.0/(1+i+j);
  double *dA, *dL, *dY; cudaMalloc(&dA, 8192); cudaMalloc(&dL, 8192); cudaMalloc(&dY, 8192);
  cudaMemcpy(dA, A.data(), 8192, cudaMemcpyHostToDevice);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1); float ms;
  k_wc2<<<1,32>>>(dA, dL, dY, 1);
  cudaEventRecord(e0); k_wc2<<<1,32>>>(dA, dL, dY, 20); cudaEventRecord(e1); cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms, e0, e1); printf("smem warp chol+inv: %.2f us\n", ms * 50);
  std::vector<double> L(1024), Y(1024);
  cudaMemcpy(L.data(), dL, 8192, cudaMemcpyDeviceToHost); cudaMemcpy(Y.data(), dY, 8192, cudaMemcpyDeviceToHost);
  double e = 0, e2 = 0;
  for (int i = 0; i < 32; ++i) for (int j = 0; j < 32; ++j) {
    double s = 0, t = 0; for (int k = 0; k <= std::min(i,j); ++k) s += L[i*32+k]*L[j*32+k];
    for (int k = 0; k < 32; ++k) t += L[i*32+k] * Y[k*32+j];
    e = std::max(e, std::abs(s - A[i*32+j])); e2 = std::max(e2, std::abs(t - (i==j)));
  }
  printf("LL^T - A %.2e  L Y - I %.2e\n", e, e2);
  return 0;
}
