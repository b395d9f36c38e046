// k_band_fb_vec on a synthetic band (nt = 224, wb = 1, identity-ish factor) with phase timing (diagnostics).

#include <cstdio>
#include <vector>
#include "../paper_2101_12164_b200/csrc/nsp_kernels.cu"
void nsp_count_launch() {}
int main() {
  const int nt = 224, wb = 1;
  std::vector<double> T((size_t)nt * (wb + 1) * 4096, 0.0);
  for (int I = 0; I < nt; ++I) for (int r = 0; r < 64; ++r) T[((size_t)I * (wb + 1)) * 4096 + r * 64 + r] = 1.0;
  double *dT, *buf; TriSys* dsys;
  cudaMalloc(&dT, T.size() * 8); cudaMalloc(&buf, nt * 64 * 8); cudaMalloc(&dsys, sizeof(TriSys));
  cudaMemcpy(dT, T.data(), T.size() * 8, cudaMemcpyHostToDevice);
  TriSys sy{dT, nt, wb, 0}; cudaMemcpy(dsys, &sy, sizeof(sy), cudaMemcpyHostToDevice);
  { std::vector<double> b0(nt * 64, 1.0); cudaMemcpy(buf, b0.data(), nt * 64 * 8, cudaMemcpyHostToDevice); }
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int r = 0; r < 3; ++r) nspk::tri_fb(dsys, 1, buf, 1, 1, true, true, 0, wb);

  cudaEventRecord(e0); nspk::tri_fb(dsys, 1, buf, 1, 1, true, true, 0, wb); cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);

  std::vector<double> x(nt * 64); cudaMemcpy(x.data(), buf, nt * 64 * 8, cudaMemcpyDeviceToHost);
  printf("vec band solve %.3f ms (%.2f us per product) %s\n", ms, ms * 1e3 / (2 * (2 * nt - 1)), cudaGetErrorString(cudaGetLastError()));
  return 0;
}
