// Microbenchmark of the small / tall-skinny kernels of nsp_blas.cu in isolation (diagnostics).
#include <cstdio>
#include <vector>
#include <random>
#include <cmath>
#include <algorithm>
#include "../paper_2101_12164_b200/csrc/nsp_blas.cu"
void nsp_count_launch() {}
int main() {
  const int sp = 128; const int64_t n = 14287;
  std::vector<double> hG(sp * sp);
  std::mt19937_64 g(1); std::normal_distribution<double> nd;
  std::vector<double> W(n * sp);
  for (auto& x : W) x = nd(g);
  double *dW, *dG, *dT, *dws, *dP; BcgStatus* dst;
  cudaMalloc(&dW, n * sp * 8); cudaMalloc(&dP, n * sp * 8); cudaMalloc(&dG, sp * sp * 8); cudaMalloc(&dT, sp * sp * 8);
  cudaMalloc(&dws, nspb::gram_ws_doubles(n, sp, sp) * 8); cudaMalloc(&dst, sizeof(BcgStatus));
  cudaMemcpy(dW, W.data(), n * sp * 8, cudaMemcpyHostToDevice);
  BcgStatus h{}; h.width = sp; cudaMemcpy(dst, &h, sizeof(h), cudaMemcpyHostToDevice);
  cudaStream_t st; cudaStreamCreate(&st);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  auto timeit = [&](const char* name, auto fn) {
    for (int i = 0; i < 3; ++i) fn();
    cudaEventRecord(e0, st);
    for (int i = 0; i < 20; ++i) fn();
    cudaEventRecord(e1, st); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("%-20s %8.2f us  (%s)\n", name, ms * 1000 / 20, cudaGetErrorString(cudaGetLastError()));
  };
  // correctness of small_chol on a well-conditioned Gram
  {
    std::vector<double> Gh(sp * sp);
    nspb::gram(dW, sp, sp, dW, sp, sp, n, dG, sp, dws, st);
    cudaMemcpy(Gh.data(), dG, sp * sp * 8, cudaMemcpyDeviceToHost);
    std::vector<double> T(sp * sp), Di(sp * sp);
    nspb::small_chol(dG, sp, 1, sp, 1e-14, dT, dst, st); cudaMemcpy(T.data(), dT, sp * sp * 8, cudaMemcpyDeviceToHost);
    nspb::small_chol(dG, sp, 0, -1, 0.0, dT, dst, st); cudaMemcpy(Di.data(), dT, sp * sp * 8, cudaMemcpyDeviceToHost);
    double e1 = 0, e2 = 0;
    for (int i = 0; i < sp; ++i) for (int j = 0; j < sp; ++j) {
      double a = 0, b = 0;
      for (int k = 0; k < sp; ++k) { b += Di[i * sp + k] * Gh[k * sp + j]; }
      for (int k = 0; k < sp; ++k) for (int l = 0; l < sp; ++l) a += T[k * sp + i] * Gh[k * sp + l] * T[l * sp + j];
      e1 = std::max(e1, std::abs(a - (i == j))); e2 = std::max(e2, std::abs(b - (i == j)));
    }
    printf("check T^T G T - I: %.3e   Dinv G - I: %.3e  (%s)\n", e1, e2, cudaGetErrorString(cudaGetLastError()));
  }
  timeit("gram WtW", [&] { nspb::gram(dW, sp, sp, dW, sp, sp, n, dG, sp, dws, st); });
  timeit("gram2 P[Q|R]", [&] { nspb::gram2(dW, sp, sp, dW, dP, sp, sp, n, dG, dT, sp, dws, st); });
  timeit("small_chol mode1", [&] { nspb::small_chol(dG, sp, 1, sp, 1e-14, dT, dst, st); });
  timeit("small_chol mode0", [&] { nspb::small_chol(dG, sp, 0, -1, 0.0, dT, dst, st); });
  timeit("small_eig gated", [&] { nspb::small_eig(dG, sp, sp, dP, sp + 1, dT, dT, &dst->fallback, st); });
  timeit("panel n x s", [&] { nspb::panel(dP, sp, nullptr, 0, dW, sp, dT, sp, sp, sp, n, 1.0, nullptr, st); });
  timeit("panel s x s", [&] { nspb::panel(dP, sp, nullptr, 0, dG, sp, dT, sp, sp, sp, sp, 1.0, nullptr, st); });
  h.fallback = 1; cudaMemcpy(dst, &h, sizeof(h), cudaMemcpyHostToDevice);
  timeit("small_eig (run)", [&] { nspb::small_eig(dG, sp, sp, dP, sp + 1, dT, dT, nullptr, st); });
  return 0;
}
