// Old vs 148-SM-balanced tall-skinny kernels: correctness and timing (diagnostics).
#include <cstdio>
#include <vector>
#include <random>
#include <cmath>
#include <algorithm>
#include "../paper_2101_12164_b200/csrc/nsp_blas.cu"
#include "nsp_ts_experiment.cu"
void nsp_count_launch() {}
int main() {
  for (int sp : {128, 64}) {
  const int64_t n = 14287;
  std::vector<double> Wh(n * sp), Ph(n * sp), Mh(sp * sp);
  std::mt19937_64 g(1); std::normal_distribution<double> nd;
  for (auto& x : Wh) x = nd(g);
  for (auto& x : Ph) x = nd(g);
  for (auto& x : Mh) x = nd(g);
  double *dW, *dP, *dM, *dO1, *dO2, *dG1, *dG2, *dws, *dnp1, *dnp2, *dr1, *dr2;
  cudaMalloc(&dW, n * sp * 8); cudaMalloc(&dP, n * sp * 8); cudaMalloc(&dM, sp * sp * 8);
  cudaMalloc(&dO1, n * sp * 8); cudaMalloc(&dO2, n * sp * 8); cudaMalloc(&dG1, 2 * sp * sp * 8); cudaMalloc(&dG2, 2 * sp * sp * 8);
  size_t wsd = std::max(nspb::gram_ws_doubles(n, sp, sp), nspb::ts_gram_ws_doubles(sp, sp));
  cudaMalloc(&dws, wsd * 8); cudaMalloc(&dnp1, ((n + 7) / 8 + 1) * sp * 8); cudaMalloc(&dnp2, ((n + 7) / 8 + 1) * sp * 8);
  cudaMalloc(&dr1, sp * 8); cudaMalloc(&dr2, sp * 8);
  cudaMemcpy(dW, Wh.data(), n * sp * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(dP, Ph.data(), n * sp * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(dM, Mh.data(), sp * sp * 8, cudaMemcpyHostToDevice);
  cudaStream_t st; cudaStreamCreate(&st);
  auto cmp = [&](const char* nm, double* a, double* b, size_t cnt) {
    std::vector<double> x(cnt), y(cnt); cudaMemcpy(x.data(), a, cnt * 8, cudaMemcpyDeviceToHost); cudaMemcpy(y.data(), b, cnt * 8, cudaMemcpyDeviceToHost);
    double num = 0, den = 0; for (size_t i = 0; i < cnt; ++i) { num += (x[i] - y[i]) * (x[i] - y[i]); den += y[i] * y[i]; }
    printf("sp %d %-12s rel diff %.3e\n", sp, nm, std::sqrt(num / den));
  };
  nspb::gram(dW, sp, sp, dW, sp, sp, n, dG1, sp, dws, st);
  nspb::ts_gram(dW, sp, sp, dW, sp, sp, n, true, dG2, sp, dws, st);
  cmp("gram sym", dG2, dG1, sp * sp);
  nspb::gram2(dW, sp, sp, dP, dW, sp, sp, n, dG1, dG1 + sp * sp, sp, dws, st);
  nspb::ts_gram2(dW, sp, sp, dP, dW, sp, sp, n, dG2, dG2 + sp * sp, sp, dws, st);
  cmp("gram2", dG2, dG1, 2 * sp * sp);
  PanelArgs a0{dO1, sp, dP, sp, dW, sp, dM, sp, -1.0, nullptr};
  nspb::panel(dO1, sp, dP, sp, dW, sp, dM, sp, sp, sp, n, -1.0, dnp1, st);
  nspb::colsq_reduce(dnp1, (int)((n + 63) / 64), sp, dr1, st);
  PanelArgs b0{dO2, sp, dP, sp, dW, sp, dM, sp, -1.0, dnp2};
  nspb::ts_panel2(b0, nullptr, sp, sp, n, st);
  nspb::colsq_reduce(dnp2, (int)((n + 7) / 8), sp, dr2, st);
  cmp("panel", dO2, dO1, n * sp);
  cmp("colsq", dr2, dr1, sp);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  auto timeit = [&](const char* name, auto fn) {
    for (int i = 0; i < 3; ++i) fn();
    cudaEventRecord(e0, st);
    for (int i = 0; i < 20; ++i) fn();
    cudaEventRecord(e1, st); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("sp %d %-22s %8.2f us (%s)\n", sp, name, ms * 1000 / 20, cudaGetErrorString(cudaGetLastError()));
  };
  timeit("gram (old)", [&] { nspb::gram(dW, sp, sp, dW, sp, sp, n, dG1, sp, dws, st); });
  timeit("ts_gram sym", [&] { nspb::ts_gram(dW, sp, sp, dW, sp, sp, n, true, dG2, sp, dws, st); });
  timeit("ts_gram", [&] { nspb::ts_gram(dW, sp, sp, dP, sp, sp, n, false, dG2, sp, dws, st); });
  timeit("gram2 (old)", [&] { nspb::gram2(dW, sp, sp, dP, dW, sp, sp, n, dG1, dG1 + sp * sp, sp, dws, st); });
  timeit("ts_gram2", [&] { nspb::ts_gram2(dW, sp, sp, dP, dW, sp, sp, n, dG2, dG2 + sp * sp, sp, dws, st); });
  PanelArgs x0{dO1, sp, dO1, sp, dW, sp, dM, sp, 1.0, nullptr}, x1{dO2, sp, dO2, sp, dP, sp, dM, sp, -1.0, dnp1};
  timeit("panel2 (old)", [&] { nspb::panel2(x0, &x1, sp, sp, n, st); });
  PanelArgs y1{dO2, sp, dO2, sp, dP, sp, dM, sp, -1.0, dnp2};
  timeit("ts_panel2", [&] { nspb::ts_panel2(x0, &y1, sp, sp, n, st); });
  timeit("panel (old)", [&] { nspb::panel(dO1, sp, nullptr, 0, dW, sp, dM, sp, sp, sp, n, 1.0, nullptr, st); });
  PanelArgs z0{dO1, sp, nullptr, 0, dW, sp, dM, sp, 1.0, nullptr};
  timeit("ts_panel", [&] { nspb::ts_panel2(z0, nullptr, sp, sp, n, st); });
  }
  return 0;
}
