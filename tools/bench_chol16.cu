// Phase timing (clock64) and wall timing of the s x s Cholesky kernels (diagnostics).
#define NSP_CHOL_PROF
#include <cstdio>
#include <vector>
#include <random>
#include <cmath>
#include <algorithm>
#include "../paper_2101_12164_b200/csrc/nsp_blas.cu"
#include "../paper_2101_12164_b200/csrc/nsp_small.cu"
void nsp_count_launch() {}
void nsp_count_path(int) {}
thread_local int nsp_force_generic = 0;
int main() {
  const int sp = 128; const int64_t n = 4096;
  std::vector<double> W(n * sp);
  std::mt19937_64 g(1); std::normal_distribution<double> nd;
  for (auto& x : W) x = nd(g);
  double *dW, *dG, *dL, *dT, *dws; BcgStatus* dst;
  cudaMalloc(&dW, n * sp * 8); cudaMalloc(&dG, sp * sp * 8); cudaMalloc(&dL, sp * sp * 8); cudaMalloc(&dT, sp * sp * 8);
  cudaMalloc(&dws, nspb::gram_ws_doubles(n, sp, sp) * 8); cudaMalloc(&dst, sizeof(BcgStatus));
  cudaMemcpy(dW, W.data(), n * sp * 8, cudaMemcpyHostToDevice);
  BcgStatus h{}; h.width = sp; cudaMemcpy(dst, &h, sizeof(h), cudaMemcpyHostToDevice);
  cudaStream_t st; cudaStreamCreate(&st);
  nspb::gram(dW, sp, sp, dW, sp, sp, n, dG, sp, dws, st);
  std::vector<double> Gh(sp * sp), T(sp * sp), Di(sp * sp);
  cudaMemcpy(Gh.data(), dG, sp * sp * 8, cudaMemcpyDeviceToHost);
  nspb::chol_fac(dG, sp, 1, sp, 1e-14, dL, dst, st);
  nspb::chol_solve(dL, sp, nullptr, 0, dT, sp, 1.0, false, true, &dst->fallback, st);
  cudaMemcpy(T.data(), dT, sp * sp * 8, cudaMemcpyDeviceToHost);
  nspb::chol_fac(dG, sp, 0, -1, 0.0, dL, dst, st);
  nspb::chol_solve(dL, sp, dG, sp, dT, sp, 1.0, true, true, nullptr, st);
  cudaMemcpy(Di.data(), dT, sp * sp * 8, cudaMemcpyDeviceToHost);
  BcgStatus hb; cudaMemcpy(&hb, dst, sizeof(hb), cudaMemcpyDeviceToHost);
  double e1 = 0, e2 = 0;
  for (int i = 0; i < sp; ++i) for (int j = 0; j < sp; ++j) {
    double a = 0;
    for (int k = 0; k < sp; ++k) for (int l = 0; l < sp; ++l) a += T[k * sp + i] * Gh[k * sp + l] * T[l * sp + j];
    e1 = std::max(e1, std::abs(a - (i == j))); e2 = std::max(e2, std::abs(Di[i * sp + j] - (i == j)));
  }
  printf("check T^T G T - I: %.3e   chol_solve(G) - I: %.3e  fallback %d indef %d width %d (%s)\n", e1, e2,
         hb.fallback, hb.indefinite, hb.width, cudaGetErrorString(cudaGetLastError()));
  for (int r = 0; r < 3; ++r) nspb::chol_fac(dG, sp, 1, sp, 1e-14, dL, dst, st);
  cudaStreamSynchronize(st);
  long long pr[128];
  cudaMemcpyFromSymbol(pr, g_chol_prof, sizeof(pr));
  printf("warp_chol16 (block 1): load %lld  columns %lld  X %lld\n", pr[65] - pr[64], pr[66] - pr[65], pr[67] - pr[66]);
  printf("load %lld\n", pr[1] - pr[0]);
  long long prev = pr[1];
  for (int s = 0; s < 8; ++s) { printf("step %d: C+A %lld  panel %lld\n", s, pr[2 + 2 * s] - prev, pr[3 + 2 * s] - pr[2 + 2 * s]); prev = pr[3 + 2 * s]; }
  printf("store %lld total %lld cycles\n", pr[40] - prev, pr[40] - pr[0]);
  cudaEvent_t e0, ev1; cudaEventCreate(&e0); cudaEventCreate(&ev1);
  auto timeit = [&](const char* name, auto fn) {
    for (int i = 0; i < 3; ++i) fn();
    cudaEventRecord(e0, st);
    for (int i = 0; i < 50; ++i) fn();
    cudaEventRecord(ev1, st); cudaEventSynchronize(ev1);
    float ms; cudaEventElapsedTime(&ms, e0, ev1);
    printf("%-22s %8.2f us per launch (back-to-back, includes launch gaps)\n", name, ms * 1000 / 50);
  };
  {  // fused chol + solve against the two-launch form
    double *dA2, *dT2;
    cudaMalloc(&dA2, sp * sp * 8); cudaMalloc(&dT2, sp * sp * 8);
    std::vector<double> a(sp * sp), b(sp * sp);
    nspb::chol_fac(dG, sp, 0, -1, 0.0, dL, dst, st);
    nspb::chol_solve(dL, sp, dG, sp, dT, sp, 1.0, true, true, nullptr, st);
    nspb::chol_fac_solve(dG, sp, 0, -1, 0.0, dL, dst, dG, sp, dT2, sp, 1.0, true, true, st);
    cudaMemcpy(a.data(), dT, sp * sp * 8, cudaMemcpyDeviceToHost);
    cudaMemcpy(b.data(), dT2, sp * sp * 8, cudaMemcpyDeviceToHost);
    double m0 = 0; for (int i = 0; i < sp * sp; ++i) m0 = std::max(m0, std::abs(a[i] - b[i]));
    nspb::chol_fac(dG, sp, 1, sp, 1e-14, dL, dst, st);
    nspb::chol_solve(dL, sp, nullptr, 0, dT, sp, 1.0, false, true, &dst->fallback, st);
    nspb::chol_fac_solve(dG, sp, 1, sp, 1e-14, dL, dst, nullptr, 0, dT2, sp, 1.0, false, true, st);
    cudaMemcpy(a.data(), dT, sp * sp * 8, cudaMemcpyDeviceToHost);
    cudaMemcpy(b.data(), dT2, sp * sp * 8, cudaMemcpyDeviceToHost);
    double m1 = 0; for (int i = 0; i < sp * sp; ++i) m1 = std::max(m1, std::abs(a[i] - b[i]));
    printf("fused vs two-launch: D^-1 G max diff %.3e, T max diff %.3e (%s)\n", m0, m1,
           cudaGetErrorString(cudaGetLastError()));
    timeit("chol_fac_solve mode0", [&] { nspb::chol_fac_solve(dG, sp, 0, -1, 0.0, dL, dst, dG, sp, dT2, sp, 1.0, true, true, st); });
    timeit("chol_fac_solve mode1", [&] { nspb::chol_fac_solve(dG, sp, 1, sp, 1e-14, dL, dst, nullptr, 0, dT2, sp, 1.0, false, true, st); });
  }
  timeit("chol_fac mode1", [&] { nspb::chol_fac(dG, sp, 1, sp, 1e-14, dL, dst, st); });
  timeit("chol_solve fwd+bwd", [&] { nspb::chol_solve(dL, sp, dG, sp, dT, sp, 1.0, true, true, nullptr, st); });
  timeit("chol_solve bwd(I)", [&] { nspb::chol_solve(dL, sp, nullptr, 0, dT, sp, 1.0, false, true, nullptr, st); });
  timeit("small_chol mode0 (old)", [&] { nspb::small_chol(dG, sp, 0, -1, 0.0, dT, dst, st); });
  timeit("small_chol mode1 (old)", [&] { nspb::small_chol(dG, sp, 1, sp, 1e-14, dT, dst, st); });
  timeit("panel s x s (old alpha)", [&] { nspb::panel(dT, sp, nullptr, 0, dG, sp, dL, sp, sp, sp, sp, 1.0, nullptr, st); });
  timeit("empty-ish (sqrt_vec)", [&] { nspb::sqrt_vec(dT, dT, 1, st); });
  return 0;
}
