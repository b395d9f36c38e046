// k_symm microbenchmark on cfg2-like shapes (64 blocks x 7 tile rows, s = 128): compile with
// -DNSP_DMMA_VOLATILE / -DNSP_MMA_PIPE to compare variants (diagnostics).
#include <cstdio>
#include <vector>
#include <random>
#include "../paper_2101_12164_b200/csrc/nsp_kernels.cu"
void nsp_count_launch() {}
int main(int argc, char** argv) {
  const int nsub = 64, ntb = 7, ld = 128;
  std::vector<FacSub> subs(nsub);
  std::vector<int2> items;
  int64_t dense_tiles = 0, rows = 0;
  for (int j = 0; j < nsub; ++j) {
    FacSub f{}; f.ntb = ntb; f.dense_off = dense_tiles; f.wvu_row = rows; f.b = ntb * 64;
    subs[j] = f; dense_tiles += ntb * (ntb + 1) / 2; rows += ntb * 64;
    for (int I = 0; I < ntb; ++I) items.push_back(make_int2(j, I));
  }
  std::vector<double> M(dense_tiles * NSP_MINV_TILE), W(rows * ld);
  std::mt19937_64 g(1); std::normal_distribution<double> nd;
  for (auto& x : M) x = nd(g);
  for (auto& x : W) x = nd(g);
  FacSub* dsub; int2* dit; double *dM, *dW, *dU, *flush;
  cudaMalloc(&dsub, nsub * sizeof(FacSub)); cudaMalloc(&dit, items.size() * sizeof(int2));
  cudaMalloc(&dM, M.size() * 8); cudaMalloc(&dW, W.size() * 8); cudaMalloc(&dU, W.size() * 8);
  cudaMalloc(&flush, 256 << 20);
  cudaMemcpy(dsub, subs.data(), nsub * sizeof(FacSub), cudaMemcpyHostToDevice);
  cudaMemcpy(dit, items.data(), items.size() * sizeof(int2), cudaMemcpyHostToDevice);
  cudaMemcpy(dM, M.data(), M.size() * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(dW, W.data(), W.size() * 8, cudaMemcpyHostToDevice);
  cudaStream_t st; cudaStreamCreate(&st);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const double flops = 2.0 * nsub * (ntb * 64.0) * (ntb * 64.0) * ld;
  for (int nit : {74, 148, 222, 296, 370, 444, 448}) {
    float best = 1e9;
    for (int r = 0; r < 8; ++r) {
      cudaMemsetAsync(flush, r, 256 << 20, st);
      cudaEventRecord(e0, st);
      nspk::symm(dsub, dit, nit, dM, dW, dU, ld, 32, st);
      cudaEventRecord(e1, st); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      if (r >= 3) best = std::min(best, ms);
    }
    printf("items %d (CTAs %d, waves %.2f): %.1f us, %.2f us per CTA-wave\n", nit, 4 * nit, 4.0 * nit / 296, best * 1e3,
           best * 1e3 / ((4 * nit + 295) / 296));
  }
  for (int cw : {64, 32}) {
    float best = 1e9, tot = 0;
    for (int r = 0; r < 13; ++r) {
      cudaMemsetAsync(flush, r, 256 << 20, st);
      cudaEventRecord(e0, st);
      nspk::symm(dsub, dit, (int)items.size(), dM, dW, dU, ld, cw, st);
      cudaEventRecord(e1, st); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      if (r >= 3) { best = std::min(best, ms); tot += ms; }
    }
    printf("%s%s cw %d: best %.1f us (%.2f TFLOP/s), mean %.1f us  %s\n", VARIANT, "", cw, best * 1e3,
           flops / (best * 1e-3) / 1e12, tot / 10 * 1e3, cudaGetErrorString(cudaGetLastError()));
  }
  // checksum
  std::vector<double> U(W.size()); cudaMemcpy(U.data(), dU, U.size() * 8, cudaMemcpyDeviceToHost);
  double cs = 0; for (size_t i = 0; i < U.size(); i += 997) cs += U[i];
  printf("checksum %.12e\n", cs);
  return 0;
}
