// Gram partials on a chunk-major padded layout (32-column chunks, 36 doubles per row: [chunk][row][36])
// fed by TMA bulk copies (one per chunk per slab) vs the library's k_gram_partial on row-major blocks.
// Diagnostics for the block-CG state layout (cfg2 shapes: n = 14287, s = 128).
#include <cstdio>
#include <vector>
#include <random>
#include <cmath>
#include <algorithm>
#include "../paper_2101_12164_b200/csrc/nsp_blas.cu"
void nsp_count_launch() {}
namespace {
constexpr int CL = 36;            // chunk row stride
constexpr int SL = 32;            // slab rows
constexpr int NSG = 4;            // stages
// partial (64 x 64 tile (tm, tn)) over a row chunk; A, B chunk-major with n rows
__global__ void __launch_bounds__(256) k_gram_cm(const double* __restrict__ A, const double* __restrict__ B, int64_t n,
                                                 int64_t rpc, double* __restrict__ part, int ntm, int ntn) {
  extern __shared__ __align__(128) double sm[];
  constexpr int OPS = 2 * SL * CL;        // one operand slab: 2 chunks x 32 rows x 36
  constexpr int STG = 2 * OPS;
  __shared__ __align__(8) uint64_t bar[NSG];
  const int tile = blockIdx.x, tm = tile / ntn, tn = tile - tm * ntn;
  const int64_t r0 = blockIdx.y * rpc, r1 = min(n, r0 + rpc);
  const int nslab = r1 > r0 ? (int)((r1 - r0 + SL - 1) / SL) : 0;
  if (threadIdx.x == 0) {
    for (int i = 0; i < NSG; ++i) mbar_init(&bar[i], 1);
    fence_mbar_init();
  }
  __syncthreads();
  auto issue = [&](int q) {   // thread 0: 4 bulk copies (A chunks 2tm, 2tm+1; B chunks 2tn, 2tn+1)
    double* st = sm + (q % NSG) * STG;
    const int64_t r = r0 + (int64_t)q * SL;
    const int rows = (int)(r1 - r < SL ? r1 - r : SL);
    const unsigned bytes = rows * CL * 8;
    fence_proxy_async();
    mbar_expect_copy(&bar[q % NSG], st, A + (2 * tm) * n * CL + r * CL, bytes);
    mbar_add_copy(&bar[q % NSG], st + SL * CL, A + (2 * tm + 1) * n * CL + r * CL, bytes);
    mbar_add_copy(&bar[q % NSG], st + OPS, B + (2 * tn) * n * CL + r * CL, bytes);
    mbar_add_copy(&bar[q % NSG], st + OPS + SL * CL, B + (2 * tn + 1) * n * CL + r * CL, bytes);
  };
  if (threadIdx.x == 0)
    for (int q = 0; q < NSG - 1 && q < nslab; ++q) issue(q);
  double acc[2][4][2];
  acc_zero(acc);
  const int warp = threadIdx.x >> 5;
  const int m0 = (warp >> 1) * 16, n0 = (warp & 1) * 32;
  const int ca = m0 >> 5, cb = n0 >> 5;
  for (int q = 0; q < nslab; ++q) {
    mbar_wait(&bar[q % NSG], (q / NSG) & 1);
    __syncthreads();
    if (threadIdx.x == 0 && q + NSG - 1 < nslab) issue(q + NSG - 1);
    const double* st = sm + (q % NSG) * STG;
    const int64_t r = r0 + (int64_t)q * SL;
    const int rows = (int)(r1 - r < SL ? r1 - r : SL);
    const int K = (rows + 3) & ~3;   // (ragged last slab: rows beyond `rows` hold stale data -> zero them first)
    if (rows < SL) {   // zero-fill stale rows of this stage (generic proxy; the stage is re-armed later)
      for (int e = threadIdx.x; e < (SL - rows) * 4 * CL; e += 256) {
        const int part4 = e / ((SL - rows) * CL), w = e - part4 * (SL - rows) * CL;
        double* base = (double*)st + part4 * SL * CL;   // A0, A1, B0, B1 chunk slabs
        base[rows * CL + w] = 0.0;
      }
      __syncthreads();
    }
    // per-warp chunk base: A[m][k] = As[k * 36 + (m - 32 ca)], B[k][n] likewise
    const double* Aw = st + ca * SL * CL - 32 * ca;
    const double* Bw = st + OPS + cb * SL * CL - 32 * cb;
    cta_mma<4, true, false>(Aw, CL, Bw, CL, acc, K);
  }
  double* out = part + ((int64_t)blockIdx.y * ntm * ntn + tile) * 4096;
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int rr = acc_row<4>(i), cc = acc_col<4>(j);
      *reinterpret_cast<double2*>(out + rr * 64 + cc) = make_double2(acc[i][j][0], acc[i][j][1]);
    }
}
}  // namespace
int main() {
  const int64_t n = 14287; const int sp = 128;
  std::vector<double> X(n * sp), Y(n * sp);
  std::mt19937_64 g(1); std::normal_distribution<double> nd;
  for (auto& x : X) x = nd(g);
  for (auto& x : Y) x = nd(g);
  std::vector<double> Xc(4 * n * CL, 0.0), Yc(4 * n * CL, 0.0);
  for (int64_t r = 0; r < n; ++r) for (int c = 0; c < sp; ++c) { Xc[(c / 32) * n * CL + r * CL + c % 32] = X[r * sp + c]; Yc[(c / 32) * n * CL + r * CL + c % 32] = Y[r * sp + c]; }
  double *dX, *dY, *dXc, *dYc, *dG1, *dG2, *dws, *dws2;
  cudaMalloc(&dX, X.size() * 8); cudaMalloc(&dY, Y.size() * 8); cudaMalloc(&dXc, Xc.size() * 8); cudaMalloc(&dYc, Yc.size() * 8);
  cudaMalloc(&dG1, sp * sp * 8); cudaMalloc(&dG2, sp * sp * 8);
  size_t wsd = nspb::gram_ws_doubles(n, sp, sp);
  cudaMalloc(&dws, wsd * 8); cudaMalloc(&dws2, wsd * 8);
  cudaMemcpy(dX, X.data(), X.size() * 8, cudaMemcpyHostToDevice); cudaMemcpy(dY, Y.data(), Y.size() * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(dXc, Xc.data(), Xc.size() * 8, cudaMemcpyHostToDevice); cudaMemcpy(dYc, Yc.data(), Yc.size() * 8, cudaMemcpyHostToDevice);
  cudaStream_t st; cudaStreamCreate(&st);
  const int ntm = 2, ntn = 2, nch = nspb::gram_chunks(n, 4);
  int64_t rpc = (n + nch - 1) / nch; rpc = ((rpc + SL - 1) / SL) * SL;
  const size_t smem = NSG * 2 * 2 * SL * CL * 8;
  cudaFuncSetAttribute(k_gram_cm, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  auto cm = [&] {
    k_gram_cm<<<dim3(4, nch), 256, smem, st>>>(dXc, dYc, n, rpc, dws2, ntm, ntn);
    k_gram_reduce<<<dim3(ntn * 4, ntm * 4), dim3(16, 16, 4), 0, st>>>(dws2, nch, ntm, ntn, ntn, dG2, nullptr, sp);
  };
  nspb::gram(dX, sp, sp, dY, sp, sp, n, dG1, sp, dws, st);
  cm();
  std::vector<double> G1(sp * sp), G2(sp * sp);
  cudaMemcpy(G1.data(), dG1, G1.size() * 8, cudaMemcpyDeviceToHost); cudaMemcpy(G2.data(), dG2, G2.size() * 8, cudaMemcpyDeviceToHost);
  double md = 0, mx = 0; for (int i = 0; i < sp * sp; ++i) { md = std::max(md, std::fabs(G1[i] - G2[i])); mx = std::max(mx, std::fabs(G1[i])); }
  printf("chunk-major TMA gram vs library: max |diff| / max %.3e (%s)\n", md / mx, cudaGetErrorString(cudaGetLastError()));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  auto timeit = [&](const char* name, auto fn) {
    for (int i = 0; i < 3; ++i) fn();
    cudaEventRecord(e0, st);
    for (int i = 0; i < 20; ++i) fn();
    cudaEventRecord(e1, st); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("%-34s %8.2f us\n", name, ms * 1000 / 20);
  };
  timeit("library gram (row-major, cp.async)", [&] { nspb::gram(dX, sp, sp, dY, sp, sp, n, dG1, sp, dws, st); });
  timeit("chunk-major gram (TMA)", cm);
  return 0;
}
