// Gram with the FULL 128 x 128 output per CTA (16 warps, 32 x 32 per warp: 16 DMMA per 8 fragment
// loads), each row slab read once, 3-stage cp.async ring, cluster-of-8 DSMEM reduction of the partials,
// then a small fixed-order reduce of the 18 cluster partials.  vs the library gram (cfg2 shapes).
#include <cstdio>
#include <vector>
#include <random>
#include <cmath>
#include <algorithm>
#include <cooperative_groups.h>
#include "../paper_2101_12164_b200/csrc/nsp_blas.cu"
namespace cg = cooperative_groups;
void nsp_count_launch() {}
namespace {
constexpr int SLR = 32;      // rows per slab
constexpr int LD = 132;      // padded row stride (128 + 4)
constexpr int NST = 3;       // stages
constexpr int CLS = 8;       // cluster size
__global__ void __cluster_dims__(CLS, 1, 1) __launch_bounds__(512)
k_gram_full(const double* __restrict__ A, const double* __restrict__ B, int64_t n, int64_t rpc, double* __restrict__ part) {
  extern __shared__ __align__(16) double sm[];
  constexpr int OPS = SLR * LD;
  constexpr int STG = 2 * OPS;
  const int64_t r0 = blockIdx.x * rpc, r1 = min(n, r0 + rpc);
  const int nslab = r1 > r0 ? (int)((r1 - r0 + SLR - 1) / SLR) : 0;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, t = lane & 3;
  const int m0 = (warp >> 2) * 32, n0 = (warp & 3) * 32;
  auto issue = [&](int q) {
    double* st = sm + (q % NST) * STG;
    const int64_t r = r0 + (int64_t)q * SLR;
    const int64_t nv = r1 - r;
    for (int e = tid; e < SLR * 64; e += 512) {   // 32 rows x 64 16-byte chunks per operand
      const int rr = e >> 6, q2 = e & 63;
      const bool v = rr < nv;
      const int64_t off = v ? (r + rr) * 128 + 2 * q2 : 0;
      unsigned sa = (unsigned)__cvta_generic_to_shared(st + rr * LD + 2 * q2);
      unsigned sb = (unsigned)__cvta_generic_to_shared(st + OPS + rr * LD + 2 * q2);
      int sz = v ? 16 : 0;
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(sa), "l"(A + off), "r"(sz));
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(sb), "l"(B + off), "r"(sz));
    }
  };
  for (int q = 0; q < NST - 1; ++q) {
    if (q < nslab) issue(q);
    cp_commit();
  }
  double acc[4][4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  for (int q = 0; q < nslab; ++q) {
    cp_wait<NST - 2>();
    __syncthreads();
    if (q + NST - 1 < nslab) issue(q + NST - 1);
    cp_commit();
    const double* As = sm + (q % NST) * STG;
    const double* Bs = As + OPS;
#pragma unroll 2
    for (int k = 0; k < SLR; k += 4) {
      double a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = As[(k + t) * LD + m0 + 8 * i + g];   // A^T: A[m][k] = X[k][m]
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = Bs[(k + t) * LD + n0 + 8 * j + g];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) dmma(acc[i][j][0], acc[i][j][1], a[i], b[j]);
    }
  }
  cp_wait<0>();
  __syncthreads();
  // partial 128 x 128 to smem (row-major, ld 128), then cluster reduction over DSMEM in rank order
  double* P = sm;
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int rr = m0 + 8 * i + g, cc = n0 + 8 * j + 2 * t;
      P[rr * 128 + cc] = acc[i][j][0];
      P[rr * 128 + cc + 1] = acc[i][j][1];
    }
  cg::cluster_group cl = cg::this_cluster();
  cl.sync();
  const int rank = cl.block_rank();
  // this CTA reduces rows [16 rank, 16 rank + 16): 2048 doubles, 4 per thread
  double* out = part + (int64_t)(blockIdx.x / CLS) * 16384;
  for (int e = tid; e < 2048; e += 512) {
    const int idx = rank * 2048 + e;
    double s = 0.0;
#pragma unroll
    for (int c = 0; c < CLS; ++c) s += cl.map_shared_rank(P, c)[idx];
    out[idx] = s;
  }
  cl.sync();
}
__global__ void k_gram_full_reduce(const double* __restrict__ part, int np, double* __restrict__ out, int ldo) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= 16384) return;
  double s = 0.0;
  for (int p = 0; p < np; ++p) s += part[(int64_t)p * 16384 + e];
  out[(e >> 7) * ldo + (e & 127)] = s;
}
}  // namespace
int main() {
  const int64_t n = 14287; const int sp = 128;
  std::vector<double> X(n * sp), Y(n * sp);
  std::mt19937_64 gg(1); std::normal_distribution<double> nd;
  for (auto& x : X) x = nd(gg);
  for (auto& x : Y) x = nd(gg);
  double *dX, *dY, *dG1, *dG2, *dws, *dpart;
  cudaMalloc(&dX, X.size() * 8); cudaMalloc(&dY, Y.size() * 8);
  cudaMalloc(&dG1, sp * sp * 8); cudaMalloc(&dG2, sp * sp * 8);
  cudaMalloc(&dws, nspb::gram_ws_doubles(n, sp, sp) * 8); cudaMalloc(&dpart, 32 * 16384 * 8);
  cudaMemcpy(dX, X.data(), X.size() * 8, cudaMemcpyHostToDevice); cudaMemcpy(dY, Y.data(), Y.size() * 8, cudaMemcpyHostToDevice);
  cudaStream_t st; cudaStreamCreate(&st);
  const int nblk = 144;
  int64_t rpc = (n + nblk - 1) / nblk;
  const size_t smem = NST * 2 * SLR * LD * 8;
  printf("smem %zu\n", smem);
  cudaFuncSetAttribute(k_gram_full, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  auto full = [&] {
    k_gram_full<<<nblk, 512, smem, st>>>(dX, dY, n, rpc, dpart);
    k_gram_full_reduce<<<64, 256, 0, st>>>(dpart, nblk / CLS, dG2, sp);
  };
  nspb::gram(dX, sp, sp, dY, sp, sp, n, dG1, sp, dws, st);
  full();
  cudaStreamSynchronize(st);
  printf("launch: %s\n", cudaGetErrorString(cudaGetLastError()));
  std::vector<double> G1(sp * sp), G2(sp * sp);
  cudaMemcpy(G1.data(), dG1, G1.size() * 8, cudaMemcpyDeviceToHost); cudaMemcpy(G2.data(), dG2, G2.size() * 8, cudaMemcpyDeviceToHost);
  double md = 0, mx = 0; for (int i = 0; i < sp * sp; ++i) { md = std::max(md, std::fabs(G1[i] - G2[i])); mx = std::max(mx, std::fabs(G1[i])); }
  printf("full-tile gram vs library: max |diff| / max %.3e\n", md / mx);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  auto timeit = [&](const char* name, auto fn) {
    for (int i = 0; i < 3; ++i) fn();
    cudaEventRecord(e0, st);
    for (int i = 0; i < 20; ++i) fn();
    cudaEventRecord(e1, st); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("%-40s %8.2f us\n", name, ms * 1000 / 20);
  };
  timeit("library gram", [&] { nspb::gram(dX, sp, sp, dY, sp, sp, n, dG1, sp, dws, st); });
  timeit("full-tile gram + cluster reduce", full);
  timeit("  (partial kernel only)", [&] { k_gram_full<<<nblk, 512, smem, st>>>(dX, dY, n, rpc, dpart); });
  return 0;
}
