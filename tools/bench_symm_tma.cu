// k_symm variant: the S_j^{-1} tiles stored PADDED (64 x 68) in global memory so that each stage's
// M tile is ONE 34.8 KB bulk copy (TMA, mbarrier) instead of 2048 cp.async; W tiles stay cp.async.
// Diagnostics: compares against nspk::symm on cfg2-like shapes (64 blocks x 7 tile rows, s = 128).
#include <cstdio>
#include <vector>
#include <random>
#include "../paper_2101_12164_b200/csrc/nsp_kernels.cu"
void nsp_count_launch() {}
constexpr int LDP = 68;
constexpr int TPAD = 64 * LDP;
template <int CW>
__global__ void __launch_bounds__(256) k_symm_t(const FacSub* __restrict__ subs, const int2* __restrict__ items,
                                                const double* __restrict__ minvp, const double* __restrict__ W,
                                                double* __restrict__ U, int ldw) {
  constexpr int NF = CW / 16;
  constexpr int LDV = CW + 4;
  constexpr int STAGE = TPAD + 64 * LDV;
  extern __shared__ __align__(128) double sm[];
  __shared__ __align__(8) uint64_t bar[2];
  const int2 it = items[blockIdx.x];
  const FacSub sb = subs[it.x];
  const int I = it.y, ntb = sb.ntb;
  const int c0 = blockIdx.y * CW;
  const double* Mb = minvp + sb.dense_off * TPAD;
  const double* Wb = W + sb.wvu_row * (int64_t)ldw + c0;
  auto mt = [&](int J) {
    return J <= I ? Mb + ((int64_t)I * (I + 1) / 2 + J) * TPAD : Mb + ((int64_t)J * (J + 1) / 2 + I) * TPAD;
  };
  if (threadIdx.x == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    fence_mbar_init();
  }
  __syncthreads();
  auto issue = [&](int J) {
    double* Ms = sm + (J & 1) * STAGE;
    if (threadIdx.x == 0) {
      fence_proxy_async();
      mbar_expect_copy(&bar[J & 1], Ms, mt(J), TPAD * 8);
    }
    cp_block(Ms + TPAD, LDV, Wb + (int64_t)J * 64 * ldw, ldw, 64, CW);
  };
  double acc[2][NF][2];
  acc_zero(acc);
  issue(0);
  cp_commit();
  for (int J = 0; J < ntb; ++J) {
    cp_wait<0>();
    mbar_wait(&bar[J & 1], (J >> 1) & 1);
    __syncthreads();
    if (J + 1 < ntb) issue(J + 1);
    cp_commit();
    const double* Ms = sm + (J & 1) * STAGE;
    if (J <= I) cta_mma<NF, false, false>(Ms, LDP, Ms + TPAD, LDV, acc);
    else cta_mma<NF, true, false>(Ms, LDP, Ms + TPAD, LDV, acc);
  }
  double* out = U + (sb.wvu_row + (int64_t)I * 64) * ldw + c0;
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < NF; ++j) {
      const int r = acc_row<NF>(i), c = acc_col<NF>(j);
      *reinterpret_cast<double2*>(out + (int64_t)r * ldw + c) = make_double2(acc[i][j][0], acc[i][j][1]);
    }
}
// both operands by TMA: W stored chunk-major padded ([chunk][row][36]) so a 64 x 32 W tile is contiguous
template <int CW>
__global__ void __launch_bounds__(256) k_symm_tt(const FacSub* __restrict__ subs, const int2* __restrict__ items,
                                                 const double* __restrict__ minvp, const double* __restrict__ Wc,
                                                 double* __restrict__ U, int ldw, int64_t rows) {
  constexpr int NF = CW / 16;
  constexpr int LDV = CW + 4;
  constexpr int STAGE = TPAD + 64 * LDV;
  extern __shared__ __align__(128) double sm[];
  __shared__ __align__(8) uint64_t bar[2];
  const int2 it = items[blockIdx.x];
  const FacSub sb = subs[it.x];
  const int I = it.y, ntb = sb.ntb;
  const int c0 = blockIdx.y * CW;
  const double* Mb = minvp + sb.dense_off * TPAD;
  const double* Wb = Wc + (int64_t)blockIdx.y * rows * LDV + sb.wvu_row * LDV;
  auto mt = [&](int J) {
    return J <= I ? Mb + ((int64_t)I * (I + 1) / 2 + J) * TPAD : Mb + ((int64_t)J * (J + 1) / 2 + I) * TPAD;
  };
  if (threadIdx.x == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    fence_mbar_init();
  }
  __syncthreads();
  auto issue = [&](int J) {
    double* Ms = sm + (J & 1) * STAGE;
    if (threadIdx.x == 0) {
      fence_proxy_async();
      mbar_expect_copy(&bar[J & 1], Ms, mt(J), TPAD * 8);
      mbar_add_copy(&bar[J & 1], Ms + TPAD, Wb + (int64_t)J * 64 * LDV, 64 * LDV * 8);
    }
  };
  double acc[2][NF][2];
  acc_zero(acc);
  issue(0);
  for (int J = 0; J < ntb; ++J) {
    mbar_wait(&bar[J & 1], (J >> 1) & 1);
    __syncthreads();
    if (J + 1 < ntb) issue(J + 1);
    const double* Ms = sm + (J & 1) * STAGE;
    if (J <= I) cta_mma<NF, false, false>(Ms, LDP, Ms + TPAD, LDV, acc);
    else cta_mma<NF, true, false>(Ms, LDP, Ms + TPAD, LDV, acc);
  }
  double* out = U + (sb.wvu_row + (int64_t)I * 64) * ldw + c0;
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < NF; ++j) {
      const int r = acc_row<NF>(i), c = acc_col<NF>(j);
      *reinterpret_cast<double2*>(out + (int64_t)r * ldw + c) = make_double2(acc[i][j][0], acc[i][j][1]);
    }
}
int main() {
  const int nsub = 64, ntb = 7, ld = 128;
  std::vector<FacSub> subs(nsub);
  std::vector<int2> items;
  int64_t dense_tiles = 0, rows = 0;
  for (int j = 0; j < nsub; ++j) {
    FacSub f{}; f.ntb = ntb; f.dense_off = dense_tiles; f.wvu_row = rows; f.b = ntb * 64;
    subs[j] = f; dense_tiles += ntb * (ntb + 1) / 2; rows += ntb * 64;
    for (int I = 0; I < ntb; ++I) items.push_back(make_int2(j, I));
  }
  std::vector<double> M(dense_tiles * 4096), Mp(dense_tiles * TPAD, 0.0), W(rows * ld);   // library: padded
  std::mt19937_64 g(1); std::normal_distribution<double> nd;
  for (auto& x : M) x = nd(g);
  for (auto& x : W) x = nd(g);
  for (int64_t t = 0; t < dense_tiles; ++t)
    for (int r = 0; r < 64; ++r) for (int c = 0; c < 64; ++c) Mp[t * TPAD + r * LDP + c] = M[t * 4096 + r * 64 + c];
  FacSub* dsub; int2* dit; double *dM, *dMp, *dW, *dU, *dU2, *flush;
  cudaMalloc(&dsub, nsub * sizeof(FacSub)); cudaMalloc(&dit, items.size() * sizeof(int2));
  cudaMalloc(&dM, M.size() * 8); cudaMalloc(&dMp, Mp.size() * 8); cudaMalloc(&dW, W.size() * 8);
  cudaMalloc(&dU, W.size() * 8); cudaMalloc(&dU2, W.size() * 8); cudaMalloc(&flush, 256 << 20);
  cudaMemcpy(dsub, subs.data(), nsub * sizeof(FacSub), cudaMemcpyHostToDevice);
  cudaMemcpy(dit, items.data(), items.size() * sizeof(int2), cudaMemcpyHostToDevice);
  cudaMemcpy(dM, M.data(), M.size() * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(dMp, Mp.data(), Mp.size() * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(dW, W.data(), W.size() * 8, cudaMemcpyHostToDevice);
  cudaStream_t st; cudaStreamCreate(&st);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const double flops = 2.0 * nsub * (ntb * 64.0) * (ntb * 64.0) * ld;
  const size_t smem = 2 * (TPAD + 64 * 36) * sizeof(double);
  const size_t smem64 = 2 * (TPAD + 64 * 68) * sizeof(double);
  cudaFuncSetAttribute(k_symm_t<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaFuncSetAttribute(k_symm_t<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem64);
  // chunk-major padded copy of W for the full-TMA variant
  std::vector<double> Wcm((size_t)(ld / 32) * rows * 36, 0.0);
  for (int64_t r = 0; r < rows; ++r) for (int c = 0; c < ld; ++c) Wcm[(size_t)(c / 32) * rows * 36 + r * 36 + (c % 32)] = W[r * ld + c];
  double* dWc; cudaMalloc(&dWc, Wcm.size() * 8); cudaMemcpy(dWc, Wcm.data(), Wcm.size() * 8, cudaMemcpyHostToDevice);
  double* dU3; cudaMalloc(&dU3, W.size() * 8);
  cudaFuncSetAttribute(k_symm_tt<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  for (int v = 0; v < 4; ++v) {
    float best = 1e9;
    for (int r = 0; r < 13; ++r) {
      cudaMemsetAsync(flush, r, 256 << 20, st);
      cudaEventRecord(e0, st);
      if (v == 0) nspk::symm(dsub, dit, (int)items.size(), dMp, dW, dU, ld, 32, st);
      else if (v == 1) k_symm_t<32><<<dim3((unsigned)items.size(), ld / 32), 256, smem, st>>>(dsub, dit, dMp, dW, dU2, ld);
      else if (v == 2) k_symm_t<64><<<dim3((unsigned)items.size(), ld / 64), 256, smem64, st>>>(dsub, dit, dMp, dW, dU2, ld);
      else k_symm_tt<32><<<dim3((unsigned)items.size(), ld / 32), 256, smem, st>>>(dsub, dit, dMp, dWc, dU3, ld, rows);
      cudaEventRecord(e1, st); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      if (r >= 3) best = std::min(best, ms);
    }
    printf("%s: best %.1f us (%.2f TFLOP/s)  %s\n", v == 3 ? "TMA-M + TMA-W (chunk-major W)" : v == 2 ? "TMA-M cw 64" : v ? "TMA-M (padded tiles)" : "library k_symm", best * 1e3,
           flops / (best * 1e-3) / 1e12, cudaGetErrorString(cudaGetLastError()));
  }
  std::vector<double> U(W.size()), U2(W.size());
  cudaMemcpy(U.data(), dU, U.size() * 8, cudaMemcpyDeviceToHost);
  cudaMemcpy(U2.data(), dU2, U2.size() * 8, cudaMemcpyDeviceToHost);
  double md = 0, mx = 0;
  for (size_t i = 0; i < U.size(); ++i) { md = std::max(md, std::fabs(U[i] - U2[i])); mx = std::max(mx, std::fabs(U[i])); }
  printf("max |diff| / max %.3e\n", md / mx);
  std::vector<double> U3(W.size());
  cudaMemcpy(U3.data(), dU3, U3.size() * 8, cudaMemcpyDeviceToHost);
  md = 0; for (size_t i = 0; i < U.size(); ++i) md = std::max(md, std::fabs(U[i] - U3[i]));
  printf("full-TMA max |diff| / max %.3e\n", md / mx);
  return 0;
}
