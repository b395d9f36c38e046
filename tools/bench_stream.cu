// Single-CTA streaming of 32 KB tiles into shared memory (diagnostics): cp.async 16-byte ring vs
// TMA bulk copies (cp.async.bulk + mbarrier), to size the per-SM bandwidth of a sequential sweep.
#include <cstdio>
#include <cuda_runtime.h>
#include <cstdint>
__device__ __forceinline__ void cp16(void* s, const void* g) {
  unsigned a = (unsigned)__cvta_generic_to_shared(s);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(a), "l"(g));
}
template <int NS>
__global__ void k_cpasync(const double* src, int ntiles, double* out) {
  extern __shared__ double sm[];
  double acc = 0;
  auto issue = [&](int t) {
    double* dst = sm + (t % NS) * 4096;
    const double* g = src + (size_t)t * 4096;
    for (int c = threadIdx.x; c < 2048; c += blockDim.x) cp16(dst + 2 * c, g + 2 * c);
  };
  for (int p = 0; p < NS - 1; ++p) { if (p < ntiles) issue(p); asm volatile("cp.async.commit_group;\n"); }
  for (int t = 0; t < ntiles; ++t) {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(NS - 2));
    __syncthreads();
    if (t + NS - 1 < ntiles) issue(t + NS - 1);
    asm volatile("cp.async.commit_group;\n");
    acc += sm[(t % NS) * 4096 + threadIdx.x];
  }
  if (acc == 1.2345) out[0] = acc;
}
template <int NS>
__global__ void k_bulk(const double* src, int ntiles, double* out) {
  extern __shared__ __align__(128) double sm2[];
  __shared__ __align__(8) unsigned long long bar[NS];
  double acc = 0;
  if (threadIdx.x == 0)
    for (int i = 0; i < NS; ++i) {
      unsigned a = (unsigned)__cvta_generic_to_shared(&bar[i]);
      asm volatile("mbarrier.init.shared.b64 [%0], 1;\n" ::"r"(a));
    }
  __syncthreads();
  auto issue = [&](int t) {
    if (threadIdx.x != 0) return;
    const int sl = t % NS;
    unsigned b = (unsigned)__cvta_generic_to_shared(&bar[sl]);
    unsigned d = (unsigned)__cvta_generic_to_shared(sm2 + sl * 4096);
    asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;\n" ::"r"(b), "r"(32768));
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n"
                 ::"r"(d), "l"(src + (size_t)t * 4096), "r"(32768), "r"(b) : "memory");
  };
  for (int p = 0; p < NS - 1 && p < ntiles; ++p) issue(p);
  for (int t = 0; t < ntiles; ++t) {
    const int sl = t % NS;
    const unsigned phase = (t / NS) & 1;
    unsigned b = (unsigned)__cvta_generic_to_shared(&bar[sl]);
    asm volatile("{\n .reg .pred p;\n W: mbarrier.try_wait.parity.shared.b64 p, [%0], %1;\n @!p bra W;\n}\n" ::"r"(b), "r"(phase));
    acc += sm2[sl * 4096 + threadIdx.x];
    __syncthreads();
    if (t + NS - 1 < ntiles) issue(t + NS - 1);
  }
  if (acc == 1.2345) out[0] = acc;
}
int main() {
  const int ntiles = 894;
  double *src, *out;
  cudaMalloc(&src, (size_t)ntiles * 4096 * 8); cudaMalloc(&out, 8);
  cudaMemset(src, 0, (size_t)ntiles * 4096 * 8);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  auto run = [&](const char* nm, auto kern, size_t smem) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    kern<<<1, 256, smem>>>(src, ntiles, out);
    cudaEventRecord(e0); kern<<<1, 256, smem>>>(src, ntiles, out); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("%-16s %.3f ms  %.2f us/tile  %.1f GB/s  (%s)\n", nm, ms, ms * 1e3 / ntiles, ntiles * 32768.0 / (ms * 1e-3) / 1e9,
           cudaGetErrorString(cudaGetLastError()));
  };
  run("cp.async NS=2", k_cpasync<2>, 2 * 32768);
  run("cp.async NS=6", k_cpasync<6>, 6 * 32768);
  run("bulk NS=2", k_bulk<2>, 2 * 32768);
  run("bulk NS=4", k_bulk<4>, 4 * 32768);
  run("bulk NS=6", k_bulk<6>, 6 * 32768);
  return 0;
}
