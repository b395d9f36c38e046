// fp64 tensor-pipe helpers: mma.sync m8n8k4 f64 (SASS DMMA.8x8x4 on sm_100a; tcgen05 has
// no f64 kind, SURVEY.md §0 finding 4) and cp.async staging.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <cstdlib>
#include <map>
#include <mutex>
#include <utility>

namespace nspd {

// Dynamic shared memory above 48 KB is an opt-in per (kernel, DEVICE): cached per device so a
// second device in the same process gets its own attribute (a process-wide flag would skip it).
inline void smem_optin(const void* f, size_t bytes) {
  static std::mutex mu;
  static std::map<std::pair<const void*, int>, size_t> done;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(mu);
  size_t& have = done[std::make_pair(f, dev)];
  if (have >= bytes) return;
  cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  have = bytes;
}

// SM count of the current device (grid sizing: one wave = SMs x resident CTAs), cached per device.
inline int num_sms() {
  static int cache[64] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) dev = 0;
  if (!cache[dev]) {
    int n = 0;
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    cache[dev] = n > 0 ? n : 148;
  }
  return cache[dev];
}

// D = A(8x4, row) * B(4x8, col) + C.  Fragment ownership (lane = 4*g + t):
//   a = A[g][t], b = B[t][g], c = {C[g][2t], C[g][2t+1]}.
// Not `volatile`: the MMA is a pure function of its register operands, so the compiler may hoist
// the next fragments' shared-memory loads above it (software pipelining).
__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
#ifdef NSP_DMMA_VOLATILE
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
#else
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
      : "+d"(c0), "+d"(c1)
      : "d"(a), "d"(b));
#endif
}

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

// CTA (8 warps) computes a 64 x (16*NF) product tile:
//   acc += A(64 x K) * B(K x 16NF),
//   A[m][k] = TA ? As[k*lda + m] : As[m*lda + k];  B[k][n] = TB ? Bs[n*ldb + k] : Bs[k*ldb + n].
// Warp w owns rows 16*(w>>1) .. +16 (2 m-fragments) and cols 8*NF*(w&1) .. +8NF (NF n-fragments).
// acc[i][j][e] <-> C[16*(w>>1) + 8i + g][8*NF*(w&1) + 8j + 2t + e].
template <int NF, bool TA, bool TB>
__device__ __forceinline__ void cta_mma(const double* __restrict__ As, int lda, const double* __restrict__ Bs,
                                        int ldb, double (&acc)[2][NF][2], int K = 64, int wsel = -1) {
  const int lane = threadIdx.x & 31, warp = wsel >= 0 ? wsel : (int)(threadIdx.x >> 5);
  const int g = lane >> 2, t = lane & 3;
  const int m0 = (warp >> 1) * 16, n0 = (warp & 1) * NF * 8;
#pragma unroll 4
  for (int k = 0; k < K; k += 4) {
    double a[2], b[NF];
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      const int m = m0 + i * 8 + g, kk = k + t;
      a[i] = TA ? As[kk * lda + m] : As[m * lda + kk];
    }
#pragma unroll
    for (int j = 0; j < NF; ++j) {
      const int n = n0 + j * 8 + g, kk = k + t;
      b[j] = TB ? Bs[n * ldb + kk] : Bs[kk * ldb + n];
    }
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
      for (int j = 0; j < NF; ++j) dmma(acc[i][j][0], acc[i][j][1], a[i], b[j]);
  }
}

template <int NF>
__device__ __forceinline__ void acc_zero(double (&acc)[2][NF][2]) {
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < NF; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
}

// Row / column of accumulator element (i, j, e) for the calling thread.
template <int NF>
__device__ __forceinline__ int acc_row(int i, int wsel = -1) {
  const int lane = threadIdx.x & 31, warp = wsel >= 0 ? wsel : (int)(threadIdx.x >> 5);
  return (warp >> 1) * 16 + i * 8 + (lane >> 2);
}
template <int NF>
__device__ __forceinline__ int acc_col(int j, int wsel = -1) {
  const int lane = threadIdx.x & 31, warp = wsel >= 0 ? wsel : (int)(threadIdx.x >> 5);
  return (warp & 1) * NF * 8 + j * 8 + 2 * (lane & 3);
}

// Async copy of a rows x cols (cols multiple of 2) row-major global block (ld gld) into smem (ld sld).
__device__ __forceinline__ void cp_block(double* s, int sld, const double* g, int64_t gld, int rows, int cols) {
  const int chunks_per_row = cols / 2;
  const int total = rows * chunks_per_row;
  for (int c = threadIdx.x; c < total; c += blockDim.x) {
    const int r = c / chunks_per_row, q = c - r * chunks_per_row;
    cp_async16(s + r * sld + 2 * q, g + r * gld + 2 * q);
  }
}

// bulk shared -> global store (TMA store, bulk-group completion); 16-byte aligned, size % 16 == 0.
// The writing threads fence their shared-memory stores to the async proxy (fence_proxy_async) and
// synchronise before the issue; the issuing thread waits for its group before the kernel exits.
__device__ __forceinline__ void bulk_store(void* gdst, const void* ssrc, unsigned bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;\n" ::"l"(gdst),
               "r"((unsigned)__cvta_generic_to_shared(ssrc)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_store_commit_wait() {   // the source may be reused / the CTA may exit
  asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
  asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory");
}

// mbarrier + bulk-copy (TMA, cp.async.bulk) helpers
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared.b64 [%0], %1;\n" ::"r"((unsigned)__cvta_generic_to_shared(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_copy(uint64_t* bar, void* dst, const void* src, unsigned bytes) {
  const unsigned b = (unsigned)__cvta_generic_to_shared(bar);
  asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;\n" ::"r"(b), "r"(bytes));
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                   (unsigned)__cvta_generic_to_shared(dst)),
               "l"(src), "r"(bytes), "r"(b)
               : "memory");
}
__device__ __forceinline__ void mbar_add_copy(uint64_t* bar, void* dst, const void* src, unsigned bytes) {
  const unsigned b = (unsigned)__cvta_generic_to_shared(bar);
  asm volatile("mbarrier.expect_tx.relaxed.cta.shared::cta.b64 [%0], %1;\n" ::"r"(b), "r"(bytes));
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                   (unsigned)__cvta_generic_to_shared(dst)),
               "l"(src), "r"(bytes), "r"(b)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned phase) {
  const unsigned b = (unsigned)__cvta_generic_to_shared(bar);
  asm volatile("{\n .reg .pred p;\n W: mbarrier.try_wait.parity.shared.b64 p, [%0], %1;\n @!p bra W;\n}\n" ::"r"(b),
               "r"(phase));
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"((unsigned)__cvta_generic_to_shared(bar)) : "memory");
}
__device__ __forceinline__ void mbar_expect(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;\n" ::"r"((unsigned)__cvta_generic_to_shared(bar)),
               "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_copy(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                   (unsigned)__cvta_generic_to_shared(dst)),
               "l"(src), "r"(bytes), "r"((unsigned)__cvta_generic_to_shared(bar))
               : "memory");
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory"); }
__device__ __forceinline__ void fence_mbar_init() { asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory"); }

// Programmatic dependent launch (PDL): hot-loop kernels start with pdl_wait() (griddepcontrol.wait:
// blocks until the preceding kernel in the stream has completed and its writes are visible; a no-op
// for a normal launch) and are launched with launch_k(), which sets the programmatic-serialisation
// attribute so that the next grid is launched while the previous one drains (NSP_PDL=0 disables).
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;\n" ::: "memory"); }

inline bool pdl_enabled() {
  static const bool on = [] {
    const char* e = getenv("NSP_PDL");
    return !(e && e[0] == '0');
  }();
  return on;
}

template <typename... KArgs, typename... Args>
inline cudaError_t launch_k(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                            Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

}  // namespace nspd
