// tcgen05 kind::i8 microbenchmark + layout check (sm_100a).
//  (1) correctness: D(128 x N, int32, TMEM) = A(128 x K) B(K x N) with A, B in the no-swizzle
//      core-matrix layout (8 rows x 16 bytes = 128 B per core matrix), B K-major or MN-major;
//      compared with a host integer product.
//  (2) throughput of the Ozaki pattern: 7 A slices x 7 B slices, the 28 products with i + j <= 8
//      into 7 TMEM accumulators of N columns, per K-step of 32; cycles per K-step vs 28 x floor.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/bench_i8mma tools/bench_i8mma.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <vector>
#include <random>
#include <cuda_runtime.h>

#define CK(x)                                                                   \
  do {                                                                          \
    cudaError_t e_ = (x);                                                       \
    if (e_ != cudaSuccess) {                                                    \
      printf("CUDA %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); \
      exit(1);                                                                  \
    }                                                                           \
  } while (0)

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// no-swizzle smem matrix descriptor (sm_100 version 1)
__device__ __forceinline__ uint64_t sdesc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((addr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;   // version
  return d;                 // base offset 0, lbo mode 0, layout SWIZZLE_NONE (0)
}
// instruction descriptor: kind::i8, s8 x s8 -> s32
__host__ __device__ constexpr uint32_t idesc_i8(int M, int N, int a_mn, int b_mn) {
  return (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)a_mn << 15) | ((uint32_t)b_mn << 16) |
         ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
__device__ __forceinline__ void mma_i8(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
      "l"(da), "l"(db), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ bool elect_one() {
  uint32_t p = 0;
  asm volatile("{\n .reg .pred P;\n elect.sync _|P, 0xffffffff;\n selp.b32 %0, 1, 0, P;\n}\n" : "=r"(p));
  return p != 0;
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned c) {
  asm volatile("mbarrier.init.shared.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(c));
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned ph) {
  asm volatile("{\n .reg .pred p;\n W: mbarrier.try_wait.parity.shared.b64 p, [%0], %1;\n @!p bra W;\n}\n" ::"r"(
                   smem_u32(bar)),
               "r"(ph) : "memory");
}
__device__ __forceinline__ void tmem_alloc(uint32_t* dst, int ncols) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(dst)), "r"(ncols));
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
}
__device__ __forceinline__ void tmem_dealloc(uint32_t t, int ncols) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(t), "r"(ncols));
}
__device__ __forceinline__ void ld16(uint32_t taddr, uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
        "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
}

// ---------------------------------------------------------------- (1) correctness
// A: 128 x K int8, blob [g=M/8][h=K/16][8][16]; B K-major: N x K blob [g][h][8][16];
// B MN-major (bmn): element B(k, n) stored at blob [h'=K/8][g'=N/16][8 k][16 n]  (core = 8 k x 16 n).
__global__ void k_check(const int8_t* A, const int8_t* B, int32_t* D, int N, int K, int bmn, int lbo_b, int sbo_b,
                        int kstep_b) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  int8_t* As = (int8_t*)sm;
  int8_t* Bs = As + 128 * K;
  for (int i = threadIdx.x; i < 128 * K; i += blockDim.x) As[i] = A[i];
  for (int i = threadIdx.x; i < N * K; i += blockDim.x) Bs[i] = B[i];
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (threadIdx.x < 32) tmem_alloc(&tbase, 256);
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t t0 = tbase;
  if (threadIdx.x == 0) {
    const uint32_t id = idesc_i8(128, N, 0, bmn);
    for (int k = 0; k < K / 32; ++k) {
      const uint64_t da = sdesc(smem_u32(As) + k * 256, 128, (K / 16) * 128);
      const uint64_t db = sdesc(smem_u32(Bs) + k * kstep_b, lbo_b, sbo_b);
      mma_i8(t0, da, db, id, k > 0);
    }
    mma_commit(&bar);
  }
  mbar_wait(&bar, 0);
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int c = 0; c < N; c += 16) {
    uint32_t v[16];
    ld16(t0 + ((uint32_t)(32 * w) << 16) + c, v);
    for (int q = 0; q < 16; ++q) D[(32 * w + lane) * N + c + q] = (int32_t)v[q];
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  if (threadIdx.x < 32) tmem_dealloc(t0, 256);
}

// ---------------------------------------------------------------- (2) Ozaki-pattern throughput
template <int N>
__global__ void k_rate(int reps, int KC, long long* cyc, int32_t* sink) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  int8_t* As = (int8_t*)sm;               // 7 slices x 128 x KC
  int8_t* Bs = As + 7 * 128 * KC;         // 7 slices x N x KC
  for (int i = threadIdx.x; i < 7 * (128 + N) * KC; i += blockDim.x) As[i] = (int8_t)((i * 37) & 7) - 3;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (threadIdx.x < 32) tmem_alloc(&tbase, 512);
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t t0 = tbase;
  if (threadIdx.x == 0) {
    const uint32_t id = idesc_i8(128, N, 0, 0);
    const long long c0 = clock64();
    for (int r = 0; r < reps; ++r)
      for (int k = 0; k < KC / 32; ++k)
        for (int i = 0; i < 7; ++i)
          for (int j = 0; i + j < 7; ++j) {
            const uint64_t da = sdesc(smem_u32(As + i * 128 * KC) + k * 256, 128, (KC / 16) * 128);
            const uint64_t db = sdesc(smem_u32(Bs + j * N * KC) + k * 256, 128, (KC / 16) * 128);
            mma_i8(t0 + (uint32_t)((i + j) * N), da, db, id, (r | k) > 0);
          }
    mma_commit(&bar);
    mbar_wait(&bar, 0);
    cyc[blockIdx.x] = clock64() - c0;
  }
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  uint32_t v[16];
  ld16(t0 + ((uint32_t)(32 * (threadIdx.x >> 5)) << 16), v);
  if (v[0] == 0x7fffffff) sink[0] = v[1];
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  if (threadIdx.x < 32) tmem_dealloc(t0, 512);
}

// tight issue: descriptors precomputed, loops unrolled (i, j compile-time)
template <int N, int KC>
__global__ void k_rate2(int reps, long long* cyc, int32_t* sink) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  int8_t* As = (int8_t*)sm;
  int8_t* Bs = As + 7 * 128 * KC;
  for (int i = threadIdx.x; i < 7 * (128 + N) * KC; i += blockDim.x) As[i] = (int8_t)((i * 37) & 7) - 3;
  if (threadIdx.x < 32 && elect_one()) {
    mbar_init(&bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (threadIdx.x < 32) tmem_alloc(&tbase, 512);
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t t0 = tbase;
  if (threadIdx.x == 0) {
    constexpr uint32_t id = idesc_i8(128, N, 0, 0);
    const uint64_t a0 = sdesc(smem_u32(As), 128, (KC / 16) * 128);
    const uint64_t b0 = sdesc(smem_u32(Bs), 128, (KC / 16) * 128);
    const long long c0 = clock64();
    for (int r = 0; r < reps; ++r) {
#pragma unroll
      for (int k = 0; k < KC / 32; ++k)
#pragma unroll
        for (int i = 0; i < 7; ++i)
#pragma unroll
          for (int j = 0; i + j < 7; ++j)
            mma_i8(t0 + (uint32_t)((i + j) * N), a0 + (uint64_t)((i * 128 * KC + k * 256) >> 4),
                   b0 + (uint64_t)((j * N * KC + k * 256) >> 4), id, (r | k) > 0);
    }
    mma_commit(&bar);
    mbar_wait(&bar, 0);
    cyc[blockIdx.x] = clock64() - c0;
  }
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  uint32_t v[16];
  ld16(t0 + ((uint32_t)(32 * (threadIdx.x >> 5)) << 16), v);
  if (v[0] == 0x7fffffff) sink[0] = v[1];
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  if (threadIdx.x < 32) tmem_dealloc(t0, 512);
}
// single accumulator, N up to 256: the plain floor
template <int N, int KC>
__global__ void k_rate1(int reps, long long* cyc, int32_t* sink) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  int8_t* As = (int8_t*)sm;
  int8_t* Bs = As + 128 * KC;
  for (int i = threadIdx.x; i < (128 + N) * KC; i += blockDim.x) As[i] = (int8_t)((i * 37) & 7) - 3;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (threadIdx.x < 32) tmem_alloc(&tbase, 512);
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t t0 = tbase;
  if (threadIdx.x == 0) {
    constexpr uint32_t id = idesc_i8(128, N, 0, 0);
    const uint64_t a0 = sdesc(smem_u32(As), 128, (KC / 16) * 128);
    const uint64_t b0 = sdesc(smem_u32(Bs), 128, (KC / 16) * 128);
    const long long c0 = clock64();
    for (int r = 0; r < reps; ++r) {
#pragma unroll
      for (int k = 0; k < KC / 32; ++k)
        mma_i8(t0, a0 + (uint64_t)((k * 256) >> 4), b0 + (uint64_t)((k * 256) >> 4), id, (r | k) > 0);
    }
    mma_commit(&bar);
    mbar_wait(&bar, 0);
    cyc[blockIdx.x] = clock64() - c0;
  }
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  uint32_t v[16];
  ld16(t0 + ((uint32_t)(32 * (threadIdx.x >> 5)) << 16), v);
  if (v[0] == 0x7fffffff) sink[0] = v[1];
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  if (threadIdx.x < 32) tmem_dealloc(t0, 512);
}

// B MN-major (core = 8 k x 16 n; blob [k/8][n/16][8][16]): per-MMA cost
template <int N, int KC>
__global__ void k_rate_mn(int reps, long long* cyc, int32_t* sink) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  int8_t* As = (int8_t*)sm;
  int8_t* Bs = As + 7 * 128 * KC;
  for (int i = threadIdx.x; i < 7 * (128 + N) * KC; i += blockDim.x) As[i] = (int8_t)((i * 37) & 7) - 3;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (threadIdx.x < 32) tmem_alloc(&tbase, 512);
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t t0 = tbase;
  if (threadIdx.x < 32 && elect_one()) {
    constexpr uint32_t id = idesc_i8(128, N, 0, 1);
    const uint64_t a0 = sdesc(smem_u32(As), 128, (KC / 16) * 128);
    const uint64_t b0 = sdesc(smem_u32(Bs), (N / 16) * 128, 128);
    const long long c0 = clock64();
    for (int r = 0; r < reps; ++r) {
#pragma unroll
      for (int k = 0; k < KC / 32; ++k)
#pragma unroll
        for (int i = 0; i < 7; ++i)
#pragma unroll
          for (int j = 0; i + j < 7; ++j)
            mma_i8(t0 + (uint32_t)((i + j) * N), a0 + (uint64_t)((i * 128 * KC + k * 256) >> 4),
                   b0 + (uint64_t)((j * N * KC + k * 4 * (N / 16) * 128) >> 4), id, (r | k) > 0);
    }
    mma_commit(&bar);
    mbar_wait(&bar, 0);
    cyc[blockIdx.x] = clock64() - c0;
  }
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  uint32_t v[16];
  ld16(t0 + ((uint32_t)(32 * (threadIdx.x >> 5)) << 16), v);
  if (v[0] == 0x7fffffff) sink[0] = v[1];
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  if (threadIdx.x < 32) tmem_dealloc(t0, 512);
}

// ---------------------------------------------------------------- A operand in TMEM (tcgen05.cp 128x256b)
__device__ __forceinline__ void mma_i8_ts(uint32_t tmem_d, uint32_t tmem_a, uint64_t db, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(tmem_d),
      "r"(tmem_a), "l"(db), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void tc_cp(uint32_t taddr, uint64_t sd) {
  asm volatile("tcgen05.cp.cta_group::1.128x256b [%0], %1;\n" ::"r"(taddr), "l"(sd));
}
// correctness: A (128 x K) staged smem -> TMEM per K-step of 32 (8 columns), then TS MMA
__global__ void k_check_ts(const int8_t* A, const int8_t* B, int32_t* D, int N, int K) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  int8_t* As = (int8_t*)sm;
  int8_t* Bs = As + 128 * K;
  for (int i = threadIdx.x; i < 128 * K; i += blockDim.x) As[i] = A[i];
  for (int i = threadIdx.x; i < N * K; i += blockDim.x) Bs[i] = B[i];
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (threadIdx.x < 32) tmem_alloc(&tbase, 512);
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t t0 = tbase;
  if (threadIdx.x < 32 && elect_one()) {
    const uint32_t id = idesc_i8(128, N, 0, 0);
    for (int k = 0; k < K / 32; ++k) {
      const uint32_t ta = t0 + 256 + (k & 1) * 8;   // A staging columns 256.. (double buffer)
      tc_cp(ta, sdesc(smem_u32(As) + k * 256, 128, (K / 16) * 128));
      const uint64_t db = sdesc(smem_u32(Bs) + k * 256, 128, (K / 16) * 128);
      mma_i8_ts(t0, ta, db, id, k > 0);
    }
    mma_commit(&bar);
  }
  mbar_wait(&bar, 0);
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int c = 0; c < N; c += 16) {
    uint32_t v[16];
    ld16(t0 + ((uint32_t)(32 * w) << 16) + c, v);
    for (int q = 0; q < 16; ++q) D[(32 * w + lane) * N + c + q] = (int32_t)v[q];
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  if (threadIdx.x < 32) tmem_dealloc(t0, 512);
}
// rate: Ozaki pattern, A slices 0..NT-1 from TMEM (cp per K-step, double-buffered), the rest from smem
template <int NT, int KC>
__global__ void k_rate_ts(int reps, long long* cyc, int32_t* sink) {
  constexpr int N = 64;
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  int8_t* As = (int8_t*)sm;
  int8_t* Bs = As + 7 * 128 * KC;
  for (int i = threadIdx.x; i < 7 * (128 + N) * KC; i += blockDim.x) As[i] = (int8_t)((i * 37) & 7) - 3;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (threadIdx.x < 32) tmem_alloc(&tbase, 512);
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t t0 = tbase;
  if (threadIdx.x < 32 && elect_one()) {
    constexpr uint32_t id = idesc_i8(128, N, 0, 0);
    const uint64_t a0 = sdesc(smem_u32(As), 128, (KC / 16) * 128);
    const uint64_t b0 = sdesc(smem_u32(Bs), 128, (KC / 16) * 128);
    const long long c0 = clock64();
    int buf = 0;
    for (int r = 0; r < reps; ++r) {
#pragma unroll
      for (int k = 0; k < KC / 32; ++k) {
        const uint32_t ta = t0 + 448 + buf * (8 * NT);
#pragma unroll
        for (int i = 0; i < NT; ++i) tc_cp(ta + 8 * i, a0 + (uint64_t)((i * 128 * KC + k * 256) >> 4));
#pragma unroll
        for (int i = 0; i < 7; ++i)
#pragma unroll
          for (int j = 0; i + j < 7; ++j) {
            const uint64_t db = b0 + (uint64_t)((j * N * KC + k * 256) >> 4);
            if (i < NT) mma_i8_ts(t0 + (uint32_t)((i + j) * N), ta + 8 * i, db, id, (r | k) > 0);
            else mma_i8(t0 + (uint32_t)((i + j) * N), a0 + (uint64_t)((i * 128 * KC + k * 256) >> 4), db, id, (r | k) > 0);
          }
        buf ^= 1;
      }
    }
    mma_commit(&bar);
    mbar_wait(&bar, 0);
    cyc[blockIdx.x] = clock64() - c0;
  }
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  uint32_t v[16];
  ld16(t0 + ((uint32_t)(32 * (threadIdx.x >> 5)) << 16), v);
  if (v[0] == 0x7fffffff) sink[0] = v[1];
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  if (threadIdx.x < 32) tmem_dealloc(t0, 512);
}

// ---------------------------------------------------------------- weight-stationary form with the B collector
#define WS_MMA(QUAL, d, a, b, id, acc)                                                                  \
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"                                       \
               "tcgen05.mma.ws.cta_group::1.kind::i8" QUAL " [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d), "l"(a), \
               "l"(b), "r"(id), "r"((uint32_t)(acc)))
// D_t (t = 0, 1) = A_t B: the first MMA fills the B collector, the second reuses it
__global__ void k_check_ws(const int8_t* A, const int8_t* B, int32_t* D, int K) {
  constexpr int N = 64;
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  int8_t* As = (int8_t*)sm;            // two A operands of 128 x K
  int8_t* Bs = As + 2 * 128 * K;
  for (int i = threadIdx.x; i < 2 * 128 * K; i += blockDim.x) As[i] = A[i];
  for (int i = threadIdx.x; i < N * K; i += blockDim.x) Bs[i] = B[i];
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (threadIdx.x < 32) tmem_alloc(&tbase, 256);
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t t0 = tbase;
  if (threadIdx.x < 32 && elect_one()) {
    const uint32_t id = idesc_i8(128, N, 0, 0);
    for (int k = 0; k < K / 32; ++k) {
      const uint64_t db = sdesc(smem_u32(Bs) + k * 256, 128, (K / 16) * 128);
      const uint64_t da0 = sdesc(smem_u32(As) + k * 256, 128, (K / 16) * 128);
      const uint64_t da1 = sdesc(smem_u32(As + 128 * K) + k * 256, 128, (K / 16) * 128);
      WS_MMA(".collector::b0::fill", t0, da0, db, id, k > 0);
      WS_MMA(".collector::b0::lastuse", t0 + N, da1, db, id, k > 0);
    }
    mma_commit(&bar);
  }
  mbar_wait(&bar, 0);
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int c = 0; c < 2 * N; c += 16) {
    uint32_t v[16];
    ld16(t0 + ((uint32_t)(32 * w) << 16) + c, v);
    for (int q = 0; q < 16; ++q) D[(32 * w + lane) * 2 * N + c + q] = (int32_t)v[q];
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  if (threadIdx.x < 32) tmem_dealloc(t0, 256);
}
// Ozaki pattern in weight-stationary order: for each B slice j, the 7 - j products with A slices i share it
template <int KC, bool COLL>
__global__ void k_rate_ws(int reps, long long* cyc, int32_t* sink) {
  constexpr int N = 64;
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  int8_t* As = (int8_t*)sm;
  int8_t* Bs = As + 7 * 128 * KC;
  for (int i = threadIdx.x; i < 7 * (128 + N) * KC; i += blockDim.x) As[i] = (int8_t)((i * 37) & 7) - 3;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (threadIdx.x < 32) tmem_alloc(&tbase, 512);
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t t0 = tbase;
  if (threadIdx.x < 32 && elect_one()) {
    constexpr uint32_t id = idesc_i8(128, N, 0, 0);
    const uint64_t a0 = sdesc(smem_u32(As), 128, (KC / 16) * 128);
    const uint64_t b0 = sdesc(smem_u32(Bs), 128, (KC / 16) * 128);
    const long long c0 = clock64();
    for (int r = 0; r < reps; ++r) {
#pragma unroll
      for (int k = 0; k < KC / 32; ++k)
#pragma unroll
        for (int j = 0; j < 7; ++j)
#pragma unroll
          for (int i = 0; i + j < 7; ++i) {
            const uint64_t da = a0 + (uint64_t)((i * 128 * KC + k * 256) >> 4);
            const uint64_t db = b0 + (uint64_t)((j * N * KC + k * 256) >> 4);
            const uint32_t dd = t0 + (uint32_t)((i + j) * N);
            const uint32_t acc = (r | k) > 0;
            if (!COLL || j == 6) WS_MMA("", dd, da, db, id, acc);
            else if (i == 0) WS_MMA(".collector::b0::fill", dd, da, db, id, acc);
            else if (i + j == 6) WS_MMA(".collector::b0::lastuse", dd, da, db, id, acc);
            else WS_MMA(".collector::b0::use", dd, da, db, id, acc);
          }
    }
    mma_commit(&bar);
    mbar_wait(&bar, 0);
    cyc[blockIdx.x] = clock64() - c0;
  }
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  uint32_t v[16];
  ld16(t0 + ((uint32_t)(32 * (threadIdx.x >> 5)) << 16), v);
  if (v[0] == 0x7fffffff) sink[0] = v[1];
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  if (threadIdx.x < 32) tmem_dealloc(t0, 512);
}

int main() {
  std::mt19937 rng(7);
  std::uniform_int_distribution<int> dist(-128, 127);
  int fails = 0;
  for (int bmn = 0; bmn < 2; ++bmn)
    for (int N : {64, 128}) {
      const int K = 128;
      std::vector<int8_t> a(128 * K), b(N * K), ab(128 * K), bb(N * K);
      for (auto& x : a) x = (int8_t)dist(rng);
      for (auto& x : b) x = (int8_t)dist(rng);   // logical B(k, n) = b[n*K + k]
      for (int m = 0; m < 128; ++m)
        for (int k = 0; k < K; ++k) ab[((m / 8) * (K / 16) + k / 16) * 128 + (m % 8) * 16 + k % 16] = a[m * K + k];
      int lbo, sbo, kstep;
      if (!bmn) {
        for (int n = 0; n < N; ++n)
          for (int k = 0; k < K; ++k) bb[((n / 8) * (K / 16) + k / 16) * 128 + (n % 8) * 16 + k % 16] = b[n * K + k];
        lbo = 128, sbo = (K / 16) * 128, kstep = 256;
      } else {   // core = 8 k x 16 n; blob [k/8][n/16][8][16]
        for (int n = 0; n < N; ++n)
          for (int k = 0; k < K; ++k) bb[((k / 8) * (N / 16) + n / 16) * 128 + (k % 8) * 16 + n % 16] = b[n * K + k];
        // MN-major: SBO = stride between MN core groups (16 n), LBO = stride between K core groups (8 k)
        sbo = 128, lbo = (N / 16) * 128, kstep = 4 * (N / 16) * 128;
      }
      int8_t *dA, *dB;
      int32_t* dD;
      CK(cudaMalloc(&dA, ab.size()));
      CK(cudaMalloc(&dB, bb.size()));
      CK(cudaMalloc(&dD, 128 * N * 4));
      CK(cudaMemcpy(dA, ab.data(), ab.size(), cudaMemcpyHostToDevice));
      CK(cudaMemcpy(dB, bb.data(), bb.size(), cudaMemcpyHostToDevice));
      CK(cudaMemset(dD, 0, 128 * N * 4));
      k_check<<<1, 128, 128 * K + N * K>>>(dA, dB, dD, N, K, bmn, lbo, sbo, kstep);
      CK(cudaDeviceSynchronize());
      std::vector<int32_t> d(128 * N);
      CK(cudaMemcpy(d.data(), dD, d.size() * 4, cudaMemcpyDeviceToHost));
      int bad = 0;
      for (int m = 0; m < 128; ++m)
        for (int n = 0; n < N; ++n) {
          int32_t ref = 0;
          for (int k = 0; k < K; ++k) ref += (int32_t)a[m * K + k] * b[n * K + k];
          if (ref != d[m * N + n]) {
            if (bad < 4) printf("  mismatch bmn=%d N=%d (%d,%d): got %d ref %d\n", bmn, N, m, n, d[m * N + n], ref);
            ++bad;
          }
        }
      printf("check B %s N=%d: %s (%d bad)\n", bmn ? "MN-major" : "K-major", N, bad ? "FAIL" : "ok", bad);
      fails += bad != 0;
      cudaFree(dA);
      cudaFree(dB);
      cudaFree(dD);
    }
  {
    const int N = 64, K = 128;
    std::vector<int8_t> a(128 * K), b(N * K), ab(128 * K), bb(N * K);
    for (auto& x : a) x = (int8_t)dist(rng);
    for (auto& x : b) x = (int8_t)dist(rng);
    for (int m = 0; m < 128; ++m)
      for (int k = 0; k < K; ++k) ab[((m / 8) * (K / 16) + k / 16) * 128 + (m % 8) * 16 + k % 16] = a[m * K + k];
    for (int n = 0; n < N; ++n)
      for (int k = 0; k < K; ++k) bb[((n / 8) * (K / 16) + k / 16) * 128 + (n % 8) * 16 + k % 16] = b[n * K + k];
    int8_t *dA, *dB;
    int32_t* dD;
    CK(cudaMalloc(&dA, ab.size()));
    CK(cudaMalloc(&dB, bb.size()));
    CK(cudaMalloc(&dD, 128 * N * 4));
    CK(cudaMemcpy(dA, ab.data(), ab.size(), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dB, bb.data(), bb.size(), cudaMemcpyHostToDevice));
    k_check_ts<<<1, 128, 128 * K + N * K>>>(dA, dB, dD, N, K);
    CK(cudaDeviceSynchronize());
    std::vector<int32_t> d(128 * N);
    CK(cudaMemcpy(d.data(), dD, d.size() * 4, cudaMemcpyDeviceToHost));
    int bad = 0;
    for (int m = 0; m < 128; ++m)
      for (int n = 0; n < N; ++n) {
        int32_t ref = 0;
        for (int k = 0; k < K; ++k) ref += (int32_t)a[m * K + k] * b[n * K + k];
        if (ref != d[m * N + n]) {
          if (bad < 4) printf("  TS mismatch (%d,%d): got %d ref %d\n", m, n, d[m * N + n], ref);
          ++bad;
        }
      }
    printf("check TS (A in TMEM via tcgen05.cp) N=64: %s (%d bad)\n", bad ? "FAIL" : "ok", bad);
    fails += bad != 0;
  }
  {   // weight-stationary MMA with the B collector
    const int N = 64, K = 64;
    std::vector<int8_t> a(2 * 128 * K), b(N * K), ab(2 * 128 * K), bb(N * K);
    for (auto& x : a) x = (int8_t)dist(rng);
    for (auto& x : b) x = (int8_t)dist(rng);
    for (int t = 0; t < 2; ++t)
      for (int m = 0; m < 128; ++m)
        for (int k = 0; k < K; ++k)
          ab[t * 128 * K + ((m / 8) * (K / 16) + k / 16) * 128 + (m % 8) * 16 + k % 16] = a[(t * 128 + m) * K + k];
    for (int n = 0; n < N; ++n)
      for (int k = 0; k < K; ++k) bb[((n / 8) * (K / 16) + k / 16) * 128 + (n % 8) * 16 + k % 16] = b[n * K + k];
    int8_t *dA, *dB;
    int32_t* dD;
    CK(cudaMalloc(&dA, ab.size()));
    CK(cudaMalloc(&dB, bb.size()));
    CK(cudaMalloc(&dD, 128 * 2 * N * 4));
    CK(cudaMemcpy(dA, ab.data(), ab.size(), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dB, bb.data(), bb.size(), cudaMemcpyHostToDevice));
    k_check_ws<<<1, 128, 2 * 128 * K + N * K>>>(dA, dB, dD, K);
    CK(cudaDeviceSynchronize());
    std::vector<int32_t> d(128 * 2 * N);
    CK(cudaMemcpy(d.data(), dD, d.size() * 4, cudaMemcpyDeviceToHost));
    int bad = 0;
    for (int t = 0; t < 2; ++t)
      for (int m = 0; m < 128; ++m)
        for (int n = 0; n < N; ++n) {
          int32_t ref = 0;
          for (int k = 0; k < K; ++k) ref += (int32_t)a[(t * 128 + m) * K + k] * b[n * K + k];
          if (ref != d[m * 2 * N + t * N + n]) {
            if (bad < 4) printf("  WS mismatch t=%d (%d,%d): got %d ref %d\n", t, m, n, d[m * 2 * N + t * N + n], ref);
            ++bad;
          }
        }
    printf("check WS (B collector fill / lastuse) N=64: %s (%d bad)\n", bad ? "FAIL" : "ok", bad);
    fails += bad != 0;
  }
  long long* dc;
  int32_t* sink;
  CK(cudaMalloc(&dc, 1024 * 8));
  CK(cudaMalloc(&sink, 64));
  const int KC = 64, reps = 64;
  auto run = [&](auto kern, int N, int grid) {
    const int smem = 7 * (128 + N) * KC;
    CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    kern<<<grid, 128, smem>>>(reps, KC, dc, sink);
    CK(cudaDeviceSynchronize());
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    kern<<<grid, 128, smem>>>(reps, KC, dc, sink);
    cudaEventRecord(e1);
    CK(cudaDeviceSynchronize());
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    std::vector<long long> c(grid);
    CK(cudaMemcpy(c.data(), dc, grid * 8, cudaMemcpyDeviceToHost));
    const double steps = (double)reps * (KC / 32);
    const double macs = (double)grid * steps * 28 * 128.0 * N * 32;
    printf("rate N=%d grid=%d: %.1f cycles per K-step (28 MMAs; floor %d) -> %.1f cyc/MMA; %.2f TOPS (events %.3f ms)\n",
           N, grid, c[0] / steps, 28 * 128 * N / 256, c[0] / steps / 28, 2 * macs / (ms * 1e-3) / 1e12, ms);
  };
  run(k_rate<64>, 64, 1);
  run(k_rate<64>, 64, 148);
  run(k_rate<32>, 32, 148);

  auto run2 = [&](auto kern, int N, int KC, int nmma, int reps2, int smem, const char* name) {
    CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    kern<<<148, 128, smem>>>(reps2, dc, sink);
    CK(cudaDeviceSynchronize());
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    kern<<<148, 128, smem>>>(reps2, dc, sink);
    cudaEventRecord(e1);
    CK(cudaDeviceSynchronize());
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    long long c;
    CK(cudaMemcpy(&c, dc, 8, cudaMemcpyDeviceToHost));
    const double steps = (double)reps2 * (KC / 32);
    const double macs = 148.0 * steps * nmma * 128.0 * N * 32;
    printf("%s N=%d KC=%d: %.1f cyc per K-step (%d MMAs, floor %d) = %.1f cyc/MMA; %.0f TOPS at events %.3f ms\n", name, N,
           KC, c / steps, nmma, nmma * 128 * N / 256, c / steps / nmma, 2 * macs / (ms * 1e-3) / 1e12, ms);
  };
  run2(k_rate2<64, 64>, 64, 64, 28, 256, 7 * (128 + 64) * 64, "ozaki-tight");
  run2(k_rate2<64, 128>, 64, 128, 28, 128, 7 * (128 + 64) * 128, "ozaki-tight");
  run2(k_rate2<32, 128>, 32, 128, 28, 128, 7 * (128 + 32) * 128, "ozaki-tight");
  run2(k_rate_mn<64, 64>, 64, 64, 28, 256, 7 * (128 + 64) * 64, "ozaki-MN-B");
  run2(k_rate_ws<64, false>, 64, 64, 28, 256, 7 * (128 + 64) * 64, "ozaki-WS");
  run2(k_rate_ws<64, true>, 64, 64, 28, 256, 7 * (128 + 64) * 64, "ozaki-WS-collector");
  run2(k_rate_ts<1, 64>, 64, 64, 28, 256, 7 * (128 + 64) * 64, "ozaki-TS1");
  run2(k_rate_ts<2, 64>, 64, 64, 28, 256, 7 * (128 + 64) * 64, "ozaki-TS2");
  run2(k_rate_ts<3, 64>, 64, 64, 28, 256, 7 * (128 + 64) * 64, "ozaki-TS3");
  run2(k_rate1<64, 128>, 64, 128, 1, 4096, (128 + 64) * 128, "single");
  run2(k_rate1<128, 128>, 128, 128, 1, 4096, (128 + 128) * 128, "single");
  run2(k_rate1<256, 128>, 256, 128, 1, 4096, (128 + 256) * 128, "single");
  printf("%s\n", fails ? "LAYOUT CHECK FAILED" : "layout checks ok");
  return 0;
}
