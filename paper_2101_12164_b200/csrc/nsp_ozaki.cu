// a2+a3 (U_j = S_j^{-1} W_j for every block; the product that the boundary-last
// ordering of reading R1 leaves, "factorized cheaply in parallel") on the 5th-generation
// INT8 tensor cores (tcgen05.mma kind::i8, accumulators in TMEM) with fp64 accuracy: the Ozaki
// splitting (DESIGN.md §6 "k_oz_symm", reading R10).
//
//   M_j = S_j^{-1} is symmetric positive definite.  With D = diag(delta_n), delta_n = 2^e_n and
//   e_n = floor(log2(M_nn)/2), the symmetrically scaled Mt = D^{-1} M D^{-1} has Mt_nn in [1, 4) and
//   |Mt_kn| <= sqrt(Mt_kk Mt_nn) < 4, so ONE power-of-two scale mu_j per block serves every entry and the scaling
//   is the same for a stored lower tile read as itself (K-major) or transposed (MN-major): only the
//   lower tiles are sliced, as in k_symm.  Wt = D W.  Each column c of Wt (per block) gets its own
//   power-of-two scale sigma_c.  Every scaled entry x (|x| < 1/2) is the 56-bit fixed-point integer
//   X = rint(x 2^55) = sum_{i=1..7} d_i 256^{7-i}, d_i signed bytes (|d_1| <= 64).  Then
//     sum_k Wt(k,c) Mt(k,n) = sigma_c mu_j 2^-110 sum_{i,j} 256^{14-i-j} sum_k dW_i(c,k) dM_j(k,n)
//   and the 28 int8 products with i + j <= 8 are accumulated EXACTLY in int32 (7 accumulators, one per
//   diagonal i + j; |sum| <= (64 * 128 + 6 * 128^2) b_j < 2^31 for b_j < 20,000: ntb <= 300 checked at setup); the dropped
//   diagonals i + j >= 9 are below 2^-57 sigma_c mu_j sqrt(b) (under fp64 rounding of the result).
//   The epilogue forms u = sum_D 2^{2-8D} acc_D in fp64 (least significant first) and scales by the
//   powers of two: U(n, c) = delta_n sigma_c mu_j u.
//
// Layouts (no-swizzle canonical UMMA core matrices: 8 rows x 16 bytes, 128 contiguous bytes):
//   M slices (setup, constant): stored lower tile (I, J) of block j (same index as the S_j^{-1} tiles,
//     dense_off + I(I+1)/2 + J), 7 slices x 4096 B, slice = [r/8][c/16][r%8][c%16] (r, c: tile row, col).
//   W^T slices (per apply): per W/V/U 64-row tile T and column tile ct (128 columns), 7 slices x 8192 B,
//     slice = [c/8][k/16][c%8][k%16] (c: column within ct, k: row within the tile).
// CTA work unit: (block j, output tile row I, column tile ct): D(c, n) = sum_K Wt_K^T Mt_(K, I)
//   A operand = W^T slices (M = 128 columns c, K-major), B operand = Mt column tile I (N = 64 rows n):
//   for K <= I the stored tile (I, K) read K-major, for K > I the stored tile (K, I) read MN-major.
#include <climits>
#include <cstdio>
#include "nsp_internal.h"
#include "nsp_dmma.cuh"

using namespace nspd;

namespace {
constexpr int OZ_NS = 7;                 // slices
constexpr int OZ_MT = OZ_NS * 4096;      // bytes: sliced 64 x 64 M tile
constexpr int OZ_AT = OZ_NS * 8192;      // bytes: sliced 128 x 64 W^T tile
constexpr int OZ_NST = 2;                // pipeline stages
constexpr int OZ_TS = 4;                 // A slices staged in TMEM (7 x 64 accumulator + 2 x 4 x 8 = 512 columns)
constexpr int OZ_SMEM = OZ_NST * (OZ_AT + OZ_MT) + 1024;

__device__ __forceinline__ uint32_t s_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// no-swizzle shared-memory matrix descriptor (sm_100, version 1): start, leading / stride byte offsets
__device__ __forceinline__ uint64_t umma_desc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((addr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | ((uint64_t)1 << 46);
}
// instruction descriptor kind::i8: s8 x s8 -> s32, M = 128, N = 64, A K-major, B K-major / MN-major
constexpr uint32_t oz_idesc(int b_mn) {
  return (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)b_mn << 16) | ((uint32_t)(64 >> 3) << 17) |
         ((uint32_t)(128 >> 4) << 24);
}
__device__ __forceinline__ void mma_i8(uint32_t d, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d),
      "l"(a), "l"(b), "r"(id), "r"(acc));
}
// A operand in TMEM (columns [ta, ta + 8)), B from shared memory
__device__ __forceinline__ void mma_i8_ts(uint32_t d, uint32_t ta, uint64_t b, uint32_t id, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(d),
      "r"(ta), "l"(b), "r"(id), "r"(acc));
}
// weight-stationary form: the B operand can be held in collector buffer b0 across consecutive MMAs (fill /
// use / lastuse), so the 7 - j products that share B slice j read it from shared memory once
#define OZ_WS_SS(QUAL, d, a, b, id, acc)                                                                 \
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"                                     \
               "tcgen05.mma.ws.cta_group::1.kind::i8" QUAL " [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d), "l"(a), \
               "l"(b), "r"(id), "r"((uint32_t)(acc)))
#define OZ_WS_TS(QUAL, d, a, b, id, acc)                                                                   \
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"                                       \
               "tcgen05.mma.ws.cta_group::1.kind::i8" QUAL " [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(d), "r"(a), \
               "l"(b), "r"(id), "r"((uint32_t)(acc)))
__device__ __forceinline__ void mma_ws(int coll, bool ts, uint32_t d, uint32_t ta, uint64_t a, uint64_t b,
                                       uint32_t id, uint32_t acc) {
  // coll: 0 none, 1 fill, 2 use, 3 lastuse
  if (ts) {
    if (coll == 1) OZ_WS_TS(".collector::b0::fill", d, ta, b, id, acc);
    else if (coll == 2) OZ_WS_TS(".collector::b0::use", d, ta, b, id, acc);
    else if (coll == 3) OZ_WS_TS(".collector::b0::lastuse", d, ta, b, id, acc);
    else OZ_WS_TS("", d, ta, b, id, acc);
  } else {
    if (coll == 1) OZ_WS_SS(".collector::b0::fill", d, a, b, id, acc);
    else if (coll == 2) OZ_WS_SS(".collector::b0::use", d, a, b, id, acc);
    else if (coll == 3) OZ_WS_SS(".collector::b0::lastuse", d, a, b, id, acc);
    else OZ_WS_SS("", d, a, b, id, acc);
  }
}
// shared memory (canonical K-major, 128 rows x 32 bytes) -> TMEM (128 lanes x 8 columns)
__device__ __forceinline__ void tc_cp(uint32_t ta, uint64_t sd) {
  asm volatile("tcgen05.cp.cta_group::1.128x256b [%0], %1;\n" ::"r"(ta), "l"(sd));
}
// bulk copy with an L2 cache policy (createpolicy: evict_last keeps the W^T slices of the running blocks -
// re-read by every unit of the block - resident against the stream of M tiles)
__device__ __forceinline__ uint64_t l2_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;\n" : "=l"(p));
  return p;
}
__device__ __forceinline__ void bulk_copy_hint(void* dst, const void* src, unsigned bytes, uint64_t* bar, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;\n" ::"r"(
          s_u32(dst)),
      "l"(src), "r"(bytes), "r"(s_u32(bar)), "l"(pol)
      : "memory");
}
// cluster of CL CTAs: the W^T slices of a K tile are multicast (each CTA fetches 1/CL of them for all), the
// stage is freed when every CTA's MMAs have read it (commit multicast to every CTA's empty barrier)
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;\n" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}
__device__ __forceinline__ void bulk_copy_mc(void* dst, const void* src, unsigned bytes, uint64_t* bar, uint16_t mask) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster [%0], [%1], %2, [%3], %4;\n" ::"r"(
          s_u32(dst)),
      "l"(src), "r"(bytes), "r"(s_u32(bar)), "h"(mask)
      : "memory");
}
__device__ __forceinline__ void mma_commit_mc(uint64_t* bar, uint16_t mask) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n" ::"r"(
                   s_u32(bar)),
               "h"(mask)
               : "memory");
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(s_u32(bar))
               : "memory");
}
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory"); }
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory"); }
__device__ __forceinline__ bool elect_one() {
  uint32_t p = 0;
  asm volatile("{\n .reg .pred P;\n elect.sync _|P, 0xffffffff;\n selp.b32 %0, 1, 0, P;\n}\n" : "=r"(p));
  return p != 0;
}
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
        "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_ld_wait() { asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory"); }

// X = rint(x 2^55) (|x| < 1/2) as 7 signed base-256 digits, most significant first
__device__ __forceinline__ void oz_digits(double x, int (&d)[OZ_NS]) {
  long long X = __double2ll_rn(x);
#pragma unroll
  for (int i = OZ_NS - 1; i > 0; --i) {
    const int lo = (int)(signed char)(X & 0xFF);
    d[i] = lo;
    X = (X - lo) >> 8;
  }
  d[0] = (int)X;
}
// exponent e with |v| < 2^e for every v of a set whose max is m (m >= 0): frexp exponent
__device__ __forceinline__ int oz_exp_above(double m) {
  if (!(m > 0.0)) return INT_MIN / 4;
  int e;
  frexp(m, &e);   // m = f 2^e, f in [0.5, 1)  ->  m < 2^e
  return e;
}

// ---------------------------------------------------------------- setup kernels
// e_n = floor(log2(M_nn) / 2) per W/V/U row (delta_n = 2^e_n); grid (nsub, max_ntb), 64 threads
__global__ void k_oz_dexp(const FacSub* __restrict__ subs, const double* __restrict__ minv, int* __restrict__ dexp) {
  const FacSub sb = subs[blockIdx.x];
  const int I = blockIdx.y;
  if (I >= sb.ntb) return;
  const int i = threadIdx.x;
  const double m = minv[(sb.dense_off + (int64_t)I * (I + 1) / 2 + I) * NSP_MINV_TILE + i * NSP_MINV_LD + i];
  int e = 0;
  if (m > 0.0 && isfinite(m)) {
    int x;
    frexp(m, &x);   // m in [2^(x-1), 2^x)
    e = (x - 1) >= 0 ? (x - 1) / 2 : -((2 - x) / 2);   // floor((x - 1) / 2)
  }
  dexp[sb.wvu_row + (int64_t)I * 64 + i] = e;
}

// mu_j exponent: max over the block's stored tiles of |M_rc| / (delta_r delta_c); items = (j, I)
__global__ void __launch_bounds__(256) k_oz_mexp(const FacSub* __restrict__ subs, const int2* __restrict__ items,
                                                 const double* __restrict__ minv, const int* __restrict__ dexp,
                                                 int* __restrict__ mexp) {
  const int2 it = items[blockIdx.x];
  const FacSub sb = subs[it.x];
  const int I = it.y;
  __shared__ double red[8];
  double mx = 0.0;
  for (int J = 0; J <= I; ++J) {
    const double* T = minv + (sb.dense_off + (int64_t)I * (I + 1) / 2 + J) * NSP_MINV_TILE;
    for (int e = threadIdx.x; e < 4096; e += 256) {
      const int r = e >> 6, c = e & 63;
      const int er = dexp[sb.wvu_row + (int64_t)I * 64 + r], ec = dexp[sb.wvu_row + (int64_t)J * 64 + c];
      mx = fmax(mx, fabs(ldexp(T[r * NSP_MINV_LD + c], -er - ec)));
    }
  }
  for (int o = 16; o; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mx;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < 8; ++w) mx = fmax(mx, red[w]);
    atomicMax(&mexp[it.x], oz_exp_above(mx) + 1);   // |Mt| / mu < 1/2
  }
}

// slices of the stored lower tiles; items = (j, I), 256 threads = 64 rows x 4 column groups of 16
// mz[t]: the number of leading slices of stored tile t that are zero in every entry (the tile's entries are
// small against the block scale mu_j: the far-apart boundary points of S_j^{-1}); the product skips their MMAs
// and their bytes (bitwise the same result: the skipped digit products are exact zeros)
__global__ void __launch_bounds__(256) k_oz_slice_m(const FacSub* __restrict__ subs, const int2* __restrict__ items,
                                                    const double* __restrict__ minv, const int* __restrict__ dexp,
                                                    const int* __restrict__ mexp, int8_t* __restrict__ msl,
                                                    int8_t* __restrict__ mz) {
  __shared__ int zmin;
  const int2 it = items[blockIdx.x];
  const FacSub sb = subs[it.x];
  const int I = it.y, mu = mexp[it.x];
  const int r = threadIdx.x >> 2, h = threadIdx.x & 3;
  const int er = dexp[sb.wvu_row + (int64_t)I * 64 + r];
  for (int J = 0; J <= I; ++J) {
    const int64_t t = sb.dense_off + (int64_t)I * (I + 1) / 2 + J;
    const double* T = minv + t * NSP_MINV_TILE + r * NSP_MINV_LD + 16 * h;
    uint32_t pk[OZ_NS][4];
#pragma unroll
    for (int i = 0; i < OZ_NS; ++i) pk[i][0] = pk[i][1] = pk[i][2] = pk[i][3] = 0u;
#pragma unroll
    for (int q = 0; q < 16; ++q) {
      const int ec = dexp[sb.wvu_row + (int64_t)J * 64 + 16 * h + q];
      int d[OZ_NS];
      oz_digits(ldexp(T[q], 55 - er - ec - mu), d);
#pragma unroll
      for (int i = 0; i < OZ_NS; ++i) pk[i][q >> 2] |= ((uint32_t)(d[i] & 0xFF)) << (8 * (q & 3));
    }
    int8_t* out = msl + t * OZ_MT + ((r >> 3) * 4 + h) * 128 + (r & 7) * 16;
#pragma unroll
    for (int i = 0; i < OZ_NS; ++i)
      *reinterpret_cast<uint4*>(out + i * 4096) = make_uint4(pk[i][0], pk[i][1], pk[i][2], pk[i][3]);
    int z = 0;   // leading all-zero slices of this thread's 16 entries
    while (z < OZ_NS - 1 && (pk[z][0] | pk[z][1] | pk[z][2] | pk[z][3]) == 0u) ++z;
    if (threadIdx.x == 0) zmin = OZ_NS;
    __syncthreads();
    atomicMin(&zmin, z);
    __syncthreads();
    if (threadIdx.x == 0) mz[t] = (int8_t)zmin;
    __syncthreads();
  }
}

// ---------------------------------------------------------------- per-apply W^T slices
// W chunk-major padded (column c of W/V/U row r at W + (c/32) cs + r * 36 + c % 32), nch chunks.
// (1) column exponents: grid (items, nct * 4), 256 threads (lane = column of the 32-column group q of column
// tile ct, warp = 8 rows of the item's 64-row tile); the max over the block's tiles is an integer atomicMax
// of exponents (order-independent: deterministic).  sexp must hold INT_MIN-ish on entry.
__global__ void __launch_bounds__(256) k_oz_wmax(const FacSub* __restrict__ subs, const int2* __restrict__ items,
                                                 const double* __restrict__ W, int64_t cs, int nch, int nct,
                                                 const int* __restrict__ dexp, int* __restrict__ sexp) {
  pdl_wait();
  const int2 it = items[blockIdx.x];
  const FacSub sb = subs[it.x];
  const int ct = blockIdx.y >> 2, q = blockIdx.y & 3;
  const int chunk = ct * 4 + q;
  if (chunk >= nch) return;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t r0 = sb.wvu_row + (int64_t)it.y * 64 + warp * 8;
  const double* Wc = W + (int64_t)chunk * cs + r0 * 36 + lane;
  double mx = 0.0;
#pragma unroll
  for (int k = 0; k < 8; ++k) mx = fmax(mx, fabs(ldexp(Wc[k * 36], dexp[r0 + k])));
  __shared__ double red[8][33];
  red[warp][lane] = mx;
  __syncthreads();
  if (warp == 0) {
#pragma unroll
    for (int w = 1; w < 8; ++w) mx = fmax(mx, red[w][lane]);
    if (mx > 0.0) atomicMax(&sexp[((int64_t)it.x * nct + ct) * 128 + q * 32 + lane], oz_exp_above(mx) + 1);
  }
}
// (2) slices: grid (items, nct * 4), 128 threads (lane = column, warp = 16-row group h of the tile)
__global__ void __launch_bounds__(128) k_oz_slice_w(const FacSub* __restrict__ subs, const int2* __restrict__ items,
                                                    const double* __restrict__ W, int64_t cs, int nch, int nct,
                                                    const int* __restrict__ dexp, const int* __restrict__ sexp,
                                                    int8_t* __restrict__ wsl) {
  pdl_wait();
  const int2 it = items[blockIdx.x];
  const FacSub sb = subs[it.x];
  const int ct = blockIdx.y >> 2, q = blockIdx.y & 3;
  const int chunk = ct * 4 + q;
  const int lane = threadIdx.x & 31, h = threadIdx.x >> 5;
  const int cc = q * 32 + lane;   // column within the column tile
  uint32_t pk[OZ_NS][4];
#pragma unroll
  for (int i = 0; i < OZ_NS; ++i) pk[i][0] = pk[i][1] = pk[i][2] = pk[i][3] = 0u;
  if (chunk < nch) {
    int e = sexp[((int64_t)it.x * nct + ct) * 128 + cc];
    if (e < -4000) e = 0;   // all-zero column
    const int64_t r0 = sb.wvu_row + (int64_t)it.y * 64 + h * 16;
    const double* Wc = W + (int64_t)chunk * cs + r0 * 36 + lane;
    double w[16];
#pragma unroll
    for (int kk = 0; kk < 16; ++kk) w[kk] = Wc[kk * 36];
#pragma unroll
    for (int kk = 0; kk < 16; ++kk) {
      int d[OZ_NS];
      oz_digits(ldexp(w[kk], 55 + dexp[r0 + kk] - e), d);
#pragma unroll
      for (int i = 0; i < OZ_NS; ++i) pk[i][kk >> 2] |= ((uint32_t)(d[i] & 0xFF)) << (8 * (kk & 3));
    }
  }
  const int64_t T = sb.wvu_row / 64 + it.y;   // W/V/U tile
  int8_t* out = wsl + (T * nct + ct) * (int64_t)OZ_AT + ((cc >> 3) * 4 + h) * 128 + (cc & 7) * 16;
#pragma unroll
  for (int i = 0; i < OZ_NS; ++i)
    *reinterpret_cast<uint4*>(out + i * 8192) = make_uint4(pk[i][0], pk[i][1], pk[i][2], pk[i][3]);
}

// ---------------------------------------------------------------- the tcgen05 product
// Persistent, one CTA per SM (TMEM: 7 accumulators x 64 columns of 512).  Warp 0: bulk-copy producer;
// warp 1: TMEM owner + MMA issuer; warps 2..9: epilogue (TMEM lane quarter = warp % 4, 32 of the 64 rows n).
// Work unit t in [0, nitems * nct): item t % nitems, column tile t / nitems.
// K-tile order of a unit (block j, output tile row I): natural 0, 1, ..., or (diagnostic NSP_OZ_DBG bit 8)
// I, I + 1, I - 1, I + 2, I - 2, ... in which the two readers of a stored tile (a, b) reach it at the same
// step.  With the dynamic unit counter the units of one block run side by side and either order re-reads
// the stored tiles from L2 (cfg5 DRAM per launch 69 GB -> 49.2 GB natural / 46.9 GB symmetric against
// 45.2 GB unique; time 26.2 vs 26.5 ms: the natural order is kept).
struct OzKOrder {
  int I, ntb, lo, hi, side, K;
  __device__ OzKOrder(int I_, int ntb_, bool natural) : I(I_), ntb(ntb_), lo(I_ - 1), hi(I_ + 1), side(0) {
    K = natural ? 0 : I_;
    if (natural) lo = -2;   // marks the natural order
  }
  __device__ void next() {
    if (lo == -2) {
      ++K;
      return;
    }
    if ((side == 0 && hi < ntb) || lo < 0) {
      K = hi++;
      side = 1;
    } else {
      K = lo--;
      side = 0;
    }
  }
};

// CL = 2: clusters of two CTAs take pair units (block j, tile rows I0, I0 + 1) from items = (j, I0) (I0 even);
// the second CTA of a pair whose I0 + 1 = ntb_j recomputes tile I0 and discards it (the multicast protocol
// needs both CTAs to walk the same K loop)
template <int CL>
__global__ void __launch_bounds__(320, 1) k_oz_symm(const FacSub* __restrict__ subs, const int2* __restrict__ items,
                                                    int nitems, int nct, const int8_t* __restrict__ msl,
                                                    const int8_t* __restrict__ wsl, const int* __restrict__ dexp,
                                                    const int* __restrict__ mexp, const int* __restrict__ sexp,
                                                    double* __restrict__ U, int64_t cs, int nch, int dbg,
                                                    int* __restrict__ uctr, const int8_t* __restrict__ mz) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ __align__(8) uint64_t full[OZ_NST], empty[OZ_NST], tfull, tempty, ufull[4], uempty[4];
  __shared__ uint32_t tbase;
  __shared__ int uring[4];
  uint8_t* base = (uint8_t*)(((uintptr_t)sm + 1023) & ~(uintptr_t)1023);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nunits = nitems * nct;
  const int crank = CL == 2 ? (int)cluster_rank() : 0;
  const int cid = blockIdx.x / CL, ncl = gridDim.x / CL;
  if (threadIdx.x == 0) {
    for (int s = 0; s < OZ_NST; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], CL);
    }
    mbar_init(&tfull, 1);
    mbar_init(&tempty, 8);
    for (int q = 0; q < 4; ++q) {
      mbar_init(&ufull[q], 1);
      mbar_init(&uempty[q], 9);
    }
    fence_mbar_init();
  }
  // work units: dynamic (uctr: one atomic grab per unit, in order, so the units of one block run side by side
  // and share their W^T and M tiles through L2; also no tail imbalance) or the static cid, cid + ncl, ...;
  // the producer publishes every unit index to the MMA and epilogue warps through a 4-deep ring
  const bool dyn = CL == 1 && uctr != nullptr;
  int ustat = cid, uslot = 0;
  uint32_t uph = 0;
  auto publish = [&]() -> int {   // producer thread
    const int u = dyn ? atomicAdd(uctr, 1) : ustat;
    ustat += ncl;
    mbar_wait(&uempty[uslot], uph ^ 1);
    *(volatile int*)&uring[uslot] = u;
    mbar_arrive(&ufull[uslot]);
    if (++uslot == 4) uslot = 0, uph ^= 1;
    return u;
  };
  auto receive = [&]() -> int {   // every lane of a consumer warp
    mbar_wait(&ufull[uslot], uph);
    const int u = *(volatile int*)&uring[uslot];
    __syncwarp();
    if (lane == 0) mbar_arrive(&uempty[uslot]);
    if (++uslot == 4) uslot = 0, uph ^= 1;
    return u;
  };
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(s_u32(&tbase)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  tc_fence_before();
  if (CL == 2) cluster_sync_all();   // the peer's barriers exist before any multicast targets them
  else __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tbase;
  pdl_wait();
  if (warp == 0) {
    if (elect_one()) {   // producer
      int st = 0;
      uint32_t ph = 0;
      const bool hint = (dbg & 4) == 0;
      const uint64_t pol = l2_evict_last();
      for (int u = publish(); u < nunits; u = publish()) {
        const int2 it = items[u % nitems];
        const int ct = u / nitems;
        const FacSub sb = subs[it.x];
        const int I = min(it.y + crank, sb.ntb - 1);
        const int64_t T0 = sb.wvu_row / 64;
        OzKOrder ko(I, sb.ntb, CL == 2 || !(dbg & 8));
        for (int step = 0; step < sb.ntb; ++step, ko.next()) {
          const int K = ko.K;
          const int64_t t = sb.dense_off + (K <= I ? (int64_t)I * (I + 1) / 2 + K : (int64_t)K * (K + 1) / 2 + I);
          // leading zero slices are neither loaded nor multiplied (all of them on a unit's first K tile, whose
          // products initialise the accumulators)
          const int zt = (mz && step > 0) ? mz[t] : 0;
          // with zt zero B slices only the W^T slices i <= 6 - zt meet a product (i + j < 7, j >= zt): the
          // rest are not loaded either (diagnostic bit 64 loads all 7)
          const int abytes = (CL == 1 && !(dbg & 64)) ? (OZ_NS - zt) * 8192 : OZ_AT;
          mbar_wait(&empty[st], ph ^ 1);
          uint8_t* As = base + st * (OZ_AT + OZ_MT);
          mbar_expect(&full[st], ((dbg & 1) ? 0 : abytes) + ((dbg & 2) ? 0 : OZ_MT - zt * 4096) + ((dbg & 3) == 3 ? 16 : 0));
          const int8_t* Ag = wsl + ((T0 + K) * nct + ct) * (int64_t)OZ_AT;
          if (CL == 2) {
            if (!(dbg & 1))
              bulk_copy_mc(As + crank * (OZ_AT / 2), Ag + crank * (OZ_AT / 2), OZ_AT / 2, &full[st], (uint16_t)3);
          } else if (!(dbg & 1)) {
            if (hint) bulk_copy_hint(As, Ag, abytes, &full[st], pol);
            else bulk_copy(As, Ag, abytes, &full[st]);
          }
          if (!(dbg & 2))
            bulk_copy(As + OZ_AT + zt * 4096, msl + t * OZ_MT + zt * 4096, OZ_MT - zt * 4096, &full[st]);
          if ((dbg & 3) == 3) bulk_copy(As, wsl, 16, &full[st]);
          if (++st == OZ_NST) st = 0, ph ^= 1;
        }
      }
    }
  } else if (warp == 1) {
    int st = 0;
    uint32_t ph = 0, tph = 0;
#ifdef NSP_OZ_PROF
    long long t_tmem = 0, t_full = 0, t_all = clock64();
#endif
    constexpr uint32_t ID_K = oz_idesc(0), ID_MN = oz_idesc(1);
    // diagnostic bit 16: the B-stationary order with collector reuse (tcgen05.mma.ws) - parity-clean and faster
    // in isolation (tools/bench_i8mma.cu: 1,344 -> 1,177 cycles per K-step for the all-SS form) but slower here
    // combined with the TMEM-sourced A slices (cfg5 27.25 vs 25.93 ms per launch): off
    const bool ws = (dbg & 16) != 0;
    for (int u = receive(); u < nunits; u = receive()) {
      const int2 it = items[u % nitems];
      const int ntb = subs[it.x].ntb;
      const int I = min(it.y + crank, ntb - 1);
#ifdef NSP_OZ_PROF
      long long t0 = clock64();
#endif
      mbar_wait(&tempty, tph ^ 1);   // the epilogue has drained the previous unit's accumulators
#ifdef NSP_OZ_PROF
      t_tmem += clock64() - t0;
#endif
      tc_fence_after();
      OzKOrder ko(I, ntb, CL == 2 || !(dbg & 8));
      for (int step = 0; step < ntb; ++step, ko.next()) {
        const int K = ko.K;
        const int zt = (mz && step > 0)
                           ? mz[subs[it.x].dense_off + (K <= I ? (int64_t)I * (I + 1) / 2 + K : (int64_t)K * (K + 1) / 2 + I)]
                           : 0;
#ifdef NSP_OZ_PROF
        long long t1 = clock64();
#endif
        mbar_wait(&full[st], ph);
#ifdef NSP_OZ_PROF
        t_full += clock64() - t1;
#endif
        tc_fence_after();
        if (elect_one()) {
          const uint32_t a0 = s_u32(base + st * (OZ_AT + OZ_MT)), b0 = a0 + OZ_AT;
          const bool mn = K > I;
          const uint32_t id = mn ? ID_MN : ID_K;
#pragma unroll
          for (int k = 0; k < 2; ++k) {
            // the OZ_TS most-used A slices (slice i feeds 7 - i products) are staged in TMEM (tcgen05.cp,
            // 8 columns each, double-buffered per K-step in columns 448..511): a TMEM-sourced MMA skips the
            // 4 KB shared-memory A read that holds the SS form at 48 instead of 32 cycles (measured,
            // tools/bench_i8mma.cu: 1344 -> 1120 cycles per K-step of 28 products)
            const uint32_t ta = tmem + 448u + (uint32_t)(k * 8 * OZ_TS);
#pragma unroll
            for (int i = 0; i < OZ_TS; ++i) tc_cp(ta + 8 * i, umma_desc(a0 + i * 8192 + k * 256, 128, 512));
            if (ws) {   // B-stationary order: j outer, the products sharing B slice j read it once (collector b0)
#pragma unroll
              for (int j = 0; j < OZ_NS; ++j) {
                const uint64_t db = mn ? umma_desc(b0 + j * 4096 + k * 2048, 512, 128)
                                       : umma_desc(b0 + j * 4096 + k * 256, 128, 512);
#pragma unroll
                for (int i = 0; i + j < OZ_NS; ++i) {
                  const uint32_t dd = tmem + (uint32_t)((i + j) * 64);
                  const int coll = (j == OZ_NS - 1) ? 0 : (i == 0 ? 1 : (i + j == OZ_NS - 1 ? 3 : 2));
                  mma_ws(coll, i < OZ_TS, dd, ta + 8 * i, umma_desc(a0 + i * 8192 + k * 256, 128, 512), db, id,
                         (step | k | j) != 0);   // the first product into diagonal i + j is the one with j = 0
                }
              }
            } else {
#pragma unroll
              for (int i = 0; i < OZ_NS; ++i)
#pragma unroll
                for (int j = 0; i + j < OZ_NS; ++j) {
                  const uint64_t db = mn ? umma_desc(b0 + j * 4096 + k * 2048, 512, 128)
                                         : umma_desc(b0 + j * 4096 + k * 256, 128, 512);
                  const uint32_t dd = tmem + (uint32_t)((i + j) * 64);
                  if (j < zt) continue;   // a zero B slice (never on step 0)
                  if (i < OZ_TS) mma_i8_ts(dd, ta + 8 * i, db, id, (step | k | i) != 0);
                  else mma_i8(dd, umma_desc(a0 + i * 8192 + k * 256, 128, 512), db, id, (step | k | i) != 0);
                }
            }
          }
          if (CL == 2) mma_commit_mc(&empty[st], (uint16_t)3);   // frees the stage in both CTAs' accounting
          else mma_commit(&empty[st]);   // frees the stage once these MMAs have read it
          if (step == ntb - 1) mma_commit(&tfull);
        }
        __syncwarp();
        if (++st == OZ_NST) st = 0, ph ^= 1;
      }
      tph ^= 1;
    }
#ifdef NSP_OZ_PROF
    if (lane == 0 && uctr) {
      atomicAdd((unsigned long long*)(uctr + 64), (unsigned long long)t_tmem);
      atomicAdd((unsigned long long*)(uctr + 66), (unsigned long long)t_full);
      atomicAdd((unsigned long long*)(uctr + 68), (unsigned long long)(clock64() - t_all));
    }
#endif
  } else {   // epilogue warps 2..9: TMEM lane quarter warp % 4, n-column half (warp - 2) / 4
    const int qd = warp & 3;
    const int half = (warp - 2) >> 2;
    const int cc = qd * 32 + lane;
    uint32_t tph = 0;
    for (int u = receive(); u < nunits; u = receive()) {
      const int2 it = items[u % nitems];
      const int ct = u / nitems;
      const FacSub sb = subs[it.x];
      const int I = it.y + crank;
      const int chunk = (I < sb.ntb) ? ct * 4 + qd : nch;   // a discarded duplicate tile: no stores
      const int ex = sexp[((int64_t)it.x * nct + ct) * 128 + cc] + mexp[it.x];
      const int64_t row0 = sb.wvu_row + (int64_t)I * 64;
      double* out = U + (int64_t)chunk * cs + row0 * 36 + lane;
      mbar_wait(&tfull, tph);
      tc_fence_after();
#pragma unroll 1
      for (int nb = 2 * half; nb < 2 * half + 2; ++nb) {
        uint32_t v[OZ_NS][16];
#pragma unroll
        for (int a = 0; a < OZ_NS; ++a)
          tmem_ld16(tmem + ((uint32_t)(qd * 32) << 16) + (uint32_t)(a * 64 + nb * 16), v[a]);
        tmem_ld_wait();
        if (chunk < nch) {
#pragma unroll
          for (int nn = 0; nn < 16; ++nn) {
            // diagonal a carries weight 2^(-14-8a): the three leading diagonals combine exactly into an int64
            // (< 2^48, exact in fp64), the four trailing ones into a second (< 2^56)
            const long long hi = ((long long)(int)v[0][nn] << 16) + ((long long)(int)v[1][nn] << 8) + (int)v[2][nn];
            const long long lo = ((long long)(int)v[3][nn] << 24) + ((long long)(int)v[4][nn] << 16) +
                                 ((long long)(int)v[5][nn] << 8) + (int)v[6][nn];
            const double acc = fma((double)hi, 0x1p-30, (double)lo * 0x1p-62);
            const int n = nb * 16 + nn;
            const int E = ex + dexp[row0 + n];
            out[(int64_t)n * 36] = (E >= -1022 && E <= 1023) ? acc * __longlong_as_double((long long)(E + 1023) << 52)
                                                             : ldexp(acc, E);
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty);
      tph ^= 1;
    }
  }
  tc_fence_before();
  if (CL == 2) cluster_sync_all();   // no CTA leaves while its peer may still multicast / commit into it
  else __syncthreads();
  if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tmem));
}

// ---------------------------------------------------------------- register-staged variant (opt-in, slower)
// The four most-used W^T slices reach TMEM from REGISTERS (tcgen05.st by the epilogue warps, which are idle
// while the tensor core runs), not through shared memory: the shared-memory port - the binding resource of
// k_oz_symm (per K-step 96 KB of MMA / copy reads + 42 KB of TMA writes at 128 B/clk) - then carries only
// slices 4..6 and the M tile (per K-step 80 KB reads + 26 KB writes), and the tensor pipe runs no tcgen05.cp:
// 6 x 48 + 22 x 32 = 992 cycles per K-step instead of 1,120.  TMEM: 7 x 64 accumulator columns + 2 buffers
// x 4 slices x 8 columns.  Per K-step g the stagers fill buffer g & 1 (afull, 8 warp arrivals) once the MMAs
// of step g - 2 have released it (afree, one commit); the W^T rows are prefetched into registers one K-step
// ahead.  The first K-step of unit u + 1 is staged before unit u's epilogue, so the tensor core restarts as
// soon as the accumulators are drained.
constexpr int RS_NST = 3;
constexpr int RS_AT = 3 * 8192;                  // slices 4..6 of the W^T tile
constexpr int RS_STAGE = RS_AT + OZ_MT;
constexpr int RS_SMEM = RS_NST * RS_STAGE + 1024;

__device__ __forceinline__ void tmem_st8(uint32_t taddr, uint4 a, uint4 b) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};\n" ::"r"(taddr), "r"(a.x),
               "r"(a.y), "r"(a.z), "r"(a.w), "r"(b.x), "r"(b.y), "r"(b.z), "r"(b.w)
               : "memory");
}
__device__ __forceinline__ void tmem_st_wait() { asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory"); }

struct OzStep {   // position in a CTA's (unit, K tile, K-step) sequence
  int u, K, k, ntb;
  int2 it;
  bool valid;
};

__global__ void __launch_bounds__(320, 1) k_oz_symm_rs(const FacSub* __restrict__ subs, const int2* __restrict__ items,
                                                       int nitems, int nct, const int8_t* __restrict__ msl,
                                                       const int8_t* __restrict__ wsl, const int* __restrict__ dexp,
                                                       const int* __restrict__ mexp, const int* __restrict__ sexp,
                                                       double* __restrict__ U, int64_t cs, int nch) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ __align__(8) uint64_t full[RS_NST], empty[RS_NST], afull[2], afree[2], tfull, tempty;
  __shared__ uint32_t tbase;
  uint8_t* base = (uint8_t*)(((uintptr_t)sm + 1023) & ~(uintptr_t)1023);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nunits = nitems * nct;
  if (threadIdx.x == 0) {
    for (int s = 0; s < RS_NST; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&afull[b], 8);
      mbar_init(&afree[b], 1);
    }
    mbar_init(&tfull, 1);
    mbar_init(&tempty, 8);
    fence_mbar_init();
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(s_u32(&tbase)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tbase;
  pdl_wait();
  if (warp == 0) {
    if (elect_one()) {   // producer: slices 4..6 of the W^T tile + the stored M tile per K tile
      int st = 0;
      uint32_t ph = 0;
      for (int u = blockIdx.x; u < nunits; u += gridDim.x) {
        const int2 it = items[u % nitems];
        const int ct = u / nitems;
        const FacSub sb = subs[it.x];
        const int I = it.y;
        const int64_t T0 = sb.wvu_row / 64;
        for (int K = 0; K < sb.ntb; ++K) {
          mbar_wait(&empty[st], ph ^ 1);
          uint8_t* As = base + st * RS_STAGE;
          mbar_expect(&full[st], RS_AT + OZ_MT);
          bulk_copy(As, wsl + ((T0 + K) * nct + ct) * (int64_t)OZ_AT + 4 * 8192, RS_AT, &full[st]);
          const int64_t t = sb.dense_off + (K <= I ? (int64_t)I * (I + 1) / 2 + K : (int64_t)K * (K + 1) / 2 + I);
          bulk_copy(As + RS_AT, msl + t * OZ_MT, OZ_MT, &full[st]);
          if (++st == RS_NST) st = 0, ph ^= 1;
        }
      }
    }
  } else if (warp == 1) {   // MMA issuer
    int st = 0;
    uint32_t ph = 0, tph = 0, g = 0;
    constexpr uint32_t ID_K = oz_idesc(0), ID_MN = oz_idesc(1);
    for (int u = blockIdx.x; u < nunits; u += gridDim.x) {
      const int2 it = items[u % nitems];
      const int I = it.y, ntb = subs[it.x].ntb;
      mbar_wait(&tempty, tph ^ 1);   // the epilogue has drained the previous unit's accumulators
      tc_fence_after();
      for (int K = 0; K < ntb; ++K) {
        mbar_wait(&full[st], ph);
        const uint32_t a0 = s_u32(base + st * RS_STAGE), b0 = a0 + RS_AT;
        const bool mn = K > I;
        const uint32_t id = mn ? ID_MN : ID_K;
#pragma unroll
        for (int k = 0; k < 2; ++k, ++g) {
          const uint32_t b = g & 1;
          mbar_wait(&afull[b], (g >> 1) & 1);
          tc_fence_after();
          if (elect_one()) {
            const uint32_t ta = tmem + 448u + 32u * b;
#pragma unroll
            for (int i = 0; i < OZ_NS; ++i)
#pragma unroll
              for (int j = 0; i + j < OZ_NS; ++j) {
                const uint64_t db = mn ? umma_desc(b0 + j * 4096 + k * 2048, 512, 128)
                                       : umma_desc(b0 + j * 4096 + k * 256, 128, 512);
                const uint32_t dd = tmem + (uint32_t)((i + j) * 64);
                if (i < 4) mma_i8_ts(dd, ta + 8 * i, db, id, (K | k | i) != 0);
                else mma_i8(dd, umma_desc(a0 + (i - 4) * 8192 + k * 256, 128, 512), db, id, (K | k | i) != 0);
              }
            mma_commit(&afree[b]);                 // the staging buffer is free once these MMAs have read it
            if (k == 1) mma_commit(&empty[st]);    // and the shared-memory stage after the second K-step
            if (k == 1 && K == ntb - 1) mma_commit(&tfull);
          }
          __syncwarp();
        }
        if (++st == RS_NST) st = 0, ph ^= 1;
      }
      tph ^= 1;
    }
  } else {   // warps 2..9: stage W^T slices {2 grp, 2 grp + 1} into TMEM; epilogue half grp
    const int qd = warp & 3;
    const int grp = (warp - 2) >> 2;
    const int cc = qd * 32 + lane;
    auto first_of = [&](int u) {
      OzStep p;
      p.u = u;
      p.K = 0;
      p.k = 0;
      p.valid = u < nunits;
      if (p.valid) {
        p.it = items[u % nitems];
        p.ntb = subs[p.it.x].ntb;
      }
      return p;
    };
    auto advance = [&](OzStep p) {
      if (++p.k == 2) {
        p.k = 0;
        if (++p.K == p.ntb) return first_of(p.u + gridDim.x);
      }
      return p;
    };
    auto load = [&](const OzStep& p, uint4 (&r)[4]) {
      const FacSub sb = subs[p.it.x];
      const int ct = p.u / nitems;
      const int8_t* Ag = wsl + ((sb.wvu_row / 64 + p.K) * nct + ct) * (int64_t)OZ_AT +
                         ((cc >> 3) * 4 + 2 * p.k) * 128 + (cc & 7) * 16;
#pragma unroll
      for (int sl = 0; sl < 2; ++sl) {
        const int8_t* q = Ag + (2 * grp + sl) * 8192;
        r[2 * sl] = __ldg(reinterpret_cast<const uint4*>(q));
        r[2 * sl + 1] = __ldg(reinterpret_cast<const uint4*>(q + 128));
      }
    };
    auto epilogue = [&](int u, uint32_t tph) {
      const int2 it = items[u % nitems];
      const int ct = u / nitems;
      const FacSub sb = subs[it.x];
      const int I = it.y;
      const int chunk = ct * 4 + qd;
      const int ex = sexp[((int64_t)it.x * nct + ct) * 128 + cc] + mexp[it.x];
      const int64_t row0 = sb.wvu_row + (int64_t)I * 64;
      double* out = U + (int64_t)chunk * cs + row0 * 36 + lane;
      mbar_wait(&tfull, tph);
      tc_fence_after();
#pragma unroll 1
      for (int nb = 2 * grp; nb < 2 * grp + 2; ++nb) {
        uint32_t v[OZ_NS][16];
#pragma unroll
        for (int a = 0; a < OZ_NS; ++a)
          tmem_ld16(tmem + ((uint32_t)(qd * 32) << 16) + (uint32_t)(a * 64 + nb * 16), v[a]);
        tmem_ld_wait();
        if (chunk < nch) {
#pragma unroll
          for (int nn = 0; nn < 16; ++nn) {
            const long long hi = ((long long)(int)v[0][nn] << 16) + ((long long)(int)v[1][nn] << 8) + (int)v[2][nn];
            const long long lo = ((long long)(int)v[3][nn] << 24) + ((long long)(int)v[4][nn] << 16) +
                                 ((long long)(int)v[5][nn] << 8) + (int)v[6][nn];
            const double acc = fma((double)hi, 0x1p-30, (double)lo * 0x1p-62);
            const int n = nb * 16 + nn;
            const int E = ex + dexp[row0 + n];
            out[(int64_t)n * 36] = (E >= -1022 && E <= 1023) ? acc * __longlong_as_double((long long)(E + 1023) << 52)
                                                             : ldexp(acc, E);
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty);
    };
    OzStep cur = first_of(blockIdx.x);
    OzStep nx1 = cur.valid ? advance(cur) : cur;
    uint4 rn[4], rn2[4];
    if (cur.valid) load(cur, rn);
    if (nx1.valid) load(nx1, rn2);
    uint32_t g = 0, tph = 0;
    int pend = -1;   // unit whose epilogue is due
    while (cur.valid) {
      uint4 rc[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) rc[q] = rn[q], rn[q] = rn2[q];
      const OzStep nxt = nx1;
      const OzStep nx2 = nx1.valid ? advance(nx1) : nx1;
      if (nx2.valid) load(nx2, rn2);   // two K-steps ahead
      const uint32_t b = g & 1;
      mbar_wait(&afree[b], ((g >> 1) & 1) ^ 1);
      tc_fence_after();
      const uint32_t ta = tmem + ((uint32_t)(qd * 32) << 16) + 448u + 32u * b + 16u * grp;
      tmem_st8(ta, rc[0], rc[1]);
      tmem_st8(ta + 8, rc[2], rc[3]);
      tmem_st_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&afull[b]);
      ++g;
      if (cur.K == 0 && cur.k == 0 && pend >= 0) {   // the next unit's first step is staged: drain the last
        epilogue(pend, tph);
        tph ^= 1;
      }
      if (cur.K == 0 && cur.k == 0) pend = cur.u;
      cur = nxt;
      nx1 = nx2;
    }
    if (pend >= 0) epilogue(pend, tph);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tmem));
}

// ---------------------------------------------------------------- register-staged variant 2 (opt-in, slower)
// NSP_OZ_KERNEL=3; parity-clean, measured 28.6 vs 26.2 ms per cfg5 launch (profiles/r02_ab_oz_register_staged2.txt).
// As k_oz_symm_rs, but the four most-used W^T slices are staged by four DEDICATED warps (one per TMEM lane
// quarter) that keep three K-steps of them in registers (loads issued two K-steps ahead of their st), so the
// staging never waits on a load; the epilogue warps only drain the accumulators; units come from the dynamic
// counter through the shared-memory ring (13 consumer warps).  Tensor pipe per K-step: 22 TMEM-A + 6
// shared-memory-A MMAs, no copies (992 instead of 1,120 cycles).
__device__ __forceinline__ void tmem_ld8(uint32_t taddr, uint32_t (&v)[8]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n"
               : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
               : "r"(taddr));
}

__global__ void __launch_bounds__(448, 1) k_oz_symm_rs2(const FacSub* __restrict__ subs, const int2* __restrict__ items,
                                                        int nitems, int nct, const int8_t* __restrict__ msl,
                                                        const int8_t* __restrict__ wsl, const int* __restrict__ dexp,
                                                        const int* __restrict__ mexp, const int* __restrict__ sexp,
                                                        double* __restrict__ U, int64_t cs, int nch,
                                                        int* __restrict__ uctr) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ __align__(8) uint64_t full[RS_NST], empty[RS_NST], afull[2], afree[2], tfull, tempty, ufull[4], uempty[4];
  __shared__ uint32_t tbase;
  __shared__ int uring[4];
  uint8_t* base = (uint8_t*)(((uintptr_t)sm + 1023) & ~(uintptr_t)1023);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nunits = nitems * nct;
  if (threadIdx.x == 0) {
    for (int s = 0; s < RS_NST; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&afull[b], 4);
      mbar_init(&afree[b], 1);
    }
    mbar_init(&tfull, 1);
    mbar_init(&tempty, 8);
    for (int q = 0; q < 4; ++q) {
      mbar_init(&ufull[q], 1);
      mbar_init(&uempty[q], 13);
    }
    fence_mbar_init();
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(s_u32(&tbase)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tbase;
  pdl_wait();
  int uslot = 0;
  uint32_t uph = 0;
  int ustat = blockIdx.x;
  auto publish = [&]() -> int {
    const int u = uctr ? atomicAdd(uctr, 1) : ustat;
    ustat += gridDim.x;
    mbar_wait(&uempty[uslot], uph ^ 1);
    *(volatile int*)&uring[uslot] = u;
    mbar_arrive(&ufull[uslot]);
    if (++uslot == 4) uslot = 0, uph ^= 1;
    return u;
  };
  auto receive = [&]() -> int {
    mbar_wait(&ufull[uslot], uph);
    const int u = *(volatile int*)&uring[uslot];
    __syncwarp();
    if (lane == 0) mbar_arrive(&uempty[uslot]);
    if (++uslot == 4) uslot = 0, uph ^= 1;
    return u;
  };
  if (warp == 0) {
    if (elect_one()) {   // producer: slices 4..6 of the W^T tile + the stored M tile per K tile
      int st = 0;
      uint32_t ph = 0;
      const uint64_t pol = l2_evict_last();
      for (int u = publish(); u < nunits; u = publish()) {
        const int2 it = items[u % nitems];
        const int ct = u / nitems;
        const FacSub sb = subs[it.x];
        const int I = it.y;
        const int64_t T0 = sb.wvu_row / 64;
        for (int K = 0; K < sb.ntb; ++K) {
          mbar_wait(&empty[st], ph ^ 1);
          uint8_t* As = base + st * RS_STAGE;
          mbar_expect(&full[st], RS_AT + OZ_MT);
          bulk_copy_hint(As, wsl + ((T0 + K) * nct + ct) * (int64_t)OZ_AT + 4 * 8192, RS_AT, &full[st], pol);
          const int64_t t = sb.dense_off + (K <= I ? (int64_t)I * (I + 1) / 2 + K : (int64_t)K * (K + 1) / 2 + I);
          bulk_copy(As + RS_AT, msl + t * OZ_MT, OZ_MT, &full[st]);
          if (++st == RS_NST) st = 0, ph ^= 1;
        }
      }
    }
  } else if (warp == 1) {   // MMA issuer
    int st = 0;
    uint32_t ph = 0, tph = 0, g = 0;
    constexpr uint32_t ID_K = oz_idesc(0), ID_MN = oz_idesc(1);
    for (int u = receive(); u < nunits; u = receive()) {
      const int2 it = items[u % nitems];
      const int I = it.y, ntb = subs[it.x].ntb;
      mbar_wait(&tempty, tph ^ 1);
      tc_fence_after();
      for (int K = 0; K < ntb; ++K) {
        mbar_wait(&full[st], ph);
        const uint32_t a0 = s_u32(base + st * RS_STAGE), b0 = a0 + RS_AT;
        const bool mn = K > I;
        const uint32_t id = mn ? ID_MN : ID_K;
#pragma unroll
        for (int k = 0; k < 2; ++k, ++g) {
          const uint32_t b = g & 1;
          mbar_wait(&afull[b], (g >> 1) & 1);
          tc_fence_after();
          if (elect_one()) {
            const uint32_t ta = tmem + 448u + 32u * b;
#pragma unroll
            for (int i = 0; i < OZ_NS; ++i)
#pragma unroll
              for (int j = 0; i + j < OZ_NS; ++j) {
                const uint64_t db = mn ? umma_desc(b0 + j * 4096 + k * 2048, 512, 128)
                                       : umma_desc(b0 + j * 4096 + k * 256, 128, 512);
                const uint32_t dd = tmem + (uint32_t)((i + j) * 64);
                if (i < 4) mma_i8_ts(dd, ta + 8 * i, db, id, (K | k | i) != 0);
                else mma_i8(dd, umma_desc(a0 + (i - 4) * 8192 + k * 256, 128, 512), db, id, (K | k | i) != 0);
              }
            mma_commit(&afree[b]);
            if (k == 1) mma_commit(&empty[st]);
            if (k == 1 && K == ntb - 1) mma_commit(&tfull);
          }
          __syncwarp();
        }
        if (++st == RS_NST) st = 0, ph ^= 1;
      }
      tph ^= 1;
    }
  } else if (warp < 10) {   // epilogue warps 2..9
    const int qd = warp & 3;
    const int half = (warp - 2) >> 2;
    const int cc = qd * 32 + lane;
    uint32_t tph = 0;
    for (int u = receive(); u < nunits; u = receive()) {
      const int2 it = items[u % nitems];
      const int ct = u / nitems;
      const FacSub sb = subs[it.x];
      const int I = it.y;
      const int chunk = ct * 4 + qd;
      const int ex = sexp[((int64_t)it.x * nct + ct) * 128 + cc] + mexp[it.x];
      const int64_t row0 = sb.wvu_row + (int64_t)I * 64;
      double* out = U + (int64_t)chunk * cs + row0 * 36 + lane;
      mbar_wait(&tfull, tph);
      tc_fence_after();
#pragma unroll 1
      for (int nb = 4 * half; nb < 4 * half + 4; ++nb) {
        uint32_t v[OZ_NS][8];
#pragma unroll
        for (int a = 0; a < OZ_NS; ++a) tmem_ld8(tmem + ((uint32_t)(qd * 32) << 16) + (uint32_t)(a * 64 + nb * 8), v[a]);
        tmem_ld_wait();
        if (chunk < nch) {
#pragma unroll
          for (int nn = 0; nn < 8; ++nn) {
            const long long hi = ((long long)(int)v[0][nn] << 16) + ((long long)(int)v[1][nn] << 8) + (int)v[2][nn];
            const long long lo = ((long long)(int)v[3][nn] << 24) + ((long long)(int)v[4][nn] << 16) +
                                 ((long long)(int)v[5][nn] << 8) + (int)v[6][nn];
            const double acc = fma((double)hi, 0x1p-30, (double)lo * 0x1p-62);
            const int n = nb * 8 + nn;
            const int E = ex + dexp[row0 + n];
            out[(int64_t)n * 36] = (E >= -1022 && E <= 1023) ? acc * __longlong_as_double((long long)(E + 1023) << 52)
                                                             : ldexp(acc, E);
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty);
      tph ^= 1;
    }
  } else {   // stager warps 10..13: TMEM lane quarter warp % 4, the four most-used W^T slices of every K-step
    const int qd = warp & 3;
    const int cc = qd * 32 + lane;
    const int64_t roff = ((cc >> 3) * 4) * 128 + (cc & 7) * 16;   // row cc's bytes inside a slice (K-step 0)
    // step iterator (unit u, K tile, K-step k); the next unit is received when a unit's steps are exhausted
    int u = receive();
    int ntb = 0, K = 0, k = 0;
    const int8_t* ub = nullptr;   // W^T slices of the unit's first K tile, row cc
    auto set_unit = [&]() {
      if (u < nunits) {
        const int2 it = items[u % nitems];
        const FacSub sb = subs[it.x];
        ntb = sb.ntb;
        ub = wsl + ((sb.wvu_row / 64) * nct + u / nitems) * (int64_t)OZ_AT + roff;
      }
      K = 0;
      k = 0;
    };
    set_unit();
    // the iterator position of the NEXT load
    auto load = [&](uint4 (&r)[8]) -> bool {
      if (u >= nunits) return false;
      const int8_t* q = ub + (int64_t)K * nct * OZ_AT + k * 256;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        r[2 * i] = __ldg(reinterpret_cast<const uint4*>(q + i * 8192));
        r[2 * i + 1] = __ldg(reinterpret_cast<const uint4*>(q + i * 8192 + 128));
      }
      if (++k == 2) {
        k = 0;
        if (++K == ntb) {
          u = receive();
          set_unit();
        }
      }
      return true;
    };
    uint32_t g = 0;
    auto stage = [&](const uint4 (&r)[8]) {
      const uint32_t b = g & 1;
      mbar_wait(&afree[b], ((g >> 1) & 1) ^ 1);
      tc_fence_after();
      const uint32_t ta = tmem + ((uint32_t)(qd * 32) << 16) + 448u + 32u * b;
#pragma unroll
      for (int i = 0; i < 4; ++i) tmem_st8(ta + 8 * i, r[2 * i], r[2 * i + 1]);
      tmem_st_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&afull[b]);
      ++g;
    };
    uint4 r0[8], r1[8], r2[8];
    bool v0 = load(r0), v1 = load(r1), v2;
    while (v0) {
      v2 = load(r2);
      stage(r0);
      if (!v1) break;
      v0 = load(r0);
      stage(r1);
      if (!v2) break;
      v1 = load(r1);
      stage(r2);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tmem));
}

// ---------------------------------------------------------------- s = 1: the matrix-vector product on the slices
// u_j = S_j^{-1} w_j for one column (the outer PCG's apply) from the same int8 slices, read once per stored tile
// (k_symv1's symmetric single read: the CTA of stored row I forms M_IJ w_J for row I and M_IJ^T w_I for row J).
// Each entry is decoded exactly: X = rint(2^55 Mt) = hi 2^32 + lo from its 7 digits, (double)hi 2^32 + (double)lo
// (exact parts, one rounding); u_n = delta_n mu_j 2^-55 sum_k X_nk (delta_k w_k).  7 instead of 8.5 bytes per stored
// entry (no fp64 tile padding).  Partials are scaled in the fixed-order reduce.
__global__ void __launch_bounds__(256, 2) k_oz_symv1(const FacSub* __restrict__ subs, const int2* __restrict__ items,
                                                  const int8_t* __restrict__ msl, const int* __restrict__ dexp,
                                                  const double* __restrict__ W, int ldw, int max_ntb,
                                                  double* __restrict__ P) {
  pdl_wait();
  extern __shared__ double wv[];            // ntb x 64: delta_k w_k of the block
  __shared__ double cpart[8][64];
  const int2 it = items[blockIdx.x];
  const FacSub sb = subs[it.x];
  const int I = it.y, ntb = sb.ntb;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int rr = lane >> 2, h = lane & 3;   // row 8 warp + rr, columns 16 h .. 16 h + 15
  const double* Wb = W + sb.wvu_row * (int64_t)ldw;
  const int* dx = dexp + sb.wvu_row;
  const int64_t gt0 = sb.wvu_row / 64;
  for (int e = tid; e < ntb * 64; e += 256) wv[e] = ldexp(Wb[(int64_t)e * ldw], dx[e]);
  __syncthreads();
  const double wr = wv[I * 64 + warp * 8 + rr];   // this lane's row of w_I (column part)
  double racc = 0.0;
  for (int J = 0; J <= I; ++J) {
    const int8_t* T = msl + (sb.dense_off + (int64_t)I * (I + 1) / 2 + J) * OZ_MT + (warp * 4 + h) * 128 + rr * 16;
    uint4 q[OZ_NS];
#pragma unroll
    for (int i = 0; i < OZ_NS; ++i) q[i] = __ldg(reinterpret_cast<const uint4*>(T + i * 4096));
    const double* v = wv + J * 64 + 16 * h;
    double cval[16];
#pragma unroll
    for (int b = 0; b < 16; ++b) {
      const int w32 = b >> 2, sh = 8 * (b & 3);
      auto dig = [&](int i) {
        const uint32_t word = w32 == 0 ? q[i].x : w32 == 1 ? q[i].y : w32 == 2 ? q[i].z : q[i].w;
        return (int)(int8_t)(word >> sh);
      };
      const int hi = (dig(0) << 16) + (dig(1) << 8) + dig(2);
      const long long lo = ((long long)dig(3) << 24) + (dig(4) << 16) + (dig(5) << 8) + dig(6);
      const double x = fma((double)hi, 0x1p32, (double)lo);
      racc = fma(x, v[b], racc);
      cval[b] = x * wr;
    }
    if (J < I) {   // column part: sum over the tile's 64 rows (8 in this warp, then the 8 warps), fixed order
#pragma unroll
      for (int b = 0; b < 16; ++b) {
        double t = cval[b];
        t += __shfl_xor_sync(0xffffffffu, t, 4);
        t += __shfl_xor_sync(0xffffffffu, t, 8);
        t += __shfl_xor_sync(0xffffffffu, t, 16);
        cval[b] = t;
      }
      if (rr == 0) {
#pragma unroll
        for (int b = 0; b < 16; ++b) cpart[warp][16 * h + b] = cval[b];
      }
      __syncthreads();
      if (tid < 64) {
        double sum = 0.0;
#pragma unroll
        for (int w = 0; w < 8; ++w) sum += cpart[w][tid];
        P[((gt0 + J) * max_ntb + I) * 64 + tid] = sum;
      }
      __syncthreads();
    }
  }
  racc += __shfl_xor_sync(0xffffffffu, racc, 1);
  racc += __shfl_xor_sync(0xffffffffu, racc, 2);
  if (h == 0) P[((gt0 + I) * max_ntb + I) * 64 + warp * 8 + rr] = racc;
}

__global__ void k_oz_symv_reduce(const FacSub* __restrict__ subs, const int2* __restrict__ items, int max_ntb,
                                 const double* __restrict__ P, const int* __restrict__ dexp,
                                 const int* __restrict__ mexp, double* __restrict__ U, int ldw) {
  pdl_wait();
  const int2 it = items[blockIdx.x];
  const FacSub sb = subs[it.x];
  const int J = it.y, ntb = sb.ntb;
  const int64_t gt = sb.wvu_row / 64 + J;
  const double* p = P + gt * max_ntb * 64 + threadIdx.x;
  double sum = 0.0;
  for (int I = J; I < ntb; ++I) sum += p[I * 64];
  const int64_t row = sb.wvu_row + (int64_t)J * 64 + threadIdx.x;
  U[row * ldw] = ldexp(sum, dexp[row] + mexp[it.x] - 55);
}
}  // namespace

namespace nspk {

size_t oz_mslice_bytes(int64_t dense_tiles) { return (size_t)dense_tiles * OZ_MT; }
size_t oz_wslice_bytes(int64_t wvu_rows, int s) {
  const int nct = (s + 127) / 128;
  return (size_t)(wvu_rows / 64) * nct * OZ_AT;
}

// setup: dexp (wvu_rows ints), mexp (nsub ints), msl (oz_mslice_bytes) from the S_j^{-1} tiles
void oz_setup(const FacSub* subs, int nsub, int max_ntb, const int2* items, int nitems, const double* minv,
              int* dexp, int* mexp, int8_t* msl, int8_t* mz, cudaStream_t st) {
  if (nsub <= 0 || nitems <= 0) return;
  nsp_count_launch();
  k_oz_dexp<<<dim3(nsub, max_ntb), 64, 0, st>>>(subs, minv, dexp);
  cudaMemsetAsync(mexp, 0x80, (size_t)nsub * sizeof(int), st);   // INT_MIN-ish
  nsp_count_launch();
  k_oz_mexp<<<nitems, 256, 0, st>>>(subs, items, minv, dexp, mexp);
  nsp_count_launch();
  k_oz_slice_m<<<nitems, 256, 0, st>>>(subs, items, minv, dexp, mexp, msl, mz);
}

void oz_symv1(const FacSub* subs, const int2* items, int nitems, int max_ntb, const int8_t* msl, const int* dexp,
              const int* mexp, const double* W, int ldw, double* U, double* P, cudaStream_t st) {
  if (nitems <= 0) return;
  const size_t smem = (size_t)max_ntb * 64 * sizeof(double);
  if (smem > 48 * 1024) smem_optin((const void*)k_oz_symv1, smem);
  nsp_count_launch();
  launch_k(k_oz_symv1, dim3(nitems), dim3(256), smem, st, subs, items, msl, dexp, W, ldw, max_ntb, P);
  nsp_count_launch();
  launch_k(k_oz_symv_reduce, dim3(nitems), dim3(64), 0, st, subs, items, max_ntb, (const double*)P, dexp, mexp, U, ldw);
}

void oz_slice_w(const FacSub* subs, const int2* items, int nitems, int nsub, int s, int nch, const double* W,
                int64_t cs, const int* dexp, int8_t* wsl, int* sexp, cudaStream_t st, bool have_exp) {
  if (nitems <= 0) return;
  const int nct = (s + 127) / 128;
  if (!have_exp) {   // the column exponents were not folded into a1 (spmm_cs_oz): a pass of their own
    cudaMemsetAsync(sexp, 0x80, (size_t)nsub * nct * 128 * sizeof(int), st);
    nsp_count_launch();
    launch_k(k_oz_wmax, dim3(nitems, nct * 4), dim3(256), 0, st, subs, items, W, cs, nch, nct, dexp, sexp);
  }
  nsp_count_launch();
  launch_k(k_oz_slice_w, dim3(nitems, nct * 4), dim3(128), 0, st, subs, items, W, cs, nch, nct, dexp,
           (const int*)sexp, wsl);
}

void oz_product(const FacSub* subs, const int2* items, int nitems, int s, int nch, double* U, int64_t cs,
                const int* dexp, const int* mexp, const int8_t* msl, const int8_t* wsl, const int* sexp,
                cudaStream_t st, const int2* pairs, int npairs, int* uctr, const int8_t* mz) {
  if (nitems <= 0) return;
  const int nct = (s + 127) / 128;
  // diagnostics: bits 1 / 2 skip the A / B loads, 4 drops the L2 evict-last hint, 8 the symmetric K order
  static const int dbg = getenv("NSP_OZ_DBG") ? atoi(getenv("NSP_OZ_DBG")) : 0;
  // clusters of two CTAs sharing the W^T slices by multicast: parity-clean but measured no faster (cfg5 apply
  // 33.9 vs 33.4 ms: the L2 -> SM traffic does not bind; the shared-memory port does), opt-in NSP_OZ_CLUSTER=1
  static const bool cl_on = getenv("NSP_OZ_CLUSTER") && getenv("NSP_OZ_CLUSTER")[0] == '1';
  if (pairs && npairs > 0 && cl_on) {
    smem_optin((const void*)k_oz_symm<2>, OZ_SMEM);
    const int units = npairs * nct;
    int grid = 2 * (units < num_sms() / 2 ? units : num_sms() / 2);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(320);
    cfg.dynamicSmemBytes = OZ_SMEM;
    cfg.stream = st;
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 2;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[1].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
    cfg.attrs = at;
    cfg.numAttrs = 2;
    nsp_count_launch();
    cudaLaunchKernelEx(&cfg, k_oz_symm<2>, subs, pairs, npairs, nct, msl, wsl, dexp, mexp, sexp, U, cs, nch, dbg,
                       (int*)nullptr, (dbg & 48) ? (const int8_t*)nullptr : mz);
    return;
  }
  // NSP_OZ_KERNEL=2: the register-staged variant k_oz_symm_rs - parity-clean, measured SLOWER (cfg5 apply
  // 39.0 vs 33.5 ms: the stagers' W^T loads sit on the critical path of every K-step), opt-in only
  static const int kv = getenv("NSP_OZ_KERNEL") ? atoi(getenv("NSP_OZ_KERNEL")) : 1;
  const int units = nitems * nct;
  if (kv == 3) {
    static const bool stat3 = getenv("NSP_OZ_STATIC") && getenv("NSP_OZ_STATIC")[0] == '1';
    if (uctr && !stat3) cudaMemsetAsync(uctr, 0, sizeof(int), st);
    smem_optin((const void*)k_oz_symm_rs2, RS_SMEM);
    const int grid = units < num_sms() ? units : num_sms();
    nsp_count_launch();
    launch_k(k_oz_symm_rs2, dim3(grid), dim3(448), (size_t)RS_SMEM, st, subs, items, nitems, nct, msl, wsl, dexp,
             mexp, sexp, U, cs, nch, stat3 ? (int*)nullptr : uctr);
    return;
  }
  if (kv == 2 && !(dbg & 3)) {
    smem_optin((const void*)k_oz_symm_rs, RS_SMEM);
    const int grid = units < num_sms() ? units : num_sms();
    nsp_count_launch();
    launch_k(k_oz_symm_rs, dim3(grid), dim3(320), (size_t)RS_SMEM, st, subs, items, nitems, nct, msl, wsl, dexp,
             mexp, sexp, U, cs, nch);
    return;
  }
  smem_optin((const void*)k_oz_symm<1>, OZ_SMEM);
  const int grid = units < num_sms() ? units : num_sms();
  nsp_count_launch();
  static const bool stat = getenv("NSP_OZ_STATIC") && getenv("NSP_OZ_STATIC")[0] == '1';
  if (uctr && !stat) cudaMemsetAsync(uctr, 0, sizeof(int), st);
#ifdef NSP_OZ_PROF
  if (uctr) cudaMemsetAsync(uctr + 64, 0, 64, st);
#endif
  launch_k(k_oz_symm<1>, dim3(grid), dim3(320), (size_t)OZ_SMEM, st, subs, items, nitems, nct, msl, wsl, dexp, mexp,
           sexp, U, cs, nch, dbg, stat ? (int*)nullptr : uctr, (dbg & 48) ? (const int8_t*)nullptr : mz);
#ifdef NSP_OZ_PROF
  if (uctr) {
    unsigned long long h[3];
    cudaMemcpyAsync(h, uctr + 64, 24, cudaMemcpyDeviceToHost, st);
    cudaStreamSynchronize(st);
    fprintf(stderr, "[oz prof] MMA warp per CTA: tempty wait %.3f, full wait %.3f, total %.3f Mcycles (grid %d)\n",
            h[0] / 1e6 / grid, h[1] / 1e6 / grid, h[2] / 1e6 / grid, grid);
  }
#endif
}

}  // namespace nspk
