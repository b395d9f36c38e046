// Tall-skinny and small dense fp64 kernels of the block-CG / Nystrom steps (§8(a) rows a6-a11,
// d1): Gram contractions and panel updates on the DMMA pipe (north_star (c)), one-CTA s x s
// Cholesky / triangular inverse / Jacobi eigensolver, small GEMMs.  All reductions are
// fixed-order two-stage (no fp64 atomics): results are bitwise reproducible (reading C17).
#include <algorithm>
#include <cstdio>
#include <cooperative_groups.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "nsp_blas.h"
#include "../../include/nsp.h"
#include "nsp_dmma.cuh"

using namespace nspd;

#ifndef NSP_GR
#define NSP_GR 32
#endif
#ifndef NSP_GNS
#define NSP_GNS 3
#endif
#ifndef NSP_GCTAS_PER_SM
#define NSP_GCTAS_PER_SM 2
#endif
namespace {

__device__ __forceinline__ void cp_async16_zf(void* smem, const void* gmem, bool valid) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  int sz = valid ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(sz));
}

// rows x cols block (cols even) from row-major global (ld gld) into smem (ld sld), rows >= nvalid
// zero-filled.
__device__ __forceinline__ void cp_block_zf(double* s, int sld, const double* g, int64_t gld, int rows, int cols,
                                            int64_t nvalid) {
  const int cpr = cols / 2;
  const int total = rows * cpr;
  for (int c = threadIdx.x; c < total; c += blockDim.x) {
    const int r = c / cpr, q = c - r * cpr;
    const bool v = r < nvalid;
    cp_async16_zf(s + r * sld + 2 * q, v ? (const void*)(g + r * gld + 2 * q) : (const void*)g, v);
  }
}

constexpr int GR = NSP_GR;     // rows per Gram slab
constexpr int LDS = 68;    // smem stride for 64-wide tiles

// part[(chunk * ntm * ntn + tm * ntn + tn) * 4096 + i * 64 + j]
//   = sum_{r in chunk} Xa[r][64 tm + i] * Xb[r][64 tn + j]
// One wave of CTAs (tiles x chunks <= 2 x SMs, two per SM), each streaming its contiguous row chunk
// through a GNS-stage cp.async ring of 32-row slabs (one barrier per slab), so the slab loads are
// in flight GNS-1 slabs ahead of the DMMA work.
constexpr int GNS = NSP_GNS;
// CL > 1: the grid's chunk dimension is split into clusters of CL CTAs (one thread-block cluster each);
// after its slab loop every CTA parks its 64 x 64 partial in shared memory and the cluster sums the CL
// partials through distributed shared memory (each CTA a 64/CL-row slice, ranks in order), so the
// partial buffer - and the k_gram_reduce that follows - holds CL x fewer chunks.
template <int CL>
__global__ void __launch_bounds__(256) k_gram_partial(const double* __restrict__ Xa, int lda,
                                                      const double* __restrict__ Xb, const double* __restrict__ Xb2,
                                                      int ldb, int ntn1, int64_t n,
                                                      int64_t rows_per_chunk, double* __restrict__ part, int ntm,
                                                      int ntn, int sym) {
  pdl_wait();
  extern __shared__ double sm[];
  constexpr int STG = 2 * GR * LDS;
  const int tile = blockIdx.x;
  int tm = tile / ntn, tn = tile - tm * ntn;
  if (sym == 1) {   // Xa == Xb: only the tiles tm <= tn, enumerated row by row
    tm = 0;
    int rem = tile;
    while (rem >= ntn - tm) {
      rem -= ntn - tm;
      ++tm;
    }
    tn = tm + rem;
  } else if (sym == 2) {   // [D | E]: the lower tiles tn <= tm of D (its only consumer is chol), then all of E
    const int nlo = ntm * (ntm + 1) / 2;
    if (tile < nlo) {
      tm = 0;
      while ((tm + 1) * (tm + 2) / 2 <= tile) ++tm;
      tn = tile - tm * (tm + 1) / 2;
    } else {
      const int u = tile - nlo;
      tm = u / ntn1;
      tn = ntn1 + (u - tm * ntn1);
    }
  }
  const int64_t r0 = blockIdx.y * rows_per_chunk;
  const int64_t r1 = min(n, r0 + rows_per_chunk);
  double acc[2][4][2];
  acc_zero(acc);
  const double* A0 = Xa + 64 * tm;
  const double* B0 = tn < ntn1 ? Xb + 64 * tn : Xb2 + 64 * (tn - ntn1);
  const int nslab = r1 > r0 ? (int)((r1 - r0 + GR - 1) / GR) : 0;
  auto issue = [&](int q) {
    double* st = sm + (q % GNS) * STG;
    const int64_t r = r0 + (int64_t)q * GR;
    cp_block_zf(st, LDS, A0 + r * lda, lda, GR, 64, r1 - r);
    cp_block_zf(st + GR * LDS, LDS, B0 + r * ldb, ldb, GR, 64, r1 - r);
  };
#pragma unroll
  for (int q = 0; q < GNS - 1; ++q) {
    if (q < nslab) issue(q);
    cp_commit();
  }
  for (int q = 0; q < nslab; ++q) {
    cp_wait<GNS - 2>();
    __syncthreads();
    if (q + GNS - 1 < nslab) issue(q + GNS - 1);
    cp_commit();
    const double* st = sm + (q % GNS) * STG;
    cta_mma<4, true, false>(st, LDS, st + GR * LDS, LDS, acc, GR);
  }
  if constexpr (CL == 1) {
    double* out = part + ((int64_t)blockIdx.y * gridDim.x + tile) * 4096;
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int rr = acc_row<4>(i), cc = acc_col<4>(j);
        *reinterpret_cast<double2*>(out + rr * 64 + cc) = make_double2(acc[i][j][0], acc[i][j][1]);
      }
  } else {
    namespace cg = cooperative_groups;
    cg::cluster_group cluster = cg::this_cluster();
    cp_wait<0>();
    __syncthreads();   // the slab ring is free
    double* mine = sm;   // 64 x 64 partial of this CTA
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int rr = acc_row<4>(i), cc = acc_col<4>(j);
        *reinterpret_cast<double2*>(mine + rr * 64 + cc) = make_double2(acc[i][j][0], acc[i][j][1]);
      }
    cluster.sync();
    const int rank = (int)cluster.block_rank();
    constexpr int SL = 4096 / CL;   // this CTA's slice of the tile (64 / CL rows)
    double* out = part + ((int64_t)(blockIdx.y / CL) * gridDim.x + tile) * 4096 + rank * SL;
    for (int e = threadIdx.x; e < SL; e += blockDim.x) {
      double v = 0.0;
#pragma unroll
      for (int q = 0; q < CL; ++q) v += cluster.map_shared_rank(mine, q)[rank * SL + e];
      out[e] = v;
    }
    cluster.sync();   // no CTA leaves while another may still read its shared memory
  }
}

// out (or out2 for column tiles >= ntn1) = sum over chunks, 4 chunk groups per element combined
// in fixed order (deterministic)
// sym: the partials hold only the tiles tm <= tn (Xa == Xb); element (i, j) of a lower tile is read
// transposed from its upper partner, so the output is exactly symmetric
__global__ void k_gram_reduce(const double* __restrict__ part, int nchunks, int ntm, int ntn, int ntn1,
                              double* out, double* out2, int ldo, int sym) {
  pdl_wait();
  __shared__ double red[4][16][17];
  // a 16 x 16 output block below the diagonal (sym) is read transposed from its upper partner with the
  // threads swapped (coalesced reads) and written transposed; diagonal blocks pick (min, max) per element
  const int bi = blockIdx.y * 16, bj = blockIdx.x * 16;
  const bool tr = (sym == 1 && bi > bj) || (sym == 2 && bi < bj && bj < ntn1 * 64);   // mirrored blocks
  const int i = tr ? bi + threadIdx.x : bi + threadIdx.y;
  const int j = tr ? bj + threadIdx.y : bj + threadIdx.x;
  const int g = threadIdx.z;
  double s = 0.0;
  if (i < ntm * 64 && j < ntn * 64) {
    int64_t off;
    int64_t stride;
    if (sym == 1) {
      const int a = min(i, j), b = max(i, j);   // (i, j) and (j, i) read the same partial entry
      const int ta = a >> 6, tb = b >> 6;
      off = (int64_t)(ta * ntn - ta * (ta - 1) / 2 + (tb - ta)) * 4096 + (a & 63) * 64 + (b & 63);
      stride = (int64_t)(ntm * (ntm + 1) / 2) * 4096;
    } else if (sym == 2) {
      const int nlo = ntm * (ntm + 1) / 2;
      if (j < ntn1 * 64) {                        // D: the lower partial, mirrored above the diagonal
        const int a = max(i, j), b = min(i, j);
        const int ta = a >> 6, tb = b >> 6;
        off = (int64_t)(ta * (ta + 1) / 2 + tb) * 4096 + (a & 63) * 64 + (b & 63);
      } else {
        off = (int64_t)(nlo + (i >> 6) * ntn1 + ((j >> 6) - ntn1)) * 4096 + (i & 63) * 64 + (j & 63);
      }
      stride = (int64_t)(nlo + ntm * ntn1) * 4096;
    } else {
      off = (int64_t)((i >> 6) * ntn + (j >> 6)) * 4096 + (i & 63) * 64 + (j & 63);
      stride = (int64_t)ntm * ntn * 4096;
    }
    for (int c = g; c < nchunks; c += 4) s += part[off + c * stride];
  }
  red[g][threadIdx.y][threadIdx.x] = s;
  __syncthreads();
  if (g == 0 && i < ntm * 64 && j < ntn * 64) {
    const double v = red[0][threadIdx.y][threadIdx.x] + red[1][threadIdx.y][threadIdx.x] +
                     red[2][threadIdx.y][threadIdx.x] + red[3][threadIdx.y][threadIdx.x];
    const int j1 = j - ntn1 * 64;
    if (j1 < 0) out[(int64_t)i * ldo + j] = v;
    else out2[(int64_t)i * ldo + j1] = v;
  }
}

// Out[r][c] = (Cin ? Cin[r][c] : 0) + sgn * sum_k In[r][k] M[k][c];   r < n, c in this 64-col tile.
// blockIdx.z selects one of two independent argument sets (X += P alpha and R -= Q alpha in one launch).
// normpart (optional): normpart[rowtile * ldo + c] = sum over the tile's rows of Out[r][c]^2.
__global__ void __launch_bounds__(256) k_panel(PanelArgs pa0, PanelArgs pa1, int kdim, int64_t n) {
  pdl_wait();
  const PanelArgs& pa = blockIdx.z ? pa1 : pa0;
  double* Out = pa.Out;
  const int ldo = pa.ldo, ldc = pa.ldc, ldi = pa.ldi, ldm = pa.ldm;
  const double* Cin = pa.Cin;
  const double* __restrict__ In = pa.In;
  const double* __restrict__ M = pa.M;
  const double sgn = pa.sgn;
  double* normpart = pa.normpart;
  extern __shared__ double sm[];
  constexpr int LDA = 36;
  double* As[2] = {sm, sm + 64 * LDA};
  double* Bs[2] = {sm + 2 * 64 * LDA, sm + 2 * 64 * LDA + 32 * LDS};
  const int64_t r0 = blockIdx.x * 64ll;
  const int c0 = blockIdx.y * 64;
  const int64_t nv = n - r0;
  const bool upper = pa.upper_unless && *pa.upper_unless == 0;
  double acc[2][4][2];
  acc_zero(acc);
  const int nk = (kdim + 31) / 32;
  if (nk > 0) {
    cp_block_zf(As[0], LDA, In + r0 * ldi, ldi, 64, 32, nv);
    cp_block(Bs[0], LDS, M + c0, ldm, 32, 64);
    cp_commit();
  }
  for (int kb = 0; kb < nk; ++kb) {
    const int b = kb & 1;
    cp_wait<0>();
    __syncthreads();
    if (kb + 1 < nk) {
      cp_block_zf(As[b ^ 1], LDA, In + r0 * ldi + (kb + 1) * 32, ldi, 64, 32, nv);
      cp_block(Bs[b ^ 1], LDS, M + (int64_t)(kb + 1) * 32 * ldm + c0, ldm, 32, 64);
      cp_commit();
    }
    // upper-triangular M: a warp's columns c0 + 32 (warp & 1) .. + 31 see zeros for k > their last column
    if (!(upper && kb * 32 > c0 + (int)(threadIdx.x >> 5 & 1) * 32 + 31))
      cta_mma<4, false, false>(As[b], LDA, Bs[b], LDS, acc, 32);
  }
  __syncthreads();   // smem reused below
  double* sq = sm;  // reuse: 64 x 65 squares
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int rr = acc_row<4>(i), cc = acc_col<4>(j);
      const int64_t r = r0 + rr;
      double v0 = 0.0, v1 = 0.0;
      if (r < n) {
        v0 = sgn * acc[i][j][0];
        v1 = sgn * acc[i][j][1];
        if (Cin) {
          const double2 cv = *reinterpret_cast<const double2*>(Cin + r * ldc + c0 + cc);
          v0 += cv.x;
          v1 += cv.y;
        }
        *reinterpret_cast<double2*>(Out + r * ldo + c0 + cc) = make_double2(v0, v1);
      }
      if (normpart) {
        sq[rr * 65 + cc] = v0 * v0;
        sq[rr * 65 + cc + 1] = v1 * v1;
      }
    }
  if (normpart) {
    __syncthreads();
    if (threadIdx.x < 64) {
      double s = 0.0;
      for (int rr = 0; rr < 64; ++rr) s += sq[rr * 65 + threadIdx.x];
      normpart[blockIdx.x * (int64_t)ldo + c0 + threadIdx.x] = s;
    }
  }
}

// The same panel for the 128-column case (s x s multiplier M with s = 128) as ONE wave: one CTA per
// SM, each owning a contiguous range of 16-row groups (balanced to +-1 group, where 64-row tiles
// quantise to 2 tiles on some SMs and 1 on others), M resident in shared memory (read once per CTA),
// In streamed through a PNS-stage ring of 64 x PKC chunks (64 x 64, 2 stages: half the barriers of
// 64 x 32 x 4 stages, panel 30.5 -> 29.9 us, cfg2 25.85 -> 25.58 ms), 16 warps = 4 row groups x 4 column quarters
// of a 64 x 128 pass; Cin prefetched into registers at the start of each pass.  normpart (optional):
// one row per CTA, the column sums of squares over its rows (fixed order).
#ifndef NSP_PANEL_NW
#define NSP_PANEL_NW 16
#endif
#ifndef NSP_PNS
#define NSP_PNS 2
#endif
#ifndef NSP_PKC
#define NSP_PKC 64
#endif
constexpr int PKC = NSP_PKC, PSPP = 128 / PKC;   // chunk width, chunks per 64-row pass
constexpr int PLDM = 132, PLDA = PKC + 4, PNS = NSP_PNS;
template <int NW>
__global__ void __launch_bounds__(NW * 32, 1) k_panel_rows(PanelArgs pa, int64_t n, int64_t ngroups) {
  // NW = 16: warps = 4 row groups x 4 column quarters (16 x 32 per warp); NW = 8: 4 row groups x 2
  // column halves (16 x 64 per warp: twice the products per loaded A fragment)
  constexpr int NF = NW == 16 ? 4 : 8;
  pdl_wait();
  extern __shared__ __align__(16) double sm[];
  double* Ms = sm;                  // 128 x PLDM
  double* Ar = sm + 128 * PLDM;     // PNS x 64 x PLDA
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int rg = NW == 16 ? warp >> 2 : warp >> 1;
  const int cb = NW == 16 ? (warp & 3) * 32 : (warp & 1) * 64;
  const int64_t g0 = (int64_t)blockIdx.x * ngroups / gridDim.x;
  const int64_t g1 = (int64_t)(blockIdx.x + 1) * ngroups / gridDim.x;
  const int64_t r0 = g0 * 16, r1 = min(n, g1 * 16);
  const int npass = r1 > r0 ? (int)((r1 - r0 + 63) / 64) : 0;
  const int nsteps = npass * PSPP;
  const double* __restrict__ In = pa.In;
  const bool upper = pa.upper_unless && *pa.upper_unless == 0;
  auto issue = [&](int q) {
    const int64_t rp = r0 + (int64_t)(q / PSPP) * 64;
    cp_block_zf(Ar + (q % PNS) * 64 * PLDA, PLDA, In + rp * pa.ldi + (q % PSPP) * PKC, pa.ldi, 64, PKC, r1 - rp);
  };
  // M rows [0, PKC) travel with the first chunk; the rest in a group of their own, waited for one step
  // later (PNS == 2: the first product does not wait for the whole 128 KB multiplier)
  static_assert(PNS == 2, "prologue assumes a 2-stage ring");
  cp_block(Ms, PLDM, pa.M, pa.ldm, PKC, 128);
  if (nsteps > 0) issue(0);
  cp_commit();
  cp_block(Ms + PKC * PLDM, PLDM, pa.M + (int64_t)PKC * pa.ldm, pa.ldm, 128 - PKC, 128);
  cp_commit();
  double acc[2][NF][2];
  acc_zero(acc);
  double sq[NF][2];
#pragma unroll
  for (int j = 0; j < NF; ++j) sq[j][0] = sq[j][1] = 0.0;
  double2 cin[2][NF];
  for (int q = 0; q < nsteps; ++q) {
    const int kc = q % PSPP;
    const int64_t rp = r0 + (int64_t)(q / PSPP) * 64;
    if (kc == 0) {   // this pass's Cin, in flight behind the pass's four chunk products
#pragma unroll
      for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int j = 0; j < NF; ++j) {
          const int64_t r = rp + rg * 16 + acc_row<NF>(i, 0);
          const int c = cb + acc_col<NF>(j, 0);
          cin[i][j] = (pa.Cin && r < r1) ? *reinterpret_cast<const double2*>(pa.Cin + r * pa.ldc + c)
                                         : make_double2(0.0, 0.0);
        }
    }
    if (q == 0) cp_wait<1>();   // chunk 0 and M's first rows (the rest of M may still be in flight)
    else cp_wait<0>();
    __syncthreads();
    if (q + PNS - 1 < nsteps) issue(q + PNS - 1);
    cp_commit();
    const double* As = Ar + (q % PNS) * 64 * PLDA;
    // a warp whose 16-row group lies past the range skips its products (the DMMA pipe is the limit), and so
    // does a warp whose columns see an all-zero chunk of an upper-triangular M
    if (rp + rg * 16 < r1 && !(upper && kc * PKC > cb + NF * 8 - 1))
      cta_mma<NF, false, false>(As + rg * 16 * PLDA, PLDA, Ms + kc * PKC * PLDM + cb, PLDM, acc, PKC, 0);
    if (kc == PSPP - 1) {
#pragma unroll
      for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int j = 0; j < NF; ++j) {
          const int64_t r = rp + rg * 16 + acc_row<NF>(i, 0);
          const int c = cb + acc_col<NF>(j, 0);
          if (r < r1) {
            const double v0 = pa.sgn * acc[i][j][0] + cin[i][j].x;
            const double v1 = pa.sgn * acc[i][j][1] + cin[i][j].y;
            *reinterpret_cast<double2*>(pa.Out + r * pa.ldo + c) = make_double2(v0, v1);
            sq[j][0] += v0 * v0;
            sq[j][1] += v1 * v1;
          }
        }
      acc_zero(acc);
    }
  }
  if (!pa.normpart) return;
  // column sums of squares: butterfly over the 8 row lanes, then the 4 row-group warps in order
#pragma unroll
  for (int j = 0; j < NF; ++j)
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      double v = sq[j][e];
      v += __shfl_xor_sync(0xffffffffu, v, 4);
      v += __shfl_xor_sync(0xffffffffu, v, 8);
      v += __shfl_xor_sync(0xffffffffu, v, 16);
      sq[j][e] = v;
    }
  cp_wait<0>();
  __syncthreads();   // the ring is free
  double* red = Ar;  // 4 x 128
  if (lane < 4) {
#pragma unroll
    for (int j = 0; j < NF; ++j) {
      const int c = cb + acc_col<NF>(j, 0);
      red[rg * 128 + c] = sq[j][0];
      red[rg * 128 + c + 1] = sq[j][1];
    }
  }
  __syncthreads();
  if (threadIdx.x < 128)
    pa.normpart[blockIdx.x * (int64_t)pa.ldo + threadIdx.x] =
        ((red[threadIdx.x] + red[128 + threadIdx.x]) + red[256 + threadIdx.x]) + red[384 + threadIdx.x];
}

// The s = 128 panel with TWO CTAs per SM: CTA 2g + h owns the rows of group g (one contiguous range of
// 16-row groups per pair, as k_panel_rows) and the output columns 64h .. 64h + 63, so its share of the
// multiplier M[:, 64h:64h+64] (68 KB) and a 2-stage ring of 64 x 32 In chunks fit twice per SM.  8 warps
// = 4 row groups x 2 column quarters (16 x 32 per warp); 4 k-chunks per 64-row pass.  While one CTA of an
// SM waits at a barrier or in its epilogue the other's products keep the DMMA pipe busy (k_panel_rows:
// one 16-warp CTA per SM, every warp in lockstep).  normpart as k_panel_rows (row g, 128 columns).
constexpr int HKC = 32, HLDM = 68, HLDA = 36, HSPP = 128 / HKC;
// PR = rows per pass (64: 8 warps = 4 row groups x 2 column quarters of 32; 32: 2 row groups x 4 column
// groups of 16 - finer passes for small n, where a 64-row pass over a 96-row range wastes half a pass)
template <int PR>
__global__ void __launch_bounds__(256, 2) k_panel_half(PanelArgs pa, int64_t n, int64_t ngroups) {
  constexpr int NF = PR == 64 ? 4 : 2;
  constexpr int NRG = PR / 16;              // row groups per pass
  constexpr int CW = 64 / (8 / NRG);        // columns per warp: 32 (PR 64) or 16 (PR 32)
  pdl_wait();
  extern __shared__ __align__(16) double sm[];
  double* Ms = sm;                  // 128 x HLDM: M[:, c0 .. c0 + 64)
  double* Ar = sm + 128 * HLDM;     // 2 x PR x HLDA
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int rg = warp / (8 / NRG), cb = (warp % (8 / NRG)) * CW;
  const int grp = blockIdx.x >> 1, c0 = (blockIdx.x & 1) * 64;
  const int ngrp = gridDim.x >> 1;
  const int64_t g0 = (int64_t)grp * ngroups / ngrp;
  const int64_t g1 = (int64_t)(grp + 1) * ngroups / ngrp;
  const int64_t r0 = g0 * 16, r1 = min(n, g1 * 16);
  const int npass = r1 > r0 ? (int)((r1 - r0 + PR - 1) / PR) : 0;
  const int nsteps = npass * HSPP;
  const double* __restrict__ In = pa.In;
  auto issue = [&](int q) {
    const int64_t rp = r0 + (int64_t)(q / HSPP) * PR;
    cp_block_zf(Ar + (q & 1) * PR * HLDA, HLDA, In + rp * pa.ldi + (q % HSPP) * HKC, pa.ldi, PR, HKC, r1 - rp);
  };
  cp_block(Ms, HLDM, pa.M + c0, pa.ldm, 128, 64);
  if (nsteps > 0) issue(0);
  cp_commit();
  double acc[2][NF][2];
  acc_zero(acc);
  double sq[NF][2];
#pragma unroll
  for (int j = 0; j < NF; ++j) sq[j][0] = sq[j][1] = 0.0;
  double2 cin[2][NF];
  for (int q = 0; q < nsteps; ++q) {
    const int kc = q % HSPP;
    const int64_t rp = r0 + (int64_t)(q / HSPP) * PR;
    if (kc == 0) {
#pragma unroll
      for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int j = 0; j < NF; ++j) {
          const int64_t r = rp + rg * 16 + acc_row<NF>(i, 0);
          const int c = c0 + cb + acc_col<NF>(j, 0);
          cin[i][j] = (pa.Cin && r < r1) ? *reinterpret_cast<const double2*>(pa.Cin + r * pa.ldc + c)
                                         : make_double2(0.0, 0.0);
        }
    }
    cp_wait<0>();
    __syncthreads();
    if (q + 1 < nsteps) issue(q + 1);
    cp_commit();
    const double* As = Ar + (q & 1) * PR * HLDA;
    if (rp + rg * 16 < r1)
      cta_mma<NF, false, false>(As + rg * 16 * HLDA, HLDA, Ms + kc * HKC * HLDM + cb, HLDM, acc, HKC, 0);
    if (kc == HSPP - 1) {
#pragma unroll
      for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int j = 0; j < NF; ++j) {
          const int64_t r = rp + rg * 16 + acc_row<NF>(i, 0);
          const int c = c0 + cb + acc_col<NF>(j, 0);
          if (r < r1) {
            const double v0 = pa.sgn * acc[i][j][0] + cin[i][j].x;
            const double v1 = pa.sgn * acc[i][j][1] + cin[i][j].y;
            *reinterpret_cast<double2*>(pa.Out + r * pa.ldo + c) = make_double2(v0, v1);
            sq[j][0] += v0 * v0;
            sq[j][1] += v1 * v1;
          }
        }
      acc_zero(acc);
    }
  }
  if (!pa.normpart) return;
#pragma unroll
  for (int j = 0; j < NF; ++j)
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      double v = sq[j][e];
      v += __shfl_xor_sync(0xffffffffu, v, 4);
      v += __shfl_xor_sync(0xffffffffu, v, 8);
      v += __shfl_xor_sync(0xffffffffu, v, 16);
      sq[j][e] = v;
    }
  cp_wait<0>();
  __syncthreads();
  double* red = Ar;   // NRG x 64
  if (lane < 4) {
#pragma unroll
    for (int j = 0; j < NF; ++j) {
      const int c = cb + acc_col<NF>(j, 0);
      red[rg * 64 + c] = sq[j][0];
      red[rg * 64 + c + 1] = sq[j][1];
    }
  }
  __syncthreads();
  if (threadIdx.x < 64) {
    double v = red[threadIdx.x];
#pragma unroll
    for (int q = 1; q < NRG; ++q) v += red[q * 64 + threadIdx.x];
    pa.normpart[grp * (int64_t)pa.ldo + c0 + threadIdx.x] = v;
  }
}

// Fused s = 128 panel + Gram partial (rows a8+a10 / a10+a11 of the block-CG iteration, one pass over
// the tall blocks instead of two):
//   Out = Cin + sgn In M   (the panel of k_panel_rows)   and   G_cta = Aop^T Out over the CTA's rows,
// Aop = In (GMODE 0: R -= Q alpha with F = Q^T R_new, M = I) or Out (GMODE 1: W = R + P beta with W^T W,
// only the tiles on / above the diagonal).  One CTA per SM (16 warps) owning a contiguous range of 16-row
// groups, M resident in shared memory, 32-row passes: the pass's In tile is staged in shared memory
// from registers that were loaded during the previous pass (the global loads of pass p+1 are in flight
// while pass p computes), the panel product runs as 2 x 8 warps of 16 x 16 outputs, the Out tile goes
// to global memory AND to shared memory, and the Gram accumulates 32 x 32 blocks per warp in registers
// across all passes.  Each CTA writes its Gram partial in k_gram_reduce's tile layout (full 2 x 2 tiles,
// or the 3 upper tiles) and, optionally, the column sums of squares of Out (the convergence norms) in
// k_panel_rows' normpart layout: fixed-order sums throughout (reading C17).
constexpr int FG_LD = 132;
template <int GMODE>
__global__ void __launch_bounds__(512, 1) k_panel_gram(PanelArgs pa, int64_t n, int64_t ngroups,
                                                      double* __restrict__ gpart) {
  pdl_wait();
  extern __shared__ __align__(16) double sm[];
  double* Ms = sm;                       // 128 x FG_LD
  double* Is = Ms + 128 * FG_LD;         // 32 x FG_LD: In rows of the pass
  double* Os = Is + 32 * FG_LD;          // 32 x FG_LD: Out rows of the pass
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, t = lane & 3;
  const int64_t g0 = (int64_t)blockIdx.x * ngroups / gridDim.x;
  const int64_t g1 = (int64_t)(blockIdx.x + 1) * ngroups / gridDim.x;
  const int64_t r0 = g0 * 16, r1 = min(n, g1 * 16);
  const int npass = r1 > r0 ? (int)((r1 - r0 + 31) / 32) : 0;
  const double* __restrict__ In = pa.In;
  // M by cp.async (waited for before the first product)
  cp_block(Ms, FG_LD, pa.M, pa.ldm, 128, 128);
  cp_commit();
  // In prefetch: 32 x 128 doubles per pass = 4 double2 per thread (coalesced rows)
  double2 pre[4];
  auto load_in = [&](int p) {
    const int64_t rb = r0 + (int64_t)p * 32;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int e = 2 * tid + 1024 * k, rr = e >> 7, cc = e & 127;
      const int64_t r = rb + rr;
      pre[k] = (p < npass && r < r1) ? *reinterpret_cast<const double2*>(In + r * pa.ldi + cc) : make_double2(0.0, 0.0);
    }
  };
  load_in(0);
  // panel warp layout: rows 16 * rg .. +16, cols 16 * cg .. +16
  const int rg = warp >> 3, cg = warp & 7;
  // Gram warp layout: 32 x 32 block (bi, bj) of the 128 x 128 output
  const int bi = warp >> 2, bj = warp & 3;
  const bool gact = GMODE == 0 || bi <= bj;   // symmetric: the blocks on / above the diagonal
  double gacc[4][4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) gacc[i][j][0] = gacc[i][j][1] = 0.0;
  double sq[2][2];
  sq[0][0] = sq[0][1] = sq[1][0] = sq[1][1] = 0.0;
  cp_wait<0>();
  for (int p = 0; p < npass; ++p) {
    const int64_t rb = r0 + (int64_t)p * 32;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int e = 2 * tid + 1024 * k, rr = e >> 7, cc = e & 127;
      *reinterpret_cast<double2*>(Is + rr * FG_LD + cc) = pre[k];
    }
    // this pass's Cin rows into Os by cp.async (Os is free until the epilogue), in flight behind the product
    if (pa.Cin) cp_block_zf(Os, FG_LD, pa.Cin + rb * pa.ldc, pa.ldc, 32, 128, r1 - rb);
    cp_commit();
    load_in(p + 1);   // next pass's In (zeros past the range)
    __syncthreads();  // Is complete (and M on the first pass)
    double acc[2][2][2];
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
      for (int j = 0; j < 2; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
#pragma unroll 4
    for (int k = 0; k < 128; k += 4) {
      double a[2], b[2];
#pragma unroll
      for (int i = 0; i < 2; ++i) a[i] = Is[(rg * 16 + i * 8 + g) * FG_LD + k + t];
#pragma unroll
      for (int j = 0; j < 2; ++j) b[j] = Ms[(k + t) * FG_LD + cg * 16 + j * 8 + g];
#pragma unroll
      for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int j = 0; j < 2; ++j) dmma(acc[i][j][0], acc[i][j][1], a[i], b[j]);
    }
    cp_wait<0>();
    __syncthreads();  // Cin rows in Os visible to every thread
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const int rr = rg * 16 + i * 8 + g;
        const int64_t r = rb + rr;
        const int c = cg * 16 + j * 8 + 2 * t;
        double v0 = 0.0, v1 = 0.0;
        if (r < r1) {
          const double2 cv = pa.Cin ? *reinterpret_cast<const double2*>(Os + rr * FG_LD + c) : make_double2(0.0, 0.0);
          v0 = pa.sgn * acc[i][j][0] + cv.x;
          v1 = pa.sgn * acc[i][j][1] + cv.y;
          *reinterpret_cast<double2*>(pa.Out + r * pa.ldo + c) = make_double2(v0, v1);
          sq[j][0] += v0 * v0;
          sq[j][1] += v1 * v1;
        }
        *reinterpret_cast<double2*>(Os + rr * FG_LD + c) = make_double2(v0, v1);
      }
    __syncthreads();  // Os complete
    if (gact) {
      const double* Aop = GMODE == 0 ? Is : Os;
#pragma unroll
      for (int k = 0; k < 32; k += 4) {
        double a[4], b[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) a[i] = Aop[(k + t) * FG_LD + bi * 32 + i * 8 + g];
#pragma unroll
        for (int j = 0; j < 4; ++j) b[j] = Os[(k + t) * FG_LD + bj * 32 + j * 8 + g];
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) dmma(gacc[i][j][0], gacc[i][j][1], a[i], b[j]);
      }
    }
    __syncthreads();  // Is / Os free for the next pass
  }
  // Gram partial: tile (tm, tn) of 64 x 64 -> k_gram_reduce's layout (GMODE 1: upper tiles 0,1,2 = (0,0),(0,1),(1,1))
  if (gact) {
    const int tm = bi >> 1, tn = bj >> 1;
    const int ntiles = GMODE == 0 ? 4 : 3;
    const int tile = GMODE == 0 ? tm * 2 + tn : (tm == 0 ? tn : 2);
    double* out = gpart + ((int64_t)blockIdx.x * ntiles + tile) * 4096;
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int rr = (bi & 1) * 32 + i * 8 + g, cc = (bj & 1) * 32 + j * 8 + 2 * t;
        *reinterpret_cast<double2*>(out + rr * 64 + cc) = make_double2(gacc[i][j][0], gacc[i][j][1]);
      }
  }
  if (!pa.normpart) return;
  // column sums of squares: the 8 row lanes by butterfly, then the two row-group warps in order
#pragma unroll
  for (int j = 0; j < 2; ++j)
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      double v = sq[j][e];
      v += __shfl_xor_sync(0xffffffffu, v, 4);
      v += __shfl_xor_sync(0xffffffffu, v, 8);
      v += __shfl_xor_sync(0xffffffffu, v, 16);
      sq[j][e] = v;
    }
  double* red = Is;   // 2 x 128
  if (lane < 4) {
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const int c = cg * 16 + j * 8 + 2 * lane;
      red[rg * 128 + c] = sq[j][0];
      red[rg * 128 + c + 1] = sq[j][1];
    }
  }
  __syncthreads();
  if (tid < 128) pa.normpart[blockIdx.x * (int64_t)pa.ldo + tid] = red[tid] + red[128 + tid];
}

// column sums of squares of X (n x s), partial per 64-row tile (fixed order)
__global__ void k_colsq_partial(const double* __restrict__ X, int ldx, int64_t n, int s, double* part, int ldp) {
  pdl_wait();
  const int c = threadIdx.x;
  const int64_t r0 = blockIdx.x * 64ll;
  if (c >= ldp) return;
  double acc = 0.0;
  if (c < s)
    for (int r = 0; r < 64 && r0 + r < n; ++r) {
      const double v = X[(r0 + r) * ldx + c];
      acc += v * v;
    }
  part[blockIdx.x * (int64_t)ldp + c] = acc;
}

// sum over row tiles -> out[c]; thread (c, g) sums tiles t = g mod 8 in order, then the 8
// group sums are added in fixed order (deterministic)
__global__ void k_colsq_reduce(const double* __restrict__ part, int ntiles, int ldp, double* out) {
  pdl_wait();
  __shared__ double red[8][128];
  const int c = threadIdx.x, g = threadIdx.y;
  double s = 0.0;
  if (c < ldp)
    for (int t = g; t < ntiles; t += 8) s += part[t * (int64_t)ldp + c];
  red[g][c] = s;
  __syncthreads();
  if (g == 0 && c < ldp) {
    double v = 0.0;
    for (int q = 0; q < 8; ++q) v += red[q][c];
    out[c] = v;
  }
}

// convergence: relres_j = sqrt(rsq_j) / bnorm_j; max over j < s (columns with bnorm 0 count as 0)
__global__ void k_converge(const double* rsq, const double* bnorm, int s, double tol, BcgStatus* st,
                           double* hist_slot) {
  pdl_wait();
  __shared__ double red[256];
  double m = 0.0;
  bool bad = false;
  for (int c = threadIdx.x; c < s; c += blockDim.x) {
    const double r = sqrt(rsq[c]);
    if (!isfinite(r)) bad = true;
    const double v = bnorm[c] > 0.0 ? r / bnorm[c] : 0.0;
    m = fmax(m, v);
  }
  red[threadIdx.x] = m;
  if (bad) st->nonfinite = 1;
  __syncthreads();
  for (int w = 128; w > 0; w >>= 1) {
    if (threadIdx.x < w) red[threadIdx.x] = fmax(red[threadIdx.x], red[threadIdx.x + w]);
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    st->relres = red[0];
    st->converged = red[0] <= tol ? 1 : 0;
    if (hist_slot) *hist_slot = red[0];
  }
}

// k_colsq_reduce + k_converge in one launch (single rank: the column norms need no allreduce)
__global__ void k_colsq_converge(const double* __restrict__ part, int ntiles, int ldp, double* rsq,
                                 const double* __restrict__ bnorm, int s, double tol, BcgStatus* st) {
  pdl_wait();
  __shared__ double red[8][128];
  __shared__ double mx[128];
  const int c = threadIdx.x, g = threadIdx.y;
  double sum = 0.0;
  if (c < ldp)
    for (int t = g; t < ntiles; t += 8) sum += part[t * (int64_t)ldp + c];
  red[g][c] = sum;
  __syncthreads();
  if (g == 0) {
    double v = 0.0, m = 0.0;
    bool bad = false;
    if (c < ldp) {
      for (int q = 0; q < 8; ++q) v += red[q][c];
      rsq[c] = v;
      if (c < s) {
        const double r = sqrt(v);
        if (!isfinite(r)) bad = true;
        m = bnorm[c] > 0.0 ? r / bnorm[c] : 0.0;
      }
    }
    if (bad) st->nonfinite = 1;
    mx[c] = m;
  }
  __syncthreads();
  if (g == 0 && c < 32) {
    double m = fmax(fmax(mx[c], mx[c + 32]), fmax(mx[c + 64], mx[c + 96]));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
    if (c == 0) {
      st->relres = m;
      st->converged = m <= tol ? 1 : 0;
    }
  }
}

__global__ void k_sqrt_vec(const double* in, double* out, int n) {
  pdl_wait();
  const int i = threadIdx.x + blockIdx.x * blockDim.x;
  if (i < n) out[i] = sqrt(in[i]);
}

// ---------------------------------------------------------------------------------------------
// one-CTA (8 warps) blocked Cholesky of an sp x sp SPD matrix (sp <= 128, multiple of 8) and of
// the inverse of its factor, latency-oriented: 8x8 diagonal blocks are factored (and inverted)
// by one thread entirely in registers (rsqrt.approx + 2 Newton steps, no divisions); the 8-column
// panel is solved row-parallel; the rank-8 trailing update runs on the DMMA pipe (m8n8k4 tiles);
// X = L^{-1} is formed block row by block row on the DMMA pipe.  3 barriers per 8 columns.
// Rows / cols >= nact (nact < 0: st->width) are replaced by the identity.
//  mode 0 (D = P^T S P): pivot <= 0 -> st->indefinite; Out = D^{-1} = X^T X.
//  mode 1 (G = W^T W, orth): pivot test min d_i > tau max d_i (reading C3) else st->fallback;
//          Out = T = X^T (so that P = W T = W R^{-1}, G = R^T R).
// Storage: As (lower) = L; As (upper, off-diagonal 8x8 blocks) = T = X^T; Di[b] = X_bb (8x8).
// ---------------------------------------------------------------------------------------------
namespace sc {
constexpr int LDA = 132;
__device__ __forceinline__ double rsqrt_nr(double d) {
  double r;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(d));
  const double h = 0.5 * d;
  r = r * fma(-h * r, r, 1.5);
  r = r * fma(-h * r, r, 1.5);
  return r;
}
}  // namespace sc

__global__ void __launch_bounds__(256) k_small_chol(const double* __restrict__ Ain, int sp, int mode, int nact,
                                                    double tau, double* __restrict__ Out, BcgStatus* st) {
  using sc::LDA;
  extern __shared__ double sm[];
  double* As = sm;                  // sp x LDA
  double* Di = sm + 128 * LDA;      // 16 x 64: X_bb = inv(L_bb), row-major 8x8
  double* Sc = Di + 16 * 64;        // 8 warps x 64 scratch
  __shared__ double piv[128];
  __shared__ int s_fail;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, t = lane & 3;
  const int NB = sp / 8;
  const int width = nact < 0 ? st->width : nact;
  if (tid == 0) s_fail = 0;
  for (int e = tid; e < sp * sp; e += 256) {
    const int i = e / sp, j = e - i * sp;
    double v = Ain[e];
    if (i >= width || j >= width) v = (i == j) ? 1.0 : 0.0;
    As[i * LDA + j] = v;
  }
  __syncthreads();
  // ============================ Cholesky
  for (int kb = 0; kb < NB; ++kb) {
    const int c0 = 8 * kb;
    if (tid == 0) {
      double a[8][8], x[8][8], il[8];
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) a[i][j] = (j <= i) ? As[(c0 + i) * LDA + c0 + j] : 0.0;
      bool fail = false;
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        double d = a[c][c];
        piv[c0 + c] = d;
        if (!(d > 0.0)) {
          fail = true;
          d = 1.0;
        }
        const double r = sc::rsqrt_nr(d);
        il[c] = r;
        a[c][c] = d * r;
#pragma unroll
        for (int i = c + 1; i < 8; ++i) a[i][c] *= r;
#pragma unroll
        for (int j = c + 1; j < 8; ++j)
#pragma unroll
          for (int i = j; i < 8; ++i) a[i][j] = fma(-a[i][c], a[j][c], a[i][j]);
      }
      // x = inv(L) (lower), right-looking
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) x[i][j] = (i == j) ? 1.0 : 0.0;
#pragma unroll
      for (int k = 0; k < 8; ++k) {
#pragma unroll
        for (int j = 0; j <= k; ++j) x[k][j] *= il[k];
#pragma unroll
        for (int i = k + 1; i < 8; ++i)
#pragma unroll
          for (int j = 0; j <= k; ++j) x[i][j] = fma(-a[i][k], x[k][j], x[i][j]);
      }
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          As[(c0 + i) * LDA + c0 + j] = (j <= i) ? a[i][j] : 0.0;
          Di[kb * 64 + i * 8 + j] = (j <= i) ? x[i][j] : 0.0;
        }
      if (fail) s_fail = 1;
    }
    __syncthreads();
    if (s_fail) break;
    // panel: L[i][c0..c0+8) = A[i][c0..c0+8) X_kk^T, one row per thread
    for (int i = c0 + 8 + tid; i < sp; i += 256) {
      double a[8], o[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) a[k] = As[i * LDA + c0 + k];
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        double sacc = 0.0;
#pragma unroll
        for (int k = 0; k <= j; ++k) sacc = fma(a[k], Di[kb * 64 + j * 8 + k], sacc);
        o[j] = sacc;
      }
#pragma unroll
      for (int j = 0; j < 8; ++j) As[i * LDA + c0 + j] = o[j];
    }
    __syncthreads();
    // trailing update on 8x8 tiles: A_IJ -= L_I,kb L_J,kb^T (I >= J > kb), one tile per warp-task
    const int m = NB - 1 - kb;
    const int ntile = m * (m + 1) / 2;
    for (int task = warp; task < ntile; task += 8) {
      // decode (q, p), p <= q, from the linear index
      int q = (int)((sqrtf(8.0f * task + 1.0f) - 1.0f) * 0.5f);
      while (q * (q + 1) / 2 > task) --q;
      while ((q + 1) * (q + 2) / 2 <= task) ++q;
      const int p = task - q * (q + 1) / 2;
      const int I = kb + 1 + q, J = kb + 1 + p;
      const double* LI = As + (8 * I) * LDA + c0;
      const double* LJ = As + (8 * J) * LDA + c0;
      double c0v = 0.0, c1v = 0.0;
#pragma unroll
      for (int k = 0; k < 8; k += 4) dmma(c0v, c1v, LI[g * LDA + k + t], LJ[g * LDA + k + t]);
      double* dst = As + (8 * I + g) * LDA + 8 * J + 2 * t;
      dst[0] -= c0v;
      dst[1] -= c1v;
    }
    __syncthreads();
  }
  if (s_fail) {
    if (tid == 0) {
      if (mode == 0) st->indefinite = 1;
      else st->fallback = 1;
    }
    return;
  }
  if (mode == 1) {
    double mn = piv[0], mx = piv[0];
    for (int i = 1; i < width; ++i) {
      mn = fmin(mn, piv[i]);
      mx = fmax(mx, piv[i]);
    }
    if (!(mn > tau * mx)) {
      if (tid == 0) st->fallback = 1;
      return;
    }
    if (tid == 0) {
      st->fallback = 0;
      st->width = width;
    }
  }
  if (mode == 2) {  // R = L^T (upper), G = R^T R
    if (tid == 0) st->fallback = 0;
    for (int e = tid; e < sp * sp; e += 256) {
      const int p = e / sp, q = e - p * sp;
      Out[e] = (q >= p) ? As[q * LDA + p] : 0.0;
    }
    return;
  }
  // ============================ X = L^{-1}, block row by block row:
  // X_IJ = -X_II sum_{K=J}^{I-1} L_IK X_KJ  (J < I);  stored transposed: As[8J + c][8I + r] = X_IJ[r][c]
  double* scr = Sc + warp * 64;
  for (int I = 1; I < NB; ++I) {
    for (int J = warp; J < I; J += 8) {
      double c0v = 0.0, c1v = 0.0;
      for (int K = J; K < I; ++K) {
        const double* LIK = As + (8 * I) * LDA + 8 * K;          // A[m][k] = LIK[m][k]
#pragma unroll
        for (int k = 0; k < 8; k += 4) {
          // B[k][n] = X_KJ[k][n]: K == J -> Di[J]; else T block (J, K): X_KJ[k][n] = As[8J + n][8K + k]
          const double b = (K == J) ? Di[J * 64 + (k + t) * 8 + g] : As[(8 * J + g) * LDA + 8 * K + k + t];
          dmma(c0v, c1v, LIK[g * LDA + k + t], b);
        }
      }
      // scr = tmp (8x8, row-major), then X_IJ = -X_II tmp
      scr[g * 8 + 2 * t] = c0v;
      scr[g * 8 + 2 * t + 1] = c1v;
      __syncwarp();
      double d0 = 0.0, d1 = 0.0;
#pragma unroll
      for (int k = 0; k < 8; k += 4) dmma(d0, d1, Di[I * 64 + g * 8 + k + t], scr[(k + t) * 8 + g]);
      __syncwarp();
      As[(8 * J + 2 * t) * LDA + 8 * I + g] = -d0;
      As[(8 * J + 2 * t + 1) * LDA + 8 * I + g] = -d1;
    }
    __syncthreads();
  }
  // T[p][q] = X[q][p]
  auto Tval = [&](int p, int q) -> double {
    const int bp = p >> 3, bq = q >> 3;
    if (bp == bq) return Di[bp * 64 + (q & 7) * 8 + (p & 7)];
    if (bp < bq) return As[p * LDA + q];
    return 0.0;
  };
  if (mode == 1) {
    for (int e = tid; e < sp * sp; e += 256) {
      const int p = e / sp, q = e - p * sp;
      Out[e] = Tval(p, q);
    }
    return;
  }
  // D^{-1} = X^T X on 8x8 tiles: Dinv_IJ = sum_{K >= J} X_KI^T X_KJ   (I <= J), mirrored
  const int ntile = NB * (NB + 1) / 2;
  for (int task = warp; task < ntile; task += 8) {
    int q = (int)((sqrtf(8.0f * task + 1.0f) - 1.0f) * 0.5f);
    while (q * (q + 1) / 2 > task) --q;
    while ((q + 1) * (q + 2) / 2 <= task) ++q;
    const int I = task - q * (q + 1) / 2, J = q;  // I <= J
    double c0v = 0.0, c1v = 0.0;
    for (int K = J; K < NB; ++K) {
#pragma unroll
      for (int k = 0; k < 8; k += 4) {
        // A[m][k] = X_KI[k][m] = T[8I + m][8K + k];  B[k][n] = X_KJ[k][n] = T[8J + n][8K + k]
        const double a = Tval(8 * I + g, 8 * K + k + t);
        const double b = Tval(8 * J + g, 8 * K + k + t);
        dmma(c0v, c1v, a, b);
      }
    }
    const int r = 8 * I + g, cc = 8 * J + 2 * t;
    Out[r * sp + cc] = c0v;
    Out[r * sp + cc + 1] = c1v;
    Out[cc * sp + r] = c0v;
    Out[(cc + 1) * sp + r] = c1v;
  }
}

// ---------------------------------------------------------------------------------------------
// one-CTA cyclic (round-robin) parallel Jacobi eigensolver of a symmetric n x n matrix (n <= 128,
// padded to even ne).  Everything stays in shared memory: A packed upper-triangular (the two-sided
// rotation keeps it symmetric; 66 KB at ne = 128) and a row slice of V transposed (Vt[k][i - i0] =
// V_ik).  The grid's CTAs all run the IDENTICAL A iteration (same instructions on the same data, so
// bitwise the same rotations) and each accumulates only its own rows of V: V's shared-memory
// traffic, the bound of a one-CTA Jacobi, is split across the grid with no communication.  One
// round = ne/2 disjoint rotations: phase 1 (one thread per pair) computes (c, s) and rotates its
// own 2 x 2 diagonal block (Golub-Van Loan Alg. 8.4.1 formulas, a_pq <- 0); phase 2 applies
// J_k^T B J_l to every off-diagonal 2 x 2 block (k < l) in ONE pass and rotates V.  Two barriers
// per round.  Outputs eigenvalues (descending) and eigenvectors (columns, same order).  `gate`
// (optional): run only if *gate != 0.  Vwork is unused (kept for the call signature).
// ---------------------------------------------------------------------------------------------
#ifdef NSP_EIG_PROF
__device__ int g_eig_sweeps;
#endif
__global__ void __launch_bounds__(1024) k_small_eig(const double* __restrict__ Ain, int lda, int n,
                                                    double* Vwork, int ldv, double* lam, double* Vsorted,
                                                    const int* gate, double tau, double* Tout, int spT,
                                                    BcgStatus* stw) {
  pdl_wait();
  (void)Vwork;
  (void)ldv;
  if (gate && *gate == 0) return;
  extern __shared__ double sm[];
  const int ne = n + (n & 1);
  const int npair = ne / 2;
  double* Ap = sm;                              // packed upper triangle, ne (ne + 1) / 2
  const int rp = (ne + gridDim.x - 1) / gridDim.x;      // V rows per CTA
  const int i0 = blockIdx.x * rp, i1 = min(ne, i0 + rp);
  double* Vt = sm + ne * (ne + 1) / 2;          // ne x rp, Vt[k * rp + (i - i0)]
  __shared__ double2 csn[64];                   // (c, s) per pair
  __shared__ int2 pq[64];                       // (p, q) per pair, p < q
  __shared__ double red[2][32];
  __shared__ int order[128];
  const int tid = threadIdx.x, nt = blockDim.x;
  auto tri = [ne](int a, int b) -> int {      // a <= b
    return a * ne - (a * (a - 1)) / 2 + (b - a);
  };
  auto at = [&](int a, int b) -> double& { return a <= b ? Ap[tri(a, b)] : Ap[tri(b, a)]; };
  for (int e = tid; e < ne * ne; e += nt) {
    const int i = e / ne, j = e - i * ne;
    if (i <= j) Ap[tri(i, j)] = (i < n && j < n) ? Ain[i * lda + j] : 0.0;
  }
  for (int e = tid; e < ne * rp; e += nt) {
    const int k = e / rp, i = i0 + (e - k * rp);
    Vt[e] = (i == k) ? 1.0 : 0.0;
  }
  __syncthreads();
  const int nblk = npair * (npair - 1) / 2;     // off-diagonal pair blocks k < l (<= 2016 < 2 nt)
  const int vk_stride = nt / rp, vi = tid % rp, vk0 = tid / rp;   // V rotation: row i0 + vi, pairs vk0 + j stride
  int bk[2], bl[2];                             // this thread's blocks, fixed across rounds
#pragma unroll
  for (int u = 0; u < 2; ++u) {
    int k = 0, rem = tid + u * nt;
    while (k < npair && rem >= npair - 1 - k) {
      rem -= npair - 1 - k;
      ++k;
    }
    bk[u] = k;
    bl[u] = k + 1 + rem;
  }
  double prev_offs = 0.0;
  for (int sweep = 0; sweep < 60; ++sweep) {
    // off-diagonal and total norms (symmetric: off-diagonal entries count twice)
    // the off-diagonal sum of squares is accumulated on its own - NOT as (all - diagonal), whose
    // cancellation leaves a ~1e-16 ||A||^2 noise floor above the 1e-28 target (round 2: the Nystrom C,
    // diagonal-dominated at convergence, ran all 60 sweeps)
    double off = 0.0, tot = 0.0;
    for (int e = tid; e < ne * ne; e += nt) {
      const int i = e / ne, j = e - i * ne;
      if (j < i) continue;
      const double v = Ap[tri(i, j)];
      if (i == j) tot += v * v;
      else off += v * v;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      off += __shfl_xor_sync(0xffffffffu, off, o);
      tot += __shfl_xor_sync(0xffffffffu, tot, o);
    }
    if ((tid & 31) == 0) {
      red[0][tid >> 5] = off;
      red[1][tid >> 5] = tot;
    }
    __syncthreads();
    double offs = 0.0, tots = 0.0;
    for (int w = 0; w < nt / 32; ++w) {       // fixed order: identical on every thread
      offs += red[0][w];
      tots += red[1][w];
    }
    __syncthreads();
    // off-diagonal entries stored once: ||A||_F^2 = sum diag^2 + 2 sum upper^2
    offs = 2.0 * offs;
    tots = tots + offs;
    if (!(offs > 1e-28 * tots) || tots == 0.0) break;
    const double tot_sweep = tots;
    // rounding floor: the off-diagonal norm has stopped falling (a sweep no longer halves it) at a level
    // already below 1e-12 ||A||_F - the 1e-14 target is under the attainable floor for this matrix and
    // further sweeps only cost time (round 2: C and T of Nystrom took the full 60 sweeps, 15 ms each)
    if (sweep > 0 && offs > 0.5 * prev_offs && offs <= 1e-24 * tots) break;
    prev_offs = offs;
#ifdef NSP_EIG_PROF
    if (tid == 0) g_eig_sweeps = sweep + 1;
#ifdef NSP_EIG_TRACE
    if (tid == 0 && blockIdx.x == 0) printf("sweep %d off/tot %.3e\n", sweep, offs / tots);
#endif
#endif
    for (int round = 0; round < ne - 1; ++round) {
      // phase 1: tournament pairing (position 0 fixed, the others rotate), rotation parameters,
      // the pair's own 2 x 2 diagonal block
      if (tid < npair) {
        auto who = [&](int pos) -> int { return pos == 0 ? 0 : 1 + (pos - 1 + round) % (ne - 1); };
        int p = who(tid), q = who(ne - 1 - tid);
        if (p > q) {
          const int t = p;
          p = q;
          q = t;
        }
        pq[tid] = make_int2(p, q);
        double& app = Ap[tri(p, p)];
        double& aqq = Ap[tri(q, q)];
        double& apq = Ap[tri(p, q)];
        double c = 1.0, s = 0.0;
        const double a_pq = apq, a_pp = app, a_qq = aqq;
        // rotate unless a_pq is negligible relative to its diagonal pair OR to the whole matrix (|a_pq| <=
        // 1e-17 ||A||_F: rounding noise that rotations between tiny diagonal entries would otherwise keep
        // regenerating elsewhere, so the sweeps never reached the off-norm target)
        if (fabs(a_pq) > 1e-300 && a_pq * a_pq > 1e-36 * fabs(a_pp * a_qq) && a_pq * a_pq > 1e-34 * tot_sweep) {
          // t = sign(th) / (|th| + sqrt(th^2 + 1)), th = d / (2 a_pq), d = a_qq - a_pp, written
          // as t = 2 a_pq sign(d) / (|d| + sqrt(d^2 + 4 a_pq^2)): one sqrt, one divide
          const double d = a_qq - a_pp;
          const double num = d >= 0 ? 2.0 * a_pq : -2.0 * a_pq;
          const double t = num / (fabs(d) + sqrt(d * d + 4.0 * a_pq * a_pq));
          c = rsqrt(t * t + 1.0);
          s = t * c;
          app = a_pp - t * a_pq;
          aqq = a_qq + t * a_pq;
          apq = 0.0;
        }
        csn[tid] = make_double2(c, s);
      }
      __syncthreads();
      // phase 2a: off-diagonal blocks B = A[{pk, qk}, {pl, ql}] <- J_k^T B J_l, J = [[c, s], [-s, c]]
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        if (tid + u * nt >= nblk) break;
        const int k = bk[u], l = bl[u];
        const int2 Pk = pq[k], Pl = pq[l];
        const double2 Ck = csn[k], Cl = csn[l];
        const int pk = Pk.x, qk = Pk.y, pl = Pl.x, ql = Pl.y;
        const double ck = Ck.x, sk = Ck.y, cl = Cl.x, sl = Cl.y;
        double& b00 = at(pk, pl);
        double& b01 = at(pk, ql);
        double& b10 = at(qk, pl);
        double& b11 = at(qk, ql);
        // rows (J_k^T): r_p = c b_p - s b_q, r_q = s b_p + c b_q
        const double r00 = ck * b00 - sk * b10, r01 = ck * b01 - sk * b11;
        const double r10 = sk * b00 + ck * b10, r11 = sk * b01 + ck * b11;
        // columns (J_l): col_p = c col_p - s col_q, col_q = s col_p + c col_q
        b00 = cl * r00 - sl * r01;
        b01 = sl * r00 + cl * r01;
        b10 = cl * r10 - sl * r11;
        b11 = sl * r10 + cl * r11;
      }
      // phase 2b: V <- V J (V transposed: columns p, q are rows of Vt, contiguous)
      if (tid < vk_stride * rp)
        for (int k = vk0; k < npair; k += vk_stride) {
          const int2 P = pq[k];
          const double2 C = csn[k];
          const int p = P.x, q = P.y;
          const double c = C.x, s = C.y;
          const double vp = Vt[p * rp + vi], vq = Vt[q * rp + vi];
          Vt[p * rp + vi] = c * vp - s * vq;
          Vt[q * rp + vi] = s * vp + c * vq;
        }
      __syncthreads();
    }
  }
  // sort descending (stable by index) - rank by counting
  if (tid < n) {
    const double li = Ap[tri(tid, tid)];
    int r = 0;
    for (int j = 0; j < n; ++j) {
      const double lj = Ap[tri(j, j)];
      if (lj > li || (lj == li && j < tid)) ++r;
    }
    order[r] = tid;
  }
  __syncthreads();
  if (tid < n && blockIdx.x == 0) lam[tid] = Ap[tri(order[tid], order[tid])];
  const int nr = max(0, min(i1, n) - i0);
  for (int e = tid; e < nr * n; e += nt) {
    const int i = e / n, k = e - i * n;
    Vsorted[(i0 + i) * n + k] = Vt[order[k] * rp + i];
  }
  if (Tout) {   // orth's eigen fallback (reading C3): keep lambda > tau lambda_max, T = V_keep Lambda^{-1/2}
    __shared__ double ls[128];
    __shared__ int wk;
    if (tid < n) ls[tid] = Ap[tri(order[tid], order[tid])];
    __syncthreads();
    if (tid == 0) {
      int cnt = 0;
      if (ls[0] > 0)
        for (int k = 0; k < n; ++k)
          if (ls[k] > tau * ls[0]) ++cnt;
      wk = cnt;
      if (blockIdx.x == 0) stw->width = cnt;
    }
    __syncthreads();
    const int w = wk;
    for (int e = tid; e < nr * spT; e += nt) {   // this CTA's rows of V
      const int i = e / spT, k = e - i * spT;
      Tout[(int64_t)(i0 + i) * spT + k] = k < w ? Vt[order[k] * rp + i] / sqrt(ls[k]) : 0.0;
    }
    if (blockIdx.x == 0)
      for (int e = tid; e < (spT - n) * spT; e += nt) Tout[(int64_t)n * spT + e] = 0.0;   // rows >= n
  }
}


// C = alpha * op(A) op(B) + beta * C, all sp-ish small (m x n, inner k), row-major, FMA.
__global__ void k_small_gemm(int m, int n, int k, double alpha, const double* A, int lda, int ta, const double* B,
                             int ldb, int tb, double beta, double* Cm, int ldc) {
  pdl_wait();
  const int i = blockIdx.y * 16 + threadIdx.y;
  const int j = blockIdx.x * 16 + threadIdx.x;
  if (i >= m || j >= n) return;
  double s = 0.0;
  for (int q = 0; q < k; ++q) {
    const double a = ta ? A[q * lda + i] : A[i * lda + q];
    const double b = tb ? B[j * ldb + q] : B[q * ldb + j];
    s = fma(a, b, s);
  }
  Cm[i * ldc + j] = alpha * s + (beta != 0.0 ? beta * Cm[i * ldc + j] : 0.0);
}

// A <- (A + A^T) / 2 (n x n, ld), plus shift on the diagonal
__global__ void k_small_sym(double* A, int n, int ld, double shift) {
  const int i = blockIdx.y * 16 + threadIdx.y, j = blockIdx.x * 16 + threadIdx.x;
  if (i >= n || j > i) return;
  const double v = 0.5 * (A[i * ld + j] + A[j * ld + i]);
  A[i * ld + j] = v + (i == j ? shift : 0.0);
  A[j * ld + i] = v + (i == j ? shift : 0.0);
}
// M[i][k] = V[i][k] * colscale[k] for k < r, 0 for k >= r (n rows, ld)
__global__ void k_scale_cols(const double* V, int ldv, const double* colscale, int r, int n, int ncols, double* M,
                             int ldm, int mode) {
  pdl_wait();
  const int i = blockIdx.y * 16 + threadIdx.y, k = blockIdx.x * 16 + threadIdx.x;
  if (i >= n || k >= ncols) return;
  double v = 0.0;
  if (k < r) {
    const double sc = colscale[k];
    v = mode == 3 ? V[i * ldv + k] : V[i * ldv + k] * (mode == 0 ? sc : (mode == 1 ? 1.0 / sqrt(sc) : sqrt(sc)));
  }
  M[i * ldm + k] = v;
}

// rows i < r scaled by d[i], rows r <= i < nrows zeroed
__global__ void k_scale_rows(double* G, int ld, const double* d, int r, int nrows, int ncols) {
  pdl_wait();
  const int i = blockIdx.y * 16 + threadIdx.y, j = blockIdx.x * 16 + threadIdx.x;
  if (i >= nrows || j >= ncols) return;
  G[i * ld + j] = i < r ? G[i * ld + j] * d[i] : 0.0;
}

// copy with ld change and zero padding: dst[r][c] = c < s ? src[r][c] : 0 (c < ldd)
// one Chebyshev step after t = A d: x += d; r -= t; d' = c1 d + c2 r (new r)
__global__ void k_cheb_update(double* __restrict__ x, double* __restrict__ r, const double* __restrict__ d,
                              const double* __restrict__ t, double* __restrict__ dn, double c1, double c2, int64_t n,
                              int want_d) {
  pdl_wait();
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double di = d[i];
  x[i] += di;
  const double ri = r[i] - t[i];
  r[i] = ri;
  if (want_d) dn[i] = fma(c1, di, c2 * ri);
}

__global__ void k_copy_pad(const double* src, int lds, double* dst, int ldd, int64_t n, int s, double scale) {
  pdl_wait();
  const int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t r = idx / ldd;
  const int c = (int)(idx - r * ldd);
  if (r >= n) return;
  dst[r * ldd + c] = c < s ? scale * src[r * lds + c] : 0.0;
}

}  // namespace

namespace nspb {

static int gram_ctas() { return NSP_GCTAS_PER_SM * num_sms(); }   // Gram CTAs: two resident per SM

int gram_chunks(int64_t n, int ntiles) {   // one wave: tiles x chunks <= NSP_GCTAS_PER_SM x SMs CTAs
  int64_t ch = (n + GR - 1) / GR;
  const int64_t cap = gram_ctas() / ntiles;
  if (ch > cap) ch = cap;
  return (int)(ch < 1 ? 1 : ch);
}

size_t gram_ws_doubles(int64_t n, int sa, int sb) {
  // every launch uses chunks x tiles <= max(gram_ctas(), tiles) partial tiles (the symmetric Gram has
  // fewer tiles and so more chunks than the two-operand one); the fused panel + Gram (s = 128) writes
  // 4 tiles per SM
  const int ntm = (sa + 63) / 64, ntn = 2 * ((sb + 63) / 64);
  (void)n;
  return (size_t)std::max(std::max(gram_ctas(), 4 * num_sms()), ntm * ntn) * 4096;
}

bool panel_gram_shape_ok(int s, int64_t n) { return s == 128 && n >= (int64_t)64 * num_sms(); }

int nsp_fused_pg_mode = 0;   // nsp_dev_set_fused_pg: 0 production threshold, 1 force (shape ok), 2 never
bool panel_gram_ok(int s, int64_t n) {
  static const bool off = [] {
    const char* e = getenv("NSP_FUSED_PG");
    return e && e[0] == '0';
  }();
  if (nsp_fused_pg_mode == 1) return panel_gram_shape_ok(s, n);
  if (nsp_fused_pg_mode == 2) return false;
  // Not used by default: measured NOT faster.  The tall-skinny passes are DMMA-bound (s / 8 = 16 flop/B
  // at s = 128), so reading each block once saves HBM bytes that are not the binding resource, while
  // the fused pass does the panel and the Gram flops back to back in one CTA per SM.  cfg2 (97 rows / SM):
  // 51 + 53 us against 25 + 26 + 9 us (block CG 464 vs 438 us per iteration); cfg5 (12.4k rows / SM):
  // 4.26 + 4.50 ms against 2.19 + 2.0 and 2.19 + 1.5 ms (block CG 97.3 vs 96.8 ms per iteration)
  // (profiles/r02_ab_*.jsonl, r02_launches_*).  nsp_dev_set_fused_pg(1) forces it (parity tests).
  (void)n;
  return !off && false;
}


int panel_gram(double* Out, const double* Cin, const double* In, const double* M, int64_t n, double sgn,
               double* normpart, int gmode, double* gram_out, double* ws, cudaStream_t st) {
  const int nsm = num_sms();
  PanelArgs a{Out, 128, Cin, 128, In, 128, M, 128, sgn, normpart};
  const size_t smem = (size_t)(128 + 32 + 32) * FG_LD * sizeof(double);
  nsp_count_path(NSP_PATH_PANEL_GRAM);
  if (gmode == 0) {
    smem_optin((const void*)k_panel_gram<0>, smem);
    nsp_count_launch();
    launch_k(k_panel_gram<0>, dim3(nsm), dim3(512), smem, st, a, n, (n + 15) / 16, ws);
  } else {
    smem_optin((const void*)k_panel_gram<1>, smem);
    nsp_count_launch();
    launch_k(k_panel_gram<1>, dim3(nsm), dim3(512), smem, st, a, n, (n + 15) / 16, ws);
  }
  nsp_count_launch();
  launch_k(k_gram_reduce, dim3(8, 8), dim3(16, 16, 4), 0, st, (const double*)ws, nsm, 2, 2, 2, gram_out,
           (double*)nullptr, 128, gmode == 0 ? 0 : 1);
  return nsm;
}

void gram2(const double* Xa, int lda, int sa, const double* Xb, const double* Xb2, int ldb, int sb, int64_t n,
           double* out, double* out2, int ldo, double* ws, cudaStream_t st, bool lower_first) {
  const int ntm = (sa + 63) / 64, ntn1 = (sb + 63) / 64;
  const int ntn = Xb2 ? 2 * ntn1 : ntn1;
  // Xa == Xb (W^T W, Y^T Y): only the tiles on and above the diagonal (3 of 4 at s = 128)
  static const bool sym_env_off = getenv("NSP_GRAM_NOSYM") != nullptr;
  const bool sym_off = sym_env_off || nsp_force_generic;
  int sym = (!sym_off && !Xb2 && Xa == Xb && lda == ldb && sa == sb && ntm > 1) ? 1 : 0;
  // [D | E] with D read only through its lower triangle: D's upper tiles are mirrored, not computed
  if (!sym_off && lower_first && Xb2 && ntn1 == ntm && ntm > 1) sym = 2;
  nsp_count_path(sym == 1 ? NSP_PATH_GRAM_SYM : sym == 2 ? NSP_PATH_GRAM_DE : NSP_PATH_GRAM_FULL);
  const int ntiles = sym == 1 ? ntm * (ntm + 1) / 2 : sym == 2 ? ntm * (ntm + 1) / 2 + ntm * ntn1 : ntm * ntn;
  int nch = gram_chunks(n, ntiles);
  // NSP_GRAM_CL=8: clusters of 8 chunk-CTAs pre-sum their partials in distributed shared memory (8x fewer
  // partials to reduce) - parity-clean but measured SLOWER end to end (the 8-CTA co-scheduling of
  // 104 KB-smem CTAs costs more than the reduce saves), so off by default
  static const int gcl_env = [] {
    const char* e = getenv("NSP_GRAM_CL");
    return e ? atoi(e) : 1;   // off by default: measured slower (cfg2 414 vs 397 us, cfg5 101 vs 97 ms per iteration)
  }();
  const int gcl = (gcl_env == 8 && nch >= 16 && !nsp_force_generic) ? 8 : 1;
  if (gcl > 1) nch = (nch / gcl) * gcl;
  int64_t rpc = (n + nch - 1) / nch;
  rpc = ((rpc + GR - 1) / GR) * GR;
  const size_t smem = GNS * 2 * GR * LDS * sizeof(double);
  if (gcl > 1) {
    smem_optin((const void*)k_gram_partial<8>, smem);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(ntiles, nch);
    cfg.blockDim = dim3(256);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
    at[1].id = cudaLaunchAttributeClusterDimension;
    at[1].val.clusterDim.x = 1;
    at[1].val.clusterDim.y = 8;
    at[1].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 2;
    nsp_count_launch();
    cudaLaunchKernelEx(&cfg, k_gram_partial<8>, Xa, lda, Xb, Xb2, ldb, ntn1, n, rpc, ws, ntm, ntn, sym);
  } else {
    smem_optin((const void*)k_gram_partial<1>, smem);
    nsp_count_launch();
    launch_k(k_gram_partial<1>, dim3(dim3(ntiles, nch)), dim3(256), smem, st, Xa, lda, Xb, Xb2, ldb, ntn1, n, rpc, ws, ntm, ntn, sym);
  }
  { nsp_count_launch(); launch_k(k_gram_reduce, dim3(dim3(ntn * 4, ntm * 4)), dim3(dim3(16, 16, 4)), 0, st, ws, nch / gcl, ntm, ntn, ntn1, out, out2, ldo, sym); }
}

void gram(const double* Xa, int lda, int sa, const double* Xb, int ldb, int sb, int64_t n, double* out, int ldo,
          double* ws, cudaStream_t st) {
  gram2(Xa, lda, sa, Xb, nullptr, ldb, sb, n, out, nullptr, ldo, ws, st);
}

void panel2(const PanelArgs& a0, const PanelArgs* a1, int kdim, int ncols, int64_t n, cudaStream_t st) {
  if (n <= 0) return;
  const size_t smem = (2 * 64 * 36 + 2 * 32 * LDS) * sizeof(double);
  smem_optin((const void*)k_panel, smem);
  dim3 grid((unsigned)((n + 63) / 64), (ncols + 63) / 64, a1 ? 2 : 1);
  { nsp_count_launch(); launch_k(k_panel, dim3(grid), dim3(256), smem, st, a0, a1 ? *a1 : a0, kdim, n); }
}

int panel(double* Out, int ldo, const double* Cin, int ldc, const double* In, int ldi, const double* M, int ldm,
          int kdim, int ncols, int64_t n, double sgn, double* normpart, cudaStream_t st, const int* upper_unless) {
  PanelArgs a{Out, ldo, Cin, ldc, In, ldi, M, ldm, sgn, normpart, upper_unless};
  const int nsm = num_sms();
  static const bool rows_off = [] {
    const char* e = getenv("NSP_PANEL_ROWS");
    return e && e[0] == '0';
  }();
  // one-wave row-range panel: s = 128 and at least one 64-row pass per SM (normpart rows = CTAs)
  static const int half_mode = [] {   // NSP_PANEL_HALF: 0 off, 1 two CTAs / SM with 64-row passes, 2 with 32-row
    const char* e = getenv("NSP_PANEL_HALF");
    return e ? atoi(e) : 0;
  }();
  if (half_mode && !rows_off && !nsp_force_generic && kdim == 128 && ncols == 128 && n >= (int64_t)64 * nsm &&
      ldo >= 128) {
    nsp_count_path(NSP_PATH_PANEL_ROWS);
    if (half_mode == 2) {
      const size_t smem = (128 * HLDM + 2 * 32 * HLDA) * sizeof(double);
      smem_optin((const void*)k_panel_half<32>, smem);
      nsp_count_launch();
      launch_k(k_panel_half<32>, dim3(2 * nsm), dim3(256), smem, st, a, n, (n + 15) / 16);
    } else {
      const size_t smem = (128 * HLDM + 2 * 64 * HLDA) * sizeof(double);
      smem_optin((const void*)k_panel_half<64>, smem);
      nsp_count_launch();
      launch_k(k_panel_half<64>, dim3(2 * nsm), dim3(256), smem, st, a, n, (n + 15) / 16);
    }
    return nsm;
  }
  if (!rows_off && !nsp_force_generic && kdim == 128 && ncols == 128 && n >= (int64_t)64 * nsm && ldo >= 128) {
    nsp_count_path(NSP_PATH_PANEL_ROWS);
    const size_t smem = (128 * PLDM + PNS * 64 * PLDA) * sizeof(double);
    smem_optin((const void*)k_panel_rows<NSP_PANEL_NW>, smem);
    { nsp_count_launch(); launch_k(k_panel_rows<NSP_PANEL_NW>, dim3(nsm), dim3(NSP_PANEL_NW * 32), smem, st, a, n, (n + 15) / 16); }
    return nsm;
  }
  nsp_count_path(NSP_PATH_PANEL_TILES);
  panel2(a, nullptr, kdim, ncols, n, st);
  return (int)((n + 63) / 64);
}

void colsq(const double* X, int ldx, int64_t n, int s, int ldp, double* part, double* out, cudaStream_t st) {
  const int nt = (int)std::max<int64_t>(1, (n + 63) / 64);   // n = 0 (a rank with no Gram rows): zeros
  { nsp_count_launch(); launch_k(k_colsq_partial, dim3(nt), dim3(ldp), 0, st, X, ldx, n, s, part, ldp); }
  { nsp_count_launch(); launch_k(k_colsq_reduce, dim3(1), dim3(dim3(128, 8)), 0, st, part, nt, ldp, out); }
}

void colsq_reduce(const double* part, int ntiles, int ldp, double* out, cudaStream_t st) {
  { nsp_count_launch(); launch_k(k_colsq_reduce, dim3(1), dim3(dim3(128, 8)), 0, st, part, ntiles, ldp, out); }
}

void sqrt_vec(const double* in, double* out, int n, cudaStream_t st) {
  { nsp_count_launch(); launch_k(k_sqrt_vec, dim3((n + 255) / 256), dim3(256), 0, st, in, out, n); }
}

void colsq_converge(const double* part, int ntiles, int ldp, double* rsq, const double* bnorm, int s, double tol,
                    BcgStatus* stt, cudaStream_t st) {
  { nsp_count_launch(); launch_k(k_colsq_converge, dim3(1), dim3(128, 8), 0, st, part, ntiles, ldp, rsq, bnorm, s, tol, stt); }
}

void converge(const double* rsq, const double* bnorm, int s, double tol, BcgStatus* stt, double* hist_slot,
              cudaStream_t st) {
  { nsp_count_launch(); launch_k(k_converge, dim3(1), dim3(256), 0, st, rsq, bnorm, s, tol, stt, hist_slot); }
}

void small_chol(const double* A, int sp, int mode, int nact, double tau, double* Out, BcgStatus* stt,
                cudaStream_t st) {
  const size_t smem = (size_t)(128 * sc::LDA + 16 * 64 + 8 * 64) * sizeof(double);
  smem_optin((const void*)k_small_chol, smem);
  { nsp_count_launch(); k_small_chol<<<1, 256, smem, st>>>(A, sp, mode, nact, tau, Out, stt); }
}

void small_eig(const double* A, int lda, int n, double* Vwork, int ldv, double* lam, double* Vsorted,
               const int* gate, cudaStream_t st, double tau, double* T, int spT, BcgStatus* stw) {
  const int ne = n + (n & 1);
  const int g = ne >= 128 ? 8 : ne >= 64 ? 4 : 1;   // V row slices (rp = ne / g rows each)
  const int rp = (ne + g - 1) / g;
  const size_t smem = (size_t)(ne * (ne + 1) / 2 + ne * rp) * sizeof(double);
  smem_optin((const void*)k_small_eig, smem);
  { nsp_count_launch(); launch_k(k_small_eig, dim3(g), dim3(1024), smem, st, A, lda, n, Vwork, ldv, lam, Vsorted, gate, tau, T, spT, stw); }
#ifdef NSP_EIG_PROF
  cudaStreamCaptureStatus cst = cudaStreamCaptureStatusNone;
  cudaStreamIsCapturing(st, &cst);
  if (cst == cudaStreamCaptureStatusNone) {   // diagnostics build: sweeps of this (eager) call
    cudaStreamSynchronize(st);
    int sw = 0;
    cudaMemcpyFromSymbol(&sw, g_eig_sweeps, sizeof(int));
    fprintf(stderr, "[nsp eig] n = %d: %d sweeps\n", n, sw);
  }
#endif
}


void small_gemm(int m, int n, int k, double alpha, const double* A, int lda, bool ta, const double* B, int ldb,
                bool tb, double beta, double* C, int ldc, cudaStream_t st) {
  dim3 grid((n + 15) / 16, (m + 15) / 16);
  { nsp_count_launch(); launch_k(k_small_gemm, dim3(grid), dim3(dim3(16, 16)), 0, st, m, n, k, alpha, A, lda, ta, B, ldb, tb, beta, C, ldc); }
}

void cheb_update(double* x, double* r, const double* d, const double* t, double* dn, double c1, double c2, int64_t n,
                 bool want_d, cudaStream_t st) {
  if (n <= 0) return;
  { nsp_count_launch(); launch_k(k_cheb_update, dim3((unsigned)((n + 255) / 256)), dim3(256), 0, st, x, r, d, t, dn, c1, c2, n, want_d ? 1 : 0); }
}

void copy_pad(const double* src, int lds, double* dst, int ldd, int64_t n, int s, double scale, cudaStream_t st) {
  const int64_t tot = n * ldd;
  if (tot <= 0) return;
  { nsp_count_launch(); launch_k(k_copy_pad, dim3((unsigned)((tot + 255) / 256)), dim3(256), 0, st, src, lds, dst, ldd, n, s, scale); }
}

void scale_rows(double* G, int ld, const double* d, int r, int nrows, int ncols, cudaStream_t st) {
  dim3 grid((ncols + 15) / 16, (nrows + 15) / 16);
  { nsp_count_launch(); launch_k(k_scale_rows, dim3(grid), dim3(dim3(16, 16)), 0, st, G, ld, d, r, nrows, ncols); }
}

void small_sym(double* A, int n, int ld, double shift, cudaStream_t st) {
  dim3 grid((n + 15) / 16, (n + 15) / 16);
  { nsp_count_launch(); k_small_sym<<<grid, dim3(16, 16), 0, st>>>(A, n, ld, shift); }
}

void scale_cols(const double* V, int ldv, const double* colscale, int r, int n, int ncols, double* M, int ldm,
                int mode, cudaStream_t st) {
  dim3 grid((ncols + 15) / 16, (n + 15) / 16);
  { nsp_count_launch(); launch_k(k_scale_cols, dim3(grid), dim3(dim3(16, 16)), 0, st, V, ldv, colscale, r, n, ncols, M, ldm, mode); }
}

}  // namespace nspb
