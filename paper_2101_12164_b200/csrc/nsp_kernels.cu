#include <climits>
// Device kernels of the S_G apply and the setup factorisation (north_star (a), (b); §8(a) rows
// a1-a5, s0).  fp64 throughout; dense tile products on the DMMA pipe (mma.sync f64).
#include <cuda_runtime.h>
#include <algorithm>
#include <cstdlib>
#include <stdint.h>

#include "nsp_dmma.cuh"
#include "nsp_internal.h"

using namespace nspd;

namespace {

constexpr int LDT = 68;  // smem row stride (doubles) of a 64x64 tile: conflict-free fragment loads

// ---------------------------------------------------------------------------------------------
// setup helpers
// ---------------------------------------------------------------------------------------------
__global__ void k_scatter(double* base, const int64_t* idx, const double* val, int64_t cnt) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < cnt) base[idx[i]] = val[i];
}

__global__ void k_pad_identity(double* base, const int64_t* tile_idx, const int* first_row, int cnt) {
  pdl_wait();
  int t = blockIdx.x;
  if (t >= cnt) return;
  double* T = base + tile_idx[t] * NSP_TILE_ELEMS;
  for (int r = first_row[t] + threadIdx.x; r < NSP_TILE; r += blockDim.x) T[r * NSP_TILE + r] = 1.0;
}

// ---------------------------------------------------------------------------------------------
// s0: right-looking tile Cholesky of one block per CTA (eq:cholesky).
// Column tile K: potrf(L_KK) in smem -> inv(L_KK) stored in the diagonal slot; panel
// L_IK = A_IK inv(L_KK)^T for every structurally nonzero tile below; trailing update
// A_ab -= L_aK L_bK^T for all panel pairs a >= b.  Structural pattern: band tiles
// (0 < I-K <= wb), border tiles (I' with border_first[I'] <= K), then the dense tail.
// ---------------------------------------------------------------------------------------------
__device__ __forceinline__ double* band_tile(const FacSub& sb, double* band, int I, int K) {
  return band + (sb.band_off + (int64_t)K * (sb.wb + 1) + (I - K)) * NSP_TILE_ELEMS;
}
__device__ __forceinline__ double* border_tile(const FacSub& sb, double* scratch, int Ib, int K) {
  return scratch + (sb.border_off + (int64_t)Ib * sb.nt1 + K) * NSP_TILE_ELEMS;
}
__device__ __forceinline__ double* dense_tile(const FacSub& sb, double* dense, int I, int J) {
  return dense + (sb.dense_off + (int64_t)I * (I + 1) / 2 + J) * NSP_TILE_ELEMS;
}

__global__ void __launch_bounds__(256) k_tile_cholesky(const FacSub* __restrict__ subs, double* band,
                                                       double* dense, double* scratch,
                                                       const int* __restrict__ border_first, int* status) {
  extern __shared__ double sm[];
  double* Ds = sm;                    // diag tile / factor
  double* Li = sm + 64 * LDT;         // inv(L_KK)
  double* As = sm + 2 * 64 * LDT;     // panel operand a
  double* Bs0 = sm + 3 * 64 * LDT;    // panel operand b (double buffered)
  double* Bs1 = sm + 4 * 64 * LDT;
  __shared__ double colv[64];
  __shared__ int s_fail;
  __shared__ short plist[2048];       // panel list: encoded tile refs (band: I-K in [1,wb]; border: 4096+I')

  const FacSub sb = subs[blockIdx.x];
  const int* bfirst = border_first + sb.border_first_off;
  const int NT = sb.nt1 + sb.ntb;
  const int tid = threadIdx.x;
  if (tid == 0) s_fail = 0;

  for (int K = 0; K < NT; ++K) {
    const bool dphase = K >= sb.nt1;
    const int Kd = K - sb.nt1;
    double* Dg = dphase ? dense_tile(sb, dense, Kd, Kd) : band_tile(sb, band, K, K);
    // ---- load diag tile (lower part used)
    for (int e = tid; e < 4096; e += 256) Ds[(e >> 6) * LDT + (e & 63)] = Dg[e];
    __syncthreads();
    // ---- unblocked Cholesky (2 barriers per column)
    for (int c = 0; c < 64; ++c) {
      const double d = Ds[c * LDT + c];
      if (!(d > 0.0)) {
        if (tid == 0) {
          s_fail = 1;
          status[sb.status_idx] = K * 64 + c + 1;  // 1-based local row in the padded ordering
        }
        break;
      }
      const double l = sqrt(d);
      if (tid > c && tid < 64) colv[tid] = Ds[tid * LDT + c] / l;
      __syncthreads();
      for (int e = tid; e < 64 * 64; e += 256) {
        const int r = e >> 6, q = e & 63;
        if (q > c && r >= q) Ds[r * LDT + q] -= colv[r] * colv[q];
      }
      if (tid > c && tid < 64) Ds[tid * LDT + c] = colv[tid];
      if (tid == 0) Ds[c * LDT + c] = l;
      __syncthreads();
    }
    __syncthreads();
    if (s_fail) return;
    // ---- inverse of the lower-triangular factor: thread j < 64 solves L x = e_j (column j of inv)
    if (tid < 64) {
      const int j = tid;
      for (int i = 0; i < 64; ++i) {
        double v;
        if (i < j) {
          v = 0.0;
        } else {
          double sacc = (i == j) ? 1.0 : 0.0;
          for (int k = j; k < i; ++k) sacc -= Ds[i * LDT + k] * Li[k * LDT + j];
          v = sacc / Ds[i * LDT + i];
        }
        Li[i * LDT + j] = v;
      }
    }
    __syncthreads();
    for (int e = tid; e < 4096; e += 256) Dg[e] = Li[(e >> 6) * LDT + (e & 63)];
    // ---- panel list
    int np = 0;
    if (!dphase) {
      const int imax = min(K + sb.wb, sb.nt1 - 1);
      for (int I = K + 1; I <= imax; ++I) {
        if (tid == 0) plist[np] = (short)(I - K);
        ++np;
      }
      for (int Ib = 0; Ib < sb.ntb; ++Ib)
        if (bfirst[Ib] <= K) {
          if (tid == 0) plist[np] = (short)(4096 + Ib);
          ++np;
        }
    } else {
      for (int Ib = Kd + 1; Ib < sb.ntb; ++Ib) {
        if (tid == 0) plist[np] = (short)(4096 + Ib);
        ++np;
      }
    }
    __syncthreads();
    auto ptile = [&](int p) -> double* {
      const int code = plist[p];
      if (code < 4096) return band_tile(sb, band, K + code, K);
      const int Ib = code - 4096;
      return dphase ? dense_tile(sb, dense, Ib, Kd) : border_tile(sb, scratch, Ib, K);
    };
    // ---- panel solve: T <- T inv(L_KK)^T
    for (int p = 0; p < np; ++p) {
      double* Tg = ptile(p);
      cp_block(As, LDT, Tg, 64, 64, 64);
      cp_commit();
      cp_wait<0>();
      __syncthreads();
      double acc[2][4][2];
      acc_zero(acc);
      cta_mma<4, false, true>(As, LDT, Li, LDT, acc);
#pragma unroll
      for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int r = acc_row<4>(i), c = acc_col<4>(j);
          *reinterpret_cast<double2*>(Tg + r * 64 + c) = make_double2(acc[i][j][0], acc[i][j][1]);
        }
      __syncthreads();
    }
    __threadfence();
    __syncthreads();
    // ---- trailing update: dest(a, b) -= P_a P_b^T, a >= b
    for (int a = 0; a < np; ++a) {
      const int ca = plist[a];
      cp_block(As, LDT, ptile(a), 64, 64, 64);
      cp_block(Bs0, LDT, ptile(0), 64, 64, 64);
      cp_commit();
      for (int b = 0; b <= a; ++b) {
        double* Bcur = (b & 1) ? Bs1 : Bs0;
        if (b + 1 <= a) {
          cp_block((b & 1) ? Bs0 : Bs1, LDT, ptile(b + 1), 64, 64, 64);
          cp_commit();
          cp_wait<1>();
        } else {
          cp_wait<0>();
        }
        __syncthreads();
        // destination tile
        const int cb = plist[b];
        double* dst;
        if (ca < 4096) {                        // band x band
          dst = band_tile(sb, band, K + ca, K + cb);
        } else if (!dphase && cb < 4096) {      // border x band
          dst = border_tile(sb, scratch, ca - 4096, K + cb);
        } else if (!dphase) {                   // border x border -> dense (S22)
          dst = dense_tile(sb, dense, ca - 4096, cb - 4096);
        } else {
          dst = dense_tile(sb, dense, ca - 4096, cb - 4096);
        }
        double acc[2][4][2];
        acc_zero(acc);
        cta_mma<4, false, true>(As, LDT, Bcur, LDT, acc);
#pragma unroll
        for (int i = 0; i < 2; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const int r = acc_row<4>(i), c = acc_col<4>(j);
            double2* q = reinterpret_cast<double2*>(dst + r * 64 + c);
            double2 v = *q;
            v.x -= acc[i][j][0];
            v.y -= acc[i][j][1];
            *q = v;
          }
        __syncthreads();
      }
    }
    __threadfence();
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------------------------
// a1 / a4 / a5: CSR SpMM on row-major s-wide fp64 blocks.  Warp per row; the row's column
// indices and values are loaded once lane-parallel and broadcast by shuffle (register staging);
// each lane owns columns lane, lane+32, ... so every X-row read is a coalesced 8s-byte segment.
// ---------------------------------------------------------------------------------------------
// Column c of a row lives at row * ld + (c / 32) * cs + c % 32: cs = 32 for row-major blocks, cs = rows * 36
// for the chunk-major padded W/V/U layout (each 64 x 32 tile contiguous: one bulk copy in k_symm).
template <int NQ>
__global__ void __launch_bounds__(256) k_spmm(int64_t rows, const int32_t* __restrict__ rp,
                                              const int32_t* __restrict__ ci, const double* __restrict__ va,
                                              const double* __restrict__ X, int ldx,
                                              const double* __restrict__ U, int ldu, int64_t ucs, int64_t split,
                                              double* __restrict__ Y, int ldy, int64_t ycs, int ypad, int s, int mode,
                                              int zero_pad) {
  pdl_wait();
  const int64_t row = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (row >= rows) return;
  const int beg = rp[row], end = rp[row + 1];
  double acc[NQ];
#pragma unroll
  for (int q = 0; q < NQ; ++q) acc[q] = 0.0;
  for (int base = beg; base < end; base += 32) {
    const int k = base + lane;
    const int c = k < end ? ci[k] : 0;
    const double v = k < end ? va[k] : 0.0;
    const int cnt = min(32, end - base);
    for (int q = 0; q < cnt; ++q) {
      const int64_t col = __shfl_sync(0xffffffffu, c, q);
      double a = __shfl_sync(0xffffffffu, v, q);
      const double* src;
      if (mode == 0 || mode == 4 || col < split) {
        if (mode == 2) continue;
        src = X + col * ldx;
      } else {
        if (mode == 3) continue;
        src = U + (col - split) * ldu;
        if (mode == 2) a = -a;
      }
      const int64_t cs = (mode == 0 || mode == 4 || col < split) ? 32 : ucs;
#pragma unroll
      for (int qq = 0; qq < NQ; ++qq) {
        const int cc = lane + 32 * qq;
        if (cc < s) acc[qq] = fma(a, __ldg(src + qq * cs + lane), acc[qq]);
      }
    }
  }
  double* y = Y + row * ldy;
#pragma unroll
  for (int qq = 0; qq < NQ; ++qq) {
    const int cc = lane + 32 * qq;
    double* yc = y + qq * ycs + lane;
    if (cc < s) *yc = mode == 4 ? *yc + acc[qq] : acc[qq];
    else if (zero_pad && cc < ypad) *yc = 0.0;
  }
  if (zero_pad)
    for (int cc = 32 * NQ + lane; cc < ypad; cc += 32) y[(cc >> 5) * ycs + (cc & 31)] = 0.0;
}

// The same SpMM with 16-byte (double2) loads: lane l owns the column pairs (2l, 2l+1) + 64q, so one
// warp instruction moves a 512-byte row segment and an s = 128 row takes two loads per nonzero instead
// of four.  At most 32 registers (8 CTAs of 256 threads per SM: full occupancy hides the dependent
// row-pointer -> index -> row-load chain).  Requires even s and even leading dimensions / chunk strides
// (16-byte aligned rows).
// OZ (a1 feeding the INT8 a2+a3, reading R10): the CTA's 8 rows lie in one 64-row W/V/U tile (rows is a
// multiple of 64), so the per-(block, column) scale exponents of the W^T slices are reduced over the 8 rows in
// shared memory and folded into ozse[block * 128 * nct + c] by integer atomicMax (order-independent); ozdx:
// delta exponent per row, oztb: block of each tile.
template <int NQ2, bool OZ = false>
__global__ void __launch_bounds__(256, NQ2 <= 2 ? 8 : 4) k_spmm2(int64_t rows, const int32_t* __restrict__ rp,
                                               const int32_t* __restrict__ ci, const double* __restrict__ va,
                                               const double* __restrict__ X, int ldx,
                                               const double* __restrict__ U, int ldu, int64_t ucs, int64_t split,
                                               double* __restrict__ Y, int ldy, int64_t ycs, int ypad, int s, int mode,
                                               int zero_pad, const int* __restrict__ ozdx = nullptr,
                                               const int* __restrict__ oztb = nullptr, int* __restrict__ ozse = nullptr,
                                               int ozn = 0) {
  pdl_wait();
  const int64_t row = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (!OZ && row >= rows) return;
  const int beg = rp[row], end = rp[row + 1];
  double2 acc[NQ2];
#pragma unroll
  for (int q = 0; q < NQ2; ++q) acc[q] = make_double2(0.0, 0.0);
  // element offset of column pair (2 lane + 64 q) in a layout with 32-column chunks of stride cs
  auto off = [&](int q, int64_t cs) -> int64_t {
    const int c = 2 * lane + 64 * q;
    return (int64_t)(c >> 5) * cs + (c & 31);
  };
  auto src_of = [&](int64_t col, double& a, int64_t& cs) -> const double* {
    if (mode == 0 || mode == 4 || col < split) {
      if (mode == 2) return nullptr;
      cs = 32;
      return X + col * ldx;
    }
    if (mode == 3) return nullptr;
    if (mode == 2) a = -a;
    cs = ucs;
    return U + (col - split) * ldu;
  };
  for (int base = beg; base < end; base += 32) {
    const int k = base + lane;
    const int c = k < end ? ci[k] : 0;
    const double v = k < end ? va[k] : 0.0;
    const int cnt = min(32, end - base);
    for (int q = 0; q < cnt; ++q) {
      const int64_t c0 = __shfl_sync(0xffffffffu, c, q);
      double a0 = __shfl_sync(0xffffffffu, v, q);
      int64_t cs0 = 32;
      const double* s0 = src_of(c0, a0, cs0);
      if (s0) {
#pragma unroll
        for (int qq = 0; qq < NQ2; ++qq) {
          if (2 * lane + 64 * qq < s) {
            const double2 x0 = __ldg(reinterpret_cast<const double2*>(s0 + off(qq, cs0)));
            acc[qq].x = fma(a0, x0.x, acc[qq].x);
            acc[qq].y = fma(a0, x0.y, acc[qq].y);
          }
        }
      }
    }
  }
  double* y = Y + row * ldy;
#pragma unroll
  for (int qq = 0; qq < NQ2; ++qq) {
    const int cc = 2 * lane + 64 * qq;
    double2* yc = reinterpret_cast<double2*>(y + off(qq, ycs));
    if (cc < s) {
      if (mode == 4) {
        const double2 o = *yc;
        *yc = make_double2(o.x + acc[qq].x, o.y + acc[qq].y);
      } else {
        *yc = acc[qq];
      }
    } else if (zero_pad && cc < ypad) {
      *yc = make_double2(0.0, 0.0);
    }
  }
  if (zero_pad)
    for (int cc = 64 * NQ2 + 2 * lane; cc < ypad; cc += 64)
      *reinterpret_cast<double2*>(y + (int64_t)(cc >> 5) * ycs + (cc & 31)) = make_double2(0.0, 0.0);
  if constexpr (OZ) {
    __shared__ int ex[8][64 * NQ2];
    const int w = threadIdx.x >> 5, d = ozdx[row];
    auto ex_of = [&](double v) {
      const double a = fabs(ldexp(v, d));
      int e;
      frexp(a, &e);
      return a > 0.0 ? e + 1 : INT_MIN / 2;   // |v delta| / 2^e < 1/2
    };
#pragma unroll
    for (int qq = 0; qq < NQ2; ++qq) {
      const int cc = 2 * lane + 64 * qq;
      ex[w][cc] = cc < s ? ex_of(acc[qq].x) : INT_MIN / 2;
      ex[w][cc + 1] = cc + 1 < s ? ex_of(acc[qq].y) : INT_MIN / 2;
    }
    __syncthreads();
    const int64_t blk = oztb[(row - w) / 64];
    for (int c = threadIdx.x; c < s; c += 256) {
      int m = ex[0][c];
#pragma unroll
      for (int r = 1; r < 8; ++r) m = max(m, ex[r][c]);
      if (m > INT_MIN / 2) atomicMax(&ozse[blk * ozn + c], m);
    }
  }
}

// One step of the fixed Chebyshev iteration for A_G^{-1} (reading R7; one rank) fused with its sparse
// product: per row, t = (A_G d)[row] over the A_G prefix of the AGG2 row (cols < split), then the
// elementwise update x += d, r -= t, d' = c1 d + c2 r of the same row - one pass instead of an SpMM that
// writes t and an update that reads it back.  Same summation order as k_spmv / k_spmm2 + k_cheb_update
// (bitwise the same iterate).  s = 1: G lanes per row; s > 1: a warp per row, column pairs per lane.
template <int G>
__global__ void __launch_bounds__(256) k_cheb_step_vec(int64_t rows, const int32_t* __restrict__ rp,
                                                       const int32_t* __restrict__ ci, const double* __restrict__ va,
                                                       int64_t split, const double* __restrict__ d,
                                                       double* __restrict__ x, double* __restrict__ r,
                                                       double* __restrict__ dn, double c1, double c2, int want_d) {
  pdl_wait();
  const int64_t row = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) / G;
  const int sub = threadIdx.x & (G - 1);
  double acc = 0.0;
  if (row < rows) {
    const int beg = rp[row], end = rp[row + 1];
    for (int k = beg + sub; k < end; k += G) {
      const int64_t col = ci[k];
      if (col < split) acc = fma(va[k], __ldg(d + col), acc);
    }
  }
#pragma unroll
  for (int o = G / 2; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if (row >= rows || sub != 0) return;
  const double di = d[row];
  x[row] += di;
  const double ri = r[row] - acc;
  r[row] = ri;
  if (want_d) dn[row] = fma(c1, di, c2 * ri);
}

// s = 1 on the sliced-ELL copy of A_G: one thread per row, the slice's entries column-major (coalesced
// 32-row segments), no row-pointer hop before the index loads: the dependent chain is index -> d gather.
__global__ void __launch_bounds__(256) k_cheb_step_sell(int64_t rows, const int64_t* __restrict__ sptr,
                                                        const int32_t* __restrict__ col, const double* __restrict__ val,
                                                        const double* __restrict__ d, double* __restrict__ x,
                                                        double* __restrict__ r, double* __restrict__ dn, double c1,
                                                        double c2, int want_d) {
  pdl_wait();
  const int64_t row = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (row >= rows) return;
  const int64_t sl = row >> 5;
  const int lane = (int)(row & 31);
  const int64_t b = sptr[sl];
  const int w = (int)((sptr[sl + 1] - b) >> 5);
  double acc = 0.0;
#pragma unroll 4
  for (int j = 0; j < w; ++j) {
    const int c = col[b + j * 32 + lane];
    if (c >= 0) acc = fma(val[b + j * 32 + lane], __ldg(d + c), acc);
  }
  const double di = d[row];
  x[row] += di;
  const double ri = r[row] - acc;
  r[row] = ri;
  if (want_d) dn[row] = fma(c1, di, c2 * ri);
}

// The same step with A_G's values dictionary-coded (one byte per entry into a table of the <= 255 distinct
// values, built in setup when A_G has that few - every constant-coefficient stencil): 5 instead of 12 bytes
// per stored entry, the values bitwise the same.
__global__ void __launch_bounds__(256) k_cheb_step_sell_dict(int64_t rows, const int64_t* __restrict__ sptr,
                                                             const int32_t* __restrict__ col,
                                                             const uint8_t* __restrict__ code,
                                                             const double* __restrict__ tab,
                                                             const double* __restrict__ d, double* __restrict__ x,
                                                             double* __restrict__ r, double* __restrict__ dn,
                                                             double c1, double c2, int want_d) {
  __shared__ double st[256];
  st[threadIdx.x] = tab[threadIdx.x];
  pdl_wait();
  __syncthreads();
  const int64_t row = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (row >= rows) return;
  const int64_t sl = row >> 5;
  const int lane = (int)(row & 31);
  const int64_t b = sptr[sl];
  const int w = (int)((sptr[sl + 1] - b) >> 5);
  double acc = 0.0;
#pragma unroll 4
  for (int j = 0; j < w; ++j) {
    const int c = col[b + j * 32 + lane];
    if (c >= 0) acc = fma(st[code[b + j * 32 + lane]], __ldg(d + c), acc);
  }
  const double di = d[row];
  x[row] += di;
  const double ri = r[row] - acc;
  r[row] = ri;
  if (want_d) dn[row] = fma(c1, di, c2 * ri);
}

// Three-term form of the same Chebyshev iteration (x only): with d_{k-1} = x_k - x_{k-1} and
// r_k = b - A x_k the step x_{k+1} = x_k + d_k, d_k = c1 d_{k-1} + c2 r_k becomes
//   x_{k+1} = x_k + c1 (x_k - x_{k-1}) + c2 (b - A x_k),
// the same polynomial in A with 4 instead of 6 block passes per step (reads x_k, x_{k-1}, b; writes x_{k+1}
// over x_{k-1}, which no other row reads).  xn may alias xp.
template <int NQ2>
__global__ void __launch_bounds__(256, NQ2 <= 2 ? 8 : 4) k_cheb3_step_blk(int64_t rows, const int32_t* __restrict__ rp,
                                                        const int32_t* __restrict__ ci, const double* __restrict__ va,
                                                        int64_t split, const double* __restrict__ xk, int ld,
                                                        const double* xp, const double* __restrict__ b,
                                                        double* xn, double c1, double c2) {
  pdl_wait();
  const int64_t row = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (row >= rows) return;
  const int beg = rp[row], end = rp[row + 1];
  double2 acc[NQ2];
#pragma unroll
  for (int q = 0; q < NQ2; ++q) acc[q] = make_double2(0.0, 0.0);
  for (int base = beg; base < end; base += 32) {
    const int k = base + lane;
    const int c = k < end ? ci[k] : 0;
    const double v = k < end ? va[k] : 0.0;
    const int cnt = min(32, end - base);
    for (int q = 0; q < cnt; ++q) {
      const int64_t col = __shfl_sync(0xffffffffu, c, q);
      const double a = __shfl_sync(0xffffffffu, v, q);
      if (col >= split) continue;
      const double* src = xk + col * ld;
#pragma unroll
      for (int qq = 0; qq < NQ2; ++qq) {
        const int cc = 2 * lane + 64 * qq;
        if (cc < ld) {
          const double2 dv = __ldg(reinterpret_cast<const double2*>(src + cc));
          acc[qq].x = fma(a, dv.x, acc[qq].x);
          acc[qq].y = fma(a, dv.y, acc[qq].y);
        }
      }
    }
  }
  const int64_t o = row * ld;
#pragma unroll
  for (int qq = 0; qq < NQ2; ++qq) {
    const int cc = 2 * lane + 64 * qq;
    if (cc >= ld) continue;
    const double2 xi = *reinterpret_cast<const double2*>(xk + o + cc);
    const double2 xo = *reinterpret_cast<const double2*>(xp + o + cc);
    const double2 bi = __ldg(reinterpret_cast<const double2*>(b + o + cc));
    double2 y;
    y.x = xi.x + fma(c1, xi.x - xo.x, c2 * (bi.x - acc[qq].x));
    y.y = xi.y + fma(c1, xi.y - xo.y, c2 * (bi.y - acc[qq].y));
    *reinterpret_cast<double2*>(xn + o + cc) = y;
  }
}

// s = 1, sliced ELL (values direct or dictionary-coded): one thread per row
__global__ void __launch_bounds__(256) k_cheb3_step_sell(int64_t rows, const int64_t* __restrict__ sptr,
                                                         const int32_t* __restrict__ col,
                                                         const double* __restrict__ val,
                                                         const uint8_t* __restrict__ code,
                                                         const double* __restrict__ tab,
                                                         const double* __restrict__ xk, const double* xp,
                                                         const double* __restrict__ b, double* xn, double c1,
                                                         double c2) {
  __shared__ double stab[256];
  if (code) stab[threadIdx.x] = tab[threadIdx.x];
  pdl_wait();
  __syncthreads();
  const int64_t row = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (row >= rows) return;
  const int64_t sl = row >> 5;
  const int lane = (int)(row & 31);
  const int64_t b0 = sptr[sl];
  const int w = (int)((sptr[sl + 1] - b0) >> 5);
  double acc = 0.0;
  if (code) {
#pragma unroll 4
    for (int j = 0; j < w; ++j) {
      const int c = col[b0 + j * 32 + lane];
      if (c >= 0) acc = fma(stab[code[b0 + j * 32 + lane]], __ldg(xk + c), acc);
    }
  } else {
#pragma unroll 4
    for (int j = 0; j < w; ++j) {
      const int c = col[b0 + j * 32 + lane];
      if (c >= 0) acc = fma(val[b0 + j * 32 + lane], __ldg(xk + c), acc);
    }
  }
  const double xi = xk[row];
  xn[row] = xi + fma(c1, xi - xp[row], c2 * (b[row] - acc));
}

template <int NQ2>
__global__ void __launch_bounds__(256, NQ2 <= 2 ? 8 : 4) k_cheb_step_blk(int64_t rows, const int32_t* __restrict__ rp,
                                                       const int32_t* __restrict__ ci, const double* __restrict__ va,
                                                       int64_t split, const double* __restrict__ d, int ld,
                                                       double* __restrict__ x, double* __restrict__ r,
                                                       double* __restrict__ dn, double c1, double c2, int want_d) {
  pdl_wait();
  const int64_t row = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (row >= rows) return;
  const int beg = rp[row], end = rp[row + 1];
  double2 acc[NQ2];
#pragma unroll
  for (int q = 0; q < NQ2; ++q) acc[q] = make_double2(0.0, 0.0);
  for (int base = beg; base < end; base += 32) {
    const int k = base + lane;
    const int c = k < end ? ci[k] : 0;
    const double v = k < end ? va[k] : 0.0;
    const int cnt = min(32, end - base);
    for (int q = 0; q < cnt; ++q) {
      const int64_t col = __shfl_sync(0xffffffffu, c, q);
      const double a = __shfl_sync(0xffffffffu, v, q);
      if (col >= split) continue;
      const double* src = d + col * ld;
#pragma unroll
      for (int qq = 0; qq < NQ2; ++qq) {
        const int cc = 2 * lane + 64 * qq;
        if (cc < ld) {
          const double2 dv = __ldg(reinterpret_cast<const double2*>(src + cc));
          acc[qq].x = fma(a, dv.x, acc[qq].x);
          acc[qq].y = fma(a, dv.y, acc[qq].y);
        }
      }
    }
  }
  const int64_t o = row * ld;
#pragma unroll
  for (int qq = 0; qq < NQ2; ++qq) {
    const int cc = 2 * lane + 64 * qq;
    if (cc >= ld) continue;
    const double2 di = *reinterpret_cast<const double2*>(d + o + cc);
    double2 xi = *reinterpret_cast<const double2*>(x + o + cc);
    double2 ri = *reinterpret_cast<const double2*>(r + o + cc);
    xi.x += di.x;
    xi.y += di.y;
    ri.x = ri.x - acc[qq].x;
    ri.y = ri.y - acc[qq].y;
    *reinterpret_cast<double2*>(x + o + cc) = xi;
    *reinterpret_cast<double2*>(r + o + cc) = ri;
    if (want_d) *reinterpret_cast<double2*>(dn + o + cc) = make_double2(fma(c1, di.x, c2 * ri.x), fma(c1, di.y, c2 * ri.y));
  }
}

// One right-hand side (s = 1): the same modes as k_spmm, G lanes per row (several rows per warp),
// the lanes take the row's nonzeros in parallel (independent gathers of x) and combine them with a
// G-lane butterfly (fixed order).  k_spmm's lane-over-columns layout would leave 31 of 32 lanes idle
// and serialise one dependent gather per nonzero.
template <int G>
__global__ void __launch_bounds__(256) k_spmv(int64_t rows, const int32_t* __restrict__ rp,
                                              const int32_t* __restrict__ ci, const double* __restrict__ va,
                                              const double* __restrict__ X, int ldx,
                                              const double* __restrict__ U, int ldu, int64_t split,
                                              double* __restrict__ Y, int ldy, int mode, int zero_pad) {
  pdl_wait();
  const int64_t row = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) / G;
  const int sub = threadIdx.x & (G - 1);
  double acc = 0.0;
  if (row < rows) {
    const int beg = rp[row], end = rp[row + 1];
    for (int k = beg + sub; k < end; k += G) {
      const int64_t col = ci[k];
      double a = va[k];
      if (mode == 0 || mode == 4 || col < split) {
        if (mode == 2) continue;
        acc = fma(a, __ldg(X + col * ldx), acc);
      } else {
        if (mode == 3) continue;
        if (mode == 2) a = -a;
        acc = fma(a, __ldg(U + (col - split) * ldu), acc);
      }
    }
  }
#pragma unroll
  for (int o = G / 2; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if (row >= rows) return;
  double* y = Y + row * ldy;
  if (sub == 0) y[0] = mode == 4 ? y[0] + acc : acc;
  if (zero_pad)
    for (int cc = 1 + sub; cc < ldy; cc += G) y[cc] = 0.0;
}

// ---------------------------------------------------------------------------------------------
// a2 + a3: batched forward and backward triangular solves with the boundary-layer factor
// L22_j of every block, all blocks (x column chunks) in one launch.  Blocked by 64-row tiles
// ("levels"): V_I = inv(L_II) (W_I - sum_{J<I} L_IJ V_J);  U_I = inv(L_II)^T (V_I - sum_{J>I}
// L_JI^T U_J).  In place in the W/V/U buffer.  (L_II^{-1} precomputed by the setup.)
// ---------------------------------------------------------------------------------------------
template <int CW>
__global__ void __launch_bounds__(256) k_trsm_fb(const FacSub* __restrict__ subs,
                                                 const double* __restrict__ dense, double* wvu, int ldw) {
  constexpr int NF = CW / 16;
  constexpr int LDV = CW + 4;
  extern __shared__ double sm[];
  double* Ls0 = sm;
  double* Ls1 = sm + 64 * LDT;
  double* Vs0 = sm + 2 * 64 * LDT;
  double* Vs1 = Vs0 + 64 * LDV;
  const FacSub sb = subs[blockIdx.x];
  const int ntb = sb.ntb;
  if (ntb == 0) return;
  const int c0 = blockIdx.y * CW;
  const double* T = dense + sb.dense_off * NSP_TILE_ELEMS;
  double* Wb = wvu + sb.wvu_row * (int64_t)ldw + c0;
  auto tile = [&](int I, int J) { return T + ((int64_t)I * (I + 1) / 2 + J) * NSP_TILE_ELEMS; };
  double acc[2][NF][2];

  // ------------------------- forward sweep
  for (int I = 0; I < ntb; ++I) {
    acc_zero(acc);
    if (I > 0) {
      cp_block(Ls0, LDT, tile(I, 0), 64, 64, 64);
      cp_block(Vs0, LDV, Wb, ldw, 64, CW);
      cp_commit();
      for (int J = 0; J < I; ++J) {
        double* Lc = (J & 1) ? Ls1 : Ls0;
        double* Vc = (J & 1) ? Vs1 : Vs0;
        if (J + 1 < I) {
          cp_block((J & 1) ? Ls0 : Ls1, LDT, tile(I, J + 1), 64, 64, 64);
          cp_block((J & 1) ? Vs0 : Vs1, LDV, Wb + (int64_t)(J + 1) * 64 * ldw, ldw, 64, CW);
          cp_commit();
          cp_wait<1>();
        } else {
          cp_wait<0>();
        }
        __syncthreads();
        cta_mma<NF, false, false>(Lc, LDT, Vc, LDV, acc);
        __syncthreads();
      }
    }
    // residual R = W_I - acc (in Vs1), then V_I = inv(L_II) R
    cp_block(Ls0, LDT, tile(I, I), 64, 64, 64);
    cp_block(Vs0, LDV, Wb + (int64_t)I * 64 * ldw, ldw, 64, CW);
    cp_commit();
    cp_wait<0>();
    __syncthreads();
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
      for (int j = 0; j < NF; ++j) {
        const int r = acc_row<NF>(i), c = acc_col<NF>(j);
        Vs1[r * LDV + c] = Vs0[r * LDV + c] - acc[i][j][0];
        Vs1[r * LDV + c + 1] = Vs0[r * LDV + c + 1] - acc[i][j][1];
      }
    __syncthreads();
    acc_zero(acc);
    cta_mma<NF, false, false>(Ls0, LDT, Vs1, LDV, acc);
    double* out = Wb + (int64_t)I * 64 * ldw;
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
      for (int j = 0; j < NF; ++j) {
        const int r = acc_row<NF>(i), c = acc_col<NF>(j);
        *reinterpret_cast<double2*>(out + (int64_t)r * ldw + c) = make_double2(acc[i][j][0], acc[i][j][1]);
      }
    __threadfence();
    __syncthreads();
  }
  // ------------------------- backward sweep
  for (int I = ntb - 1; I >= 0; --I) {
    acc_zero(acc);
    if (I < ntb - 1) {
      cp_block(Ls0, LDT, tile(I + 1, I), 64, 64, 64);
      cp_block(Vs0, LDV, Wb + (int64_t)(I + 1) * 64 * ldw, ldw, 64, CW);
      cp_commit();
      int it = 0;
      for (int J = I + 1; J < ntb; ++J, ++it) {
        double* Lc = (it & 1) ? Ls1 : Ls0;
        double* Vc = (it & 1) ? Vs1 : Vs0;
        if (J + 1 < ntb) {
          cp_block((it & 1) ? Ls0 : Ls1, LDT, tile(J + 1, I), 64, 64, 64);
          cp_block((it & 1) ? Vs0 : Vs1, LDV, Wb + (int64_t)(J + 1) * 64 * ldw, ldw, 64, CW);
          cp_commit();
          cp_wait<1>();
        } else {
          cp_wait<0>();
        }
        __syncthreads();
        cta_mma<NF, true, false>(Lc, LDT, Vc, LDV, acc);
        __syncthreads();
      }
    }
    cp_block(Ls0, LDT, tile(I, I), 64, 64, 64);
    cp_block(Vs0, LDV, Wb + (int64_t)I * 64 * ldw, ldw, 64, CW);
    cp_commit();
    cp_wait<0>();
    __syncthreads();
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
      for (int j = 0; j < NF; ++j) {
        const int r = acc_row<NF>(i), c = acc_col<NF>(j);
        Vs1[r * LDV + c] = Vs0[r * LDV + c] - acc[i][j][0];
        Vs1[r * LDV + c + 1] = Vs0[r * LDV + c + 1] - acc[i][j][1];
      }
    __syncthreads();
    acc_zero(acc);
    cta_mma<NF, true, false>(Ls0, LDT, Vs1, LDV, acc);
    double* out = Wb + (int64_t)I * 64 * ldw;
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
      for (int j = 0; j < NF; ++j) {
        const int r = acc_row<NF>(i), c = acc_col<NF>(j);
        *reinterpret_cast<double2*>(out + (int64_t)r * ldw + c) = make_double2(acc[i][j][0], acc[i][j][1]);
      }
    __threadfence();
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------------------------
// s0 (setup, after the factorisation): explicit M_j = S_j^{-1} = L22^{-T} L22^{-1} of every block's
// boundary-layer Schur complement, lower tiles in the L22 tile layout (diagonal tiles full).
// One CTA per (block, tile column C): tile column C of M = L^{-T} L^{-1} E_C computed in place in
// M's own tile column (forward sweep from tile row C, backward sweep down to C).
// ---------------------------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_l22_inverse(const FacSub* __restrict__ subs, const double* __restrict__ dense,
                                                     double* minv) {
  constexpr int NF = 4;
  constexpr int LDV = 68;
  extern __shared__ double sm[];
  double* Ls0 = sm;
  double* Ls1 = sm + 64 * LDT;
  double* Vs0 = sm + 2 * 64 * LDT;
  double* Vs1 = Vs0 + 64 * LDV;
  const FacSub sb = subs[blockIdx.x];
  const int ntb = sb.ntb, C = blockIdx.y;
  if (C >= ntb) return;
  const double* T = dense + sb.dense_off * NSP_TILE_ELEMS;
  double* Mb = minv + sb.dense_off * NSP_MINV_TILE;
  auto tile = [&](int I, int J) { return T + ((int64_t)I * (I + 1) / 2 + J) * NSP_TILE_ELEMS; };
  auto vt = [&](int I) { return Mb + ((int64_t)I * (I + 1) / 2 + C) * NSP_MINV_TILE; };   // row tile I of the RHS
  for (int I = C; I < ntb; ++I)
    for (int e = threadIdx.x; e < 4096; e += 256)
      vt(I)[(e >> 6) * NSP_MINV_LD + (e & 63)] = (I == C && (e >> 6) == (e & 63)) ? 1.0 : 0.0;
  __threadfence_block();
  __syncthreads();
  double acc[2][NF][2];
  for (int I = C; I < ntb; ++I) {   // forward: V_I = inv(L_II) (E_I - sum_{C<=J<I} L_IJ V_J)
    acc_zero(acc);
    if (I > C) {
      cp_block(Ls0, LDT, tile(I, C), 64, 64, 64);
      cp_block(Vs0, LDV, vt(C), NSP_MINV_LD, 64, 64);
      cp_commit();
      for (int J = C, it = 0; J < I; ++J, ++it) {
        double* Lc = (it & 1) ? Ls1 : Ls0;
        double* Vc = (it & 1) ? Vs1 : Vs0;
        if (J + 1 < I) {
          cp_block((it & 1) ? Ls0 : Ls1, LDT, tile(I, J + 1), 64, 64, 64);
          cp_block((it & 1) ? Vs0 : Vs1, LDV, vt(J + 1), NSP_MINV_LD, 64, 64);
          cp_commit();
          cp_wait<1>();
        } else {
          cp_wait<0>();
        }
        __syncthreads();
        cta_mma<NF, false, false>(Lc, LDT, Vc, LDV, acc);
        __syncthreads();
      }
    }
    cp_block(Ls0, LDT, tile(I, I), 64, 64, 64);
    cp_block(Vs0, LDV, vt(I), NSP_MINV_LD, 64, 64);
    cp_commit();
    cp_wait<0>();
    __syncthreads();
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
      for (int j = 0; j < NF; ++j) {
        const int r = acc_row<NF>(i), c = acc_col<NF>(j);
        Vs1[r * LDV + c] = Vs0[r * LDV + c] - acc[i][j][0];
        Vs1[r * LDV + c + 1] = Vs0[r * LDV + c + 1] - acc[i][j][1];
      }
    __syncthreads();
    acc_zero(acc);
    cta_mma<NF, false, false>(Ls0, LDT, Vs1, LDV, acc);
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
      for (int j = 0; j < NF; ++j) {
        const int r = acc_row<NF>(i), c = acc_col<NF>(j);
        *reinterpret_cast<double2*>(vt(I) + r * NSP_MINV_LD + c) = make_double2(acc[i][j][0], acc[i][j][1]);
      }
    __threadfence_block();
    __syncthreads();
  }
  for (int I = ntb - 1; I >= C; --I) {   // backward: U_I = inv(L_II)^T (V_I - sum_{J>I} L_JI^T U_J)
    acc_zero(acc);
    if (I < ntb - 1) {
      cp_block(Ls0, LDT, tile(I + 1, I), 64, 64, 64);
      cp_block(Vs0, LDV, vt(I + 1), NSP_MINV_LD, 64, 64);
      cp_commit();
      int it = 0;
      for (int J = I + 1; J < ntb; ++J, ++it) {
        double* Lc = (it & 1) ? Ls1 : Ls0;
        double* Vc = (it & 1) ? Vs1 : Vs0;
        if (J + 1 < ntb) {
          cp_block((it & 1) ? Ls0 : Ls1, LDT, tile(J + 1, I), 64, 64, 64);
          cp_block((it & 1) ? Vs0 : Vs1, LDV, vt(J + 1), NSP_MINV_LD, 64, 64);
          cp_commit();
          cp_wait<1>();
        } else {
          cp_wait<0>();
        }
        __syncthreads();
        cta_mma<NF, true, false>(Lc, LDT, Vc, LDV, acc);
        __syncthreads();
      }
    }
    cp_block(Ls0, LDT, tile(I, I), 64, 64, 64);
    cp_block(Vs0, LDV, vt(I), NSP_MINV_LD, 64, 64);
    cp_commit();
    cp_wait<0>();
    __syncthreads();
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
      for (int j = 0; j < NF; ++j) {
        const int r = acc_row<NF>(i), c = acc_col<NF>(j);
        Vs1[r * LDV + c] = Vs0[r * LDV + c] - acc[i][j][0];
        Vs1[r * LDV + c + 1] = Vs0[r * LDV + c + 1] - acc[i][j][1];
      }
    __syncthreads();
    acc_zero(acc);
    cta_mma<NF, true, false>(Ls0, LDT, Vs1, LDV, acc);
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
      for (int j = 0; j < NF; ++j) {
        const int r = acc_row<NF>(i), c = acc_col<NF>(j);
        *reinterpret_cast<double2*>(vt(I) + r * NSP_MINV_LD + c) = make_double2(acc[i][j][0], acc[i][j][1]);
      }
    __threadfence_block();
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------------------------
// a2 + a3 as ONE symmetric product per block: U_j = M_j W_j, M_j = S_j^{-1} (= L22^{-T} L22^{-1}
// W_j, the two triangular sweeps of north_star (b) with the factor's inverse precomputed in the
// setup).  No dependency chain: one CTA per (block, output tile row I, column chunk) computes
// U_I = sum_{J<=I} M_IJ W_J + sum_{J>I} M_JI^T W_J from the stored lower tiles (each stored tile
// serves two output rows; they meet in L2).  Same flops as the sweeps, half the factor bytes.
// items[x] = (block, I); W, U: W/V/U-layout buffers (ld ldw), out of place.
// ---------------------------------------------------------------------------------------------
template <int CW, bool CM>
__global__ void __launch_bounds__(256) k_symm(const FacSub* __restrict__ subs, const int2* __restrict__ items,
                                              const double* __restrict__ minv, const double* __restrict__ W,
                                              double* __restrict__ U, int ldw, int64_t cs) {
  // CM (chunk-major padded W/U, ldw = CW + 4, cs = chunk stride): the W tile of a stage is contiguous too,
  // so both operands arrive by bulk copy (TMA) on one mbarrier; otherwise W by cp.async
  constexpr int NF = CW / 16;
  constexpr int LDV = CW + 4;
  constexpr int STAGE = NSP_MINV_TILE + 64 * LDV;   // one (M tile, W tile) pair
  extern __shared__ __align__(128) double sm[];
  __shared__ __align__(8) uint64_t bar[2];
  // CM: grid (chunks, items) - the chunk CTAs of one item are adjacent in launch order, so they read
  // each S_j^{-1} tile from L2 within the same wave
  const int bx = CM ? blockIdx.y : blockIdx.x, by = CM ? blockIdx.x : blockIdx.y;
  const int2 it = items[bx];
  const FacSub sb = subs[it.x];
  const int I = it.y, ntb = sb.ntb;
  const int c0 = by * CW;
  const double* Mb = minv + sb.dense_off * NSP_MINV_TILE;
  const double* Wb = CM ? W + by * cs + sb.wvu_row * (int64_t)LDV : W + sb.wvu_row * (int64_t)ldw + c0;
  auto mt = [&](int J) {   // stored tile holding block (I, J) (transposed when J > I)
    return J <= I ? Mb + ((int64_t)I * (I + 1) / 2 + J) * NSP_MINV_TILE
                  : Mb + ((int64_t)J * (J + 1) / 2 + I) * NSP_MINV_TILE;
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
      // the stage's full byte count is expected (arrive.expect_tx) BEFORE any of its copies is issued,
      // so the phase cannot complete on a partial byte count
      mbar_expect(&bar[J & 1], NSP_MINV_TILE * 8 + (CM ? 64 * LDV * 8 : 0));
      bulk_copy(Ms, mt(J), NSP_MINV_TILE * 8, &bar[J & 1]);
      if (CM) bulk_copy(Ms + NSP_MINV_TILE, Wb + (int64_t)J * 64 * LDV, 64 * LDV * 8, &bar[J & 1]);
    }
    if (!CM) cp_block(Ms + NSP_MINV_TILE, LDV, Wb + (int64_t)J * 64 * ldw, ldw, 64, CW);
  };
  double acc[2][NF][2];
  acc_zero(acc);
  // the S_j^{-1} tiles are constant: stage 0's M tile is requested BEFORE waiting for the producer of
  // W (programmatic dependent launch), so its latency hides behind the previous kernel's tail
  // (stage 0 expects M and W bytes up front: the W copy issued after pdl_wait() only completes it)
  if (threadIdx.x == 0) {
    mbar_expect(&bar[0], NSP_MINV_TILE * 8 + (CM ? 64 * LDV * 8 : 0));
    bulk_copy(sm, mt(0), NSP_MINV_TILE * 8, &bar[0]);
  }
  pdl_wait();
  if (CM) {
    if (threadIdx.x == 0) bulk_copy(sm + NSP_MINV_TILE, Wb, 64 * LDV * 8, &bar[0]);
  } else {
    cp_block(sm + NSP_MINV_TILE, LDV, Wb, ldw, 64, CW);
  }
  cp_commit();
  for (int J = 0; J < ntb; ++J) {
    if (!CM) cp_wait<0>();
    mbar_wait(&bar[J & 1], (J >> 1) & 1);
    __syncthreads();   // stage J complete for every thread; stage J + 1 free (its last reader was J - 1)
    if (J + 1 < ntb) issue(J + 1);
    if (!CM) cp_commit();
    const double* Ms = sm + (J & 1) * STAGE;
    if (J <= I) cta_mma<NF, false, false>(Ms, NSP_MINV_LD, Ms + NSP_MINV_TILE, LDV, acc);
    else cta_mma<NF, true, false>(Ms, NSP_MINV_LD, Ms + NSP_MINV_TILE, LDV, acc);
  }
  double* out = CM ? U + by * cs + (sb.wvu_row + (int64_t)I * 64) * LDV
                   : U + (sb.wvu_row + (int64_t)I * 64) * ldw + c0;
  const int ldo = CM ? LDV : ldw;
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < NF; ++j) {
      const int r = acc_row<NF>(i), c = acc_col<NF>(j);
      *reinterpret_cast<double2*>(out + (int64_t)r * ldo + c) = make_double2(acc[i][j][0], acc[i][j][1]);
    }
}

// Persistent form of k_symm (chunk-major W/U): 2 CTAs per SM walk the work units u = item * nch + chunk
// (chunk fastest, so the chunk CTAs of one item still share each S_j^{-1} tile through L2) with ONE
// 2-stage TMA ring that runs across unit boundaries - the first stage of the next unit is in flight while
// the current one finishes its last product and writes its U tile, instead of every CTA paying its own
// prologue and epilogue.
template <int CW>
__global__ void __launch_bounds__(256, 2) k_symm_p(const FacSub* __restrict__ subs, const int2* __restrict__ items,
                                                   int nitems, int nch, const double* __restrict__ minv,
                                                   const double* __restrict__ W, double* __restrict__ U, int64_t cs) {
  constexpr int NF = CW / 16;
  constexpr int LDV = CW + 4;
  constexpr int STAGE = NSP_MINV_TILE + 64 * LDV;
  extern __shared__ __align__(128) double sm[];
  __shared__ __align__(8) uint64_t bar[2];
  const int64_t total = (int64_t)nitems * nch;
  struct Unit {
    const double* Mb;
    const double* Wb;
    double* out;
    int I, ntb;
  };
  auto unit = [&](int64_t u) {
    const int2 it = items[u / nch];
    const int by = (int)(u % nch);
    const FacSub sb = subs[it.x];
    Unit r;
    r.Mb = minv + sb.dense_off * NSP_MINV_TILE;
    r.Wb = W + by * cs + sb.wvu_row * (int64_t)LDV;
    r.out = U + by * cs + (sb.wvu_row + (int64_t)it.y * 64) * LDV;
    r.I = it.y;
    r.ntb = sb.ntb;
    return r;
  };
  auto mt = [](const Unit& q, int J) {
    return J <= q.I ? q.Mb + ((int64_t)q.I * (q.I + 1) / 2 + J) * NSP_MINV_TILE
                    : q.Mb + ((int64_t)J * (J + 1) / 2 + q.I) * NSP_MINV_TILE;
  };
  if (threadIdx.x == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    fence_mbar_init();
  }
  __syncthreads();
  int64_t u = blockIdx.x;
  if (u >= total) {
    pdl_wait();
    return;
  }
  Unit cur = unit(u);
  // stage 0: the constant M tile before the programmatic-launch wait, W after it
  if (threadIdx.x == 0) {
    mbar_expect(&bar[0], NSP_MINV_TILE * 8 + 64 * LDV * 8);
    bulk_copy(sm, mt(cur, 0), NSP_MINV_TILE * 8, &bar[0]);
  }
  pdl_wait();
  if (threadIdx.x == 0) bulk_copy(sm + NSP_MINV_TILE, cur.Wb, 64 * LDV * 8, &bar[0]);
  double acc[2][NF][2];
  acc_zero(acc);
  unsigned g = 0;   // global step: stage g & 1, phase (g >> 1) & 1
  while (true) {
    const int64_t un = u + gridDim.x;
    const bool has_next = un < total;
    Unit nxt;
    if (has_next) nxt = unit(un);
    for (int J = 0; J < cur.ntb; ++J, ++g) {
      mbar_wait(&bar[g & 1], (g >> 1) & 1);
      __syncthreads();   // stage g complete for every thread; stage g + 1 free (its last reader was g - 1)
      if (threadIdx.x == 0) {
        const bool more = J + 1 < cur.ntb;
        if (more || has_next) {
          const Unit& q = more ? cur : nxt;
          const int Jn = more ? J + 1 : 0;
          double* Ms = sm + ((g + 1) & 1) * STAGE;
          fence_proxy_async();
          mbar_expect(&bar[(g + 1) & 1], NSP_MINV_TILE * 8 + 64 * LDV * 8);
          bulk_copy(Ms, mt(q, Jn), NSP_MINV_TILE * 8, &bar[(g + 1) & 1]);
          bulk_copy(Ms + NSP_MINV_TILE, q.Wb + (int64_t)Jn * 64 * LDV, 64 * LDV * 8, &bar[(g + 1) & 1]);
        }
      }
      const double* Ms = sm + (g & 1) * STAGE;
      if (J <= cur.I) cta_mma<NF, false, false>(Ms, NSP_MINV_LD, Ms + NSP_MINV_TILE, LDV, acc);
      else cta_mma<NF, true, false>(Ms, NSP_MINV_LD, Ms + NSP_MINV_TILE, LDV, acc);
    }
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
      for (int j = 0; j < NF; ++j) {
        const int r = acc_row<NF>(i), c = acc_col<NF>(j);
        *reinterpret_cast<double2*>(cur.out + (int64_t)r * LDV + c) = make_double2(acc[i][j][0], acc[i][j][1]);
      }
    acc_zero(acc);
    if (!has_next) break;
    u = un;
    cur = nxt;
  }
}

// ---------------------------------------------------------------------------------------------
// a2 + a3 for ONE right-hand side (the outer PCG, s = 1): u_j = S_j^{-1} w_j as a symmetric
// matrix-VECTOR product streaming the stored lower tiles of S_j^{-1} once from HBM / L2 with
// coalesced loads straight into registers (no DMMA: a tile product would do 32x the work for one
// column).  One CTA per (block, output tile row I).  J <= I: row dot products (warp w owns rows
// 8w..8w+7, lanes along the row); J > I: the stored tile (J, I) transposed, column dot products
// (thread t owns column t & 63 over a quarter of the rows).  Fixed combination order.
// ---------------------------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_symv(const FacSub* __restrict__ subs, const int2* __restrict__ items,
                                              const double* __restrict__ minv, const double* __restrict__ W, int ldw,
                                              double* __restrict__ U) {
  extern __shared__ double wv[];            // ntb x 64 right-hand side of the block
  __shared__ double cpart[4][64];
  const int2 it = items[blockIdx.x];
  const FacSub sb = subs[it.x];
  const int I = it.y, ntb = sb.ntb;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, col = tid & 63, grp = tid >> 6;
  const double* Mb = minv + sb.dense_off * NSP_MINV_TILE;
  const double* Wb = W + sb.wvu_row * (int64_t)ldw;
  for (int e = tid; e < ntb * 64; e += 256) wv[e] = Wb[(int64_t)e * ldw];
  __syncthreads();
  double r8[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) r8[i] = 0.0;
  double cacc = 0.0;
  for (int J = 0; J < ntb; ++J) {
    const double* v = wv + J * 64;
    if (J <= I) {
      const double* T = Mb + ((int64_t)I * (I + 1) / 2 + J) * NSP_MINV_TILE;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const double* row = T + (warp * 8 + i) * NSP_MINV_LD;
        r8[i] = fma(__ldg(row + lane), v[lane], r8[i]);
        r8[i] = fma(__ldg(row + lane + 32), v[lane + 32], r8[i]);
      }
    } else {
      const double* T = Mb + ((int64_t)J * (J + 1) / 2 + I) * NSP_MINV_TILE;
#pragma unroll
      for (int i = 0; i < 16; ++i) cacc = fma(__ldg(T + (grp * 16 + i) * NSP_MINV_LD + col), v[grp * 16 + i], cacc);
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1)
#pragma unroll
    for (int i = 0; i < 8; ++i) r8[i] += __shfl_xor_sync(0xffffffffu, r8[i], o);
  cpart[grp][col] = cacc;
  __syncthreads();
  if (lane < 8) {
    const int r = warp * 8 + lane;
    double mine = r8[0];
#pragma unroll
    for (int i = 1; i < 8; ++i)
      if (lane == i) mine = r8[i];
    const double u = mine + ((cpart[0][r] + cpart[1][r]) + (cpart[2][r] + cpart[3][r]));
    U[(sb.wvu_row + (int64_t)I * 64 + r) * ldw] = u;
  }
}

// Same product reading every stored tile ONCE (k_symv reads each off-diagonal tile twice: as
// (I, J) for row I and transposed for row J).  The CTA of stored tile row I multiplies each tile
// (I, J), J <= I, from registers both ways: M_IJ w_J accumulates into output row I, and for J < I the
// column product M_IJ^T w_I (8 warps' partial sums combined in fixed order) is written to the
// partial slot P[(tile J) * max_ntb + I]; the row sum goes to P[(tile I) * max_ntb + I].
// k_symv_reduce then forms u_J = sum_{I >= J} P[J][I] in ascending I (deterministic).
__global__ void __launch_bounds__(256) k_symv1(const FacSub* __restrict__ subs, const int2* __restrict__ items,
                                               const double* __restrict__ minv, const double* __restrict__ W, int ldw,
                                               int max_ntb, double* __restrict__ P) {
  pdl_wait();
  extern __shared__ double wv[];            // ntb x 64 right-hand side of the block
  __shared__ double cpart[8][64];
  const int2 it = items[blockIdx.x];
  const FacSub sb = subs[it.x];
  const int I = it.y, ntb = sb.ntb;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const double* Mb = minv + sb.dense_off * NSP_MINV_TILE;
  const double* Wb = W + sb.wvu_row * (int64_t)ldw;
  const int64_t gt0 = sb.wvu_row / 64;
  for (int e = tid; e < ntb * 64; e += 256) wv[e] = Wb[(int64_t)e * ldw];
  __syncthreads();
  const double* wI = wv + I * 64;
  double r8[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) r8[i] = 0.0;
  for (int J = 0; J <= I; ++J) {
    const double* T = Mb + ((int64_t)I * (I + 1) / 2 + J) * NSP_MINV_TILE;
    const double* v = wv + J * 64;
    const double v0 = v[lane], v1 = v[lane + 32];
    double c0 = 0.0, c1 = 0.0;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int row = warp * 8 + i;
      const double t0 = __ldg(T + row * NSP_MINV_LD + lane), t1 = __ldg(T + row * NSP_MINV_LD + lane + 32);
      r8[i] = fma(t0, v0, fma(t1, v1, r8[i]));
      const double wr = wI[row];
      c0 = fma(t0, wr, c0);
      c1 = fma(t1, wr, c1);
    }
    if (J < I) {
      cpart[warp][lane] = c0;
      cpart[warp][lane + 32] = c1;
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
#pragma unroll
  for (int o = 16; o > 0; o >>= 1)
#pragma unroll
    for (int i = 0; i < 8; ++i) r8[i] += __shfl_xor_sync(0xffffffffu, r8[i], o);
  if (lane < 8) {
    double mine = r8[0];
#pragma unroll
    for (int i = 1; i < 8; ++i)
      if (lane == i) mine = r8[i];
    P[((gt0 + I) * max_ntb + I) * 64 + warp * 8 + lane] = mine;
  }
}

__global__ void k_symv_reduce(const FacSub* __restrict__ subs, const int2* __restrict__ items, int max_ntb,
                              const double* __restrict__ P, double* __restrict__ U, int ldw) {
  pdl_wait();
  const int2 it = items[blockIdx.x];
  const FacSub sb = subs[it.x];
  const int J = it.y, ntb = sb.ntb;
  const int64_t gt = sb.wvu_row / 64 + J;
  const double* p = P + gt * max_ntb * 64 + threadIdx.x;
  double sum = 0.0;
  for (int I = J; I < ntb; ++I) sum += p[I * 64];
  U[(sb.wvu_row + (int64_t)J * 64 + threadIdx.x) * ldw] = sum;
}

// ---------------------------------------------------------------------------------------------
// Generic batched forward + backward triangular solves on tiled factors (one system per blockIdx.x,
// column chunks on blockIdx.y): dense lower tiles (wb < 0: tile(I,J) = T + I(I+1)/2 + J) or band
// tiles (tile(I,J) = T + J(wb+1) + (I-J), 0 <= I-J <= wb).  Used for A_G^{-1} (band) and for the
// interior blocks A_11 (band) of the full A_I solves; diagonal tiles hold inv(L_II).
// ---------------------------------------------------------------------------------------------
template <int CW>
__global__ void __launch_bounds__(256) k_tri_fb(const TriSys* __restrict__ sys, double* buf, int ldw, int fwd,
                                                int bwd) {
  constexpr int NF = CW / 16;
  constexpr int LDV = CW + 4;
  extern __shared__ double sm[];
  double* Ls0 = sm;
  double* Ls1 = sm + 64 * LDT;
  double* Vs0 = sm + 2 * 64 * LDT;
  double* Vs1 = Vs0 + 64 * LDV;
  const TriSys sy = sys[blockIdx.x];
  const int nt = sy.nt, wb = sy.wb;
  if (nt == 0) return;
  const int c0 = blockIdx.y * CW;
  const double* T = sy.T;
  double* Wb = buf + sy.row0 * (int64_t)ldw + c0;
  auto tile = [&](int I, int J) -> const double* {
    return wb < 0 ? T + ((int64_t)I * (I + 1) / 2 + J) * NSP_TILE_ELEMS
                  : T + ((int64_t)J * (wb + 1) + (I - J)) * NSP_TILE_ELEMS;
  };
  double acc[2][NF][2];
  if (fwd)
    for (int I = 0; I < nt; ++I) {
      acc_zero(acc);
      const int jlo = wb < 0 ? 0 : max(0, I - wb);
      if (I > jlo) {
        cp_block(Ls0, LDT, tile(I, jlo), 64, 64, 64);
        cp_block(Vs0, LDV, Wb + (int64_t)jlo * 64 * ldw, ldw, 64, CW);
        cp_commit();
        for (int J = jlo, it = 0; J < I; ++J, ++it) {
          double* Lc = (it & 1) ? Ls1 : Ls0;
          double* Vc = (it & 1) ? Vs1 : Vs0;
          if (J + 1 < I) {
            cp_block((it & 1) ? Ls0 : Ls1, LDT, tile(I, J + 1), 64, 64, 64);
            cp_block((it & 1) ? Vs0 : Vs1, LDV, Wb + (int64_t)(J + 1) * 64 * ldw, ldw, 64, CW);
            cp_commit();
            cp_wait<1>();
          } else {
            cp_wait<0>();
          }
          __syncthreads();
          cta_mma<NF, false, false>(Lc, LDT, Vc, LDV, acc);
          __syncthreads();
        }
      }
      cp_block(Ls0, LDT, tile(I, I), 64, 64, 64);
      cp_block(Vs0, LDV, Wb + (int64_t)I * 64 * ldw, ldw, 64, CW);
      cp_commit();
      cp_wait<0>();
      __syncthreads();
#pragma unroll
      for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int j = 0; j < NF; ++j) {
          const int r = acc_row<NF>(i), c = acc_col<NF>(j);
          Vs1[r * LDV + c] = Vs0[r * LDV + c] - acc[i][j][0];
          Vs1[r * LDV + c + 1] = Vs0[r * LDV + c + 1] - acc[i][j][1];
        }
      __syncthreads();
      acc_zero(acc);
      cta_mma<NF, false, false>(Ls0, LDT, Vs1, LDV, acc);
      double* out = Wb + (int64_t)I * 64 * ldw;
#pragma unroll
      for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int j = 0; j < NF; ++j) {
          const int r = acc_row<NF>(i), c = acc_col<NF>(j);
          *reinterpret_cast<double2*>(out + (int64_t)r * ldw + c) = make_double2(acc[i][j][0], acc[i][j][1]);
        }
      __threadfence();
      __syncthreads();
    }
  if (bwd)
    for (int I = nt - 1; I >= 0; --I) {
      acc_zero(acc);
      const int jhi = wb < 0 ? nt - 1 : min(nt - 1, I + wb);
      if (I < jhi) {
        cp_block(Ls0, LDT, tile(I + 1, I), 64, 64, 64);
        cp_block(Vs0, LDV, Wb + (int64_t)(I + 1) * 64 * ldw, ldw, 64, CW);
        cp_commit();
        int it = 0;
        for (int J = I + 1; J <= jhi; ++J, ++it) {
          double* Lc = (it & 1) ? Ls1 : Ls0;
          double* Vc = (it & 1) ? Vs1 : Vs0;
          if (J + 1 <= jhi) {
            cp_block((it & 1) ? Ls0 : Ls1, LDT, tile(J + 1, I), 64, 64, 64);
            cp_block((it & 1) ? Vs0 : Vs1, LDV, Wb + (int64_t)(J + 1) * 64 * ldw, ldw, 64, CW);
            cp_commit();
            cp_wait<1>();
          } else {
            cp_wait<0>();
          }
          __syncthreads();
          cta_mma<NF, true, false>(Lc, LDT, Vc, LDV, acc);
          __syncthreads();
        }
      }
      cp_block(Ls0, LDT, tile(I, I), 64, 64, 64);
      cp_block(Vs0, LDV, Wb + (int64_t)I * 64 * ldw, ldw, 64, CW);
      cp_commit();
      cp_wait<0>();
      __syncthreads();
#pragma unroll
      for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int j = 0; j < NF; ++j) {
          const int r = acc_row<NF>(i), c = acc_col<NF>(j);
          Vs1[r * LDV + c] = Vs0[r * LDV + c] - acc[i][j][0];
          Vs1[r * LDV + c + 1] = Vs0[r * LDV + c + 1] - acc[i][j][1];
        }
      __syncthreads();
      acc_zero(acc);
      cta_mma<NF, true, false>(Ls0, LDT, Vs1, LDV, acc);
      double* out = Wb + (int64_t)I * 64 * ldw;
#pragma unroll
      for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int j = 0; j < NF; ++j) {
          const int r = acc_row<NF>(i), c = acc_col<NF>(j);
          *reinterpret_cast<double2*>(out + (int64_t)r * ldw + c) = make_double2(acc[i][j][0], acc[i][j][1]);
        }
      __threadfence();
      __syncthreads();
    }
}

// ---------------------------------------------------------------------------------------------
// Narrow-band forward + backward triangular solves (wb <= WBM tiles, e.g. the A_G factor of the 2D
// configs, RCM bandwidth 16): the sweep is a chain of (row I, tile J) products whose factor tiles
// do not depend on the solution, so they (and the right-hand-side tile of each row) stream through
// an NS-stage cp.async ring issued NS-1 products ahead, while the last WBM + 1 solution tiles stay
// in shared memory (no reload).  One barrier per product, one more per row.  Same arithmetic as
// k_tri_fb (diagonal tiles hold inv(L_II)), bitwise the same products in the same order.
// ---------------------------------------------------------------------------------------------
template <int CW, int NS, int WBM>
__global__ void __launch_bounds__(256) k_band_fb(const TriSys* __restrict__ sys, double* buf, int ldw, int fwd,
                                                 int bwd) {
  constexpr int NF = CW / 16;
  constexpr int LDV = CW + 4;
  constexpr int NV = WBM + 1;
  extern __shared__ double sm[];
  double* Lr = sm;                               // NS x (64 x LDT)
  double* Wr = sm + NS * 64 * LDT;               // NS x (64 x LDV): right-hand side tile of a diag step
  double* Vr = Wr + NS * 64 * LDV;               // NV x (64 x LDV): latest solution tiles
  const TriSys sy = sys[blockIdx.x];
  const int nt = sy.nt, wb = sy.wb;
  if (nt == 0) return;
  const int c0 = blockIdx.y * CW;
  const double* T = sy.T;
  double* Wb = buf + sy.row0 * (int64_t)ldw + c0;
  auto tile = [&](int I, int J) -> const double* { return T + ((int64_t)J * (wb + 1) + (I - J)) * NSP_TILE_ELEMS; };
  double acc[2][NF][2];
  for (int pass = 0; pass < 2; ++pass) {
    const bool fw = pass == 0;
    if (fw ? !fwd : !bwd) continue;
    // product cursor over the sweep: row I, then its off-diagonal tiles, then the diagonal
    // forward: J = max(0, I - wb) .. I - 1, then I;  backward (rows descending): J = I + 1 .. min(nt-1, I + wb), then I
    auto first_j = [&](int I) { return fw ? max(0, I - wb) : I + 1; };
    auto last_off = [&](int I) { return fw ? I - 1 : min(nt - 1, I + wb); };
    auto next_row = [&](int I) { return fw ? I + 1 : I - 1; };
    int iI = fw ? 0 : nt - 1, iJ = first_j(iI);   // issue cursor (iJ > last_off => diagonal)
    int ip = 0;
    auto issue = [&]() {
      if (fw ? iI >= nt : iI < 0) return;
      double* Ls = Lr + (ip % NS) * 64 * LDT;
      const bool diag = iJ > last_off(iI);
      if (!diag) {
        cp_block(Ls, LDT, fw ? tile(iI, iJ) : tile(iJ, iI), 64, 64, 64);
        ++iJ;
      } else {
        cp_block(Ls, LDT, tile(iI, iI), 64, 64, 64);
        cp_block(Wr + (ip % NS) * 64 * LDV, LDV, Wb + (int64_t)iI * 64 * ldw, ldw, 64, CW);
        iI = next_row(iI);
        iJ = (fw ? iI < nt : iI >= 0) ? first_j(iI) : 0;
      }
      ++ip;
    };
#pragma unroll 1
    for (int p = 0; p < NS - 1; ++p) {
      issue();
      cp_commit();
    }
    int I = fw ? 0 : nt - 1, J = first_j(I);
    acc_zero(acc);
    for (int q = 0;; ++q) {
      if (fw ? I >= nt : I < 0) break;
      cp_wait<NS - 2>();
      __syncthreads();
      issue();
      cp_commit();
      const double* Ls = Lr + (q % NS) * 64 * LDT;
      if (J <= last_off(I)) {   // acc += L_IJ V_J (forward) / L_JI^T U_J (backward)
        const double* Vs = Vr + (J % NV) * 64 * LDV;
        if (fw) cta_mma<NF, false, false>(Ls, LDT, Vs, LDV, acc);
        else cta_mma<NF, true, false>(Ls, LDT, Vs, LDV, acc);
        ++J;
        continue;
      }
      // diagonal: R = W_I - acc (in place in the stage), V_I = inv(L_II) R (forward) / inv(L_II)^T R
      double* Ws = Wr + (q % NS) * 64 * LDV;
#pragma unroll
      for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int j = 0; j < NF; ++j) {
          const int r = acc_row<NF>(i), c = acc_col<NF>(j);
          Ws[r * LDV + c] -= acc[i][j][0];
          Ws[r * LDV + c + 1] -= acc[i][j][1];
        }
      __syncthreads();
      acc_zero(acc);
      if (fw) cta_mma<NF, false, false>(Ls, LDT, Ws, LDV, acc);
      else cta_mma<NF, true, false>(Ls, LDT, Ws, LDV, acc);
      double* Vs = Vr + (I % NV) * 64 * LDV;
      double* out = Wb + (int64_t)I * 64 * ldw;
#pragma unroll
      for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int j = 0; j < NF; ++j) {
          const int r = acc_row<NF>(i), c = acc_col<NF>(j);
          Vs[r * LDV + c] = acc[i][j][0];
          Vs[r * LDV + c + 1] = acc[i][j][1];
          *reinterpret_cast<double2*>(out + (int64_t)r * ldw + c) = make_double2(acc[i][j][0], acc[i][j][1]);
        }
      acc_zero(acc);
      I = next_row(I);
      J = (fw ? I < nt : I >= 0) ? first_j(I) : 0;
    }
    cp_wait<0>();
    __threadfence();
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------------------------
// Single right-hand side (s = 1, the outer PCG's A_G^{-1}) narrow-band forward + backward solve:
// the same product chain as k_band_fb, as 64 x 64 matrix-VECTOR products on the FMA pipe (a DMMA
// tile product would do 32x the work for one column).  Factor tiles (32 KB, contiguous) and the
// right-hand-side tile stream into an NS-stage ring by TMA bulk copies (cp.async.bulk + mbarrier,
// one elected thread), issued NS-1 products ahead; the last WBM + 1 solution vectors stay in shared
// memory.  Row products (forward): warp w owns rows 8w..8w+7, lanes run along the row (conflict-
// free), butterfly reduction.  Column products (backward, L^T): thread t owns column t & 63 for a
// quarter of the rows, the 4 partials meet in shared memory.  Same operations in a fixed order.
// buf (ld 1) holds the right-hand side on entry and the solution on exit.
// ---------------------------------------------------------------------------------------------
// 8 dot products per warp: v[rr] (per-lane partials of row rr) -> the full sum of row
// 4 bit4 + 2 bit3 + bit2 of the lane, in lanes with (lane & 3) == 0 (and their 3 neighbours)
__device__ __forceinline__ double warp_reduce8(double v[8], int lane) {
  {
    const bool up = lane & 16;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const double rcv = __shfl_xor_sync(0xffffffffu, up ? v[i] : v[i + 4], 16);
      v[i] = (up ? v[i + 4] : v[i]) + rcv;
    }
  }
  {
    const bool up = lane & 8;
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      const double rcv = __shfl_xor_sync(0xffffffffu, up ? v[i] : v[i + 2], 8);
      v[i] = (up ? v[i + 2] : v[i]) + rcv;
    }
  }
  {
    const bool up = lane & 4;
    const double rcv = __shfl_xor_sync(0xffffffffu, up ? v[0] : v[1], 4);
    v[0] = (up ? v[1] : v[0]) + rcv;
  }
  v[0] += __shfl_xor_sync(0xffffffffu, v[0], 2);
  v[0] += __shfl_xor_sync(0xffffffffu, v[0], 1);
  return v[0];
}
__device__ __forceinline__ int warp_reduce8_row(int lane) {
  return 4 * ((lane >> 4) & 1) + 2 * ((lane >> 3) & 1) + ((lane >> 2) & 1);
}

// s > 1 (32-column chunks, ldw a multiple of 32 with zero padding columns): the P-step recurrence on
// the DMMA pipe.  The spike tiles and the right-hand-side tiles do not depend on the recurrence, so
// they stream through a 2-deep cp.async ring one step ahead; the running 64 x 32 coupling block stays
// in shared memory.  One CTA per column chunk.
__global__ void __launch_bounds__(256) k_spike_tail_mma(const double* __restrict__ spk,
                                                        const int* __restrict__ chunk_first, int P, double* buf,
                                                        int ldw, int fwd) {
  pdl_wait();
  constexpr int LDX = 36;
  extern __shared__ __align__(16) double sm[];
  double* Ss = sm;                       // 2 x 64 x LDT
  double* Ys = sm + 2 * 64 * LDT;        // 2 x 64 x LDX (right-hand side tile of the step)
  double* Xs = Ys + 2 * 64 * LDX;        // 64 x LDX: the previous step's result
  const int c0 = blockIdx.x * 32;
  const int nstep = P - 1;
  auto tile_of = [&](int j) { return fwd ? chunk_first[j + 2] - 1 : chunk_first[P - 2 - j]; };
  auto src_of = [&](int j) { return fwd ? chunk_first[j + 1] - 1 : chunk_first[P - 1 - j]; };
  auto issue = [&](int j) {
    const int t = tile_of(j);
    cp_block(Ss + (j & 1) * 64 * LDT, LDT, spk + (int64_t)t * 4096, 64, 64, 64);
    cp_block(Ys + (j & 1) * 64 * LDX, LDX, buf + (int64_t)t * 64 * ldw + c0, ldw, 64, 32);
  };
  cp_block(Xs, LDX, buf + (int64_t)src_of(0) * 64 * ldw + c0, ldw, 64, 32);
  issue(0);
  cp_commit();
  double acc[2][2][2];
  for (int j = 0; j < nstep; ++j) {
    cp_wait<0>();
    __syncthreads();
    if (j + 1 < nstep) issue(j + 1);
    cp_commit();
    acc_zero(acc);
    cta_mma<2, false, false>(Ss + (j & 1) * 64 * LDT, LDT, Xs, LDX, acc, 64);
    __syncthreads();   // every read of Xs done
    const double* Y = Ys + (j & 1) * 64 * LDX;
    double* out = buf + (int64_t)tile_of(j) * 64 * ldw + c0;
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        const int r = acc_row<2>(i), c = acc_col<2>(q);
        const double v0 = Y[r * LDX + c] - acc[i][q][0], v1 = Y[r * LDX + c + 1] - acc[i][q][1];
        Xs[r * LDX + c] = v0;
        Xs[r * LDX + c + 1] = v1;
        *reinterpret_cast<double2*>(out + (int64_t)r * ldw + c) = make_double2(v0, v1);
      }
  }
}

// s > 1: every remaining tile row in parallel, grid (tile rows, 32-column chunks), DMMA product
__global__ void __launch_bounds__(256) k_spike_update_mma(const double* __restrict__ spk,
                                                          const int* __restrict__ chunk_first,
                                                          const int* __restrict__ tile_chunk, int P, double* buf,
                                                          int ldw, int fwd) {
  pdl_wait();
  constexpr int LDX = 36;
  extern __shared__ __align__(16) double sm[];
  double* Ss = sm;
  double* Xs = sm + 64 * LDT;
  const int I = blockIdx.x;
  const int c0 = blockIdx.y * 32;
  const int k = tile_chunk[I];
  int src;
  if (fwd) {
    if (k == 0 || I == chunk_first[k + 1] - 1) return;
    src = chunk_first[k] - 1;
  } else {
    if (k == P - 1 || I == chunk_first[k]) return;
    src = chunk_first[k + 1];
  }
  cp_block(Ss, LDT, spk + (int64_t)I * 4096, 64, 64, 64);
  cp_block(Xs, LDX, buf + (int64_t)src * 64 * ldw + c0, ldw, 64, 32);
  cp_commit();
  cp_wait<0>();
  __syncthreads();
  double acc[2][2][2];
  acc_zero(acc);
  cta_mma<2, false, false>(Ss, LDT, Xs, LDX, acc, 64);
  double* out = buf + (int64_t)I * 64 * ldw + c0;
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const int r = acc_row<2>(i), c = acc_col<2>(q);
      double2* o = reinterpret_cast<double2*>(out + (int64_t)r * ldw + c);
      const double2 cur = *o;
      *o = make_double2(cur.x - acc[i][q][0], cur.y - acc[i][q][1]);
    }
}

template <int NS, int WBM>
__global__ void __launch_bounds__(256) k_band_fb_vec(const TriSys* __restrict__ sys, double* buf, int fwd, int bwd) {
  constexpr int NV = WBM + 1;
  extern __shared__ __align__(128) double sm[];
  double* Lr = sm;                          // NS x 4096 (contiguous 64 x 64 tiles)
  double* Wr = sm + NS * 4096;              // NS x 64 (rhs tile of a diagonal step)
  double* Vr = Wr + NS * 64;                // NV x 64
  double* Pp = Vr + NV * 64;                // 4 x 64 column partials
  double* Rs = Pp + 4 * 64;                 // 64 residual
  __shared__ __align__(8) uint64_t bar[NS];
  const TriSys sy = sys[blockIdx.x];
  const int nt = sy.nt, wb = sy.wb;
  if (nt == 0) return;
  const double* T = sy.T;
  double* Wb = buf + sy.row0;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int col = tid & 63, grp = tid >> 6;
  const int myrow = warp_reduce8_row(lane);   // forward: the row whose sum this lane holds
  auto tile = [&](int I, int J) -> const double* { return T + ((int64_t)J * (wb + 1) + (I - J)) * NSP_TILE_ELEMS; };
  if (tid == 0)
    for (int i = 0; i < NS; ++i) mbar_init(&bar[i], 1);
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  __syncthreads();
  unsigned uses[NS];   // completed phases per slot (thread-uniform)
#pragma unroll
  for (int i = 0; i < NS; ++i) uses[i] = 0;
  for (int pass = 0; pass < 2; ++pass) {
    const bool fw = pass == 0;
    if (fw ? !fwd : !bwd) continue;
    auto first_j = [&](int I) { return fw ? max(0, I - wb) : I + 1; };
    auto last_off = [&](int I) { return fw ? I - 1 : min(nt - 1, I + wb); };
    auto next_row = [&](int I) { return fw ? I + 1 : I - 1; };
    int iI = fw ? 0 : nt - 1, iJ = first_j(iI), ip = 0;
    auto issue = [&]() {   // one product's tiles into slot ip % NS (thread 0 issues)
      if (fw ? iI >= nt : iI < 0) return;
      const int sl = ip % NS;
      if (iJ <= last_off(iI)) {
        if (tid == 0) mbar_expect_copy(&bar[sl], Lr + sl * 4096, fw ? tile(iI, iJ) : tile(iJ, iI), 32768);
        ++iJ;
      } else {
        if (tid == 0) {
          mbar_expect(&bar[sl], 32768 + 512);   // full stage bytes before either copy is issued
          bulk_copy(Lr + sl * 4096, tile(iI, iI), 32768, &bar[sl]);
          bulk_copy(Wr + sl * 64, Wb + (int64_t)iI * 64, 512, &bar[sl]);
        }
        iI = next_row(iI);
        iJ = (fw ? iI < nt : iI >= 0) ? first_j(iI) : 0;
      }
      ++ip;
    };
    for (int p = 0; p < NS - 1; ++p) issue();
    int I = fw ? 0 : nt - 1, J = first_j(I);
    double racc = 0.0;   // forward: lane j of warp w holds the sum of row 8w + j (after reduction)
    double cacc = 0.0;   // backward: column partial (col, grp)
    for (int q = 0;; ++q) {
      if (fw ? I >= nt : I < 0) break;
      const int sl = q % NS;
      mbar_wait(&bar[sl], uses[sl] & 1);
      ++uses[sl];
      __syncthreads();          // every thread is done with the slot the next issue overwrites
      issue();
      const double* L = Lr + sl * 4096;
      const bool diag = J > last_off(I);
      const double* v = diag ? nullptr : Vr + (J % NV) * 64;
      if (diag) {                // residual R = W_I - acc
        if (fw) {
          if ((lane & 3) == 0) Rs[warp * 8 + myrow] = Wr[sl * 64 + warp * 8 + myrow] - racc;
        } else {
          Pp[grp * 64 + col] = cacc;
          __syncthreads();
          if (tid < 64) Rs[tid] = Wr[sl * 64 + tid] - ((Pp[tid] + Pp[64 + tid]) + (Pp[128 + tid] + Pp[192 + tid]));
        }
        __syncthreads();
        v = Rs;
      }
      if (fw) {                  // y_r = sum_c L[r][c] v[c], rows 8w .. 8w+7
        double p8[8];
        const double v0 = v[lane], v1 = v[lane + 32];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const double* Lrow = L + (warp * 8 + i) * 64;
          p8[i] = fma(Lrow[lane], v0, Lrow[lane + 32] * v1);
        }
        const double mine = warp_reduce8(p8, lane);   // row 8 warp + myrow, on lanes with (lane & 3) == 0
        if (!diag) {
          racc += mine;
        } else if ((lane & 3) == 0) {
          Vr[(I % NV) * 64 + warp * 8 + myrow] = mine;
          Wb[(int64_t)I * 64 + warp * 8 + myrow] = mine;
        }
      } else {                   // y_c = sum_r L[r][c] v[r], rows 16 grp .. 16 grp + 15
        double y = 0.0;
#pragma unroll
        for (int i = 0; i < 16; ++i) y = fma(L[(grp * 16 + i) * 64 + col], v[grp * 16 + i], y);
        if (!diag) {
          cacc += y;
        } else {
          Pp[grp * 64 + col] = y;
          __syncthreads();
          if (tid < 64) {
            const double u = (Pp[tid] + Pp[64 + tid]) + (Pp[128 + tid] + Pp[192 + tid]);
            Vr[(I % NV) * 64 + tid] = u;
            Wb[(int64_t)I * 64 + tid] = u;
          }
        }
      }
      if (diag) {
        racc = 0.0;
        cacc = 0.0;
        I = next_row(I);
        J = (fw ? I < nt : I >= 0) ? first_j(I) : 0;
      } else {
        ++J;
      }
    }
    __threadfence();
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------------------------
// One-column chunk sweeps of the partitioned A_G solve (wb <= 1) as ONE matrix-vector product per tile
// row: forward y_I = X_II w_I - G_I y_{I-1} with G_I = X_II L_{I,I-1}; backward y_I = X_II^T w_I -
// H_I y_{I+1} with H_I = X_II^T L_{I+1,I}^T (X_II = L_II^{-1}; Xd / Gc tiles formed in setup by
// k_band_prep, row-dot layout for both directions).  The same triangular solve reassociated: the
// recurrence carries one product per row instead of two, and the row's two products are one fused dot
// product (one warp reduction).  One CTA per chunk; the tiles and the rhs tile of the next NS - 1 rows
// stream in by TMA bulk copies.
// ---------------------------------------------------------------------------------------------
template <int NS>
__global__ void __launch_bounds__(256) k_band_rec_vec(const TriSys* __restrict__ sys, const double* __restrict__ Xd,
                                                      int64_t xstride, const double* __restrict__ Gc, double* buf,
                                                      int fwd) {
  pdl_wait();
  extern __shared__ __align__(128) double sm[];
  double* Tr = sm;                 // NS x (Xd tile, Gc tile)
  double* Wr = sm + NS * 8192;     // NS x 64 rhs
  double* Vr = Wr + NS * 64;       // 2 x 64: y of the previous row (ping-pong)
  __shared__ __align__(8) uint64_t bar[NS];
  const TriSys sy = sys[blockIdx.x];
  const int nt = sy.nt;
  if (nt == 0) return;
  const int64_t t0 = sy.row0 / 64;   // global tile index of the chunk's first row
  double* Wb = buf + sy.row0;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int myrow = warp_reduce8_row(lane);
  if (tid == 0)
    for (int i = 0; i < NS; ++i) mbar_init(&bar[i], 1);
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  __syncthreads();
  auto row_of = [&](int q) { return fwd ? q : nt - 1 - q; };   // q-th step's local tile row
  auto issue = [&](int q) {
    if (q >= nt || tid != 0) return;
    const int sl = q % NS, I = row_of(q);
    mbar_expect(&bar[sl], 32768 + (q > 0 ? 32768 : 0) + 512);   // full stage bytes first, then the copies
    bulk_copy(Tr + sl * 8192, Xd + (t0 + I) * xstride * 4096, 32768, &bar[sl]);
    if (q > 0) bulk_copy(Tr + sl * 8192 + 4096, Gc + (t0 + I) * 4096, 32768, &bar[sl]);
    bulk_copy(Wr + sl * 64, Wb + (int64_t)I * 64, 512, &bar[sl]);
  };
  for (int q = 0; q < NS - 1; ++q) issue(q);
  for (int q = 0; q < nt; ++q) {
    const int sl = q % NS, I = row_of(q);
    mbar_wait(&bar[sl], (q / NS) & 1);
    __syncthreads();   // the slot issued next was last read at step q - 1; y_{q-1} is in Vr
    issue(q + NS - 1);
    const double* X = Tr + sl * 8192;
    const double* G = X + 4096;
    const double* w = Wr + sl * 64;
    const double* yp = Vr + ((q + 1) & 1) * 64;
    const double w0 = w[lane], w1 = w[lane + 32];
    double p8[8];
    if (q > 0) {
      const double y0 = yp[lane], y1 = yp[lane + 32];
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const double* xr = X + (warp * 8 + i) * 64;
        const double* gr = G + (warp * 8 + i) * 64;
        p8[i] = fma(xr[lane], w0, fma(xr[lane + 32], w1, -fma(gr[lane], y0, gr[lane + 32] * y1)));
      }
    } else {
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const double* xr = X + (warp * 8 + i) * 64;
        p8[i] = fma(xr[lane], w0, xr[lane + 32] * w1);
      }
    }
    const double y = warp_reduce8(p8, lane);
    if ((lane & 3) == 0) {
      Vr[(q & 1) * 64 + warp * 8 + myrow] = y;
      Wb[(int64_t)I * 64 + warp * 8 + myrow] = y;
    }
  }
  __threadfence();
}

// The same reassociated chunk sweep for s > 1 (CW-column slices, DMMA): per tile row
// V_I = Xd_I W_I - Gc_I V_prev as two 64 x 64 x CW tile products into two accumulators, one CTA
// barrier per row; the next row's two tiles and rhs tile are staged by cp.async behind this row's
// products (2 stages).  Xd / Gc as in k_band_rec_vec.
template <int CW>
__global__ void __launch_bounds__(256) k_band_rec(const TriSys* __restrict__ sys, const double* __restrict__ Xd,
                                                  int64_t xstride, const double* __restrict__ Gc, double* buf, int ldw,
                                                  int fwd) {
  pdl_wait();
  constexpr int NF = CW / 16;
  constexpr int LDV = CW + 4;
  extern __shared__ double sm[];
  double* Xs = sm;                    // 2 x 64 x LDT
  double* Gs = Xs + 2 * 64 * LDT;     // 2 x 64 x LDT
  double* Ws = Gs + 2 * 64 * LDT;     // 2 x 64 x LDV
  double* Vs = Ws + 2 * 64 * LDV;     // 2 x 64 x LDV (ping-pong: the previous row's solution)
  const TriSys sy = sys[blockIdx.x];
  const int nt = sy.nt;
  if (nt == 0) return;
  const int64_t t0 = sy.row0 / 64;
  const int c0 = blockIdx.y * CW;
  double* Wb = buf + sy.row0 * (int64_t)ldw + c0;
  auto row_of = [&](int q) { return fwd ? q : nt - 1 - q; };
  auto issue = [&](int q) {
    if (q >= nt) return;
    const int sl = q & 1, I = row_of(q);
    cp_block(Xs + sl * 64 * LDT, LDT, Xd + (t0 + I) * xstride * 4096, 64, 64, 64);
    if (q > 0) cp_block(Gs + sl * 64 * LDT, LDT, Gc + (t0 + I) * 4096, 64, 64, 64);
    cp_block(Ws + sl * 64 * LDV, LDV, Wb + (int64_t)I * 64 * ldw, ldw, 64, CW);
  };
  issue(0);
  cp_commit();
  for (int q = 0; q < nt; ++q) {
    const int sl = q & 1, I = row_of(q);
    cp_wait<0>();
    __syncthreads();   // stage q landed; V of row q - 1 visible; stage q + 1's slot was last read at q - 1
    issue(q + 1);
    cp_commit();
    double acc[2][NF][2], accg[2][NF][2];
    acc_zero(acc);
    acc_zero(accg);
    cta_mma<NF, false, false>(Xs + sl * 64 * LDT, LDT, Ws + sl * 64 * LDV, LDV, acc);
    if (q > 0) cta_mma<NF, false, false>(Gs + sl * 64 * LDT, LDT, Vs + ((q + 1) & 1) * 64 * LDV, LDV, accg);
    double* Vo = Vs + (q & 1) * 64 * LDV;
    double* out = Wb + (int64_t)I * 64 * ldw;
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
      for (int j = 0; j < NF; ++j) {
        const int r = acc_row<NF>(i), c = acc_col<NF>(j);
        const double v0 = acc[i][j][0] - accg[i][j][0], v1 = acc[i][j][1] - accg[i][j][1];
        Vo[r * LDV + c] = v0;
        Vo[r * LDV + c + 1] = v1;
        *reinterpret_cast<double2*>(out + (int64_t)r * ldw + c) = make_double2(v0, v1);
      }
  }
  cp_wait<0>();
  __threadfence();
}

// Setup for k_band_rec_vec: per tile row I of the band (wb <= 1, diagonal tiles hold X_II = L_II^{-1})
//   XF_I = X_II, GF_I = X_II L_{I,I-1} (I >= 1), XB_I = X_II^T, GB_I = X_II^T L_{I+1,I}^T (I <= nt - 2)
// one CTA per tile row, plain FMA products (setup).
__global__ void __launch_bounds__(256) k_band_prep(const double* __restrict__ T, int nt, int wb, double* XF, double* GF,
                                                   double* XB, double* GB) {
  __shared__ double Xs[64][65];
  const int I = blockIdx.x, tid = threadIdx.x;
  auto tile = [&](int r, int c) { return T + ((int64_t)c * (wb + 1) + (r - c)) * NSP_TILE_ELEMS; };
  const double* Xg = tile(I, I);
  for (int e = tid; e < 4096; e += 256) {
    Xs[e >> 6][e & 63] = Xg[e];
    if (XF) XF[(int64_t)I * 4096 + e] = Xg[e];
    XB[(int64_t)I * 4096 + e] = Xg[(e & 63) * 64 + (e >> 6)];
  }
  __syncthreads();
  const double* Lf = (wb >= 1 && I >= 1) ? tile(I, I - 1) : nullptr;        // L_{I,I-1}
  const double* Lb = (wb >= 1 && I + 1 < nt) ? tile(I + 1, I) : nullptr;    // L_{I+1,I}
  for (int e = tid; e < 4096; e += 256) {
    const int r = e >> 6, cc = e & 63;
    double gf = 0.0, gb = 0.0;
    for (int k = 0; k < 64; ++k) {
      if (Lf) gf = fma(Xs[r][k], Lf[k * 64 + cc], gf);    // (X_II L_{I,I-1})[r][c]
      if (Lb) gb = fma(Xs[k][r], Lb[cc * 64 + k], gb);    // (X_II^T L_{I+1,I}^T)[r][c]
    }
    GF[(int64_t)I * 4096 + e] = gf;
    GB[(int64_t)I * 4096 + e] = gb;
  }
}

// ---------------------------------------------------------------------------------------------
// Partitioned ("spike") narrow-band solve of the A_G factor.  The band rows are cut into P chunks of
// consecutive 64-row tiles; chunk k couples to chunk k-1 only through one factor tile C_k (first tile
// row of k x last tile column of k-1).  With the spikes S_k = L_kk^{-1} [C_k; 0] and
// T_k = L_kk^{-T} [0; C_{k+1}^T] formed in setup:
//   forward:  y_k = L_kk^{-1} b_k (all chunks in parallel);  x_k = y_k - S_k x_{k-1}[last tile]
//   backward: z_k = L_kk^{-T} x_k (parallel);                 u_k = z_k - T_k u_{k+1}[first tile]
// the coupling tiles ride a P-step recurrence (k_spike_tail), the rest is one parallel update
// (k_spike_update).  Exact in exact arithmetic; a reordering of the same triangular solve.
// tile_chunk[I] = chunk of tile row I; chunk_first[k] = first tile row of chunk k (chunk_first[P] = nt)
// spk: rows of the band buffer x 64 (S_k rows for the forward spikes, T_k rows for the backward).
// ---------------------------------------------------------------------------------------------
__device__ __forceinline__ void spike_tile_product(const double* __restrict__ Sg, const double* __restrict__ Xg,
                                                   int ldw, double* __restrict__ Og, int ncols, double* sm) {
  // Og (64 x ncols, ld ldw) -= Sg (64 x 64, ld 64) * Xg (64 x ncols, ld ldw); ncols <= 32, both operands
  // staged in shared memory (dynamic, 50 KB)
  double* Ss = sm;              // 64 x 65
  double* Xs = sm + 64 * 65;    // 64 x 33
  for (int e = threadIdx.x; e < 4096; e += 256) Ss[(e >> 6) * 65 + (e & 63)] = __ldg(Sg + e);
  for (int e = threadIdx.x; e < 64 * ncols; e += 256) {
    const int r = e / ncols, cc = e - r * ncols;
    Xs[r * 33 + cc] = Xg[(int64_t)r * ldw + cc];
  }
  __syncthreads();
  for (int e = threadIdx.x; e < 64 * ncols; e += 256) {
    const int r = e / ncols, cc = e - r * ncols;
    double acc = 0.0;
#pragma unroll 8
    for (int k = 0; k < 64; ++k) acc = fma(Ss[r * 65 + k], Xs[k * 33 + cc], acc);
    Og[(int64_t)r * ldw + cc] -= acc;
  }
  __syncthreads();
}

// sequential over chunks (one CTA per 32-column chunk): the coupling tiles
__global__ void __launch_bounds__(256) k_spike_tail(const double* __restrict__ spk, const int* __restrict__ chunk_first,
                                                    int P, double* buf, int ldw, int s, int fwd) {
  extern __shared__ double sm[];
  const int c0 = blockIdx.x * 32;
  const int ncols = min(32, s - c0);
  if (fwd) {
    for (int k = 1; k < P; ++k) {   // x_k[last] -= S_k[last rows] x_{k-1}[last]
      const int last = chunk_first[k + 1] - 1, prev = chunk_first[k] - 1;
      spike_tile_product(spk + (int64_t)last * 64 * 64, buf + (int64_t)prev * 64 * ldw + c0, ldw,
                         buf + (int64_t)last * 64 * ldw + c0, ncols, sm);
      __threadfence_block();
    }
  } else {
    for (int k = P - 2; k >= 0; --k) {   // u_k[first] -= T_k[first rows] u_{k+1}[first]
      const int first = chunk_first[k], nxt = chunk_first[k + 1];
      spike_tile_product(spk + (int64_t)first * 64 * 64, buf + (int64_t)nxt * 64 * ldw + c0, ldw,
                         buf + (int64_t)first * 64 * ldw + c0, ncols, sm);
      __threadfence_block();
    }
  }
}

// one column (s = 1, ld 1): the same P-step recurrence as a matrix-vector chain.  The spike tiles
// do not depend on the recurrence, so they stream through a 2-deep TMA ring while the previous
// step computes; the running 64-vector stays in shared memory; each warp owns 8 rows (coalesced
// 32-lane row reads, transposed shuffle reduction: 9 shuffles for 8 dot products).
__global__ void __launch_bounds__(256) k_spike_tail_vec(const double* __restrict__ spk,
                                                        const int* __restrict__ chunk_first, int P,
                                                        double* buf, int fwd) {
  pdl_wait();
  extern __shared__ __align__(128) double sm[];   // 3 x 4096 spike tiles (ring)
  __shared__ double xs[2][64];                     // ping-pong: the coupling vector of the previous step
  __shared__ __align__(8) uint64_t bar[3];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int nstep = P - 1;
  // step j: the tile row updated (and whose spike rows are used) and the tile row it reads
  auto tile_of = [&](int j) { return fwd ? chunk_first[j + 2] - 1 : chunk_first[P - 2 - j]; };
  auto src_of = [&](int j) { return fwd ? chunk_first[j + 1] - 1 : chunk_first[P - 1 - j]; };
  if (tid == 0) {
    for (int i = 0; i < 3; ++i) mbar_init(&bar[i], 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  if (tid == 0) {
    for (int j = 0; j < 3 && j < nstep; ++j)
      mbar_expect_copy(&bar[j], sm + j * 4096, spk + (int64_t)tile_of(j) * 4096, 4096 * 8);
  }
  if (tid < 64) xs[0][tid] = buf[(int64_t)src_of(0) * 64 + tid];
  __syncthreads();
  const int myrow = 8 * warp + warp_reduce8_row(lane);
  for (int j = 0; j < nstep; ++j) {
    const int t = tile_of(j);
    const double y = (lane & 3) == 0 ? buf[(int64_t)t * 64 + myrow] : 0.0;
    const int b = j % 3;
    mbar_wait(&bar[b], (j / 3) & 1);
    const double* S = sm + b * 4096;
    const double x0 = xs[j & 1][lane], x1 = xs[j & 1][lane + 32];
    double v[8];
#pragma unroll
    for (int rr = 0; rr < 8; ++rr) {
      const double* Sr = S + (8 * warp + rr) * 64;
      v[rr] = fma(Sr[lane], x0, Sr[lane + 32] * x1);
    }
    v[0] = warp_reduce8(v, lane);
    if ((lane & 3) == 0) {
      const double o = y - v[0];
      xs[(j + 1) & 1][myrow] = o;
      buf[(int64_t)t * 64 + myrow] = o;
    }
    __syncthreads();   // xs of this step visible; every read of ring slot b (and of xs[j & 1]) is done
    if (tid == 0 && j + 3 < nstep) {
      asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
      mbar_expect_copy(&bar[b], sm + b * 4096, spk + (int64_t)tile_of(j + 3) * 4096, 4096 * 8);
    }
  }
}

// one column: every remaining tile row in parallel, one CTA per tile row, spike rows read straight
// from global memory (each warp 8 rows, coalesced), no shared-memory staging
__global__ void __launch_bounds__(256) k_spike_update_vec(const double* __restrict__ spk,
                                                          const int* __restrict__ chunk_first,
                                                          const int* __restrict__ tile_chunk, int P, double* buf,
                                                          int fwd) {
  pdl_wait();
  const int I = blockIdx.x;
  const int k = tile_chunk[I];
  int src;
  if (fwd) {
    if (k == 0 || I == chunk_first[k + 1] - 1) return;
    src = chunk_first[k] - 1;
  } else {
    if (k == P - 1 || I == chunk_first[k]) return;
    src = chunk_first[k + 1];
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const double* xg = buf + (int64_t)src * 64;
  const double x0 = xg[lane], x1 = xg[lane + 32];
  const double* S = spk + (int64_t)I * 4096;
  double v[8];
#pragma unroll
  for (int rr = 0; rr < 8; ++rr) {
    const double* Sr = S + (8 * warp + rr) * 64;
    v[rr] = fma(__ldg(Sr + lane), x0, __ldg(Sr + lane + 32) * x1);
  }
  const double d = warp_reduce8(v, lane);
  if ((lane & 3) == 0) buf[(int64_t)I * 64 + 8 * warp + warp_reduce8_row(lane)] -= d;
}

// all remaining tile rows in parallel: grid (tile rows, 32-column chunks)
__global__ void __launch_bounds__(256) k_spike_update(const double* __restrict__ spk, const int* __restrict__ chunk_first,
                                                      const int* __restrict__ tile_chunk, int P, double* buf, int ldw,
                                                      int s, int fwd) {
  extern __shared__ double sm[];
  const int I = blockIdx.x;
  const int c0 = blockIdx.y * 32;
  const int ncols = min(32, s - c0);
  const int k = tile_chunk[I];
  if (fwd) {
    if (k == 0 || I == chunk_first[k + 1] - 1) return;   // chunk 0 is final; the last tile came from the tail
    const int prev = chunk_first[k] - 1;
    spike_tile_product(spk + (int64_t)I * 64 * 64, buf + (int64_t)prev * 64 * ldw + c0, ldw,
                       buf + (int64_t)I * 64 * ldw + c0, ncols, sm);
  } else {
    if (k == P - 1 || I == chunk_first[k]) return;
    const int nxt = chunk_first[k + 1];
    spike_tile_product(spk + (int64_t)I * 64 * 64, buf + (int64_t)nxt * 64 * ldw + c0, ldw,
                       buf + (int64_t)I * 64 * ldw + c0, ncols, sm);
  }
}

// Philox4x32-10 (Salmon et al., SC'11; Random123 constants) + the Box-Muller cosine branch, the same
// stream layout as nsp_inputs/philox.py (reading C7): counter = (e lo, e hi, stream, 0), key = seed.
__global__ void k_philox_gaussian(double* __restrict__ out, int64_t rows, int s, int ld,
                                  const int64_t* __restrict__ gidx, uint64_t seed, uint32_t stream) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= rows * ld) return;
  const int64_t r = i / ld;
  const int j = (int)(i - r * ld);
  if (j >= s) {
    out[i] = 0.0;
    return;
  }
  const uint64_t e = (uint64_t)gidx[r] * (uint64_t)s + (uint64_t)j;
  uint32_t c0 = (uint32_t)e, c1 = (uint32_t)(e >> 32), c2 = stream, c3 = 0u;
  uint32_t k0 = (uint32_t)seed, k1 = (uint32_t)(seed >> 32);
#pragma unroll
  for (int q = 0; q < 10; ++q) {
    const uint64_t p0 = 0xD2511F53ull * c0, p1 = 0xCD9E8D57ull * c2;
    const uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0, hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
    c0 = hi1 ^ c1 ^ k0;
    c1 = lo1;
    c2 = hi0 ^ c3 ^ k1;
    c3 = lo0;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  const double scale = 1.0 / 9007199254740992.0;   // 2^-53
  const double u1 = ((double)(((uint64_t)(c0 >> 5)) * 67108864ull + (c1 >> 6)) + 0.5) * scale;
  const double u2 = ((double)(((uint64_t)(c2 >> 5)) * 67108864ull + (c3 >> 6)) + 0.5) * scale;
  out[i] = sqrt(-2.0 * log(u1)) * cos(2.0 * 3.141592653589793 * u2);
}

// row gather / scatter between an n x s block (ld lds) and a padded buffer (ld ldd):
// gather: dst[r][c] = idx[r] >= 0 && c < s ? scale * src[idx[r]][c] : 0  for r < rows, c < ldd
// scatter: dst[idx[r]][c] = src[r][c]   (c < s, idx[r] >= 0)
__global__ void k_gather_rows(const double* __restrict__ src, int lds, const int32_t* __restrict__ idx, int64_t rows,
                              double* dst, int ldd, int s, double scale) {
  pdl_wait();
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t r = e / ldd;
  const int c = (int)(e - r * ldd);
  if (r >= rows) return;
  const int32_t k = idx[r];
  dst[r * ldd + c] = (k >= 0 && c < s) ? scale * src[(int64_t)k * lds + c] : 0.0;
}
__global__ void k_scatter_rows(const double* __restrict__ src, int lds, const int32_t* __restrict__ idx, int64_t rows,
                               double* dst, int ldd, int s, int accumulate) {
  pdl_wait();
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t r = e / s;
  const int c = (int)(e - r * s);
  if (r >= rows) return;
  const int32_t k = idx[r];
  if (k < 0) return;
  if (accumulate) dst[(int64_t)k * ldd + c] += src[r * lds + c];
  else dst[(int64_t)k * ldd + c] = src[r * lds + c];
}

}  // namespace

namespace nspk {

void scatter(double* base, const int64_t* idx, const double* val, int64_t cnt, cudaStream_t st) {
  if (cnt <= 0) return;
  { nsp_count_launch(); k_scatter<<<(unsigned)((cnt + 255) / 256), 256, 0, st>>>(base, idx, val, cnt); }
}

void set_pad_identity(double* base, const int64_t* tile_idx, const int* first_row, int cnt, cudaStream_t st) {
  if (cnt <= 0) return;
  { nsp_count_launch(); launch_k(k_pad_identity, dim3(cnt), dim3(64), 0, st, base, tile_idx, first_row, cnt); }
}

void tile_cholesky(const FacSub* subs, int nsub, double* band, double* dense, double* scratch,
                   const int* border_first, int* status, cudaStream_t st) {
  if (nsub <= 0) return;
  const size_t smem = 5 * 64 * LDT * sizeof(double);
  smem_optin((const void*)k_tile_cholesky, (size_t)((int)smem));
  { nsp_count_launch(); k_tile_cholesky<<<nsub, 256, smem, st>>>(subs, band, dense, scratch, border_first, status); }
}

bool spmm_cs_oz(const DevCSR& A, const double* X, int ldx, double* Y, int64_t ycs, int ypad, int s,
                const int* ozdx, const int* oztb, int* ozse, cudaStream_t st) {
  if (A.rows <= 0 || A.rows % 64 || s % 2 || ldx % 2 || ycs % 2 || ypad % 2 || s > 256) return false;
  const unsigned blocks = (unsigned)(A.rows / 8);
  const int ozn = 128 * ((s + 127) / 128);
  const int nq2 = (s + 63) / 64;
  nsp_count_launch();
  if (nq2 == 1)
    launch_k(k_spmm2<1, true>, dim3(blocks), dim3(256), 0, st, A.rows, A.rowptr, A.col, A.val, X, ldx, nullptr, 0,
             (int64_t)32, (int64_t)0, Y, 36, ycs, ypad, s, 0, 1, ozdx, oztb, ozse, ozn);
  else if (nq2 == 2)
    launch_k(k_spmm2<2, true>, dim3(blocks), dim3(256), 0, st, A.rows, A.rowptr, A.col, A.val, X, ldx, nullptr, 0,
             (int64_t)32, (int64_t)0, Y, 36, ycs, ypad, s, 0, 1, ozdx, oztb, ozse, ozn);
  else
    launch_k(k_spmm2<4, true>, dim3(blocks), dim3(256), 0, st, A.rows, A.rowptr, A.col, A.val, X, ldx, nullptr, 0,
             (int64_t)32, (int64_t)0, Y, 36, ycs, ypad, s, 0, 1, ozdx, oztb, ozse, ozn);
  return true;
}

void spmm_cs(const DevCSR& A, const double* X, int ldx, const double* U, int ldu, int64_t ucs, int64_t split,
             double* Y, int ldy, int64_t ycs, int ypad, int s, int mode, bool zero_pad, cudaStream_t st) {
  if (A.rows <= 0) return;
  const unsigned blocks = (unsigned)((A.rows * 32 + 255) / 256);
  if (s == 1 && ycs == 32 && ucs == 32) {
    static const int G = [] {
      const char* e = getenv("NSP_SPMV_G");
      const int g = e ? atoi(e) : 8;
      return (g == 2 || g == 4) ? g : 8;
    }();
    nsp_count_launch();
    if (G == 2)
      launch_k(k_spmv<2>, dim3((unsigned)((A.rows * 2 + 255) / 256)), dim3(256), 0, st, A.rows, A.rowptr, A.col, A.val, X, ldx, U, ldu, split, Y, ldy, mode, zero_pad);
    else if (G == 4)
      launch_k(k_spmv<4>, dim3((unsigned)((A.rows * 4 + 255) / 256)), dim3(256), 0, st, A.rows, A.rowptr, A.col, A.val, X, ldx, U, ldu, split, Y, ldy, mode, zero_pad);
    else
      launch_k(k_spmv<8>, dim3((unsigned)((A.rows * 8 + 255) / 256)), dim3(256), 0, st, A.rows, A.rowptr, A.col, A.val, X, ldx, U, ldu, split, Y, ldy, mode, zero_pad);
    return;
  }
  static const int vmode = [] {
    const char* e = getenv("NSP_SPMM_V");
    return e ? atoi(e) : 2;
  }();
  // 16-byte loads when every row segment is 16-byte aligned (even s, even strides)
  if (vmode == 2 && s % 2 == 0 && ldx % 2 == 0 && ldu % 2 == 0 && ucs % 2 == 0 && ldy % 2 == 0 && ycs % 2 == 0 &&
      ypad % 2 == 0 && s <= 256) {
    const int nq2 = (s + 63) / 64;
    if (nq2 == 1)
      { nsp_count_launch(); launch_k(k_spmm2<1>, dim3(blocks), dim3(256), 0, st, A.rows, A.rowptr, A.col, A.val, X, ldx, U, ldu, ucs, split, Y, ldy, ycs, ypad, s, mode, zero_pad, (const int*)nullptr, (const int*)nullptr, (int*)nullptr, 0); }
    else if (nq2 == 2)
      { nsp_count_launch(); launch_k(k_spmm2<2>, dim3(blocks), dim3(256), 0, st, A.rows, A.rowptr, A.col, A.val, X, ldx, U, ldu, ucs, split, Y, ldy, ycs, ypad, s, mode, zero_pad, (const int*)nullptr, (const int*)nullptr, (int*)nullptr, 0); }
    else
      { nsp_count_launch(); launch_k(k_spmm2<4>, dim3(blocks), dim3(256), 0, st, A.rows, A.rowptr, A.col, A.val, X, ldx, U, ldu, ucs, split, Y, ldy, ycs, ypad, s, mode, zero_pad, (const int*)nullptr, (const int*)nullptr, (int*)nullptr, 0); }
    return;
  }
  if (s <= 32)
    { nsp_count_launch(); launch_k(k_spmm<1>, dim3(blocks), dim3(256), 0, st, A.rows, A.rowptr, A.col, A.val, X, ldx, U, ldu, ucs, split, Y, ldy, ycs, ypad, s, mode, zero_pad); }
  else if (s <= 64)
    { nsp_count_launch(); launch_k(k_spmm<2>, dim3(blocks), dim3(256), 0, st, A.rows, A.rowptr, A.col, A.val, X, ldx, U, ldu, ucs, split, Y, ldy, ycs, ypad, s, mode, zero_pad); }
  else if (s <= 128)
    { nsp_count_launch(); launch_k(k_spmm<4>, dim3(blocks), dim3(256), 0, st, A.rows, A.rowptr, A.col, A.val, X, ldx, U, ldu, ucs, split, Y, ldy, ycs, ypad, s, mode, zero_pad); }
  else
    { nsp_count_launch(); launch_k(k_spmm<8>, dim3(blocks), dim3(256), 0, st, A.rows, A.rowptr, A.col, A.val, X, ldx, U, ldu, ucs, split, Y, ldy, ycs, ypad, s, mode, zero_pad); }
}

void spmm(const DevCSR& A, const double* X, int ldx, const double* U, int ldu, int64_t split, double* Y,
          int ldy, int s, int mode, bool zero_pad, cudaStream_t st) {
  spmm_cs(A, X, ldx, U, ldu, 32, split, Y, ldy, 32, ldy, s, mode, zero_pad, st);
}

void cheb_step(const DevCSR& A, int64_t split, const double* d, int ld, int s, double* x, double* r, double* dn,
               double c1, double c2, bool want_d, cudaStream_t st) {
  if (A.rows <= 0) return;
  if (s == 1 && ld == 1) {
    // lanes per row: cfg5 outer PCG (M_2, 91 its) 15.04 / 17.56 / 23.34 ms per iteration with 4 / 8 / 16
    // lanes (the unfused SpMV + update: 16.54 ms)
    static const int G = [] {
      const char* e = getenv("NSP_CHEB_G");
      const int g = e ? atoi(e) : 4;
      return (g == 2 || g == 8 || g == 16) ? g : 4;
    }();
    nsp_count_launch();
    if (G == 2)
      launch_k(k_cheb_step_vec<2>, dim3((unsigned)((A.rows * 2 + 255) / 256)), dim3(256), 0, st, A.rows, A.rowptr,
               A.col, A.val, split, d, x, r, dn, c1, c2, want_d ? 1 : 0);
    else if (G == 4)
      launch_k(k_cheb_step_vec<4>, dim3((unsigned)((A.rows * 4 + 255) / 256)), dim3(256), 0, st, A.rows, A.rowptr,
               A.col, A.val, split, d, x, r, dn, c1, c2, want_d ? 1 : 0);
    else if (G == 16)
      launch_k(k_cheb_step_vec<16>, dim3((unsigned)((A.rows * 16 + 255) / 256)), dim3(256), 0, st, A.rows, A.rowptr,
               A.col, A.val, split, d, x, r, dn, c1, c2, want_d ? 1 : 0);
    else
      launch_k(k_cheb_step_vec<8>, dim3((unsigned)((A.rows * 8 + 255) / 256)), dim3(256), 0, st, A.rows, A.rowptr,
               A.col, A.val, split, d, x, r, dn, c1, c2, want_d ? 1 : 0);
    return;
  }
  const unsigned blocks = (unsigned)((A.rows * 32 + 255) / 256);
  const int nq2 = (ld + 63) / 64;
  nsp_count_launch();
  if (nq2 <= 1)
    launch_k(k_cheb_step_blk<1>, dim3(blocks), dim3(256), 0, st, A.rows, A.rowptr, A.col, A.val, split, d, ld, x, r, dn, c1,
             c2, want_d ? 1 : 0);
  else if (nq2 == 2)
    launch_k(k_cheb_step_blk<2>, dim3(blocks), dim3(256), 0, st, A.rows, A.rowptr, A.col, A.val, split, d, ld, x, r, dn, c1,
             c2, want_d ? 1 : 0);
  else
    launch_k(k_cheb_step_blk<4>, dim3(blocks), dim3(256), 0, st, A.rows, A.rowptr, A.col, A.val, split, d, ld, x, r, dn, c1,
             c2, want_d ? 1 : 0);
}

void cheb3_step(const DevCSR& A, int64_t split, const double* xk, int ld, int s, const double* xp, const double* b,
                double* xn, double c1, double c2, cudaStream_t st, const int64_t* sptr, const int32_t* scol,
                const double* sval, const uint8_t* code, const double* tab) {
  if (A.rows <= 0 && !(s == 1 && sptr)) return;
  if (s == 1 && ld == 1) {
    const int64_t rows = split;
    nsp_count_launch();
    launch_k(k_cheb3_step_sell, dim3((unsigned)((rows + 255) / 256)), dim3(256), 0, st, rows, sptr, scol, sval, code,
             tab, xk, xp, b, xn, c1, c2);
    return;
  }
  const unsigned blocks = (unsigned)((A.rows * 32 + 255) / 256);
  const int nq2 = (ld + 63) / 64;
  nsp_count_launch();
  if (nq2 == 1)
    launch_k(k_cheb3_step_blk<1>, dim3(blocks), dim3(256), 0, st, A.rows, A.rowptr, A.col, A.val, split, xk, ld, xp, b,
             xn, c1, c2);
  else if (nq2 == 2)
    launch_k(k_cheb3_step_blk<2>, dim3(blocks), dim3(256), 0, st, A.rows, A.rowptr, A.col, A.val, split, xk, ld, xp, b,
             xn, c1, c2);
  else
    launch_k(k_cheb3_step_blk<4>, dim3(blocks), dim3(256), 0, st, A.rows, A.rowptr, A.col, A.val, split, xk, ld, xp, b,
             xn, c1, c2);
}

void cheb_step_sell(int64_t rows, const int64_t* sptr, const int32_t* col, const double* val, const double* d,
                    double* x, double* r, double* dn, double c1, double c2, bool want_d, cudaStream_t st,
                    const uint8_t* code, const double* tab) {
  if (rows <= 0) return;
  if (code && tab) {
    nsp_count_launch();
    launch_k(k_cheb_step_sell_dict, dim3((unsigned)((rows + 255) / 256)), dim3(256), 0, st, rows, sptr, col, code, tab,
             d, x, r, dn, c1, c2, want_d ? 1 : 0);
    return;
  }
  nsp_count_launch();
  launch_k(k_cheb_step_sell, dim3((unsigned)((rows + 255) / 256)), dim3(256), 0, st, rows, sptr, col, val, d, x, r, dn,
           c1, c2, want_d ? 1 : 0);
}

void philox_gaussian(double* out, int64_t rows, int s, int ld, const int64_t* gidx, uint64_t seed, uint32_t stream,
                     cudaStream_t st) {
  const int64_t tot = rows * ld;
  if (tot <= 0) return;
  nsp_count_launch();
  k_philox_gaussian<<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(out, rows, s, ld, gidx, seed, stream);
}

void band_prep(const double* T, int nt, int wb, double* XF, double* GF, double* XB, double* GB, cudaStream_t st) {
  if (nt <= 0) return;
  nsp_count_launch();
  k_band_prep<<<nt, 256, 0, st>>>(T, nt, wb, XF, GF, XB, GB);
}

void band_rec(const TriSys* sys, int nsys, const double* Xd, int64_t xstride, const double* Gc, double* buf, int ldw,
              bool fwd, cudaStream_t st) {
  if (nsys <= 0) return;
  // few independent sweeps: 16-wide column slices double the CTAs (as in tri_fb)
  if (nsys * (ldw / 32) < 2 * num_sms()) {
    const size_t smem = (4 * 64 * LDT + 4 * 64 * 20) * sizeof(double);
    smem_optin((const void*)k_band_rec<16>, (size_t)((int)smem));
    nsp_count_launch();
    launch_k(k_band_rec<16>, dim3(dim3(nsys, ldw / 16)), dim3(256), smem, st, sys, Xd, xstride, Gc, buf, ldw, fwd ? 1 : 0);
    return;
  }
  const size_t smem = (4 * 64 * LDT + 4 * 64 * 36) * sizeof(double);
  smem_optin((const void*)k_band_rec<32>, (size_t)((int)smem));
  nsp_count_launch();
  launch_k(k_band_rec<32>, dim3(dim3(nsys, ldw / 32)), dim3(256), smem, st, sys, Xd, xstride, Gc, buf, ldw, fwd ? 1 : 0);
}

void band_rec_vec(const TriSys* sys, int nsys, const double* Xd, int64_t xstride, const double* Gc, double* buf, bool fwd,
                  cudaStream_t st) {
  if (nsys <= 0) return;
  constexpr int NS = 3;
  const size_t smem = (NS * 8192 + NS * 64 + 2 * 64) * sizeof(double);
  smem_optin((const void*)k_band_rec_vec<NS>, (size_t)((int)smem));
  nsp_count_launch();
  launch_k(k_band_rec_vec<NS>, dim3(nsys), dim3(256), smem, st, sys, Xd, xstride, Gc, buf, fwd ? 1 : 0);
}

void tri_fb(const TriSys* sys, int nsys, double* buf, int ldw, int cw, bool fwd, bool bwd, cudaStream_t st,
            int wbmax) {
  if (nsys <= 0) return;
  dim3 grid(nsys, ldw / cw);
  if (wbmax >= 0 && wbmax <= 2 && cw == 1 && ldw == 1 && !getenv("NSP_NO_BAND")) {   // one column: matvec chain
    constexpr int NS = 4;
    const size_t smem = (NS * 4096 + NS * 64 + 3 * 64 + 4 * 64 + 64) * sizeof(double);
    smem_optin((const void*)k_band_fb_vec<NS, 2>, (size_t)((int)smem));
    { nsp_count_launch(); k_band_fb_vec<NS, 2><<<nsys, 256, smem, st>>>(sys, buf, fwd, bwd); }
    return;
  }
  if (cw == 1) cw = 32;   // generic kernels: at least one 32-wide column chunk
  grid = dim3(nsys, ldw >= 32 ? ldw / cw : 1);
  if (wbmax >= 0 && wbmax <= 2 && cw == 32 && nsys * (ldw / 32) < 2 * num_sms() && !getenv("NSP_NO_BAND")) {
    // few independent sweeps (e.g. the single A_G system): 16-wide column chunks double the CTAs
    constexpr int NS = 3;
    const size_t smem = (NS * 64 * LDT + NS * 64 * 20 + 3 * 64 * 20) * sizeof(double);
    smem_optin((const void*)k_band_fb<16, NS, 2>, (size_t)((int)smem));
    { nsp_count_launch(); k_band_fb<16, NS, 2><<<dim3(nsys, ldw / 16), 256, smem, st>>>(sys, buf, ldw, fwd, bwd); }
    return;
  }
  if (wbmax >= 0 && wbmax <= 2 && cw == 32 && !getenv("NSP_NO_BAND")) {   // narrow band: deep-prefetch kernel
    constexpr int NS = 3;
    const size_t smem = (NS * 64 * LDT + NS * 64 * 36 + 3 * 64 * 36) * sizeof(double);
    smem_optin((const void*)k_band_fb<32, NS, 2>, (size_t)((int)smem));
    { nsp_count_launch(); k_band_fb<32, NS, 2><<<grid, 256, smem, st>>>(sys, buf, ldw, fwd, bwd); }
    return;
  }
  if (cw == 64) {
    const size_t smem = (2 * 64 * LDT + 2 * 64 * (64 + 4)) * sizeof(double);
    smem_optin((const void*)k_tri_fb<64>, (size_t)((int)smem));
    { nsp_count_launch(); k_tri_fb<64><<<grid, 256, smem, st>>>(sys, buf, ldw, fwd, bwd); }
  } else {
    const size_t smem = (2 * 64 * LDT + 2 * 64 * (32 + 4)) * sizeof(double);
    smem_optin((const void*)k_tri_fb<32>, (size_t)((int)smem));
    { nsp_count_launch(); k_tri_fb<32><<<grid, 256, smem, st>>>(sys, buf, ldw, fwd, bwd); }
  }
}

void spike_tail(const double* spk, const int* chunk_first, int P, double* buf, int ldw, int s, bool fwd,
                cudaStream_t st) {
  if (P <= 1) return;
  const size_t smem = (64 * 65 + 64 * 33) * sizeof(double);
  smem_optin((const void*)k_spike_tail, (size_t)((int)smem));
    smem_optin((const void*)k_spike_update, (size_t)((int)smem));
  if (s == 1 && ldw == 1) {
    smem_optin((const void*)k_spike_tail_vec, (size_t)(3 * 4096 * 8));
    { nsp_count_launch(); launch_k(k_spike_tail_vec, dim3(1), dim3(256), 3 * 4096 * 8, st, spk, chunk_first, P, buf, fwd); }
    return;
  }
  if (ldw % 32 == 0 && !getenv("NSP_SPIKE_OLD")) {
    const size_t sm2 = (2 * 64 * LDT + 3 * 64 * 36) * sizeof(double);
    smem_optin((const void*)k_spike_tail_mma, (size_t)((int)sm2));
    { nsp_count_launch(); launch_k(k_spike_tail_mma, dim3(ldw / 32), dim3(256), sm2, st, spk, chunk_first, P, buf, ldw, fwd ? 1 : 0); }
    return;
  }
  { nsp_count_launch(); k_spike_tail<<<(s + 31) / 32, 256, smem, st>>>(spk, chunk_first, P, buf, ldw, s, fwd); }
}

void spike_update(const double* spk, const int* chunk_first, const int* tile_chunk, int P, int nt, double* buf,
                  int ldw, int s, bool fwd, cudaStream_t st) {
  if (P <= 1) return;
  if (s == 1 && ldw == 1) {
    { nsp_count_launch(); launch_k(k_spike_update_vec, dim3(nt), dim3(256), 0, st, spk, chunk_first, tile_chunk, P, buf, fwd); }
    return;
  }
  if (ldw % 32 == 0 && !getenv("NSP_SPIKE_OLD")) {
    const size_t sm2 = (64 * LDT + 64 * 36) * sizeof(double);
    smem_optin((const void*)k_spike_update_mma, (size_t)((int)sm2));
    { nsp_count_launch(); launch_k(k_spike_update_mma, dim3(nt, ldw / 32), dim3(256), sm2, st, spk, chunk_first, tile_chunk, P, buf, ldw, fwd ? 1 : 0); }
    return;
  }
  const size_t smem = (64 * 65 + 64 * 33) * sizeof(double);   // attribute set with k_spike_tail (called first)
  { nsp_count_launch(); k_spike_update<<<dim3(nt, (s + 31) / 32), 256, smem, st>>>(spk, chunk_first, tile_chunk, P,
                                                                                    buf, ldw, s, fwd); }
}

void gather_rows(const double* src, int lds, const int32_t* idx, int64_t rows, double* dst, int ldd, int s,
                 double scale, cudaStream_t st) {
  const int64_t tot = rows * ldd;
  if (tot <= 0) return;
  { nsp_count_launch(); launch_k(k_gather_rows, dim3((unsigned)((tot + 255) / 256)), dim3(256), 0, st, src, lds, idx, rows, dst, ldd, s, scale); }
}

void scatter_rows(const double* src, int lds, const int32_t* idx, int64_t rows, double* dst, int ldd, int s,
                  bool accumulate, cudaStream_t st) {
  const int64_t tot = rows * s;
  if (tot <= 0) return;
  { nsp_count_launch(); launch_k(k_scatter_rows, dim3((unsigned)((tot + 255) / 256)), dim3(256), 0, st, src, lds, idx, rows, dst, ldd, s, accumulate); }
}

void l22_inverse(const FacSub* subs, int nsub, int max_ntb, const double* dense, double* minv, cudaStream_t st) {
  if (nsub <= 0 || max_ntb <= 0) return;
  const size_t smem = (2 * 64 * LDT + 2 * 64 * 68) * sizeof(double);
  smem_optin((const void*)k_l22_inverse, (size_t)((int)smem));
  { nsp_count_launch(); k_l22_inverse<<<dim3(nsub, max_ntb), 256, smem, st>>>(subs, dense, minv); }
}

void symm(const FacSub* subs, const int2* items, int nitems, const double* minv, const double* W, double* U, int ldw,
          int cw, cudaStream_t st, int64_t cm_stride) {
  if (nitems <= 0) return;
  // 2 stages, one barrier per K step: the padded M tile by one bulk copy (TMA); the W tile by one bulk
  // copy too when W/U are chunk-major (cm_stride > 0: ldw = 36 per 32-column chunk), else by cp.async.
  // Measured on cfg2 shapes (tools/bench_symm_tma.cu): 135.1 us (both cp.async) -> 122.9 (TMA M) ->
  // 112.6 us (TMA M + W, 29.2 TFLOP/s); 64-wide / 3-stage / half-tile variants are slower.
  const size_t smem = 2 * (NSP_MINV_TILE + 64 * (cw + 4)) * sizeof(double);
  static const bool persist = [] {
    const char* e = getenv("NSP_SYMM_PERSIST");
    return e && e[0] == '1';
  }();
  if (cm_stride > 0 && persist) {   // persistent: 2 CTAs per SM over (item, chunk) units
    const size_t sm2 = 2 * (NSP_MINV_TILE + 64 * 36) * sizeof(double);
    smem_optin((const void*)k_symm_p<32>, sm2);
    const int nch = ldw / 32;
    const int64_t total = (int64_t)nitems * nch;
    const int grid = (int)std::min<int64_t>(total, 2 * (int64_t)num_sms());
    nsp_count_launch();
    launch_k(k_symm_p<32>, dim3(grid), dim3(256), sm2, st, subs, items, nitems, nch, minv, W, U, cm_stride);
    return;
  }
  if (cm_stride > 0) {   // ldw = the logical padded width (a multiple of 32), one CTA column per chunk
    const dim3 grid(ldw / 32, nitems);
    smem_optin((const void*)k_symm<32, true>, (size_t)((int)(2 * (NSP_MINV_TILE + 64 * 36) * sizeof(double))));
    { nsp_count_launch(); launch_k(k_symm<32, true>, grid, dim3(256), 2 * (NSP_MINV_TILE + 64 * 36) * sizeof(double), st, subs, items, minv, W, U, 36, cm_stride); }
    return;
  }
  dim3 grid(nitems, ldw / cw);
  if (cw == 64) {
    smem_optin((const void*)k_symm<64, false>, (size_t)((int)smem));
    { nsp_count_launch(); launch_k(k_symm<64, false>, dim3(grid), dim3(256), smem, st, subs, items, minv, W, U, ldw, (int64_t)0); }
  } else {
    smem_optin((const void*)k_symm<32, false>, (size_t)((int)smem));
    { nsp_count_launch(); launch_k(k_symm<32, false>, dim3(grid), dim3(256), smem, st, subs, items, minv, W, U, ldw, (int64_t)0); }
  }
}

void symv(const FacSub* subs, const int2* items, int nitems, int max_ntb, const double* minv, const double* W, int ldw,
          double* U, cudaStream_t st) {
  if (nitems <= 0) return;
  const size_t smem = (size_t)max_ntb * 64 * sizeof(double);
  if (smem > 48 * 1024) {
    static size_t attr = 0;
    if (attr < smem) {
      smem_optin((const void*)k_symv, (size_t)((int)smem));
      attr = smem;
    }
  }
  { nsp_count_launch(); k_symv<<<nitems, 256, smem, st>>>(subs, items, minv, W, ldw, U); }
}

void symv1(const FacSub* subs, const int2* items, int nitems, int max_ntb, const double* minv, const double* W, int ldw,
           double* U, double* P, cudaStream_t st) {
  if (nitems <= 0) return;
  const size_t smem = (size_t)max_ntb * 64 * sizeof(double);
  if (smem > 48 * 1024) {
    static size_t attr = 0;
    if (attr < smem) {
      smem_optin((const void*)k_symv1, (size_t)((int)smem));
      attr = smem;
    }
  }
  { nsp_count_launch(); launch_k(k_symv1, dim3(nitems), dim3(256), smem, st, subs, items, minv, W, ldw, max_ntb, P); }
  { nsp_count_launch(); launch_k(k_symv_reduce, dim3(nitems), dim3(64), 0, st, subs, items, max_ntb, P, U, ldw); }
}

void trsm_fb(const FacSub* subs, int nsub, const double* dense, double* wvu, int ldw, int cw, cudaStream_t st) {
  if (nsub <= 0) return;
  dim3 grid(nsub, ldw / cw);
  if (cw == 64) {
    const size_t smem = (2 * 64 * LDT + 2 * 64 * (64 + 4)) * sizeof(double);
    smem_optin((const void*)k_trsm_fb<64>, (size_t)((int)smem));
    { nsp_count_launch(); k_trsm_fb<64><<<grid, 256, smem, st>>>(subs, dense, wvu, ldw); }
  } else {
    const size_t smem = (2 * 64 * LDT + 2 * 64 * (32 + 4)) * sizeof(double);
    smem_optin((const void*)k_trsm_fb<32>, (size_t)((int)smem));
    { nsp_count_launch(); k_trsm_fb<32><<<grid, 256, smem, st>>>(subs, dense, wvu, ldw); }
  }
}

}  // namespace nspk
