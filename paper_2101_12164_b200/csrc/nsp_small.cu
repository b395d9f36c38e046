// a7 / a10 / a11 s x s Cholesky and its application (§8(a) rows a7, a10, a11; north_star (c) "small
// s x s Cholesky and solve kernels"), latency-oriented for s <= 128:
//  k_chol16   one CTA, 8 warps.  16-column blocks; the 16 x 16 diagonal block is factored by ONE warp
//             in registers (no CTA barrier inside) together with X_kk = L_kk^{-1}; the panel
//             L_ik = A_ik X_kk^T and the rank-16 trailing update run on the DMMA pipe.  Look-ahead:
//             warp 0 updates and factors the NEXT diagonal block while warps 1-7 finish the trailing
//             update, so the serial chain per block is one warp factorisation + the panel.  The
//             diagonal factorisation has a single call site (instruction-cache friendly).
//  k_chol_solve  sp/8 CTAs, each solving for 8 right-hand-side columns with L staged in shared
//             memory; 16-row blocks, the diagonal block as a product with X_kk, the off-diagonal
//             updates on the DMMA pipe.
// Pivot semantics follow reading C3 (orth: min pivot > tau * max pivot) and SPEC.md:263 (D: a
// pivot <= 0 is an indefinite search space).
#include <cuda_runtime.h>
#include <stdint.h>

#include "nsp_blas.h"
#include "../../include/nsp.h"
#include "nsp_dmma.cuh"

using namespace nspd;

namespace {

constexpr int LDA = 132;   // smem row stride of the s x s matrix

__device__ __forceinline__ double rsqrt_nr(double d) {
  double r;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(d));
  const double h = 0.5 * d;
  r = r * fma(-h * r, r, 1.5);
  r = r * fma(-h * r, r, 1.5);
  return r;
}

#ifdef NSP_CHOL_PROF
__device__ long long g_chol_prof[128];
#define CPROF(i) \
  if (threadIdx.x == 0) g_chol_prof[i] = clock64();
#else
#define CPROF(i)
#endif
#ifdef NSP_CHOL_PROF
#define WPROF(k) \
  if (lane == 0 && c0 == 16) g_chol_prof[64 + (k)] = clock64();
#else
#define WPROF(k)
#endif

// One warp: factor the 16 x 16 diagonal block at (c0, c0) of As in place (lower = L), write
// X = L^{-1} (16 x 16 row-major, lower) to Xd and the pivots (before the square root) to piv.  A
// non-positive pivot is replaced by 1 (deterministic continuation) and reported by `false`.
// Lane l holds row l >> 1, columns 8 (l & 1) .. + 7 in registers.
__device__ __noinline__ bool warp_chol16(double* As, int c0, double* Xd, double* piv, double* colv, double* invd) {
  const int lane = threadIdx.x & 31;
  const int r = lane >> 1, h = lane & 1;
  double* B = As + c0 * LDA + c0;
  WPROF(0)
  double v[8];
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const int j = 8 * h + q;
    v[q] = (j <= r) ? B[r * LDA + j] : 0.0;
  }
  bool ok = true;
  WPROF(1)
#ifndef NSP_CHOL_NOPIPE
  // software-pipelined: the owner of row c+1 forms the next pivot from its own registers right after
  // column c is scaled (d_{c+1} = a_{c+1,c+1} - l_{c+1,c}^2, bitwise the value the trailing update
  // below produces), so the next pivot broadcast + rsqrt overlap this column's smem broadcast/update.
  double d = __shfl_sync(0xffffffffu, v[0], 0);
#pragma unroll
  for (int c = 0; c < 16; ++c) {
    const int hc = c >> 3, qc = c & 7;
    const double held = v[qc];
    if (lane == 0) piv[c0 + c] = d;
    if (!(d > 0.0)) {
      ok = false;
      d = 1.0;
    }
    const double rs = rsqrt_nr(d);
    double lv = 0.0;   // L(r, c) on the lanes holding column c (zero above the diagonal)
    if (h == hc) lv = (r > c) ? held * rs : ((r == c) ? d * rs : 0.0);
    double dnext = 0.0;
    if (c < 15) {
      const int c1 = c + 1, h1 = c1 >> 3, q1 = c1 & 7;
      const double l1 = __shfl_sync(0xffffffffu, lv, 2 * c1 + hc);    // L(c+1, c)
      const double dn = fma(-l1, l1, v[q1]);                           // valid on lane 2(c+1)+h1
      dnext = __shfl_sync(0xffffffffu, dn, 2 * c1 + h1);
    }
    if (h == hc) {
      if (r >= c) v[qc] = lv;
      colv[r] = lv;
    }
    if (lane == 0) invd[c] = rs;
    __syncwarp();
    const double li = colv[r];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int j = 8 * h + q;
      if (j > c && j <= r) v[q] = fma(-li, colv[j], v[q]);
    }
    __syncwarp();
    d = dnext;
  }
#else
#pragma unroll
  for (int c = 0; c < 16; ++c) {
    const int hc = c >> 3, qc = c & 7;
    const double held = v[qc];
    double d = __shfl_sync(0xffffffffu, held, 2 * c + hc);
    if (lane == 0) piv[c0 + c] = d;
    if (!(d > 0.0)) {
      ok = false;
      d = 1.0;
    }
    const double rs = rsqrt_nr(d);
    if (h == hc) {
      if (r > c) v[qc] = held * rs;
      else if (r == c) v[qc] = d * rs;
      colv[r] = (r >= c) ? v[qc] : 0.0;
    }
    if (lane == 0) invd[c] = rs;
    __syncwarp();
    const double li = colv[r];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int j = 8 * h + q;
      if (j > c && j <= r) v[q] = fma(-li, colv[j], v[q]);
    }
    __syncwarp();
  }
#endif
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const int j = 8 * h + q;
    if (j <= r) B[r * LDA + j] = v[q];
  }
  __syncwarp();
  WPROF(2)
  // X = L^{-1} by 8 x 8 blocks: lanes 0-7 / 8-15 invert L11 / L22 (one column each), then
  // X21 = -X22 (L21 X11) on all 32 lanes (two entries each)
  if (lane < 16) {
    const int blk = lane >> 3, j = lane & 7, o = 8 * blk;
    double x[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      double s = (i == j) ? 1.0 : 0.0;
#pragma unroll
      for (int k = 0; k < i; ++k)
        if (k >= j) s = fma(-B[(o + i) * LDA + o + k], x[k], s);
      x[i] = (i >= j) ? s * invd[o + i] : 0.0;
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      Xd[(o + i) * 16 + o + j] = x[i];
      Xd[(o + i) * 16 + 8 * (1 - blk) + j] = 0.0;
    }
  }
  __syncwarp();
  {
    const int i = lane >> 2, jj = 2 * (lane & 3);
    double m0 = 0.0, m1 = 0.0;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const double l = B[(8 + i) * LDA + k];
      m0 = fma(l, Xd[k * 16 + jj], m0);
      m1 = fma(l, Xd[k * 16 + jj + 1], m1);
    }
    __syncwarp();
    Xd[(8 + i) * 16 + jj] = m0;
    Xd[(8 + i) * 16 + jj + 1] = m1;
    __syncwarp();
    double x0 = 0.0, x1 = 0.0;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const double xk = Xd[(8 + i) * 16 + 8 + k];
      x0 = fma(xk, Xd[(8 + k) * 16 + jj], x0);
      x1 = fma(xk, Xd[(8 + k) * 16 + jj + 1], x1);
    }
    __syncwarp();
    Xd[(8 + i) * 16 + jj] = -x0;
    Xd[(8 + i) * 16 + jj + 1] = -x1;
  }
  __syncwarp();
  WPROF(3)
  return ok;
}


// One THREAD: factor the 8 x 8 lower block at B (ld LDA) in registers - pivots (before the square root)
// to piv, L in place (lower), X = L^{-1} (lower, zeros above) to Xo (ld 16).  A non-positive pivot is
// replaced by 1 (deterministic continuation) and reported by `false`.  The dependency chain per column
// is one reciprocal square root and one update (no shuffles, no shared-memory round trips).
__device__ __forceinline__ bool fac8(double* B, double* Xo, double* piv) {
  double a[8][8], x[8][8], il[8];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) a[i][j] = (j <= i) ? B[i * LDA + j] : 0.0;
  bool ok = true;
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    double d = a[c][c];
    piv[c] = d;
    if (!(d > 0.0)) {
      ok = false;
      d = 1.0;
    }
    const double r = rsqrt_nr(d);
    il[c] = r;
    a[c][c] = d * r;
#pragma unroll
    for (int i = c + 1; i < 8; ++i) a[i][c] *= r;
#pragma unroll
    for (int j = c + 1; j < 8; ++j)
#pragma unroll
      for (int i = j; i < 8; ++i) a[i][j] = fma(-a[i][c], a[j][c], a[i][j]);
  }
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
      if (j <= i) B[i * LDA + j] = a[i][j];
      Xo[i * 16 + j] = (j <= i) ? x[i][j] : 0.0;
    }
  return ok;
}

// Warp 0: the 16 x 16 diagonal block at (c0, c0) as 2 x 2 blocks of 8 - L11 by one thread (fac8),
// L21 = A21 X11^T and A22 - L21 L21^T row-parallel on 8 lanes, L22 by one thread, X21 = -X22 L21 X11
// row-parallel.  Same outputs as warp_chol16: L in place (lower), X = L^{-1} to Xd (16 x 16 row-major,
// zero above the diagonal), pivots to piv.  Kept behind NSP_CHOL_FAST8: measured SLOWER than the
// warp-wide column loop (a 128 x 128 factorisation 94.2k vs 67.9k cycles, gpurun_out r02b) - one
// thread's dependent fp64 chain (rsqrt + Newton, the 8 x 8 inverse) costs more than the warp's
// shuffles.
__device__ __noinline__ bool diag16_fast(double* As, int c0, double* Xd, double* piv) {
  const int lane = threadIdx.x & 31;
  double* B = As + c0 * LDA + c0;
  int ok = 1;
  if (lane == 0) ok = fac8(B, Xd, piv + c0);
  __syncwarp();
  double l[8];
  if (lane < 8) {   // row 8 + lane of L21 = A21 X11^T
    double a[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) a[k] = B[(8 + lane) * LDA + k];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      double s = 0.0;
#pragma unroll
      for (int k = 0; k <= j; ++k) s = fma(a[k], Xd[j * 16 + k], s);
      l[j] = s;
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) B[(8 + lane) * LDA + j] = l[j];
  }
  __syncwarp();
  if (lane < 8) {   // A22[lane][j] -= L21[lane] . L21[j], j <= lane
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      if (j <= lane) {
        double s = 0.0;
#pragma unroll
        for (int k = 0; k < 8; ++k) s = fma(l[k], B[(8 + j) * LDA + k], s);
        B[(8 + lane) * LDA + 8 + j] -= s;
      }
    }
  }
  __syncwarp();
  if (lane == 0) ok &= fac8(B + 8 * LDA + 8, Xd + 8 * 16 + 8, piv + c0 + 8) ? 1 : 0;
  __syncwarp();
  if (lane < 8) {   // T = L21 X11 (row lane), then X21 = -X22 T
    double tr[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      double s = 0.0;
#pragma unroll
      for (int k = j; k < 8; ++k) s = fma(l[k], Xd[k * 16 + j], s);
      tr[j] = s;
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) Xd[(8 + lane) * 16 + j] = tr[j];   // T row (the X21 slot, overwritten below)
  }
  __syncwarp();
  double xr[8];
  if (lane < 8) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      double s = 0.0;
#pragma unroll
      for (int m = 0; m <= lane; ++m) s = fma(Xd[(8 + lane) * 16 + 8 + m], Xd[(8 + m) * 16 + j], s);
      xr[j] = -s;
    }
  }
  __syncwarp();
  if (lane < 8) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      Xd[(8 + lane) * 16 + j] = xr[j];
      Xd[lane * 16 + 8 + j] = 0.0;
    }
  }
  __syncwarp();
  return __shfl_sync(0xffffffffu, ok, 0) != 0;
}

// Output Lp (sp x sp): strictly-lower off-diagonal blocks = L, diagonal 16 x 16 blocks = X_kk
// (lower, zero above the diagonal); the strictly-upper 16 x 16 blocks are NOT written.  Rows / cols >= nact (nact < 0: st->width) are replaced by the identity.
//  mode 0: a pivot <= 0 -> st->indefinite.
//  mode 1: pivot test min d_i > tau max d_i over i < nact (reading C3), else st->fallback = 1;
//          success: st->fallback = 0, st->width = nact.
#ifndef NSP_CF_T
#define NSP_CF_T 256
#endif
constexpr int CF_T = NSP_CF_T;   // threads per k_chol16 CTA (512 measured slower: 35.4 -> 36.7 us)
// Solve for the 8 right-hand-side columns c0.. of op(B) with L staged in shared memory (Ls, ld LD:
// strictly-lower blocks = L, diagonal 16 x 16 blocks = X_kk = L_kk^{-1}), x: sp x 8 (ld 10) staging;
// Out[:, c0..c0+8) = sgn * op(B).  op = L^{-T} L^{-1} (fwd && bwd), L^{-1} (fwd), L^{-T} (bwd); B == nullptr:
// the identity.  Per 16-row block: x_kb <- X_kk x_kb (warps 0, 1), then the other rows' updates on the
// DMMA pipe (8-row groups over the CTA's warps).  NT threads.
template <int NT>
__device__ __forceinline__ void solve8(const double* Ls, int LD, double* x, int sp, const double* __restrict__ B,
                                       int ldb, double* __restrict__ Out, int ldo, double sgn, int fwd, int bwd,
                                       int c0) {
  constexpr int LX = 10;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, t = lane & 3;
  const int NB = sp / 16;
  if (fwd)
    for (int kb = 0; kb < NB; ++kb) {
      const int b0 = 16 * kb;
      double d0 = 0.0, d1 = 0.0;
      if (warp < 2) {
#pragma unroll
        for (int k = 0; k < 16; k += 4)
          dmma(d0, d1, Ls[(b0 + 8 * warp + g) * LD + b0 + k + t], x[(b0 + k + t) * LX + g]);
      }
      __syncthreads();
      if (warp < 2) {
        x[(b0 + 8 * warp + g) * LX + 2 * t] = d0;
        x[(b0 + 8 * warp + g) * LX + 2 * t + 1] = d1;
      }
      __syncthreads();
      for (int grp = warp; grp < (sp - b0 - 16) / 8; grp += NT / 32) {
        const int row0 = b0 + 16 + 8 * grp;
        double a0 = 0.0, a1 = 0.0;
#pragma unroll
        for (int k = 0; k < 16; k += 4) dmma(a0, a1, Ls[(row0 + g) * LD + b0 + k + t], x[(b0 + k + t) * LX + g]);
        x[(row0 + g) * LX + 2 * t] -= a0;
        x[(row0 + g) * LX + 2 * t + 1] -= a1;
      }
      __syncthreads();
    }
  if (bwd)
    for (int kb = NB - 1; kb >= 0; --kb) {
      const int b0 = 16 * kb;
      double d0 = 0.0, d1 = 0.0;
      if (warp < 2) {
#pragma unroll
        for (int k = 0; k < 16; k += 4)
          dmma(d0, d1, Ls[(b0 + k + t) * LD + b0 + 8 * warp + g], x[(b0 + k + t) * LX + g]);
      }
      __syncthreads();
      if (warp < 2) {
        x[(b0 + 8 * warp + g) * LX + 2 * t] = d0;
        x[(b0 + 8 * warp + g) * LX + 2 * t + 1] = d1;
      }
      __syncthreads();
      for (int grp = warp; grp < b0 / 8; grp += NT / 32) {
        const int row0 = 8 * grp;
        double a0 = 0.0, a1 = 0.0;
#pragma unroll
        for (int k = 0; k < 16; k += 4) dmma(a0, a1, Ls[(b0 + k + t) * LD + row0 + g], x[(b0 + k + t) * LX + g]);
        x[(row0 + g) * LX + 2 * t] -= a0;
        x[(row0 + g) * LX + 2 * t + 1] -= a1;
      }
      __syncthreads();
    }
  for (int e = tid; e < sp * 8; e += NT) {
    const int i = e >> 3, cc = e & 7;
    Out[(int64_t)i * ldo + c0 + cc] = sgn * x[i * LX + cc];
  }
}

// Fused s x s Cholesky + solve (sxs.Out != nullptr): the grid's sp / 8 CTAs each run the IDENTICAL
// factorisation (same instructions on the same data - bitwise the same factor) and then solve for
// their own 8 right-hand-side columns with the factor still in shared memory, so the solve needs no
// second launch and no factor round trip; CTA 0 alone writes Lp and the status.  Skipped (no output)
// when the factorisation fails (mode 0) or the pivot test sends orth to the eigen fallback (mode 1).
struct SxsSolve {
  const double* B;
  int ldb;
  double* Out;
  int ldo;
  double sgn;
  int fwd, bwd;
};

__global__ void __launch_bounds__(CF_T) k_chol16(const double* __restrict__ Ain, int sp, int mode, int nact,
                                                double tau, double* __restrict__ Lp, BcgStatus* st, SxsSolve sxs) {
  pdl_wait();
  extern __shared__ double sm[];
  double* As = sm;                 // 128 x LDA
  double* Di = sm + 128 * LDA;     // 8 x 256: X_kk
  double* xs = Di + 8 * 256;       // fused solve: sp x 10 right-hand-side staging
  const bool lead = blockIdx.x == 0;
  __shared__ double piv[128];
  __shared__ double colv[16], invd[16];
  __shared__ int s_fail, s_skip;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, t = lane & 3;
  const int width = nact < 0 ? st->width : nact;
  const int NB = sp / 16;
  CPROF(0)
  {  // one bulk copy (TMA) per row of the lower triangle, all on one mbarrier, then the identity fix-up
    __shared__ __align__(8) uint64_t lbar;
    if (tid == 0) {
      mbar_init(&lbar, sp);
      fence_mbar_init();
    }
    __syncthreads();
    if (tid < sp) mbar_expect_copy(&lbar, As + tid * LDA, Ain + (int64_t)tid * sp, 8u * ((tid + 2) & ~1));
    mbar_wait(&lbar, 0);
    __syncthreads();
    if (width < sp)
      for (int e = tid; e < sp * sp; e += CF_T) {
        const int i = e / sp, j = e - i * sp;
        if (j <= i && (i >= width || j >= width)) As[i * LDA + j] = (i == j) ? 1.0 : 0.0;
      }
  }
  if (tid == 0) s_fail = 0;
  __syncthreads();
  CPROF(1)
  auto tile_update = [&](int I, int J, int c0) {   // A_IJ -= L_I,kb L_J,kb^T (8 x 8, k = 16)
    double c0v = 0.0, c1v = 0.0;
#pragma unroll
    for (int k = 0; k < 16; k += 4)
      dmma(c0v, c1v, As[(8 * I + g) * LDA + c0 + k + t], As[(8 * J + g) * LDA + c0 + k + t]);
    double* dst = As + (8 * I + g) * LDA + 8 * J + 2 * t;
    dst[0] -= c0v;
    dst[1] -= c1v;
  };
  for (int step = 0; step < NB; ++step) {
    // (C) trailing update with panel step-1; warp 0: next diagonal block first, then factor it (A)
    if (step > 0) {
      const int kb = step - 1, c0 = 16 * kb;
      const int b8 = 2 * step, m = 2 * NB - b8;
      if (warp == 0) {
        tile_update(b8, b8, c0);
        tile_update(b8 + 1, b8, c0);
        tile_update(b8 + 1, b8 + 1, c0);
        __syncwarp();
      } else {
        const int ntile = m * (m + 1) / 2;
        for (int task = warp - 1; task < ntile; task += CF_T / 32 - 1) {
          int q = (int)((sqrtf(8.0f * task + 1.0f) - 1.0f) * 0.5f);
          while (q * (q + 1) / 2 > task) --q;
          while ((q + 1) * (q + 2) / 2 <= task) ++q;
          const int p = task - q * (q + 1) / 2;
          if (q <= 1) continue;   // tiles of the next diagonal block: warp 0
          tile_update(b8 + q, b8 + p, c0);
        }
      }
    }
    if (warp == 0) {   // (A) the only call site of the diagonal factorisation
#ifdef NSP_CHOL_FAST8   // measured slower (tools/bench_chol16.cu: 94.2k vs 67.9k cycles per 128 x 128)
      const bool ok = diag16_fast(As, 16 * step, Di + step * 256, piv);
#else
      const bool ok = warp_chol16(As, 16 * step, Di + step * 256, piv, colv, invd);
#endif
      if (!ok && lane == 0) s_fail = 1;
    }
    __syncthreads();
    CPROF(2 + 2 * step)
    if (s_fail) break;
    // (B) panel: L_ik = A_ik X_kk^T for the rows below the block, 8-row groups, in place
    const int c0 = 16 * step;
    const int ngrp = (sp - c0 - 16) / 8;
    for (int grp = warp; grp < ngrp; grp += CF_T / 32) {
      const int row0 = c0 + 16 + 8 * grp;
      double acc[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
#pragma unroll
      for (int k = 0; k < 16; k += 4) {
        const double a = As[(row0 + g) * LDA + c0 + k + t];
#pragma unroll
        for (int nf = 0; nf < 2; ++nf) dmma(acc[nf][0], acc[nf][1], a, Di[step * 256 + (nf * 8 + g) * 16 + k + t]);
      }
      __syncwarp();
#pragma unroll
      for (int nf = 0; nf < 2; ++nf) {
        As[(row0 + g) * LDA + c0 + nf * 8 + 2 * t] = acc[nf][0];
        As[(row0 + g) * LDA + c0 + nf * 8 + 2 * t + 1] = acc[nf][1];
      }
    }
    __syncthreads();
    CPROF(3 + 2 * step)
  }
  if (warp == 0) {   // status: warp-parallel min / max of the pivots
    if (mode == 0) {
      if (lane == 0) s_skip = s_fail;
      if (lane == 0 && s_fail && lead) st->indefinite = 1;
    } else {
      double mn = 1e308, mx = 0.0;
      for (int i = lane; i < width; i += 32) {
        mn = fmin(mn, piv[i]);
        mx = fmax(mx, piv[i]);
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        mn = fmin(mn, __shfl_xor_sync(0xffffffffu, mn, o));
        mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
      }
      if (lane == 0) {
        const bool fb = s_fail != 0 || !(mn > tau * mx);
        s_skip = fb ? 1 : 0;
        if (lead) {
          st->fallback = fb ? 1 : 0;
          if (!fb) st->width = width;
        }
      }
    }
  }
  // output: X_kk (zero above its diagonal) overwrites L_kk in As, then every row's stored part
  // (columns < 16 (bi + 1); the strictly-upper blocks are not written) leaves by one bulk copy
  for (int e = tid; e < NB * 256; e += CF_T) {
    const int b = e >> 8, r = (e >> 4) & 15, c2 = e & 15;
    As[(16 * b + r) * LDA + 16 * b + c2] = c2 <= r ? Di[b * 256 + r * 16 + c2] : 0.0;
  }
  fence_proxy_async();
  __syncthreads();
  if (lead && tid < sp) bulk_store(Lp + (int64_t)tid * sp, As + tid * LDA, 16u * ((tid >> 4) + 1) * 8u);
  if (sxs.Out && !s_skip) {   // fused solve for this CTA's 8 columns (As is only read from here on)
    const int c0 = blockIdx.x * 8;
    for (int e = tid; e < sp * 8; e += CF_T) {
      const int i = e >> 3, c = e & 7;
      xs[i * 10 + c] = sxs.B ? sxs.B[(int64_t)i * sxs.ldb + c0 + c] : (i == c0 + c ? 1.0 : 0.0);
    }
    __syncthreads();
    solve8<CF_T>(As, LDA, xs, sp, sxs.B, sxs.ldb, sxs.Out, sxs.ldo, sxs.sgn, sxs.fwd, sxs.bwd, c0);
  }
  if (lead && tid < sp) bulk_store_commit_wait();
  CPROF(40)
}

// Out[:, 8b..8b+8) = sgn * op(B)[:, 8b..8b+8), op = L^{-T} L^{-1} (fwd && bwd), L^{-1} (fwd) or L^{-T}
// (bwd); B == nullptr: the identity.  One CTA (4 warps) per 8 right-hand-side columns.  Lp staged
// in smem; per 16-row block: x_kb <- X_kk x_kb (16 x 16 x 8 product, 2 DMMA m-fragments), then
// the remaining rows x_i -= L_i,kb x_kb on the DMMA pipe (8-row fragments over the 4 warps).
// gate (optional): skip when *gate != 0.
#ifndef NSP_CS_T
#define NSP_CS_T 256
#endif
constexpr int CS_T = NSP_CS_T;   // threads per k_chol_solve CTA (8 warps: the rows-below updates in 2 rounds)
__global__ void __launch_bounds__(CS_T) k_chol_solve(const double* __restrict__ Lp, int sp,
                                                    const double* __restrict__ B, int ldb, double* __restrict__ Out,
                                                    int ldo, double sgn, int fwd, int bwd, const int* gate) {
  pdl_wait();
  if (gate && *gate) return;
  extern __shared__ double sm[];
  const int LD = sp + 2;
  double* Ls = sm;                 // sp x LD (zero above the diagonal)
  double* x = sm + sp * LD;        // sp x 8 (+pad 2 -> ld 10)
  constexpr int LX = 10;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, t = lane & 3;
  const int c0 = blockIdx.x * 8;
  // Lp row i up to the end of its diagonal block by one bulk copy (TMA, one mbarrier); the columns
  // beyond (the strictly-upper blocks, never written by k_chol16) are zero-filled
  __shared__ __align__(8) uint64_t lbar;
  if (tid == 0) {
    mbar_init(&lbar, sp);
    fence_mbar_init();
  }
  __syncthreads();
  for (int i = tid; i < sp; i += CS_T) {
    const int w = 16 * ((i >> 4) + 1);
    mbar_expect_copy(&lbar, Ls + i * LD, Lp + (int64_t)i * sp, 8u * w);
    for (int j = w; j < sp; ++j) Ls[i * LD + j] = 0.0;
  }
  for (int e = tid; e < sp * 8; e += CS_T) {
    const int i = e >> 3, c = e & 7;
    x[i * LX + c] = B ? B[(int64_t)i * ldb + c0 + c] : (i == c0 + c ? 1.0 : 0.0);
  }
  mbar_wait(&lbar, 0);
  __syncthreads();
  const int NB = sp / 16;
  if (fwd)
    for (int kb = 0; kb < NB; ++kb) {
      const int b0 = 16 * kb;
      // x_kb <- X_kk x_kb : warps 0, 1 take the two 8-row halves (m8 n8 k16)
      double d0 = 0.0, d1 = 0.0;
      if (warp < 2) {
#pragma unroll
        for (int k = 0; k < 16; k += 4)
          dmma(d0, d1, Ls[(b0 + 8 * warp + g) * LD + b0 + k + t], x[(b0 + k + t) * LX + g]);
      }
      __syncthreads();
      if (warp < 2) {
        x[(b0 + 8 * warp + g) * LX + 2 * t] = d0;
        x[(b0 + 8 * warp + g) * LX + 2 * t + 1] = d1;
      }
      __syncthreads();
      // x_i -= L_i,kb x_kb for the rows below, 8-row groups
      for (int grp = warp; grp < (sp - b0 - 16) / 8; grp += CS_T / 32) {
        const int row0 = b0 + 16 + 8 * grp;
        double a0 = 0.0, a1 = 0.0;
#pragma unroll
        for (int k = 0; k < 16; k += 4)
          dmma(a0, a1, Ls[(row0 + g) * LD + b0 + k + t], x[(b0 + k + t) * LX + g]);
        x[(row0 + g) * LX + 2 * t] -= a0;
        x[(row0 + g) * LX + 2 * t + 1] -= a1;
      }
      __syncthreads();
    }
  if (bwd)
    for (int kb = NB - 1; kb >= 0; --kb) {
      const int b0 = 16 * kb;
      // x_kb <- X_kk^T x_kb
      double d0 = 0.0, d1 = 0.0;
      if (warp < 2) {
#pragma unroll
        for (int k = 0; k < 16; k += 4)
          dmma(d0, d1, Ls[(b0 + k + t) * LD + b0 + 8 * warp + g], x[(b0 + k + t) * LX + g]);
      }
      __syncthreads();
      if (warp < 2) {
        x[(b0 + 8 * warp + g) * LX + 2 * t] = d0;
        x[(b0 + 8 * warp + g) * LX + 2 * t + 1] = d1;
      }
      __syncthreads();
      // x_i -= L_kb,i^T x_kb for the rows above
      for (int grp = warp; grp < b0 / 8; grp += CS_T / 32) {
        const int row0 = 8 * grp;
        double a0 = 0.0, a1 = 0.0;
#pragma unroll
        for (int k = 0; k < 16; k += 4)
          dmma(a0, a1, Ls[(b0 + k + t) * LD + row0 + g], x[(b0 + k + t) * LX + g]);
        x[(row0 + g) * LX + 2 * t] -= a0;
        x[(row0 + g) * LX + 2 * t + 1] -= a1;
      }
      __syncthreads();
    }
  for (int e = tid; e < sp * 8; e += CS_T) {
    const int i = e >> 3, cc = e & 7;
    Out[(int64_t)i * ldo + c0 + cc] = sgn * x[i * LX + cc];
  }
}

}  // namespace

namespace nspb {

void chol_fac(const double* A, int sp, int mode, int nact, double tau, double* Lp, BcgStatus* stt, cudaStream_t st) {
  // sp = s rounded up to 64 (the block-CG padding): 64 or 128
  const size_t smem = (size_t)(128 * LDA + 8 * 256 + 128 * 10) * sizeof(double);
  smem_optin((const void*)k_chol16, smem);
  nsp_count_launch();
  launch_k(k_chol16, dim3(1), dim3(CF_T), smem, st, A, sp, mode, nact, tau, Lp, stt, SxsSolve{});
}

void chol_fac_solve(const double* A, int sp, int mode, int nact, double tau, double* Lp, BcgStatus* stt,
                    const double* B, int ldb, double* Out, int ldo, double sgn, bool fwd, bool bwd, cudaStream_t st) {
  const size_t smem = (size_t)(128 * LDA + 8 * 256 + 128 * 10) * sizeof(double);
  smem_optin((const void*)k_chol16, smem);
  nsp_count_launch();
  nsp_count_path(NSP_PATH_CHOL_SOLVE);
  launch_k(k_chol16, dim3(sp / 8), dim3(CF_T), smem, st, A, sp, mode, nact, tau, Lp, stt,
           SxsSolve{B, ldb, Out, ldo, sgn, fwd ? 1 : 0, bwd ? 1 : 0});
}

void chol_solve(const double* Lp, int sp, const double* B, int ldb, double* Out, int ldo, double sgn, bool fwd,
                bool bwd, const int* gate, cudaStream_t st) {
  const size_t smem = (size_t)(sp * (sp + 2) + sp * 10) * sizeof(double);
  smem_optin((const void*)k_chol_solve, (size_t)((int)((128 * 130 + 128 * 10) * sizeof(double))));
  nsp_count_launch();
  launch_k(k_chol_solve, dim3(sp / 8), dim3(CS_T), smem, st, Lp, sp, B, ldb, Out, ldo, sgn, fwd, bwd, gate);
}

}  // namespace nspb
