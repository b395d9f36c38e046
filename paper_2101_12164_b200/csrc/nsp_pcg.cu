// Outer PCG on the border system and the full solve of A x = b (§8(a) row d3):
//   f   = b_G - A_GI A_I^{-1} b_I                       (eq:A_LDLT PAPER.md:381-385, eq:Sx=b PAPER.md:415-420)
//   w   = PCG(S_G, f, M),  M in {I, A_G^{-1} (eq:S1), M_2 = A_G^{-1} + Z Sigma Z^T (eq:left_prec_mat)}
//   x_I = A_I^{-1} (b_I - A_IG w),  x_G = w,  un-permuted to the original order.
// PCG is the textbook preconditioned CG, x_0 = 0, stopping on the recurrence residual
// ||r_k|| / ||f|| <= tol (reading C9); iteration count = S_G applications.
//
// A_I_j^{-1} on a full interior vector uses the block elimination of the setup's ordering
// (I1 = interior rows, B = boundary layer, L22 L22^T = A_BB - A_B1 A_11^{-1} A_1B):
//   y_B = L22^{-T} L22^{-1} (r_B - A_B1 A_11^{-1} r_1),   y_1 = A_11^{-1} (r_1 - A_1B y_B)
// with A_11^{-1} the band factor (k_tri_fb) and L22 the dense trailing factor (k_trsm_fb).
// Every scalar of the iteration stays on the device; one small status read per iteration.
// All reductions are fixed-order two-stage (no fp64 atomics; reading C17).
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <cstring>

#include "nsp_blas.h"
#include "nsp_dmma.cuh"
#include "nsp_solver.h"
#include "nsp_comm.h"

using nspd::launch_k;
using nspd::pdl_wait;

namespace {

constexpr int RT = 256;             // threads per reduction CTA
constexpr int RPB = 512;            // rows per partial-sum chunk (2 per thread: many CTAs, short chains)
constexpr int GT_ROWS = 64;         // rows per Z^T r chunk
constexpr int PCG_CHUNK = 8;        // PCG iterations per host status check (one CUDA graph)

// part[b*2 + q] = sum over chunk b of a_q . b_q (q = 0, 1; a2 may be null)
__global__ void __launch_bounds__(RT) k_dot2_partial(const double* __restrict__ a1, const double* __restrict__ b1,
                                                     const double* __restrict__ a2, const double* __restrict__ b2,
                                                     int64_t n, double* __restrict__ part) {
  pdl_wait();
  __shared__ double red[2][RT];
  const int64_t r0 = (int64_t)blockIdx.x * RPB;
  double s1 = 0.0, s2 = 0.0;
  for (int64_t r = r0 + threadIdx.x; r < min(n, r0 + RPB); r += RT) {
    s1 = fma(a1[r], b1[r], s1);
    if (a2) s2 = fma(a2[r], b2[r], s2);
  }
  red[0][threadIdx.x] = s1;
  red[1][threadIdx.x] = s2;
  __syncthreads();
  for (int w = RT / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w) {
      red[0][threadIdx.x] += red[0][threadIdx.x + w];
      red[1][threadIdx.x] += red[1][threadIdx.x + w];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    part[blockIdx.x * 2] = red[0][0];
    part[blockIdx.x * 2 + 1] = red[1][0];
  }
}

// Scalar slots of the iteration (device doubles):
//   sc[0], sc[1]: r.z (ping-pong by iteration parity)   sc[2]: p.q   sc[3]: r.r   sc[4]: ||f||
// mode 0: out slot = sum (q = 0);   mode 1: out slot = sum (q = 0), status relres / converged from
// sum = r.r;  mode 2: ||f|| (sqrt of sum) and the initial status.
__device__ __forceinline__ void dot_status(double v, int mode, double* sc, int slot, double tol, BcgStatus* st,
                                           double* hist, int hist_mod);
__global__ void __launch_bounds__(RT) k_dot_reduce(const double* __restrict__ part, int nblk, double* sc, int slot,
                                                   int mode, double tol, BcgStatus* st, double* hist,
                                                   int hist_mod) {
  pdl_wait();
  __shared__ double red[RT];
  if (mode == 1 && st->done) return;   // read by every thread before thread 0 can write it
  double s = 0.0;
  for (int b = threadIdx.x; b < nblk; b += RT) s += part[b * 2];
  red[threadIdx.x] = s;
  __syncthreads();
  for (int w = RT / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x != 0) return;
  // nblk < 0: the sum was formed beforehand (several ranks: summed over ranks) in sc[-nblk - 1]
  const double v = nblk < 0 ? sc[-nblk - 1] : red[0];
  dot_status(v, mode, sc, slot, tol, st, hist, hist_mod);
}

// the scalar / status update of k_dot_reduce for the reduced value v (one thread)
__device__ __forceinline__ void dot_status(double v, int mode, double* sc, int slot, double tol, BcgStatus* st,
                                           double* hist, int hist_mod) {
  if (mode == 0) {
    sc[slot] = v;
  } else if (mode == 1) {
    sc[slot] = v;
    const double fn = sc[4];
    const double rel = fn > 0.0 ? sqrt(v) / fn : 0.0;
    st->relres = rel;
    st->converged = rel <= tol ? 1 : 0;
    if (!isfinite(v)) st->nonfinite = 1;
    const int it = ++st->iters;
    hist[hist_mod > 0 ? (it - 1) % hist_mod : it - 1] = rel;
    st->done = (st->converged || st->nonfinite || st->indefinite || it >= st->maxit) ? 1 : 0;
  } else {
    sc[4] = sqrt(v);
    st->relres = v > 0.0 ? 1.0 : 0.0;
    st->converged = v > 0.0 ? 0 : 1;
    if (!isfinite(v)) st->nonfinite = 1;
    st->iters = 0;
    st->done = (st->converged || st->nonfinite || st->maxit <= 0) ? 1 : 0;
  }
}

// Fixed-order sum of nblk chunk partials (stride 2), evaluated identically by every CTA that needs
// it: warp 0 loads lane-strided, then a fixed xor tree; the result is broadcast through smem.
__device__ __forceinline__ double cta_sum_partials(const double* __restrict__ part, int nblk, double* bcast) {
  if (nblk < 0) return part[0];   // already reduced (several ranks: summed over ranks)
  if (threadIdx.x < 32) {
    double v = 0.0;
    for (int b = threadIdx.x; b < nblk; b += 32) v += part[b * 2];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (threadIdx.x == 0) *bcast = v;
  }
  __syncthreads();
  return *bcast;
}

// alpha = (r.z) / (p.q) with the p.q reduction folded in (sum of the partials);  x += alpha p;
// r -= alpha q;  partial r.r.  p.q <= 0 -> indefinite.
__global__ void __launch_bounds__(RT) k_pcg_xr_f(double* __restrict__ x, double* __restrict__ r,
                                                 const double* __restrict__ p, const double* __restrict__ q,
                                                 int64_t n, double* sc, int cur,
                                                 const double* __restrict__ pq_part, int nblk,
                                                 double* __restrict__ part, BcgStatus* st, int64_t ngram,
                                                 unsigned* done_ctr, double tol, double* hist, int hist_mod) {
  pdl_wait();
  __shared__ double red[RT];
  __shared__ double bc;
  __shared__ bool last;
  if (st->done) return;
  const double pq = cta_sum_partials(pq_part, nblk, &bc);
  const double alpha = pq > 0.0 ? sc[cur] / pq : 0.0;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    sc[2] = pq;
    if (!(pq > 0.0)) st->indefinite = 1;
  }
  const int64_t r0 = (int64_t)blockIdx.x * RPB;
  double s = 0.0;
  for (int64_t i = r0 + threadIdx.x; i < min(n, r0 + RPB); i += RT) {
    x[i] = fma(alpha, p[i], x[i]);
    const double v = fma(-alpha, q[i], r[i]);
    r[i] = v;
    if (i < ngram) s = fma(v, v, s);   // several ranks: the shared rows count on rank 0 only
  }
  red[threadIdx.x] = s;
  __syncthreads();
  for (int w = RT / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) part[blockIdx.x * 2] = red[0];
  if (!done_ctr) return;
  // one rank: the LAST CTA to finish sums the r.r partials in k_dot_reduce's fixed order (bitwise the same
  // value) and updates the status - no separate reduce launch
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = atomicAdd(done_ctr, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!last) return;
  __threadfence();
  const int nblk_out = (int)gridDim.x;
  double t = 0.0;
  for (int b = threadIdx.x; b < nblk_out; b += RT) t += ((volatile double*)part)[b * 2];
  red[threadIdx.x] = t;
  __syncthreads();
  for (int w = RT / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    *done_ctr = 0u;
    dot_status(red[0], 1, sc, 3, tol, st, hist, hist_mod);
  }
}

// p = z + beta p with the r.z reduction folded in: rz_new = sum(partials), beta = rz_new / sc[cur];
// CTA 0 stores rz_new in sc[cur ^ 1] for the next iteration's alpha
__global__ void __launch_bounds__(RT) k_pcg_p_f(double* __restrict__ p, const double* __restrict__ z, int64_t n,
                                                double* sc, int cur, const double* __restrict__ rz_part, int nblk,
                                                const BcgStatus* st) {
  pdl_wait();
  __shared__ double bc;
  if (st->done) return;
  const double rz = cta_sum_partials(rz_part, nblk, &bc);
  const double beta = rz / sc[cur];
  if (blockIdx.x == 0 && threadIdx.x == 0) sc[cur ^ 1] = rz;
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) p[i] = fma(beta, p[i], z[i]);
}

// y[i*ldy] = a[i*lda] + alpha * b[i*ldb]
__global__ void k_axpy_strided(double* y, int ldy, const double* a, int lda, const double* b, int ldb, double alpha,
                               int64_t n) {
  pdl_wait();
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) y[i * ldy] = fma(alpha, b[i * ldb], a[i * lda]);
}

// part[chunk*128 + k] = sum over chunk rows of Z[row][k] * r[row]  (k < rk)
__global__ void __launch_bounds__(256) k_gemvt_partial(const double* __restrict__ Z, int ldz,
                                                       const double* __restrict__ r, int64_t n, int rk,
                                                       double* __restrict__ part, int64_t rows_per_cta) {
  pdl_wait();
  // chunk of GT_ROWS rows; warp w takes rows w, w + 8, ...; lane covers columns lane + 32 j (j < 4),
  // so every row read is one coalesced 1 KB line; the 8 warp partials are summed in fixed order
  // each CTA owns a contiguous range of rows_per_cta rows (a multiple of GT_ROWS; a bounded grid, so
  // the single-CTA reduce sums at most a few hundred partials)
  __shared__ double red[8][128];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int64_t r0 = (int64_t)blockIdx.x * rows_per_cta;
  const int64_t r1 = min(n, r0 + rows_per_cta);
  double acc[4] = {0.0, 0.0, 0.0, 0.0};
  for (int64_t i = r0 + wid; i < r1; i += 8) {
    const double ri = r[i];
    const double* zr = Z + i * ldz;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int k = lane + 32 * j;
      if (k < rk) acc[j] = fma(__ldg(zr + k), ri, acc[j]);
    }
  }
#pragma unroll
  for (int j = 0; j < 4; ++j) red[wid][lane + 32 * j] = acc[j];
  __syncthreads();
  if (threadIdx.x < 128) {
    double s = 0.0;
#pragma unroll
    for (int w = 0; w < 8; ++w) s += red[w][threadIdx.x];
    part[blockIdx.x * 128 + threadIdx.x] = s;
  }
}

// g[k] = sigma[k] * sum_chunks part[chunk][k]  (fixed order: 8 interleaved partial sums, combined
// in group order)
__global__ void __launch_bounds__(1024) k_gemvt_reduce(const double* __restrict__ part, int nchunks,
                                                       const double* __restrict__ sigma, int rk,
                                                       double* __restrict__ g) {
  pdl_wait();
  __shared__ double red[8][128];
  const int k = threadIdx.x & 127, grp = threadIdx.x >> 7;
  double s = 0.0;
#pragma unroll 4
  for (int b = grp; b < nchunks; b += 8) s += part[b * 128 + k];
  red[grp][k] = s;
  __syncthreads();
  if (threadIdx.x < rk) {
    double t = 0.0;
#pragma unroll
    for (int q = 0; q < 8; ++q) t += red[q][k];
    g[k] = sigma ? sigma[k] * t : t;
  }
}

// y[row] += sum_k Z[row][k] g[k]   (warp per row, 16-byte loads of column pairs, butterfly sum)
__global__ void __launch_bounds__(256) k_gemv_add(const double* __restrict__ Z, int ldz, const double* __restrict__ g,
                                                  int rk, int64_t n, double* __restrict__ y) {
  pdl_wait();
  const int64_t row = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (row >= n) return;
  double s = 0.0;
  for (int k = 2 * lane; k < rk; k += 64) {
    const double2 z = __ldg(reinterpret_cast<const double2*>(Z + row * ldz + k));
    s = fma(z.x, g[k], s);
    if (k + 1 < rk) s = fma(z.y, g[k + 1], s);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) y[row] += s;
}

// bounded Z^T r grid: at most 4 CTAs per SM, each a contiguous multiple of GT_ROWS rows
static unsigned gemvt_grid(int64_t n, int64_t* rows_per_cta) {
  const int64_t cap = 4 * (int64_t)nspd::num_sms();
  int64_t nch = std::max<int64_t>(1, (n + GT_ROWS - 1) / GT_ROWS);
  if (nch > cap) nch = cap;
  int64_t rpc = (n + nch - 1) / nch;
  rpc = std::max<int64_t>(GT_ROWS, ((rpc + GT_ROWS - 1) / GT_ROWS) * GT_ROWS);
  *rows_per_cta = rpc;
  return (unsigned)std::max<int64_t>(1, (n + rpc - 1) / rpc);
}

// WHILE-node control of the device-driven PCG loop: repeat until the iteration stopped itself
__global__ void k_pcg_loop_ctl(const BcgStatus* st, cudaGraphConditionalHandle h) {
  cudaGraphSetConditional(h, st->done ? 0u : 1u);
}

unsigned nblk_of(int64_t n) { return (unsigned)std::max<int64_t>(1, (n + RPB - 1) / RPB); }
unsigned grid1(int64_t n, int t) { return (unsigned)std::max<int64_t>(1, (n + t - 1) / t); }

}  // namespace

namespace nspi {

struct PcgWs {
  double *f, *w, *r, *z, *p, *q, *tmp, *t2, *eg;   // n_G vectors; eg: k x k (A-DEF2 solve, column 0)
  double *bB, *wvu, *tmpB;                 // W/V/U rows x 32
  double *i1r, *i1buf;                     // band rows x 32
  double *agbuf, *apply_wvu, *part, *part2, *gpart, *g, *sc, *hist;
  BcgStatus* st;
  unsigned* ctr;   // last-CTA counter of k_pcg_xr_f (zero between uses)
};

static size_t pcg_layout(const nsp_ctx* c, char* base, PcgWs* out) {
  size_t off = 0;
  auto take = [&](size_t nd) {
    off = (off + 255) & ~size_t(255);
    double* p = base ? (double*)(base + off) : nullptr;
    off += nd * 8;
    return p;
  };
  PcgWs w{};
  const size_t nG = (size_t)std::max<int64_t>(c->nG, 1);
  w.f = take(nG);
  w.w = take(nG);
  w.r = take(nG);
  w.z = take(nG);
  w.p = take(nG);
  w.q = take(nG);
  w.tmp = take(nG);
  w.t2 = take(nG);
  w.eg = take(2 * 128 * 128);
  const size_t wr = (size_t)std::max<int64_t>(c->wvu_rows, 1) * 32;
  w.bB = take(wr);
  w.wvu = take(wr);
  w.tmpB = take(wr);
  const size_t ir = (size_t)std::max<int64_t>(c->i1_rows, 1) * 32;
  w.i1r = take(ir);
  w.i1buf = take(ir);
  w.agbuf = take(c->has_ag ? ag_ws_doubles(c, 1) : 1);
  w.apply_wvu = take(apply_ws_bytes(c, 1) / 8 + 1);
  w.part = take((size_t)2 * nblk_of(std::max<int64_t>(c->nG, 1)) + 2);
  w.part2 = take((size_t)2 * nblk_of(std::max<int64_t>(c->nG, 1)) + 2);
  w.gpart = take((size_t)128 * grid1(std::max<int64_t>(c->nG, 1), GT_ROWS));
  w.g = take(128);
  w.sc = take(16);
  w.hist = take(PCG_CHUNK);
  w.st = (BcgStatus*)take(sizeof(BcgStatus) / 8 + 1);
  w.ctr = (unsigned*)take(1);
  if (out) *out = w;
  return ((off + 255) & ~size_t(255)) + 256;
}

size_t pcg_ws_bytes(const nsp_ctx* c) { return pcg_layout(c, nullptr, nullptr); }

// Rows that enter inner products: all local rows on one rank; with several ranks the private rows of every
// rank plus the shared rows once (rank 0), SURVEY.md §8(e) - the shared rows are the trailing local rows.
static int64_t dot_rows(const nsp_ctx* c) { return (c->nranks <= 1 || c->rank == 0) ? c->nG : c->n_priv; }

// out slot = a . b over the first n rows (several ranks: summed over ranks by one allreduce of the scalar)
static nsp_status dot(nsp_ctx* c, const double* a, const double* b, int64_t n, PcgWs& w, int slot) {
  const unsigned nb = nblk_of(n);
  nsp_count_launch();
  launch_k(k_dot2_partial, dim3(nb), dim3(RT), 0, c->stream, a, b, nullptr, nullptr, n, w.part);
  nsp_count_launch();
  launch_k(k_dot_reduce, dim3(1), dim3(RT), 0, c->stream, w.part, (int)nb, w.sc, slot, 0, 0.0, w.st, w.hist, PCG_CHUNK);
  return c->nranks > 1 ? comm_allreduce(c, w.sc + slot, 1) : NSP_OK;
}

// z = M r for the PCG preconditioner (0: identity copy, 1: A_G^{-1}, 2: M_2)
static nsp_status pcg_precond(nsp_ctx* c, int which, const double* r, double* z, PcgWs& w) {
  const int64_t n = c->nG;
  if (which == 0) {
    NSP_CUDA_TRY(c, cudaMemcpyAsync(z, r, (size_t)n * 8, cudaMemcpyDeviceToDevice, c->stream));
    return NSP_OK;
  }
  // M_2: the low-rank coefficient g = Sigma Z^T r does not depend on A_G^{-1} r, so it runs on a forked
  // side stream (a graph branch when captured) while the A_G solve - a latency-bound chain on a few
  // SMs - runs on the context stream; z += Z g after the join (one rank: the allreduce of g of several
  // ranks stays on the context stream)
  const bool fork2 = which == 2 && c->nys_rank > 0 && c->side_stream && c->ev_fork && c->ev_join && c->nranks == 1;
  if (fork2) {
    NSP_CUDA_TRY(c, cudaEventRecord(c->ev_fork, c->stream));
    NSP_CUDA_TRY(c, cudaStreamWaitEvent(c->side_stream, c->ev_fork, 0));
    int64_t rpc;
    const unsigned nch = gemvt_grid(n, &rpc);
    nsp_count_launch();
    launch_k(k_gemvt_partial, dim3(nch), dim3(256), 0, c->side_stream, c->d_Z, c->nys_ld, r, n, c->nys_rank, w.gpart, rpc);
    nsp_count_launch();
    launch_k(k_gemvt_reduce, dim3(1), dim3(1024), 0, c->side_stream, w.gpart, (int)nch, c->d_sigma, c->nys_rank, w.g);
    NSP_CUDA_TRY(c, cudaEventRecord(c->ev_join, c->side_stream));
  }
  nsp_status e = ag_solve(c, r, 1, z, 1, 1, w.agbuf);
  if (e != NSP_OK) return e;
  if (fork2) {
    NSP_CUDA_TRY(c, cudaStreamWaitEvent(c->stream, c->ev_join, 0));
    nsp_count_launch();
    launch_k(k_gemv_add, dim3(grid1(n * 32, 256)), dim3(256), 0, c->stream, c->d_Z, c->nys_ld, w.g, c->nys_rank, n, z);
    NSP_CUDA_TRY(c, cudaGetLastError());
    return NSP_OK;
  }
  if (which == 3 && c->nys_rank > 0) {
    // M_A-DEF2 r = A_G^{-1} r + Z E^{-1} Z^T (r - S_G A_G^{-1} r),  E = Z^T S_G Z (reading R5)
    const int kp = c->nys_ld, rk = c->nys_rank;
    if ((e = apply_into(c, z, 1, w.t2, 1, 1, 1, w.apply_wvu)) != NSP_OK) return e;     // S_G A_G^{-1} r
    nsp_count_launch();
    launch_k(k_axpy_strided, dim3(grid1(n, 256)), dim3(256), 0, c->stream, w.t2, 1, r, 1, w.t2, 1, -1.0, n);   // d = r - S t
    int64_t rpc;
    const unsigned nch = gemvt_grid(n, &rpc);
    nsp_count_launch();
    launch_k(k_gemvt_partial, dim3(nch), dim3(256), 0, c->stream, c->d_Z, kp, w.t2, n, rk, w.gpart, rpc);
    double* G = w.eg;                 // kp x kp, column 0 = Z^T d
    double* H = w.eg + 128 * 128;     // kp x kp, column 0 = E^{-1} Z^T d
    NSP_CUDA_TRY(c, cudaMemsetAsync(G, 0, (size_t)kp * kp * 8, c->stream));
    nsp_count_launch();
    launch_k(k_gemvt_reduce, dim3(1), dim3(1024), 0, c->stream, w.gpart, (int)nch, nullptr, rk, w.g);
    NSP_CUDA_TRY(c, cudaMemcpy2DAsync(G, kp * 8, w.g, 8, 8, rk, cudaMemcpyDeviceToDevice, c->stream));
    nspb::chol_solve(c->d_ELp, kp, G, kp, H, kp, 1.0, true, true, nullptr, c->stream);
    NSP_CUDA_TRY(c, cudaMemcpy2DAsync(w.g, 8, H, kp * 8, 8, rk, cudaMemcpyDeviceToDevice, c->stream));
    nsp_count_launch();
    launch_k(k_gemv_add, dim3(grid1(n * 32, 256)), dim3(256), 0, c->stream, c->d_Z, kp, w.g, rk, n, z);
  }
  if (which == 2 && c->nys_rank > 0) {
    const int64_t ng = dot_rows(c);
    int64_t rpc;
    const unsigned nch = gemvt_grid(ng, &rpc);
    nsp_count_launch();
    launch_k(k_gemvt_partial, dim3(nch), dim3(256), 0, c->stream, c->d_Z, c->nys_ld, r, ng, c->nys_rank, w.gpart, rpc);
    nsp_count_launch();
    launch_k(k_gemvt_reduce, dim3(1), dim3(1024), 0, c->stream, w.gpart, (int)nch, c->d_sigma, c->nys_rank, w.g);
    if (c->nranks > 1 && (e = comm_allreduce(c, w.g, c->nys_rank)) != NSP_OK) return e;
    nsp_count_launch();
    launch_k(k_gemv_add, dim3(grid1(n * 32, 256)), dim3(256), 0, c->stream, c->d_Z, c->nys_ld, w.g, c->nys_rank, n, z);
  }
  NSP_CUDA_TRY(c, cudaGetLastError());
  return NSP_OK;
}

// wvu (W/V/U rows, ld 32) = A_I^{-1}-restricted-to-B of (rB ; r1):  y_B = L22^{-T} L22^{-1}(r_B - A_B1 A_11^{-1} r_1)
// i1r holds r_1 (band rows, ld 32), bB holds r_B; i1buf is overwritten with A_11^{-1} r_1.
static nsp_status interior_boundary_solve(nsp_ctx* c, PcgWs& w) {
  NSP_CUDA_TRY(c, cudaMemcpyAsync(w.i1buf, w.i1r, (size_t)c->i1_rows * 32 * 8, cudaMemcpyDeviceToDevice, c->stream));
  nspk::tri_fb(c->d_i1sys, c->nsub, w.i1buf, 32, 32, true, true, c->stream, c->i1_wbmax);
  nspk::spmm(c->CB, w.bB, 32, w.i1buf, 32, c->wvu_rows, w.wvu, 32, 1, 1, true, c->stream);
  if (c->d_minv) {   // y_B = S_j^{-1}(...) in place (k_symv1 reads w.wvu, its reduce writes it; partial
                     // slots in the apply workspace, idle here)
    double* P = w.apply_wvu + 2 * c->wvu_rows * 32;
    P = (double*)(((uintptr_t)P + 255) & ~(uintptr_t)255);
    nspk::symv1(c->d_subs, c->d_items, c->n_items, c->max_ntb, c->d_minv, w.wvu, 32, w.wvu, P, c->stream);
  } else {
    nspk::trsm_fb(c->d_subs, c->nsub, c->d_dense, w.wvu, 32, 32, c->stream);
  }
  NSP_CUDA_TRY(c, cudaGetLastError());
  return NSP_OK;
}

static nsp_status read_st(nsp_ctx* c, BcgStatus* d, BcgStatus* h) {
  NSP_CUDA_TRY(c, cudaMemcpyAsync(h, d, sizeof(BcgStatus), cudaMemcpyDeviceToHost, c->stream));
  NSP_CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  return NSP_OK;
}

nsp_status pcg_impl(nsp_ctx* c, const double* b, double* x, double tol, int maxit, int precond, PcgWs& w,
                    nsp_report* rep) {
  cudaStream_t st = c->stream;
  {
    const char* xfe = getenv("NSP_XFORK");
    if (precond == 2 && !(xfe && xfe[0] == '0')) {   // side stream for the M_2 low-rank branch
      if (!c->side_stream) NSP_CUDA_TRY(c, cudaStreamCreateWithFlags(&c->side_stream, cudaStreamNonBlocking));
      if (!c->ev_fork) NSP_CUDA_TRY(c, cudaEventCreateWithFlags(&c->ev_fork, cudaEventDisableTiming));
      if (!c->ev_join) NSP_CUDA_TRY(c, cudaEventCreateWithFlags(&c->ev_join, cudaEventDisableTiming));
    }
  }
  const int64_t n = c->nG;
  BcgStatus* hs = (BcgStatus*)c->h_status;
  nsp_status e;
  // several ranks: each rank reduces its own blocks, the S_G applies and A_G^{-1}
  // (Chebyshev) are sharded with their shared-row allreduce, inner products run over dot_rows and are
  // summed over ranks; the loop runs eagerly with one status read per iteration
  const bool multi = c->nranks > 1;
  const int64_t ng = dot_rows(c);
  // ---- reduction to the border: f = b_G - A_GI A_I^{-1} b_I
  nspk::gather_rows(b, 1, c->d_i1_src, c->i1_rows, w.i1r, 32, 1, 1.0, st);
  nspk::gather_rows(b, 1, c->d_b_src, c->wvu_rows, w.bB, 32, 1, 1.0, st);
  if ((e = interior_boundary_solve(c, w)) != NSP_OK) return e;
  nspk::spmm(c->AGG2, nullptr, 0, w.wvu, 32, n, w.tmp, 1, 1, 2, false, st);      // K-part: A_GI y_B
  if (multi && (e = finish_shared_rows(c, nullptr, 1, w.tmp, 1, 1, false)) != NSP_OK) return e;
  nspk::gather_rows(b, 1, c->d_g_src, n, w.f, 1, 1, 1.0, st);
  if (n > 0) {
    nsp_count_launch();
    launch_k(k_axpy_strided, dim3(grid1(n, 256)), dim3(256), 0, st, w.f, 1, w.f, 1, w.tmp, 1, -1.0, n);
  }
  // ---- PCG on S_G w = f
  BcgStatus init{};
  init.maxit = maxit;
  std::memcpy(hs, &init, sizeof(init));
  NSP_CUDA_TRY(c, cudaMemcpyAsync(w.st, hs, sizeof(BcgStatus), cudaMemcpyHostToDevice, st));
  NSP_CUDA_TRY(c, cudaMemsetAsync(w.w, 0, (size_t)std::max<int64_t>(n, 1) * 8, st));
  NSP_CUDA_TRY(c, cudaMemsetAsync(w.ctr, 0, sizeof(unsigned), st));
  NSP_CUDA_TRY(c, cudaMemcpyAsync(w.r, w.f, (size_t)n * 8, cudaMemcpyDeviceToDevice, st));
  if (multi) {   // ||f||^2 summed over ranks (slot 5), then the status from it
    if ((e = dot(c, w.f, w.f, ng, w, 5)) != NSP_OK) return e;
    nsp_count_launch();
    launch_k(k_dot_reduce, dim3(1), dim3(RT), 0, st, w.part, -6, w.sc, 4, 2, tol, w.st, w.hist, PCG_CHUNK);
  } else {
    const unsigned nb = nblk_of(n);
    nsp_count_launch();
    launch_k(k_dot2_partial, dim3(nb), dim3(RT), 0, st, w.f, w.f, nullptr, nullptr, n, w.part);
    nsp_count_launch();
    launch_k(k_dot_reduce, dim3(1), dim3(RT), 0, st, w.part, (int)nb, w.sc, 4, 2, tol, w.st, w.hist, PCG_CHUNK);
  }
  if ((e = read_st(c, w.st, hs)) != NSP_OK) return e;
  if (rep && rep->hist && rep->hist_cap > 0) rep->hist[0] = hs->relres;
  int iters = 0;
  double relres = hs->relres;
  nsp_status ret = hs->converged ? NSP_OK : NSP_NOT_CONVERGED;
  if (!hs->converged) {
    if ((e = pcg_precond(c, precond, w.r, w.z, w)) != NSP_OK) return e;
    NSP_CUDA_TRY(c, cudaMemcpyAsync(w.p, w.z, (size_t)n * 8, cudaMemcpyDeviceToDevice, st));
    if ((e = dot(c, w.r, w.z, ng, w, 0)) != NSP_OK) return e;
    int cur = 0;
    // one iteration, enqueued; stops itself on the device once st->done is set (converged, p^T S p
    // <= 0, non-finite, or maxit), so PCG_CHUNK iterations run between host status checks and the
    // chunk is one cached CUDA graph (single rank, no profiling, NSP_GRAPH != 0)
    double* hist_dev = w.hist;   // PCG_CHUNK ring (chunk path) or the full history (WHILE graph)
    int hist_mod = PCG_CHUNK;
    auto iteration = [&](cudaStream_t q) -> nsp_status {
      nsp_status e2;
      if ((e2 = apply_into(c, w.p, 1, w.q, 1, 1, 1, w.apply_wvu)) != NSP_OK) return e2;   // q = S_G p
      const unsigned nb = nblk_of(n);
      if (multi) {   // the same steps with every scalar summed over ranks before use (slots 6, 7, 8)
        if ((e2 = dot(c, w.p, w.q, ng, w, 6)) != NSP_OK) return e2;                           // p.q
        nsp_count_launch();
        launch_k(k_pcg_xr_f, dim3(nb), dim3(RT), 0, q, w.w, w.r, w.p, w.q, n, w.sc, cur, (const double*)(w.sc + 6), -1,
                 w.part2, w.st, ng, (unsigned*)nullptr, tol, hist_dev, hist_mod);
        nsp_count_launch();
        launch_k(k_dot_reduce, dim3(1), dim3(RT), 0, q, w.part2, (int)nb, w.sc, 7, 0, 0.0, w.st, hist_dev, hist_mod);
        if ((e2 = comm_allreduce(c, w.sc + 7, 1)) != NSP_OK) return e2;                       // r.r
        nsp_count_launch();
        launch_k(k_dot_reduce, dim3(1), dim3(RT), 0, q, w.part2, -8, w.sc, 3, 1, tol, w.st, hist_dev, hist_mod);
        if ((e2 = pcg_precond(c, precond, w.r, w.z, w)) != NSP_OK) return e2;
        if ((e2 = dot(c, w.r, w.z, ng, w, 8)) != NSP_OK) return e2;                           // r.z
        nsp_count_launch();
        launch_k(k_pcg_p_f, dim3(grid1(n, RT)), dim3(RT), 0, q, w.p, w.z, n, w.sc, cur, (const double*)(w.sc + 8), -1,
                 w.st);
        cur ^= 1;
        return NSP_OK;
      }
      // p.q partials; their sum is taken inside k_pcg_xr_f (every CTA, same order)
      nsp_count_launch();
      launch_k(k_dot2_partial, dim3(nb), dim3(RT), 0, q, w.p, w.q, nullptr, nullptr, n, w.part);
      nsp_count_launch();
      launch_k(k_pcg_xr_f, dim3(nb), dim3(RT), 0, q, w.w, w.r, w.p, w.q, n, w.sc, cur, w.part, (int)nb, w.part2, w.st,
               n, w.ctr, tol, hist_dev, hist_mod);   // + the r.r reduce and status (last CTA)
      if ((e2 = pcg_precond(c, precond, w.r, w.z, w)) != NSP_OK) return e2;
      // r.z partials; the sum (and beta) inside k_pcg_p_f
      nsp_count_launch();
      launch_k(k_dot2_partial, dim3(nb), dim3(RT), 0, q, w.r, w.z, nullptr, nullptr, n, w.part);
      nsp_count_launch();
      launch_k(k_pcg_p_f, dim3(grid1(n, RT)), dim3(RT), 0, q, w.p, w.z, n, w.sc, cur, w.part, (int)nb, w.st);
      cur ^= 1;
      return NSP_OK;
    };
    const char* genv = getenv("NSP_GRAPH");
    const bool use_graph = !multi && !c->prof_on && !(genv && genv[0] == '0');
    const PcgKey key{w.w, n, precond, tol, maxit, c->nys_rank, c->d_Z, c->d_ELp, c->nys_gen};
    double hbuf[PCG_CHUNK];
    // device-driven loop (default): ONE launch of a graph whose WHILE node repeats the iteration
    // until st->done; the chunked graph below is the fallback (and NSP_GRAPH=1)
    bool loop_done = false;
    if (use_graph && !(genv && genv[0] == '1') && !c->pcg_no_while) {
      if (c->phist_cap < maxit + 1) {
        if (c->d_phist) cudaFree(c->d_phist);
        c->d_phist = nullptr;
        c->phist_cap = 0;
        NSP_CUDA_TRY(c, cudaMalloc(&c->d_phist, (size_t)(maxit + 1) * sizeof(double)));
        c->phist_cap = maxit + 1;
        if (c->pcg_wgraph) {
          cudaGraphExecDestroy(c->pcg_wgraph);
          c->pcg_wgraph = nullptr;
        }
      }
      auto build_while = [&]() -> cudaError_t {
        if (c->pcg_wgraph) {
          cudaGraphExecDestroy(c->pcg_wgraph);
          c->pcg_wgraph = nullptr;
        }
        cudaError_t ce;
        if (!c->gstream && (ce = cudaStreamCreateWithFlags(&c->gstream, cudaStreamNonBlocking)) != cudaSuccess) return ce;
        cudaGraph_t g = nullptr;
        if ((ce = cudaGraphCreate(&g, 0)) != cudaSuccess) return ce;
        cudaGraphConditionalHandle hcond;
        cudaGraphNodeParams np = {};
        np.type = cudaGraphNodeTypeConditional;
        np.conditional.type = cudaGraphCondTypeWhile;
        np.conditional.size = 1;
        cudaGraphNode_t wnode;
        if ((ce = cudaGraphConditionalHandleCreate(&hcond, g, 1, cudaGraphCondAssignDefault)) != cudaSuccess ||
            (np.conditional.handle = hcond, ce = cudaGraphAddNode(&wnode, g, nullptr, 0, &np)) != cudaSuccess) {
          cudaGraphDestroy(g);
          return ce;
        }
        if ((ce = cudaStreamBeginCaptureToGraph(c->gstream, np.conditional.phGraph_out[0], nullptr, nullptr, 0,
                                                cudaStreamCaptureModeRelaxed)) != cudaSuccess) {
          cudaGraphDestroy(g);
          return ce;
        }
        c->stream = c->gstream;
        c->capturing = true;
        hist_dev = c->d_phist;
        hist_mod = 0;
        const int cur0 = cur;
        const long long l0 = nsp_launch_count();
        nsp_status ec = iteration(c->gstream);
        if (ec == NSP_OK) ec = iteration(c->gstream);   // two per body: the r.z ping-pong returns to cur0
        if (ec == NSP_OK) {
          nsp_count_launch();
          k_pcg_loop_ctl<<<1, 1, 0, c->gstream>>>(w.st, hcond);
        }
        cur = cur0;
        hist_dev = w.hist;
        hist_mod = PCG_CHUNK;
        cudaGraph_t gout = nullptr;
        const cudaError_t ce2 = cudaStreamEndCapture(c->gstream, &gout);
        c->stream = st;
        c->capturing = false;
        c->pcg_wbody_kernels = nsp_launch_count() - l0;
        nsp_count_launches(-c->pcg_wbody_kernels);
        if (ec != NSP_OK || ce2 != cudaSuccess) {
          cudaGraphDestroy(g);
          return ce2 != cudaSuccess ? ce2 : cudaErrorUnknown;
        }
        cudaGraphExec_t gx = nullptr;
        ce = cudaGraphInstantiate(&gx, g, 0);
        cudaGraphDestroy(g);
        if (ce != cudaSuccess) return ce;
        c->pcg_wgraph = gx;
        c->pcg_wkey = key;
        return cudaSuccess;
      };
      if (!(c->pcg_wgraph && c->pcg_wkey == key) && build_while() != cudaSuccess) {
        (void)cudaGetLastError();
        c->pcg_no_while = true;
      } else {
        NSP_CUDA_TRY(c, cudaGraphLaunch(c->pcg_wgraph, st));
        if ((e = read_st(c, w.st, hs)) != NSP_OK) return e;
        const int done = hs->iters;
        // kernels actually run: two iterations per body pass (the second a no-op pass when the
        // first stopped); count the body per pass
        nsp_count_launches(c->pcg_wbody_kernels * (long long)((done + 2) / 2));
        if (rep && rep->hist && rep->hist_cap > 1) {
          const int m = std::min(done, rep->hist_cap - 1);
          if (m > 0) NSP_CUDA_TRY(c, cudaMemcpy(rep->hist + 1, c->d_phist, (size_t)m * sizeof(double),
                                                cudaMemcpyDeviceToHost));
        }
        iters = done;
        relres = hs->relres;
        if (hs->indefinite) {
          ret = NSP_ERR_INDEFINITE;
          c->err = "nsp_pcg: p^T S_G p <= 0";
        } else if (hs->nonfinite) {
          ret = NSP_ERR_NUMERICAL;
          c->err = "nsp_pcg: non-finite residual";
        } else if (hs->converged) {
          ret = NSP_OK;
        }
        loop_done = true;
      }
    }
    while (!loop_done) {
      if (use_graph) {
        if (!(c->pcg_graph && c->pcg_key == key)) {
          if (!c->gstream) NSP_CUDA_TRY(c, cudaStreamCreateWithFlags(&c->gstream, cudaStreamNonBlocking));
          if (c->pcg_graph) {
            cudaGraphExecDestroy(c->pcg_graph);
            c->pcg_graph = nullptr;
          }
          cudaGraph_t g = nullptr;
          c->stream = c->gstream;
          c->capturing = true;
          const long long l0 = nsp_launch_count();
          NSP_CUDA_TRY(c, cudaStreamBeginCapture(c->gstream, cudaStreamCaptureModeRelaxed));
          nsp_status ec = NSP_OK;
          for (int j = 0; j < PCG_CHUNK && ec == NSP_OK; ++j) ec = iteration(c->gstream);
          cudaError_t ce = cudaStreamEndCapture(c->gstream, &g);
          c->stream = st;
          c->capturing = false;
          c->pcg_graph_kernels = nsp_launch_count() - l0;
          nsp_count_launches(-c->pcg_graph_kernels);
          if (ec != NSP_OK) return ec;
          NSP_CUDA_TRY(c, ce);
          cudaGraphExec_t gx = nullptr;
          NSP_CUDA_TRY(c, cudaGraphInstantiate(&gx, g, 0));
          cudaGraphDestroy(g);
          c->pcg_graph = gx;
          c->pcg_key = key;
        }
        NSP_CUDA_TRY(c, cudaGraphLaunch(c->pcg_graph, st));
        nsp_count_launches(c->pcg_graph_kernels);
      } else {
        // several ranks: one iteration per status read (every rank runs the same collective sequence and
        // stops on the same, bit-identical, replicated decision)
        for (int j = 0; j < (multi ? 1 : PCG_CHUNK); ++j)
          if ((e = iteration(st)) != NSP_OK) return e;
      }
      NSP_CUDA_TRY(c, cudaMemcpyAsync(hbuf, w.hist, sizeof(hbuf), cudaMemcpyDeviceToHost, st));
      if ((e = read_st(c, w.st, hs)) != NSP_OK) return e;
      for (int it = iters; it < hs->iters; ++it)
        if (rep && rep->hist && it + 1 < rep->hist_cap) rep->hist[it + 1] = hbuf[it % PCG_CHUNK];
      iters = hs->iters;
      relres = hs->relres;
      if (hs->indefinite) {
        ret = NSP_ERR_INDEFINITE;
        c->err = "nsp_pcg: p^T S_G p <= 0";
        break;
      }
      if (hs->nonfinite) {
        ret = NSP_ERR_NUMERICAL;
        c->err = "nsp_pcg: non-finite residual";
        break;
      }
      if (hs->converged) {
        ret = NSP_OK;
        break;
      }
      if (hs->done || iters >= maxit) break;
    }
  }
  // ---- back-substitution: x_I = A_I^{-1}(b_I - A_IG w), x_G = w, un-permute
  nspk::gather_rows(b, 1, c->d_i1_src, c->i1_rows, w.i1r, 32, 1, 1.0, st);
  nspk::gather_rows(b, 1, c->d_b_src, c->wvu_rows, w.bB, 32, 1, 1.0, st);
  nspk::spmm(c->A2G, w.w, 1, nullptr, 0, 0, w.tmpB, 32, 1, 0, true, st);            // A_IG w (B rows)
  if (c->wvu_rows > 0) {
    nsp_count_launch();
    launch_k(k_axpy_strided, dim3(grid1(c->wvu_rows, 256)), dim3(256), 0, st, w.bB, 32, w.bB, 32, w.tmpB, 32, -1.0, c->wvu_rows);
  }
  if ((e = interior_boundary_solve(c, w)) != NSP_OK) return e;                       // y_B in wvu
  nspk::spmm(c->C1, w.i1r, 32, w.wvu, 32, c->i1_rows, w.i1buf, 32, 1, 1, true, st); // r_1 - A_1B y_B
  nspk::tri_fb(c->d_i1sys, c->nsub, w.i1buf, 32, 32, true, true, st, c->i1_wbmax);               // y_1
  if (multi) NSP_CUDA_TRY(c, cudaMemsetAsync(x, 0, (size_t)c->n * 8, st));
  nspk::scatter_rows(w.i1buf, 32, c->d_i1_src, c->i1_rows, x, 1, 1, false, st);
  nspk::scatter_rows(w.wvu, 32, c->d_b_src, c->wvu_rows, x, 1, 1, false, st);
  nspk::scatter_rows(w.w, 1, c->d_g_src, ng, x, 1, 1, false, st);   // shared Gamma rows once (rank 0)
  // several ranks: every rank wrote its own rows (zero elsewhere); one allreduce assembles x on all ranks
  if (multi && (e = comm_allreduce(c, x, (size_t)c->n)) != NSP_OK) return e;
  NSP_CUDA_TRY(c, cudaStreamSynchronize(st));
  NSP_CUDA_TRY(c, cudaGetLastError());
  if (rep) {
    rep->iters = iters;
    rep->converged = ret == NSP_OK;
    rep->status = ret;
    rep->relres = relres;
  }
  return ret;
}

}  // namespace nspi

using namespace nspi;

extern "C" nsp_status nsp_pcg(nsp_ctx* c, const double* b, double* x, double tol, int maxit, int precond, void* ws,
                              nsp_report* rep) {
  NspNvtx nvtx_range_("nsp_pcg");
  if (!c || !b || !x || maxit < 0 || precond < 0 || precond > 3) {
    if (c) c->err = "nsp_pcg: bad arguments (precond in {0, 1, 2, 3})";
    return NSP_ERR_ARG;
  }
  if (c->nranks != 1 && precond == 3) {
    c->err = "nsp_pcg: M_A-DEF2 (precond 3) is single-rank";
    return NSP_ERR_STATE;
  }
  if (precond >= 1 && !c->has_ag) {
    c->err = "nsp_pcg: the A_G^{-1} / M_2 preconditioner needs the A_G factor (opts.factor_gamma = 1)";
    return NSP_ERR_STATE;
  }
  if (precond == 3 && c->nys_rank > 0) {
    nsp_status ea = adef_prepare(c);
    if (ea != NSP_OK) return ea;
  }
  if (precond == 3 && c->nys_rank > 0 && !c->adef_ok) {
    c->err = "nsp_pcg: E = Z^T S_G Z not positive definite (M_A-DEF2 unavailable)";
    return NSP_ERR_STATE;
  }
  if (precond >= 2 && c->nys_rank < 0) {
    c->err = "nsp_pcg: M_2 requested before nsp_nystrom";
    return NSP_ERR_STATE;
  }
  char* base;
  nsp_status e = get_ws(c, ws, pcg_ws_bytes(c), &base);
  if (e != NSP_OK) return e;
  PcgWs w;
  pcg_layout(c, base, &w);
  return pcg_impl(c, b, x, tol, maxit, precond, w, rep);
}
