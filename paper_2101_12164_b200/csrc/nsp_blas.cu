// Tall-skinny and small dense fp64 kernels of the block-CG / Nystrom steps (§8(a) rows a6-a11,
// d1): Gram contractions and panel updates on the DMMA pipe (north_star (c)), one-CTA s x s
// Cholesky / triangular inverse / Jacobi eigensolver, small GEMMs.  All reductions are
// fixed-order two-stage (no fp64 atomics): results are bitwise reproducible (reading C17).
#include <cuda_runtime.h>
#include <stdint.h>

#include "nsp_blas.h"
#include "nsp_dmma.cuh"

using namespace nspd;

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

constexpr int GR = 32;     // rows per Gram slab
constexpr int LDS = 68;    // smem stride for 64-wide tiles

// part[(chunk * ntm * ntn + tm * ntn + tn) * 4096 + i * 64 + j]
//   = sum_{r in chunk} Xa[r][64 tm + i] * Xb[r][64 tn + j]
__global__ void __launch_bounds__(256) k_gram_partial(const double* __restrict__ Xa, int lda,
                                                      const double* __restrict__ Xb, int ldb, int64_t n,
                                                      int64_t rows_per_chunk, double* __restrict__ part, int ntm,
                                                      int ntn) {
  extern __shared__ double sm[];
  double* As[2] = {sm, sm + GR * LDS};
  double* Bs[2] = {sm + 2 * GR * LDS, sm + 3 * GR * LDS};
  const int tile = blockIdx.x;
  const int tm = tile / ntn, tn = tile - tm * ntn;
  const int64_t r0 = blockIdx.y * rows_per_chunk;
  const int64_t r1 = min(n, r0 + rows_per_chunk);
  double acc[2][4][2];
  acc_zero(acc);
  const double* A0 = Xa + 64 * tm;
  const double* B0 = Xb + 64 * tn;
  int buf = 0;
  if (r0 < r1) {
    cp_block_zf(As[0], LDS, A0 + r0 * lda, lda, GR, 64, r1 - r0);
    cp_block_zf(Bs[0], LDS, B0 + r0 * ldb, ldb, GR, 64, r1 - r0);
    cp_commit();
  }
  for (int64_t r = r0; r < r1; r += GR) {
    const int64_t rn = r + GR;
    if (rn < r1) {
      cp_block_zf(As[buf ^ 1], LDS, A0 + rn * lda, lda, GR, 64, r1 - rn);
      cp_block_zf(Bs[buf ^ 1], LDS, B0 + rn * ldb, ldb, GR, 64, r1 - rn);
      cp_commit();
      cp_wait<1>();
    } else {
      cp_wait<0>();
    }
    __syncthreads();
    cta_mma<4, true, false>(As[buf], LDS, Bs[buf], LDS, acc, GR);
    __syncthreads();
    buf ^= 1;
  }
  double* out = part + ((int64_t)blockIdx.y * ntm * ntn + tile) * 4096;
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int rr = acc_row<4>(i), cc = acc_col<4>(j);
      *reinterpret_cast<double2*>(out + rr * 64 + cc) = make_double2(acc[i][j][0], acc[i][j][1]);
    }
}

__global__ void k_gram_reduce(const double* __restrict__ part, int nchunks, int ntm, int ntn, double* out,
                              int ldo) {
  const int i = blockIdx.y * 16 + threadIdx.y;
  const int j = blockIdx.x * 16 + threadIdx.x;
  if (i >= ntm * 64 || j >= ntn * 64) return;
  const int64_t off = (int64_t)((i >> 6) * ntn + (j >> 6)) * 4096 + (i & 63) * 64 + (j & 63);
  const int64_t stride = (int64_t)ntm * ntn * 4096;
  double s = 0.0;
  for (int c = 0; c < nchunks; ++c) s += part[off + c * stride];
  out[(int64_t)i * ldo + j] = s;
}

// Out[r][c] = (Cin ? Cin[r][c] : 0) + sgn * sum_k In[r][k] M[k][c];   r < n, c in this 64-col tile.
// normpart (optional): normpart[rowtile * ldo + c] = sum over the tile's rows of Out[r][c]^2.
__global__ void __launch_bounds__(256) k_panel(double* Out, int ldo, const double* Cin, int ldc,
                                               const double* __restrict__ In, int ldi, const double* __restrict__ M,
                                               int ldm, int kdim, int64_t n, double sgn, double* normpart) {
  extern __shared__ double sm[];
  constexpr int LDA = 36;
  double* As[2] = {sm, sm + 64 * LDA};
  double* Bs[2] = {sm + 2 * 64 * LDA, sm + 2 * 64 * LDA + 32 * LDS};
  const int64_t r0 = blockIdx.x * 64ll;
  const int c0 = blockIdx.y * 64;
  const int64_t nv = n - r0;
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
    if (kb + 1 < nk) {
      cp_block_zf(As[b ^ 1], LDA, In + r0 * ldi + (kb + 1) * 32, ldi, 64, 32, nv);
      cp_block(Bs[b ^ 1], LDS, M + (int64_t)(kb + 1) * 32 * ldm + c0, ldm, 32, 64);
      cp_commit();
      cp_wait<1>();
    } else {
      cp_wait<0>();
    }
    __syncthreads();
    cta_mma<4, false, false>(As[b], LDA, Bs[b], LDS, acc, 32);
    __syncthreads();
  }
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

// column sums of squares of X (n x s), partial per 64-row tile (fixed order)
__global__ void k_colsq_partial(const double* __restrict__ X, int ldx, int64_t n, int s, double* part, int ldp) {
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

// sum over row tiles -> out[c]
__global__ void k_colsq_reduce(const double* __restrict__ part, int ntiles, int ldp, double* out) {
  const int c = threadIdx.x;
  if (c >= ldp) return;
  double s = 0.0;
  for (int t = 0; t < ntiles; ++t) s += part[t * (int64_t)ldp + c];
  out[c] = s;
}

// convergence: relres_j = sqrt(rsq_j) / bnorm_j; max over j < s (columns with bnorm 0 count as 0)
__global__ void k_converge(const double* rsq, const double* bnorm, int s, double tol, BcgStatus* st,
                           double* hist_slot) {
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

__global__ void k_sqrt_vec(const double* in, double* out, int n) {
  const int i = threadIdx.x + blockIdx.x * blockDim.x;
  if (i < n) out[i] = sqrt(in[i]);
}

// ---------------------------------------------------------------------------------------------
// one-CTA Cholesky of an sp x sp SPD matrix with pivot record, and the inverse of its factor.
// mode 0 (D = P^T S P): rows/cols >= width replaced by identity; pivot <= 0 -> indefinite flag.
// mode 1 (G = W^T W, orth): pivot test  min d_i > tau * max d_i  (reading C3); failure -> fallback.
// Outputs: L (lower, ld sp), Linv (lower, ld sp); mode 1 also T = Linv^T (P = W T = W R^{-1}).
// ---------------------------------------------------------------------------------------------
__global__ void __launch_bounds__(1024) k_small_chol(const double* __restrict__ Ain, int sp, int mode, int nact,
                                                     double tau, double* Lout, double* Linv, double* Tout,
                                                     BcgStatus* st) {
  extern __shared__ double sm[];
  const int ld = sp + 1;
  double* A = sm;                       // sp x ld
  double* X = sm + sp * ld;             // packed lower: row i at i(i+1)/2
  __shared__ double colv[256];
  __shared__ double piv[256];
  __shared__ int fail;
  const int tid = threadIdx.x, nt = blockDim.x;
  const int width = nact < 0 ? st->width : nact;
  if (tid == 0) fail = 0;
  for (int e = tid; e < sp * sp; e += nt) {
    const int i = e / sp, j = e - i * sp;
    double v = Ain[e];
    if (i >= width || j >= width) v = (i == j) ? 1.0 : 0.0;
    A[i * ld + j] = v;
  }
  __syncthreads();
  for (int c = 0; c < sp; ++c) {
    const double d = A[c * ld + c];
    if (tid == 0) piv[c] = d;
    if (!(d > 0.0)) {
      if (tid == 0) fail = 1;
      break;
    }
    const double l = sqrt(d);
    for (int i = c + 1 + tid; i < sp; i += nt) colv[i] = A[i * ld + c] / l;
    __syncthreads();
    const int m = sp - c - 1;
    for (int e = tid; e < m * m; e += nt) {
      const int i = c + 1 + e / m, j = c + 1 + e % m;
      if (j <= i) A[i * ld + j] -= colv[i] * colv[j];
    }
    for (int i = c + 1 + tid; i < sp; i += nt) A[i * ld + c] = colv[i];
    if (tid == 0) A[c * ld + c] = l;
    __syncthreads();
  }
  __syncthreads();
  bool ok = !fail;
  if (ok && mode == 1) {
    double mn = piv[0], mx = piv[0];
    for (int i = 1; i < width; ++i) {
      mn = fmin(mn, piv[i]);
      mx = fmax(mx, piv[i]);
    }
    ok = mn > tau * mx;
  }
  if (!ok) {
    if (tid == 0) {
      if (mode == 0) st->indefinite = 1;
      else st->fallback = 1;
    }
    return;
  }
  if (tid == 0 && mode == 1) {
    st->fallback = 0;
    st->width = width;
  }
  // inverse of lower L: right-looking forward substitution on X = I
  for (int e = tid; e < sp * (sp + 1) / 2; e += nt) X[e] = 0.0;
  __syncthreads();
  for (int i = tid; i < sp; i += nt) X[i * (i + 1) / 2 + i] = 1.0;
  __syncthreads();
  for (int k = 0; k < sp; ++k) {
    const double lkk = A[k * ld + k];
    for (int cc = tid; cc <= k; cc += nt) X[k * (k + 1) / 2 + cc] /= lkk;
    __syncthreads();
    const int m = sp - k - 1;
    for (int e = tid; e < m * (k + 1); e += nt) {
      const int i = k + 1 + e / (k + 1), cc = e % (k + 1);
      X[i * (i + 1) / 2 + cc] -= A[i * ld + k] * X[k * (k + 1) / 2 + cc];
    }
    __syncthreads();
  }
  for (int e = tid; e < sp * sp; e += nt) {
    const int i = e / sp, j = e - i * sp;
    const double lv = (j <= i) ? A[i * ld + j] : 0.0;
    const double xv = (j <= i) ? X[i * (i + 1) / 2 + j] : 0.0;
    if (Lout) Lout[e] = lv;
    if (Linv) Linv[e] = xv;
    if (Tout) Tout[j * sp + i] = xv;  // T = Linv^T
  }
}

// ---------------------------------------------------------------------------------------------
// one-CTA cyclic (round-robin) parallel Jacobi eigensolver of a symmetric n x n matrix (n <= 256,
// padded to even).  A in smem, V in global.  Outputs eigenvalues (descending) and eigenvectors
// (columns, same order).  `gate` (optional): run only if *gate != 0.
// ---------------------------------------------------------------------------------------------
__global__ void __launch_bounds__(1024) k_small_eig(const double* __restrict__ Ain, int lda, int n,
                                                    double* V, int ldv, double* lam, double* Vsorted,
                                                    const int* gate) {
  if (gate && *gate == 0) return;
  extern __shared__ double sm[];
  const int ne = n + (n & 1);
  const int ld = ne + 1;
  double* A = sm;
  __shared__ double cs[128], sn[128];
  __shared__ int pp[128], qq[128];
  __shared__ double red[1024];
  __shared__ int order[256];
  const int tid = threadIdx.x, nt = blockDim.x;
  for (int e = tid; e < ne * ne; e += nt) {
    const int i = e / ne, j = e - i * ne;
    A[i * ld + j] = (i < n && j < n) ? Ain[i * lda + j] : 0.0;
    V[i * ldv + j] = (i == j) ? 1.0 : 0.0;
  }
  __syncthreads();
  const int npair = ne / 2;
  for (int sweep = 0; sweep < 60; ++sweep) {
    // off-diagonal and total norms
    double off = 0.0, tot = 0.0;
    for (int e = tid; e < ne * ne; e += nt) {
      const int i = e / ne, j = e - i * ne;
      const double v = A[i * ld + j];
      tot += v * v;
      if (i != j) off += v * v;
    }
    red[tid] = off;
    __syncthreads();
    for (int w = nt / 2; w > 0; w >>= 1) {
      if (tid < w) red[tid] += red[tid + w];
      __syncthreads();
    }
    const double offs = red[0];
    __syncthreads();
    red[tid] = tot;
    __syncthreads();
    for (int w = nt / 2; w > 0; w >>= 1) {
      if (tid < w) red[tid] += red[tid + w];
      __syncthreads();
    }
    const double tots = red[0];
    __syncthreads();
    if (!(offs > 1e-32 * tots) || tots == 0.0) break;
    for (int round = 0; round < ne - 1; ++round) {
      // tournament pairing: positions 0..ne-1, element 0 fixed, others rotate
      if (tid < npair) {
        auto who = [&](int pos) -> int { return pos == 0 ? 0 : 1 + (pos - 1 + round) % (ne - 1); };
        int p = who(tid), q = who(ne - 1 - tid);
        if (p > q) {
          const int t = p;
          p = q;
          q = t;
        }
        pp[tid] = p;
        qq[tid] = q;
        const double apq = A[p * ld + q];
        double c = 1.0, s = 0.0;
        if (fabs(apq) > 1e-300) {
          const double th = (A[q * ld + q] - A[p * ld + p]) / (2.0 * apq);
          const double t = (th >= 0 ? 1.0 : -1.0) / (fabs(th) + sqrt(th * th + 1.0));
          c = 1.0 / sqrt(t * t + 1.0);
          s = t * c;
        }
        cs[tid] = c;
        sn[tid] = s;
      }
      __syncthreads();
      // columns: A <- A J ; V <- V J
      for (int e = tid; e < npair * ne; e += nt) {
        const int k = e / ne, i = e - k * ne;
        const int p = pp[k], q = qq[k];
        const double c = cs[k], s = sn[k];
        const double ap = A[i * ld + p], aq = A[i * ld + q];
        A[i * ld + p] = c * ap - s * aq;
        A[i * ld + q] = s * ap + c * aq;
        const double vp = V[i * ldv + p], vq = V[i * ldv + q];
        V[i * ldv + p] = c * vp - s * vq;
        V[i * ldv + q] = s * vp + c * vq;
      }
      __syncthreads();
      // rows: A <- J^T A
      for (int e = tid; e < npair * ne; e += nt) {
        const int k = e / ne, j = e - k * ne;
        const int p = pp[k], q = qq[k];
        const double c = cs[k], s = sn[k];
        const double ap = A[p * ld + j], aq = A[q * ld + j];
        A[p * ld + j] = c * ap - s * aq;
        A[q * ld + j] = s * ap + c * aq;
      }
      __syncthreads();
    }
  }
  // sort descending (stable by index) - rank by counting
  if (tid < n) {
    const double li = A[tid * ld + tid];
    int r = 0;
    for (int j = 0; j < n; ++j) {
      const double lj = A[j * ld + j];
      if (lj > li || (lj == li && j < tid)) ++r;
    }
    order[r] = tid;
  }
  __syncthreads();
  if (tid < n) lam[tid] = A[order[tid] * ld + order[tid]];
  __syncthreads();
  for (int e = tid; e < n * n; e += nt) {
    const int i = e / n, k = e - i * n;
    Vsorted[i * n + k] = V[i * ldv + order[k]];
  }
}

// orth fallback: keep eigenvalues > tau * lambda_max (lam descending, only the first s are real);
// T[:, k] = V[:, k] / sqrt(lam_k) for k < width, zero otherwise.
__global__ void k_orth_from_eig(const double* lam, const double* Vs, int n, int sp, double tau, double* T,
                                BcgStatus* st) {
  if (!st->fallback) return;
  __shared__ int w;
  if (threadIdx.x == 0) {
    const double lmax = lam[0];
    int c = 0;
    if (lmax > 0)
      for (int k = 0; k < n; ++k)
        if (lam[k] > tau * lmax) ++c;
    w = c;
    st->width = c;
  }
  __syncthreads();
  for (int e = threadIdx.x; e < sp * sp; e += blockDim.x) {
    const int i = e / sp, k = e - i * sp;
    double v = 0.0;
    if (i < n && k < w) v = Vs[i * n + k] / sqrt(lam[k]);
    T[e] = v;
  }
}

// C = alpha * op(A) op(B) + beta * C, all sp-ish small (m x n, inner k), row-major, FMA.
__global__ void k_small_gemm(int m, int n, int k, double alpha, const double* A, int lda, int ta, const double* B,
                             int ldb, int tb, double beta, double* Cm, int ldc) {
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

// copy with ld change and zero padding: dst[r][c] = c < s ? src[r][c] : 0 (c < ldd)
__global__ void k_copy_pad(const double* src, int lds, double* dst, int ldd, int64_t n, int s, double scale) {
  const int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t r = idx / ldd;
  const int c = (int)(idx - r * ldd);
  if (r >= n) return;
  dst[r * ldd + c] = c < s ? scale * src[r * lds + c] : 0.0;
}

}  // namespace

namespace nspb {

static void set_smem(const void* f, size_t bytes) {
  cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
}

int gram_chunks(int64_t n, int ntiles) {
  int64_t ch = (n + 255) / 256;
  const int64_t cap = (296 + ntiles - 1) / ntiles;
  if (ch > cap) ch = cap;
  return (int)(ch < 1 ? 1 : ch);
}

size_t gram_ws_doubles(int64_t n, int sa, int sb) {
  const int ntm = (sa + 63) / 64, ntn = (sb + 63) / 64;
  return (size_t)gram_chunks(n, ntm * ntn) * ntm * ntn * 4096;
}

void gram(const double* Xa, int lda, int sa, const double* Xb, int ldb, int sb, int64_t n, double* out, int ldo,
          double* ws, cudaStream_t st) {
  const int ntm = (sa + 63) / 64, ntn = (sb + 63) / 64;
  const int nch = gram_chunks(n, ntm * ntn);
  int64_t rpc = (n + nch - 1) / nch;
  rpc = ((rpc + GR - 1) / GR) * GR;
  const size_t smem = 4 * GR * LDS * sizeof(double);
  static bool attr = false;
  if (!attr) {
    set_smem((const void*)k_gram_partial, smem);
    attr = true;
  }
  { nsp_count_launch(); k_gram_partial<<<dim3(ntm * ntn, nch), 256, smem, st>>>(Xa, lda, Xb, ldb, n, rpc, ws, ntm, ntn); }
  { nsp_count_launch(); k_gram_reduce<<<dim3(ntn * 4, ntm * 4), dim3(16, 16), 0, st>>>(ws, nch, ntm, ntn, out, ldo); }
}

void panel(double* Out, int ldo, const double* Cin, int ldc, const double* In, int ldi, const double* M, int ldm,
           int kdim, int ncols, int64_t n, double sgn, double* normpart, cudaStream_t st) {
  if (n <= 0) return;
  const size_t smem = (2 * 64 * 36 + 2 * 32 * LDS) * sizeof(double);
  static bool attr = false;
  if (!attr) {
    set_smem((const void*)k_panel, smem);
    attr = true;
  }
  dim3 grid((unsigned)((n + 63) / 64), (ncols + 63) / 64);
  { nsp_count_launch(); k_panel<<<grid, 256, smem, st>>>(Out, ldo, Cin, ldc, In, ldi, M, ldm, kdim, n, sgn, normpart); }
}

void colsq(const double* X, int ldx, int64_t n, int s, int ldp, double* part, double* out, cudaStream_t st) {
  const int nt = (int)((n + 63) / 64);
  { nsp_count_launch(); k_colsq_partial<<<nt, ldp, 0, st>>>(X, ldx, n, s, part, ldp); }
  { nsp_count_launch(); k_colsq_reduce<<<1, ldp, 0, st>>>(part, nt, ldp, out); }
}

void colsq_reduce(const double* part, int ntiles, int ldp, double* out, cudaStream_t st) {
  { nsp_count_launch(); k_colsq_reduce<<<1, ldp, 0, st>>>(part, ntiles, ldp, out); }
}

void sqrt_vec(const double* in, double* out, int n, cudaStream_t st) {
  { nsp_count_launch(); k_sqrt_vec<<<(n + 255) / 256, 256, 0, st>>>(in, out, n); }
}

void converge(const double* rsq, const double* bnorm, int s, double tol, BcgStatus* stt, double* hist_slot,
              cudaStream_t st) {
  { nsp_count_launch(); k_converge<<<1, 256, 0, st>>>(rsq, bnorm, s, tol, stt, hist_slot); }
}

void small_chol(const double* A, int sp, int mode, int nact, double tau, double* L, double* Linv, double* T,
                BcgStatus* stt, cudaStream_t st) {
  const size_t smem = ((size_t)sp * (sp + 1) + (size_t)sp * (sp + 1) / 2) * sizeof(double);
  set_smem((const void*)k_small_chol, smem);
  { nsp_count_launch(); k_small_chol<<<1, 1024, smem, st>>>(A, sp, mode, nact, tau, L, Linv, T, stt); }
}

void small_eig(const double* A, int lda, int n, double* Vwork, int ldv, double* lam, double* Vsorted,
               const int* gate, cudaStream_t st) {
  const int ne = n + (n & 1);
  const size_t smem = (size_t)ne * (ne + 1) * sizeof(double);
  set_smem((const void*)k_small_eig, smem);
  { nsp_count_launch(); k_small_eig<<<1, 1024, smem, st>>>(A, lda, n, Vwork, ldv, lam, Vsorted, gate); }
}

void orth_from_eig(const double* lam, const double* Vs, int n, int sp, double tau, double* T, BcgStatus* stt,
                   cudaStream_t st) {
  { nsp_count_launch(); k_orth_from_eig<<<1, 1024, 0, st>>>(lam, Vs, n, sp, tau, T, stt); }
}

void small_gemm(int m, int n, int k, double alpha, const double* A, int lda, bool ta, const double* B, int ldb,
                bool tb, double beta, double* C, int ldc, cudaStream_t st) {
  dim3 grid((n + 15) / 16, (m + 15) / 16);
  { nsp_count_launch(); k_small_gemm<<<grid, dim3(16, 16), 0, st>>>(m, n, k, alpha, A, lda, ta, B, ldb, tb, beta, C, ldc); }
}

void copy_pad(const double* src, int lds, double* dst, int ldd, int64_t n, int s, double scale, cudaStream_t st) {
  const int64_t tot = n * ldd;
  if (tot <= 0) return;
  { nsp_count_launch(); k_copy_pad<<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(src, lds, dst, ldd, n, s, scale); }
}

}  // namespace nspb
