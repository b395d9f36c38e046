// Tall-skinny / small dense fp64 kernels (nsp_blas.cu).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

// device-resident per-solve status (read back once per iteration)
struct BcgStatus {
  int width;        // active direction-block width s'
  int indefinite;   // chol(P^T S P) failed
  int fallback;     // orth used the eigen fallback
  int converged;
  int nonfinite;
  int done;       // PCG: the iteration stopped (converged / breakdown / maxit); later kernels no-op
  int iters;      // PCG: iterations taken (device count)
  int maxit;      // PCG: iteration cap
  int nfallback;  // block CG (device-driven loop): eigen-fallback count
  int pad_;
  double relres;    // max_j ||R_j|| / ||B_j||
  double scalar[6]; // PCG scalars
};

void nsp_count_launch();
// dispatch-path evidence counters (NSP_PATH_* in include/nsp.h): incremented at dispatch (eager or captured)
void nsp_count_path(int id);
// kernel-level tests (nsp_dev_*): force the generic kernels instead of the shape-specialised ones
// (0 = production dispatch, 1 = generic k_panel / full-tile Gram); set only around a test call
extern thread_local int nsp_force_generic;

struct PanelArgs {
  double* Out;
  int ldo;
  const double* Cin;
  int ldc;
  const double* In;
  int ldi;
  const double* M;
  int ldm;
  double sgn;
  double* normpart;
  // optional: when non-null and *upper_unless == 0, M is upper triangular (M[k][c] = 0 for k > c: orth's
  // T = R^{-1} after a successful Cholesky-QR) and the all-zero k-chunks of M are skipped per warp
  const int* upper_unless;
};

namespace nspb {
int gram_chunks(int64_t n, int ntiles);
size_t gram_ws_doubles(int64_t n, int sa, int sb);
// out (ld ldo) = Xa(n x sa)^T Xb(n x sb); sa, sb multiples of 64 (columns padded)
void gram(const double* Xa, int lda, int sa, const double* Xb, int ldb, int sb, int64_t n, double* out, int ldo,
          double* ws, cudaStream_t st);
// Out = Cin + sgn * In(n x kdim) M(kdim x ncols); ncols multiple of 64, kdim multiple of 32
// out = Xa^T Xb, out2 = Xa^T Xb2 (shared left operand, one pass)
void gram2(const double* Xa, int lda, int sa, const double* Xb, const double* Xb2, int ldb, int sb, int64_t n,
           double* out, double* out2, int ldo, double* ws, cudaStream_t st, bool lower_first = false);
// two independent panels in one launch (a1 may be null)
void panel2(const PanelArgs& a0, const PanelArgs* a1, int kdim, int ncols, int64_t n, cudaStream_t st);
// returns the number of normpart rows written (row tiles, or CTAs of the one-wave s = 128 kernel)
int panel(double* Out, int ldo, const double* Cin, int ldc, const double* In, int ldi, const double* M, int ldm,
          int kdim, int ncols, int64_t n, double sgn, double* normpart, cudaStream_t st,
          const int* upper_unless = nullptr);
// fused panel + Gram (s = 128, ld 128, n >= 64 x SMs, single rank): Out = Cin + sgn In M and
// gram_out = In^T Out (gmode 0) or Out^T Out (gmode 1, exactly symmetric); normpart (nullable): column
// sums of squares of Out, one row per CTA (returns the row count).  ws: gram_ws_doubles.
bool panel_gram_ok(int s, int64_t n);          // the production choice (large n)
bool panel_gram_shape_ok(int s, int64_t n);    // the kernel's shape requirement (kernel-level tests)
extern int nsp_fused_pg_mode;                  // 0 production, 1 force whenever the shape allows, 2 never
int panel_gram(double* Out, const double* Cin, const double* In, const double* M, int64_t n, double sgn,
               double* normpart, int gmode, double* gram_out, double* ws, cudaStream_t st);
void colsq(const double* X, int ldx, int64_t n, int s, int ldp, double* part, double* out, cudaStream_t st);
void colsq_reduce(const double* part, int ntiles, int ldp, double* out, cudaStream_t st);
void sqrt_vec(const double* in, double* out, int n, cudaStream_t st);
void colsq_converge(const double* part, int ntiles, int ldp, double* rsq, const double* bnorm, int s, double tol,
                    BcgStatus* stt, cudaStream_t st);
void converge(const double* rsq, const double* bnorm, int s, double tol, BcgStatus* stt, double* hist_slot,
              cudaStream_t st);
// mode 0: D (pivot <= 0 -> indefinite), Out = D^{-1}; mode 1: orth Gram (pivot test -> fallback),
// Out = T = R^{-1} with G = R^T R; mode 2: Out = R (upper), pivot <= 0 -> fallback.  nact < 0: active width read from stt->width; rows/cols >= nact
// are replaced by the identity.  sp <= 128, multiple of 32.
void small_chol(const double* A, int sp, int mode, int nact, double tau, double* Out, BcgStatus* stt,
                cudaStream_t st);
// latency-oriented s x s Cholesky (nsp_small.cu): Lp = L with the 16 x 16 diagonal blocks replaced
// by their inverses.  mode 0: pivot <= 0 -> indefinite; mode 1: pivot test (tau) -> fallback, else
// width = nact.  sp multiple of 16, <= 128.
void chol_fac(const double* A, int sp, int mode, int nact, double tau, double* Lp, BcgStatus* stt,
              cudaStream_t st);
// chol_fac + chol_solve fused (sp / 8 CTAs, each factoring redundantly and solving 8 columns): Lp and
// the status as chol_fac; Out = sgn * op(B) unless the factorisation failed (mode 0) or the pivot test
// chose the eigen fallback (mode 1), in which case Out is not written.
void chol_fac_solve(const double* A, int sp, int mode, int nact, double tau, double* Lp, BcgStatus* stt,
                    const double* B, int ldb, double* Out, int ldo, double sgn, bool fwd, bool bwd, cudaStream_t st);
// Out = sgn * op(B) (B == nullptr: identity), op = L^{-T}L^{-1} (fwd && bwd), L^{-1} (fwd), L^{-T} (bwd);
// sp / 8 CTAs (8 columns each); skipped when gate && *gate.
void chol_solve(const double* Lp, int sp, const double* B, int ldb, double* Out, int ldo, double sgn, bool fwd,
                bool bwd, const int* gate, cudaStream_t st);
void small_eig(const double* A, int lda, int n, double* Vwork, int ldv, double* lam, double* Vsorted,
               const int* gate, cudaStream_t st,
               double tau = 0.0, double* T = nullptr, int spT = 0, BcgStatus* stw = nullptr);
void small_gemm(int m, int n, int k, double alpha, const double* A, int lda, bool ta, const double* B, int ldb,
                bool tb, double beta, double* C, int ldc, cudaStream_t st);
void scale_rows(double* G, int ld, const double* d, int r, int nrows, int ncols, cudaStream_t st);
void small_sym(double* A, int n, int ld, double shift, cudaStream_t st);
// M[:, k] = V[:, k] * f(colscale[k]) for k < r (f: mode 0 x, 1 1/sqrt(x), 2 sqrt(x), 3 copy), zero for r <= k < ncols
void scale_cols(const double* V, int ldv, const double* colscale, int r, int n, int ncols, double* M, int ldm,
                int mode, cudaStream_t st);
void cheb_update(double* x, double* r, const double* d, const double* t, double* dn, double c1, double c2, int64_t n,
                 bool want_d, cudaStream_t st);
void copy_pad(const double* src, int lds, double* dst, int ldd, int64_t n, int s, double scale, cudaStream_t st);
}  // namespace nspb
