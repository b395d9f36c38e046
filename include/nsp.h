/* nsp.h - C ABI of the B200-native Nystrom-Schur block-CG hot path
 * (arXiv 2101.12164, "Nystrom-Schur two-level preconditioner").
 *
 * Problem (§1 eq:linear_system): A x = b, A sparse SPD, permuted
 * to doubly bordered block diagonal (DBBD) form by a caller-supplied partition
 * (§2.3 eq:perm_A):
 *     P^T A P = [[A_I, A_IG], [A_GI, A_G]],   A_I = diag(A_I_0, ..., A_I_{K-1}).
 * Border Schur complement (eq:schur_complement):
 *     S_G = A_G - sum_j A_GI_j A_I_j^{-1} A_I_jG.
 * Nystrom-Schur preconditioner M_2 = A_G^{-1} + Z Sigma Z^T (PAPER.md:937-943
 * eq:left_prec_mat, Alg. 2).
 *
 * Conventions (all entry points):
 *  - Host inputs (nsp_csr arrays, part) are copied by nsp_setup; the caller may
 *    free them on return.
 *  - Blocks X, Y, B, Omega are DEVICE pointers owned by the caller, on
 *    opts.device, fp64, ROW-MAJOR with leading dimension s, n_gamma_local rows,
 *    Gamma rows ordered as nsp_gamma_index() reports (single rank: ascending
 *    original node id, reading C10).
 *  - All work is enqueued on opts.stream (a cudaStream_t, may be NULL = legacy
 *    default stream).  nsp_schur_apply / nsp_kgamma_apply are asynchronous.  The
 *    single-rank solvers run their iterations as ONE device-driven CUDA graph
 *    (a WHILE node with the stop test on the device) and synchronise the
 *    stream once per solve; the multi-rank block CG reads a small status
 *    block once per iteration.  All solvers synchronise at exit.
 *  - ws: optional caller-owned device workspace of nsp_workspace_bytes(s)
 *    bytes; NULL makes the context allocate (and keep) its own.
 *  - Errors: every call returns an nsp_status; on a negative status
 *    nsp_last_error(ctx) holds a one-line message.  No CPU fallback exists: if
 *    the CUDA device or kernels are unavailable the calls fail with NSP_ERR_CUDA.
 */
#ifndef NSP_H
#define NSP_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  NSP_OK = 0,
  NSP_NOT_CONVERGED = 1,        /* maxit reached; not an error */
  NSP_ERR_ARG = -1,             /* invalid argument / malformed CSR / partition */
  NSP_ERR_NOT_SPD = -2,         /* Cholesky pivot <= 0 in A_I_j or A_G */
  NSP_ERR_INDEFINITE = -3,      /* block CG: chol(P^T S P) failed; PCG: p^T S p <= 0 */
  NSP_ERR_STAGNATION = -4,      /* all search directions deflated before convergence */
  NSP_ERR_RANK_COLLAPSE = -5,   /* Nystrom: no eigenvalue of C >= eps (M_2 -> A_G^{-1}) */
  NSP_ERR_NUMERICAL = -6,       /* non-finite values */
  NSP_ERR_STATE = -7,           /* call order (e.g. pcg with M_2 before nsp_nystrom) */
  NSP_ERR_CUDA = -8,
  NSP_ERR_NCCL = -9,
  NSP_ERR_OOM = -10
} nsp_status;

typedef struct nsp_ctx nsp_ctx;

/* Sparse SPD matrix, full symmetric storage, HOST arrays.  rowptr int64[n+1],
 * colidx int32[nnz] strictly increasing within each row, val fp64[nnz]. */
typedef struct {
  int64_t n;
  const int64_t* rowptr;
  const int32_t* colidx;
  const double* val;
} nsp_csr;

typedef struct {
  int device;            /* CUDA device ordinal */
  void* stream;          /* cudaStream_t (e.g. torch.cuda.current_stream().cuda_stream) */
  int nranks, rank;      /* multi-GPU: ranks own contiguous ranges of block ids */
  const void* nccl_id;   /* 128-byte ncclUniqueId shared by all ranks; NULL if nranks == 1 */
  int bcg_precond;       /* block-CG preconditioner: 0 = none (M = I), 1 = A_G^{-1} (reading C2) */
  int factor_gamma;      /* 1 = factor A_G in nsp_setup (needed by M_2, bcg_precond=1, pcg) */
  double orth_tau;       /* rank-revealing threshold tau of orth() (reading C3), default 1e-14 */
  double nys_eps_rel;    /* Nystrom eigenvalue split eps = nys_eps_rel * lambda_max(C) (reading C6), 1e-12 */
  size_t scratch_bytes;  /* device scratch budget for the setup factorisation; 0 = auto */
  int verbose;
  void* local_group;     /* testing only: nsp_local_group_create(nranks) handle shared by nranks host
                            threads driving ranks on ONE device (replaces NCCL); NULL otherwise */
  int apply_kernel;      /* a2+a3 of the S_G apply: 0 = one symmetric product with the explicit
                            S_j^{-1} = L22^{-T} L22^{-1} tiles formed in setup (default): for s >= 48
                            on the INT8 tensor cores with fp64 accuracy (tcgen05 kind::i8, Ozaki
                            splitting of the D-scaled tiles into 7 int8 slices, reading R10; built in
                            setup when the device budget allows, env NSP_OZAKI=0 disables), else the
                            fp64 DMMA product; 1 = the two batched triangular sweeps with L22 (no extra
                            memory); 2 = the fp64 DMMA product only; 3 = the INT8 path for every s > 1 */
  int nys_power;         /* q >= 0: q-power iteration Nystrom (eq:power PAPER.md:204-212), G = B_H^q Omega
                            with the columns orthonormalised between applications; 0 = Alg. 2 as written */
  int nys_form;          /* inner system of nsp_nystrom: 0 = the border system S_G X = K_G G, Y = A_G X
                            (reading C1, default); 1 = the paper-literal S_I X = A_IG G, Y = A_GI X
                            (eq:SI) by block PCG preconditioned by A_I;
                            read by nsp_setup (builds A_I on the interior layout), single rank;
                            2 = M_3: Nystrom of S_I^{-1} itself (eq:internal_term_lr_approximation_2,
                            eq:left_prec_mat2): Y = S_I^{-1} Omega_I by block PCG, Z = A_G^{-1} A_GI V,
                            Omega is then n x (rank + oversample) in ORIGINAL order (interior rows used),
                            no power steps;
                            3 = M_1 (eq:prec1S): Nystrom of R_G^{-T} A_GI S_I^{-1} A_IG
                            R_G^{-1} (eq:lr_approximation_S-1_A-I) with R_G the A_G Cholesky factor of
                            the setup (ordering: ag_order), Z = R_G^{-1} U; Omega is n_gamma x s in
                            R_G's row order (the Gamma order when ag_order = 1); power steps allowed.
                            nsp_pcg precond 2 / 3 then apply M_1 / M_A-DEF1 */
  int ag_order;          /* ordering of the A_G factor (factor_gamma): 0 = reverse Cuthill-McKee band
                            (default); 1 = the natural Gamma order (nsp_gamma_index), so that
                            R_G = chol(A_G) exactly as written (dense-ish band: small n_G only) */
  int ag_solver;         /* how A_G^{-1} is applied (factor_gamma): 0 = auto (the band Cholesky factor
                            when it fits the device budget, else 2); 1 = band Cholesky factor only
                            (NSP_ERR_OOM when it does not fit); 2 = a fixed-degree Chebyshev iteration
                            on A_G ("an iterative solver to solve linear systems with
                            A_G ... A_G is typically well conditioned"), spectrum bounds from a setup
                            Lanczos run, degree for a 1e-15 relative error bound; a fixed polynomial,
                            so M_2 stays one symmetric operator for the outer PCG.  M_1 (nys_form 3)
                            needs the factor (1 or a fitting auto). */
} nsp_opts;

/* Solver / setup report; caller-owned.  hist / widths are optional caller
 * buffers (NULL or cap 0 = not recorded). */
typedef struct {
  int iters;             /* S_G applications inside the loop (reading C4) */
  int converged;
  int status;
  double relres;         /* final max_j ||R_j|| / ||B_j||  (block CG) or ||r||/||f|| (PCG) */
  double* hist;  int hist_cap;     /* relres per iteration (index 0 = initial) */
  int* widths;   int widths_cap;   /* active direction-block width per iteration */
  int bad_block;                   /* NOT_SPD: block id (-1 = A_G) */
  long long bad_pivot;             /* NOT_SPD: original node id of the failing pivot */
  int rank;                        /* Nystrom: rank of the approximation (min(r, k)) */
  int fallbacks;                   /* block CG: eigen-fallback orthonormalisations */
  double t_ms[8];                  /* setup: [0] host analysis, [1] H2D, [2] GPU factor, [3] A_G factor,
                                      [4] S_j^{-1} tiles (apply_kernel 0), [5] their INT8
                                      slices (reading R10) */
} nsp_report;

void nsp_default_opts(nsp_opts* o);

/* nsp_setup: validate A and part (NSP_ERR_ARG names the offending entry:
 * unsorted / out-of-range colidx, asymmetry, part outside {-1} U [0,K),
 * separator property violation (i, j, b_i, b_j)); build the DBBD permutation
 * (blocks 0..K-1 in ascending original index, then Gamma ascending; PAPER.md
 * eq:perm_A); order each block interior-first / boundary-layer-last; copy to
 * the device and run the GPU numeric factorisation of every A_I_j in one
 * launch per batch ("factorized cheaply in parallel"), plus
 * A_G (eq:cholesky PAPER.md:443-446) when opts.factor_gamma.  rep may be NULL;
 * on NSP_ERR_NOT_SPD it receives bad_block / bad_pivot. */
nsp_status nsp_setup(const nsp_csr* A, const int32_t* part, int K, const nsp_opts* opts,
                     nsp_ctx** out, nsp_report* rep);

nsp_status nsp_dims(const nsp_ctx* ctx, int64_t* n, int64_t* n_gamma, int64_t* n_gamma_local,
                    int* K_local);

/* ---- multi-GPU sharding ----
 * Rank r of G owns the contiguous block range [rK/G, (r+1)K/G) (a subtree of a depth-first ND leaf
 * numbering).  Its local Gamma rows are its PRIVATE rows (every adjacent block is its own and no
 * A_G neighbour is private to another rank) followed by the SHARED rows (all other Gamma rows,
 * replicated on every rank), each group in ascending original id.  Per S_G apply the shared rows'
 * per-rank partials are summed by one allreduce; Gram matrices and column norms are summed over
 * the private rows of every rank plus the shared rows once (rank 0's partial).
 * nsp_shard_plan: HOST-ONLY (no device needed) computation of that plan for (nranks, rank):
 * gamma_local (nullable, capacity >= n_private + n_shared) receives the original ids.
 * Returns NSP_ERR_ARG on a malformed part / rank. */
nsp_status nsp_shard_plan(const nsp_csr* A, const int32_t* part, int K, int nranks, int rank,
                          int64_t* n_private, int64_t* n_shared, int64_t* gamma_local, int* blk0, int* nblk);
/* n_private / n_shared local Gamma rows and the local block range of a context. */
nsp_status nsp_shard_info(const nsp_ctx* ctx, int64_t* n_private, int64_t* n_shared, int* blk0, int* nblk);
/* 128-byte ncclUniqueId for opts.nccl_id (call on one rank, broadcast to all); NSP_ERR_NCCL if
 * libnccl.so.2 cannot be loaded. */
nsp_status nsp_nccl_unique_id(void* out128);
/* The NCCL branch's call sequence (dlopen of libnccl.so.2, ncclGetUniqueId, ncclCommInitRank, in-place
 * ncclAllReduce(ncclDouble, ncclSum) on a stream, ncclCommDestroy) on a ONE-rank communicator on `device`:
 * count (> 0) fp64 values go through the allreduce and must come back unchanged; *max_abs_err (HOST pointer)
 * receives the largest deviation (0 expected).  SURVEY.md 8(e): a one-GPU box cannot run two ranks, this is
 * the hardware check of the production collective.  NSP_ERR_NCCL if NCCL cannot be loaded or a call fails. */
nsp_status nsp_nccl_selftest(int device, size_t count, double* max_abs_err);
/* Testing the sharded path on one device: a group for nranks (<= 16) host threads; each thread sets
 * opts.local_group, opts.nranks, opts.rank and calls nsp_setup / the solvers concurrently.  The
 * allreduce is then two host barriers around a rank-ordered device sum (no kernel waits on another
 * rank's kernel).  Destroy after every context of the group. */
void* nsp_local_group_create(int nranks);
void nsp_local_group_destroy(void* group);
/* orig_index: host int64[n_gamma_local]; local Gamma row -> original node id. */
nsp_status nsp_gamma_index(const nsp_ctx* ctx, int64_t* orig_index);
nsp_status nsp_workspace_bytes(const nsp_ctx* ctx, int s, size_t* bytes);
/* factor statistics: host int64[12] = {n_I, n_boundary_layer (sum b_j), L22 entries streamed per
 * apply (padded tiles), factor tiles, nnz(A_G), nnz(A_GI), max b_j, A_G bandwidth, sum b_j^2,
 * sum b_j, local blocks, W/V/U rows} */
nsp_status nsp_stats(const nsp_ctx* ctx, int64_t* stats12);
/* INT8 a2+a3 work per apply and 128-column tile (reading R10): host int64[3] = {int8 slice products
 * (128 x 64 x 64 each) k_oz_symm executes with the leading-zero-slice skip, the same count with all 28
 * products per (unit, K tile), unique bytes of the stored S_j^-1 tile slices it reads (skip applied)};
 * all 0 when the INT8 slices were not built.  Host-only; NSP_ERR_ARG on NULL. */
nsp_status nsp_ozaki_stats(const nsp_ctx* ctx, int64_t* out3);
/* Live timing of the batched factor-sweep kernel (a2+a3): enable = 1 records a CUDA event pair
 * around every launch on the context stream; nsp_profile_read synchronises the stream and
 * returns the summed duration and launch count since the last read. */
nsp_status nsp_profile(nsp_ctx* ctx, int enable);
nsp_status nsp_profile_read(nsp_ctx* ctx, double* sweep_ms, long long* sweeps);

/* Y = S_G X (eq:schur_complement), X, Y device n_gamma_local x s row-major; X != Y.
 * Steps: W = A_IG X (boundary-layer rows), V = L_j^{-1} W, U = L_j^{-T} V for all
 * blocks in one launch, Y = A_G X - A_GI U (north_star (a), (b)). */
nsp_status nsp_schur_apply(nsp_ctx* ctx, const double* X, double* Y, int s, void* ws);
/* Y = K_G X = A_GI A_I^{-1} A_IG X (the border contribution; Alg. 2 steps 2-4 via reading C1). */
nsp_status nsp_kgamma_apply(nsp_ctx* ctx, const double* X, double* Y, int s, void* ws);

/* Y = A_G X (Alg. 2 step 4 under reading C1: Y = A_G X after the border solve). */
nsp_status nsp_gamma_apply(nsp_ctx* ctx, const double* X, double* Y, int s);

/* Breakdown-free block CG on S_G X = B (reading C3/C4),
 * X0 = 0, stop when max_j ||R_j||/||B_j|| <= tol.  Returns NSP_OK,
 * NSP_NOT_CONVERGED, NSP_ERR_INDEFINITE, NSP_ERR_STAGNATION or NSP_ERR_NUMERICAL. */
nsp_status nsp_block_cg(nsp_ctx* ctx, const double* B, double* X, int s, double tol, int maxit,
                        void* ws, nsp_report* rep);

/* Alg. 2 steps 1-12 (opts.nys_power = q > 0: first q power steps G <- orth(B_H G),
 * each one block solve; rep->iters = total inner iterations): B = K_G Omega; block CG to tol_inner;
 * Y = A_G X; thin Cholesky-QR2 of Y; C = sym(Omega^T Y); EVD split at eps; T; EVD of T;
 * U~ = Q W(:,1:k); Z = A_G^{-1} U~; keeps (Z, Sigma) in ctx for nsp_pcg.
 * Omega: device n_gamma_local x (rank+oversample) row-major, or NULL: generated on the device from
 * `seed` (Philox4x32-10 stream 0, Box-Muller; the row index is the global Gamma index, so it equals
 * nsp_inputs.philox.gaussian_block(seed, 0, n_gamma, s) up to the last-ulp rounding of log / cos;
 * reading C7).  NULL is accepted for nys_form 0 / 1 (NSP_ERR_ARG for the M_3 / M_1 forms). */
nsp_status nsp_nystrom(nsp_ctx* ctx, int rank, int oversample, uint64_t seed, const double* Omega,
                       double tol_inner, int maxit_inner, void* ws, nsp_report* rep);
/* sigma: host double[>= rank]; rank_out: approximation rank. */
nsp_status nsp_nystrom_sigma(const nsp_ctx* ctx, double* sigma, int* rank_out);
/* Y = M X for M in {0: identity, 1: A_G^{-1}, 2: M_2 (M_1 / M_3 after nys_form 3 / 2),
 * 3: R_G^{-T} (X in the Gamma order, Y in R_G's row order), 4: R_G^{-1} (X in R_G's row order, Y in the
 * Gamma order)}, A_G = R_G^T R_G the setup's A_G factor (opts.ag_order); device n_gamma_local x s. */
nsp_status nsp_precond_apply(nsp_ctx* ctx, int which, const double* X, double* Y, int s, void* ws);

/* Full solve A x = b through eq:A_LDLT: f = b_G - A_GI A_I^{-1} b_I; PCG on
 * S_G w = f (eq:Sx=b) with precond {0 none, 1 A_G^{-1} (S~_1), 2 M_2, 3 M_A-DEF2 =
 * A_G^{-1} + Z E^{-1} Z^T (I - S_G A_G^{-1}), E = Z^T S_G Z (the adapted-deflation variant of M_2,
 * eq:deflation_comp_from_low_rank / PAPER.md:961-962, reading R5; non-symmetric)}; with
 * opts.nys_form 2 / 3 the pair (2, 3) is (M_3, M_A-DEF3) / (M_1, M_A-DEF1) - the same forms built on
 * that variant's Z; x_I = A_I^{-1}(b_I - A_IG w); un-permute.  b, x: device fp64[n] in ORIGINAL order.
 * The iteration runs as one device-driven CUDA graph (single rank); rep->hist gets the recurrence
 * residual of every iteration.  Single rank only (NSP_ERR_STATE for nranks > 1).
 * Returns NSP_ERR_STATE for 2 / 3 before nsp_nystrom. */
nsp_status nsp_pcg(nsp_ctx* ctx, const double* b, double* x, double tol, int maxit, int precond,
                   void* ws, nsp_report* rep);

/* Switch the block-CG preconditioner of an existing context (opts.bcg_precond, reading C2):
 * 0 = none (M = I), 1 = A_G^{-1} (needs the A_G factor / Chebyshev operator: opts.factor_gamma at
 * setup, else NSP_ERR_STATE).  The workspace size (nsp_workspace_bytes) does not depend on it. */
nsp_status nsp_set_bcg_precond(nsp_ctx* ctx, int precond);

/* ---- evidence and kernel-level testing ----
 * Dispatch-path counters: how many times each shape-specialised path was DISPATCHED in this process
 * (an eager launch or a capture into a CUDA graph that is then replayed).  Tests read deltas to
 * assert that the bench's code path (e.g. the one-wave s = 128 panel, the symmetric Gram) is the
 * one their oracle comparison exercised.  out: host long long[n]; returns NSP_PATH_COUNT. */
enum {
  NSP_PATH_PANEL_ROWS = 0,   /* k_panel_rows: s = 128 one-wave row-range panel (n >= 64 x SMs) */
  NSP_PATH_PANEL_TILES = 1,  /* k_panel: 64 x 64 tile panel (any s, any n) */
  NSP_PATH_GRAM_SYM = 2,     /* Gram X^T X computing only the tiles on / above the diagonal */
  NSP_PATH_GRAM_DE = 3,      /* [D | E] = P^T [Q | R] with D's upper tiles mirrored */
  NSP_PATH_GRAM_FULL = 4,    /* Gram with every output tile computed */
  NSP_PATH_SYMM = 5,         /* a2+a3 as the symmetric S_j^{-1} product (k_symm) */
  NSP_PATH_SWEEPS = 6,       /* a2+a3 as two batched triangular sweeps (k_trsm_fb) */
  NSP_PATH_SYMV = 7,         /* a2+a3 for one column (k_symv1) */
  NSP_PATH_PANEL_GRAM = 8,   /* fused panel + Gram partial (R -= Q alpha with Q^T R; W = R + P beta with W^T W) */
  NSP_PATH_CHOL_SOLVE = 9,   /* fused s x s Cholesky + triangular solve (one launch) */
  NSP_PATH_OZAKI = 10,       /* a2+a3 on the INT8 tensor cores (k_oz_slice_w + k_oz_symm, reading R10) */
  NSP_PATH_COUNT = 16
};
int nsp_path_counters(long long* out, int n);

/* Kernel-level test entry points for the block-CG building blocks (rows a6, a8, a10, a11) on caller
 * device data, stream-ordered on `stream` (cudaStream_t), synchronous on return.  Blocks are n x s
 * row-major with ld = s, s in {64, 128}.  path: 0 = the production dispatch, 1 = the generic
 * kernels (64 x 64 tile panel, full-tile Gram).
 *  nsp_dev_panel: Out = Cin + sgn * In M (M s x s; Cin may be NULL = 0, may alias Out);
 *                 colsq (nullable, device double[s]) = column sums of squares of Out in the kernel's
 *                 fixed reduction order.
 *  nsp_dev_gram:  out = Xa^T Xb (s x s); with Xb2 != NULL also out2 = Xa^T Xb2; lower_first: out is
 *                 only read through its lower triangle (D of [D | E]). */
nsp_status nsp_dev_panel(double* Out, const double* Cin, const double* In, const double* M, int64_t n, int s,
                         double sgn, double* colsq, int path, void* stream);
nsp_status nsp_dev_gram(const double* Xa, const double* Xb, const double* Xb2, int64_t n, int s, double* out,
                        double* out2, int lower_first, int path, void* stream);
/*  nsp_dev_panel_gram: the fused s = 128 pass (n >= 64 x SMs, else NSP_ERR_ARG): Out = Cin + sgn In M and
 *                 gram = In^T Out (gmode 0: the R -= Q alpha, F = Q^T R pass) or Out^T Out (gmode 1: the
 *                 W = R + P beta, W^T W pass; exactly symmetric); colsq as nsp_dev_panel. */
/*  nsp_dev_philox_gaussian: out (device rows x s, row-major) = the device Omega generator of nsp_nystrom
 *                 (Omega == NULL) for the global rows row0 .. row0+rows-1 and Philox stream `stream_id`. */
nsp_status nsp_dev_philox_gaussian(double* out, int64_t rows, int s, uint64_t seed, unsigned stream_id, int64_t row0,
                                   void* stream);
/*  nsp_dev_set_fused_pg: process-wide choice of the fused s = 128 panel + Gram pass in block CG for the
 *                 contexts' NEXT graph captures: 0 = production (off: measured not faster),
 *                 1 = whenever the shape allows (n >= 64 x SMs; the oracle parity test), 2 = never. */
nsp_status nsp_dev_set_fused_pg(int mode);
nsp_status nsp_dev_panel_gram(double* Out, const double* Cin, const double* In, const double* M, int64_t n,
                              double sgn, int gmode, double* gram, double* colsq, void* stream);

const char* nsp_last_error(const nsp_ctx* ctx);
/* Number of device kernels this library has launched in the process (evidence counter). */
long long nsp_kernel_launches(void);
void nsp_destroy(nsp_ctx* ctx);

#ifdef __cplusplus
}
#endif
#endif /* NSP_H */
