// Internal data layout of the nsp context (DESIGN.md §"Data layout in HBM").
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <vector>

#include "../../include/nsp.h"
#include <nvtx3/nvToolsExt.h>

// NVTX range around an ABI call (tracing: visible in nsys / ncu --nvtx timelines; header-only NVTX3,
// a no-op unless a tool is attached)
struct NspNvtx {
  explicit NspNvtx(const char* name) { nvtxRangePushA(name); }
  ~NspNvtx() { nvtxRangePop(); }
};

#define NSP_TILE 64          // factor tile edge (rows = cols)
#define NSP_TILE_ELEMS (NSP_TILE * NSP_TILE)
// S_j^{-1} tiles are stored PADDED (64 rows x 68 doubles): one stored tile is one contiguous bulk copy
// (TMA) into the bank-conflict-free shared-memory layout of the DMMA fragments
#define NSP_MINV_LD 68
#define NSP_MINV_TILE (NSP_TILE * NSP_MINV_LD)

// Per-block factor layout (one entry per local block j, and one for A_G).
// Local ordering of block j: [I1 (band order, n1 rows, padded to nt1*64)]
// [B = boundary layer (b rows, padded to ntb*64)].  Tiles are 64x64 row-major.
//  band tile (I, K), 0 <= I-K <= wb, I < nt1:   band[band_off + K*(wb+1) + (I-K)]
//  border tile (I', K), I' < ntb, K < nt1:      scratch[border_off + I'*nt1 + K]
//  dense tile (I', J'), J' <= I' < ntb:         dense[dense_off + I'(I'+1)/2 + J']
// Diagonal tiles hold inv(L_KK) after factorisation.
struct FacSub {
  int nt1, ntb, wb, pad_;
  int64_t band_off;      // tiles
  int64_t dense_off;     // tiles
  int64_t border_off;    // tiles, relative to the batch scratch base (-1 if none)
  int64_t wvu_row;       // first row of this block in the W/V/U buffer (ntb*64 rows)
  int n1, b;             // true sizes
  int border_first_off;  // index into border_first[] (ntb entries)
  int status_idx;        // index into the factor status array
};

// A batched triangular system for k_tri_fb: tiles at T (dense lower if wb < 0, else band of
// half-width wb tiles), nt tile rows, rows row0.. of the right-hand-side buffer.
struct TriSys {
  const double* T;
  int nt, wb;
  int64_t row0;
};

struct DevCSR {   // device CSR with int32 row pointers (nnz < 2^31 checked)
  int64_t rows = 0, nnz = 0;
  int32_t* rowptr = nullptr;
  int32_t* col = nullptr;
  double* val = nullptr;
};

struct HostCSR32 {
  std::vector<int32_t> rowptr, col;
  std::vector<double> val;
};

// key of the cached block-CG iteration graph (nsp_solver.cu)
struct PcgKey {
  const double* w = nullptr;
  int64_t n = 0;
  int precond = -1;
  double tol = 0;
  int maxit = 0;
  int rank = 0;
  const void* Z = nullptr;     // Nystrom basis / E factor buffers (re-allocated by a new nsp_nystrom)
  const void* E = nullptr;
  long long gen = 0;
  bool operator==(const PcgKey& o) const {
    return w == o.w && n == o.n && precond == o.precond && tol == o.tol && maxit == o.maxit && rank == o.rank &&
           Z == o.Z && E == o.E && gen == o.gen;
  }
};
struct GraphKey {
  const void* X = nullptr;
  int64_t n = 0;
  int s = 0;
  double tol = 0.0;
  int kind = 0, usem = 0;
  double tau = 0.0;
  int af = 0;   // apply-first structure (reading R9)
  bool operator==(const GraphKey& o) const {
    return X == o.X && n == o.n && s == o.s && tol == o.tol && kind == o.kind && usem == o.usem && tau == o.tau &&
           af == o.af;
  }
};

struct nsp_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  nsp_opts opts{};
  int nranks = 1, rank = 0;
  int64_t n = 0, nG = 0;          // global n, local Gamma rows
  int64_t nG_global = 0;
  int K = 0, nsub = 0, blk0 = 0;  // local blocks [blk0, blk0+nsub)
  std::string err;

  std::vector<int64_t> gamma;     // local Gamma row -> original id
  std::vector<int64_t> gamma_gidx;  // local Gamma row -> global Gamma index (ascending original id)
  std::vector<FacSub> subs;       // host copy
  std::vector<int64_t> sub_n;     // |block j|

  // device factor storage
  FacSub* d_subs = nullptr;
  double* d_band = nullptr;   int64_t band_tiles = 0;
  double* d_dense = nullptr;  int64_t dense_tiles = 0;
  int* d_border_first = nullptr;
  int64_t wvu_rows = 0;       // total W/V/U rows (sum ntb*64)
  int max_ntb = 0;

  // Gamma-side sparse operators
  // a2+a3 as one symmetric product (opts.apply_kernel = 0): M_j = S_j^{-1} tiles + work items
  double* d_minv = nullptr;
  int2* d_items = nullptr;
  int n_items = 0;
  int n_items_sh = 0;         // several ranks: items [0, n_items_sh) belong to blocks coupled to shared rows
  // a2+a3 on the INT8 tensor cores (nsp_ozaki.cu, reading R10): D-scaled S_j^{-1} lower tiles as 7 int8
  // slices each, per-row delta exponents, per-block mu exponents
  int8_t* d_oz_msl = nullptr;
  int* d_oz_dexp = nullptr;
  int* d_oz_mexp = nullptr;
  int* d_oz_tblk = nullptr;   // W/V/U tile -> local block
  int2* d_oz_pairs = nullptr; // (block, even tile row I0): the two-CTA cluster work units
  int n_oz_pairs = 0;
  int* d_oz_ctr = nullptr;    // k_oz_symm's dynamic work counter (reset before every launch)
  int8_t* d_oz_mz = nullptr;  // per stored tile: leading all-zero slices (skipped by the product)
  // int8 slice products (128 x 64 x 64 each) one column tile of an apply executes: with the leading-zero
  // skip (natural K order, the unit's first K tile unskipped) and the full 28 per (unit, K tile)
  int64_t oz_prod_exec = 0, oz_prod_full = 0;
  int64_t oz_slice_bytes = 0;   // unique bytes of the stored-tile slices one column tile reads (skip applied)
  DevCSR A2G;                 // rows: W/V/U rows; cols: local Gamma
  DevCSR AGG2;                // rows: local Gamma; cols < nG: A_G, cols >= nG: -A_GI (W/V/U row + nG)
  DevCSR AGSH;                // multi-rank: shared x shared part of A_G (rows/cols relative to n_priv)
  DevCSR AGO;                 // one rank: A_G alone (the cols < nG prefix of every AGG2 row) - the
                              // Chebyshev A_G^{-1} steps read only these entries
  // the same A_G as sliced ELL (32-row slices, column-major within a slice, width = the slice's longest
  // row, col -1 = padding): the s = 1 Chebyshev step, one thread per row with no row-pointer hop
  int64_t* d_sell_ptr = nullptr;   // nslices + 1 element offsets
  int32_t* d_sell_col = nullptr;
  double* d_sell_val = nullptr;
  uint8_t* d_sell_code = nullptr;   // dictionary-coded values (<= 255 distinct) and their table, or null
  double* d_sell_tab = nullptr;
  int64_t n_priv = 0;         // local Gamma rows [0, n_priv) private, [n_priv, nG) shared (replicated)
  struct NspComm* comm = nullptr;

  // A_G factor (band, RCM order): rows of the band buffer -> local Gamma index (-1 = padding)
  bool has_ag = false;
  // or A_G^{-1} by a fixed Chebyshev iteration ("an iterative solver to solve linear
  // systems with A_G"; opts.ag_solver): spectrum bounds [cheb_a, cheb_b], K steps, per-step coefficients
  bool ag_cheb = false;
  double cheb_a = 0.0, cheb_b = 0.0;
  int cheb_K = 0;
  std::vector<double> cheb_c1, cheb_c2;
  double* d_gband = nullptr;  int64_t gband_tiles = 0;
  TriSys* d_gsys = nullptr;   int g_nt = 0, g_wb = 0;
  int32_t* d_gperm = nullptr;     // band row -> Gamma row (size g_nt*64)
  int32_t* d_gperm_inv = nullptr; // Gamma row -> band row
  // partitioned A_G solve (narrow band, setup_gamma_factor): P chunk systems + spikes
  int g_P = 0;
  TriSys* d_gchunks = nullptr;
  int* d_gchunk_first = nullptr;   // P + 1
  int* d_gtile_chunk = nullptr;    // g_nt
  double* d_gGF = nullptr;         // g_nt tiles each (g_P > 1, wb <= 1): k_band_rec operands
  double* d_gXB = nullptr;
  double* d_gGB = nullptr;
  double* d_gspkF = nullptr;       // g_nt*64 x 64: S_k rows
  double* d_gspkB = nullptr;       // g_nt*64 x 64: T_k rows

  // Nystrom-Schur M_2 = A_G^{-1} + Z Sigma Z^T (Alg. 2 steps 11-12)
  double* d_Z = nullptr;          // nG x nys_ld
  double* d_sigma = nullptr;      // nys_ld
  int nys_rank = -1, nys_ld = 0;
  long long nys_gen = 0;   // bumped by every nsp_nystrom
  double* d_ELp = nullptr;        // Cholesky (k_chol16 packed) of E = Z^T S_G Z for M_A-DEF2
  bool adef_ok = false;
  bool adef_ready = false;        // E of the current Z formed (lazily, on the first M_A-DEF2 use)
  std::vector<double> h_sigma;

  // full-system solve (nsp_pcg; eq:A_LDLT PAPER.md:381-385): every block's interior rows I1 in
  // band order (padded to nt1*64 rows, blocks concatenated), its band factor L11 as a TriSys,
  // original-id maps, and the block couplings as CSRs with a leading identity part:
  //   CB rows = W/V/U rows:  [ I | -A_B1 ]  (cols < wvu_rows: identity, cols >= wvu_rows: band row)
  //   C1 rows = band rows:   [ I | -A_1B ]  (cols < i1_rows: identity, cols >= i1_rows: W/V/U row)
  int64_t i1_rows = 0;
  int i1_wbmax = -1;          // largest band half-width (tiles) of the I1 factors
  TriSys* d_i1sys = nullptr;
  int32_t* d_i1_src = nullptr;
  int32_t* d_b_src = nullptr;
  int32_t* d_g_src = nullptr;
  DevCSR CB, C1;
  DevCSR AII;                 // opts.nys_form 1/2: A_I on the interior layout (+ the -I coupling of B rows)
  int32_t* d_int_src = nullptr;   // interior layout row -> original id (-1 padding)

  // statistics
  int64_t n_I = 0, n_bl = 0, nnz_AG = 0, nnz_AGI = 0, max_b = 0, ag_bw = 0;

  // internal workspace (when caller passes ws == NULL)
  void* ws_int = nullptr; size_t ws_int_bytes = 0;
  // small pinned host status
  void* h_status = nullptr;

  // cached CUDA graph of one block-CG iteration (tail + head), captured on gstream
  cudaGraphExec_t bcg_graph = nullptr;
  GraphKey bcg_key;
  long long bcg_graph_kernels = 0;   // kernel nodes per launch of bcg_graph (launch evidence counter)
  // cached device-driven block-CG loop: one graph whose WHILE node repeats tail + head + loop
  // control until the device-side stop test fires (one host sync per solve)
  cudaGraphExec_t bcg_wgraph = nullptr;
  GraphKey bcg_wkey;
  int bcg_wmaxit = 0;
  long long bcg_wbody_kernels = 0;
  double* d_bhist = nullptr;   // per-iteration relres (device), capacity bhist_cap
  int* d_bwidth = nullptr;     // per-iteration active width (device)
  int bhist_cap = 0;
  bool bcg_no_while = false;   // the WHILE graph could not be built: per-iteration graphs
  // cached device-driven PCG loop (WHILE node around two iterations + loop control)
  cudaGraphExec_t pcg_wgraph = nullptr;
  PcgKey pcg_wkey;
  long long pcg_wbody_kernels = 0;
  double* d_phist = nullptr;
  int phist_cap = 0;
  bool pcg_no_while = false;
  // cached CUDA graph of PCG_CHUNK outer-PCG iterations
  cudaGraphExec_t pcg_graph = nullptr;
  PcgKey pcg_key;
  long long pcg_graph_kernels = 0;
  cudaStream_t gstream = nullptr;
  cudaStream_t side_stream = nullptr;   // block CG: the deferred X update (forked, joined before orth)
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  cudaStream_t comm_stream = nullptr;   // several ranks: the shared-row allreduce, overlapped with the apply
  cudaEvent_t ev_cfork = nullptr, ev_cjoin = nullptr;
  cudaStream_t apply_stream = nullptr;  // block CG: S_G W on a forked branch while W^T W / chol run (R9)
  cudaEvent_t ev_afork = nullptr, ev_ajoin = nullptr;
  bool capturing = false;          // block CG is capturing its iteration graph
  bool gprof_in_graph = false;     // the cached graph records gprof_ev around a2+a3
  cudaEvent_t gprof_ev[2] = {nullptr, nullptr};
  double gprof_ms = 0.0;
  long long gprof_n = 0;
  // live kernel timing (nsp_profile): event pairs around the factor-sweep launches
  int prof_on = 0;
  std::vector<cudaEvent_t> prof_ev;   // 2 per record
  int prof_used = 0;
  int64_t sum_b2 = 0, sum_b = 0;
};

// number of device kernels launched by this library (evidence counter)
void nsp_count_launch();
void nsp_count_launches(long long k);   // kernels executed by a graph launch
long long nsp_launch_count();

// kernel launchers (nsp_kernels.cu)
namespace nspk {
void scatter(double* base, const int64_t* idx, const double* val, int64_t cnt, cudaStream_t st);
void set_pad_identity(double* base, const int64_t* tile_idx, const int* first_row, int cnt, cudaStream_t st);
void tile_cholesky(const FacSub* subs, int nsub, double* band, double* dense, double* scratch,
                   const int* border_first, int* status, cudaStream_t st);
// Y[r, c] (c < s) = sum_k val_k * X(col_k, c); mode 0: Y = A X (X ld ldx);
// mode 1: Y = A [X ; U] with cols >= split reading U (ld ldu) at col-split;
// mode 2: Y = -(cols >= split part only)  (K_G apply); mode 3: cols < split only (A_G X);
// mode 4: Y += A X
// Y ld ldy; columns s..ldy-1 of Y are written with 0 when zero_pad.
// chunk strides: column c at row * ld + (c / 32) * cs + c % 32 (cs = 32: row-major)
void spmm_cs(const DevCSR& A, const double* X, int ldx, const double* U, int ldu, int64_t ucs, int64_t split,
             double* Y, int ldy, int64_t ycs, int ypad, int s, int mode, bool zero_pad, cudaStream_t st);
// a1 for the INT8 a2+a3 (mode 0, chunk-major W, ld 36): also folds the per-(block, column) W^T scale exponents
// into ozse (atomicMax; ozse pre-filled with INT_MIN-ish); false (nothing launched) when the shape is not eligible
bool spmm_cs_oz(const DevCSR& A, const double* X, int ldx, double* Y, int64_t ycs, int ypad, int s,
                const int* ozdx, const int* oztb, int* ozse, cudaStream_t st);
void spmm(const DevCSR& A, const double* X, int ldx, const double* U, int ldu, int64_t split,
          double* Y, int ldy, int s, int mode, bool zero_pad, cudaStream_t st);
void trsm_fb(const FacSub* subs, int nsub, const double* dense, double* wvu, int ldw, int cw,
             cudaStream_t st);
// setup: M_j = S_j^{-1} = L22^{-T} L22^{-1} tiles (same layout as the L22 tiles)
void l22_inverse(const FacSub* subs, int nsub, int max_ntb, const double* dense, double* minv, cudaStream_t st);
// a2+a3 as U_j = M_j W_j (items = (block, tile row)), W -> U out of place
void symm(const FacSub* subs, const int2* items, int nitems, const double* minv, const double* W, double* U, int ldw,
          int cw, cudaStream_t st,
          int64_t cm_stride = 0);
// wbmax: largest band half-width (tiles) of the systems, -1 unknown; <= 2 with cw 32 selects k_band_fb
// a2+a3 on the INT8 tensor cores (Ozaki splitting, nsp_ozaki.cu)
size_t oz_mslice_bytes(int64_t dense_tiles);
size_t oz_wslice_bytes(int64_t wvu_rows, int s);
void oz_setup(const FacSub* subs, int nsub, int max_ntb, const int2* items, int nitems, const double* minv,
              int* dexp, int* mexp, int8_t* msl, int8_t* mz, cudaStream_t st);
// W^T slices of every block (chunk-major W, nch chunks, s columns) -> wsl, sexp (nsub * nct * 128 ints)
void oz_slice_w(const FacSub* subs, const int2* items, int nitems, int nsub, int s, int nch, const double* W,
                int64_t cs, const int* dexp, int8_t* wsl, int* sexp, cudaStream_t st, bool have_exp = false);
// U = S_j^{-1} W for the items [0, nitems) from the slices (chunk-major U)
// s = 1: u_j = S_j^{-1} w_j from the slices (one column, ld ldw; P: partial slots as k_symv1)
void oz_symv1(const FacSub* subs, const int2* items, int nitems, int max_ntb, const int8_t* msl, const int* dexp,
              const int* mexp, const double* W, int ldw, double* U, double* P, cudaStream_t st);
// pairs (j, I0), I0 even, covering the same items: clusters of two CTAs share the W^T slices (multicast)
void oz_product(const FacSub* subs, const int2* items, int nitems, int s, int nch, double* U, int64_t cs,
                const int* dexp, const int* mexp, const int8_t* msl, const int8_t* wsl, const int* sexp,
                cudaStream_t st, const int2* pairs = nullptr, int npairs = 0, int* uctr = nullptr,
                const int8_t* mz = nullptr);
// a2+a3 for one column (ld ldw, column 0): u_j = S_j^{-1} w_j, matrix-vector (s = 1)
void symv(const FacSub* subs, const int2* items, int nitems, int max_ntb, const double* minv, const double* W, int ldw,
          double* U, cudaStream_t st);
void symv1(const FacSub* subs, const int2* items, int nitems, int max_ntb, const double* minv, const double* W, int ldw,
           double* U, double* P, cudaStream_t st);
// partitioned A_G solve, one column: the reassociated chunk sweeps (k_band_rec_vec) and their setup
void band_prep(const double* T, int nt, int wb, double* XF, double* GF, double* XB, double* GB, cudaStream_t st);
// Xd tile of row I at Xd + I * xstride * 4096 (the band's own diagonal tiles: xstride = wb + 1)
void band_rec_vec(const TriSys* sys, int nsys, const double* Xd, int64_t xstride, const double* Gc, double* buf, bool fwd,
                  cudaStream_t st);
void band_rec(const TriSys* sys, int nsys, const double* Xd, int64_t xstride, const double* Gc, double* buf, int ldw,
              bool fwd, cudaStream_t st);
void tri_fb(const TriSys* sys, int nsys, double* buf, int ldw, int cw, bool fwd, bool bwd, cudaStream_t st,
            int wbmax = -1);
// partitioned narrow-band solve of the A_G factor: coupling-tile recurrence / parallel spike update
void spike_tail(const double* spk, const int* chunk_first, int P, double* buf, int ldw, int s, bool fwd,
                cudaStream_t st);
void spike_update(const double* spk, const int* chunk_first, const int* tile_chunk, int P, int nt, double* buf,
                  int ldw, int s, bool fwd, cudaStream_t st);
void gather_rows(const double* src, int lds, const int32_t* idx, int64_t rows, double* dst, int ldd, int s,
                 double scale, cudaStream_t st);
void scatter_rows(const double* src, int lds, const int32_t* idx, int64_t rows, double* dst, int ldd, int s,
                  bool accumulate, cudaStream_t st);
// one fused Chebyshev step (one rank): t = A_G d (the cols < split prefix of A's rows), x += d, r -= t,
// dn = c1 d + c2 r; blocks n x ld row-major (ld = 1 with s = 1)
void cheb_step(const DevCSR& A, int64_t split, const double* d, int ld, int s, double* x, double* r, double* dn,
               double c1, double c2, bool want_d, cudaStream_t st);
// the s = 1 step on the sliced-ELL A_G (rows = n_G)
// three-term Chebyshev step x_{k+1} = x_k + c1 (x_k - x_{k-1}) + c2 (b - A x_k) (rows of A with cols < split; s = 1:
// the sliced ELL copy of A_G over `split` rows); xn may alias xp
void cheb3_step(const DevCSR& A, int64_t split, const double* xk, int ld, int s, const double* xp, const double* b,
                double* xn, double c1, double c2, cudaStream_t st, const int64_t* sptr = nullptr,
                const int32_t* scol = nullptr, const double* sval = nullptr, const uint8_t* code = nullptr,
                const double* tab = nullptr);
void cheb_step_sell(int64_t rows, const int64_t* sptr, const int32_t* col, const double* val, const double* d,
                    double* x, double* r, double* dn, double c1, double c2, bool want_d, cudaStream_t st,
                    const uint8_t* code = nullptr, const double* tab = nullptr);
// Gaussian block on the device, bit-compatible with nsp_inputs.philox.gaussian_block (reading C7):
// out[r * ld + j] (j < s; columns s..ld-1 zeroed) = N(0,1) from Philox4x32-10 counter (gidx[r] * s + j,
// stream, 0), key = seed, Box-Muller cosine branch.  gidx: device int64 row indices.
void philox_gaussian(double* out, int64_t rows, int s, int ld, const int64_t* gidx, uint64_t seed, uint32_t stream,
                     cudaStream_t st);
}  // namespace nspk

#define NSP_CUDA_TRY(ctx, call)                                                   \
  do {                                                                            \
    cudaError_t e_ = (call);                                                      \
    if (e_ != cudaSuccess) {                                                      \
      (ctx)->err = std::string("CUDA error: ") + cudaGetErrorString(e_) + " at " + \
                   __FILE__ + ":" + std::to_string(__LINE__);                     \
      return NSP_ERR_CUDA;                                                        \
    }                                                                             \
  } while (0)
