// Breakdown-free block CG on S_G X = B (PAPER.md:1212-1216 [JiL17, Ole80]; readings C3/C4), the
// Nystrom-Schur construction (Alg. 2) and the outer PCG (eq:Sx=b) - host
// drivers enqueueing the device kernels on the context stream.  One small device->host status
// read per iteration (the convergence / breakdown flags); everything else stays on the device.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <map>
#include <vector>
#include <cstring>
#include <string>

#include "nsp_blas.h"
#include "nsp_comm.h"
#include "nsp_solver.h"

namespace nspi {

// NSP_TRACE=1: CUDA-event phase timing of block CG, printed to stderr at exit (diagnostics only)
struct Tracer {
  bool on = false;
  cudaStream_t st = nullptr;
  std::vector<cudaEvent_t> ev;
  std::vector<const char*> lab;
  std::vector<double> host_us;
  std::chrono::steady_clock::time_point t0;
  void init(cudaStream_t s) {
    const char* e = getenv("NSP_TRACE");
    on = e && e[0] == '1';
    st = s;
    t0 = std::chrono::steady_clock::now();
  }
  void mark(const char* l) {
    if (!on) return;
    cudaEvent_t e;
    cudaEventCreate(&e);
    cudaEventRecord(e, st);
    ev.push_back(e);
    lab.push_back(l);
    host_us.push_back(std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count());
  }
  void report() {
    if (!on || ev.size() < 2) return;
    cudaStreamSynchronize(st);
    std::map<std::string, std::pair<double, int>> agg, hagg;
    for (size_t i = 1; i < ev.size(); ++i) {
      float ms = 0;
      cudaEventElapsedTime(&ms, ev[i - 1], ev[i]);
      auto& a = agg[lab[i]];
      a.first += ms;
      a.second++;
      auto& h = hagg[lab[i]];
      h.first += host_us[i] - host_us[i - 1];
      h.second++;
    }
    for (auto& kv : agg)
      fprintf(stderr, "[nsp trace] %-14s gpu %9.3f ms  host %9.3f ms  n=%d\n", kv.first.c_str(), kv.second.first,
              hagg[kv.first].first / 1000.0, kv.second.second);
    for (auto e : ev) cudaEventDestroy(e);
    ev.clear();
    lab.clear();
    host_us.clear();
  }
};

struct Carver {
  char* p;
  size_t off = 0;
  explicit Carver(char* base) : p(base) {}
  double* take(size_t ndoubles) {
    off = (off + 255) & ~size_t(255);
    double* r = (double*)(p + off);
    off += ndoubles * 8;
    return r;
  }
};

// Operator of the block CG: kind 0 = S_G on the n_G border rows (reading C1, the default), kind 1 =
// the paper-literal S_I on the interior rows (eq:SI; interior layout = all blocks' band rows, then
// all boundary-layer rows; padding rows stay zero) preconditioned by A_I.
struct BcgWs {
  int sp, kind;
  int64_t n;
  double *X, *R, *P, *Q, *W, *Z, *QW;
  double *tG, *hB, *wB, *agb;   // kind 1 scratch
  double *D, *E, *F, *G, *Ld, *Ldi, *T, *al, *be, *tmp, *Vw, *Vs, *lam, *bnorm, *rsq, *gram, *npart, *wvu;
  BcgStatus* st;
};

static int sp_of(int s) { return ((s + 63) / 64) * 64; }
size_t ag_ws_doubles(const nsp_ctx* c, int s);

static size_t bcg_layout(const nsp_ctx* c, int s, char* base, BcgWs* w, int kind = 0) {
  const int sp = sp_of(s);
  const int64_t n = kind ? c->i1_rows + c->wvu_rows : c->nG;
  Carver cv(base ? base : (char*)nullptr);
  BcgWs t{};
  t.sp = sp;
  t.kind = kind;
  t.n = n;
  const size_t blk = (size_t)std::max<int64_t>(n, 1) * sp;
  t.X = cv.take(blk);
  t.R = cv.take(blk);
  t.P = cv.take(blk);
  t.Q = cv.take(blk);
  t.W = cv.take(blk);
  // Z exists whenever M = A_G^{-1} is possible (nsp_set_bcg_precond may switch M after setup)
  t.Z = ((kind || c->opts.bcg_precond || c->has_ag) ? cv.take(blk) : nullptr);
  t.QW = cv.take(blk);   // S_G W of the apply-first iteration (reading R9)
  if (kind) {
    t.tG = cv.take((size_t)std::max<int64_t>(c->nG, 1) * sp);
    t.hB = cv.take((size_t)std::max<int64_t>(c->wvu_rows, 1) * sp);
    t.wB = cv.take((size_t)std::max<int64_t>(c->wvu_rows, 1) * sp);
    t.agb = cv.take(c->has_ag ? ag_ws_doubles(c, sp) : 1);
  }
  const size_t sm = (size_t)sp * sp;
  t.D = cv.take(sm);
  t.E = cv.take(sm);
  t.F = cv.take(sm);
  t.G = cv.take(sm);
  t.Ld = cv.take(sm);
  t.Ldi = cv.take(sm);
  t.T = cv.take(sm);
  t.al = cv.take(sm);
  t.be = cv.take(sm);
  t.tmp = cv.take(sm);
  t.Vw = cv.take((size_t)(sp + 1) * (sp + 1));
  t.Vs = cv.take(sm);
  t.lam = cv.take(sp);
  t.bnorm = cv.take(sp);
  t.rsq = cv.take(sp);
  t.gram = cv.take(nspb::gram_ws_doubles(n, sp, sp));
  t.npart = cv.take((size_t)((n + 63) / 64 + 1) * sp);
  t.wvu = cv.take(std::max(apply_ws_bytes(c, sp) / 8 + 1, c->has_ag ? ag_ws_doubles(c, sp) : 0));
  t.st = (BcgStatus*)cv.take(sizeof(BcgStatus) / 8 + 1);
  if (w) *w = t;
  return ((cv.off + 255) & ~size_t(255)) + 256;   // 256-aligned: callers carve more after it
}

size_t solver_ws_bytes(const nsp_ctx* c, int s) { return bcg_layout(c, s, nullptr, nullptr); }

void solver_free(nsp_ctx*) {}

static nsp_status read_status(nsp_ctx* c, BcgStatus* d, BcgStatus* h) {
  NSP_CUDA_TRY(c, cudaMemcpyAsync(h, d, sizeof(BcgStatus), cudaMemcpyDeviceToHost, c->stream));
  NSP_CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  return NSP_OK;
}

// Rows of the local block that enter Grams and norms: all local rows on one rank; with several
// ranks the private rows of every rank plus the shared rows once (rank 0), SURVEY.md §8(e).
static int64_t gram_rows(const nsp_ctx* c) { return (c->nranks <= 1 || c->rank == 0) ? c->nG : c->n_priv; }
static int64_t gram_rows(const nsp_ctx* c, const BcgWs& w) { return w.kind ? w.n : gram_rows(c); }

static bool fused_sxs() {
  static const bool on = [] {
    const char* e = getenv("NSP_FUSED_SXS");
    return !(e && e[0] == '0');
  }();
  return on;
}

// orth(Wm): Gram, Cholesky-QR with pivot test, eigen fallback; P = Wm T (reading C3)
static nsp_status orth(nsp_ctx* c, BcgWs& w, const double* Wm, int s, double* Pout,
                       cudaEvent_t join_before_panel = nullptr, bool gram_done = false, bool no_panel = false) {
  const int sp = w.sp;
  const int64_t n = w.n;
  cudaStream_t st = c->stream;
  if (!gram_done) {   // (gram_done: G = W^T W already formed by the fused W = Z + P beta pass)
    nspb::gram(Wm, sp, sp, Wm, sp, sp, gram_rows(c, w), w.G, sp, w.gram, st);
    nsp_status e = comm_allreduce(c, w.G, (size_t)sp * sp);
    if (e != NSP_OK) return e;
  }
  // CholQR with the pivot test (k_chol16 mode 1), T = R^{-1} = L^{-T} (skipped on fallback): one fused
  // launch (every CTA factors, then forms 8 columns of T), or the two-launch form with NSP_FUSED_SXS=0
  if (fused_sxs()) {
    nspb::chol_fac_solve(w.G, sp, 1, s, c->opts.orth_tau, w.Ldi, w.st, nullptr, 0, w.T, sp, 1.0, false, true, st);
  } else {
    nspb::chol_fac(w.G, sp, 1, s, c->opts.orth_tau, w.Ldi, w.st, st);
    nspb::chol_solve(w.Ldi, sp, nullptr, 0, w.T, sp, 1.0, false, true, &w.st->fallback, st);
  }
  // eigen fallback (gated on the pivot test): EVD and T = V_keep Lambda^{-1/2} in one launch
  nspb::small_eig(w.G, sp, s, w.Vw, sp + 1, w.lam, w.Vs, &w.st->fallback, st, c->opts.orth_tau, w.T, sp, w.st);
  if (no_panel) return NSP_OK;   // (apply-first: the caller forms P = W T and Q = (S W) T together)
  if (join_before_panel) NSP_CUDA_TRY(c, cudaStreamWaitEvent(st, join_before_panel, 0));   // X += P alpha done
  // P = W T; T upper triangular unless the eigen fallback fired (its zero chunks skipped, bitwise the same)
  nspb::panel(Pout, sp, nullptr, 0, Wm, sp, w.T, sp, sp, sp, n, 1.0, nullptr, st, &w.st->fallback);
  return NSP_OK;
}

// Z = M R
static nsp_status precond(nsp_ctx* c, const double* R, double* Z, int ld, int s, double* wvu);

// A_I^{-1} R on the interior layout, s columns (ld sp): per block, y_B = S_j^{-1}(r_B - A_B1 A_11^{-1}
// r_1), y_1 = A_11^{-1}(r_1 - A_1B y_B) (the block elimination of reading R3 with s right-hand sides)
static nsp_status ai_solve(nsp_ctx* c, BcgWs& w, const double* R, double* Z) {
  const int sp = w.sp;
  cudaStream_t st = c->stream;
  const int cw = 32;
  double* Z1 = Z;
  double* ZB = Z + c->i1_rows * (int64_t)sp;
  const double* R1 = R;
  const double* RB = R + c->i1_rows * (int64_t)sp;
  NSP_CUDA_TRY(c, cudaMemcpyAsync(Z1, R1, (size_t)c->i1_rows * sp * 8, cudaMemcpyDeviceToDevice, st));
  nspk::tri_fb(c->d_i1sys, c->nsub, Z1, sp, cw, true, true, st, c->i1_wbmax);                              // A_11^{-1} r_1
  nspk::spmm(c->CB, RB, sp, Z1, sp, c->wvu_rows, w.wB, sp, sp, 1, false, st);                  // r_B - A_B1 t_1
  if (c->d_minv) {
    nspk::symm(c->d_subs, c->d_items, c->n_items, c->d_minv, w.wB, ZB, sp, cw, st);           // y_B
  } else {
    nspk::trsm_fb(c->d_subs, c->nsub, c->d_dense, w.wB, sp, cw, st);
    NSP_CUDA_TRY(c, cudaMemcpyAsync(ZB, w.wB, (size_t)c->wvu_rows * sp * 8, cudaMemcpyDeviceToDevice, st));
  }
  nspk::spmm(c->C1, R1, sp, ZB, sp, c->i1_rows, Z1, sp, sp, 1, false, st);                     // r_1 - A_1B y_B
  nspk::tri_fb(c->d_i1sys, c->nsub, Z1, sp, cw, true, true, st, c->i1_wbmax);                              // y_1
  NSP_CUDA_TRY(c, cudaGetLastError());
  return NSP_OK;
}

// Q = S_I P = A_I P - A_IG A_G^{-1} A_GI P (eq:SI) on the interior layout
static nsp_status si_apply(nsp_ctx* c, BcgWs& w, const double* P, double* Q, int s) {
  const int sp = w.sp;
  cudaStream_t st = c->stream;
  const double* PB = P + c->i1_rows * (int64_t)sp;
  nspk::spmm(c->AGG2, nullptr, 0, PB, sp, c->nG, w.tG, sp, s, 2, true, st);                   // A_GI P_B
  nsp_status e = ag_solve(c, w.tG, sp, w.tG, sp, s, w.agb);                                    // A_G^{-1}
  if (e != NSP_OK) return e;
  nspk::spmm(c->A2G, w.tG, sp, nullptr, 0, 0, w.hB, sp, s, 0, true, st);                        // A_IG t
  nspk::spmm(c->AII, P, sp, w.hB, sp, w.n, Q, sp, s, 1, true, st);                             // A_I P - [0; h_B]
  NSP_CUDA_TRY(c, cudaGetLastError());
  return NSP_OK;
}

static nsp_status op_apply(nsp_ctx* c, BcgWs& w, const double* P, double* Q, int s) {
  if (w.kind) return si_apply(c, w, P, Q, s);
  return apply_into(c, P, w.sp, Q, w.sp, s, 1, w.wvu);
}

static nsp_status op_precond(nsp_ctx* c, BcgWs& w, const double* R, double* Z, int s) {
  if (w.kind) return ai_solve(c, w, R, Z);
  return precond(c, R, Z, w.sp, s, w.wvu);
}

// Device-driven block-CG loop control (end of every iteration of the WHILE-node body): count the
// iteration, record relres / width / fallback, and stop on the same tests, in the same order, as the
// host loop (indefinite, non-finite, all directions deflated, converged, maxit).
__global__ void k_bcg_loop_ctl(BcgStatus* st, double* hist, int* widths, int maxit,
                               cudaGraphConditionalHandle h) {
  asm volatile("griddepcontrol.wait;\n" ::: "memory");
  const int it = ++st->iters;          // completed iterations
  hist[it] = st->relres;
  widths[it - 1] = st->width;
  st->nfallback += st->fallback;
  const bool stop = st->indefinite || st->nonfinite || st->width == 0 || st->converged || it >= maxit;
  cudaGraphSetConditional(h, stop ? 0u : 1u);
}
__global__ void k_bcg_loop_init(BcgStatus* st, int iters) {
  st->iters = iters;
  st->nfallback = 0;
}

nsp_status block_cg_impl(nsp_ctx* c, const double* B, int ldb, double* Xout, int ldx, int s, double tol, int maxit,
                         BcgWs& w, nsp_report* rep) {
  const int sp = w.sp;
  const int64_t n = w.n;
  cudaStream_t st = c->stream;
  BcgStatus* hs = (BcgStatus*)c->h_status;
  const bool usem = w.kind ? true : c->opts.bcg_precond != 0;
  int iters = 0, fallbacks = 0;
  nsp_status ret = NSP_NOT_CONVERGED;
  Tracer tr;
  tr.init(st);
  tr.mark("start");
  // init: X = 0, R = B, bnorm
  NSP_CUDA_TRY(c, cudaMemsetAsync(w.X, 0, (size_t)n * sp * 8, st));
  nspb::copy_pad(B, ldb, w.R, sp, n, s, 1.0, st);
  const int64_t ng = gram_rows(c, w);
  const bool multi = c->nranks > 1;
  // fused tall-skinny passes (s = 128, single rank, one-wave shapes): R -= Q alpha with F = Q^T R (M = I)
  // and W = Z + P beta with W^T W - each tall block read once per use (NSP_FUSED_PG=0: separate kernels)
  const bool fuse_pg = !multi && nspb::panel_gram_ok(sp, n);
  nsp_status e;
  nspb::colsq(w.R, sp, ng, s, sp, w.npart, w.rsq, st);
  if ((e = comm_allreduce(c, w.rsq, sp)) != NSP_OK) return e;
  nspb::sqrt_vec(w.rsq, w.bnorm, sp, st);
  BcgStatus init{};
  init.width = s;
  std::memcpy(hs, &init, sizeof(init));
  NSP_CUDA_TRY(c, cudaMemcpyAsync(w.st, hs, sizeof(BcgStatus), cudaMemcpyHostToDevice, st));
  nspb::converge(w.rsq, w.bnorm, s, tol, w.st, nullptr, st);
  e = read_status(c, w.st, hs);
  if (e != NSP_OK) return e;
  if (rep && rep->hist && rep->hist_cap > 0) rep->hist[0] = hs->relres;
  double relres = hs->relres;
  double* Zr = usem ? w.Z : w.R;
  // head: a1-a8 (Q = S P, D|E, chol(D), alpha, X/R update, norms, convergence) + the status copy
  // apply-first (reading R9; one rank, small n_G where the iteration is latency-bound): the tail applies
  // S_G to W = Z + P beta on a forked branch while W^T W, its Cholesky and T = L^{-T} run, then forms
  // P = W T and Q = (S_G W) T in one panel launch - Q = S_G P by linearity - and the head skips its apply
  const char* afe = getenv("NSP_APPLY_FIRST");
  const bool apply_first = !multi && !tr.on && w.kind == 0 &&
                           (afe ? afe[0] == '1' : n <= 65536);
  bool skip_apply = false;   // the head's Q was formed by the preceding tail
  auto head = [&](bool copy_status) -> nsp_status {
    cudaStream_t q = c->stream;
    nsp_status e2;
    tr.mark("loop");
    if (!skip_apply && (e2 = op_apply(c, w, w.P, w.Q, s)) != NSP_OK) return e2;
    tr.mark("apply");
    nspb::gram2(w.P, sp, sp, w.Q, w.R, sp, sp, ng, w.D, w.E, sp, w.gram, q, true);   // D: lower tiles (chol)
    if (multi) {   // D and E are adjacent in the workspace: one allreduce
      if ((e2 = comm_allreduce(c, w.D, (size_t)2 * sp * sp)) != NSP_OK) return e2;
    }
    tr.mark("gram_DE");
    if (fused_sxs()) {   // D = L L^T and alpha = D^{-1} E in one launch
      nspb::chol_fac_solve(w.D, sp, 0, -1, 0.0, w.Ld, w.st, w.E, sp, w.al, sp, 1.0, true, true, q);
      tr.mark("chol_D");
    } else {
      nspb::chol_fac(w.D, sp, 0, -1, 0.0, w.Ld, w.st, q);        // D = L L^T
      tr.mark("chol_D");
      nspb::chol_solve(w.Ld, sp, w.E, sp, w.al, sp, 1.0, true, true, nullptr, q);   // alpha = D^{-1} E
    }
    tr.mark("alpha");
    // R -= Q alpha here; X += P alpha is deferred to the next tail (x_update), off the critical path
    const int npt = (fuse_pg && !usem)
                        ? nspb::panel_gram(w.R, w.R, w.Q, w.al, n, -1.0, w.npart, 0, w.F, w.gram, q)   // + F = Q^T R
                        : nspb::panel(w.R, sp, w.R, sp, w.Q, sp, w.al, sp, sp, sp, n, -1.0, multi ? nullptr : w.npart, q);
    if (multi) {
      nspb::colsq(w.R, sp, ng, s, sp, w.npart, w.rsq, q);
      if ((e2 = comm_allreduce(c, w.rsq, sp)) != NSP_OK) return e2;
      nspb::converge(w.rsq, w.bnorm, s, tol, w.st, nullptr, q);
    } else {
      nspb::colsq_converge(w.npart, npt, sp, w.rsq, w.bnorm, s, tol, w.st, q);
    }
    tr.mark("XR_update");
    if (copy_status) NSP_CUDA_TRY(c, cudaMemcpyAsync(hs, w.st, sizeof(BcgStatus), cudaMemcpyDeviceToHost, q));
    NSP_CUDA_TRY(c, cudaGetLastError());
    return NSP_OK;
  };
  // X += P alpha of the previous head.  X is read by nothing inside the loop, so (single rank, no
  // tracing) the panel runs on a side stream forked from the context stream and joined only before
  // orth overwrites P: it overlaps the tail's small s x s kernels.  Inside a captured graph the
  // fork / join become graph edges.
  const char* xfe = getenv("NSP_XFORK");
  const bool xfork = !tr.on && !(xfe && xfe[0] == '0');   // (several ranks too: no collective in it)
  if (xfork) {
    if (!c->side_stream) NSP_CUDA_TRY(c, cudaStreamCreateWithFlags(&c->side_stream, cudaStreamNonBlocking));
    if (!c->ev_fork) NSP_CUDA_TRY(c, cudaEventCreateWithFlags(&c->ev_fork, cudaEventDisableTiming));
    if (!c->ev_join) NSP_CUDA_TRY(c, cudaEventCreateWithFlags(&c->ev_join, cudaEventDisableTiming));
  }
  auto x_update = [&](bool fork) -> nsp_status {
    if (!fork) {
      nspb::panel(w.X, sp, w.X, sp, w.P, sp, w.al, sp, sp, sp, n, 1.0, nullptr, c->stream);
      return NSP_OK;
    }
    NSP_CUDA_TRY(c, cudaEventRecord(c->ev_fork, c->stream));
    NSP_CUDA_TRY(c, cudaStreamWaitEvent(c->side_stream, c->ev_fork, 0));
    nspb::panel(w.X, sp, w.X, sp, w.P, sp, w.al, sp, sp, sp, n, 1.0, nullptr, c->side_stream);
    NSP_CUDA_TRY(c, cudaEventRecord(c->ev_join, c->side_stream));
    return NSP_OK;
  };
  // tail: a9-a11 (X += P alpha, Z = M R, F = Q^T Z, beta, W = Z + P beta, P = orth(W))
  auto tail = [&]() -> nsp_status {
    cudaStream_t q = c->stream;
    nsp_status e2;
    if ((e2 = x_update(xfork)) != NSP_OK) return e2;
    if (usem && (e2 = op_precond(c, w, w.R, w.Z, s)) != NSP_OK) return e2;
    if (!(fuse_pg && !usem)) {   // (fused: F = Q^T R came with the head's R update)
      nspb::gram(w.Q, sp, sp, Zr, sp, sp, ng, w.F, sp, w.gram, q);
      if ((e2 = comm_allreduce(c, w.F, (size_t)sp * sp)) != NSP_OK) return e2;
    }
    nspb::chol_solve(w.Ld, sp, w.F, sp, w.be, sp, -1.0, true, true, nullptr, q);  // beta = -D^{-1} F
    tr.mark("beta");
    if (fuse_pg) nspb::panel_gram(w.W, Zr, w.P, w.be, n, 1.0, nullptr, 1, w.G, w.gram, q);   // + G = W^T W
    else nspb::panel(w.W, sp, Zr, sp, w.P, sp, w.be, sp, sp, sp, n, 1.0, nullptr, q);
    tr.mark("W");
    if (apply_first) {
      if (!c->apply_stream) NSP_CUDA_TRY(c, cudaStreamCreateWithFlags(&c->apply_stream, cudaStreamNonBlocking));
      if (!c->ev_afork) NSP_CUDA_TRY(c, cudaEventCreateWithFlags(&c->ev_afork, cudaEventDisableTiming));
      if (!c->ev_ajoin) NSP_CUDA_TRY(c, cudaEventCreateWithFlags(&c->ev_ajoin, cudaEventDisableTiming));
      NSP_CUDA_TRY(c, cudaEventRecord(c->ev_afork, q));
      NSP_CUDA_TRY(c, cudaStreamWaitEvent(c->apply_stream, c->ev_afork, 0));
      c->stream = c->apply_stream;   // the apply's kernels go to the forked branch (a graph branch when captured)
      e2 = op_apply(c, w, w.W, w.QW, s);
      c->stream = q;
      if (e2 != NSP_OK) return e2;
      NSP_CUDA_TRY(c, cudaEventRecord(c->ev_ajoin, c->apply_stream));
      if ((e2 = orth(c, w, w.W, s, w.P, nullptr, fuse_pg, true)) != NSP_OK) return e2;   // G, chol, T (or eig)
      if (xfork) NSP_CUDA_TRY(c, cudaStreamWaitEvent(q, c->ev_join, 0));                // X += P alpha done
      NSP_CUDA_TRY(c, cudaStreamWaitEvent(q, c->ev_ajoin, 0));                           // S_G W done
      PanelArgs pp{w.P, sp, nullptr, 0, w.W, sp, w.T, sp, 1.0, nullptr, &w.st->fallback};
      PanelArgs pq{w.Q, sp, nullptr, 0, w.QW, sp, w.T, sp, 1.0, nullptr, &w.st->fallback};
      nspb::panel2(pp, &pq, sp, sp, n, q);   // P = W T and Q = (S_G W) T, one launch
      skip_apply = true;
    } else {
      if ((e2 = orth(c, w, w.W, s, w.P, xfork ? c->ev_join : nullptr, fuse_pg)) != NSP_OK) return e2;
      skip_apply = false;
    }
    tr.mark("orth");
    return NSP_OK;
  };
  // One CUDA graph for tail + head of every iteration after the first (launch-bound loop;
  // single rank, no tracing, NSP_GRAPH != 0): captured on a private stream, launched on the
  // context stream, cached in the context while the workspace / s / tol / operator are unchanged.
  const char* genv = getenv("NSP_GRAPH");
  const bool use_graph = !multi && !tr.on && !(genv && genv[0] == '0');
  cudaGraphExec_t gexec = nullptr;
  if (use_graph) {
    const GraphKey key{w.X, n, s, tol, w.kind, usem ? 1 : 0, c->opts.orth_tau, apply_first ? 1 : 0};
    if (c->bcg_graph && c->bcg_key == key) gexec = c->bcg_graph;
  }
  const bool heads_run = !hs->converged && maxit > 0;
  if (hs->converged) {
    ret = NSP_OK;
  } else {
    if (usem) {
      NSP_CUDA_TRY(c, cudaMemsetAsync(w.Z, 0, (size_t)n * sp * 8, st));
      if ((e = op_precond(c, w, w.R, w.Z, s)) != NSP_OK) return e;
    }
    if ((e = orth(c, w, Zr, s, w.P)) != NSP_OK) return e;
    // device-driven loop (default; NSP_GRAPH=1 keeps the per-iteration graph, profiling and tracing
    // use it too): iteration 0 eagerly, then ONE graph launch whose WHILE node runs tail + head +
    // k_bcg_loop_ctl until the stop test fires
    const bool use_while = use_graph && !c->prof_on && !(genv && genv[0] == '1') && maxit > 1;
    bool stop = false;
    auto run_iters = [&](int it0, int it1) -> nsp_status {
      nsp_status e;
      for (int it = it0; it < it1; ++it) {
        if (it == 0 || !use_graph) {
          if (it > 0 && (e = tail()) != NSP_OK) return e;
          if ((e = head(true)) != NSP_OK) return e;
        } else {
          if (!gexec) {
            if (!c->gstream) NSP_CUDA_TRY(c, cudaStreamCreateWithFlags(&c->gstream, cudaStreamNonBlocking));
            if (c->bcg_graph) {
              cudaGraphExecDestroy(c->bcg_graph);
              c->bcg_graph = nullptr;
            }
            cudaGraph_t g = nullptr;
            c->stream = c->gstream;
            c->capturing = true;
            c->gprof_in_graph = false;
            const long long l0 = nsp_launch_count();
            NSP_CUDA_TRY(c, cudaStreamBeginCapture(c->gstream, cudaStreamCaptureModeRelaxed));
            nsp_status ec = tail();
            if (ec == NSP_OK) ec = head(true);
            cudaError_t ce = cudaStreamEndCapture(c->gstream, &g);
            c->stream = st;
            c->capturing = false;
            c->bcg_graph_kernels = nsp_launch_count() - l0;   // captured, not executed
            nsp_count_launches(-c->bcg_graph_kernels);
            if (ec != NSP_OK) return ec;
            NSP_CUDA_TRY(c, ce);
            NSP_CUDA_TRY(c, cudaGraphInstantiate(&gexec, g, 0));
            cudaGraphDestroy(g);
            c->bcg_graph = gexec;
            c->bcg_key = GraphKey{w.X, n, s, tol, w.kind, usem ? 1 : 0, c->opts.orth_tau, apply_first ? 1 : 0};
          }
          NSP_CUDA_TRY(c, cudaGraphLaunch(gexec, st));
          nsp_count_launches(c->bcg_graph_kernels);
        }
        NSP_CUDA_TRY(c, cudaStreamSynchronize(st));
        if (it > 0 && use_graph && c->prof_on && c->gprof_in_graph) {
          float ms = 0.f;
          NSP_CUDA_TRY(c, cudaEventElapsedTime(&ms, c->gprof_ev[0], c->gprof_ev[1]));
          c->gprof_ms += ms;
          c->gprof_n += 1;
        }
        tr.mark("sync");
        iters = it + 1;
        fallbacks += hs->fallback;
        relres = hs->relres;
        if (rep && rep->hist && it + 1 < rep->hist_cap) rep->hist[it + 1] = hs->relres;
        if (rep && rep->widths && it < rep->widths_cap) rep->widths[it] = hs->width;
        if (hs->indefinite) {
          ret = NSP_ERR_INDEFINITE;
          c->err = "nsp_block_cg: chol(P^T S P) failed (S_G not SPD on the search space)";
          stop = true;
          return NSP_OK;
        }
        if (hs->nonfinite) {
          ret = NSP_ERR_NUMERICAL;
          c->err = "nsp_block_cg: non-finite residual";
          stop = true;
          return NSP_OK;
        }
        if (hs->width == 0) {
          ret = NSP_ERR_STAGNATION;
          c->err = "nsp_block_cg: all search directions deflated";
          stop = true;
          return NSP_OK;
        }
        if (hs->converged) {
          ret = NSP_OK;
          stop = true;
          return NSP_OK;
        }
      }
      return NSP_OK;
    };
    if ((e = run_iters(0, use_while ? 1 : maxit)) != NSP_OK) return e;
    if (use_while && !stop && c->bcg_no_while) {
      if ((e = run_iters(1, maxit)) != NSP_OK) return e;
    } else if (use_while && !stop) {
      if (c->bhist_cap < maxit + 1) {
        if (c->d_bhist) cudaFree(c->d_bhist);
        if (c->d_bwidth) cudaFree(c->d_bwidth);
        c->d_bhist = nullptr;
        c->d_bwidth = nullptr;
        c->bhist_cap = 0;
        NSP_CUDA_TRY(c, cudaMalloc(&c->d_bhist, (size_t)(maxit + 1) * sizeof(double)));
        NSP_CUDA_TRY(c, cudaMalloc(&c->d_bwidth, (size_t)(maxit + 1) * sizeof(int)));
        c->bhist_cap = maxit + 1;
        if (c->bcg_wgraph) {   // baked-in pointers changed
          cudaGraphExecDestroy(c->bcg_wgraph);
          c->bcg_wgraph = nullptr;
        }
      }
      const GraphKey key{w.X, n, s, tol, w.kind, usem ? 1 : 0, c->opts.orth_tau, apply_first ? 1 : 0};
      // build (or reuse) the WHILE graph; any CUDA error while building it (a node type the
      // conditional body does not support) falls back to the per-iteration graph for good
      auto build_while = [&]() -> cudaError_t {
        if (c->bcg_wgraph) {
          cudaGraphExecDestroy(c->bcg_wgraph);
          c->bcg_wgraph = nullptr;
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
        cudaGraph_t body = np.conditional.phGraph_out[0];
        if ((ce = cudaStreamBeginCaptureToGraph(c->gstream, body, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed)) !=
            cudaSuccess) {
          cudaGraphDestroy(g);
          return ce;
        }
        c->stream = c->gstream;
        c->capturing = true;
        const long long l0 = nsp_launch_count();
        nsp_status ec = tail();
        if (ec == NSP_OK) ec = head(false);
        if (ec == NSP_OK) {
          nsp_count_launch();
          k_bcg_loop_ctl<<<1, 1, 0, c->gstream>>>(w.st, c->d_bhist, c->d_bwidth, maxit, hcond);
        }
        cudaGraph_t gout = nullptr;
        const cudaError_t ce2 = cudaStreamEndCapture(c->gstream, &gout);
        c->stream = st;
        c->capturing = false;
        c->bcg_wbody_kernels = nsp_launch_count() - l0;
        nsp_count_launches(-c->bcg_wbody_kernels);
        if (ec != NSP_OK || ce2 != cudaSuccess) {
          cudaGraphDestroy(g);
          return ce2 != cudaSuccess ? ce2 : cudaErrorUnknown;
        }
        cudaGraphExec_t gx = nullptr;
        ce = cudaGraphInstantiate(&gx, g, 0);
        cudaGraphDestroy(g);
        if (ce != cudaSuccess) return ce;
        c->bcg_wgraph = gx;
        c->bcg_wkey = key;
        c->bcg_wmaxit = maxit;
        return cudaSuccess;
      };
      if (!(c->bcg_wgraph && c->bcg_wkey == key && c->bcg_wmaxit == maxit) && build_while() != cudaSuccess) {
        (void)cudaGetLastError();
        c->bcg_no_while = true;
        if (c->opts.verbose) fprintf(stderr, "[nsp] device-driven block-CG loop unavailable; per-iteration graphs\n");
        if ((e = run_iters(1, maxit)) != NSP_OK) return e;
        goto copy_out;
      }
      nsp_count_launch();
      k_bcg_loop_init<<<1, 1, 0, st>>>(w.st, 1);
      NSP_CUDA_TRY(c, cudaGraphLaunch(c->bcg_wgraph, st));
      NSP_CUDA_TRY(c, cudaMemcpyAsync(hs, w.st, sizeof(BcgStatus), cudaMemcpyDeviceToHost, st));
      NSP_CUDA_TRY(c, cudaStreamSynchronize(st));
      const int done = hs->iters;   // >= 2
      nsp_count_launches(c->bcg_wbody_kernels * (long long)(done - 1));
      if (rep && rep->hist && rep->hist_cap > 2) {
        const int m = std::min(done, rep->hist_cap - 1) - 1;   // entries 2 .. min(done, cap-1)
        if (m > 0) NSP_CUDA_TRY(c, cudaMemcpy(rep->hist + 2, c->d_bhist + 2, (size_t)m * sizeof(double),
                                              cudaMemcpyDeviceToHost));
      }
      if (rep && rep->widths && rep->widths_cap > 1) {
        const int m = std::min(done, rep->widths_cap) - 1;     // entries 1 .. min(done, cap) - 1
        if (m > 0) NSP_CUDA_TRY(c, cudaMemcpy(rep->widths + 1, c->d_bwidth + 1, (size_t)m * sizeof(int),
                                              cudaMemcpyDeviceToHost));
      }
      iters = done;
      fallbacks += hs->nfallback;
      relres = hs->relres;
      if (hs->indefinite) {
        ret = NSP_ERR_INDEFINITE;
        c->err = "nsp_block_cg: chol(P^T S P) failed (S_G not SPD on the search space)";
      } else if (hs->nonfinite) {
        ret = NSP_ERR_NUMERICAL;
        c->err = "nsp_block_cg: non-finite residual";
      } else if (hs->width == 0) {
        ret = NSP_ERR_STAGNATION;
        c->err = "nsp_block_cg: all search directions deflated";
      } else if (hs->converged) {
        ret = NSP_OK;
      }
    }
  }
copy_out:
  // the last head's X += P alpha (every earlier one ran in the following tail)
  if (heads_run) {
    if ((e = x_update(false)) != NSP_OK) return e;
  }
  // copy X out
  nspb::copy_pad(w.X, sp, Xout, ldx, n, s, 1.0, st);
  tr.mark("end");
  tr.report();
  NSP_CUDA_TRY(c, cudaStreamSynchronize(st));
  NSP_CUDA_TRY(c, cudaGetLastError());
  if (rep) {
    rep->iters = iters;
    rep->converged = ret == NSP_OK;
    rep->status = ret;
    rep->relres = relres;
    rep->fallbacks = fallbacks;
  }
  return ret;
}

// ---------------------------------------------------------------------------------------------
// A_G^{-1} X (eq:S1): rows gathered into RCM band order, band forward + backward sweeps, scattered
// back.  buf: g_nt*64 x ld_pad(s, 32) doubles.
// ---------------------------------------------------------------------------------------------
static int cheb_ld(int s) { return s == 1 ? 1 : ld_pad(s, 32); }
size_t ag_ws_doubles(const nsp_ctx* c, int s) {
  if (c->ag_cheb) return (size_t)5 * std::max<int64_t>(c->nG, 1) * cheb_ld(s) + 5 * 64;
  return (size_t)c->g_nt * 64 * ld_pad(s, 32) + 64;
}

// A_G^{-1} X by the fixed Chebyshev iteration of the setup (Saad Alg. 12.1):
// r = x0 = X, d = r / theta, then K times { t = A_G d; x += d; r -= t; d' = c1_k d + c2_k r } - one
// CSR SpMM (A_G part of AGG2) and one fused elementwise pass per step.  X may alias Y.
static nsp_status ag_cheb(nsp_ctx* c, const double* X, int ldx, double* Y, int ldy, int s, double* buf) {
  const int ld = cheb_ld(s);
  const int64_t n = c->nG;
  const size_t blk = (size_t)std::max<int64_t>(n, 1) * ld;
  double* xw = buf;
  double* r = buf + blk;
  double* d0 = buf + 2 * blk;
  double* d1 = buf + 3 * blk;
  double* t = buf + 4 * blk;
  cudaStream_t st = c->stream;
  if (n == 0) return NSP_OK;
  nspb::copy_pad(X, ldx, r, ld, n, s, 1.0, st);
  const double theta = 0.5 * (c->cheb_b + c->cheb_a);
  // one rank: the three-term (x-only) form of the same polynomial, 4 instead of 6 block passes per step
  static const bool three_off = getenv("NSP_CHEB3") && getenv("NSP_CHEB3")[0] == '0';
  const bool s1_sell = ld == 1 && c->d_sell_ptr;
  if (c->nranks == 1 && !three_off && c->cheb_K >= 1 && (s1_sell || (ld > 1 && ld % 2 == 0 && c->AGO.rows))) {
    // x_0 = 0, x_1 = d_0 = b / theta, then K - 1 steps x_{k+1} = x_k + c1_{k-1} (x_k - x_{k-1}) + c2_{k-1} (b - A x_k)
    double* xk = d0;   // x_1
    double* xo = xw;   // x_0 = 0 (overwritten by x_2)
    nspb::copy_pad(X, ldx, xk, ld, n, s, 1.0 / theta, st);
    NSP_CUDA_TRY(c, cudaMemsetAsync(xo, 0, blk * 8, st));
    for (int k = 1; k < c->cheb_K; ++k) {
      nspk::cheb3_step(c->AGO, n, xk, ld, s, xo, r, xo, c->cheb_c1[k - 1], c->cheb_c2[k - 1], st, c->d_sell_ptr,
                       c->d_sell_col, c->d_sell_val, c->d_sell_code, c->d_sell_tab);
      std::swap(xk, xo);
    }
    nspb::copy_pad(xk, ld, Y, ldy, n, s, 1.0, st);
    NSP_CUDA_TRY(c, cudaGetLastError());
    return NSP_OK;
  }
  nspb::copy_pad(X, ldx, d0, ld, n, s, 1.0 / theta, st);
  NSP_CUDA_TRY(c, cudaMemsetAsync(xw, 0, blk * 8, st));
  static const bool fused_off = getenv("NSP_CHEB_FUSED") && getenv("NSP_CHEB_FUSED")[0] == '0';
  for (int k = 0; k < c->cheb_K; ++k) {
    static const bool sell_off = getenv("NSP_CHEB_SELL") && getenv("NSP_CHEB_SELL")[0] == '0';
    if (c->nranks == 1 && !fused_off && ld == 1 && c->d_sell_ptr && !sell_off) {   // s = 1: sliced ELL
      nspk::cheb_step_sell(n, c->d_sell_ptr, c->d_sell_col, c->d_sell_val, d0, xw, r, d1, c->cheb_c1[k],
                           c->cheb_c2[k], k + 1 < c->cheb_K, st, c->d_sell_code, c->d_sell_tab);
      std::swap(d0, d1);
      continue;
    }
    if (c->nranks == 1 && !fused_off && (ld == 1 || ld % 2 == 0)) {   // product and update in one pass
      nspk::cheb_step(c->AGO.rows ? c->AGO : c->AGG2, n, d0, ld, s, xw, r, d1, c->cheb_c1[k], c->cheb_c2[k],
                      k + 1 < c->cheb_K, st);
      std::swap(d0, d1);
      continue;
    }
    nspk::spmm(c->AGG2, d0, ld, nullptr, 0, n, t, ld, s, 3, true, st);   // t = A_G d
    if (c->nranks > 1) {   // shared rows: sum the per-rank partials, add the shared x shared term
      nsp_status e = finish_shared_rows(c, d0, ld, t, ld, s, true);
      if (e != NSP_OK) return e;
    }
    nspb::cheb_update(xw, r, d0, t, d1, c->cheb_c1[k], c->cheb_c2[k], (int64_t)n * ld, k + 1 < c->cheb_K, st);
    std::swap(d0, d1);
  }
  nspb::copy_pad(xw, ld, Y, ldy, n, s, 1.0, st);
  NSP_CUDA_TRY(c, cudaGetLastError());
  return NSP_OK;
}

// Triangular solves with the A_G factor A_G = R_G^T R_G, R_G = L^T P (P: the band ordering; L the
// band Cholesky factor).  X is either in the Gamma order (x_gamma: rows gathered through P) or already
// in R_G's row space (the band order, rows 0..n_G-1); likewise Y (y_gamma: scattered back through
// P^T).  fwd: L^{-1}, bwd: L^{-T}; both: A_G^{-1} (eq:S1).  So R_G^{-T} x = fwd (x_gamma, band out),
// R_G^{-1} y = bwd (band in, y_gamma out).  buf: g_nt*64 x ld_pad(s, 32) doubles.
nsp_status ag_tri(nsp_ctx* c, const double* X, int ldx, bool x_gamma, double* Y, int ldy, bool y_gamma, int s,
                  bool fwd, bool bwd, double* buf) {
  if (!c->has_ag) {
    c->err = "A_G^{-1} needs the A_G factor: set opts.factor_gamma = 1";
    return NSP_ERR_STATE;
  }
  if (c->ag_cheb) {
    if (fwd && bwd && x_gamma && y_gamma) return ag_cheb(c, X, ldx, Y, ldy, s, buf);
    c->err = "R_G^{-1} / R_G^{-T} need the A_G band factor (opts.ag_solver 1); A_G^{-1} is a Chebyshev iteration here";
    return NSP_ERR_STATE;
  }
  const bool vec = s == 1 && c->g_wb <= 2;   // one column, narrow band: matrix-vector chain kernel
  const int ldw = vec ? 1 : ld_pad(s, 32);
  const int64_t rows = (int64_t)c->g_nt * 64;
  if (x_gamma) {
    nspk::gather_rows(X, ldx, c->d_gperm, rows, buf, ldw, s, 1.0, c->stream);
  } else {
    nspb::copy_pad(X, ldx, buf, ldw, c->nG, s, 1.0, c->stream);
    if (rows > c->nG)
      NSP_CUDA_TRY(c, cudaMemsetAsync(buf + c->nG * (int64_t)ldw, 0, (size_t)(rows - c->nG) * ldw * 8, c->stream));
  }
  if (c->g_P > 1) {   // partitioned: P chunk sweeps in parallel + spike corrections
    const int cw = vec ? 1 : 32, P = c->g_P;
    static const bool rec_off = getenv("NSP_BAND_NOREC") != nullptr;
    // the reassociated one-product-per-row chunk sweeps (k_band_rec_vec / k_band_rec)
    const bool rec = c->d_gGF && !rec_off && (vec || ldw % 32 == 0);
    if (fwd) {
      if (rec && vec) nspk::band_rec_vec(c->d_gchunks, P, c->d_gband, c->g_wb + 1, c->d_gGF, buf, true, c->stream);
      else if (rec) nspk::band_rec(c->d_gchunks, P, c->d_gband, c->g_wb + 1, c->d_gGF, buf, ldw, true, c->stream);
      else nspk::tri_fb(c->d_gchunks, P, buf, ldw, cw, true, false, c->stream, c->g_wb);
      nspk::spike_tail(c->d_gspkF, c->d_gchunk_first, P, buf, ldw, s, true, c->stream);
      nspk::spike_update(c->d_gspkF, c->d_gchunk_first, c->d_gtile_chunk, P, c->g_nt, buf, ldw, s, true, c->stream);
    }
    if (bwd) {
      if (rec && vec) nspk::band_rec_vec(c->d_gchunks, P, c->d_gXB, 1, c->d_gGB, buf, false, c->stream);
      else if (rec) nspk::band_rec(c->d_gchunks, P, c->d_gXB, 1, c->d_gGB, buf, ldw, false, c->stream);
      else nspk::tri_fb(c->d_gchunks, P, buf, ldw, cw, false, true, c->stream, c->g_wb);
      nspk::spike_tail(c->d_gspkB, c->d_gchunk_first, P, buf, ldw, s, false, c->stream);
      nspk::spike_update(c->d_gspkB, c->d_gchunk_first, c->d_gtile_chunk, P, c->g_nt, buf, ldw, s, false, c->stream);
    }
  } else {
    nspk::tri_fb(c->d_gsys, 1, buf, ldw, vec ? 1 : 32, fwd, bwd, c->stream, c->g_wb);
  }
  if (y_gamma) nspk::scatter_rows(buf, ldw, c->d_gperm, rows, Y, ldy, s, false, c->stream);
  else nspb::copy_pad(buf, ldw, Y, ldy, c->nG, s, 1.0, c->stream);
  NSP_CUDA_TRY(c, cudaGetLastError());
  return NSP_OK;
}

nsp_status ag_solve(nsp_ctx* c, const double* X, int ldx, double* Y, int ldy, int s, double* buf) {
  return ag_tri(c, X, ldx, true, Y, ldy, true, s, true, true, buf);
}

// Y = M_2 X = A_G^{-1} X + Z (Sigma (Z^T X))   (Alg. 2 step 12, eq:left_prec_mat)
// ws: ag_ws + 2 * 64*64... small buffers carved by the caller
nsp_status m2_apply(nsp_ctx* c, const double* X, int ldx, double* Y, int ldy, int s, double* buf, double* gsm,
                    double* gws) {
  nsp_status e = ag_solve(c, X, ldx, Y, ldy, s, buf);
  if (e != NSP_OK) return e;
  if (c->nys_rank > 0) {
    // G = Z^T X (nys_ld x sp), G <- diag(sigma) G, Y += Z G
    const int sp = ((s + 63) / 64) * 64;
    nspb::gram(c->d_Z, c->nys_ld, c->nys_ld, X, ldx, sp, gram_rows(c), gsm, sp, gws, c->stream);
    if (c->nranks > 1) {
      e = comm_allreduce(c, gsm, (size_t)c->nys_ld * sp);
      if (e != NSP_OK) return e;
    }
    nspb::scale_rows(gsm, sp, c->d_sigma, c->nys_rank, c->nys_ld, sp, c->stream);
    PanelArgs pa{Y, ldy, Y, ldy, c->d_Z, c->nys_ld, gsm, sp, 1.0, nullptr};
    nspb::panel2(pa, nullptr, c->nys_ld, sp, c->nG, c->stream);
  }
  NSP_CUDA_TRY(c, cudaGetLastError());
  return NSP_OK;
}

static nsp_status precond(nsp_ctx* c, const double* R, double* Z, int ld, int s, double* buf) {
  return ag_solve(c, R, ld, Z, ld, s, buf);
}

nsp_status adef_prepare(nsp_ctx* c) {
  if (c->adef_ready || c->nys_rank <= 0) return NSP_OK;
  const int kp = c->nys_ld, rk = c->nys_rank;
  const int64_t n = c->nG;
  cudaStream_t st = c->stream;
  const size_t nb = (size_t)std::max<int64_t>(n, 1) * kp;
  double *SZ = nullptr, *wvu = nullptr, *G = nullptr, *gw = nullptr;
  BcgStatus* dst = nullptr;
  auto release = [&]() {
    cudaFree(SZ);
    cudaFree(wvu);
    cudaFree(G);
    cudaFree(gw);
    cudaFree(dst);
  };
  if (cudaMalloc((void**)&SZ, nb * 8) != cudaSuccess || cudaMalloc((void**)&wvu, apply_ws_bytes(c, kp)) != cudaSuccess ||
      cudaMalloc((void**)&G, (size_t)kp * kp * 8) != cudaSuccess ||
      cudaMalloc((void**)&gw, nspb::gram_ws_doubles(n, kp, kp) * 8) != cudaSuccess ||
      cudaMalloc((void**)&dst, sizeof(BcgStatus)) != cudaSuccess) {
    release();
    c->err = "adef_prepare: out of device memory";
    return NSP_ERR_OOM;
  }
  BcgStatus* hs = (BcgStatus*)c->h_status;
  *hs = BcgStatus{};
  nsp_status e = NSP_OK;
  if (cudaMemcpyAsync(dst, hs, sizeof(BcgStatus), cudaMemcpyHostToDevice, st) != cudaSuccess) e = NSP_ERR_CUDA;
  if (e == NSP_OK) e = apply_into(c, c->d_Z, kp, SZ, kp, rk, 1, wvu);   // S_G Z
  if (e == NSP_OK) {
    nspb::gram(c->d_Z, kp, kp, SZ, kp, kp, gram_rows(c), G, kp, gw, st);
    if (c->nranks > 1) e = comm_allreduce(c, G, (size_t)kp * kp);
  }
  if (e == NSP_OK) {
    nspb::small_sym(G, rk, kp, 0.0, st);
    if (cudaMalloc((void**)&c->d_ELp, (size_t)kp * kp * 8) != cudaSuccess) e = NSP_ERR_OOM;
  }
  if (e == NSP_OK) {
    nspb::chol_fac(G, kp, 0, rk, 0.0, c->d_ELp, dst, st);
    if (cudaMemcpyAsync(hs, dst, sizeof(BcgStatus), cudaMemcpyDeviceToHost, st) != cudaSuccess ||
        cudaStreamSynchronize(st) != cudaSuccess)
      e = NSP_ERR_CUDA;
  }
  release();
  if (e != NSP_OK) return e;
  c->adef_ok = !hs->indefinite;
  c->adef_ready = true;
  c->nys_gen += 1;   // the cached PCG graphs bake in d_ELp
  return NSP_OK;
}

}  // namespace nspi

using namespace nspi;

extern "C" {

nsp_status nsp_block_cg(nsp_ctx* c, const double* B, double* X, int s, double tol, int maxit, void* ws,
                        nsp_report* rep) {
  NspNvtx nvtx_range_("nsp_block_cg");
  if (!c || !B || !X || s <= 0 || s > 128 || maxit < 0) {
    if (c) c->err = "nsp_block_cg: bad arguments (1 <= s <= 128)";
    return NSP_ERR_ARG;
  }
  char* base;
  nsp_status e = get_ws(c, ws, solver_ws_bytes(c, s), &base);
  if (e != NSP_OK) return e;
  BcgWs w;
  bcg_layout(c, s, base, &w);
  return block_cg_impl(c, B, s, X, s, s, tol, maxit, w, rep);
}

// Alg. 2 with readings C1 (border system), C5 (U~ = Q W), C6 (symmetrised C,
// eps split, descending T eigenpairs, rank = min(r, k)).
nsp_status nsp_nystrom(nsp_ctx* c, int rank, int oversample, uint64_t seed, const double* Omega, double tol_inner,
                       int maxit_inner, void* ws, nsp_report* rep) {
  NspNvtx nvtx_range_("nsp_nystrom");
  const int s = rank + oversample;
  if (!c || rank <= 0 || oversample < 0 || s > 128 || maxit_inner < 0) {
    if (c) c->err = "nsp_nystrom: bad arguments (rank > 0, rank + oversample <= 128)";
    return NSP_ERR_ARG;
  }
  if (!Omega && (c->opts.nys_form == 2 || c->opts.nys_form == 3)) {
    c->err = "nsp_nystrom: the M_3 / M_1 forms take an explicit Omega (device generation covers the Gamma-indexed forms)";
    return NSP_ERR_ARG;
  }
  if (!c->has_ag) {
    c->err = "nsp_nystrom: M_2 needs the A_G factor (opts.factor_gamma = 1)";
    return NSP_ERR_STATE;
  }
  const int sp = sp_of(s);
  const int64_t n = c->nG;
  cudaStream_t st = c->stream;
  const size_t blk = (size_t)std::max<int64_t>(n, 1) * sp, sm = (size_t)sp * sp;
  // form 0: border system (reading C1); 1: paper-literal S_I system (eq:SI); 2: M_3 - Nystrom of S_I^{-1}
  // itself (eq:internal_term_lr_approximation_2 / eq:left_prec_mat2), Omega then n x s in original order
  const int form = (c->opts.nys_form >= 1 && c->opts.nys_form <= 3) ? c->opts.nys_form : 0;
  if (form == 3 && c->nranks != 1) {
    c->err = "nsp_nystrom: the M_1 form (nys_form 3) is single-rank";
    return NSP_ERR_STATE;
  }
  // NSP_NYS_TRACE=1: host wall time per phase (stream synchronised; diagnostics only)
  static const bool ntr = getenv("NSP_NYS_TRACE") && getenv("NSP_NYS_TRACE")[0] == '1';
  auto nyt0 = std::chrono::steady_clock::now();
  auto nymark = [&](const char* lab) {
    if (!ntr) return;
    cudaStreamSynchronize(c->stream);
    const auto t1 = std::chrono::steady_clock::now();
    fprintf(stderr, "[nsp nys] %-10s %8.3f ms\n", lab, std::chrono::duration<double, std::milli>(t1 - nyt0).count());
    nyt0 = t1;
  };
  // several ranks (form 0): every Gram is summed over the private rows of every rank plus the shared rows
  // once (gram_rows) and allreduced; the s x s steps are then replicated bit-identically; A_G X completes
  // its shared rows with one allreduce; A_G^{-1} is the sharded Chebyshev operator
  const bool multi = c->nranks > 1;
  if ((form == 1 || form == 2) && (c->nranks != 1 || c->AII.rows == 0)) {
    c->err = "nsp_nystrom: the S_I forms need opts.nys_form set at nsp_setup (single rank)";
    return NSP_ERR_STATE;
  }
  const int64_t n_int = c->i1_rows + c->wvu_rows;
  const bool si = form == 1 || form == 2;   // inner system on the interior layout (S_I)
  const size_t iblk = si ? (size_t)std::max<int64_t>(n_int, 1) * sp : 0;
  const size_t bcg_bytes = bcg_layout(c, s, nullptr, nullptr, si ? 1 : 0);
  const size_t extra =
      (6 * blk + (form == 2 ? 4 : 2) * iblk + 16 * sm + 8 * sp + (size_t)(sp + 1) * (sp + 1)) * 8 + 64 * 256;
  char* base;
  nsp_status e = get_ws(c, ws, bcg_bytes + extra, &base);
  if (e != NSP_OK) return e;
  BcgWs w;
  bcg_layout(c, s, base, &w, si ? 1 : 0);
  Carver cv(base + bcg_bytes);
  double* Om = cv.take(blk);
  double* Bn = cv.take(blk);
  double* Xn = cv.take(blk);
  double* Y = cv.take(blk);
  double* Qa = cv.take(blk);
  double* Qb = cv.take(blk);
  double* G = cv.take(sm);
  double* Rk = cv.take(sm);
  double* Tk = cv.take(sm);
  double* Racc = cv.take(sm);
  double* Rtmp = cv.take(sm);
  double* C = cv.take(sm);
  double* VC = cv.take(sm);
  double* Vsc = cv.take(sm);
  double* M1 = cv.take(sm);
  double* Tm = cv.take(sm);
  double* VT = cv.take(sm);
  double* Wc = cv.take(sm);
  double* Vw = cv.take((size_t)(sp + 1) * (sp + 1));
  double* lamC = cv.take(sp);
  double* lamT = cv.take(sp);
  double* Fi = si ? cv.take(iblk) : nullptr;   // S_I forms: right-hand side / solution (interior layout)
  double* Xi = si ? cv.take(iblk) : nullptr;
  double* Qa2 = form == 2 ? cv.take(iblk) : nullptr;   // M_3: Cholesky-QR of the n_int-row Y
  double* Qb2 = form == 2 ? cv.take(iblk) : nullptr;
  BcgStatus* hs = (BcgStatus*)c->h_status;
  // Cholesky-QR2 of Yin -> Q (returned, one of Qa / Qb), R in Racc (shifted Cholesky-QR3 when the
  // first Gram is numerically singular)
  auto cholqr = [&](const double* Yin, const double** Qres, int64_t nr = -1, double* QA = nullptr,
                    double* QB = nullptr) -> nsp_status {
    if (nr < 0) nr = n;
    if (!QA) {
      QA = Qa;
      QB = Qb;
    }
    NSP_CUDA_TRY(c, cudaMemsetAsync(Racc, 0, sm * 8, st));
    const double* Qin = Yin;
    double* Qout = QA;
    int passes = 2;
    const int64_t ngr = (multi && nr == n) ? gram_rows(c) : nr;
    for (int pass = 0; pass < passes; ++pass) {
      nspb::gram(Qin, sp, sp, Qin, sp, sp, ngr, G, sp, w.gram, st);
      if (multi) {
        nsp_status ea = comm_allreduce(c, G, sm);
        if (ea != NSP_OK) return ea;
      }
      nspb::small_chol(G, sp, 2, s, 0.0, Rk, w.st, st);
      if (pass == 0) {
        nsp_status e2 = read_status(c, w.st, hs);
        if (e2 != NSP_OK) return e2;
        if (hs->fallback) {  // shift = 11 (n s + s(s+1)) u ||Y||_F^2 (shifted CholeskyQR)
          std::vector<double> gd(sm);
          NSP_CUDA_TRY(c, cudaMemcpy(gd.data(), G, sm * 8, cudaMemcpyDeviceToHost));
          double tr = 0.0;
          for (int i = 0; i < s; ++i) tr += gd[(size_t)i * sp + i];
          const double shift = 11.0 * ((double)nr * s + (double)s * (s + 1)) * 1.1102230246251565e-16 * tr;
          nspb::small_sym(G, s, sp, shift, st);
          nspb::small_chol(G, sp, 2, s, 0.0, Rk, w.st, st);
          passes = 3;
        }
      }
      nspb::small_chol(G, sp, 1, s, 0.0, Tk, w.st, st);      // T = R^{-1}
      PanelArgs pa{Qout, sp, nullptr, 0, Qin, sp, Tk, sp, 1.0, nullptr};
      nspb::panel2(pa, nullptr, sp, sp, nr, st);
      if (pass == 0) {
        NSP_CUDA_TRY(c, cudaMemcpyAsync(Racc, Rk, sm * 8, cudaMemcpyDeviceToDevice, st));
      } else {
        nspb::small_gemm(s, s, s, 1.0, Rk, sp, false, Racc, sp, false, 0.0, Rtmp, sp, st);
        NSP_CUDA_TRY(c, cudaMemcpyAsync(Racc, Rtmp, sm * 8, cudaMemcpyDeviceToDevice, st));
      }
      Qin = Qout;
      Qout = (Qout == QA) ? QB : QA;
    }
    nsp_status e2 = read_status(c, w.st, hs);
    if (e2 != NSP_OK) return e2;
    if (hs->fallback) {
      c->err = "nsp_nystrom: Cholesky-QR failed";
      return NSP_ERR_NUMERICAL;
    }
    *Qres = Qin;
    return NSP_OK;
  };
  // G = Omega; q power steps G <- orth(B_H G) (eq:power PAPER.md:204-212), then Alg. 2 steps 1-4 on G
  if (Omega) {
    nspb::copy_pad(Omega, s, Om, sp, n, s, 1.0, st);
  } else {   // Omega generated on the device: Philox stream 0 at the rows' global Gamma indices (reading C7)
    int64_t* dg = nullptr;
    NSP_CUDA_TRY(c, cudaMallocAsync((void**)&dg, (size_t)std::max<int64_t>(n, 1) * 8, st));
    NSP_CUDA_TRY(c, cudaMemcpyAsync(dg, c->gamma_gidx.data(), (size_t)n * 8, cudaMemcpyHostToDevice, st));
    nspk::philox_gaussian(Om, n, s, sp, dg, seed, 0u, st);
    NSP_CUDA_TRY(c, cudaFreeAsync(dg, st));
  }
  const int q = c->opts.nys_power > 0 ? c->opts.nys_power : 0;
  nsp_report brep{};
  int total_iters = 0;
  nsp_status sb = NSP_OK;
  if (form == 2) {   // M_3: Y = S_I^{-1} Omega_I (block PCG on S_I, A_I preconditioner), no power steps
    nspk::gather_rows(Omega, s, c->d_int_src, n_int, Fi, sp, s, 1.0, st);
    brep = nsp_report{};
    if (rep) {
      brep.hist = rep->hist;
      brep.hist_cap = rep->hist_cap;
      brep.widths = rep->widths;
      brep.widths_cap = rep->widths_cap;
    }
    nsp_status sbi = block_cg_impl(c, Fi, sp, Xi, sp, s, tol_inner, maxit_inner, w, &brep);
    if (sbi < 0) return sbi;
    if (sbi == NSP_NOT_CONVERGED) sb = NSP_NOT_CONVERGED;
    total_iters += brep.iters;
  }
  for (int pw = 0; form != 2 && pw <= q; ++pw) {
    if (form == 1) {   // paper-literal: F = A_IG G, S_I X = F (block PCG, A_I), Y = A_GI X
      NSP_CUDA_TRY(c, cudaMemsetAsync(Fi, 0, (size_t)c->i1_rows * sp * 8, st));
      nspk::spmm(c->A2G, Om, sp, nullptr, 0, 0, Fi + c->i1_rows * (int64_t)sp, sp, s, 0, true, st);
      brep = nsp_report{};
      if (rep && pw == q) {
        brep.hist = rep->hist;
        brep.hist_cap = rep->hist_cap;
        brep.widths = rep->widths;
        brep.widths_cap = rep->widths_cap;
      }
      nsp_status sbi = block_cg_impl(c, Fi, sp, Xi, sp, s, tol_inner, maxit_inner, w, &brep);
      if (sbi < 0) return sbi;
      if (sbi == NSP_NOT_CONVERGED) sb = NSP_NOT_CONVERGED;
      total_iters += brep.iters;
      nspk::spmm(c->AGG2, nullptr, 0, Xi + c->i1_rows * (int64_t)sp, sp, n, Y, sp, s, 2, true, st);
      if (pw < q) {
        const double* Qp = nullptr;
        if ((e = cholqr(Y, &Qp)) != NSP_OK) return e;
        NSP_CUDA_TRY(c, cudaMemcpyAsync(Om, Qp, blk * 8, cudaMemcpyDeviceToDevice, st));
      }
      continue;
    }
    nymark("start");
    // steps 1-2: B = K_G G  (reading C1); M_1 (form 3): the operator is R_G^{-T} B_H R_G^{-1}, so the
    // sketch enters as R_G^{-1} G (eq:lr_approximation_S-1_A-I)
    const double* Gin = Om;
    if (form == 3) {
      NSP_CUDA_TRY(c, cudaMemsetAsync(Qa, 0, blk * 8, st));   // padding columns stay zero
      if ((e = ag_tri(c, Om, sp, false, Qa, sp, true, s, false, true, w.wvu)) != NSP_OK) return e;
      Gin = Qa;
    }
    if ((e = apply_into(c, Gin, sp, Bn, sp, s, 2, w.wvu)) != NSP_OK) return e;
    nymark("K_G Omega");
    // step 3: S_G X = B by breakdown-free block CG to tol_inner
    brep = nsp_report{};
    if (rep && pw == q) {
      brep.hist = rep->hist;
      brep.hist_cap = rep->hist_cap;
      brep.widths = rep->widths;
      brep.widths_cap = rep->widths_cap;
    }
    nsp_status sbi = block_cg_impl(c, Bn, sp, Xn, sp, s, tol_inner, maxit_inner, w, &brep);
    if (sbi < 0) return sbi;
    if (sbi == NSP_NOT_CONVERGED) sb = NSP_NOT_CONVERGED;
    total_iters += brep.iters;
    nymark("block CG");
    // step 4: Y = A_G X  (M_1: Y = R_G^{-T} A_G X, in R_G's row space)
    nspk::spmm(c->AGG2, Xn, sp, nullptr, 0, n, Y, sp, s, 3, true, st);
    if (multi && (e = finish_shared_rows(c, Xn, sp, Y, sp, s, true)) != NSP_OK) return e;
    if (form == 3 && (e = ag_tri(c, Y, sp, true, Y, sp, false, s, true, false, w.wvu)) != NSP_OK) return e;
    if (pw < q) {   // power step: G <- orthonormal basis of Y
      const double* Qp = nullptr;
      if ((e = cholqr(Y, &Qp)) != NSP_OK) return e;
      NSP_CUDA_TRY(c, cudaMemcpyAsync(Om, Qp, blk * 8, cudaMemcpyDeviceToDevice, st));
    }
  }
  brep.iters = total_iters;
  // the Nystrom operands: G (sketch) and Y = B G with nY rows (M_3: the interior layout)
  const int64_t nY = form == 2 ? n_int : n;
  const double* Gs = form == 2 ? Fi : Om;
  const double* Ys = form == 2 ? Xi : Y;
  nymark("A_G X");
  // step 5: Y = Q R
  const double* Q = nullptr;
  if ((e = (form == 2 ? cholqr(Ys, &Q, nY, Qa2, Qb2) : cholqr(Ys, &Q))) != NSP_OK) return e;
  nymark("CholQR2");
  // step 6: C = Omega^T Y, symmetrised (reading C6)
  nspb::gram(Gs, sp, sp, Ys, sp, sp, multi ? gram_rows(c) : nY, C, sp, w.gram, st);
  if (multi && (e = comm_allreduce(c, C, sm)) != NSP_OK) return e;
  nspb::small_sym(C, s, sp, 0.0, st);
  if (const char* dump = getenv("NSP_DUMP_C")) {   // diagnostics: C (s x s, ld sp) as raw fp64
    std::vector<double> hc((size_t)sp * sp);
    cudaMemcpy(hc.data(), C, hc.size() * 8, cudaMemcpyDeviceToHost);
    if (FILE* f = fopen(dump, "wb")) {
      fwrite(hc.data(), 8, hc.size(), f);
      fclose(f);
    }
  }
  // step 7: EVD of C, split at eps = nys_eps_rel * lambda_max
  nspb::small_eig(C, sp, s, Vw, sp + 1, lamC, VC, nullptr, st);
  std::vector<double> hl(s);
  NSP_CUDA_TRY(c, cudaMemcpyAsync(hl.data(), lamC, s * 8, cudaMemcpyDeviceToHost, st));
  NSP_CUDA_TRY(c, cudaStreamSynchronize(st));
  int r = 0;
  if (hl[0] > 0.0)
    for (int i = 0; i < s; ++i)
      if (hl[i] >= c->opts.nys_eps_rel * hl[0]) ++r;
  const int rk = std::min(r, rank);
  // release any previous approximation
  if (c->d_Z) cudaFree(c->d_Z);
  if (c->d_sigma) cudaFree(c->d_sigma);
  c->d_Z = nullptr;
  c->d_sigma = nullptr;
  c->nys_rank = 0;
  c->nys_gen += 1;   // invalidates the cached PCG graph
  c->h_sigma.clear();
  nsp_status ret = sb == NSP_NOT_CONVERGED ? NSP_NOT_CONVERGED : NSP_OK;
  if (rk > 0) {
    nymark("C + EVD");
    // step 8: T = R V1 D1^{-1} V1^T R^T = M1 M1^T with M1 = R V1 D1^{-1/2}
    NSP_CUDA_TRY(c, cudaMemsetAsync(Vsc, 0, sm * 8, st));
    nspb::scale_cols(VC, s, lamC, r, s, sp, Vsc, sp, 1, st);
    nspb::small_gemm(s, r, s, 1.0, Racc, sp, false, Vsc, sp, false, 0.0, M1, sp, st);
    NSP_CUDA_TRY(c, cudaMemsetAsync(Tm, 0, sm * 8, st));
    nspb::small_gemm(s, s, r, 1.0, M1, sp, false, M1, sp, true, 0.0, Tm, sp, st);
    nspb::small_sym(Tm, s, sp, 0.0, st);
    // step 9: EVD of T, descending
    nspb::small_eig(Tm, sp, s, Vw, sp + 1, lamT, VT, nullptr, st);
    // step 10: U~ = Q W(:, 1:k)  (reading C5)
    const int kp = ((rk + 63) / 64) * 64;
    double* U = form == 2 ? Fi : Bn;  // reuse (nY x kp, kp <= sp; the sketch is no longer needed)
    NSP_CUDA_TRY(c, cudaMemsetAsync(Wc, 0, sm * 8, st));
    nspb::scale_cols(VT, s, lamT, rk, s, kp, Wc, kp, 3, st);
    PanelArgs pu{U, kp, nullptr, 0, Q, sp, Wc, kp, 1.0, nullptr};
    nspb::panel2(pu, nullptr, sp, kp, nY, st);
    nymark("T, EVD, U");
    // step 11: Z = A_G^{-1} U~  (M_3: Z^ = A_G^{-1} A_GI V^, eq:left_prec_mat2)
    NSP_CUDA_TRY(c, cudaMalloc((void**)&c->d_Z, (size_t)std::max<int64_t>(n, 1) * kp * 8));
    NSP_CUDA_TRY(c, cudaMemsetAsync(c->d_Z, 0, (size_t)std::max<int64_t>(n, 1) * kp * 8, st));
    if (form == 2) {
      nspk::spmm(c->AGG2, nullptr, 0, U + c->i1_rows * (int64_t)kp, kp, n, Bn, kp, rk, 2, true, st);
      if ((e = ag_solve(c, Bn, kp, c->d_Z, kp, rk, w.wvu)) != NSP_OK) return e;
    } else if (form == 3) {   // M_1: Z = R_G^{-1} U (eq:prec1S)
      if ((e = ag_tri(c, U, kp, false, c->d_Z, kp, true, rk, false, true, w.wvu)) != NSP_OK) return e;
    } else if ((e = ag_solve(c, U, kp, c->d_Z, kp, rk, w.wvu)) != NSP_OK) {
      return e;
    }
    NSP_CUDA_TRY(c, cudaMalloc((void**)&c->d_sigma, kp * 8));
    NSP_CUDA_TRY(c, cudaMemsetAsync(c->d_sigma, 0, kp * 8, st));
    NSP_CUDA_TRY(c, cudaMemcpyAsync(c->d_sigma, lamT, rk * 8, cudaMemcpyDeviceToDevice, st));
    c->h_sigma.resize(rk);
    NSP_CUDA_TRY(c, cudaMemcpyAsync(c->h_sigma.data(), lamT, rk * 8, cudaMemcpyDeviceToHost, st));
    NSP_CUDA_TRY(c, cudaStreamSynchronize(st));
    c->nys_rank = rk;
    c->nys_ld = kp;
    nymark("Z = A_G^-1 U");
    // M_A-DEF2 (reading R5): E = Z^T S_G Z is formed lazily, on the first nsp_pcg(precond = 3) (adef_prepare):
    // one S_G block apply on Z that the M_2 / M_1 / M_3 paths never need
    if (c->d_ELp) cudaFree(c->d_ELp);
    c->d_ELp = nullptr;
    c->adef_ok = false;
    c->adef_ready = false;
  } else {
    ret = NSP_ERR_RANK_COLLAPSE;
    c->err = "nsp_nystrom: no eigenvalue of C >= eps (M_2 degenerates to A_G^{-1})";
  }
  nymark("E = Z^T S Z");
  NSP_CUDA_TRY(c, cudaGetLastError());
  if (rep) {
    rep->iters = brep.iters;
    rep->converged = brep.converged;
    rep->relres = brep.relres;
    rep->fallbacks = brep.fallbacks;
    rep->rank = c->nys_rank;
    rep->status = ret;
  }
  return ret;
}

nsp_status nsp_nystrom_sigma(const nsp_ctx* c, double* sigma, int* rank_out) {
  if (!c || !rank_out) return NSP_ERR_ARG;
  if (c->nys_rank < 0) return NSP_ERR_STATE;
  *rank_out = c->nys_rank;
  if (sigma)
    for (int i = 0; i < c->nys_rank; ++i) sigma[i] = c->h_sigma[i];
  return NSP_OK;
}

nsp_status nsp_precond_apply(nsp_ctx* c, int which, const double* X, double* Y, int s, void* ws) {
  NspNvtx nvtx_range_("nsp_precond_apply");
  if (!c || !X || !Y || s <= 0 || s > 128 || which < 0 || which > 4) return NSP_ERR_ARG;
  if (which == 0) {
    NSP_CUDA_TRY(c, cudaMemcpyAsync(Y, X, (size_t)c->nG * s * 8, cudaMemcpyDeviceToDevice, c->stream));
    return NSP_OK;
  }
  if (which == 2 && c->nys_rank < 0) {
    c->err = "nsp_precond_apply: M_2 requested before nsp_nystrom";
    return NSP_ERR_STATE;
  }
  const int sp = sp_of(s);
  const size_t blk = (size_t)std::max<int64_t>(c->nG, 1) * sp;
  const size_t need = (ag_ws_doubles(c, s) + (size_t)128 * sp + nspb::gram_ws_doubles(c->nG, 128, sp) + 2 * blk +
                       2048) * 8;
  char* base;
  nsp_status e = get_ws(c, ws, need, &base);
  if (e != NSP_OK) return e;
  Carver cv(base);
  double* buf = cv.take(ag_ws_doubles(c, s));
  double* gsm = cv.take((size_t)128 * sp);
  double* gws = cv.take(nspb::gram_ws_doubles(c->nG, 128, sp));
  double* Xp = cv.take(blk);
  double* Yp = cv.take(blk);
  if (which == 1) return ag_solve(c, X, s, Y, s, s, buf);
  if (which == 3) return ag_tri(c, X, s, true, Y, s, false, s, true, false, buf);   // R_G^{-T}: Gamma -> R_G rows
  if (which == 4) return ag_tri(c, X, s, false, Y, s, true, s, false, true, buf);   // R_G^{-1}: R_G rows -> Gamma
  nspb::copy_pad(X, s, Xp, sp, c->nG, s, 1.0, c->stream);
  NSP_CUDA_TRY(c, cudaMemsetAsync(Yp, 0, blk * 8, c->stream));
  if ((e = m2_apply(c, Xp, sp, Yp, sp, s, buf, gsm, gws)) != NSP_OK) return e;
  nspb::copy_pad(Yp, sp, Y, s, c->nG, s, 1.0, c->stream);
  NSP_CUDA_TRY(c, cudaGetLastError());
  return NSP_OK;
}

}
