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

struct BcgWs {
  int sp;
  double *X, *R, *P, *Q, *W, *Z;
  double *D, *E, *F, *G, *Ld, *Ldi, *T, *al, *be, *tmp, *Vw, *Vs, *lam, *bnorm, *rsq, *gram, *npart, *wvu;
  BcgStatus* st;
};

static int sp_of(int s) { return ((s + 63) / 64) * 64; }

static size_t bcg_layout(const nsp_ctx* c, int s, char* base, BcgWs* w) {
  const int sp = sp_of(s);
  const int64_t n = c->nG;
  Carver cv(base ? base : (char*)nullptr);
  BcgWs t{};
  t.sp = sp;
  const size_t blk = (size_t)std::max<int64_t>(n, 1) * sp;
  t.X = cv.take(blk);
  t.R = cv.take(blk);
  t.P = cv.take(blk);
  t.Q = cv.take(blk);
  t.W = cv.take(blk);
  t.Z = (c->opts.bcg_precond ? cv.take(blk) : nullptr);
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
  t.wvu = cv.take(apply_ws_bytes(c, sp) / 8 + 1);
  t.st = (BcgStatus*)cv.take(sizeof(BcgStatus) / 8 + 1);
  if (w) *w = t;
  return cv.off + 256;
}

size_t solver_ws_bytes(const nsp_ctx* c, int s) { return bcg_layout(c, s, nullptr, nullptr); }

void solver_free(nsp_ctx*) {}

static nsp_status read_status(nsp_ctx* c, BcgStatus* d, BcgStatus* h) {
  NSP_CUDA_TRY(c, cudaMemcpyAsync(h, d, sizeof(BcgStatus), cudaMemcpyDeviceToHost, c->stream));
  NSP_CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  return NSP_OK;
}

// orth(Wm): Gram, Cholesky-QR with pivot test, eigen fallback; P = Wm T (reading C3)
static void orth(nsp_ctx* c, BcgWs& w, const double* Wm, int s, double* Pout) {
  const int sp = w.sp;
  const int64_t n = c->nG;
  cudaStream_t st = c->stream;
  nspb::gram(Wm, sp, sp, Wm, sp, sp, n, w.G, sp, w.gram, st);
  nspb::small_chol(w.G, sp, 1, s, c->opts.orth_tau, w.T, w.st, st);
  nspb::small_eig(w.G, sp, s, w.Vw, sp + 1, w.lam, w.Vs, &w.st->fallback, st);
  nspb::orth_from_eig(w.lam, w.Vs, s, sp, c->opts.orth_tau, w.T, w.st, st);
  nspb::panel(Pout, sp, nullptr, 0, Wm, sp, w.T, sp, sp, sp, n, 1.0, nullptr, st);
}

// Z = M R
static nsp_status precond(nsp_ctx* c, const double* R, double* Z, int ld, int s, double* wvu);

nsp_status block_cg_impl(nsp_ctx* c, const double* B, int ldb, double* Xout, int ldx, int s, double tol, int maxit,
                         BcgWs& w, nsp_report* rep) {
  const int sp = w.sp;
  const int64_t n = c->nG;
  cudaStream_t st = c->stream;
  BcgStatus* hs = (BcgStatus*)c->h_status;
  const bool usem = c->opts.bcg_precond != 0;
  int iters = 0, fallbacks = 0;
  nsp_status ret = NSP_NOT_CONVERGED;
  Tracer tr;
  tr.init(st);
  tr.mark("start");
  // init: X = 0, R = B, bnorm
  NSP_CUDA_TRY(c, cudaMemsetAsync(w.X, 0, (size_t)n * sp * 8, st));
  nspb::copy_pad(B, ldb, w.R, sp, n, s, 1.0, st);
  nspb::colsq(w.R, sp, n, s, sp, w.npart, w.rsq, st);
  nspb::sqrt_vec(w.rsq, w.bnorm, sp, st);
  BcgStatus init{};
  init.width = s;
  std::memcpy(hs, &init, sizeof(init));
  NSP_CUDA_TRY(c, cudaMemcpyAsync(w.st, hs, sizeof(BcgStatus), cudaMemcpyHostToDevice, st));
  nspb::converge(w.rsq, w.bnorm, s, tol, w.st, nullptr, st);
  nsp_status e = read_status(c, w.st, hs);
  if (e != NSP_OK) return e;
  if (rep && rep->hist && rep->hist_cap > 0) rep->hist[0] = hs->relres;
  double relres = hs->relres;
  if (hs->converged) {
    ret = NSP_OK;
  } else {
    double* Zr = w.R;
    if (usem) {
      if ((e = precond(c, w.R, w.Z, sp, s, w.wvu)) != NSP_OK) return e;
      Zr = w.Z;
    }
    orth(c, w, Zr, s, w.P);
    for (int it = 0; it < maxit; ++it) {
      // a1-a5: Q = S_G P
      tr.mark("loop");
      if ((e = apply_into(c, w.P, sp, w.Q, sp, s, 1, w.wvu)) != NSP_OK) return e;
      tr.mark("apply");
      // a6: D = P^T Q, E = P^T R
      nspb::gram2(w.P, sp, sp, w.Q, w.R, sp, sp, n, w.D, w.E, sp, w.gram, st);
      tr.mark("gram_DE");
      // a7: chol(D), alpha = D^{-1} E
      nspb::small_chol(w.D, sp, 0, -1, 0.0, w.Ldi, w.st, st);   // Ldi = D^{-1}
      tr.mark("chol_D");
      nspb::panel(w.al, sp, nullptr, 0, w.Ldi, sp, w.E, sp, sp, sp, sp, 1.0, nullptr, st);
      tr.mark("alpha");
      // a8: X += P alpha, R -= Q alpha, column norms
      {
        PanelArgs px{w.X, sp, w.X, sp, w.P, sp, w.al, sp, 1.0, nullptr};
        PanelArgs pr{w.R, sp, w.R, sp, w.Q, sp, w.al, sp, -1.0, w.npart};
        nspb::panel2(px, &pr, sp, sp, n, st);
      }
      nspb::colsq_reduce(w.npart, (int)((n + 63) / 64), sp, w.rsq, st);
      double* hslot = nullptr;
      nspb::converge(w.rsq, w.bnorm, s, tol, w.st, hslot, st);
      tr.mark("XR_update");
      NSP_CUDA_TRY(c, cudaGetLastError());
      if ((e = read_status(c, w.st, hs)) != NSP_OK) return e;
      tr.mark("sync");
      iters = it + 1;
      fallbacks += hs->fallback;
      relres = hs->relres;
      if (rep && rep->hist && it + 1 < rep->hist_cap) rep->hist[it + 1] = hs->relres;
      if (rep && rep->widths && it < rep->widths_cap) rep->widths[it] = hs->width;
      if (hs->indefinite) {
        ret = NSP_ERR_INDEFINITE;
        c->err = "nsp_block_cg: chol(P^T S P) failed (S_G not SPD on the search space)";
        break;
      }
      if (hs->nonfinite) {
        ret = NSP_ERR_NUMERICAL;
        c->err = "nsp_block_cg: non-finite residual";
        break;
      }
      if (hs->width == 0) {
        ret = NSP_ERR_STAGNATION;
        c->err = "nsp_block_cg: all search directions deflated";
        break;
      }
      if (hs->converged) {
        ret = NSP_OK;
        break;
      }
      // a9: Z = M R
      Zr = w.R;
      if (usem) {
        if ((e = precond(c, w.R, w.Z, sp, s, w.wvu)) != NSP_OK) return e;
        Zr = w.Z;
      }
      // a10: F = Q^T Z, beta = -D^{-1} F, W = Z + P beta
      nspb::gram(w.Q, sp, sp, Zr, sp, sp, n, w.F, sp, w.gram, st);
      nspb::panel(w.be, sp, nullptr, 0, w.Ldi, sp, w.F, sp, sp, sp, sp, -1.0, nullptr, st);
      tr.mark("beta");
      nspb::panel(w.W, sp, Zr, sp, w.P, sp, w.be, sp, sp, sp, n, 1.0, nullptr, st);
      tr.mark("W");
      // a11: P = orth(W)
      orth(c, w, w.W, s, w.P);
      tr.mark("orth");
    }
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

static nsp_status precond(nsp_ctx* c, const double* R, double* Z, int ld, int s, double* wvu) {
  (void)R;
  (void)Z;
  (void)ld;
  (void)s;
  (void)wvu;
  c->err = "block-CG preconditioner A_G^{-1} requires the A_G factor (not built)";
  return NSP_ERR_STATE;
}

}  // namespace nspi

using namespace nspi;

extern "C" {

nsp_status nsp_block_cg(nsp_ctx* c, const double* B, double* X, int s, double tol, int maxit, void* ws,
                        nsp_report* rep) {
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

nsp_status nsp_nystrom(nsp_ctx* c, int, int, const double*, double, int, void*, nsp_report*) {
  if (c) c->err = "nsp_nystrom: not built";
  return NSP_ERR_STATE;
}
nsp_status nsp_nystrom_sigma(const nsp_ctx*, double*, int*) { return NSP_ERR_STATE; }
nsp_status nsp_precond_apply(nsp_ctx*, int, const double*, double*, int, void*) { return NSP_ERR_STATE; }
nsp_status nsp_pcg(nsp_ctx*, const double*, double*, double, int, int, void*, nsp_report*) { return NSP_ERR_STATE; }
}
