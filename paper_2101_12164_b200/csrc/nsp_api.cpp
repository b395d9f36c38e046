// Context queries, workspace management and the S_G / K_G block applies (§8(a) rows a0-a5).
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "nsp_comm.h"
#include "nsp_internal.h"
#include "nsp_solver.h"
#include "nsp_blas.h"

namespace nspi {

static int device_sms(int dev) {   // SM count per device (cached)
  static int cache[64] = {0};
  if (dev < 0 || dev >= 64) dev = 0;
  if (!cache[dev]) {
    int n = 0;
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    cache[dev] = n > 0 ? n : 148;
  }
  return cache[dev];
}

int pick_cw(const nsp_ctx* c, int s) {
  const int tiles64 = (s + 63) / 64;
  if (const char* e = getenv("NSP_CW")) return atoi(e) == 64 && s > 32 ? 64 : 32;   // tuning override
  if (c->d_minv) return 32;   // k_symm: 32-wide chunks run 2 CTAs/SM (faster at every measured shape)
  return (s > 32 && (int64_t)c->nsub * tiles64 >= 2 * device_sms(c->device)) ? 64 : 32;
}

int ld_pad(int s, int cw) { return ((s + cw - 1) / cw) * cw; }

size_t apply_ws_bytes_base(const nsp_ctx* c, int s);

// a2+a3 on the INT8 tensor cores for this width (reading R10): apply_kernel 0 from s >= 48 (NSP_OZ_MIN_S),
// apply_kernel 3 for every s > 1
bool use_ozaki(const nsp_ctx* c, int s) {
  if (!c->d_oz_msl || s <= 1) return false;
  if (c->opts.apply_kernel == 3) return true;
  static const int min_s = getenv("NSP_OZ_MIN_S") ? atoi(getenv("NSP_OZ_MIN_S")) : 48;
  return c->opts.apply_kernel == 0 && s >= min_s;
}

// byte offset of the INT8 W^T slices / column exponents inside the apply workspace
static size_t oz_ws_offset(const nsp_ctx* c, int s) {
  const int cw = pick_cw(c, s);
  size_t b = c->d_minv ? (size_t)c->wvu_rows * (ld_pad(s, cw) / 32) * 36 * 8 * 2 + 512
                       : (size_t)c->wvu_rows * ld_pad(s, cw) * 8 + 512;
  if (c->d_minv) b += (size_t)c->wvu_rows * c->max_ntb * 8 + 256;
  return (b + 1023) & ~(size_t)1023;
}

size_t apply_ws_bytes(const nsp_ctx* c, int s) {
  if (use_ozaki(c, s)) {
    const int nct = (s + 127) / 128;
    return oz_ws_offset(c, s) + nspk::oz_wslice_bytes(c->wvu_rows, s) + (size_t)c->nsub * nct * 128 * 4 + 1024;
  }
  return apply_ws_bytes_base(c, s);
}

size_t apply_ws_bytes_base(const nsp_ctx* c, int s) {
  const int cw = pick_cw(c, s);
  // W and U; with the S_j^{-1} tiles the chunk-major padded layout (36 doubles per row per 32-col chunk)
  size_t b = c->d_minv ? (size_t)c->wvu_rows * (ld_pad(s, cw) / 32) * 36 * 8 * 2 + 512
                       : (size_t)c->wvu_rows * ld_pad(s, cw) * 8 + 512;
  // k_symv1 partial slots (s = 1; reserved for every s: callers size one workspace for several widths)
  if (c->d_minv) b += (size_t)c->wvu_rows * c->max_ntb * 8 + 256;
  return b;
}

nsp_status get_ws(nsp_ctx* c, void* ws, size_t need, char** out) {
  if (ws) {
    *out = (char*)ws;
    return NSP_OK;
  }
  if (c->ws_int_bytes < need) {
    if (c->ws_int) cudaFree(c->ws_int);
    c->ws_int = nullptr;
    c->ws_int_bytes = 0;
    NSP_CUDA_TRY(c, cudaMalloc(&c->ws_int, need));
    c->ws_int_bytes = need;
  }
  *out = (char*)c->ws_int;
  return NSP_OK;
}

// Y = S_G X (mode 1) or K_G X (mode 2); wvu: workspace of apply_ws_bytes.
nsp_status apply_into(nsp_ctx* c, const double* X, int ldx, double* Y, int ldy, int s, int mode, double* wvu) {
  const int cw = pick_cw(c, s);
  const int ldw = ld_pad(s, cw);
  // chunk-major padded W/U (s > 1 with the S_j^{-1} tiles): a 64 x 32 tile of W is one contiguous bulk copy
  const bool cm = c->d_minv && s > 1;
  const int64_t cs = (int64_t)c->wvu_rows * 36;
  // a1: W = A_IG X on the boundary-layer rows (zero padding rows / columns); on the INT8 a2+a3 path it also
  // reduces the W^T slices' per-(block, column) scale exponents (no separate pass over W)
  const bool ozp = cm && use_ozaki(c, s);
  int8_t* oz_wsl = ozp ? (int8_t*)((char*)wvu + oz_ws_offset(c, s)) : nullptr;
  int* oz_sexp = ozp ? (int*)(oz_wsl + nspk::oz_wslice_bytes(c->wvu_rows, s)) : nullptr;
  bool oz_have_exp = false;
  if (ozp) {
    NSP_CUDA_TRY(c, cudaMemsetAsync(oz_sexp, 0x80, (size_t)c->nsub * ((s + 127) / 128) * 128 * sizeof(int), c->stream));
    oz_have_exp = nspk::spmm_cs_oz(c->A2G, X, ldx, wvu, cs, ldw, s, c->d_oz_dexp, c->d_oz_tblk, oz_sexp, c->stream);
  }
  if (oz_have_exp) {
  } else if (cm) nspk::spmm_cs(c->A2G, X, ldx, nullptr, 0, 32, 0, wvu, 36, cs, ldw, s, 0, true, c->stream);
  else nspk::spmm(c->A2G, X, ldx, nullptr, 0, 0, wvu, ldw, s, 0, true, c->stream);
  // a2 + a3: U = L22^{-T} L22^{-1} W for every block, one launch: either as one symmetric product
  // with the setup's S_j^{-1} tiles (k_symm, no dependency chain) or as the two batched sweeps
  // live timing of the a2+a3 kernel: an event pair per eager call, or (inside the captured block-CG
  // graph) the context's dedicated pair, read after every graph launch (nsp_solver.cu)
  const bool gprof = c->prof_on && c->capturing;
  const bool prof = !gprof && c->prof_on && (size_t)(c->prof_used + 2) <= c->prof_ev.size();
  // the pair brackets the dominant kernel: the whole a2+a3 (DMMA product, sweeps, s = 1 product) or, on the
  // INT8 path, the tensor-core product k_oz_symm after the W^T slicing
  const bool oz1 = c->d_minv && s > 1 && use_ozaki(c, s);
  auto mark_start = [&]() {
    if (gprof) cudaEventRecordWithFlags(c->gprof_ev[0], c->stream, cudaEventRecordExternal);   // a graph node
    if (prof) cudaEventRecord(c->prof_ev[c->prof_used], c->stream);
  };
  if (!oz1) mark_start();
  double* U = wvu;
  // several ranks, s > 1 (SURVEY.md §8(e) budget: "process the subdomains adjacent to shared separators
  // first and launch the allreduce on a second stream"): the blocks coupled to shared rows are multiplied
  // first, their shared-row partials formed and allreduced on the comm stream while the other blocks'
  // products and the private rows' a4+a5 run on the context stream
  static const bool ovl_off = getenv("NSP_COMM_OVERLAP") && getenv("NSP_COMM_OVERLAP")[0] == '0';
  if (c->nranks > 1 && c->d_minv && s > 1 && !gprof && !prof && !ovl_off) {
    U = cm ? wvu + (int64_t)(ldw / 32) * cs : wvu + c->wvu_rows * (int64_t)ldw;
    const int nsh_it = c->n_items_sh, nrest = c->n_items - c->n_items_sh;
    const int64_t nsh = c->nG - c->n_priv;
    cudaStream_t main = c->stream;
    const bool oz = use_ozaki(c, s);
    int8_t* wsl = oz_wsl;
    int* sexp = oz_sexp;
    auto prod = [&](const int2* its, int nit) {
      if (oz) nspk::oz_product(c->d_subs, its, nit, s, ldw / 32, U, cs, c->d_oz_dexp, c->d_oz_mexp, c->d_oz_msl,
                               wsl, sexp, main, nullptr, 0, c->d_oz_ctr, c->d_oz_mz);
      else nspk::symm(c->d_subs, its, nit, c->d_minv, wvu, U, ldw, cw, main, cs);
    };
    nsp_count_path(oz ? NSP_PATH_OZAKI : NSP_PATH_SYMM);
    if (oz)
      nspk::oz_slice_w(c->d_subs, c->d_items, c->n_items, c->nsub, s, ldw / 32, wvu, cs, c->d_oz_dexp, wsl, sexp,
                       main, oz_have_exp);
    prod(c->d_items, nsh_it);
    DevCSR shr = c->AGG2;   // the shared rows' slice of the a4+a5 operator
    shr.rows = nsh;
    shr.rowptr = c->AGG2.rowptr + c->n_priv;
    if (cm) nspk::spmm_cs(shr, X, ldx, U, 36, cs, c->nG, Y + c->n_priv * (int64_t)ldy, ldy, 32, ldy, s, mode, true, main);
    else nspk::spmm(shr, X, ldx, U, ldw, c->nG, Y + c->n_priv * (int64_t)ldy, ldy, s, mode, true, main);
    if (!c->comm_stream) NSP_CUDA_TRY(c, cudaStreamCreateWithFlags(&c->comm_stream, cudaStreamNonBlocking));
    if (!c->ev_cfork) NSP_CUDA_TRY(c, cudaEventCreateWithFlags(&c->ev_cfork, cudaEventDisableTiming));
    if (!c->ev_cjoin) NSP_CUDA_TRY(c, cudaEventCreateWithFlags(&c->ev_cjoin, cudaEventDisableTiming));
    NSP_CUDA_TRY(c, cudaEventRecord(c->ev_cfork, main));
    NSP_CUDA_TRY(c, cudaStreamWaitEvent(c->comm_stream, c->ev_cfork, 0));
    c->stream = c->comm_stream;
    nsp_status e = finish_shared_rows(c, X, ldx, Y, ldy, s, mode != 2);   // allreduce + shared x shared A_G
    c->stream = main;
    if (e != NSP_OK) return e;
    NSP_CUDA_TRY(c, cudaEventRecord(c->ev_cjoin, c->comm_stream));
    if (nrest > 0) prod(c->d_items + nsh_it, nrest);
    DevCSR prv = c->AGG2;   // the private rows
    prv.rows = c->n_priv;
    if (cm) nspk::spmm_cs(prv, X, ldx, U, 36, cs, c->nG, Y, ldy, 32, ldy, s, mode, true, main);
    else nspk::spmm(prv, X, ldx, U, ldw, c->nG, Y, ldy, s, mode, true, main);
    NSP_CUDA_TRY(c, cudaStreamWaitEvent(main, c->ev_cjoin, 0));
    NSP_CUDA_TRY(c, cudaGetLastError());
    return NSP_OK;
  }
  if (c->d_minv) {
    U = cm ? wvu + (int64_t)(ldw / 32) * cs : wvu + c->wvu_rows * (int64_t)ldw;
    if (s == 1) {   // one right-hand side (outer PCG): memory-bound matrix-vector form, tiles read once
      double* P = U + c->wvu_rows * (int64_t)ldw;
      P = (double*)(((uintptr_t)P + 255) & ~(uintptr_t)255);
      nsp_count_path(NSP_PATH_SYMV);
      // NSP_OZ_SYMV=1: the product from the INT8 slices, decoded per entry - parity-clean but measured slower
      // (cfg5 outer PCG 20.1 vs 12.2 ms per iteration: the decode, not the bytes, binds); opt-in only
      static const bool oz_symv = getenv("NSP_OZ_SYMV") && getenv("NSP_OZ_SYMV")[0] == '1';
      if (getenv("NSP_SYMV2")) nspk::symv(c->d_subs, c->d_items, c->n_items, c->max_ntb, c->d_minv, wvu, ldw, U, c->stream);
      else if (c->d_oz_msl && oz_symv && c->opts.apply_kernel != 2)   // the INT8 slices, decoded (7 B per entry)
        nspk::oz_symv1(c->d_subs, c->d_items, c->n_items, c->max_ntb, c->d_oz_msl, c->d_oz_dexp, c->d_oz_mexp, wvu, ldw,
                       U, P, c->stream);
      else nspk::symv1(c->d_subs, c->d_items, c->n_items, c->max_ntb, c->d_minv, wvu, ldw, U, P, c->stream);
    } else if (use_ozaki(c, s)) {
      nsp_count_path(NSP_PATH_OZAKI);
      int8_t* wsl = oz_wsl;
      int* sexp = oz_sexp;
      nspk::oz_slice_w(c->d_subs, c->d_items, c->n_items, c->nsub, s, ldw / 32, wvu, cs, c->d_oz_dexp, wsl, sexp,
                       c->stream, oz_have_exp);
      mark_start();
      nspk::oz_product(c->d_subs, c->d_items, c->n_items, s, ldw / 32, U, cs, c->d_oz_dexp, c->d_oz_mexp,
                       c->d_oz_msl, wsl, sexp, c->stream, c->d_oz_pairs, c->n_oz_pairs, c->d_oz_ctr, c->d_oz_mz);
    } else {
      nsp_count_path(NSP_PATH_SYMM);
      nspk::symm(c->d_subs, c->d_items, c->n_items, c->d_minv, wvu, U, ldw, cw, c->stream, cs);
    }
  } else {
    nsp_count_path(NSP_PATH_SWEEPS);
    nspk::trsm_fb(c->d_subs, c->nsub, c->d_dense, wvu, ldw, cw, c->stream);
  }
  if (gprof) {
    cudaEventRecordWithFlags(c->gprof_ev[1], c->stream, cudaEventRecordExternal);
    c->gprof_in_graph = true;
  }
  if (prof) {
    cudaEventRecord(c->prof_ev[c->prof_used + 1], c->stream);
    c->prof_used += 2;
  }
  // a4 + a5: Y = A_G X - A_GI U (fused), or Y = A_GI U
  if (cm) nspk::spmm_cs(c->AGG2, X, ldx, U, 36, cs, c->nG, Y, ldy, 32, ldy, s, mode, true, c->stream);
  else nspk::spmm(c->AGG2, X, ldx, U, ldw, c->nG, Y, ldy, s, mode, true, c->stream);
  NSP_CUDA_TRY(c, cudaGetLastError());
  return finish_shared_rows(c, X, ldx, Y, ldy, s, mode != 2);
}

// Multi-rank: the shared rows of Y hold this rank's partial; sum the partials over ranks (one
// allreduce) and add the shared x shared A_G term (identically on every rank).  No-op for 1 rank.
nsp_status finish_shared_rows(nsp_ctx* c, const double* X, int ldx, double* Y, int ldy, int s, bool ag_term) {
  if (c->nranks <= 1) return NSP_OK;
  const int64_t nsh = c->nG - c->n_priv;
  if (nsh <= 0) return NSP_OK;
  nsp_status e = comm_allreduce(c, Y + c->n_priv * (int64_t)ldy, (size_t)nsh * ldy);
  if (e != NSP_OK) return e;
  if (ag_term)
    nspk::spmm(c->AGSH, X + c->n_priv * (int64_t)ldx, ldx, nullptr, 0, 0, Y + c->n_priv * (int64_t)ldy, ldy, s, 4,
               false, c->stream);
  NSP_CUDA_TRY(c, cudaGetLastError());
  return NSP_OK;
}

}  // namespace nspi

using namespace nspi;

extern "C" {

nsp_status nsp_dims(const nsp_ctx* c, int64_t* n, int64_t* n_gamma, int64_t* n_gamma_local, int* K_local) {
  if (!c) return NSP_ERR_ARG;
  if (n) *n = c->n;
  if (n_gamma) *n_gamma = c->nG_global;
  if (n_gamma_local) *n_gamma_local = c->nG;
  if (K_local) *K_local = c->nsub;
  return NSP_OK;
}

nsp_status nsp_shard_info(const nsp_ctx* c, int64_t* n_private, int64_t* n_shared, int* blk0, int* nblk) {
  if (!c) return NSP_ERR_ARG;
  if (n_private) *n_private = c->n_priv;
  if (n_shared) *n_shared = c->nG - c->n_priv;
  if (blk0) *blk0 = c->blk0;
  if (nblk) *nblk = c->nsub;
  return NSP_OK;
}

nsp_status nsp_gamma_index(const nsp_ctx* c, int64_t* orig) {
  if (!c || !orig) return NSP_ERR_ARG;
  std::memcpy(orig, c->gamma.data(), c->gamma.size() * sizeof(int64_t));
  return NSP_OK;
}

nsp_status nsp_profile(nsp_ctx* c, int enable) {
  if (!c) return NSP_ERR_ARG;
  if (enable && c->prof_ev.empty()) {
    c->prof_ev.resize(2 * 4096);
    for (auto& e : c->prof_ev) NSP_CUDA_TRY(c, cudaEventCreate(&e));
    for (auto& e : c->gprof_ev) NSP_CUDA_TRY(c, cudaEventCreate(&e));
  }
  if (c->prof_on != enable && c->bcg_graph) {   // the cached graph bakes in (or omits) the timing events
    cudaGraphExecDestroy(c->bcg_graph);
    c->bcg_graph = nullptr;
  }
  c->gprof_ms = 0.0;
  c->gprof_n = 0;
  c->prof_on = enable;
  c->prof_used = 0;
  return NSP_OK;
}

nsp_status nsp_profile_read(nsp_ctx* c, double* sweep_ms, long long* sweeps) {
  if (!c) return NSP_ERR_ARG;
  NSP_CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  double tot = 0.0;
  for (int k = 0; k + 1 < c->prof_used; k += 2) {
    float ms = 0.f;
    NSP_CUDA_TRY(c, cudaEventElapsedTime(&ms, c->prof_ev[k], c->prof_ev[k + 1]));
    tot += ms;
  }
  if (sweep_ms) *sweep_ms = tot + c->gprof_ms;
  if (sweeps) *sweeps = c->prof_used / 2 + c->gprof_n;
  c->prof_used = 0;
  c->gprof_ms = 0.0;
  c->gprof_n = 0;
  return NSP_OK;
}

nsp_status nsp_stats(const nsp_ctx* c, int64_t* st) {
  if (!c || !st) return NSP_ERR_ARG;
  int64_t l22 = 0;
  for (const FacSub& f : c->subs) l22 += (int64_t)f.ntb * (f.ntb + 1) / 2 * NSP_TILE_ELEMS;
  st[0] = c->n_I;
  st[1] = c->n_bl;
  st[2] = l22;
  st[3] = c->band_tiles + c->dense_tiles;
  st[4] = c->nnz_AG;
  st[5] = c->nnz_AGI;
  st[6] = c->max_b;
  st[7] = c->ag_bw;
  st[8] = c->sum_b2;
  st[9] = c->sum_b;
  st[10] = c->nsub;
  st[11] = c->wvu_rows;
  return NSP_OK;
}

nsp_status nsp_ozaki_stats(const nsp_ctx* c, int64_t* out) {
  if (!c || !out) return NSP_ERR_ARG;
  out[0] = c->d_oz_msl ? c->oz_prod_exec : 0;
  out[1] = c->d_oz_msl ? c->oz_prod_full : 0;
  out[2] = c->d_oz_msl ? c->oz_slice_bytes : 0;
  return NSP_OK;
}

nsp_status nsp_workspace_bytes(const nsp_ctx* c, int s, size_t* bytes) {
  if (!c || !bytes || s <= 0) return NSP_ERR_ARG;
  *bytes = solver_ws_bytes(c, s);
  return NSP_OK;
}

nsp_status nsp_schur_apply(nsp_ctx* c, const double* X, double* Y, int s, void* ws) {
  NspNvtx nvtx_range_("nsp_schur_apply");
  if (!c || !X || !Y || s <= 0 || s > 256) return NSP_ERR_ARG;
  char* w;
  nsp_status st = get_ws(c, ws, apply_ws_bytes(c, s), &w);
  if (st != NSP_OK) return st;
  return apply_into(c, X, s, Y, s, s, 1, (double*)w);
}

nsp_status nsp_kgamma_apply(nsp_ctx* c, const double* X, double* Y, int s, void* ws) {
  NspNvtx nvtx_range_("nsp_kgamma_apply");
  if (!c || !X || !Y || s <= 0 || s > 256) return NSP_ERR_ARG;
  char* w;
  nsp_status st = get_ws(c, ws, apply_ws_bytes(c, s), &w);
  if (st != NSP_OK) return st;
  return apply_into(c, X, s, Y, s, s, 2, (double*)w);
}

nsp_status nsp_gamma_apply(nsp_ctx* c, const double* X, double* Y, int s) {
  NspNvtx nvtx_range_("nsp_gamma_apply");
  if (!c || !X || !Y || s <= 0 || s > 256) return NSP_ERR_ARG;
  nspk::spmm(c->AGG2, X, s, nullptr, 0, c->nG, Y, s, s, 3, false, c->stream);
  NSP_CUDA_TRY(c, cudaGetLastError());
  return finish_shared_rows(c, X, s, Y, s, s, true);
}

nsp_status nsp_set_bcg_precond(nsp_ctx* c, int precond) {
  if (!c || precond < 0 || precond > 1) return NSP_ERR_ARG;
  if (precond == 1 && !c->has_ag) {
    c->err = "nsp_set_bcg_precond: M = A_G^{-1} needs the A_G operator (opts.factor_gamma at setup)";
    return NSP_ERR_STATE;
  }
  c->opts.bcg_precond = precond;   // the cached iteration graphs are keyed on it (rebuilt on change)
  return NSP_OK;
}

nsp_status nsp_dev_panel(double* Out, const double* Cin, const double* In, const double* M, int64_t n, int s,
                         double sgn, double* colsq, int path, void* stream) {
  if (n < 0 || (s != 64 && s != 128) || path < 0 || path > 1) return NSP_ERR_ARG;
  cudaStream_t st = (cudaStream_t)stream;
  if (n == 0) {   // empty block: nothing to update, zero column sums
    if (colsq && cudaMemsetAsync(colsq, 0, (size_t)s * 8, st) != cudaSuccess) return NSP_ERR_CUDA;
    return cudaStreamSynchronize(st) == cudaSuccess ? NSP_OK : NSP_ERR_CUDA;
  }
  if (!Out || !In || !M) return NSP_ERR_ARG;
  double* part = nullptr;
  if (colsq && cudaMalloc(&part, (size_t)(std::max<int64_t>((n + 63) / 64, 1024) + 1) * s * 8) != cudaSuccess)
    return NSP_ERR_CUDA;
  nsp_force_generic = path;
  const int npt = nspb::panel(Out, s, Cin, s, In, s, M, s, s, s, n, sgn, part, st);
  nsp_force_generic = 0;
  if (colsq) nspb::colsq_reduce(part, npt, s, colsq, st);
  const cudaError_t e = cudaStreamSynchronize(st);
  if (part) cudaFree(part);
  return e == cudaSuccess && cudaGetLastError() == cudaSuccess ? NSP_OK : NSP_ERR_CUDA;
}

nsp_status nsp_dev_gram(const double* Xa, const double* Xb, const double* Xb2, int64_t n, int s, double* out,
                        double* out2, int lower_first, int path, void* stream) {
  if (!out || (Xb2 && !out2) || n < 0 || (s != 64 && s != 128) || path < 0 || path > 1) return NSP_ERR_ARG;
  cudaStream_t st = (cudaStream_t)stream;
  if (n == 0) {   // empty contraction: zero Gram
    if (cudaMemsetAsync(out, 0, (size_t)s * s * 8, st) != cudaSuccess) return NSP_ERR_CUDA;
    if (out2 && cudaMemsetAsync(out2, 0, (size_t)s * s * 8, st) != cudaSuccess) return NSP_ERR_CUDA;
    return cudaStreamSynchronize(st) == cudaSuccess ? NSP_OK : NSP_ERR_CUDA;
  }
  if (!Xa || !Xb) return NSP_ERR_ARG;
  double* ws = nullptr;
  if (cudaMalloc(&ws, nspb::gram_ws_doubles(n, s, s) * 8) != cudaSuccess) return NSP_ERR_CUDA;
  nsp_force_generic = path;
  nspb::gram2(Xa, s, s, Xb, Xb2, s, s, n, out, out2, s, ws, st, lower_first != 0);
  nsp_force_generic = 0;
  const cudaError_t e = cudaStreamSynchronize(st);
  cudaFree(ws);
  return e == cudaSuccess && cudaGetLastError() == cudaSuccess ? NSP_OK : NSP_ERR_CUDA;
}

nsp_status nsp_dev_panel_gram(double* Out, const double* Cin, const double* In, const double* M, int64_t n,
                              double sgn, int gmode, double* gram, double* colsq, void* stream) {
  if (!Out || !In || !M || !gram || (gmode != 0 && gmode != 1) || !nspb::panel_gram_shape_ok(128, n)) return NSP_ERR_ARG;
  cudaStream_t st = (cudaStream_t)stream;
  double *ws = nullptr, *part = nullptr;
  if (cudaMalloc(&ws, nspb::gram_ws_doubles(n, 128, 128) * 8) != cudaSuccess) return NSP_ERR_CUDA;
  if (colsq && cudaMalloc(&part, (size_t)((n + 63) / 64 + 1) * 128 * 8) != cudaSuccess) {
    cudaFree(ws);
    return NSP_ERR_CUDA;
  }
  const int npt = nspb::panel_gram(Out, Cin, In, M, n, sgn, part, gmode, gram, ws, st);
  if (colsq) nspb::colsq_reduce(part, npt, 128, colsq, st);
  const cudaError_t e = cudaStreamSynchronize(st);
  cudaFree(ws);
  if (part) cudaFree(part);
  return e == cudaSuccess && cudaGetLastError() == cudaSuccess ? NSP_OK : NSP_ERR_CUDA;
}

nsp_status nsp_dev_philox_gaussian(double* out, int64_t rows, int s, uint64_t seed, unsigned stream_id, int64_t row0,
                                   void* stream) {
  if (!out || rows < 0 || s <= 0 || row0 < 0) return NSP_ERR_ARG;
  if (rows == 0) return NSP_OK;
  cudaStream_t st = (cudaStream_t)stream;
  std::vector<int64_t> g((size_t)rows);
  for (int64_t r = 0; r < rows; ++r) g[(size_t)r] = row0 + r;
  int64_t* dg = nullptr;
  if (cudaMalloc((void**)&dg, (size_t)rows * 8) != cudaSuccess) return NSP_ERR_CUDA;
  cudaMemcpy(dg, g.data(), (size_t)rows * 8, cudaMemcpyHostToDevice);
  nspk::philox_gaussian(out, rows, s, s, dg, seed, stream_id, st);
  const cudaError_t e = cudaStreamSynchronize(st);
  cudaFree(dg);
  return e == cudaSuccess && cudaGetLastError() == cudaSuccess ? NSP_OK : NSP_ERR_CUDA;
}

nsp_status nsp_dev_set_fused_pg(int mode) {
  if (mode < 0 || mode > 2) return NSP_ERR_ARG;
  nspb::nsp_fused_pg_mode = mode;
  return NSP_OK;
}

const char* nsp_last_error(const nsp_ctx* c) { return c ? c->err.c_str() : "null context"; }

void nsp_destroy(nsp_ctx* c) {
  if (!c) return;
  auto fr = [](void* p) {
    if (p) cudaFree(p);
  };
  fr(c->d_subs);
  fr(c->d_band);
  fr(c->d_dense);
  fr(c->d_border_first);
  fr(c->d_gband);
  fr(c->d_gsys);
  fr(c->d_gperm);
  fr(c->d_gperm_inv);
  fr(c->d_gchunks);
  fr(c->d_gchunk_first);
  fr(c->d_gtile_chunk);
  fr(c->d_gspkF);
  fr(c->d_gGF);
  fr(c->d_gXB);
  fr(c->d_gGB);
  fr(c->d_gspkB);
  fr(c->d_i1sys);
  fr(c->d_minv);
  fr(c->d_oz_msl);
  fr(c->d_oz_dexp);
  fr(c->d_oz_mexp);
  fr(c->d_oz_tblk);
  fr(c->d_oz_pairs);
  fr(c->d_oz_ctr);
  fr(c->d_oz_mz);
  fr(c->d_sell_code);
  fr(c->d_sell_tab);
  fr(c->d_items);
  fr(c->d_i1_src);
  fr(c->d_b_src);
  fr(c->d_g_src);
  fr(c->d_Z);
  fr(c->d_ELp);
  fr(c->d_int_src);
  fr(c->d_sigma);
  fr(c->d_sell_ptr);
  fr(c->d_sell_col);
  fr(c->d_sell_val);
  comm_free(c);
  if (c->bcg_graph) cudaGraphExecDestroy(c->bcg_graph);
  if (c->pcg_graph) cudaGraphExecDestroy(c->pcg_graph);
  if (c->bcg_wgraph) cudaGraphExecDestroy(c->bcg_wgraph);
  if (c->pcg_wgraph) cudaGraphExecDestroy(c->pcg_wgraph);
  if (c->d_phist) cudaFree(c->d_phist);
  if (c->d_bhist) cudaFree(c->d_bhist);
  if (c->d_bwidth) cudaFree(c->d_bwidth);
  if (c->gstream) cudaStreamDestroy(c->gstream);
  if (c->side_stream) cudaStreamDestroy(c->side_stream);
  if (c->apply_stream) cudaStreamDestroy(c->apply_stream);
  if (c->comm_stream) cudaStreamDestroy(c->comm_stream);
  if (c->ev_cfork) cudaEventDestroy(c->ev_cfork);
  if (c->ev_cjoin) cudaEventDestroy(c->ev_cjoin);
  if (c->ev_afork) cudaEventDestroy(c->ev_afork);
  if (c->ev_ajoin) cudaEventDestroy(c->ev_ajoin);
  if (c->ev_fork) cudaEventDestroy(c->ev_fork);
  if (c->ev_join) cudaEventDestroy(c->ev_join);
  for (DevCSR* m : {&c->A2G, &c->AGG2, &c->AGSH, &c->AGO, &c->CB, &c->C1, &c->AII}) {
    fr(m->rowptr);
    fr(m->col);
    fr(m->val);
  }
  fr(c->ws_int);
  for (auto& e : c->prof_ev) cudaEventDestroy(e);
  if (!c->prof_ev.empty())
    for (auto& e : c->gprof_ev) cudaEventDestroy(e);
  if (c->h_status) cudaFreeHost(c->h_status);
  solver_free(c);
  delete c;
}

}  // extern "C"

#include <atomic>
static std::atomic<long long> g_launches{0};
static std::atomic<long long> g_path[NSP_PATH_COUNT];
thread_local int nsp_force_generic = 0;
void nsp_count_path(int id) {
  if (id >= 0 && id < NSP_PATH_COUNT) g_path[id].fetch_add(1, std::memory_order_relaxed);
}
extern "C" int nsp_path_counters(long long* out, int n) {
  if (!out) return NSP_PATH_COUNT;
  for (int i = 0; i < n && i < NSP_PATH_COUNT; ++i) out[i] = g_path[i].load();
  return NSP_PATH_COUNT;
}
void nsp_count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }
void nsp_count_launches(long long k) { g_launches.fetch_add(k, std::memory_order_relaxed); }
long long nsp_launch_count() { return g_launches.load(); }
extern "C" long long nsp_kernel_launches(void) { return g_launches.load(); }
