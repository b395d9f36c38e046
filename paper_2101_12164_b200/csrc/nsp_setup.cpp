#include <cstdio>
// nsp_setup: host analysis (validation, DBBD permutation, per-block ordering, tile layout), the
// host->device copy, and the GPU numeric factorisation (§8(a) row s0).
//
// DBBD (PAPER.md:369-378 eq:perm_A): blocks 0..K-1 in ascending original index, then Gamma in
// ascending original index (reading C10).  Inside block j the interior is split into
//   I1 = nodes with no Gamma neighbour (ordered natural or RCM, whichever has the smaller
//        bandwidth) and
//   B  = boundary layer (nodes with a Gamma neighbour), ordered last.
// Since A_I_jG is nonzero only on the B rows, L_j^{-1} A_I_jG X is nonzero only on the B rows
// and equals L22^{-1} W_B, where L22 = chol(A_BB - A_B1 A_11^{-1} A_1B) is the trailing block of
// the Cholesky factor of A_I_j in this ordering; A_GI_j reads only the B rows of
// L_j^{-T} L_j^{-1} (.) which equal L22^{-T} L22^{-1} W_B.  The hot path therefore streams only
// the dense trailing factor L22.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <numeric>
#include <string>
#include <vector>

#include <omp.h>

#include "nsp_comm.h"
#include "nsp_internal.h"

using nspi::comm_init;

namespace {

using Clock = std::chrono::steady_clock;
double ms_since(Clock::time_point t0) {
  return std::chrono::duration<double, std::milli>(Clock::now() - t0).count();
}

// Reverse Cuthill-McKee on a local graph (adjacency in CSR), George-Liu pseudo-peripheral root.
std::vector<int> rcm_order(int n, const std::vector<int>& rp, const std::vector<int>& ci) {
  std::vector<int> order;
  order.reserve(n);
  std::vector<char> vis(n, 0);
  std::vector<int> deg(n);
  for (int i = 0; i < n; ++i) deg[i] = rp[i + 1] - rp[i];
  std::vector<int> level(n, -1), q;
  auto bfs_levels = [&](int root, int& ecc, int& last_min) {
    // BFS restricted to unvisited component; returns eccentricity and min-degree node of last level
    q.clear();
    q.push_back(root);
    level[root] = 0;
    size_t h = 0;
    while (h < q.size()) {
      int v = q[h++];
      for (int k = rp[v]; k < rp[v + 1]; ++k) {
        int u = ci[k];
        if (!vis[u] && level[u] < 0) {
          level[u] = level[v] + 1;
          q.push_back(u);
        }
      }
    }
    ecc = level[q.back()];
    last_min = q.back();
    for (int v : q)
      if (level[v] == ecc && deg[v] < deg[last_min]) last_min = v;
    for (int v : q) level[v] = -1;
  };
  for (int start = 0; start < n; ++start) {
    if (vis[start]) continue;
    // min degree node of this component
    int root = start;
    {
      int e, lm;
      bfs_levels(start, e, lm);
      for (int v : q)
        if (deg[v] < deg[root]) root = v;
    }
    int ecc, lm;
    bfs_levels(root, ecc, lm);
    for (int it = 0; it < 8; ++it) {
      int ecc2, lm2;
      bfs_levels(lm, ecc2, lm2);
      if (ecc2 > ecc) {
        root = lm;
        ecc = ecc2;
        lm = lm2;
      } else {
        break;
      }
    }
    // Cuthill-McKee BFS from root, neighbours by ascending degree
    size_t h = order.size();
    order.push_back(root);
    vis[root] = 1;
    std::vector<int> nb;
    while (h < order.size()) {
      int v = order[h++];
      nb.clear();
      for (int k = rp[v]; k < rp[v + 1]; ++k)
        if (!vis[ci[k]]) nb.push_back(ci[k]);
      std::sort(nb.begin(), nb.end(), [&](int a, int b) { return deg[a] != deg[b] ? deg[a] < deg[b] : a < b; });
      for (int u : nb)
        if (!vis[u]) {
          vis[u] = 1;
          order.push_back(u);
        }
    }
  }
  std::reverse(order.begin(), order.end());
  return order;
}

int bandwidth(int n, const std::vector<int>& rp, const std::vector<int>& ci, const std::vector<int>& pos) {
  int bw = 0;
  for (int v = 0; v < n; ++v)
    for (int k = rp[v]; k < rp[v + 1]; ++k) bw = std::max(bw, std::abs(pos[v] - pos[ci[k]]));
  return bw;
}

struct SubHost {
  int j = 0;                       // global block id
  std::vector<int64_t> nodes;      // original ids in the new local order: I1 (n1) then B (b)
  int n1 = 0, b = 0, bw = 0, wb = 0, nt1 = 0, ntb = 0;
  bool rcm = false;
  std::vector<int> border_first;   // per B tile: first column tile with a nonzero
  // entries (lower triangle) in tile storage, indices relative to the region base
  std::vector<int64_t> band_idx, dense_idx, border_idx;
  std::vector<double> band_val, dense_val, border_val;
};

template <class T>
nsp_status upload(nsp_ctx* c, T** dptr, const std::vector<T>& h) {
  *dptr = nullptr;
  if (h.empty()) return NSP_OK;
  NSP_CUDA_TRY(c, cudaMalloc((void**)dptr, h.size() * sizeof(T)));
  NSP_CUDA_TRY(c, cudaMemcpy(*dptr, h.data(), h.size() * sizeof(T), cudaMemcpyHostToDevice));
  return NSP_OK;
}

nsp_status upload_csr(nsp_ctx* c, DevCSR& d, const HostCSR32& h) {
  d.rows = (int64_t)h.rowptr.size() - 1;
  d.nnz = (int64_t)h.col.size();
  nsp_status st;
  if ((st = upload(c, &d.rowptr, h.rowptr)) != NSP_OK) return st;
  if ((st = upload(c, &d.col, h.col)) != NSP_OK) return st;
  if ((st = upload(c, &d.val, h.val)) != NSP_OK) return st;
  return NSP_OK;
}

}  // namespace

extern "C" void nsp_default_opts(nsp_opts* o) {
  std::memset(o, 0, sizeof(*o));
  o->device = 0;
  o->stream = nullptr;
  o->nranks = 1;
  o->rank = 0;
  o->nccl_id = nullptr;
  o->bcg_precond = 0;
  o->factor_gamma = 0;
  o->orth_tau = 1e-14;
  o->nys_eps_rel = 1e-12;
  o->scratch_bytes = 0;
  o->verbose = 0;
}

static nsp_status fail(nsp_ctx* c, nsp_status st, const std::string& msg) {
  c->err = msg;
  return st;
}

nsp_status nsp_setup_impl(nsp_ctx* c, const nsp_csr* A, const int32_t* part, int K, nsp_report* rep);
static nsp_status validate_inputs(nsp_ctx* c, const nsp_csr* A, const int32_t* part, int K);

// A_G^{-1} by a fixed Chebyshev iteration.  Host: A_G's rows in the local Gamma
// order; the upper spectrum bound is min(Gershgorin, 1.05 x the top Lanczos Ritz value), the lower
// one the bottom Ritz value / 1.05 (Lanczos from a fixed start vector, 120 steps, no
// reorthogonalisation: the extreme Ritz values converge first); the degree K makes the Chebyshev
// error bound 2 q^K <= 1e-15, q = (sqrt(kappa) - 1) / (sqrt(kappa) + 1) (Saad, Alg. 12.1).
static double tridiag_count_below(const std::vector<double>& al, const std::vector<double>& be, double x) {
  // Sturm count: eigenvalues of the symmetric tridiagonal (al, be) smaller than x
  int cnt = 0;
  double d = 1.0;
  for (size_t i = 0; i < al.size(); ++i) {
    const double b2 = i ? be[i - 1] * be[i - 1] : 0.0;
    d = al[i] - x - (i ? b2 / d : 0.0);
    if (d == 0.0) d = -1e-300;
    if (d < 0.0) ++cnt;
  }
  return cnt;
}

// glist: the Gamma rows the spectrum bounds are taken over, gpos: original id -> position in glist.  One
// rank: the local rows.  Several ranks: the GLOBAL Gamma set (every rank derives the same bounds and
// coefficients - the polynomial is one operator on the whole border; its applications are sharded).
static nsp_status setup_gamma_cheb(nsp_ctx* c, const nsp_csr* A, const int32_t* part,
                                   const std::vector<int32_t>& gpos_local, const std::vector<int64_t>* glist_in = nullptr) {
  std::vector<int32_t> gpos_glob;
  const std::vector<int64_t>& glist = glist_in ? *glist_in : c->gamma;
  if (glist_in) {
    gpos_glob.assign(A->n, -1);
    for (size_t g = 0; g < glist.size(); ++g) gpos_glob[glist[g]] = (int32_t)g;
  }
  const std::vector<int32_t>& gpos = glist_in ? gpos_glob : gpos_local;
  const int64_t nG = (int64_t)glist.size();
  const int64_t* rp = A->rowptr;
  const int32_t* ci = A->colidx;
  const double* va = A->val;
  std::vector<int64_t> grp(nG + 1, 0);
  for (int64_t g = 0; g < nG; ++g) {
    const int64_t v = glist[g];
    int64_t k = 0;
    for (int64_t q = rp[v]; q < rp[v + 1]; ++q)
      if (part[ci[q]] < 0) ++k;
    grp[g + 1] = grp[g] + k;
  }
  std::vector<int32_t> gci(grp[nG]);
  std::vector<double> gva(grp[nG]);
  double gersh = 0.0;
#pragma omp parallel for schedule(static) reduction(max : gersh)
  for (int64_t g = 0; g < nG; ++g) {
    const int64_t v = glist[g];
    int64_t k = grp[g];
    double rs = 0.0;
    for (int64_t q = rp[v]; q < rp[v + 1]; ++q)
      if (part[ci[q]] < 0) {
        gci[k] = gpos[ci[q]];
        gva[k++] = va[q];
        rs += std::fabs(va[q]);
      }
    gersh = std::max(gersh, rs);
  }
  auto spmv = [&](const std::vector<double>& x, std::vector<double>& y) {
#pragma omp parallel for schedule(static)
    for (int64_t g = 0; g < nG; ++g) {
      double s = 0.0;
      for (int64_t k = grp[g]; k < grp[g + 1]; ++k) s += gva[k] * x[gci[k]];
      y[g] = s;
    }
  };
  const int m = (int)std::min<int64_t>(120, nG);
  std::vector<double> v(nG), vp(nG, 0.0), w(nG), al, be;
  uint64_t st = 0x9E3779B97F4A7C15ull;
  double nrm = 0.0;
  for (int64_t g = 0; g < nG; ++g) {
    st = st * 6364136223846793005ull + 1442695040888963407ull;
    v[g] = (double)(st >> 11) * (1.0 / 9007199254740992.0) - 0.5;
    nrm += v[g] * v[g];
  }
  nrm = std::sqrt(nrm);
  for (auto& x : v) x /= nrm;
  double b = 0.0;
  for (int k = 0; k < m; ++k) {
    spmv(v, w);
    double a = 0.0;
    for (int64_t g = 0; g < nG; ++g) {
      w[g] -= b * vp[g];
      a += v[g] * w[g];
    }
    double bn = 0.0;
    for (int64_t g = 0; g < nG; ++g) {
      w[g] -= a * v[g];
      bn += w[g] * w[g];
    }
    bn = std::sqrt(bn);
    al.push_back(a);
    if (k + 1 == m || bn <= 1e-14 * std::fabs(a)) break;
    be.push_back(bn);
    b = bn;
    for (int64_t g = 0; g < nG; ++g) {
      vp[g] = v[g];
      v[g] = w[g] / bn;
    }
  }
  be.resize(al.size() - 1);
  // extreme Ritz values by bisection on the Sturm count
  double lo = -gersh - 1.0, hi = gersh + 1.0;
  for (int it = 0; it < 200; ++it) {
    const double mid = 0.5 * (lo + hi);
    if (tridiag_count_below(al, be, mid) >= 1) hi = mid;
    else lo = mid;
  }
  const double tmin = hi;
  lo = -gersh - 1.0;
  hi = gersh + 1.0;
  for (int it = 0; it < 200; ++it) {
    const double mid = 0.5 * (lo + hi);
    if (tridiag_count_below(al, be, mid) >= (double)al.size()) hi = mid;
    else lo = mid;
  }
  const double tmax = hi;
  if (!(tmin > 0.0)) return fail(c, NSP_ERR_NOT_SPD, "nsp_setup: A_G Lanczos estimate not positive (A_G not SPD?)");
  const double a = tmin / 1.05, bb = std::min(gersh, 1.05 * tmax);
  const double kappa = bb / a;
  const double q = (std::sqrt(kappa) - 1.0) / (std::sqrt(kappa) + 1.0);
  const int K = (int)std::ceil(std::log(2.0 / 1e-15) / std::log(1.0 / std::max(q, 1e-300)));
  if (K > 4000)
    return fail(c, NSP_ERR_OOM, "nsp_setup: A_G too ill-conditioned for the Chebyshev solver (kappa " +
                                    std::to_string(kappa) + ") and its band factor does not fit");
  c->cheb_a = a;
  c->cheb_b = bb;
  c->cheb_K = std::max(K, 1);
  const double theta = 0.5 * (bb + a), delta = 0.5 * (bb - a), sigma1 = theta / delta;
  c->cheb_c1.assign(c->cheb_K, 0.0);
  c->cheb_c2.assign(c->cheb_K, 0.0);
  double rho = 1.0 / sigma1;
  for (int k = 0; k < c->cheb_K; ++k) {   // d_{k+1} = rho_{k+1} rho_k d_k + (2 rho_{k+1} / delta) r_{k+1}
    const double rn = 1.0 / (2.0 * sigma1 - rho);
    c->cheb_c1[k] = rn * rho;
    c->cheb_c2[k] = 2.0 * rn / delta;
    rho = rn;
  }
  c->ag_cheb = true;
  c->has_ag = true;
  c->ag_bw = -c->cheb_K;   // nsp_stats: negative = Chebyshev degree
  if (c->opts.verbose)
    fprintf(stderr, "[nsp] A_G^{-1}: Chebyshev on [%.4g, %.4g] (kappa %.1f), K = %d\n", a, bb, kappa, c->cheb_K);
  return NSP_OK;
}

// Cholesky factor of A_G (eq:cholesky) for the first-level preconditioner
// S~_1^{-1} = A_G^{-1} (eq:S1) and M_2: RCM band ordering of the Gamma graph, band tiles, the same
// GPU tile-Cholesky kernel as the blocks (a band-only block).
static nsp_status setup_gamma_factor(nsp_ctx* c, const nsp_csr* A, const int32_t* part,
                                     const std::vector<int32_t>& gpos, nsp_report* rep) {
  const int64_t nG = c->nG;
  if (nG == 0) return NSP_OK;
  if (nG > INT32_MAX) return fail(c, NSP_ERR_ARG, "A_G too large");
  const int64_t* rp = A->rowptr;
  const int32_t* ci = A->colidx;
  const double* va = A->val;
  std::vector<int> arp(nG + 1, 0), aci;
  for (int64_t g = 0; g < nG; ++g) {
    const int64_t v = c->gamma[g];
    for (int64_t q = rp[v]; q < rp[v + 1]; ++q) {
      const int64_t u = ci[q];
      if (u != v && part[u] < 0 && va[q] != 0.0) aci.push_back(gpos[u]);
    }
    arp[g + 1] = (int)aci.size();
  }
  std::vector<int> ord;
  if (c->opts.ag_order == 1) {   // natural Gamma order: R_G = chol(A_G) as written (M_1 parity, small n_G)
    ord.resize(nG);
    for (int64_t k = 0; k < nG; ++k) ord[k] = (int)k;
  } else {
    ord = rcm_order((int)nG, arp, aci);
  }
  std::vector<int> pos(nG);
  for (int64_t k = 0; k < nG; ++k) pos[ord[k]] = (int)k;
  const int bw = bandwidth((int)nG, arp, aci, pos);
  c->ag_bw = bw;
  const int nt = (int)((nG + NSP_TILE - 1) / NSP_TILE);
  const int wb = std::min(nt - 1, (bw + NSP_TILE - 1) / NSP_TILE);
  const int64_t tiles = (int64_t)nt * (wb + 1);
  size_t free_b = 0, total_b = 0;
  NSP_CUDA_TRY(c, cudaMemGetInfo(&free_b, &total_b));
  if ((double)tiles * NSP_TILE_ELEMS * 8 > 0.4 * (double)free_b)
    return fail(c, NSP_ERR_OOM, "nsp_setup: A_G band factor (RCM bandwidth " + std::to_string(bw) +
                                    ") exceeds the device budget (opts.ag_solver 0 / 2: Chebyshev iteration)");
  std::vector<int64_t> idx;
  std::vector<double> val;
  for (int64_t g = 0; g < nG; ++g) {
    const int64_t v = c->gamma[g];
    const int li = pos[g];
    for (int64_t q = rp[v]; q < rp[v + 1]; ++q) {
      const int64_t u = ci[q];
      if (part[u] >= 0) continue;
      const int lj = pos[gpos[u]];
      if (lj > li) continue;
      const int I = li / NSP_TILE, Kt = lj / NSP_TILE;
      idx.push_back(((int64_t)Kt * (wb + 1) + (I - Kt)) * NSP_TILE_ELEMS + (li % NSP_TILE) * NSP_TILE + lj % NSP_TILE);
      val.push_back(va[q]);
    }
  }
  NSP_CUDA_TRY(c, cudaMalloc((void**)&c->d_gband, (size_t)tiles * NSP_TILE_ELEMS * 8));
  NSP_CUDA_TRY(c, cudaMemsetAsync(c->d_gband, 0, (size_t)tiles * NSP_TILE_ELEMS * 8, c->stream));
  c->gband_tiles = tiles;
  int64_t* d_idx = nullptr;
  double* d_val = nullptr;
  nsp_status st;
  if ((st = upload(c, &d_idx, idx)) != NSP_OK) return st;
  if ((st = upload(c, &d_val, val)) != NSP_OK) return st;
  nspk::scatter(c->d_gband, d_idx, d_val, (int64_t)idx.size(), c->stream);
  if (nG % NSP_TILE) {
    std::vector<int64_t> ti{(int64_t)(nt - 1) * (wb + 1)};
    std::vector<int> fr{(int)(nG % NSP_TILE)};
    int64_t* d_t = nullptr;
    int* d_f = nullptr;
    if ((st = upload(c, &d_t, ti)) != NSP_OK) return st;
    if ((st = upload(c, &d_f, fr)) != NSP_OK) return st;
    nspk::set_pad_identity(c->d_gband, d_t, d_f, 1, c->stream);
    NSP_CUDA_TRY(c, cudaStreamSynchronize(c->stream));
    cudaFree(d_t);
    cudaFree(d_f);
  }
  FacSub F{};
  F.nt1 = nt;
  F.ntb = 0;
  F.wb = wb;
  F.n1 = (int)nG;
  F.status_idx = 0;
  std::vector<FacSub> fv{F};
  std::vector<int> bf{0};
  FacSub* d_f = nullptr;
  int* d_bf = nullptr;
  int* d_stat = nullptr;
  if ((st = upload(c, &d_f, fv)) != NSP_OK) return st;
  if ((st = upload(c, &d_bf, bf)) != NSP_OK) return st;
  NSP_CUDA_TRY(c, cudaMalloc((void**)&d_stat, sizeof(int)));
  NSP_CUDA_TRY(c, cudaMemsetAsync(d_stat, 0, sizeof(int), c->stream));
  nspk::tile_cholesky(d_f, 1, c->d_gband, nullptr, nullptr, d_bf, d_stat, c->stream);
  NSP_CUDA_TRY(c, cudaGetLastError());
  int hstat = 0;
  NSP_CUDA_TRY(c, cudaMemcpyAsync(&hstat, d_stat, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
  NSP_CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  cudaFree(d_idx);
  cudaFree(d_val);
  cudaFree(d_f);
  cudaFree(d_bf);
  cudaFree(d_stat);
  if (hstat != 0) {
    const int r = hstat - 1;
    const int64_t orig = r < nG ? c->gamma[ord[r]] : -1;
    if (rep) {
      rep->bad_block = -1;
      rep->bad_pivot = orig;
      rep->status = NSP_ERR_NOT_SPD;
    }
    return fail(c, NSP_ERR_NOT_SPD, "nsp_setup: A_G not SPD (pivot at node " + std::to_string(orig) + ")");
  }
  std::vector<int32_t> gp((size_t)nt * NSP_TILE, -1), gpi(nG);
  for (int64_t g = 0; g < nG; ++g) {
    gp[pos[g]] = (int32_t)g;
    gpi[g] = pos[g];
  }
  if ((st = upload(c, &c->d_gperm, gp)) != NSP_OK) return st;
  if ((st = upload(c, &c->d_gperm_inv, gpi)) != NSP_OK) return st;
  std::vector<TriSys> ts{TriSys{c->d_gband, nt, wb, 0}};
  if ((st = upload(c, &c->d_gsys, ts)) != NSP_OK) return st;
  c->g_nt = nt;
  c->g_wb = wb;
  c->has_ag = true;
  // partitioned solve (narrow band: the chunks couple through exactly one factor tile): P chunk
  // systems and the spikes S_k = L_kk^{-1}[C_k; 0], T_k = L_kk^{-T}[0; C_{k+1}^T] (nsp_kernels.cu)
  if (wb <= 1 && nt >= 16 && !getenv("NSP_NO_SPIKE")) {
    int P = (int)std::sqrt((double)nt);
    P = std::max(2, std::min(32, P));
    std::vector<int> first(P + 1), tchunk(nt);
    for (int k = 0; k <= P; ++k) first[k] = (int)((int64_t)k * nt / P);
    for (int k = 0; k < P; ++k)
      for (int I = first[k]; I < first[k + 1]; ++I) tchunk[I] = k;
    std::vector<TriSys> ch(P);
    for (int k = 0; k < P; ++k)
      ch[k] = TriSys{c->d_gband + (int64_t)first[k] * (wb + 1) * NSP_TILE_ELEMS, first[k + 1] - first[k], wb,
                     (int64_t)first[k] * 64};
    if ((st = upload(c, &c->d_gchunks, ch)) != NSP_OK) return st;
    if ((st = upload(c, &c->d_gchunk_first, first)) != NSP_OK) return st;
    if ((st = upload(c, &c->d_gtile_chunk, tchunk)) != NSP_OK) return st;
    const size_t sb = (size_t)nt * 64 * 64 * 8;
    NSP_CUDA_TRY(c, cudaMalloc((void**)&c->d_gspkF, sb));
    NSP_CUDA_TRY(c, cudaMalloc((void**)&c->d_gspkB, sb));
    NSP_CUDA_TRY(c, cudaMemsetAsync(c->d_gspkF, 0, sb, c->stream));
    NSP_CUDA_TRY(c, cudaMemsetAsync(c->d_gspkB, 0, sb, c->stream));
    std::vector<double> tl(NSP_TILE_ELEMS), tt(NSP_TILE_ELEMS);
    for (int k = 1; k < P; ++k) {   // C_k = factor tile (first[k], first[k] - 1)
      const double* Ck = c->d_gband + ((int64_t)(first[k] - 1) * (wb + 1) + 1) * NSP_TILE_ELEMS;
      NSP_CUDA_TRY(c, cudaMemcpyAsync(c->d_gspkF + (int64_t)first[k] * 64 * 64, Ck, NSP_TILE_ELEMS * 8,
                                      cudaMemcpyDeviceToDevice, c->stream));
      NSP_CUDA_TRY(c, cudaMemcpy(tl.data(), Ck, NSP_TILE_ELEMS * 8, cudaMemcpyDeviceToHost));
      for (int i = 0; i < 64; ++i)
        for (int j = 0; j < 64; ++j) tt[i * 64 + j] = tl[j * 64 + i];
      NSP_CUDA_TRY(c, cudaMemcpy(c->d_gspkB + (int64_t)(first[k] - 1) * 64 * 64, tt.data(), NSP_TILE_ELEMS * 8,
                                 cudaMemcpyHostToDevice));
    }
    nspk::tri_fb(c->d_gchunks + 1, P - 1, c->d_gspkF, 64, 32, true, false, c->stream, wb);   // S_k, k >= 1
    nspk::tri_fb(c->d_gchunks, P - 1, c->d_gspkB, 64, 32, false, true, c->stream, wb);       // T_k, k <= P-2
    // reassociated sweeps: X_II L_{I,I-1}, X_II^T, X_II^T L_{I+1,I}^T per tile row (X_II: the band's own)
    const size_t tb = (size_t)nt * NSP_TILE_ELEMS * 8;
    NSP_CUDA_TRY(c, cudaMalloc((void**)&c->d_gGF, tb));
    NSP_CUDA_TRY(c, cudaMalloc((void**)&c->d_gXB, tb));
    NSP_CUDA_TRY(c, cudaMalloc((void**)&c->d_gGB, tb));
    nspk::band_prep(c->d_gband, nt, wb, nullptr, c->d_gGF, c->d_gXB, c->d_gGB, c->stream);
    NSP_CUDA_TRY(c, cudaStreamSynchronize(c->stream));
    NSP_CUDA_TRY(c, cudaGetLastError());
    c->g_P = P;
  }
  return NSP_OK;
}

// ---------------------------------------------------------------------------------------------
// Shard plan: rank r owns the contiguous block range [rK/G, (r+1)K/G) - a subtree of
// the depth-first ND leaf numbering.  A Gamma row is PRIVATE to r when every block adjacent to it is
// owned by r and none of its A_G neighbours is private to another rank; every other Gamma row is
// SHARED (replicated on all ranks, its S_G value completed by one allreduce of per-rank partials).
// With G = 1 every Gamma row is private (ascending original id, reading C10).  Host only.
// ---------------------------------------------------------------------------------------------
struct ShardPlan {
  int blk0 = 0, nblk = 0;
  std::vector<int64_t> priv, shared;   // original ids, ascending
};

static int block_owner_of(int j, int K, int G) {
  // largest q with floor(qK/G) <= j
  int q = (int)(((int64_t)j * G + G - 1) / K);
  while (q > 0 && (int64_t)q * K / G > j) --q;
  while (q + 1 < G && (int64_t)(q + 1) * K / G <= j) ++q;
  return q;
}

static bool make_shard_plan(const nsp_csr* A, const int32_t* part, int K, int G, int r, ShardPlan& P,
                            std::string& err) {
  if (G < 1 || G > 64 || r < 0 || r >= G) {
    err = "nsp_setup: nranks must be in [1, 64] and 0 <= rank < nranks";
    return false;
  }
  const int64_t n = A->n;
  const int64_t* rp = A->rowptr;
  const int32_t* ci = A->colidx;
  const double* va = A->val;
  P.blk0 = (int)((int64_t)r * K / G);
  P.nblk = (int)((int64_t)(r + 1) * K / G) - P.blk0;
  P.priv.clear();
  P.shared.clear();
  if (G == 1) {
    for (int64_t i = 0; i < n; ++i)
      if (part[i] < 0) P.priv.push_back(i);
    return true;
  }
  std::vector<int> owner(K);
  for (int j = 0; j < K; ++j) owner[j] = block_owner_of(j, K, G);
  std::vector<int> cand(n, -2);   // -2: not Gamma, -1: shared, >= 0: private candidate of that rank
#pragma omp parallel for schedule(dynamic, 4096)
  for (int64_t g = 0; g < n; ++g) {
    if (part[g] >= 0) continue;
    uint64_t mask = 0;
    for (int64_t q = rp[g]; q < rp[g + 1]; ++q) {
      const int64_t u = ci[q];
      if (part[u] >= 0 && va[q] != 0.0) mask |= 1ull << owner[part[u]];
    }
    cand[g] = __builtin_popcountll(mask) == 1 ? __builtin_ctzll(mask) : -1;
  }
  std::vector<char> demote(n, 0);
#pragma omp parallel for schedule(dynamic, 4096)
  for (int64_t g = 0; g < n; ++g) {
    if (cand[g] < 0) continue;
    for (int64_t q = rp[g]; q < rp[g + 1]; ++q) {
      const int64_t h = ci[q];
      if (h != g && cand[h] >= 0 && cand[h] != cand[g] && va[q] != 0.0) {
        demote[g] = 1;
        break;
      }
    }
  }
  for (int64_t g = 0; g < n; ++g) {
    if (cand[g] == -2) continue;
    const int o = demote[g] ? -1 : cand[g];
    if (o < 0) P.shared.push_back(g);
    else if (o == r) P.priv.push_back(g);
  }
  return true;
}

extern "C" nsp_status nsp_shard_plan(const nsp_csr* A, const int32_t* part, int K, int nranks, int rank,
                                     int64_t* n_private, int64_t* n_shared, int64_t* gamma_local, int* blk0,
                                     int* nblk) {
  if (!A || !part || K <= 0 || A->n <= 0) return NSP_ERR_ARG;
  for (int64_t i = 0; i < A->n; ++i)
    if (part[i] < -1 || part[i] >= K) return NSP_ERR_ARG;
  ShardPlan P;
  std::string err;
  if (!make_shard_plan(A, part, K, nranks, rank, P, err)) return NSP_ERR_ARG;
  if (n_private) *n_private = (int64_t)P.priv.size();
  if (n_shared) *n_shared = (int64_t)P.shared.size();
  if (gamma_local) {
    std::copy(P.priv.begin(), P.priv.end(), gamma_local);
    std::copy(P.shared.begin(), P.shared.end(), gamma_local + P.priv.size());
  }
  if (blk0) *blk0 = P.blk0;
  if (nblk) *nblk = P.nblk;
  return NSP_OK;
}

extern "C" nsp_status nsp_setup(const nsp_csr* A, const int32_t* part, int K, const nsp_opts* opts,
                                nsp_ctx** out, nsp_report* rep) {
  NspNvtx nvtx_range_("nsp_setup");
  if (!out) return NSP_ERR_ARG;
  *out = nullptr;
  nsp_ctx* c = new nsp_ctx();
  if (opts) c->opts = *opts;
  else nsp_default_opts(&c->opts);
  if (const char* ev = getenv("NSP_VERBOSE")) c->opts.verbose = ev[0] == '1';   // diagnostics
  *out = c;
  if (!A || !part || K <= 0) return fail(c, NSP_ERR_ARG, "nsp_setup: null A/part or K <= 0");
  c->device = c->opts.device;
  c->stream = (cudaStream_t)c->opts.stream;
  c->nranks = c->opts.nranks > 0 ? c->opts.nranks : 1;
  c->rank = c->opts.rank;
  if (c->nranks > 1 && (c->opts.factor_gamma || c->opts.bcg_precond) &&
      (c->opts.ag_solver == 1 || c->opts.nys_form != 0))
    return fail(c, NSP_ERR_ARG, "nsp_setup: with several ranks A_G^{-1} is the sharded Chebyshev operator "
                                "(ag_solver 0 / 2) and nys_form must be 0");
  nsp_status vs = validate_inputs(c, A, part, K);   // host-only: errors reported without a device
  if (vs != NSP_OK) return vs;
  NSP_CUDA_TRY(c, cudaSetDevice(c->device));
  nsp_status st = nsp_setup_impl(c, A, part, K, rep);
  if (st != NSP_OK) return st;
  return comm_init(c);
}

// Host-only input validation (SPEC.md:30-31 CSR, SPEC.md:135 separator property): runs before
// any device call, so malformed inputs are reported with NSP_ERR_ARG even without a GPU.
static nsp_status validate_inputs(nsp_ctx* c, const nsp_csr* A, const int32_t* part, int K) {
  const int64_t n = A->n;
  const int64_t* rp = A->rowptr;
  const int32_t* ci = A->colidx;
  const double* va = A->val;
  if (n <= 0 || !rp || !ci || !va) return fail(c, NSP_ERR_ARG, "nsp_setup: empty or null CSR");
  if (rp[0] != 0) return fail(c, NSP_ERR_ARG, "nsp_setup: rowptr[0] != 0");
  if (c->opts.ag_order < 0 || c->opts.ag_order > 1) return fail(c, NSP_ERR_ARG, "nsp_setup: ag_order must be 0 or 1");
  if (c->opts.ag_solver < 0 || c->opts.ag_solver > 2) return fail(c, NSP_ERR_ARG, "nsp_setup: ag_solver must be 0..2");
  if (c->opts.nys_form < 0 || c->opts.nys_form > 3) return fail(c, NSP_ERR_ARG, "nsp_setup: nys_form must be 0..3");
  // ---------------- validation
  std::string verr;
  int64_t bad_row = -1;
#pragma omp parallel for schedule(dynamic, 4096)
  for (int64_t i = 0; i < n; ++i) {
    if (bad_row >= 0) continue;
    bool ok = rp[i + 1] >= rp[i];
    for (int64_t q = rp[i]; ok && q < rp[i + 1]; ++q) {
      if (ci[q] < 0 || ci[q] >= n) ok = false;
      else if (q > rp[i] && ci[q] <= ci[q - 1]) ok = false;
    }
    if (!ok) {
#pragma omp critical
      if (bad_row < 0 || i < bad_row) bad_row = i;
    }
  }
  if (bad_row >= 0)
    return fail(c, NSP_ERR_ARG, "nsp_setup: row " + std::to_string(bad_row) +
                                    " has out-of-range or unsorted column indices");
  for (int64_t i = 0; i < n; ++i)
    if (part[i] < -1 || part[i] >= K)
      return fail(c, NSP_ERR_ARG, "nsp_setup: part[" + std::to_string(i) + "] = " + std::to_string(part[i]) +
                                      " not in {-1} U [0, K)");
  int64_t asym = -1, asym_j = -1, sep_i = -1, sep_j = -1;
#pragma omp parallel for schedule(dynamic, 4096)
  for (int64_t i = 0; i < n; ++i) {
    for (int64_t q = rp[i]; q < rp[i + 1]; ++q) {
      const int64_t j = ci[q];
      // symmetric value check via binary search in row j
      const int32_t* b = ci + rp[j];
      const int32_t* e = ci + rp[j + 1];
      const int32_t* f = std::lower_bound(b, e, (int32_t)i);
      if (f == e || *f != i || va[rp[j] + (f - b)] != va[q]) {
#pragma omp critical
        if (asym < 0) {
          asym = i;
          asym_j = j;
        }
      }
      if (va[q] != 0.0 && part[i] >= 0 && part[j] >= 0 && part[i] != part[j]) {
#pragma omp critical
        if (sep_i < 0) {
          sep_i = i;
          sep_j = j;
        }
      }
    }
  }
  if (asym >= 0)
    return fail(c, NSP_ERR_ARG, "nsp_setup: matrix not symmetric at (" + std::to_string(asym) + ", " +
                                    std::to_string(asym_j) + ")");
  if (sep_i >= 0)
    return fail(c, NSP_ERR_ARG, "nsp_setup: separator property violated at entry (" + std::to_string(sep_i) +
                                    ", " + std::to_string(sep_j) + ") between blocks " +
                                    std::to_string(part[sep_i]) + " and " + std::to_string(part[sep_j]));

  return NSP_OK;
}

nsp_status nsp_setup_impl(nsp_ctx* c, const nsp_csr* A, const int32_t* part, int K, nsp_report* rep) {
  auto t0 = Clock::now();
  const int64_t n = A->n;
  const int64_t* rp = A->rowptr;
  const int32_t* ci = A->colidx;
  const double* va = A->val;
  if (n <= 0 || !rp || !ci || !va) return fail(c, NSP_ERR_ARG, "nsp_setup: empty or null CSR");
  if (rp[0] != 0) return fail(c, NSP_ERR_ARG, "nsp_setup: rowptr[0] != 0");
  c->n = n;
  c->K = K;
  // ---------------- shard plan + DBBD index maps (local blocks [B0, B0 + KL), local Gamma rows =
  // private then shared)
  ShardPlan plan;
  {
    std::string perr;
    if (!make_shard_plan(A, part, K, c->nranks, c->rank, plan, perr)) return fail(c, NSP_ERR_ARG, perr);
  }
  const int B0 = plan.blk0, KL = plan.nblk;
  std::vector<int32_t> gpos(n, -1), lpos(n, -1), bidx(n, -1);
  std::vector<std::vector<int64_t>> blocks(KL);
  c->gamma = plan.priv;
  c->gamma.insert(c->gamma.end(), plan.shared.begin(), plan.shared.end());
  for (size_t g = 0; g < c->gamma.size(); ++g) gpos[c->gamma[g]] = (int32_t)g;
  int64_t nG_global = 0;
  for (int64_t i = 0; i < n; ++i) {
    if (part[i] < 0) ++nG_global;
    else if (part[i] >= B0 && part[i] < B0 + KL) blocks[part[i] - B0].push_back(i);
  }
  c->nG = (int64_t)c->gamma.size();
  c->nG_global = nG_global;
  {   // global Gamma index (position in ascending original id) of every local row: the row index of a
      // device-generated Omega (nsp_nystrom with Omega == NULL; reading C7)
    std::vector<int64_t> gall;
    gall.reserve((size_t)nG_global);
    for (int64_t i = 0; i < n; ++i)
      if (part[i] < 0) gall.push_back(i);
    c->gamma_gidx.resize(c->gamma.size());
    for (size_t g = 0; g < c->gamma.size(); ++g)
      c->gamma_gidx[g] = std::lower_bound(gall.begin(), gall.end(), c->gamma[g]) - gall.begin();
  }
  c->n_priv = (int64_t)plan.priv.size();
  c->blk0 = B0;
  c->nsub = KL;
  std::vector<SubHost> sh(KL);
  c->sub_n.resize(KL);
  for (int j = 0; j < KL; ++j) c->sub_n[j] = (int64_t)blocks[j].size();

  // ---------------- per-block ordering (I1 band order, B last)
#pragma omp parallel for schedule(dynamic, 1)
  for (int j = 0; j < KL; ++j) {
    SubHost& S = sh[j];
    S.j = B0 + j;
    const auto& nodes = blocks[j];
    const int nj = (int)nodes.size();
    std::vector<int64_t> I1, Bn;
    for (int64_t v : nodes) {
      bool bl = false;
      for (int64_t q = rp[v]; q < rp[v + 1]; ++q)
        if (part[ci[q]] < 0 && va[q] != 0.0) {
          bl = true;
          break;
        }
      (bl ? Bn : I1).push_back(v);
    }
    S.n1 = (int)I1.size();
    S.b = (int)Bn.size();
    // local index of I1 nodes (natural order)
    for (int k = 0; k < S.n1; ++k) lpos[I1[k]] = k;
    std::vector<int> arp(S.n1 + 1, 0), aci;
    for (int k = 0; k < S.n1; ++k) {
      const int64_t v = I1[k];
      for (int64_t q = rp[v]; q < rp[v + 1]; ++q) {
        const int64_t u = ci[q];
        if (u != v && part[u] == S.j && lpos[u] >= 0 && va[q] != 0.0) {
          // u in I1? (B nodes have lpos -1 at this point)
          aci.push_back(lpos[u]);
        }
      }
      arp[k + 1] = (int)aci.size();
    }
    std::vector<int> pos_nat(S.n1);
    std::iota(pos_nat.begin(), pos_nat.end(), 0);
    const int bw_nat = bandwidth(S.n1, arp, aci, pos_nat);
    std::vector<int> ord = rcm_order(S.n1, arp, aci);
    std::vector<int> pos_rcm(S.n1);
    for (int k = 0; k < S.n1; ++k) pos_rcm[ord[k]] = k;
    const int bw_rcm = bandwidth(S.n1, arp, aci, pos_rcm);
    S.rcm = bw_rcm < bw_nat;
    const std::vector<int>& pos = S.rcm ? pos_rcm : pos_nat;
    S.bw = S.rcm ? bw_rcm : bw_nat;
    S.nodes.assign(nj, -1);
    for (int k = 0; k < S.n1; ++k) S.nodes[pos[k]] = I1[k];
    for (int k = 0; k < S.n1; ++k) lpos[S.nodes[k]] = k;  // final I1 positions
    // B order: by first I1 coupling position, then original id
    std::vector<std::pair<int, int64_t>> bkey(S.b);
    for (int k = 0; k < S.b; ++k) {
      const int64_t v = Bn[k];
      int first = S.n1;
      for (int64_t q = rp[v]; q < rp[v + 1]; ++q) {
        const int64_t u = ci[q];
        if (part[u] == S.j && lpos[u] >= 0 && va[q] != 0.0) first = std::min(first, lpos[u]);
      }
      bkey[k] = {first, v};
    }
    std::sort(bkey.begin(), bkey.end());
    S.nt1 = (S.n1 + NSP_TILE - 1) / NSP_TILE;
    S.ntb = (S.b + NSP_TILE - 1) / NSP_TILE;
    S.wb = S.nt1 > 0 ? std::min(S.nt1 - 1, (S.bw + NSP_TILE - 1) / NSP_TILE) : 0;
    S.border_first.assign(S.ntb, S.nt1);
    for (int k = 0; k < S.b; ++k) {
      S.nodes[S.n1 + k] = bkey[k].second;
      lpos[bkey[k].second] = S.nt1 * NSP_TILE + k;  // padded local index
      bidx[bkey[k].second] = k;
      const int ft = bkey[k].first < S.n1 ? bkey[k].first / NSP_TILE : S.nt1;
      S.border_first[k / NSP_TILE] = std::min(S.border_first[k / NSP_TILE], ft);
    }
  }

  // ---------------- offsets, scratch batches
  c->subs.resize(KL);
  int64_t band_tiles = 0, dense_tiles = 0, wvu_rows = 0;
  std::vector<int> border_first_all;
  c->max_ntb = 0;
  c->n_I = 0;
  c->n_bl = 0;
  c->max_b = 0;
  for (int j = 0; j < KL; ++j) {
    const SubHost& S = sh[j];
    FacSub& F = c->subs[j];
    F.nt1 = S.nt1;
    F.ntb = S.ntb;
    F.wb = S.wb;
    F.pad_ = 0;
    F.n1 = S.n1;
    F.b = S.b;
    F.band_off = band_tiles;
    F.dense_off = dense_tiles;
    F.wvu_row = wvu_rows;
    F.border_first_off = (int)border_first_all.size();
    F.status_idx = j;
    F.border_off = -1;
    border_first_all.insert(border_first_all.end(), S.border_first.begin(), S.border_first.end());
    band_tiles += (int64_t)S.nt1 * (S.wb + 1);
    dense_tiles += (int64_t)S.ntb * (S.ntb + 1) / 2;
    wvu_rows += (int64_t)S.ntb * NSP_TILE;
    c->max_ntb = std::max(c->max_ntb, S.ntb);
    c->n_I += S.n1 + S.b;
    c->n_bl += S.b;
    c->max_b = std::max<int64_t>(c->max_b, S.b);
    c->sum_b2 += (int64_t)S.b * S.b;
    c->sum_b += S.b;
  }
  c->band_tiles = band_tiles;
  c->dense_tiles = dense_tiles;
  c->wvu_rows = wvu_rows;
  size_t free_b = 0, total_b = 0;
  NSP_CUDA_TRY(c, cudaMemGetInfo(&free_b, &total_b));
  const size_t persist = (size_t)(band_tiles + dense_tiles) * NSP_TILE_ELEMS * 8;
  if (persist > free_b) return fail(c, NSP_ERR_OOM, "nsp_setup: factor storage exceeds free device memory");
  size_t budget = c->opts.scratch_bytes;
  if (budget == 0) budget = (size_t)((free_b - persist) * 0.5);
  std::vector<std::pair<int, int>> batches;  // [j0, j1)
  {
    int j0 = 0;
    int64_t acc = 0;
    for (int j = 0; j < KL; ++j) {
      const int64_t t = (int64_t)sh[j].ntb * sh[j].nt1;
      if (j > j0 && (size_t)(acc + t) * NSP_TILE_ELEMS * 8 > budget) {
        batches.push_back({j0, j});
        j0 = j;
        acc = 0;
      }
      c->subs[j].border_off = acc;
      acc += t;
    }
    batches.push_back({j0, KL});
  }
  int64_t max_batch_tiles = 0;
  for (auto& bt : batches) {
    int64_t acc = 0;
    for (int j = bt.first; j < bt.second; ++j) acc += (int64_t)sh[j].ntb * sh[j].nt1;
    max_batch_tiles = std::max(max_batch_tiles, acc);
  }
  if ((size_t)max_batch_tiles * NSP_TILE_ELEMS * 8 > free_b - persist)
    return fail(c, NSP_ERR_OOM, "nsp_setup: a single block's border scratch exceeds free device memory");

  // ---------------- tile entries (lower triangle of A_I_j in the new ordering)
#pragma omp parallel for schedule(dynamic, 1)
  for (int j = 0; j < KL; ++j) {
    SubHost& S = sh[j];
    const FacSub& F = c->subs[j];
    const int nj = (int)S.nodes.size();
    const int off1 = S.nt1 * NSP_TILE;
    for (int k = 0; k < nj; ++k) {
      const int64_t v = S.nodes[k];
      const int li = lpos[v];
      for (int64_t q = rp[v]; q < rp[v + 1]; ++q) {
        const int64_t u = ci[q];
        if (part[u] != B0 + j) continue;
        const int lj = lpos[u];
        if (lj > li) continue;
        const double a = va[q];
        if (li < off1) {  // I1 x I1 -> band
          const int I = li / NSP_TILE, Kt = lj / NSP_TILE;
          S.band_idx.push_back((F.band_off + (int64_t)Kt * (S.wb + 1) + (I - Kt)) * NSP_TILE_ELEMS +
                               (li % NSP_TILE) * NSP_TILE + lj % NSP_TILE);
          S.band_val.push_back(a);
        } else if (lj < off1) {  // B x I1 -> border scratch (batch relative)
          const int bi = li - off1;
          const int Ib = bi / NSP_TILE, Kt = lj / NSP_TILE;
          S.border_idx.push_back((F.border_off + (int64_t)Ib * S.nt1 + Kt) * NSP_TILE_ELEMS +
                                 (bi % NSP_TILE) * NSP_TILE + lj % NSP_TILE);
          S.border_val.push_back(a);
        } else {  // B x B -> dense
          const int bi = li - off1, bj = lj - off1;
          const int Ib = bi / NSP_TILE, Jb = bj / NSP_TILE;
          S.dense_idx.push_back((F.dense_off + (int64_t)Ib * (Ib + 1) / 2 + Jb) * NSP_TILE_ELEMS +
                                (bi % NSP_TILE) * NSP_TILE + bj % NSP_TILE);
          S.dense_val.push_back(a);
        }
      }
    }
  }

  // ---------------- Gamma-side CSRs
  HostCSR32 A2G, AGG2;
  A2G.rowptr.assign(wvu_rows + 1, 0);
  {
    // rows of W/V/U: block j, border k -> row wvu_row + k; padded rows empty
    std::vector<int64_t> rowsrc(wvu_rows, -1);
    for (int j = 0; j < KL; ++j)
      for (int k = 0; k < sh[j].b; ++k) rowsrc[c->subs[j].wvu_row + k] = sh[j].nodes[sh[j].n1 + k];
    std::vector<std::pair<int32_t, double>> ent;
    for (int64_t r = 0; r < wvu_rows; ++r) {
      const int64_t v = rowsrc[r];
      if (v >= 0) {
        ent.clear();
        for (int64_t q = rp[v]; q < rp[v + 1]; ++q)
          if (part[ci[q]] < 0 && va[q] != 0.0) {
            if (gpos[ci[q]] < 0) return fail(c, NSP_ERR_ARG, "nsp_setup: shard plan misses a Gamma neighbour");
            ent.push_back({gpos[ci[q]], va[q]});
          }
        std::sort(ent.begin(), ent.end());
        for (auto& e : ent) {
          A2G.col.push_back(e.first);
          A2G.val.push_back(e.second);
        }
      }
      A2G.rowptr[r + 1] = (int32_t)A2G.col.size();
    }
  }
  // AGG2: private rows hold every entry; shared rows hold this rank's PARTIAL (A_G entries to its
  // private rows, -A_GI entries to its own blocks); the shared x shared part of A_G goes to AGSH,
  // applied after the allreduce of the partials (identically on every rank).
  AGG2.rowptr.assign(c->nG + 1, 0);
  HostCSR32 AGSH;
  const int64_t nsh = c->nG - c->n_priv;
  AGSH.rowptr.assign(nsh + 1, 0);
  c->nnz_AG = 0;
  c->nnz_AGI = 0;
  {
    std::vector<std::pair<int64_t, double>> ent, esh;
    for (int64_t g = 0; g < c->nG; ++g) {
      const int64_t v = c->gamma[g];
      const bool shared_row = g >= c->n_priv;
      ent.clear();
      esh.clear();
      for (int64_t q = rp[v]; q < rp[v + 1]; ++q) {
        const int64_t u = ci[q];
        if (va[q] == 0.0 && u != v) continue;
        if (part[u] < 0) {
          if (gpos[u] < 0) continue;                            // private row of another rank
          if (shared_row && gpos[u] >= c->n_priv) {
            esh.push_back({gpos[u] - c->n_priv, va[q]});
          } else {
            ent.push_back({gpos[u], va[q]});
          }
          c->nnz_AG++;
        } else {
          if (part[u] < B0 || part[u] >= B0 + KL) continue;     // block of another rank
          ent.push_back({c->nG + c->subs[part[u] - B0].wvu_row + bidx[u], -va[q]});
          c->nnz_AGI++;
        }
      }
      if (shared_row) {
        std::sort(esh.begin(), esh.end());
        for (auto& e : esh) {
          AGSH.col.push_back((int32_t)e.first);
          AGSH.val.push_back(e.second);
        }
        AGSH.rowptr[g - c->n_priv + 1] = (int32_t)AGSH.col.size();
      }
      std::sort(ent.begin(), ent.end());
      for (auto& e : ent) {
        if (e.first > INT32_MAX) return fail(c, NSP_ERR_ARG, "nsp_setup: W/V/U index exceeds int32");
        AGG2.col.push_back((int32_t)e.first);
        AGG2.val.push_back(e.second);
      }
      AGG2.rowptr[g + 1] = (int32_t)AGG2.col.size();
    }
  }
  // ---------------- full-system solve maps (nsp_pcg): band rows, original-id maps, [I | -A_B1], [I | -A_1B]
  std::vector<int64_t> i1_row0(KL);
  int64_t i1_rows = 0;
  for (int j = 0; j < KL; ++j) {
    i1_row0[j] = i1_rows;
    i1_rows += (int64_t)sh[j].nt1 * NSP_TILE;
  }
  if (i1_rows + wvu_rows > INT32_MAX) return fail(c, NSP_ERR_ARG, "nsp_setup: interior rows exceed int32");
  c->i1_rows = i1_rows;
  c->i1_wbmax = 0;
  for (int j = 0; j < KL; ++j) c->i1_wbmax = std::max(c->i1_wbmax, sh[j].wb);
  std::vector<int32_t> i1_src(i1_rows, -1), b_src(wvu_rows, -1), g_src(c->nG);
  for (int64_t g = 0; g < c->nG; ++g) g_src[g] = (int32_t)c->gamma[g];
  HostCSR32 CB, C1;
  CB.rowptr.assign(wvu_rows + 1, 0);
  C1.rowptr.assign(i1_rows + 1, 0);
  {
    std::vector<int32_t> cnt_b(wvu_rows, 0), cnt_1(i1_rows, 0);
    for (int j = 0; j < KL; ++j) {
      const SubHost& S = sh[j];
      for (int k = 0; k < S.n1; ++k) i1_src[i1_row0[j] + k] = (int32_t)S.nodes[k];
      for (int k = 0; k < S.b; ++k) b_src[c->subs[j].wvu_row + k] = (int32_t)S.nodes[S.n1 + k];
    }
    // row r of CB: identity then -A_B1 (band columns ascending); row of C1: identity then -A_1B
    auto row_entries = [&](int64_t v, int j, bool from_b, std::vector<std::pair<int32_t, double>>& ent) {
      ent.clear();
      for (int64_t q = rp[v]; q < rp[v + 1]; ++q) {
        const int64_t u = ci[q];
        if (part[u] != B0 + j || u == v || va[q] == 0.0) continue;
        const bool u_b = bidx[u] >= 0;
        if (from_b && !u_b) ent.push_back({(int32_t)(wvu_rows + i1_row0[j] + lpos[u]), -va[q]});
        if (!from_b && u_b) ent.push_back({(int32_t)(i1_rows + c->subs[j].wvu_row + bidx[u]), -va[q]});
      }
      std::sort(ent.begin(), ent.end());
    };
    std::vector<std::pair<int32_t, double>> ent;
    for (int64_t r = 0; r < wvu_rows; ++r) {
      if (b_src[r] >= 0) {
        const int64_t v = b_src[r];
        CB.col.push_back((int32_t)r);
        CB.val.push_back(1.0);
        row_entries(v, part[v] - B0, true, ent);
        for (auto& e : ent) {
          CB.col.push_back(e.first);
          CB.val.push_back(e.second);
        }
      }
      CB.rowptr[r + 1] = (int32_t)CB.col.size();
    }
    for (int64_t r = 0; r < i1_rows; ++r) {
      if (i1_src[r] >= 0) {
        const int64_t v = i1_src[r];
        C1.col.push_back((int32_t)r);
        C1.val.push_back(1.0);
        row_entries(v, part[v] - B0, false, ent);
        for (auto& e : ent) {
          C1.col.push_back(e.first);
          C1.val.push_back(e.second);
        }
      }
      C1.rowptr[r + 1] = (int32_t)C1.col.size();
    }
  }
  // ---------------- A_I on the interior layout (band rows, then W/V/U rows) for the paper-literal
  // S_I inner system (opts.nys_form == 1): every B row carries one extra entry (n_int + row, -1)
  // so that "A_I P - [0; h_B]" is a single SpMM pass
  HostCSR32 AII;
  if ((c->opts.nys_form == 1 || c->opts.nys_form == 2) && c->nranks == 1) {
    const int64_t n_int = i1_rows + wvu_rows;
    if (n_int + wvu_rows > INT32_MAX) return fail(c, NSP_ERR_ARG, "nsp_setup: interior rows exceed int32");
    auto iidx = [&](int64_t u, int jl) -> int32_t {
      return bidx[u] >= 0 ? (int32_t)(i1_rows + c->subs[jl].wvu_row + bidx[u]) : (int32_t)(i1_row0[jl] + lpos[u]);
    };
    AII.rowptr.assign(n_int + 1, 0);
    std::vector<std::pair<int32_t, double>> ent;
    for (int64_t r = 0; r < n_int; ++r) {
      const bool isb = r >= i1_rows;
      const int64_t v = isb ? b_src[r - i1_rows] : i1_src[r];
      if (v >= 0) {
        const int jl = part[v] - B0;
        ent.clear();
        for (int64_t q = rp[v]; q < rp[v + 1]; ++q) {
          const int64_t u = ci[q];
          if (part[u] != part[v] || (va[q] == 0.0 && u != v)) continue;
          ent.push_back({iidx(u, jl), va[q]});
        }
        std::sort(ent.begin(), ent.end());
        for (auto& e : ent) {
          AII.col.push_back(e.first);
          AII.val.push_back(e.second);
        }
        if (isb) {
          AII.col.push_back((int32_t)(n_int + (r - i1_rows)));
          AII.val.push_back(-1.0);
        }
      }
      AII.rowptr[r + 1] = (int32_t)AII.col.size();
    }
  }
  const double t_host = ms_since(t0);

  // ---------------- device upload
  auto t1 = Clock::now();
  nsp_status st;
  if ((st = upload_csr(c, c->A2G, A2G)) != NSP_OK) return st;
  if ((st = upload_csr(c, c->AGG2, AGG2)) != NSP_OK) return st;
  if ((st = upload_csr(c, c->AGSH, AGSH)) != NSP_OK) return st;
  if (c->nranks == 1 && c->opts.factor_gamma) {   // A_G alone for the Chebyshev steps (rows are col-sorted)
    HostCSR32 AGO;
    AGO.rowptr.assign(c->nG + 1, 0);
    for (int64_t g = 0; g < c->nG; ++g) {
      for (int32_t q = AGG2.rowptr[g]; q < AGG2.rowptr[g + 1] && AGG2.col[q] < c->nG; ++q) {
        AGO.col.push_back(AGG2.col[q]);
        AGO.val.push_back(AGG2.val[q]);
      }
      AGO.rowptr[g + 1] = (int32_t)AGO.col.size();
    }
    if ((st = upload_csr(c, c->AGO, AGO)) != NSP_OK) return st;
    // sliced ELL copy (32-row slices, column-major inside a slice)
    const int64_t nsl = (c->nG + 31) / 32;
    std::vector<int64_t> sptr(nsl + 1, 0);
    for (int64_t q = 0; q < nsl; ++q) {
      int w = 0;
      for (int64_t g = q * 32; g < std::min<int64_t>(c->nG, q * 32 + 32); ++g)
        w = std::max(w, AGO.rowptr[g + 1] - AGO.rowptr[g]);
      sptr[q + 1] = sptr[q] + (int64_t)w * 32;
    }
    std::vector<int32_t> scol(sptr[nsl], -1);
    std::vector<double> sval(sptr[nsl], 0.0);
    for (int64_t g = 0; g < c->nG; ++g) {
      const int64_t q = g / 32, lane = g % 32;
      for (int32_t k = AGO.rowptr[g]; k < AGO.rowptr[g + 1]; ++k) {
        const int64_t e = sptr[q] + (int64_t)(k - AGO.rowptr[g]) * 32 + lane;
        scol[e] = AGO.col[k];
        sval[e] = AGO.val[k];
      }
    }
    if ((st = upload(c, &c->d_sell_ptr, sptr)) != NSP_OK) return st;
    if ((st = upload(c, &c->d_sell_col, scol)) != NSP_OK) return st;
    if ((st = upload(c, &c->d_sell_val, sval)) != NSP_OK) return st;
    {   // dictionary coding of the values when A_G has at most 255 distinct ones (code 255: padding)
      std::vector<double> tab;
      std::vector<uint8_t> code(sval.size(), 255);
      bool ok = true;
      for (size_t e = 0; e < sval.size() && ok; ++e) {
        if (scol[e] < 0) continue;
        size_t t = 0;
        while (t < tab.size() && std::memcmp(&tab[t], &sval[e], sizeof(double)) != 0) ++t;   // bitwise
        if (t == tab.size()) {
          if (tab.size() == 255) ok = false;
          else tab.push_back(sval[e]);
        }
        code[e] = (uint8_t)t;
      }
      const char* de = getenv("NSP_SELL_DICT");
      if (ok && !(de && de[0] == '0')) {
        tab.resize(256, 0.0);
        if ((st = upload(c, &c->d_sell_code, code)) != NSP_OK) return st;
        if ((st = upload(c, &c->d_sell_tab, tab)) != NSP_OK) return st;
      }
    }
  }
  if ((st = upload_csr(c, c->CB, CB)) != NSP_OK) return st;
  if (!AII.rowptr.empty()) {
    if ((st = upload_csr(c, c->AII, AII)) != NSP_OK) return st;
    std::vector<int32_t> isrc(i1_src);   // interior layout row -> original id (-1 padding)
    isrc.insert(isrc.end(), b_src.begin(), b_src.end());
    if ((st = upload(c, &c->d_int_src, isrc)) != NSP_OK) return st;
  }
  if ((st = upload_csr(c, c->C1, C1)) != NSP_OK) return st;
  if ((st = upload(c, &c->d_i1_src, i1_src)) != NSP_OK) return st;
  if ((st = upload(c, &c->d_b_src, b_src)) != NSP_OK) return st;
  if ((st = upload(c, &c->d_g_src, g_src)) != NSP_OK) return st;
  if ((st = upload(c, &c->d_subs, c->subs)) != NSP_OK) return st;
  std::vector<int> bf = border_first_all;
  if (bf.empty()) bf.push_back(0);
  if ((st = upload(c, &c->d_border_first, bf)) != NSP_OK) return st;
  if (band_tiles > 0) {
    NSP_CUDA_TRY(c, cudaMalloc((void**)&c->d_band, (size_t)band_tiles * NSP_TILE_ELEMS * 8));
    NSP_CUDA_TRY(c, cudaMemsetAsync(c->d_band, 0, (size_t)band_tiles * NSP_TILE_ELEMS * 8, c->stream));
  }
  {
    std::vector<TriSys> ts(KL);
    for (int j = 0; j < KL; ++j)
      ts[j] = TriSys{c->d_band ? c->d_band + c->subs[j].band_off * NSP_TILE_ELEMS : nullptr, sh[j].nt1, sh[j].wb,
                     i1_row0[j]};
    if ((st = upload(c, &c->d_i1sys, ts)) != NSP_OK) return st;
  }
  if (dense_tiles > 0) {
    NSP_CUDA_TRY(c, cudaMalloc((void**)&c->d_dense, (size_t)dense_tiles * NSP_TILE_ELEMS * 8));
    NSP_CUDA_TRY(c, cudaMemsetAsync(c->d_dense, 0, (size_t)dense_tiles * NSP_TILE_ELEMS * 8, c->stream));
  }
  // entries: upload in chunks through one staging pair
  const int64_t CH = 1 << 24;
  int64_t* d_idx = nullptr;
  double* d_val = nullptr;
  NSP_CUDA_TRY(c, cudaMalloc((void**)&d_idx, CH * 8));
  NSP_CUDA_TRY(c, cudaMalloc((void**)&d_val, CH * 8));
  std::vector<int64_t> hidx;
  std::vector<double> hval;
  auto flush_entries = [&](double* base) -> nsp_status {
    for (int64_t s0 = 0; s0 < (int64_t)hidx.size(); s0 += CH) {
      const int64_t cnt = std::min<int64_t>(CH, (int64_t)hidx.size() - s0);
      NSP_CUDA_TRY(c, cudaMemcpyAsync(d_idx, hidx.data() + s0, cnt * 8, cudaMemcpyHostToDevice, c->stream));
      NSP_CUDA_TRY(c, cudaMemcpyAsync(d_val, hval.data() + s0, cnt * 8, cudaMemcpyHostToDevice, c->stream));
      nspk::scatter(base, d_idx, d_val, cnt, c->stream);
      NSP_CUDA_TRY(c, cudaStreamSynchronize(c->stream));
    }
    hidx.clear();
    hval.clear();
    return NSP_OK;
  };
  for (int j = 0; j < KL; ++j) {
    hidx.insert(hidx.end(), sh[j].band_idx.begin(), sh[j].band_idx.end());
    hval.insert(hval.end(), sh[j].band_val.begin(), sh[j].band_val.end());
    std::vector<int64_t>().swap(sh[j].band_idx);
    std::vector<double>().swap(sh[j].band_val);
  }
  if ((st = flush_entries(c->d_band)) != NSP_OK) return st;
  for (int j = 0; j < KL; ++j) {
    hidx.insert(hidx.end(), sh[j].dense_idx.begin(), sh[j].dense_idx.end());
    hval.insert(hval.end(), sh[j].dense_val.begin(), sh[j].dense_val.end());
    std::vector<int64_t>().swap(sh[j].dense_idx);
    std::vector<double>().swap(sh[j].dense_val);
  }
  if ((st = flush_entries(c->d_dense)) != NSP_OK) return st;
  // identity on padded diagonal rows
  {
    std::vector<int64_t> bt, dt;
    std::vector<int> bfr, dfr;
    for (int j = 0; j < KL; ++j) {
      const SubHost& S = sh[j];
      if (S.nt1 > 0 && S.n1 % NSP_TILE) {
        bt.push_back(c->subs[j].band_off + (int64_t)(S.nt1 - 1) * (S.wb + 1));
        bfr.push_back(S.n1 % NSP_TILE);
      }
      if (S.ntb > 0 && S.b % NSP_TILE) {
        const int I = S.ntb - 1;
        dt.push_back(c->subs[j].dense_off + (int64_t)I * (I + 1) / 2 + I);
        dfr.push_back(S.b % NSP_TILE);
      }
    }
    int64_t* d_t = nullptr;
    int* d_f = nullptr;
    if (!bt.empty()) {
      if ((st = upload(c, &d_t, bt)) != NSP_OK) return st;
      if ((st = upload(c, &d_f, bfr)) != NSP_OK) return st;
      nspk::set_pad_identity(c->d_band, d_t, d_f, (int)bt.size(), c->stream);
      NSP_CUDA_TRY(c, cudaStreamSynchronize(c->stream));
      cudaFree(d_t);
      cudaFree(d_f);
    }
    if (!dt.empty()) {
      if ((st = upload(c, &d_t, dt)) != NSP_OK) return st;
      if ((st = upload(c, &d_f, dfr)) != NSP_OK) return st;
      nspk::set_pad_identity(c->d_dense, d_t, d_f, (int)dt.size(), c->stream);
      NSP_CUDA_TRY(c, cudaStreamSynchronize(c->stream));
      cudaFree(d_t);
      cudaFree(d_f);
    }
  }
  const double t_h2d = ms_since(t1);

  // ---------------- GPU factorisation, batch by batch
  auto t2 = Clock::now();
  double* d_scratch = nullptr;
  if (max_batch_tiles > 0)
    NSP_CUDA_TRY(c, cudaMalloc((void**)&d_scratch, (size_t)max_batch_tiles * NSP_TILE_ELEMS * 8));
  int* d_status = nullptr;
  NSP_CUDA_TRY(c, cudaMalloc((void**)&d_status, KL * sizeof(int)));
  NSP_CUDA_TRY(c, cudaMemsetAsync(d_status, 0, KL * sizeof(int), c->stream));
  for (auto& bt : batches) {
    int64_t tiles = 0;
    for (int j = bt.first; j < bt.second; ++j) {
      tiles += (int64_t)sh[j].ntb * sh[j].nt1;
      hidx.insert(hidx.end(), sh[j].border_idx.begin(), sh[j].border_idx.end());
      hval.insert(hval.end(), sh[j].border_val.begin(), sh[j].border_val.end());
      std::vector<int64_t>().swap(sh[j].border_idx);
      std::vector<double>().swap(sh[j].border_val);
    }
    if (tiles > 0) NSP_CUDA_TRY(c, cudaMemsetAsync(d_scratch, 0, (size_t)tiles * NSP_TILE_ELEMS * 8, c->stream));
    if ((st = flush_entries(d_scratch)) != NSP_OK) return st;
    nspk::tile_cholesky(c->d_subs + bt.first, bt.second - bt.first, c->d_band, c->d_dense, d_scratch,
                        c->d_border_first, d_status, c->stream);
    NSP_CUDA_TRY(c, cudaGetLastError());
  }
  NSP_CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  std::vector<int> hstat(KL);
  NSP_CUDA_TRY(c, cudaMemcpy(hstat.data(), d_status, KL * sizeof(int), cudaMemcpyDeviceToHost));
  cudaFree(d_status);
  cudaFree(d_scratch);
  cudaFree(d_idx);
  cudaFree(d_val);
  const double t_fac = ms_since(t2);
  for (int j = 0; j < KL; ++j)
    if (hstat[j] != 0) {
      const int lrow = hstat[j] - 1;
      const SubHost& S = sh[j];
      int64_t orig = -1;
      if (lrow < S.n1) orig = S.nodes[lrow];
      else if (lrow >= S.nt1 * NSP_TILE && lrow - S.nt1 * NSP_TILE < S.b) orig = S.nodes[S.n1 + lrow - S.nt1 * NSP_TILE];
      if (rep) {
        rep->bad_block = B0 + j;
        rep->bad_pivot = orig;
        rep->status = NSP_ERR_NOT_SPD;
      }
      return fail(c, NSP_ERR_NOT_SPD, "nsp_setup: A_I_" + std::to_string(j) + " not SPD (pivot at node " +
                                          std::to_string(orig) + ")");
    }
  // ---------------- explicit S_j^{-1} tiles for the one-product a2+a3 (opts.apply_kernel == 0)
  if (c->opts.apply_kernel != 1 && dense_tiles > 0) {
    const size_t bytes = (size_t)dense_tiles * NSP_MINV_TILE * 8;
    size_t fr = 0, tot = 0;
    NSP_CUDA_TRY(c, cudaMemGetInfo(&fr, &tot));
    if (bytes < fr / 2) {   // otherwise stay with the L22 sweeps (apply_kernel 1)
      NSP_CUDA_TRY(c, cudaMalloc((void**)&c->d_minv, bytes));
      nspk::l22_inverse(c->d_subs, c->nsub, c->max_ntb, c->d_dense, c->d_minv, c->stream);
      NSP_CUDA_TRY(c, cudaGetLastError());
      // several ranks: the blocks coupled to a SHARED Gamma row first (their U feeds the shared-row
      // partials, so the shared-row allreduce can start while the other blocks' products run)
      std::vector<char> blk_sh(KL, 0);
      if (c->nranks > 1)
        for (int j = 0; j < KL; ++j)
          for (int64_t r = c->subs[j].wvu_row; r < c->subs[j].wvu_row + sh[j].b && !blk_sh[j]; ++r)
            for (int32_t q = A2G.rowptr[r]; q < A2G.rowptr[r + 1]; ++q)
              if (A2G.col[q] >= c->n_priv) {
                blk_sh[j] = 1;
                break;
              }
      std::vector<int2> items;
      for (int pass = 0; pass < 2; ++pass)
        for (int j = 0; j < KL; ++j)
          if (blk_sh[j] == (pass == 0 ? 1 : 0))
            for (int I = 0; I < sh[j].ntb; ++I) items.push_back(make_int2(j, I));
      c->n_items = (int)items.size();
      c->n_items_sh = 0;
      for (int j = 0; j < KL; ++j)
        if (blk_sh[j]) c->n_items_sh += sh[j].ntb;
      if ((st = upload(c, &c->d_items, items)) != NSP_OK) return st;
      NSP_CUDA_TRY(c, cudaStreamSynchronize(c->stream));
      // the L22 tiles are not read again once S_j^{-1} exists (a2+a3, the full solve's y_B and the S_I
      // forms' block elimination all use S_j^{-1}): release them (cfg5: 42 GB)
      cudaFree(c->d_dense);
      c->d_dense = nullptr;
    }
  }
  const double t_fac_all = ms_since(t2);
  // ---------------- INT8 tensor-core slices of the S_j^{-1} tiles (reading R10; apply_kernel 0 / 3):
  // D-scaled lower tiles as 7 int8 slices each (a quarter of the fp64 tiles' bytes... 7/8 of their
  // lower-triangle bytes); the fp64 tiles stay (s = 1 products, the S_I forms).  Skipped when the
  // device budget does not allow it (a2+a3 then stays on the DMMA k_symm) or when a block is so large
  // that the int32 diagonal sums could overflow (b_j > 300 tiles).
  double t_oz = 0.0;
  {
    const char* oe = getenv("NSP_OZAKI");
    const bool oz_on = !(oe && oe[0] == '0');
    if (c->d_minv && oz_on && (c->opts.apply_kernel == 0 || c->opts.apply_kernel == 3) && c->max_ntb <= 300 &&
        c->n_items > 0) {
      auto t4 = Clock::now();
      const size_t mb = nspk::oz_mslice_bytes(dense_tiles);
      size_t fr = 0, tot = 0;
      NSP_CUDA_TRY(c, cudaMemGetInfo(&fr, &tot));
      const char* re = getenv("NSP_OZ_RESERVE_GB");
      const size_t reserve = (size_t)((re ? atof(re) : 12.0) * 1073741824.0);
      if (mb + reserve < fr) {
        NSP_CUDA_TRY(c, cudaMalloc((void**)&c->d_oz_msl, mb));
        NSP_CUDA_TRY(c, cudaMalloc((void**)&c->d_oz_dexp, (size_t)c->wvu_rows * sizeof(int)));
        NSP_CUDA_TRY(c, cudaMalloc((void**)&c->d_oz_mexp, (size_t)c->nsub * sizeof(int)));
        {
          std::vector<int> tb((size_t)(c->wvu_rows / 64), 0);
          for (int j = 0; j < c->nsub; ++j)
            for (int I = 0; I < c->subs[j].ntb; ++I) tb[(size_t)(c->subs[j].wvu_row / 64 + I)] = j;
          if ((st = upload(c, &c->d_oz_tblk, tb)) != NSP_OK) return st;
          std::vector<int2> pr;
          for (int j = 0; j < c->nsub; ++j)
            for (int I = 0; I < c->subs[j].ntb; I += 2) pr.push_back(make_int2(j, I));
          c->n_oz_pairs = (int)pr.size();
          NSP_CUDA_TRY(c, cudaMalloc((void**)&c->d_oz_ctr, 1024));   // [0]: the counter; [64..69]: NSP_OZ_PROF diagnostics
          if (!pr.empty() && (st = upload(c, &c->d_oz_pairs, pr)) != NSP_OK) return st;
        }
        NSP_CUDA_TRY(c, cudaMalloc((void**)&c->d_oz_mz, (size_t)dense_tiles));
        nspk::oz_setup(c->d_subs, c->nsub, c->max_ntb, c->d_items, c->n_items, c->d_minv, c->d_oz_dexp,
                       c->d_oz_mexp, c->d_oz_msl, c->d_oz_mz, c->stream);
        NSP_CUDA_TRY(c, cudaGetLastError());
        NSP_CUDA_TRY(c, cudaStreamSynchronize(c->stream));
        {   // executed slice products per column tile (k_oz_symm's K loop: natural order, tile K = 0 unskipped,
            // product (i, j) with i + j < 7 dropped when B slice j < mz[t]) - the bench's roofline counts these
          std::vector<int8_t> hz((size_t)dense_tiles);
          NSP_CUDA_TRY(c, cudaMemcpy(hz.data(), c->d_oz_mz, hz.size(), cudaMemcpyDeviceToHost));
          int64_t ex = 0, full = 0, sl = 0;
          for (const FacSub& f : c->subs)
            for (int I = 0; I < f.ntb; ++I)
              for (int K = 0; K < f.ntb; ++K) {
                if (K <= I)   // unique slice bytes: a tile with J = 0 is also read whole (as a unit's first K tile)
                  sl += 4096 * (7 - (K == 0 ? 0 : std::max(0, std::min(7, (int)hz[(size_t)(f.dense_off + (int64_t)I * (I + 1) / 2 + K)]))));
                const int64_t t = f.dense_off + (K <= I ? (int64_t)I * (I + 1) / 2 + K : (int64_t)K * (K + 1) / 2 + I);
                const int z = K == 0 ? 0 : std::max(0, std::min(7, (int)hz[(size_t)t]));
                full += 28;
                ex += 28 - (7 * z - z * (z - 1) / 2);
              }
          c->oz_prod_exec = ex;
          c->oz_prod_full = full;
          c->oz_slice_bytes = sl;
        if (c->opts.verbose || getenv("NSP_VERBOSE")) {   // how many slices the product skips
          long long cnt[8] = {0};
          for (int8_t z : hz) cnt[z < 0 ? 0 : (z > 7 ? 7 : z)]++;
          fprintf(stderr, "[nsp] INT8 slices: stored tiles by leading zero slices 0..6:");
          for (int q = 0; q < 7; ++q) fprintf(stderr, " %lld", cnt[q]);
          fprintf(stderr, "\n");
        }
        }
      } else if (c->opts.verbose) {
        fprintf(stderr, "nsp_setup: INT8 slices (%.1f GB) skipped: %.1f GB free, %.1f GB reserve\n", mb / 1e9,
                fr / 1e9, reserve / 1e9);
      }
      t_oz = ms_since(t4);
    }
  }
  double t_ag = 0.0;
  if (c->opts.factor_gamma) {
    auto t3 = Clock::now();
    nsp_status sg;
    if (c->nranks > 1) {   // sharded: the Chebyshev polynomial of the global A_G, applied on local rows
      std::vector<int64_t> gall;
      gall.reserve((size_t)c->nG_global);
      for (int64_t i = 0; i < A->n; ++i)
        if (part[i] < 0) gall.push_back(i);
      sg = setup_gamma_cheb(c, A, part, gpos, &gall);
    } else {
      sg = c->opts.ag_solver == 2 ? NSP_ERR_OOM : setup_gamma_factor(c, A, part, gpos, rep);
      if (sg == NSP_ERR_OOM && c->opts.ag_solver != 1) {
        (void)cudaGetLastError();
        sg = setup_gamma_cheb(c, A, part, gpos);
        if (sg == NSP_OK) c->err.clear();
      }
    }
    if (sg != NSP_OK) return sg;
    t_ag = ms_since(t3);
  }
  if (rep) {
    rep->status = NSP_OK;
    rep->t_ms[3] = t_ag;
    rep->t_ms[0] = t_host;
    rep->t_ms[1] = t_h2d;
    rep->t_ms[2] = t_fac;
    rep->t_ms[4] = t_fac_all - t_fac;   // S_j^{-1} tiles
    rep->t_ms[5] = t_oz;                // their INT8 slices
  }
  NSP_CUDA_TRY(c, cudaMallocHost(&c->h_status, 4096));
  return NSP_OK;
}
