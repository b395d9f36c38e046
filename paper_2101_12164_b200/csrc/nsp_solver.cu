// Block CG / Nystrom / PCG drivers (placeholder until the solver kernels land).
#include "nsp_solver.h"

namespace nspi {
size_t solver_ws_bytes(const nsp_ctx* c, int s) { return apply_ws_bytes(c, s); }
void solver_free(nsp_ctx*) {}
}  // namespace nspi

extern "C" {
nsp_status nsp_block_cg(nsp_ctx* c, const double*, double*, int, double, int, void*, nsp_report*) {
  if (c) c->err = "nsp_block_cg: not built";
  return NSP_ERR_STATE;
}
nsp_status nsp_nystrom(nsp_ctx* c, int, int, const double*, double, int, void*, nsp_report*) {
  if (c) c->err = "nsp_nystrom: not built";
  return NSP_ERR_STATE;
}
nsp_status nsp_nystrom_sigma(const nsp_ctx*, double*, int*) { return NSP_ERR_STATE; }
nsp_status nsp_precond_apply(nsp_ctx*, int, const double*, double*, int, void*) { return NSP_ERR_STATE; }
nsp_status nsp_pcg(nsp_ctx*, const double*, double*, double, int, int, void*, nsp_report*) { return NSP_ERR_STATE; }
}
