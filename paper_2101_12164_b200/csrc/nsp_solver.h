// Solver-side internals shared by nsp_api.cpp and nsp_solver.cu.
#pragma once
#include "nsp_internal.h"

namespace nspi {
int pick_cw(const nsp_ctx* c, int s);
int ld_pad(int s, int cw);
size_t apply_ws_bytes(const nsp_ctx* c, int s);
bool use_ozaki(const nsp_ctx* c, int s);
nsp_status get_ws(nsp_ctx* c, void* ws, size_t need, char** out);
nsp_status finish_shared_rows(nsp_ctx* c, const double* X, int ldx, double* Y, int ldy, int s, bool ag_term);
nsp_status apply_into(nsp_ctx* c, const double* X, int ldx, double* Y, int ldy, int s, int mode, double* wvu);
size_t solver_ws_bytes(const nsp_ctx* c, int s);
void solver_free(nsp_ctx* c);
}  // namespace nspi

namespace nspi {
size_t ag_ws_doubles(const nsp_ctx* c, int s);
// Y = A_G^{-1} X (band factor of A_G; eq:S1), buf: ag_ws_doubles(c, s) doubles
nsp_status ag_solve(nsp_ctx* c, const double* X, int ldx, double* Y, int ldy, int s, double* buf);
nsp_status ag_tri(nsp_ctx* c, const double* X, int ldx, bool x_gamma, double* Y, int ldy, bool y_gamma, int s,
                  bool fwd, bool bwd, double* buf);
// M_A-DEF2 (reading R5): E = Z^T S_G Z and its Cholesky factor for the current Nystrom basis, formed once
// on first use (one S_G block apply on Z); sets adef_ok
nsp_status adef_prepare(nsp_ctx* c);
}  // namespace nspi
