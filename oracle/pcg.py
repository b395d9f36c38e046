"""Outer PCG on the border system S_G w = f (PAPER.md:415-420 eq:Sx=b) with a
preconditioner (M_2, A_G^{-1} or none), and the full solve of A x = b through
the block LDL^T factorisation (PAPER.md:381-385 eq:A_LDLT):

    f   = b_G - A_GI A_I^{-1} b_I
    w   = PCG(S_G, f, M)
    x_I = A_I^{-1} (b_I - A_IG w),   x_G = w,   then un-permute.

PCG is the textbook preconditioned conjugate gradient (the
method whose error obeys eq:k-th_error_cg), x0 = 0, stopping on the recurrence
residual ||r_k|| / ||f|| <= tol (reading C9).  Iteration count = number of S_G
applications.
"""
from __future__ import annotations

import numpy as np

from .schur import SchurOracle


def pcg(apply_S, f: np.ndarray, tol: float, maxit: int, apply_M=None, record_x=False):
    """Preconditioned CG on S_Gamma w = f (the CG of PAPER.md:37-58 / eq:k-th_error_cg; the paper gives no
    pseudo-code, so textbook PCG, reading C9): x_0 = 0, stop on ||r_k|| / ||f|| <= tol (recurrence residual)."""
    f = np.asarray(f, dtype=np.float64)
    x = np.zeros_like(f)
    r = f.copy()
    fn = np.linalg.norm(f)
    info = {"iters": 0, "relres": [1.0 if fn > 0 else 0.0], "status": 1, "xs": []}
    if fn == 0:
        info["status"] = 0
        return x, info
    z = apply_M(r) if apply_M is not None else r.copy()
    p = z.copy()
    rz = r @ z
    for _ in range(maxit):
        q = apply_S(p)
        pq = p @ q
        if not pq > 0:
            info["status"] = -3
            return x, info
        a = rz / pq
        x = x + a * p
        r = r - a * q
        info["iters"] += 1
        rel = np.linalg.norm(r) / fn
        info["relres"].append(float(rel))
        if record_x:
            info["xs"].append(x.copy())
        if rel <= tol:
            info["status"] = 0
            return x, info
        z = apply_M(r) if apply_M is not None else r.copy()
        rz_new = r @ z
        p = z + (rz_new / rz) * p
        rz = rz_new
    return x, info


def solve_full_system(S: SchurOracle, b: np.ndarray, tol: float, maxit: int, apply_M=None):
    """Full solve A x = b through the block factorisation eq:A_LDLT and eq:Sx=b
    (PAPER.md:415-420): f = b_G - A_GI A_I^{-1} b_I, PCG on S_Gamma w = f, x_I = A_I^{-1}(b_I - A_IG w)."""
    d = S.d
    b = np.asarray(b, dtype=np.float64)
    b_G = b[d.gamma]
    b_I = [b[blk] for blk in d.blocks]
    y_I = S.solve_AI(b_I)
    f = b_G.copy()
    for j in range(d.K):
        f -= S.A_GI(j) @ y_I[j]
    w, info = pcg(S.apply, f, tol, maxit, apply_M)
    x = np.zeros_like(b)
    x[d.gamma] = w
    for j in range(d.K):
        x[d.blocks[j]] = S.solve_AI_block(j, b_I[j] - d.A_IG[j] @ w)
    return x, info
