"""Breakdown-free block (P)CG ("breakdown-free block PCG
method [JiL17, Ole80]"; PAPER.md:902-907 one system with k+p right-hand sides).

The paper gives no details of the breakdown-free variant; this follows reading
C3 step by step:

    R0 = B (X0 = 0);  Z0 = M R0;  P0 = orth(Z0)
    loop:  Q = S P;  D = P^T Q;  alpha = D^{-1} P^T R
           X += P alpha;  R -= Q alpha;  iters += 1
           stop if max_j ||R_j|| / ||B_j|| <= tol          (reading C4)
           Z = M R;  beta = -D^{-1} Q^T Z;  P = orth(Z + P beta)

orth(W): Gram G = W^T W; plain Cholesky G = R^T R recording the pivots
d_i = r_ii^2; if every d_i > 0 and min_i d_i > tau * max_i d_i, P = W R^{-1}
(Cholesky-QR); otherwise the eigen fallback G = V L V^T keeps the eigenvalues
l > tau * l_max and P = W V_keep L_keep^{-1/2} (active width s' <= s).
Columns with ||B_j|| = 0 count as converged.  Iteration count = number of S
applications inside the loop.
"""
from __future__ import annotations

import numpy as np

NSP_OK = 0
NSP_NOT_CONVERGED = 1
NSP_ERR_INDEFINITE = -3
NSP_ERR_STAGNATION = -4


def cholesky_pivots(G: np.ndarray):
    """Plain right-looking Cholesky of a small SPD matrix: returns (R upper, pivots, ok)."""
    s = G.shape[0]
    R = np.zeros_like(G)
    piv = np.zeros(s)
    for i in range(s):
        d = G[i, i] - R[:i, i] @ R[:i, i]
        piv[i] = d
        if not d > 0.0:
            return R, piv[: i + 1], False
        R[i, i] = np.sqrt(d)
        R[i, i + 1:] = (G[i, i + 1:] - R[:i, i] @ R[:i, i + 1:]) / R[i, i]
    return R, piv, True


def inner_fp64(A: np.ndarray, B: np.ndarray) -> np.ndarray:
    """Block inner product A^T B in fp64 (BLAS)."""
    return A.T @ B


def inner_extended(A: np.ndarray, B: np.ndarray) -> np.ndarray:
    """Block inner product A^T B accumulated in the host's extended precision (x87 80-bit long double),
    rounded once to fp64 (reading R8: the Gram accuracy the GPU's chunked fixed-order sums reach)."""
    return (A.astype(np.longdouble).T @ B.astype(np.longdouble)).astype(np.float64)


def orth(W: np.ndarray, tau: float = 1e-14, inner=inner_fp64):
    """Rank-revealing orthonormalisation of the direction block (reading C3).
    Returns (P, width, used_fallback)."""
    G = inner(W, W)
    R, piv, ok = cholesky_pivots(G)
    if ok and piv.min() > tau * piv.max():
        # P = W R^{-1}: solve P R = W row by row (R upper triangular)
        P = np.linalg.solve(R.T, W.T).T
        return P, W.shape[1], False
    lam, V = np.linalg.eigh(G)
    if not lam.max() > 0.0:
        return W[:, :0], 0, True
    keep = lam > tau * lam.max()
    P = (W @ V[:, keep]) / np.sqrt(lam[keep])
    return P, int(keep.sum()), True


def bf_bcg(apply_S, B: np.ndarray, tol: float, maxit: int, apply_M=None, tau: float = 1e-14,
           X0=None, inner=inner_fp64):
    """Breakdown-free block (P)CG of the module docstring (reading C3 step by step,
    stopping rule reading C4): returns (X, info) with info = iters, status, relres history, widths.
    inner: the block inner product used for every Gram (P^T Q, P^T R, Q^T Z, W^T W); inner_extended
    accumulates them in extended precision (reading R8)."""
    B = np.asarray(B, dtype=np.float64)
    n, s = B.shape
    X = np.zeros_like(B) if X0 is None else np.array(X0, dtype=np.float64)
    R = B - apply_S(X) if X0 is not None else B.copy()
    bnorm = np.linalg.norm(B, axis=0)
    safe = np.where(bnorm > 0, bnorm, 1.0)

    def relres(R):
        rr = np.linalg.norm(R, axis=0) / safe
        rr[bnorm == 0] = 0.0
        return rr

    info = {"iters": 0, "widths": [], "relres": [float(relres(R).max()) if s else 0.0],
            "fallbacks": 0, "status": NSP_NOT_CONVERGED}
    if s == 0 or relres(R).max() <= tol:
        info["status"] = NSP_OK
        return X, info
    Z = apply_M(R) if apply_M is not None else R
    P, w, fb = orth(Z, tau, inner)
    info["fallbacks"] += int(fb)
    for _ in range(maxit):
        if w == 0:
            info["status"] = NSP_ERR_STAGNATION
            return X, info
        info["widths"].append(w)
        Q = apply_S(P)
        D = inner(P, Q)
        _, _, ok = cholesky_pivots(D)
        if not ok:
            info["status"] = NSP_ERR_INDEFINITE
            return X, info
        alpha = np.linalg.solve(D, inner(P, R))
        X = X + P @ alpha
        R = R - Q @ alpha
        info["iters"] += 1
        rr = relres(R)
        info["relres"].append(float(rr.max()))
        if rr.max() <= tol:
            info["status"] = NSP_OK
            return X, info
        Z = apply_M(R) if apply_M is not None else R
        beta = -np.linalg.solve(D, inner(Q, Z))
        P, w, fb = orth(Z + P @ beta, tau, inner)
        info["fallbacks"] += int(fb)
    return X, info
