"""Nystrom-Schur preconditioner M_2 = A_G^{-1} + Z Sigma Z^T (PAPER.md:965-989,
Alg. 2 "Construction of the Nystrom-Schur preconditioner"; eq:left_prec_mat
PAPER.md:937-943; Alg. 1).

Step by step in the paper's order, with the DESIGN.md readings:
  1  G = Omega (n_G x (k+p) Gaussian, passed in; reading C7)
  2-4 Y = A_GI S_I^{-1} A_IG G, computed through the equivalent border system
     (reading C1, from Woodbury eq:S-1 PAPER.md:807-813):
        B = K_G G;  solve S_G X = B by BF block CG to tol_inner;  Y = A_G X
  5  Y = Q R  (Householder QR, sign-normalised so diag(R) >= 0)
  6  C = G^T Y, symmetrised (C + C^T)/2 (reading C6)
  7  EVD C = V1 D1 V1^T + V2 D2 V2^T, D1 = eigenvalues >= eps = eps_rel * lambda_max(C)
  8  T = R V1 D1^{-1} V1^T R^T (symmetrised)
  9  EVD T = W E W^T, descending
  10 U~ = Q W(:, 1:k), Sigma = E(1:k)   (reading C5: Q, not "YW"; rank = min(r, k))
  11 solve A_G Z = U~
  12 M_2 r = A_G^{-1} r + Z Sigma Z^T r
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import scipy.linalg as sla

from .bcg import bf_bcg
from .schur import SchurOracle

NSP_ERR_RANK_COLLAPSE = -5


@dataclass
class NystromResult:
    Z: np.ndarray          # n_G x r
    sigma: np.ndarray      # r, descending
    U: np.ndarray          # n_G x r (orthonormal)
    rank: int
    bcg: dict
    status: int


def nystrom_from_Y(Omega: np.ndarray, Y: np.ndarray, k: int, eps_rel: float = 1e-12):
    """Alg. 2 steps 5-10 on given (Omega, Y). Returns (U, sigma, r_C)."""
    Q, R = np.linalg.qr(Y)                               # step 5
    sgn = np.where(np.diag(R) < 0, -1.0, 1.0)
    Q, R = Q * sgn, (R.T * sgn).T
    C = Omega.T @ Y                                      # step 6
    C = 0.5 * (C + C.T)
    d, V = np.linalg.eigh(C)                             # step 7
    if d.size == 0 or not d.max() > 0:
        return Q[:, :0], np.zeros(0), 0
    keep = d >= eps_rel * d.max()
    V1, D1 = V[:, keep], d[keep]
    T = R @ V1 @ np.diag(1.0 / D1) @ V1.T @ R.T          # step 8
    T = 0.5 * (T + T.T)
    e, W = np.linalg.eigh(T)                             # step 9
    order = np.argsort(-e, kind="stable")
    e, W = e[order], W[:, order]
    r = min(int(keep.sum()), k)                          # rank = min(r, k)
    U = Q @ W[:, :r]                                     # step 10 (reading C5)
    return U, e[:r], int(keep.sum())


def orthonormalize(Y: np.ndarray) -> np.ndarray:
    """Q factor of a Householder QR with diag(R) >= 0 (the orthonormalisation between power steps,
    PAPER.md:209-211 "orthonormalize the columns between applications of B")."""
    Q, R = np.linalg.qr(Y)
    return Q * np.where(np.diag(R) < 0, -1.0, 1.0)


def apply_BH(S: SchurOracle, G: np.ndarray, tol_inner, maxit_inner, precond, tau, exact_inner):
    """Y = B_H G = A_GI S_I^{-1} A_IG G through the border system (reading C1): B = K_G G, solve
    S_G X = B (BF block CG to tol_inner, or exactly), Y = A_G X.  Returns (Y, block-CG info)."""
    B = S.k_gamma(G)
    if exact_inner:
        X = np.linalg.solve(S.dense(), B)
        info = {"iters": 0, "status": 0, "widths": []}
    else:
        M = S.solve_AG if precond == "AG" else None
        X, info = bf_bcg(S.apply, B, tol_inner, maxit_inner, M, tau)
    return S.d.A_G @ X, info


def nystrom_schur(S: SchurOracle, Omega: np.ndarray, k: int, tol_inner: float = 0.1,
                  maxit_inner: int = 1000, precond: str = "none", tau: float = 1e-14,
                  eps_rel: float = 1e-12, exact_inner: bool = False, q: int = 0) -> NystromResult:
    """q >= 0: q-power iteration Nystrom (eq:power PAPER.md:204-212): G = B_H^q Omega with the
    columns orthonormalised between applications of B_H; q = 0 is Alg. 2 as written.  bcg['iters'] is
    the total inner iteration count over the q + 1 block solves, bcg['iters_each'] the list."""
    G = Omega
    its = []
    for _ in range(q):                                    # power steps
        Yp, info = apply_BH(S, G, tol_inner, maxit_inner, precond, tau, exact_inner)
        its.append(info["iters"])
        G = orthonormalize(Yp)
    Y, info = apply_BH(S, G, tol_inner, maxit_inner, precond, tau, exact_inner)   # steps 1-4
    its.append(info["iters"])
    info = dict(info, iters=sum(its), iters_each=its)
    U, sigma, rC = nystrom_from_Y(G, Y, k, eps_rel)
    status = 0 if rC > 0 else NSP_ERR_RANK_COLLAPSE
    Z = S.solve_AG(U) if U.shape[1] else U               # step 11
    return NystromResult(Z, sigma, U, U.shape[1], info, status)


def apply_M2(S: SchurOracle, Z: np.ndarray, sigma: np.ndarray, r: np.ndarray) -> np.ndarray:
    """Alg. 2 step 12: M_2 r = A_G^{-1} r + Z (Sigma (Z^T r))."""
    out = S.solve_AG(r)
    if Z.shape[1]:
        out = out + Z @ (sigma * (Z.T @ r)) if r.ndim == 1 else out + Z @ (sigma[:, None] * (Z.T @ r))
    return out


def apply_ADEF2(S: SchurOracle, Z: np.ndarray, r: np.ndarray) -> np.ndarray:
    """M_A-DEF2 r = A_G^{-1} r + Z E^{-1} Z^T (r - S_G A_G^{-1} r), E = Z^T S_G Z: the adapted-deflation
    form (eq:adapted_deflation_prec PAPER.md:295-306, eq:deflation_comp_from_low_rank)
    built from M_2's basis Z = A_G^{-1} W ("in a similar way ... M_A-DEF2"; DESIGN.md
    reading R5: in the R_G-scaled space Y = R_G^{-T} W, so R_G^{-1} Y = Z and every R_G cancels)."""
    t = S.solve_AG(r)
    if Z.shape[1] == 0:
        return t
    E = Z.T @ S.apply(Z)
    E = 0.5 * (E + E.T)
    return t + Z @ np.linalg.solve(E, Z.T @ (r - S.apply(t)))


def chol_R_gamma(S: SchurOracle) -> np.ndarray:
    """R_G: the upper Cholesky factor of A_G = R_G^T R_G (eq:cholesky PAPER.md:443-446) in the Gamma
    order of the DBBD (dense; oracle sizes)."""
    return np.linalg.cholesky(S.d.A_G.toarray()).T


def nystrom_m1(S: SchurOracle, Omega: np.ndarray, k: int, tol_inner: float = 0.1, maxit_inner: int = 1000,
               precond: str = "none", tau: float = 1e-14, eps_rel: float = 1e-12, exact_inner: bool = False,
               q: int = 0) -> NystromResult:
    """M_1 (eq:prec1S PAPER.md:846-852).  Alg. 1's Nystrom steps applied to the operator
    R_G^{-T} A_GI S_I^{-1} A_IG R_G^{-1} ~ U Sigma U^T (eq:lr_approximation_S-1_A-I PAPER.md:836-840),
    R_G the A_G Cholesky factor (chol_R_gamma); Omega lives in R_G's row space.  The operator is applied
    as R_G^{-T} B_H R_G^{-1} with B_H = A_GI S_I^{-1} A_IG through the border system (reading C1,
    apply_BH).  Then Z = R_G^{-1} U (eq:prec1S "Z_k = R_G^{-1} U_k") and
    M_1 r = A_G^{-1} r + Z Sigma Z^T r - the form of apply_M2 with this (Z, Sigma)."""
    R = chol_R_gamma(S)
    G = Omega
    its = []

    def op(Gx):
        Yp, info = apply_BH(S, sla.solve_triangular(R, Gx, lower=False), tol_inner, maxit_inner, precond, tau,
                            exact_inner)
        return sla.solve_triangular(R, Yp, trans="T", lower=False), info

    for _ in range(q):                                    # power steps (eq:power) on the same operator
        Yp, info = op(G)
        its.append(info["iters"])
        G = orthonormalize(Yp)
    Y, info = op(G)
    its.append(info["iters"])
    info = dict(info, iters=sum(its), iters_each=its)
    U, sigma, rC = nystrom_from_Y(G, Y, k, eps_rel)
    status = 0 if rC > 0 else NSP_ERR_RANK_COLLAPSE
    Z = sla.solve_triangular(R, U, lower=False) if U.shape[1] else U
    return NystromResult(Z, sigma, U, U.shape[1], info, status)


def apply_M1(S: SchurOracle, Z: np.ndarray, sigma: np.ndarray, r: np.ndarray) -> np.ndarray:
    """eq:prec1S: M_1 r = R_G^{-1} (I + U Sigma U^T) R_G^{-T} r = A_G^{-1} r + Z Sigma Z^T r, Z = R_G^{-1} U."""
    return apply_M2(S, Z, sigma, r)


def apply_ADEF1(S: SchurOracle, Z: np.ndarray, r: np.ndarray) -> np.ndarray:
    """M_A-DEF1 = R_G^{-1} P_A-DEF1 R_G^{-T} (eq:deflation_comp_from_low_rank PAPER.md:871-886,
    eq:our_two_level_preconditioner PAPER.md:887-893) with Q = U E^{-1} U^T, E = U^T R_G^{-T} S_G R_G^{-1} U:
    since R_G^{-1} R_G^{-T} = A_G^{-1} and R_G^{-1} U = Z,
    M r = A_G^{-1} r + Z E^{-1} Z^T (r - S_G A_G^{-1} r), E = Z^T S_G Z - apply_ADEF2's form on M_1's Z."""
    return apply_ADEF2(S, Z, r)
