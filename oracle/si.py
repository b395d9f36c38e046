"""The paper-literal inner system of Alg. 2: the interior Schur complement

    S_I = A_I - A_IG A_G^{-1} A_GI        (eq:SI)

solved with k+p right-hand sides F = A_IG G (step 2) by the breakdown-free block PCG "preconditioned
by the block diagonal matrix A_I", then Y = A_GI X (step 4) and steps
5-12 exactly as in `nystrom.py` (the build's default is the equivalent border
system of reading C1).  Interior vectors are stacked block by block in the DBBD order (blocks 0..K-1,
each in ascending original index).
"""
from __future__ import annotations

import numpy as np
import scipy.sparse as sp

from .bcg import bf_bcg
from .nystrom import NSP_ERR_RANK_COLLAPSE, NystromResult, nystrom_from_Y, orthonormalize
from .schur import SchurOracle


class SIOperator:
    def __init__(self, S: SchurOracle):
        self.S = S
        d = S.d
        self.sizes = [b.size for b in d.blocks]
        self.offs = np.concatenate([[0], np.cumsum(self.sizes)]).astype(np.int64)
        self.n_I = int(self.offs[-1])
        self.A_I = sp.block_diag([d.A_I[j] for j in range(d.K) if d.A_I[j].shape[0]] or [sp.csr_matrix((0, 0))],
                                 format="csr")
        self.A_IG = sp.vstack([d.A_IG[j] for j in range(d.K)], format="csr")   # n_I x n_G

    def apply(self, V: np.ndarray) -> np.ndarray:
        """S_I V = A_I V - A_IG A_G^{-1} A_GI V (eq:SI)."""
        return self.A_I @ V - self.A_IG @ self.S.solve_AG(self.A_IG.T @ V)

    def solve_AI(self, R: np.ndarray) -> np.ndarray:
        """A_I^{-1} R block by block (the preconditioner of PAPER.md:1181)."""
        out = np.empty_like(R)
        for j in range(self.S.d.K):
            a, b = self.offs[j], self.offs[j + 1]
            if b > a:
                out[a:b] = self.S.solve_AI_block(j, R[a:b])
        return out


def nystrom_schur_si(S: SchurOracle, Omega: np.ndarray, k: int, tol_inner: float = 0.1,
                     maxit_inner: int = 1000, precond: bool = True, tau: float = 1e-14,
                     eps_rel: float = 1e-12, q: int = 0) -> NystromResult:
    """Alg. 2 with the paper-literal inner system: F = A_IG G, S_I X = F by the block
    PCG preconditioned by A_I (eq:SI PAPER.md:814-819), Y = A_GI X,
    then steps 5-12 as nystrom.nystrom_schur."""
    op = SIOperator(S)
    G = Omega
    its = []
    for step in range(q + 1):
        F = op.A_IG @ G                                                    # step 2
        X, info = bf_bcg(op.apply, F, tol_inner, maxit_inner,
                         op.solve_AI if precond else None, tau)           # step 3
        its.append(info["iters"])
        Y = op.A_IG.T @ X                                                  # step 4: Y = A_GI X
        if step < q:
            G = orthonormalize(Y)
    info = dict(info, iters=sum(its), iters_each=its)
    U, sigma, rC = nystrom_from_Y(G, Y, k, eps_rel)
    status = 0 if rC > 0 else NSP_ERR_RANK_COLLAPSE
    Z = S.solve_AG(U) if U.shape[1] else U
    return NystromResult(Z, sigma, U, U.shape[1], info, status)


def interior_rows(S: SchurOracle) -> np.ndarray:
    """Original node ids of the interior rows in the DBBD order (blocks 0..K-1, ascending ids)."""
    return np.concatenate([b for b in S.d.blocks]) if S.d.K else np.zeros(0, dtype=np.int64)


def nystrom_si_inverse(S: SchurOracle, Omega_full: np.ndarray, k: int, tol_inner: float = 0.1,
                       maxit_inner: int = 1000, precond: bool = True, tau: float = 1e-14,
                       eps_rel: float = 1e-12, exact_inner: bool = False) -> NystromResult:
    """M_3 (eq:internal_term_lr_approximation_2, eq:left_prec_mat2): Nystrom of
    S_I^{-1} ~ V Sigma V^T with the sketch Omega_I (the interior rows of Omega_full, n x s in the
    original order): Y = S_I^{-1} Omega_I (block PCG, A_I preconditioner), Alg. 1 steps on (Omega_I, Y),
    then Z^ = A_G^{-1} A_GI V and M_3 = A_G^{-1} + Z^ Sigma Z^^T."""
    op = SIOperator(S)
    Om = np.ascontiguousarray(Omega_full[interior_rows(S)])
    if exact_inner:
        SI = op.A_I.toarray() - op.A_IG.toarray() @ np.linalg.solve(S.d.A_G.toarray(), op.A_IG.T.toarray())
        Y = np.linalg.solve(SI, Om)
        info = {"iters": 0, "status": 0, "widths": []}
    else:
        Y, info = bf_bcg(op.apply, Om, tol_inner, maxit_inner, op.solve_AI if precond else None, tau)
    V, sigma, rC = nystrom_from_Y(Om, Y, k, eps_rel)
    status = 0 if rC > 0 else NSP_ERR_RANK_COLLAPSE
    Z = S.solve_AG(op.A_IG.T @ V) if V.shape[1] else V
    return NystromResult(Z, sigma, V, V.shape[1], info, status)
