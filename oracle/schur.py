"""Border Schur complement S_G = A_G - A_GI A_I^{-1} A_IG (PAPER.md:387-390,
§2.3 eq:schur_complement), explicit (dense) and implicit (applied through
per-block direct solves), plus K_G := A_GI A_I^{-1} A_IG (the border
contribution; SURVEY.md §0 notation) and A_G^{-1} (the first-level
preconditioner S~_1^{-1}, PAPER.md:422-428 eq:S1).

A_I is block diagonal (eq:perm_A), so A_I^{-1} acts block by block:
A_GI A_I^{-1} A_IG X = sum_j A_GI_j A_I_j^{-1} A_I_jG X.  Each A_I_j^{-1} is a
library sparse direct solve (scipy SuperLU) used as a primitive step.
"""
from __future__ import annotations

import numpy as np
import scipy.sparse as sp
import scipy.sparse.linalg as spla

from .dbbd import DBBD


def _lu(M: sp.csr_matrix):
    return spla.splu(sp.csc_matrix(M), permc_spec="MMD_AT_PLUS_A",
                     diag_pivot_thresh=0.0, options={"SymmetricMode": True})


def _map(fn, items, threads: int):
    """[fn(i) for i in items], evaluated by `threads` host threads (SuperLU's solve releases the GIL);
    results come back in item order, so every caller combines them in the same fixed order as the
    serial loop (bitwise-identical output for any thread count)."""
    items = list(items)
    if threads <= 1 or len(items) <= 1:
        return [fn(i) for i in items]
    from concurrent.futures import ThreadPoolExecutor
    with ThreadPoolExecutor(max_workers=threads) as ex:
        return list(ex.map(fn, items))


class SchurOracle:
    def __init__(self, d: DBBD, blocks_needed=None, threads: int = 1):
        self.d = d
        self._lu = {}
        self._lu_G = None
        self._A_GI = None
        self._rows = {}
        self.blocks_needed = blocks_needed
        self.threads = threads

    # --- A_I_j^{-1} -----------------------------------------------------
    def lu_block(self, j: int):
        """Factor A_I_j (sparse LU as a library primitive; "factorized cheaply in parallel")."""
        if j not in self._lu:
            self._lu[j] = _lu(self.d.A_I[j]) if self.d.A_I[j].shape[0] > 0 else None
        return self._lu[j]

    def solve_AI_block(self, j: int, R: np.ndarray) -> np.ndarray:
        """A_I_j^{-1} R with the block factor."""
        lu = self.lu_block(j)
        if lu is None:
            return np.zeros_like(R)
        return lu.solve(np.ascontiguousarray(R))

    def A_GI(self, j: int) -> sp.csr_matrix:
        """A_{Gamma I_j} = A_{I_j Gamma}^T (eq:perm_A PAPER.md:371-380)."""
        if self._A_GI is None:
            self._A_GI = [None] * self.d.K
        if self._A_GI[j] is None:
            self._A_GI[j] = self.d.A_IG[j].T.tocsr()
        return self._A_GI[j]

    def gamma_rows(self, j: int) -> np.ndarray:
        """Gamma rows coupled to block j (the nonzero rows of A_GI_j = the nonzero columns of A_I_jG)."""
        if j not in self._rows:
            self._rows[j] = np.flatnonzero(np.diff(self.A_GI(j).indptr))
        return self._rows[j]

    # --- K_G X = A_GI A_I^{-1} A_IG X -------------------------------------
    def k_gamma_block(self, j: int, X: np.ndarray):
        """Block j's term A_GI_j A_I_j^{-1} A_I_jG X on its coupled Gamma rows (rows, values), or None."""
        F = self.d.A_IG[j] @ X                     # A_I_jG X   (Alg. 2 step 2)
        if not np.any(F):
            return None
        U = self.solve_AI_block(j, F)              # A_I_j^{-1} F
        r = self.gamma_rows(j)
        return r, self.A_GI(j)[r] @ U              # A_GI_j U   (Alg. 2 step 4)

    def k_gamma(self, X: np.ndarray, blocks=None) -> np.ndarray:
        """K_Gamma X = sum_j A_GI_j A_I_j^{-1} A_I_j_G X (reading C1, the A_Gamma-free part of
        eq:schur_complement), summed in ascending j.  blocks: restrict the sum to these blocks (a
        bounded timing sample of a large config)."""
        X = np.asarray(X, dtype=np.float64)
        out = np.zeros((self.d.n_gamma,) + X.shape[1:])
        js = range(self.d.K) if blocks is None else sorted(blocks)
        for t in _map(lambda j: self.k_gamma_block(j, X), js, self.threads):
            if t is not None:
                out[t[0]] += t[1]
        return out

    # --- S_G X (eq:schur_complement) ---------------------------------------
    def apply(self, X: np.ndarray) -> np.ndarray:
        """S_Gamma X = A_Gamma X - K_Gamma X (eq:schur_complement PAPER.md:387-390), implicitly."""
        return self.d.A_G @ np.asarray(X, dtype=np.float64) - self.k_gamma(X)

    def apply_rows(self, X: np.ndarray, rows: np.ndarray) -> np.ndarray:
        """(S_G X)[rows, :] computed one output row at a time: only the blocks
        adjacent to a sampled Gamma row contribute to it."""
        X = np.asarray(X, dtype=np.float64)
        rows = np.asarray(rows)
        out = np.asarray(self.d.A_G[rows] @ X)
        for j in range(self.d.K):
            AGIj = self.A_GI(j)[rows]
            if AGIj.nnz == 0:
                continue
            F = self.d.A_IG[j] @ X
            U = self.solve_AI_block(j, F)
            out -= AGIj @ U
        return out

    def factor_all(self):
        """Factor every A_I_j (in parallel over blocks when threads > 1)."""
        _map(self.lu_block, range(self.d.K), self.threads)

    # --- explicit dense S_G (tiny cases only) ------------------------------
    def dense(self) -> np.ndarray:
        """The explicit S_Gamma (eq:schur_complement PAPER.md:387-390) by dense elimination, tiny cases only."""
        S = self.d.A_G.toarray()
        for j in range(self.d.K):
            if self.d.A_I[j].shape[0] == 0:
                continue
            AIj = self.d.A_I[j].toarray()
            AIGj = self.d.A_IG[j].toarray()
            S -= AIGj.T @ np.linalg.solve(AIj, AIGj)
        return S

    # --- A_G^{-1} (eq:S1) ---------------------------------------------------
    def solve_AG(self, R: np.ndarray) -> np.ndarray:
        """A_Gamma^{-1} R (S~_1 of eq:S1) by a direct sparse solve."""
        if self._lu_G is None:
            self._lu_G = _lu(self.d.A_G)
        return self._lu_G.solve(np.ascontiguousarray(R, dtype=np.float64))

    # --- A_I^{-1} on a full interior vector (block by block) ---------------
    def solve_AI(self, r_I: list) -> list:
        """Block-diagonal A_I^{-1} applied block by block."""
        return [self.solve_AI_block(j, r_I[j]) for j in range(self.d.K)]


def schur_rows(A: sp.csr_matrix, part: np.ndarray, X: np.ndarray, rows_gamma: np.ndarray) -> np.ndarray:
    """(S_G X)[g, :] for the given Gamma rows, straight from eq:schur_complement
    written out row by row:  (A_G X)[g] - sum_{j adjacent to g} A_GI_j[g, :] A_I_j^{-1} A_I_jG X,
    touching only the blocks adjacent to the sampled rows (for full-size configs where the full
    DBBD is too large to extract).  X: n_G x s in the Gamma order of ascending original id
    (reading C10); rows_gamma: original node ids of the sampled Gamma rows."""
    A = sp.csr_matrix(A)
    part = np.asarray(part)
    gamma = np.flatnonzero(part < 0)
    gpos = np.full(A.shape[0], -1, dtype=np.int64)
    gpos[gamma] = np.arange(gamma.size)
    X = np.asarray(X, dtype=np.float64)
    out = np.zeros((len(rows_gamma), X.shape[1]))
    for r, g in enumerate(rows_gamma):
        cols = A.indices[A.indptr[g]:A.indptr[g + 1]]
        vals = A.data[A.indptr[g]:A.indptr[g + 1]]
        gam = part[cols] < 0
        out[r] = vals[gam] @ X[gpos[cols[gam]]]                       # (A_G X)[g]
        for j in np.unique(part[cols[~gam]]):
            blk = np.flatnonzero(part == j)
            AIj = A[blk][:, blk]
            AjG = A[blk][:, gamma]                                     # A_I_jG
            U = _lu(AIj).solve(np.ascontiguousarray(AjG @ X))          # A_I_j^{-1} A_I_jG X
            a_g = A[g][:, blk].toarray().ravel()                       # A_GI_j[g, :]
            out[r] -= a_g @ U
    return out


class LocalSchurOracle:
    """S_Gamma assembled from dense LOCAL blocks (SURVEY.md §8(c) oracle step 2, "explicit, for cfg2"):
    eq:schur_complement written out block by block,

        S_Gamma = A_Gamma - sum_j E_j^T K_j E_j,   K_j = F_j^T A_I_j^{-1} F_j,   F_j = A_I_jG[:, G_j],

    where G_j is the set of Gamma rows coupled to block j and E_j selects them.  K_j is formed once
    (A_I_j^{-1} by the same library sparse factor as SchurOracle) and every apply is then |G_j| x |G_j|
    dense products: fast enough for full-size cfg2 block CG on the host.  Test infrastructure only."""

    def __init__(self, d: DBBD, threads: int = 1, schur: SchurOracle | None = None):
        self.d = d
        self.S = schur if schur is not None else SchurOracle(d, threads=threads)
        self.S.threads = threads

        def form(j):
            r = self.S.gamma_rows(j)
            if r.size == 0 or d.A_I[j].shape[0] == 0:
                return r, np.zeros((r.size, r.size))
            F = d.A_IG[j][:, r].toarray()                   # F_j = A_I_jG restricted to G_j
            return r, F.T @ self.S.solve_AI_block(j, F)    # K_j = F_j^T A_I_j^{-1} F_j

        self.rows, self.K = zip(*_map(form, range(d.K), threads)) if d.K else ((), ())

    def k_gamma(self, X: np.ndarray) -> np.ndarray:
        """K_Gamma X = sum_j E_j^T K_j E_j X, ascending j."""
        X = np.asarray(X, dtype=np.float64)
        out = np.zeros((self.d.n_gamma,) + X.shape[1:])
        for r, Kj in zip(self.rows, self.K):
            if r.size:
                out[r] += Kj @ X[r]
        return out

    def apply(self, X: np.ndarray) -> np.ndarray:
        """S_Gamma X = A_Gamma X - K_Gamma X (eq:schur_complement PAPER.md:387-390)."""
        return self.d.A_G @ np.asarray(X, dtype=np.float64) - self.k_gamma(X)
