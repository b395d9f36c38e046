"""Doubly bordered block diagonal (DBBD) form of A from a partition vector.

PAPER.md:369-378 (§2.3, eq:perm_A): P^T A P = [[A_I, A_IG], [A_GI, A_G]] with
A_I block diagonal.  Reading C10: permutation = [block 0 nodes in
ascending original index, ..., block K-1, Gamma nodes in ascending original
index].  The separator property (no entry couples two different
blocks) is checked by brute force over all nonzeros.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import scipy.sparse as sp


@dataclass
class DBBD:
    n: int
    K: int
    gamma: np.ndarray              # original ids of Gamma nodes (ascending)
    blocks: list                   # blocks[j] = original ids of block j (ascending)
    A_I: list                      # A_I[j]: scipy csr, |blk_j| x |blk_j|
    A_IG: list                     # A_IG[j]: scipy csr, |blk_j| x n_G
    A_G: sp.csr_matrix             # n_G x n_G
    perm: np.ndarray               # new -> old

    @property
    def n_gamma(self) -> int:
        """Size of the border Gamma (eq:perm_A PAPER.md:371-380)."""
        return int(self.gamma.size)

    @property
    def A_GI(self) -> list:
        """The border rows A_{Gamma I_j} = A_{I_j Gamma}^T of eq:perm_A."""
        return [m.T.tocsr() for m in self.A_IG]


def dbbd(A: sp.csr_matrix, part: np.ndarray, K: int, blocks=None) -> DBBD:
    """Doubly bordered block diagonal form of A (eq:perm_A PAPER.md:371-380): the K interior blocks
    A_I_j (part == j), the border Gamma (part == -1, ascending id; reading C10) and the couplings.
    blocks (optional): extract A_I_j / A_I_jG only for these block ids (the others are None) - a bounded
    timing sample of a config too large to extract whole; the separator check still covers all of A."""
    A = sp.csr_matrix(A)
    n = A.shape[0]
    if A.shape != (n, n):
        raise ValueError("A must be square")
    part = np.asarray(part)
    if part.shape != (n,):
        raise ValueError("part must have n entries")
    if np.any((part < -1) | (part >= K)):
        raise ValueError("part entries must be -1 or a block id in [0, K)")
    if (A - A.T).count_nonzero() != 0:
        raise ValueError("A must be symmetric")
    coo = A.tocoo()
    bi, bj = part[coo.row], part[coo.col]
    bad = (bi >= 0) & (bj >= 0) & (bi != bj) & (coo.data != 0)
    if np.any(bad):
        k = int(np.flatnonzero(bad)[0])
        raise ValueError(f"separator property violated at entry ({coo.row[k]}, {coo.col[k]}) "
                         f"between blocks {bi[k]} and {bj[k]}")
    gamma = np.flatnonzero(part < 0)
    want = set(range(K)) if blocks is None else set(int(j) for j in blocks)
    if blocks is None:
        blks = [np.flatnonzero(part == j) for j in range(K)]
    else:   # one stable sort instead of K scans: block j's ids are ascending within its run
        order = np.argsort(part, kind="stable")
        starts = np.searchsorted(part[order], np.arange(K + 1))
        blks = [order[starts[j]:starts[j + 1]] for j in range(K)]
    A_I = [A[b][:, b].tocsr() if j in want else None for j, b in enumerate(blks)]
    A_IG = [A[b][:, gamma].tocsr() if j in want else None for j, b in enumerate(blks)]
    A_G = A[gamma][:, gamma].tocsr()
    perm = np.concatenate(blks + [gamma])
    return DBBD(n, K, gamma, blks, A_I, A_IG, A_G, perm)
