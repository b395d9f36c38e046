"""Measured comparison for DESIGN.md §7 (the 3D apply's flop floor): per-block flops per right-hand side of
the sparse-factor solve restricted to the boundary layer (forward + backward over the reach of the B rows in L,
SuperLU factor with MMD / COLAMD ordering) against the dense S_j^{-1} product (2 b_j^2), on cfg5 blocks.
    python tools/nd_flop_count.py"""
import sys, time
sys.path.insert(0, '/root/repo')
import numpy as np, scipy.sparse as sp, scipy.sparse.linalg as spla
from nsp_inputs import problems as P
pr = P.make("cfg5")
A = pr.A.to_scipy()
blocks = [0, 300, 511]
gamma = np.flatnonzero(pr.part < 0)
for j in blocks:
    blk = np.flatnonzero(pr.part == j)
    AI = A[blk][:, blk].tocsr(); AIG = A[blk][:, gamma].tocsr()
    n = AI.shape[0]
    B = np.flatnonzero(np.diff(AIG.tocsr().indptr))          # boundary-layer rows
    for spec in ["MMD_AT_PLUS_A", "COLAMD"]:
        lu = spla.splu(sp.csc_matrix(AI), permc_spec=spec, diag_pivot_thresh=0.0, options={"SymmetricMode": True})
        L = lu.L.tocsc()
        perm = lu.perm_c   # column perm: A[:, perm_c]... position of original node i in factor order
        pos = np.empty(n, dtype=np.int64); pos[perm] = np.arange(n)
        # reach of B rows in the forward solve: closure under "column k updates rows L[k+1:, k]"
        reach = np.zeros(n, dtype=bool)
        start = np.sort(pos[B])
        reach[start] = True
        indptr, indices = L.indptr, L.indices
        for k in range(n):
            if reach[k]:
                reach[indices[indptr[k]:indptr[k + 1]]] = True
        colnnz = np.diff(indptr)
        f_fwd = 2 * colnnz[reach].sum()
        # backward solve restricted to B: needs u at rows that feed B through L^T, i.e. the same reach set
        # (u_k depends on u_i for i > k with L[i,k] != 0; only rows in B are wanted -> ancestors of B = reach)
        f_bwd = 2 * colnnz[reach].sum()
        print(f"block {j} ({spec}): n={n} b={B.size} nnz(L)={L.nnz} reach={reach.sum()} "
              f"ND-solve flops/RHS={f_fwd + f_bwd:.3e} dense S^-1 flops/RHS={2 * B.size**2:.3e} "
              f"ratio={(2 * B.size**2) / (f_fwd + f_bwd):.2f}", flush=True)
