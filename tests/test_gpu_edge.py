"""Degenerate and ragged cases through the C ABI on the GPU (parity against the dense
oracle S_G): an all-boundary block (n1 = 0), a block with no boundary layer (an isolated node, b = 0),
empty blocks, a separator node adjacent to no block, ragged s (1 ... 128, not multiples of the tile
widths), both apply kernels, block CG, and the full solve with every preconditioner."""
import numpy as np
import pytest
import scipy.sparse as sp
import torch

import oracle as O
from nsp_inputs import philox
from nsp_inputs.problems import CSR, laplacian
from paper_2101_12164_b200 import Context

pytestmark = pytest.mark.gpu


def _degenerate():
    m = 14
    L = laplacian((m, m)).to_scipy()
    A = sp.block_diag([L, sp.csr_matrix(np.array([[2.0]]))]).tocsr()   # + an isolated node
    A.sort_indices()
    n = A.shape[0]
    part = np.full(n, -1, dtype=np.int32)
    idx = lambda y, x: y * m + x
    for y in range(m):
        for x in range(m):
            part[idx(y, x)] = 0 if y < 6 else (-1 if y == 6 else 1)
    part[idx(6, 7)] = 2                                    # all-boundary block (n1 = 0)
    part[idx(5, 7)] = -1
    part[idx(7, 7)] = -1
    for y, x in [(0, 13), (0, 12), (1, 13)]:                # (0, 13): Gamma node with no adjacent block
        part[idx(y, x)] = -1
    part[n - 1] = 3                                         # no boundary layer (b = 0)
    K = 6                                                   # blocks 4, 5 empty
    csr = CSR(n, A.indptr.astype(np.int64), A.indices.astype(np.int32), A.data.astype(np.float64))
    return csr, part, K


@pytest.fixture(scope="module")
def deg():
    csr, part, K = _degenerate()
    d = O.dbbd(csr.to_scipy(), part, K)
    S = O.SchurOracle(d)
    return csr, part, K, d, S, S.dense()


def _dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).to("cuda", torch.float64)


def _rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


@pytest.mark.parametrize("apply_kernel", [0, 1])
@pytest.mark.parametrize("s", [1, 7, 33, 64, 100, 128])
def test_degenerate_apply(deg, s, apply_kernel):
    csr, part, K, d, S, Sd = deg
    ctx = Context(csr.rowptr, csr.colidx, csr.val, part, K, apply_kernel=apply_kernel)
    X = philox.gaussian_block(2, 9, d.n_gamma, s)
    Y = torch.empty(d.n_gamma, s, dtype=torch.float64, device="cuda")
    ctx.schur_apply(_dev(X), Y)
    assert _rel(Y.cpu().numpy(), Sd @ X) <= 1e-12
    ctx.close()


def test_degenerate_block_cg_and_pcg(deg):
    csr, part, K, d, S, Sd = deg
    ctx = Context(csr.rowptr, csr.colidx, csr.val, part, K, factor_gamma=True)
    s = 5
    B = philox.gaussian_block(3, 9, d.n_gamma, s)
    X = torch.zeros(d.n_gamma, s, dtype=torch.float64, device="cuda")
    rep = ctx.block_cg(_dev(B), X, 1e-12, 200)
    assert rep["converged"]
    assert _rel(X.cpu().numpy(), np.linalg.solve(Sd, B)) <= 1e-10
    Om = philox.gaussian_block(0, 0, d.n_gamma, 8)
    ctx.nystrom(6, 2, _dev(Om), 1e-10, 200)
    b = philox.gaussian(5, 1, csr.n)
    xd = np.linalg.solve(csr.to_scipy().toarray(), b)
    for prec in (0, 1, 2):
        x = torch.zeros(csr.n, dtype=torch.float64, device="cuda")
        r = ctx.pcg(_dev(b), x, 1e-12, 500, precond=prec)
        assert r["converged"], (prec, r)
        assert _rel(x.cpu().numpy(), xd) <= 1e-9, prec
    ctx.close()


def test_round2_abi_error_paths():
    """Round-2 entry points fail loudly on bad use: M = A_G^{-1} without the A_G operator (NSP_ERR_STATE),
    an out-of-range M, an explicit-Omega-only Nystrom form called with Omega = NULL (NSP_ERR_ARG), kernel
    entries with unsupported widths / too-small fused shapes (NSP_ERR_ARG), a bad fused-pass mode."""
    from paper_2101_12164_b200 import nsp
    from paper_2101_12164_b200.nsp import NspError
    from nsp_inputs import problems as P
    pr = P.make("cfg1")
    ctx = Context(pr.A.rowptr, pr.A.colidx, pr.A.val, pr.part, pr.K)
    with pytest.raises(NspError, match="NSP_ERR_STATE"):
        ctx.set_bcg_precond(1)
    with pytest.raises(NspError, match="NSP_ERR_ARG"):
        ctx.set_bcg_precond(2)
    ctx.close()
    ctx = Context(pr.A.rowptr, pr.A.colidx, pr.A.val, pr.part, pr.K, factor_gamma=True, nys_form=3, ag_order=1)
    with pytest.raises(NspError, match="NSP_ERR_ARG"):
        ctx.nystrom(pr.rank, pr.oversample, None, 0.1, 50)
    ctx.close()
    X = torch.zeros(100, 32, dtype=torch.float64, device="cuda")
    M = torch.zeros(32, 32, dtype=torch.float64, device="cuda")
    with pytest.raises(NspError):
        nsp.dev_panel(X, None, X, M, 1.0)                     # s = 32: not a supported width
    Y = torch.zeros(100, 128, dtype=torch.float64, device="cuda")
    G = torch.zeros(128, 128, dtype=torch.float64, device="cuda")
    with pytest.raises(NspError):
        nsp.dev_panel_gram(Y, None, Y, G, 1.0, 0, G)          # n < 64 x SMs: no fused shape
    with pytest.raises(NspError):
        nsp.dev_set_fused_pg(3)


def test_block_cg_precond_switch_reuses_context():
    """nsp_set_bcg_precond switches M on one context (the bench times both modes on one cfg5 context):
    each mode gives the same iterations and X as a context built for that mode (bitwise: same kernels)."""
    from nsp_inputs import problems as P
    pr = P.make("cfg2s")
    d = O.dbbd(pr.A.to_scipy(), pr.part, pr.K)
    B = _dev(O.SchurOracle(d).k_gamma(pr.omega()))
    ctx = Context(pr.A.rowptr, pr.A.colidx, pr.A.val, pr.part, pr.K, factor_gamma=True)
    out = {}
    for m in (0, 1, 0):
        ctx.set_bcg_precond(m)
        X = torch.zeros_like(B)
        rep = ctx.block_cg(B, X, pr.tol_bcg, 500)
        out.setdefault(m, []).append((rep["iters"], X.cpu().numpy()))
    ctx.close()
    assert out[0][0][0] == out[0][1][0] and np.array_equal(out[0][0][1], out[0][1][1])
    ref = Context(pr.A.rowptr, pr.A.colidx, pr.A.val, pr.part, pr.K, bcg_precond=1)
    X = torch.zeros_like(B)
    rep = ref.block_cg(B, X, pr.tol_bcg, 500)
    ref.close()
    assert rep["iters"] == out[1][0][0] and np.array_equal(X.cpu().numpy(), out[1][0][1])
