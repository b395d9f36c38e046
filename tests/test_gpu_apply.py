"""GPU parity of the S_G / K_G block applies (north_star: S_G X within 1e-12 relative Frobenius)
against the oracle, through the C ABI."""
import numpy as np
import pytest
import torch

from tests.gpu_util import block, context, dev, problem, relfro
from tests.test_oracle_pins import _closed_form_modes, _single_separator

pytestmark = pytest.mark.gpu

CASES = [("cfg1", 30), ("cfg1", 1), ("cfg1", 7), ("cfg2s", 32), ("cfg2s", 100), ("cfg3s", 16),
         ("cfg3s", 64), ("cfg4s", 24), ("cfg5s", 32), ("cfg5s", 128)]


@pytest.mark.parametrize("apply_kernel", [0, 1, 2])
@pytest.mark.parametrize("name,s", CASES)
def test_schur_apply_parity(name, s, apply_kernel):
    """apply_kernel 0: a2+a3 as one product with the explicit S_j^{-1} tiles (INT8 tensor cores for
    s >= 48, reading R10); 1: the L22 sweeps; 2: the fp64 DMMA product only."""
    pr, d, S = problem(name)
    ctx = context(pr, apply_kernel=apply_kernel)
    X = block(d.n_gamma, s)
    Y = torch.empty(d.n_gamma, s, dtype=torch.float64, device="cuda")
    ctx.schur_apply(dev(X), Y)
    torch.cuda.synchronize()
    ref = S.apply(X)
    assert relfro(Y.cpu().numpy(), ref) <= 1e-12
    Yk = torch.empty_like(Y)
    ctx.kgamma_apply(dev(X), Yk)
    assert relfro(Yk.cpu().numpy(), S.k_gamma(X)) <= 1e-12
    ctx.close()


@pytest.mark.parametrize("dims,axis,c", [((16, 12), 1, 5), ((64, 64), 0, 32), ((9, 6, 5), 0, 3),
                                         ((70, 130), 0, 35)])
def test_schur_apply_closed_form(dims, axis, c):
    """S_G v_j = lambda_j v_j on a single separator (SURVEY.md §8(c) pin), on the GPU directly."""
    A, part = _single_separator(dims, axis, c)
    from paper_2101_12164_b200 import Context
    ctx = Context(A.rowptr, A.colidx, A.val, part, 2)
    lam, V, _, _ = _closed_form_modes(dims, axis, c)
    Y = torch.empty(V.shape, dtype=torch.float64, device="cuda")
    ctx.schur_apply(dev(V), Y)
    assert np.max(np.abs(Y.cpu().numpy() - V * lam)) < 1e-12 * lam.max()
    ctx.close()


@pytest.mark.parametrize("apply_kernel", [0, 1])
def test_apply_deterministic(apply_kernel):
    pr, d, S = problem("cfg2s")
    ctx = context(pr, apply_kernel=apply_kernel)
    X = dev(block(d.n_gamma, 32))
    Y1 = torch.empty_like(X)
    Y2 = torch.empty_like(X)
    ctx.schur_apply(X, Y1)
    ctx.schur_apply(X, Y2)
    assert torch.equal(Y1, Y2)
    ctx.close()
