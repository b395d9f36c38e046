"""GPU parity of A_G^{-1}, the A_G^{-1}-preconditioned block CG, the Nystrom step (Alg. 2) and the
two-level preconditioner M_2 (north_star: Nystrom eigenvalues within 1e-8) against the oracle."""
import numpy as np
import pytest
import torch

import oracle as O
from oracle.nystrom import apply_M2
from tests.gpu_util import block, context, dev, problem, relfro

pytestmark = pytest.mark.gpu

NAMES = ["cfg1", "cfg2s", "cfg5s", "cfg4s"]


@pytest.mark.parametrize("name", NAMES)
def test_ag_solve_parity(name):
    pr, d, S = problem(name)
    ctx = context(pr, factor_gamma=True)
    for s in [1, 5, 64]:
        X = block(d.n_gamma, s, seed=11)
        Y = torch.empty(d.n_gamma, s, dtype=torch.float64, device="cuda")
        ctx.precond_apply(1, dev(X), Y)
        assert relfro(Y.cpu().numpy(), S.solve_AG(X)) <= 1e-12
    ctx.close()


@pytest.mark.parametrize("name", ["cfg1", "cfg2s", "cfg5s"])
def test_bcg_precond_AG_parity(name):
    """Reading C2, M = A_G^{-1} (paper-analog): iteration counts +-1, iterates at equal counts."""
    pr, d, S = problem(name)
    B = S.k_gamma(pr.omega())
    Xo, io = O.bf_bcg(S.apply, B, pr.tol_bcg, 500, S.solve_AG)
    ctx = context(pr, bcg_precond=1)
    X = torch.zeros(d.n_gamma, pr.s, dtype=torch.float64, device="cuda")
    rep = ctx.block_cg(dev(B), X, pr.tol_bcg, 500)
    assert rep["converged"] and abs(rep["iters"] - io["iters"]) <= 1, (rep["iters"], io["iters"])
    X2 = torch.zeros_like(X)
    ctx.block_cg(dev(B), X2, 0.0, io["iters"])
    assert relfro(X2.cpu().numpy(), Xo) <= 1e-8
    ctx.close()


@pytest.mark.parametrize("name", ["cfg1", "cfg2s", "cfg5s"])
def test_nystrom_parity(name):
    """Sigma (top rank) and M_2 r at equal inner iteration counts (reading C16): <= 1e-8."""
    pr, d, S = problem(name)
    Om = pr.omega()
    ref = O.nystrom_schur(S, Om, pr.rank, pr.tol_bcg, 500)
    it = ref.bcg["iters"]
    ctx = context(pr, factor_gamma=True)
    rep = ctx.nystrom(pr.rank, pr.oversample, dev(Om), 0.0, it)
    assert rep["iters"] == it and rep["rank"] == ref.rank
    sig = ctx.nystrom_sigma()
    assert np.max(np.abs(sig - ref.sigma) / ref.sigma) <= 1e-8, (sig[:4], ref.sigma[:4])
    # M_2 on probes
    R = block(d.n_gamma, 64, seed=21)
    Y = torch.empty(d.n_gamma, 64, dtype=torch.float64, device="cuda")
    ctx.precond_apply(2, dev(R), Y)
    Yref = apply_M2(S, ref.Z, ref.sigma, R)
    assert relfro(Y.cpu().numpy(), Yref) <= 1e-8
    # free-running inner solve: iteration count within +-1
    rep2 = ctx.nystrom(pr.rank, pr.oversample, dev(Om), pr.tol_bcg, 500)
    assert abs(rep2["iters"] - it) <= 1
    ctx.close()


def test_nystrom_exact_single_separator_gpu():
    """Exactness pin on the GPU: s >= rank(B_H) -> U Sigma U^T = B_H; top eigenvalues = closed form."""
    from tests.test_oracle_pins import _closed_form_modes, _single_separator
    from nsp_inputs import philox
    from paper_2101_12164_b200 import Context
    dims, axis, c = (13, 24), 0, 6
    A, part = _single_separator(dims, axis, c)
    d = O.dbbd(A.to_scipy(), part, 2)
    nG = d.n_gamma
    ctx = Context(A.rowptr, A.colidx, A.val, part, 2, factor_gamma=True)
    Om = philox.gaussian_block(0, 0, nG, nG)
    ctx.nystrom(nG, 0, dev(Om), 1e-14, 200)
    sig = ctx.nystrom_sigma()
    _, _, mu, ff = _closed_form_modes(dims, axis, c)
    lam_bh = np.sort((2 + mu) * ff / (2 + mu - ff))[::-1]
    assert np.allclose(sig[:5], lam_bh[:5], rtol=1e-8)
    ctx.close()


@pytest.mark.parametrize("name,kfix", [("cfg1", 3), ("cfg2s", 5), ("cfg5s", 4)])
def test_nystrom_power_parity(name, kfix):
    """q-power Nystrom (eq:power PAPER.md:204-212), q = 1 and 2: Sigma and M_2 probes at equal inner
    iteration counts (kfix per block solve, tol 0) within 1e-8 of the oracle."""
    from paper_2101_12164_b200 import Context
    pr, d, S = problem(name)
    Om = pr.omega()
    R = block(d.n_gamma, 16, seed=23)
    for q in (1, 2):
        ref = O.nystrom_schur(S, Om, pr.rank, 0.0, kfix, q=q)
        assert ref.bcg["iters_each"] == [kfix] * (q + 1)
        ctx = Context(pr.A.rowptr, pr.A.colidx, pr.A.val, pr.part, pr.K, factor_gamma=True, nys_power=q)
        rep = ctx.nystrom(pr.rank, pr.oversample, dev(Om), 0.0, kfix)
        assert rep["iters"] == (q + 1) * kfix and rep["rank"] == ref.rank
        sig = ctx.nystrom_sigma()
        assert np.max(np.abs(sig - ref.sigma) / ref.sigma) <= 1e-8, (q, sig[:3], ref.sigma[:3])
        Y = torch.empty(d.n_gamma, 16, dtype=torch.float64, device="cuda")
        ctx.precond_apply(2, dev(R), Y)
        assert relfro(Y.cpu().numpy(), apply_M2(S, ref.Z, ref.sigma, R)) <= 1e-8
        ctx.close()


@pytest.mark.parametrize("name", ["cfg1", "cfg2s", "cfg5s"])
def test_nystrom_si_form_parity(name):
    """The paper-literal inner system (eq:SI; Alg. 2 steps 2-4; block PCG preconditioned by A_I,
    PAPER.md:1181) on the GPU against oracle.si: free-running inner iteration count within +-1, Sigma and
    M_2 probes within 1e-8 at equal counts (reading C16)."""
    from paper_2101_12164_b200 import Context
    pr, d, S = problem(name)
    Om = pr.omega()
    ref = O.nystrom_schur_si(S, Om, pr.rank, pr.tol_bcg, 500)
    ctx = Context(pr.A.rowptr, pr.A.colidx, pr.A.val, pr.part, pr.K, factor_gamma=True, nys_form=1)
    rep = ctx.nystrom(pr.rank, pr.oversample, dev(Om), pr.tol_bcg, 500)
    assert rep["converged"] and abs(rep["iters"] - ref.bcg["iters"]) <= 1, (rep["iters"], ref.bcg["iters"])
    k = ref.bcg["iters"]
    ref0 = O.nystrom_schur_si(S, Om, pr.rank, 0.0, k)
    rep0 = ctx.nystrom(pr.rank, pr.oversample, dev(Om), 0.0, k)
    assert rep0["iters"] == k and rep0["rank"] == ref0.rank
    sig = ctx.nystrom_sigma()
    assert np.max(np.abs(sig - ref0.sigma) / ref0.sigma) <= 1e-8, (sig[:3], ref0.sigma[:3])
    R = block(d.n_gamma, 16, seed=29)
    Y = torch.empty(d.n_gamma, 16, dtype=torch.float64, device="cuda")
    ctx.precond_apply(2, dev(R), Y)
    assert relfro(Y.cpu().numpy(), apply_M2(S, ref0.Z, ref0.sigma, R)) <= 1e-8
    ctx.close()


@pytest.mark.parametrize("name", ["cfg1", "cfg2s", "cfg5s"])
def test_nystrom_m3_parity(name):
    """M_3 (Nystrom of S_I^{-1}, eq:left_prec_mat2; opts.nys_form = 2): inner count within +-1, Sigma and
    M_3 / M_A-DEF3 probes at equal counts within 1e-8 of oracle.si.nystrom_si_inverse."""
    from oracle.nystrom import apply_ADEF2
    from paper_2101_12164_b200 import Context
    from nsp_inputs import philox
    pr, d, S = problem(name)
    Om = philox.gaussian_block(0, 5, pr.n, pr.s)     # n x s sketch in the original order (interior rows used)
    ref = O.nystrom_si_inverse(S, Om, pr.rank, pr.tol_bcg, 500)
    ctx = Context(pr.A.rowptr, pr.A.colidx, pr.A.val, pr.part, pr.K, factor_gamma=True, nys_form=2)
    rep = ctx.nystrom(pr.rank, pr.oversample, dev(Om), pr.tol_bcg, 500)
    assert rep["converged"] and abs(rep["iters"] - ref.bcg["iters"]) <= 1, (rep["iters"], ref.bcg["iters"])
    k = ref.bcg["iters"]
    ref0 = O.nystrom_si_inverse(S, Om, pr.rank, 0.0, k)
    rep0 = ctx.nystrom(pr.rank, pr.oversample, dev(Om), 0.0, k)
    assert rep0["iters"] == k and rep0["rank"] == ref0.rank
    sig = ctx.nystrom_sigma()
    assert np.max(np.abs(sig - ref0.sigma) / ref0.sigma) <= 1e-8, (sig[:3], ref0.sigma[:3])
    R = block(d.n_gamma, 8, seed=31)
    Y = torch.empty(d.n_gamma, 8, dtype=torch.float64, device="cuda")
    ctx.precond_apply(2, dev(R), Y)
    assert relfro(Y.cpu().numpy(), apply_M2(S, ref0.Z, ref0.sigma, R)) <= 1e-8
    # M_A-DEF3 through the full solve at equal PCG counts
    b = pr.rhs()
    xo, io = O.solve_full_system(S, b, 1e-8, 2000, lambda r: apply_ADEF2(S, ref0.Z, r))
    x = torch.zeros(pr.n, dtype=torch.float64, device="cuda")
    rp = ctx.pcg(dev(b), x, 0.0, io["iters"], precond=3)
    assert rp["iters"] == io["iters"]
    assert relfro(x.cpu().numpy(), xo) <= 1e-8
    ctx.close()


@pytest.mark.parametrize("name", ["cfg1", "cfg2s", "cfg5s"])
def test_nystrom_m1_parity(name):
    """M_1 (eq:prec1S; opts.nys_form = 3) with the A_G factor in the natural Gamma order (ag_order = 1), so
    R_G = chol(A_G) is the oracle's factor: inner count within +-1; Sigma, M_1 probes and the M_1 /
    M_A-DEF1 full solves at equal counts within 1e-8 of oracle.nystrom.nystrom_m1."""
    from oracle.nystrom import apply_ADEF1, apply_M1
    pr, d, S = problem(name)
    Om = pr.omega()
    ref = O.nystrom_m1(S, Om, pr.rank, pr.tol_bcg, 500)
    ctx = context(pr, factor_gamma=True, nys_form=3, ag_order=1)
    rep = ctx.nystrom(pr.rank, pr.oversample, dev(Om), pr.tol_bcg, 500)
    assert rep["converged"] and abs(rep["iters"] - ref.bcg["iters"]) <= 1, (rep["iters"], ref.bcg["iters"])
    k = ref.bcg["iters"]
    ref0 = O.nystrom_m1(S, Om, pr.rank, 0.0, k)
    rep0 = ctx.nystrom(pr.rank, pr.oversample, dev(Om), 0.0, k)
    assert rep0["iters"] == k and rep0["rank"] == ref0.rank
    sig = ctx.nystrom_sigma()
    assert np.max(np.abs(sig - ref0.sigma) / ref0.sigma) <= 1e-8, (sig[:3], ref0.sigma[:3])
    R = block(d.n_gamma, 8, seed=33)
    Y = torch.empty(d.n_gamma, 8, dtype=torch.float64, device="cuda")
    ctx.precond_apply(2, dev(R), Y)
    assert relfro(Y.cpu().numpy(), apply_M1(S, ref0.Z, ref0.sigma, R)) <= 1e-8
    b = pr.rhs()
    for prec, fn in ((2, lambda r: apply_M1(S, ref0.Z, ref0.sigma, r)), (3, lambda r: apply_ADEF1(S, ref0.Z, r))):
        xo, io = O.solve_full_system(S, b, 1e-8, 2000, fn)
        x = torch.zeros(pr.n, dtype=torch.float64, device="cuda")
        rp = ctx.pcg(dev(b), x, 1e-8, 2000, precond=prec)
        assert rp["converged"] and abs(rp["iters"] - io["iters"]) <= 1, (prec, rp["iters"], io["iters"])
        x2 = torch.zeros_like(x)
        rp2 = ctx.pcg(dev(b), x2, 0.0, io["iters"], precond=prec)
        assert rp2["iters"] == io["iters"]
        assert relfro(x2.cpu().numpy(), xo) <= 1e-8
    ctx.close()


@pytest.mark.parametrize("order", [0, 1])
def test_nystrom_m1_full_rank_closed_form_gpu(order):
    """M_1 at full rank on cfg1 (inner solve to 1e-13; s = rank(B_H) = 125 of n_G = 127: the separator
    crossing has no interior neighbour, so B_H has zero eigenvalues, and Nystrom with s >= rank is exact):
    the dominant Sigma equal 1/lambda - 1 for the generalized eigenvalues S_G v = lambda A_G v (closed form
    below eq:Rt_S-1_R, independent of R_G's ordering: RCM (0) and natural (1) factors), and M_1 ~ S_G^{-1}:
    the outer PCG needs at most a few iterations.  Tolerance: with s = rank the sketch Omega^T A Omega is
    square and its condition number (1e6 natural, 9e8 RCM for this Omega, computed in fp64 on the host)
    multiplies the 1e-13 inner residual into Sigma (1e6 x 1e-13 = 1e-7; measured 3.5e-8 once the block CG's
    rounding association changed, reading R9): the top 20 are compared at 1e-7 (natural) / 1e-4
    (RCM; the oracle with exact solves and an RCM-ordered R_G already loses 1e-11 there)."""
    import scipy.linalg as sl
    from nsp_inputs import philox
    pr, d, S = problem("cfg1")
    n = d.n_gamma
    lam = sl.eigh(S.dense(), d.A_G.toarray(), eigvals_only=True)
    ref = np.sort(1.0 / lam - 1.0)[::-1]
    rk = int((ref > 1e-10 * ref[0]).sum())
    assert 100 <= rk < n
    Om = philox.gaussian_block(3, 0, n, rk)
    ctx = context(pr, factor_gamma=True, nys_form=3, ag_order=order)
    ctx.nystrom(rk, 0, dev(Om), 1e-13, 200)
    sig = ctx.nystrom_sigma()
    assert len(sig) == rk
    assert np.allclose(sig[:20], ref[:20], rtol=1e-7 if order == 1 else 1e-4), (sig[:4], ref[:4])
    b = pr.rhs()
    x = torch.zeros(pr.n, dtype=torch.float64, device="cuda")
    rp = ctx.pcg(dev(b), x, 1e-8, 50, precond=2)
    assert rp["converged"] and rp["iters"] <= 4, rp["iters"]
    ctx.close()


@pytest.mark.parametrize("name", NAMES)
def test_ag_chebyshev_parity(name):
    """A_G^{-1} by the fixed Chebyshev iteration (opts.ag_solver = 2; "an iterative
    solver to solve linear systems with A_G"): relative error <= 1e-12 against the oracle's direct
    solve, for s = 1, 5, 64 (the degree is set for a 1e-15 error bound)."""
    pr, d, S = problem(name)
    ctx = context(pr, factor_gamma=True, ag_solver=2)
    assert ctx.stats()["ag_bw"] < 0      # Chebyshev degree reported as -K
    for s in [1, 5, 64]:
        X = block(d.n_gamma, s, seed=12)
        Y = torch.empty(d.n_gamma, s, dtype=torch.float64, device="cuda")
        ctx.precond_apply(1, dev(X), Y)
        assert relfro(Y.cpu().numpy(), S.solve_AG(X)) <= 1e-12
    ctx.close()


@pytest.mark.parametrize("name", ["cfg1", "cfg5s"])
def test_m2_pcg_with_chebyshev_ag(name):
    """M_2 built and applied with the Chebyshev A_G^{-1} (the cfg5 route: its band factor does not fit):
    Sigma, and the outer PCG at equal iteration counts, within 1e-8 of the oracle (direct A_G^{-1})."""
    pr, d, S = problem(name)
    Om = pr.omega()
    ref = O.nystrom_schur(S, Om, pr.rank, pr.tol_bcg, 500)
    k = ref.bcg["iters"]
    ctx = context(pr, factor_gamma=True, ag_solver=2)
    rep = ctx.nystrom(pr.rank, pr.oversample, dev(Om), 0.0, k)
    assert rep["iters"] == k and rep["rank"] == ref.rank
    sig = ctx.nystrom_sigma()
    assert np.max(np.abs(sig - ref.sigma) / ref.sigma) <= 1e-8
    b = pr.rhs()
    xo, io = O.solve_full_system(S, b, 1e-8, 2000, lambda r: apply_M2(S, ref.Z, ref.sigma, r))
    x = torch.zeros(pr.n, dtype=torch.float64, device="cuda")
    rp = ctx.pcg(dev(b), x, 1e-8, 2000, precond=2)
    assert rp["converged"] and abs(rp["iters"] - io["iters"]) <= 1
    x2 = torch.zeros_like(x)
    ctx.pcg(dev(b), x2, 0.0, io["iters"], precond=2)
    assert relfro(x2.cpu().numpy(), xo) <= 1e-8
    ctx.close()


@pytest.mark.parametrize("spikes", [True, False])
def test_ag_partitioned_band_parity(spikes, monkeypatch):
    """The partitioned ("spike") A_G band solve (nt >= 16 tile rows, band <= 1 tile: cfg2m) against the
    oracle's direct solve and against the unpartitioned sweep (NSP_NO_SPIKE=1): s = 1 (matrix-vector
    chain kernels; partitioned: the reassociated one-product recurrence k_band_rec_vec), 7 and 64 (DMMA
    spike recurrence / update), relative error <= 1e-12."""
    if not spikes:
        monkeypatch.setenv("NSP_NO_SPIKE", "1")
    pr, d, S = problem("cfg2m")
    assert d.n_gamma >= 16 * 64
    ctx = context(pr, factor_gamma=True, ag_solver=1)
    assert 0 < ctx.stats()["ag_bw"] <= 64        # band of at most one tile: the partition applies
    for s in [1, 7, 64]:
        X = block(d.n_gamma, s, seed=13)
        Y = torch.empty(d.n_gamma, s, dtype=torch.float64, device="cuda")
        ctx.precond_apply(1, dev(X), Y)
        assert relfro(Y.cpu().numpy(), S.solve_AG(X)) <= 1e-12, s
        # the halves (M_1): R^{-T} then R^{-1} gives A_G^{-1} too
        Z = torch.empty_like(Y)
        W = torch.empty_like(Y)
        ctx.precond_apply(3, dev(X), Z)
        ctx.precond_apply(4, Z, W)
        assert relfro(W.cpu().numpy(), S.solve_AG(X)) <= 1e-12, s
    ctx.close()


def test_bcg_paper_analog_cfg2m():
    """Block CG with M = A_G^{-1} (reading C2) through the partitioned band solve at s = 32: iteration
    count within +-1 of the oracle, iterates at equal counts within 1e-8."""
    pr, d, S = problem("cfg2m")
    B = S.k_gamma(pr.omega())
    Xo, io = O.bf_bcg(S.apply, B, pr.tol_bcg, 500, S.solve_AG)
    ctx = context(pr, bcg_precond=1)
    X = torch.zeros(d.n_gamma, pr.s, dtype=torch.float64, device="cuda")
    rep = ctx.block_cg(dev(B), X, pr.tol_bcg, 500)
    assert rep["converged"] and abs(rep["iters"] - io["iters"]) <= 1, (rep["iters"], io["iters"])
    X2 = torch.zeros_like(X)
    ctx.block_cg(dev(B), X2, 0.0, io["iters"])
    assert relfro(X2.cpu().numpy(), Xo) <= 1e-8
    ctx.close()


@pytest.mark.parametrize("name,kfix", [("cfg1", 3), ("cfg5s", 4)])
def test_nystrom_m1_power_parity(name, kfix):
    """M_1 (nys_form 3, natural-order R_G) with q = 1 power step (eq:power on R_G^{-T} B_H R_G^{-1}): Sigma
    and M_1 probes at equal inner counts within 1e-8 of oracle.nystrom.nystrom_m1(q=1)."""
    from oracle.nystrom import apply_M1
    pr, d, S = problem(name)
    Om = pr.omega()
    ref = O.nystrom_m1(S, Om, pr.rank, 0.0, kfix, q=1)
    ctx = context(pr, factor_gamma=True, nys_form=3, ag_order=1, nys_power=1)
    rep = ctx.nystrom(pr.rank, pr.oversample, dev(Om), 0.0, kfix)
    assert rep["iters"] == 2 * kfix and rep["rank"] == ref.rank
    sig = ctx.nystrom_sigma()
    assert np.max(np.abs(sig - ref.sigma) / ref.sigma) <= 1e-8, (sig[:3], ref.sigma[:3])
    R = block(d.n_gamma, 8, seed=29)
    Y = torch.empty(d.n_gamma, 8, dtype=torch.float64, device="cuda")
    ctx.precond_apply(2, dev(R), Y)
    assert relfro(Y.cpu().numpy(), apply_M1(S, ref.Z, ref.sigma, R)) <= 1e-8
    ctx.close()


def test_m1_rcm_factor_pcg_cfg5s():
    """M_1 with the default RCM-ordered factor (its Nystrom approximation differs from the oracle's by
    the orthogonal similarity between the two R_G, reading R6): the outer PCG converges with a true
    residual <= 1e-6 and within 20 % of the natural-order M_1's iteration count."""
    pr, d, S = problem("cfg5s")
    b = pr.rhs()
    its = {}
    for order in (0, 1):
        ctx = context(pr, factor_gamma=True, nys_form=3, ag_order=order)
        ctx.nystrom(pr.rank, pr.oversample, dev(pr.omega()), pr.tol_bcg, 500)
        x = torch.zeros(pr.n, dtype=torch.float64, device="cuda")
        rp = ctx.pcg(dev(b), x, 1e-8, 2000, precond=2)
        assert rp["converged"]
        A = pr.A.to_scipy()
        xg = x.cpu().numpy()
        assert np.linalg.norm(b - A @ xg) / np.linalg.norm(b) <= 1e-6
        its[order] = rp["iters"]
        ctx.close()
    assert abs(its[0] - its[1]) <= max(2, 0.2 * its[1]), its


def test_nystrom_device_omega_cfg2s():
    """nsp_nystrom with Omega == NULL (generated on the device from the seed, reading C7) reproduces the
    run with the host-generated Omega: same inner count, Sigma within 1e-8."""
    pr, d, S = problem("cfg2s")
    ctx = context(pr, factor_gamma=True)
    r1 = ctx.nystrom(pr.rank, pr.oversample, dev(pr.omega()), pr.tol_bcg, 500)
    sig1 = ctx.nystrom_sigma()
    r2 = ctx.nystrom(pr.rank, pr.oversample, None, pr.tol_bcg, 500, seed=0)
    sig2 = ctx.nystrom_sigma()
    assert abs(r1["iters"] - r2["iters"]) <= 1 and r1["rank"] == r2["rank"]
    assert np.max(np.abs(sig1 - sig2) / np.abs(sig1)) <= 1e-8
    ctx.close()
