"""Pins of the CPU oracle against things other than itself (closed forms,
brute-force elimination, exact-arithmetic termination, exactness).  CPU only.

Each test names the passage (PAPER.md line / SURVEY.md §8(c) pin table) that
fixes the expected value.
"""
import math
import os

import numpy as np
import pytest
import scipy.sparse as sp

import oracle as O
from oracle.bcg import NSP_OK, NSP_ERR_STAGNATION
from oracle.nystrom import apply_M2, nystrom_from_Y
from nsp_inputs import philox
from nsp_inputs import problems as P

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


# ---------------------------------------------------------------------------
# inputs
# ---------------------------------------------------------------------------

def test_philox_known_answers():
    """Random123 KAT vectors (tests/golden/philox4x32_10_kat.txt)."""
    for line in open(os.path.join(GOLDEN, "philox4x32_10_kat.txt")):
        if line.startswith("#") or not line.strip():
            continue
        w = [int(x, 16) for x in line.split()]
        out = philox.philox4x32_10(np.array([w[:4]], dtype=np.uint32), (w[4], w[5]))[0]
        assert [int(x) for x in out] == w[6:10]


def test_gaussian_moments_and_determinism():
    g = philox.gaussian(0, 0, 200_000)
    assert abs(g.mean()) < 4 / math.sqrt(g.size) * 1.5
    assert abs(g.var() - 1) < 0.02
    assert np.array_equal(g[:1000], philox.gaussian(0, 0, 1000))
    assert not np.array_equal(g[:1000], philox.gaussian(1, 0, 1000))


@pytest.mark.parametrize("dims,coef", [((13, 9), None), ((12, 10), [1.0, 1e-3]), ((6, 5, 4), None)])
def test_laplacian_closed_form_spectrum(dims, coef):
    """north_star: eigenvalues sum_d c_d 4 sin^2(pi k_d / (2(m_d+1)))."""
    A = P.laplacian(dims, coef).to_scipy().toarray()
    assert np.array_equal(A, A.T)
    coef = coef or [1.0] * len(dims)
    grids = np.meshgrid(*[c * 4 * np.sin(np.pi * np.arange(1, m + 1) / (2 * (m + 1))) ** 2
                          for m, c in zip(dims, coef)], indexing="ij")
    lam = np.sort(sum(grids).ravel())
    assert np.max(np.abs(np.linalg.eigvalsh(A) - lam)) < 1e-12 * lam.max()


def test_cfg1_partition_sizes():
    """BASELINE.json configs[0] n_G = 127; C11 blocks 1024/992/992/961 (tests/golden/cfg_sizes.txt)."""
    for line in open(os.path.join(GOLDEN, "cfg_sizes.txt")):
        if line.startswith("#") or not line.strip():
            continue
        name, n, nnz, ng, K, sizes = line.split()
        pr = P.make(name)
        assert pr.n == int(n) and pr.A.nnz == int(nnz) and pr.n_gamma == int(ng) and pr.K == int(K)
        assert list(np.bincount(pr.part[pr.part >= 0])) == [int(x) for x in sizes.split(",")]


def test_separator_property_bruteforce():
    """no entry couples two different blocks (checked entry by entry)."""
    for name in ["cfg1", "cfg3s", "cfg4s"]:
        pr = P.make(name)
        A = pr.A
        for i in range(0, A.n, 7):
            for q in range(A.rowptr[i], A.rowptr[i + 1]):
                j = A.colidx[q]
                bi, bj = pr.part[i], pr.part[j]
                assert bi < 0 or bj < 0 or bi == bj
    # and dbbd rejects a violation
    A = P.laplacian((4, 4)).to_scipy()
    part = np.zeros(16, dtype=np.int32)
    part[1] = 1
    with pytest.raises(ValueError, match="separator property"):
        O.dbbd(A, part, 2)


# ---------------------------------------------------------------------------
# S_G
# ---------------------------------------------------------------------------

def _single_separator(dims, axis, c):
    """Box with one separator plane at index c along `axis` (reading: SURVEY.md §8(c) pin table)."""
    pr_A = P.laplacian(dims)
    idx = np.indices(dims)[axis].ravel()
    part = np.where(idx < c, 0, np.where(idx > c, 1, -1)).astype(np.int32)
    return pr_A, part


def _closed_form_modes(dims, axis, c):
    m = dims[axis]
    w1, w2 = c, m - c - 1
    plane = [dims[a] for a in range(len(dims)) if a != axis]
    js = np.meshgrid(*[np.arange(1, p + 1) for p in plane], indexing="ij")
    js = [j.ravel() for j in js]
    mu = sum(4 * np.sin(np.pi * j / (2 * (p + 1))) ** 2 for j, p in zip(js, plane))
    theta = np.arccosh(1 + mu / 2)
    f = lambda w: np.sinh(w * theta) / np.sinh((w + 1) * theta)  # noqa: E731
    lam = 2 + mu - f(w1) - f(w2)
    # eigenvectors: tensor DST-I modes on the plane, Gamma nodes in ascending original index
    coords = np.meshgrid(*[np.arange(1, p + 1) for p in plane], indexing="ij")
    coords = [x.ravel() for x in coords]
    V = np.ones((coords[0].size, js[0].size))
    for x, j, p in zip(coords, js, plane):
        V *= np.sin(np.pi * np.outer(x, j) / (p + 1))
    V /= np.linalg.norm(V, axis=0)
    return lam, V, mu, f(w1) + f(w2)


@pytest.mark.parametrize("dims,axis,c", [((9, 7), 0, 4), ((16, 12), 1, 5), ((64, 64), 0, 32), ((9, 6, 5), 0, 3)])
def test_schur_single_separator_closed_form(dims, axis, c):
    """S_G v_j = lambda_j v_j, lambda_j = 2 + mu_j - f(w1) - f(w2)."""
    A, part = _single_separator(dims, axis, c)
    d = O.dbbd(A.to_scipy(), part, 2)
    S = O.SchurOracle(d)
    lam, V, _, _ = _closed_form_modes(dims, axis, c)
    SV = S.apply(V)
    assert np.max(np.abs(SV - V * lam)) < 1e-12 * lam.max()


@pytest.mark.parametrize("dims,axis,c", [((9, 7), 0, 4), ((9, 6, 5), 0, 3)])
def test_related_spectra_closed_form(dims, axis, c):
    """eig(A_G^{-1} S_G) = 1 - (f1+f2)/(2+mu) in (0,1];
    eig(B_H) = (2+mu)(f1+f2)/(2+mu-f1-f2), B_H = A_GI S_I^{-1} A_IG."""
    A, part = _single_separator(dims, axis, c)
    d = O.dbbd(A.to_scipy(), part, 2)
    S = O.SchurOracle(d)
    lam, V, mu, ff = _closed_form_modes(dims, axis, c)
    Sd = S.dense()
    AG = d.A_G.toarray()
    ev = np.sort(np.linalg.eigvals(np.linalg.solve(AG, Sd)).real)
    assert np.allclose(ev, np.sort(1 - ff / (2 + mu)), atol=1e-12)
    assert ev.max() <= 1 + 1e-12
    BH = AG @ np.linalg.solve(Sd, AG) - AG          # finding 1: B_H = A_G S_G^{-1} A_G - A_G
    eb = np.sort(np.linalg.eigvalsh(0.5 * (BH + BH.T)))
    assert np.allclose(eb, np.sort((2 + mu) * ff / (2 + mu - ff)), rtol=1e-10, atol=1e-12)


def _gauss_eliminate_schur(Afull, nI):
    """Brute force: Gaussian elimination (pure Python loops) of the first nI unknowns."""
    n = len(Afull)
    M = [list(map(float, row)) for row in Afull]
    for k in range(nI):
        piv = M[k][k]
        for i in range(k + 1, n):
            if M[i][k] != 0.0:
                l = M[i][k] / piv
                for j in range(k, n):
                    M[i][j] -= l * M[k][j]
    return np.array([row[nI:] for row in M[nI:]])


@pytest.mark.parametrize("dims,K", [((7, 6), 4), ((5, 4, 4), 4)])
def test_schur_bruteforce_elimination(dims, K):
    """north_star: dense brute-force S_G by Gaussian elimination on tiny grids."""
    A = P.laplacian(dims).to_scipy()
    part = P.geometric_nd(dims, K)
    d = O.dbbd(A, part, K)
    Ad = A.toarray()[np.ix_(d.perm, d.perm)]
    S_bf = _gauss_eliminate_schur(Ad.tolist(), d.n - d.n_gamma)
    S = O.SchurOracle(d)
    assert np.max(np.abs(S.dense() - S_bf)) < 1e-13 * np.abs(S_bf).max()
    X = np.random.default_rng(0).standard_normal((d.n_gamma, 3))
    assert np.max(np.abs(S.apply(X) - S_bf @ X)) < 1e-13 * np.abs(S_bf @ X).max()
    rows = np.array([0, d.n_gamma // 2, d.n_gamma - 1])
    assert np.max(np.abs(S.apply_rows(X, rows) - (S_bf @ X)[rows])) < 1e-13 * np.abs(S_bf @ X).max()


@pytest.mark.parametrize("dims,axis,c", [((9, 7), 0, 4), ((16, 12), 1, 5), ((9, 6, 5), 0, 3)])
def test_local_schur_single_separator_closed_form(dims, axis, c):
    """LocalSchurOracle (S_G from dense local blocks, the full-size cfg2 oracle) against the closed-form
    single-separator spectrum: S_G v_j = lambda_j v_j."""
    A, part = _single_separator(dims, axis, c)
    d = O.dbbd(A.to_scipy(), part, 2)
    lam, V, _, _ = _closed_form_modes(dims, axis, c)
    L = O.LocalSchurOracle(d)
    assert np.max(np.abs(L.apply(V) - V * lam)) < 1e-12 * lam.max()


@pytest.mark.parametrize("dims,K", [((7, 6), 4), ((5, 4, 4), 4)])
def test_local_schur_bruteforce_elimination(dims, K):
    """LocalSchurOracle against brute-force Gaussian elimination (pure Python loops) on tiny grids."""
    A = P.laplacian(dims).to_scipy()
    part = P.geometric_nd(dims, K)
    d = O.dbbd(A, part, K)
    Ad = A.toarray()[np.ix_(d.perm, d.perm)]
    S_bf = _gauss_eliminate_schur(Ad.tolist(), d.n - d.n_gamma)
    X = np.random.default_rng(0).standard_normal((d.n_gamma, 3))
    L = O.LocalSchurOracle(d)
    assert np.max(np.abs(L.apply(X) - S_bf @ X)) < 1e-13 * np.abs(S_bf @ X).max()


def test_oracle_threads_bitwise_identical():
    """The thread pool only distributes independent blocks; sums stay in ascending block order, so
    the result is bitwise identical to the serial loop (any thread count)."""
    pr = P.make("cfg2s")
    d = O.dbbd(pr.A.to_scipy(), pr.part, pr.K)
    X = pr.omega()
    Y1 = O.SchurOracle(d).apply(X)
    Y4 = O.SchurOracle(d, threads=4).apply(X)
    assert np.array_equal(Y1, Y4)
    assert np.array_equal(O.LocalSchurOracle(d).apply(X), O.LocalSchurOracle(d, threads=4).apply(X))
    # subset sums: K_G over a block subset = the sum of its blocks' terms
    S = O.SchurOracle(d)
    parts = S.k_gamma(X, blocks=range(0, d.K, 2)) + S.k_gamma(X, blocks=range(1, d.K, 2))
    assert np.max(np.abs(parts - S.k_gamma(X))) <= 1e-13 * np.abs(parts).max()


def test_schur_decoupled_and_arrow():
    """A_GI = 0 -> S_G = A_G; arrow matrix -> a_GG - sum a_i^2/d_i."""
    A = sp.csr_matrix(np.diag([2.0, 3.0, 4.0, 5.0]))
    d = O.dbbd(A, np.array([0, 0, 1, -1], dtype=np.int32), 2)
    assert np.allclose(O.SchurOracle(d).dense(), [[5.0]])
    dvals = np.array([2.0, 3.0, 4.0, 5.0])
    a = np.array([0.5, -1.0, 0.25, 0.75])
    Ad = np.zeros((5, 5))
    Ad[:4, :4] = np.diag(dvals)
    Ad[4, :4] = Ad[:4, 4] = a
    Ad[4, 4] = 10.0
    d = O.dbbd(sp.csr_matrix(Ad), np.array([0, 1, 2, 3, -1], dtype=np.int32), 4)
    assert abs(O.SchurOracle(d).dense()[0, 0] - (10.0 - np.sum(a * a / dvals))) < 1e-14


def _dense_blocks(d):
    nI = d.n - d.n_gamma
    AI = np.zeros((nI, nI))
    AIG = np.zeros((nI, d.n_gamma))
    o = 0
    for j in range(d.K):
        m = d.blocks[j].size
        AI[o:o + m, o:o + m] = d.A_I[j].toarray()
        AIG[o:o + m] = d.A_IG[j].toarray()
        o += m
    return AI, AIG, d.A_G.toarray()


def test_woodbury_and_reading_C1_identity():
    """eq:S-1 and reading C1: A_G S_G^{-1} K_G Om = A_GI S_I^{-1} A_IG Om."""
    pr = P.make("cfg1")
    d = O.dbbd(pr.A.to_scipy(), pr.part, pr.K)
    S = O.SchurOracle(d)
    AI, AIG, AG = _dense_blocks(d)
    SI = AI - AIG @ np.linalg.solve(AG, AIG.T)                      # eq:SI
    Sg = AG - AIG.T @ np.linalg.solve(AI, AIG)                       # eq:schur_complement
    lhs = np.linalg.inv(Sg)
    rhs = np.linalg.inv(AG) + np.linalg.solve(AG, AIG.T @ np.linalg.solve(SI, AIG @ np.linalg.inv(AG)))
    assert np.max(np.abs(lhs - rhs)) < 1e-12 * np.abs(lhs).max()
    Om = pr.omega()
    Y_paper = AIG.T @ np.linalg.solve(SI, AIG @ Om)                  # Alg. 2 steps 2-4 literally
    Y_c1 = AG @ np.linalg.solve(Sg, S.k_gamma(Om))                   # reading C1
    assert np.max(np.abs(Y_paper - Y_c1)) < 1e-12 * np.abs(Y_paper).max()


# ---------------------------------------------------------------------------
# block CG
# ---------------------------------------------------------------------------

def test_bcg_exact_termination_cfg1():
    """north_star: block CG converges within ceil(n_G/s) iterations in exact arithmetic;
    active widths sum to n_G (30+30+30+30+7 = 127)."""
    pr = P.make("cfg1")
    d = O.dbbd(pr.A.to_scipy(), pr.part, pr.K)
    S = O.SchurOracle(d)
    B = S.k_gamma(pr.omega())
    X, info = O.bf_bcg(S.apply, B, 1e-12, 50)
    assert info["status"] == NSP_OK
    assert info["iters"] <= math.ceil(d.n_gamma / pr.s)
    assert sum(info["widths"]) == d.n_gamma
    assert np.max(np.abs(X - np.linalg.solve(S.dense(), B))) < 1e-10 * np.abs(X).max()
    X1, info1 = O.bf_bcg(S.apply, B, pr.tol_bcg, 50)
    assert info1["iters"] == 5 and info1["widths"] == [30, 30, 30, 30, 7]


def test_bcg_s1_is_textbook_cg():
    """block CG with s = 1 produces the CG iterates."""
    pr = P.make("cfg2s")
    d = O.dbbd(pr.A.to_scipy(), pr.part, pr.K)
    S = O.SchurOracle(d)
    b = pr.omega()[:, :1]
    for k in [3, 10, 25]:
        Xb, ib = O.bf_bcg(S.apply, b, 0.0, k)
        xc, ic = O.pcg(lambda v: S.apply(v[:, None])[:, 0], b[:, 0], 0.0, k)
        assert ib["iters"] == ic["iters"] == k
        assert np.max(np.abs(Xb[:, 0] - xc)) < 1e-10 * np.abs(xc).max()


def test_bcg_identity_and_duplicates():
    """S = I -> 1 iteration; two identical columns -> width drops by one."""
    B = np.random.default_rng(1).standard_normal((40, 5))
    X, info = O.bf_bcg(lambda V: V, B, 1e-12, 10)
    assert info["iters"] == 1 and np.allclose(X, B)
    Dg = np.arange(1.0, 21.0)
    B = np.random.default_rng(2).standard_normal((20, 4))
    B[:, 3] = B[:, 1]
    X, info = O.bf_bcg(lambda V: Dg[:, None] * V, B, 1e-10, 30)
    assert info["status"] == NSP_OK
    assert info["widths"][0] == 3
    assert np.allclose(X[:, 3], X[:, 1])
    assert np.max(np.abs(X - B / Dg[:, None])) < 1e-9


def test_bcg_zero_rhs_and_stagnation():
    B = np.zeros((10, 3))
    X, info = O.bf_bcg(lambda V: V, B, 0.1, 5)
    assert info["status"] == NSP_OK and info["iters"] == 0
    # directions all deflated: S = 0 on the span -> D singular is reported, not hidden
    B = np.random.default_rng(0).standard_normal((10, 2))
    _, info = O.bf_bcg(lambda V: 0 * V, B, 1e-3, 5)
    assert info["status"] != NSP_OK


def test_inner_extended_error_bound():
    """oracle.bcg.inner_extended (reading R8) against the exact inner product (rational arithmetic): the
    error obeys the dot-product bound with the EXTENDED unit roundoff, |err| <= n u_ext sum |a_i b_i|
    + u_64 |exact| (one final rounding), and on a cancellation-heavy case it is far below the fp64 error."""
    from fractions import Fraction
    from oracle.bcg import inner_extended
    u_ext = float(np.finfo(np.longdouble).eps)
    assert u_ext < 1e-18, "inner_extended needs an extended long double"
    rng = np.random.default_rng(5)
    n = 4000
    a = rng.standard_normal(n) * np.exp(rng.uniform(-5, 5, n))
    b = rng.standard_normal(n)
    b[-1] = -(a[:-1] @ b[:-1]) / a[-1]          # heavy cancellation in column 0
    A, Bm = a[:, None], np.stack([b, np.abs(rng.standard_normal(n))], axis=1)
    got = inner_extended(A, Bm)[0]
    f64 = (A.T @ Bm)[0]
    for j in range(2):
        exact = float(sum(Fraction(x) * Fraction(y) for x, y in zip(a, Bm[:, j])))
        mag = float(np.sum(np.abs(a * Bm[:, j])))
        err = abs(got[j] - exact)
        assert err <= n * u_ext * mag + np.spacing(abs(exact)), (j, err, n * u_ext * mag)
        if j == 0:
            assert err < abs(f64[j] - exact) / 100, (err, abs(f64[j] - exact))


def test_bcg_extended_inner_structural_pins():
    """bf_bcg with extended-precision Grams keeps the exact-arithmetic pins: cfg1 terminates in
    ceil(n_G/s) iterations with widths 30+30+30+30+7 = n_G; s = 1 is textbook CG."""
    from oracle.bcg import inner_extended
    pr = P.make("cfg1")
    d = O.dbbd(pr.A.to_scipy(), pr.part, pr.K)
    S = O.SchurOracle(d)
    B = S.k_gamma(pr.omega())
    X, info = O.bf_bcg(S.apply, B, 1e-12, 50, inner=inner_extended)
    assert info["iters"] <= math.ceil(d.n_gamma / pr.s) and sum(info["widths"]) == d.n_gamma
    assert np.max(np.abs(X - np.linalg.solve(S.dense(), B))) < 1e-10 * np.abs(X).max()
    b = B[:, :1]
    Xb, _ = O.bf_bcg(S.apply, b, 0.0, 10, inner=inner_extended)
    xc, _ = O.pcg(lambda v: S.apply(v[:, None])[:, 0], b[:, 0], 0.0, 10)
    assert np.max(np.abs(Xb[:, 0] - xc)) < 1e-10 * np.abs(xc).max()


def test_orth_fallback_rank():
    rng = np.random.default_rng(3)
    W = rng.standard_normal((50, 6))
    W[:, 5] = W[:, 0] + W[:, 2]
    P_, w, fb = O.orth(W)
    assert fb and w == 5
    assert np.allclose(P_.T @ P_, np.eye(5), atol=1e-12)
    P2, w2, fb2 = O.orth(W[:, :5])
    assert not fb2 and w2 == 5 and np.allclose(P2.T @ P2, np.eye(5), atol=1e-12)


def test_pcg_cg_error_bound():
    """eq:k-th_error_cg at every step, unpreconditioned CG on S_G."""
    pr = P.make("cfg1")
    d = O.dbbd(pr.A.to_scipy(), pr.part, pr.K)
    S = O.SchurOracle(d)
    Sd = S.dense()
    ev = np.linalg.eigvalsh(Sd)
    kap = ev.max() / ev.min()
    f = pr.omega()[:, 0]
    xs = np.linalg.solve(Sd, f)
    _, info = O.pcg(lambda v: Sd @ v, f, 1e-12, 200, record_x=True)
    e0 = math.sqrt(xs @ Sd @ xs)
    rho = (math.sqrt(kap) - 1) / (math.sqrt(kap) + 1)
    for k, x in enumerate(info["xs"], start=1):
        e = x - xs
        assert math.sqrt(e @ Sd @ e) <= 2 * e0 * rho ** k * (1 + 1e-8) + 1e-12


# ---------------------------------------------------------------------------
# Nystrom, M_2, PCG
# ---------------------------------------------------------------------------

def test_nystrom_rank1_and_exactness():
    """SPEC.md:342/356; exact on rank <= k; rank = min(r, k)."""
    rng = np.random.default_rng(4)
    u = rng.standard_normal(30)
    u /= np.linalg.norm(u)
    Bm = np.outer(u, u)
    Om = rng.standard_normal((30, 3))
    U, sig, rC = nystrom_from_Y(Om, Bm @ Om, 1)
    assert rC == 1 and abs(sig[0] - 1) < 1e-12 and abs(abs(U[:, 0] @ u) - 1) < 1e-12
    V = np.linalg.qr(rng.standard_normal((30, 4)))[0]
    Bm = V @ np.diag([5.0, 3.0, 2.0, 0.5]) @ V.T
    Om = rng.standard_normal((30, 7))
    U, sig, rC = nystrom_from_Y(Om, Bm @ Om, 7)
    assert rC == 4 and U.shape[1] == 4
    assert np.max(np.abs(U @ np.diag(sig) @ U.T - Bm)) < 1e-12


def test_nystrom_exact_on_single_separator_line():
    """north_star: exact Nystrom reconstruction when s >= rank(B_H) with an exact inner
    solve (24-node separator line); top eigenvalues match the closed form of eig(B_H)."""
    dims, axis, c = (13, 24), 0, 6
    A, part = _single_separator(dims, axis, c)
    d = O.dbbd(A.to_scipy(), part, 2)
    S = O.SchurOracle(d)
    nG = d.n_gamma
    Om = philox.gaussian_block(0, 0, nG, nG)
    res = O.nystrom_schur(S, Om, nG, exact_inner=True)
    AG = d.A_G.toarray()
    BH = AG @ np.linalg.solve(S.dense(), AG) - AG
    rec = res.U @ np.diag(res.sigma) @ res.U.T
    assert np.max(np.abs(rec - BH)) < 1e-9 * np.abs(BH).max()
    _, _, mu, ff = _closed_form_modes(dims, axis, c)
    lam_bh = np.sort((2 + mu) * ff / (2 + mu - ff))[::-1]
    assert np.allclose(res.sigma[:5], lam_bh[:5], rtol=1e-9)


def test_m2_exact_gives_one_pcg_iteration_and_Z0():
    """eq:S-1: with k = n_G and an exact inner solve, M_2 = S_G^{-1} -> PCG converges in 1
    iteration; with Z = 0, M_2 = A_G^{-1}."""
    pr = P.make("cfg1")
    d = O.dbbd(pr.A.to_scipy(), pr.part, pr.K)
    S = O.SchurOracle(d)
    Om = philox.gaussian_block(0, 0, d.n_gamma, d.n_gamma)
    res = O.nystrom_schur(S, Om, d.n_gamma, exact_inner=True)
    M = lambda r: apply_M2(S, res.Z, res.sigma, r)  # noqa: E731
    Sd = S.dense()
    assert np.max(np.abs(M(np.eye(d.n_gamma)) @ Sd - np.eye(d.n_gamma))) < 1e-9
    f = pr.omega()[:, 0]
    _, info = O.pcg(S.apply, f, 1e-8, 10, M)
    assert info["iters"] == 1
    r = pr.omega()[:, 1]
    assert np.allclose(apply_M2(S, np.zeros((d.n_gamma, 0)), np.zeros(0), r), np.linalg.solve(d.A_G.toarray(), r))


def test_full_solve_matches_dense_direct():
    """solve_full_system vs a dense direct solve."""
    pr = P.make("cfg1")
    A = pr.A.to_scipy()
    d = O.dbbd(A, pr.part, pr.K)
    S = O.SchurOracle(d)
    xs = pr.xstar()
    b = A @ xs
    res = O.nystrom_schur(S, pr.omega(), pr.rank, pr.tol_bcg)
    M = lambda r: apply_M2(S, res.Z, res.sigma, r)  # noqa: E731
    x, info = O.solve_full_system(S, b, 1e-12, 500, M)
    xd = np.linalg.solve(A.toarray(), b)
    assert info["status"] == 0
    assert np.linalg.norm(x - xd) / np.linalg.norm(xd) < 1e-10
    # M_2 is symmetric (SPEC.md:463 probe)
    rng = np.random.default_rng(5)
    u, v = rng.standard_normal(d.n_gamma), rng.standard_normal(d.n_gamma)
    assert abs(u @ M(v) - v @ M(u)) < 1e-12 * abs(u @ M(v))


def test_schur_rows_single_separator_closed_form():
    """oracle.schur.schur_rows (the row-by-row definition used for full-size sampled parity) against
    the single-separator closed form S_G v_j = lambda_j v_j (SURVEY.md §8(c) pin table)."""
    from oracle.schur import schur_rows
    dims, axis, c = (16, 12), 1, 5
    A, part = _single_separator(dims, axis, c)
    lam, V, _, _ = _closed_form_modes(dims, axis, c)
    gamma = np.flatnonzero(part < 0)
    rows = gamma[[0, 3, gamma.size - 1]]
    Y = schur_rows(A.to_scipy(), part, V, rows)
    assert np.max(np.abs(Y - (V * lam)[[0, 3, gamma.size - 1]])) < 1e-13 * lam.max()


def test_power_nystrom_converges_to_closed_form():
    """eq:power: with exact inner solves, q-power iteration with s < rank(B_H)
    approaches the closed-form top eigenvalues of B_H monotonically in q (the top-k subspace is
    resolved better; eq:bound_theta_k PAPER.md:1026-1027)."""
    dims, axis, c = (13, 24), 0, 6
    A, part = _single_separator(dims, axis, c)
    d = O.dbbd(A.to_scipy(), part, 2)
    S = O.SchurOracle(d)
    _, _, mu, ff = _closed_form_modes(dims, axis, c)
    lam_bh = np.sort((2 + mu) * ff / (2 + mu - ff))[::-1]
    Om = philox.gaussian_block(0, 0, d.n_gamma, 8)
    errs = []
    for q in range(4):
        r = O.nystrom_schur(S, Om, 4, exact_inner=True, q=q)
        errs.append(np.max(np.abs(r.sigma[:4] - lam_bh[:4]) / lam_bh[:4]))
    assert all(errs[i + 1] <= errs[i] * 1.0001 for i in range(3)), errs
    assert errs[3] < 1e-2 * errs[0], errs


def test_si_formulation_matches_border_formulation():
    """Reading C1 at the level of the whole Nystrom step: with exact inner solves, the paper-literal
    S_I system (eq:SI, Alg. 2 steps 2-4) and the border system give the same Y = B_H G, hence the same
    Sigma; S_I itself is checked against the dense definition A_I - A_IG A_G^{-1} A_GI."""
    pr = P.make("cfg1")
    d = O.dbbd(pr.A.to_scipy(), pr.part, pr.K)
    S = O.SchurOracle(d)
    op = O.SIOperator(S)
    V = philox.gaussian_block(4, 9, op.n_I, 3)
    SI = op.A_I.toarray() - op.A_IG.toarray() @ np.linalg.solve(d.A_G.toarray(), op.A_IG.T.toarray())
    assert np.allclose(op.apply(V), SI @ V, rtol=0, atol=1e-12 * np.abs(SI @ V).max())
    Om = pr.omega()
    a = O.nystrom_schur_si(S, Om, pr.rank, tol_inner=1e-13, maxit_inner=2000)
    b = O.nystrom_schur(S, Om, pr.rank, exact_inner=True)
    assert np.max(np.abs(a.sigma - b.sigma) / b.sigma) < 1e-9


def test_si_block_pcg_iterations_cfg1():
    """Context (parity unpinned): the S_I block PCG (A_I preconditioner) at tol 0.1 converges in a few
    iterations on cfg1 (the paper's it_SI are 24-72 on its matrices, tab:blockvsclassic)."""
    pr = P.make("cfg1")
    d = O.dbbd(pr.A.to_scipy(), pr.part, pr.K)
    r = O.nystrom_schur_si(O.SchurOracle(d), pr.omega(), pr.rank, tol_inner=0.1)
    assert r.bcg["status"] == 0 and 1 <= r.bcg["iters"] <= 20 and r.rank == pr.rank


def test_adef2_exact_deflation_space():
    """M_A-DEF2 (reading R5): if Z spans an exact invariant subspace of A_G^{-1} S_G (the GEVP eq:GEVP
    eigenvectors), the A-DEF preconditioned operator maps those directions to themselves: M S_G z = z
    (eq:adapted_deflation_prec: P_A-DEF A Z = Z), and on the complement it equals A_G^{-1} S_G."""
    import scipy.linalg as sl
    from oracle.nystrom import apply_ADEF2
    pr = P.make("cfg1")
    d = O.dbbd(pr.A.to_scipy(), pr.part, pr.K)
    S = O.SchurOracle(d)
    Sd = S.dense()
    AG = d.A_G.toarray()
    lam, V = sl.eigh(Sd, AG)                  # S v = lam A_G v (eq:GEVP)
    Z = V[:, :6]                              # smallest generalized eigenpairs
    MS = np.column_stack([apply_ADEF2(S, Z, Sd[:, j]) for j in range(Sd.shape[0])])
    assert np.allclose(MS @ Z, Z, atol=1e-10)
    v = V[:, 20]                              # a direction outside span(Z): A_G^{-1} S v = lam v
    assert np.allclose(MS @ v, lam[20] * v, atol=1e-10 * np.abs(v).max())


def test_m3_exact_gives_one_pcg_iteration():
    """M_3 (eq:left_prec_mat2): with s = n_I and an exact inner solve the Nystrom approximation of S_I^{-1}
    is exact, so M_3 = A_G^{-1} + A_G^{-1} A_GI S_I^{-1} A_IG A_G^{-1} = S_G^{-1} (Woodbury eq:S-1,
    PAPER.md:807-813) and the outer PCG converges in one iteration."""
    from oracle.nystrom import apply_M2
    dims, axis, c = (5, 9), 0, 2
    A, part = _single_separator(dims, axis, c)
    d = O.dbbd(A.to_scipy(), part, 2)
    S = O.SchurOracle(d)
    nI = A.n - d.n_gamma
    Om = philox.gaussian_block(0, 0, A.n, nI)
    r = O.nystrom_si_inverse(S, Om, nI, exact_inner=True)
    assert r.rank == nI
    b = philox.gaussian(5, 1, A.n)
    x, info = O.solve_full_system(S, b, 1e-10, 50, lambda v: apply_M2(S, r.Z, r.sigma, v))
    assert info["iters"] <= 1 + 1 and np.allclose(x, np.linalg.solve(A.to_scipy().toarray(), b), atol=1e-9)


def test_rt_s_inverse_r_identity():
    """eq:Rt_S-1_R: R_G S_G^{-1} R_G^T = I + R_G^{-T} A_GI S_I^{-1} A_IG R_G^{-1}, checked
    with dense matrices built by elimination (independent of the Nystrom code), and the eigenvalue map
    stated below it: (lambda, u) of R_G^{-T} S_G R_G^{-1} <-> (1/lambda - 1, u)."""
    import scipy.linalg as sl
    from oracle.nystrom import chol_R_gamma
    pr = P.make("cfg1")
    d = O.dbbd(pr.A.to_scipy(), pr.part, pr.K)
    S = O.SchurOracle(d)
    Sd = S.dense()
    R = chol_R_gamma(S)
    assert np.allclose(R.T @ R, d.A_G.toarray(), atol=1e-12)
    A = pr.A.to_scipy().toarray()
    perm = d.perm
    Ap = A[np.ix_(perm, perm)]
    nI = A.shape[0] - d.n_gamma
    AI, AIG, AGI = Ap[:nI, :nI], Ap[:nI, nI:], Ap[nI:, :nI]
    SI = AI - AIG @ np.linalg.solve(d.A_G.toarray(), AGI)          # eq:SI
    Ri = np.linalg.inv(R)
    lhs = R @ np.linalg.solve(Sd, R.T)
    rhs = np.eye(d.n_gamma) + Ri.T @ AGI @ np.linalg.solve(SI, AIG) @ Ri
    assert np.allclose(lhs, rhs, atol=1e-9 * np.abs(lhs).max())
    lam = np.sort(np.linalg.eigvalsh(Ri.T @ Sd @ Ri))
    mu = np.sort(np.linalg.eigvalsh(0.5 * (rhs + rhs.T) - np.eye(d.n_gamma)))
    assert np.allclose(np.sort(1.0 / lam - 1.0), mu, rtol=1e-8, atol=1e-10)


def test_m1_full_rank_closed_form_and_exact():
    """M_1 (eq:prec1S): with s = n_G and an exact inner solve the Nystrom approximation of
    R_G^{-T} A_GI S_I^{-1} A_IG R_G^{-1} is its EVD, so Sigma equals 1/lambda - 1 for the generalized
    eigenvalues S_G v = lambda A_G v (eq:GEVP; the map below eq:Rt_S-1_R) and M_1 = S_G^{-1}
    (M_1 S_G = I)."""
    import scipy.linalg as sl
    from oracle.nystrom import apply_M1
    pr = P.make("cfg1")
    d = O.dbbd(pr.A.to_scipy(), pr.part, pr.K)
    S = O.SchurOracle(d)
    n = d.n_gamma
    Om = philox.gaussian_block(3, 0, n, n)
    r = O.nystrom_m1(S, Om, n, exact_inner=True)
    lam = sl.eigh(S.dense(), d.A_G.toarray(), eigvals_only=True)   # ascending
    ref = np.sort(1.0 / lam - 1.0)[::-1]
    keep = ref > 1e-12 * ref[0]
    assert r.rank >= keep.sum() - 1
    m = min(r.rank, int(keep.sum()))
    assert np.allclose(r.sigma[:m], ref[:m], rtol=1e-7, atol=1e-9 * ref[0])
    Sd = S.dense()
    MS = apply_M1(S, r.Z, r.sigma, Sd)
    assert np.allclose(MS, np.eye(n), atol=1e-7)


def test_m1_low_rank_matches_adef1_deflation():
    """M_A-DEF1 (eq:deflation_comp_from_low_rank / eq:our_two_level_preconditioner) built on an exact
    truncated EVD (s = n_G, exact inner solve, k < n_G): the preconditioned operator maps span(Z) onto
    itself identically (P_A-DEF A Z = Z), while M_1 maps it to Z (I + Sigma) / (1 + Sigma) = Z too
    (the adapted-deflation property stated after eq:prec1S)."""
    from oracle.nystrom import apply_ADEF1, apply_M1
    pr = P.make("cfg1")
    d = O.dbbd(pr.A.to_scipy(), pr.part, pr.K)
    S = O.SchurOracle(d)
    n = d.n_gamma
    Om = philox.gaussian_block(4, 0, n, n)
    r = O.nystrom_m1(S, Om, 10, exact_inner=True)
    assert r.rank == 10
    Sd = S.dense()
    MS1 = apply_M1(S, r.Z, r.sigma, Sd @ r.Z)
    MSd = apply_ADEF1(S, r.Z, Sd @ r.Z)
    assert np.allclose(MS1, r.Z, atol=1e-8 * np.abs(r.Z).max())
    assert np.allclose(MSd, r.Z, atol=1e-8 * np.abs(r.Z).max())
