"""a2+a3 on the INT8 tensor cores (tcgen05 kind::i8, Ozaki splitting of the D-scaled S_j^{-1} tiles,
DESIGN.md reading R10) against the oracle: the S_G / K_G applies within the north_star's 1e-12 relative
Frobenius (eq:schur_complement PAPER.md:387-396), forced on for every width (apply_kernel 3, including
s > 128: two column tiles, and ragged s), elementwise agreement with the fp64 DMMA product, determinism,
and the dispatch evidence (path counter)."""
import numpy as np
import pytest
import torch

import paper_2101_12164_b200.nsp as nsp
from tests.gpu_util import block, context, dev, problem, relfro

pytestmark = pytest.mark.gpu

CASES = [("cfg1", 7), ("cfg1", 30), ("cfg2s", 100), ("cfg2s", 128), ("cfg2s", 200), ("cfg3s", 64),
         ("cfg4s", 96), ("cfg5s", 128), ("cfg5s", 33)]


@pytest.mark.parametrize("name,s", CASES)
def test_ozaki_apply_parity(name, s):
    pr, d, S = problem(name)
    ctx = context(pr, apply_kernel=3)
    X = block(d.n_gamma, s)
    Y = torch.empty(d.n_gamma, s, dtype=torch.float64, device="cuda")
    c0 = nsp.path_counters()
    ctx.schur_apply(dev(X), Y)
    torch.cuda.synchronize()
    c1 = nsp.path_counters()
    assert c1["ozaki"] > c0["ozaki"], "the INT8 tensor-core a2+a3 was not dispatched"
    ref = S.apply(X)
    err = relfro(Y.cpu().numpy(), ref)
    print(f"{name} s={s}: S_G X rel. Frobenius error {err:.2e}")
    assert err <= 1e-12
    Yk = torch.empty_like(Y)
    ctx.kgamma_apply(dev(X), Yk)
    assert relfro(Yk.cpu().numpy(), S.k_gamma(X)) <= 1e-12
    ctx.close()


@pytest.mark.parametrize("name,s", [("cfg2s", 128), ("cfg5s", 100)])
def test_ozaki_matches_dmma_elementwise(name, s):
    """K_G X (the a2+a3 result through A_GI) from the INT8 path and from the fp64 DMMA product agree
    entry by entry to the fp64 rounding level of the product (|diff| <= 1e-13 max|K_G X| per column)."""
    pr, d, S = problem(name)
    X = dev(block(d.n_gamma, s))
    out = []
    for ak in (3, 2):
        ctx = context(pr, apply_kernel=ak)
        Y = torch.empty(d.n_gamma, s, dtype=torch.float64, device="cuda")
        ctx.kgamma_apply(X, Y)
        torch.cuda.synchronize()
        out.append(Y.cpu().numpy())
        ctx.close()
    diff = np.abs(out[0] - out[1]).max(axis=0) / np.abs(out[1]).max(axis=0)
    print(f"{name} s={s}: max column-relative |INT8 - DMMA| {diff.max():.2e}")
    assert diff.max() <= 1e-13


def test_ozaki_deterministic():
    pr, d, S = problem("cfg2s")
    ctx = context(pr, apply_kernel=3)
    X = dev(block(d.n_gamma, 128))
    Y1 = torch.empty_like(X)
    Y2 = torch.empty_like(X)
    ctx.schur_apply(X, Y1)
    ctx.schur_apply(X, Y2)
    torch.cuda.synchronize()
    assert torch.equal(Y1, Y2)
    ctx.close()


def test_ozaki_scale_extremes():
    """Columns of wildly different magnitude (1e-150 .. 1e150) and an all-zero column: the per-column
    power-of-two scales keep every column at full relative accuracy."""
    pr, d, S = problem("cfg2s")
    ctx = context(pr, apply_kernel=3)
    X = block(d.n_gamma, 64)
    X[:, 1] *= 1e150
    X[:, 2] *= 1e-150
    X[:, 3] = 0.0
    Y = torch.empty(d.n_gamma, 64, dtype=torch.float64, device="cuda")
    ctx.schur_apply(dev(X), Y)
    torch.cuda.synchronize()
    Yh = Y.cpu().numpy()
    ref = S.apply(X)
    for c in range(64):
        nr = np.linalg.norm(ref[:, c])
        if nr == 0:
            assert np.all(Yh[:, c] == 0)
        else:
            assert np.linalg.norm(Yh[:, c] - ref[:, c]) / nr <= 1e-12, c
    ctx.close()


def test_ozaki_cluster_multicast_variant():
    """The two-CTA cluster variant (W^T slices multicast, NSP_OZ_CLUSTER=1, opt-in) gives the bitwise same
    result as the one-CTA kernel (same products, same epilogue; only the data movement differs), including
    blocks with an odd tile count (the pair's second CTA recomputes and discards)."""
    import subprocess, sys, os
    code = (
        "import numpy as np, torch, sys\n"
        "sys.path.insert(0, %r)\n"
        "from tests.gpu_util import block, context, dev, problem\n"
        "pr, d, S = problem('cfg2s')\n"
        "ctx = context(pr, apply_kernel=3)\n"
        "X = dev(block(d.n_gamma, 128))\n"
        "Y = torch.empty_like(X)\n"
        "ctx.schur_apply(X, Y)\n"
        "torch.cuda.synchronize()\n"
        "np.save(sys.argv[1], Y.cpu().numpy())\n" % os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import tempfile
    outs = []
    with tempfile.TemporaryDirectory() as td:
        for cl in ("0", "1"):
            f = os.path.join(td, f"y{cl}.npy")
            env = dict(os.environ, NSP_OZ_CLUSTER=cl)
            r = subprocess.run([sys.executable, "-c", code, f], env=env, capture_output=True, text=True, timeout=600)
            assert r.returncode == 0, r.stderr[-2000:]
            outs.append(np.load(f))
    assert np.array_equal(outs[0], outs[1])


def test_ozaki_register_staged_variant():
    """The register-staged kernel (NSP_OZ_KERNEL=2, opt-in) computes the identical digit products: bitwise the
    same S_G X as the default kernel."""
    import subprocess, sys, os, tempfile
    code = (
        "import numpy as np, torch, sys\n"
        "sys.path.insert(0, %r)\n"
        "from tests.gpu_util import block, context, dev, problem\n"
        "pr, d, S = problem('cfg5s')\n"
        "ctx = context(pr, apply_kernel=3)\n"
        "X = dev(block(d.n_gamma, 128))\n"
        "Y = torch.empty_like(X)\n"
        "ctx.schur_apply(X, Y)\n"
        "torch.cuda.synchronize()\n"
        "np.save(sys.argv[1], Y.cpu().numpy())\n" % os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    outs = []
    with tempfile.TemporaryDirectory() as td:
        for kv in ("1", "2"):
            f = os.path.join(td, f"y{kv}.npy")
            env = dict(os.environ, NSP_OZ_KERNEL=kv)
            r = subprocess.run([sys.executable, "-c", code, f], env=env, capture_output=True, text=True, timeout=600)
            assert r.returncode == 0, r.stderr[-2000:]
            outs.append(np.load(f))
    assert np.array_equal(outs[0], outs[1])


@pytest.mark.parametrize("name", ["cfg2s", "cfg5s"])
def test_ozaki_work_counts(name):
    """nsp_ozaki_stats (the bench's INT8 roofline numerator): 28 slice products per (unit, K tile), i.e.
    28 sum ntb_j^2 in all; the executed count (leading-zero-slice skip) is no larger and no smaller than the
    count of units' first K tiles (never skipped); the unique slice bytes lie between those two bounds too."""
    pr, d, S = problem(name)
    ctx = context(pr, apply_kernel=3)
    st = ctx.stats()
    oz = ctx.ozaki_stats()
    t_l, t_w = st["l22_entries"] // 4096, st["wvu_rows"] // 64
    assert oz["slice_products_full"] == 28 * (2 * t_l - t_w)
    assert 28 * t_w <= oz["slice_products_executed"] <= oz["slice_products_full"]
    assert 7 * 4096 * t_w <= oz["m_slice_bytes"] <= 7 * 4096 * t_l
    print(f"{name}: executed {oz['slice_products_executed']} of {oz['slice_products_full']} slice products, "
          f"slice bytes {oz['m_slice_bytes']} of {7 * 4096 * t_l}")
    ctx.close()
