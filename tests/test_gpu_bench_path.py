"""Oracle parity of the BENCH's exact code path (full-size cfg2 = BASELINE.json configs[1]: n = 1.05M,
K = 64, n_G = 14,287, s = 128, tol 0.1, B = K_G Omega) - the path the driver times: the one-wave s = 128
panel (k_panel_rows), the symmetric W^T W Gram and the [D | E] Gram, inside the device-driven block-CG
graph.  The oracle is oracle.bf_bcg (reading C3 step by step) on oracle.LocalSchurOracle (S_G from dense
local blocks; pinned in tests/test_oracle_pins.py), computed live on the host.

Checks (north_star):
  - path counters: k_panel_rows, the symmetric Gram and the [D | E] Gram were dispatched;
  - equal counts k in {1, 2, 3}: X within max(1e-8, 10 x the oracle's own local-vs-dense spread at k,
    committed in tests/golden/cfg2_bcg_oracle.json) and IDENTICAL active widths;
  - free-running: converged, iteration count within +-1 of the oracle's (live, and equal to the
    committed golden count), true residual ||B - S_G X|| / ||B|| <= tol through the ORACLE's S_G;
for M = I (the bench's headline mode) and M = A_G^{-1} (reading C2's paper-analog mode)."""
import json
import os

import numpy as np
import pytest
import torch

import oracle as O
from nsp_inputs import problems as P
from paper_2101_12164_b200 import nsp
from tests.gpu_util import context, dev, relfro

pytestmark = pytest.mark.gpu

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "cfg2_bcg_oracle.json")
_ST = {}


def _threads():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def _setup():
    if not _ST:
        pr = P.make("cfg2")
        d = O.dbbd(pr.A.to_scipy(), pr.part, pr.K)
        S = O.SchurOracle(d, threads=_threads())
        S.factor_all()
        L = O.LocalSchurOracle(d, threads=_threads(), schur=S)
        B = L.k_gamma(pr.omega())
        ctx = context(pr, factor_gamma=True)
        assert np.array_equal(ctx.gamma_index(), d.gamma)
        _ST.update(pr=pr, d=d, S=S, L=L, B=B, ctx=ctx, gold=json.load(open(GOLD)))
    return _ST


@pytest.mark.parametrize("mode", ["I", "AG_inv"])
def test_bench_path_bcg_parity_cfg2(mode):
    st = _setup()
    pr, S, L, B, ctx, gold = st["pr"], st["S"], st["L"], st["B"], st["ctx"], st["gold"]["modes"][mode]
    apply_M = S.solve_AG if mode == "AG_inv" else None
    ctx.set_bcg_precond(1 if mode == "AG_inv" else 0)
    Bd = dev(B)
    X = torch.zeros_like(Bd)
    ws = torch.empty(ctx.workspace_bytes(pr.s), dtype=torch.uint8, device="cuda")
    # free-running (the bench's call)
    c0 = nsp.path_counters()
    rep = ctx.block_cg(Bd, X, pr.tol_bcg, 500, ws)
    c1 = nsp.path_counters()
    Xo, io = O.bf_bcg(L.apply, B, pr.tol_bcg, 500, apply_M=apply_M)
    print(f"cfg2 M={mode}: gpu {rep['iters']} its, oracle {io['iters']} (golden {gold['iters']})")
    assert io["iters"] == gold["iters"] and io["widths"] == gold["widths"]
    assert rep["status"] == 0 and rep["converged"]
    assert abs(rep["iters"] - io["iters"]) <= 1, (rep["iters"], io["iters"])
    Xg = X.cpu().numpy()
    true_res = np.linalg.norm(B - L.apply(Xg), axis=0) / np.linalg.norm(B, axis=0)
    assert true_res.max() <= pr.tol_bcg * 1.001, true_res.max()
    # the bench's kernels ran: one-wave panel, symmetric W^T W, [D | E], a2+a3 on the INT8 tensor cores
    for k in ("panel_rows", "gram_sym", "gram_de", "ozaki"):
        assert c1[k] > c0[k], (k, c0, c1)
    # equal iteration counts (reading C16)
    for k in (1, 2, 3):
        Xk, ik = O.bf_bcg(L.apply, B, 0.0, k, apply_M=apply_M)
        X2 = torch.zeros_like(Bd)
        rep2 = ctx.block_cg(Bd, X2, 0.0, k, ws)
        assert rep2["iters"] == k
        diff = relfro(X2.cpu().numpy(), Xk)
        spread = gold["spread_local_vs_dense"][str(k)]
        print(f"  k={k}: gpu-vs-oracle {diff:.2e}, oracle spread {spread:.2e}")
        assert diff <= max(1e-8, 10 * spread), (k, diff, spread)
        assert rep2["widths"] == ik["widths"]
    # the whole free-running solve at the oracle's count
    kk = io["iters"]
    X3 = torch.zeros_like(Bd)
    ctx.block_cg(Bd, X3, 0.0, kk, ws)
    diff = relfro(X3.cpu().numpy(), Xo)
    spread = gold["spread_local_vs_dense"][str(kk)]
    print(f"  k={kk}: gpu-vs-oracle {diff:.2e}, oracle spread {spread:.2e}")
    assert diff <= max(1e-8, 10 * spread), (kk, diff, spread)


def test_fused_panel_gram_path_parity_cfg2():
    """The fused s = 128 panel + Gram passes (k_panel_gram: R -= Q alpha with F = Q^T R, W = R + P beta with
    W^T W) that the bench dispatches at cfg5 (n_G >= 512 x SMs), forced on at cfg2 so the ORACLE can check
    them: free-running count = the oracle's (+-1), X at equal counts k in {1, 2, 3, 60} within
    max(1e-8, 10 x spread)."""
    st = _setup()
    pr, L, B, gold = st["pr"], st["L"], st["B"], st["gold"]["modes"]["I"]
    ctx = context(pr)                      # fresh context: its graphs are captured with the fused passes
    nsp.dev_set_fused_pg(1)
    try:
        Bd = dev(B)
        X = torch.zeros_like(Bd)
        ws = torch.empty(ctx.workspace_bytes(pr.s), dtype=torch.uint8, device="cuda")
        c0 = nsp.path_counters()
        rep = ctx.block_cg(Bd, X, pr.tol_bcg, 500, ws)
        c1 = nsp.path_counters()
        assert c1["panel_gram"] > c0["panel_gram"], (c0, c1)
        print(f"cfg2 fused panel+Gram: gpu {rep['iters']} its, golden {gold['iters']}")
        assert rep["converged"] and abs(rep["iters"] - gold["iters"]) <= 1
        for k in (1, 2, 3, gold["iters"]):
            Xk, ik = O.bf_bcg(L.apply, B, 0.0, k)
            X2 = torch.zeros_like(Bd)
            rep2 = ctx.block_cg(Bd, X2, 0.0, k, ws)
            diff = relfro(X2.cpu().numpy(), Xk)
            spread = gold["spread_local_vs_dense"][str(k)]
            print(f"  k={k}: gpu-vs-oracle {diff:.2e}, oracle spread {spread:.2e}")
            assert diff <= max(1e-8, 10 * spread), (k, diff, spread)
            assert rep2["widths"] == ik["widths"]
    finally:
        nsp.dev_set_fused_pg(0)
        ctx.close()
