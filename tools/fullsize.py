"""Full-size BASELINE.json configs on one B200 (the bench's launch configuration): setup time and
memory, S_G apply time, block CG to tol, sampled-row parity of the apply (when a reference row
function is passed in - tests/test_gpu_fullsize.py passes the oracle's
row-by-row definition, true residual of the block-CG solution through the parity-checked apply.
    python tools/fullsize.py cfg2 cfg3 cfg4 cfg5 [--rows 6]"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch

from nsp_inputs import philox
from nsp_inputs import problems as P
from paper_2101_12164_b200 import build as B
from paper_2101_12164_b200 import nsp


def run_pcg(name, maxit=5000):
    """Nystrom (Alg. 2) + outer PCG with M_2 at full size; x checked against x* (b = A x*) or by the
    true residual ||b - A x|| / ||b|| (host CSR matvec)."""
    B.build()
    pr = P.make(name)
    t0 = time.perf_counter()
    ctx = nsp.Context(pr.A.rowptr, pr.A.colidx, pr.A.val, pr.part, pr.K, factor_gamma=True)
    torch.cuda.synchronize()
    t_setup = time.perf_counter() - t0
    Om = torch.from_numpy(pr.omega()).cuda()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    rn = ctx.nystrom(pr.rank, pr.oversample, Om, pr.tol_bcg, 1000)
    torch.cuda.synchronize()
    t_nys = time.perf_counter() - t0
    b = pr.rhs()
    st = ctx.stats()
    out = dict(config=name, setup_s=round(t_setup, 2), ag_factor_ms=round(ctx.setup_report["t_ms"][3], 1),
               ag_solver=("chebyshev K=%d" % -st["ag_bw"]) if st["ag_bw"] < 0 else "band (RCM bw %d)" % st["ag_bw"],
               nystrom_s=round(t_nys, 3), nystrom_inner_iters=rn["iters"], nystrom_rank=rn["rank"],
               sigma_top=[float(x) for x in ctx.nystrom_sigma()[:3]])
    A = pr.A.to_scipy()
    precs = [int(x) for x in os.environ.get("NSP_PRECS", "1,2,3").split(",")]
    for prec in precs:   # S~_1, M_2, M_A-DEF2
        x = torch.zeros(pr.n, dtype=torch.float64, device="cuda")
        bd = torch.from_numpy(b).cuda()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        rep = ctx.pcg(bd, x, pr.tol_pcg, maxit, precond=prec)
        torch.cuda.synchronize()
        t = time.perf_counter() - t0
        xh = x.cpu().numpy()
        out[f"pcg_M{prec}"] = dict(iters=rep["iters"], converged=rep["converged"], s=round(t, 3),
                                   true_relres=float(np.linalg.norm(b - A @ xh) / np.linalg.norm(b)))
    ctx.close()
    return out


def run_pcg_plain(name, maxit=20000):
    """Outer PCG on the full system without a preconditioner (precond 0) at full size - for configs
    whose A_G band factor does not fit (cfg5): interior band + S_j^{-1} factors only."""
    B.build()
    pr = P.make(name)
    t0 = time.perf_counter()
    ctx = nsp.Context(pr.A.rowptr, pr.A.colidx, pr.A.val, pr.part, pr.K)
    torch.cuda.synchronize()
    t_setup = time.perf_counter() - t0
    b = pr.rhs()
    x = torch.zeros(pr.n, dtype=torch.float64, device="cuda")
    bd = torch.from_numpy(b).cuda()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    rep = ctx.pcg(bd, x, pr.tol_pcg or 1e-8, maxit, precond=0)
    torch.cuda.synchronize()
    t = time.perf_counter() - t0
    xh = x.cpu().numpy()
    A = pr.A.to_scipy()
    out = dict(config=name, setup_s=round(t_setup, 2), pcg_M0=dict(iters=rep["iters"], converged=rep["converged"],
               s=round(t, 3), true_relres=float(np.linalg.norm(b - A @ xh) / np.linalg.norm(b)),
               x_err=float(np.linalg.norm(xh - pr.xstar()) / np.linalg.norm(pr.xstar()))))
    ctx.close()
    return out


def run(name, nrows=6, maxit=1000, apply_kernel=0, ref_rows=None):
    """ref_rows(A, part, X, global_ids) -> reference rows of S_G X (the oracle's row-by-row definition,
    passed in by tests/test_gpu_fullsize.py; this diagnostics tool never imports the oracle itself)."""
    B.build()
    t0 = time.perf_counter()
    pr = P.make(name)
    t_gen = time.perf_counter() - t0
    free0 = torch.cuda.mem_get_info()[0]
    t0 = time.perf_counter()
    ctx = nsp.Context(pr.A.rowptr, pr.A.colidx, pr.A.val, pr.part, pr.K, apply_kernel=apply_kernel)
    torch.cuda.synchronize()
    t_setup = time.perf_counter() - t0
    used_setup = free0 - torch.cuda.mem_get_info()[0]
    s, nG = pr.s, ctx.n_gamma_local
    st = ctx.stats()
    X = torch.from_numpy(philox.gaussian_block(5, 9, nG, s)).cuda()
    Y = torch.empty_like(X)
    wsb = torch.empty(ctx.workspace_bytes(s), dtype=torch.uint8, device="cuda")
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for i in range(6):
        ev0.record()
        ctx.schur_apply(X, Y, wsb)
        ev1.record()
        torch.cuda.synchronize()
        if i:
            ts.append(ev0.elapsed_time(ev1))
    t_apply = float(np.median(ts))
    # sampled-row parity against a reference row function supplied by the caller (the tests)
    rng = np.random.default_rng(7)
    pick = np.sort(rng.choice(nG, size=min(nrows, nG), replace=False))
    gid = ctx.gamma_index()[pick]
    rel, t_oracle = None, 0.0
    if ref_rows is not None:
        t0 = time.perf_counter()
        ref = ref_rows(pr.A.to_scipy(), pr.part, X.cpu().numpy(), gid)
        t_oracle = time.perf_counter() - t0
        got = Y.cpu().numpy()[pick]
        rel = float(np.linalg.norm(got - ref) / np.linalg.norm(ref))
    # block CG on B = K_G Omega to tol
    Om = torch.from_numpy(pr.omega()).cuda()
    Bm = torch.empty_like(Om)
    ctx.kgamma_apply(Om, Bm, wsb)
    Xs = torch.zeros_like(Om)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    rep = ctx.block_cg(Bm, Xs, pr.tol_bcg, maxit, wsb)
    torch.cuda.synchronize()
    t_bcg = time.perf_counter() - t0
    R = torch.empty_like(Om)
    ctx.schur_apply(Xs, R, wsb)
    true_res = float(((Bm - R).norm(dim=0) / Bm.norm(dim=0)).max())
    out = dict(config=name, n=pr.n, nnz=pr.A.nnz, K=pr.K, s=s, n_gamma=nG, gen_s=round(t_gen, 1),
               setup_s=round(t_setup, 2), setup_ms=[round(x, 1) for x in ctx.setup_report["t_ms"][:5]],
               device_mem_gb=round(used_setup / 2**30, 2), boundary_rows=st["sum_b"], sum_b2=st["sum_b2"],
               apply_ms=round(t_apply, 3), rhs_applies_per_s=round(s / (t_apply * 1e-3), 1),
               apply_tflops=round(2.0 * st["sum_b2"] * s / (t_apply * 1e-3) / 1e12, 2),
               sampled_rows=len(pick), sampled_rel_err=rel, oracle_rows_s=round(t_oracle, 1),
               bcg_iters=rep["iters"], bcg_converged=rep["converged"], bcg_relres=rep["relres"],
               bcg_true_relres=true_res, bcg_s=round(t_bcg, 3), tol=pr.tol_bcg,
               widths_tail=rep["widths"][-3:])
    ctx.close()
    return out


if __name__ == "__main__":
    nrows = int(sys.argv[sys.argv.index("--rows") + 1]) if "--rows" in sys.argv else 6
    if "--pcg0" in sys.argv:
        for name in [a for a in sys.argv[1:] if a.startswith("cfg")]:
            print(json.dumps(run_pcg_plain(name)), flush=True)
        sys.exit(0)
    if "--pcg" in sys.argv:
        for name in [a for a in sys.argv[1:] if a.startswith("cfg")]:
            print(json.dumps(run_pcg(name)), flush=True)
        sys.exit(0)
    for name in [a for a in sys.argv[1:] if a.startswith("cfg")]:
        try:
            print(json.dumps(run(name, nrows)), flush=True)
        except Exception as e:  # report and continue with the next config
            print(json.dumps({"config": name, "error": repr(e)[:400]}), flush=True)
        torch.cuda.empty_cache()
