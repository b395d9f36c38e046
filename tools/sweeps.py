"""Synthetic sweeps mirroring the paper's tab:compare_tolerance (eps_SI), tab:rank_variation (k) and
tab:oversampling_variation (p) on the B200 path: inner
block-CG iterations (it_S), outer PCG iterations with M_2 to 1e-8 (it_PCG), Nystrom and PCG times.
    python tools/sweeps.py cfg2 [--what tol,rank,over]"""
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


def one(ctx, pr, k, p, tol_inner, bcg_precond_ctx=None, maxit=5000):
    Om = torch.from_numpy(philox.gaussian_block(0, philox.STREAM_OMEGA, ctx.n_gamma, k + p)).cuda()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    rn = ctx.nystrom(k, p, Om, tol_inner, 1000)
    torch.cuda.synchronize()
    t_nys = time.perf_counter() - t0
    b = torch.from_numpy(pr.rhs()).cuda()
    x = torch.zeros_like(b)
    t0 = time.perf_counter()
    rp = ctx.pcg(b, x, pr.tol_pcg or 1e-8, maxit, precond=2)
    torch.cuda.synchronize()
    t_pcg = time.perf_counter() - t0
    return dict(k=k, p=p, eps_SI=tol_inner, it_S=rn["iters"], rank=rn["rank"], nystrom_s=round(t_nys, 3),
                it_PCG=rp["iters"], pcg_converged=rp["converged"], pcg_s=round(t_pcg, 3))


def variants(pr, tol_inner=0.1):
    """tab:compare_variations analog: it_total = inner block-CG iterations + outer
    PCG iterations for M_1, M_A-DEF1, M_2, M_A-DEF2, M_3, M_A-DEF3, and S~_1 (A_G^{-1} alone)."""
    out = {}
    b = torch.from_numpy(pr.rhs()).cuda()
    for form, lab in ((3, "1"), (0, "2"), (2, "3")):
        ctx = nsp.Context(pr.A.rowptr, pr.A.colidx, pr.A.val, pr.part, pr.K, factor_gamma=True, nys_form=form)
        rows = pr.n if form == 2 else ctx.n_gamma
        Om = torch.from_numpy(philox.gaussian_block(0, 5 if form == 2 else philox.STREAM_OMEGA, rows, pr.s)).cuda()
        rn = ctx.nystrom(pr.rank, pr.oversample, Om, tol_inner, 1000)
        for prec, name in ((2, f"M{lab}"), (3, f"M_A-DEF{lab}")):
            x = torch.zeros_like(b)
            r = ctx.pcg(b, x, pr.tol_pcg or 1e-8, 20000, precond=prec)
            out[name] = dict(it_inner=rn["iters"], it_pcg=r["iters"], it_total=rn["iters"] + r["iters"],
                             converged=r["converged"])
        if form == 0:
            x = torch.zeros_like(b)
            r = ctx.pcg(b, x, pr.tol_pcg or 1e-8, 20000, precond=1)
            out["S1"] = dict(it_pcg=r["iters"], it_total=r["iters"], converged=r["converged"])
        ctx.close()
    return out


def main():
    B.build()
    name = sys.argv[1] if len(sys.argv) > 1 and sys.argv[1].startswith("cfg") else "cfg2"
    what = sys.argv[sys.argv.index("--what") + 1].split(",") if "--what" in sys.argv else ["tol", "rank", "over"]
    pr = P.make(name)
    out = {"config": name}
    if "variants" in what:
        out["variants"] = variants(pr)
        print(json.dumps(out), flush=True)
        return
    for prec in (0, 1):   # reading C2: block CG with M = I and M = A_G^{-1}
        ctx = nsp.Context(pr.A.rowptr, pr.A.colidx, pr.A.val, pr.part, pr.K, factor_gamma=True, bcg_precond=prec)
        k0, p0 = pr.rank, pr.oversample
        if "tol" in what:
            out[f"tol_M{prec}"] = [one(ctx, pr, k0, p0, e) for e in (0.8, 0.5, 0.3, 0.1, 0.01)]
        if "rank" in what:
            out[f"rank_M{prec}"] = [one(ctx, pr, k, max(0, min(p0, 128 - k)), 0.1) for k in (5, 10, 20, 40, 80, 100)]
        if "over" in what:
            out[f"over_M{prec}"] = [one(ctx, pr, 20, p, 0.1) for p in (0, 5, 10, 20, 40)]
        ctx.close()
        print(json.dumps(out), flush=True)
    # unpreconditioned and A_G^{-1} (S~_1) references
    ctx = nsp.Context(pr.A.rowptr, pr.A.colidx, pr.A.val, pr.part, pr.K, factor_gamma=True)
    b = torch.from_numpy(pr.rhs()).cuda()
    for prec in (0, 1):
        x = torch.zeros_like(b)
        r = ctx.pcg(b, x, pr.tol_pcg or 1e-8, 20000, precond=prec)
        out[f"pcg_M{prec}_only"] = dict(iters=r["iters"], converged=r["converged"])
    ctx.close()
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
