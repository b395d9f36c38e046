"""Time the A_G^{-1} band solve (nsp_precond_apply which=1) and the S_G apply at s = 1, 32, 128 (diagnostics)."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from nsp_inputs import problems as P
from paper_2101_12164_b200 import nsp, build as B
B.build()
name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
pr = P.make(name)
ctx = nsp.Context(pr.A.rowptr, pr.A.colidx, pr.A.val, pr.part, pr.K, factor_gamma=True)
st = ctx.stats()
out = {"config": name, "ag_bw": st["ag_bw"], "n_gamma": ctx.n_gamma}
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for s in (1, 32, 128):
    X = torch.randn(ctx.n_gamma, s, dtype=torch.float64, device="cuda")
    Y = torch.empty_like(X)
    for which, lab in ((1, "ag_solve"), (-1, "schur_apply")):
        ts = []
        for i in range(8):
            e0.record()
            if which == 1:
                ctx.precond_apply(1, X, Y)
            else:
                ctx.schur_apply(X, Y)
            e1.record(); torch.cuda.synchronize()
            if i >= 3: ts.append(e0.elapsed_time(e1))
        out[f"{lab}_s{s}_ms"] = round(min(ts), 4)
print(json.dumps(out))
