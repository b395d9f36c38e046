"""Time A_G^{-1} (precond_apply 1) on a config, s = 1 and s = 100 (diagnostics)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from nsp_inputs import problems as P
from paper_2101_12164_b200 import nsp
name = sys.argv[1] if len(sys.argv) > 1 else "cfg5"
pr = P.make(name)
ctx = nsp.Context(pr.A.rowptr, pr.A.colidx, pr.A.val, pr.part, pr.K, factor_gamma=True,
                  ag_solver=int(os.environ.get("AGS", "0")))
print("stats", ctx.stats()["ag_bw"], flush=True)
n = ctx.n_gamma
for s in (1, 100):
    X = torch.randn(n, s, dtype=torch.float64, device="cuda"); Y = torch.empty_like(X)
    ws = torch.empty(ctx.workspace_bytes(128) // 8 + 1, dtype=torch.float64, device="cuda")
    ctx.precond_apply(1, X, Y); torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3): ctx.precond_apply(1, X, Y)
    e1.record(); torch.cuda.synchronize()
    print(name, "s", s, "A_G^-1 ms", e0.elapsed_time(e1) / 3, flush=True)
