"""One A_G^{-1} solve at s (for ncu launch lists; diagnostics)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from nsp_inputs import problems as P
from paper_2101_12164_b200 import nsp, build as B
B.build()
pr = P.make(sys.argv[1] if len(sys.argv) > 1 else "cfg2")
s = int(sys.argv[2]) if len(sys.argv) > 2 else 128
ctx = nsp.Context(pr.A.rowptr, pr.A.colidx, pr.A.val, pr.part, pr.K, factor_gamma=True)
X = torch.randn(ctx.n_gamma, s, dtype=torch.float64, device="cuda")
Y = torch.empty_like(X)
for _ in range(2):
    ctx.precond_apply(1, X, Y)
torch.cuda.synchronize()
print("ok")
