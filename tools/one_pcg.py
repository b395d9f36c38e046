"""Nystrom + a few outer PCG iterations with M_2 on a config (for ncu launch lists; diagnostics)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from nsp_inputs import problems as P
from paper_2101_12164_b200 import nsp, build as B
B.build()
pr = P.make(sys.argv[1] if len(sys.argv) > 1 else "cfg2")
its = int(sys.argv[2]) if len(sys.argv) > 2 else 10
ctx = nsp.Context(pr.A.rowptr, pr.A.colidx, pr.A.val, pr.part, pr.K, factor_gamma=True)
Om = torch.from_numpy(pr.omega()).cuda()
ctx.nystrom(pr.rank, pr.oversample, Om, pr.tol_bcg, 1000)
b = torch.from_numpy(pr.rhs()).cuda()
x = torch.zeros_like(b)
ctx.pcg(b, x, 0.0, its, precond=2)
torch.cuda.synchronize()
print("ok")
