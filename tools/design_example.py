"""The DESIGN.md usage example, runnable (diagnostics)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2101_12164_b200 import Context
from nsp_inputs import problems as P                     # any SPD CSR + a DBBD partition works
pr = P.make("cfg2")                                      # A (CSR, host), part[i] in [0, K) or -1 (Γ)
ctx = Context(pr.A.rowptr, pr.A.colidx, pr.A.val, pr.part, pr.K,
              factor_gamma=True)                         # setup: A_I_j factors, S_j^-1 tiles, A_Γ factor
nG, s = ctx.n_gamma, pr.s
Om = torch.randn(nG, s, dtype=torch.float64, device="cuda")
B = torch.empty_like(Om); X = torch.zeros_like(Om)
ctx.kgamma_apply(Om, B)                                  # a0: B = K_Γ Ω
rep = ctx.block_cg(B, X, 0.1, 500)                       # a1-a11: S_Γ X = B, breakdown-free block CG
rn = ctx.nystrom(100, 28, Om, 0.1, 500)                  # d1-d2: Alg. 2, builds M_2 in the context
b = torch.from_numpy(pr.rhs()).cuda(); x = torch.zeros_like(b)
rp = ctx.pcg(b, x, 1e-8, 5000, precond=2)                # d3: full solve A x = b with M_2
ctx.close()
print("iters", rep["iters"], "nystrom rank", rn["rank"], "pcg", rp["iters"], rp["converged"])
