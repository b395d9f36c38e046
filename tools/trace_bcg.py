"""Phase timing of one cfg block-CG solve (NSP_TRACE=1 event tracer in libnsp)."""
import os, sys, time
os.environ["NSP_TRACE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from nsp_inputs import problems as P
from paper_2101_12164_b200 import Context
name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
pr = P.make(name)
ctx = Context(pr.A.rowptr, pr.A.colidx, pr.A.val, pr.part, pr.K)
Om = torch.from_numpy(pr.omega()).cuda()
B = torch.empty_like(Om); X = torch.empty_like(Om)
ctx.kgamma_apply(Om, B)
for rep in range(2):
    torch.cuda.synchronize(); t = time.perf_counter()
    r = ctx.block_cg(B, X, pr.tol_bcg, 1000)
    torch.cuda.synchronize(); print("wall ms", (time.perf_counter() - t) * 1e3, "iters", r["iters"], file=sys.stderr)
