"""Diagnostics: the bench's call sequence on one config (steps, profiling pass, applies, e2e, paper-analog,
then Nystrom twice) with the time of every Nystrom call - to locate a slowdown that appears only after it."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from nsp_inputs import problems as P  # noqa: E402
from paper_2101_12164_b200 import nsp  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
pr = P.make(name)
ctx = nsp.Context(pr.A.rowptr, pr.A.colidx, pr.A.val, pr.part, pr.K, factor_gamma=True)
Om = torch.from_numpy(pr.omega()).cuda()
B, X, Y = torch.empty_like(Om), torch.empty_like(Om), torch.empty_like(Om)
ws = torch.empty(ctx.workspace_bytes(pr.s), dtype=torch.uint8, device="cuda")


def nys(tag):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    r = ctx.nystrom(pr.rank, pr.oversample, Om, pr.tol_bcg, 1000)
    torch.cuda.synchronize()
    print(f"{tag}: nystrom {(time.perf_counter() - t0) * 1e3:.2f} ms ({r['iters']} its)", flush=True)


def step():
    ctx.kgamma_apply(Om, B, ws)
    r = ctx.block_cg(B, X, pr.tol_bcg, 1000, ws)
    ctx.gamma_apply(X, Y)
    return r


nys("fresh")
nys("fresh again")
for _ in range(5):
    step()
nys("after steps")
ctx.profile(True)
for _ in range(3):
    step()
ctx.profile_read()
ctx.profile(False)
nys("after profile pass")
ctx.set_bcg_precond(1)
for _ in range(3):
    step()
ctx.set_bcg_precond(0)
nys("after analog")
nys("after analog again")
