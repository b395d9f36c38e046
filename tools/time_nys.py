"""Nystrom timing (diagnostics): repeated nsp_nystrom on one config after warm-up, wall time with a
device sync on both sides, plus the block-CG time of the same inner solve.
    python tools/time_nys.py cfg2 [reps]"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from nsp_inputs import problems as P  # noqa: E402
from paper_2101_12164_b200 import nsp  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 4
pr = P.make(name)
ctx = nsp.Context(pr.A.rowptr, pr.A.colidx, pr.A.val, pr.part, pr.K, factor_gamma=True)
Om = torch.from_numpy(pr.omega()).cuda()
for r in range(reps):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    rn = ctx.nystrom(pr.rank, pr.oversample, Om, pr.tol_bcg, 1000)
    torch.cuda.synchronize()
    print(f"{name} nystrom call {r}: {(time.perf_counter() - t0) * 1e3:.2f} ms, {rn['iters']} inner its", flush=True)
B = torch.empty_like(Om)
X = torch.empty_like(Om)
ctx.kgamma_apply(Om, B)
for r in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    rep = ctx.block_cg(B, X, pr.tol_bcg, 1000)
    torch.cuda.synchronize()
    print(f"{name} block_cg call {r}: {(time.perf_counter() - t0) * 1e3:.2f} ms, {rep['iters']} its", flush=True)
