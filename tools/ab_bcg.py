"""A/B timing (diagnostics): block CG time-to-tol (M = I and, with --analog, M = A_G^-1) and the S_G
apply on one config, median of repeated solves after warm-up, L2 flushed before each.  The kernel
variants are selected by environment variables read once per process (NSP_FUSED_SXS, NSP_FUSED_PG,
NSP_SPMM_V, ...), so each variant is its own process:
    NSP_FUSED_PG=0 python tools/ab_bcg.py cfg2 [reps] [--analog]"""
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from nsp_inputs import problems as P  # noqa: E402
from paper_2101_12164_b200 import nsp  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
reps = int(sys.argv[2]) if len(sys.argv) > 2 and sys.argv[2].isdigit() else 9
pr = P.make(name)
ctx = nsp.Context(pr.A.rowptr, pr.A.colidx, pr.A.val, pr.part, pr.K, factor_gamma="--analog" in sys.argv)
s = pr.s
Om = torch.from_numpy(pr.omega()).cuda()
B = torch.empty_like(Om)
X = torch.empty_like(Om)
ws = torch.empty(ctx.workspace_bytes(s), dtype=torch.uint8, device="cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
ctx.kgamma_apply(Om, B, ws)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)


def timed(fn, n):
    out = []
    for _ in range(n):
        flush.zero_()
        e0.record()
        r = fn()
        e1.record()
        torch.cuda.synchronize()
        out.append((e0.elapsed_time(e1), r))
    return out


res = {"config": name, "env": {k: v for k, v in os.environ.items() if k.startswith("NSP_")}}
for mode in ([0, 1] if "--analog" in sys.argv else [0]):
    ctx.set_bcg_precond(mode)
    timed(lambda: ctx.block_cg(B, X, pr.tol_bcg, 1000, ws), 3)
    t = timed(lambda: ctx.block_cg(B, X, pr.tol_bcg, 1000, ws), reps)
    med = statistics.median(x for x, _ in t)
    its = t[-1][1]["iters"]
    res[f"bcg_M{mode}"] = {"ms": round(med, 3), "iters": its, "us_per_iter": round(med / its * 1e3, 1)}
P_ = torch.randn_like(Om)
Q_ = torch.empty_like(Om)
t = timed(lambda: ctx.schur_apply(P_, Q_, ws), reps + 3)[3:]
res["apply_ms"] = round(statistics.median(x for x, _ in t), 4)
print(json.dumps(res), flush=True)
