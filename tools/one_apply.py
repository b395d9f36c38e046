"""S_G applies at width s with a chosen apply_kernel, timed with CUDA events (and for ncu launch lists):
python tools/one_apply.py cfg2 128 3 [reps]."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from nsp_inputs import problems as P
from paper_2101_12164_b200 import nsp, build as B
B.build()
pr = P.make(sys.argv[1] if len(sys.argv) > 1 else "cfg2")
s = int(sys.argv[2]) if len(sys.argv) > 2 else 128
ak = int(sys.argv[3]) if len(sys.argv) > 3 else 0
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 10
ctx = nsp.Context(pr.A.rowptr, pr.A.colidx, pr.A.val, pr.part, pr.K, apply_kernel=ak)
X = torch.randn(ctx.n_gamma, s, dtype=torch.float64, device="cuda")
Y = torch.empty_like(X)
ws = torch.empty(ctx.workspace_bytes(s), dtype=torch.uint8, device="cuda")
ctx.schur_apply(X, Y, ws)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(reps):
    ctx.schur_apply(X, Y, ws)
e1.record()
torch.cuda.synchronize()
print(f"{pr.name if hasattr(pr, 'name') else sys.argv[1]} s={s} apply_kernel={ak}: {e0.elapsed_time(e1) / reps:.4f} ms per S_G apply")
