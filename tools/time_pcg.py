"""Median time of the outer PCG (precond 2 = M_2) over repeated solves after warm-up (diagnostics).
    python tools/time_pcg.py cfg2 [reps]"""
import os, sys, time, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from nsp_inputs import problems as P
from paper_2101_12164_b200 import nsp
name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 7
pr = P.make(name)
ctx = nsp.Context(pr.A.rowptr, pr.A.colidx, pr.A.val, pr.part, pr.K, factor_gamma=True)
ctx.nystrom(pr.rank, pr.oversample, torch.from_numpy(pr.omega()).cuda(), pr.tol_bcg, 1000)
b = torch.from_numpy(pr.rhs()).cuda()
for prec in [int(x) for x in os.environ.get('NSP_PRECS', '2,1').split(',')]:
    ts, its = [], None
    for r in range(reps + int(os.environ.get('NSP_PCG_WARM', '2'))):
        x = torch.zeros_like(b)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        rep = ctx.pcg(b, x, pr.tol_pcg or 1e-8, 20000, precond=prec)
        torch.cuda.synchronize()
        if r >= int(os.environ.get('NSP_PCG_WARM', '2')):
            ts.append(time.perf_counter() - t0)
        its = rep["iters"]
    med = statistics.median(ts)
    print(f"{name} precond {prec}: {its} its, median {med * 1e3:.2f} ms, {med / its * 1e6:.1f} us/it", flush=True)
