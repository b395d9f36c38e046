"""Diagnostic (GPU): cfg2s block CG with a duplicated and a zero right-hand-side column
at tol 1e-6 - per-iteration relres / widths of the GPU vs the oracle, and X at equal counts, to locate
where the free-running counts diverge.  Also the same without the degenerate columns."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))   # (tests/: may use the oracle)
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle as O  # noqa: E402
from tests.gpu_util import block, context, dev, problem, relfro  # noqa: E402


def run(B, tol, label, ks):
    pr, d, S = problem("cfg2s")
    ctx = context(pr)
    Xo, io = O.bf_bcg(S.apply, B, tol, 500)
    X = torch.zeros(d.n_gamma, B.shape[1], dtype=torch.float64, device="cuda")
    rep = ctx.block_cg(dev(B), X, tol, 500)
    print(f"{label}: gpu {rep['iters']} its fb {rep['fallbacks']}  oracle {io['iters']} fb {io['fallbacks']}")
    h_g, h_o = rep["hist"], io["relres"]
    for i in range(0, min(len(h_g), len(h_o)), 10):
        print(f"   it {i:4d} gpu {h_g[i]:.6e} oracle {h_o[i]:.6e} ratio {h_g[i] / h_o[i]:.6f}")
    print("   widths gpu", rep["widths"][:5], rep["widths"][-5:], " oracle", io["widths"][:5], io["widths"][-5:])
    for k in ks:
        Xk, ik = O.bf_bcg(S.apply, B, 0.0, k)
        X2 = torch.zeros_like(X)
        ctx.block_cg(dev(B), X2, 0.0, k)
        Xs, _ = O.bf_bcg(lambda V: S.dense() @ V, B, 0.0, k)
        print(f"   k={k}: gpu-vs-oracle {relfro(X2.cpu().numpy(), Xk):.3e}  oracle spread {relfro(Xs, Xk):.3e}")
    ctx.close()


if __name__ == "__main__":
    pr, d, S = problem("cfg2s")
    B = block(d.n_gamma, 8)
    run(B.copy(), 1e-6, "cfg2s 8 distinct columns", [1, 5, 20, 60, 100])
    B[:, 5] = B[:, 2]
    B[:, 7] = 0.0
    run(B, 1e-6, "cfg2s duplicate + zero column", [1, 5, 20, 60, 100, 130])
