"""Writes tests/golden/cfg2_bcg_oracle.json: the ORACLE's breakdown-free block-CG run on the full-size
cfg2 workload (BASELINE.json configs[1]: 1024^2 anisotropic, K = 64, s = 128, tol 0.1, B = K_G Omega,
Omega = Philox seed 0), for M = I and M = A_G^{-1} (reading C2): iteration counts, active widths,
relres history, and the oracle's own evaluation-order spread of X at equal counts.

Calls only oracle/ and nsp_inputs/ (no CUDA path).  The spread compares two exact evaluations of the
same operator - S_G assembled from dense local blocks (LocalSchurOracle, the test's oracle) against the
fully dense S_G (A_G - sum_j E_j^T K_j E_j accumulated into one n_G x n_G matrix) - running the same
algorithm (oracle.bf_bcg): it is the rounding sensitivity of block CG itself on this workload
(DESIGN.md "Parity tolerances").

    python tests/golden/make_cfg2_bcg.py [threads]
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import oracle as O  # noqa: E402
from nsp_inputs import problems as P  # noqa: E402


def relfro(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def main():
    threads = int(sys.argv[1]) if len(sys.argv) > 1 else (os.cpu_count() or 1)
    t0 = time.time()
    pr = P.make("cfg2")
    d = O.dbbd(pr.A.to_scipy(), pr.part, pr.K)
    S = O.SchurOracle(d, threads=threads)
    S.factor_all()
    L = O.LocalSchurOracle(d, threads=threads, schur=S)
    print(f"oracle setup {time.time() - t0:.1f} s", flush=True)
    B = L.k_gamma(pr.omega())
    Sd = d.A_G.toarray()
    for r, Kj in zip(L.rows, L.K):
        Sd[np.ix_(r, r)] -= Kj
    out = {"config": "cfg2", "s": pr.s, "tol": pr.tol_bcg, "n_gamma": d.n_gamma, "omega_seed": 0,
           "generator": "tests/golden/make_cfg2_bcg.py (oracle.bf_bcg on oracle.LocalSchurOracle)", "modes": {}}
    for mode, apply_M in [("I", None), ("AG_inv", S.solve_AG)]:
        t0 = time.time()
        X, info = O.bf_bcg(L.apply, B, pr.tol_bcg, 500, apply_M=apply_M)
        it = info["iters"]
        spread = {}
        for k in sorted({1, 2, 3, it // 2, it}):
            Xl, _ = O.bf_bcg(L.apply, B, 0.0, k, apply_M=apply_M)
            Xd, _ = O.bf_bcg(lambda V: Sd @ V, B, 0.0, k, apply_M=apply_M)
            spread[str(k)] = relfro(Xd, Xl)
        out["modes"][mode] = {"iters": it, "status": info["status"], "widths": info["widths"],
                              "relres": info["relres"], "fallbacks": info["fallbacks"],
                              "spread_local_vs_dense": spread}
        print(mode, it, spread, f"{time.time() - t0:.1f} s", flush=True)
    with open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "cfg2_bcg_oracle.json"), "w") as f:
        json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
