"""Parity at BASELINE.json's full size, in the bench's launch configuration (cfg2: n = 1.05M, K = 64,
s = 128): sampled rows of S_G X against the oracle's row-by-row definition (<= 1e-12), and the
block-CG solution meeting tol on the true residual through the (parity-checked) GPU apply."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_cfg2_fullsize_sampled_parity():
    from tools.fullsize import run
    r = run("cfg2", nrows=8)
    assert r["sampled_rel_err"] <= 1e-12, r
    assert r["bcg_converged"] and r["bcg_true_relres"] <= r["tol"] * 1.01, r
