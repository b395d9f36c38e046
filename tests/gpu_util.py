"""Shared helpers of the -m gpu parity tests (inputs from nsp_inputs, expected values from oracle/)."""
import numpy as np
import torch

import oracle as O
from nsp_inputs import philox
from nsp_inputs import problems as P
from paper_2101_12164_b200 import Context

_CACHE = {}


def problem(name):
    if name not in _CACHE:
        pr = P.make(name)
        d = O.dbbd(pr.A.to_scipy(), pr.part, pr.K)
        _CACHE[name] = (pr, d, O.SchurOracle(d))
    return _CACHE[name]


def context(pr, **kw):
    return Context(pr.A.rowptr, pr.A.colidx, pr.A.val, pr.part, pr.K, **kw)


def block(rows, cols, seed=7, stream=9):
    return philox.gaussian_block(seed, stream, rows, cols)


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).to("cuda", torch.float64)


def relfro(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))
