"""Host-side input validation of nsp_setup (SPEC.md:30-31 CSR well-formedness, SPEC.md:135 separator
property, part range): runs before any device call, so it is checked here on CPU through the raw C ABI
(NSP_ERR_ARG with a message naming the offending entry)."""
import ctypes as C

import numpy as np
import pytest

from nsp_inputs import problems as P
from paper_2101_12164_b200 import nsp


def _setup(rowptr, colidx, val, part, K, **opts):
    lib = nsp.load_library()
    rp = np.ascontiguousarray(rowptr, dtype=np.int64)
    ci = np.ascontiguousarray(colidx, dtype=np.int32)
    va = np.ascontiguousarray(val, dtype=np.float64)
    pa = np.ascontiguousarray(part, dtype=np.int32)
    csr = nsp.nsp_csr(rp.size - 1, rp.ctypes.data, ci.ctypes.data, va.ctypes.data)
    o = nsp.nsp_opts()
    lib.nsp_default_opts(C.byref(o))
    for k, v in opts.items():
        setattr(o, k, v)
    ctx = C.c_void_p()
    st = lib.nsp_setup(C.byref(csr), pa.ctypes.data, K, C.byref(o), C.byref(ctx), None)
    msg = lib.nsp_last_error(ctx).decode()
    lib.nsp_destroy(ctx)
    return st, msg


@pytest.fixture(scope="module")
def cfg1():
    return P.make("cfg1")


def test_separator_violation_named(cfg1):
    part = cfg1.part.copy()
    g = np.flatnonzero(part < 0)[5]          # put a separator node into a block: couples two blocks
    nb = cfg1.A.colidx[cfg1.A.rowptr[g]:cfg1.A.rowptr[g + 1]]
    blocks = sorted(set(part[nb][part[nb] >= 0].tolist()))
    part[g] = blocks[0]
    st, msg = _setup(cfg1.A.rowptr, cfg1.A.colidx, cfg1.A.val, part, cfg1.K)
    assert st == -1 and "separator property violated" in msg, msg


def test_part_out_of_range(cfg1):
    part = cfg1.part.copy()
    part[17] = cfg1.K
    st, msg = _setup(cfg1.A.rowptr, cfg1.A.colidx, cfg1.A.val, part, cfg1.K)
    assert st == -1 and "part[17]" in msg, msg


def test_unsorted_and_out_of_range_columns(cfg1):
    ci = cfg1.A.colidx.copy()
    r = 100
    a, b = cfg1.A.rowptr[r], cfg1.A.rowptr[r + 1]
    ci[a:b] = ci[a:b][::-1]
    st, msg = _setup(cfg1.A.rowptr, ci, cfg1.A.val, cfg1.part, cfg1.K)
    assert st == -1 and "row 100" in msg, msg
    ci = cfg1.A.colidx.copy()
    ci[-1] = cfg1.n + 5
    st, msg = _setup(cfg1.A.rowptr, ci, cfg1.A.val, cfg1.part, cfg1.K)
    assert st == -1 and "out-of-range" in msg, msg


def test_asymmetric(cfg1):
    va = cfg1.A.val.copy()
    r = 200
    q = cfg1.A.rowptr[r] + 1 if cfg1.A.colidx[cfg1.A.rowptr[r]] != r else cfg1.A.rowptr[r] + 1
    va[q] *= 1.5
    st, msg = _setup(cfg1.A.rowptr, cfg1.A.colidx, va, cfg1.part, cfg1.K)
    assert st == -1 and "not symmetric" in msg, msg


def test_empty_matrix():
    st, msg = _setup(np.zeros(1, np.int64), np.zeros(0, np.int32), np.zeros(0), np.zeros(0, np.int32), 1)
    assert st == -1, msg


@pytest.mark.parametrize("field,value", [("ag_order", 2), ("ag_order", -1), ("ag_solver", 3), ("nys_form", 4),
                                         ("nys_form", -1)])
def test_option_ranges(cfg1, field, value):
    """Out-of-range options (opts.ag_order 0..1, ag_solver 0..2, nys_form 0..3) are rejected on the host."""
    st, msg = _setup(cfg1.A.rowptr, cfg1.A.colidx, cfg1.A.val, cfg1.part, cfg1.K, **{field: value})
    assert st == -1 and field in msg, msg
