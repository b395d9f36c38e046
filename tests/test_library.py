"""CPU checks of the C-ABI boundary: libnsp.so builds for sm_100a, loads, and exports every
symbol include/nsp.h declares; the binding refuses to run without a GPU (no CPU fallback)."""
import ctypes
import os
import re

import pytest

from paper_2101_12164_b200 import build as B
from paper_2101_12164_b200 import nsp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "nsp.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(nsp_[a-z_0-9]+)\s*\(", src)))


def test_header_symbols_exported():
    B.build()
    lib = ctypes.CDLL(B.LIB)
    decl = _declared()
    assert "nsp_setup" in decl and "nsp_block_cg" in decl and "nsp_pcg" in decl
    for name in decl:
        assert hasattr(lib, name), f"{name} declared in nsp.h but not exported"
    assert sorted(nsp.EXPORTED) == decl


def test_sass_has_dmma():
    import subprocess
    B.build()
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", B.LIB], capture_output=True, text=True).stdout
    assert "DMMA" in out, "fp64 tensor-pipe (DMMA) instructions missing from libnsp.so"
    # a2+a3 on the 5th-generation tensor cores (reading R10): tcgen05 kind::i8 MMAs (SS and TMEM-A forms),
    # smem -> TMEM copies, TMEM loads, and the bulk copies that feed them
    for m in ("UTCIMMA", "UTCCP", "LDTM", "UBLKCP"):
        assert m in out, f"{m} missing from libnsp.so"
    assert "sm_100a" in subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-lelf", B.LIB],
                                       capture_output=True, text=True).stdout


def test_no_cpu_fallback():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from nsp_inputs import problems as P
    pr = P.make("cfg1")
    with pytest.raises(RuntimeError, match="CUDA"):
        nsp.Context(pr.A.rowptr, pr.A.colidx, pr.A.val, pr.part, pr.K)


def test_default_opts_abi():
    lib = nsp.load_library()
    o = nsp.nsp_opts()
    lib.nsp_default_opts(ctypes.byref(o))
    assert o.nranks == 1 and o.orth_tau == 1e-14 and o.nys_eps_rel == 1e-12
