"""CPU oracle for the Nystrom-Schur block-CG hot path (arXiv 2101.12164).

TEST INFRASTRUCTURE ONLY.  Plain, slow, obviously-correct fp64 numpy/scipy
implementations of what the hot path computes, each function citing the paper
passage it follows.  Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s
`cpu_baseline` / `--impl reference` legs may import anything from here; the
product package `paper_2101_12164_b200` never does, and this package never
imports the product package (they share no code; only `nsp_inputs` - the seeded
input generators - serves both).

Pin status (DESIGN.md §"Oracle pins"): every function below is pinned by a
`-m "not gpu"` test in tests/test_oracle_pins.py against something other than
itself (closed forms, brute-force elimination, exact-arithmetic termination,
exactness) except where a docstring says "parity unpinned".
"""
from .dbbd import DBBD, dbbd  # noqa: F401
from .schur import LocalSchurOracle, SchurOracle  # noqa: F401
from .bcg import bf_bcg, orth  # noqa: F401
from .nystrom import nystrom_schur, nystrom_m1, NystromResult  # noqa: F401
from .pcg import pcg, solve_full_system  # noqa: F401
from .si import SIOperator, interior_rows, nystrom_schur_si, nystrom_si_inverse  # noqa: F401
