"""B200-native Nystrom-Schur block-CG hot path (arXiv 2101.12164).

The product is the C-ABI library `libnsp.so` (include/nsp.h); `nsp` is the thin
ctypes binding (argument marshalling only).  There is no CPU fallback: if the
library or a CUDA device is missing, every call raises.
"""
from .nsp import Context, NspError, load_library  # noqa: F401
