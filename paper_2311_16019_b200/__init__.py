"""paper_2311_16019_b200 — B200-native (sm_100a) sketched-and-truncated block Krylov
solver for the low-rank Sylvester equation A X + X B = C1 C2^T (arXiv 2311.16019, Alg. 1).

The product is the C-ABI shared library `libsylvsketch.so` (include/sylv_sketch.h);
this package is a thin ctypes binding (api.py) plus its build script (build.py).
"""
from .api import (SylvSketch, SylvError, Operator, Config, Stats, stencil_operator,  # noqa: F401
                  csr_operator, operators_for, from_config, load_library, version, LIB_PATH, SYMBOLS,
                  partition, Comm, LocalGroup, nccl_comm, wrap_nccl)
