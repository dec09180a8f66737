"""CPU fp64 ORACLE for the sketched-and-truncated block Arnoldi method (arXiv 2311.16019).

*** TEST INFRASTRUCTURE ONLY. ***  Only `tests/`, `__graft_entry__.smoke()` and
`bench.py`'s cpu_baseline / `--impl reference` legs may import or execute
anything under `oracle/`.  The product path (`paper_2311_16019_b200/`) never
imports it and has no CPU fallback; the two share no code, only the seeded input
generators in `synth/` (which hold none of the method's arithmetic).

Plain, slow, obviously-correct NumPy/SciPy in fp64.  Every function cites the
PAPER.md passage it follows (``P:<line>`` = line of /root/reference/PAPER.md;
Alg. 1 = ``alg:whitening_krylov`` P:878-914).  Readings of garbled or silent
passages are listed in DESIGN.md §"Readings" and are cited here as (R<n>).

Modules
  sparse_sign  — the hashed sparse-sign embedding S (R1: the paper uses SRDCT,
                 BASELINE.json mandates sparse-sign with 8 nnz/column).
  operators    — the convection-diffusion stencils (assembled by Kronecker sums)
                 and CSR operators; B^T by explicit transpose.
  alg1         — Alg. 1 step by step: truncated block Arnoldi (MGS, Householder),
                 incremental sketched QR (CGS2), projected Sylvester solve,
                 sketched residual, check schedule, two-pass reconstruction,
                 true residual.
  alg2         — the paper's comparison methods: Alg. 2 (truncated Arnoldi without a
                 sketch, Prop. 3.2 residual bound) and the full Arnoldi /
                 Galerkin method.

Pins (tests/test_oracle_*.py, `-m "not gpu"`) tie each part to mathematics the
paper fixes; see DESIGN.md §"Oracle pins".  Parts with no pin say
"parity unpinned" in their docstring.
"""
from . import sparse_sign, operators, alg1, alg2  # noqa: F401
