"""Seeded synthetic input generators shared by the oracle tests and the CUDA path.

This package holds NO arithmetic of the method (no operator application, no
orthogonalisation, no sketch, no projected solve).  It only draws the random
inputs that BASELINE.json's configs describe and tabulates the config sizes:

* the right-hand-side factors C1, C2 (iid N(0,1), PCG64 seeds, optional column
  normalisation), and
* the banded random CSR matrices of config c4 (a random *input*, not the method).

Both `oracle/` and `paper_2311_16019_b200/` consume these; neither imports the
other.
"""
from .inputs import (CONFIGS, Config, ZETA, SKETCH_SEEDS, TOL, make_rhs, banded_csr,  # noqa: F401
                     config_csr, get_config, small_config)
