"""Coefficient matrices A, B^T of A X + X B = C1 C2^T (oracle side, assembled explicitly).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Convection-diffusion operator L(u) = -nu*Laplace(u) + w.grad(u) (P:972-975,
eq. condiff_op), discretised by centred finite differences on the unit square /
cube with homogeneous Dirichlet BCs, N interior nodes per direction, h = 1/(N+1),
nu = 1, lexicographic ordering with x fastest (readings R14-R16 in DESIGN.md;
BASELINE.json configs 0-3).

The oracle assembles the 1-D factor
    T(w) = tridiag(-1/h^2 - w/(2h),  2/h^2,  -1/h^2 + w/(2h))   [(i,i-1), (i,i), (i,i+1)]
and Kronecker-sums it: 2-D  A = I (x) T(w_x) + T(w_y) (x) I ; 3-D analogously.
B^T is formed by an explicit sparse transpose (the GPU path uses the equivalent
"stencil with -w" identity; the oracle deliberately does not).
"""
from __future__ import annotations

import numpy as np
import scipy.sparse as sp


def tridiag_1d(N: int, w: float, nu: float = 1.0) -> sp.csr_matrix:
    h = 1.0 / (N + 1)
    lower = np.full(N - 1, -nu / h**2 - w / (2 * h))
    main = np.full(N, 2.0 * nu / h**2)
    upper = np.full(N - 1, -nu / h**2 + w / (2 * h))
    return sp.diags([lower, main, upper], [-1, 0, 1], shape=(N, N), format="csr")


def stencil_matrix(N: int, w, nu: float = 1.0) -> sp.csr_matrix:
    """Centred-FD matrix of -nu*Laplace + w.grad on N^dim interior nodes (dim = len(w))."""
    dim = len(w)
    I = sp.identity(N, format="csr")
    factors = [tridiag_1d(N, float(wi), nu) for wi in w]
    if dim == 2:
        A = sp.kron(I, factors[0]) + sp.kron(factors[1], I)
    elif dim == 3:
        A = (sp.kron(sp.kron(I, I), factors[0]) + sp.kron(sp.kron(I, factors[1]), I)
             + sp.kron(sp.kron(factors[2], I), I))
    else:
        raise ValueError("dim must be 2 or 3")
    return sp.csr_matrix(A)


def csr_from_triplet(trip, n: int) -> sp.csr_matrix:
    row_ptr, col, val = trip
    return sp.csr_matrix((val, col.astype(np.int64), row_ptr), shape=(n, n))


def operator_pair(cfg, csr_pair=None):
    """(A, B^T, B) as scipy CSR for a synth.Config.  For 'csr' configs pass the
    (A, B) triplets from synth.config_csr (or they are generated here)."""
    if cfg.kind.startswith("stencil"):
        A = stencil_matrix(cfg.N, cfg.wA)
        B = stencil_matrix(cfg.N, cfg.wB)
    else:
        if csr_pair is None:
            from synth.inputs import config_csr
            csr_pair = config_csr(cfg)
        A = csr_from_triplet(csr_pair[0], cfg.n)
        B = csr_from_triplet(csr_pair[1], cfg.n)
    return A, sp.csr_matrix(B.T), B
