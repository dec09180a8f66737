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


def variable_fd_matrix(dim: int, N: int, nu: float, wfun) -> sp.csr_matrix:
    """-nu Laplace + w . grad with a variable field w (the paper's Ex. 6.1 / 6.3
    operators), centred differences, Dirichlet, h = 1/(N+1), x fastest: assembled as
        A = nu L + sum_e diag(w_e(nodes)) D_e
    with L the Kronecker-sum Laplacian (stencil_matrix with w = 0) and D_e the Kronecker
    embedding of the 1-D central difference tridiag(-1, 0, 1) / (2h) along direction e.
    (The GPU receives the same operator as a CSR matrix assembled point by point in synth/;
    the pin test checks the two agree.)"""
    h = 1.0 / (N + 1)
    I = sp.identity(N, format="csr")
    D1 = sp.diags([-np.ones(N - 1), np.ones(N - 1)], [-1, 1], shape=(N, N), format="csr") / (2 * h)
    L = stencil_matrix(N, (0.0,) * dim, nu=nu)
    g = np.arange(1, N + 1) * h
    if dim == 2:
        Y, X = np.meshgrid(g, g, indexing="ij")
        w = wfun(X.ravel(), Y.ravel())
        Ds = [sp.kron(I, D1), sp.kron(D1, I)]
    else:
        Z, Y, X = np.meshgrid(g, g, g, indexing="ij")
        w = wfun(X.ravel(), Y.ravel(), Z.ravel())
        Ds = [sp.kron(sp.kron(I, I), D1), sp.kron(sp.kron(I, D1), I), sp.kron(sp.kron(D1, I), I)]
    A = L
    for e in range(dim):
        A = A + sp.diags(w[e]) @ Ds[e]
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
    elif getattr(cfg, "fd_dim", 0):
        from synth.inputs import VELOCITY              # the problem's velocity fields (input data)
        A = variable_fd_matrix(cfg.fd_dim, cfg.fd_N, cfg.nu, VELOCITY[cfg.wA_field])
        B = variable_fd_matrix(cfg.fd_dim, cfg.fd_N, cfg.nu, VELOCITY[cfg.wB_field])
    else:
        if csr_pair is None:
            from synth.inputs import config_csr
            csr_pair = config_csr(cfg)
        A = csr_from_triplet(csr_pair[0], cfg.n)
        B = csr_from_triplet(csr_pair[1], cfg.n)
    return A, sp.csr_matrix(B.T), B
