"""Pins for oracle/operators.py and the synth CSR generator.

* Stencil assembly (Kronecker sums) vs a pure-Python loop over grid nodes that
  writes the centred-difference formula of -Laplace(u) + w.grad(u) directly.
* Closed-form spectrum of the 1-D factor tridiag(a, b, c):
  lambda_j = b + 2 sqrt(ac) cos(j pi/(N+1))  (catches a sign or index error in w/(2h)).
* B^T of a constant-coefficient central-difference stencil equals the stencil with -w
   -- the identity the GPU path relies on.
* CSR generator: band, distinct columns, diagonal = sum|offdiag| + 1, sorted rows.
"""
import math

import numpy as np
import pytest
import scipy.sparse as sp

from oracle import operators
from synth import inputs


def _loop_stencil(N, w):
    dim = len(w)
    h = 1.0 / (N + 1)
    n = N ** dim
    A = sp.lil_matrix((n, n))
    strides = [N ** e for e in range(dim)]
    for idx in range(n):
        coords = [(idx // strides[e]) % N for e in range(dim)]
        A[idx, idx] = 2.0 * dim / h**2
        for e in range(dim):
            if coords[e] + 1 < N:      # u_{x+e}
                A[idx, idx + strides[e]] += -1.0 / h**2 + w[e] / (2 * h)
            if coords[e] - 1 >= 0:     # u_{x-e}
                A[idx, idx - strides[e]] += -1.0 / h**2 - w[e] / (2 * h)
    return A.tocsr()


@pytest.mark.parametrize("N,w", [(5, (10.0, -3.0)), (4, (20.0, 20.0, 20.0)), (3, (-10.0, 10.0, 5.0))])
def test_stencil_matches_loop(N, w):
    A = operators.stencil_matrix(N, w)
    B = _loop_stencil(N, w)
    assert abs(A - B).max() < 1e-9 * abs(B).max()


def test_1d_factor_spectrum():
    N, w = 40, 7.0
    h = 1.0 / (N + 1)
    T = operators.tridiag_1d(N, w).toarray()
    a, b, c = -1 / h**2 - w / (2 * h), 2 / h**2, -1 / h**2 + w / (2 * h)
    lam = np.sort(b + 2 * math.sqrt(a * c) * np.cos(np.arange(1, N + 1) * math.pi / (N + 1)))
    got = np.sort(np.linalg.eigvals(T).real)
    assert np.allclose(got, lam, rtol=1e-9)
    assert T[1, 0] == pytest.approx(a) and T[0, 1] == pytest.approx(c)


def test_2d_spectrum_is_kronecker_sum():
    N, w = 9, (3.0, -5.0)
    A = operators.stencil_matrix(N, w).toarray()
    l1 = np.linalg.eigvals(operators.tridiag_1d(N, w[0]).toarray()).real
    l2 = np.linalg.eigvals(operators.tridiag_1d(N, w[1]).toarray()).real
    want = np.sort((l1[:, None] + l2[None, :]).ravel())
    assert np.allclose(np.sort(np.linalg.eigvals(A).real), want, rtol=1e-9)


@pytest.mark.parametrize("N,w", [(6, (-5.0, 5.0)), (4, (-10.0, 10.0, 5.0))])
def test_transpose_is_negated_convection(N, w):
    B = operators.stencil_matrix(N, w)
    Bneg = operators.stencil_matrix(N, tuple(-x for x in w))
    assert abs(B.T - Bneg).max() < 1e-9 * abs(B).max()


def test_banded_csr_properties():
    n, m, band = 3000, 20, 64
    rp, col, val = inputs.banded_csr(n, m, band, seed=1)
    assert rp.dtype == np.int64 and col.dtype == np.int32
    assert np.all(np.diff(rp) == m + 1)
    C = col.reshape(n, m + 1).astype(np.int64)
    V = val.reshape(n, m + 1)
    i = np.arange(n)[:, None]
    assert np.all(np.diff(C, axis=1) > 0)                     # sorted, distinct
    assert np.all(np.abs(C - i) <= band)
    isdiag = C == i
    assert np.all(isdiag.sum(axis=1) == 1)
    diag = V[isdiag]
    off = np.where(isdiag, 0.0, np.abs(V)).sum(axis=1)
    assert np.allclose(diag, off + 1.0)
    # deterministic for the seed, different across seeds
    rp2, col2, val2 = inputs.banded_csr(n, m, band, seed=1)
    assert np.array_equal(col, col2) and np.array_equal(val, val2)
    assert not np.array_equal(col, inputs.banded_csr(n, m, band, seed=2)[1])
