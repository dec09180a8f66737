"""Pins for the paper-workload parts of the oracle:

  variable-coefficient operators (Ex. 6.1 / 6.3): the oracle's Kronecker assembly
      nu L + sum_e diag(w_e) D_e equals synth's point-by-point CSR (the GPU's input) and reduces
      to the constant-coefficient stencil (itself pinned in test_oracle_operators) for constant w;
      a hand-computed row of the 2-D operator
  SRDCT (R2): the orthonormal DCT-II equals the explicit cosine matrix on small n; the
      sketch preserves norms in expectation with the sqrt(n/s) scale (and the printed sqrt(s/n)
      does not); sigma^2(S V) of random orthonormal V lies near the Marchenko-Pastur edges
"""
import math

import numpy as np
import pytest
import scipy.sparse as sp

from oracle import alg1, operators
from oracle.srdct import SRDCT
from synth import inputs


@pytest.mark.parametrize("dim,N,nu,field", [(2, 9, 0.01, "ex61_B"), (2, 7, 0.1, "ex61_A"), (3, 6, 0.005, "ex63_A"),
                                            (3, 5, 0.005, "ex63_B")])
def test_variable_fd_operator_matches_synth_csr(dim, N, nu, field):
    A = operators.variable_fd_matrix(dim, N, nu, inputs.VELOCITY[field])
    rp, ci, v = inputs.fd_csr(dim, N, nu, field)
    B = sp.csr_matrix((v, ci.astype(np.int64), rp), shape=A.shape)
    assert abs(A - B).max() <= 1e-12 * abs(A).max()


def test_variable_fd_constant_field_is_the_stencil():
    A = operators.variable_fd_matrix(2, 8, 1.0, inputs.VELOCITY["ex61_A"])     # w = (1, 1)
    assert abs(A - operators.stencil_matrix(8, (1.0, 1.0))).max() <= 1e-12 * abs(A).max()


def test_variable_fd_hand_computed_row():
    """Row of node (i, j) = (2, 3) (1-based, h = 1/(N+1)) of -nu Lap + w . grad, w = ex61_B."""
    N, nu = 6, 0.1
    h = 1.0 / (N + 1)
    A = operators.variable_fd_matrix(2, N, nu, inputs.VELOCITY["ex61_B"]).toarray()
    i, j = 2, 3
    x, y = i * h, j * h
    wx, wy = 3 * y * (1 - x * x), -2 * x * (1 - y * y)
    row = (i - 1) + N * (j - 1)
    want = {row: 4 * nu / h ** 2, row - 1: -nu / h ** 2 - wx / (2 * h), row + 1: -nu / h ** 2 + wx / (2 * h),
            row - N: -nu / h ** 2 - wy / (2 * h), row + N: -nu / h ** 2 + wy / (2 * h)}
    got = {c: A[row, c] for c in np.nonzero(A[row])[0]}
    assert set(got) == set(want)
    for c in want:
        assert got[c] == pytest.approx(want[c], rel=1e-13)


def test_dct_is_the_orthonormal_cosine_transform():
    n = 37
    k = np.arange(n)[:, None]
    i = np.arange(n)[None, :]
    Nmat = np.sqrt(2.0 / n) * np.cos(np.pi * k * (2 * i + 1) / (2 * n))
    Nmat[0] /= np.sqrt(2.0)
    rng = np.random.default_rng(0)
    X = rng.standard_normal((n, 3))
    S = SRDCT(n, n, np.ones(n), np.arange(n))                 # D = I, E = I, scale 1
    assert np.allclose(S @ X, Nmat @ X, atol=1e-13)
    assert np.allclose(Nmat @ Nmat.T, np.eye(n), atol=1e-13)


def test_srdct_norm_in_expectation_and_scale_reading():
    n, s = 2000, 200
    rng = np.random.default_rng(1)
    x = rng.standard_normal(n)
    ratios = []
    for seed in range(40):
        S = SRDCT(n, s, inputs.srdct_signs(n, seed), inputs.srdct_rows(n, s, seed))
        ratios.append(float(np.linalg.norm(S @ x) ** 2 / (x @ x)))
    assert abs(np.mean(ratios) - 1.0) < 0.05                   # sqrt(n/s) (R2)
    assert np.mean(ratios) * (s / n) ** 2 < 0.05               # the printed sqrt(s/n) would shrink by s/n


@pytest.mark.parametrize("n,m,s", [(20000, 100, 400), (90000, 100, 1200)])
def test_srdct_embedding_edges(n, m, s):
    rng = np.random.default_rng(2)
    V, _ = np.linalg.qr(rng.standard_normal((n, m)))
    S = SRDCT(n, s, inputs.srdct_signs(n, 11), inputs.srdct_rows(n, s, 11))
    sv = np.linalg.svd(S @ V, compute_uv=False) ** 2
    lo, hi = (1 - math.sqrt(m / s)) ** 2, (1 + math.sqrt(m / s)) ** 2
    assert sv.min() > lo - 0.1 and sv.max() < hi + 0.2


def test_paper_config_runs_alg1_with_srdct():
    """Alg. 1 on a small Ex. 6.1-type problem with the SRDCT: the sketched QR relation and the
    explicit sketched residual hold for this S as for the sparse sign (they hold for any S)."""
    cfg = inputs.get_config("ex61_nu0.1").replace(fd_N=20, n=400, d_max=40, s=200, k=4)
    A, Bt, B = operators.operator_pair(cfg)
    C1, C2 = inputs.make_rhs(cfg)
    o = alg1.SylvesterSketchedKrylov.from_config(cfg, C1=C1, C2=C2, keep_basis=True)
    d = 12
    o.step(d)
    res = o.residual(d)
    U = np.concatenate([o.U.U[i] for i in range(1, d + 2)], axis=1)
    S_U, S_V = alg1.sketch_pair(cfg)
    SU = S_U @ U
    assert np.linalg.norm(o.U.Q @ o.U.T - SU) <= 1e-11 * np.linalg.norm(SU)
    m = d
    V = np.concatenate([o.V.U[i] for i in range(1, d + 1)], axis=1)
    import scipy.linalg as sla
    Uh = sla.solve_triangular(o.U.T[:m, :m], U[:, :m].T, trans="T", lower=False).T
    Vh = sla.solve_triangular(o.V.T[:m, :m], V.T, trans="T", lower=False).T
    X = Uh @ res.Y @ Vh.T
    R = A @ X + (B.T @ X.T).T - C1 @ C2.T
    SRS = S_U @ (S_V @ R.T).T
    assert res.rho == pytest.approx(np.linalg.norm(SRS), rel=1e-9)
