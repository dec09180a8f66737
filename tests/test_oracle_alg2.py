"""Pins for oracle/alg2.py: Alg. 2 (truncated Arnoldi, no sketch) and the full
Arnoldi / Galerkin method, against what the paper and the mathematics fix.

  residual form   for X = U_d Y V_d^T with H_d Y + Y G_d^T = E1 b1 b2^T E1^T, the dense residual
                  equals U_d Y E_d g^T V_{d+1}^T + U_{d+1} h E_d^T Y V_d^T (eq. residualform_po,
                  P:221-228, proof of Prop. 3.2) -- closed form, any k
  Prop. 3.2       ||R_d^tr||_F <= sqrt(dr)(||Y E_d g^T|| + ||h E_d^T Y||)
  Galerkin        full method: Y equals an independently built Galerkin solution (orthonormal
                  bases from block powers + numpy QR) and rho = ||R||_F exactly
  same basis      Alg. 2's truncated recurrence equals Alg. 1's (oracle/alg1.py, an independent
                  implementation of the same lines 3-8): H_und and the window blocks agree
  two-pass        replay = retained-basis product
"""
import math

import numpy as np
import pytest
import scipy.linalg as sla
import scipy.sparse as sp

from oracle import alg1, alg2, operators, sparse_sign
from synth import inputs


def _small(N=10, r=2, k=2, d_max=20, wA=(10.0, 10.0), wB=(-5.0, 5.0)):
    cfg = inputs.small_config("stencil2d", N=N, r=r, k=k, d_max=d_max, wA=wA, wB=wB)
    A, Bt, B = operators.operator_pair(cfg)
    C1, C2 = inputs.make_rhs(cfg)
    return cfg, A, Bt, B, C1, C2


def _dense_R(A, B, C1, C2, X):
    return A @ X + (B.T @ X.T).T - C1 @ C2.T


@pytest.mark.parametrize("k,r", [(2, 2), (3, 1), (1, 3)])
def test_residual_form_and_prop32_bound(k, r):
    cfg, A, Bt, B, C1, C2 = _small(N=12, r=r, k=k)
    d = 10
    o = alg2.TruncatedArnoldiSylvester(A, Bt, C1, C2, k, keep_basis=True)
    o.step(d)
    res = o.residual(d)
    m = d * r
    U = np.concatenate([o.U.U[i] for i in range(1, d + 2)], axis=1)
    V = np.concatenate([o.V.U[i] for i in range(1, d + 2)], axis=1)
    Y = res.Y
    X = U[:, :m] @ Y @ V[:, :m].T
    R = _dense_R(A, B, C1, C2, X)
    h, g = o.U.H[(d + 1, d)], o.V.H[(d + 1, d)]
    form = U[:, :m] @ (Y[:, m - r:] @ g.T) @ V[:, m:].T + U[:, m:] @ (h @ Y[m - r:, :]) @ V[:, :m].T
    assert np.linalg.norm(R - form) <= 1e-9 * np.linalg.norm(R)
    nR = np.linalg.norm(R)
    assert nR <= res.rho * (1 + 1e-12)
    assert res.rho_rel == pytest.approx(res.rho / np.linalg.norm(C1 @ C2.T), rel=1e-12)
    # the bound is not the exact norm under truncation (U_d not orthonormal)
    exact = math.sqrt(np.linalg.norm(Y[:, m - r:] @ g.T) ** 2 + np.linalg.norm(h @ Y[m - r:]) ** 2)
    assert res.rho > 1.5 * exact


def test_full_method_is_galerkin_and_rho_is_exact():
    cfg, A, Bt, B, C1, C2 = _small(N=8, r=2, k=50, d_max=8)
    d, r = 7, 2
    o = alg2.TruncatedArnoldiSylvester(A, Bt, C1, C2, k=50, full=True, keep_basis=True)
    o.step(d)
    res = o.residual(d)
    X1, X2 = o.solution(d, res.Y, rank_tol=0.0)

    def basis(M, C):
        blocks, Z = [], C
        for _ in range(d):
            blocks.append(Z)
            Z = np.asarray(M @ Z)
        return np.linalg.qr(np.concatenate(blocks, axis=1))[0]

    Uo, Vo = basis(A, C1), basis(Bt, C2)
    Yg = sla.solve_sylvester(Uo.T @ (A @ Uo), (Vo.T @ (B.T @ Vo)).T, (Uo.T @ C1) @ (C2.T @ Vo))
    Xg = Uo @ Yg @ Vo.T
    X = X1 @ X2.T
    assert np.linalg.norm(X - Xg) <= 1e-8 * np.linalg.norm(Xg)
    assert res.rho == pytest.approx(np.linalg.norm(_dense_R(A, B, C1, C2, X)), rel=1e-8)
    U = np.concatenate([o.U.U[i] for i in range(1, d + 2)], axis=1)
    assert np.allclose(U.T @ U, np.eye(U.shape[1]), atol=1e-12)


def test_truncated_basis_equals_alg1_basis():
    """Alg. 1 and Alg. 2 build the SAME truncated basis (lines 3-8 of both); the two oracle
    modules implement it independently, so H_und and the window blocks must agree."""
    cfg, A, Bt, B, C1, C2 = _small(N=16, r=2, k=3, d_max=30)
    d = 20
    o2 = alg2.TruncatedArnoldiSylvester(A, Bt, C1, C2, 3)
    S = sparse_sign.matrix(cfg.n, 4 * 30 * 2, 8, 11)
    s1 = alg1.Sequence(A, C1, S, k=3)
    o2.step(d)
    for _ in range(d):
        s1.step()
    for (i, j), h in s1.H.items():
        assert np.allclose(o2.U.H[(i, j)], h, rtol=0, atol=1e-10 * max(1.0, np.abs(h).max()))
    for i in range(d + 2 - 3, d + 2):
        assert np.allclose(o2.U.U[i], s1.U[i], atol=1e-11)


@pytest.mark.parametrize("full", [False, True])
def test_replay_equals_retained_basis(full):
    cfg, A, Bt, B, C1, C2 = _small(N=10, r=2, k=2 if not full else 40)
    d = 9
    o = alg2.TruncatedArnoldiSylvester(A, Bt, C1, C2, 2 if not full else 40, full=full, keep_basis=True)
    o.step(d)
    res = o.residual(d)
    X1, X2 = o.solution(d, res.Y, rank_tol=0.0)
    m = d * 2
    U = np.concatenate([o.U.U[i] for i in range(1, d + 1)], axis=1)
    V = np.concatenate([o.V.U[i] for i in range(1, d + 1)], axis=1)
    X = U @ res.Y @ V.T
    assert np.linalg.norm(X1 @ X2.T - X) <= 1e-10 * np.linalg.norm(X)


def test_solve_driver_and_bound_at_d_star():
    """The R9 driver runs on Alg. 2 too: at its d*, the true residual of the returned solution
    is below the Prop. 3.2 bound, hence below tol ||C1 C2^T||.  (On c0 the bound, with its
    sqrt(dr) factor and the truncation delay, stalls near 2e-4 by d = 300, so Alg. 2 is run to
    1e-3 here; the full method reaches the BJ tolerance 1e-6 with its exact residual.)"""
    cfg = inputs.get_config("c0")
    A, _, B = operators.operator_pair(cfg)
    o = alg2.TruncatedArnoldiSylvester.from_config(cfg)
    res = alg1.solve(o, 1e-3, cfg.d_max)
    assert res.converged
    X1, X2 = o.solution(res.d_star, res.Y)
    _, rel = alg1.true_residual(A, B, o.C1, o.C2, X1, X2)
    assert rel <= res.rho_rel * (1 + 1e-6) and rel < 1e-3
    of = alg2.TruncatedArnoldiSylvester.from_config(cfg, full=True)
    rf = alg1.solve(of, cfg.tol, cfg.d_max)
    assert rf.converged
    X1, X2 = of.solution(rf.d_star, rf.Y)
    _, rel = alg1.true_residual(A, B, of.C1, of.C2, X1, X2)
    assert rel == pytest.approx(rf.rho_rel, rel=1e-3) and rel < cfg.tol
