"""Pins for oracle/alg1.py against what the paper and the mathematics fix.

Each test would fail on a plausible mistake in the oracle (dropped term, wrong
sign/index, transposed operand, unhatted residual coefficients, wrong T_1, ...).

  exactness       dr = n, any injective S, no truncation  -> X_d = Kronecker solution
  galerkin        S = I, k >= d  -> X_d equals an independently built Galerkin
                  solution (orthonormal Krylov basis via numpy QR) and rho = ||R||_F
                  
  sketched rho    rho == ||S_U (A X + X B - C1 C2^T) S_V^T||_F for the truncated,
                  sketched run (eq. resnorm_sk P:323-326 with hatted coefficients, R4)
  S-Galerkin      Uhat^T S^T S R S_V^T S_V Vhat = 0
  arnoldi         A U_d = U_{d+1} H_und_d; window orthonormality
  prop 2.1        S U_{d+1} = Q T, Q^T Q = I, T = R of positive-diagonal QR(S U_{d+1})
  whitened M      [T_d|T_H] H_und T_d^{-1} = Q_d^T S A U_d T_d^{-1}
  T_1 / beta      beta_1 = tau_1 ell (R3)
  two-pass        replay = retained-basis product
  breakdown       C1 = C2 = eigenvector of symmetric A = B -> X = C1 C2^T / (2 lambda)
  true residual   factored formula == dense ||A X + X B - C1 C2^T||_F
  schedule        R9 lists
"""
import math

import numpy as np
import pytest
import scipy.linalg as sla
import scipy.sparse as sp

from oracle import alg1, operators, sparse_sign
from synth import inputs


def _small(N=8, r=2, k=2, d_max=20, s=None, wA=(10.0, 10.0), wB=(-5.0, 5.0), seed_c=0):
    cfg = inputs.small_config("stencil2d", N=N, r=r, k=k, d_max=d_max, s=s, wA=wA, wB=wB, seed_c=seed_c)
    A, Bt, B = operators.operator_pair(cfg)
    C1, C2 = inputs.make_rhs(cfg)
    return cfg, A, Bt, B, C1, C2


def _kron_solution(A, B, C1, C2):
    n = A.shape[0]
    Ad, Bd = A.toarray(), B.toarray()
    K = np.kron(np.eye(n), Ad) + np.kron(Bd.T, np.eye(n))      # (I (x) A + B^T (x) I) vec X
    x = np.linalg.solve(K, (C1 @ C2.T).reshape(-1, order="F"))
    return x.reshape(n, n, order="F")


def _retained(obj, d):
    U = np.concatenate([obj.U.U[i] for i in range(1, d + 1)], axis=1)
    V = np.concatenate([obj.V.U[i] for i in range(1, d + 1)], axis=1)
    return U, V


def test_exactness_when_space_is_exhausted():
    cfg, A, Bt, B, C1, C2 = _small(N=4, r=2, k=50, d_max=8)       # n = 16, dr = 16 at d = 8
    S_U = sparse_sign.matrix(cfg.n, 80, 8, 11)
    S_V = sparse_sign.matrix(cfg.n, 80, 8, 12)
    o = alg1.SylvesterSketchedKrylov(A, Bt, C1, C2, S_U, S_V, k=50)
    o.step(8)
    res = o.residual(8)
    X1, X2 = o.solution(8, res.Y, rank_tol=0.0)
    X = _kron_solution(A, B, C1, C2)
    assert np.linalg.norm(X1 @ X2.T - X) <= 1e-8 * np.linalg.norm(X)
    assert res.rho_rel < 1e-8


def test_galerkin_special_case_identity_sketch():
    cfg, A, Bt, B, C1, C2 = _small(N=8, r=2, k=50, d_max=6)
    n, d, r = cfg.n, 6, 2
    I = sp.identity(n, format="csr")
    o = alg1.SylvesterSketchedKrylov(A, Bt, C1, C2, I, I, k=50)
    o.step(d)
    res = o.residual(d)
    X1, X2 = o.solution(d, res.Y, rank_tol=0.0)
    # independent Galerkin: orthonormal bases of K_d(A, C1), K_d(B^T, C2) from the power basis
    def basis(M, C):
        blocks, Z = [], C
        for _ in range(d):
            blocks.append(Z)
            Z = np.asarray(M @ Z)
        Q, _ = np.linalg.qr(np.concatenate(blocks, axis=1))
        return Q
    Uo, Vo = basis(A, C1), basis(Bt, C2)
    Yg = sla.solve_sylvester(Uo.T @ (A @ Uo), (Vo.T @ (B.T @ Vo)).T, (Uo.T @ C1) @ (C2.T @ Vo))
    Xg = Uo @ Yg @ Vo.T
    X = X1 @ X2.T
    assert np.linalg.norm(X - Xg) <= 1e-8 * np.linalg.norm(Xg)
    R = A @ X + (B.T @ X.T).T - C1 @ C2.T
    assert res.rho == pytest.approx(np.linalg.norm(R), rel=1e-8)
    # T = I when S = I and the basis is orthonormal
    assert np.allclose(o.U.T[:d * r, :d * r], np.eye(d * r), atol=1e-10)


@pytest.mark.parametrize("k,r", [(2, 2), (3, 1), (1, 3)])
def test_sketched_residual_identity_and_galerkin_condition(k, r):
    cfg, A, Bt, B, C1, C2 = _small(N=12, r=r, k=k, d_max=14)
    d = 10
    s = 8 * math.ceil(4 * (d + 1) * r / 8)
    S_U = sparse_sign.matrix(cfg.n, s, 8, 11)
    S_V = sparse_sign.matrix(cfg.n, s, 8, 12)
    o = alg1.SylvesterSketchedKrylov(A, Bt, C1, C2, S_U, S_V, k=k)
    o.U.keep_basis = o.V.keep_basis = True
    o.step(d)
    res = o.residual(d)
    U, V = _retained(o, d)
    m = d * r
    Uh = sla.solve_triangular(o.U.T[:m, :m], U.T, trans="T", lower=False).T      # U T^{-1}
    Vh = sla.solve_triangular(o.V.T[:m, :m], V.T, trans="T", lower=False).T
    X = Uh @ res.Y @ Vh.T
    R = A @ X + (B.T @ X.T).T - C1 @ C2.T
    SRS = np.asarray(S_U @ (S_V @ R.T).T)
    assert res.rho == pytest.approx(np.linalg.norm(SRS), rel=1e-9)
    # the paper's literal (unhatted) coefficients do NOT give the sketched residual norm
    hU, hV = o.U.H[(d + 1, d)], o.V.H[(d + 1, d)]
    lit = math.sqrt(np.linalg.norm(hU @ res.Y[m - r:]) ** 2 + np.linalg.norm(res.Y[:, m - r:] @ hV.T) ** 2)
    assert abs(lit - res.rho) > 1e-3 * res.rho
    # S^T S - Galerkin condition
    G = (S_U @ Uh).T @ SRS @ (S_V @ Vh)
    assert np.linalg.norm(G) <= 1e-9 * np.linalg.norm(SRS) * np.linalg.norm(S_U @ Uh, 2) * np.linalg.norm(S_V @ Vh, 2)
    # two-pass replay equals the retained-basis product
    X1, X2 = o.solution(d, res.Y, rank_tol=0.0)
    assert np.linalg.norm(X1 @ X2.T - X) <= 1e-10 * np.linalg.norm(X)


def test_arnoldi_and_sketched_qr_relations():
    cfg, A, Bt, B, C1, C2 = _small(N=16, r=2, k=2, d_max=20)
    d, r = 15, 2
    S = sparse_sign.matrix(cfg.n, 4 * 20 * r, 8, 11)
    seq = alg1.Sequence(A, C1, S, k=2, keep_basis=True)
    for _ in range(d):
        seq.step()
    U = np.concatenate([seq.U[i] for i in range(1, d + 2)], axis=1)
    # truncated Arnoldi relation A U_d = U_{d+1} H_und_d
    lhs = A @ U[:, :d * r]
    assert np.linalg.norm(lhs - U @ seq.Hbar(d)) <= 1e-12 * np.linalg.norm(lhs)
    # local orthonormality inside the window; unit-norm blocks
    for j in range(1, d + 2):
        assert np.allclose(seq.U[j].T @ seq.U[j], np.eye(r), atol=1e-12)
        for i in range(max(1, j - 2 + 1), j):
            assert np.abs(seq.U[i].T @ seq.U[j]).max() < 1e-12
    # global orthogonality is NOT maintained (truncation): U_1 vs U_{d+1}
    assert np.abs(seq.U[1].T @ seq.U[d + 1]).max() > 1e-6
    # Prop. 2.1: S U_{d+1} = Q T with orthonormal Q, T = positive-diag R of the QR
    SU = np.asarray(S @ U)
    assert np.linalg.norm(seq.Q @ seq.T - SU) <= 1e-12 * np.linalg.norm(SU)
    assert np.allclose(seq.Q.T @ seq.Q, np.eye(U.shape[1]), atol=1e-12)
    _, Rref = alg1.qr_pos(SU)
    assert np.linalg.norm(seq.T - Rref) <= 1e-9 * np.linalg.norm(Rref)
    assert np.allclose(np.tril(seq.T, -1), 0) and np.all(np.diag(seq.T) > 0)
    # whitened projected matrix: direct formula = Q_d^T (S A U_d) T_d^{-1}
    M, hhat = seq.projected(d)
    m = d * r
    ref = seq.Q[:, :m].T @ np.asarray(S @ lhs)
    ref = sla.solve_triangular(seq.T[:m, :m], ref.T, trans="T", lower=False).T
    assert np.linalg.norm(M - ref) <= 1e-10 * np.linalg.norm(ref)
    # M is block upper Hessenberg (r subdiagonals)
    assert np.abs(np.tril(M, -r - 1)).max() <= 1e-10 * np.abs(M).max()
    # beta_1 = tau_1 ell (R3)
    tau1 = seq.T[:r, :r]
    assert np.allclose(seq.beta, tau1 @ seq.ell, rtol=1e-12, atol=1e-12 * np.abs(seq.beta).max())


def test_breakdown_on_invariant_subspace_closed_form():
    N = 10
    A = operators.stencil_matrix(N, (0.0, 0.0))                 # symmetric Laplacian, B = A
    x = np.arange(1, N + 1) / (N + 1)
    v = np.kron(np.sin(2 * np.pi * x), np.sin(np.pi * x))[:, None] * 3.0
    lam = float((v.T @ (A @ v)).item() / (v.T @ v).item())
    S_U = sparse_sign.matrix(N * N, 64, 8, 11)
    S_V = sparse_sign.matrix(N * N, 64, 8, 12)
    o = alg1.SylvesterSketchedKrylov(A, A, v, v, S_U, S_V, k=2)
    o.step(1)
    assert o.breakdown
    res = o.residual(1)
    X1, X2 = o.solution(1, res.Y, rank_tol=0.0)
    X = v @ v.T / (2 * lam)
    assert np.linalg.norm(X1 @ X2.T - X) <= 1e-10 * np.linalg.norm(X)
    assert res.rho_rel < 1e-10


def test_true_residual_matches_dense():
    cfg, A, Bt, B, C1, C2 = _small(N=9, r=2, k=2, d_max=10)
    rng = np.random.default_rng(3)
    X1, X2 = rng.standard_normal((cfg.n, 5)), rng.standard_normal((cfg.n, 5))
    X = X1 @ X2.T
    R = A @ X + (B.T @ X.T).T - C1 @ C2.T
    res, rel = alg1.true_residual(A, B, C1, C2, X1, X2)
    assert res == pytest.approx(np.linalg.norm(R), rel=1e-10)
    assert rel == pytest.approx(np.linalg.norm(R) / np.linalg.norm(C1 @ C2.T), rel=1e-10)
    for chunk in (7, 32, 80):                  # row-blocked R-factors (TSQR), ragged last block
        res_c, rel_c = alg1.true_residual(A, B, C1, C2, X1, X2, chunk=chunk)
        assert res_c == pytest.approx(np.linalg.norm(R), rel=1e-10)
        assert rel_c == pytest.approx(rel, rel=1e-10)


def test_check_schedule():
    s8 = alg1.check_schedule(8, 600)
    assert s8 == [10, 20, 30, 40, 50, 60, 70, 80, 90, 100, 120, 140, 170, 200, 230, 270, 320, 370, 430, 500,
                  580, 600]
    s4 = alg1.check_schedule(4, 1500)
    assert s4[:20] == list(range(10, 201, 10)) and s4[20] == 230
    assert s4[-1] == 1500
    s1 = alg1.check_schedule(1, 300)
    assert s1 == list(range(10, 301, 10))
    assert alg1.check_schedule(8, 7) == [7]


class _FakeRun:
    """A stand-in for SylvesterSketchedKrylov with a prescribed rho_rel(d) (search logic only)."""

    def __init__(self, rho, r=4, singular=()):
        self.rho, self.r, self.d, self.breakdown = rho, r, 0, False
        self.singular, self.calls = set(singular), []

    def step(self):
        self.d += 1

    def residual(self, d):
        self.calls.append(d)
        if d in self.singular:
            return alg1.CheckResult(d, math.nan, math.nan, None, True)
        return alg1.CheckResult(d, self.rho(d), self.rho(d), None, False)


@pytest.mark.parametrize("rate,r", [(0.985, 4), (0.97, 8), (0.991, 4), (0.9, 1)])
def test_search_finds_the_first_crossing_of_a_monotone_rho(rate, r):
    """R9 search (schedule + prediction + safeguarded regula falsi) on a strictly decreasing
    rho_rel(d): d* is exactly the first d with rho_rel < tol (brute force), with no more
    projected solves than the plain schedule + bisection would use."""
    tol, d_max = 1e-6, 1500
    rho = lambda d: 0.3 * rate ** d * (1 + 0.2 / (1 + d))   # strictly decreasing
    first = next(d for d in range(1, d_max + 1) if rho(d) < tol)
    fake = _FakeRun(rho, r=r)
    res = alg1.solve(fake, tol, d_max, keep_Y=False)
    assert res.converged and res.d_star == first
    sched = alg1.check_schedule(r, d_max)
    n_sched = next(i for i, d in enumerate(sched) if d >= first) + 1
    lo = max([0] + [d for d in sched if d < first])
    hi = min(d for d in sched if d >= first)
    n_bisect = 0
    while hi - lo > 1:
        mid = (lo + hi) // 2
        lo, hi = (lo, mid) if rho(mid) < tol else (mid, hi)
        n_bisect += 1
    assert len(fake.calls) <= n_sched + n_bisect


def test_search_is_a_valid_crossing_with_bumps_and_singular_checks():
    """Non-monotone rho_rel (bumps near tol) and numerically failed checks: the returned d*
    passes, the check just below it (if made) failed, and every failed check is skipped."""
    tol = 1e-6
    rho = lambda d: 2e-3 * 0.99 ** d * (1 + 0.05 * math.sin(d))
    fake = _FakeRun(rho, r=4, singular={779, 780, 781, 800})
    res = alg1.solve(fake, tol, 1500, keep_Y=False)
    assert res.converged and rho(res.d_star) < tol and res.d_star not in fake.singular
    below = [d for d in fake.calls if d < res.d_star and d not in fake.singular]
    assert below and rho(max(below)) >= tol
    assert max(below) == res.d_star - 1 or all(d not in fake.calls for d in range(max(below) + 1, res.d_star))


def test_skipping_keeps_a_valid_check_every_50_steps():
    """R9 (round 2): inside the every-10 regime a check is skipped only while the next one lies
    at most 50 steps past the last valid check.  A slowly decaying rho (r = 1, so the regime
    runs to d_max: Ex. 6.1's shape) whose early checks predict a crossing far past d_max must
    still be checked every <= 50 steps and reach its true crossing — without the bound the
    search jumped from d = 270 straight to d_max."""
    tol, d_max = 1e-6, 800
    rho = lambda d: 0.1 * math.exp(-0.012 * d) if d < 600 else 0.1 * math.exp(-7.2) * math.exp(-0.09 * (d - 600))
    first = next(d for d in range(1, d_max + 1) if rho(d) < tol)
    fake = _FakeRun(rho, r=1)
    res = alg1.solve(fake, tol, d_max, keep_Y=False)
    assert res.converged and res.d_star == first
    valid = sorted(d for d in fake.calls if d <= first)
    gaps = [b - a for a, b in zip(valid, valid[1:])]
    assert max(gaps) <= 50, gaps


def test_c0_regression_expectation():
    """Not a pin (parity unpinned for d* on the BJ configs): c0 converges near the
    survey-time expectation d* = 107 with a true residual of the same order."""
    cfg = inputs.get_config("c0")
    o = alg1.SylvesterSketchedKrylov.from_config(cfg)
    res = alg1.solve(o, cfg.tol, cfg.d_max)
    assert res.converged and 100 <= res.d_star <= 115
    X1, X2 = o.solution(res.d_star, res.Y)
    A, _, B = operators.operator_pair(cfg)
    _, rel = alg1.true_residual(A, B, o.C1, o.C2, X1, X2)
    assert rel < 5e-6


@pytest.mark.parametrize("k", [2, 20])
def test_sketched_residual_within_embedding_bound(k):
    """Paper P:185-188: if S_U, S_V are eps-subspace embeddings of the Krylov
    spaces that contain the residual's column and row spaces (R = A X + X B - C1 C2^T has
    columns in span(U_{d+1}) and rows in span(V_{d+1})), the sketched residual norm lies in
    [(1 - eps_U)(1 - eps_V), (1 + eps_U)(1 + eps_V)] ||R||_F.  eps is measured directly from
    the singular values of S Q (Q an orthonormal basis of the retained blocks), the true R
    from the dense reconstruction of the oracle's X (rank_tol = 0: no truncation), so this
    pins rho, the solution and the basis together against an independent bound."""
    d = 10
    cfg, A, Bt, B, C1, C2 = _small(N=10, r=1, k=k, d_max=d + 2, s=400)
    obj = alg1.SylvesterSketchedKrylov.from_config(cfg, C1=C1, C2=C2, keep_basis=True)
    obj.step(d)
    res = obj.residual(d)
    X1, X2 = obj.solution(d, res.Y, rank_tol=0.0)
    R = A @ (X1 @ X2.T) + (X1 @ X2.T) @ B.toarray() - C1 @ C2.T
    nR = np.linalg.norm(R)
    S_U = sparse_sign.matrix(cfg.n, cfg.s, cfg.zeta, cfg.seed_u).toarray()
    S_V = sparse_sign.matrix(cfg.n, cfg.s, cfg.zeta, cfg.seed_v).toarray()
    # the residual lives in span(U_{d+1}) (x) span(V_{d+1}) (exactly, up to rounding)
    QU = np.linalg.qr(np.concatenate([obj.U.U[i] for i in range(1, d + 2)], axis=1))[0]
    QV = np.linalg.qr(np.concatenate([obj.V.U[i] for i in range(1, d + 2)], axis=1))[0]
    assert np.linalg.norm(R - QU @ (QU.T @ R) @ QV @ QV.T) <= 1e-8 * nR
    sU = np.linalg.svd(S_U @ QU, compute_uv=False)
    sV = np.linalg.svd(S_V @ QV, compute_uv=False)
    eU = max(abs(sU.max() - 1), abs(1 - sU.min()))
    eV = max(abs(sV.max() - 1), abs(1 - sV.min()))
    assert eU < 1 and eV < 1
    assert res.rho == pytest.approx(np.linalg.norm(S_U @ R @ S_V.T), rel=1e-9)
    assert (1 - eU) * (1 - eV) * nR * (1 - 1e-9) <= res.rho <= (1 + eU) * (1 + eV) * nR * (1 + 1e-9)


def test_truncation_rank_and_factors_on_a_known_spectrum():
    """R12: Y ~ Y1 Y2^T keeps sigma_i > rank_tol * sigma_1.  Pinned with a Y whose
    SVD is fixed by construction (orthogonal factors from a seeded QR, singular values that
    straddle the threshold 1e-12 sigma_1 in both directions): l is the known count, and
    X1 X2^T equals the whitened bases times the known best rank-l approximation,
    Uhat Y_l Vhat^T with Uhat = U_d T_U^{-1} (retained blocks)."""
    cfg, A, Bt, B, C1, C2 = _small(N=10, r=2, k=2, d_max=12)
    d, r = 8, 2
    m = d * r
    obj = alg1.SylvesterSketchedKrylov.from_config(cfg, C1=C1, C2=C2, keep_basis=True)
    obj.step(d)
    rng = np.random.default_rng(7)
    Qa, _ = np.linalg.qr(rng.standard_normal((m, m)))
    Qb, _ = np.linalg.qr(rng.standard_normal((m, m)))
    sig = np.array([3.0, 1e-2, 1e-5, 1e-8, 9e-12, 4e-12, 2e-12, 1e-12, 5e-13, 1e-14] + [0.0] * (m - 10))
    ell = int(np.sum(sig > 1e-12 * 3.0))          # sigma_i > 3e-12: 3.0 ... 4e-12 -> 6
    assert ell == 6
    Y = (Qa * sig[None, :]) @ Qb.T
    X1, X2 = obj.solution(d, Y, rank_tol=1e-12)
    assert X1.shape[1] == ell and X2.shape[1] == ell
    U, V = _retained(obj, d)
    Uh = sla.solve_triangular(obj.U.T[:m, :m], U.T, trans="T", lower=False).T
    Vh = sla.solve_triangular(obj.V.T[:m, :m], V.T, trans="T", lower=False).T
    Yl = (Qa[:, :ell] * sig[None, :ell]) @ Qb[:, :ell].T
    ref = Uh @ Yl @ Vh.T
    assert np.linalg.norm(X1 @ X2.T - ref) <= 1e-10 * np.linalg.norm(ref)
    # balanced split: ||X1 e_i|| / ||X2 e_i|| = ||Uhat Qa e_i|| / ||Vhat Qb e_i|| (sqrt(sigma) on both);
    # only for the well-separated sigma_1..sigma_4 (singular vectors of the clustered 1e-12
    # values are determined only to eps sigma_1 / gap)
    for i in range(4):
        want = np.linalg.norm(Uh @ Qa[:, i]) / np.linalg.norm(Vh @ Qb[:, i])
        assert np.linalg.norm(X1[:, i]) / np.linalg.norm(X2[:, i]) == pytest.approx(want, rel=1e-6)
    # rank_tol = 0 keeps every singular value the SVD returns as positive (the exact zeros
    # come back as rounding-level positives)
    X1f, _ = obj.solution(d, Y, rank_tol=0.0)
    assert X1f.shape[1] >= 10


def test_cond_T_equals_condition_of_the_sketched_basis():
    """Sequence.cond_T(d) = kappa(T_d) = kappa(S U_d) (Prop. 2.1: S U_d = Q_d T_d, Q_d orthonormal),
    checked against the explicitly sketched retained basis; T_d grows ill-conditioned with d
    under truncation (the loss of global orthogonality the paper discusses)."""
    cfg, A, Bt, B, C1, C2 = _small(N=16, r=2, k=2, d_max=40)
    S = sparse_sign.matrix(cfg.n, cfg.s, cfg.zeta, cfg.seed_u)
    seq = alg1.Sequence(A, C1, S, k=2, keep_basis=True)
    for _ in range(30):
        seq.step()
    conds = []
    for d in (5, 15, 30):
        U = np.concatenate([seq.U[i] for i in range(1, d + 1)], axis=1)
        want = np.linalg.cond(np.asarray(S @ U))
        assert seq.cond_T(d) == pytest.approx(want, rel=1e-6)
        conds.append(want)
    assert conds[0] < conds[1] < conds[2]


# ---- f3: sketched inner products inside the truncated Gram-Schmidt -------------------

@pytest.mark.parametrize("k,r", [(2, 2), (3, 1)])
def test_sketched_gs_basis_relations(k, r):
    """Sketched-GS oracle: window blocks S-orthonormal ((S U_i)^T (S U_j) = delta_ij
    inside the window), the truncated Arnoldi relation A U_d = U_{d+1} H_und_d (an
    algebraic identity of the recurrence), Prop. 2.1 (S U = Q T), and rho equal to the
    explicitly sketched residual ||S_U R S_V^T||_F (the whitened relations hold for any basis)."""
    cfg, A, Bt, B, C1, C2 = _small(N=12, r=r, k=k, d_max=14)
    d = 10
    s = 8 * math.ceil(4 * (d + 1) * r / 8)
    S_U = sparse_sign.matrix(cfg.n, s, 8, 11)
    S_V = sparse_sign.matrix(cfg.n, s, 8, 12)
    o = alg1.SylvesterSketchedKrylov(A, Bt, C1, C2, S_U, S_V, k=k, sketched_gs=True)
    o.U.keep_basis = o.V.keep_basis = True
    o.step(d)
    U = np.concatenate([o.U.U[i] for i in range(1, d + 2)], axis=1)
    SU = np.asarray(S_U @ U)
    for j in range(1, d + 2):
        for i in range(max(1, j - k + 1), j + 1):
            G = SU[:, (i - 1) * r:i * r].T @ SU[:, (j - 1) * r:j * r]
            assert np.allclose(G, np.eye(r) if i == j else 0.0, atol=1e-11)
    # Euclidean orthonormality is NOT what this basis has
    assert np.abs(o.U.U[d + 1].T @ o.U.U[d + 1] - np.eye(r)).max() > 1e-3
    lhs = A @ U[:, :d * r]
    assert np.linalg.norm(lhs - U @ o.U.Hbar(d)) <= 1e-11 * np.linalg.norm(lhs)
    assert np.linalg.norm(o.U.Q @ o.U.T - SU) <= 1e-11 * np.linalg.norm(SU)
    res = o.residual(d)
    m = d * r
    V = np.concatenate([o.V.U[i] for i in range(1, d + 1)], axis=1)
    Uh = sla.solve_triangular(o.U.T[:m, :m], U[:, :m].T, trans="T", lower=False).T
    Vh = sla.solve_triangular(o.V.T[:m, :m], V.T, trans="T", lower=False).T
    X = Uh @ res.Y @ Vh.T
    R = A @ X + (B.T @ X.T).T - C1 @ C2.T
    assert res.rho == pytest.approx(np.linalg.norm(np.asarray(S_U @ (S_V @ R.T).T)), rel=1e-9)
    X1, X2 = o.solution(d, res.Y, rank_tol=0.0)
    assert np.linalg.norm(X1 @ X2.T - X) <= 1e-9 * np.linalg.norm(X)


def test_sketched_gs_with_identity_sketch_is_galerkin():
    """S = I, k >= d: the sketched inner product is the Euclidean one, the basis orthonormal, and
    the method reduces to the full Arnoldi / Galerkin method: Y and rho equal the
    oracle/alg2 full method's."""
    from oracle import alg2
    cfg, A, Bt, B, C1, C2 = _small(N=8, r=2, k=50, d_max=8)
    d = 6
    I = sp.identity(cfg.n, format="csr")
    o = alg1.SylvesterSketchedKrylov(A, Bt, C1, C2, I, I, k=50, sketched_gs=True)
    o.step(d)
    f = alg2.TruncatedArnoldiSylvester(A, Bt, C1, C2, k=50, full=True)
    f.step(d)
    ro, rf = o.residual(d), f.residual(d)
    assert ro.rho == pytest.approx(rf.rho, rel=1e-8)
    assert np.linalg.norm(ro.Y - rf.Y) <= 1e-8 * np.linalg.norm(rf.Y)
