"""Alg. 2 (truncated Arnoldi for Sylvester, no sketch) and the full Arnoldi (Galerkin)
comparison method, plain fp64, step by step.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Follows PAPER.md Appendix A, Alg. 2 (`alg:standardinnerprod_krylov`), line by line:
  line 1      U_1 beta_1 = C_1, V_1 beta_2 = C_2 (skinny QR, positive diagonal, R10)
  lines 3-9   W~ = A U_d; for i = max(1, d-k+1) .. d: h_{i,d} = U_i^T W~, W~ -= U_i h_{i,d}
              (MGS, the window of R5); U_{d+1} h_{d+1,d} = W~ (skinny QR)
  line 11     H_d Y + Y G_d^T = E_1 beta_1 beta_2^T E_1^T   (eq. reduced_tr, P:245-247;
              H_d = the square dr x dr part of H_und_d)
  line 12     rho = sqrt(dr) (||Y E_d g_{d+1,d}^T||_F + ||h_{d+1,d} E_d^T Y||_F)
              (Prop. 3.2: an upper bound of the true residual norm ||R_d^tr||_F)
  lines 17-18 truncated SVD of Y (R12), X^(1) = U_d Y_1, X^(2) = V_d Y_2 by the two-pass replay

The full Arnoldi method (eq. full; Galerkin) is the same recurrence with
k >= d and one reorthogonalisation sweep (the second MGS pass adds its coefficients to h_{i,d};
standard practice, needed for orthonormal bases in floating point), for which the residual norm
is exact: ||R_d||_F^2 = ||h_{d+1,d} E_d^T Y||_F^2 + ||Y E_d g_{d+1,d}^T||_F^2 (R13: the
printed E_{d+1} is E_d).

Stopping quantity (R8 reading applied to both): rho_rel = rho / ||beta_1 beta_2^T||_F
(= rho / ||C_1 C_2^T||_F, U_1 and V_1 being orthonormal).
"""
from __future__ import annotations

import math
import time
from typing import Dict, Tuple

import numpy as np
import scipy.linalg as sla

from .alg1 import CheckResult, RANK_TOL, qr_pos


class PlainSequence:
    """One Krylov sequence of Alg. 2 lines 1-8: K_d(M, C) with k-truncated MGS (optionally
    reorthogonalised: the full method)."""

    def __init__(self, M, C: np.ndarray, k: int, reorth: bool = False, keep_basis: bool = False):
        self.M, self.k, self.reorth, self.keep_basis = M, k, reorth, keep_basis
        self.C = np.array(C, dtype=np.float64)
        self.n, self.r = self.C.shape
        U1, self.beta = qr_pos(self.C)                          # line 1
        self.U: Dict[int, np.ndarray] = {1: U1}
        self.H: Dict[Tuple[int, int], np.ndarray] = {}
        self.Wnorm: Dict[int, float] = {}
        self.d = 0
        self.breakdown = False

    def step(self) -> None:
        d = self.d + 1
        W = np.asarray(self.M @ self.U[d])                      # line 3
        self.Wnorm[d] = float(np.linalg.norm(W))
        window = range(max(1, d - self.k + 1), d + 1)
        for i in window:                                        # lines 4-7 (MGS)
            h = self.U[i].T @ W
            W = W - self.U[i] @ h
            self.H[(i, d)] = h
        if self.reorth:                                         # full method: second sweep
            for i in window:
                h = self.U[i].T @ W
                W = W - self.U[i] @ h
                self.H[(i, d)] = self.H[(i, d)] + h
        Unew, hsub = qr_pos(W)                                  # line 8
        self.H[(d + 1, d)] = hsub
        if np.min(np.abs(np.diag(hsub))) <= 1e-14 * self.Wnorm[d]:   # R11
            self.breakdown = True
        self.U[d + 1] = Unew
        if not self.keep_basis:
            for i in list(self.U):
                if i < d + 2 - self.k:
                    del self.U[i]
        self.d = d

    def Hsq(self, d: int) -> np.ndarray:
        """H_d: the leading dr x dr (square) part of H_und_d (block upper Hessenberg, banded)."""
        r = self.r
        Hm = np.zeros((d * r, d * r))
        for j in range(1, d + 1):
            for i in range(max(1, j - self.k + 1), min(j + 1, d) + 1):
                Hm[(i - 1) * r:i * r, (j - 1) * r:j * r] = self.H[(i, j)]
        return Hm

    def replay(self, Z: np.ndarray, d: int) -> np.ndarray:
        """X = U_d Z regenerating U_1..U_d from C and the stored h_{i,j}: U_1 =
        C beta^{-1}; U_{j+1} = (M U_j - sum_i U_i h_{i,j}) h_{j+1,j}^{-1}."""
        r, k = self.r, self.k
        U = {1: sla.solve_triangular(self.beta, self.C.T, trans="T", lower=False).T}
        X = U[1] @ Z[0:r]
        for j in range(1, d):
            W = np.asarray(self.M @ U[j])
            for i in range(max(1, j - k + 1), j + 1):
                W = W - U[i] @ self.H[(i, j)]
            U[j + 1] = sla.solve_triangular(self.H[(j + 1, j)], W.T, trans="T", lower=False).T
            X = X + U[j + 1] @ Z[j * r:(j + 1) * r]
            for i in list(U):
                if i < j + 2 - k:
                    del U[i]
        return X


class TruncatedArnoldiSylvester:
    """Alg. 2 (full=False) or the full Arnoldi / Galerkin method (full=True) for
    A X + X B = C1 C2^T.  residual(d) returns the method's stopping quantity:
    Alg. 2: the Prop. 3.2 bound; full: the exact residual norm (both relative, R8)."""

    def __init__(self, A, Bt, C1, C2, k: int, full: bool = False, keep_basis: bool = False):
        self.full = full
        self.U = PlainSequence(A, C1, k, reorth=full, keep_basis=keep_basis)
        self.V = PlainSequence(Bt, C2, k, reorth=full, keep_basis=keep_basis)
        self.r = self.U.r
        self.C1, self.C2 = np.asarray(C1), np.asarray(C2)
        self.rhs_norm = float(np.linalg.norm(self.U.beta @ self.V.beta.T))
        self.d = 0

    @classmethod
    def from_config(cls, cfg, full=False, C1=None, C2=None, csr_pair=None, keep_basis=False, k=None):
        from synth.inputs import make_rhs
        from . import operators
        A, Bt, _ = operators.operator_pair(cfg, csr_pair)
        if C1 is None:
            C1, C2 = make_rhs(cfg)
        kk = k if k is not None else (cfg.d_max + 1 if full else cfg.k)
        return cls(A, Bt, C1, C2, kk, full=full, keep_basis=keep_basis)

    def step(self, nsteps: int = 1) -> None:
        for _ in range(nsteps):
            self.U.step()
            self.V.step()
            self.d += 1

    @property
    def breakdown(self) -> bool:
        return self.U.breakdown or self.V.breakdown

    def solve_projected(self, d: int):
        r, m = self.r, d * self.r
        F = np.zeros((m, m))
        F[:r, :r] = self.U.beta @ self.V.beta.T                 # E_1 beta_1 beta_2^T E_1^T
        return sla.solve_sylvester(self.U.Hsq(d), self.V.Hsq(d).T, F)   # line 11

    def residual(self, d: int) -> CheckResult:
        assert 1 <= d <= self.d
        t0 = time.perf_counter()
        r, m = self.r, d * self.r
        try:
            Y = self.solve_projected(d)
        except (np.linalg.LinAlgError, ValueError):
            return CheckResult(d, math.nan, math.nan, None, True, time.perf_counter() - t0)
        if not np.all(np.isfinite(Y)):
            return CheckResult(d, math.nan, math.nan, None, True, time.perf_counter() - t0)
        a = float(np.linalg.norm(Y[:, m - r:] @ self.V.H[(d + 1, d)].T))     # ||Y E_d g^T||
        b = float(np.linalg.norm(self.U.H[(d + 1, d)] @ Y[m - r:, :]))       # ||h E_d^T Y||
        if self.full:
            rho = math.sqrt(a * a + b * b)                                     # P:240-242 (exact)
        else:
            rho = math.sqrt(m) * (a + b)                                       # line 12, Prop. 3.2
        return CheckResult(d, rho, rho / self.rhs_norm, Y, False, time.perf_counter() - t0)

    def solution(self, d: int, Y: np.ndarray, rank_tol: float = RANK_TOL):
        """Lines 17-18: Y ~ Y1 Y2^T (truncated SVD, balanced sqrt(Sigma), R12), X1 = U_d Y1 and
        X2 = V_d Y2 by the two-pass replay (no T: the bases are Euclidean-orthonormal blockwise)."""
        W, sig, Zt = np.linalg.svd(Y)
        if sig.size == 0 or sig[0] == 0:
            return np.zeros((self.U.n, 0)), np.zeros((self.V.n, 0))
        ell = int(np.count_nonzero(sig > rank_tol * sig[0]))
        Y1 = W[:, :ell] * np.sqrt(sig[:ell])[None, :]
        Y2 = Zt[:ell].T * np.sqrt(sig[:ell])[None, :]
        return self.U.replay(Y1, d), self.V.replay(Y2, d)
