"""Alg. 1 (sketched-and-truncated block Arnoldi for Sylvester), plain fp64, step by step.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Follows PAPER.md Alg. 1 line by line in the paper's order and
notation, with the readings listed in DESIGN.md §"Readings" (R2-R13) where the
printed text is garbled or silent.  Library primitives used as steps: sparse
products (scipy.sparse), Householder QR (numpy.linalg.qr = LAPACK geqrf/orgqr),
triangular solves, SVD, Bartels-Stewart (scipy.linalg.solve_sylvester).

Notation:
  U_i        basis blocks (n x r) of K_d(A, C1);  V_i of K_d(B^T, C2)
  h_{i,j}    truncated-Gram-Schmidt coefficients (r x r), H_d / H_underline_d
  S U_{d+1} = Q_{d+1} T_{d+1},  T_{d+1} = [[T_d, T_H], [0, tau_{d+1}]]   (Prop. 2.1)
  M_U = T_d H_d T_d^{-1} + T_H h_{d+1,d} tau_d^{-1} E_d^T = [T_d | T_H] H_und T_d^{-1}
  hhat = tau_{d+1} h_{d+1,d} tau_d^{-1}       (R4: the paper prints h_{d+1,d})
"""
from __future__ import annotations

import dataclasses
import math
import time
from typing import Dict, List, Optional, Tuple

import numpy as np
import scipy.linalg as sla

from . import sparse_sign
from . import operators

BREAKDOWN_RTOL = 1e-14      # R11: min diag h_{d+1,d} <= 1e-14 ||W~||_F
RANK_TOL = 1e-12            # R12: keep sigma_i > RANK_TOL * sigma_1 in Y ~ Y1 Y2^T


def qr_pos(X: np.ndarray) -> Tuple[np.ndarray, np.ndarray]:
    """Skinny Householder QR with positive-diagonal R (R10)."""
    Q, R = np.linalg.qr(X, mode="reduced")
    sg = np.sign(np.diag(R))
    sg[sg == 0] = 1.0
    return Q * sg[None, :], R * sg[:, None]


class Sequence:
    """One Krylov sequence of Alg. 1: K_d(M, C) with sketch S (M = A or B^T).

    State after `d` completed steps: blocks U_1..U_{d+1} (only the last k kept,
    unless keep_basis), all coefficients h_{i,j} (j <= d), the sketched basis Q
    (s x (d+1)r, orthonormal) and T_{d+1} ((d+1)r square, upper triangular).
    """

    def __init__(self, M, C: np.ndarray, S, k: int, keep_basis: bool = False, sketched_gs: bool = False):
        self.M, self.S, self.k = M, S, k
        # f3: "use the sketched inner product also in the computation of the truncated
        # bases": h_{i,d} = (S U_i)^T (S W~) and the new block S-orthonormal, (S U)^T (S U) = I
        self.sketched_gs = sketched_gs
        self.n, self.r = C.shape
        self.C = np.array(C, dtype=np.float64)
        self.keep_basis = keep_basis
        # Alg. 1 line 1: U_1 ell = C (skinny QR), Q_1 beta = S C.
        if sketched_gs:                                         # U_1 ell = C, S-orthonormal U_1
            _, self.ell = qr_pos(np.asarray(S @ self.C))
            U1 = sla.solve_triangular(self.ell, self.C.T, trans="T", lower=False).T
        else:
            U1, self.ell = qr_pos(self.C)
        _, self.beta = qr_pos(S @ self.C)
        # R3: T_1 = tau_1 = R(S U_1) (= beta ell^{-1}); the paper prints T_1 = beta.
        Q1, tau1 = qr_pos(np.asarray(S @ U1))
        self.Q = Q1
        self.T = tau1.copy()
        self.U: Dict[int, np.ndarray] = {1: U1}
        self.H: Dict[Tuple[int, int], np.ndarray] = {}
        self.d = 0
        self.breakdown = False
        self.Wnorm: Dict[int, float] = {}

    # ---- Alg. 1 lines 3-9 for this sequence -------------------------------------------
    def step(self) -> None:
        d = self.d + 1
        k, r = self.k, self.r
        W = np.asarray(self.M @ self.U[d])                      # line 3: W~ = A U_d
        if self.sketched_gs:
            return self._step_sketched_gs(d, W)
        self.Wnorm[d] = float(np.linalg.norm(W))
        for i in range(max(1, d - k + 1), d + 1):               # lines 4-7, R5 window
            h = self.U[i].T @ W                                 # h_{i,d} = U_i^T W~
            W = W - self.U[i] @ h                               # W~ = W~ - U_i h_{i,d}  (MGS order)
            self.H[(i, d)] = h
        Unew, hsub = qr_pos(W)                                  # line 8: U_{d+1} h_{d+1,d} = W~
        self.H[(d + 1, d)] = hsub
        if np.min(np.abs(np.diag(hsub))) <= BREAKDOWN_RTOL * self.Wnorm[d]:
            self.breakdown = True
        self._update_sketched_qr(d, Unew)

    def _step_sketched_gs(self, d: int, W: np.ndarray) -> None:
        """f3: lines 4-8 with the sketched inner product <x, y>_S = (S x)^T (S y): the
        window blocks are S-orthonormal, h_{i,d} = (S U_i)^T (S W~) (MGS order), and
        U_{d+1} h_{d+1,d} = W~ with (S U_{d+1})^T (S U_{d+1}) = I, i.e. h_{d+1,d} = R of the
        positive-diagonal QR of S W~ (R10).  No inner product in R^n.  The breakdown test
        (R11) measures W~ in the sketched norm."""
        k = self.k
        S = self.S
        SW = np.asarray(S @ W)
        self.Wnorm[d] = float(np.linalg.norm(SW))
        for i in range(max(1, d - k + 1), d + 1):
            SUi = np.asarray(S @ self.U[i])
            h = SUi.T @ SW                                      # h_{i,d} = <U_i, W~>_S
            W = W - self.U[i] @ h
            SW = SW - SUi @ h
            self.H[(i, d)] = h
        _, hsub = qr_pos(np.asarray(S @ W))                     # S-normalisation of the new block
        Unew = sla.solve_triangular(hsub, W.T, trans="T", lower=False).T
        self.H[(d + 1, d)] = hsub
        if np.min(np.abs(np.diag(hsub))) <= BREAKDOWN_RTOL * self.Wnorm[d]:
            self.breakdown = True
        self._update_sketched_qr(d, Unew)

    def _update_sketched_qr(self, d: int, Unew: np.ndarray) -> None:
        k, r = self.k, self.r
        # line 9: Q_{d+1} T_{d+1} = S [U_d, U_{d+1}], update only.
        w = np.asarray(self.S @ Unew)
        c1 = self.Q.T @ w
        w = w - self.Q @ c1                                     # CGS, pass 1
        c2 = self.Q.T @ w
        w = w - self.Q @ c2                                     # CGS, pass 2 (reorthogonalisation)
        q, tau = qr_pos(w)
        m = self.T.shape[0]
        T = np.zeros((m + r, m + r))
        T[:m, :m] = self.T
        T[:m, m:] = c1 + c2                                     # T_H
        T[m:, m:] = tau                                         # tau_{d+1}
        self.T = T
        self.Q = np.concatenate([self.Q, q], axis=1)
        self.U[d + 1] = Unew
        if not self.keep_basis:                                 # only the window survives
            for i in list(self.U):
                if i < d + 2 - k:
                    del self.U[i]
        self.d = d

    # ---- small matrices -----------------------------------------------------------------
    def Hbar(self, d: int) -> np.ndarray:
        """H_underline_d, (d+1)r x dr, block upper Hessenberg and banded."""
        r = self.r
        Hb = np.zeros(((d + 1) * r, d * r))
        for j in range(1, d + 1):
            for i in range(max(1, j - self.k + 1), j + 2):
                Hb[(i - 1) * r:i * r, (j - 1) * r:j * r] = self.H[(i, j)]
        return Hb

    def block(self, X: np.ndarray, i: int, j: int) -> np.ndarray:
        r = self.r
        return X[(i - 1) * r:i * r, (j - 1) * r:j * r]

    def projected(self, d: int):
        """M = [T_d | T_H] H_und_d T_d^{-1} (R6: direct form, = Q_d^T (S A U_d) T_d^{-1},
        equal to Hhat_d + Hhat E_d^T of P:199-203 / line 10) and hhat (R4)."""
        r, m = self.r, d * self.r
        T1 = self.T[:m + r, :m + r]
        Td = T1[:m, :m]
        X = T1[:m, :] @ self.Hbar(d)
        Mt = sla.solve_triangular(Td, X.T, trans="T", lower=False)   # (X T_d^{-1})^T
        M = Mt.T
        tau_d = self.block(T1, d, d)
        tau_d1 = self.block(T1, d + 1, d + 1)
        hhat = tau_d1 @ self.H[(d + 1, d)] @ np.linalg.inv(tau_d)
        return M, hhat

    def cond_T(self, d: int) -> float:
        m = d * self.r
        return float(np.linalg.cond(self.T[:m, :m]))

    # ---- second pass -----------------------------------------------------
    def replay(self, Z: np.ndarray, d: int) -> np.ndarray:
        """X = U_d Z regenerating U_1..U_d from C and the stored h_{i,j}: no inner
        products.  U_1 = C ell^{-1}; U_{j+1} = (M U_j - sum U_i h_{i,j}) h_{j+1,j}^{-1}
        (the same for the sketched-GS basis: only the coefficients differ)."""
        r, k = self.r, self.k
        U = {1: sla.solve_triangular(self.ell, self.C.T, trans="T", lower=False).T}
        X = U[1] @ Z[0:r]
        for j in range(1, d):
            W = np.asarray(self.M @ U[j])
            for i in range(max(1, j - k + 1), j + 1):
                W = W - U[i] @ self.H[(i, j)]
            U[j + 1] = sla.solve_triangular(self.H[(j + 1, j)], W.T, trans="T", lower=False).T
            Zj = Z[j * r:(j + 1) * r]
            for i0 in range(0, X.shape[0], 1 << 20):          # X += U_{j+1} Z_{j+1} (row blocks:
                X[i0:i0 + (1 << 20)] += U[j + 1][i0:i0 + (1 << 20)] @ Zj   # memory only, same sums)
            for i in list(U):
                if i < j + 2 - k:
                    del U[i]
        return X


@dataclasses.dataclass
class CheckResult:
    d: int
    rho: float
    rho_rel: float
    Y: Optional[np.ndarray] = None
    singular: bool = False
    seconds: float = 0.0


def sketch_pair(cfg):
    """(S_U, S_V) of a config: the hashed sparse-sign embeddings (R1, seeds seed_u / seed_v), or
    the paper's SRDCT (R2) with the signs and rows synth/ draws from the same seeds."""
    if getattr(cfg, "sketch", "sparse_sign") == "srdct":
        from synth.inputs import srdct_rows, srdct_signs
        from .srdct import SRDCT
        return tuple(SRDCT(cfg.n, cfg.s, srdct_signs(cfg.n, sd), srdct_rows(cfg.n, cfg.s, sd))
                     for sd in (cfg.seed_u, cfg.seed_v))
    return (sparse_sign.matrix(cfg.n, cfg.s, cfg.zeta, cfg.seed_u),
            sparse_sign.matrix(cfg.n, cfg.s, cfg.zeta, cfg.seed_v))


class SylvesterSketchedKrylov:
    """Both sequences of Alg. 1 plus the projected solve, the check and the solution."""

    def __init__(self, A, Bt, C1, C2, S_U, S_V, k: int, sketched_gs: bool = False):
        self.U = Sequence(A, C1, S_U, k, sketched_gs=sketched_gs)
        self.V = Sequence(Bt, C2, S_V, k, sketched_gs=sketched_gs)
        self.A, self.Bt = A, Bt
        self.C1, self.C2 = np.asarray(C1), np.asarray(C2)
        self.r = self.U.r
        self.rhs_norm = float(np.linalg.norm(self.U.beta @ self.V.beta.T))   # R8: ||beta1 beta2^T||_F
        self.d = 0

    @classmethod
    def from_config(cls, cfg, C1=None, C2=None, csr_pair=None, keep_basis=False, sketched_gs=False):
        from synth.inputs import make_rhs
        A, Bt, _ = operators.operator_pair(cfg, csr_pair)
        if C1 is None:
            C1, C2 = make_rhs(cfg)
        S_U, S_V = sketch_pair(cfg)
        obj = cls(A, Bt, C1, C2, S_U, S_V, cfg.k, sketched_gs=sketched_gs)
        obj.U.keep_basis = obj.V.keep_basis = keep_basis
        obj.cfg = cfg
        return obj

    def step(self, nsteps: int = 1) -> None:
        for _ in range(nsteps):
            self.U.step()
            self.V.step()
            self.d += 1

    @property
    def breakdown(self) -> bool:
        return self.U.breakdown or self.V.breakdown

    def residual(self, d: int) -> CheckResult:
        """Alg. 1 lines 12-13 at d (<= steps done): solve eq. (reduced_sk) by
        Bartels-Stewart and evaluate rho with the hatted coefficients (R4)."""
        assert 1 <= d <= self.d
        t0 = time.perf_counter()
        r, m = self.r, d * self.r
        MU, hhat = self.U.projected(d)
        MV, ghat = self.V.projected(d)
        F = np.zeros((m, m))
        F[:r, :r] = self.U.beta @ self.V.beta.T                   # E_1 beta_1 beta_2^T E_1^T
        try:
            Y = sla.solve_sylvester(MU, MV.T, F)                   # M_U Y + Y M_V^T = F
        except (np.linalg.LinAlgError, ValueError):
            return CheckResult(d, math.nan, math.nan, None, True, time.perf_counter() - t0)
        if not np.all(np.isfinite(Y)):
            return CheckResult(d, math.nan, math.nan, None, True, time.perf_counter() - t0)
        rho = math.sqrt(np.linalg.norm(hhat @ Y[m - r:, :]) ** 2 + np.linalg.norm(Y[:, m - r:] @ ghat.T) ** 2)
        return CheckResult(d, rho, rho / self.rhs_norm, Y, False, time.perf_counter() - t0)

    def solution(self, d: int, Y: np.ndarray, rank_tol: float = RANK_TOL):
        """Alg. 1 lines 19-20 (R12): Y ~ Y1 Y2^T by truncated SVD (balanced
        sqrt(Sigma)), X1 = U_d T_U^{-1} Y1, X2 = V_d T_V^{-1} Y2 by the two-pass replay."""
        r, m = self.r, d * self.r
        W, sig, Zt = np.linalg.svd(Y)
        if sig.size == 0 or sig[0] == 0:
            return np.zeros((self.U.n, 0)), np.zeros((self.V.n, 0))
        ell = int(np.count_nonzero(sig > rank_tol * sig[0]))
        Y1 = W[:, :ell] * np.sqrt(sig[:ell])[None, :]
        Y2 = Zt[:ell].T * np.sqrt(sig[:ell])[None, :]
        Z1 = sla.solve_triangular(self.U.T[:m, :m], Y1, lower=False)
        Z2 = sla.solve_triangular(self.V.T[:m, :m], Y2, lower=False)
        return self.U.replay(Z1, d), self.V.replay(Z2, d)


def check_schedule(r: int, d_max: int) -> List[int]:
    """Canonical check schedule (R9; the p of Alg. 1 line 11 made explicit).  The paper
    solves the projected equation every p iterations, p = 10 in its experiments
    (P:979): every 10 steps while d*r <= 800; then
    d_next = 10*ceil(1.15*d_prev/10); d_max always included.  The bisection of solve()
    then recovers the smallest passing d inside the last bracket."""
    out, d = [], 10
    while d <= d_max and d * r <= 800:
        out.append(d)
        d += 10
    d = out[-1] if out else 10
    while True:
        d = 10 * math.ceil(1.15 * d / 10)
        if d >= d_max:
            break
        if not out or d > out[-1]:
            out.append(d)
    if not out or out[-1] != d_max:
        out.append(d_max)
    return [x for x in out if x <= d_max]


@dataclasses.dataclass
class SolveResult:
    d_star: int
    rho_rel: float
    converged: bool
    history: List[CheckResult]
    Y: Optional[np.ndarray]
    step_seconds: float
    solve_seconds: float


def _predict_crossing(d1: int, r1: float, d2: int, r2: float, tol: float) -> float:
    """Log-linear extrapolation of rho_rel through (d1, r1), (d2, r2) to rho_rel = tol."""
    if not (r1 > r2 > 0) or not math.isfinite(r1) or d2 <= d1:
        return math.nan
    slope = (math.log(r2) - math.log(r1)) / (d2 - d1)
    return d2 + (math.log(tol) - math.log(r2)) / slope


def solve(obj: SylvesterSketchedKrylov, tol: float, d_max: int, keep_Y=True) -> SolveResult:
    """Step + scheduled checks + search for the first crossing (R9).  d* = smallest d in the
    final bracket with rho_rel < tol (strict).  Breakdown: solve at the current d (R11).

    Schedule: check_schedule(); past its every-10 regime, when the log-linear extrapolation of
    the last two valid checks puts the crossing d_hat before the next scheduled check, the
    next check is at max(d_last + 1, ceil(d_hat) + 2) instead; inside the every-10 regime a
    check is skipped while d_hat lies more than 10 steps past it, the next check is still in
    that regime and lies at most 50 steps past the last valid check (round 2: the cheap early
    checks; skipping into the geometric regime overshot c1's crossing by 250 steps in a
    simulation on the goldens' rho(d), so it is not done; without the 50-step bound Ex. 6.1
    nu = 0.001 (r = 1: the every-10 regime reaches d_max = 800) skipped from d = 270 to 800,
    where rho_rel = 3.5 (kappa(T) ~ 1e16), and found no crossing).  Search on the bracket
    (d_fail, d_pass]: regula falsi on log rho_rel (x = lo + (log r_lo - log tol) /
    (log r_lo - log r_hi) (hi - lo), checked at ceil(x) clamped into the bracket, or at hi - 1 when
that is within 2 of hi), a bisection
    step after two steps that did not halve the bracket; a check that fails numerically
    (singular) is replaced by the nearest d in the bracket (mid, mid+1, mid-1, mid+2, ...).
    With rho_rel monotone on the bracket, every such search returns the bisection's d*."""
    sched = check_schedule(obj.r, d_max)
    hist: List[CheckResult] = []
    seen: List[Tuple[int, float]] = []
    t_step = t_solve = 0.0
    d_fail, passing = 0, None
    skips = 0
    for idx in range(len(sched)):
        if len(seen) >= 2:
            (d1, r1), (d2, r2) = seen[-2], seen[-1]
            dh = _predict_crossing(d1, r1, d2, r2, tol)
            if math.isfinite(dh) and sched[idx] * obj.r > 800 and dh + 2 < sched[idx]:
                sched[idx] = max(d2 + 1, math.ceil(dh) + 2)
            elif (math.isfinite(dh) and dh - 10 > sched[idx] and idx + 1 < len(sched)
                  and sched[idx + 1] * obj.r <= 800 and sched[idx + 1] - d2 <= 50):
                continue          # every-10 regime: crossing predicted > 10 steps past: skip (R9)
        dc = sched[idx]
        t0 = time.perf_counter()
        while obj.d < dc and not obj.breakdown:
            obj.step()
        t_step += time.perf_counter() - t0
        dc = min(dc, obj.d)
        res = obj.residual(dc)
        t_solve += res.seconds
        hist.append(res)
        if res.singular:
            skips += 1
            if skips >= 5:
                break
            continue
        skips = 0
        if math.isfinite(res.rho_rel):
            seen.append((dc, res.rho_rel))
        if res.rho_rel < tol or obj.breakdown:
            passing = res
            break
        d_fail = dc
    if passing is None:
        last = next((h for h in reversed(hist) if not h.singular), None)
        return SolveResult(obj.d, last.rho_rel if last else math.nan, False, hist,
                           last.Y if last else None, t_step, t_solve)
    lo, best = d_fail, passing
    hi = passing.d
    r_lo = next((r for d, r in seen if d == lo), math.nan)
    r_hi = passing.rho_rel
    slow = 0
    while hi - lo > 1 and not obj.breakdown:
        mid0 = (lo + hi) // 2
        if slow < 2 and math.isfinite(r_lo) and math.isfinite(r_hi) and r_lo > r_hi > 0:
            x = lo + (math.log(r_lo) - math.log(tol)) / (math.log(r_lo) - math.log(r_hi)) * (hi - lo)
            mid0 = min(hi - 1, max(lo + 1, math.ceil(x)))
            if hi - mid0 <= 2:               # crossing predicted just below hi: settle it at once
                mid0 = hi - 1
        res = None
        for t in range(8):
            cand = mid0 + ((t + 1) // 2 if t % 2 else -(t // 2))
            if cand <= lo or cand >= hi:
                continue
            r = obj.residual(cand)
            t_solve += r.seconds
            hist.append(r)
            if not r.singular and math.isfinite(r.rho_rel):
                res = r
                break
        width = hi - lo
        if res is None:
            lo, r_lo = mid0, math.nan
            continue
        if res.rho_rel < tol:
            hi, r_hi, best = res.d, res.rho_rel, res
        else:
            lo, r_lo = res.d, res.rho_rel
        slow = slow + 1 if 2 * (hi - lo) > width else 0
    return SolveResult(best.d, best.rho_rel, True, hist, best.Y if keep_Y else None, t_step, t_solve)


def rfactor_rows(n: int, rows_of, chunk: Optional[int] = None) -> np.ndarray:
    """Householder R-factor of an n-row matrix given by rows_of(slice) (numpy.linalg.qr).
    chunk: R of [M_1; M_2; ...] = R of the stacked per-block R-factors (up to row signs,
    which the residual norm below does not see) — the same factor without holding M whole."""
    if chunk is None or chunk >= n:
        return np.linalg.qr(rows_of(slice(0, n)), mode="r")
    parts = [np.linalg.qr(rows_of(slice(i, min(n, i + chunk))), mode="r") for i in range(0, n, chunk)]
    return np.linalg.qr(np.concatenate(parts, axis=0), mode="r")


def residual_rfactor_L(A, X1, C1, chunk: Optional[int] = None) -> np.ndarray:
    """R-factor of L = [A X1, X1, C1] (O8 below)."""
    Acsr = A.tocsr()
    return rfactor_rows(X1.shape[0], lambda sl: np.concatenate([np.asarray(Acsr[sl] @ X1), X1[sl], C1[sl]], axis=1),
                        chunk)


def residual_rfactor_R(B, X2, C2, chunk: Optional[int] = None) -> np.ndarray:
    """R-factor of R = [X2, B^T X2, C2] (O8 below)."""
    Bt = B.T.tocsr()
    return rfactor_rows(X2.shape[0], lambda sl: np.concatenate([X2[sl], np.asarray(Bt[sl] @ X2), C2[sl]], axis=1),
                        chunk)


def residual_from_rfactors(RL, RR, l: int, C1, C2) -> Tuple[float, float]:
    """||R_L N R_R^T||_F with N = diag(I_l, I_l, -I_r), and its ratio to ||C1 C2^T||_F."""
    N = np.diag(np.concatenate([np.ones(2 * l), -np.ones(C1.shape[1])]))
    res = float(np.linalg.norm(RL @ N @ RR.T))
    rc = float(np.linalg.norm(np.linalg.qr(C1, mode="r") @ np.linalg.qr(C2, mode="r").T))
    return res, res / rc


def true_residual(A, B, C1, C2, X1, X2, chunk: Optional[int] = None) -> Tuple[float, float]:
    """||A X + X B - C1 C2^T||_F and its ratio to ||C1 C2^T||_F for X = X1 X2^T,
    without Gram matrices: L = [A X1, X1, C1], R = [X2, B^T X2, C2], N = diag(I, I, -I),
    A X + X B - C1 C2^T = L N R^T, so the norm is ||R_L N R_R^T||_F with Householder R-factors.
    chunk: row-blocked R-factors (see rfactor_rows)."""
    RL = residual_rfactor_L(A, X1, C1, chunk)
    RR = residual_rfactor_R(B, X2, C2, chunk)
    return residual_from_rfactors(RL, RR, X1.shape[1], C1, C2)
