"""Host-side a6 logic of the library (no GPU): the projected matrix builder and the
Bartels-Stewart solve, checked against the oracle's formulas / scipy on the same data."""
import numpy as np
import scipy.linalg as sla

import paper_2311_16019_b200 as pkg
from oracle import alg1, operators, sparse_sign
from synth import inputs


def _lib_layout_H(seq, d, r, k):
    H = np.zeros((d + 1, k + 1, r, r))
    for j in range(1, d + 1):
        nwin = min(k, j)
        for i in range(nwin):
            H[j, i] = seq.H[(j - nwin + 1 + i, j)]
        H[j, k] = seq.H[(j + 1, j)]
    return H


def test_projected_matrix_matches_oracle():
    cfg = inputs.small_config("stencil2d", N=14, r=2, k=3, d_max=20)
    A, Bt, B = operators.operator_pair(cfg)
    C1, _ = inputs.make_rhs(cfg)
    S = sparse_sign.matrix(cfg.n, cfg.s, 8, 11)
    seq = alg1.Sequence(A, C1, S, k=3)
    d = 12
    for _ in range(d):
        seq.step()
    M_ref, _ = seq.projected(d)
    T = np.asfortranarray(seq.T)
    M = pkg.api.host_projected(d, 2, 3, T, _lib_layout_H(seq, d, 2, 3))
    assert np.linalg.norm(M - M_ref) <= 1e-12 * np.linalg.norm(M_ref)


def test_bartels_stewart_matches_scipy():
    rng = np.random.default_rng(0)
    m, r = 60, 3
    MU = rng.standard_normal((m, m)) + 12 * np.eye(m)
    MV = rng.standard_normal((m, m)) + 9 * np.eye(m)
    B = rng.standard_normal((r, r))
    F = np.zeros((m, m))
    F[:r, :r] = B
    Y = pkg.api.host_sylvester(MU, MV, B)
    assert np.linalg.norm(MU @ Y + Y @ MV.T - F) <= 1e-12 * np.linalg.norm(F) * 10
    assert np.allclose(Y, sla.solve_sylvester(MU, MV.T, F), rtol=1e-10, atol=1e-13)
