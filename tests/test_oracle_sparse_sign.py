"""Pins for oracle/sparse_sign.py (the hashed sparse-sign embedding S).

The paper fixes only what an epsilon-subspace embedding must do; the
construction itself is reading R1.  Pins:
  * structure: exactly one nonzero per bucket per column, entries +-1/sqrt(zeta),
    hence ||S e_j|| = 1 exactly; distinct slots within a 32-row group;
  * an independent scalar re-derivation of the hash on a few columns (guards the
    vectorised uint64 masking);
  * uniformity of the row map (chi-square) and of the signs;
  * E||Sx||^2 = ||x||^2 (closed form: each column has unit norm and the signs are
    balanced, so the Monte-Carlo mean over seeds converges to 1);
  * subspace-embedding behaviour: singular values of S V for random orthonormal V
    fall inside the Marchenko-Pastur edges (1 +- sqrt(m/s))^2 up to a small margin.
"""
import math

import numpy as np
import pytest

from oracle import sparse_sign


def _scalar_entry(j, t, s, zeta, seed):
    M = 0xFFFFFFFF

    def mix(x):
        x &= M
        x ^= x >> 16
        x = (x * 0x7FEB352D) & M
        x ^= x >> 15
        x = (x * 0x846CA68B) & M
        x ^= x >> 16
        return x

    sd = (seed ^ (seed >> 32)) & M
    m, lane = j >> 5, j & 31

    def G(q):
        return mix(mix((((m * zeta + t) << 2) | q) & M) ^ sd)

    b = s // zeta
    base = (G(0) * b) >> 32
    a = 2 * (G(1) & 15) + 1
    c = (G(1) >> 4) & 31
    slot = (base + ((a * lane + c) & 31)) % b
    val = (-1.0 if (G(2) >> lane) & 1 else 1.0) / math.sqrt(zeta)
    return t * b + slot, val


@pytest.mark.parametrize("n,s,zeta,seed", [(1000, 400, 8, 11), (4096, 1200, 8, 12), (77, 48, 4, 3)])
def test_structure(n, s, zeta, seed):
    S = sparse_sign.matrix(n, s, zeta, seed).tocsc()
    b = s // zeta
    assert S.shape == (s, n)
    assert np.all(np.diff(S.indptr) == zeta)          # no two buckets collide (disjoint row ranges)
    vals = np.abs(S.data)
    assert np.allclose(vals, 1 / math.sqrt(zeta), rtol=0, atol=0)
    for jj in [0, 1, n // 2, n - 1]:
        rows = S.indices[S.indptr[jj]:S.indptr[jj + 1]]
        assert sorted(rows // b) == list(range(zeta))
    col_norm = np.sqrt(np.asarray(S.multiply(S).sum(axis=0))).ravel()
    assert np.allclose(col_norm, 1.0, rtol=0, atol=4e-16)


def test_matches_scalar_rederivation():
    n, s, zeta, seed = 5000, 1600, 8, (7 << 32) + 11
    S = sparse_sign.matrix(n, s, zeta, seed).tocsc()
    for j in [0, 31, 32, 33, 1234, 4999]:
        want = sorted(_scalar_entry(j, t, s, zeta, seed) for t in range(zeta))
        rows = S.indices[S.indptr[j]:S.indptr[j + 1]]
        vals = S.data[S.indptr[j]:S.indptr[j + 1]]
        got = sorted(zip(rows.tolist(), vals.tolist()))
        assert got == want


def test_group_slots_distinct():
    s, zeta, seed = 2400 * 8, 8, 11
    b = s // zeta
    j = np.arange(32 * 50)
    for t in range(zeta):
        rows, _ = sparse_sign.entries(j, t, s, zeta, seed)
        grp = rows.reshape(50, 32)
        for g in grp:
            assert len(set(g.tolist())) == 32
            assert np.all(g // b == t)


def test_uniform_rows_and_signs():
    n, s, zeta, seed = 320000, 8000, 8, 11
    S = sparse_sign.matrix(n, s, zeta, seed).tocsr()
    counts = np.diff(S.indptr)                       # nonzeros per sketch row
    expected = n * zeta / s
    b = s // zeta
    chi2 = float(((counts - expected) ** 2 / expected).sum())
    # a 32-row group covers 32 consecutive slots of a bucket exactly once, so a slot's
    # count is Binomial(n/32, 32/b): E[chi2] = s (1 - 32/b)
    mean = s * (1 - 32 / b)
    assert abs(chi2 - mean) < 8 * math.sqrt(2 * s)
    pos = float((S.data > 0).mean())
    assert abs(pos - 0.5) < 6 * math.sqrt(0.25 / S.data.size)


def test_norm_preserved_in_expectation():
    rng = np.random.default_rng(0)
    n, s, zeta = 3000, 320, 8
    x = rng.standard_normal(n)
    ratios = [float(np.linalg.norm(sparse_sign.matrix(n, s, zeta, seed) @ x) ** 2 / (x @ x))
              for seed in range(60)]
    # Var of ||Sx||^2/||x||^2 is O(1/s); 60 draws -> standard error ~ sqrt(2/s/60)
    assert abs(np.mean(ratios) - 1.0) < 4 * math.sqrt(2.0 / s / 60) + 1e-3


@pytest.mark.parametrize("n,m,s", [(20000, 100, 400), (40000, 200, 1600)])
def test_marchenko_pastur_edges(n, m, s):
    rng = np.random.default_rng(1)
    V, _ = np.linalg.qr(rng.standard_normal((n, m)))
    S = sparse_sign.matrix(n, s, 8, 11)
    sv = np.linalg.svd(S @ V, compute_uv=False) ** 2
    lo, hi = (1 - math.sqrt(m / s)) ** 2, (1 + math.sqrt(m / s)) ** 2
    assert sv.min() > lo - 0.08 and sv.max() < hi + 0.15


def test_apply_hashed_equals_materialised_product():
    rng = np.random.default_rng(5)
    n, s, r = 10007, 640, 3
    X = rng.standard_normal((n, r))
    S = sparse_sign.matrix(n, s, 8, 12)
    got = sparse_sign.apply_hashed(X, s, 8, 12, chunk=3000)
    assert np.allclose(got, S @ X, rtol=1e-13, atol=1e-13 * np.abs(X).sum())
