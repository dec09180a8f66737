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


def _mp_edges(m, s):
    return (1 - math.sqrt(m / s)) ** 2, (1 + math.sqrt(m / s)) ** 2


def _sine_modes(N, dims, freqs):
    """Orthonormal basis of low-frequency Dirichlet sine modes on an N^dims grid (x fastest)."""
    x = np.arange(1, N + 1) / (N + 1)
    import itertools
    cols = []
    for f in itertools.product(*[range(1, q + 1) for q in freqs]):
        v = np.ones(1)
        for a in reversed(f):                  # last factor varies slowest (z), first fastest (x)
            v = np.kron(v, np.sin(np.pi * a * x))
        cols.append(v)
    Q, _ = np.linalg.qr(np.array(cols).T)
    return Q


@pytest.mark.parametrize("dims,N,freqs,seed", [(2, 128, (10, 10), 11), (2, 128, (10, 10), 12),
                                               (3, 32, (5, 5, 8), 11), (3, 32, (5, 5, 8), 12)])
def test_embedding_on_smooth_structured_subspaces(dims, N, freqs, seed):
    """P:117-127 (epsilon-subspace embedding) on the subspaces the method actually sketches:
    smooth low-frequency modes, where neighbouring rows (one 32-row hash group) carry nearly
    equal values.  sigma^2(S Q) must stay inside the Marchenko-Pastur edges (s = 4m, the BJ
    ratio) with the same margins as for random subspaces.  Negative control: the same S with
    its signs dropped (|S|) sums the smooth rows coherently and fails by two orders."""
    Q = _sine_modes(N, dims, freqs)
    m = Q.shape[1]
    s = 4 * m
    S = sparse_sign.matrix(Q.shape[0], s, 8, seed)
    sv = np.linalg.svd(S @ Q, compute_uv=False) ** 2
    lo, hi = _mp_edges(m, s)
    assert sv.min() > lo - 0.08 and sv.max() < hi + 0.15
    sv_bad = np.linalg.svd(abs(S) @ Q, compute_uv=False) ** 2
    assert sv_bad.max() > 10 * hi


@pytest.mark.parametrize("kind,N,r,d,seed", [("stencil2d", 64, 1, 100, 11), ("stencil3d", 24, 4, 50, 11),
                                             ("stencil3d", 24, 4, 50, 12)])
def test_embedding_on_krylov_subspaces(kind, N, r, d, seed):
    """The embedding pin on orthonormalised Krylov bases K_d(A, C1) of the BJ operator families
    (c0's 2-D operator; a 24^3 slice of c2/c3's 3-D operator), built here by plain block
    Arnoldi with full reorthogonalisation (independent of alg1): sigma^2(S Q) inside the MP edges at s = 4 d r."""
    from oracle import operators
    from synth import inputs
    cfg = (inputs.get_config("c0") if kind == "stencil2d" else
           inputs.small_config(kind, N=N, r=r, k=2, d_max=d))
    A, _, _ = operators.operator_pair(cfg)
    C1, _ = inputs.make_rhs(cfg)
    Q, _ = np.linalg.qr(C1)                    # full block Arnoldi, reorthogonalised twice
    for _ in range(d - 1):
        W = np.asarray(A @ Q[:, -r:])
        for _ in range(2):
            W -= Q @ (Q.T @ W)
        q, _ = np.linalg.qr(W)
        Q = np.concatenate([Q, q], axis=1)
    m = Q.shape[1]
    s = 8 * math.ceil(4 * m / 8)
    S = sparse_sign.matrix(Q.shape[0], s, 8, seed)
    sv = np.linalg.svd(S @ Q, compute_uv=False) ** 2
    lo, hi = _mp_edges(m, s)
    assert m == d * r and np.allclose(Q.T @ Q, np.eye(m), atol=1e-10)
    assert sv.min() > lo - 0.08 and sv.max() < hi + 0.15
