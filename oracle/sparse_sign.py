"""Hashed sparse-sign subspace embedding S (s x n), materialised (oracle only).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

The paper sketches with an SRDCT; BASELINE.json's north star replaces it
by a sparse-sign embedding with zeta = 8 nonzeros per column generated from a
seeded hash, S never stored on the GPU (reading R1 in DESIGN.md).  The paper's
requirement on S is only the epsilon-subspace-embedding property,
and Prop. 2.1 / eqs. (reduced_sk), (resnorm_sk) hold for any S.

Definition (DESIGN.md §"Sparse-sign hash"; uint32 arithmetic mod 2^32):

    mix32(x)  = x ^= x>>16; x *= 0x7feb352d; x ^= x>>15; x *= 0x846ca68b; x ^= x>>16
    seed32    = (seed ^ (seed >> 32)) & 0xffffffff
    G(m,t,q)  = mix32( mix32( ((m*zeta + t) << 2) | q ) ^ seed32 )
    b         = s / zeta                      (bucket height; s % zeta == 0)

  Row j of the operand belongs to group m = j >> 5, lane l = j & 31.  For each
  bucket t in [0, zeta):
    base  = (G(m,t,0) * b) >> 32              (in [0, b))
    a     = 2*(G(m,t,1) & 15) + 1,  c = (G(m,t,1) >> 4) & 31
    slot  = (base + ((a*l + c) & 31)) mod b
    S[t*b + slot, j] = (bit l of G(m,t,2) ? -1 : +1) / sqrt(zeta)

Each column has exactly one nonzero in each of the zeta buckets (so ||S e_j|| = 1),
and the 32 rows of a group land in 32 distinct slots of every bucket when b >= 32.
"""
from __future__ import annotations

import math

import numpy as np
import scipy.sparse as sp

def mix32(x: np.ndarray) -> np.ndarray:
    """lowbias32 integer finaliser on uint32 values (numpy uint32 arithmetic wraps mod 2^32)."""
    x = np.asarray(x, dtype=np.uint32).copy()
    x ^= x >> np.uint32(16)
    x *= np.uint32(0x7FEB352D)
    x ^= x >> np.uint32(15)
    x *= np.uint32(0x846CA68B)
    x ^= x >> np.uint32(16)
    return x


def seed32(seed: int) -> np.uint32:
    seed = int(seed) & 0xFFFFFFFFFFFFFFFF
    return np.uint32((seed ^ (seed >> 32)) & 0xFFFFFFFF)


def group_hash(m: np.ndarray, t: int, q: int, zeta: int, seed: int) -> np.ndarray:
    """G(m, t, q) = mix32(mix32(((m*zeta + t) << 2) | q) ^ seed32), uint32."""
    m = np.asarray(m, dtype=np.uint32)
    key = ((m * np.uint32(zeta) + np.uint32(t)) << np.uint32(2)) | np.uint32(q)
    return mix32(mix32(key) ^ seed32(seed))


def entries(j: np.ndarray, t: int, s: int, zeta: int, seed: int):
    """(row index in [0,s), value) of the bucket-t nonzero of columns j (vectorised)."""
    if s % zeta:
        raise ValueError("s must be a multiple of zeta")
    b = s // zeta
    j = np.asarray(j, dtype=np.int64)
    if j.size == 0:
        return np.zeros(0, dtype=np.int64), np.zeros(0)
    m = j >> 5
    lane = (j & 31).astype(np.uint32)
    m0 = int(m.min())
    groups = np.arange(m0, int(m.max()) + 1, dtype=np.int64)
    gi = m - m0                                   # the three group hashes, once per 32-row group
    g0 = group_hash(groups, t, 0, zeta, seed)[gi].astype(np.uint64)
    g1 = group_hash(groups, t, 1, zeta, seed)[gi]
    g2 = group_hash(groups, t, 2, zeta, seed)[gi]
    base = ((g0 * np.uint64(b)) >> np.uint64(32)).astype(np.int64)
    a = np.uint32(2) * (g1 & np.uint32(15)) + np.uint32(1)
    c = (g1 >> np.uint32(4)) & np.uint32(31)
    slot = (base + ((a * lane + c) & np.uint32(31)).astype(np.int64)) % b
    row = t * b + slot
    neg = (g2 >> lane) & np.uint32(1)
    val = np.where(neg == 1, -1.0, 1.0) / math.sqrt(zeta)
    return row, val


def matrix(n: int, s: int, zeta: int, seed: int, chunk: int = 1 << 22) -> sp.csc_matrix:
    """Materialise S as a scipy CSC matrix (s x n, exactly zeta stored entries per column,
    row indices increasing because bucket t occupies rows [t*b, (t+1)*b))."""
    rows = np.empty((n, zeta), dtype=np.int64)
    vals = np.empty((n, zeta), dtype=np.float64)
    for j0 in range(0, n, chunk):
        j = np.arange(j0, min(n, j0 + chunk), dtype=np.int64)
        for t in range(zeta):
            rows[j0:j0 + j.size, t], vals[j0:j0 + j.size, t] = entries(j, t, s, zeta, seed)
    indptr = np.arange(0, n * zeta + 1, zeta, dtype=np.int64)
    return sp.csc_matrix((vals.reshape(-1), rows.reshape(-1), indptr), shape=(s, n))


def apply(S: sp.spmatrix, X: np.ndarray) -> np.ndarray:
    """S X for an n x r block (the plain sparse product)."""
    return np.asarray(S @ X)


def apply_hashed(X: np.ndarray, s: int, zeta: int, seed: int, chunk: int = 1 << 21) -> np.ndarray:
    """S X without materialising S (same definition; for the full-size configs):
    (S X)[row_t(j), :] += val_t(j) X[j, :] summed with np.bincount per bucket/column."""
    X = np.asarray(X, dtype=np.float64)
    if X.ndim == 1:
        X = X[:, None]
    n, r = X.shape
    out = np.zeros((s, r))
    for j0 in range(0, n, chunk):
        j = np.arange(j0, min(n, j0 + chunk), dtype=np.int64)
        for t in range(zeta):
            rows, vals = entries(j, t, s, zeta, seed)
            for c in range(r):
                out[:, c] += np.bincount(rows, weights=vals * X[j, c], minlength=s)
    return out
