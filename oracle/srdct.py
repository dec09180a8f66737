"""The paper's sketch: subsampled randomized discrete cosine transform (SRDCT), applied
(not materialised).  TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

    S = sqrt(n/s) D N E   (P:965 prints sqrt(s/n); reading R2: sqrt(n/s) makes E||S x||^2 = ||x||^2)

E = diag of Rademacher signs, N = the orthonormal DCT-II (scipy.fft.dct(type=2, norm="ortho"),
the transform MATLAB's dct computes), D = selection of s rows.  The random signs and rows are
drawn by synth/ (inputs of the method, shared by both sides): srdct_signs / srdct_rows.
"""
from __future__ import annotations

import math

import numpy as np
import scipy.fft


class SRDCT:
    """S as an operator: S @ X for an n x r block (or an n-vector)."""

    def __init__(self, n: int, s: int, signs: np.ndarray, rows: np.ndarray):
        self.n, self.s = n, s
        self.shape = (s, n)
        self.signs = np.asarray(signs, dtype=np.float64)
        self.rows = np.asarray(rows, dtype=np.int64)
        assert self.signs.shape == (n,) and self.rows.shape == (s,)
        self.scale = math.sqrt(n / s)

    def __matmul__(self, X):
        X = np.asarray(X, dtype=np.float64)
        vec = X.ndim == 1
        if vec:
            X = X[:, None]
        Y = scipy.fft.dct(self.signs[:, None] * X, type=2, norm="ortho", axis=0)   # N E X
        out = self.scale * Y[self.rows]                                            # sqrt(n/s) D
        return out[:, 0] if vec else out
