"""Config table and seeded input generators (BASELINE.json `configs`).

No arithmetic of the method lives here (see package docstring).
"""
from __future__ import annotations

import dataclasses
import math
from typing import Optional, Tuple

import numpy as np

ZETA = 8            # sparse-sign nonzeros per column (BASELINE.json north_star / configs)
SKETCH_SEEDS = (11, 12)   # S_U, S_V seeds (SURVEY.md §8(c) "independent seeds", proposed defaults)
TOL = 1e-6          # sketched relative residual target (BASELINE.json configs)


@dataclasses.dataclass(frozen=True)
class Config:
    """One workload.  `kind` is 'stencil2d', 'stencil3d' or 'csr'.

    Stencil operators are -Laplace(u) + w.grad(u) on the unit square/cube with
    homogeneous Dirichlet BCs, N interior nodes per direction, h = 1/(N+1),
    central differences (BASELINE.json configs 0-3).
    """
    name: str
    kind: str
    n: int
    r: int
    k: int
    d_max: int
    s: int
    N: int = 0
    wA: Tuple[float, ...] = ()
    wB: Tuple[float, ...] = ()
    normalize_c: bool = False
    seed_c: int = 0
    # CSR (config 4)
    csr_nnz_off: int = 0
    csr_band: int = 0
    seed_a: int = 1
    seed_b: int = 2
    zeta: int = ZETA
    seed_u: int = SKETCH_SEEDS[0]
    seed_v: int = SKETCH_SEEDS[1]
    tol: float = TOL

    @property
    def dim(self) -> int:
        return {"stencil2d": 2, "stencil3d": 3}.get(self.kind, 0)

    def replace(self, **kw) -> "Config":
        return dataclasses.replace(self, **kw)


def _stencil(name, dim, N, wA, wB, r, k, d_max, normalize=False, seed_c=0):
    n = N ** dim
    return Config(name=name, kind=f"stencil{dim}d", n=n, r=r, k=k, d_max=d_max,
                  s=4 * d_max * r, N=N, wA=tuple(float(x) for x in wA),
                  wB=tuple(float(x) for x in wB), normalize_c=normalize, seed_c=seed_c)


CONFIGS = {
    # BASELINE.json configs[0..4]; s = 4*d_max*r, zeta = 8, seeds (11, 12), tol 1e-6.
    "c0": _stencil("c0", 2, 64, (10, 10), (-5, 5), r=1, k=2, d_max=300),
    "c1": _stencil("c1", 2, 512, (50, 50), (-20, 30), r=4, k=2, d_max=1500, normalize=True),
    "c2": _stencil("c2", 3, 128, (20, 20, 20), (-10, 10, 5), r=4, k=2, d_max=800),
    "c3": _stencil("c3", 3, 256, (20, 20, 20), (-10, 10, 5), r=8, k=3, d_max=600),
    "c4": Config(name="c4", kind="csr", n=2 ** 22, r=2, k=2, d_max=400, s=4 * 400 * 2,
                 csr_nnz_off=20, csr_band=4096, seed_a=1, seed_b=2),
}


def get_config(name: str) -> Config:
    return CONFIGS[name]


def make_rhs(cfg: Config) -> Tuple[np.ndarray, np.ndarray]:
    """C1, C2: n x r, iid N(0,1) from numpy PCG64(seed_c); C1 drawn first, then C2,
    row-major.  Config c1 normalises each column to unit 2-norm."""
    rng = np.random.Generator(np.random.PCG64(cfg.seed_c))
    C1 = rng.standard_normal((cfg.n, cfg.r))
    C2 = rng.standard_normal((cfg.n, cfg.r))
    if cfg.normalize_c:
        C1 /= np.linalg.norm(C1, axis=0, keepdims=True)
        C2 /= np.linalg.norm(C2, axis=0, keepdims=True)
    return np.ascontiguousarray(C1), np.ascontiguousarray(C2)


def banded_csr(n: int, nnz_off: int, band: int, seed: int):
    """Random banded nonsymmetric CSR matrix of BASELINE.json config 4.

    Row i: `nnz_off` distinct off-diagonal columns uniform in
    [max(0,i-band), min(n-1,i+band)] minus {i}; rows with duplicate draws are
    redrawn; values N(0,1)/sqrt(nnz_off); diagonal = sum|offdiag| + 1, so every
    Gershgorin disc lies in Re >= 1.  Returns (row_ptr int64[n+1], col int32[nnz],
    val float64[nnz]) with sorted column indices (nnz = n*(nnz_off+1)).
    Requires every row to have at least nnz_off candidates (n > nnz_off, band >= nnz_off).
    """
    if n <= nnz_off or 2 * band < nnz_off:
        raise ValueError("band too narrow for nnz_off distinct columns")
    rng = np.random.Generator(np.random.PCG64(seed))
    i = np.arange(n, dtype=np.int64)
    lo = np.maximum(0, i - band)
    hi = np.minimum(n - 1, i + band)
    cnt = hi - lo                      # candidates excluding the diagonal
    if np.any(cnt < nnz_off):
        raise ValueError("band too narrow near the boundary")

    def draw(rows):
        u = rng.integers(0, cnt[rows, None], size=(rows.size, nnz_off), dtype=np.int64)
        c = lo[rows, None] + u
        c += (c >= i[rows, None])      # skip the diagonal
        c.sort(axis=1)
        return c

    cols = draw(i)
    while True:
        dup = np.nonzero(np.any(cols[:, 1:] == cols[:, :-1], axis=1))[0]
        if dup.size == 0:
            break
        cols[dup] = draw(dup)
    vals = rng.standard_normal((n, nnz_off)) / math.sqrt(nnz_off)
    diag = np.abs(vals).sum(axis=1) + 1.0
    # insert the diagonal in sorted position
    allc = np.concatenate([cols, i[:, None]], axis=1)
    allv = np.concatenate([vals, diag[:, None]], axis=1)
    order = np.argsort(allc, axis=1, kind="stable")
    allc = np.take_along_axis(allc, order, axis=1)
    allv = np.take_along_axis(allv, order, axis=1)
    m = nnz_off + 1
    row_ptr = np.arange(n + 1, dtype=np.int64) * m
    return row_ptr, allc.reshape(-1).astype(np.int32), np.ascontiguousarray(allv.reshape(-1))


def config_csr(cfg: Config):
    """(A, B) CSR triplets for a 'csr' config (seeds seed_a, seed_b)."""
    A = banded_csr(cfg.n, cfg.csr_nnz_off, cfg.csr_band, cfg.seed_a)
    B = banded_csr(cfg.n, cfg.csr_nnz_off, cfg.csr_band, cfg.seed_b)
    return A, B


def small_config(kind="stencil2d", N=12, r=2, k=2, d_max=20, s: Optional[int] = None,
                 wA=None, wB=None, n=None, nnz_off=6, band=20, **kw) -> Config:
    """Test-sized config (same families, smaller sizes)."""
    if kind.startswith("stencil"):
        dim = 2 if kind == "stencil2d" else 3
        wA = wA if wA is not None else ((10.0, 10.0) if dim == 2 else (20.0, 20.0, 20.0))
        wB = wB if wB is not None else ((-5.0, 5.0) if dim == 2 else (-10.0, 10.0, 5.0))
        nn = N ** dim
        return Config(name=f"small-{kind}-{N}", kind=kind, n=nn, r=r, k=k, d_max=d_max,
                      s=s if s is not None else 4 * d_max * r, N=N, wA=tuple(wA), wB=tuple(wB), **kw)
    nn = n if n is not None else 5000
    return Config(name=f"small-csr-{nn}", kind="csr", n=nn, r=r, k=k, d_max=d_max,
                  s=s if s is not None else 4 * d_max * r, csr_nnz_off=nnz_off, csr_band=band, **kw)
