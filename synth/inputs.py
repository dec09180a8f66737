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
    # paper workloads: variable-coefficient convection-diffusion assembled as
    # CSR (kind 'csr'): fd_dim 2/3, N interior nodes per direction, viscosity nu, named
    # velocity fields (VELOCITY below) for A and B
    fd_dim: int = 0
    fd_N: int = 0
    nu: float = 1.0
    wA_field: str = ""
    wB_field: str = ""
    sketch: str = "sparse_sign"     # or "srdct" (the paper's subsampled randomized DCT)
    normalize_rhs: str = ""         # "" | "columns" (c1) | "unit" (each of C1, C2 to unit Frobenius norm)

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


# Velocity fields of the paper's experiments (problem data, not the method): w(x, y[, z]) at the
# grid points, arrays in, tuple of arrays out.
VELOCITY = {
    "ex61_A": lambda x, y: (np.ones_like(x), np.ones_like(x)),                       # w_A = (1, 1)
    "ex61_B": lambda x, y: (3 * y * (1 - x ** 2), -2 * x * (1 - y ** 2)),            # w_B
    "ex63_A": lambda x, y, z: (x * np.sin(x), y * np.cos(y), np.exp(z ** 2 - 1)),   # w_A
    "ex63_B": lambda x, y, z: ((1 - x ** 2) * y * z, np.ones_like(x), np.exp(z)),   # w_B
}


def _paper_61(nu, N=300):
    n = N * N
    # maxit = 600, but tab1:ex2 reports d = 766/770 for nu = 0.001: d_max = 800 there (R26)
    return Config(name=f"ex61_nu{nu:g}", kind="csr", n=n, r=1, k=10, d_max=600 if nu > 0.005 else 800, s=1200,
                  fd_dim=2, fd_N=N, nu=nu,
                  wA_field="ex61_A", wB_field="ex61_B", sketch="srdct", normalize_rhs="unit")


def _paper_63(N):
    n = N ** 3
    return Config(name=f"ex63_n{n}", kind="csr", n=n, r=1, k=3, d_max=250, s=500, fd_dim=3, fd_N=N, nu=0.005,
                  wA_field="ex63_A", wB_field="ex63_B", sketch="srdct", normalize_rhs="unit")


# The paper's own workloads (P:969-979 Ex. 6.1, table tab1:ex2; P:1120-1128 Ex. 6.3, table tab1:ex3):
# seeded N(0,1) right-hand sides stand in for MATLAB rng('default') (d comparable qualitatively only).
PAPER_CONFIGS = {c.name: c for c in [_paper_61(0.1), _paper_61(0.01), _paper_61(0.001)]
                 + [_paper_63(N) for N in (50, 60, 70, 80, 90, 100)]}


def get_config(name: str) -> Config:
    return CONFIGS[name] if name in CONFIGS else PAPER_CONFIGS[name]


def make_rhs(cfg: Config) -> Tuple[np.ndarray, np.ndarray]:
    """C1, C2: n x r, iid N(0,1) from numpy PCG64(seed_c); C1 drawn first, then C2,
    row-major.  Config c1 normalises each column to unit 2-norm."""
    rng = np.random.Generator(np.random.PCG64(cfg.seed_c))
    C1 = rng.standard_normal((cfg.n, cfg.r))
    C2 = rng.standard_normal((cfg.n, cfg.r))
    if cfg.normalize_c:
        C1 /= np.linalg.norm(C1, axis=0, keepdims=True)
        C2 /= np.linalg.norm(C2, axis=0, keepdims=True)
    if cfg.normalize_rhs == "unit":                   # P:977 (c1, c2 unit norm) / P:1122 (||c1 c2^T|| = 1)
        C1 /= np.linalg.norm(C1)
        C2 /= np.linalg.norm(C2)
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


def fd_csr(dim: int, N: int, nu: float, field: str):
    """Centred finite differences of L(u) = -nu Lap u + w . grad u (eq. condiff_op) on the
    unit square / cube, N interior nodes per direction, h = 1/(N+1), homogeneous Dirichlet, x
    fastest (R14), w = VELOCITY[field] evaluated at the node: row (i, j[, l]) has the diagonal
    2 dim nu / h^2 and, per direction e, the neighbours -nu/h^2 -+ w_e / (2h) (minus side / plus
    side).  Assembled stencil-point by stencil-point; returns the CSR triplet with sorted columns."""
    h = 1.0 / (N + 1)
    g = np.arange(1, N + 1) * h
    if dim == 2:
        Y, X = np.meshgrid(g, g, indexing="ij")      # row index = x + N y (x fastest)
        coords = (X.ravel(), Y.ravel())
        idx = [np.tile(np.arange(N), N), np.repeat(np.arange(N), N)]
    else:
        Z, Y, X = np.meshgrid(g, g, g, indexing="ij")
        coords = (X.ravel(), Y.ravel(), Z.ravel())
        idx = [np.tile(np.arange(N), N * N), np.tile(np.repeat(np.arange(N), N), N), np.repeat(np.arange(N), N * N)]
    w = VELOCITY[field](*coords)
    n = N ** dim
    rows = np.arange(n, dtype=np.int64)
    R, Cc, V = [rows], [rows], [np.full(n, 2.0 * dim * nu / h ** 2)]
    stride = 1
    for e in range(dim):
        for sgn in (-1, 1):
            ok = (idx[e] > 0) if sgn < 0 else (idx[e] < N - 1)
            R.append(rows[ok])
            Cc.append(rows[ok] + sgn * stride)
            V.append(-nu / h ** 2 + sgn * w[e][ok] / (2 * h))
        stride *= N
    R, Cc, V = np.concatenate(R), np.concatenate(Cc), np.concatenate(V)
    order = np.lexsort((Cc, R))
    R, Cc, V = R[order], Cc[order], V[order]
    row_ptr = np.zeros(n + 1, dtype=np.int64)
    np.add.at(row_ptr, R + 1, 1)
    return np.cumsum(row_ptr), Cc.astype(np.int32), np.ascontiguousarray(V)


def config_csr(cfg: Config):
    """(A, B) CSR triplets for a 'csr' config: the banded random matrices (seeds seed_a, seed_b),
    or the paper's variable-coefficient operators (fd_dim > 0)."""
    if cfg.fd_dim:
        return (fd_csr(cfg.fd_dim, cfg.fd_N, cfg.nu, cfg.wA_field),
                fd_csr(cfg.fd_dim, cfg.fd_N, cfg.nu, cfg.wB_field))
    A = banded_csr(cfg.n, cfg.csr_nnz_off, cfg.csr_band, cfg.seed_a)
    B = banded_csr(cfg.n, cfg.csr_nnz_off, cfg.csr_band, cfg.seed_b)
    return A, B


def srdct_signs(n: int, seed: int) -> np.ndarray:
    """The Rademacher diagonal E of the SRDCT sketch: n signs +-1 (int8) from numpy
    PCG64(seed + 7919).  A random number of the method, passed to both sides as an input."""
    rng = np.random.Generator(np.random.PCG64(seed + 7919))
    return np.where(rng.integers(0, 2, size=n) == 1, 1, -1).astype(np.int8)


def srdct_rows(n: int, s: int, seed: int) -> np.ndarray:
    """The row selection D of the SRDCT sketch: s distinct rows of [0, n), drawn with numpy
    PCG64(seed) and sorted.  A random number of the method, passed to both sides as an input."""
    rng = np.random.Generator(np.random.PCG64(seed))
    return np.sort(rng.choice(n, size=s, replace=False)).astype(np.int64)


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
