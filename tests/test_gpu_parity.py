"""GPU parity: the CUDA path (through the C ABI) against the CPU fp64 oracle on the
same seeded inputs.  Tolerances (BASELINE.json north star):
  sketch of a fixed block          1e-12 relative (max-norm)
  per-step rho_rel (first 50 steps) 1e-8 relative
  small matrices H, T, beta, and the window blocks U_j: 1e-9 relative (Frobenius)
  d* within +-2, true relative residual within 10% of the oracle's at the same d.
Sizes span several CTAs and a ragged tail (n not a multiple of the rows per CTA).
"""
import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

from oracle import alg1, operators, sparse_sign  # noqa: E402
from synth import inputs  # noqa: E402


def _pkg():
    import paper_2311_16019_b200 as pkg
    return pkg


CASES = {
    "2d-r1": dict(kind="stencil2d", N=23, r=1, k=2, d_max=60),
    "2d-r4": dict(kind="stencil2d", N=37, r=4, k=2, d_max=60),
    "3d-r8k3": dict(kind="stencil3d", N=19, r=8, k=3, d_max=55),
    # even N: the 2.5-D TMA passes (tiles 32 x 4, ragged in x and y)
    "3d-r8k3-tma": dict(kind="stencil3d", N=34, r=8, k=3, d_max=55),
    "3d-r8k2-tma": dict(kind="stencil3d", N=20, r=8, k=2, d_max=55),
    "3d-r8k4-tma": dict(kind="stencil3d", N=26, r=8, k=4, d_max=55),
    "3d-r4k2-tma": dict(kind="stencil3d", N=34, r=4, k=2, d_max=55),
    "3d-r4k3-tma": dict(kind="stencil3d", N=20, r=4, k=3, d_max=55),
    "3d-r4k4-tma": dict(kind="stencil3d", N=18, r=4, k=4, d_max=55),
    "3d-r2k1": dict(kind="stencil3d", N=11, r=2, k=1, d_max=55),
    "csr-r2": dict(kind="csr", n=20011, nnz_off=20, band=300, r=2, k=2, d_max=55),
    "csr-r4k4": dict(kind="csr", n=5003, nnz_off=6, band=40, r=4, k=4, d_max=55),
}


def _setup(name, keep_basis=False):
    cfg = inputs.small_config(**CASES[name])
    csr = inputs.config_csr(cfg) if cfg.kind == "csr" else None
    C1, C2 = inputs.make_rhs(cfg)
    orc = alg1.SylvesterSketchedKrylov.from_config(cfg, C1=C1, C2=C2, csr_pair=csr, keep_basis=keep_basis)
    gpu = _pkg().from_config(cfg, C1=torch.from_numpy(C1).cuda(), C2=torch.from_numpy(C2).cuda(), csr_pair=csr,
                             stream=torch.cuda.current_stream().cuda_stream)
    return cfg, csr, C1, C2, orc, gpu


def _rho_close(rr, ro):
    """1e-8 relative while rho_rel >= 1e-9 (three decades below tol = 1e-6); below that the
    iteration has converged past the tolerance and rho is rounding noise: both must be tiny."""
    if ro >= 1e-9:
        # 1e-8 relative, with the rounding floor of a quantity normalised by ||C1 C2^T||
        # (~1e-16 times the conditioning; 1e-15 absolute) below rho_rel ~ 1e-7
        return abs(rr - ro) <= max(1e-8 * ro, 1e-15)
    return abs(rr - ro) <= 1e-12


def _rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


@pytest.mark.parametrize("name", list(CASES))
def test_sketch_of_fixed_block(name):
    cfg = inputs.small_config(**CASES[name])
    gpu = _setup(name)[-1]
    rng = np.random.default_rng(7)
    for which, seed in ((0, cfg.seed_u), (1, cfg.seed_v)):
        X = rng.standard_normal((cfg.n, cfg.r))
        got = gpu.apply_sketch(which, torch.from_numpy(X).cuda())
        want = sparse_sign.matrix(cfg.n, cfg.s, cfg.zeta, seed) @ X
        assert np.abs(got - want).max() <= 1e-12 * np.abs(want).max()


@pytest.mark.parametrize("name", list(CASES))
def test_per_step_rho_and_small_matrices(name):
    cfg, csr, C1, C2, orc, gpu = _setup(name, keep_basis=True)
    bad = []
    for d in range(1, 51):
        gpu.step(1)
        orc.step(1)
        _, rr = gpu.residual(d)
        ro = orc.residual(d).rho_rel
        if not _rho_close(rr, ro):
            bad.append((d, rr, ro))
    assert not bad, bad[:5]
    for which, seq in ((0, orc.U), (1, orc.V)):
        d = 12
        H, T, beta = gpu.get_small(which, d)
        m = d * cfg.r
        assert _rel(H, seq.Hbar(d)) <= 1e-9
        assert _rel(T, seq.T[:m + cfg.r, :m + cfg.r]) <= 1e-9
        assert _rel(beta, seq.beta) <= 1e-12


@pytest.mark.parametrize("name", list(CASES))
def test_window_blocks(name):
    """The normalised window blocks U_j = Z_j R_j equal the oracle's Householder/MGS blocks
    (before convergence: d = 5 for the fast-converging CSR cases, 15 otherwise)."""
    cfg, csr, C1, C2, orc, gpu = _setup(name, keep_basis=True)
    d = 5 if cfg.kind == "csr" else 15
    gpu.step(d)
    orc.step(d)
    for which, seq in ((0, orc.U), (1, orc.V)):
        for j in range(d + 2 - cfg.k, d + 2):
            Ug = gpu.get_block(which, j)
            assert _rel(Ug, seq.U[j]) <= 1e-9, (which, j)


def test_csr_ring_multi_tile():
    """Sliding-ring SELL pass 1 (k_pass1_sell_ring) with several tiles per CTA and a ragged last
    one: band 6000 at r = 2 gives tiles of 1024 rows; 450011 rows = 3 tiles for each of the 148
    CTAs.  Window blocks and per-step rho against the oracle."""
    CASES["csr-ring"] = dict(kind="csr", n=450011, nnz_off=12, band=6000, r=2, k=2, d_max=30)
    try:
        cfg, csr, C1, C2, orc, gpu = _setup("csr-ring", keep_basis=True)
    finally:
        del CASES["csr-ring"]
    for d in range(1, 7):
        gpu.step(1)
        orc.step(1)
        _, rr = gpu.residual(d)
        ro = orc.residual(d).rho_rel
        assert _rho_close(rr, ro), (d, rr, ro)
    for which, seq in ((0, orc.U), (1, orc.V)):
        for j in range(6 + 2 - cfg.k, 6 + 2):
            assert _rel(gpu.get_block(which, j), seq.U[j]) <= 1e-9, (which, j)


@pytest.mark.parametrize("name", ["2d-r1", "csr-r2", "3d-r8k3", "3d-r8k3-tma"])
def test_solution_and_true_residual(name):
    cfg, csr, C1, C2, orc, gpu = _setup(name)
    d = 6 if cfg.kind == "csr" else 30          # the banded CSR case converges in ~8 steps
    gpu.step(d)
    orc.step(d)
    res = orc.residual(d)
    _, rr = gpu.residual(d)
    assert res.rho_rel > 1e-9 and _rho_close(rr, res.rho_rel)
    X1o, X2o = orc.solution(d, res.Y)
    max_rank = X1o.shape[1] + 8
    X1, X2, rank = gpu.solution(d, max_rank)
    assert abs(rank - X1o.shape[1]) <= 1
    A, _, B = operators.operator_pair(cfg, csr)
    _, tro = alg1.true_residual(A, B, C1, C2, X1o, X2o)
    _, trg = alg1.true_residual(A, B, C1, C2, X1[:, :rank], X2[:, :rank])
    assert abs(trg - tro) <= 0.1 * tro
    Xo = X1o @ X2o.T
    Xg = X1[:, :rank] @ X2[:, :rank].T
    assert _rel(Xg, Xo) <= 1e-6


def test_full_solve_c0_matches_oracle():
    cfg = inputs.get_config("c0")
    C1, C2 = inputs.make_rhs(cfg)
    orc = alg1.SylvesterSketchedKrylov.from_config(cfg, C1=C1, C2=C2)
    ro = alg1.solve(orc, cfg.tol, cfg.d_max)
    gpu = _pkg().from_config(cfg, C1=C1, C2=C2)
    d_star, rr, st = gpu.solve()
    assert st == 0 and ro.converged
    assert abs(d_star - ro.d_star) <= 2
    X1o, X2o = orc.solution(ro.d_star, ro.Y)
    X1, X2, rank = gpu.solution(d_star, X1o.shape[1] + 16)
    A, _, B = operators.operator_pair(cfg)
    _, tro = alg1.true_residual(A, B, C1, C2, X1o, X2o)
    _, trg = alg1.true_residual(A, B, C1, C2, X1[:, :rank], X2[:, :rank])
    assert abs(trg - tro) <= 0.1 * tro


def test_edge_tiny_n_and_small_buckets():
    """n = 16 < 32 rows (one partial warp group), b = s/zeta = 6 < 32 slots per bucket."""
    cfg = inputs.small_config("stencil2d", N=4, r=1, k=2, d_max=5, s=48)
    C1, C2 = inputs.make_rhs(cfg)
    orc = alg1.SylvesterSketchedKrylov.from_config(cfg, C1=C1, C2=C2)
    gpu = _pkg().from_config(cfg, C1=C1, C2=C2)
    for d in range(1, 5):
        gpu.step(1)
        orc.step(1)
        _, rr = gpu.residual(d)
        ro = orc.residual(d).rho_rel
        assert abs(rr - ro) <= 1e-8 * ro


def test_breakdown_closed_form():
    N = 10
    x = np.arange(1, N + 1) / (N + 1)
    v = np.kron(np.sin(2 * np.pi * x), np.sin(np.pi * x))[:, None] * 3.0
    A = operators.stencil_matrix(N, (0.0, 0.0))
    lam = float((v.T @ (A @ v)).item() / (v.T @ v).item())
    pkg = _pkg()
    op = pkg.stencil_operator("stencil2d", N, (0.0, 0.0))
    gpu = pkg.SylvSketch(op, op, v, v, r=1, k=2, d_max=10, s=64)
    d, st = gpu.step(3)
    assert st == 5 and d == 1          # SYLV_E_BREAKDOWN at d = 1
    _, rr = gpu.residual(1)
    assert rr < 1e-10
    X1, X2, rank = gpu.solution(1, 2)
    X = v @ v.T / (2 * lam)
    assert _rel(X1[:, :rank] @ X2[:, :rank].T, X) <= 1e-10


@pytest.mark.parametrize("name", ["c0", "c1", "c2", "c3", "c4"])
def test_sketch_full_config_sizes(name):
    """S X at every BASELINE config's (n, r, s), both seeds, vs the oracle's hashed S."""
    cfg = inputs.get_config(name)
    rng = np.random.default_rng(11)
    X = rng.standard_normal((cfg.n, cfg.r))
    Xd = torch.from_numpy(X).cuda()
    pkg = _pkg()
    # build a context with the config's sizes but a 1-step d_max (no stepping happens)
    if cfg.kind.startswith("stencil"):
        A = pkg.stencil_operator(cfg.kind, cfg.N, cfg.wA)
    else:
        A = pkg.stencil_operator("stencil2d", 2048, (0.0, 0.0))   # n = 2^22 = c4's n
    C1 = torch.from_numpy(rng.standard_normal((cfg.n, cfg.r))).cuda()
    gpu = pkg.SylvSketch(A, A, C1, C1, r=cfg.r, k=cfg.k, d_max=2, s=cfg.s, seed_u=cfg.seed_u,
                         seed_v=cfg.seed_v)
    for which, seed in ((0, cfg.seed_u), (1, cfg.seed_v)):
        got = gpu.apply_sketch(which, Xd)
        want = sparse_sign.apply_hashed(X, cfg.s, cfg.zeta, seed)
        assert np.abs(got - want).max() <= 1e-12 * np.abs(want).max()
    gpu.close()


# k = 1 (orthogonalise against the newest block only): the recurrence loses conditioning within
# ~40 steps at r = 8, so it is checked against the generic passes over 20 steps, not in the
# 50-step oracle parity window
TMA_ONLY = {"3d-r8k1-tma": dict(kind="stencil3d", N=22, r=8, k=1, d_max=55)}


@pytest.mark.parametrize("name", ["3d-r8k3-tma", "3d-r8k4-tma", "3d-r4k2-tma", "3d-r4k3-tma", "3d-r4k4-tma",
                                  "3d-r8k1-tma"])
def test_tma_passes_match_generic_passes(name):
    """The 2.5-D TMA passes and the generic DMMA passes compute the same recurrence: window
    blocks and per-step rho agree to rounding (1e-12 relative) over 20 steps."""
    cfg = inputs.small_config(**{**CASES, **TMA_ONLY}[name])
    C1, C2 = inputs.make_rhs(cfg)
    st = torch.cuda.current_stream().cuda_stream
    a = _pkg().from_config(cfg, C1=torch.from_numpy(C1).cuda(), C2=torch.from_numpy(C2).cuda(), stream=st)
    b = _pkg().from_config(cfg, C1=torch.from_numpy(C1).cuda(), C2=torch.from_numpy(C2).cuda(), stream=st,
                           tma=False)
    for d in range(1, 21):
        a.step(1)
        b.step(1)
        ra, rb = a.residual(d)[1], b.residual(d)[1]
        assert abs(ra - rb) <= 1e-12 * rb + 1e-15, (d, ra, rb)
    for which in (0, 1):
        for j in range(22 - cfg.k, 22):
            assert _rel(a.get_block(which, j), b.get_block(which, j)) <= 1e-12, (which, j)



@pytest.mark.parametrize("name,ds", [("2d-r1", (20, 40, 55)), ("3d-r8k3", (10, 30, 50)), ("csr-r4k4", (3, 5))])
def test_device_projected_solve_matches_host(name, ds):
    """the device sign-function solve of M_U Y + Y M_V^T = E1 b1 b2^T E1^T
    gives the same sketched residual as the host Bartels-Stewart solve (1e-7 relative: the
    Newton sign iteration's forward error, several decades below the 1e-6 stopping
    tolerance), on the same device-built basis."""
    cfg, csr, C1, C2, orc, _ = _setup(name)
    st = torch.cuda.current_stream().cuda_stream
    g = _pkg().from_config(cfg, C1=torch.from_numpy(C1).cuda(), C2=torch.from_numpy(C2).cuda(), csr_pair=csr,
                           stream=st, proj="gpu")
    h = _pkg().from_config(cfg, C1=torch.from_numpy(C1).cuda(), C2=torch.from_numpy(C2).cuda(), csr_pair=csr,
                           stream=st, proj="host")
    done = 0
    for d in ds:
        g.step(d - done)
        h.step(d - done)
        orc.step(d - done)
        done = d
        rg, rh = g.residual(d)[1], h.residual(d)[1]
        ro = orc.residual(d).rho_rel
        assert abs(rg - rh) <= 1e-7 * rh, (d, rg, rh)
        assert abs(rg - ro) <= 1e-7 * ro, (d, rg, ro)      # and the oracle's
    s = g.stats()
    assert s["gpu_solves"] == len(ds) and s["gpu_solve_fallbacks"] == 0
    # the solution from the device-solved Y equals the host-solved one
    X1g, X2g, kg = g.solution(done, 64)
    X1h, X2h, kh = h.solution(done, 64)
    assert kg == kh
    assert _rel(X1g @ X2g.T, X1h @ X2h.T) <= 1e-6


def test_c0_full_solve_with_device_projected_solves():
    cfg = inputs.get_config("c0")
    C1, C2 = inputs.make_rhs(cfg)
    g = _pkg().from_config(cfg, C1=torch.from_numpy(C1).cuda(), C2=torch.from_numpy(C2).cuda(),
                           stream=torch.cuda.current_stream().cuda_stream, proj="gpu")
    d, rr, _ = g.solve()
    assert abs(d - 107) <= 2 and rr < cfg.tol
    assert g.stats()["gpu_solve_fallbacks"] == 0


@pytest.mark.parametrize("name", ["3d-r8k3", "2d-r4", "3d-r4k2-tma"])
def test_dmma_sweeps_match_fma_sweeps(name, monkeypatch):
    """a5's CGS2 sweeps of Q on the fp64 tensor cores (k_qtw_mma / k_qc_mma, R >= 4) and the FMA
    kernels (SYLV_QMMA=0, read at init) build the same sketched QR: T and rho agree to rounding
    over 30 steps (s = 880 for 3d-r4k2-tma: a ragged 16-row tail)."""
    cfg = inputs.small_config(**CASES[name])
    C1, C2 = inputs.make_rhs(cfg)
    st = torch.cuda.current_stream().cuda_stream
    a = _pkg().from_config(cfg, C1=torch.from_numpy(C1).cuda(), C2=torch.from_numpy(C2).cuda(), stream=st)
    monkeypatch.setenv("SYLV_QMMA", "0")
    b = _pkg().from_config(cfg, C1=torch.from_numpy(C1).cuda(), C2=torch.from_numpy(C2).cuda(), stream=st)
    a.step(30)
    b.step(30)
    for d in (5, 17, 30):
        ra, rb = a.residual(d)[1], b.residual(d)[1]
        assert abs(ra - rb) <= 1e-10 * rb + 1e-15, (d, ra, rb)
    for which in (0, 1):
        _, Ta, _ = a.get_small(which, 30)
        _, Tb, _ = b.get_small(which, 30)
        assert _rel(Ta, Tb) <= 1e-12, which


@pytest.mark.parametrize("name,ds", [("2d-r1", (20, 40, 55)), ("3d-r8k3", (10, 30, 50)), ("2d-r4", (15, 45)),
                                     ("csr-r4k4", (3, 5))])
def test_device_eig_solve_matches_oracle(name, ds, monkeypatch):
    """f1 (round 2): the certified eigendecomposition solve (cuSOLVER Xgeev + ZGEMM applies +
    iterative refinement to a rounding-level projected residual; SYLV_EIG=2 forces it ahead of
    the sign iteration) gives the ORACLE's sketched residual (1e-7 relative, several decades
    below tol) and the host solve's solution."""
    cfg, csr, C1, C2, orc, _ = _setup(name)
    st = torch.cuda.current_stream().cuda_stream
    monkeypatch.setenv("SYLV_EIG", "2")
    g = _pkg().from_config(cfg, C1=torch.from_numpy(C1).cuda(), C2=torch.from_numpy(C2).cuda(), csr_pair=csr,
                           stream=st, proj="gpu")
    monkeypatch.delenv("SYLV_EIG")
    h = _pkg().from_config(cfg, C1=torch.from_numpy(C1).cuda(), C2=torch.from_numpy(C2).cuda(), csr_pair=csr,
                           stream=st, proj="host")
    done = 0
    for d in ds:
        g.step(d - done)
        h.step(d - done)
        orc.step(d - done)
        done = d
        rg = g.residual(d)[1]
        ro = orc.residual(d).rho_rel
        assert abs(rg - ro) <= 1e-7 * ro, (d, rg, ro)
    s = g.stats()
    assert s["gpu_solves"] == len(ds) and s["gpu_solve_fallbacks"] == 0
    X1g, X2g, kg = g.solution(done, 64)
    X1h, X2h, kh = h.solution(done, 64)
    assert kg == kh
    assert _rel(X1g @ X2g.T, X1h @ X2h.T) <= 1e-6
