"""GPU parity of the comparison methods against oracle/alg2.py, through the C ABI:

  method "truncated"  Alg. 2: the same truncated basis as Alg. 1 without a
                      sketch; rho = the Prop. 3.2 bound sqrt(dr)(||Y E_d g^T|| + ||h E_d^T Y||)
  method "full"       full Arnoldi / Galerkin: block CGS2 against every
                      retained block; rho = the exact residual norm

Tolerances as for Alg. 1 (BASELINE.json north star): per-step rho_rel 1e-8 relative (R19
floors), H_und 1e-9, d* within +-2, true residual within 10 % of the oracle's at the same d.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

from oracle import alg1, alg2, operators  # noqa: E402
from synth import inputs  # noqa: E402

CASES = {
    "2d-r4": dict(kind="stencil2d", N=37, r=4, k=2, d_max=60),
    "2d-r1": dict(kind="stencil2d", N=23, r=1, k=2, d_max=60),
    "3d-r8k3-tma": dict(kind="stencil3d", N=34, r=8, k=3, d_max=55),
    "3d-r4k2": dict(kind="stencil3d", N=21, r=4, k=2, d_max=55),
    "csr-r2": dict(kind="csr", n=20011, nnz_off=20, band=300, r=2, k=2, d_max=55),
}


def _rho_close(rr, ro):
    if ro >= 1e-9:
        return abs(rr - ro) <= max(1e-8 * ro, 1e-15)
    return abs(rr - ro) <= 1e-12


def _setup(name, method):
    import paper_2311_16019_b200 as pkg
    cfg = inputs.small_config(**CASES[name])
    csr = inputs.config_csr(cfg) if cfg.kind == "csr" else None
    C1, C2 = inputs.make_rhs(cfg)
    full = method == "full"
    orc = alg2.TruncatedArnoldiSylvester.from_config(cfg, full=full, C1=C1, C2=C2, csr_pair=csr)
    gpu = pkg.from_config(cfg, C1=torch.from_numpy(C1).cuda(), C2=torch.from_numpy(C2).cuda(), csr_pair=csr,
                          stream=torch.cuda.current_stream().cuda_stream, method=method)
    return cfg, csr, C1, C2, orc, gpu


@pytest.mark.parametrize("method", ["truncated", "full"])
@pytest.mark.parametrize("name", list(CASES))
def test_per_step_rho_and_H_match_oracle(name, method):
    cfg, csr, C1, C2, orc, gpu = _setup(name, method)
    D = 30
    gpu.step(D)
    orc.step(D)
    bad = []
    for d in range(1, D + 1):
        _, rr = gpu.residual(d)
        ro = orc.residual(d).rho_rel
        if not _rho_close(rr, ro):
            bad.append((d, rr, ro))
    assert not bad, bad[:5]
    r = cfg.r
    for which, seq in ((0, orc.U), (1, orc.V)):
        H, T, beta = gpu.get_small(which, D)
        Ho = np.zeros(((D + 1) * r, D * r))
        for (i, j), h in seq.H.items():
            if j <= D:
                Ho[(i - 1) * r:i * r, (j - 1) * r:j * r] = h
        assert np.linalg.norm(H - Ho) <= 1e-9 * np.linalg.norm(Ho)
        assert np.allclose(T, np.eye(T.shape[0]))                 # no sketch: T = I
        assert np.allclose(beta, seq.beta, rtol=1e-12, atol=1e-12 * np.abs(seq.beta).max())
    gpu.close()


@pytest.mark.parametrize("method", ["truncated", "full"])
@pytest.mark.parametrize("name", ["2d-r4", "3d-r8k3-tma", "csr-r2"])
def test_solution_and_true_residual_match_oracle(name, method):
    cfg, csr, C1, C2, orc, gpu = _setup(name, method)
    d = 25
    gpu.step(d)
    orc.step(d)
    res = orc.residual(d)
    X1o, X2o = orc.solution(d, res.Y)
    mr = d * cfg.r
    X1 = torch.zeros((cfg.n, mr), dtype=torch.float64, device="cuda")
    X2 = torch.zeros((cfg.n, mr), dtype=torch.float64, device="cuda")
    gpu.residual(d)
    _, _, rank = gpu.solution(d, mr, X1, X2)
    X1h, X2h = X1[:, :rank].cpu().numpy(), X2[:, :rank].cpu().numpy()
    A, _, B = operators.operator_pair(cfg, csr)
    _, rel_o = alg1.true_residual(A, B, C1, C2, X1o, X2o)
    _, rel_g = alg1.true_residual(A, B, C1, C2, X1h, X2h)
    assert abs(rel_g - rel_o) <= 0.10 * rel_o
    Xo = X1o @ X2o.T
    assert np.linalg.norm(X1h @ X2h.T - Xo) <= 1e-6 * np.linalg.norm(Xo)
    gpu.close()


@pytest.mark.parametrize("method,tol", [("truncated", 1e-3), ("full", 1e-6)])
def test_c0_time_to_tolerance_matches_oracle(method, tol):
    """d* of the R9 driver on c0 (n = 4096) for both comparison methods vs the oracle's
    (Alg. 2's bound reaches ~2e-4 at best on c0, so it is driven to 1e-3)."""
    import paper_2311_16019_b200 as pkg
    cfg = inputs.get_config("c0").replace(tol=tol)
    C1, C2 = inputs.make_rhs(cfg)
    orc = alg2.TruncatedArnoldiSylvester.from_config(cfg, full=method == "full")
    ro = alg1.solve(orc, tol, cfg.d_max, keep_Y=False)
    gpu = pkg.from_config(cfg, C1=torch.from_numpy(C1).cuda(), C2=torch.from_numpy(C2).cuda(),
                          stream=torch.cuda.current_stream().cuda_stream, method=method)
    d, rr, st = gpu.solve()
    assert st == 0 and ro.converged
    assert abs(d - ro.d_star) <= 2 and rr < tol
    gpu.close()


def test_full_method_basis_is_orthonormal_at_c2_slice():
    """The full method keeps the Euclidean basis orthonormal (CGS2): U^T U = I over 40 blocks of a
    3-D convection-diffusion case (get_block reads the retained, normalised blocks)."""
    import paper_2311_16019_b200 as pkg
    cfg = inputs.small_config("stencil3d", N=40, r=4, k=2, d_max=45)
    C1, C2 = inputs.make_rhs(cfg)
    gpu = pkg.from_config(cfg, C1=torch.from_numpy(C1).cuda(), C2=torch.from_numpy(C2).cuda(),
                          stream=torch.cuda.current_stream().cuda_stream, method="full")
    gpu.step(40)
    U = np.concatenate([gpu.get_block(0, j) for j in range(1, 42)], axis=1)
    assert np.abs(U.T @ U - np.eye(U.shape[1])).max() < 1e-12
    gpu.close()
