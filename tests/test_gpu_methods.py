"""GPU parity of the comparison methods (oracle/alg2.py) and of the sketched-GS
variant (f3: oracle/alg1.py with sketched_gs=True), through the C ABI:

  method "truncated"  Alg. 2: the same truncated basis as Alg. 1 without a
                      sketch; rho = the Prop. 3.2 bound sqrt(dr)(||Y E_d g^T|| + ||h E_d^T Y||)
  method "full"       full Arnoldi / Galerkin: block CGS2 against every
                      retained block; rho = the exact residual norm
  method "sketched_gs" Alg. 1 with the sketched inner product in the truncated GS

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


# ---- f3: sketched inner products inside the truncated GS (method "sketched_gs") -------

SGS_CASES = ["2d-r4", "2d-r1", "3d-r8k3-tma", "3d-r4k2", "csr-r2"]


def _setup_sgs(name):
    import paper_2311_16019_b200 as pkg
    cfg = inputs.small_config(**CASES[name])
    csr = inputs.config_csr(cfg) if cfg.kind == "csr" else None
    C1, C2 = inputs.make_rhs(cfg)
    orc = alg1.SylvesterSketchedKrylov.from_config(cfg, C1=C1, C2=C2, csr_pair=csr, sketched_gs=True)
    gpu = pkg.from_config(cfg, C1=torch.from_numpy(C1).cuda(), C2=torch.from_numpy(C2).cuda(), csr_pair=csr,
                          stream=torch.cuda.current_stream().cuda_stream, method="sketched_gs")
    return cfg, csr, C1, C2, orc, gpu


@pytest.mark.parametrize("name", SGS_CASES)
def test_sketched_gs_matches_oracle(name):
    cfg, csr, C1, C2, orc, gpu = _setup_sgs(name)
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
    # H and T are compared while the iteration has not converged (rho_rel >= 1e-9, R19): past
    # that, W' is rounding noise and S W' formed from sketches (GPU) and by sketching W' (oracle)
    # differ at noise level (rho is invariant to the normalisation of the noise block)
    Dc = max(d for d in range(1, D + 1) if orc.residual(d).rho_rel >= 1e-9)
    for which, seq in ((0, orc.U), (1, orc.V)):
        H, T, beta = gpu.get_small(which, Dc)
        Ho = seq.Hbar(Dc)
        assert np.linalg.norm(H - Ho) <= 1e-9 * np.linalg.norm(Ho)
        To = seq.T[:(Dc + 1) * r, :(Dc + 1) * r]
        assert np.linalg.norm(T - To) <= 1e-9 * np.linalg.norm(To)
    # solution and true residual at d = D
    res = orc.residual(D)
    X1o, X2o = orc.solution(D, res.Y)
    mr = D * r
    X1 = torch.zeros((cfg.n, mr), dtype=torch.float64, device="cuda")
    X2 = torch.zeros((cfg.n, mr), dtype=torch.float64, device="cuda")
    gpu.residual(D)
    _, _, rank = gpu.solution(D, mr, X1, X2)
    A, _, B = operators.operator_pair(cfg, csr)
    _, rel_o = alg1.true_residual(A, B, C1, C2, X1o, X2o)
    _, rel_g = alg1.true_residual(A, B, C1, C2, X1[:, :rank].cpu().numpy(), X2[:, :rank].cpu().numpy())
    assert abs(rel_g - rel_o) <= 0.10 * rel_o
    gpu.close()


def test_sketched_gs_c0_time_to_tolerance_matches_oracle():
    import paper_2311_16019_b200 as pkg
    cfg = inputs.get_config("c0")
    C1, C2 = inputs.make_rhs(cfg)
    orc = alg1.SylvesterSketchedKrylov.from_config(cfg, sketched_gs=True)
    ro = alg1.solve(orc, cfg.tol, cfg.d_max, keep_Y=False)
    gpu = pkg.from_config(cfg, C1=torch.from_numpy(C1).cuda(), C2=torch.from_numpy(C2).cuda(),
                          stream=torch.cuda.current_stream().cuda_stream, method="sketched_gs")
    d, rr, st = gpu.solve()
    assert st == 0 and ro.converged and abs(d - ro.d_star) <= 2 and rr < cfg.tol
    gpu.close()


@pytest.mark.parametrize("kind,P", [("stencil3d", 2), ("stencil2d", 3), ("csr", 2)])
def test_sketched_gs_sharded_equals_unsharded(kind, P):
    """Row-sharded sketched-GS contexts (virtual ranks of one GPU, sylv_local_group): the only
    collective per step is the allreduce of the sketch of the matvec (S is linear in rows); rho
    per step and T equal the unsharded run."""
    import threading
    import paper_2311_16019_b200 as pkg
    args = {"stencil3d": dict(kind="stencil3d", N=24, r=4, k=2, d_max=30),
            "stencil2d": dict(kind="stencil2d", N=48, r=2, k=3, d_max=30),
            "csr": dict(kind="csr", n=6400, nnz_off=6, band=60, r=2, k=2, d_max=30)}[kind]
    cfg = inputs.small_config(**args)
    csr = inputs.config_csr(cfg) if cfg.kind == "csr" else None
    C1, C2 = inputs.make_rhs(cfg)
    D = 20
    ref = pkg.from_config(cfg, C1=torch.from_numpy(C1).cuda(), C2=torch.from_numpy(C2).cuda(), csr_pair=csr,
                          method="sketched_gs")
    ref.step(D)
    want = [ref.residual(d)[1] for d in range(1, D + 1)]
    Tw = ref.get_small(0, D)[1]
    ref.close()
    group = pkg.LocalGroup(P)
    out, errs = [None] * P, []

    def run(rank):
        try:
            torch.cuda.set_device(0)
            rb, re_ = pkg.partition(cfg, P, rank)
            comm = group.comm(rank)
            st = torch.cuda.Stream()
            g = pkg.from_config(cfg, C1=torch.from_numpy(np.ascontiguousarray(C1[rb:re_])).cuda(),
                                C2=torch.from_numpy(np.ascontiguousarray(C2[rb:re_])).cuda(), csr_pair=csr,
                                stream=st.cuda_stream, comm=comm, row_range=(rb, re_), method="sketched_gs")
            g.step(D)
            out[rank] = ([g.residual(d)[1] for d in range(1, D + 1)], g.get_small(0, D)[1])
            g.close()
            comm.close()
        except Exception as e:  # pragma: no cover
            errs.append(e)

    th = [threading.Thread(target=run, args=(q,)) for q in range(P)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=600)
    group.close()
    assert not errs, errs
    for rr, T in out:
        # the sharded sketch sums in a different order: per-step rho to the north-star 1e-8 with
        # the R19 rounding floors (as the Alg. 1 sharded tests)
        assert all(_rho_close(a, b) for a, b in zip(rr, want)), list(zip(rr, want))
        Dc = max(d for d in range(1, D + 1) if want[d - 1] >= 1e-9)
        m = (Dc + 1) * cfg.r
        assert np.linalg.norm(T[:m, :m] - Tw[:m, :m]) <= 1e-9 * np.linalg.norm(Tw[:m, :m])


# ---- f4: the paper's workloads (variable-coefficient operators as CSR, k up to 10, SRDCT) -----

def _paper_small(name, **kw):
    return inputs.get_config(name).replace(**kw)


@pytest.mark.parametrize("n,s", [(4096, 400), (90000, 1200), (20011, 500)])
def test_srdct_sketch_of_fixed_block(n, s):
    """S X on the GPU (cuFFT DCT-II + the selected rows) vs the oracle's scipy DCT (R2)."""
    import paper_2311_16019_b200 as pkg
    from oracle.srdct import SRDCT
    N = int(round(n ** 0.5))
    cfg = (inputs.get_config("ex61_nu0.1").replace(fd_N=N, n=N * N, s=s, d_max=s // 2 - 1)
           if N * N == n else inputs.small_config("csr", n=n, r=1, k=2, d_max=s // 2 - 1, s=s, sketch="srdct"))
    csr = inputs.config_csr(cfg)
    C1, C2 = inputs.make_rhs(cfg)
    gpu = pkg.from_config(cfg, C1=torch.from_numpy(C1).cuda(), C2=torch.from_numpy(C2).cuda(), csr_pair=csr,
                          stream=torch.cuda.current_stream().cuda_stream)
    rng = np.random.default_rng(3)
    X = rng.standard_normal((cfg.n, 1))
    for which, sd in ((0, cfg.seed_u), (1, cfg.seed_v)):
        S = SRDCT(cfg.n, s, inputs.srdct_signs(cfg.n, sd), inputs.srdct_rows(cfg.n, s, sd))
        got = gpu.apply_sketch(which, torch.from_numpy(X).cuda())
        want = S @ X
        assert np.abs(got - want).max() <= 1e-12 * np.abs(want).max()
    gpu.close()


@pytest.mark.parametrize("case", [
    dict(name="ex61_nu0.01", fd_N=45, n=45 * 45, s=480, d_max=100, k=10),                 # k = 10, SRDCT
    dict(name="ex61_nu0.1", fd_N=40, n=1600, s=400, d_max=100, k=7, sketch="sparse_sign"),  # k = 7, sparse sign
    dict(name="ex63_n125000", fd_N=14, n=14 ** 3, s=400, d_max=90, k=3),                  # 3-D variable w, SRDCT
])
def test_paper_workload_rho_matches_oracle(case):
    import paper_2311_16019_b200 as pkg
    case = dict(case)
    cfg = _paper_small(case.pop("name"), **case)
    csr = inputs.config_csr(cfg)
    C1, C2 = inputs.make_rhs(cfg)
    orc = alg1.SylvesterSketchedKrylov.from_config(cfg, C1=C1, C2=C2)
    gpu = pkg.from_config(cfg, C1=torch.from_numpy(C1).cuda(), C2=torch.from_numpy(C2).cuda(), csr_pair=csr,
                          stream=torch.cuda.current_stream().cuda_stream)
    D = 40
    gpu.step(D)
    orc.step(D)
    bad = [(d, gpu.residual(d)[1], orc.residual(d).rho_rel) for d in range(1, D + 1)]
    bad = [b for b in bad if not _rho_close(b[1], b[2])]
    assert not bad, bad[:5]
    gpu.close()
