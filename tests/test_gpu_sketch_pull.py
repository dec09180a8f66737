"""The pull formulation of the sparse-sign sketch (csrc/sketch_pull.cuh) against the oracle.

The kernel sorts each bucket's 32-row groups by window base once (hash-only data) and gathers
instead of scattering; it must produce the same S·X as the oracle's hashed S (1e-12 relative,
BASELINE north star) for every r, ragged n (a partial last group), the smallest bucket it is
used for (b = 64), many L2 chunks (SYLV_PULL_CHUNK forces tiny chunks so that bases repeat
across chunk boundaries), and the per-step rho of Alg. 1 must match the oracle (1e-8) when
the whole step runs with it.  The push kernel (k_sketch_cols) is the same check's other arm.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

from oracle import alg1, sparse_sign  # noqa: E402
from synth import inputs  # noqa: E402


def _pkg():
    import paper_2311_16019_b200 as pkg
    return pkg


# (kind, N, r, s): n = N^2 (2-D) or N^3 (3-D); b = s / 8
SHAPES = {
    "2d-r1-ragged": ("stencil2d", 45, 1, 8 * 64),        # n = 2025 (63 groups + 9 rows), b = 64
    "2d-r2-b100": ("stencil2d", 61, 2, 8 * 100),         # n = 3721
    "3d-r4": ("stencil3d", 23, 4, 8 * 150),              # n = 12167 (ragged)
    "3d-r8": ("stencil3d", 26, 8, 8 * 333),              # n = 17576, b = 333 (odd)
}


def _ctx(kind, N, r, s):
    pkg = _pkg()
    A = pkg.stencil_operator(kind, N, (1.0, 2.0, 3.0) if kind == "stencil3d" else (1.0, 2.0))
    n = N ** 3 if kind == "stencil3d" else N * N
    C = torch.from_numpy(np.random.default_rng(3).standard_normal((n, r))).cuda()
    return pkg.SylvSketch(A, A, C, C, r=r, k=2, d_max=2, s=s, seed_u=11, seed_v=12), n


@pytest.mark.parametrize("chunk,bpw", [(None, None), ("7", None), (None, "1"), ("7", "8"), ("3", "5"), ("2", "16")])
@pytest.mark.parametrize("name", list(SHAPES))
def test_pull_sketch_matches_oracle(name, chunk, bpw, monkeypatch):
    """chunk: 32-row groups per L2 chunk; bpw: window bases per warp (strip bpw + 31 slots)."""
    kind, N, r, s = SHAPES[name]
    monkeypatch.setenv("SYLV_SKETCH", "pull")
    if chunk:
        monkeypatch.setenv("SYLV_PULL_CHUNK", chunk)
    if bpw:
        monkeypatch.setenv("SYLV_PULL_BPW", bpw)
    gpu, n = _ctx(kind, N, r, s)
    X = np.random.default_rng(5).standard_normal((n, r))
    for which, seed in ((0, 11), (1, 12)):
        got = gpu.apply_sketch(which, torch.from_numpy(X).cuda())
        want = sparse_sign.matrix(n, s, 8, seed) @ X
        assert np.abs(got - want).max() <= 1e-12 * np.abs(want).max(), (name, which)
    # wider r than the context's R goes through temporary strips
    if r < 8:
        X8 = np.random.default_rng(6).standard_normal((n, 8))
        got = gpu.apply_sketch(0, torch.from_numpy(X8).cuda())
        want = sparse_sign.matrix(n, s, 8, 11) @ X8
        assert np.abs(got - want).max() <= 1e-12 * np.abs(want).max()
    gpu.close()


def test_pull_and_push_agree_and_are_deterministic(monkeypatch):
    kind, N, r, s = SHAPES["3d-r8"]
    X = torch.from_numpy(np.random.default_rng(9).standard_normal((N ** 3, r))).cuda()
    out = {}
    for mode in ("pull", "cols"):
        monkeypatch.setenv("SYLV_SKETCH", mode)
        gpu, _ = _ctx(kind, N, r, s)
        a = gpu.apply_sketch(0, X)
        b = gpu.apply_sketch(0, X)
        np.testing.assert_array_equal(a, b)      # fixed summation order
        out[mode] = a
        gpu.close()
    assert np.abs(out["pull"] - out["cols"]).max() <= 1e-13 * np.abs(out["cols"]).max()


@pytest.mark.parametrize("case", [
    dict(kind="stencil3d", N=26, r=8, k=3, d_max=50),
    dict(kind="csr", n=5003, nnz_off=6, band=40, r=4, k=4, d_max=50),
])
def test_pull_sketch_per_step_rho(case, monkeypatch):
    monkeypatch.setenv("SYLV_SKETCH", "pull")
    monkeypatch.setenv("SYLV_PULL_CHUNK", "5")
    cfg = inputs.small_config(**case)
    csr = inputs.config_csr(cfg) if cfg.kind == "csr" else None
    C1, C2 = inputs.make_rhs(cfg)
    orc = alg1.SylvesterSketchedKrylov.from_config(cfg, C1=C1, C2=C2, csr_pair=csr)
    gpu = _pkg().from_config(cfg, C1=torch.from_numpy(C1).cuda(), C2=torch.from_numpy(C2).cuda(), csr_pair=csr,
                             stream=torch.cuda.current_stream().cuda_stream)
    bad = []
    for d in range(1, 41):
        gpu.step(1)
        orc.step(1)
        rr = gpu.residual(d)[1]
        ro = orc.residual(d).rho_rel
        ok = abs(rr - ro) <= 1e-8 * ro if ro >= 1e-9 else abs(rr - ro) <= 1e-12
        if not ok:
            bad.append((d, rr, ro))
    gpu.close()
    assert not bad, bad[:5]
