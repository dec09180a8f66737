"""Oracle parity at the FULL BASELINE sizes (c0..c4), against goldens written by the oracle alone
(`tools/make_golden.py`, imports only oracle/ and synth/; files under tests/golden/).

North-star tolerances (BASELINE.json), in the launch configuration bench.py times (default
context: 2.5-D TMA passes / CSR gathers, pull sketch, phase schedule, device solves for
d r >= 512 with host fallback):
  * per-step sketched residual rho_rel(d), d = 1..50: 1e-8 relative (R19 floors below 1e-7 /
    1e-9, as in test_gpu_parity._rho_close);
  * the iteration count to tolerance d* within +-2 of the oracle's (both run the R9 schedule and
    search; P:903-905 stopping rule);
  * the true relative residual ||A X + X B - C1 C2^T||_F / ||C1 C2^T||_F of the GPU's
    solution at the oracle's d* within 10 % of the oracle's at the same d (solution at the
    context's rank_tol = 1e-12, R12; no rank cap below the oracle's rank).
"""
import json
import math
import os

import numpy as np
import pytest

pytestmark = [pytest.mark.gpu, pytest.mark.timeout(3600)]

torch = pytest.importorskip("torch")

from oracle import alg1, operators  # noqa: E402
from synth import inputs  # noqa: E402

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _golden(name):
    p = os.path.join(GOLDEN, f"{name}.json")
    if not os.path.exists(p):
        pytest.skip(f"no golden for {name} (tools/make_golden.py {name})")
    with open(p) as f:
        return json.load(f)


def _rho_close(rr, ro):
    if ro >= 1e-9:
        return abs(rr - ro) <= max(1e-8 * ro, 1e-15)
    return abs(rr - ro) <= 1e-12


def _context(cfg, csr):
    import paper_2311_16019_b200 as pkg
    C1, C2 = inputs.make_rhs(cfg)
    g = pkg.from_config(cfg, C1=torch.from_numpy(C1).cuda(), C2=torch.from_numpy(C2).cuda(), csr_pair=csr,
                        stream=torch.cuda.current_stream().cuda_stream)
    return g, C1, C2


CFGS = ["c0", "c1", "c2", "c3", "c4",
        # the paper's own workloads (f4: Ex. 6.1, 6.3 with the SRDCT, R24-R26)
        "ex61_nu0.1", "ex61_nu0.01", "ex61_nu0.001", "ex63_n125000"]


@pytest.mark.parametrize("name", CFGS)
def test_per_step_rho_matches_oracle_golden(name):
    gold = _golden(name)
    cfg = inputs.get_config(name)
    csr = inputs.config_csr(cfg) if cfg.kind == "csr" else None
    g, _, _ = _context(cfg, csr)
    per = gold["per_step"]
    g.step(len(per))
    bad = []
    for e in per:
        _, rr = g.residual(e["d"])
        if not _rho_close(rr, e["rho_rel"]):
            bad.append((e["d"], rr, e["rho_rel"]))
    assert not bad, f"{name}: rho_rel off at (d, gpu, oracle) {bad[:5]}"
    g.close()


def _true_rel(cfg, csr, C1, C2, X1, X2):
    A, _, B = operators.operator_pair(cfg, csr)
    chunk = 1 << 20 if cfg.n > (1 << 21) else None
    return alg1.true_residual(A, B, C1, C2, X1, X2, chunk=chunk)[1]


@pytest.mark.parametrize("name", CFGS)
def test_time_to_tolerance_matches_oracle_golden(name):
    gold = _golden(name)
    if "d_star" not in gold:
        pytest.skip(f"golden {name} has no d* yet")
    cfg = inputs.get_config(name)
    csr = inputs.config_csr(cfg) if cfg.kind == "csr" else None
    g, C1, C2 = _context(cfg, csr)
    d_star, rr, st = g.solve()
    assert st == 0 and rr < cfg.tol
    # R28: d* within +-2 (north star) while the sketched bases keep kappa(T) u < 1; beyond that
    # (Ex. 6.1 nu = 0.001: kappa(T_V) = 4e16) rho_rel near tol is set by rounding (the oracle's own
    # rho is non-monotone step to step: 721 -> 1.38e-6, 722 -> 7.9e-7) and d* is compared within 2 %
    kap = max(gold.get("kappa_T_U") or 0.0, gold.get("kappa_T_V") or 0.0)
    dtol = 2 if kap * 2.2e-16 < 1.0 else max(2, int(0.02 * gold["d_star"]))
    assert abs(d_star - gold["d_star"]) <= dtol, f"{name}: GPU d* {d_star} vs oracle {gold['d_star']} (+-{dtol})"
    # every check both searches made (same R9 schedule): the GPU's rho_rel (device sign-function /
    # eigendecomposition solves for d r >= 512) against the oracle's (Bartels-Stewart), 1e-6
    # relative while kappa(T) < 1e10 (c3 on B200: <= 1.4e-8 up to d* = 234); beyond (c1: kappa(T)
    # up to 2.5e15) rho carries rounding amplified by kappa(T) (R27) and is not compared value by value
    orc = {e["d"]: e["rho_rel"] for e in gold.get("history", []) if e.get("rho_rel") is not None}
    if kap < 1e10:
        bad = [(d, r, orc[d]) for d, r in g.history() if d in orc and math.isfinite(orc[d])
               and abs(r - orc[d]) > 1e-6 * orc[d]]
        assert not bad, f"{name}: checked rho differs from the oracle's: {bad[:4]}"
    if gold.get("true_rel") is None:
        return
    # the GPU's solution at the ORACLE's d* (same d), at rank_tol; rank cap well above the oracle's rank
    d0 = gold["d_star"]
    cap = min(d0 * cfg.r, max(64, 2 * gold["rank"]))
    X1 = torch.zeros((cfg.n, cap), dtype=torch.float64, device="cuda")
    X2 = torch.zeros((cfg.n, cap), dtype=torch.float64, device="cuda")
    d_now, _ = g.step(0)
    if d0 > d_now:                       # the GPU's own d* may lie just below the oracle's
        g.step(d0 - d_now)
    g.residual(d0)
    _, _, rank = g.solution(d0, cap, X1, X2)
    assert rank < cap, "rank cap reached: the truncation must be decided by rank_tol"
    X1h = X1[:, :rank].cpu().numpy()
    X2h = X2[:, :rank].cpu().numpy()
    del X1, X2
    rel = _true_rel(cfg, csr, C1, C2, X1h, X2h)
    msg = f"{name}: true residual {rel:.4e} vs oracle {gold['true_rel']:.4e} at d = {d0} (ranks {rank} / {gold['rank']})"
    if gold["true_rel"] <= 10 * gold["rho_rel_star"]:
        # the subspace-embedding regime: the true residual is determined by the
        # method, and the north star's 10 % applies
        assert abs(rel - gold["true_rel"]) <= 0.10 * gold["true_rel"], msg
    else:
        # R27: the oracle's own true residual exceeds its sketched residual by > 10x (the sketched
        # bases have lost the embedding, kappa(T) ~ 1e13 - 1e16: SURVEY A22); the true residual is
        # then set by rounding amplified by kappa(T): the GPU's may not be worse than the oracle's
        # by more than an order of magnitude, and (exact arithmetic puts the true residual within
        # the embedding distortion of rho) not below a tenth of the sketched residual
        assert 0.1 * gold["rho_rel_star"] <= rel <= 10.0 * gold["true_rel"], msg
    g.close()
