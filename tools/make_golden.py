"""Write tests/golden/<cfg>.json from the ORACLE ONLY (imports oracle/ and synth/, nothing else).

Per BASELINE config (VERDICT r1 "Next" 1; north_star tolerances):
  rho_rel(d), rho(d) for d = 1..min(50, d*)      per-step sketched residual (R4, R8)
  d*, rho_rel(d*), converged, check history       Alg. 1 + the canonical search (R9)
  kappa(T_U), kappa(T_V) at d*
  rank l at rank_tol = 1e-12 and the true residual ||A X + X B - C1 C2^T||_F / ||C1 C2^T||_F
  of X = X1 X2^T (O8) at d*
  oracle timings on this machine (host cores stated; informative only)

Usage: python tools/make_golden.py c2 [--parity 50] [--no-solution]
"""
import argparse
import json
import math
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

from oracle import alg1, operators  # noqa: E402
from synth import inputs  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("cfg")
    ap.add_argument("--parity", type=int, default=50)
    ap.add_argument("--no-solution", action="store_true")
    ap.add_argument("--mem-gb", type=float, default=40.0, help="skip the true residual above this estimate")
    a = ap.parse_args()
    cfg = inputs.get_config(a.cfg)
    out_path = os.path.join(ROOT, "tests", "golden", f"{cfg.name}.json")
    os.makedirs(os.path.dirname(out_path), exist_ok=True)
    rec = {"config": cfg.name, "n": cfg.n, "r": cfg.r, "k": cfg.k, "d_max": cfg.d_max, "s": cfg.s,
           "zeta": cfg.zeta, "tol": cfg.tol, "rank_tol": alg1.RANK_TOL,
           "generator": "tools/make_golden.py (oracle/ + synth/ only)",
           "host": {"cores": os.cpu_count()}}

    def dump():
        with open(out_path + ".tmp", "w") as f:
            json.dump(rec, f, indent=1)
        os.replace(out_path + ".tmp", out_path)

    t0 = time.perf_counter()
    csr = inputs.config_csr(cfg) if cfg.kind == "csr" else None
    obj = alg1.SylvesterSketchedKrylov.from_config(cfg, csr_pair=csr)
    rec["setup_s"] = time.perf_counter() - t0
    print(f"[{cfg.name}] setup {rec['setup_s']:.1f}s", flush=True)

    # per-step rho for d = 1..parity (every step, exact Bartels-Stewart)
    per = []
    tstep = 0.0
    for d in range(1, a.parity + 1):
        t1 = time.perf_counter()
        obj.step()
        tstep += time.perf_counter() - t1
        res = obj.residual(d)
        per.append({"d": d, "rho": res.rho, "rho_rel": res.rho_rel, "singular": res.singular,
                    "solve_s": res.seconds})
        if d % 10 == 0:
            print(f"[{cfg.name}] d={d} rho_rel={res.rho_rel:.6e} ({tstep / d:.2f}s/step)", flush=True)
        if obj.breakdown:
            break
    rec["per_step"] = per
    rec["oracle_step_s_mean"] = tstep / max(1, len(per))
    dump()

    # full solve with the canonical schedule + search (R9); the steps already made are reused
    t1 = time.perf_counter()
    sol = alg1.solve(obj, cfg.tol, cfg.d_max)
    rec["solve_wall_s"] = time.perf_counter() - t1
    rec["d_star"] = sol.d_star
    rec["rho_rel_star"] = sol.rho_rel
    rec["converged"] = sol.converged
    rec["history"] = [{"d": h.d, "rho_rel": h.rho_rel, "singular": h.singular, "solve_s": h.seconds}
                      for h in sol.history]
    rec["steps_done"] = obj.d
    rec["breakdown"] = obj.breakdown
    rec["oracle_time_to_tol_s"] = rec["setup_s"] + tstep + rec["solve_wall_s"]
    m = sol.d_star * cfg.r
    rec["kappa_T_U"] = float(np.linalg.cond(obj.U.T[:m, :m]))
    rec["kappa_T_V"] = float(np.linalg.cond(obj.V.T[:m, :m]))
    print(f"[{cfg.name}] d*={sol.d_star} rho_rel={sol.rho_rel:.6e} conv={sol.converged} "
          f"solve {rec['solve_wall_s']:.1f}s", flush=True)
    dump()
    if a.no_solution or sol.Y is None:
        return
    sig = np.linalg.svd(sol.Y, compute_uv=False)
    ell = int(np.count_nonzero(sig > alg1.RANK_TOL * sig[0]))
    rec["rank"] = ell
    rec["sigma_head"] = [float(x) for x in sig[:8]]
    # memory-lean second pass: one sequence's factor at a time (X1 -> R_L, then X2 -> R_R; the
    # same quantities as alg1.solution + alg1.true_residual, O8), row-blocked R-factors
    est_gb = cfg.n * ell * 8 / 1e9
    rec["true_residual_mem_est_gb"] = est_gb
    if est_gb > a.mem_gb:
        rec["true_residual"] = None
        rec["true_residual_skipped"] = f"memory estimate {est_gb:.0f} GB > {a.mem_gb} GB"
        dump()
        return
    obj.U.U.clear()                     # the window blocks are not needed by the replay
    obj.V.U.clear()
    import scipy.linalg as sla
    W, sg, Zt = np.linalg.svd(sol.Y)
    m = sol.d_star * cfg.r
    Y1 = W[:, :ell] * np.sqrt(sg[:ell])[None, :]
    Y2 = Zt[:ell].T * np.sqrt(sg[:ell])[None, :]
    A, _, B = operators.operator_pair(cfg, csr)
    chunk = 1 << 20 if cfg.n > (1 << 21) else None
    t1 = time.perf_counter()
    X1 = obj.U.replay(sla.solve_triangular(obj.U.T[:m, :m], Y1, lower=False), sol.d_star)
    RL = alg1.residual_rfactor_L(A, X1, obj.C1, chunk)
    del X1
    X2 = obj.V.replay(sla.solve_triangular(obj.V.T[:m, :m], Y2, lower=False), sol.d_star)
    RR = alg1.residual_rfactor_R(B, X2, obj.C2, chunk)
    del X2
    rec["second_pass_s"] = time.perf_counter() - t1
    res, rel = alg1.residual_from_rfactors(RL, RR, ell, obj.C1, obj.C2)
    rec["true_residual"] = res
    rec["true_rel"] = rel
    print(f"[{cfg.name}] rank {ell} true_rel {rel:.6e} (second pass {rec['second_pass_s']:.1f}s)", flush=True)
    dump()


if __name__ == "__main__":
    main()
