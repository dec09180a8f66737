"""Rank of the truncated solution at rank_tol = 1e-12 (R12) at d* for each config (development probe)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2311_16019_b200 as pkg
from synth import inputs
for name in sys.argv[1:]:
    cfg = inputs.get_config(name)
    csr = inputs.config_csr(cfg) if cfg.kind == "csr" else None
    C1, C2 = inputs.make_rhs(cfg)
    g = pkg.from_config(cfg, C1=torch.from_numpy(C1).cuda(), C2=torch.from_numpy(C2).cuda(), csr_pair=csr,
                        stream=torch.cuda.current_stream().cuda_stream)
    t0 = time.perf_counter()
    d, rr, st = g.solve()
    t1 = time.perf_counter()
    cap = min(d * cfg.r, int(os.environ.get("CAP", "256")))
    X1 = torch.zeros((cfg.n, cap), dtype=torch.float64, device="cuda")
    X2 = torch.zeros((cfg.n, cap), dtype=torch.float64, device="cuda")
    t2 = time.perf_counter()
    _, _, rank = g.solution(d, cap, X1, X2)
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    print(f"{name}: d*={d} rho_rel={rr:.4e} solve {t1-t0:.2f}s rank {rank} (cap {cap}) second pass {t3-t2:.2f}s "
          f"stats {g.stats()}", flush=True)
    print("history", g.history(), flush=True)
    del X1, X2
    g.close()
    torch.cuda.empty_cache()
