"""Time to tolerance of the full solve (step + check schedule + bisection) for one config:
GPU step time and host projected-solve time separately (development probe)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2311_16019_b200 as pkg
from synth import inputs
name = sys.argv[1]
cfg = inputs.get_config(name)
if len(sys.argv) > 2:
    cfg = cfg.replace(d_max=int(sys.argv[2]), s=4 * int(sys.argv[2]) * cfg.r)
csr = inputs.config_csr(cfg) if cfg.kind == "csr" else None
C1, C2 = inputs.make_rhs(cfg)
torch.cuda.synchronize()
t0 = time.perf_counter()
g = pkg.from_config(cfg, C1=torch.from_numpy(C1).cuda(), C2=torch.from_numpy(C2).cuda(), csr_pair=csr,
                    stream=torch.cuda.current_stream().cuda_stream)
torch.cuda.synchronize()
t1 = time.perf_counter()
try:
    d, rr, st = g.solve()
except Exception as e:
    print("solve error", e)
    d, rr, st = -1, float("nan"), -1
torch.cuda.synchronize()
t2 = time.perf_counter()
s = g.stats()
print(f"{name}: d*={d} rho_rel={rr:.3e} status={st} init {t1-t0:.2f}s solve {t2-t1:.2f}s approx {s.get('gpu_approx_checks')} "
      f"(host solves {s['host_solves']} taking {s['host_solve_s']:.2f}s; steps {s['steps']})", flush=True)
print("history", g.history())
print("last_error", g.last_error())
