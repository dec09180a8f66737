"""Second pass (sylv_sketch_solution) phase times at a config's d* (development probe)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["SYLV_TRACE_INIT"] = "1"
import torch
import paper_2311_16019_b200 as pkg
from synth import inputs
name = sys.argv[1] if len(sys.argv) > 1 else "c3"
d = int(sys.argv[2]) if len(sys.argv) > 2 else 234
cfg = inputs.get_config(name)
C1, C2 = inputs.make_rhs(cfg)
g = pkg.from_config(cfg, C1=torch.from_numpy(C1).cuda(), C2=torch.from_numpy(C2).cuda(),
                    stream=torch.cuda.current_stream().cuda_stream)
g.step(d)
t0 = time.perf_counter(); g.residual(d); print("residual", time.perf_counter() - t0, flush=True)
for mr in (32, 8):
    X1 = torch.empty((cfg.n, mr), dtype=torch.float64, device="cuda")
    X2 = torch.empty((cfg.n, mr), dtype=torch.float64, device="cuda")
    torch.cuda.synchronize(); t0 = time.perf_counter()
    _, _, rk = g.solution(d, mr, X1, X2)
    torch.cuda.synchronize(); print("solution max_rank", mr, "rank", rk, time.perf_counter() - t0, flush=True)
