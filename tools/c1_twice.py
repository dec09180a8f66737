"""Two c1 solves in one process: the second context reuses the first one's pooled device
memory (development probe for reads of uninitialised memory)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2311_16019_b200 as pkg
from synth import inputs
cfg = inputs.get_config(sys.argv[1] if len(sys.argv) > 1 else "c1")
C1, C2 = inputs.make_rhs(cfg)
st = torch.cuda.Stream()
for it in range(2):
    g = pkg.from_config(cfg, C1=torch.from_numpy(C1).cuda(), C2=torch.from_numpy(C2).cuda(), stream=st.cuda_stream)
    t0 = time.perf_counter()
    d, rr, s = g.solve()
    s2 = g.stats()
    print(it, "d*", d, rr, s, f"{time.perf_counter()-t0:.1f}s", "gpu_solves", s2["gpu_solves"], "fallbacks",
          s2.get("gpu_solve_fallbacks"), flush=True)
    print("history", [(a, f"{b:.4e}") for a, b in g.history()[-14:]], flush=True)
    g.close()
