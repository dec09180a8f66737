import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, numpy as np
import paper_2311_16019_b200 as pkg
from synth import inputs
cfg = inputs.get_config("c1")
C1, C2 = inputs.make_rhs(cfg)
st = torch.cuda.current_stream().cuda_stream
g = pkg.from_config(cfg, C1=torch.from_numpy(C1).cuda(), C2=torch.from_numpy(C2).cuda(), stream=st, proj="gpu")
h = pkg.from_config(cfg, C1=torch.from_numpy(C1).cuda(), C2=torch.from_numpy(C2).cuda(), stream=st, proj="host")
done = 0
for d in (150, 300, 500, 700, 780, 781, 789):
    g.step(d - done); h.step(d - done); done = d
    t0 = time.time(); rg = g.residual(d)[1]; tg = time.time() - t0
    t0 = time.time(); rh = h.residual(d)[1]; th = time.time() - t0
    s = g.stats()
    print(f"d={d} gpu {rg:.6e} ({tg:.2f}s, solves {s['gpu_solves']} fb {s['gpu_solve_fallbacks']}) host {rh:.6e} ({th:.2f}s) rel {abs(rg-rh)/rh:.2e} | {g.last_error()}", flush=True)
