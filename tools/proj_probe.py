import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, numpy as np
import paper_2311_16019_b200 as pkg
from synth import inputs
cfg = inputs.small_config(kind="stencil2d", N=23, r=1, k=2, d_max=60)
C1, C2 = inputs.make_rhs(cfg)
st = torch.cuda.current_stream().cuda_stream
for proj in ("gpu", "host"):
    g = pkg.from_config(cfg, C1=torch.from_numpy(C1).cuda(), C2=torch.from_numpy(C2).cuda(), stream=st, proj=proj)
    g.step(40)
    print(proj, g.residual(40), g.stats()["gpu_solves"], g.stats()["gpu_solve_fallbacks"], g.last_error(), flush=True)
