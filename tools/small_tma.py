"""Development probe: a few block steps of a small 3-D r=8 case (TMA pass path)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2311_16019_b200 as pkg
from synth import inputs
N = int(sys.argv[1]) if len(sys.argv) > 1 else 20
k = int(sys.argv[2]) if len(sys.argv) > 2 else 2
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 4
cfg = inputs.small_config(kind="stencil3d", N=N, r=8, k=k, d_max=20)
C1, C2 = inputs.make_rhs(cfg)
g = pkg.from_config(cfg, C1=torch.from_numpy(C1).cuda(), C2=torch.from_numpy(C2).cuda(),
                    stream=torch.cuda.current_stream().cuda_stream, serial=True)
for i in range(steps):
    print(N, k, i + 1, g.step(1), flush=True)
