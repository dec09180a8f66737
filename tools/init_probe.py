import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, numpy as np
import paper_2311_16019_b200 as pkg
from synth import inputs
cfg = inputs.get_config(sys.argv[1] if len(sys.argv) > 1 else "c3")
C1, C2 = inputs.make_rhs(cfg)
d1, d2 = torch.from_numpy(C1).cuda(), torch.from_numpy(C2).cuda()
h1, h2 = torch.from_numpy(C1).pin_memory(), torch.from_numpy(C2).pin_memory()
st = torch.cuda.current_stream().cuda_stream
for it in range(3):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    g = pkg.from_config(cfg, C1=d1 if it < 2 else h1, C2=d2 if it < 2 else h2, stream=st)
    torch.cuda.synchronize(); t1 = time.perf_counter()
    g.step(1); torch.cuda.synchronize(); t2 = time.perf_counter()
    g.close(); torch.cuda.synchronize(); t3 = time.perf_counter()
    print(f"it {it}: init {t1-t0:.3f}s first step {t2-t1:.3f}s close {t3-t2:.3f}s", flush=True)
