import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, numpy as np
import paper_2311_16019_b200 as pkg
from synth import inputs
cfg = inputs.get_config("c3")
C1, C2 = inputs.make_rhs(cfg)
st = torch.cuda.current_stream().cuda_stream
d1, d2 = torch.from_numpy(C1).cuda(), torch.from_numpy(C2).cuda()
g = pkg.from_config(cfg, C1=d1, C2=d2, stream=st); g.step(5); g.close(); torch.cuda.empty_cache()
for it in range(3):
    C1h = torch.from_numpy(C1).pin_memory(); C2h = torch.from_numpy(C2).pin_memory()
    torch.cuda.synchronize(); t0 = time.perf_counter()
    s2 = pkg.from_config(cfg, C1=C1h, C2=C2h, stream=st)
    torch.cuda.synchronize(); t1 = time.perf_counter()
    s2.step(23); torch.cuda.synchronize(); t2 = time.perf_counter()
    rr = s2.residual(23); torch.cuda.synchronize(); t3 = time.perf_counter()
    s2.close(); t4 = time.perf_counter()
    print(f"it {it}: init {t1-t0:.3f} steps {t2-t1:.3f} residual {t3-t2:.3f} close {t4-t3:.3f}", flush=True)
