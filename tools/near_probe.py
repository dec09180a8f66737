"""Step a config to d0 (default d* - 30), then run N more steps (development probe for the
sketch-space kernels near d*; run under ncu with --launch-skip)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2311_16019_b200 as pkg
from synth import inputs
name, d0, nn = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
cfg = inputs.get_config(name)
csr = inputs.config_csr(cfg) if cfg.kind == "csr" else None
C1, C2 = inputs.make_rhs(cfg)
g = pkg.from_config(cfg, C1=torch.from_numpy(C1).cuda(), C2=torch.from_numpy(C2).cuda(), csr_pair=csr,
                    stream=torch.cuda.current_stream().cuda_stream, serial=True)
g.step(d0)
torch.cuda.synchronize()
l0 = g.stats()["launches"]
print("launches before", l0, flush=True)
torch.cuda.nvtx.range_push("probe")
g.step(nn)
torch.cuda.synchronize()
torch.cuda.nvtx.range_pop()
print("launches after", g.stats()["launches"], flush=True)
