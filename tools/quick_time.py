"""Quick device timing of block steps for one config (development probe)."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2311_16019_b200 as pkg
from synth import inputs

name = sys.argv[1] if len(sys.argv) > 1 else "c3"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 10
cfg = inputs.get_config(name)
t0 = time.time()
csr = inputs.config_csr(cfg) if cfg.kind == "csr" else None
C1, C2 = inputs.make_rhs(cfg)
print(f"{name}: gen {time.time()-t0:.1f}s", flush=True)
t0 = time.time()
serial = "serial" in sys.argv[3:]
notma = "notma" in sys.argv[3:]
g = pkg.from_config(cfg, C1=torch.from_numpy(C1).cuda(), C2=torch.from_numpy(C2).cuda(), csr_pair=csr, timing=True,
                    stream=torch.cuda.current_stream().cuda_stream, serial=serial, tma=not notma)
print("serial" if serial else "two streams")
torch.cuda.synchronize(); print(f"init {time.time()-t0:.2f}s", flush=True)
g.step(3); g.reset_stats()
torch.cuda.synchronize()
e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
e0.record(); d, st = g.step(steps); e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1)
s = g.stats()
R, K, n = cfg.r, cfg.k, cfg.n
print(f"{name} {steps} steps: {ms:.2f} ms total, {ms/steps:.3f} ms/step, d={d}")
for k in ("pass1", "pass2", "skqr", "sketch"):
    nn = s['n_'+k]
    if nn: print(f"  {k}: {s['ms_'+k]/nn*1e3:.1f} us/launch over {nn}")
bp1 = 8*n*R*K; bp2 = 8*n*R*(K+1)
if s['n_pass1']: print(f"  pass1 alg GB/s {bp1/(s['ms_pass1']/s['n_pass1']*1e-3)/1e9:.0f}; pass2 alg GB/s {bp2/(s['ms_pass2']/s['n_pass2']*1e-3)/1e9:.0f}")
t0=time.time(); rho, rr = g.residual(d); print(f"residual d={d} rho_rel={rr:.3e} host {time.time()-t0:.2f}s")
