"""c1 near the crossing: rho_rel(d) from host Bartels-Stewart vs the device sign-function
solve, on the same steps (development probe)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2311_16019_b200 as pkg
from synth import inputs
cfg = inputs.get_config("c1")
C1, C2 = inputs.make_rhs(cfg)
ds = [int(x) for x in sys.argv[1].split(",")] if len(sys.argv) > 1 else [700, 760, 780, 790, 800, 820, 840]
ctx = {}
for mode in ("host", "gpu"):
    g = pkg.from_config(cfg, C1=torch.from_numpy(C1).cuda(), C2=torch.from_numpy(C2).cuda(),
                        stream=torch.cuda.current_stream().cuda_stream, proj=mode)
    g.step(max(ds) + 1)
    ctx[mode] = g
for d in ds:
    out = []
    for mode in ("host", "gpu"):
        t0 = time.perf_counter()
        try:
            rho, rr = ctx[mode].residual(d)
        except Exception as e:
            rr = float("nan")
        out.append((mode, rr, time.perf_counter() - t0))
    print(d, " ".join(f"{m}: {rr:.6e} ({t:.1f}s)" for m, rr, t in out), flush=True)
print("gpu stats", {k: v for k, v in ctx["gpu"].stats().items() if "solve" in k})
