"""Host Bartels-Stewart at c1 sizes: the two Schur decompositions serial vs on two threads."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2311_16019_b200 as pkg
from synth import inputs
cfg = inputs.get_config("c1")
C1, C2 = inputs.make_rhs(cfg)
g = pkg.from_config(cfg, C1=torch.from_numpy(C1).cuda(), C2=torch.from_numpy(C2).cuda(),
                    stream=torch.cuda.current_stream().cuda_stream, proj="host")
g.step(800)
print("cores", os.cpu_count(), flush=True)
for d in (500, 782):
    for mode in ("serial", "threads", "serial", "threads"):
        if mode == "serial":
            os.environ["SYLV_HOST_SERIAL"] = "1"
        else:
            os.environ.pop("SYLV_HOST_SERIAL", None)
        t0 = time.perf_counter()
        rho, rr = g.residual(d)
        print(d, mode, f"{time.perf_counter() - t0:.2f}s", rr, flush=True)
