"""Development probe: P virtual ranks (LocalGroup) on one GPU, a few steps."""
import sys, os, threading, time, faulthandler
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
faulthandler.dump_traceback_later(50, exit=True)
import numpy as np, torch
import paper_2311_16019_b200 as pkg
from synth import inputs
N, r, k, P, steps = (int(x) for x in sys.argv[1:6])
tma = len(sys.argv) < 7 or sys.argv[6] != "notma"
cfg = inputs.small_config(kind="stencil3d", N=N, r=r, k=k, d_max=20)
C1, C2 = inputs.make_rhs(cfg)
grp = pkg.LocalGroup(P)
def worker(rank):
    torch.cuda.set_device(0)
    b, e = pkg.partition(cfg, P, rank)
    comm = grp.comm(rank)
    st = torch.cuda.Stream()
    print(f"rank {rank} rows {b}:{e} init", flush=True)
    g = pkg.from_config(cfg, C1=torch.from_numpy(C1[b:e]).cuda(), C2=torch.from_numpy(C2[b:e]).cuda(),
                        stream=st.cuda_stream, comm=comm, row_range=(b, e), tma=tma)
    print(f"rank {rank} init done", flush=True)
    for d in range(1, steps + 1):
        g.step(1)
        print(f"rank {rank} step {d} rho {g.residual(d)[1]:.6e}", flush=True)
    g.close(); comm.close()
th = [threading.Thread(target=worker, args=(i,)) for i in range(P)]
[t.start() for t in th]; [t.join() for t in th]
print("done")
