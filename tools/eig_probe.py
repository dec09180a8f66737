"""Development probe (not product): is an eigendecomposition-based projected Sylvester solve
with iterative refinement accurate on c1's projected matrices, where the device sign iteration
fails (M_V has eigenvalues with Re < 0)?  Steps c1 to d, takes T and H from the context,
forms M_U, M_V with the host a6 helper, solves with host Bartels-Stewart (reference) and with
torch.linalg.eig on the GPU + refinement, and prints the differences and times.

    python tools/eig_probe.py c1 780
"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2311_16019_b200 as pkg  # noqa: E402
from synth import inputs  # noqa: E402

name, d = sys.argv[1], int(sys.argv[2])
cfg = inputs.get_config(name)
C1, C2 = inputs.make_rhs(cfg)
g = pkg.from_config(cfg, C1=torch.from_numpy(C1).cuda(), C2=torch.from_numpy(C2).cuda(),
                    stream=torch.cuda.current_stream().cuda_stream)
g.step(d)
r, k = cfg.r, cfg.k
m = d * r
HU, TU, bU = g.get_small(0, d)
HV, TV, bV = g.get_small(1, d)
MU = pkg.api.host_projected(d, r, k, TU, HU)
MV = pkg.api.host_projected(d, r, k, TV, HV)
Bm = bU @ bV.T
t0 = time.perf_counter()
Yref = pkg.api.host_sylvester(MU, MV, Bm)
t1 = time.perf_counter()
F = np.zeros((m, m))
F[:r, :r] = Bm
print(f"{name} d={d} m={m}: host BS {t1 - t0:.2f} s; |Yref| {np.linalg.norm(Yref):.3e}; "
      f"host residual {np.linalg.norm(MU @ Yref + Yref @ MV.T - F) / np.linalg.norm(F):.2e}", flush=True)

dev = torch.device("cuda")
A = torch.from_numpy(MU).to(dev)
B = torch.from_numpy(MV.T.copy()).to(dev)
Fd = torch.from_numpy(F).to(dev)
for rep in range(2):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    la, VA = torch.linalg.eig(A)
    lb, VB = torch.linalg.eig(B)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    LUa = torch.linalg.lu_factor(VA)
    LUb = torch.linalg.lu_factor(VB)
    den = la[:, None] + lb[None, :]

    def apply(R):
        G = torch.linalg.lu_solve(*LUa, R.to(torch.complex128))          # VA^-1 R
        G = G @ VB                                                        # (VA^-1 R) VB
        G = G / den
        K = VA @ G
        # K VB^-1 = (VB^-T K^T)^T
        Y = torch.linalg.lu_solve(*LUb, K.transpose(0, 1), adjoint=False, left=True) if False else \
            torch.linalg.lu_solve(*LUb, K, left=False)
        return Y.real

    Y = apply(Fd)
    hist = []
    for it in range(8):
        Rres = Fd - A @ Y - Y @ B
        rn = (torch.linalg.norm(Rres) / torch.linalg.norm(Fd)).item()
        hist.append(rn)
        if rn < 1e-14 or (it > 1 and rn > 0.5 * hist[-2]):
            break
        Y = Y + apply(Rres)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    Yn = Y.cpu().numpy()
    cva = torch.linalg.cond(VA).item()
    cvb = torch.linalg.cond(VB).item()
    ylast = np.linalg.norm(Yn[-r:, :] - Yref[-r:, :]) / np.linalg.norm(Yref[-r:, :])
    ycol = np.linalg.norm(Yn[:, -r:] - Yref[:, -r:]) / np.linalg.norm(Yref[:, -r:])
    print(f"rep {rep}: eig {t1 - t0:.2f} s, LU+refine {t2 - t1:.2f} s; kappa(VA) {cva:.2e} kappa(VB) {cvb:.2e}; "
          f"min |la+lb| {den.abs().min().item():.3e}; residual history {['%.1e' % h for h in hist]}; "
          f"|Y-Yref|/|Yref| {np.linalg.norm(Yn - Yref) / np.linalg.norm(Yref):.2e}, last rows {ylast:.2e}, "
          f"last cols {ycol:.2e}", flush=True)
    print("  eig real parts: MU min", la.real.min().item(), "MV^T min", lb.real.min().item(), flush=True)
g.close()
