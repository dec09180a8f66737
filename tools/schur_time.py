import time, os, numpy as np, scipy.linalg as sla
print("cores", os.cpu_count())
rng = np.random.default_rng(0)
for m in (2000, 3100):
    A = rng.standard_normal((m, m))
    t0 = time.perf_counter(); T, Z = sla.schur(A); print("schur", m, time.perf_counter() - t0, flush=True)
    t0 = time.perf_counter(); H = sla.hessenberg(A); print("hessenberg", m, time.perf_counter() - t0, flush=True)
    t0 = time.perf_counter(); U, s, Vt = np.linalg.svd(A); print("svd", m, time.perf_counter() - t0, flush=True)
