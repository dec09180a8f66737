"""Development probe: cuBLAS DGEMM throughput (through torch) for the second pass's X accumulation
shape X^T (l x n) += M^T (l x kk) U^T (kk x n) against a square DGEMM (fp64 ceiling on B200)."""
import time

import torch

dev = torch.device("cuda")


def bench(m, k, n, reps=5, transb=False):
    a = torch.randn(m, k, dtype=torch.float64, device=dev)
    b = torch.randn(n, k, dtype=torch.float64, device=dev).t() if transb else torch.randn(k, n, dtype=torch.float64, device=dev)
    c = torch.zeros(m, n, dtype=torch.float64, device=dev)
    c.addmm_(a, b)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        c.addmm_(a, b)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    print(f"m={m} k={k} n={n} transb={transb}: {ms:.2f} ms, {2 * m * k * n / ms / 1e9:.1f} TF/s", flush=True)
    del a, b, c
    torch.cuda.empty_cache()


bench(8192, 8192, 8192)
for k in (256, 512, 1024):
    bench(216, k, 1 << 23, transb=True)
bench(256, 256, 1 << 23, transb=True)
