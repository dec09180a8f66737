import torch, time
torch.backends.cuda.preferred_linalg_library("cusolver")
for m in (512, 1024, 2048, 4096):
    A = torch.randn(m, m, dtype=torch.float64, device="cuda") + m * torch.eye(m, dtype=torch.float64, device="cuda")
    B = torch.randn(m, m, dtype=torch.float64, device="cuda")
    for _ in range(2):
        torch.linalg.lu_factor(A); A @ B; torch.linalg.inv(A)
    torch.cuda.synchronize()
    def t(f, n=5):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        for _ in range(n): f()
        torch.cuda.synchronize(); return (time.perf_counter() - t0) / n * 1e3
    tl = t(lambda: torch.linalg.lu_factor(A))
    LU, piv = torch.linalg.lu_factor(A)
    ts = t(lambda: torch.linalg.lu_solve(LU, piv, B))
    tg = t(lambda: A @ B)
    ti = t(lambda: torch.linalg.inv(A))
    print(f"m={m}: getrf {tl:.2f} ms, getrs(m rhs) {ts:.2f} ms, dgemm {tg:.2f} ms ({2*m**3/tg/1e9:.1f} TF), inv {ti:.2f} ms", flush=True)
