"""Full-size checks in the configuration bench.py times (BASELINE configs, default context:
2.5-D TMA passes / CSR gathers, pull sketch, phase schedule), through properties the paper fixes
at any size — the oracle cannot run these sizes step by step:

  * Arnoldi relation of the truncated basis (Alg. 1 lines 3-8):
        A U_d = sum_{i=d-k+1}^{d} U_i h_{i,d} + U_{d+1} h_{d+1,d}
    with A applied on the host by the oracle's own sparse operator (scipy), the blocks and the
    H columns from the library;
  * orthonormality of the k+1 window blocks (CGS + CholQR, R5);
  * the sketched QR relation S [U_1 .. U_{d+1}] = Q_{d+1} T_{d+1} (Prop. 2.1):
    its Gram restricted to the new block, (S U_{d+1})^T (S U_{d+1}) = T[:, new]^T T[:, new],
    with S U_{d+1} from the library's apply_sketch (itself checked against the oracle's
    hashed S at every config size in test_gpu_parity).
Tolerances: 1e-11 relative (Arnoldi), 1e-10 (orthonormality, sketch Gram) — rounding of
O(n)-term sums at n up to 1.7e7.
"""
import numpy as np
import pytest

pytestmark = [pytest.mark.gpu, pytest.mark.timeout(1800)]

torch = pytest.importorskip("torch")

from oracle import operators  # noqa: E402
from synth import inputs  # noqa: E402


def _rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


@pytest.mark.parametrize("name,seqs", [("c3", (0, 1)), ("c2", (0, 1)), ("c4", (0, 1)), ("c1", (0, 1))])
def test_fullsize_invariants(name, seqs):
    import paper_2311_16019_b200 as pkg
    cfg = inputs.get_config(name)
    csr = inputs.config_csr(cfg) if cfg.kind == "csr" else None
    C1, C2 = inputs.make_rhs(cfg)
    g = pkg.from_config(cfg, C1=torch.from_numpy(C1).cuda(), C2=torch.from_numpy(C2).cuda(), csr_pair=csr,
                        stream=torch.cuda.current_stream().cuda_stream)
    d, k, r = 5, cfg.k, cfg.r
    g.step(d)
    A, Bt, _ = operators.operator_pair(cfg, csr)
    for which in seqs:
        M = A if which == 0 else Bt
        H, T, _ = g.get_small(which, d)
        blocks = {j: g.get_block(which, j) for j in range(d + 1 - k, d + 2)}
        # Arnoldi relation for column block d
        lhs = M @ blocks[d]
        rhs = np.zeros_like(lhs)
        for i in range(max(1, d - k + 1), d + 2):
            rhs += blocks[i] @ H[(i - 1) * r:i * r, (d - 1) * r:d * r]
        assert _rel(rhs, lhs) <= 1e-11, (name, which, _rel(rhs, lhs))
        # orthonormal window
        W = np.concatenate([blocks[j] for j in sorted(blocks)], axis=1)
        G = W.T @ W
        assert np.abs(G - np.eye(G.shape[0])).max() <= 1e-10, (name, which, np.abs(G - np.eye(G.shape[0])).max())
        # sketched QR relation for the new block
        SU = g.apply_sketch(which, torch.from_numpy(np.ascontiguousarray(blocks[d + 1])).cuda())
        Tn = T[:(d + 1) * r, d * r:(d + 1) * r]
        assert _rel(SU.T @ SU, Tn.T @ Tn) <= 1e-10, (name, which, _rel(SU.T @ SU, Tn.T @ Tn))
        del blocks, W, lhs, rhs
    g.close()


@pytest.mark.parametrize("name,P", [("c3", 2), ("c4", 3)])
def test_fullsize_sharded_matches_unsharded(name, P):
    """The row-sharded path (virtual ranks of one process, the same code as NCCL ranks) at a
    full BASELINE size: per-step rho and T equal the unsharded run up to reduction order."""
    import threading
    import paper_2311_16019_b200 as pkg
    cfg = inputs.get_config(name)
    csr = inputs.config_csr(cfg) if cfg.kind == "csr" else None
    C1, C2 = inputs.make_rhs(cfg)
    nsteps = 6
    g = pkg.from_config(cfg, C1=torch.from_numpy(C1).cuda(), C2=torch.from_numpy(C2).cuda(), csr_pair=csr,
                        stream=torch.cuda.current_stream().cuda_stream)
    rho1 = []
    for d in range(1, nsteps + 1):
        g.step(1)
        rho1.append(g.residual(d)[1])
    T1 = g.get_small(0, nsteps)[1]
    g.close()
    torch.cuda.empty_cache()
    grp = pkg.LocalGroup(P)
    out, errs = [None] * P, []

    def worker(rank):
        try:
            torch.cuda.set_device(0)
            b, e = pkg.partition(cfg, P, rank)
            comm = grp.comm(rank)
            st = torch.cuda.Stream()
            h = pkg.from_config(cfg, C1=torch.from_numpy(C1[b:e]).cuda(), C2=torch.from_numpy(C2[b:e]).cuda(),
                                csr_pair=csr, stream=st.cuda_stream, comm=comm, row_range=(b, e))
            rho = []
            for d in range(1, nsteps + 1):
                h.step(1)
                rho.append(h.residual(d)[1])
            out[rank] = (rho, h.get_small(0, nsteps)[1])
            h.close()
            comm.close()
        except Exception as ex:  # surfaced below
            errs.append((rank, ex))

    th = [threading.Thread(target=worker, args=(r,)) for r in range(P)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=900)
    grp.close()
    assert not errs, errs
    for rho, T in out:
        for d, (a, b) in enumerate(zip(rho, rho1), 1):
            assert abs(a - b) <= 1e-10 * b + 1e-15, (name, d, a, b)
        assert _rel(T, T1) <= 1e-10
