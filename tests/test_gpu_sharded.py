"""Row-sharded contexts on one GPU.

P virtual ranks of ONE process (sylv_local_group_create; one host thread per rank, every
rank's kernels on its own streams, transports = plain device sums/copies ordered by CUDA
events, no kernel waits on another) run the same code path as NCCL ranks: halo exchange of
each new block's boundary planes/lines, allreduce of the Gram-Schmidt inner products and
Grams, allreduce of the partial sketches (S hashed on GLOBAL rows); CSR operators are split
into 32-row-group ranges with band-wide ghost rows.  The sharded run must
reproduce the unsharded GPU run up to reduction order (1e-10 relative on rho and on the
basis blocks) and the CPU oracle to the parity tolerance (rho 1e-8 relative, d <= 50).
The NCCL transport itself is exercised at world size 1 (one GPU per gpurun call).
"""
import ctypes as C
import threading

import numpy as np
import pytest

pytestmark = [pytest.mark.gpu, pytest.mark.timeout(1200)]

torch = pytest.importorskip("torch")

from oracle import alg1  # noqa: E402
from synth import inputs  # noqa: E402


def _pkg():
    import paper_2311_16019_b200 as pkg
    return pkg


CASES = {
    # (config, ranks, tma)
    "3d-r8k3-tma-P2": (dict(kind="stencil3d", N=34, r=8, k=3, d_max=40), 2, True),
    "3d-r8k3-tma-P3": (dict(kind="stencil3d", N=34, r=8, k=3, d_max=40), 3, True),
    "3d-r8k2-generic-P2": (dict(kind="stencil3d", N=32, r=8, k=2, d_max=40), 2, False),
    "3d-r4k2-P4": (dict(kind="stencil3d", N=32, r=4, k=2, d_max=40), 4, True),
    "2d-r4k2-P3": (dict(kind="stencil2d", N=64, r=4, k=2, d_max=40), 3, True),
    "2d-r1k2-P2": (dict(kind="stencil2d", N=64, r=1, k=2, d_max=40), 2, True),
    # pull sketch (sketch_pull.cuh) on shards: global group offsets m0 > 0 in the sorted lists
    "3d-r8k3-tma-P3-pull": (dict(kind="stencil3d", N=34, r=8, k=3, d_max=40), 3, True, "pull"),
    "2d-r4k2-P3-pull": (dict(kind="stencil2d", N=64, r=4, k=2, d_max=40), 3, True, "pull"),
    # row-sharded CSR (c4's decomposition): ghost rows = band, global CSR on every rank
    "csr-r2k2-P2": (dict(kind="csr", n=20011, nnz_off=20, band=300, r=2, k=2, d_max=40), 2, True),
    "csr-r4k3-P3": (dict(kind="csr", n=9001, nnz_off=6, band=500, r=4, k=3, d_max=40), 3, True),
    "csr-r1k2-P4": (dict(kind="csr", n=6007, nnz_off=6, band=100, r=1, k=2, d_max=40), 4, True),
}
NSTEPS = 16


def _rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def _unsharded(cfg, C1, C2, tma, nsteps):
    g = _pkg().from_config(cfg, C1=torch.from_numpy(C1).cuda(), C2=torch.from_numpy(C2).cuda(),
                           stream=torch.cuda.current_stream().cuda_stream, tma=tma)
    rho = []
    for d in range(1, nsteps + 1):
        g.step(1)
        rho.append(g.residual(d)[1])
    blocks = {w: [g.get_block(w, j) for j in range(nsteps + 2 - cfg.k, nsteps + 2)] for w in (0, 1)}
    sk = g.apply_sketch(0, torch.from_numpy(C1).cuda())
    g.close()
    return rho, blocks, sk


def _sharded(cfg, C1, C2, P, tma, nsteps, solution_rank=0):
    pkg = _pkg()
    grp = pkg.LocalGroup(P)
    out = [None] * P
    errs = []

    def worker(rank):
        try:
            torch.cuda.set_device(0)
            b, e = pkg.partition(cfg, P, rank)
            comm = grp.comm(rank)
            st = torch.cuda.Stream()
            g = pkg.from_config(cfg, C1=torch.from_numpy(C1[b:e]).cuda(), C2=torch.from_numpy(C2[b:e]).cuda(),
                                stream=st.cuda_stream, comm=comm, row_range=(b, e), tma=tma)
            rho = []
            for d in range(1, nsteps + 1):
                g.step(1)
                rho.append(g.residual(d)[1])
            blocks = {w: [g.get_block(w, j) for j in range(nsteps + 2 - cfg.k, nsteps + 2)] for w in (0, 1)}
            sk = g.apply_sketch(0, torch.from_numpy(C1[b:e]).cuda())
            H, T, beta = g.get_small(0, nsteps)
            X1, X2, rk = g.solution(nsteps, solution_rank) if solution_rank else (None, None, 0)
            out[rank] = dict(rows=(b, e), rho=rho, blocks=blocks, sk=sk, H=H, T=T, X1=X1, X2=X2, rank=rk)
            g.close()
            comm.close()
        except Exception as ex:  # surfaced below
            errs.append((rank, ex))

    th = [threading.Thread(target=worker, args=(r,)) for r in range(P)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=600)
    grp.close()
    assert not errs, errs
    return out


@pytest.mark.parametrize("name", list(CASES))
def test_sharded_equals_unsharded(name, monkeypatch):
    kw, P, tma = CASES[name][:3]
    if len(CASES[name]) > 3:
        monkeypatch.setenv("SYLV_SKETCH", CASES[name][3])
    cfg = inputs.small_config(**kw)
    C1, C2 = inputs.make_rhs(cfg)
    rho1, blocks1, sk1 = _unsharded(cfg, C1, C2, tma, NSTEPS)
    shards = _sharded(cfg, C1, C2, P, tma, NSTEPS)
    # row ranges tile [0, n) in rank order
    assert shards[0]["rows"][0] == 0 and shards[-1]["rows"][1] == cfg.n
    assert all(shards[i]["rows"][1] == shards[i + 1]["rows"][0] for i in range(P - 1))
    for sh in shards:
        # every rank reaches the same (replicated) projected quantities
        np.testing.assert_array_equal(sh["rho"], shards[0]["rho"])
        np.testing.assert_array_equal(sh["T"], shards[0]["T"])
        # rho_rel is normalised by ||C1 C2^T||: the reduction-order rounding of the sharded
        # sums is ~1e-16 of that scale, so below rho_rel ~ 1e-6 an absolute floor applies
        for d, (a, b) in enumerate(zip(sh["rho"], rho1), 1):
            assert abs(a - b) <= 1e-10 * b + 1e-15, (name, d, a, b)
        assert _rel(sh["sk"], sk1) <= 1e-12
    for w in (0, 1):
        for i in range(cfg.k):
            full = np.concatenate([sh["blocks"][w][i] for sh in shards])
            assert _rel(full, blocks1[w][i]) <= 1e-10, (name, w, i)


@pytest.mark.parametrize("name", ["3d-r8k3-tma-P3", "csr-r2k2-P2"])
def test_sharded_matches_oracle_and_solution(name):
    kw, P, tma = CASES[name][:3]
    cfg = inputs.small_config(**kw)
    C1, C2 = inputs.make_rhs(cfg)
    csr = inputs.config_csr(cfg) if cfg.kind == "csr" else None
    orc = alg1.SylvesterSketchedKrylov.from_config(cfg, C1=C1, C2=C2, csr_pair=csr)
    ro = []
    for d in range(1, NSTEPS + 1):
        orc.step(1)
        ro.append(orc.residual(d).rho_rel)
    shards = _sharded(cfg, C1, C2, P, tma, NSTEPS, solution_rank=48)
    # the parity rule of test_gpu_parity._rho_close: 1e-8 relative while rho_rel >= 1e-9
    # (three decades below tol), rounding-noise floor 1e-12 below that
    for d, (a, b) in enumerate(zip(shards[0]["rho"], ro), 1):
        assert abs(a - b) <= (max(1e-8 * b, 1e-15) if b >= 1e-9 else 1e-12), (d, a, b)
    # the factored solution, assembled from the ranks' rows, equals the unsharded one
    g = _pkg().from_config(cfg, C1=torch.from_numpy(C1).cuda(), C2=torch.from_numpy(C2).cuda(),
                           stream=torch.cuda.current_stream().cuda_stream)
    g.step(NSTEPS)
    g.residual(NSTEPS)
    X1, X2, rk = g.solution(NSTEPS, 48)
    g.close()
    assert all(sh["rank"] == rk for sh in shards)
    Xs1 = np.concatenate([np.asarray(sh["X1"]) for sh in shards])
    Xs2 = np.concatenate([np.asarray(sh["X2"]) for sh in shards])
    assert _rel(Xs1 @ Xs2.T, np.asarray(X1) @ np.asarray(X2).T) <= 1e-9


def test_nccl_transport_world_size_one():
    """The NCCL transport (communicator split per channel, allreduce, halo with no
    neighbours) at world size 1 reproduces the unsharded context bit for bit."""
    pkg = _pkg()
    lib = pkg.load_library()
    uid = (C.c_uint8 * 128)()
    assert lib.sylv_comm_nccl_unique_id(uid) == 0
    h = C.c_void_p()
    assert lib.sylv_comm_create_nccl(1, 0, uid, C.byref(h)) == 0
    comm = pkg.Comm(h)
    cfg = inputs.small_config(kind="stencil3d", N=34, r=8, k=3, d_max=40)
    C1, C2 = inputs.make_rhs(cfg)
    st = torch.cuda.current_stream().cuda_stream
    a = pkg.from_config(cfg, C1=torch.from_numpy(C1).cuda(), C2=torch.from_numpy(C2).cuda(), stream=st, comm=comm,
                        row_range=(0, cfg.n))
    b = pkg.from_config(cfg, C1=torch.from_numpy(C1).cuda(), C2=torch.from_numpy(C2).cuda(), stream=st)
    for d in range(1, 11):
        a.step(1)
        b.step(1)
        assert a.residual(d)[1] == b.residual(d)[1]
    a.close()
    b.close()
    comm.close()


def test_csr_operator_passed_already_transposed():
    """sylv_operator.is_transposed: passing B^T's CSR arrays (no device transpose) gives the same
    iteration as passing B (the library transposes on the device)."""
    import scipy.sparse as sp
    pkg = _pkg()
    cfg = inputs.small_config(kind="csr", n=5003, nnz_off=6, band=40, r=2, k=2, d_max=30)
    (ra, ca, va), (rb, cb, vb) = inputs.config_csr(cfg)
    C1, C2 = inputs.make_rhs(cfg)
    Bt = sp.csr_matrix((vb, cb.astype(np.int64), rb), shape=(cfg.n, cfg.n)).T.tocsr()
    Bt.sort_indices()
    runs = []
    for transposed in (False, True):
        A = pkg.csr_operator(cfg.n, ra, ca, va)
        Bop = (pkg.csr_operator(cfg.n, Bt.indptr.astype(np.int64), Bt.indices.astype(np.int32), Bt.data,
                                is_transposed=True) if transposed else pkg.csr_operator(cfg.n, rb, cb, vb))
        g = pkg.SylvSketch(A[0], Bop[0], torch.from_numpy(C1).cuda(), torch.from_numpy(C2).cuda(), r=cfg.r, k=cfg.k,
                           d_max=cfg.d_max, s=cfg.s, keep=[A[1], Bop[1]])
        g.step(15)
        runs.append([g.residual(d)[1] for d in range(1, 16)])
        g.close()
    np.testing.assert_allclose(runs[1], runs[0], rtol=1e-12, atol=1e-18)


def test_wrap_caller_owned_nccl_communicator(tmp_path):
    """sylv_comm_wrap_nccl over torch's own NCCL communicator (world size 1): a sharded-path
    context runs on it, and destroying the library's comm leaves torch's usable."""
    import os
    import torch.distributed as dist
    pkg = _pkg()
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29531")
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        t = torch.ones(1, device="cuda")
        dist.all_reduce(t)                                   # creates torch's communicator
        pg = dist.distributed_c10d._get_default_group()
        try:
            ptr = pg._get_backend(torch.device("cuda"))._comm_ptr()
        except Exception as e:                               # pragma: no cover (older torch)
            pytest.skip(f"torch does not expose its ncclComm_t: {e}")
        comm = pkg.wrap_nccl(ptr)
        cfg = inputs.small_config(kind="stencil3d", N=16, r=4, k=2, d_max=20)
        C1, C2 = inputs.make_rhs(cfg)
        g = pkg.from_config(cfg, C1=torch.from_numpy(C1).cuda(), C2=torch.from_numpy(C2).cuda(), comm=comm,
                            row_range=(0, cfg.n))
        g.step(8)
        rr = g.residual(8)[1]
        g.close()
        comm.close()
        ref = pkg.from_config(cfg, C1=torch.from_numpy(C1).cuda(), C2=torch.from_numpy(C2).cuda())
        ref.step(8)
        assert rr == pytest.approx(ref.residual(8)[1], rel=1e-12)
        ref.close()
        dist.all_reduce(t)                                   # torch's communicator still works
        torch.cuda.synchronize()
        assert t.item() == 1.0
    finally:
        dist.destroy_process_group()
