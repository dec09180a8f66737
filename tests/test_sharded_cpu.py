"""The row-sharded decomposition of SURVEY §8(e) on CPU: world size 2 and 3 with gloo.

Each rank holds only its z-slab (3-D stencil) or row range (CSR, c4's decomposition) of every
basis block (rows from the library's own host partition function, sylv_partition), and
emulates in NumPy exactly the exchange steps the sharded CUDA path performs (engine.cu /
comm.cuh):
  * halo: the ghost planes (stencil: N^2 rows; CSR: band = max |col - row| rows) of the
    newest block come from the neighbour ranks (send/recv), and the operator rows of the
    slab are applied to [ghost_lo; Z_loc; ghost_hi];
  * Gram-Schmidt inner products and the Gram of W' are allreduced (sum), the r x r
    normalisation (CholQR) is then identical on every rank;
  * the partial sketch S[:, rows_loc] W_loc uses GLOBAL row indices and is allreduced
    (S is linear in rows), the sketch-space QR is replicated (mode "replicated"), or
    reduce-scattered so each rank keeps s/P rows of Q and w, with the CGS2 coefficient vectors
    and the CholQR Gram allreduced (mode "sharded_sketch": the engine's default for several
    ranks when P divides s);
  * mode "sketched_gs" (f3): the Gram-Schmidt coefficients and the normalisation come
    from the allreduced sketch of the matvec (no inner product over the n rows at all).
The assembled H_und_d, T_d and beta must equal the single-process oracle's (which never
splits rows) to rounding (1e-10), on every rank.  This pins the decomposition itself
(which data crosses ranks, and global hashing) without a GPU.
"""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

from oracle import alg1, operators, sparse_sign  # noqa: E402
from synth import inputs  # noqa: E402

CFGS = {
    "stencil3d": dict(kind="stencil3d", N=12, r=2, k=2, d_max=12),
    # row-sharded CSR (c4's decomposition): halo width = the band max |col - row|
    "csr": dict(kind="csr", n=3001, nnz_off=6, band=200, r=2, k=2, d_max=12),
}
NSTEPS = 8


def _halo_width(cfg, M):
    if cfg.kind == "stencil3d":
        return cfg.N * cfg.N
    if cfg.kind == "stencil2d":
        return cfg.N
    coo = M.tocoo()
    return int(np.abs(coo.col - coo.row).max())


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _allreduce(x):
    t = torch.from_numpy(np.ascontiguousarray(x))
    dist.all_reduce(t)
    return t.numpy()


def _halo(Z, plane, rank, world):
    """Ghost planes of Z (local rows) from the neighbours: (lower ghost, upper ghost)."""
    lo = np.zeros((plane, Z.shape[1]))
    hi = np.zeros((plane, Z.shape[1]))
    ops = []
    send_first = torch.from_numpy(np.ascontiguousarray(Z[:plane]))
    send_last = torch.from_numpy(np.ascontiguousarray(Z[-plane:]))
    recv_lo = torch.zeros(plane, Z.shape[1], dtype=torch.float64)
    recv_hi = torch.zeros(plane, Z.shape[1], dtype=torch.float64)
    if rank > 0:
        ops += [dist.P2POp(dist.isend, send_first, rank - 1), dist.P2POp(dist.irecv, recv_lo, rank - 1)]
    if rank < world - 1:
        ops += [dist.P2POp(dist.isend, send_last, rank + 1), dist.P2POp(dist.irecv, recv_hi, rank + 1)]
    if ops:
        for req in dist.batch_isend_irecv(ops):
            req.wait()
    if rank > 0:
        lo = recv_lo.numpy()
    if rank < world - 1:
        hi = recv_hi.numpy()
    return lo, hi


def _cholqr2_sharded(w):
    """CholQR2 of a row-sharded s x r block: Grams allreduced, each rank keeps its rows."""
    G = _allreduce(w.T @ w)
    t1 = np.linalg.cholesky(G).T
    w1 = np.linalg.solve(t1.T, w.T).T
    G2 = _allreduce(w1.T @ w1)
    t2 = np.linalg.cholesky(G2).T
    return np.linalg.solve(t2.T, w1.T).T, t2 @ t1


class ShardedSequence:
    """One Krylov sequence of Alg. 1 on this rank's slab (lines 1 and 3-9)."""

    def __init__(self, M, C, rows, plane, seed, cfg, rank, world, mode="replicated"):
        b, e = rows
        self.mode = mode
        self.rows, self.plane, self.rank, self.world, self.k, self.r = rows, plane, rank, world, cfg.k, cfg.r
        self.sl = slice(rank * cfg.s // world, (rank + 1) * cfg.s // world)   # this rank's sketch rows
        n = M.shape[0]
        ext = np.arange(max(0, b - plane), min(n, e + plane))
        self.M_loc = M[b:e][:, ext].toarray()                 # slab rows, columns incl. ghost planes
        self.has_lo, self.has_hi = b > 0, e < n
        j = np.arange(b, e)
        self.S_loc = np.zeros((cfg.s, e - b))                 # columns of S for the GLOBAL rows b..e-1
        for t in range(cfg.zeta):
            row, val = sparse_sign.entries(j, t, cfg.s, cfg.zeta, seed)
            self.S_loc[row, np.arange(e - b)] = val
        Cl = C[b:e]
        SC = _allreduce(self.S_loc @ Cl)
        _, self.beta = alg1.qr_pos(SC)
        if mode == "sketched_gs":                             # U_1 = C R(S C)^{-1}: S-orthonormal
            ell = self.beta
        else:
            G = _allreduce(Cl.T @ Cl)
            ell = np.linalg.cholesky(G).T                     # U_1 ell = C (CholQR)
        self.U = {1: np.linalg.solve(ell.T, Cl.T).T}
        if mode == "sharded_sketch":                          # this rank's rows of Q_1
            self.Q, self.T = _cholqr2_sharded(_allreduce(self.S_loc @ self.U[1])[self.sl])
        else:
            self.Q, self.T = alg1.qr_pos(_allreduce(self.S_loc @ self.U[1]))
        self.H = {}
        self.d = 0

    def apply(self, Z):
        lo, hi = _halo(Z, self.plane, self.rank, self.world)
        parts = ([lo] if self.has_lo else []) + [Z] + ([hi] if self.has_hi else [])
        return self.M_loc @ np.concatenate(parts)

    def step(self):
        d = self.d + 1
        W = self.apply(self.U[d])
        window = range(max(1, d - self.k + 1), d + 1)
        if self.mode == "sketched_gs":
            # coefficients from sketches only (one allreduce of the sketch of the matvec)
            SW = _allreduce(self.S_loc @ W)
            SU = {i: _allreduce(self.S_loc @ self.U[i]) for i in window}
            for i in window:
                h = SU[i].T @ SW
                W = W - self.U[i] @ h
                SW = SW - SU[i] @ h
                self.H[(i, d)] = h
            _, hs = alg1.qr_pos(SW)
        else:
            for i in window:
                h = _allreduce(self.U[i].T @ W)
                W = W - self.U[i] @ h
                self.H[(i, d)] = h
            G = _allreduce(W.T @ W)
            hs = np.linalg.cholesky(G).T
        self.H[(d + 1, d)] = hs
        Unew = np.linalg.solve(hs.T, W.T).T
        w = _allreduce(self.S_loc @ Unew)
        if self.mode == "sharded_sketch":
            # reduce-scatter: this rank's rows of the summed sketch; CGS2 over the local rows of Q
            # with the m r coefficients allreduced, CholQR2 with the Gram allreduced
            w = w[self.sl]
            c1 = _allreduce(self.Q.T @ w)
            w = w - self.Q @ c1
            c2 = _allreduce(self.Q.T @ w)
            w = w - self.Q @ c2
            q, tau = _cholqr2_sharded(w)
        else:
            c1 = self.Q.T @ w
            w = w - self.Q @ c1
            c2 = self.Q.T @ w
            w = w - self.Q @ c2
            q, tau = alg1.qr_pos(w)
        m, r = self.T.shape[0], self.r
        T = np.zeros((m + r, m + r))
        T[:m, :m], T[:m, m:], T[m:, m:] = self.T, c1 + c2, tau
        self.T, self.Q = T, np.concatenate([self.Q, q], axis=1)
        self.U[d + 1] = Unew
        self.d = d

    def Hbar(self, d):
        r = self.r
        Hb = np.zeros(((d + 1) * r, d * r))
        for j in range(1, d + 1):
            for i in range(max(1, j - self.k + 1), j + 2):
                Hb[(i - 1) * r:i * r, (j - 1) * r:j * r] = self.H[(i, j)]
        return Hb


def _worker(rank, world, port, q, kind, mode):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2311_16019_b200 as pkg
        cfg = inputs.small_config(**CFGS[kind])
        rows = pkg.partition(cfg, world, rank)               # the library's host partition
        A, Bt, _ = operators.operator_pair(cfg)
        C1, C2 = inputs.make_rhs(cfg)
        U = ShardedSequence(A, C1, rows, _halo_width(cfg, A), cfg.seed_u, cfg, rank, world, mode)
        V = ShardedSequence(Bt, C2, rows, _halo_width(cfg, Bt), cfg.seed_v, cfg, rank, world, mode)
        for _ in range(NSTEPS):
            U.step()
            V.step()
        q.put((rank, rows, U.Hbar(NSTEPS), U.T, U.beta, V.Hbar(NSTEPS), V.T, V.beta))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("kind,world,mode", [("stencil3d", 2, "replicated"), ("stencil3d", 3, "replicated"),
                                             ("csr", 2, "replicated"), ("csr", 3, "replicated"),
                                             ("stencil3d", 2, "sharded_sketch"), ("csr", 4, "sharded_sketch"),
                                             ("stencil3d", 2, "sketched_gs"), ("csr", 3, "sketched_gs")])
def test_sharded_decomposition_matches_oracle(kind, world, mode):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q, kind, mode)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    cfg = inputs.small_config(**CFGS[kind])
    orc = alg1.SylvesterSketchedKrylov.from_config(cfg, sketched_gs=mode == "sketched_gs")
    orc.step(NSTEPS)
    res.sort()
    assert res[0][1][0] == 0 and res[-1][1][1] == cfg.n
    assert all(res[i][1][1] == res[i + 1][1][0] for i in range(world - 1))
    for (_, rows, HU, TU, bU, HV, TV, bV) in res:
        for got, want in ((HU, orc.U.Hbar(NSTEPS)), (TU, orc.U.T), (bU, orc.U.beta),
                          (HV, orc.V.Hbar(NSTEPS)), (TV, orc.V.T), (bV, orc.V.beta)):
            assert np.linalg.norm(got - want) <= 1e-10 * np.linalg.norm(want), rows
