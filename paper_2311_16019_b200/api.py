"""ctypes binding of include/sylv_sketch.h (argument marshalling only).

Every step of the method runs inside libsylvsketch.so (CUDA kernels for sm_100a plus
the host projected solve).  There is no CPU fallback: if the shared library is
missing or no CUDA device is present, construction raises.
"""
from __future__ import annotations

import ctypes as C
import glob
import importlib.util
import os
from typing import Optional, Tuple

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libsylvsketch.so")

STATUS = {0: "OK", 1: "E_INVALID", 2: "E_NOMEM", 3: "E_CUDA", 4: "E_NCCL", 5: "E_BREAKDOWN",
          6: "E_SINGULAR", 7: "E_NOT_CONVERGED", 8: "E_STATE", 9: "E_LOST_INDEP", 10: "E_LAPACK"}
OK, E_BREAKDOWN, E_SINGULAR, E_NOT_CONVERGED, E_LOST_INDEP = 0, 5, 6, 7, 9
OP_STENCIL2D, OP_STENCIL3D, OP_CSR = 1, 2, 3


class SylvError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status


class Operator(C.Structure):
    _fields_ = [("kind", C.c_int32), ("n", C.c_int64), ("grid", C.c_int32 * 3), ("nu", C.c_double),
                ("w", C.c_double * 3), ("row_ptr", C.c_void_p), ("col_idx", C.c_void_p),
                ("val", C.c_void_p), ("nnz", C.c_int64), ("is_transposed", C.c_int32)]


class Config(C.Structure):
    _fields_ = [("r", C.c_int32), ("k", C.c_int32), ("d_max", C.c_int32), ("zeta", C.c_int32),
                ("s", C.c_int64), ("seed_u", C.c_uint64), ("seed_v", C.c_uint64), ("tol", C.c_double),
                ("rank_tol", C.c_double), ("chunk", C.c_int32), ("flags", C.c_int32),
                ("row_begin", C.c_int64), ("row_end", C.c_int64), ("method", C.c_int32),
                ("sketch_kind", C.c_int32), ("srdct_signs_u", C.c_void_p), ("srdct_signs_v", C.c_void_p),
                ("srdct_rows_u", C.c_void_p), ("srdct_rows_v", C.c_void_p)]


METHODS = {"sketched": 0, "truncated": 1, "full": 2, "sketched_gs": 3}   # SYLV_METHOD_* (include/sylv_sketch.h)


class Stats(C.Structure):
    _fields_ = [("launches", C.c_int64), ("steps", C.c_int64), ("ms_pass1", C.c_double),
                ("ms_pass2", C.c_double), ("n_pass1", C.c_int64), ("n_pass2", C.c_int64),
                ("ms_skqr", C.c_double), ("n_skqr", C.c_int64), ("ms_sketch", C.c_double),
                ("n_sketch", C.c_int64), ("host_solve_s", C.c_double),
                ("host_solves", C.c_int64), ("kappa_T_u", C.c_double), ("kappa_T_v", C.c_double),
                ("gpu_solves", C.c_int64), ("gpu_solve_s", C.c_double), ("gpu_solve_fallbacks", C.c_int64),
                ("gpu_approx_checks", C.c_int64)]

    def as_dict(self):
        return {f: getattr(self, f) for f, _ in self._fields_}


_lib = None
SYMBOLS = ["sylv_sketch_init", "sylv_sketch_step", "sylv_sketch_residual", "sylv_sketch_solution",
           "sylv_sketch_solve", "sylv_sketch_apply_sketch", "sylv_sketch_get_small",
           "sylv_sketch_get_block", "sylv_sketch_history", "sylv_sketch_stats",
           "sylv_sketch_reset_stats", "sylv_sketch_last_error", "sylv_sketch_destroy",
           "sylv_set_lapack_path", "sylv_version", "sylv_host_projected", "sylv_host_sylvester",
           "sylv_partition", "sylv_comm_nccl_unique_id", "sylv_comm_create_nccl", "sylv_comm_wrap_nccl",
           "sylv_local_group_create",
           "sylv_local_group_destroy", "sylv_comm_create_local", "sylv_comm_destroy"]


def lapack_path() -> str:
    spec = importlib.util.find_spec("scipy")
    if spec is None or not spec.submodule_search_locations:
        raise SylvError(10, "scipy (bundled OpenBLAS/LAPACK) not found")
    site = os.path.dirname(list(spec.submodule_search_locations)[0])
    hits = sorted(glob.glob(os.path.join(site, "scipy.libs", "libscipy_openblas*.so")))
    if not hits:
        raise SylvError(10, "libscipy_openblas*.so not found next to scipy")
    return hits[0]


def load_library(path: str = LIB_PATH):
    """Load libsylvsketch.so (no fallback: raises if absent).  SYLV_LIB_PATH: a development
    A/B build of the same library (build.build(out=..., extra=[...]))."""
    global _lib
    if _lib is not None:
        return _lib
    path = os.environ.get("SYLV_LIB_PATH", path)
    if not os.path.exists(path):
        raise SylvError(3, f"{path} missing: run `python -m paper_2311_16019_b200.build` "
                           "(or __graft_entry__.build())")
    lib = C.CDLL(path)
    P = C.c_void_p
    lib.sylv_sketch_init.argtypes = [C.POINTER(Operator), C.POINTER(Operator), P, P, C.POINTER(Config), P, P,
                                     C.POINTER(P)]
    lib.sylv_sketch_step.argtypes = [P, C.c_int32, C.POINTER(C.c_int32)]
    lib.sylv_sketch_residual.argtypes = [P, C.c_int32, C.POINTER(C.c_double), C.POINTER(C.c_double)]
    lib.sylv_sketch_solution.argtypes = [P, C.c_int32, P, P, C.c_int64, C.c_int32, C.POINTER(C.c_int32)]
    lib.sylv_sketch_solve.argtypes = [P, C.POINTER(C.c_int32), C.POINTER(C.c_double)]
    lib.sylv_sketch_apply_sketch.argtypes = [P, C.c_int32, P, C.c_int32, P]
    lib.sylv_sketch_get_small.argtypes = [P, C.c_int32, C.c_int32, P, P, P]
    lib.sylv_sketch_get_block.argtypes = [P, C.c_int32, C.c_int32, P]
    lib.sylv_sketch_history.argtypes = [P, C.c_int32, P, P, C.POINTER(C.c_int32)]
    lib.sylv_sketch_stats.argtypes = [P, C.POINTER(Stats)]
    lib.sylv_sketch_reset_stats.argtypes = [P]
    lib.sylv_sketch_reset_stats.restype = None
    lib.sylv_sketch_last_error.argtypes = [P]
    lib.sylv_sketch_last_error.restype = C.c_char_p
    lib.sylv_sketch_destroy.argtypes = [P]
    lib.sylv_sketch_destroy.restype = None
    lib.sylv_set_lapack_path.argtypes = [C.c_char_p]
    lib.sylv_version.restype = C.c_char_p
    lib.sylv_host_projected.argtypes = [C.c_int32, C.c_int32, C.c_int32, P, C.c_int64, P, P]
    lib.sylv_host_projected.restype = C.c_int
    lib.sylv_host_sylvester.argtypes = [C.c_int32, C.c_int32, P, P, P, P]
    lib.sylv_host_sylvester.restype = C.c_int
    lib.sylv_partition.argtypes = [C.c_int32, C.c_int32, C.c_int64, C.c_int32, C.c_int32,
                                   C.POINTER(C.c_int64), C.POINTER(C.c_int64)]
    lib.sylv_partition.restype = C.c_int
    lib.sylv_comm_nccl_unique_id.argtypes = [P]
    lib.sylv_comm_nccl_unique_id.restype = C.c_int
    lib.sylv_comm_create_nccl.argtypes = [C.c_int32, C.c_int32, P, C.POINTER(P)]
    lib.sylv_comm_create_nccl.restype = C.c_int
    lib.sylv_comm_wrap_nccl.argtypes = [P, C.POINTER(P)]
    lib.sylv_comm_wrap_nccl.restype = C.c_int
    lib.sylv_local_group_create.argtypes = [C.c_int32, C.POINTER(P)]
    lib.sylv_local_group_create.restype = C.c_int
    lib.sylv_local_group_destroy.argtypes = [P]
    lib.sylv_local_group_destroy.restype = None
    lib.sylv_comm_create_local.argtypes = [P, C.c_int32, C.POINTER(P)]
    lib.sylv_comm_create_local.restype = C.c_int
    lib.sylv_comm_destroy.argtypes = [P]
    lib.sylv_comm_destroy.restype = None
    for name in SYMBOLS[:11]:
        if name not in ("sylv_sketch_reset_stats",):
            getattr(lib, name).restype = C.c_int
    lib.sylv_set_lapack_path.restype = C.c_int
    st = lib.sylv_set_lapack_path(lapack_path().encode())
    if st != 0:
        raise SylvError(st, "could not load host LAPACK")
    _lib = lib
    return lib


def _ptr(x, shape=None, dtype=np.float64, out=False) -> Tuple[int, object]:
    """(address, keep-alive) for a C-contiguous torch tensor or numpy array.

    The C ABI takes raw double* (int64/int32 for CSR arrays): a wrong dtype or shape would
    make the library read or write past the buffer, so both are checked here.  `shape`
    (rows, cols) is the layout the ABI expects; CUDA tensors must live on the current
    device.  Inputs may be converted (numpy copy); outputs (out=True) never are, since a
    silent copy would receive the result and be dropped."""
    if x is None:
        return 0, None
    if hasattr(x, "data_ptr"):           # torch.Tensor
        import torch
        tdt = {np.float64: torch.float64, np.int64: torch.int64, np.int32: torch.int32}[dtype]
        if x.dtype != tdt:
            raise TypeError(f"tensor must be {tdt}, got {x.dtype}")
        if not x.is_contiguous():
            raise ValueError("tensor must be contiguous")
        if x.is_cuda and x.device.index != torch.cuda.current_device():
            raise ValueError(f"tensor is on {x.device}, the current device is cuda:{torch.cuda.current_device()}")
        if shape is not None and tuple(x.shape) != tuple(shape):
            raise ValueError(f"expected shape {tuple(shape)}, got {tuple(x.shape)}")
        return x.data_ptr(), x
    if out:
        if not isinstance(x, np.ndarray) or x.dtype != dtype or not x.flags.c_contiguous or not x.flags.writeable:
            raise ValueError(f"output must be a writeable C-contiguous {np.dtype(dtype).name} numpy array")
        a = x
    else:
        a = np.ascontiguousarray(x, dtype=dtype)
    if shape is not None and tuple(a.shape) != tuple(shape):
        raise ValueError(f"expected shape {tuple(shape)}, got {tuple(a.shape)}")
    return a.ctypes.data, a


def stencil_operator(kind: str, N: int, w, nu: float = 1.0) -> Operator:
    op = Operator()
    op.kind = OP_STENCIL2D if kind == "stencil2d" else OP_STENCIL3D
    dim = 2 if kind == "stencil2d" else 3
    op.n = N ** dim
    op.grid[0] = N
    op.nu = nu
    for i, v in enumerate(w):
        op.w[i] = float(v)
    return op


def csr_operator(n: int, row_ptr, col_idx, val, is_transposed: bool = False):
    """CSR descriptor (host or device arrays).  For the operator B, is_transposed = True means the
    arrays already hold B^T (no device transpose at init)."""
    op = Operator()
    op.kind = OP_CSR
    op.n = n
    op.is_transposed = 1 if is_transposed else 0
    keep = []
    for name, arr, dt in (("row_ptr", row_ptr, np.int64), ("col_idx", col_idx, np.int32), ("val", val, np.float64)):
        p, k = _ptr(arr, dtype=dt)
        setattr(op, name, p)
        keep.append(k)
    op.nnz = int(len(val) if not hasattr(val, "numel") else val.numel())
    return op, keep


class SylvSketch:
    """One solver context (both Krylov sequences).  Mirrors the C ABI one to one."""

    def __init__(self, A: Operator, B: Operator, C1, C2, *, r: int, k: int, d_max: int, s: int,
                 zeta: int = 8, seed_u: int = 11, seed_v: int = 12, tol: float = 1e-6,
                 rank_tol: float = 1e-12, chunk: int = 0, timing: bool = False, stream=None,
                 keep=None, serial: bool = False, tma: bool = True, comm: "Comm" = None,
                 proj: str = "auto", method: str = "sketched",
                 row_range: Optional[Tuple[int, int]] = None, srdct=None):
        self.lib = load_library()
        self.cfg = Config(r=r, k=k, d_max=d_max, zeta=zeta, s=s, seed_u=seed_u, seed_v=seed_v, tol=tol,
                          rank_tol=rank_tol, chunk=chunk, flags=(1 if timing else 0) | (2 if serial else 0) | (0 if tma else 4)
                          | {"auto": 0, "gpu": 8, "host": 16}[proj],
                          row_begin=row_range[0] if row_range else 0, row_end=row_range[1] if row_range else 0,
                          method=METHODS[method])
        self.method = method
        if srdct is not None:     # ((signs_u, rows_u), (signs_v, rows_v)): the SRDCT sketch
            (su, ru), (sv, rv) = srdct
            self._srdct = [np.ascontiguousarray(a, dtype=t) for a, t in
                           ((su, np.int8), (sv, np.int8), (ru, np.int64), (rv, np.int64))]
            if any(a.shape != (int(A.n),) for a in self._srdct[:2]) or any(a.shape != (s,) for a in self._srdct[2:]):
                raise ValueError("SRDCT: n signs and s rows per sequence")
            self.cfg.sketch_kind = 1
            self.cfg.srdct_signs_u, self.cfg.srdct_signs_v, self.cfg.srdct_rows_u, self.cfg.srdct_rows_v = (
                a.ctypes.data for a in self._srdct)
        self.n, self.r, self.s = int(A.n), r, s     # n: this context's (local) rows, set below
        self._keep = [A, B, keep]
        n_loc = int(row_range[1] - row_range[0]) if row_range else int(A.n)
        p1, k1 = _ptr(C1, shape=(n_loc, r))
        p2, k2 = _ptr(C2, shape=(n_loc, r))
        self._ctx = C.c_void_p()
        st = C.c_void_p(stream) if stream is not None else None
        self._comm = comm
        if comm is not None and row_range is None:
            raise ValueError("a sharded context needs row_range=(begin, end) (see partition())")
        self.n_global = int(A.n)
        if row_range:
            self.n = int(row_range[1] - row_range[0])
        status = self.lib.sylv_sketch_init(C.byref(A), C.byref(B), p1, p2, C.byref(self.cfg),
                                           comm.handle if comm is not None else None, st, C.byref(self._ctx))
        if status != OK:
            msg = self._err()
            self.close()
            raise SylvError(status, msg)

    def last_error(self) -> str:
        return self._err()

    # -- helpers
    def _err(self) -> str:
        return self.lib.sylv_sketch_last_error(self._ctx).decode() if self._ctx else "init failed"

    def _check(self, status: int, allow=()):
        if status != OK and status not in allow:
            raise SylvError(status, self._err())
        return status

    def close(self):
        if getattr(self, "_ctx", None):
            self.lib.sylv_sketch_destroy(self._ctx)
            self._ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- ABI
    def step(self, nsteps: int = 1) -> Tuple[int, int]:
        d = C.c_int32()
        st = self._check(self.lib.sylv_sketch_step(self._ctx, nsteps, C.byref(d)),
                         allow=(E_BREAKDOWN, E_NOT_CONVERGED, E_LOST_INDEP))
        return d.value, st

    def residual(self, d: int) -> Tuple[float, float]:
        rho, rr = C.c_double(), C.c_double()
        self._check(self.lib.sylv_sketch_residual(self._ctx, d, C.byref(rho), C.byref(rr)))
        return rho.value, rr.value

    def solve(self) -> Tuple[int, float, int]:
        ds, rr = C.c_int32(), C.c_double()
        st = self._check(self.lib.sylv_sketch_solve(self._ctx, C.byref(ds), C.byref(rr)), allow=(E_NOT_CONVERGED,))
        return ds.value, rr.value, st

    def solution(self, d: int, max_rank: int, X1=None, X2=None) -> Tuple[object, object, int]:
        if X1 is None:
            X1 = np.zeros((self.n, max_rank))
            X2 = np.zeros((self.n, max_rank))
        p1, _ = _ptr(X1, shape=(self.n, max_rank), out=True)
        p2, _ = _ptr(X2, shape=(self.n, max_rank), out=True)
        rank = C.c_int32()
        self._check(self.lib.sylv_sketch_solution(self._ctx, d, p1, p2, max_rank, max_rank, C.byref(rank)))
        return X1, X2, rank.value

    def apply_sketch(self, which: int, X, out=None):
        r = int(X.shape[1])
        if out is None:
            out = np.zeros((self.s, r))
        px, _ = _ptr(X, shape=(self.n, r))
        po, _ = _ptr(out, shape=(self.s, r), out=True)
        self._check(self.lib.sylv_sketch_apply_sketch(self._ctx, which, px, r, po))
        return out

    def get_small(self, which: int, d: int):
        r, m = self.r, d * self.r
        H = np.zeros((m + r, m))
        T = np.zeros((m + r, m + r))
        beta = np.zeros((r, r))
        self._check(self.lib.sylv_sketch_get_small(self._ctx, which, d, H.ctypes.data, T.ctypes.data,
                                                   beta.ctypes.data))
        return H, T, beta

    def get_block(self, which: int, j: int, out=None):
        if out is None:
            out = np.zeros((self.n, self.r))
        p, _ = _ptr(out, shape=(self.n, self.r), out=True)
        self._check(self.lib.sylv_sketch_get_block(self._ctx, which, j, p))
        return out

    def history(self):
        cnt = C.c_int32()
        self.lib.sylv_sketch_history(self._ctx, 0, None, None, C.byref(cnt))
        n = cnt.value
        d = np.zeros(n, dtype=np.int32)
        rr = np.zeros(n)
        self.lib.sylv_sketch_history(self._ctx, n, d.ctypes.data, rr.ctypes.data, C.byref(cnt))
        return list(zip(d.tolist(), rr.tolist()))

    def stats(self) -> dict:
        s = Stats()
        self._check(self.lib.sylv_sketch_stats(self._ctx, C.byref(s)))
        return s.as_dict()

    def reset_stats(self):
        self.lib.sylv_sketch_reset_stats(self._ctx)


def operators_for(cfg, csr_pair=None):
    """(A, B, keepalive) C-ABI operator descriptors for a synth.Config (B, not B^T)."""
    if cfg.kind.startswith("stencil"):
        return stencil_operator(cfg.kind, cfg.N, cfg.wA), stencil_operator(cfg.kind, cfg.N, cfg.wB), None
    if csr_pair is None:
        from synth.inputs import config_csr
        csr_pair = config_csr(cfg)
    (ra, ca, va), (rb, cb, vb) = csr_pair
    A, ka = csr_operator(cfg.n, ra, ca, va)
    B, kb = csr_operator(cfg.n, rb, cb, vb)
    return A, B, (ka, kb)


def partition(cfg, nranks: int, rank: int) -> Tuple[int, int]:
    """sylv_partition: this rank's global rows [begin, end) of a config (stencil: whole
    planes/lines; CSR: multiples of 32 rows)."""
    lib = load_library()
    kind = {"stencil2d": OP_STENCIL2D, "stencil3d": OP_STENCIL3D, "csr": OP_CSR}.get(cfg.kind)
    if kind is None:
        raise SylvError(1, f"unknown operator kind {cfg.kind}")
    b, e = C.c_int64(), C.c_int64()
    st = lib.sylv_partition(kind, cfg.N if kind != OP_CSR else 1, cfg.n, nranks, rank, C.byref(b), C.byref(e))
    if st != OK:
        raise SylvError(st, f"cannot split {cfg.name} over {nranks} ranks")
    return b.value, e.value


class Comm:
    """A sylv_comm* transport handle (NCCL, or one virtual rank of a LocalGroup)."""

    def __init__(self, handle, keep=None):
        self.handle = handle
        self._keep = keep

    def close(self):
        if getattr(self, "handle", None):
            load_library().sylv_comm_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class LocalGroup:
    """nranks virtual ranks in this process on one GPU (sylv_local_group_create); drive
    rank i's context from its own host thread (the C calls release the GIL)."""

    def __init__(self, nranks: int):
        self.lib = load_library()
        self.nranks = nranks
        self.handle = C.c_void_p()
        st = self.lib.sylv_local_group_create(nranks, C.byref(self.handle))
        if st != OK:
            raise SylvError(st, "sylv_local_group_create")

    def comm(self, rank: int) -> Comm:
        h = C.c_void_p()
        st = self.lib.sylv_comm_create_local(self.handle, rank, C.byref(h))
        if st != OK:
            raise SylvError(st, "sylv_comm_create_local")
        return Comm(h, keep=self)

    def close(self):
        if getattr(self, "handle", None):
            self.lib.sylv_local_group_destroy(self.handle)
            self.handle = None


def nccl_comm(group=None) -> Comm:
    """NCCL transport for the calling rank of a torch.distributed group: rank 0 draws the
    unique id (sylv_comm_nccl_unique_id), torch broadcasts the 128 bytes, every rank joins."""
    import torch
    import torch.distributed as dist
    lib = load_library()
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    uid = (C.c_uint8 * 128)()
    if rank == 0:
        st = lib.sylv_comm_nccl_unique_id(uid)
        if st != OK:
            raise SylvError(st, "sylv_comm_nccl_unique_id (libnccl.so.2 not loadable?)")
    dev = torch.device("cuda", torch.cuda.current_device()) if dist.get_backend(group) == "nccl" else "cpu"
    t = torch.tensor(list(bytes(uid)), dtype=torch.uint8, device=dev)
    dist.broadcast(t, src=0, group=group)
    raw = bytes(t.cpu().tolist())
    uid2 = (C.c_uint8 * 128).from_buffer_copy(raw)
    h = C.c_void_p()
    st = lib.sylv_comm_create_nccl(world, rank, uid2, C.byref(h))
    if st != OK:
        raise SylvError(st, "sylv_comm_create_nccl")
    return Comm(h)


def wrap_nccl(nccl_comm_ptr: int) -> Comm:
    """NCCL transport over a communicator the caller owns (an ncclComm_t address): the library
    splits its channels from it and never destroys it (sylv_comm_wrap_nccl)."""
    lib = load_library()
    h = C.c_void_p()
    st = lib.sylv_comm_wrap_nccl(C.c_void_p(nccl_comm_ptr), C.byref(h))
    if st != OK:
        raise SylvError(st, "sylv_comm_wrap_nccl")
    return Comm(h)


def from_config(cfg, C1=None, C2=None, csr_pair=None, timing=False, stream=None, **kw) -> SylvSketch:
    if C1 is None:
        from synth.inputs import make_rhs
        C1, C2 = make_rhs(cfg)
    A, B, keep = operators_for(cfg, csr_pair)
    if getattr(cfg, "sketch", "sparse_sign") == "srdct" and "srdct" not in kw:
        from synth.inputs import srdct_rows, srdct_signs     # the sketch's random numbers (inputs)
        kw["srdct"] = tuple((srdct_signs(cfg.n, sd), srdct_rows(cfg.n, cfg.s, sd)) for sd in (cfg.seed_u, cfg.seed_v))
    return SylvSketch(A, B, C1, C2, r=cfg.r, k=cfg.k, d_max=cfg.d_max, s=cfg.s, zeta=cfg.zeta,
                      seed_u=cfg.seed_u, seed_v=cfg.seed_v, tol=cfg.tol, timing=timing, stream=stream,
                      keep=keep, **kw)


def host_projected(d: int, r: int, k: int, T: np.ndarray, H: np.ndarray) -> np.ndarray:
    """Host a6 helper (no GPU): M = [T_d|T_H] H_und T_d^{-1}; T col-major (F-order) array."""
    lib = load_library()
    T = np.asfortranarray(T, dtype=np.float64)
    H = np.ascontiguousarray(H, dtype=np.float64)
    M = np.zeros((d * r, d * r), order="F")
    st = lib.sylv_host_projected(d, r, k, T.ctypes.data, T.shape[0], H.ctypes.data, M.ctypes.data)
    if st != OK:
        raise SylvError(st, "sylv_host_projected failed")
    return M


def host_sylvester(MU: np.ndarray, MV: np.ndarray, B: np.ndarray) -> np.ndarray:
    """Host a6 helper (no GPU): Y with MU Y + Y MV^T = E1 B E1^T."""
    lib = load_library()
    m, r = MU.shape[0], B.shape[0]
    a = np.asfortranarray(MU, dtype=np.float64).copy(order="F")
    b = np.asfortranarray(MV, dtype=np.float64).copy(order="F")
    Bc = np.ascontiguousarray(B, dtype=np.float64)
    Y = np.zeros((m, m), order="F")
    st = lib.sylv_host_sylvester(m, r, a.ctypes.data, b.ctypes.data, Bc.ctypes.data, Y.ctypes.data)
    if st != OK:
        raise SylvError(st, "sylv_host_sylvester failed")
    return Y


def version() -> str:
    return load_library().sylv_version().decode()
