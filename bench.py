#!/usr/bin/env python
"""Benchmark: Krylov block steps/s of Alg. 1 (both sequences)
on a BASELINE.json config, through the C ABI of libsylvsketch.so.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config c3] [--impl ours|reference]

One "step" = one block step d -> d+1 of BOTH Krylov sequences: SpMM + k-truncated block
Gram-Schmidt + CholQR normalisation + hashed sparse-sign sketch + sketch-space QR update.
The host projected solve (a6) and the second pass (a7) are timed separately (--ttt).
Prints ONE JSON line (rank 0).  See DESIGN.md §Measurement for every field.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "time-to-rel.residual 1e-6 (s); Krylov block-steps/s; HBM GB/s vs 8 TB/s peak"
UNIT = "block-steps/s"
NOMINAL_HBM_GBS = 8000.0


def _peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def _workload_desc(cfg):
    if cfg.kind.startswith("stencil"):
        dim = cfg.dim
        return (f"{cfg.name}: {dim}-D convection-diffusion {cfg.N}^{dim} (n={cfg.n}), w_A={cfg.wA}, w_B={cfg.wB}, "
                f"r={cfg.r}, k={cfg.k}, s={cfg.s}, zeta={cfg.zeta}, fp64")
    return (f"{cfg.name}: banded random CSR n={cfg.n}, {cfg.csr_nnz_off}+1 nnz/row, band +-{cfg.csr_band}, "
            f"r={cfg.r}, k={cfg.k}, s={cfg.s}, zeta={cfg.zeta}, fp64")


def algorithmic_bytes(cfg, n=None):
    """Per block step (both sequences): stencil B_n = 2*8*n*r*(2k+1);
    CSR B_n = 2*[12 nnz + 4(n+1) + 8 n r (2k+3)].  Per launch: pass 1 reads k blocks,
    pass 2 reads k blocks and writes 1 (stencil; CSR pass 1 also reads A and writes A Z,
    pass 2 reads A Z)."""
    n = cfg.n if n is None else n          # sharded: this rank's rows
    r, k = cfg.r, cfg.k
    blk = 8 * n * r
    if cfg.kind == "csr":
        nnz = n * (cfg.csr_nnz_off + 1)
        mat = 12 * nnz + 4 * (n + 1)
        p1 = mat + blk * (k + 1)          # A, Z_d gathers (counted once), k-1 other window blocks, write AZ
        p2 = blk * (k + 1) + blk          # read AZ + k window blocks, write W'
        return {"pass1": p1, "pass2": p2, "sketch": blk, "step": 2 * (p1 + p2)}
    p1 = blk * k
    p2 = blk * (k + 1)
    # the sketch kernel reads the new block once (8 n r bytes); not part of SURVEY's B_n,
    # which assumes the sketch fused into pass 2
    return {"pass1": p1, "pass2": p2, "sketch": blk, "step": 2 * (p1 + p2)}


class ClockSampler:
    """nvidia-smi clocks / throttle reasons every 200 ms around and during the timed region:
    one looping nvidia-smi process (the profiling recipe's clocks line), started before the
    region — spawning a process per sample stalls kernel launches of short runs — and
    stopped after it."""
    Q = ("timestamp,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0):
        self.index = index
        self.rows = []
        self._p = None
        self.t0 = self.t1 = None

    def region(self, start: bool):
        """Mark the start / end of the timed region (wall clock)."""
        if start:
            self.t0 = time.time()
        else:
            self.t1 = time.time()

    def __enter__(self):
        try:
            self._p = subprocess.Popen(["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                                        "--format=csv,noheader,nounits", "-lms", "200"],
                                       stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            time.sleep(0.5)                       # spawn + first sample before the timed region
        except Exception:
            self._p = None
        return self

    def __exit__(self, *a):
        if self._p is None:
            return
        time.sleep(0.25)                          # one more sample after the region
        self._p.terminate()
        try:
            out, _ = self._p.communicate(timeout=5)
        except Exception:
            self._p.kill()
            out = ""
        for line in (out or "").splitlines():
            if line.strip():
                self.rows.append([x.strip() for x in line.split(",")])

    def summary(self):
        import datetime
        rows = []
        for r in self.rows:
            try:
                ts = datetime.datetime.strptime(r[0], "%Y/%m/%d %H:%M:%S.%f").timestamp()
            except Exception:
                continue
            rows.append((ts, r[1:]))
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        # samples inside the timed region (+-0.2 s); a region shorter than the 200 ms sampling
        # period gets the sample nearest to it
        t0, t1 = self.t0 or rows[0][0], self.t1 or rows[-1][0]
        inside = [v for ts, v in rows if t0 - 0.2 <= ts <= t1 + 0.2]
        if not inside:
            inside = [min(rows, key=lambda tv: min(abs(tv[0] - t0), abs(tv[0] - t1)))[1]]
        sm = [float(r[0]) for r in inside if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in inside if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in inside for i in range(4) if len(r) > 4 + i and r[4 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(inside), "samples_total": len(rows),
                "how": "one looping nvidia-smi (-lms 200) started before and stopped after the timed region"}


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def _golden(name):
    """The oracle's golden record of a config (tests/golden/<cfg>.json, written by
    tools/make_golden.py from oracle/ alone): d*, rank, oracle timings on the build host."""
    p = os.path.join(ROOT, "tests", "golden", f"{name}.json")
    if not os.path.exists(p):
        return None
    with open(p) as f:
        return json.load(f)


def _rank_cap(cfg, d, gold):
    """Column capacity of the solution buffers: above the rank at rank_tol (the oracle's rank
    from the golden, x1.5), so the truncation is decided by rank_tol, not by the buffer."""
    want = int(1.1 * gold["rank"]) + 8 if gold and gold.get("rank") else 256
    return max(1, min(d * cfg.r, want))


def traffic_for(cfg_name, kernel):
    p = os.path.join(ROOT, "profiles", "traffic.json")
    if not os.path.exists(p):
        return None
    with open(p) as f:
        d = json.load(f)
    v = d.get(cfg_name, {}).get(kernel)
    return v


def oracle_steps(cfg, nsteps, budget_s, warmup=0):
    """The CPU oracle as it stands: setup (excluded), then up to `nsteps` block steps
    (stops early once budget_s is exceeded).  Returns (steps, seconds, setup_s)."""
    from oracle import alg1
    from synth import inputs
    t0 = time.perf_counter()
    csr = inputs.config_csr(cfg) if cfg.kind == "csr" else None
    C1, C2 = inputs.make_rhs(cfg)
    orc = alg1.SylvesterSketchedKrylov.from_config(cfg, C1=C1, C2=C2, csr_pair=csr)
    setup = time.perf_counter() - t0
    for _ in range(warmup):
        orc.step(1)
    t0 = time.perf_counter()
    done = 0
    while done < nsteps:
        orc.step(1)
        done += 1
        if time.perf_counter() - t0 > budget_s:
            break
    return done, time.perf_counter() - t0, setup


def run_reference(args, cfg):
    ws, rank, _ = dist_env()
    if rank != 0:
        return 0
    import torch  # noqa: F401  (threads report only)
    cores = os.cpu_count()
    budget = float(os.environ.get("SYLV_REF_BUDGET_S", "150"))
    steps, secs, setup = oracle_steps(cfg, args.steps, budget, warmup=0)
    v = steps / secs
    sample = (f"{steps} oracle block steps (both sequences) of {cfg.name} from d=1 after a {setup:.0f} s oracle setup "
              f"(excluded); stops early after {budget:.0f} s (warm-up steps skipped: the oracle has no caches to warm)")
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": ws, "steps": steps,
            "warmup": 0, "requested_steps": args.steps, "ms_per_step": 1e3 * secs / steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": {"workload": _workload_desc(cfg)},
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": sample},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def _warm_solvers(cfg, stream):
    """Untimed: one small solve through each device projected solver (sign iteration and the
    certified eigendecomposition, SYLV_EIG=2) and the host one, so the time to tolerance does not
    include first-touch costs of the solver libraries (cuSOLVER's Xgeev: ~25 s on a fresh box)."""
    import torch
    import paper_2311_16019_b200 as pkg
    from synth import inputs
    small = inputs.small_config(kind="stencil2d", N=23, r=cfg.r, k=2, d_max=70)
    C1, C2 = inputs.make_rhs(small)
    for eig, proj in (("2", "gpu"), ("1", "gpu"), ("1", "host")):
        old = os.environ.get("SYLV_EIG")
        os.environ["SYLV_EIG"] = eig
        try:
            w = pkg.from_config(small, C1=torch.from_numpy(C1).cuda(), C2=torch.from_numpy(C2).cuda(),
                                stream=stream.cuda_stream, proj=proj)
        finally:
            if old is None:
                os.environ.pop("SYLV_EIG")
            else:
                os.environ["SYLV_EIG"] = old
        w.step(64)
        w.residual(64)
        X = torch.zeros((small.n, 64), dtype=torch.float64, device="cuda")
        w.solution(64, 64, X, X.clone())
        w.close()
    torch.cuda.synchronize()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default=os.environ.get("SYLV_BENCH_CONFIG", "c3"))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-ttt", action="store_true", help="skip the time-to-tolerance solve")
    ap.add_argument("--no-near", action="store_true", help="skip the timed window near d*")
    args = ap.parse_args()

    from synth import inputs
    cfg = inputs.get_config(args.config)
    if args.impl == "reference":
        return run_reference(args, cfg)

    import numpy as np
    import torch
    import paper_2311_16019_b200 as pkg

    ws, rank, local = dist_env()
    if ws > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        torch.cuda.set_device(0)
    dev = torch.device("cuda", torch.cuda.current_device())
    stream = torch.cuda.current_stream()

    assert args.warmup >= 3 or os.environ.get("SYLV_ALLOW_SHORT_WARMUP"), "W >= 3 warm-up steps required"
    if args.warmup + args.steps > cfg.d_max:
        raise SystemExit(f"warmup+steps must be <= d_max={cfg.d_max}")

    # ---- inputs (synthetic, seeded).  N > 1: the config is row-sharded over the ranks
    # (z-slabs / y-lines) through the NCCL transport, strong scaling;
    # SYLV_BENCH_REPLICAS=1 runs independent replicas instead (weak scaling).
    csr = inputs.config_csr(cfg) if cfg.kind == "csr" else None
    C1, C2 = inputs.make_rhs(cfg)
    sharded = ws > 1 and not os.environ.get("SYLV_BENCH_REPLICAS")
    shard_kw = {}
    if sharded:
        comm = pkg.nccl_comm()
        rb, re_ = pkg.partition(cfg, ws, rank)
        C1, C2 = np.ascontiguousarray(C1[rb:re_]), np.ascontiguousarray(C2[rb:re_])
        shard_kw = dict(comm=comm, row_range=(rb, re_))
    C1d = torch.from_numpy(C1).to(dev)
    C2d = torch.from_numpy(C2).to(dev)
    solver = pkg.from_config(cfg, C1=C1d, C2=C2d, csr_pair=csr, timing=True, stream=stream.cuda_stream, **shard_kw)
    # per-kernel attribution run (serial stream, CUDA events around each launch), untimed
    attr = pkg.from_config(cfg, C1=C1d, C2=C2d, csr_pair=csr, timing=True, stream=stream.cuda_stream, serial=True,
                           **shard_kw)
    attr.step(args.warmup)
    attr.reset_stats()
    attr.step(min(args.steps, 10))
    torch.cuda.synchronize()
    attr_stats = attr.stats()
    attr.close()

    def barrier():
        if ws > 1:
            torch.distributed.barrier()

    solver.step(args.warmup)
    torch.cuda.synchronize()
    solver.reset_stats()
    l0 = solver.stats()["launches"]
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        barrier()
        torch.cuda.synchronize()
        clk.region(True)
        e0.record(stream)
        d_done, st = solver.step(args.steps)
        e1.record(stream)
        torch.cuda.synchronize()
        clk.region(False)
        barrier()
    ms = e0.elapsed_time(e1)
    stats = attr_stats
    launches = solver.stats()["launches"] - l0
    if ws > 1:
        t = torch.tensor([ms], device=dev, dtype=torch.float64)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        ms = float(t.item())
    solver.close()
    torch.cuda.empty_cache()

    # whole-job block steps/s: sharded ranks advance ONE problem together (strong scaling);
    # replicas each advance their own copy (weak scaling)
    value = (1 if sharded else ws) * args.steps / (ms * 1e-3)
    ab = algorithmic_bytes(cfg, C1.shape[0])     # per rank (= whole problem unless sharded)
    ab_job = algorithmic_bytes(cfg)
    peak, peak_src = _peaks()
    p2_ms = stats["ms_pass2"] / max(1, stats["n_pass2"])
    p1_ms = stats["ms_pass1"] / max(1, stats["n_pass1"])
    sk_ms = stats["ms_sketch"] / max(1, stats["n_sketch"])
    # dominant kernel = the largest per-launch device time among the hot-path kernels
    # (each launches once per sequence per step); times are CUDA events on the launching
    # stream (serial mode: no overlap inflates them)
    cand = {"pass1": p1_ms, "pass2": p2_ms, "sketch": sk_ms}
    dom = max(cand, key=cand.get)
    dom_ms, dom_bytes = cand[dom], ab[dom]
    achieved = dom_bytes / (dom_ms * 1e-3) / 1e9
    traffic = traffic_for(cfg.name, dom)
    # aggregate over the job's GPUs, against the aggregate peak
    step_gbs = (ab_job["step"] if sharded else ab["step"] * ws) / (ms / args.steps * 1e-3) / 1e9

    # ---- time to tolerance (BASELINE metric's first part): full solve with the canonical
    # check schedule (R9): init from device C + steps + projected solves + search,
    # then the second pass (a7) at the context's rank_tol (no rank cap below the rank)
    ttt = None
    gold = _golden(cfg.name)
    if not args.no_ttt:
        _warm_solvers(cfg, stream)
        barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        s3 = pkg.from_config(cfg, C1=C1d, C2=C2d, csr_pair=csr, stream=stream.cuda_stream, **shard_kw)
        d_star, rr_star, st_star = s3.solve()
        torch.cuda.synchronize()
        el = time.perf_counter() - t0
        st3 = s3.stats()
        sec = None
        if st_star == 0:
            mr = _rank_cap(cfg, d_star, gold)
            X1o = torch.empty((C1.shape[0], mr), dtype=torch.float64, device=dev)
            X2o = torch.empty((C1.shape[0], mr), dtype=torch.float64, device=dev)
            torch.cuda.synchronize()
            t2 = time.perf_counter()
            _, _, rk = s3.solution(d_star, mr, X1o, X2o)
            torch.cuda.synchronize()
            sec = {"seconds": time.perf_counter() - t2, "rank": rk, "max_rank": mr, "rank_tol": 1e-12,
                   "capped": rk >= mr,
                   "what": "sylv_sketch_solution(d*): SVD truncation of Y at rank_tol + replay of d* block steps "
                           "per sequence (pass 2 with stored coefficients) + X accumulation, device outputs"}
            del X1o, X2o
        s3.close()
        torch.cuda.empty_cache()
        if ws > 1:
            t = torch.tensor([el], device=dev, dtype=torch.float64)
            torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
            el = float(t.item())
        ttt = {"seconds": el, "d_star": d_star, "rho_rel": rr_star, "converged": st_star == 0,
               "oracle_d_star": gold.get("d_star") if gold else None,
               "block_steps": st3["steps"], "host_solves": st3["host_solves"], "host_solve_s": st3["host_solve_s"],
               "gpu_solves": st3["gpu_solves"], "gpu_solve_s": st3["gpu_solve_s"], "second_pass": sec,
               "region": "wall clock: context init from device-resident C1, C2 + sylv_sketch_solve (steps, "
                         "canonical check schedule, projected solves: host Bartels-Stewart for d r < 512, device "
                         "sign-function iteration above, search of the last bracket); max over ranks"}

    # ---- steps near d* (the regime that decides time to tolerance: m = d r sketch-space
    # columns, the CGS2 sweeps of Q grow with d): a second timed window d* - 30 .. d* - 10
    near = None
    dref = (ttt or {}).get("d_star") or (gold or {}).get("d_star")
    if not args.no_near and dref and dref - 30 > args.warmup:
        d0, nn = dref - 30, 20
        s4 = pkg.from_config(cfg, C1=C1d, C2=C2d, csr_pair=csr, timing=True, stream=stream.cuda_stream, **shard_kw)
        s4.step(d0)
        torch.cuda.synchronize()
        barrier()
        e0.record(stream)
        s4.step(nn)
        e1.record(stream)
        torch.cuda.synchronize()
        ms_n = e0.elapsed_time(e1)
        s4.close()
        if ws > 1:
            t = torch.tensor([ms_n], device=dev, dtype=torch.float64)
            torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
            ms_n = float(t.item())
        # per-kernel split near d* (serial attribution context, CUDA events per launch)
        s5 = pkg.from_config(cfg, C1=C1d, C2=C2d, csr_pair=csr, timing=True, stream=stream.cuda_stream, serial=True,
                             **shard_kw)
        s5.step(d0)
        s5.reset_stats()
        s5.step(10)
        torch.cuda.synchronize()
        a5 = s5.stats()
        s5.close()
        torch.cuda.empty_cache()
        m_mid = (d0 + 5) * cfg.r
        q_bytes = 8 * cfg.s * m_mid                     # one sweep of Q (s x m), per sequence
        skqr_ms = a5["ms_skqr"] / max(1, a5["n_skqr"])
        sk_ms_n = a5["ms_sketch"] / max(1, a5["n_sketch"])
        qr_ms = max(1e-6, skqr_ms - sk_ms_n)           # the QR update alone (the skqr events include the sketch)
        step_b = (ab_job["step"] if sharded else ab["step"] * ws)
        near = {"d_range": [d0 + 1, d0 + nn], "value": (1 if sharded else ws) * nn / (ms_n * 1e-3),
                "unit": UNIT, "ms_per_step": ms_n / nn,
                "step_roofline_frac": step_b / (ms_n / nn * 1e-3) / 1e9 / (peak * ws),
                "kernels_ms": {"pass1": a5["ms_pass1"] / max(1, a5["n_pass1"]),
                               "pass2": a5["ms_pass2"] / max(1, a5["n_pass2"]),
                               "sketch": a5["ms_sketch"] / max(1, a5["n_sketch"]), "skqr": skqr_ms},
                "skqr": {"m": m_mid, "Q_sweeps": 4, "bytes_per_launch": 4 * q_bytes, "ms": qr_ms,
                         "GBps": 4 * q_bytes / (qr_ms * 1e-3) / 1e9,
                         "frac": 4 * q_bytes / (qr_ms * 1e-3) / 1e9 / peak,
                         "what": "sketch-space QR update (a5) alone: block CGS2 = 4 sweeps of Q (Q^T w, Q c "
                                 "twice) + CholQR2 + T column, per sequence (skqr events minus the sketch)"}}

    # ---- end to end through the C ABI with HOST buffers: init from pinned host C1, C2
    # (H2D inside), sylv_sketch_solve to tolerance, and the solution X1, X2 (rank_tol) into
    # pinned host buffers (D2H inside) — the calls a user makes, wall clock, max over ranks
    e2e = None
    if not args.no_e2e:
        C1h = torch.from_numpy(C1).pin_memory()
        C2h = torch.from_numpy(C2).pin_memory()
        mr = _rank_cap(cfg, (ttt or {}).get("d_star") or cfg.d_max, gold)
        X1h = torch.empty((C1.shape[0], mr), dtype=torch.float64).pin_memory()
        X2h = torch.empty((C1.shape[0], mr), dtype=torch.float64).pin_memory()
        barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        s2 = pkg.from_config(cfg, C1=C1h, C2=C2h, csr_pair=csr, stream=stream.cuda_stream, **shard_kw)
        d_e, rr_e, st_e = s2.solve()
        rk = 0
        if st_e == 0:
            _, _, rk = s2.solution(d_e, mr, X1h.numpy(), X2h.numpy())
        torch.cuda.synchronize()
        el = time.perf_counter() - t0
        nst = s2.stats()["steps"]
        s2.close()
        if ws > 1:
            t = torch.tensor([el], device=dev, dtype=torch.float64)
            torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
            el = float(t.item())
        mirror = 2 * 8 * ((cfg.k + 1) * cfg.r ** 2 + cfg.r * ((nst // 2 + 1) * cfg.r + cfg.r))
        e2e = {"value": (1 if sharded else ws) * nst / el, "unit": UNIT, "seconds": el, "d_star": d_e,
               "rho_rel": rr_e, "rank": rk, "max_rank": mr,
               "h2d_bytes_per_step": int(2 * 8 * C1.shape[0] * cfg.r * (1 if sharded else ws) / max(1, nst)),
               "d2h_bytes_per_step": int(mirror + 2 * 8 * C1.shape[0] * mr * (1 if sharded else ws) / max(1, nst)),
               "region": "init(pinned host C1, C2: H2D) + sylv_sketch_solve to rho_rel < tol (all block steps, "
                         "projected solves, search) + sylv_sketch_solution(d*) at rank_tol into pinned host X1, X2 "
                         "(D2H); value = block steps run / wall clock, max over ranks"}
        del X1h, X2h

    cpu = None
    if rank == 0 and not args.no_cpu_baseline:
        budget = float(os.environ.get("SYLV_CPU_BUDGET_S", "30"))
        steps_o, secs_o, setup_o = oracle_steps(cfg, 50, budget)
        cpu = {"value": steps_o / secs_o, "unit": UNIT, "cores": os.cpu_count(), "kind": "oracle",
               "sample": f"{steps_o} oracle block steps (both sequences) of {cfg.name} from d=1, "
                         f"after {setup_o:.0f} s oracle setup (excluded); ~{budget:.0f} s budget"}
        if gold and gold.get("oracle_time_to_tol_s"):
            # the oracle's whole run to tolerance (setup + steps + its schedule of Bartels-Stewart
            # solves + search), measured once by tools/make_golden.py on the build container
            cpu["time_to_tolerance"] = {
                "seconds": gold["oracle_time_to_tol_s"], "d_star": gold.get("d_star"),
                "cores": gold.get("host", {}).get("cores"), "solve_s": gold.get("solve_wall_s"),
                "second_pass_s": gold.get("second_pass_s"),
                "where": "build container (tests/golden, tools/make_golden.py), not this box",
                "extrapolated_on_this_box_s": (gold.get("steps_done", gold["d_star"]) / (steps_o / secs_o)
                                               + sum(h.get("solve_s", 0.0) for h in gold.get("history", []))
                                               if gold.get("d_star") else None),
                "extrapolation": "this box's oracle step rate x the golden's steps + the golden's "
                                 "projected-solve seconds (solves not re-timed here)"}

    clk_sum = clk.summary()
    l2_peak = 6300 * (clk_sum.get("sm_mhz") or 1965.0) * 1e6 / 1e9   # GB/s
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
            "scaling": "strong" if sharded else "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": _workload_desc(cfg), "d_range": [args.warmup + 1, args.warmup + args.steps],
                       "parallelism": ((f"row-sharded z-slabs x{ws} (NCCL halo + allreduce)" if cfg.kind.startswith("stencil")
                                        else f"row-sharded 32-row-group ranges x{ws} (NCCL band halo + allreduce)") if sharded
                                       else "replicas" if ws > 1 else "single GPU"),
                       "l2": "inputs larger than L2 (window of k+1 blocks per sequence >> 126 MB)"
                       if 8 * cfg.n * cfg.r * (cfg.k + 1) > 126e6 else "working set may be L2-resident"},
            "roofline": {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic, "peak_source": peak_src,
                         "bytes_per_launch": dom_bytes, "avg_launch_ms": dom_ms,
                         "kernels": {k: {"ms": v, "GBps": ab[k] / (v * 1e-3) / 1e9,
                                         "frac": ab[k] / (v * 1e-3) / 1e9 / peak} for k, v in cand.items()},
                         "skqr_ms": stats["ms_skqr"] / max(1, stats["n_skqr"]),
                         "sketch_l2": {"bytes_per_launch": cfg.zeta * ab["sketch"],
                                       "GBps": cfg.zeta * ab["sketch"] / (sk_ms * 1e-3) / 1e9,
                                       "peak": l2_peak, "frac": cfg.zeta * ab["sketch"] / (sk_ms * 1e-3) / 1e9 / l2_peak,
                                       "peak_source": "LTS throughput cap ~6300 B/cycle full chip (B300_MICROARCH.md, "
                                                      "measured on B300; same L2 design) x median SM clock under load",
                                       "what": "pull sketch (sketch_pull.cuh): every element of the new block "
                                               "is read zeta times from L2 (once per bucket); bound by L2->SM "
                                               "bandwidth, not HBM (ncu lts__throughput, profiles/)"},
                         "note": ("sketch: hashed sparse-sign gather, bounded by L2 bandwidth (zeta reads "
                                  "per element), not by HBM" if dom == "sketch" else "")},
            "step_roofline": {"bytes_per_step": ab_job["step"] if sharded else ab["step"] * ws, "GBps": step_gbs,
                              "frac": step_gbs / (peak * ws), "frac_of_8TBps": step_gbs / (NOMINAL_HBM_GBS * ws),
                              "what": "SURVEY §8(d) B_n per block step (both sequences) / device step time"},
            "time_to_tolerance": ttt, "near_dstar": near,
            "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches,
            "clocks": clk_sum,
        }
        print(json.dumps(line), flush=True)
    if ws > 1:
        torch.distributed.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
