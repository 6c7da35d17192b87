#!/usr/bin/env python
"""Benchmark: trajectory problems solved per second at a fixed number of AM
sweeps (BASELINE.json metric), on 1..8 B200s, plus the FP64-pipe roofline.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config c1] [--impl ours|reference]

A step is one pass of the hot path over one goal batch: solve (fixed sweeps,
tol=0 as the reference's bench-kernels uses) + fused scoring/argmin.
* value: device-resident inputs, CUDA events on the launching stream around
  each step, L2 flushed between steps (256 MiB write), max over ranks.
* e2e:   the public API from pinned host buffers (planner.plan_batch ->
  bmpc_plan_host: H2D, solve, score, D2H inside the timed region).
* roofline: algorithmic fp64 work of the persistent AM kernel
  (W(n,m,nb) slots per instance per sweep; 2 flops per
  slot) / its CUDA-event duration, against the DFMA peak measured live.
Multi-GPU (torchrun): --scaling weak (default; each rank a whole config: its
own block of l goal columns of one shared scene, or its own scenes) or strong
(the BASELINE config split over the ranks as dist.plan_sharded does); the
shards' results are all-gathered inside the timed step (the only collective),
and e2e runs dist.plan_sharded.
--impl reference: the reference's own CPU path -- its batchmpc package (build-time
copy, oracle/_ref/pkg) with its compiled Cython kernels, BatchSolver.solve +
planner scoring -- on all host cores, one BLAS thread per process.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "trajectory problems solved/sec (fixed AM iters)"


def work_slots(n: int, m: int, nb: int) -> int:
    """Algorithmic fp64-pipe slots per instance per AM sweep."""
    return 33 * m * n + 97 * n + 21 * n * nb + 3 * nb * nb + 24 * nb


# ---------------------------------------------------------------- clocks ----
class ClockSampler:
    """SM clock + throttle reasons sampled through NVML every ~2 ms while the
    timed region runs (nvidia-smi's own query path is too slow for a
    millisecond-scale step); falls back to nvidia-smi when NVML is missing."""

    REASONS = {  # NVML clocks-event-reason bits
        "hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
        "sw_power_cap": 0x4,
    }

    def __init__(self, index: int, period_ms: float = 2.0):
        self.index, self.period, self.rows, self._stop = index, period_ms, [], threading.Event()
        self.t = None
        self.max_mhz = None

    def _run(self):
        try:
            import pynvml as N

            N.nvmlInit()
            h = N.nvmlDeviceGetHandleByIndex(self.index)
            self.max_mhz = N.nvmlDeviceGetMaxClockInfo(h, N.NVML_CLOCK_SM)
            get_reasons = getattr(N, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
                N.nvmlDeviceGetCurrentClocksThrottleReasons
            while not self._stop.is_set():
                self.rows.append((N.nvmlDeviceGetClockInfo(h, N.NVML_CLOCK_SM), int(get_reasons(h))))
                self._stop.wait(self.period / 1000.0)
            N.nvmlShutdown()
        except Exception:
            q = "clocks.sm,clocks.max.sm"
            while not self._stop.is_set():
                r = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                    "--format=csv,noheader,nounits"], capture_output=True, text=True)
                if r.returncode == 0 and r.stdout.strip():
                    sm, mx = (float(s) for s in r.stdout.strip().split(","))
                    self.max_mhz = mx
                    self.rows.append((sm, 0))
                self._stop.wait(0.1)

    def __enter__(self):
        self.t = threading.Thread(target=self._run, daemon=True)
        self.t.start()
        time.sleep(0.05)
        return self

    def __exit__(self, *exc):
        self._stop.set()
        self.t.join(timeout=10)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["no samples"]}
        reasons = sorted({name for _, bits in self.rows for name, bit in self.REASONS.items() if bits & bit})
        return {"sm_mhz": statistics.median(r[0] for r in self.rows), "sm_max_mhz": self.max_mhz,
                "reasons": reasons, "samples": len(self.rows), "source": "nvml"}


def _coll_device(dev):
    """Device of the bench's scalar collectives: the GPU under NCCL, host under gloo."""
    import torch.distributed as dist

    return dev if dist.get_backend() == "nccl" else "cpu"


# ------------------------------------------------------------- workloads ----
def make_step_workload(cfg_name: str, world: int, rank: int, scaling: str = "weak"):
    """(config, this rank's SceneBatch, global column offset, the full job).

    weak: every rank a whole config's worth -- one scene of world*l goals with
    rank owning a contiguous block of l columns, or its own set of scenes;
    strong: the BASELINE config itself split over the ranks -- contiguous goal
    columns of its one scene (c1/c2) or contiguous scene blocks (c3/c4),
    exactly as dist.plan_sharded partitions it."""
    from paper_2109_10392_b200.dist import shard_range
    from paper_2109_10392_b200.scenes import CONFIGS, make_workload

    cfg = CONFIGS[cfg_name]
    if scaling == "strong":
        full = make_workload(cfg_name)
        if cfg.scenes == 1:
            lo, hi = shard_range(cfg.l, rank, world)
            return cfg, full.columns(lo, hi), lo, full
        lo, hi = shard_range(cfg.scenes, rank, world)
        return cfg, full.scenes(lo, hi), 0, full
    if cfg.scenes == 1:
        # one scene, world * l goals; rank owns a contiguous block of l columns
        full = make_workload(cfg_name, l=cfg.l * world)
        return cfg, full.columns(rank * cfg.l, (rank + 1) * cfg.l), rank * cfg.l, full
    W = make_workload(cfg_name, seed0=rank * cfg.scenes)
    return cfg, W, 0, None


# ------------------------------------------------------------ CPU baseline ----
# The reference's own CPU path: its batchmpc package (build-time copy in
# oracle/_ref/pkg, with its Cython kernels compiled from /root/reference) running
# BatchSolver.solve(tol=0) + its planner scoring (sample_plan / filter_candidates
# / rank) over disjoint goal blocks of one scene, one process per host core, one
# BLAS thread each.  Each worker builds the scene and the
# solver (KKT factorisation) once, outside the timed region.  When the package
# copy is absent the oracle's restatement (oracle/am_oracle.py + its C kernels)
# stands in.
REF_PKG = ROOT / "oracle" / "_ref" / "pkg"


def _cpu_kind() -> str:
    if (REF_PKG / "batchmpc" / "solver.py").exists() and any((REF_PKG / "batchmpc" / "kernels").glob("_speedups*.so")):
        return "refpkg"
    return "c"


def _cpu_sample_text(kind: str) -> str:
    return ("the reference's own batchmpc.BatchSolver.solve + planner scoring (oracle/_ref/pkg: its sources, its "
            "Cython kernels compiled from /root/reference)" if kind == "refpkg"
            else "oracle/am_oracle.py (solver.py restated op for op) + am_oracle.c kernels")


_W = {}


def _cpu_init(cfg_name, goals, kind):
    from threadpoolctl import threadpool_limits

    from paper_2109_10392_b200.scenes import CONFIGS, make_workload

    cfg = CONFIGS[cfg_name]
    W = make_workload(cfg_name, l=goals, scenes=1)
    _W.update(cfg=cfg, W=W, kind=kind)
    if kind == "refpkg":
        sys.path.insert(0, str(REF_PKG))
        import batchmpc as B
        from batchmpc import planner as RP
        from batchmpc.solver import BatchSolver, ProblemBatch

        grid = B.build_time_grid(0.0, cfg.t_f, cfg.n)
        basis = B.build_basis(grid, cfg.degree)
        _W.update(solver=BatchSolver(basis, B.build_constant_matrices(basis, cfg.m), 1.0), PB=ProblemBatch,
                  RP=RP)
    else:
        sys.path.insert(0, str(ROOT / "oracle"))
        import am_oracle as O

        _W["solver"] = O.OracleSolver(cfg.n, cfg.t_f, cfg.degree, cfg.m)
    # after every BLAS is loaded (numpy's and scipy's own OpenBLAS), kept for the
    # worker's lifetime: one thread per process
    _W["limits"] = threadpool_limits(1)


def _cpu_job(args):
    lo, hi, iters = args
    W, solver = _W["W"], _W["solver"]
    t = time.perf_counter()
    if _W["kind"] == "refpkg":
        RP = _W["RP"]
        batch = _W["PB"](l=hi - lo, xi_x=W.xi_x[0], xi_y=W.xi_y[0], a=W.a, b=W.b, v_min=W.v_min,
                         v_max=W.v_max, a_max=W.a_max, b_xy=np.ascontiguousarray(W.b_xy[:, lo:hi]),
                         b_psi=np.ascontiguousarray(W.b_psi[:, lo:hi]))
        st, info = solver.solve(batch, max_iter=iters, tol=0.0)
        bs = solver.basis
        xd, yd = bs.Pdot @ st.c_x, bs.Pdot @ st.c_y
        plan = RP.RankedPlan(goals=[None] * batch.l, x=bs.P @ st.c_x, y=bs.P @ st.c_y, psi=bs.P @ st.c_psi,
                             psidot=bs.Pdot @ st.c_psi, v=np.sqrt(xd ** 2 + yd ** 2),
                             xddot=bs.Pddot @ st.c_x, yddot=bs.Pddot @ st.c_y,
                             residuals=info.residual_history[-1])
        RP.filter_candidates(plan, batch, RP.FilterLimits())
        RP.rank(plan, RP.MetaCostSpec("cruise", v_cruise=20.0))
        best = plan.best_index
    else:
        r = solver.solve(W.xi_x[0], W.xi_y[0], W.b_xy[:, lo:hi], W.b_psi[:, lo:hi], W.a, W.b, W.v_min,
                         W.v_max, W.a_max, iters, kernel="c")
        best = solver.score(r, W.xi_x[0], W.xi_y[0], W.a, W.b, kind="cruise", v_cruise=20.0)["best_index"]
    return time.perf_counter() - t, hi - lo, best


def cpu_reference_rate(cfg_name: str, goals: int, iters: int, steps: int, warmup: int):
    """Problems/s of the reference CPU path on `goals` goal columns of scene 0
    split over every host core: mean over `steps` timed passes (wall clock
    around the pool map) after `warmup` passes.  Returns (rate, per-step
    seconds, processes, kind)."""
    import multiprocessing as mp

    kind = _cpu_kind()
    procs = min(os.cpu_count() or 1, goals)
    per = int(math.ceil(goals / procs))
    jobs = [(i * per, min(goals, (i + 1) * per), iters) for i in range(procs) if i * per < goals]
    times = []
    for v in ("OPENBLAS_NUM_THREADS", "OMP_NUM_THREADS", "MKL_NUM_THREADS"):
        os.environ[v] = "1"  # inherited by the spawned workers
    with mp.get_context("spawn").Pool(len(jobs), initializer=_cpu_init, initargs=(cfg_name, goals, kind)) as pool:
        pool.map(_cpu_job, [(0, 1, 1)] * len(jobs))  # imports, first-touch
        for _ in range(warmup):
            pool.map(_cpu_job, jobs)
        for _ in range(steps):
            t0 = time.perf_counter()
            pool.map(_cpu_job, jobs)
            times.append(time.perf_counter() - t0)
    return goals * len(times) / sum(times), times, len(jobs), kind


# ---------------------------------------------------------------- our arm ----
def run_ours(args, rank, world, local_rank):
    import ctypes

    import torch

    from paper_2109_10392_b200 import _native as nat
    from paper_2109_10392_b200 import device as D
    from paper_2109_10392_b200 import make_solver
    from paper_2109_10392_b200.planner import FilterLimits, MetaCostSpec, _spec_struct, plan_batch

    local_rank = local_rank % max(1, torch.cuda.device_count())  # see main(): gloo smoke test
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    cfg, W, offset, full = make_step_workload(args.config, world, rank, args.scaling)
    iters = args.iters or cfg.iters
    solver = make_solver(W.n, W.t_f, W.degree, W.m)
    ctx = solver._context()
    lib = nat.load()
    L = W.L
    nb, n = solver.basis.n_b, solver.basis.grid.n
    spec = MetaCostSpec("cruise", v_cruise=20.0)
    limits = FilterLimits()
    sspec = _spec_struct(spec, limits)
    stream = torch.cuda.current_stream()
    sp = ctypes.c_void_p(stream.cuda_stream)

    prob = D.DeviceProblem.from_host(n, W.xi_x, W.xi_y, W.b_xy, W.b_psi, W.l, W.a, W.b, W.v_min,
                                     W.v_max, W.a_max, device=dev)
    pstruct = prob.c_struct()
    sol = D.alloc_solution(nb, n, L, iters, False, dev)
    sc = D.alloc_score(L, prob.S, dev)
    prec = 1 if args.precision == "fp32" else 0
    opts = nat.SolveOpts(max_iter=iters, tol=0.0, precision=prec)
    # the device API without host synchronisation: the early-stop decision stays
    # on the device and {iterations, converged} land in status_dev
    status_dev = torch.zeros(2, dtype=torch.int32, device=dev)
    opts_async = nat.SolveOpts(max_iter=iters, tol=0.0, precision=prec, status_dev=status_dev.data_ptr())
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    # pack_xi, [obstacle_boxes when culling: m >= 24], am_solve (+ fused scoring),
    # early_stop, am_solve (early-stop re-run: exits at once when there is none), argmin
    launches_per_step = 5 + (1 if W.m >= int(os.environ.get("BMPC_CULL_MIN_M", "24")) else 0)

    # N > 1: the step ends with the shards' result exchange (dist.plan_sharded's
    # collective, here on device tensors so nothing waits on the host): one
    # scene -> (cost, global index, n_feasible) of each rank's feasible winner;
    # scenes -> every scene's (best, argmin_all, argmin_hc, n_feasible) row.
    # The {iterations, converged} status rides along (the cross-shard early-stop
    # rule: at tol = 0 no rank converges, checked after the timed loop).
    gathered = None
    if world > 1:
        import torch.distributed as dist

        cdev = _coll_device(dev)
        rec_len = 5 if W.S == 1 else 4 * W.S + 2
        gathered = torch.empty(world, rec_len, dtype=torch.float64, device=cdev)

    def exchange():
        if W.S == 1:
            b = sc.best_index[0]
            bc = sc.meta_cost[b.clamp(min=0)]
            rec = torch.stack([torch.where(b >= 0, bc, torch.full_like(bc, float("inf"))),
                               torch.where(b >= 0, (b + offset).double(), torch.full_like(bc, -1.0)),
                               sc.n_feasible[0].double(), status_dev[0].double(), status_dev[1].double()])
        else:
            rec = torch.cat([torch.stack([sc.best_index, sc.argmin_all, sc.argmin_hc, sc.n_feasible]).double().ravel(),
                             status_dev.double()])
        if gathered.device.type == "cuda":
            dist.all_gather_into_tensor(gathered, rec)
        else:
            dist.all_gather(list(gathered.unbind(0)), rec.cpu())

    def step():
        # the residual history is not requested (plan_batch does not return it)
        out = D.solution_struct(sol)
        out.history = None
        nat.check(lib.bmpc_plan(ctx, ctypes.byref(pstruct), ctypes.byref(opts_async), ctypes.byref(out),
                                ctypes.byref(sspec), ctypes.byref(D.score_struct(sc)), sp))
        if world > 1:
            exchange()
        return out

    def kernel_only():
        out = D.solution_struct(sol)
        out.history = None  # as in the step
        nat.check(lib.bmpc_sweeps(ctx, ctypes.byref(pstruct), ctypes.byref(opts), iters, 0, 0, None,
                                  0, ctypes.byref(out), sp))

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    with ClockSampler(local_rank) as clk:
        torch.cuda.synchronize()
        if world > 1:
            torch.distributed.barrier()
        for i in range(args.steps):
            flush.fill_(float(i))
            ev[i][0].record(stream)
            step()
            ev[i][1].record(stream)
        torch.cuda.synchronize()
        if world > 1:
            torch.distributed.barrier()
    step_ms = [a.elapsed_time(b) for a, b in ev]
    t_local = sum(step_ms)
    best_global = None
    total_L = L
    if world > 1:
        from paper_2109_10392_b200.dist import merge_winners

        g = gathered.cpu().numpy()
        assert (g[:, -1] == 0).all(), "a shard converged at tol = 0: the step would need the re-run"
        if W.S == 1:
            best_global, _ = merge_winners(g[:, :3])
        tt = torch.tensor([t_local, float(L)], dtype=torch.float64, device=_coll_device(dev))
        tl = [torch.empty_like(tt) for _ in range(world)]
        torch.distributed.all_gather(tl, tt)
        t_max = max(float(x[0]) for x in tl)
        total_L = int(sum(float(x[1]) for x in tl))
    else:
        t_max = t_local
    total_problems = total_L * args.steps
    value = total_problems / (t_max / 1e3)

    # roofline: the persistent AM kernel alone
    kk = []
    for i in range(max(3, args.steps)):
        flush.fill_(float(i))
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        kernel_only()
        b.record(stream)
        torch.cuda.synchronize()
        kk.append(a.elapsed_time(b))
    k_ms = statistics.median(kk)
    flops = 2.0 * work_slots(n, W.m, nb) * L * iters
    peak = D.peak_fp64_tflops(5)
    achieved = flops / (k_ms * 1e-3) / 1e12

    # e2e through the public API from host buffers
    pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory().numpy()  # noqa: E731

    class _H:
        pass

    H = _H()
    H.xi_x, H.xi_y, H.b_xy, H.b_psi = pin(W.xi_x), pin(W.xi_y), pin(W.b_xy), pin(W.b_psi)
    H.l, H.S, H.a, H.b, H.v_min, H.v_max, H.a_max = W.l, W.S, W.a, W.b, W.v_min, W.v_max, W.a_max
    job = None
    if world > 1:
        from paper_2109_10392_b200.dist import plan_sharded

        # the whole job every rank passes to plan_sharded (weak c3/c4: the
        # ranks' consecutive seed blocks are one stacked batch)
        from paper_2109_10392_b200.scenes import make_workload

        job = full if full is not None else make_workload(args.config, scenes=cfg.scenes * world)

    def e2e_call(src):
        if job is not None:
            return plan_sharded(solver, job, max_iter=iters, tol=0.0, spec=spec, limits=limits,
                                precision=args.precision)
        return plan_batch(solver, src, max_iter=iters, tol=0.0, spec=spec, limits=limits,
                          precision=args.precision)

    def timed_e2e(src, steps):
        r = None
        for _ in range(args.warmup):  # as the timed loop: the previous result stays alive
            r = e2e_call(src)
        ms = []
        for i in range(steps):
            flush.fill_(float(i))
            torch.cuda.synchronize()
            if world > 1:
                torch.distributed.barrier()
            t0 = time.perf_counter()
            r = e2e_call(src)
            ms.append((time.perf_counter() - t0) * 1e3)
        return ms, r

    e2e_ms, res = timed_e2e(H, args.steps)
    best_e2e = res.best_index[0]
    e2e_local = sum(e2e_ms)
    if world > 1:
        tt = torch.tensor([e2e_local], dtype=torch.float64, device=_coll_device(dev))
        torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
        e2e_local = float(tt.item())
    e2e_value = total_problems / (e2e_local / 1e3)
    h2d = sum(a.nbytes for a in (H.xi_x, H.xi_y, H.b_xy, H.b_psi))
    d2h = 3 * nb * L * 8 + 3 * L * 8 + 3 * L * 8 + L + 4 * W.S * 8
    # the same call from ordinary (pageable) numpy arrays, as the reference API
    # passes them, and BatchSolver.solve end to end (reference-shaped: host
    # arrays in, AmState + SolveInfo out)
    extra = {}
    if world == 1:
        pg_ms, _ = timed_e2e(W, args.steps)
        extra["e2e_pageable"] = {"value": L * args.steps / (sum(pg_ms) / 1e3), "unit": "problems/s",
                                 "ms_per_step": sum(pg_ms) / args.steps,
                                 "path": "plan_batch from pageable numpy inputs (staged copies in)"}
        from paper_2109_10392_b200.solver import ProblemBatch

        src = (ProblemBatch(l=W.l, xi_x=W.xi_x[0], xi_y=W.xi_y[0], a=W.a, b=W.b, v_min=W.v_min,
                            v_max=W.v_max, a_max=W.a_max, b_xy=W.b_xy, b_psi=W.b_psi)
               if W.S == 1 else W)
        sv_ms = []
        for i in range(args.warmup + min(args.steps, 5)):
            flush.fill_(float(i))
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            st, info = solver.solve(src, max_iter=iters, tol=0.0)
            _ = (st.c_x, info.residual_history[-1])
            if i >= args.warmup:
                sv_ms.append((time.perf_counter() - t0) * 1e3)
        extra["e2e_solve"] = {"value": L * len(sv_ms) / (sum(sv_ms) / 1e3), "unit": "problems/s",
                              "ms_per_step": sum(sv_ms) / len(sv_ms),
                              "path": "BatchSolver.solve(batch, max_iter, tol=0) from pageable numpy: "
                                      "coefficients, multipliers and the final residuals on the host; "
                                      "v / alpha / d / alpha_a / d_a left on the device until read; "
                                      "no scoring"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        goals = min(cfg.l, 1024)  # bounded sample: scene 0, at most 1024 goals of this config
        rate, times, used, kind = cpu_reference_rate(args.config, goals, iters, steps=3, warmup=1)
        cpu = {"value": rate, "unit": "problems/s", "cores": used,
               "kind": "reference" if kind == "refpkg" else "port",
               "sample": f"{args.config} scene 0, {goals} goals x {iters} sweeps + scoring per pass, split "
                         f"over {used} processes (1 BLAS thread each), mean of {len(times)} passes "
                         f"({statistics.mean(times):.2f}s each); " + _cpu_sample_text(kind)}
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "problems/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": t_max / args.steps,
            "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None,
            "dtype": "f64" if prec == 0 else "f32+f64 (fp32 sample passes, fp64 QPs / G / multipliers)",
            "data": "synthetic (seeded scene generator, paper_2109_10392_b200/scenes.py)",
            "config": {"workload": args.config, "problems_per_step": total_L,
                       "problems_per_gpu": L, "iters": iters, "n": n,
                       "m": W.m, "n_b": nb, "scenes_per_gpu": W.S, "tol": 0.0,
                       "l2": "flushed between steps (256 MiB write)",
                       "parallelism": f"{'goal-column' if W.S == 1 else 'scene'} shards x{world} "
                                      f"({args.scaling} scaling)"},
            "roofline": roofline_entry(args, achieved, peak, k_ms, t_max / args.steps, n, W.m, nb),
            "e2e": {"value": e2e_value, "unit": "problems/s", "h2d_bytes_per_step": int(h2d),
                    "d2h_bytes_per_step": int(d2h), "ms_per_step": e2e_local / args.steps,
                    "path": "plan_batch -> bmpc_plan_host: page-locked inputs read in place over "
                            "the host link by the kernels, results back in one copy into a "
                            "pinned block"},
            **extra,
            "gpu_launches": launches_per_step * args.steps,
            "clocks": clk.summary(),
            "cpu_baseline": cpu,
            "best_index_scene0": best_global if world > 1 and W.S == 1 else best_e2e,
        }
        print(json.dumps(line))


def roofline_entry(args, achieved, peak, k_ms, step_ms, n, m, nb):
    """FP64-pipe roofline of the persistent AM kernel.  `achieved` counts the
    canonical algorithmic work W of SURVEY.md section 8d; `traffic` and the
    measured fp64-pipe activity come from the committed ncu capture of the same
    config (profiles/ncu_<config>_<precision>.json) when there is one."""
    r = {"bound": "fp64", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
         "frac": achieved / peak, "traffic": None, "kernel": "am_solve_kernel", "kernel_ms": k_ms,
         "kernel_share_of_step": k_ms / step_ms,
         "work": f"2*W(n,m,nb)*L*iters, canonical W={work_slots(n, m, nb)} fp64 slots per "
                 f"instance-sweep (SURVEY.md 8d)",
         "kernel_timing": "CUDA events on the bench stream around bmpc_sweeps launches "
                          "(same inputs, L2 flushed), median",
         "peak_source": "measured live: DFMA microbenchmark (csrc/peak.cu)",
         "note": "frac = canonical algorithmic work per second over the FP64 peak; the kernel "
                 "executes less than W (exact-form obstacle/acceleration blocks: an outside test "
                 "per obstacle term; obstacles culled by bounding boxes when m >= 24; whole obstacle slots "
                 "skipped while every sample stays within its recorded clearance), so frac "
                 "can exceed 1 on obstacle-heavy configs; frac_executed is the executed fp64 "
                 "flops over the peak (ncu capture of the same config, profiles/ncu_<config>_"
                 "<precision>.json)"}
    if args.precision == "fp32":
        # the fp32 mode runs the per-sample passes on the FP32 pipe (148 SMs x 128
        # FFMA lanes: twice the DFMA lanes) and the QPs / Gram terms in fp64, so
        # the canonical work is also quoted against the FP32 peak
        r["bound"] = "fp32+fp64"
        r["peak_fp32"] = 2.0 * peak
        r["frac_vs_fp32_peak"] = achieved / (2.0 * peak)
        r["note"] += ("; fp32 mode: the per-sample passes (sampling, atan2, sin/cos, the three "
                      "blocks and their residual contractions) run in fp32, the QP steps, Gram terms "
                      "of G and the multipliers in fp64; peak_fp32 = 2 x the measured DFMA peak "
                      "(FFMA lanes per SM = 2 x DFMA lanes on B200)")
    prof = ROOT / "profiles" / f"ncu_{args.config}_{args.precision}.json"
    if prof.exists():
        d = json.loads(prof.read_text())
        r["traffic"] = d["dram_read_bytes"] + d["dram_write_bytes"]
        r["traffic_unit"] = "bytes per launch (ncu dram__bytes_read+write)"
        r["ncu"] = {k: d[k] for k in ("report", "kernel", "fp64_pipe_active_pct", "issue_active_per_cycle",
                                        "warps_active_per_cycle", "duration_ms", "registers_per_thread",
                                        "fp64_thread_ops_per_cycle", "fp64_slot_frac_executed",
                                        "fp64_flop_frac_executed", "note") if k in d}
        if "fp64_flop_frac_executed" in d:
            # executed fp64 work (ncu SASS counts of DFMA x2 + DMUL + DADD per elapsed
            # cycle, over the DFMA lanes' peak): the pipe's real utilisation, next to
            # the canonical-W fraction above (which credits the work the exact-form
            # obstacle block and the culling never execute)
            r["frac_executed"] = d["fp64_flop_frac_executed"]
            r["achieved_executed"] = d["fp64_flop_frac_executed"] * peak
    return r


# ---------------------------------------------------------- reference arm ----
def run_reference(args, rank, world):
    """--impl reference: the reference's own CPU path (see cpu_reference_rate) on
    this host's cores, on a bounded sample of the same workload per step; rank 0
    only under torchrun."""
    if rank != 0:
        return
    from paper_2109_10392_b200.scenes import CONFIGS

    cfg = CONFIGS[args.config]
    iters = args.iters or cfg.iters
    goals = min(cfg.l, 1024)  # bounded sample of the workload per step: scene 0
    value, times, used, kind = cpu_reference_rate(args.config, goals, iters, args.steps, args.warmup)
    n, m, nb = cfg.n, cfg.m, cfg.degree + 1
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "problems/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * sum(times) / len(times), "higher_is_better": True, "scaling": args.scaling,
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded scene generator, paper_2109_10392_b200/scenes.py)",
        "config": {"workload": args.config, "problems_per_step": goals, "problems_per_gpu": goals, "iters": iters,
                   "n": n, "m": m, "n_b": nb, "scenes_per_gpu": 1, "tol": 0.0},
        "cpu_baseline": {"value": value, "unit": "problems/s", "cores": used,
                         "kind": "reference" if kind == "refpkg" else "port",
                         "sample": f"{args.config} scene 0, {goals} goals x {iters} sweeps + scoring per "
                                   f"step over {used} processes (1 BLAS thread each); " + _cpu_sample_text(kind)},
        "e2e": {"value": value, "unit": "problems/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c1")
    ap.add_argument("--iters", type=int, default=0)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"],
                    help="weak: a whole config per GPU; strong: the BASELINE config split over the GPUs")
    ap.add_argument("--precision", default="fp64", choices=["fp64", "fp32"],
                    help="fp32: fp32 sample passes, fp64 QPs / G / multipliers (tolerance in DESIGN.md)")
    args = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1 and args.impl == "ours":
        import torch
        import torch.distributed as dist

        # one process per GPU over NCCL; BMPC_DIST_BACKEND=gloo lets a single-GPU
        # box smoke-test the multi-rank plumbing (ranks then share the device and
        # the tiny collectives run on host tensors)
        backend = os.environ.get("BMPC_DIST_BACKEND", "nccl")
        dev_index = local_rank % max(1, torch.cuda.device_count())
        torch.cuda.set_device(dev_index)
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", dev_index))
        else:
            dist.init_process_group(backend)
    if args.impl == "reference":
        run_reference(args, rank, world)
    else:
        run_ours(args, rank, world, local_rank)
    if world > 1 and args.impl == "ours":
        import torch.distributed as dist

        dist.destroy_process_group()


if __name__ == "__main__":
    main()
