"""Where the end-to-end plan_batch time goes (c1 by default): total vs the
device-resident bmpc_plan vs its host-side parts.  Usage: e2e_breakdown.py [--config c1]"""
import argparse
import ctypes
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2109_10392_b200 import _native as nat  # noqa: E402
from paper_2109_10392_b200 import device as D  # noqa: E402
from paper_2109_10392_b200 import make_solver  # noqa: E402
from paper_2109_10392_b200.planner import FilterLimits, MetaCostSpec, _spec_struct, plan_batch  # noqa: E402
from paper_2109_10392_b200.scenes import make_workload  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c1")
ap.add_argument("--reps", type=int, default=20)
args = ap.parse_args()
W = make_workload(args.config)
solver = make_solver(W.n, W.t_f, W.degree, W.m)
spec, limits = MetaCostSpec("cruise", v_cruise=20.0), FilterLimits()
pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory().numpy()  # noqa: E731


class H:
    pass


h = H()
h.xi_x, h.xi_y, h.b_xy, h.b_psi = pin(W.xi_x), pin(W.xi_y), pin(W.b_xy), pin(W.b_psi)
h.l, h.S, h.a, h.b, h.v_min, h.v_max, h.a_max = W.l, W.S, W.a, W.b, W.v_min, W.v_max, W.a_max


def timeit(fn, reps):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        ts.append((time.perf_counter() - t0) * 1e3)
    return float(np.median(ts))


t_plan = timeit(lambda: plan_batch(solver, h, max_iter=100, tol=0.0, spec=spec, limits=limits), args.reps)
dev = torch.device("cuda", 0)
prob = D.DeviceProblem.from_host(W.n, W.xi_x, W.xi_y, W.b_xy, W.b_psi, W.l, W.a, W.b, W.v_min, W.v_max,
                                 W.a_max, device=dev)
sol = D.alloc_solution(solver.basis.n_b, W.n, W.L, 100, False, dev)
sc = D.alloc_score(W.L, W.S, dev)
lib, ctx = nat.load(), solver._context()
opts = nat.SolveOpts(max_iter=100, tol=0.0)
sspec = _spec_struct(spec, limits)
sp = ctypes.c_void_p(D.stream_ptr())
ps = prob.c_struct()
t_dev = timeit(lambda: nat.check(lib.bmpc_plan(ctx, ctypes.byref(ps), ctypes.byref(opts),
                                               ctypes.byref(D.solution_struct(sol)), ctypes.byref(sspec),
                                               ctypes.byref(D.score_struct(sc)), sp)), args.reps)
big = torch.empty(3 * 11 * W.L, dtype=torch.float64, device=dev)
hp = torch.empty(big.numel(), dtype=torch.float64).pin_memory()
t_d2h_pin = timeit(lambda: hp.copy_(big), args.reps)
hpg = np.empty(big.numel())
t_d2h_page = timeit(lambda: hpg.__setitem__(slice(None), big.cpu().numpy()), args.reps)
print(f"{args.config}: plan_batch {t_plan:.3f} ms | device bmpc_plan {t_dev:.3f} ms | "
      f"D2H coef pinned {t_d2h_pin:.3f} ms pageable {t_d2h_page:.3f} ms")

# the C-ABI host entry alone (structs prebuilt): plan_batch minus Python
xi_x, xi_y = h.xi_x, h.xi_y
prob_h = nat.Problem(W.m, W.l, W.S, xi_x.ctypes.data, xi_y.ctypes.data, h.b_xy.ctypes.data,
                     h.b_psi.ctypes.data, W.a, W.b, W.v_min, W.v_max, W.a_max)
coef = np.empty((3, solver.basis.n_b, W.L))
res = np.empty((3, W.L))
out_h = nat.SolveOut(coef[0].ctypes.data, coef[1].ctypes.data, coef[2].ctypes.data, None, None,
                     None, None, None, res.ctypes.data, 0, 0)
meta, mr, hm = np.empty((3, W.L))
flags = np.empty(W.L, dtype=np.uint8)
best, amin, ahc, nf = np.empty((4, W.S), dtype=np.int64)
so = nat.ScoreOut(meta.ctypes.data, mr.ctypes.data, hm.ctypes.data, flags.ctypes.data,
                  best.ctypes.data, amin.ctypes.data, ahc.ctypes.data, nf.ctypes.data)
t_host = timeit(lambda: nat.check(lib.bmpc_plan_host(ctx, ctypes.byref(prob_h), ctypes.byref(opts),
                                                     ctypes.byref(out_h), ctypes.byref(sspec),
                                                     ctypes.byref(so), sp)), args.reps)
t_empty = timeit(lambda: torch.cuda.synchronize(), args.reps)
print(f"{args.config}: bmpc_plan_host (ctypes, structs prebuilt) {t_host:.3f} ms | "
      f"python plan_batch overhead {t_plan - t_host:.3f} ms | bare sync {t_empty:.3f} ms")


def host_fresh():
    coef = np.empty((3, solver.basis.n_b, W.L))
    res = np.empty((3, W.L))
    o = nat.SolveOut(coef[0].ctypes.data, coef[1].ctypes.data, coef[2].ctypes.data, None, None,
                     None, None, None, res.ctypes.data, 0, 0)
    meta, mr, hm = np.empty((3, W.L))
    flags = np.empty(W.L, dtype=np.uint8)
    best, amin, ahc, nf = np.empty((4, W.S), dtype=np.int64)
    s = nat.ScoreOut(meta.ctypes.data, mr.ctypes.data, hm.ctypes.data, flags.ctypes.data,
                     best.ctypes.data, amin.ctypes.data, ahc.ctypes.data, nf.ctypes.data)
    nat.check(lib.bmpc_plan_host(ctx, ctypes.byref(prob_h), ctypes.byref(opts), ctypes.byref(o),
                                 ctypes.byref(sspec), ctypes.byref(s), sp))


t_fresh = timeit(host_fresh, args.reps)
print(f"{args.config}: bmpc_plan_host with fresh numpy outputs {t_fresh:.3f} ms")
