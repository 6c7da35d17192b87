"""Device time of the c1 step's pieces (CUDA events, L2 flushed): the full
async bmpc_plan, bmpc_solve (no scoring), the sweeps alone."""
import ctypes
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402

from paper_2109_10392_b200 import _native as nat  # noqa: E402
from paper_2109_10392_b200 import device as D  # noqa: E402
from paper_2109_10392_b200 import make_solver  # noqa: E402
from paper_2109_10392_b200.planner import FilterLimits, MetaCostSpec, _spec_struct  # noqa: E402
from paper_2109_10392_b200.scenes import make_workload  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c1"
W = make_workload(cfg)
solver = make_solver(W.n, W.t_f, W.degree, W.m)
ctx, lib = solver._context(), nat.load()
dev = torch.device("cuda", 0)
prob = D.DeviceProblem.from_host(W.n, W.xi_x, W.xi_y, W.b_xy, W.b_psi, W.l, W.a, W.b, W.v_min, W.v_max,
                                 W.a_max, device=dev)
sol = D.alloc_solution(solver.basis.n_b, W.n, W.L, 100, False, dev)
sc = D.alloc_score(W.L, W.S, dev)
status = torch.zeros(2, dtype=torch.int32, device=dev)
opts = nat.SolveOpts(max_iter=100, tol=0.0, status_dev=status.data_ptr())
spec = _spec_struct(MetaCostSpec("cruise", v_cruise=20.0), FilterLimits())
sp = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
ps = prob.c_struct()
flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)


def out():
    o = D.solution_struct(sol)
    o.history = None
    return o


fns = {
    "plan (async)": lambda: lib.bmpc_plan(ctx, ctypes.byref(ps), ctypes.byref(opts), ctypes.byref(out()),
                                          ctypes.byref(spec), ctypes.byref(D.score_struct(sc)), sp),
    "solve (async)": lambda: lib.bmpc_solve(ctx, ctypes.byref(ps), ctypes.byref(opts), ctypes.byref(out()), sp),
    "sweeps only": lambda: lib.bmpc_sweeps(ctx, ctypes.byref(ps), ctypes.byref(opts), 100, 0, 0, None, 0,
                                           ctypes.byref(out()), sp),
}
for name, fn in fns.items():
    ts = []
    for r in range(12):
        flush.fill_(float(r))
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        assert fn() == 0
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    ts = sorted(ts[2:])
    print(f"{cfg} {name:14s} median {ts[len(ts) // 2] * 1e3:8.1f} us  min {ts[0] * 1e3:8.1f} us")
