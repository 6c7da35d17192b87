"""The C ABI from plain C: examples/plan_c.c (gcc, no Python in the loop) runs
bmpc_plan_host on a dumped c0 problem and must report what the Python API
reports for the same inputs -- bit-identical coefficients (an FNV-1a hash of
their bytes), the same best index and sweep count."""

import subprocess

import numpy as np
import pytest

from conftest import golden

pytestmark = pytest.mark.gpu


def test_plain_c_caller(cuda, tmp_path):
    from pathlib import Path

    from paper_2109_10392_b200 import make_solver
    from paper_2109_10392_b200.planner import FilterLimits, MetaCostSpec, plan_batch

    root = Path(__file__).resolve().parents[1]
    exe = tmp_path / "plan_c"
    lib = root / "paper_2109_10392_b200" / "_lib"
    subprocess.run(["gcc", "-O2", str(root / "examples" / "plan_c.c"), f"-I{root / 'include'}", f"-L{lib}",
                    "-lbatchmpc_b200", f"-Wl,-rpath,{lib}", "-o", str(exe)], check=True)
    z = golden("c0")
    n, t_f, degree, m = int(z["n"]), float(z["t_f"]), int(z["degree"]), int(z["m"])
    solver = make_solver(n, t_f, degree, m)
    b, k = solver.basis, solver.kkt
    l, iters = int(z["l"]), 60
    hdr = [n, b.n_b, m, l, iters, solver.rho_xy, float(z["a"]), float(z["b"]), float(z["v_min"]),
           float(z["v_max"]), float(z["a_max"])]
    parts = [np.array(hdr, dtype=np.float64), b.P, b.Pdot, b.Pddot, solver._tau, k.inv_axis, k.matrix_axis,
             k.inv_psi, k.matrix_psi, k.ftf_axis, np.atleast_2d(z["xi_x"])[0], np.atleast_2d(z["xi_y"])[0],
             z["b_xy"], z["b_psi"]]
    path = tmp_path / "problem.bin"
    with open(path, "wb") as fh:
        for p in parts:
            fh.write(np.ascontiguousarray(p, dtype=np.float64).tobytes())
    out = subprocess.run([str(exe), str(path)], check=True, capture_output=True, text=True).stdout.split()
    got = dict(zip(out[::2], out[1::2]))

    class Scenes:
        pass

    sc = Scenes()
    sc.xi_x, sc.xi_y = np.atleast_2d(z["xi_x"]), np.atleast_2d(z["xi_y"])
    sc.b_xy, sc.b_psi, sc.l, sc.S = z["b_xy"], z["b_psi"], l, 1
    sc.a, sc.b, sc.v_min, sc.v_max, sc.a_max = (float(z[q]) for q in ("a", "b", "v_min", "v_max", "a_max"))
    res = plan_batch(solver, sc, max_iter=iters, tol=0.0, spec=MetaCostSpec("cruise", v_cruise=20.0),
                     limits=FilterLimits())
    coef = np.concatenate([res.c_x.ravel(), res.c_y.ravel(), res.c_psi.ravel()]).astype(np.float64)
    h = 1469598103934665603
    for byte in coef.tobytes():
        h = ((h ^ byte) * 1099511628211) & 0xFFFFFFFFFFFFFFFF
    assert int(got["iterations"]) == res.iterations == iters
    assert int(got["best_index"]) == (res.best_index[0] if res.best_index[0] is not None else -1)
    assert int(got["argmin_all"]) == int(res.argmin_all[0])
    assert int(got["fnv"]) == h  # bit-identical coefficients
