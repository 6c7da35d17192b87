"""The reference's OWN solver and planner test modules, unmodified, against this
package.

``build()`` copies /root/reference/pkg/tests/{conftest,test_solver_units,
test_solver_properties,test_planner}.py (plus the ``oracles`` module their
``demo_batch`` fixture imports) into oracle/_ref/ref_tests/;
oracle/ref_suite_plugin.py aliases ``batchmpc`` to ``paper_2109_10392_b200`` so
the reference's session fixtures (pkg/tests/conftest.py:14-33) build our
BatchSolver and every solver / kernels / planner call runs on the device.

Excluded, with the reason:
  test_planner.py::TestPlannerCycle::test_slow_lead_prefers_lane_change
      needs batchmpc.harness (TOML scenario loader + IDM traffic world), which
      is out of scope (closed-loop driver, not the path)

Expected to fail, with the reason (the run must fail exactly these):
  test_solver_units.py::TestSolveContract::test_residual_trend_on_canonical_scenario
      asserts per[-1, best] <= per[0, best] for the column with the smallest
      final residual.  On the demo batch that column is a straight lane-keeping
      goal that is converged before the first sweep: both numbers are rounding
      noise (the reference itself: 4.7e-13 then 3.2e-13, tests/golden/demo.npz
      history; ours 1.2e-13 then 5.1e-13), so their order is not a property of
      the algorithm.  The rest of that test (per[-1, best] <= 1e-3) holds and
      test_noise_column_stays_at_rounding_level below pins ours below 1e-12.
"""

import os
import re
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parents[1]
SUITE = ROOT / "oracle" / "_ref" / "ref_tests"
EXCLUDED = {"test_slow_lead_prefers_lane_change": "needs batchmpc.harness (out of scope)"}
EXPECTED_FAIL = {"test_solver_units.py": {"TestSolveContract::test_residual_trend_on_canonical_scenario"}}


@pytest.mark.parametrize("module,expect", [("test_solver_units.py", 30),
                                           ("test_solver_properties.py", 8),
                                           ("test_planner.py", 29)])
def test_reference_suite(cuda, module, expect, tmp_path):
    if not (SUITE / module).exists():
        pytest.fail(f"{SUITE / module} missing: run __graft_entry__.build() where /root/reference exists")
    ini = tmp_path / "pytest.ini"
    ini.write_text("[pytest]\naddopts = -p no:cacheprovider\n")
    env = dict(os.environ, PYTHONPATH=os.pathsep.join([str(ROOT / "oracle"), str(ROOT)]),
               OPENBLAS_NUM_THREADS="1")
    desel = " and ".join(f"not {k}" for k in EXCLUDED)
    cmd = [sys.executable, "-m", "pytest", "-p", "ref_suite_plugin", "-c", str(ini),
           "--rootdir", str(SUITE), str(SUITE / module), "-q", "-rfE", "-k", desel]
    r = subprocess.run(cmd, cwd=SUITE, env=env, capture_output=True, text=True, timeout=1200)
    tail = r.stdout[-6000:] + r.stderr[-2000:]
    print(tail)
    m = re.search(r"(\d+) passed", r.stdout)
    passed = int(m.group(1)) if m else 0
    failed = set(re.findall(r"^FAILED \S+?::(\S+)", r.stdout, re.M))
    want = EXPECTED_FAIL.get(module, set())
    assert failed == want, tail
    assert r.returncode == (1 if want else 0), tail
    assert passed == expect - len(want), (passed, expect, tail)


def test_noise_column_stays_at_rounding_level(cuda):
    """The column the expected failure above looks at: converged from the start,
    its residual stays at rounding level through 150 sweeps."""
    import numpy as np

    from conftest import golden
    from paper_2109_10392_b200 import ProblemBatch, make_solver

    z = golden("demo")
    solver = make_solver(100, 10.0, 10, 10)
    b = ProblemBatch(l=11, xi_x=z["xi_x"], xi_y=z["xi_y"], a=float(z["a"]), b=float(z["b"]),
                     v_min=float(z["v_min"]), v_max=float(z["v_max"]), a_max=float(z["a_max"]),
                     b_xy=z["b_xy"], b_psi=z["b_psi"])
    _, info = solver.solve(b, max_iter=150, tol=0.0)
    per = np.array([r.max_per_instance() for r in info.residual_history])
    best = int(np.argmin(per[-1]))
    assert per[:, best].max() <= 1e-12
