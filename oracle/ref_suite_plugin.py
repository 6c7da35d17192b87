"""pytest plugin (test infrastructure): run the reference's OWN solver and
planner test files, unmodified, against this package's sm_100a classes.

SURVEY.md section 8f-2.  ``build()`` copies, from /root/reference (build
container only), the reference's test modules and the ``oracles`` module their
``demo_batch`` fixture imports into oracle/_ref/ref_tests/ (git-ignored, ships to
the GPU box like oracle/_ref's compiled kernels):

    pkg/tests/{conftest,test_solver_units,test_solver_properties,test_planner}.py
    pkg/src/batchmpc/oracles.py

This plugin (loaded with ``-p ref_suite_plugin`` before any test module is
imported) makes ``import batchmpc`` resolve to ``paper_2109_10392_b200``: the
reference's session fixtures (pkg/tests/conftest.py:14-33 -- ``solver`` is
``BatchSolver(basis, mats, rho_xy=1.0)``) then build our GPU BatchSolver, our
basis/constant matrices, and every ``batchmpc.kernels`` / ``batchmpc.planner``
call in the tests runs our device code.  ``batchmpc.oracles`` is the reference's
own module, executed inside the aliased package so its ``from .solver import``
binds to ours too.  Nothing here is on the product path.
"""

from __future__ import annotations

import importlib.util
import sys
from pathlib import Path

HERE = Path(__file__).resolve().parent
ROOT = HERE.parent
REF_TESTS = HERE / "_ref" / "ref_tests"

sys.path.insert(0, str(ROOT))

import paper_2109_10392_b200 as _pkg  # noqa: E402
from paper_2109_10392_b200 import basis, kernels, planner, solver, traffic  # noqa: E402

for _name, _mod in (("batchmpc", _pkg), ("batchmpc.basis", basis), ("batchmpc.solver", solver),
                    ("batchmpc.kernels", kernels), ("batchmpc.planner", planner),
                    ("batchmpc.traffic", traffic)):
    sys.modules[_name] = _mod
_pkg.kernels, _pkg.planner, _pkg.traffic = kernels, planner, traffic

_spec = importlib.util.spec_from_file_location("batchmpc.oracles", REF_TESTS / "oracles.py")
_oracles = importlib.util.module_from_spec(_spec)
sys.modules["batchmpc.oracles"] = _oracles
_spec.loader.exec_module(_oracles)
_pkg.oracles = _oracles
