"""bench-gpu CLI: timing.csv and run.jsonl in the reference harness formats."""

import csv
import json

import pytest

pytestmark = pytest.mark.gpu


def test_bench_gpu_cli(cuda, tmp_path):
    from paper_2109_10392_b200.bench_gpu import main

    main(["--sizes", "16", "64", "--cycles", "3", "--out-dir", str(tmp_path)])
    rows = list(csv.DictReader(open(tmp_path / "timing.csv")))
    assert [r["l"] for r in rows] == ["16", "64"] and all(r["n_solves"] == "3" for r in rows)
    assert list(rows[0]) == ["l", "n_solves", "mean", "min", "max"]
    assert all(0 < float(r["min"]) <= float(r["mean"]) <= float(r["max"]) for r in rows)
    recs = [json.loads(x) for x in open(tmp_path / "run.jsonl")]
    assert [r["cycle"] for r in recs] == [0, 1, 2]
    r = recs[0]
    assert len(r["meta_costs"]) == 64 and len(r["goal_lanes"]) == 64 and len(r["obstacles"]) == 10
    assert set(r["residuals_best"]) == {"obs", "acc", "nonhol"}
    assert len(r["residuals_best"]["obs"]) == r["residual_iters"]
