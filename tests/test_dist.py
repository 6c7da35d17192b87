"""Multi-process (gloo, world size 2) coverage of the multi-GPU host logic:
contiguous goal-column shards, the per-shard winner records and the
all-gather reduction with numpy's lowest-index tie rule.  CPU only."""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, costs, feas, out):
    import torch.distributed as dist

    from paper_2109_10392_b200.dist import allgather_winner, local_winner, shard_range

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        lo, hi = shard_range(len(costs), rank, world)
        rec = local_winner(costs[lo:hi], feas[lo:hi], lo)
        best, nf = allgather_winner(rec)
        out[rank] = (best if best is not None else -1, nf)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("case", ["random", "ties", "none_feasible", "one_shard_empty"])
def test_gloo_world2_argmin(case):
    rng = np.random.default_rng(7)
    L = 1024
    costs = rng.normal(100.0, 10.0, L)
    feas = rng.random(L) < 0.3
    if case == "ties":
        costs = np.round(costs / 10.0)  # many exact ties across both shards
    elif case == "none_feasible":
        feas[:] = False
    elif case == "one_shard_empty":
        feas[: L // 2] = False
    mgr = mp.Manager()
    out = mgr.dict()
    port = _free_port()
    mp.spawn(_worker, args=(2, port, costs, feas, out), nprocs=2, join=True)
    expect = int(np.argmin(np.where(feas, costs, np.inf))) if feas.any() else -1
    assert out[0] == out[1] == (expect, int(feas.sum()))


def _worker_payload(rank, world, port, costs, feas, coefs, out):
    import torch.distributed as dist

    from paper_2109_10392_b200.dist import allgather_winner_payload, local_winner, shard_range

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        lo, hi = shard_range(len(costs), rank, world)
        rec = local_winner(costs[lo:hi], feas[lo:hi], lo)
        i = int(rec[1]) - lo if rec[1] >= 0 else 0
        best, nf, pay = allgather_winner_payload(rec, coefs[:, :, lo + i])
        out[rank] = (best if best is not None else -1, nf, None if pay is None else pay.tolist())
    finally:
        dist.destroy_process_group()


def test_gloo_world2_winner_payload():
    """The winning column's coefficients reach every rank inside the all-gather."""
    rng = np.random.default_rng(3)
    L, nb = 512, 11
    costs = rng.normal(100.0, 10.0, L)
    feas = rng.random(L) < 0.4
    coefs = rng.normal(size=(3, nb, L))
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker_payload, args=(2, _free_port(), costs, feas, coefs, out), nprocs=2, join=True)
    expect = int(np.argmin(np.where(feas, costs, np.inf)))
    for r in (0, 1):
        best, nf, pay = out[r]
        assert best == expect and nf == int(feas.sum())
        np.testing.assert_array_equal(np.array(pay), coefs[:, :, expect])


def _worker_tol(rank, world, port, worst, tol, out):
    import torch.distributed as dist

    from paper_2109_10392_b200.dist import global_first_converged

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        out[rank] = global_first_converged(worst[rank], tol)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("case", ["global_later", "never", "nan"])
def test_gloo_world2_global_early_stop(case):
    """Per-shard worst residuals -> the single-GPU early-stop sweep count."""
    it = 30
    t = np.arange(it, dtype=np.float64)
    worst = np.stack([1.0 / (1 + t), 2.0 / (1 + t)])  # rank 1 converges later
    tol = 0.1
    if case == "never":
        tol = 1e-9
    if case == "nan":
        worst[1, 25:] = np.nan
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker_tol, args=(2, _free_port(), worst, tol, out), nprocs=2, join=True)
    g = np.max(np.where(np.isnan(worst), np.inf, worst), axis=0)
    ok = np.nonzero(g <= tol)[0]
    expect = (int(ok[0]) + 1, True) if ok.size else (it, False)
    assert out[0] == out[1] == expect
    if case == "global_later":
        assert expect[0] == 20  # rank 0 alone would stop at 10


def test_goal_and_scene_record_merges():
    """plan_sharded's record builders and merges (CPU): the three scoring masks
    with numpy's tie / NaN rules across shards, and scene-block padding."""
    from types import SimpleNamespace

    from paper_2109_10392_b200.dist import goal_records, merge_goal_records, scene_records, shard_range

    rng = np.random.default_rng(11)
    L, nb = 300, 4
    meta = np.round(rng.normal(50.0, 5.0, L))  # many exact ties
    meta[17] = np.nan
    flags = rng.integers(0, 8, L).astype(np.uint8)
    coef = rng.normal(size=(3 * nb, L))
    for world in (1, 2, 3, 7):
        rows = []
        for r in range(world):
            lo, hi = shard_range(L, r, world)
            rows.append(goal_records(meta[lo:hi], flags[lo:hi], coef[:, lo:hi], lo))
        best, a_all, a_hc, nf, cost, c = merge_goal_records(np.stack(rows))
        feas, hc = flags == 7, (flags & 5) == 5
        assert best == int(np.argmin(np.where(feas, meta, np.inf)))
        assert a_all == int(np.argmin(meta)) == 17  # NaN wins, as numpy's argmin
        assert a_hc == int(np.argmin(np.where(hc, meta, np.inf)))
        assert nf == int(feas.sum()) and cost == meta[best]
        np.testing.assert_array_equal(c, coef[:, best])
    res = SimpleNamespace(best_index=[3, None], argmin_all=np.array([1, 2]), argmin_hc=np.array([3, -1]),
                          n_feasible=np.array([5, 0]), meta_cost=np.arange(20.0),
                          c_x=np.ones((nb, 20)), c_y=2 * np.ones((nb, 20)), c_psi=3 * np.ones((nb, 20)))
    rec = scene_records(res, nb, 2, 3, 10).reshape(3, -1)
    assert rec[0, :5].tolist() == [3, 1, 3, 5, 3.0] and rec[1, 0] == -1 and rec[1, 4] == np.inf
    assert rec[2, 0] == -1 and rec[0, 5:].tolist() == [1] * nb + [2] * nb + [3] * nb
