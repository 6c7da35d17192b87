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
