"""Multi-GPU sharding (one process per GPU, torch.distributed plumbing).

The path shards without any data-path collective:

* one scene (c1/c2): contiguous goal-column blocks per rank; each rank scores
  its block and the per-shard winner records (best_cost, global_index,
  n_feasible) are all-gathered and reduced lexicographically by
  (cost, index) -- numpy's lowest-index tie rule;
* many scenes (c3/c4): contiguous scene blocks per rank; per-scene results
  are complete on the owning rank, no cross-GPU reduction.

The only collective is that tiny all-gather (a few dozen bytes per rank).
"""

from __future__ import annotations

import math

import numpy as np


def shard_range(total: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous block [lo, hi) of `total` items owned by `rank` (ceil split)."""
    per = int(math.ceil(total / world)) if world else total
    lo = min(total, rank * per)
    return lo, min(total, lo + per)


def local_winner(meta_cost: np.ndarray, feasible: np.ndarray, offset: int) -> np.ndarray:
    """(best_cost, global_index, n_feasible) of one shard; cost +inf / index -1 if none."""
    feas = np.asarray(feasible, dtype=bool)
    if feas.any():
        costs = np.where(feas, meta_cost, np.inf)
        i = int(np.argmin(costs))
        return np.array([costs[i], float(offset + i), float(feas.sum())])
    return np.array([np.inf, -1.0, 0.0])


def merge_winners(records: np.ndarray) -> tuple[int | None, int]:
    """Reduce (world, 3) winner records: lowest cost, ties to lowest global index."""
    best, best_i = math.inf, None
    total = 0
    for cost, idx, nf in records:
        total += int(nf)
        if idx < 0:
            continue
        if best_i is None or cost < best or (cost == best and idx < best_i):
            best, best_i = cost, int(idx)
    return best_i, total


def allgather_winner(record: np.ndarray, group=None) -> tuple[int | None, int]:
    """All-gather each rank's winner record and reduce (every rank gets the result).

    Uses the default process group's backend (NCCL on GPUs, gloo on CPU)."""
    import torch
    import torch.distributed as dist

    backend = dist.get_backend(group)
    dev = torch.device("cuda", torch.cuda.current_device()) if backend == "nccl" else torch.device("cpu")
    t = torch.tensor(record, dtype=torch.float64, device=dev)
    out = [torch.empty_like(t) for _ in range(dist.get_world_size(group))]
    dist.all_gather(out, t, group=group)
    recs = np.stack([o.cpu().numpy() for o in out])
    return merge_winners(recs)


def allgather_winner_payload(record: np.ndarray, payload: np.ndarray, group=None):
    """Like allgather_winner, with the winning column's data riding in the same
    all-gather: each rank contributes its local winner record
    and a fixed-size payload (e.g. the winner's coefficients, 3 n_b doubles);
    every rank gets (best global index or None, n_feasible, winner payload or
    None)."""
    import torch
    import torch.distributed as dist

    backend = dist.get_backend(group)
    dev = torch.device("cuda", torch.cuda.current_device()) if backend == "nccl" else torch.device("cpu")
    pay = np.ascontiguousarray(payload, dtype=np.float64).ravel()
    t = torch.tensor(np.concatenate([np.asarray(record, dtype=np.float64), pay]), device=dev)
    out = [torch.empty_like(t) for _ in range(dist.get_world_size(group))]
    dist.all_gather(out, t, group=group)
    rows = np.stack([o.cpu().numpy() for o in out])
    best, nf = merge_winners(rows[:, :3])
    if best is None:
        return None, nf, None
    owner = int(np.nonzero(rows[:, 1] == best)[0][0])
    return best, nf, rows[owner, 3:].reshape(np.shape(payload))


def global_first_converged(local_worst: np.ndarray, tol: float, group=None) -> tuple[int, bool]:
    """Exact global early stop across shards (solver.py:437-439): the sweep
    count and converged flag of the single-GPU solve, from each rank's worst
    residual per sweep (max over its instances, NaN propagating) -- one
    all-reduce(MAX) of the per-sweep vector.  Ranks whose local solve ran
    longer re-run this many sweeps (instances are deterministic)."""
    import torch
    import torch.distributed as dist

    backend = dist.get_backend(group)
    dev = torch.device("cuda", torch.cuda.current_device()) if backend == "nccl" else torch.device("cpu")
    w = np.asarray(local_worst, dtype=np.float64)
    # NaN is "not converged": map it to +inf before the MAX (NaN has no MAX rule)
    t = torch.tensor(np.where(np.isnan(w), np.inf, w), device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    g = t.cpu().numpy()
    ok = np.nonzero(g <= tol)[0]
    if ok.size == 0:
        return len(g), False
    return int(ok[0]) + 1, True
