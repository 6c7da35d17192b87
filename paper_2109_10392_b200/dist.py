"""Multi-GPU sharding (one process per GPU, torch.distributed plumbing).

The path shards without any data-path collective:

* one scene (c1/c2): contiguous goal-column blocks per rank; each rank scores
  its block and the per-shard winner records (best_cost, global_index,
  n_feasible) are all-gathered and reduced lexicographically by
  (cost, index) -- numpy's lowest-index tie rule;
* many scenes (c3/c4): contiguous scene blocks per rank; per-scene results
  are complete on the owning rank, no cross-GPU reduction.

The only collective is that tiny all-gather (a few dozen bytes per rank).
``plan_sharded`` is the product entry point: the planner call of
planner.plan_batch, split over the ranks of a process group, with results
identical to the single-GPU call (instance arithmetic never depends on the
shard) and the reference's global early-stop rule kept across shards
(solver.py:437-439).
"""

from __future__ import annotations

import math
from dataclasses import dataclass

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


# ------------------------------------------------------- sharded planning ----
def _group_info(group=None) -> tuple[int, int]:
    import torch.distributed as dist

    if not (dist.is_available() and dist.is_initialized()):
        return 1, 0
    return dist.get_world_size(group), dist.get_rank(group)


def allgather_rows(vec: np.ndarray, group=None) -> np.ndarray:
    """All-gather one fixed-length float64 vector per rank -> (world, len) on
    every rank (NCCL: through device memory; gloo: host tensors)."""
    import torch
    import torch.distributed as dist

    backend = dist.get_backend(group)
    dev = torch.device("cuda", torch.cuda.current_device()) if backend == "nccl" else torch.device("cpu")
    t = torch.as_tensor(np.ascontiguousarray(vec, dtype=np.float64)).to(dev)
    out = torch.empty(dist.get_world_size(group), t.numel(), dtype=torch.float64, device=dev)
    dist.all_gather_into_tensor(out, t, group=group) if backend == "nccl" else \
        dist.all_gather(list(out.unbind(0)), t, group=group)
    return out.cpu().numpy()


def scene_records(res, nb: int, S_local: int, per: int, l: int) -> np.ndarray:
    """Per-scene result rows of one rank's scene block, padded to `per` scenes:
    [best, argmin_all, argmin_hc, n_feasible, best_cost, coef(3 nb)] per scene
    (-1 / inf / NaN for None), flattened."""
    width = 5 + 3 * nb
    rows = np.full((per, width), np.nan)
    rows[:, :4] = -1.0
    rows[:, 4] = np.inf
    for s in range(S_local):
        b = res.best_index[s]
        rows[s, 0] = -1.0 if b is None else float(b)
        rows[s, 1], rows[s, 2], rows[s, 3] = res.argmin_all[s], res.argmin_hc[s], res.n_feasible[s]
        if b is not None:
            g = s * l + b
            rows[s, 4] = res.meta_cost[g]
            rows[s, 5:] = np.concatenate([res.c_x[:, g], res.c_y[:, g], res.c_psi[:, g]])
    return rows.ravel()


def goal_records(meta, flags, coef, offset: int) -> np.ndarray:
    """One rank's goal-column block of one scene: (cost, global index, count)
    winner records under the three masks of the scoring (feasible = all three
    filters, unfiltered, heading+collision only) plus the feasible winner's
    coefficients (3 nb; NaN when none)."""
    flags = np.asarray(flags)
    nb3 = coef.shape[0]
    recs = []
    for mask in (flags == 7, np.ones(flags.shape, dtype=bool), (flags & 5) == 5):
        if mask.any():
            c = np.where(mask, meta, np.inf)
            i = int(np.argmin(c))
            recs.append([c[i], float(offset + i), float(mask.sum())])
        else:
            recs.append([np.inf, -1.0, 0.0])
    f = recs[0]
    pay = coef[:, int(f[1]) - offset] if f[1] >= 0 else np.full(nb3, np.nan)
    return np.concatenate([np.ravel(recs), pay])


def merge_goal_records(rows: np.ndarray):
    """(world, 9 + 3 nb) goal records -> (best, argmin_all, argmin_hc, n_feasible,
    best_cost, winner coef or None)."""
    out = []
    for q in range(3):
        out.append(merge_winners(rows[:, 3 * q:3 * q + 3]))
    best, nf = out[0]
    cost, coef = np.inf, None
    if best is not None:
        owner = int(np.nonzero(rows[:, 1] == best)[0][0])
        cost, coef = float(rows[owner, 0]), rows[owner, 9:].copy()
    return best, out[1][0], out[2][0], nf, cost, coef


@dataclass
class ShardedPlan:
    """plan_sharded's result on every rank.  Per scene (S entries):
    best_index (None when nothing is feasible), argmin_all, argmin_hc (-1 =
    None), n_feasible, best_cost and the winner's coefficients (3, n_b) (None).
    ``local`` is this rank's own planner.PlanResult over its shard
    (``shard`` = [lo, hi) goal columns of the scene, or scenes)."""

    best_index: list
    argmin_all: np.ndarray
    argmin_hc: np.ndarray
    n_feasible: np.ndarray
    best_cost: np.ndarray
    best_coef: list
    iterations: int
    converged: bool
    mode: str            # "goals" (one scene, columns split) or "scenes"
    shard: tuple
    local: object


def _exact_sweeps(solver, sub, max_iter, tol, status, group, precision="fp64"):
    """The single-GPU early-stop sweep count across shards (solver.py:437-439).
    Every rank's local solve stopped at its own first converged sweep t_r (or
    ran max_iter).  If no rank converged, or all converged at the same sweep,
    that is the global answer; otherwise each rank re-solves without stopping,
    with its residual history, and the per-sweep worst residuals are
    all-reduced (global_first_converged)."""
    st = allgather_rows(np.array(status, dtype=np.float64), group)
    live = st[:, 1] != 2  # 2: an empty shard, no say in the decision
    its, conv = st[live, 0].astype(int), st[live, 1] > 0
    if not conv.any():
        return max_iter, False, False
    if conv.all() and (its == its[0]).all():
        return int(its[0]), True, False
    worst = np.zeros(max_iter)
    if sub is not None:
        import torch

        prob = solver._problem(sub)
        sol = solver.solve_device(prob, max_iter=max_iter, tol=-1.0, want_v=False, precision=precision)
        h = sol.history[:max_iter]
        worst = torch.nan_to_num(h, nan=float("inf")).amax(dim=(1, 2)).cpu().numpy()
    t, c = global_first_converged(worst, tol, group)
    return t, c, True


def plan_sharded(solver, scenes, max_iter: int = 100, tol: float = 0.0, spec=None, limits=None,
                 precision: str = "fp64", group=None) -> ShardedPlan:
    """planner.plan_batch over the ranks of a process group (one process per
    GPU).  One scene: contiguous goal-column blocks, the
    winner records of the three scoring masks (and the feasible winner's
    coefficients) all-gathered and reduced with numpy's tie rule.  Stacked
    scenes: contiguous scene blocks, the per-scene results all-gathered.
    Every rank passes the same full ``scenes``; results equal the single-GPU
    plan_batch's bit for bit."""
    from .planner import plan_batch

    world, rank = _group_info(group)
    xi_x, xi_y, S, l = solver.check_scenes(scenes)
    nb = solver.basis.n_b
    from .scenes import SceneBatch

    def sub_batch(xx, xy, bxy, bps, Sl, ll):
        return SceneBatch(solver.basis.grid.n, 0.0, 0, xx.shape[1] // solver.basis.grid.n, ll, Sl,
                          xx, xy, np.ascontiguousarray(bxy), np.ascontiguousarray(bps), scenes.a, scenes.b,
                          scenes.v_min, scenes.v_max, scenes.a_max, solver.rho_xy)

    if S == 1:
        mode = "goals"
        lo, hi = shard_range(l, rank, world)
        sub = sub_batch(xi_x, xi_y, scenes.b_xy[:, lo:hi], scenes.b_psi[:, lo:hi], 1, hi - lo) if hi > lo else None
    else:
        mode = "scenes"
        lo, hi = shard_range(S, rank, world)
        cols = slice(lo * l, hi * l)
        sub = sub_batch(xi_x[lo:hi], xi_y[lo:hi], scenes.b_xy[:, cols], scenes.b_psi[:, cols], hi - lo, l) \
            if hi > lo else None

    def run(iters, t):
        return plan_batch(solver, sub, max_iter=iters, tol=t, spec=spec, limits=limits,
                          precision=precision) if sub is not None else None

    res = run(max_iter, tol)
    iters, conv = max_iter, False
    if world > 1:
        status = (res.iterations, int(res.converged)) if res is not None else (max_iter, 2)
        iters, conv, rerun = _exact_sweeps(solver, sub, max_iter, tol, status, group, precision)
        if rerun or (res is not None and res.iterations != iters):
            res = run(iters, -1.0)
    elif res is not None:
        iters, conv = res.iterations, res.converged
    if mode == "goals":
        if res is not None:
            coef = np.concatenate([res.c_x, res.c_y, res.c_psi], axis=0)
            rec = goal_records(res.meta_cost, res.flags, coef, lo)
        else:
            rec = np.concatenate([np.tile([np.inf, -1.0, 0.0], 3), np.full(3 * nb, np.nan)])
        rows = allgather_rows(rec, group)[None] if world > 1 else rec[None, None]
        best, a_all, a_hc, nf, cost, coef = merge_goal_records(rows[0])
        return ShardedPlan([best], np.array([-1 if a_all is None else a_all]),
                           np.array([-1 if a_hc is None else a_hc]), np.array([nf]), np.array([cost]),
                           [None if coef is None else coef.reshape(3, nb)], iters, conv, mode, (lo, hi), res)
    per = shard_range(S, 0, world)[1]
    rec = scene_records(res, nb, hi - lo, per, l) if res is not None else scene_records(None, nb, 0, per, l)
    rows = (allgather_rows(rec, group) if world > 1 else rec[None]).reshape(-1, 5 + 3 * nb)[:S]
    best = [None if b < 0 else int(b) for b in rows[:, 0]]
    coefs = [None if b is None else rows[s, 5:].reshape(3, nb) for s, b in enumerate(best)]
    return ShardedPlan(best, rows[:, 1].astype(np.int64), rows[:, 2].astype(np.int64),
                       rows[:, 3].astype(np.int64), rows[:, 4].copy(), coefs, iters, conv, mode, (lo, hi), res)


def _better(cost, idx, best, best_i) -> bool:
    """numpy argmin order on (cost, index): a NaN cost wins (the first NaN),
    otherwise the lower cost, ties to the lower index."""
    if best_i is None:
        return True
    cn, bn = cost != cost, best != best
    if cn or bn:
        return cn and (not bn or idx < best_i)
    return cost < best or (cost == best and idx < best_i)


def merge_winners(records: np.ndarray) -> tuple[int | None, int]:
    """Reduce (world, 3) winner records: lowest cost, ties to lowest global index
    (numpy's argmin rule, planner.py:248-257, NaN included)."""
    best, best_i = math.inf, None
    total = 0
    for cost, idx, nf in records:
        total += int(nf)
        if idx < 0:
            continue
        if _better(cost, int(idx), best, best_i):
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
