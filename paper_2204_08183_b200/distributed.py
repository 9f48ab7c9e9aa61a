"""Multi-GPU drivers: one process per GPU (torchrun), torch.distributed for
the plumbing.

cross_validate_distributed — config C4: the (grid point x
replicate) tasks of the reference's cross_validate
(/root/reference/proj/src/crossval.cpp:123-216) are independent fits; they are
dealt round-robin to ranks, each rank runs its tasks on its own GPU (device
row-mask folds, no design copies), the per-task fold scores are all-gathered
and merged in TASK order exactly as the reference merges its thread slots
(crossval.cpp:176-211), so the result does not depend on the world size.
There is no data-path collective; "scaling" is weak in tasks per GPU.
"""
from __future__ import annotations

import math
import sys
from typing import Callable, List, Optional, Sequence

TaskRunner = Callable[[Sequence[int]], List[Optional[List[float]]]]


def _dist():
    # no process group can exist unless torch.distributed was imported: a
    # single-process caller does not pay the (seconds-long) torch import
    dist = sys.modules.get("torch.distributed")
    if dist is None:
        return None, 0, 1
    if dist.is_available() and dist.is_initialized():
        return dist, dist.get_rank(), dist.get_world_size()
    return None, 0, 1


def shard_tasks(n_tasks: int, rank: int, world: int) -> List[int]:
    """Round-robin deal: task t -> rank t % world."""
    return list(range(rank, n_tasks, world))


def merge_scores(grid: Sequence[float], repetitions: int,
                 scores: Sequence[Optional[Sequence[float]]]) -> dict:
    """The reference's task-ordered aggregation (crossval.cpp:176-211):
    mean and sample sd of all fold scores per grid point, failed replicates
    dropped and counted, argmax with the first on ties."""
    curve, failed = [], 0
    for gi, lam in enumerate(grid):
        vals, s = [], 0.0
        for t in range(repetitions):
            sc = scores[gi * repetitions + t]
            if sc is None:
                failed += 1
                continue
            for v in sc:
                vals.append(float(v))
                s += float(v)
        mean = s / len(vals) if vals else 0.0
        spread = 0.0
        if len(vals) > 1:
            ss = 0.0
            for v in vals:
                ss += (v - mean) * (v - mean)
            spread = math.sqrt(ss / (len(vals) - 1))
        curve.append({"strength": float(lam), "mean_loglik": mean, "spread": spread,
                      "evaluations": len(vals)})
    best = None
    for gi, pt in enumerate(curve):
        if pt["evaluations"] == 0:
            continue
        if best is None or pt["mean_loglik"] > curve[best]["mean_loglik"]:
            best = gi
    if best is None:
        raise RuntimeError("every cross-validation replicate failed; nothing to select")
    return {"curve": curve, "selected": curve[best]["strength"], "failed_replicates": failed}


def local_device() -> int:
    """This process's GPU: LOCAL_RANK (torchrun), else the current CUDA device,
    else 0 — never the global rank (wrong on multi-node jobs)."""
    import os
    if "LOCAL_RANK" in os.environ:
        return int(os.environ["LOCAL_RANK"])
    try:
        import torch
        if torch.cuda.is_available():
            return torch.cuda.current_device()
    except Exception:
        pass
    return 0


def device_task_runner(ds, model: str, penalty: str, grid, folds: int, repetitions: int,
                       seed: int, tol: float, max_cycles: int, device: int) -> TaskRunner:
    """Tasks on this rank's GPU through the C++ mirror (survscan.cv_run_tasks:
    every fold fit of the rank's tasks advances in batched multi-fit launches)."""
    import survscan

    def run(tasks):
        return list(survscan.cv_run_tasks(ds, model, penalty, list(grid), folds, repetitions, seed,
                                          list(tasks), tol=tol, max_cycles=max_cycles,
                                          devices=[device]))
    return run


def _gather_checked(dist, world, local, err):
    """All-gather (payload, error) from every rank; if any rank failed, raise
    the same error on EVERY rank (no rank is left waiting in a collective)."""
    parts = [(local, err)]
    if dist is not None and world > 1:
        parts = [None] * world
        dist.all_gather_object(parts, (local, err))
    bad = [(r, e) for r, (_, e) in enumerate(parts) if e is not None]
    if bad:
        r, e = bad[0]
        raise RuntimeError(f"rank {r} failed: {e}")
    return [p for p, _ in parts]


def _broadcast(dist, world, obj):
    if dist is None or world == 1:
        return obj
    box = [obj]
    dist.broadcast_object_list(box, src=0)
    return box[0]


def cross_validate_distributed(ds, model: str = "cox", penalty: str = "l1",
                               grid: Sequence[float] = (), folds: int = 10,
                               repetitions: int = 10, seed: int = 0, tol: float = 1e-6,
                               max_cycles: int = 1000, device: Optional[int] = None,
                               task_runner: Optional[TaskRunner] = None,
                               final_fit: bool = True) -> dict:
    """C4 across ranks.  Every rank returns the same merged result (or raises
    the same error)."""
    dist, rank, world = _dist()
    import survscan
    dev = local_device() if device is None else device
    grid = list(grid)
    if not grid:  # gamma_max sweep once, on rank 0's GPU, then broadcast
        res = None
        if rank == 0:
            try:
                res = (list(survscan.cv_grid(ds, model, device=dev)), None)
            except Exception as exc:  # noqa: BLE001 - re-raised on every rank
                res = (None, f"{type(exc).__name__}: {exc}")
        res = _broadcast(dist, world, res)
        if res[1] is not None:
            raise RuntimeError(f"rank 0 failed: {res[1]}")
        grid = res[0]
    survscan.cv_check_folds(ds, folds, repetitions, seed, len(grid))
    n_tasks = len(grid) * repetitions
    mine = shard_tasks(n_tasks, rank, world)
    if task_runner is None:
        task_runner = device_task_runner(ds, model, penalty, grid, folds, repetitions, seed, tol,
                                         max_cycles, dev)
    local, err = [], None
    try:
        local = list(zip(mine, task_runner(mine)))
    except Exception as exc:  # noqa: BLE001 - re-raised on every rank
        err = f"{type(exc).__name__}: {exc}"
    parts = _gather_checked(dist, world, local, err)
    scores: List[Optional[List[float]]] = [None] * n_tasks
    seen = 0
    for part in parts:
        for t, sc in part:
            scores[t] = None if sc is None else [float(v) for v in sc]
            seen += 1
    if seen != n_tasks:
        raise RuntimeError(f"gathered {seen} of {n_tasks} task results")
    out = merge_scores(grid, repetitions, scores)
    out["tasks_per_rank"] = len(mine)
    if final_fit:
        out["final_fit"] = survscan.fit(ds, model=model, penalty=penalty,
                                        strength=out["selected"], tol=tol, max_cycles=max_cycles,
                                        device=dev)
    return out


def bootstrap_distributed(ds, model: str, penalty: str, strength: float, coefficient: int = 0,
                          resamples: int = 200, seed: int = 0, tol: float = 1e-6,
                          max_cycles: int = 1000, device: Optional[int] = None,
                          draw_runner=None):
    """bootstrap_interval (src/crossval.cpp:218-257) with the resamples dealt
    round-robin over ranks (each rank's fits batched on its GPU), draws
    gathered and merged in resample order: the interval equals the
    single-process one for any world size."""
    dist, rank, world = _dist()
    import survscan
    if resamples < 100:
        raise ValueError("bootstrap needs at least 100 resamples")
    dev = local_device() if device is None else device
    mine = shard_tasks(resamples, rank, world)
    if draw_runner is None:
        def draw_runner(ids):
            return list(survscan.bootstrap_run(ds, model, penalty, strength, [], coefficient,
                                               list(ids), seed, tol, max_cycles, [dev]))
    local, err = [], None
    try:
        local = list(zip(mine, draw_runner(mine)))
    except Exception as exc:  # noqa: BLE001
        err = f"{type(exc).__name__}: {exc}"
    parts = _gather_checked(dist, world, local, err)
    draws = [None] * resamples
    for part in parts:
        for b, v in part:
            draws[b] = v
    return survscan.bootstrap_merge(draws, resamples)
