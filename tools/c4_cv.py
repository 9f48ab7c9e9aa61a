"""Config C4 measurement: stratified Cox, 10-fold CV x 20-point lambda grid,
N=1e6, p=1000, 1% binary, K=100 strata, through the drop-in survscan API
(device row-mask folds, batched multi-fit launches).  Used by bench.py
(secondary.c4_cv) and runnable alone:

    python tools/c4_cv.py [--n 1000000 --p 1000 --grid 20 --folds 10]
"""
from __future__ import annotations

import argparse
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def strata_of(n: int, k: int, seed: int = 7) -> np.ndarray:
    """stratum = splitmix64(seed ^ row_id) mod k (a fixed hash of the row id)."""
    x = (np.arange(n, dtype=np.uint64) ^ np.uint64(seed)) + np.uint64(0x9E3779B97F4A7C15)
    x = (x ^ (x >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
    x = (x ^ (x >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    x = x ^ (x >> np.uint64(31))
    return (x % np.uint64(k)).astype(np.int64)


def c4_dataset(n: int, p: int, strata: int, seed: int = 4, device: int = 0):
    """The C4 design (device generator, simulate_cox family, ties q=1e-3,
    administrative censoring at the 0.9 quantile) as a survscan.Dataset."""
    import survscan
    from paper_2204_08183_b200 import capi
    sim = capi.SimData(n, p, 0.01, 0.8, seed, 0.9, 1000.0, device=device)
    cols = np.repeat(np.arange(p, dtype=np.int64), np.diff(sim.col_ptr))
    rows = np.asarray(sim.row_idx, np.int64)
    return survscan.dataset_from_coo(np.asarray(sim.times), np.asarray(sim.status, np.int64),
                                     rows, cols, np.ones(len(rows)), p,
                                     strata_of(n, strata) if strata > 1 else None)


def run(n=1_000_000, p=1000, strata=100, grid_points=20, folds=10, seed=7, device=0,
        barrier=None, reduce_max=None):
    """Time-to-result of the whole C4 job on this rank set (torch.distributed
    when initialised: tasks dealt over ranks, one GPU per rank)."""
    import survscan
    from paper_2204_08183_b200 import distributed as D
    t0 = time.perf_counter()
    ds = c4_dataset(n, p, strata, device=device)
    build_s = time.perf_counter() - t0
    gmax = survscan.gamma_max(ds, "cox")
    grid = list(np.geomspace(gmax, gmax / 1000.0, grid_points))
    if barrier:
        barrier()
    t0 = time.perf_counter()
    res = D.cross_validate_distributed(ds, "cox", "l1", grid, folds=folds, repetitions=1,
                                       seed=seed, tol=1e-6, max_cycles=1000, device=device,
                                       final_fit=True)
    wall = time.perf_counter() - t0
    if reduce_max:
        wall = reduce_max(wall)
    ff = res["final_fit"]
    return {"workload": f"C4: stratified Cox ({strata} strata), {folds}-fold CV x "
                        f"{grid_points}-point L1 grid [gamma_max/1000, gamma_max], N={n}, "
                        f"p={p}, 1% binary, + final refit",
            "time_to_result_s": round(wall, 3), "dataset_build_s": round(build_s, 3),
            "fold_fits": grid_points * folds, "heldout_evaluations": grid_points * folds,
            "gamma_max": gmax, "selected": res["selected"],
            "final_fit_cycles": int(ff["cycles"]), "final_fit_nonzero": int(ff["nonzero_count"]),
            "tasks_per_rank": res.get("tasks_per_rank"),
            "path": "survscan.cross_validate pieces (cv_run_tasks: device row-mask folds, batched "
                    "multi-fit launches) dealt over ranks by distributed.cross_validate_distributed"}


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=1_000_000)
    ap.add_argument("--p", type=int, default=1000)
    ap.add_argument("--strata", type=int, default=100)
    ap.add_argument("--grid", type=int, default=20)
    ap.add_argument("--folds", type=int, default=10)
    a = ap.parse_args()
    import json
    print(json.dumps(run(a.n, a.p, a.strata, a.grid, a.folds)))
