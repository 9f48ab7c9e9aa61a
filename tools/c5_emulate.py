"""Config C5 protocol cost on one GPU: S patient shards emulated in one
process (each shard its own engine on 148/S CTAs, all in one batched launch
per cycle, cross-shard exchange inside the kernel: gss_comm_local +
gss_sharded_fit_local) against one unsharded engine with the same rows per
"GPU" (one shard's rows on 148/S CTAs).  Per-coordinate device time.

    python tools/c5_emulate.py --rows-per-shard 2000000 --p 64 --shards 2 4
"""
import argparse
import json
import os
import sys
import types

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2204_08183_b200 import capi, sharded  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--rows-per-shard", type=int, default=2_000_000)
ap.add_argument("--p", type=int, default=64)
ap.add_argument("--shards", type=int, nargs="+", default=[2, 4])
ap.add_argument("--cycles", type=int, default=3)
a = ap.parse_args()
out = {"rows_per_shard": a.rows_per_shard, "p": a.p, "cycles": a.cycles, "runs": []}
for S in a.shards:
    n = a.rows_per_shard * S
    sim = capi.SimData(n, a.p, 0.01, 0.8, 11, 0.9, 1000.0)
    ds = types.SimpleNamespace(times=np.asarray(sim.times), status=np.asarray(sim.status),
                               col_ptr=np.asarray(sim.col_ptr), row_idx=np.asarray(sim.row_idx),
                               vals=None, stratum_start=None,
                               col_indicator=np.ones(a.p, np.uint8))
    engines, bounds = sharded.shard_engines(ds, S)
    capi.comm_local(engines)
    r = capi.sharded_fit_local(engines, "l1", 2 ** 0.5, 1e-300, a.cycles)
    sh_us = r["device_seconds"] / (r["cycles"] * (a.p + 1)) * 1e6
    grid = max(1, 148 // S)
    # unsharded reference at equal rows per GPU: shard 0's rows on the same CTA count
    d0 = sharded.shard_dataset(ds, bounds[0], bounds[1], 0)
    e0 = capi.Engine(d0, "cox").set_grid(grid)
    r0 = e0.fit(penalty="l1", strength=2 ** 0.5, tol=1e-300, max_cycles=a.cycles)
    one_us = r0["device_seconds"] / (r0["cycles"] * (a.p + 1)) * 1e6
    # and the same total rows unsharded on the whole GPU
    dall = capi.Dataset(sim.times, sim.status, sim.col_ptr, sim.row_idx)
    rall = capi.Engine(dall, "cox").fit(penalty="l1", strength=2 ** 0.5, tol=1e-300,
                                         max_cycles=a.cycles)
    all_us = rall["device_seconds"] / (rall["cycles"] * (a.p + 1)) * 1e6
    out["runs"].append({"shards": S, "ctas_per_shard": grid, "rows_total": n,
                        "unsharded_us_per_coordinate_same_total_rows": round(all_us, 2),
                        "ratio_same_total": round(sh_us / all_us, 3),
                        "sharded_us_per_coordinate": round(sh_us, 2),
                        "unsharded_us_per_coordinate_same_rows_per_gpu": round(one_us, 2),
                        "ratio": round(sh_us / one_us, 3)})
    print(json.dumps(out["runs"][-1]), flush=True)
print(json.dumps(out))
