"""Config C5 at full size on ONE B200: N = 1e8 patients, p = 1e4 columns at
0.1% density (1e9 nonzeros; SURVEY.md §8d allows 0.1% for C5), cut into
`--shards` patient shards (12.5M rows each for 8) that run as one batched
launch per CCD cycle with the cross-shard exchange inside the kernel.  Each
shard is generated on the device independently; shard r's event times are
offset above shard r+1's, so the global (time desc) order is the rank order.
Reports per-coordinate device time and the objective.

    python tools/c5_full_emulated.py --shards 8 --rows-per-shard 12500000 --p 10000
"""
import argparse
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2204_08183_b200 import capi  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--shards", type=int, default=8)
ap.add_argument("--rows-per-shard", type=int, default=12_500_000)
ap.add_argument("--p", type=int, default=10_000)
ap.add_argument("--density", type=float, default=0.001)
ap.add_argument("--cycles", type=int, default=2)
ap.add_argument("--unsharded", action="store_true", help="one engine over all rows instead")
a = ap.parse_args()
S = a.shards
if a.unsharded:
    rows = S * a.rows_per_shard
    t0 = time.perf_counter()
    sim = capi.SimData(rows, a.p, a.density, 0.8, 1000, 0.9, 1000.0)
    d = capi.Dataset(sim.times, sim.status, sim.col_ptr, sim.row_idx)
    nnz = int(sim.nnz)
    del sim
    e = capi.Engine(d, "cox")
    build = time.perf_counter() - t0
    r = e.fit(penalty="l1", strength=2 ** 0.5, tol=1e-300, max_cycles=a.cycles)
    us = r["device_seconds"] / (r["cycles"] * (a.p + 1)) * 1e6
    print(json.dumps({"workload": f"unsharded on one B200: N={rows}, p={a.p}, density {a.density}, "
                                  f"{nnz} nonzeros", "build_seconds": round(build, 1),
                      "cycles": r["cycles"], "device_seconds": round(r["device_seconds"], 3),
                      "us_per_coordinate": round(us, 1),
                      "algorithmic_GBps": round((12.0 * rows + 4.0 * nnz / a.p) / (us * 1e-6) / 1e9, 1)}))
    sys.exit(0)
t0 = time.perf_counter()
engines, datasets, nnz = [], [], 0
for r in range(S):
    sim = capi.SimData(a.rows_per_shard, a.p, a.density, 0.8, 1000 + r, 0.9, 1000.0)
    t = np.asarray(sim.times) + float(S - 1 - r) * 1.0e6
    d = capi.Dataset(t, sim.status, sim.col_ptr, sim.row_idx)
    nnz += int(sim.nnz)
    del sim
    datasets.append(d)
    engines.append(capi.Engine(d, "cox"))
build = time.perf_counter() - t0
capi.comm_local(engines)
t0 = time.perf_counter()
r = capi.sharded_fit_local(engines, "l1", 2 ** 0.5, 1e-300, a.cycles)
wall = time.perf_counter() - t0
us = r["device_seconds"] / (r["cycles"] * (a.p + 1)) * 1e6
rows = S * a.rows_per_shard
print(json.dumps({"workload": f"C5 on one B200: N={rows}, p={a.p}, density {a.density}, "
                              f"{nnz} nonzeros, {S} patient shards x {148 // S} CTAs in one "
                              f"batched launch per cycle, in-kernel cross-shard exchange",
                  "build_seconds": round(build, 1), "cycles": r["cycles"],
                  "device_seconds": round(r["device_seconds"], 3), "wall_seconds": round(wall, 3),
                  "us_per_coordinate": round(us, 1),
                  "algorithmic_GBps": round((12.0 * rows + 4.0 * nnz / a.p) / (us * 1e-6) / 1e9, 1),
                  "objective": r["objective"], "nonzero": r["nonzero_count"]}))
