"""Batched multi-fit throughput probe (C4-like): K fold fits at N rows, p
columns, alone vs batched (gss_fit_batch), device time."""
import argparse
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2204_08183_b200 import capi  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=1_000_000)
ap.add_argument("--p", type=int, default=1000)
ap.add_argument("--fits", type=int, default=48)
ap.add_argument("--active", type=int, default=0)
ap.add_argument("--alone", type=int, default=2)
ap.add_argument("--max-cycles", type=int, default=4)
a = ap.parse_args()
sim = capi.SimData(a.n, a.p, 0.01, 0.8, 4, 0.9, 1000.0)
ds = capi.Dataset(sim.times, sim.status, sim.col_ptr, sim.row_idx)
rng = np.random.default_rng(1)
fold = rng.permutation(a.n) % 10
lams = np.geomspace(1.0, 100.0, 20)
specs = [((fold != (i % 10)).astype(np.uint8), lams[i % 20]) for i in range(a.fits)]
t0 = time.perf_counter()
engines = [capi.Engine(ds, "cox", row_mask=m) for m, _ in specs]
print("create %.3f s" % (time.perf_counter() - t0))
coords = 0
t0 = time.perf_counter()
res, dev = capi.fit_batch(engines, "l1", [g for _, g in specs], tol=1e-300,
                          max_cycles=a.max_cycles, max_active=a.active)
wall = time.perf_counter() - t0
coords = sum(r["cycles"] for r in res) * a.p
print("batched: %d fits x %d cycles: device %.3f s wall %.3f s -> %.0f coord/s (%.2f us/coord/fit)"
      % (a.fits, a.max_cycles, dev, wall, coords / dev, dev / coords * 1e6))
for i in range(a.alone):
    e = capi.Engine(ds, "cox", row_mask=specs[i][0])
    r = e.fit(penalty="l1", strength=specs[i][1], tol=1e-300, max_cycles=a.max_cycles)
    ms, _ = e.cycle_stats()
    c = r["cycles"] * a.p
    print("alone fit %d: device %.3f s -> %.0f coord/s (%.2f us/coord)" % (i, ms.sum() / 1e3,
          c / (ms.sum() / 1e3), ms.sum() / 1e3 / c * 1e6))
    same = res[i]
    print("   batched beta == alone(full grid)? max rel diff %.2e" %
          np.max(np.abs(same["beta"] - r["beta"]) / np.maximum(1, np.abs(r["beta"]))))
