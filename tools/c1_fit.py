"""C1 (the reference's CPU-runnable case): N=1e5, p=1000, 1%
binary, no censoring, distinct times, L1 gamma=sqrt(2), tol 1e-6 — time to fit
on one B200 (device generator: same design family, own RNG stream).

    python tools/c1_fit.py [--out f.json]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2204_08183_b200 import capi  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--out", default="")
a = ap.parse_args()
sim = capi.SimData(100_000, 1000, 0.01, 0.8, 1, 0.0, 0.0)
ds = capi.Dataset(sim.times, sim.status, sim.col_ptr, sim.row_idx)
eng = capi.Engine(ds, "cox")
eng.fit(penalty="l1", strength=2 ** 0.5)  # warm-up (module load, first launch)
t0 = time.perf_counter()
r = eng.fit(penalty="l1", strength=2 ** 0.5)
wall = time.perf_counter() - t0
ms, _ = eng.cycle_stats()
res = {"config": "C1: N=1e5, p=1000, 1%, no censoring, L1 sqrt(2), tol 1e-6",
       "cycles": int(r["cycles"]), "wall_s": wall, "device_s": float(ms.sum()) * 1e-3,
       "us_per_coordinate": float(ms.sum()) * 1e3 / (r["cycles"] * 1001),
       "nonzero": int((r["beta"] != 0).sum())}
print(json.dumps(res))
if a.out:
    json.dump(res, open(a.out, "w"), indent=1)
