"""Profiling driver for the sweep kernel (run under ncu on the GPU box).

    python tools/prof_sweep.py --n 10000000 --p 64 --mode fit --cycles 2
    python tools/prof_sweep.py --mode api --reps 20      # grad_hessian only (no updates)
"""
import argparse
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2204_08183_b200 import capi  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=10_000_000)
ap.add_argument("--p", type=int, default=64)
ap.add_argument("--density", type=float, default=0.01)
ap.add_argument("--mode", default="fit", choices=["fit", "api"])
ap.add_argument("--cycles", type=int, default=2)
ap.add_argument("--reps", type=int, default=20)
ap.add_argument("--strength", type=float, default=2 ** 0.5)
ap.add_argument("--interval", type=int, default=100)
ap.add_argument("--model", default="cox", choices=["cox", "finegray"])
a = ap.parse_args()

sim = capi.SimData(a.n, a.p, a.density, 0.8, 2, 0.9, 1000.0,
                   p_mix=0.5 if a.model == "finegray" else 0.0)
ds = capi.Dataset(sim.times, sim.status, sim.col_ptr, sim.row_idx)
eng = capi.Engine(ds, a.model, recompute_interval=a.interval)
if a.mode == "fit":
    t0 = time.perf_counter()
    r = eng.fit(penalty="l1", strength=a.strength, tol=1e-300, max_cycles=a.cycles)
    ms, acc = eng.cycle_stats()
    print("cycles", r["cycles"], "cycle_ms", ms.round(3).tolist(), "accepted", acc.tolist(),
          "wall", round(time.perf_counter() - t0, 3))
    print("per-coordinate us", (ms / (a.p + 1) * 1e3).round(2).tolist())
else:
    for j in range(a.reps):
        eng.grad_hessian(j % a.p)
    t0 = time.perf_counter()
    for j in range(a.reps):
        eng.grad_hessian(j % a.p)
    dt = (time.perf_counter() - t0) / a.reps
    print("api grad_hessian wall us/call", round(dt * 1e6, 2))
