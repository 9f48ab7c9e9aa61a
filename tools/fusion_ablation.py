"""Acceptance check 5 of the reference (tests/acceptance.cpp:196-235) on the
device: the fused derivative pass (cycle kernel, API mode) against the
separated three-pass path (gss_separated.cu), values and speed.

    python tools/fusion_ablation.py --n 10000000 --p 20 [--model finegray] [--out f.json]

Timing is wall time around synchronous C-ABI calls (each call ends in a
stream synchronize), best of 2 sweeps over the p columns, like the
reference's check.
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
ap.add_argument("--n", type=int, default=10_000_000)
ap.add_argument("--p", type=int, default=20)
ap.add_argument("--density", type=float, default=0.05)
ap.add_argument("--model", default="cox", choices=["cox", "finegray"])
ap.add_argument("--out", default="")
a = ap.parse_args()

pmix = 0.5 if a.model == "finegray" else 0.0
sim = capi.SimData(a.n, a.p, a.density, 0.8, 9500, 0.85, 1000.0, p_mix=pmix)
ds = capi.Dataset(sim.times, sim.status, sim.col_ptr, sim.row_idx)
eng = capi.Engine(ds, a.model)
eng.load_beta(np.random.default_rng(1200).uniform(-0.2, 0.2, size=a.p))
worst = 0.0
for j in range(a.p):
    f, s = eng.grad_hessian(j), eng.grad_hessian_separated(j)
    for k in ("gradient", "hessian"):
        worst = max(worst, abs(f[k] - s[k]) / max(1.0, abs(f[k]), abs(s[k])))


def sweep(fused):
    t0 = time.perf_counter()
    for j in range(a.p):
        (eng.grad_hessian if fused else eng.grad_hessian_separated)(j)
    return time.perf_counter() - t0


sep = min(sweep(False), sweep(False))
fus = min(sweep(True), sweep(True))
res = {"check": "acceptance 5: fused vs separated", "model": a.model, "n": a.n, "p": a.p,
       "density": a.density, "max_rel": worst, "fused_s": fus, "separated_s": sep,
       "fused_us_per_call": fus / a.p * 1e6, "separated_us_per_call": sep / a.p * 1e6,
       "values_ok": worst <= 1e-12, "speed_ok": fus <= 1.10 * sep}
print(json.dumps(res))
if a.out:
    with open(a.out, "w") as fh:
        json.dump(res, fh, indent=1)
