"""Cost of the round-1 patient-sharded (C5) protocol on one GPU.

Every shard is emulated in one process (LocalExchange), so the numbers show
the protocol's per-coordinate overhead (two launches + two all-gathers + the
host step per coordinate), not NVLink scaling:

    python tools/shard_protocol_bench.py --n 2000000 --p 16 --world 2 --out f.json

The unsharded engine's API grad_hessian on the same data is timed beside it.
"""
import argparse
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import oracle as orc  # noqa: E402  (test infrastructure: builds the sorted layout)
from paper_2204_08183_b200 import capi, sharded  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=2_000_000)
ap.add_argument("--p", type=int, default=16)
ap.add_argument("--density", type=float, default=0.01)
ap.add_argument("--world", type=int, default=2)
ap.add_argument("--out", default="")
a = ap.parse_args()

rng = np.random.default_rng(5)
k = rng.binomial(a.n, a.density, size=a.p)
rows = np.concatenate([rng.choice(a.n, size=c, replace=False) for c in k])
cols = np.repeat(np.arange(a.p), k)
t = np.ceil(rng.exponential(size=a.n) * 1000.0) / 1000.0
status = (rng.random(a.n) < 0.7).astype(np.int64)
ds = orc.assemble(t, status, rows, cols, np.ones(rows.size), a.p)

fitter = sharded.ShardedFit(ds, "cox", sharded.LocalExchange(a.world))
eng = capi.Engine(capi.Dataset.from_sorted(ds), "cox")
beta = np.linspace(-0.2, 0.2, a.p)
fitter.load_beta(beta)
eng.load_beta(beta)


def per_coord(f):
    for j in range(a.p):
        f(j)
    t0 = time.perf_counter()
    for j in range(a.p):
        f(j)
    return (time.perf_counter() - t0) / a.p * 1e6


sh = per_coord(fitter.grad_hessian)
un = per_coord(eng.grad_hessian)
res = {"config": "C5 protocol, shards emulated on one GPU", "n": a.n, "p": a.p,
       "density": a.density, "world": a.world,
       "sharded_us_per_coordinate": sh, "unsharded_api_us_per_coordinate": un,
       "note": "host-stepped protocol: shard aggregate launch + all-gather + shard sums "
               "launch + all-gather per coordinate; the in-kernel peer exchange is round-2 work"}
print(json.dumps(res))
if a.out:
    json.dump(res, open(a.out, "w"), indent=1)
