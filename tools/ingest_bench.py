"""Ingestion (dataset_from_coo) time: device radix sorts (gss_coo_sort) vs the
host comparison sort, same data, N rows x p columns at `density`, ties and
strata.  Writes one JSON line.

    python tools/ingest_bench.py --n 10000000 --p 100 --density 0.01
"""
import argparse
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import survscan  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=10_000_000)
ap.add_argument("--p", type=int, default=100)
ap.add_argument("--density", type=float, default=0.01)
ap.add_argument("--strata", type=int, default=100)
a = ap.parse_args()
rng = np.random.default_rng(0)
t = np.ceil(rng.exponential(size=a.n) * 1000) / 1000
s = (rng.random(a.n) < 0.8).astype(np.int64)
k = int(a.n * a.p * a.density)
rows = rng.integers(0, a.n, k)
cols = rng.integers(0, a.p, k)
key = np.unique(cols * a.n + rows)
rng.shuffle(key)
rows, cols = (key % a.n).astype(np.int64), (key // a.n).astype(np.int64)
vals = np.ones(len(key))
st = rng.integers(0, a.strata, a.n) if a.strata > 1 else None
out = {"n": a.n, "p": a.p, "nnz": int(len(key)), "strata": a.strata}
survscan.dataset_from_coo(t[:1000], s[:1000], rows[:0], cols[:0], vals[:0], a.p)  # context
for mode in ("device", "host"):
    if mode == "host":
        os.environ["SURVSCAN_HOST_INGEST"] = "1"
    t0 = time.perf_counter()
    ds = survscan.dataset_from_coo(t, s, rows, cols, vals, a.p, st)
    out[mode + "_seconds"] = round(time.perf_counter() - t0, 3)
    out[mode + "_hash"] = ds.content_hash
out["identical"] = out["device_hash"] == out["host_hash"]
out["speedup"] = round(out["host_seconds"] / out["device_seconds"], 2)
print(json.dumps(out))
