"""Event-trace analysis of one sweep launch (needs GSS_TRACE=1 at engine creation).

    GSS_TRACE=1 python tools/trace_sweep.py --n 10000000 --p 16
Events: 0 kernel start, 1 claim, 2 full armed, 3 agg start, 4 A published,
5 look-back start, 6 prefix ready, 7 consumer full seen, 8 agg seen,
9 prefix seen, 10 tile done, 11 ticket, 12 tail done.
"""
import argparse
import ctypes
import os
import sys

import numpy as np

os.environ["GSS_TRACE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2204_08183_b200 import capi  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=10_000_000)
ap.add_argument("--p", type=int, default=16)
a = ap.parse_args()

sim = capi.SimData(a.n, a.p, 0.01, 0.8, 2, 0.9, 1000.0)
ds = capi.Dataset(sim.times, sim.status, sim.col_ptr, sim.row_idx)
eng = capi.Engine(ds, "cox")
L = capi.lib()
L.gss_engine_trace.restype = ctypes.c_int64
buf = np.zeros(2 * (1 << 22), np.uint64)
for rep in range(3):
    L.gss_engine_trace(eng.h, buf.ctypes.data_as(ctypes.c_void_p), ctypes.c_int64(0))
    eng.grad_hessian(rep % a.p)
    k = L.gss_engine_trace(eng.h, buf.ctypes.data_as(ctypes.c_void_p), ctypes.c_int64(1 << 22))
ev = buf[:2 * k].reshape(-1, 2)
ts = ev[:, 0].astype(np.int64)
meta = ev[:, 1]
cta = (meta >> np.uint64(40)).astype(np.int64)
kind = ((meta >> np.uint64(32)) & np.uint64(0xff)).astype(np.int64)
tile = (meta & np.uint64(0xffffffff)).astype(np.int64)
t0 = ts.min()
ts = (ts - t0) / 1000.0  # us
print(f"events {k}, span {ts.max():.1f} us")
for e in range(13):
    m = kind == e
    if m.any():
        print(f"ev{e:2d}: n={m.sum():6d} first={ts[m].min():8.2f} last={ts[m].max():8.2f}")
# per-tile intervals
def per_tile(e):
    m = kind == e
    d = {}
    for tt, tv in zip(tile[m], ts[m]):
        d.setdefault(int(tt), tv)
    return d
P = {e: per_tile(e) for e in (2, 3, 7, 9, 10)}
def gap(e1, e2, label):
    common = sorted(set(P[e1]) & set(P[e2]))
    if not common:
        return
    g = np.array([P[e2][t] - P[e1][t] for t in common])
    print(f"{label:28s} median {np.median(g):7.2f} p90 {np.percentile(g, 90):7.2f} max {g.max():8.2f} us")
gap(2, 3, "phase-A item")
gap(7, 9, "consumer full -> prefix")
gap(9, 10, "prefix -> tile done")
gap(7, 10, "consumer tile total")
for e in (4, 5):
    m = kind == e
    if m.any():
        print("ev", e, ts[m].min())
# consumer busy per CTA
m = kind == 10
tiles_per_cta = np.bincount(cta[m])
print("tiles per CTA: max", tiles_per_cta.max())
# time profile of claims
c = np.sort(ts[kind == 2])
print("item start times quantiles (us):", np.percentile(c, [0, 10, 50, 90, 100]).round(1).tolist())
d = np.sort(ts[kind == 10])
print("tile-done quantiles (us):", np.percentile(d, [0, 10, 50, 90, 100]).round(1).tolist())
d3 = np.sort(ts[kind == 3])
print("item-done quantiles (us):", np.percentile(d3, [0, 10, 50, 90, 99, 100]).round(1).tolist())
d7 = np.sort(ts[kind == 7])
print("consumer-first-seen quantiles (us):", np.percentile(d7, [0, 10, 50, 90, 100]).round(1).tolist())
