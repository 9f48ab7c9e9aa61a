"""Per-tile processing cost (cycles from stage-ready to tile end, consumer
group thread 0) of one CCD slot in the middle of a cycle, against the tile's
features (event block ends, transform passes, column list sizes).
Needs the trace build: GSS_TRACE_BUILD=1 python -m paper_2204_08183_b200.build
then GSS_TRACE=1 GSS_DEBUG=524288 python tools/tile_cost_probe.py"""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2204_08183_b200 import capi  # noqa: E402

n, p = 10_000_000, 512
sim = capi.SimData(n, p, 0.01, 0.8, 2, 0.9, 1000.0)
ds = capi.Dataset(sim.times, sim.status, sim.col_ptr, sim.row_idx)
eng = capi.Engine(ds, "cox")
L = capi.lib()
import ctypes  # noqa: E402
L.gss_engine_trace.restype = ctypes.c_int64
eng.fit(penalty="l1", strength=2 ** 0.5, tol=1e-300, max_cycles=1)
nt = (n + 2047) // 2048
buf = np.zeros(2 * (32 << 16), np.uint64)
L.gss_engine_trace(eng.h, buf.ctypes.data_as(ctypes.c_void_p), ctypes.c_int64(32 << 16))
cost = buf[:nt].astype(np.float64)
# features from the host data (sorted order == device order without strata)
t = np.asarray(sim.times)
st = np.asarray(sim.status)
ends = np.zeros(n, bool)
ends[:-1] = t[:-1] != t[1:]
ends[-1] = True
ev_end = np.zeros(n, np.int64)
# event count at block ends
blk = np.cumsum(np.r_[0, ends[:-1]])
evc = np.bincount(blk, weights=(st == 1).astype(float))
ev_end[ends] = evc[blk[ends]] > 0
tile = np.arange(n) // 2048
be = np.bincount(tile, weights=ev_end, minlength=nt)
ok = cost > 0
X = np.c_[np.ones(ok.sum()), be[ok]]
coef, *_ = np.linalg.lstsq(X, cost[ok], rcond=None)
r = np.corrcoef(be[ok], cost[ok])[0, 1]
q = np.quantile(cost[ok], [0.1, 0.5, 0.9])
print(json.dumps({"tiles": int(ok.sum()), "cost_cycles_p10_p50_p90": q.round(0).tolist(),
                  "fit_cycles": {"intercept": round(coef[0], 1), "per_event_block_end": round(coef[1], 2)},
                  "corr_cost_block_ends": round(float(r), 3),
                  "by_region": [[int(a), round(float(cost[ok][(np.nonzero(ok)[0] >= a) & (np.nonzero(ok)[0] < a + nt // 10)].mean()), 0),
                                 round(float(be[a:a + nt // 10].mean()), 1)] for a in range(0, nt, nt // 10)]}))
