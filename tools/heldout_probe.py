"""Cost of one held-out evaluation (C4 pieces): masked engine create,
load_beta, log_likelihood, destroy, at N = 1e6, p = 1000 (one thread)."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2204_08183_b200 import capi  # noqa: E402

n, p = 1_000_000, 1000
sim = capi.SimData(n, p, 0.01, 0.8, 2, 0.9, 1000.0)
ds = capi.Dataset(sim.times, sim.status, sim.col_ptr, sim.row_idx)
rng = np.random.default_rng(1)
beta = np.where(rng.random(p) < 0.1, rng.normal(size=p) * 0.05, 0.0)
L = capi.lib()
for rep in range(4):
    mask = (rng.integers(0, 10, n) == 3).astype(np.uint8)
    t0 = time.perf_counter()
    e = capi.Engine(ds, "cox", 100, row_mask=mask)
    t1 = time.perf_counter()
    e.load_beta(beta)
    t2 = time.perf_counter()
    ll = e.log_likelihood()
    t3 = time.perf_counter()
    L.gss_engine_destroy(e.h)
    e.h = None
    t4 = time.perf_counter()
    print(f"create {1e3*(t1-t0):.1f} ms  load_beta {1e3*(t2-t1):.1f}  loglik {1e3*(t3-t2):.1f}  "
          f"destroy {1e3*(t4-t3):.1f}  ll={ll:.6f}", flush=True)
