"""Per-phase wall time of gss_dataset_pack at the C2 size (GSS_PACK_TIMING)."""
import os
import sys
import time

os.environ["GSS_PACK_TIMING"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2204_08183_b200 import capi  # noqa: E402

sim = capi.SimData(10_000_000, 5000, 0.01, 0.8, 2, 0.9, 1000.0)
for _ in range(3):
    t0 = time.perf_counter()
    d = capi.Dataset(sim.times, sim.status, sim.col_ptr, sim.row_idx)
    print("pack total s", round(time.perf_counter() - t0, 3), file=sys.stderr, flush=True)
    del d
