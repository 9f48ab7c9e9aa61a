"""Config C5 multi-process path (one process per shard, CUDA-IPC peer buffers,
the exchange inside the kernels) checked against the unsharded fit.  Runs
under torchrun with any backend; several ranks may share one GPU when an MPS
daemon runs (each rank's grid is capped so the shards' kernels co-reside):

    torchrun --nproc-per-node 2 tools/c5_multiproc.py --same-gpu --grid 74
"""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

ap = argparse.ArgumentParser()
ap.add_argument("--same-gpu", action="store_true")
ap.add_argument("--grid", type=int, default=0)
ap.add_argument("--n", type=int, default=60_000)
ap.add_argument("--p", type=int, default=8)
ap.add_argument("--tol", type=float, default=1e-12)
ap.add_argument("--sim", type=int, default=0, help="rows of a device-generated C2-family dataset "
                "(timing mode: 3 cycles, per-coordinate device time)")
a = ap.parse_args()

import torch.distributed as dist  # noqa: E402

dist.init_process_group("gloo")
rank, world = dist.get_rank(), dist.get_world_size()
dev = 0 if a.same_gpu else int(os.environ.get("LOCAL_RANK", "0"))
from paper_2204_08183_b200 import capi, sharded  # noqa: E402
from tests.test_gpu_parity import _random_sorted  # noqa: E402

if a.sim:
    import types
    sim = capi.SimData(a.sim, a.p, 0.01, 0.8, 11, 0.9, 1000.0, device=dev)
    ds = types.SimpleNamespace(times=np.asarray(sim.times), status=np.asarray(sim.status),
                               col_ptr=np.asarray(sim.col_ptr), row_idx=np.asarray(sim.row_idx),
                               vals=None, stratum_start=None, col_indicator=np.ones(a.p, np.uint8))
    r = sharded.fit_in_kernel_distributed(ds, penalty="l1", strength=2 ** 0.5, tol=1e-300,
                                          max_cycles=3, device=dev, grid=a.grid)
    us = r["device_seconds"] / (r["cycles"] * (a.p + 1)) * 1e6
    sys.stdout.write(json.dumps({"rank": rank, "world": world, "rows_total": a.sim, "p": a.p,
                                 "grid": a.grid, "us_per_coordinate": round(us, 2),
                                 "objective": r["objective"]}) + "\n")
    sys.stdout.flush()
    dist.barrier()
    dist.destroy_process_group()
    sys.exit(0)
ds = _random_sorted(a.n, a.p, 0.05, seed=123, quant=40.0, strata=3)
r = sharded.fit_in_kernel_distributed(ds, penalty="l1", strength=1.5, tol=a.tol, max_cycles=8,
                                      device=dev, recompute_interval=7, grid=a.grid)
out = {"rank": rank, "world": world, "cycles": r["cycles"], "objective": r["objective"]}
if rank == 0:
    one = capi.Engine(capi.Dataset.from_sorted(ds, device=dev), "cox", 7).fit(
        penalty="l1", strength=1.5, tol=a.tol, max_cycles=8)
    err = float(np.max(np.abs(r["beta"] - one["beta"]) / np.maximum(1.0, np.abs(one["beta"]))))
    out.update({"unsharded_cycles": one["cycles"], "max_rel_err_beta": err,
                "pass": bool(err < 1e-8 and one["cycles"] == r["cycles"])})
# one write per line: ranks share the launcher's stdout pipe
sys.stdout.write(json.dumps(out) + "\n")
sys.stdout.flush()
dist.barrier()
dist.destroy_process_group()
