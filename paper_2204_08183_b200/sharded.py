"""Config C5: one Cox/Fine-Gray fit over patients sharded across GPUs.

The rows of the global (stratum, time desc, row id) order are cut into
contiguous shards at tied-block boundaries, one shard per rank (one process
per GPU, torch.distributed).  The reverse-time scan is a prefix over ALL
patients, so every coordinate has one real exchange step:

  1. each shard's aggregate for column j (fwd tail of (e, e*x, e*x^2), the
     Fine-Gray u-weighted head, stratum flags) — gss_shard_aggregate;
  2. all-gather; each rank composes its carry as the segmented prefix of the
     earlier shards' tails (and suffix of the later shards' heads);
  3. the fused scan of its shard with that carry -> (grad_sum, hess_sum) —
     gss_shard_sums;
  4. all-gather the sums, add them in RANK order (identical bits everywhere),
     Engine::finish + coordinate_step (src/ccd.cpp:71-129) on every rank, the
     sparse update on every shard (validate-before-mutate OR-ed over ranks).

The driver is written over "local shards" + an all-gather, so the same code
runs with one shard per rank (`TorchExchange`) or with every shard in one
process on one GPU (`LocalExchange`) — the latter is how the protocol is
tested against the unsharded fit here.
"""
from __future__ import annotations

import math
from typing import List, Sequence

import numpy as np

from . import capi


class LocalExchange:
    """All shards live in this process: the all-gather is a stack."""
    def __init__(self, world: int):
        self.world = world
        self.ranks = list(range(world))

    def allgather(self, local_rows: Sequence[np.ndarray]) -> np.ndarray:
        return np.stack([np.asarray(r, np.float64) for r in local_rows])


class TorchExchange:
    """One shard per rank; torch.distributed all_gather (NCCL or gloo)."""
    def __init__(self, device=None):
        import torch
        import torch.distributed as dist
        self.dist, self.torch = dist, torch
        self.world = dist.get_world_size()
        self.ranks = [dist.get_rank()]
        self.device = device if device is not None else (
            torch.device("cuda", torch.cuda.current_device())
            if dist.get_backend() == "nccl" else torch.device("cpu"))

    def allgather(self, local_rows: Sequence[np.ndarray]) -> np.ndarray:
        t = self.torch.as_tensor(np.asarray(local_rows[0], np.float64), device=self.device)
        parts = [self.torch.empty_like(t) for _ in range(self.world)]
        self.dist.all_gather(parts, t)
        return np.stack([p.cpu().numpy() for p in parts])


def shard_bounds(times, stratum_start, world: int) -> List[int]:
    """Contiguous cuts of the sorted rows, moved forward to the next tied-block
    (or stratum) boundary so no tied block spans two shards."""
    n = len(times)
    cuts = [0]
    for r in range(1, world):
        c = max(cuts[-1], (n * r) // world)
        while 0 < c < n and times[c] == times[c - 1] and not (
                stratum_start is not None and stratum_start[c]):
            c += 1
        cuts.append(c)
    cuts.append(n)
    return cuts


def shard_dataset(ds, lo: int, hi: int, device: int):
    """capi.Dataset of sorted rows [lo, hi) of `ds` (an oracle.Sorted-like
    host layout: times, status, col_ptr, row_idx, vals, stratum_start)."""
    p = len(ds.col_ptr) - 1
    cols, rows, vals = [], [], []
    cp = [0]
    for j in range(p):
        a, b = ds.col_ptr[j], ds.col_ptr[j + 1]
        r = ds.row_idx[a:b]
        keep = (r >= lo) & (r < hi)
        rows.append(r[keep] - lo)
        vals.append(ds.vals[a:b][keep] if ds.vals is not None else np.ones(keep.sum()))
        cp.append(cp[-1] + int(keep.sum()))
    ss = np.zeros(hi - lo, np.uint8)
    if ds.stratum_start is not None:
        ss[:] = ds.stratum_start[lo:hi]
    ss[0] = 1 if lo == 0 else (ds.stratum_start[lo] if ds.stratum_start is not None else 0)
    return capi.Dataset(ds.times[lo:hi], ds.status[lo:hi], np.asarray(cp, np.int64),
                        np.concatenate(rows).astype(np.int32) if rows else np.zeros(0, np.int32),
                        np.concatenate(vals) if vals else None, ds.col_indicator, ss, device)


def _carries(aggs: np.ndarray, world: int) -> np.ndarray:
    """Per shard r: fwd carry = segmented sum of the tails of shards r* .. r-1
    (r* = last earlier shard holding a stratum start), rev carry = heads of
    shards r+1 .. r** (r** = first later shard holding a stratum start)."""
    out = np.zeros((world, 8))
    for r in range(world):
        f = np.zeros(3)
        start = 0
        for q in range(r - 1, -1, -1):
            if aggs[q][0] != 0.0:
                start = q
                break
        for q in range(start, r):
            f = f + aggs[q][1:4]
        rv = np.zeros(3)
        end = world - 1
        for q in range(r + 1, world):
            if aggs[q][0] != 0.0:
                end = q
                break
        for q in range(r + 1, end + 1):
            rv = rv + aggs[q][4:7]
        out[r, 0:3] = f
        out[r, 4:7] = rv
    return out


class ShardedFit:
    """fit_with_engine (src/ccd.cpp:131-184) over patient shards."""

    def __init__(self, ds, model: str, exchange, device: int = 0, recompute_interval: int = 100,
                 engine_factory=None):
        self.x = exchange
        self.world = exchange.world
        self.bounds = shard_bounds(ds.times, ds.stratum_start, self.world)
        if any(self.bounds[r + 1] <= self.bounds[r] for r in range(self.world)):
            # the same error on every rank before any collective (no rank waits)
            raise ValueError(f"cannot cut {len(ds.times)} rows into {self.world} non-empty "
                             f"shards at tied-block boundaries: {self.bounds}")
        self.p = len(ds.col_ptr) - 1
        self.engines, self._ds = [], []
        for r in exchange.ranks:
            lo, hi = self.bounds[r], self.bounds[r + 1]
            if engine_factory is not None:  # test stand-in for the device engine
                self.engines.append(engine_factory(ds, lo, hi))
                continue
            d = shard_dataset(ds, lo, hi, device)
            self._ds.append(d)
            self.engines.append(capi.Engine(d, model, recompute_interval))
        # delta' X_j over all patients: shard sums added in rank order
        self.fixed = self.x.allgather([e.fixed_terms() for e in self.engines]).sum(axis=0)

    # one exchange round: aggregates -> carries -> shard sums -> rank-ordered totals
    def _sums(self, column: int):
        aggs = self.x.allgather([e.shard_aggregate(column) for e in self.engines])
        car = _carries(aggs, self.world)
        local = [np.array(e.shard_sums(column, car[r]))
                 for e, r in zip(self.engines, self.x.ranks)]
        tot = self.x.allgather(local)
        s0 = s1 = 0.0
        for r in range(self.world):
            s0 += tot[r][0]
            s1 += tot[r][1]
        return s0, s1

    def grad_hessian(self, j: int):
        s0, s1 = self._sums(j)
        g = self.fixed[j] - s0
        h = min(-s1, 0.0) if not math.isnan(s1) else -s1
        return {"gradient": g, "hessian": h, "fixed_term": self.fixed[j]}

    def log_likelihood(self) -> float:
        s0, s1 = self._sums(-1)
        return s0 - s1

    def load_beta(self, beta):
        for e in self.engines:
            e.load_beta(beta)

    def fit(self, penalty="none", strength=0.0, tol=1e-6, max_cycles=1000, trust_init=1.0):
        import survscan
        p = self.p
        beta = np.zeros(p)
        hw = np.full(p, trust_init)
        self.load_beta(beta)
        pen = penalty != "none"

        def objective():
            ll = self.log_likelihood()
            if penalty == "l1":
                return ll - sum(strength * abs(b) for b in beta)
            if penalty == "l2":
                return ll - sum(b * b / (2.0 * strength) for b in beta)
            return ll

        prev = objective()
        trace, cycles, converged, skipped, violations = [prev], 0, p == 0, 0, 0
        while not converged and cycles < max_cycles:
            for j in range(p):
                gh = self.grad_hessian(j)
                nb, applied, nhw, skip = survscan.coordinate_step(
                    beta[j], gh["gradient"], gh["hessian"], penalty, strength, pen, hw[j])
                if skip:
                    skipped += 1
                    continue
                hw[j] = nhw
                if applied != 0.0:
                    over = self.x.allgather([np.array([float(e.update_validate(j, applied))])
                                             for e in self.engines])
                    if over.max() > 0:
                        raise capi.GssError(8, f"update: |x'beta| would exceed 700 (column {j})")
                    for e in self.engines:
                        e.update(j, applied)
                    beta[j] = nb
            cycles += 1
            obj = objective()
            trace.append(obj)
            if obj < prev - 1e-10:
                violations += 1
            if abs(obj - prev) / max(1.0, abs(obj)) < tol:
                converged = True
            prev = obj
        return {"beta": beta, "objective": prev, "cycles": cycles, "converged": converged,
                "objective_trace": np.array(trace), "skipped_steps": skipped,
                "monotonicity_violations": violations,
                "nonzero_count": int(np.count_nonzero(beta)), "shards": self.bounds}


# ---------------------------------------------------------------------------
# In-kernel exchange (gss_comm): the shards' cycle kernels exchange their
# aggregates over peer memory after every grid exchange, so the whole CCD fit
# runs on the device with the C++ host loop (gss_engine_fit per rank, or
# gss_sharded_fit_local for every shard of this process) — no host step per
# coordinate, no collective calls on the data path.
# ---------------------------------------------------------------------------
def shard_engines(ds, world: int, device: int = 0, ranks=None, recompute_interval: int = 100):
    """Engines over the contiguous row shards of `ds` (shard_bounds cuts)."""
    bounds = shard_bounds(ds.times, ds.stratum_start, world)
    if any(bounds[r + 1] <= bounds[r] for r in range(world)):
        raise ValueError(f"cannot cut {len(ds.times)} rows into {world} non-empty shards at "
                         f"tied-block boundaries: {bounds}")
    ranks = range(world) if ranks is None else ranks
    out = []
    for r in ranks:
        d = shard_dataset(ds, bounds[r], bounds[r + 1], device)
        e = capi.Engine(d, "cox", recompute_interval)
        e._ds_keep = d
        out.append(e)
    return out, bounds


def fit_in_kernel_local(ds, world: int, device: int = 0, penalty="l1", strength=0.0, tol=1e-6,
                        max_cycles=1000, recompute_interval: int = 100):
    """Config C5 emulated in one process: `world` shards on one GPU, one
    batched launch per cycle, cross-shard exchange inside the kernel."""
    engines, bounds = shard_engines(ds, world, device, recompute_interval=recompute_interval)
    capi.comm_local(engines)
    r = capi.sharded_fit_local(engines, penalty, strength, tol, max_cycles)
    r["shards"] = bounds
    return r


def fit_in_kernel_distributed(ds, penalty="l1", strength=0.0, tol=1e-6, max_cycles=1000,
                              device=None, recompute_interval: int = 100, grid: int = 0):
    """Config C5, one process per GPU (torchrun; any torch.distributed
    backend): rank r fits shard r.  The ranks all-gather their CUDA-IPC
    exchange-buffer handles and fixed terms with torch.distributed (no NCCL
    needed), then the exchange runs over peer memory inside the kernels."""
    import torch.distributed as dist
    world, rank = dist.get_world_size(), dist.get_rank()
    dev = device if device is not None else __import__("torch").cuda.current_device()
    comm = capi.comm_create(world, rank, dev)
    handles = [None] * world
    dist.all_gather_object(handles, capi.comm_ipc_handle(comm))
    capi.comm_connect(comm, handles)
    (eng,), bounds = shard_engines(ds, world, dev, ranks=[rank],
                                   recompute_interval=recompute_interval)
    if grid:
        eng.set_grid(grid)
    eng.attach_comm(comm)
    fixed, cmax = [None] * world, [None] * world
    dist.all_gather_object(fixed, eng.fixed_terms())
    dist.all_gather_object(cmax, eng.colmax())
    eng.set_fixed_terms(np.sum(np.stack(fixed), axis=0))  # rank-order sum (numpy: sequential)
    eng.set_colmax(np.max(np.stack(cmax), axis=0))  # one overflow bound on every shard
    dist.barrier()
    r = eng.fit(penalty=penalty, strength=strength, tol=tol, max_cycles=max_cycles)
    r["shards"] = bounds
    return r
