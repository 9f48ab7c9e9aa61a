"""Config C5's multi-process path without a GPU: the patient-sharded CCD
driver (paper_2204_08183_b200/sharded.py) over world_size-2 gloo ranks
(TorchExchange) must reproduce the unsharded oracle fit.  Each rank's shard
runs on `NumpyShard`, a dense numpy restatement of the two shard entry points
(test infrastructure standing in for the device engine's gss_shard_aggregate /
gss_shard_sums)."""
import os
import socket
import sys

import numpy as np
import pytest
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

from oracle import oracle as orc  # noqa: E402
from tests._common import TOL_BETA, TOL_DERIV, rel  # noqa: E402


def make_ds(seed=3, n=3000, p=5, strata=3):
    rng = np.random.default_rng(seed)
    rows, cols = [], []
    for j in range(p):
        r = rng.choice(n, size=rng.binomial(n, 0.1), replace=False)
        rows.append(r)
        cols.append(np.full(len(r), j))
    t = np.ceil(rng.exponential(size=n) * 30) / 30
    st = (rng.random(n) < 0.8).astype(np.int64)
    return orc.assemble(t, st, np.concatenate(rows), np.concatenate(cols),
                        np.ones(sum(len(r) for r in rows)), p,
                        strata=rng.integers(0, strata, size=n) if strata else None)


class NumpyShard:
    """Cox shard [lo, hi) of a Sorted layout (dense numpy; CPU test stand-in)."""

    def __init__(self, ds, lo, hi):
        self.lo, self.hi = lo, hi
        p = len(ds.col_ptr) - 1
        self.X = np.zeros((hi - lo, p))
        for j in range(p):
            a, b = ds.col_ptr[j], ds.col_ptr[j + 1]
            r = ds.row_idx[a:b]
            k = (r >= lo) & (r < hi)
            self.X[r[k] - lo, j] = ds.vals[a:b][k]
        self.t = ds.times[lo:hi]
        self.ev = (ds.status[lo:hi] == 1).astype(float)
        ss = np.zeros(hi - lo, bool) if ds.stratum_start is None else \
            ds.stratum_start[lo:hi].astype(bool)
        ss[0] = ss[0] or lo == 0
        self.seg = ss
        self.eta = np.zeros(hi - lo)
        # block ends: last row of each run of equal time inside a stratum
        nxt_t = np.append(self.t[1:], -1.0)
        nxt_s = np.append(self.seg[1:], True)
        self.end = (nxt_t != self.t) | nxt_s
        self.d = np.zeros(hi - lo)
        start = 0
        for i in range(hi - lo):
            if self.end[i]:
                self.d[i] = self.ev[start:i + 1].sum()
                start = i + 1

    def fixed_terms(self):
        return self.ev @ self.X

    def load_beta(self, beta):
        self.eta = self.X @ np.asarray(beta)

    def _lanes(self, j):
        e = np.exp(self.eta)
        if j < 0:
            return np.stack([e, 0 * e, 0 * e], 1)
        x = self.X[:, j]
        return np.stack([e, e * x, e * x * x], 1)

    def shard_aggregate(self, j):
        v = self._lanes(j)
        starts = np.nonzero(self.seg)[0]
        last = starts[-1] if len(starts) else 0
        out = np.zeros(8)
        out[0] = 1.0 if len(starts) else 0.0
        out[1:4] = v[last:].sum(0)
        out[7] = 1.0 if self.seg[0] else 0.0
        return out

    def shard_sums(self, j, carry):
        v = self._lanes(j)
        run = np.zeros(3) if self.seg[0] else np.asarray(carry[0:3], float).copy()
        s0 = s1 = 0.0
        for i in range(len(v)):
            if self.seg[i]:
                run = np.zeros(3)
            run = run + v[i]
            if self.end[i] and self.d[i] > 0:
                if j < 0:
                    s1 += self.d[i] * np.log(run[0])
                else:
                    g, h = run[1] / run[0], run[2] / run[0]
                    s0 += self.d[i] * g
                    s1 += self.d[i] * (h - g * g)
        if j < 0:
            s0 = float(self.ev @ self.eta)
        return s0, s1

    def update_validate(self, j, delta):
        return bool(np.any(np.abs(self.eta + self.X[:, j] * delta) > 700.0))

    def update(self, j, delta):
        self.eta = self.eta + self.X[:, j] * delta


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2204_08183_b200 import sharded
        ds = make_ds()
        f = sharded.ShardedFit(ds, "cox", sharded.TorchExchange(),
                               engine_factory=lambda d, lo, hi: NumpyShard(d, lo, hi))
        q.put((rank, f.fit(penalty="l1", strength=3.0, max_cycles=5)))
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_world_size_two_sharded_fit_matches_oracle():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    ref = orc.OracleEngine(make_ds(), "cox").fit(penalty="l1", strength=3.0, max_cycles=5)
    for rank in (0, 1):
        r = got[rank]
        assert r["cycles"] == ref["cycles"]
        assert np.max(rel(r["beta"], ref["beta"])) < TOL_BETA
        assert np.max(rel(r["objective_trace"], ref["objective_trace"])) < TOL_DERIV
    assert np.array_equal(got[0]["beta"], got[1]["beta"])  # identical steps on every rank


def test_carry_composition_segments_by_strata():
    from paper_2204_08183_b200.sharded import _carries
    aggs = np.zeros((4, 8))
    aggs[:, 1:4] = [[1, 1, 1], [2, 2, 2], [4, 4, 4], [8, 8, 8]]
    aggs[:, 4:7] = [[1, 0, 0], [2, 0, 0], [4, 0, 0], [8, 0, 0]]
    aggs[0, 0] = 1.0          # shard 0 holds the first stratum start
    aggs[2, 0] = 1.0          # a stratum starts inside shard 2
    c = _carries(aggs, 4)
    assert list(c[1, 0:3]) == [1, 1, 1]
    assert list(c[2, 0:3]) == [3, 3, 3]
    assert list(c[3, 0:3]) == [4, 4, 4]      # from shard 2's last stratum start only
    assert c[0, 4] == 2 + 4                    # rev: shard 1 whole + shard 2's head
    assert c[2, 4] == 8
