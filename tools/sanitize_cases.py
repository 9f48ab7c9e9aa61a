"""Small device workloads for compute-sanitizer (memcheck / racecheck /
synccheck) over the hand-written protocols of the cycle kernel: mbarrier ring,
named barriers, grid barrier, async-proxy fences.  Covers Cox and Fine-Gray,
API (grad_hessian / log_likelihood / grad_hessian_all) and CCD modes,
in-kernel refresh (recompute_interval=2), the exact validate-before-mutate
path and valued-column record correction, on a capped grid so CTAs hold
several tiles.

    compute-sanitizer --tool racecheck python tools/sanitize_cases.py
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import oracle as orc  # noqa: E402  (checker only)
from paper_2204_08183_b200 import capi  # noqa: E402


def data(n, p, seed, competing=0.0, valued=False, strata=None, outlier=False):
    rng = np.random.default_rng(seed)
    rows, cols, vals = [], [], []
    for j in range(p):
        r = np.sort(rng.choice(n, size=max(4, n // 20), replace=False))
        v = np.round(rng.normal(size=r.size), 2) if (valued and j % 2) else np.ones(r.size)
        v[v == 0] = 0.5
        if outlier and j == 0:
            v = v * 0 + 200.0
        rows.append(r)
        cols.append(np.full(r.size, j))
        vals.append(v)
    t = np.ceil(rng.exponential(size=n) * 20) / 20
    st = (rng.random(n) < 0.7).astype(np.int64)
    if competing:
        st[(st == 0) & (rng.random(n) < competing)] = 2
    s = None if strata is None else rng.integers(0, strata, size=n)
    return orc.assemble(t, st, np.concatenate(rows), np.concatenate(cols), np.concatenate(vals),
                        p, strata=s)


def main():
    grid = int(os.environ.get("SAN_GRID", "2"))
    n = int(os.environ.get("SAN_N", "9000"))
    for model, comp in (("cox", 0.0), ("finegray", 0.5)):
        for valued, strata in ((False, None), (True, 3)):
            ds = data(n, 5, 7, comp, valued, strata)
            dd = capi.Dataset.from_sorted(ds)
            e = capi.Engine(dd, model, recompute_interval=2).set_grid(grid)
            e.load_beta(np.linspace(-0.2, 0.2, ds.p))
            for j in range(ds.p):
                e.grad_hessian(j)
            e.log_likelihood()
            e.grad_hessian_all()
            e.update(1, 0.1)
            r = e.fit(penalty="l1", strength=0.5, max_cycles=3)
            print(model, "valued" if valued else "ind", "strata" if strata else "", "cycles",
                  r["cycles"], "obj", r["objective"], flush=True)
    # exact overflow validation path: a large value forces the exact check
    ds = data(n, 3, 9, outlier=True)
    e = capi.Engine(capi.Dataset.from_sorted(ds), "cox").set_grid(grid)
    try:
        r = e.fit(penalty="none", max_cycles=3)
        print("exact-path fit cycles", r["cycles"])
    except capi.GssError as exc:
        print("exact-path fit raised", exc.kind)
    # round 2 paths: dense-column pool (60% density), batched multi-fit,
    # in-kernel cross-shard exchange (2 local shards), device ingestion
    rng = np.random.default_rng(3)
    rows, cols, vals = [], [], []
    for j, dens in enumerate([0.6, 0.05, 0.3]):
        r = np.sort(rng.choice(n, size=int(dens * n), replace=False))
        rows.append(r)
        cols.append(np.full(r.size, j))
        vals.append(np.round(rng.normal(size=r.size), 2) + 0.01)
    t = np.ceil(rng.exponential(size=n) * 20) / 20
    st = (rng.random(n) < 0.7).astype(np.int64)
    dsd = orc.assemble(t, st, np.concatenate(rows), np.concatenate(cols), np.concatenate(vals), 3)
    for model in ("cox", "finegray"):
        e = capi.Engine(capi.Dataset.from_sorted(dsd), model, recompute_interval=3).set_grid(grid)
        e.load_beta(np.array([0.1, -0.1, 0.05]))
        for j in range(3):
            e.grad_hessian(j)
        print("dense", model, "cycles", e.fit(penalty="l1", strength=0.5, max_cycles=3)["cycles"],
              flush=True)
    ds = data(n, 5, 11)
    dd = capi.Dataset.from_sorted(ds)
    res, _ = capi.fit_batch([capi.Engine(dd, "cox"), capi.Engine(dd, "cox")], "l1", [0.5, 1.0],
                            max_cycles=3)
    print("batched fits", [r["cycles"] for r in res], flush=True)
    from paper_2204_08183_b200 import sharded
    r = sharded.fit_in_kernel_local(data(2 * n, 5, 13), 2, penalty="l1", strength=0.5,
                                    max_cycles=3, recompute_interval=4)
    print("sharded in-kernel fit cycles", r["cycles"], flush=True)
    import survscan
    dsx = survscan.dataset_from_coo(t, st, np.concatenate(rows), np.concatenate(cols),
                                    np.concatenate(vals), 3, rng.integers(0, 4, n))
    print("device ingestion nnz", dsx.nnz_total, flush=True)
    print("sanitize cases done")


if __name__ == "__main__":
    main()
