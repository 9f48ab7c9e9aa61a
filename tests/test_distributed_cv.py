"""Config C4's multi-process path without a GPU: cross-validation tasks dealt
over world_size-2 gloo ranks, scores all-gathered and merged in task order,
must equal the single-process result bit for bit, and the merged curve must
match the UNMODIFIED reference's cross_validate (oracle/_ref, CPU) on the same
data.  The per-task fits run on the C oracle (the compute stand-in here; on
a GPU box the same driver runs survscan.cv_run_tasks on each rank's device)."""
import os
import socket
import sys

import numpy as np
import pytest
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

from tests._common import load, raw  # noqa: E402

GRID = [0.05, 0.2, 0.8, 3.2]
FOLDS, REPS, SEED, TOL, MAXC = 3, 2, 11, 1e-12, 400


def _dataset(name="cox_ties"):
    import survscan
    c = load(name)
    (t, s, rows, cols, vals, p), _ = raw(c)
    return str(c["model"]), survscan.dataset_from_coo(t, s, rows, cols, vals, p), (t, s, rows,
                                                                                   cols, vals, p)


def oracle_runner(ds, model, grid):
    """Task scores with the C oracle on subset datasets (subset_rows semantics)."""
    import survscan
    from oracle import oracle as orc
    times, status = np.asarray(ds.times), np.asarray(ds.status)
    p = ds.p
    cells = [(i, j, ds.covariate(i, j)) for j in range(p) for i in range(ds.n)
             if ds.covariate(i, j) != 0.0]
    ci = np.array([c[0] for c in cells]), np.array([c[1] for c in cells]), \
        np.array([c[2] for c in cells])

    def subset(mask):
        pos = np.nonzero(mask)[0]
        remap = -np.ones(ds.n, np.int64)
        remap[pos] = np.arange(len(pos))
        sel = remap[ci[0]] >= 0
        return orc.assemble(times[pos], status[pos], remap[ci[0][sel]], ci[1][sel], ci[2][sel], p)

    def run(tasks):
        out = []
        for task in tasks:
            gi, t = task // REPS, task % REPS
            fold_of = np.array(survscan.fold_assignment(ds.n, FOLDS, SEED, gi, t))
            scores = []
            for f in range(FOLDS):
                eng = orc.OracleEngine(subset(fold_of != f), model)
                r = eng.fit(penalty="l1", strength=grid[gi], tol=TOL, max_cycles=MAXC)
                held = orc.OracleEngine(subset(fold_of == f), model)
                held.load_beta(r["beta"])
                scores.append(held.log_likelihood())
            out.append(scores)
        return out
    return run


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2204_08183_b200.distributed import cross_validate_distributed
        model, ds, _ = _dataset()
        res = cross_validate_distributed(ds, model=model, penalty="l1", grid=GRID, folds=FOLDS,
                                         repetitions=REPS, seed=SEED, tol=TOL, max_cycles=MAXC,
                                         task_runner=oracle_runner(ds, model, GRID),
                                         final_fit=False)
        q.put((rank, res))
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.fixture(scope="module")
def runs():
    from paper_2204_08183_b200.distributed import cross_validate_distributed
    model, ds, _ = _dataset()
    single = cross_validate_distributed(ds, model=model, penalty="l1", grid=GRID, folds=FOLDS,
                                        repetitions=REPS, seed=SEED, tol=TOL, max_cycles=MAXC,
                                        task_runner=oracle_runner(ds, model, GRID),
                                        final_fit=False)
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
    return single, got


def test_world_size_two_equals_single_process(runs):
    single, got = runs
    assert set(got) == {0, 1}
    for rank in (0, 1):
        res = got[rank]
        assert res["selected"] == single["selected"]
        assert res["failed_replicates"] == single["failed_replicates"]
        assert res["curve"] == single["curve"]  # bitwise: task-ordered merge
    assert got[0]["tasks_per_rank"] + got[1]["tasks_per_rank"] == len(GRID) * REPS


def test_merged_curve_matches_reference_cross_validate(runs):
    d = os.path.join(ROOT, "oracle", "_ref")
    if not os.path.isdir(d):
        pytest.skip("reference module not built")
    sys.path.insert(0, d)
    import _survscan as ref
    single, _ = runs
    model, _, (t, s, rows, cols, vals, p) = _dataset()
    rds = ref.dataset_from_coo(t, s, rows, cols, vals, p)
    cv = ref.cross_validate(rds, model=model, penalty="l1", grid=GRID, folds=FOLDS,
                            repetitions=REPS, seed=SEED, tol=TOL, max_cycles=MAXC, threads=1)
    assert cv["selected"] == single["selected"]
    for a, b in zip(single["curve"], cv["curve"]):
        assert a["evaluations"] == b["evaluations"]
        assert abs(a["mean_loglik"] - b["mean_loglik"]) <= 1e-9 * max(1.0, abs(b["mean_loglik"]))


def test_shard_tasks_covers_every_task_once():
    from paper_2204_08183_b200.distributed import shard_tasks
    for world in (1, 2, 4, 8):
        seen = sorted(t for r in range(world) for t in shard_tasks(37, r, world))
        assert seen == list(range(37))
