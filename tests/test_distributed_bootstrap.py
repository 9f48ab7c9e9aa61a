"""Bootstrap (src/crossval.cpp:218-257) dealt over world_size-2 gloo ranks:
the resamples' draws (the reference's derive_seed(seed, 0, b) row streams,
reproduced by survscan.bootstrap_indices) are fitted per rank, gathered and
merged in resample order — equal to the single-process interval and to the
UNMODIFIED reference's bootstrap_interval.  The per-resample fits run on the
C oracle here (the GPU path runs survscan.bootstrap_run on each rank's
device).  Also: a failing rank makes EVERY rank raise (no hang)."""
import os
import socket
import subprocess
import sys

import numpy as np
import pytest
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

from tests._common import load, raw  # noqa: E402

RES, SEED, LAM, COEF = 100, 17, 0.3, 2


def _data():
    import survscan
    c = load("cox_ties")
    (t, s, rows, cols, vals, p), _ = raw(c)
    return survscan.dataset_from_coo(t, s, rows, cols, vals, p), (t, s, rows, cols, vals, p)


def oracle_draws(ds):
    import survscan
    from oracle import oracle as orc
    times, status = np.asarray(ds.times), np.asarray(ds.status)
    cells = [(i, j, ds.covariate(i, j)) for j in range(ds.p) for i in range(ds.n)
             if ds.covariate(i, j) != 0.0]
    ri = np.array([c[0] for c in cells])
    cj = np.array([c[1] for c in cells])
    vv = np.array([c[2] for c in cells])

    def run(ids):
        out = []
        for b in ids:
            idx = np.asarray(survscan.bootstrap_indices(ds.n, SEED, b), np.int64)
            # subset_rows(idx, fresh_row_ids=True): repeated rows, new ids in order
            rows, cols, vals = [], [], []
            for k, i in enumerate(idx):
                sel = ri == i
                rows.append(np.full(sel.sum(), k))
                cols.append(cj[sel])
                vals.append(vv[sel])
            sub = orc.assemble(times[idx], status[idx], np.concatenate(rows), np.concatenate(cols),
                               np.concatenate(vals), ds.p)
            r = orc.OracleEngine(sub, "cox").fit(penalty="l1", strength=LAM)
            out.append(float(r["beta"][COEF]))
        return out
    return run


def _worker(rank, world, port, q, fail_rank):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2204_08183_b200.distributed import bootstrap_distributed
        ds, _ = _data()
        runner = oracle_draws(ds)
        if rank == fail_rank:
            def runner(ids):  # noqa: F811
                raise ValueError("injected failure")
        try:
            res = bootstrap_distributed(ds, "cox", "l1", LAM, coefficient=COEF, resamples=RES,
                                        seed=SEED, draw_runner=runner)
            q.put((rank, "ok", tuple(res)))
        except RuntimeError as exc:
            q.put((rank, "raised", str(exc)))
    finally:
        dist.destroy_process_group()


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _spawn(fail_rank):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q, fail_rank)) for r in range(2)]
    for p in procs:
        p.start()
    got = {}
    for _ in procs:
        r, kind, val = q.get(timeout=300)
        got[r] = (kind, val)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return got


def test_bootstrap_world_two_equals_single_and_reference():
    from paper_2204_08183_b200.distributed import bootstrap_distributed
    ds, (t, s, rows, cols, vals, p) = _data()
    single = tuple(bootstrap_distributed(ds, "cox", "l1", LAM, coefficient=COEF, resamples=RES,
                                         seed=SEED, draw_runner=oracle_draws(ds)))
    got = _spawn(fail_rank=-1)
    for r in (0, 1):
        assert got[r] == ("ok", single)  # bitwise: resample-ordered merge
    ref_dir = os.path.join(ROOT, "oracle", "_ref")
    if not os.path.isdir(ref_dir):
        pytest.skip("reference module not built")
    np.savez("/tmp/_boot_in.npz", t=t, s=s, rows=rows, cols=cols, vals=vals, p=p)
    out = subprocess.check_output([sys.executable, "-c", f"""
import sys, numpy as np
sys.path.insert(0, {ref_dir!r})
import _survscan as ref
z = np.load('/tmp/_boot_in.npz')
ds = ref.dataset_from_coo(z['t'], z['s'], z['rows'], z['cols'], z['vals'], int(z['p']))
lo, hi, f = ref.bootstrap_interval(ds, 'cox', 'l1', {LAM}, coefficient={COEF}, resamples={RES},
                                   seed={SEED}, threads=1)
print(repr(lo), repr(hi), f)
"""], text=True).split()
    lo, hi, failed = float(out[0]), float(out[1]), int(out[2])
    assert failed == single[2]
    assert abs(single[0] - lo) <= 1e-8 * max(1.0, abs(lo))
    assert abs(single[1] - hi) <= 1e-8 * max(1.0, abs(hi))


def test_failing_rank_raises_everywhere():
    got = _spawn(fail_rank=1)
    assert got[0][0] == "raised" and got[1][0] == "raised"
    assert "rank 1 failed" in got[0][1] and "injected failure" in got[0][1]
