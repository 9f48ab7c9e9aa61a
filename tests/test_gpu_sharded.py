"""Config C5 on one GPU: the patient-sharded protocol (paper_2204_08183_b200/
sharded.py) with every shard emulated in one process (LocalExchange) must
reproduce the unsharded computation — derivatives and log-likelihood to the
north-star tolerance, and fits with the same cycle counts and coefficients."""
import os

import numpy as np
import pytest

from oracle import oracle as orc
from tests._common import TOL_BETA, TOL_DERIV, rel, rel_cond
from tests.test_gpu_parity import _random_sorted

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def mods():
    from paper_2204_08183_b200 import capi, sharded
    assert capi.lib().gss_device_count() > 0
    return capi, sharded


@pytest.mark.parametrize("world", [2, 3, 5])
@pytest.mark.parametrize("n,quant,strata", [(40_000, 40.0, None), (30_001, 25.0, 4),
                                            (9_000, None, None)])
def test_sharded_derivatives_match_unsharded(mods, world, n, quant, strata):
    capi, sharded = mods
    ds = _random_sorted(n, 6, 0.05, seed=n + world, quant=quant, strata=strata)
    fitter = sharded.ShardedFit(ds, "cox", sharded.LocalExchange(world))
    ref = orc.OracleEngine(ds, "cox")
    beta = np.linspace(-0.3, 0.25, ds.p)
    fitter.load_beta(beta)
    ref.load_beta(beta)
    assert rel(fitter.log_likelihood(), ref.log_likelihood()) < TOL_DERIV
    for j in range(ds.p):
        a, b = fitter.grad_hessian(j), ref.grad_hessian(j)
        assert a["fixed_term"] == pytest.approx(b["fixed_term"], rel=1e-15)
        assert rel_cond(a["gradient"], b["gradient"], b["fixed_term"]) < TOL_DERIV, j
        assert rel(a["hessian"], b["hessian"]) < TOL_DERIV, j


@pytest.mark.parametrize("world", [1, 2, 4])
def test_sharded_fit_matches_single_device_fit(mods, world):
    capi, sharded = mods
    ds = _random_sorted(50_000, 8, 0.04, seed=77, quant=30.0)
    r1 = sharded.ShardedFit(ds, "cox", sharded.LocalExchange(world)).fit(
        penalty="l1", strength=2.0, max_cycles=6)
    r2 = orc.OracleEngine(ds, "cox").fit(penalty="l1", strength=2.0, max_cycles=6)
    assert r1["cycles"] == r2["cycles"]
    assert np.max(rel(r1["beta"], r2["beta"])) < TOL_BETA
    assert np.max(rel(r1["objective_trace"], r2["objective_trace"])) < TOL_DERIV
    assert len(r1["shards"]) == world + 1


def test_shard_cuts_respect_tied_blocks(mods):
    _, sharded = mods
    t = np.array([5, 5, 5, 4, 4, 3, 3, 3, 3, 1], float)
    cuts = sharded.shard_bounds(t, None, 3)
    assert cuts[0] == 0 and cuts[-1] == len(t)
    for c in cuts[1:-1]:
        assert c == len(t) or t[c] != t[c - 1]


@pytest.mark.parametrize("world", [2, 3, 4])
@pytest.mark.parametrize("n,quant,strata,interval", [(60_000, 40.0, None, 100),
                                                     (45_001, 25.0, 5, 100),
                                                     (20_000, None, None, 7)])
def test_in_kernel_sharded_fit_matches_oracle(mods, world, n, quant, strata, interval):
    """The in-kernel cross-shard exchange (gss_comm_local + gss_sharded_fit_local:
    every shard's cycle kernel publishes its aggregate to the others' peer
    buffers after each grid exchange) reproduces the unsharded CCD fit: same
    cycles, coefficients within 1e-8, including refreshes (interval 7) and
    strata that span shard cuts."""
    capi, sharded = mods
    ds = _random_sorted(n, 8, 0.05, seed=n + 17 * world, quant=quant, strata=strata)
    r = sharded.fit_in_kernel_local(ds, world, penalty="l1", strength=1.5, max_cycles=8,
                                    recompute_interval=interval)
    ref = orc.OracleEngine(ds, "cox", recompute_interval=interval).fit(
        penalty="l1", strength=1.5, max_cycles=8)
    assert r["cycles"] == ref["cycles"]
    assert np.max(rel(r["beta"], ref["beta"])) < TOL_BETA
    assert rel(r["objective"], ref["objective"]) < TOL_DERIV
    one = capi.Engine(capi.Dataset.from_sorted(ds), "cox", interval).fit(
        penalty="l1", strength=1.5, max_cycles=8)
    assert one["cycles"] == r["cycles"]
    assert np.max(rel(r["beta"], one["beta"])) < TOL_BETA


def test_in_kernel_shards_refuse_finegray_and_empty_cuts(mods):
    capi, sharded = mods
    ds = _random_sorted(5_000, 3, 0.05, seed=3, quant=2.0)
    with pytest.raises(ValueError):
        sharded.shard_engines(ds, 4000)
    d = capi.Dataset.from_sorted(ds)
    e = capi.Engine(d, "cox")
    assert capi.lib().gss_engine_attach_comm(e.h, None) != 0  # null comm -> error, no crash


def test_comm_init_single_rank_bootstrap(mods):
    """The multi-process path's bootstrap (NCCL unique id -> ncclCommInitRank
    -> CUDA IPC export/all-gather of the exchange buffers) on one rank; a
    one-rank communicator leaves the fit unchanged (no cross exchange)."""
    capi, sharded = mods
    ds = _random_sorted(20_000, 5, 0.05, seed=5, quant=30.0)
    uid = capi.comm_unique_id()
    assert len(uid) == 128
    comm = capi.comm_init(1, 0, uid, 0)
    assert comm.rank == (0, 1)
    d = capi.Dataset.from_sorted(ds)
    a = capi.Engine(d, "cox").attach_comm(comm).fit(penalty="l1", strength=1.0, max_cycles=5)
    b = capi.Engine(d, "cox").fit(penalty="l1", strength=1.0, max_cycles=5)
    assert a["cycles"] == b["cycles"]
    np.testing.assert_array_equal(a["beta"], b["beta"])


@pytest.mark.parametrize("world,grid", [(2, 74), (3, 49)])
def test_multiprocess_shards_under_mps(world, grid, tmp_path):
    """The one-process-per-shard path (CUDA-IPC exchange buffers connected
    through torch.distributed, system-scope flags, the exchange inside every
    rank's kernel) with all ranks on one GPU: a private MPS daemon lets the
    ranks' kernels co-reside (grids capped).  Every rank ends with the same
    objective; rank 0's coefficients match the unsharded fit."""
    import json
    import shutil
    import subprocess
    import sys
    ctl = shutil.which("nvidia-cuda-mps-control")
    if ctl is None:
        pytest.skip("no MPS control daemon on this box")
    env = dict(os.environ, CUDA_MPS_PIPE_DIRECTORY=str(tmp_path / "pipe"),
               CUDA_MPS_LOG_DIRECTORY=str(tmp_path / "log"))
    os.makedirs(env["CUDA_MPS_PIPE_DIRECTORY"])
    os.makedirs(env["CUDA_MPS_LOG_DIRECTORY"])
    if subprocess.run([ctl, "-d"], env=env).returncode != 0:
        pytest.skip("could not start a private MPS daemon")
    try:
        root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
        port = 29600 + world
        out = subprocess.run(
            [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
             f"--nproc-per-node={world}", "--master-addr", "127.0.0.1", "--master-port", str(port),
             os.path.join(root, "tools", "c5_multiproc.py"), "--same-gpu", "--grid", str(grid)],
            env=env, capture_output=True, text=True, timeout=240, cwd=root)
    finally:
        subprocess.run([ctl], input="quit\n", env=env, text=True)
    # the ranks share one stdout pipe: decode every JSON object in it, even
    # two that landed on one line
    dec, lines, i, txt = json.JSONDecoder(), [], 0, out.stdout
    while True:
        i = txt.find("{", i)
        if i < 0:
            break
        try:
            obj, i = dec.raw_decode(txt, i)
        except json.JSONDecodeError:
            i += 1
            continue
        lines.append(obj)
    assert out.returncode == 0 and len(lines) == world, out.stderr[-2000:]
    assert len({ln["objective"] for ln in lines}) == 1
    r0 = [ln for ln in lines if ln["rank"] == 0][0]
    assert r0["pass"], r0


def test_in_kernel_sharded_fit_valued_dense_and_refresh(mods):
    """Shards of a dataset with valued columns (the exp recompute and the
    valued-record correction exchange), a dense column (density >= 25%: the
    dense pool), strata spanning the cuts and in-kernel refreshes every 3
    accepted updates (max |eta| combined over shards): same cycles and
    coefficients as the oracle."""
    capi, sharded = mods
    rng = np.random.default_rng(21)
    n, p = 40_000, 6
    rows, cols, vals = [], [], []
    for j, dens in enumerate([0.05, 0.4, 0.03, 0.08, 0.02, 0.05]):
        r = np.sort(rng.choice(n, size=int(dens * n), replace=False))
        v = np.ones(r.size) if j in (2, 4) else np.round(rng.normal(size=r.size), 2) + 0.01
        rows.append(r)
        cols.append(np.full(r.size, j))
        vals.append(v)
    t = np.ceil(rng.exponential(size=n) * 30) / 30
    st = (rng.random(n) < 0.7).astype(np.int64)
    ds = orc.assemble(t, st, np.concatenate(rows), np.concatenate(cols), np.concatenate(vals), p,
                      strata=rng.integers(0, 3, n))
    for world in (2, 3):
        r = sharded.fit_in_kernel_local(ds, world, penalty="l1", strength=1.0, max_cycles=6,
                                        recompute_interval=3)
        ref = orc.OracleEngine(ds, "cox", recompute_interval=3).fit(
            penalty="l1", strength=1.0, max_cycles=6)
        assert r["cycles"] == ref["cycles"]
        assert np.max(rel(r["beta"], ref["beta"])) < TOL_BETA
        assert rel(r["objective"], ref["objective"]) < TOL_DERIV


def test_in_kernel_sharded_overflow_raises_on_every_shard(mods):
    """A step that would push |x'beta| past 700 on one row of the LAST shard
    (a censored row with the smallest time and x = 1e5, the construction of
    test_fit_overflow_mid_cycle_raises_like_reference) must stop the fit on
    every shard: the exact validation's overflow flag is OR-ed over shards in
    the kernel, and the error is the reference's OverflowError."""
    capi, sharded = mods
    rng = np.random.default_rng(77)
    n, p = 30_000, 6
    t = rng.exponential(size=n)
    status = (rng.random(n) < 0.7).astype(np.int64)
    last = int(np.argmin(t))
    status[last] = 0
    bulk = np.setdiff1d(np.arange(n), [last])
    rows, cols, vals = [], [], []
    eta = np.zeros(n)
    for j in range(p):
        r = rng.choice(bulk, size=1500, replace=False)
        v = np.round(rng.uniform(-3.0, 3.0, size=r.size), 2)
        v[v == 0] = 1.5
        eta[r] += 0.4 * v
        r = np.append(r, last)
        v = np.append(v, 1.0e5)
        o = np.argsort(r)
        rows.append(r[o])
        cols.append(np.full(r.size, j))
        vals.append(v[o])
    t = t / np.exp(eta)
    t[last] = t.min() / 2.0
    ds = orc.assemble(t, status, np.concatenate(rows), np.concatenate(cols), np.concatenate(vals), p)
    with pytest.raises(orc.OracleError) as e_ref:
        orc.OracleEngine(ds, "cox").fit(penalty="none", max_cycles=5)
    for world in (2, 3):
        with pytest.raises(capi.GssError) as e_dev:
            sharded.fit_in_kernel_local(ds, world, penalty="none", max_cycles=5)
        assert e_dev.value.kind == e_ref.value.kind == "OverflowError"
