"""The drop-in Python API (`survscan`, the reference's bindings surface,
bindings/survscan_py.cpp:105-326) on the device engine, plus parity of the
C++ drivers (fit, cross_validate, gamma_max) against the UNMODIFIED reference
module built in oracle/_ref (test infrastructure, run on the host CPU)."""
import math
import os
import sys

import numpy as np
import pytest

from tests._common import TOL_BETA, TOL_DERIV, load, raw, rel

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def ss():
    import survscan
    assert survscan.device_count() > 0
    return survscan


@pytest.fixture(scope="module")
def ref():
    d = os.path.join(ROOT, "oracle", "_ref")
    if not os.path.isdir(d):
        pytest.skip("reference module not built (oracle/build_ref.sh)")
    sys.path.insert(0, d)
    try:
        import _survscan as r
    except ImportError as exc:
        pytest.skip(f"reference module unavailable: {exc}")
    return r


@pytest.fixture(scope="module")
def fg(ss):
    return ss.simulate_finegray(n=400, p=6, density=0.2, seed=5, censoring_quantile=0.9)


def test_simulation_shape_and_determinism(ss, fg):
    ds, b1, b2 = fg
    assert ds.n == 400 and ds.p == 6 and ds.has_competing
    assert np.array_equal(b2, -b1)
    again, c1, _ = ss.simulate_finegray(n=400, p=6, density=0.2, seed=5, censoring_quantile=0.9)
    assert again.content_hash == ds.content_hash and np.array_equal(b1, c1)
    assert set(np.unique(ds.status)) <= {0, 1, 2}


def test_fit_monotone_and_finegray_reduces_to_cox(ss, fg):
    ds = fg[0]
    res = ss.fit(ds, model="finegray", penalty="l1", strength=0.05)
    assert res["converged"] and res["beta"].shape == (6,)
    tr = res["objective_trace"]
    assert all(b >= a - 1e-10 for a, b in zip(tr, tr[1:]))
    cox_ds, _ = ss.simulate_cox(n=300, p=4, density=0.2, seed=9, censoring_quantile=0.85)
    a = ss.fit(cox_ds, model="cox")
    b = ss.fit(cox_ds, model="finegray")
    assert np.max(np.abs(a["beta"] - b["beta"])) <= 1e-12


def test_loglik_gradient_finite_difference(ss, fg):
    ds = fg[0]
    beta = np.full(ds.p, 0.01)
    base = ss.log_likelihood(ds, "finegray", beta)
    assert math.isfinite(base) and base < 0
    h = 1e-5
    up, dn = beta.copy(), beta.copy()
    up[2] += h
    dn[2] -= h
    fd = (ss.log_likelihood(ds, "finegray", up) - ss.log_likelihood(ds, "finegray", dn)) / (2 * h)
    g, hess = ss.grad_hessian(ds, "finegray", beta, 2)
    assert hess <= 0 and abs(fd - g) <= 1e-6 * max(1.0, abs(g))


def test_cross_validate_gamma_max(ss, fg):
    ds = fg[0]
    cv = ss.cross_validate(ds, model="finegray", penalty="l1", folds=3, repetitions=1, seed=4)
    strengths = [pt["strength"] for pt in cv["curve"]]
    assert len(strengths) == 10 and strengths == sorted(strengths)
    assert cv["selected"] in strengths
    top = ss.gamma_max(ds, model="finegray")
    assert strengths[-1] == top and ss.auto_grid(top)[0] == top / 1000.0
    assert ss.fit(ds, model="finegray", penalty="l1", strength=top)["nonzero_count"] == 0


def test_bootstrap_interval(ss, fg):
    lo, hi, failed = ss.bootstrap_interval(fg[0], model="finegray", penalty="l1", strength=0.05,
                                           coefficient=1, resamples=100, seed=3)
    assert lo <= hi and failed == 0


def test_drop_in_caller_runs(tmp_path):
    """tests/cpp/drop_in_caller.cpp — written against the reference's C++
    Engine / CCD API — runs on the device engine."""
    import subprocess
    from paper_2204_08183_b200 import build as B
    host = os.path.join(ROOT, "paper_2204_08183_b200", "csrc", "host")
    exe = str(tmp_path / "caller")
    subprocess.check_call(["g++", "-std=c++20", "-O1", "-I" + host,
                           os.path.join(ROOT, "tests", "cpp", "drop_in_caller.cpp"),
                           "-L" + B.PKG, "-lsurvscan_b200", "-lgss", "-Wl,-rpath," + B.PKG,
                           "-o", exe])
    out = subprocess.check_output([exe], text=True)
    assert "drop-in caller ok" in out


def test_errors_surface(ss, fg):
    # (RuntimeError: once a test has imported the reference module into this
    # process, its translator also claims survscan::Error)
    with pytest.raises(RuntimeError, match="competing"):
        ss.fit(fg[0], model="cox")  # competing rows under a cox model
    with pytest.raises(RuntimeError):
        ss.grad_hessian(fg[0], "finegray", np.zeros(6), 17)


def _both(ss, ref, name):
    c = load(name)
    (t, s, rows, cols, vals, p), _ = raw(c)
    a = ss.dataset_from_coo(t, s, rows, cols, vals, p)
    b = ref.dataset_from_coo(t, s, rows, cols, vals, p)
    return str(c["model"]), a, b


@pytest.mark.parametrize("name", ["cox_small", "cox_ties", "cox_valued", "fg_small", "fg_ties"])
def test_fit_parity_with_reference_module(ss, ref, name):
    model, a, b = _both(ss, ref, name)
    for pen, lam in [("none", 0.0), ("l1", 0.5), ("l2", 2.0)]:
        ra = ss.fit(a, model=model, penalty=pen, strength=lam, tol=1e-12, max_cycles=400)
        rb = ref.fit(b, model=model, penalty=pen, strength=lam, tol=1e-12, max_cycles=400,
                     threads=1)
        assert ra["cycles"] == rb["cycles"], (pen, lam)
        assert np.max(rel(ra["beta"], rb["beta"])) < TOL_BETA
        assert rel(ra["objective"], rb["objective"]) < TOL_DERIV
        assert ra["nonzero_count"] == rb["nonzero_count"]


@pytest.mark.parametrize("name", ["cox_small", "fg_small"])
def test_gamma_max_and_loglik_parity(ss, ref, name):
    model, a, b = _both(ss, ref, name)
    assert rel(ss.gamma_max(a, model=model), ref.gamma_max(b, model=model)) < TOL_DERIV
    beta = np.linspace(-0.2, 0.2, a.p)
    assert rel(ss.log_likelihood(a, model, beta), ref.log_likelihood(b, model, beta)) < TOL_DERIV


@pytest.mark.parametrize("name,model", [("cox_ties", "cox"), ("fg_small", "finegray")])
def test_cross_validate_parity_with_reference_module(ss, ref, name, model):
    """Same seeded partitions (counter-seeded shuffles), device row-mask folds
    vs the reference's subset copies: identical curves."""
    _, a, b = _both(ss, ref, name)
    grid = list(np.geomspace(0.05, 5.0, 5))
    kw = dict(model=model, penalty="l1", grid=grid, folds=3, repetitions=2, seed=11, tol=1e-12,
              max_cycles=400)
    ca = ss.cross_validate(a, **kw)
    cb = ref.cross_validate(b, threads=1, **kw)
    assert ca["selected"] == cb["selected"]
    assert ca["failed_replicates"] == cb["failed_replicates"]
    for pa, pb in zip(ca["curve"], cb["curve"]):
        assert pa["evaluations"] == pb["evaluations"]
        assert rel(pa["mean_loglik"], pb["mean_loglik"]) < 1e-9
    assert np.max(rel(ca["final_fit"]["beta"], cb["final_fit"]["beta"])) < TOL_BETA


def test_engine_class_surface(ss):
    c = load("cox_small")
    (t, s, rows, cols, vals, p), _ = raw(c)
    ds = ss.dataset_from_coo(t, s, rows, cols, vals, p)
    eng = ss.Engine(ds, "cox", recompute_interval=3)
    eng.load_beta(c["beta_probe"])
    assert rel(eng.log_likelihood(), c["ll"]) < TOL_DERIV
    for j in range(p):
        g, h, f = eng.grad_hessian(j)
        assert rel(h, c["hess"][j]) < TOL_DERIV
    eng.load_beta(np.zeros(p))
    for j, d in [(0, 0.1), (1, -0.2), (2, 0.3)]:
        eng.update_xbeta_sparse(j, d)
    assert eng.accepted_updates == 3 and eng.refresh_count == 1
    r = eng.fit(penalty="l1", strength=0.5)
    assert rel(r["objective"], float(c["fit1_objective"])) < TOL_DERIV


def test_distributed_driver_single_rank_equals_cross_validate(ss):
    """C4 driver (one process per GPU) at world size 1 == the C++ cross_validate."""
    from paper_2204_08183_b200.distributed import cross_validate_distributed
    c = load("cox_ties")
    (t, s, rows, cols, vals, p), _ = raw(c)
    ds = ss.dataset_from_coo(t, s, rows, cols, vals, p)
    grid = [0.05, 0.4, 3.0]
    kw = dict(model="cox", penalty="l1", grid=grid, folds=3, repetitions=2, seed=5, tol=1e-10,
              max_cycles=300)
    a = cross_validate_distributed(ds, **kw)
    b = ss.cross_validate(ds, **kw)
    assert a["selected"] == b["selected"]
    for pa, pb in zip(a["curve"], b["curve"]):
        assert pa["mean_loglik"] == pb["mean_loglik"] and pa["evaluations"] == pb["evaluations"]
    assert np.array_equal(a["final_fit"]["beta"], b["final_fit"]["beta"])


@pytest.mark.parametrize("name,model,lam,coef", [("cox_ties", "cox", 0.3, 2),
                                                 ("fg_small", "finegray", 0.05, 1)])
def test_bootstrap_parity_with_reference_module(ss, ref, name, model, lam, coef):
    """bootstrap_interval (src/crossval.cpp:218-257): the same derive_seed
    draw streams, the resamples' fits batched on the device (gss_fit_batch):
    the interval equals the reference's within the coefficient tolerance."""
    _, a, b = _both(ss, ref, name)
    kw = dict(model=model, penalty="l1", strength=lam, coefficient=coef, resamples=120, seed=23,
              tol=1e-10, max_cycles=500)
    la, ha, fa = ss.bootstrap_interval(a, **kw)
    lb, hb, fb = ref.bootstrap_interval(b, threads=1, **kw)
    assert fa == fb
    assert rel(la, lb) < TOL_BETA and rel(ha, hb) < TOL_BETA
    # the per-resample draws, too (resample-ordered pieces of the rank driver)
    draws = ss.bootstrap_run(a, model, "l1", lam, [], coef, list(range(120)), 23, 1e-10, 500)
    assert tuple(ss.bootstrap_merge(draws, 120)) == (la, ha, fa)


def test_cross_validate_bit_identical_across_device_lists():
    """Acceptance #10 of the reference (tests/acceptance.cpp:346-383: results
    bit-identical across worker counts), on the device: the same CV run with
    its tasks dealt over 1, 2 or 3 device lanes (worker threads on GPU 0)
    gives identical curves, selection and final coefficients."""
    import survscan
    rng = np.random.default_rng(11)
    n, p = 6000, 10
    k = int(n * p * 0.05)
    rows, cols = rng.integers(0, n, k), rng.integers(0, p, k)
    key = np.unique(cols * n + rows)
    t = np.ceil(rng.exponential(size=n) * 30) / 30
    s = (rng.random(n) < 0.7).astype(np.int64)
    ds = survscan.dataset_from_coo(t, s, key % n, key // n, np.ones(len(key)), p,
                                   rng.integers(0, 3, n))
    kw = dict(model="cox", penalty="l1", grid=[0.5, 1.0, 2.0, 4.0, 8.0], folds=5, repetitions=2,
              seed=3)
    outs = [survscan.cross_validate(ds, devices=d, **kw) for d in ([0], [0, 0], [0, 0, 0])]
    for o in outs[1:]:
        assert o["selected"] == outs[0]["selected"]
        assert [c["mean_loglik"] for c in o["curve"]] == [c["mean_loglik"] for c in outs[0]["curve"]]
        assert np.array_equal(np.asarray(o["final_fit"]["beta"]),
                              np.asarray(outs[0]["final_fit"]["beta"]))
