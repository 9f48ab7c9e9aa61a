"""Device path vs the reference (golden fixtures) and the pinned C oracle.

All calls go through the C ABI (libgss.so, include/gss.h).  Tolerances are
the north star's (BASELINE.json): 1e-10 relative on log-likelihood, gradient
and Hessian; 1e-8 on fitted coefficients.  Gradients use the
conditioning-aware denominator of SURVEY.md §8a (tests/_common.py).
"""
import numpy as np
import pytest

from oracle import oracle as orc
from tests._common import TOL_BETA, TOL_DERIV, cases, fit_cases, load, raw, rel, rel_cond

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def capi():
    from paper_2204_08183_b200 import capi as C
    assert C.lib().gss_device_count() > 0
    return C


def _sorted(c):
    args, strata = raw(c)
    return orc.assemble(*args, strata=strata)


GOLD = [n for n in cases() if not n.startswith("ka_")]
COX = [n for n in GOLD if str(load(n)["model"]) == "cox"]


@pytest.mark.parametrize("name", cases("ka_"))
def test_known_answers(capi, name):
    c = load(name)
    ds = _sorted(c)
    eng = capi.Engine(capi.Dataset.from_sorted(ds), "cox")
    gh = eng.grad_hessian(0)
    assert gh["gradient"] == pytest.approx(float(c["grad0"][0]), abs=1e-15)
    assert gh["hessian"] == pytest.approx(float(c["hess0"][0]), abs=1e-15)
    assert eng.log_likelihood() == pytest.approx(float(c["ll0"]), rel=1e-15, abs=1e-15)


@pytest.mark.parametrize("name", GOLD)
def test_derivatives_vs_reference(capi, name):
    c = load(name)
    ds = _sorted(c)
    eng = capi.Engine(capi.Dataset.from_sorted(ds), str(c["model"]))
    assert rel(eng.log_likelihood(), c["ll0"]) < TOL_DERIV
    eng.load_beta(c["beta_probe"])
    assert rel(eng.log_likelihood(), c["ll"]) < TOL_DERIV
    for j in range(ds.p):
        gh = eng.grad_hessian(j)
        assert rel_cond(gh["gradient"], c["grad"][j], gh["fixed_term"]) < TOL_DERIV, j
        assert rel(gh["hessian"], c["hess"][j]) < TOL_DERIV, j


@pytest.mark.parametrize("name", GOLD)
def test_fits_vs_reference(capi, name):
    c = load(name)
    ds = _sorted(c)
    dd = capi.Dataset.from_sorted(ds)
    max_cycles = 200 if "strata" in c else 1000
    for k, pen, lam in fit_cases(c):
        eng = capi.Engine(dd, str(c["model"]))
        r = eng.fit(penalty=pen, strength=lam, max_cycles=max_cycles)
        assert r["cycles"] == int(c[f"fit{k}_cycles"]), (pen, lam)
        assert np.max(rel(r["beta"], c[f"fit{k}_beta"])) < TOL_BETA, (pen, lam)
        assert rel(r["objective"], c[f"fit{k}_objective"]) < TOL_DERIV
        assert np.max(rel(r["objective_trace"], c[f"fit{k}_trace"])) < TOL_DERIV


def _random_sorted(n, p, density, seed, quant=None, strata=None, valued=False, competing=0.0):
    rng = np.random.default_rng(seed)
    nnz_per_col = rng.binomial(n, density, size=p)
    rows, cols, vals = [], [], []
    for j, k in enumerate(nnz_per_col):
        r = rng.choice(n, size=k, replace=False)
        rows.append(r)
        cols.append(np.full(k, j))
        vals.append(np.round(rng.normal(size=k), 3) if valued else np.ones(k))
    rows = np.concatenate(rows)
    cols = np.concatenate(cols)
    vals = np.concatenate(vals)
    vals[vals == 0] = 0.5
    t = rng.exponential(size=n)
    if quant:
        t = np.ceil(t * quant) / quant
    status = (rng.random(n) < 0.7).astype(np.int64)
    if competing:
        status[(status == 0) & (rng.random(n) < competing)] = 2
    st = None if strata is None else rng.integers(0, strata, size=n)
    return orc.assemble(t, status, rows, cols, vals, p, strata=st)


@pytest.mark.parametrize("n,p,quant,strata,valued", [
    (100_000, 24, None, None, False),
    (150_001, 16, 100.0, None, False),
    (60_000, 12, 30.0, 7, False),
    (70_000, 10, None, None, True),
])
def test_multitile_vs_oracle(capi, n, p, quant, strata, valued):
    ds = _random_sorted(n, p, 0.02, seed=n + p, quant=quant, strata=strata, valued=valued)
    ref = orc.OracleEngine(ds, "cox")
    eng = capi.Engine(capi.Dataset.from_sorted(ds), "cox")
    beta = np.random.default_rng(3).uniform(-0.4, 0.4, size=p)
    ref.load_beta(beta)
    eng.load_beta(beta)
    assert np.max(rel(eng.xbeta(), ref.eta[:n])) < 1e-13
    assert rel(eng.log_likelihood(), ref.log_likelihood()) < TOL_DERIV
    for j in range(p):
        a, b = eng.grad_hessian(j), ref.grad_hessian(j)
        assert rel_cond(a["gradient"], b["gradient"], b["fixed_term"]) < TOL_DERIV
        assert rel(a["hessian"], b["hessian"]) < TOL_DERIV
    # fit parity at a fixed number of cycles (convergence tests a rounded objective)
    eng2 = capi.Engine(capi.Dataset.from_sorted(ds), "cox")
    ref2 = orc.OracleEngine(ds, "cox")
    r1 = eng2.fit(penalty="l1", strength=2.0, max_cycles=6)
    r2 = ref2.fit(penalty="l1", strength=2.0, max_cycles=6)
    assert r1["cycles"] == r2["cycles"]
    assert np.max(rel(r1["beta"], r2["beta"])) < TOL_BETA
    assert np.max(rel(r1["objective_trace"], r2["objective_trace"])) < TOL_DERIV


def test_row_mask_equals_subset(capi):
    """A masked engine behaves exactly like the subset_rows() dataset
    (src/dataset.cpp:268-322) — the CV fold representation."""
    ds = _random_sorted(30_000, 8, 0.05, seed=5, quant=20.0)
    mask = (np.random.default_rng(1).random(ds.n) < 0.8).astype(np.uint8)
    keep = np.nonzero(mask)[0]
    # subset in sorted order with fresh ids preserving the order
    sub_rows = np.repeat(np.arange(ds.p), np.diff(ds.col_ptr))
    remap = -np.ones(ds.n, np.int64)
    remap[keep] = np.arange(len(keep))
    sel = remap[ds.row_idx] >= 0
    sub = orc.assemble(ds.times[keep], ds.status[keep], remap[ds.row_idx[sel]], sub_rows[sel],
                       ds.vals[sel], ds.p)
    ref = orc.OracleEngine(sub, "cox")
    eng = capi.Engine(capi.Dataset.from_sorted(ds), "cox", row_mask=mask)
    beta = np.linspace(-0.3, 0.3, ds.p)
    ref.load_beta(beta)
    eng.load_beta(beta)
    assert rel(eng.log_likelihood(), ref.log_likelihood()) < TOL_DERIV
    for j in range(ds.p):
        a, b = eng.grad_hessian(j), ref.grad_hessian(j)
        assert rel_cond(a["gradient"], b["gradient"], b["fixed_term"]) < TOL_DERIV
        assert rel(a["hessian"], b["hessian"]) < TOL_DERIV


def test_update_semantics_and_refresh(capi):
    """update_xbeta_sparse: indicator multiply rule, overflow atomicity,
    refresh cadence (tests/test_engine.cpp:178-263)."""
    ds = _random_sorted(20_000, 6, 0.05, seed=9, valued=False)
    ref = orc.OracleEngine(ds, "cox", recompute_interval=3)
    eng = capi.Engine(capi.Dataset.from_sorted(ds), "cox", recompute_interval=3)
    for j, d in [(0, 0.3), (1, -0.2), (2, 0.1), (0, 0.05), (3, 0.7)]:
        ref.update(j, d)
        eng.update(j, d)
    assert eng.counters() == (5, 1)
    assert np.max(rel(eng.exp_xbeta(), ref.e[:ds.n])) < 1e-14
    assert np.max(rel(eng.xbeta(), ref.eta[:ds.n])) < 1e-14
    before = eng.xbeta()
    with pytest.raises(capi.GssError) as ei:
        eng.update(4, 800.0)
    assert ei.value.kind == "OverflowError"
    assert np.array_equal(eng.xbeta(), before)
    with pytest.raises(capi.GssError) as ei:
        eng.grad_hessian(99)
    assert ei.value.kind == "InvalidColumnError"


def test_determinism(capi):
    ds = _random_sorted(200_000, 4, 0.01, seed=11, quant=50.0)
    dd = capi.Dataset.from_sorted(ds)
    outs = []
    for _ in range(3):
        eng = capi.Engine(dd, "cox")
        eng.load_beta(np.array([0.2, -0.1, 0.3, 0.05]))
        outs.append([eng.grad_hessian(j)["gradient"] for j in range(4)] + [eng.log_likelihood()])
    assert outs[0] == outs[1] == outs[2]


@pytest.mark.parametrize("n,p,quant,strata,valued", [
    (90_000, 12, None, None, False),
    (70_001, 10, 50.0, None, True),
    (50_000, 8, 20.0, 5, False),
])
def test_finegray_multitile_vs_oracle(capi, n, p, quant, strata, valued):
    """Forward-backward (u-weighted suffix) scan across many tiles and CTAs."""
    ds = _random_sorted(n, p, 0.03, seed=7 * n + p, quant=quant, strata=strata, valued=valued,
                        competing=0.6)
    ref = orc.OracleEngine(ds, "finegray")
    eng = capi.Engine(capi.Dataset.from_sorted(ds), "finegray")
    beta = np.random.default_rng(5).uniform(-0.3, 0.3, size=p)
    ref.load_beta(beta)
    eng.load_beta(beta)
    assert rel(eng.log_likelihood(), ref.log_likelihood()) < TOL_DERIV
    for j in range(p):
        a, b = eng.grad_hessian(j), ref.grad_hessian(j)
        assert rel_cond(a["gradient"], b["gradient"], b["fixed_term"]) < TOL_DERIV, j
        assert rel(a["hessian"], b["hessian"]) < TOL_DERIV, j
    eng2 = capi.Engine(capi.Dataset.from_sorted(ds), "finegray")
    ref2 = orc.OracleEngine(ds, "finegray")
    r1 = eng2.fit(penalty="l1", strength=1.0, max_cycles=5)
    r2 = ref2.fit(penalty="l1", strength=1.0, max_cycles=5)
    assert r1["cycles"] == r2["cycles"]
    assert np.max(rel(r1["beta"], r2["beta"])) < TOL_BETA
    assert np.max(rel(r1["objective_trace"], r2["objective_trace"])) < TOL_DERIV


def test_finegray_competing_block_ends_vs_oracle(capi):
    """Tied blocks with events whose last row (the Breslow transform's row) is a
    competing row, with censoring before them (G < 1): the kernel streams
    u = 1/G on competing rows and recovers G at those block ends."""
    rng = np.random.default_rng(29)
    n, p = 80_000, 8
    t = np.ceil(rng.exponential(size=n) * 40.0) / 40.0
    status = np.where(rng.random(n) < 0.5, 1, np.where(rng.random(n) < 0.5, 2, 0))
    # sorted order is (time desc, row id asc): a block's last row has the largest id
    last = {}
    for i in range(n):
        last[t[i]] = i
    has_event = {}
    for i in range(n):
        if status[i] == 1:
            has_event[t[i]] = True
    ends = [i for tv, i in last.items() if has_event.get(tv)]
    status[ends] = 2
    assert len(ends) > 100
    per = [rng.choice(n, size=rng.binomial(n, 0.04), replace=False) for _ in range(p)]
    rows = np.concatenate(per)
    cols = np.concatenate([np.full(len(r), j) for j, r in enumerate(per)])
    ds = orc.assemble(t, status, rows, cols, np.ones(len(rows)), p)
    ref = orc.OracleEngine(ds, "finegray")
    eng = capi.Engine(capi.Dataset.from_sorted(ds), "finegray")
    beta = np.random.default_rng(31).uniform(-0.3, 0.3, size=p)
    ref.load_beta(beta)
    eng.load_beta(beta)
    assert rel(eng.log_likelihood(), ref.log_likelihood()) < TOL_DERIV
    for j in range(p):
        a, b = eng.grad_hessian(j), ref.grad_hessian(j)
        assert rel_cond(a["gradient"], b["gradient"], b["fixed_term"]) < TOL_DERIV, j
        assert rel(a["hessian"], b["hessian"]) < TOL_DERIV, j
    r1 = capi.Engine(capi.Dataset.from_sorted(ds), "finegray").fit(penalty="l1", strength=1.0,
                                                                    max_cycles=4)
    r2 = orc.OracleEngine(ds, "finegray").fit(penalty="l1", strength=1.0, max_cycles=4)
    assert r1["cycles"] == r2["cycles"]
    assert np.max(rel(r1["beta"], r2["beta"])) < TOL_BETA


def test_finegray_mask_equals_subset(capi):
    ds = _random_sorted(40_000, 6, 0.05, seed=21, quant=30.0, competing=0.5)
    mask = (np.random.default_rng(2).random(ds.n) < 0.75).astype(np.uint8)
    keep = np.nonzero(mask)[0]
    sub_cols = np.repeat(np.arange(ds.p), np.diff(ds.col_ptr))
    remap = -np.ones(ds.n, np.int64)
    remap[keep] = np.arange(len(keep))
    sel = remap[ds.row_idx] >= 0
    sub = orc.assemble(ds.times[keep], ds.status[keep], remap[ds.row_idx[sel]], sub_cols[sel],
                       ds.vals[sel], ds.p)
    ref = orc.OracleEngine(sub, "finegray")
    eng = capi.Engine(capi.Dataset.from_sorted(ds), "finegray", row_mask=mask)
    beta = np.linspace(-0.2, 0.3, ds.p)
    ref.load_beta(beta)
    eng.load_beta(beta)
    assert rel(eng.log_likelihood(), ref.log_likelihood()) < TOL_DERIV
    for j in range(ds.p):
        a, b = eng.grad_hessian(j), ref.grad_hessian(j)
        assert rel_cond(a["gradient"], b["gradient"], b["fixed_term"]) < TOL_DERIV
        assert rel(a["hessian"], b["hessian"]) < TOL_DERIV


@pytest.mark.parametrize("model", ["cox", "finegray"])
def test_row_mask_equals_subset_1m_rows(capi, model):
    """Row-masked engine above 2^20 rows (the host pack and row codes run on
    parallel threads over chunks cut at tied-block starts): 30 distinct-time
    levels per unit make tied blocks of thousands of rows that straddle the
    chunk cuts; derivatives and log-likelihood equal the oracle on the
    subset of visible rows."""
    ds = _random_sorted(1_300_000, 5, 0.01, seed=77, quant=30.0,
                        competing=0.5 if model == "finegray" else 0.0)
    mask = (np.random.default_rng(5).random(ds.n) < 0.8).astype(np.uint8)
    keep = np.nonzero(mask)[0]
    sub_cols = np.repeat(np.arange(ds.p), np.diff(ds.col_ptr))
    remap = -np.ones(ds.n, np.int64)
    remap[keep] = np.arange(len(keep))
    sel = remap[ds.row_idx] >= 0
    sub = orc.assemble(ds.times[keep], ds.status[keep], remap[ds.row_idx[sel]], sub_cols[sel],
                       ds.vals[sel], ds.p)
    ref = orc.OracleEngine(sub, model)
    dd = capi.Dataset.from_sorted(ds)
    eng = capi.Engine(dd, model, row_mask=mask)
    full = capi.Engine(dd, model)
    ref_full = orc.OracleEngine(ds, model)
    beta = np.linspace(-0.2, 0.3, ds.p)
    for e, r in ((eng, ref), (full, ref_full)):
        r.load_beta(beta)
        e.load_beta(beta)
        assert rel(e.log_likelihood(), r.log_likelihood()) < TOL_DERIV
        for j in range(ds.p):
            a, b = e.grad_hessian(j), r.grad_hessian(j)
            assert rel_cond(a["gradient"], b["gradient"], b["fixed_term"]) < TOL_DERIV
            assert rel(a["hessian"], b["hessian"]) < TOL_DERIV


def test_finegray_without_competing_is_cox(capi):
    """tests/test_engine.cpp:293-310: no status-2 rows => the Cox computation."""
    ds = _random_sorted(30_000, 5, 0.04, seed=3, quant=40.0)
    dd = capi.Dataset.from_sorted(ds)
    a, b = capi.Engine(dd, "cox"), capi.Engine(dd, "finegray")
    beta = np.array([0.1, -0.2, 0.05, 0.3, -0.1])
    a.load_beta(beta)
    b.load_beta(beta)
    for j in range(ds.p):
        assert a.grad_hessian(j) == b.grad_hessian(j)
    assert a.log_likelihood() == b.log_likelihood()
    ra = capi.Engine(dd, "cox").fit(penalty="l1", strength=1.0, max_cycles=4)
    rb = capi.Engine(dd, "finegray").fit(penalty="l1", strength=1.0, max_cycles=4)
    assert np.array_equal(ra["beta"], rb["beta"])


@pytest.mark.parametrize("model", ["cox", "finegray"])
def test_grad_hessian_all_matches_single(capi, model):
    ds = _random_sorted(60_000, 9, 0.03, seed=17, quant=25.0, competing=0.5 if model == "finegray" else 0.0)
    eng = capi.Engine(capi.Dataset.from_sorted(ds), model)
    eng.load_beta(np.linspace(-0.2, 0.2, ds.p))
    allg = eng.grad_hessian_all()
    for j in range(ds.p):
        gh = eng.grad_hessian(j)
        # same kernel, but the batched launch builds each carry from the previous
        # slot's per-tile records (another fixed summation order)
        assert rel_cond(allg["gradient"][j], gh["gradient"], gh["fixed_term"]) < 1e-13
        assert rel(allg["hessian"][j], gh["hessian"]) < 1e-13


# ---- separated (unfused) path: Engine::grad_hessian_separated (engine.cpp:244-329) ----

@pytest.mark.parametrize("model,n,p,quant,strata,valued,mask", [
    ("cox", 80_000, 10, None, None, False, False),
    ("cox", 70_001, 8, 40.0, 6, True, False),
    ("cox", 50_000, 6, 20.0, None, False, True),
    ("finegray", 60_000, 8, 30.0, None, False, False),
    ("finegray", 45_000, 6, 25.0, 4, True, True),
])
def test_separated_equals_fused(capi, model, n, p, quant, strata, valued, mask):
    """tests/test_engine.cpp:165-176 (and acceptance check 5): fused and
    separated paths coincide to 1e-12; both match the oracle to 1e-10."""
    ds = _random_sorted(n, p, 0.04, seed=5 * n + p, quant=quant, strata=strata, valued=valued,
                        competing=0.5 if model == "finegray" else 0.0)
    m = (np.random.default_rng(n).random(ds.n) < 0.8).astype(np.uint8) if mask else None
    eng = capi.Engine(capi.Dataset.from_sorted(ds), model, row_mask=m)
    eng.load_beta(np.random.default_rng(9).uniform(-0.6, 0.6, size=p))
    for j in range(p):
        a, b = eng.grad_hessian(j), eng.grad_hessian_separated(j)
        assert rel(a["gradient"], b["gradient"]) < 1e-12, j
        assert rel(a["hessian"], b["hessian"]) < 1e-12, j
        assert a["fixed_term"] == b["fixed_term"]


def test_separated_known_answers_and_errors(capi):
    """test_engine.cpp:48-61 (N=2 known answer through both paths) and :318
    (InvalidColumnError from the separated path)."""
    for name in cases("ka_"):
        c = load(name)
        ds = _sorted(c)
        eng = capi.Engine(capi.Dataset.from_sorted(ds), "cox")
        gh = eng.grad_hessian_separated(0)
        assert gh["gradient"] == pytest.approx(float(c["grad0"][0]), abs=1e-15)
        assert gh["hessian"] == pytest.approx(float(c["hess0"][0]), abs=1e-15)
        with pytest.raises(capi.GssError) as ei:
            eng.grad_hessian_separated(ds.p)
        assert ei.value.kind == "InvalidColumnError"


def test_separated_after_fit_tracks_updates(capi):
    """After a device CCD fit (in-kernel updates and refreshes) the separated
    path sees the same exp(eta) state as the fused one."""
    ds = _random_sorted(40_000, 12, 0.05, seed=77, quant=50.0)
    eng = capi.Engine(capi.Dataset.from_sorted(ds), "cox", recompute_interval=5)
    eng.fit(penalty="l1", strength=1.0, max_cycles=3)
    for j in range(ds.p):
        a, b = eng.grad_hessian(j), eng.grad_hessian_separated(j)
        assert rel_cond(a["gradient"], b["gradient"], a["fixed_term"]) < 1e-12
        assert rel(a["hessian"], b["hessian"]) < 1e-12


@pytest.mark.parametrize("model", ["cox", "finegray"])
def test_exact_overflow_validation_path_vs_oracle(capi, model):
    """One extreme value per column (|x| = 1000, on a censored row with the
    smallest time, so it sits in no event's risk set and leaves beta at the
    bulk's scale) makes the fast |x'beta| bound (max|eta| + sum |delta| *
    max|x|) pass 700 after a few updates: the kernel takes the exact
    validate-before-mutate path (src/engine.cpp:171-190: consumers check every
    touched row, one extra grid exchange) on most coordinates. Results must
    still match the oracle."""
    rng = np.random.default_rng(404)
    n, p = 40_000, 8
    t = rng.exponential(size=n)
    status = (rng.random(n) < 0.7).astype(np.int64)
    if model == "finegray":  # competing rows: the weighted (forward-backward) kernel
        status[(status == 0) & (rng.random(n) < 0.5)] = 2
    outl = np.argsort(t)[:p]  # smallest times
    status[outl] = 0
    bulk = np.setdiff1d(np.arange(n), outl)
    rows, cols, vals = [], [], []
    eta = np.zeros(n)
    for j in range(p):
        r = rng.choice(bulk, size=2000, replace=False)
        v = np.round(rng.uniform(-3.0, 3.0, size=r.size), 2)
        v[v == 0] = 1.5
        eta[r] += 0.3 * v
        r = np.append(r, outl[j])
        v = np.append(v, 1000.0)
        o = np.argsort(r)
        rows.append(r[o])
        cols.append(np.full(r.size, j))
        vals.append(v[o])
    t = t / np.exp(eta)
    t[outl] = t.min() / 2.0 - np.arange(p) * 1e-9  # keep them last in time
    t = np.ceil(t * 1e6) / 1e6
    ds = orc.assemble(t, status, np.concatenate(rows), np.concatenate(cols), np.concatenate(vals), p)
    eng = capi.Engine(capi.Dataset.from_sorted(ds), model)
    ref = orc.OracleEngine(ds, model)
    r1 = eng.fit(penalty="l1", strength=1.0, max_cycles=6)
    r2 = ref.fit(penalty="l1", strength=1.0, max_cycles=6)
    assert r1["cycles"] == r2["cycles"]
    assert np.max(rel(r1["beta"], r2["beta"])) < TOL_BETA
    assert np.max(rel(r1["objective_trace"], r2["objective_trace"])) < TOL_DERIV
    assert np.abs(r1["beta"]).sum() * 1000.0 > 700.0  # the fast bound was exceeded


@pytest.mark.parametrize("model", ["cox", "finegray"])
def test_fit_overflow_mid_cycle_raises_like_reference(capi, model):
    """An accepted step that would push some |x'beta| past 700 raises
    OverflowError from fit (validate-before-mutate, src/engine.cpp:171-190);
    on the device the error is raised inside the cycle kernel, which then
    streams the rest of the cycle without work ('dry') and must end cleanly.
    The extreme value sits on a censored row with the smallest time (in no
    event's risk set), so beta follows the bulk and 1e5 * beta overflows."""
    rng = np.random.default_rng(77)
    n, p = 30_000, 6
    t = rng.exponential(size=n)
    status = (rng.random(n) < 0.7).astype(np.int64)
    if model == "finegray":  # competing rows: the weighted (forward-backward) kernel
        status[(status == 0) & (rng.random(n) < 0.5)] = 2
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
        orc.OracleEngine(ds, model).fit(penalty="none", max_cycles=5)
    with pytest.raises(capi.GssError) as e_dev:
        capi.Engine(capi.Dataset.from_sorted(ds), model).fit(penalty="none", max_cycles=5)
    assert e_ref.value.kind == "OverflowError"
    assert e_dev.value.kind == "OverflowError"
