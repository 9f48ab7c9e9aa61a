"""Parity at the geometry the full-size fits run: many tiles per CTA.

At the benchmark sizes (C2: 4883 tiles on 148 CTAs) every CTA holds ~33
tiles, all tile groups of the consumer warps work, the control warp's
incremental carry scan runs across tiles, and CTAs beyond 64 (Cox) / 40
(Fine-Gray) tiles keep their per-tile records in global memory.  Small test
inputs give one tile per CTA unless the grid is capped: `Engine.set_grid`
(gss_engine_set_grid) puts the whole range on 1, 2, 3 or 7 CTAs here, so the
same code paths run on inputs the C oracle (oracle/oracle.c, pinned to the
reference's golden fixtures) checks in seconds.

Reference semantics: scan_kernels.hpp:74-214 (fused scan), engine.cpp:162-242
(update/finish), ccd.cpp:71-184 (CCD), censoring.cpp:39-90 (IPCW);
tests/test_engine.cpp:85-123 (parity vs the O(N^2) oracle at 1e-10).
"""
import numpy as np
import pytest

from oracle import oracle as orc
from tests._common import TOL_BETA, TOL_DERIV, cases, fit_cases, load, raw, rel, rel_cond
from tests.test_gpu_parity import _random_sorted

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def capi():
    from paper_2204_08183_b200 import capi as C
    assert C.lib().gss_device_count() > 0
    return C


GOLD = [n for n in cases() if not n.startswith("ka_")]


def _check_derivs(eng, ref, p, tol=TOL_DERIV):
    assert rel(eng.log_likelihood(), ref.log_likelihood()) < tol
    for j in range(p):
        a, b = eng.grad_hessian(j), ref.grad_hessian(j)
        assert rel_cond(a["gradient"], b["gradient"], b["fixed_term"]) < tol, j
        assert rel(a["hessian"], b["hessian"]) < tol, j
    allg = eng.grad_hessian_all()
    for j in range(p):
        b = ref.grad_hessian(j)
        assert rel_cond(allg["gradient"][j], b["gradient"], b["fixed_term"]) < tol, j
        assert rel(allg["hessian"][j], b["hessian"]) < tol, j


def _check_fit(r1, r2):
    assert r1["cycles"] == r2["cycles"]
    assert np.max(rel(r1["beta"], r2["beta"])) < TOL_BETA
    assert np.max(rel(r1["objective_trace"], r2["objective_trace"])) < TOL_DERIV


@pytest.mark.parametrize("grid", [1, 3])
@pytest.mark.parametrize("name", GOLD)
def test_goldens_on_few_ctas(capi, name, grid):
    """The reference's golden derivatives and fits with every tile of the
    dataset on 1 or 3 CTAs (all four Cox / both Fine-Gray tile groups)."""
    c = load(name)
    args, strata = raw(c)
    ds = orc.assemble(*args, strata=strata)
    dd = capi.Dataset.from_sorted(ds)
    eng = capi.Engine(dd, str(c["model"])).set_grid(grid)
    assert 1 <= eng.grid <= grid
    eng.load_beta(c["beta_probe"])
    assert rel(eng.log_likelihood(), c["ll"]) < TOL_DERIV
    for j in range(ds.p):
        gh = eng.grad_hessian(j)
        assert rel_cond(gh["gradient"], c["grad"][j], gh["fixed_term"]) < TOL_DERIV, j
        assert rel(gh["hessian"], c["hess"][j]) < TOL_DERIV, j
    max_cycles = 200 if "strata" in c else 1000
    for k, pen, lam in fit_cases(c):
        e2 = capi.Engine(dd, str(c["model"])).set_grid(grid)
        r = e2.fit(penalty=pen, strength=lam, max_cycles=max_cycles)
        assert r["cycles"] == int(c[f"fit{k}_cycles"]), (pen, lam)
        assert np.max(rel(r["beta"], c[f"fit{k}_beta"])) < TOL_BETA, (pen, lam)
        assert np.max(rel(r["objective_trace"], c[f"fit{k}_trace"])) < TOL_DERIV


# (model, n, p, quant, strata, valued, grid): tiles per CTA = ceil(n / 2048) / grid
CAPPED = [
    ("cox", 300_001, 10, 100.0, None, False, 1),   # 147 tiles on one CTA: global records
    ("cox", 300_001, 10, 100.0, None, False, 3),   # 49 per CTA: shared-memory records
    ("cox", 200_000, 8, None, None, True, 2),      # valued columns, 49 per CTA
    ("cox", 160_000, 8, 30.0, 9, False, 7),        # strata inside CTA ranges
    ("cox", 140_000, 8, 30.0, 40, True, 1),        # many strata, valued, 69 tiles on one CTA
    ("finegray", 200_000, 8, 60.0, None, False, 2),  # 49 per CTA > 40: global records
    ("finegray", 150_000, 8, None, None, True, 7),
    ("finegray", 120_000, 6, 20.0, 6, False, 3),
    ("finegray", 100_000, 6, 20.0, 25, True, 1),
]


@pytest.mark.parametrize("model,n,p,quant,strata,valued,grid", CAPPED)
def test_many_tiles_per_cta_vs_oracle(capi, model, n, p, quant, strata, valued, grid):
    ds = _random_sorted(n, p, 0.02, seed=n + 13 * p + grid, quant=quant, strata=strata,
                        valued=valued, competing=0.5 if model == "finegray" else 0.0)
    dd = capi.Dataset.from_sorted(ds)
    ref = orc.OracleEngine(ds, model)
    eng = capi.Engine(dd, model).set_grid(grid)
    beta = np.random.default_rng(n).uniform(-0.4, 0.4, size=p)
    ref.load_beta(beta)
    eng.load_beta(beta)
    _check_derivs(eng, ref, p)
    # CCD: pending-update patch, fused records, in-range carry scan, refresh
    e2 = capi.Engine(dd, model, recompute_interval=7).set_grid(grid)
    r2 = orc.OracleEngine(ds, model, recompute_interval=7)
    _check_fit(e2.fit(penalty="l1", strength=1.5, max_cycles=6),
               r2.fit(penalty="l1", strength=1.5, max_cycles=6))


@pytest.mark.parametrize("model", ["cox", "finegray"])
@pytest.mark.parametrize("grid", [2, 0])
def test_dense_columns_list_fallback(capi, model, grid):
    """Dense storage (density >= 25%, SparseColumn::make dataset.cpp:126-157):
    the 60%, 30% (all ones, hence valued) and 90% columns are read row-wise
    from the device dense pool by the scan, the pending update and the
    next-slot records.  The 20% column stays sparse but overflows the
    256-entry shared-memory list of a 2048-row tile slice, so the consumers
    read its slice from global memory.  Sparse indicator columns between."""
    rng = np.random.default_rng(99 + grid)
    n, p = 120_000, 6
    rows, cols, vals = [], [], []
    for j, dens in enumerate([0.6, 0.3, 0.01, 0.2, 0.02, 0.9]):
        r = np.sort(rng.choice(n, size=int(dens * n), replace=False))
        v = np.ones(r.size) if j in (1, 2, 4) else np.round(rng.normal(size=r.size), 2)
        v[v == 0] = 0.25
        rows.append(r)
        cols.append(np.full(r.size, j))
        vals.append(v * (0.3 if j in (0, 5) else 1.0))
    t = np.ceil(rng.exponential(size=n) * 80) / 80
    status = (rng.random(n) < 0.7).astype(np.int64)
    if model == "finegray":
        status[(status == 0) & (rng.random(n) < 0.5)] = 2
    ds = orc.assemble(t, status, np.concatenate(rows), np.concatenate(cols),
                      np.concatenate(vals), p)
    assert ds.col_indicator.tolist() == [0, 0, 1, 0, 1, 0]
    dd = capi.Dataset.from_sorted(ds)
    ref = orc.OracleEngine(ds, model)
    eng = capi.Engine(dd, model).set_grid(grid)
    beta = np.array([0.1, -0.2, 0.3, 0.05, -0.1, 0.08])
    ref.load_beta(beta)
    eng.load_beta(beta)
    _check_derivs(eng, ref, p)
    _check_fit(capi.Engine(dd, model).set_grid(grid).fit(penalty="l1", strength=2.0,
                                                         max_cycles=5),
               orc.OracleEngine(ds, model).fit(penalty="l1", strength=2.0, max_cycles=5))


@pytest.mark.parametrize("model,strata", [("cox", None), ("cox", 100), ("finegray", None),
                                          ("finegray", 30)])
def test_ccd_fit_2m_rows_vs_oracle(capi, model, strata):
    """CCD fits at N=2M (977 tiles: ~7 per CTA on the full grid), Breslow
    ties, with and without strata: equal cycle counts to convergence (tol
    1e-6, ccd.cpp:172-173), beta within 1e-8, objective traces within 1e-10."""
    ds = _random_sorted(2_000_000, 16, 0.01, seed=2024 + (strata or 0), quant=500.0,
                        strata=strata, competing=0.5 if model == "finegray" else 0.0)
    dd = capi.Dataset.from_sorted(ds)
    r1 = capi.Engine(dd, model).fit(penalty="l1", strength=3.0, max_cycles=100)
    r2 = orc.OracleEngine(ds, model).fit(penalty="l1", strength=3.0, max_cycles=100)
    assert r1["converged"] and r2["converged"]
    _check_fit(r1, r2)
    assert r1["nonzero_count"] == r2["nonzero_count"]


def _collinear(n, p, seed, competing=0.0):
    """Nearly collinear indicator columns (a shared 3% row set plus 0.3% own
    rows each): cyclic coordinate descent crawls, so a fit runs its whole
    cycle budget with every coordinate accepted every cycle."""
    rng = np.random.default_rng(seed)
    base = rng.choice(n, size=int(0.03 * n), replace=False)
    rows, cols = [], []
    for j in range(p):
        extra = rng.choice(n, size=int(0.003 * n), replace=False)
        r = np.unique(np.concatenate([base[rng.random(base.size) < 0.97], extra]))
        rows.append(r)
        cols.append(np.full(r.size, j))
    rows, cols = np.concatenate(rows), np.concatenate(cols)
    eta = np.zeros(n)
    np.add.at(eta, rows, 0.05)
    t = np.ceil(rng.exponential(size=n) / np.exp(eta) * 200) / 200
    st = (rng.random(n) < 0.7).astype(np.int64)
    if competing:
        st[(st == 0) & (rng.random(n) < competing)] = 2
    return orc.assemble(t, st, rows, cols, np.ones(len(rows)), p)


@pytest.mark.parametrize("model", ["cox", "finegray"])
def test_long_fit_frequent_refresh_vs_oracle(capi, model):
    """A long fit: 60 cycles x 24 accepted coordinates with
    recompute_interval=5 (288 in-kernel refreshes, src/engine.cpp:217).  The
    in-kernel refresh rebuilds exp(eta) from the incrementally maintained eta;
    the reference rebuilds eta = X beta (engine.cpp:156-160).  The drift must
    stay inside the coefficient tolerance over the whole fit."""
    ds = _collinear(250_000, 24, 606, competing=0.5 if model == "finegray" else 0.0)
    dd = capi.Dataset.from_sorted(ds)
    eng = capi.Engine(dd, model, recompute_interval=5).set_grid(5)
    ref = orc.OracleEngine(ds, model, recompute_interval=5)
    r1 = eng.fit(penalty="l2", strength=50.0, tol=1e-13, max_cycles=60)
    r2 = ref.fit(penalty="l2", strength=50.0, tol=1e-13, max_cycles=60)
    assert r2["cycles"] == 60 and not r2["converged"]
    _check_fit(r1, r2)
    acc, refreshes = eng.counters()
    assert acc == ref.accepted == 1440
    assert refreshes == ref.refreshes == 288
    # state after the fit: derivatives at the fitted beta still agree
    for j in (0, 11, 23):
        a, b = eng.grad_hessian(j), ref.grad_hessian(j)
        assert rel_cond(a["gradient"], b["gradient"], b["fixed_term"]) < TOL_DERIV
        assert rel(a["hessian"], b["hessian"]) < TOL_DERIV


def test_regrid_keeps_results(capi):
    """Re-partitioning an engine between calls (set_grid) keeps the state:
    the same derivatives (to summation order) on 1, 5, 64 and all CTAs."""
    ds = _random_sorted(180_000, 5, 0.03, seed=31, quant=40.0, strata=3)
    eng = capi.Engine(capi.Dataset.from_sorted(ds), "cox")
    eng.load_beta(np.array([0.2, -0.1, 0.3, 0.05, -0.2]))
    base = [eng.grad_hessian(j)["gradient"] for j in range(5)] + [eng.log_likelihood()]
    for g in (1, 5, 64, 0):
        eng.set_grid(g)
        got = [eng.grad_hessian(j)["gradient"] for j in range(5)] + [eng.log_likelihood()]
        assert np.max(rel(got, base)) < 1e-12
