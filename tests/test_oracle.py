"""Pins the C oracle (oracle/oracle.c) against the golden fixtures produced by
the real reference (tests/golden/make_golden.py) — CPU only."""
import numpy as np
import pytest

from oracle import oracle as orc
from tests._common import TOL_BETA, TOL_DERIV, cases, fit_cases, load, raw, rel, rel_cond


def _engine(c, **kw):
    args, strata = raw(c)
    ds = orc.assemble(*args, strata=strata)
    return ds, orc.OracleEngine(ds, str(c["model"]), **kw)


@pytest.mark.parametrize("name", cases("ka_"))
def test_known_answers(name):
    c = load(name)
    ds, eng = _engine(c)
    gh = eng.grad_hessian(0)
    assert gh["gradient"] == pytest.approx(float(c["grad0"][0]), abs=1e-15)
    assert gh["hessian"] == pytest.approx(float(c["hess0"][0]), abs=1e-15)
    assert eng.log_likelihood() == pytest.approx(float(c["ll0"]), rel=1e-15, abs=1e-15)
    for key, val in (("want_grad", gh["gradient"]), ("want_hess", gh["hessian"])):
        if key in c:
            assert val == pytest.approx(float(c[key]), abs=1e-15)
    if "want_fixed" in c:
        assert gh["fixed_term"] == float(c["want_fixed"])
    if "want_ll" in c:
        assert eng.log_likelihood() == pytest.approx(float(c["want_ll"]), abs=1e-15)


GOLD = [n for n in cases() if not n.startswith("ka_")]


@pytest.mark.parametrize("name", GOLD)
def test_derivatives_and_loglik(name):
    c = load(name)
    ds, eng = _engine(c)
    p = ds.p
    eng.load_beta(c["beta_probe"])
    assert rel(eng.log_likelihood(), c["ll"]) < TOL_DERIV
    for j in range(p):
        gh = eng.grad_hessian(j)
        assert rel_cond(gh["gradient"], c["grad"][j], gh["fixed_term"]) < TOL_DERIV
        assert rel(gh["hessian"], c["hess"][j]) < TOL_DERIV
    eng.load_beta(np.zeros(p))
    assert rel(eng.log_likelihood(), c["ll0"]) < TOL_DERIV


@pytest.mark.parametrize("name", GOLD)
def test_fits(name):
    c = load(name)
    for k, pen, lam in fit_cases(c):
        ds, eng = _engine(c)
        r = eng.fit(penalty=pen, strength=lam, max_cycles=1000 if "strata" not in c else 200)
        assert r["cycles"] == int(c[f"fit{k}_cycles"]), (pen, lam)
        assert np.max(rel(r["beta"], c[f"fit{k}_beta"])) < TOL_BETA, (pen, lam)
        assert rel(r["objective"], c[f"fit{k}_objective"]) < TOL_DERIV
        assert np.max(rel(r["objective_trace"], c[f"fit{k}_trace"])) < TOL_DERIV


def test_coordinate_step_known_answers():
    """tests/test_ccd.cpp:31-105 restated."""
    cs = orc.coordinate_step
    # Newton exactness: g=1, h=-2 -> raw 0.5 within halfwidth 1
    r = cs(0.0, 1.0, -2.0, 0, 0.0, False, 1.0)
    assert r["applied"] == 0.5 and r["new_halfwidth"] == 1.0
    # trust clip
    r = cs(0.0, 10.0, -1.0, 0, 0.0, False, 1.0)
    assert r["applied"] == 1.0 and r["new_halfwidth"] == 2.0
    # L1 parked at zero
    r = cs(0.0, 0.5, -1.0, 1, 1.0, True, 1.0)
    assert r["applied"] == 0.0 and r["new_halfwidth"] == 0.5 and not r["skipped"]
    # L1 leaving zero: g_eff = 3 - 1
    r = cs(0.0, 3.0, -4.0, 1, 1.0, True, 1.0)
    assert r["applied"] == 0.5
    # sign crossing clamps to -beta
    r = cs(0.2, -5.0, -1.0, 1, 1.0, True, 10.0)
    assert r["new_beta"] == 0.0 and r["applied"] == -0.2
    # flat but sloped: skipped, halfwidth kept
    r = cs(0.0, 1.0, 0.0, 0, 0.0, False, 0.7)
    assert r["skipped"] and r["new_halfwidth"] == 0.7
    # flat and zero: halve
    r = cs(0.0, 0.0, 0.0, 0, 0.0, False, 0.7)
    assert not r["skipped"] and r["new_halfwidth"] == 0.35
    # L2 rescues a flat coordinate
    r = cs(0.0, 1.0, 0.0, 2, 2.0, True, 10.0)
    assert r["applied"] == pytest.approx(2.0)
    # halfwidth floor
    r = cs(0.0, 0.0, 0.0, 0, 0.0, False, 1e-300)
    assert r["new_halfwidth"] == 1e-300


def test_cox_rejects_competing_rows():
    c = load("fg_small")
    args, _ = raw(c)
    ds = orc.assemble(*args)
    with pytest.raises(orc.OracleError) as ei:
        orc.OracleEngine(ds, "cox")
    assert ei.value.kind == "DomainError"


def test_overflow_is_rejected_atomically():
    c = load("cox_small")
    ds, eng = _engine(c)
    beta = np.zeros(ds.p)
    beta[0] = 800.0
    with pytest.raises(orc.OracleError) as ei:
        eng.load_beta(beta)
    assert ei.value.kind == "OverflowError"
    assert np.all(eng.eta[:ds.n] == 0.0)
    with pytest.raises(orc.OracleError):
        eng.update(0, 750.0)
    assert np.all(eng.eta[:ds.n] == 0.0) and eng.accepted == 0


def test_finegray_without_competing_is_cox_bitwise():
    """tests/test_engine.cpp:293-310."""
    c = load("cox_small")
    args, _ = raw(c)
    ds = orc.assemble(*args)
    a = orc.OracleEngine(ds, "cox")
    b = orc.OracleEngine(ds, "finegray")
    a.load_beta(c["beta_probe"])
    b.load_beta(c["beta_probe"])
    for j in range(ds.p):
        assert a.grad_hessian(j) == b.grad_hessian(j)
    assert a.log_likelihood() == b.log_likelihood()


def test_oracle_on_reference_c1_data():
    """The C oracle on config C1's reference-generated data (tests/golden/
    c1_ref.npz, make_c1.py) reproduces the reference's 3-cycle fit."""
    from tests.golden.make_c1 import load as load_c1
    c1 = load_c1()
    ds = orc.Sorted(c1["times"], c1["status"], np.asarray(c1["row_ids"], np.int64),
                    c1["col_ptr"], c1["row_idx"], np.ones(len(c1["row_idx"])),
                    np.ones(len(c1["col_ptr"]) - 1, np.uint8))
    r = orc.OracleEngine(ds, "cox").fit(penalty="l1", strength=float(c1["gamma"]), max_cycles=3)
    assert r["cycles"] == 3
    assert np.max(rel(r["beta"], c1["fit3_beta"])) < 1e-8
    assert rel(r["objective"], float(c1["fit3_objective"])) < 1e-10
