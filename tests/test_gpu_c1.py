"""Config C1 (BASELINE.json configs[0]) on the reference's OWN data.

tests/golden/c1_ref.npz holds simulate_cox(n=100000, p=1000, density=0.01,
seed=1) as produced by the reference binary (src/simgen.cpp:108-122, written
out through its write_sparse_coo) and the reference's L1 fit at gamma=sqrt(2)
(src/ccd.cpp:131-184): 9 cycles, 975 nonzero, objective -998899.6307083
(tests/golden/make_c1.py).  The device fit must reproduce it: equal cycles
and nonzero count, objective within 1e-10, coefficients within 1e-8.
"""
import numpy as np
import pytest

from tests._common import TOL_BETA, TOL_DERIV, rel, rel_cond
from tests.golden.make_c1 import load

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def c1():
    return load()


@pytest.fixture(scope="module")
def dev(c1):
    from paper_2204_08183_b200 import capi
    return capi, capi.Dataset(c1["times"], c1["status"], c1["col_ptr"], c1["row_idx"])


@pytest.mark.parametrize("grid", [0, 7])
def test_c1_fit_matches_reference(c1, dev, grid):
    capi, dd = dev
    r = capi.Engine(dd, "cox").set_grid(grid).fit(penalty="l1", strength=float(c1["gamma"]),
                                                 tol=1e-6, max_cycles=1000)
    assert r["cycles"] == int(c1["fit_cycles"]) == 9
    assert r["nonzero_count"] == int(c1["fit_nonzero"]) == 975
    assert rel(r["objective"], float(c1["fit_objective"])) < TOL_DERIV
    assert abs(r["objective"] - (-998899.6307083)) < 1e-4
    assert np.max(rel(r["beta"], c1["fit_beta"])) < TOL_BETA
    assert np.max(rel(r["objective_trace"], c1["fit_trace"])) < TOL_DERIV


def test_c1_derivatives_at_probe(c1, dev):
    capi, dd = dev
    eng = capi.Engine(dd, "cox")
    eng.load_beta(c1["fit3_beta"])
    assert rel(eng.log_likelihood(), float(c1["probe_ll"])) < TOL_DERIV
    for j, g, h in zip(c1["probe_cols"], c1["probe_grad"], c1["probe_hess"]):
        gh = eng.grad_hessian(int(j))
        assert rel_cond(gh["gradient"], g, gh["fixed_term"]) < TOL_DERIV
        assert rel(gh["hessian"], h) < TOL_DERIV
