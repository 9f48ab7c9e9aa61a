"""Config C5 on one GPU: the patient-sharded protocol (paper_2204_08183_b200/
sharded.py) with every shard emulated in one process (LocalExchange) must
reproduce the unsharded computation — derivatives and log-likelihood to the
north-star tolerance, and fits with the same cycle counts and coefficients."""
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
