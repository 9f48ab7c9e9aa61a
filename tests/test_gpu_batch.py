"""Batched multi-fit (gss_fit_batch): one cycle-kernel launch advances every
active fit by one CCD cycle, each on its own share of the SMs (SURVEY.md §8f
row 1).  Every batched fit must equal the same fit run
alone on the same number of CTAs bit for bit (same summation order), and the
oracle within the north-star tolerances."""
import numpy as np
import pytest

from oracle import oracle as orc
from tests._common import TOL_BETA, TOL_DERIV, rel
from tests.test_gpu_parity import _random_sorted

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def capi():
    from paper_2204_08183_b200 import capi as C
    assert C.lib().gss_device_count() > 0
    return C


def _folds(n, k, seed):
    rng = np.random.default_rng(seed)
    fold = rng.permutation(n) % k
    return [(fold != f).astype(np.uint8) for f in range(k)]


@pytest.mark.parametrize("model,strata", [("cox", None), ("cox", 12), ("finegray", None)])
def test_batch_equals_single_fits(capi, model, strata):
    ds = _random_sorted(120_000, 12, 0.03, seed=808, quant=60.0, strata=strata,
                        competing=0.5 if model == "finegray" else 0.0)
    dd = capi.Dataset.from_sorted(ds)
    masks = _folds(ds.n, 5, 3)
    lams = [0.5, 1.0, 2.0, 4.0, 8.0, 16.0]
    # 5 folds x 6 lambdas = 30 fits, 8 active at a time (18 CTAs each)
    specs = [(m, g) for m in masks for g in lams]
    engines = [capi.Engine(dd, model, row_mask=m) for m, _ in specs]
    res, dev_s = capi.fit_batch(engines, "l1", [g for _, g in specs], max_active=8)
    assert dev_s > 0
    share = engines[0].grid  # restored after the batch
    assert share == capi.Engine(dd, model).grid
    for (m, g), r in list(zip(specs, res))[::7]:
        assert not isinstance(r, Exception), r
        alone = capi.Engine(dd, model, row_mask=m).set_grid(148 // 8).fit(penalty="l1", strength=g)
        assert r["cycles"] == alone["cycles"]
        assert np.array_equal(r["beta"], alone["beta"])
        assert r["objective"] == alone["objective"]
    # and the oracle on the materialised fold
    (m, g), r = specs[9], res[9]
    keep = np.nonzero(m)[0]
    cols = np.repeat(np.arange(ds.p), np.diff(ds.col_ptr))
    remap = -np.ones(ds.n, np.int64)
    remap[keep] = np.arange(len(keep))
    sel = remap[ds.row_idx] >= 0
    st = None if ds.strata is None else ds.strata[keep]
    sub = orc.assemble(ds.times[keep], ds.status[keep], remap[ds.row_idx[sel]], cols[sel],
                       ds.vals[sel], ds.p, strata=st)
    r2 = orc.OracleEngine(sub, model).fit(penalty="l1", strength=g)
    assert r["cycles"] == r2["cycles"]
    assert np.max(rel(r["beta"], r2["beta"])) < TOL_BETA
    assert rel(r["objective"], r2["objective"]) < TOL_DERIV


def test_batch_mixed_kinds_and_failures(capi):
    """Weighted (Fine-Gray with competing rows) and unweighted fits in one
    call go to separate launches; a failing fit reports its own status and the
    others still finish."""
    ds = _random_sorted(60_000, 6, 0.04, seed=5, quant=30.0, competing=0.4)
    dd = capi.Dataset.from_sorted(ds)
    no_comp = (ds.status != 2).astype(np.uint8)
    engines = [capi.Engine(dd, "finegray"), capi.Engine(dd, "finegray", row_mask=no_comp),
               capi.Engine(dd, "finegray"), capi.Engine(dd, "cox", row_mask=no_comp)]
    res, _ = capi.fit_batch(engines, "l1", [1.0, 1.0, -1.0, 2.0])
    assert isinstance(res[2], capi.GssError) and res[2].kind == "DomainError"
    for i in (0, 1, 3):
        ref = [capi.Engine(dd, "finegray"), capi.Engine(dd, "finegray", row_mask=no_comp), None,
               capi.Engine(dd, "cox", row_mask=no_comp)][i]
        r = ref.set_grid(148 // 3).fit(penalty="l1", strength=[1.0, 1.0, 0, 2.0][i])
        assert res[i]["cycles"] == r["cycles"]
        assert np.max(rel(res[i]["beta"], r["beta"])) < 1e-12
