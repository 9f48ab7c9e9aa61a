"""Ring-protocol stress on the device: tile groups running at very different
speeds must never consume a stage two ring cycles early (mbarrier parity
aliasing).  GSS_DEBUG=1 makes the consumers skip the tile work (the same path
a fit takes after a device error, `dry` mode), so groups race ahead of each
other; before the issue-count check this deadlocked at C2 size.
"""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def capi():
    from paper_2204_08183_b200 import capi as C
    assert C.lib().gss_device_count() > 0
    return C


def _engine(capi, n, p, debug=None):
    sim = capi.SimData(n, p, 0.01, 0.8, 2, 0.9, 1000.0)
    ds = capi.Dataset(sim.times, sim.status, sim.col_ptr, sim.row_idx)
    old = os.environ.get("GSS_DEBUG")
    try:
        if debug is not None:
            os.environ["GSS_DEBUG"] = str(debug)
        eng = capi.Engine(ds, "cox")  # GSS_DEBUG is read at engine creation
    finally:
        if old is None:
            os.environ.pop("GSS_DEBUG", None)
        else:
            os.environ["GSS_DEBUG"] = old
    return sim, ds, eng


@pytest.mark.parametrize("debug", [1, 17])
def test_groups_racing_ahead_do_not_alias_stages(capi, debug):
    _, _, eng = _engine(capi, 10_000_000, 256, debug)
    # no tile work: the objective never moves (one cycle), but the launch of
    # 257 slots must complete cleanly
    r = eng.fit(penalty="l1", strength=2 ** 0.5, tol=1e-300, max_cycles=3)
    assert r["cycles"] >= 1


def test_normal_fit_after_debug_engine_is_unaffected(capi):
    sim, ds, eng = _engine(capi, 2_000_000, 32)
    r1 = eng.fit(penalty="l1", strength=2 ** 0.5, max_cycles=4)
    r2 = capi.Engine(ds, "cox").fit(penalty="l1", strength=2 ** 0.5, max_cycles=4)
    assert np.array_equal(r1["beta"], r2["beta"])  # bitwise deterministic
