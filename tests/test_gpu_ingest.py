"""Device ingestion (gss_coo_sort: CUB radix sorts) vs the host sort of
dataset_from_coo (the reference's order, src/dataset.cpp:190-262): the sorted
layouts must be identical (content hash over times, status, CSC structure,
values and stratum starts, plus the row ids), and the first-error semantics
(row / column / value / duplicate) must match message for message."""
import os

import numpy as np
import pytest

import survscan

pytestmark = pytest.mark.gpu


def _both(*args, **kw):
    os.environ["SURVSCAN_HOST_INGEST"] = "1"
    try:
        host = survscan.dataset_from_coo(*args, **kw)
    finally:
        del os.environ["SURVSCAN_HOST_INGEST"]
    dev = survscan.dataset_from_coo(*args, **kw)
    return host, dev


def _err(*args, **kw):
    msgs = []
    for host in (True, False):
        if host:
            os.environ["SURVSCAN_HOST_INGEST"] = "1"
        try:
            with pytest.raises(survscan.SurvscanError) as ei:
                survscan.dataset_from_coo(*args, **kw)
            msgs.append(str(ei.value))
        finally:
            os.environ.pop("SURVSCAN_HOST_INGEST", None)
    return msgs


def _data(n, p, density, seed, ties=100.0, strata=None, zeros=False):
    rng = np.random.default_rng(seed)
    t = np.ceil(rng.exponential(size=n) * ties) / ties
    t[rng.random(n) < 0.01] = 0.0
    s = rng.integers(0, 3, n)
    k = int(n * p * density)
    rows = rng.integers(0, n, k)
    cols = rng.integers(0, p, k)
    key = np.unique(cols * n + rows)  # distinct cells
    rng.shuffle(key)
    rows, cols = key % n, key // n
    vals = np.where(rng.random(len(key)) < 0.5, 1.0, rng.normal(size=len(key)))
    if zeros:
        vals[rng.random(len(vals)) < 0.1] = 0.0
    st = None if strata is None else rng.integers(-3, strata, n)
    return t, s, rows.astype(np.int64), cols.astype(np.int64), vals, p, st


@pytest.mark.parametrize("n,p,density,seed,ties,strata,zeros", [
    (1, 1, 1.0, 0, 10.0, None, False),
    (1000, 7, 0.05, 1, 10.0, None, False),
    (20000, 40, 0.01, 2, 100.0, 9, True),
    (300001, 30, 0.003, 3, 1000.0, 50, False),
])
def test_device_ingest_matches_host(n, p, density, seed, ties, strata, zeros):
    t, s, rows, cols, vals, p, st = _data(n, p, density, seed, ties, strata, zeros)
    host, dev = _both(t, s, rows, cols, vals, p, st)
    assert dev.n == host.n and dev.p == host.p and dev.nnz_total == host.nnz_total
    assert dev.content_hash == host.content_hash
    np.testing.assert_array_equal(dev.times, host.times)
    np.testing.assert_array_equal(dev.status, host.status)
    for j in range(min(p, 5)):
        for i in (0, n // 2, n - 1):
            assert dev.covariate(i, j) == host.covariate(i, j)


def test_device_ingest_negative_zero_time_ties_with_zero():
    t = np.array([0.0, -0.0, 0.0, 1.0])
    host, dev = _both(t, np.array([1, 1, 0, 1]), np.array([0, 1, 2, 3]), np.zeros(4, np.int64),
                      np.ones(4), 1)
    assert dev.content_hash == host.content_hash


def test_device_ingest_errors_match_host():
    t, s = np.array([3.0, 2.0, 1.0]), np.array([1, 0, 1])
    one = np.ones(3)
    # first failing entry in input order wins, with its first failing check
    for rows, cols, vals in [
        (np.array([0, 5, 1]), np.array([0, 0, 9]), one),          # row out of range
        (np.array([0, 1, -1]), np.array([0, 9, 0]), one),         # column before row
        (np.array([0, 1, 2]), np.array([0, 0, 0]), np.array([1.0, np.inf, 1.0])),
        (np.array([2, 0, 2]), np.array([1, 0, 1]), one),          # duplicate cell
    ]:
        host_msg, dev_msg = _err(t, s, rows, cols, vals, 2)
        assert host_msg == dev_msg, (host_msg, dev_msg)
