"""The drop-in boundary without a GPU: the C ABI library exports every entry
point include/gss.h declares, the C++ mirror + pybind module load, and the
host-side dataset operations behave like the reference's (CPU only)."""
import ctypes
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared(header):
    txt = open(os.path.join(ROOT, "include", header)).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(gss_[a-z0-9_]+)\s*\(", txt)))


@pytest.mark.parametrize("header", ["gss.h", "gss_sim.h"])
def test_c_abi_exports_every_declared_symbol(header):
    from paper_2204_08183_b200 import capi
    lib = capi.lib()
    names = _declared(header)
    assert len(names) >= (20 if header == "gss.h" else 3)
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing


def test_no_device_fails_loudly():
    from paper_2204_08183_b200 import capi
    if capi.lib().gss_device_count() > 0:
        pytest.skip("a device is present")
    with pytest.raises(capi.GssError) as ei:
        capi.Dataset(np.array([1.0]), np.array([1]), np.array([0, 0]), np.zeros(0, np.int32))
    assert ei.value.kind == "NoDeviceError"


def test_cpp_mirror_and_module_load():
    import survscan
    assert "sm_100a" in survscan.__version__
    for name in survscan.__all__:
        assert hasattr(survscan, name), name


def test_dataset_sorting_and_accessors():
    """sort_and_block: time desc, row id asc; absent cells are zeros
    (src/dataset.cpp:212-262)."""
    import survscan
    t = np.array([5.0, 3.0, 1.0, 4.0, 3.0])
    s = np.array([1, 0, 1, 2, 1])
    ds = survscan.dataset_from_coo(t, s, rows=np.array([0, 2, 4, 1]), cols=np.array([0, 1, 1, 0]),
                                   values=np.array([1.0, 2.0, 0.0, 1.0]), n_cols=3)
    assert ds.n == 5 and ds.p == 3 and ds.has_competing and ds.n_events == 3
    assert list(ds.times) == [5.0, 4.0, 3.0, 3.0, 1.0]
    assert list(ds.status) == [1, 2, 0, 1, 1]  # tie at 3.0 broken by row id (1 before 4)
    assert ds.nnz_total == 3  # the explicit zero is dropped
    assert ds.covariate(0, 0) == 1.0 and ds.covariate(2, 0) == 1.0 and ds.covariate(4, 1) == 2.0
    sub = ds.subset_rows([0, 2, 2, 4], fresh_row_ids=True)
    assert sub.n == 4 and list(sub.times) == [5.0, 3.0, 3.0, 1.0]
    with pytest.raises(survscan.SurvscanError):
        ds.subset_rows([2, 2], fresh_row_ids=False)
    with pytest.raises(survscan.SurvscanError):
        survscan.dataset_from_coo(t, s, rows=np.array([0, 0]), cols=np.array([1, 1]),
                                  values=np.array([1.0, 1.0]), n_cols=3)  # duplicate cell


def test_dataset_roundtrip_and_hash(tmp_path):
    import survscan
    ds, _, _ = survscan.simulate_finegray(n=300, p=5, density=0.2, seed=5, censoring_quantile=0.9)
    again, _, _ = survscan.simulate_finegray(n=300, p=5, density=0.2, seed=5,
                                             censoring_quantile=0.9)
    assert again.content_hash == ds.content_hash
    obs, coo = str(tmp_path / "d.obs"), str(tmp_path / "d.coo")
    survscan.write_sparse_coo(ds, obs, coo)
    assert survscan.load_sparse_coo(obs, coo).content_hash == ds.content_hash
    csv = str(tmp_path / "d.csv")
    survscan.write_dense_csv(ds, csv)
    assert survscan.load_dense_csv(csv).content_hash == ds.content_hash
    with pytest.raises(survscan.SurvscanError):
        survscan.load_dense_csv(str(tmp_path / "missing.csv"))


def test_stratified_dataset_layout():
    import survscan
    t = np.array([1.0, 2.0, 3.0, 4.0])
    ds = survscan.dataset_from_coo(t, np.array([1, 1, 1, 1]), rows=np.array([0]),
                                   cols=np.array([0]), values=np.array([1.0]), n_cols=1,
                                   strata=np.array([1, 0, 1, 0]))
    # stratum 0 rows (ids 1, 3) first, each stratum by time desc
    assert list(ds.times) == [4.0, 2.0, 3.0, 1.0]


def test_auto_grid_endpoints():
    import survscan
    g = survscan.auto_grid(2.0)
    assert len(g) == 10 and g[0] == 2.0 / 1000.0 and g[-1] == 2.0
    assert all(a < b for a, b in zip(g, g[1:]))
