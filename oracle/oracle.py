"""ctypes front end of the C oracle (oracle/oracle.c) plus a numpy restatement
of the reference's dataset assembly.

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline leg, always as the checker, never as the thing
measured or shipped.

`assemble` restates sort_and_block + SurvivalDataset::assemble
(/root/reference/proj/src/dataset.cpp:212-262, 172-210, 126-157):
rows sorted by decreasing time, ties by ascending original row id (optionally
grouped by ascending stratum first — strata are a rebuild feature, SURVEY.md
§8c), zero cells dropped, columns below 25% density stored sparse and marked
"indicator" when every stored value is 1.0.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "liboracle.so")

ORC_ERRORS = {0: None, 3: "DomainError", 6: "InvalidColumnError",
              7: "NonPositiveDenominatorError", 8: "OverflowError",
              9: "DegenerateCurveError"}


def build(force: bool = False) -> str:
    src = os.path.join(HERE, "oracle.c")
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < max(
            os.path.getmtime(src), os.path.getmtime(os.path.join(HERE, "oracle.h"))):
        subprocess.check_call(["gcc", "-std=c11", "-O2", "-fPIC", "-shared",
                               "-ffp-contract=off", src, "-o", LIB, "-lm"])
    return LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(build())
    return _lib


class OracleError(RuntimeError):
    def __init__(self, code: int, what: str):
        super().__init__(f"{ORC_ERRORS.get(code, code)}: {what}")
        self.code = code
        self.kind = ORC_ERRORS.get(code)


class _Data(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int64), ("p", ctypes.c_int64),
                ("times", ctypes.c_void_p), ("status", ctypes.c_void_p),
                ("col_ptr", ctypes.c_void_p), ("row_idx", ctypes.c_void_p),
                ("vals", ctypes.c_void_p), ("col_indicator", ctypes.c_void_p),
                ("stratum_start", ctypes.c_void_p)]


class _State(ctypes.Structure):
    _fields_ = [("fine_gray", ctypes.c_int), ("beta", ctypes.c_void_p),
                ("eta", ctypes.c_void_p), ("e", ctypes.c_void_p),
                ("fixed", ctypes.c_void_p), ("u", ctypes.c_void_p),
                ("g", ctypes.c_void_p), ("accepted", ctypes.c_int64),
                ("refreshes", ctypes.c_int64), ("recompute_interval", ctypes.c_int64)]


class _Fit(ctypes.Structure):
    _fields_ = [("objective", ctypes.c_double), ("cycles", ctypes.c_int64),
                ("converged", ctypes.c_int64), ("nonzero", ctypes.c_int64),
                ("skipped", ctypes.c_int64), ("violations", ctypes.c_int64)]


def _ptr(a):
    return None if a is None else a.ctypes.data


@dataclass
class Sorted:
    """Sorted dataset in the reference's in-memory layout (CSC over sorted rows)."""
    times: np.ndarray          # float64 [n]
    status: np.ndarray         # int32 [n]
    row_ids: np.ndarray        # int64 [n] original row id of each sorted position
    col_ptr: np.ndarray        # int64 [p+1]
    row_idx: np.ndarray        # int32 [nnz]
    vals: np.ndarray           # float64 [nnz]
    col_indicator: np.ndarray  # uint8 [p]
    stratum_start: np.ndarray | None = None  # uint8 [n]
    strata: np.ndarray | None = None         # int64 [n] stratum per sorted row

    @property
    def n(self):
        return len(self.times)

    @property
    def p(self):
        return len(self.col_ptr) - 1


def assemble(times, status, rows, cols, values, n_cols, strata=None) -> Sorted:
    times = np.asarray(times, dtype=np.float64)
    status = np.asarray(status, dtype=np.int32)
    rows = np.asarray(rows, dtype=np.int64)
    cols = np.asarray(cols, dtype=np.int64)
    values = np.asarray(values, dtype=np.float64)
    n = len(times)
    ids = np.arange(n, dtype=np.int64)
    keys = [ids, -times]
    if strata is not None:
        strata = np.asarray(strata, dtype=np.int64)
        keys.append(strata)
    order = np.lexsort(keys)                       # dataset.cpp:227-230
    pos_of = np.empty(n, dtype=np.int64)
    pos_of[order] = np.arange(n)
    keep = values != 0.0                           # dataset.cpp:254
    r = pos_of[rows[keep]]
    c = cols[keep]
    v = values[keep]
    o = np.lexsort((r, c))                         # per-column ascending rows
    r, c, v = r[o], c[o], v[o]
    counts = np.bincount(c, minlength=n_cols)
    col_ptr = np.zeros(n_cols + 1, dtype=np.int64)
    np.cumsum(counts, out=col_ptr[1:])
    ind = np.zeros(n_cols, dtype=np.uint8)
    for j in range(n_cols):                         # dataset.cpp:126-157
        seg = v[col_ptr[j]:col_ptr[j + 1]]
        dens = (len(seg) / n) if n else 0.0
        ind[j] = 1 if (dens < 0.25 and np.all(seg == 1.0)) else 0
    ss = None
    st_sorted = None
    if strata is not None:
        st_sorted = strata[order]
        ss = np.zeros(n, dtype=np.uint8)
        if n:
            ss[0] = 1
            ss[1:] = (st_sorted[1:] != st_sorted[:-1]).astype(np.uint8)
    return Sorted(times[order].copy(), status[order].copy(), order.astype(np.int64),
                  col_ptr, r.astype(np.int32), v.copy(), ind, ss, st_sorted)


class OracleEngine:
    """Serial restatement of survscan::Engine (engine.hpp:33-90)."""

    def __init__(self, ds: Sorted, model: str = "cox", recompute_interval: int = 100):
        self.ds = ds
        n, p = ds.n, ds.p
        self._keep = [ds.times, ds.status, ds.col_ptr, ds.row_idx, ds.vals,
                      ds.col_indicator, ds.stratum_start]
        self._d = _Data(n, p, _ptr(ds.times), _ptr(ds.status), _ptr(ds.col_ptr),
                        _ptr(ds.row_idx), _ptr(ds.vals), _ptr(ds.col_indicator),
                        _ptr(ds.stratum_start))
        self.beta = np.zeros(p + 1)
        self.eta = np.zeros(n + 1)
        self.e = np.ones(n + 1)
        self.fixed = np.zeros(p + 1)
        self.u = np.zeros(n + 1)
        self.g = np.ones(n + 1)
        fg = 1 if model in ("finegray", "fine_gray") else 0
        self._s = _State(fg, _ptr(self.beta), _ptr(self.eta), _ptr(self.e),
                         _ptr(self.fixed), _ptr(self.u), _ptr(self.g), 0, 0,
                         recompute_interval)
        self._check(lib().orc_init(ctypes.byref(self._d), ctypes.byref(self._s)), "init")

    @staticmethod
    def _check(rc, what):
        if rc:
            raise OracleError(rc, what)

    def load_beta(self, beta):
        b = np.ascontiguousarray(beta, dtype=np.float64)
        self._check(lib().orc_load_beta(ctypes.byref(self._d), ctypes.byref(self._s),
                                        ctypes.c_void_p(b.ctypes.data)), "load_beta")

    def update(self, j, delta):
        self._check(lib().orc_update(ctypes.byref(self._d), ctypes.byref(self._s),
                                     ctypes.c_int64(j), ctypes.c_double(delta)), "update")

    def grad_hessian(self, j):
        out = (ctypes.c_double * 5)()
        self._check(lib().orc_grad_hessian(
            ctypes.byref(self._d), ctypes.byref(self._s), ctypes.c_int64(j),
            ctypes.byref(out, 0), ctypes.byref(out, 8), ctypes.byref(out, 16),
            ctypes.byref(out, 24), ctypes.byref(out, 32)), "grad_hessian")
        return {"gradient": out[0], "hessian": out[1], "fixed_term": out[2],
                "grad_sum": out[3], "hess_sum": out[4]}

    def log_likelihood(self):
        out = ctypes.c_double()
        self._check(lib().orc_log_likelihood(ctypes.byref(self._d), ctypes.byref(self._s),
                                             ctypes.byref(out)), "log_likelihood")
        return out.value

    @property
    def accepted(self):
        return self._s.accepted

    @property
    def refreshes(self):
        return self._s.refreshes

    def fit(self, penalty="none", strength=0.0, exempt=(), tol=1e-6, max_cycles=1000,
            trust_init=1.0):
        kind = {"none": 0, "l1": 1, "l2": 2}[penalty]
        ex = np.zeros(self.ds.p + 1, dtype=np.uint8)
        for j in exempt:
            ex[j] = 1
        trace = np.zeros(max_cycles + 1)
        res = _Fit()
        self._check(lib().orc_fit(ctypes.byref(self._d), ctypes.byref(self._s),
                                  ctypes.c_int(kind), ctypes.c_double(strength),
                                  ctypes.c_void_p(ex.ctypes.data), ctypes.c_double(tol),
                                  ctypes.c_int64(max_cycles), ctypes.c_double(trust_init),
                                  ctypes.c_void_p(trace.ctypes.data), ctypes.byref(res)),
                    "fit")
        return {"beta": self.beta[:self.ds.p].copy(), "objective": res.objective,
                "cycles": res.cycles, "converged": bool(res.converged),
                "nonzero_count": res.nonzero, "skipped_steps": res.skipped,
                "monotonicity_violations": res.violations,
                "objective_trace": trace[:res.cycles + 1].copy()}


def coordinate_step(beta_j, grad, hess, kind, strength, penalized, halfwidth):
    """src/ccd.cpp:71-129 via the C restatement."""
    out = (ctypes.c_double * 3)()
    sk = ctypes.c_int()
    lib().orc_coordinate_step(ctypes.c_double(beta_j), ctypes.c_double(grad),
                              ctypes.c_double(hess), ctypes.c_int(kind),
                              ctypes.c_double(strength), ctypes.c_int(int(penalized)),
                              ctypes.c_double(halfwidth), ctypes.byref(out, 0),
                              ctypes.byref(out, 8), ctypes.byref(out, 16), ctypes.byref(sk))
    return {"new_beta": out[0], "applied": out[1], "new_halfwidth": out[2],
            "skipped": bool(sk.value)}
