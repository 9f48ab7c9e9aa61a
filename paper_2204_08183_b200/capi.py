"""ctypes binding of the C ABI (include/gss.h) — the thin FFI layer a host
language uses to drive the device engine.  No fallback: if libgss.so is
missing or no sm_100 device is present, calls raise.

This is also the binding shown in INTEGRATION.md for callers that cannot use
the pybind module.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

from .build import LIBGSS

GSS_STATUS = {
    1: "ParseError", 2: "SchemaError", 3: "DomainError", 4: "IndexError",
    5: "DuplicateEntryError", 6: "InvalidColumnError",
    7: "NonPositiveDenominatorError", 8: "OverflowError", 9: "DegenerateCurveError",
    10: "EmptyFoldError", 100: "CudaError", 101: "NoDeviceError", 102: "OutOfMemoryError",
}

EXPORTS = [
    "gss_last_error", "gss_version", "gss_device_count", "gss_dataset_pack",
    "gss_dataset_release", "gss_dataset_device_bytes", "gss_engine_create",
    "gss_engine_destroy", "gss_engine_load_beta", "gss_engine_update", "gss_engine_refresh",
    "gss_engine_grad_hessian", "gss_engine_log_likelihood", "gss_engine_get_beta",
    "gss_engine_get_xbeta", "gss_engine_get_exp_xbeta", "gss_engine_get_fixed_terms",
    "gss_engine_get_ipcw", "gss_engine_counters", "gss_engine_fit",
    "gss_engine_max_abs_gradient", "gss_engine_last_timing", "gss_engine_grad_hessian_all",
    "gss_engine_cycle_stats", "gss_shard_aggregate", "gss_shard_sums",
    "gss_engine_update_validate", "gss_engine_grad_hessian_separated",
    "gss_engine_set_grid", "gss_engine_grid", "gss_fit_batch",
]


class GssError(RuntimeError):
    def __init__(self, code, msg):
        self.code = code
        self.kind = GSS_STATUS.get(code, str(code))
        super().__init__(f"{self.kind}: {msg}")


class HostDataset(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int64), ("p", ctypes.c_int64),
                ("times", ctypes.c_void_p), ("status", ctypes.c_void_p),
                ("col_ptr", ctypes.c_void_p), ("row_idx", ctypes.c_void_p),
                ("vals", ctypes.c_void_p), ("col_indicator", ctypes.c_void_p),
                ("stratum_start", ctypes.c_void_p)]


class PenaltySpec(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int), ("strength", ctypes.c_double),
                ("exempt", ctypes.c_void_p)]


class FitConfig(ctypes.Structure):
    _fields_ = [("tolerance", ctypes.c_double), ("max_cycles", ctypes.c_int64),
                ("trust_init", ctypes.c_double)]


class FitResult(ctypes.Structure):
    _fields_ = [("objective", ctypes.c_double), ("cycles", ctypes.c_int64),
                ("converged", ctypes.c_int32), ("nonzero_count", ctypes.c_int64),
                ("skipped_steps", ctypes.c_int64), ("monotonicity_violations", ctypes.c_int64),
                ("wall_seconds", ctypes.c_double), ("device_seconds", ctypes.c_double)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIBGSS):
            raise ImportError(f"{LIBGSS} not built (run python -m paper_2204_08183_b200.build)")
        L = ctypes.CDLL(LIBGSS)
        L.gss_last_error.restype = ctypes.c_char_p
        L.gss_version.restype = ctypes.c_char_p
        L.gss_dataset_device_bytes.restype = ctypes.c_int64
        for name in ("gss_dataset_release", "gss_engine_destroy", "gss_comm_destroy"):
            getattr(L, name).restype = None
        _lib = L
    return _lib


def check(rc):
    if rc != 0:
        raise GssError(rc, lib().gss_last_error().decode())


def _p(a):
    return None if a is None else ctypes.c_void_p(a.ctypes.data)


class Dataset:
    """Device-packed dataset from the sorted host layout (see oracle.Sorted)."""

    def __init__(self, times, status, col_ptr, row_idx, vals=None, col_indicator=None,
                 stratum_start=None, device=0):
        self._arrs = [np.ascontiguousarray(times, np.float64),
                      np.ascontiguousarray(status, np.int32),
                      np.ascontiguousarray(col_ptr, np.int64),
                      np.ascontiguousarray(row_idx, np.int32),
                      None if vals is None else np.ascontiguousarray(vals, np.float64),
                      None if col_indicator is None else np.ascontiguousarray(col_indicator,
                                                                              np.uint8),
                      None if stratum_start is None else np.ascontiguousarray(stratum_start,
                                                                              np.uint8)]
        t, s, cp, ri, v, ci, ss = self._arrs
        self.n, self.p = len(t), len(cp) - 1
        h = HostDataset(self.n, self.p, t.ctypes.data, s.ctypes.data, cp.ctypes.data,
                        ri.ctypes.data if len(ri) else None,
                        None if v is None else v.ctypes.data,
                        None if ci is None else ci.ctypes.data,
                        None if ss is None else ss.ctypes.data)
        self.h = ctypes.c_void_p()
        check(lib().gss_dataset_pack(ctypes.byref(h), device, ctypes.byref(self.h)))

    @classmethod
    def from_sorted(cls, ds, device=0):
        return cls(ds.times, ds.status, ds.col_ptr, ds.row_idx, ds.vals, ds.col_indicator,
                   ds.stratum_start, device)

    def device_bytes(self):
        return lib().gss_dataset_device_bytes(self.h)

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.gss_dataset_release(self.h)
            self.h = None


class SimConfig(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int64), ("p", ctypes.c_int64), ("density", ctypes.c_double),
                ("beta_sparsity", ctypes.c_double), ("seed", ctypes.c_uint64),
                ("censoring_quantile", ctypes.c_double), ("time_quantum", ctypes.c_double),
                ("p_mix", ctypes.c_double)]


class SimOut(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int64), ("p", ctypes.c_int64), ("nnz", ctypes.c_int64),
                ("times", ctypes.POINTER(ctypes.c_double)),
                ("status", ctypes.POINTER(ctypes.c_int32)),
                ("col_ptr", ctypes.POINTER(ctypes.c_int64)),
                ("row_idx", ctypes.POINTER(ctypes.c_int32)),
                ("beta_true", ctypes.POINTER(ctypes.c_double))]


class SimData:
    """Benchmark-scale synthetic design in PINNED host memory (gss_sim.h).
    Arrays are zero-copy numpy views valid while this object lives."""

    def __init__(self, n, p, density=0.01, beta_sparsity=0.8, seed=0, censoring_quantile=0.0,
                 time_quantum=0.0, device=0, p_mix=0.0):
        L = lib()
        L.gss_sim_last_error.restype = ctypes.c_char_p
        self._out = SimOut()
        cfg = SimConfig(n, p, density, beta_sparsity, seed, censoring_quantile, time_quantum,
                        p_mix)
        rc = L.gss_simulate(ctypes.byref(cfg), device, ctypes.byref(self._out))
        if rc:
            raise GssError(rc, L.gss_sim_last_error().decode())
        o = self._out
        self.n, self.p, self.nnz = o.n, o.p, o.nnz
        as_np = np.ctypeslib.as_array
        self.times = as_np(o.times, shape=(o.n,))
        self.status = as_np(o.status, shape=(o.n,))
        self.col_ptr = as_np(o.col_ptr, shape=(o.p + 1,))
        self.row_idx = as_np(o.row_idx, shape=(max(o.nnz, 1),))[:o.nnz]
        self.beta_true = as_np(o.beta_true, shape=(max(o.p, 1),))[:o.p]

    def host_bytes(self):
        return (self.times.nbytes + self.status.nbytes + self.col_ptr.nbytes
                + self.row_idx.nbytes)

    def __del__(self):
        if _lib is not None and getattr(self, "_out", None) is not None:
            _lib.gss_sim_free(ctypes.byref(self._out))
            self._out = None


class Engine:
    """survscan::Engine surface over the C ABI (engine.hpp:33-90)."""

    def __init__(self, ds: Dataset, model="cox", recompute_interval=100, row_mask=None):
        self.ds = ds
        m = {"cox": 0, "finegray": 1, "fine_gray": 1}[model]
        self._mask = None if row_mask is None else np.ascontiguousarray(row_mask, np.uint8)
        self.h = ctypes.c_void_p()
        check(lib().gss_engine_create(ds.h, m, ctypes.c_int64(recompute_interval),
                                      _p(self._mask), ctypes.byref(self.h)))

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.gss_engine_destroy(self.h)
            self.h = None

    def attach_comm(self, comm):
        """gss_engine_attach_comm: this engine becomes shard `comm.rank`."""
        check(lib().gss_engine_attach_comm(self.h, comm.h))
        self._comm = comm
        return self

    def colmax(self):
        out = np.zeros(self.ds.p)
        check(lib().gss_engine_get_colmax(self.h, _p(out), ctypes.c_int64(self.ds.p)))
        return out

    def set_colmax(self, cm):
        c = np.ascontiguousarray(cm, np.float64)
        check(lib().gss_engine_set_colmax(self.h, _p(c), ctypes.c_int64(len(c))))

    def set_fixed_terms(self, fixed):
        f = np.ascontiguousarray(fixed, np.float64)
        check(lib().gss_engine_set_fixed_terms(self.h, _p(f), ctypes.c_int64(len(f))))

    def set_grid(self, grid):
        """CTAs per launch (0 = one per SM); re-partitions the tile ranges."""
        check(lib().gss_engine_set_grid(self.h, int(grid)))
        return self

    @property
    def grid(self):
        return lib().gss_engine_grid(self.h)

    def load_beta(self, beta):
        b = np.ascontiguousarray(beta, np.float64)
        check(lib().gss_engine_load_beta(self.h, _p(b), ctypes.c_int64(len(b))))

    def update(self, j, delta):
        check(lib().gss_engine_update(self.h, ctypes.c_int64(j), ctypes.c_double(delta)))

    def refresh(self):
        check(lib().gss_engine_refresh(self.h))

    def grad_hessian(self, j):
        g, h, f = ctypes.c_double(), ctypes.c_double(), ctypes.c_double()
        check(lib().gss_engine_grad_hessian(self.h, ctypes.c_int64(j), ctypes.byref(g),
                                            ctypes.byref(h), ctypes.byref(f)))
        return {"gradient": g.value, "hessian": h.value, "fixed_term": f.value}

    def grad_hessian_separated(self, j):
        """Engine::grad_hessian_separated (engine.hpp:61): the unfused path."""
        g, h, f = ctypes.c_double(), ctypes.c_double(), ctypes.c_double()
        check(lib().gss_engine_grad_hessian_separated(self.h, ctypes.c_int64(j), ctypes.byref(g),
                                                      ctypes.byref(h), ctypes.byref(f)))
        return {"gradient": g.value, "hessian": h.value, "fixed_term": f.value}

    def log_likelihood(self):
        out = ctypes.c_double()
        check(lib().gss_engine_log_likelihood(self.h, ctypes.byref(out)))
        return out.value

    def _rows(self, fn):
        out = np.empty(self.ds.n)
        check(fn(self.h, _p(out), ctypes.c_int64(self.ds.n)))
        return out

    def beta(self):
        out = np.empty(self.ds.p)
        check(lib().gss_engine_get_beta(self.h, _p(out), ctypes.c_int64(self.ds.p)))
        return out

    def xbeta(self):
        return self._rows(lib().gss_engine_get_xbeta)

    def exp_xbeta(self):
        return self._rows(lib().gss_engine_get_exp_xbeta)

    def fixed_terms(self):
        out = np.empty(self.ds.p)
        check(lib().gss_engine_get_fixed_terms(self.h, _p(out), ctypes.c_int64(self.ds.p)))
        return out

    def counters(self):
        a, r = ctypes.c_int64(), ctypes.c_int64()
        check(lib().gss_engine_counters(self.h, ctypes.byref(a), ctypes.byref(r)))
        return a.value, r.value

    def grad_hessian_all(self):
        """All columns at the current beta in one device launch."""
        g, h, f = np.empty(self.ds.p), np.empty(self.ds.p), np.empty(self.ds.p)
        check(lib().gss_engine_grad_hessian_all(self.h, _p(g), _p(h), _p(f)))
        return {"gradient": g, "hessian": h, "fixed_term": f}

    # ---- patient sharding (config C5) ----
    def shard_aggregate(self, column):
        out = np.zeros(8)
        check(lib().gss_shard_aggregate(self.h, ctypes.c_int64(column), _p(out)))
        return out

    def shard_sums(self, column, carry):
        c = np.ascontiguousarray(carry, np.float64)
        s0, s1 = ctypes.c_double(), ctypes.c_double()
        check(lib().gss_shard_sums(self.h, ctypes.c_int64(column), _p(c), ctypes.byref(s0),
                                   ctypes.byref(s1)))
        return s0.value, s1.value

    def update_validate(self, column, delta):
        over = ctypes.c_int32()
        check(lib().gss_engine_update_validate(self.h, ctypes.c_int64(column),
                                               ctypes.c_double(delta), ctypes.byref(over)))
        return bool(over.value)

    def max_abs_gradient(self):
        out = ctypes.c_double()
        check(lib().gss_engine_max_abs_gradient(self.h, ctypes.byref(out)))
        return out.value

    def fit(self, penalty="none", strength=0.0, exempt=(), tol=1e-6, max_cycles=1000,
            trust_init=1.0):
        kind = {"none": 0, "l1": 1, "l2": 2}[penalty]
        ex = None
        if len(exempt):
            ex = np.zeros(self.ds.p, np.uint8)
            ex[list(exempt)] = 1
        pen = PenaltySpec(kind, strength, None if ex is None else ex.ctypes.data)
        cfg = FitConfig(tol, max_cycles, trust_init)
        beta = np.zeros(self.ds.p)
        trace = np.zeros(max_cycles + 1)
        res = FitResult()
        check(lib().gss_engine_fit(self.h, ctypes.byref(pen), ctypes.byref(cfg), _p(beta),
                                   _p(trace), ctypes.byref(res)))
        return {"beta": beta, "objective": res.objective, "cycles": res.cycles,
                "converged": bool(res.converged), "nonzero_count": res.nonzero_count,
                "skipped_steps": res.skipped_steps,
                "monotonicity_violations": res.monotonicity_violations,
                "objective_trace": trace[:res.cycles + 1].copy(),
                "wall_seconds": res.wall_seconds, "device_seconds": res.device_seconds}

    def last_timing(self):
        ms, n = ctypes.c_double(), ctypes.c_int64()
        check(lib().gss_engine_last_timing(self.h, ctypes.byref(ms), ctypes.byref(n)))
        return ms.value, n.value

    def cycle_stats(self, max_cycles=100000):
        ms = np.zeros(max_cycles)
        acc = np.zeros(max_cycles, np.int64)
        L = lib()
        L.gss_engine_cycle_stats.restype = ctypes.c_int64
        k = L.gss_engine_cycle_stats(self.h, _p(ms), _p(acc), ctypes.c_int64(max_cycles))
        return ms[:k].copy(), acc[:k].copy()


class Comm:
    """gss_comm: one shard's handle on the in-kernel cross-shard exchange
    (config C5).  Keep it alive while its engine fits."""

    def __init__(self, h):
        self.h = h

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.gss_comm_destroy(self.h)
            self.h = None

    @property
    def rank(self):
        n, r = ctypes.c_int(), ctypes.c_int()
        check(lib().gss_comm_rank(self.h, ctypes.byref(n), ctypes.byref(r)))
        return r.value, n.value


def comm_unique_id() -> bytes:
    """gss_comm_unique_id: the NCCL bootstrap id (rank 0; broadcast it)."""
    buf = (ctypes.c_ubyte * 128)()
    check(lib().gss_comm_unique_id(buf))
    return bytes(buf)


def comm_init(nranks: int, rank: int, uid: bytes, device: int = 0) -> Comm:
    """gss_comm_init: one process per GPU (NCCL bootstrap + CUDA IPC buffers)."""
    buf = (ctypes.c_ubyte * 128).from_buffer_copy(uid[:128])
    h = ctypes.c_void_p()
    check(lib().gss_comm_init(int(nranks), int(rank), buf, int(device), ctypes.byref(h)))
    return Comm(h)


def comm_create(nranks: int, rank: int, device: int = 0) -> Comm:
    """gss_comm_create: this rank's exchange buffers (NCCL-free bootstrap)."""
    h = ctypes.c_void_p()
    check(lib().gss_comm_create(int(nranks), int(rank), int(device), ctypes.byref(h)))
    return Comm(h)


def comm_ipc_handle(comm: Comm) -> bytes:
    buf = (ctypes.c_ubyte * 128)()
    check(lib().gss_comm_ipc_handle(comm.h, buf))
    return bytes(buf)


def comm_connect(comm: Comm, handles) -> Comm:
    """gss_comm_connect: `handles` = every rank's 128-byte handle, rank order."""
    allb = b"".join(handles)
    buf = (ctypes.c_ubyte * len(allb)).from_buffer_copy(allb)
    check(lib().gss_comm_connect(comm.h, buf))
    return comm


def comm_local(engines):
    """gss_comm_local: every shard engine of this process gets a communicator
    (rank = position) and the global fixed terms."""
    k = len(engines)
    hs = (ctypes.c_void_p * k)(*[e.h.value for e in engines])
    out = (ctypes.c_void_p * k)()
    check(lib().gss_comm_local(hs, int(k), out))
    comms = [Comm(ctypes.c_void_p(out[i])) for i in range(k)]
    for e, c in zip(engines, comms):
        e._comm = c
    return comms


def sharded_fit_local(engines, penalty="l1", strength=0.0, tol=1e-6, max_cycles=1000,
                      trust_init=1.0):
    """gss_sharded_fit_local: one CCD fit over the patient shards of this
    process (all shards in one batched launch per cycle)."""
    k = len(engines)
    kind = {"none": 0, "l1": 1, "l2": 2}[penalty]
    pen = PenaltySpec(kind, float(strength), None)
    cfg = FitConfig(tol, max_cycles, trust_init)
    hs = (ctypes.c_void_p * k)(*[e.h.value for e in engines])
    beta = np.zeros(engines[0].ds.p)
    res = FitResult()
    dev_s = ctypes.c_double()
    check(lib().gss_sharded_fit_local(hs, int(k), ctypes.byref(pen), ctypes.byref(cfg), _p(beta),
                                      ctypes.byref(res), ctypes.byref(dev_s)))
    return {"beta": beta, "objective": res.objective, "cycles": res.cycles,
            "converged": bool(res.converged), "nonzero_count": res.nonzero_count,
            "skipped_steps": res.skipped_steps, "device_seconds": dev_s.value}


def fit_batch(engines, penalty="l1", strengths=None, tol=1e-6, max_cycles=1000, trust_init=1.0,
              max_active=0):
    """gss_fit_batch: fit every engine (one CCD cycle of all active fits per
    launch).  strengths: one per engine (or a scalar).  Returns (list of fit
    dicts or GssError per engine, device seconds)."""
    k = len(engines)
    if k == 0:
        return [], 0.0
    p = engines[0].ds.p
    kind = {"none": 0, "l1": 1, "l2": 2}[penalty]
    if strengths is None or np.isscalar(strengths):
        strengths = [0.0 if strengths is None else float(strengths)] * k
    pens = (PenaltySpec * k)(*[PenaltySpec(kind, float(g), None) for g in strengths])
    cfg = FitConfig(tol, max_cycles, trust_init)
    hs = (ctypes.c_void_p * k)(*[e.h.value for e in engines])
    beta = np.zeros((k, p))
    res = (FitResult * k)()
    st = np.zeros(k, np.int32)
    dev_s = ctypes.c_double()
    lib().gss_fit_batch(hs, ctypes.c_int64(k), pens, ctypes.byref(cfg), int(max_active),
                        _p(beta), res, _p(st), ctypes.byref(dev_s))
    out = []
    for i in range(k):
        if st[i]:
            out.append(GssError(int(st[i]), "batched fit %d failed" % i))
            continue
        r = res[i]
        out.append({"beta": beta[i].copy(), "objective": r.objective, "cycles": r.cycles,
                    "converged": bool(r.converged), "nonzero_count": r.nonzero_count,
                    "skipped_steps": r.skipped_steps,
                    "monotonicity_violations": r.monotonicity_violations,
                    "wall_seconds": r.wall_seconds, "device_seconds": r.device_seconds})
    return out, dev_s.value
