"""Shared helpers for the parity tests: golden fixture loading and the
parity metrics.

rel()      — the reference tests' metric |a-b|/max(1,|a|,|b|)
             (tests/test_engine.cpp:16-18; tests/acceptance.cpp:41-43).
rel_cond() — the conditioning-aware metric of SURVEY.md §8a for gradients:
             |a-b|/max(1,|a|,|b|,|fixed_term|,|grad_sum|).  g' = fixed - Σ
             cancels near the optimum; the reference disagrees with itself
             by ~3e-9 there under plain rel across chunk plans.
"""
import glob
import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")

# north_star tolerances (BASELINE.json): 1e-10 on ll/grad/hess, 1e-8 on beta
TOL_DERIV = 1e-10
TOL_BETA = 1e-8


def rel(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    return np.abs(a - b) / np.maximum(1.0, np.maximum(np.abs(a), np.abs(b)))


def rel_cond(a, b, scale):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    den = np.maximum.reduce([np.ones_like(a), np.abs(a), np.abs(b), np.abs(scale)])
    return np.abs(a - b) / den


def load(name):
    z = np.load(os.path.join(GOLDEN, name + ".npz"), allow_pickle=False)
    return {k: z[k] for k in z.files}


def cases(prefix=""):
    out = []
    for f in sorted(glob.glob(os.path.join(GOLDEN, prefix + "*.npz"))):
        name = os.path.basename(f)[:-4]
        if name != "c1_ref":  # config C1 fixture: its own tests (test_gpu_c1.py)
            out.append(name)
    return out


def raw(c):
    """(times, status, rows, cols, values, n_cols[, strata]) of a fixture."""
    args = (c["times"], c["status"], c["rows"], c["cols"], c["values"], int(c["n_cols"]))
    return args, (c["strata"] if "strata" in c else None)


def fit_cases(c):
    out = []
    names = [str(s) for s in c.get("fits", [])]
    for k, nm in enumerate(names):
        pen, lam = nm.split(":")
        out.append((k, pen, float(lam)))
    return out
