"""(Historical: written for the kernel before the control-warp restructure;
several events it reads are no longer emitted. The current per-phase
profile is GSS_DEBUG=256 / 1024 with tools/prof_sweep.py.)

Per-CTA slot timing of the cycle kernel (trace build, all CTAs, no CTA-0
event trace): how much of each coordinate is spent waiting for the slowest
CTA, and whether the same CTAs are slow every slot (static imbalance) or not.

    GSS_LIB=build_trace/libgss.so python tools/trace_ctas.py --n 10000000 --p 256
"""
import argparse
import ctypes
import os
import sys

import numpy as np

os.environ["GSS_TRACE"] = "1"
os.environ["GSS_DEBUG"] = str(int(os.environ.get("GSS_DEBUG", "0")) | 32)
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2204_08183_b200 import capi  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=10_000_000)
ap.add_argument("--p", type=int, default=256)
ap.add_argument("--model", default="cox")
a = ap.parse_args()

pmix = 0.5 if a.model == "finegray" else 0.0
sim = capi.SimData(a.n, a.p, 0.01, 0.8, 2, 0.9, 1000.0, p_mix=pmix)
ds = capi.Dataset(sim.times, sim.status, sim.col_ptr, sim.row_idx)
eng = capi.Engine(ds, a.model)
L = capi.lib()
L.gss_engine_trace.restype = ctypes.c_int64
CAP = 32 << 16
buf = np.zeros(2 * CAP, np.uint64)
eng.fit(penalty="l1", strength=2 ** 0.5, tol=1e-300, max_cycles=1)
L.gss_engine_trace(eng.h, None, ctypes.c_int64(0))
eng.fit(penalty="l1", strength=2 ** 0.5, tol=1e-300, max_cycles=1)
L.gss_engine_trace(eng.h, buf.ctypes.data_as(ctypes.c_void_p), ctypes.c_int64(CAP))
ms, acc = eng.cycle_stats()
print("cycle ms", ms.round(3).tolist(), "per coord us", (ms / (a.p + 1) * 1e3).round(2).tolist())
G = None


def region(r):
    reg = buf.reshape(-1, 2)[r * 65536:(r + 1) * 65536]
    t = reg[:, 0].astype(np.int64)
    c = (reg[:, 1] & np.uint64(0xffffffff)).astype(np.int64)
    return t, c


t30, c30 = region(31)  # consumed (slot k), index k*G + cta
nz = np.nonzero(t30)[0]
G = int(c30[nz].max()) + 1
ns = len(nz) // G
cons = t30[:ns * G].reshape(ns, G) / 1000.0
t29, _ = region(29)  # exchange arrive (exchange ordinal)
t30b, _ = region(30)  # exchange pass
nx = int((t29 != 0).sum()) // G
arr = t29[:nx * G].reshape(nx, G) / 1000.0
pas = t30b[:nx * G].reshape(nx, G) / 1000.0
print(f"G={G} slots traced={ns} exchanges={nx}")
sl = slice(ns // 4, ns - 2)
c = cons[sl]
med = np.median(c, axis=1, keepdims=True)
lag = c - med
print("consumed: max-median %.2f us, median-min %.2f us, p90-median %.2f (medians over slots)" % (
    np.median(c.max(1) - med[:, 0]), np.median(med[:, 0] - c.min(1)),
    np.median(np.percentile(c, 90, axis=1) - med[:, 0])))
mean_lag = lag.mean(0)
resid = lag - mean_lag
print("per-CTA lag: std of CTA means %.2f us, residual std %.2f us" % (mean_lag.std(), resid.std()))
order = np.argsort(mean_lag)
print("slowest CTAs (mean lag us):", [(int(i), round(float(mean_lag[i]), 2)) for i in order[-8:]])
print("fastest CTAs (mean lag us):", [(int(i), round(float(mean_lag[i]), 2)) for i in order[:8]])
last = np.argmax(c, axis=1)
u, k = np.unique(last, return_counts=True)
top = np.argsort(k)[-8:]
print("last-to-finish CTA histogram (top):", [(int(u[i]), int(k[i])) for i in top])
# slot period and where it goes, on the median CTA
period = np.median(np.diff(np.median(cons, axis=1)))
xa = arr[-(nx // 2):]
xp = pas[-(nx // 2):]
print("slot period %.2f us; exchange: last arrive -> median pass %.2f us, pass spread %.2f us" % (
    period, np.median(np.median(xp, 1) - xa.max(1)), np.median(xp.max(1) - xp.min(1))))
# pass -> next consumed on each CTA = the CTA's busy time for the next slot
if nx >= ns:
    off = nx - ns  # prologue (and refresh) exchanges precede
print("sum of tiles per CTA known on host; CTA busy (pass->consumed) estimated below")
busy = []
for s_ in range(ns // 4, ns - 2):
    # the exchange that precedes slot s_ consumption: latest pass before min consumed time
    before = pas[(pas.max(1) < cons[s_].min())]
    if len(before):
        busy.append(cons[s_] - before[-1])
if busy:
    b = np.array(busy)
    print("busy per slot (pass -> consumed): median over CTAs %.2f us, max %.2f, min %.2f" % (
        np.median(np.median(b, 1)), np.median(b.max(1)), np.median(b.min(1))))
    bm = b.mean(0)
    print("busy CTA-mean: std %.2f us; slowest" % bm.std(), [(int(i), round(float(bm[i]), 2)) for i in np.argsort(bm)[-6:]])
