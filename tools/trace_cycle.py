"""(Historical: written for the kernel before the control-warp restructure;
several events it reads are no longer emitted. The current per-phase
profile is GSS_DEBUG=256 / 1024 with tools/prof_sweep.py.)

Event trace of CTA 0 of the persistent cycle kernel (GSS_TRACE=1).

    python tools/trace_cycle.py --n 10000000 --p 64
Ring events (arg = stream position q): 20 producer issue, 23 producer passed the
same-tile progress wait, 21 consumer saw the data, 22 consumer released.
Slot events (arg = slot): 3 consumed, 7 exchange arrive, 4 exchange passed, 5 done.
Phase events of warp 0 (arg = tile): 10 patched, 11 phase 1, 12 scans, 13 transform, 14 records.
"""
import argparse
import ctypes
import os
import sys

import numpy as np

os.environ["GSS_TRACE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2204_08183_b200 import capi  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=10_000_000)
ap.add_argument("--p", type=int, default=64)
a = ap.parse_args()

sim = capi.SimData(a.n, a.p, 0.01, 0.8, 2, 0.9, 1000.0)
ds = capi.Dataset(sim.times, sim.status, sim.col_ptr, sim.row_idx)
eng = capi.Engine(ds, "cox")
L = capi.lib()
L.gss_engine_trace.restype = ctypes.c_int64
CAP = 32 << 16
buf = np.zeros(2 * CAP, np.uint64)
eng.fit(penalty="l1", strength=2 ** 0.5, tol=1e-300, max_cycles=1)
L.gss_engine_trace(eng.h, None, ctypes.c_int64(0))
eng.fit(penalty="l1", strength=2 ** 0.5, tol=1e-300, max_cycles=2)
k = L.gss_engine_trace(eng.h, buf.ctypes.data_as(ctypes.c_void_p), ctypes.c_int64(CAP))
ms, acc = eng.cycle_stats()
print("cycle ms", ms.round(3).tolist(), "per coord us", (ms / (a.p + 1) * 1e3).round(2).tolist())
ev = buf[:2 * k].reshape(-1, 2)
ev = ev[ev[:, 0] != 0]
ts = ev[:, 0].astype(np.int64)
meta = ev[:, 1]
kind = ((meta >> np.uint64(32)) & np.uint64(0xff)).astype(np.int64)
arg = (meta & np.uint64(0xffffffff)).astype(np.int64)
# keep the last launch only (positions restart per launch)
order = np.argsort(ts, kind="stable")
ts, meta = ts[order], meta[order]
kind = ((meta >> np.uint64(32)) & np.uint64(0xff)).astype(np.int64)
arg = (meta & np.uint64(0xffffffff)).astype(np.int64)
t_us = (ts - ts.min()) / 1000.0
starts = np.where((kind == 20) & (arg == 0))[0]
if len(starts) > 1:
    cut = t_us[starts[-1]]
    keep = t_us >= cut - 1e-9
    t_us, kind, arg = t_us[keep], kind[keep], arg[keep]


def by_arg(e):
    d = {}
    for a_, t_ in zip(arg[kind == e], t_us[kind == e]):
        d.setdefault(int(a_), t_)
    return d


iss, pas, got, rls = by_arg(20), by_arg(23), by_arg(21), by_arg(22)
qs = sorted(set(iss) & set(got) & set(rls))
lat = np.array([got[q] - iss[q] for q in qs])
hold = np.array([rls[q] - got[q] for q in qs])
print("load latency (issue->data seen) us: median %.2f p10 %.2f p90 %.2f" %
      (np.median(lat), np.percentile(lat, 10), np.percentile(lat, 90)))
print("consumer hold (data->release) us: median %.2f p90 %.2f" % (np.median(hold), np.percentile(hold, 90)))
pw = [iss[q] - pas[q] for q in qs if q in pas]
issue_t = np.array([iss[q] for q in qs])
print("issue gaps us: median %.3f mean %.3f" % (np.median(np.diff(issue_t)), np.mean(np.diff(issue_t))))
# producer waiting for the ring: time from the release of q-S to issue of q
S = 7  # Cox ring stages (Geo<false>::kS)
wait_ring = [iss[q] - rls[q - S] for q in qs if q - S in rls]
print("issue after release of q-S: median %.3f us" % np.median(wait_ring))
c3, c7, c4, c5 = (np.array(sorted(by_arg(e).values())) for e in (3, 7, 4, 5))
n = min(len(c3), len(c7), len(c4), len(c5))
if n > 3:
    print("slot: consume %.2f | scan+publish %.2f | barrier %.2f | step+carry %.2f  (us, medians)" % (
        np.median(c3[1:n] - c5[:n - 1]), np.median(c7[:n] - c3[:n]), np.median(c4[:n] - c7[:n]),
        np.median(c5[:n] - c4[:n])))
# warp-0 tile phases: 21 data seen -> 10 patched/xm -> 11 scans+exchange -> 12 transform -> 13 records -> 22 released
seq = sorted((t_, k_) for t_, k_ in zip(t_us, kind) if k_ in (21, 10, 11, 12, 13, 22))
names = {21: "data", 10: "patch", 11: "scan", 12: "xform", 13: "records", 22: "release"}
dur = {}
for (ta, ka), (tb, kb) in zip(seq, seq[1:]):
    nxt = {21: 10, 10: 11, 11: 12, 12: 13, 13: 22}.get(ka)
    if nxt == kb:
        dur.setdefault(names[kb], []).append(tb - ta)
print("warp-0 tile phases (median us):", {k: round(float(np.median(v)), 3) for k, v in dur.items()})
# all CTAs: slot-consumed times (event 30, region of warp 31, index slot*G + cta)
G = 148
reg = buf.reshape(-1, 2)[31 * 65536:32 * 65536]
tsc = reg[:, 0].astype(np.int64)
ctas = (reg[:, 1] & np.uint64(0xffffffff)).astype(np.int64)
valid = tsc != 0
if valid.any():
    nsl = int(valid.sum()) // G
    tt = tsc[:nsl * G].reshape(nsl, G) / 1000.0
    spread = tt.max(axis=1) - tt.min(axis=1)
    print("per-slot consumed spread over CTAs (us): median %.2f" % np.median(spread[1:]))
    rel = tt - tt.min(axis=1, keepdims=True)
    mean_rel = rel[1:].mean(axis=0)
    order = np.argsort(mean_rel)
    print("fastest CTAs", order[:6].tolist(), np.round(mean_rel[order[:6]], 2).tolist())
    print("slowest CTAs", order[-6:].tolist(), np.round(mean_rel[order[-6:]], 2).tolist())
    print("mean lag by CTA block of 16:", [round(float(mean_rel[i:i + 16].mean()), 1) for i in range(0, G, 16)])
def region(r):
    reg = buf.reshape(-1, 2)[r * 65536:(r + 1) * 65536]
    t = reg[:, 0].astype(np.int64)
    n = int((t != 0).sum()) // G
    return t[:n * G].reshape(n, G) / 1000.0
arr, pas_ = region(29), region(30)
n = min(len(arr), len(pas_))
if n > 2:
    arr, pas_ = arr[-n // 2:], pas_[-n // 2:]
    last_arrive = arr.max(axis=1)
    print("exchange: arrive spread %.2f us, last-arrive -> first pass %.2f us, -> last pass %.2f us" % (
        np.median(arr.max(1) - arr.min(1)), np.median(pas_.min(1) - last_arrive),
        np.median(pas_.max(1) - last_arrive)))
top, aft_empty, aft_issue = by_arg(24), by_arg(25), by_arg(26)
qq = sorted(set(top) & set(aft_empty) & set(iss) & set(aft_issue))
pas = {q: aft_empty[q] for q in qq}
def med(xs):
    return round(float(np.median(xs)), 3) if len(xs) else None
print("producer per position (median us): wait-empty", med([aft_empty[q] - top[q] for q in qq]),
      "| empty->issue-start", med([iss[q] - aft_empty[q] for q in qq]),
      "| progress", med([pas[q] - aft_empty[q] for q in qq]),
      "| setup", med([iss[q] - pas[q] for q in qq]),
      "| issue", med([aft_issue[q] - iss[q] for q in qq]),
      "| to next top", med([top[q + 1] - aft_issue[q] for q in qq if q + 1 in top]))
# raw timeline of one middle slot on CTA 0 (CTA 0 owns floor(ntiles/G) tiles)
tc_ = (((a.n + 2047) // 2048)) // 148
sl = 40
c5d = by_arg(5)
if sl - 1 in c5d:
    base = c5d[sl - 1]  # previous slot's control done
    print("slot %d timeline (us from previous slot done): q: issue / data / release" % sl)
    rows_ = []
    for i in range(tc_):
        q = sl * tc_ + i
        rows_.append("%2d:%6.2f/%6.2f/%6.2f" % (i, iss.get(q, np.nan) - base, got.get(q, np.nan) - base,
                                               rls.get(q, np.nan) - base))
    for j in range(0, len(rows_), 4):
        print("   " + "  ".join(rows_[j:j + 4]))
    print("   slot consumed at %.2f, exchange passed %.2f, done %.2f" % (
        by_arg(3).get(sl, np.nan) - base, by_arg(4).get(sl, np.nan) - base, c5d.get(sl, np.nan) - base))

# post-exchange breakdown on CTA 0: 4 passed -> 8 after barrier release (tid 0) -> 9 gathered -> 5 slot done
e8 = np.sort(t_us[kind == 8]); e9 = np.sort(t_us[kind == 9]); e5 = np.sort(t_us[kind == 5])
if len(e8) > 10 and len(e9) == len(e8):
    g = e9 - e8
    # pair each gather end with the next slot-done event
    d = [e5[np.searchsorted(e5, x)] - x for x in e9 if np.searchsorted(e5, x) < len(e5)]
    print("post-exchange: gather %.2f us, step+carries+sync %.2f us (medians)" % (np.median(g), np.median(d)))
