"""Summarise one `ncu --set full` capture of the cycle kernel into the JSON
that bench.py reads for roofline.traffic (profiles/ncu_cycle_summary.json).

    python tools/ncu_summary.py gpurun_out/prof_c2.ncu-rep --n 10000000 --p 5000 \
        --nnz 500005713 --command "..." -o profiles/ncu_cycle_summary.json
"""
import argparse
import csv
import json
import subprocess
import sys

ap = argparse.ArgumentParser()
ap.add_argument("report")
ap.add_argument("--n", type=float, required=True)
ap.add_argument("--p", type=int, required=True)
ap.add_argument("--nnz", type=float, required=True)
ap.add_argument("--bytes-per-row", type=float, default=12.0)
ap.add_argument("--command", default="")
ap.add_argument("--kernel", default="cycle_kernel<false>")
ap.add_argument("-o", "--out", required=True)
a = ap.parse_args()

raw = subprocess.run(["ncu", "-i", a.report, "--page", "raw", "--csv"], capture_output=True,
                     text=True, check=True).stdout
rows = list(csv.reader(raw.splitlines()))
hdr, units, vals = rows[0], rows[1], rows[2]
m = {h: (v, u) for h, u, v in zip(hdr, units, vals)}


def num(key, scale=1.0):
    v, u = m[key]
    v = float(v.replace(",", ""))
    mult = {"Tbyte": 1e12, "Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0, "ms": 1e-3,
            "us": 1e-6, "ns": 1e-9, "s": 1.0, "%": 1.0, "register/thread": 1.0}.get(u)
    if mult is None and u and ("byte" in u or u.endswith("s")):
        raise ValueError(f"unknown unit {u!r} for {key}")
    mult = mult or 1.0
    return v * mult * scale


t = num("gpu__time_duration.sum")
rd, wr = num("dram__bytes_read.sum"), num("dram__bytes_write.sum")
# algorithmic bytes of one launch: p coordinate slots + the
# objective slot; the update part (20 B per touched nonzero) is counted with
# every coordinate accepted (an upper bound: most are at C2)
per_coord = a.bytes_per_row * a.n + 4.0 * a.nnz / a.p
alg = a.p * per_coord + a.bytes_per_row * a.n + 20.0 * a.nnz
stalls = {k.replace("smsp__pcsamp_warps_issue_stalled_", ""): float(v[0])
          for k, v in m.items() if k.startswith("smsp__pcsamp_warps_issue_stalled_")
          and not k.endswith("not_issued")}
tot = sum(stalls.values()) or 1.0
out = {
    "command": a.command,
    "kernel": a.kernel,
    "launch_ms": t * 1e3,
    "dram_read_GB": rd / 1e9,
    "dram_write_GB": wr / 1e9,
    "dram_bytes_per_launch": rd + wr,
    "dram_bytes_per_coordinate": (rd + wr) / (a.p + 1),
    "algorithmic_bytes_per_launch": alg,
    "algorithmic_bytes_per_coordinate": per_coord,
    "traffic_over_algorithmic": round((rd + wr) / alg, 4),
    "dram_GBps_under_ncu": round((rd + wr) / t / 1e9, 1),
    "sm_throughput_pct": num("sm__throughput.avg.pct_of_peak_sustained_elapsed"),
    "issue_active_pct": num("smsp__issue_active.avg.pct_of_peak_sustained_active"),
    "registers_per_thread": num("launch__registers_per_thread"),
    "block": int(num("launch__block_size")),
    "grid": int(num("launch__grid_size")),
    "l2_hit_rate_pct": num("lts__t_sector_hit_rate.pct"),
    "stall_samples_pct": {k: round(100 * v / tot, 1)
                          for k, v in sorted(stalls.items(), key=lambda kv: -kv[1]) if v / tot > 0.01},
}
json.dump(out, open(a.out, "w"), indent=1)
print(json.dumps(out, indent=1))
