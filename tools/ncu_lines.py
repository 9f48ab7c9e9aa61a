"""Per-source-line warp-stall samples from an ncu report (cuda,sass view),
with the dominant stall reasons of each line.

    python tools/ncu_lines.py report.ncu-rep [top] [lo-hi line filter]
"""
import csv
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
rng = None
if len(sys.argv) > 3:
    a, b = sys.argv[3].split("-")
    rng = (int(a), int(b))
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
lines = []
cur_file = None
hdr = None
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
    if r and r[0] == "Line No":
        hdr = r
    if hdr and len(r) > 6 and r[0].isdigit():
        try:
            tot = int(r[4])
        except ValueError:
            continue
        reasons = []
        for i, h in enumerate(hdr):
            if h.startswith("stall_") and "Not Issued" not in h:
                try:
                    v = int(r[i])
                except ValueError:
                    continue
                if v:
                    reasons.append((v, h[6:]))
        reasons.sort(reverse=True)
        lines.append((tot, cur_file, int(r[0]), r[1][:90], reasons[:3]))
total = sum(x[0] for x in lines) or 1
if rng:
    lines = [x for x in lines if rng[0] <= x[2] <= rng[1]]
    lines.sort(key=lambda x: x[2])
else:
    lines.sort(reverse=True)
for s, f, ln, src, rs in lines[:top]:
    rtxt = " ".join(f"{n}:{100.0 * v / total:.1f}" for v, n in rs)
    print(f"{100.0 * s / total:5.1f}% {f}:{ln:5d}  {src:90s} [{rtxt}]")
