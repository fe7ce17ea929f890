"""Per-source-line hot spots of one kernel from an ncu report (needs a capture
made with --import-source on and a -lineinfo build).

    python tools/ncu_lines.py REPORT.ncu-rep [--top 40] [--ranges file:a-b=name ...]

Prints the lines with the most warp-stall samples (all samples, i.e. where
warps spent their time) with their executed warp instructions and the
dominant stall reasons, then totals per named line range.
"""
import argparse
import csv
import io
import subprocess
from collections import defaultdict

ap = argparse.ArgumentParser()
ap.add_argument("report")
ap.add_argument("--top", type=int, default=40)
ap.add_argument("--ranges", nargs="*", default=[])
a = ap.parse_args()

raw = subprocess.run(["ncu", "-i", a.report, "--page", "source", "--csv", "--print-source",
                      "cuda,sass"], capture_output=True, text=True).stdout
fname = None
header = None
rows = []
for rec in csv.reader(io.StringIO(raw)):
    if not rec:
        continue
    if rec[0] == "File Path":
        fname = rec[1].split("/")[-1]
        continue
    if rec[0] == "Line No":
        header = rec
        continue
    if header is None or not rec[0].strip().isdigit():
        continue
    d = dict(zip(header[2:], rec[2:]))
    # the first 'Source' is the CUDA line, the second the (empty) SASS column
    rows.append((fname, int(rec[0]), rec[1].strip(), d))


def num(x):
    try:
        return float(x)
    except (TypeError, ValueError):
        return 0.0


stall_cols = [c for c in (header or []) if c.startswith("stall_") and "Not Issued" not in c]
tot_s = sum(num(d.get("Warp Stall Sampling (All Samples)")) for *_, d in rows)
tot_i = sum(num(d.get("Instructions Executed")) for *_, d in rows)
print(f"total samples {tot_s:.0f}, warp instructions {tot_i:.0f}")
rows.sort(key=lambda r: -num(r[3].get("Warp Stall Sampling (All Samples)")))
for f, ln, src, d in rows[: a.top]:
    s = num(d.get("Warp Stall Sampling (All Samples)"))
    ins = num(d.get("Instructions Executed"))
    st = sorted(((num(d.get(c)), c[6:]) for c in stall_cols), reverse=True)[:3]
    sts = " ".join(f"{n}:{v:.0f}" for v, n in st if v)
    print(f"{100 * s / tot_s:5.1f}% {ins / max(tot_i, 1) * 100:5.1f}%i {f}:{ln:<5d} {src[:70]:70s} {sts}")
if a.ranges:
    acc = defaultdict(lambda: [0.0, 0.0])
    for f, ln, src, d in rows:
        for spec in a.ranges:
            loc, name = spec.split("=")
            ff, rng = loc.split(":")
            lo, hi = (int(x) for x in rng.split("-"))
            if f == ff and lo <= ln <= hi:
                acc[name][0] += num(d.get("Warp Stall Sampling (All Samples)"))
                acc[name][1] += num(d.get("Instructions Executed"))
    for name, (s, i) in acc.items():
        print(f"range {name:20s} samples {100 * s / tot_s:5.1f}%  instructions {100 * i / tot_i:5.1f}%")
