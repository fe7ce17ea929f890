"""Summarise an ncu --csv launch list: one line per launch with its metrics.

    python tools/ncu_csv.py gpurun_out/x.csv
"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr, recs = None, {}
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr is None or len(r) != len(hdr):
        continue
    d = dict(zip(hdr, r))
    key = (int(d["ID"]), d["Kernel Name"][:48])
    recs.setdefault(key, {})[d["Metric Name"]] = d["Metric Value"]
short = {"gpu__time_duration.sum": "ns", "dram__bytes_read.sum": "rdB",
         "dram__bytes_write.sum": "wrB", "lts__t_sector_hit_rate.pct": "l2hit%",
         "sm__warps_active.avg.pct_of_peak_sustained_active": "warps%"}
for (i, name), m in sorted(recs.items()):
    print(i, name, " ".join(f"{short.get(k, k)}={v}" for k, v in m.items()))
