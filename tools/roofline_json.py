"""gpurun_out/roof/*.csv (ncu, one rollout_kernel launch each) ->
profiles/r2/rollout_ncu.json keyed "<workload>/<rollout|train>/B<batch>"."""
import csv
import io
import json
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
out = {}
for f in sorted((ROOT / "gpurun_out" / "roof").glob("*.csv")):
    text = f.read_text()
    rows = list(csv.reader(io.StringIO(text[text.find('"ID"'):])))
    if not rows:
        continue
    h = {k: i for i, k in enumerate(rows[0])}
    vals = {}
    for r in rows[1:]:
        if len(r) < len(h):
            continue
        v = float(r[h["Metric Value"]].replace(",", ""))
        unit = r[h["Metric Unit"]]
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1, "usecond": 1e3,
                 "msecond": 1e6}.get(unit, 1)
        vals[r[h["Metric Name"]]] = v * scale
    stem = f.stem  # <workload>_rollout | <workload>_train
    wl, mode = stem.rsplit("_", 1)
    out[f"{wl}/{mode}/B1024"] = {
        "dram_bytes_read": vals.get("dram__bytes_read.sum"),
        "dram_bytes_write": vals.get("dram__bytes_write.sum"),
        "inst_executed": vals.get("smsp__inst_executed.sum"),
        "ipc": vals.get("sm__inst_executed.avg.per_cycle_active"),
        "ncu_ns": vals.get("gpu__time_duration.sum"),
        "warps_active_pct": vals.get("sm__warps_active.avg.pct_of_peak_sustained_active"),
        "issue_active_pct": vals.get("smsp__issue_active.avg.pct_of_peak_sustained_active"),
        "capture": f"ncu --metrics ... -k regex:rollout_kernel -s 3 -c 1 python bench.py "
                   f"--workload {wl}{' --mode train' if mode == 'train' else ''} (tools/roofline_capture.sh)",
    }
dst = ROOT / "profiles" / "r2" / "rollout_ncu.json"
dst.parent.mkdir(parents=True, exist_ok=True)
dst.write_text(json.dumps(out, indent=1) + "\n")
print(json.dumps(out, indent=1))
