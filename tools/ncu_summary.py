"""One-screen summary of an ncu --set full report (per profiled launch):
duration, DRAM bytes / throughput, L2 hit rate, tensor-pipe and issue
activity, occupancy limiters and the top warp-stall reasons.

    python tools/ncu_summary.py gpurun_out/x.ncu-rep > profiles/r2/x_summary.txt
"""
import csv
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "launch__occupancy_limit_registers",
        "launch__occupancy_limit_shared_mem", "launch__occupancy_limit_warps",
        "smsp__inst_executed.sum", "sm__cycles_elapsed.avg"]

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr, units = rows[0], rows[1]
for vals in rows[2:]:
    d = dict(zip(hdr, vals))
    u = dict(zip(hdr, units))
    print(f"== {d.get('Kernel Name', '?')[:110]}")
    for k in KEYS:
        if k in d:
            print(f"  {k:62s} {d[k]} {u.get(k, '')}")
    stalls = sorted(((float(v.replace(',', '') or 0), k) for k, v in d.items()
                     if k.startswith("smsp__pcsamp_warps_issue_stalled_") and "not_issued" not in k),
                    reverse=True)
    tot = sum(s for s, _ in stalls) or 1.0
    print("  top stall samples: " + ", ".join(
        f"{k.replace('smsp__pcsamp_warps_issue_stalled_', '')} {100 * s / tot:.0f}%"
        for s, k in stalls[:6]))
