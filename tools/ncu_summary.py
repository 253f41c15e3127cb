"""Summarise an ncu report (raw page): per kernel launch the duration, DRAM
bytes, pipe utilisation, occupancy and the top warp-stall reasons."""
import csv
import io
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct"]

rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[0]
for v in rows[2:]:
    d = dict(zip(h, v))
    print("==", d.get("Kernel Name", "?")[:110])
    for k in KEYS:
        if k in d:
            print(f"   {k} = {d[k]}")
    st = sorted(((float(d[k] or 0), k) for k in h if k.startswith("smsp__average_warps_issue_stalled_")
                 and k.endswith("per_issue_active.ratio")), reverse=True)[:6]
    print("   stalls: " + ", ".join(f"{k.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', '')} {x:.2f}" for x, k in st))
