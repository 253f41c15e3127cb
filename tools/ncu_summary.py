"""Write a JSON + text summary of one ncu --set full capture (profiles/)."""
import csv
import io
import json
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__occupancy_limit_shared_mem", "launch__occupancy_limit_registers", "smsp__inst_executed.sum",
        "sm__cycles_elapsed.avg.per_second", "launch__grid_size", "launch__block_size",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct"]


def main(rep, out_json, kind, level, note, workload="", alg_flops=None, exec_flops=None):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(raw)))
    h, u, v = r[0], r[1], r[2]
    d = {h[i]: (v[i], u[i]) for i in range(len(h))}
    m = {k: d[k] for k in KEYS if k in d}
    stalls = {k.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", ""): float(d[k][0])
              for k in h if "average_warps_issue_stalled" in k and "per_issue_active" in k and d[k][0]
              and float(d[k][0]) > 0.05}

    def mb(x):
        val, unit = x
        f = float(val)
        return f * {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0}.get(unit, 1.0)

    traffic = mb(m["dram__bytes_read.sum"]) + mb(m["dram__bytes_write.sum"])
    out = {"kernel_kind": kind, "level": level, "workload": workload, "algorithmic_flops": alg_flops,
           "executed_flops": exec_flops, "kernel": d.get("Kernel Name", ("", ""))[0],
           "dram_bytes_per_launch": traffic, "metrics": {k: f"{a} {b}" for k, (a, b) in m.items()},
           "stalls_per_issue": stalls, "note": note}
    json.dump(out, open(out_json, "w"), indent=1)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    a = sys.argv
    main(a[1], a[2], a[3], int(a[4]), a[5] if len(a) > 5 else "", a[6] if len(a) > 6 else "",
         float(a[7]) if len(a) > 7 else None, float(a[8]) if len(a) > 8 else None)
