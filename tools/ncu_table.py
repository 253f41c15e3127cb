"""One line per ncu report: duration, DRAM bytes, DRAM GB/s, DMMA pipe %, warps
active %, occupancy limits (profiles/ summaries of secondary kernels)."""
import csv
import io
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__occupancy_limit_shared_mem", "launch__occupancy_limit_registers", "launch__grid_size"]
SCALE = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0, "usecond": 1e-6, "msecond": 1e-3, "nsecond": 1e-9}


def row(rep):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(raw)))
    h, u, v = r[0], r[1], r[2]
    d = {h[i]: (v[i], u[i]) for i in range(len(h))}
    t = float(d[KEYS[0]][0]) * SCALE.get(d[KEYS[0]][1], 1e-6)
    rb = float(d[KEYS[1]][0]) * SCALE.get(d[KEYS[1]][1], 1.0)
    wb = float(d[KEYS[2]][0]) * SCALE.get(d[KEYS[2]][1], 1.0)
    name = d.get("Kernel Name", ("?", ""))[0][:40]
    return (f"{name:40s} {t * 1e6:8.1f} us  DRAM {(rb + wb) / 1e6:8.1f} MB  {(rb + wb) / t / 1e9:7.0f} GB/s  "
            f"DMMA {float(d[KEYS[3]][0]):5.1f}%  warps {float(d[KEYS[4]][0]):5.1f}%  regs {d[KEYS[5]][0]}  "
            f"occ(smem,regs) {d[KEYS[6]][0]},{d[KEYS[7]][0]}  grid {d[KEYS[8]][0]}")


if __name__ == "__main__":
    for rep in sys.argv[1:]:
        print(row(rep))
