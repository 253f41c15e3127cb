"""Per-launch achieved rates of one build: durations from a serial --timeline
run (H2SP_SERIAL=1 python bench.py --timeline, stderr), algorithmic work from
the plan (h2sp_plan_launches), against the measured peaks.

usage: python tools/per_launch_roofline.py TIMELINE_LOG [config] [N]"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main(path, config=2, n=None):
    import h2gen
    import paper_1705_04601_b200 as h2sp
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    hbm = float(peaks.get("hbm_gbs", 6536.7))
    fp64 = 37.0
    h = h2gen.make_config(config, N=n, with_close=False)
    plan = h2sp.Plan(h2gen.pack(h))
    lis = plan.launches()
    durs = [float(l.split()[-2]) for l in open(path) if l.startswith("timeline")]
    assert len(durs) == len(lis), (len(durs), len(lis))
    print(f"{'kind':>11} {'lvl':>3} {'items':>7} {'us':>8} {'GFLOP':>8} {'TF/s':>6} {'%DMMA':>6} {'MB':>8} {'GB/s':>7} {'%HBM':>5}")
    for li, d in zip(lis, durs):
        tf = li["flops_exec"] / (d * 1e-6) / 1e12 if d > 0 else 0.0
        gb = li["bytes"] / (d * 1e-6) / 1e9 if d > 0 else 0.0
        print(f"{li['kind']:>11} {li['level']:>3} {li['items']:>7} {d:8.1f} {li['flops_exec'] / 1e9:8.3f} {tf:6.2f} "
              f"{100 * tf / fp64:6.1f} {li['bytes'] / 1e6:8.1f} {gb:7.0f} {100 * gb / hbm:5.1f}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 2, int(sys.argv[3]) if len(sys.argv) > 3 else None)
