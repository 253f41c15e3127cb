"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list:
per-kernel totals and the launches of the last step."""
import collections
import csv
import io
import sys


def load(path):
    lines = open(path).read().splitlines()
    start = [i for i, l in enumerate(lines) if l.startswith('"ID"')][0]
    return list(csv.DictReader(io.StringIO("\n".join(lines[start:]))))


def main(path, last=None):
    rows = load(path)
    agg = collections.OrderedDict()
    for r in rows:
        n = r["Kernel Name"].split("(")[0][:70]
        agg.setdefault(n, [0, 0.0])
        agg[n][0] += 1
        agg[n][1] += float(r["Metric Value"])
    tot = sum(v[1] for v in agg.values())
    print(f"{len(rows)} launches, {tot / 1e6:.3f} ms total")
    for n, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{c:5d} {t / 1e6:9.3f} ms {100 * t / tot:5.1f}%  {n}")
    if last:
        print(f"--- last {last} launches")
        for r in rows[-last:]:
            print(f"{float(r['Metric Value']) / 1e3:8.1f} us  grid={r['Grid Size']:>14} blk={r['Block Size']:>12}  "
                  f"{r['Kernel Name'].split('(')[0][:40]}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else None)
