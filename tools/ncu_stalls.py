"""Per CUDA source line: share of warp-stall samples and the top stall reasons
(ncu -i rep --page source --csv --print-source cuda,sass > file; this file)."""
import collections
import csv
import sys


def main(path, top=25, kernel=0):
    rows = list(csv.reader(open(path)))
    his = [i for i, r in enumerate(rows) if "Warp Stall Sampling (All Samples)" in r]
    hi = his[kernel]
    end = his[kernel + 1] if kernel + 1 < len(his) else len(rows)
    hdr = rows[hi]
    iA = hdr.index("Warp Stall Sampling (All Samples)")
    reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
    ri = [hdr.index(h) for h in reasons]
    line, src = None, {}
    agg = collections.defaultdict(collections.Counter)
    for r in rows[hi + 1:end]:
        if r and r[0]:
            try:
                line = int(r[0])
            except ValueError:
                line = None
                continue
            src[line] = r[1].strip()[:80]
        elif line is not None and len(r) > iA and r[iA] not in ("", "-"):
            for h, i in zip(reasons, ri):
                try:
                    agg[line][h] += float(r[i])
                except ValueError:
                    pass
    tot = sum(sum(c.values()) for c in agg.values()) or 1
    for ln, c in sorted(agg.items(), key=lambda x: -sum(x[1].values()))[:top]:
        s = sum(c.values())
        print(f"{100 * s / tot:5.1f}% L{ln:5d} {src[ln][:58]:58s} " +
              " ".join(f"{k[6:]}={100 * v / s:.0f}" for k, v in c.most_common(4)))


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 25, int(sys.argv[3]) if len(sys.argv) > 3 else 0)
