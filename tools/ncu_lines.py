"""Aggregate ncu warp-stall samples and executed instructions per CUDA source
line (ncu -i rep --page source --csv --print-source cuda,sass)."""
import csv
import sys


def main(path, top=30):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Warp Stall Sampling (All Samples)" in r]
    out = []
    for h0 in hi:
        hdr = rows[h0]
        iA = hdr.index("Warp Stall Sampling (All Samples)")
        iE = hdr.index("Instructions Executed")
        j = h0 + 1
        cur = None
        while j < len(rows) and "Warp Stall Sampling (All Samples)" not in rows[j]:
            r = rows[j]
            if len(r) > iA and r[0]:
                cur = [r[0], r[1], 0.0, 0.0]
                out.append(cur)
            if cur is not None and len(r) > iA and not r[0] and r[iA] not in ("-", ""):
                cur[2] += float(r[iA])
                cur[3] += float(r[iE] or 0)
            j += 1
    tot = sum(o[2] for o in out) or 1
    print(f"total samples {tot:.0f}")
    for o in sorted(out, key=lambda o: -o[2])[:top]:
        print(f"{100 * o[2] / tot:5.1f}%  inst={o[3]:9.0f}  L{o[0]:>5}  {o[1].strip()[:90]}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 30)
