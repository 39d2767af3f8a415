"""Top stall-sampled SASS instructions of an ncu report (source page, sass):
    ncu -i X.ncu-rep --page source --csv --print-source sass > X.csv
    python tools/ncu_hot.py X.csv [top]
"""
import csv
import sys


def main():
    rows = list(csv.reader(open(sys.argv[1])))
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
    hdr = rows[1]
    ia, isrc, iss = hdr.index("Address"), hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)")
    data = []
    for r in rows[2:]:
        if len(r) < len(hdr):
            continue
        try:
            data.append((int(r[iss] or 0), r[ia], r[isrc]))
        except ValueError:
            pass
    tot = sum(d[0] for d in data) or 1
    idx = {d[1]: i for i, d in enumerate(data)}
    for s, a, src in sorted(data, reverse=True)[:top]:
        i = idx[a]
        prev = data[i - 1][2] if i else ""
        print(f"{100 * s / tot:5.1f}% {a} {src[:70]:70s} | prev: {prev[:50]}")


if __name__ == "__main__":
    main()
