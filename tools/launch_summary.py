"""Summarise an ncu launch list (``--metrics gpu__time_duration.sum --csv``):
per-kernel launch count, time per step and share.  Usage:
    python tools/launch_summary.py gpurun_out/launches.csv [steps] [--per-launch NAME]
"""
import collections
import csv
import sys


def load(path):
    rows = list(csv.reader(open(path)))
    hdr, data = None, []
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d["Metric Name"] == "gpu__time_duration.sum":
                data.append(d)
    return data


def main():
    path = sys.argv[1]
    steps = int(sys.argv[2]) if len(sys.argv) > 2 and sys.argv[2].isdigit() else 2
    data = load(path)
    agg = collections.defaultdict(lambda: [0, 0.0])
    for d in data:
        k = d["Kernel Name"].split("(")[0].replace("void ", "")
        agg[k][0] += 1
        agg[k][1] += float(d["Metric Value"].replace(",", ""))
    tot = sum(v[1] for v in agg.values())
    print(f"{'kernel':58s} {'launches':>8s} {'ms/step':>9s} {'share':>6s}")
    for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{k[:58]:58s} {v[0]:8d} {v[1] / 1e6 / steps:9.3f} {100 * v[1] / tot:5.1f}%")
    print(f"{'total':58s} {len(data):8d} {tot / 1e6 / steps:9.3f}")
    if "--per-launch" in sys.argv:
        name = sys.argv[sys.argv.index("--per-launch") + 1]
        ds = [d for d in data if name in d["Kernel Name"]]
        print(name, [(d["Grid Size"], round(float(d["Metric Value"]) / 1e3))
                     for d in ds[:len(ds) // steps]])


if __name__ == "__main__":
    main()
