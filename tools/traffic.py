"""Measured DRAM traffic per step and kernel class from an ncu launch list
taken with ``--metrics gpu__time_duration.sum,dram__bytes_read.sum,
dram__bytes_write.sum`` over ``tools/ncu_step.py <workload> <steps>``:

    python tools/traffic.py launches.csv <steps> <workload>   -> profiles/traffic_<workload>.json

bench.py reports the dominant class's entry as ``roofline.traffic`` (bytes
per step, the same unit as ``roofline.algorithmic_bytes_per_step``).
"""
import collections
import csv
import json
import sys
from pathlib import Path

CLASSES = [
    ("k_input_fwd", "input_fwd"), ("k_prod_block", "prod_eval"),
    ("k_sum_ws<0", "sum_fwd_tc"), ("k_group_shift<0", "sum_fwd_tc"),
    ("k_sum_fwd_simt", "sum_fwd_simt"),
    ("k_param_flow", "param_flow"), ("k_ratio", "param_flow"), ("k_pf_", "param_flow"),
    ("k_sum_ws<1", "child_flow"), ("k_group_shift<1", "child_flow"),
    ("k_child_flow", "child_flow"),
    ("k_flow_push", "accum_push"), ("k_push_ratio", "accum_push"), ("k_input_flow", "input_flow"), ("k_input_param_flow", "input_flow"),
    ("k_replica", "replica"), ("k_em", "em"), ("k_theta_to_mma", "em"),
]
UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}


def main():
    path, steps, wl = sys.argv[1], int(sys.argv[2]), sys.argv[3]
    rows = list(csv.reader(open(path)))
    hdr, per_kernel = None, collections.defaultdict(dict)
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if not hdr or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        if d["Metric Name"].startswith("dram__bytes"):
            per_kernel[(d["ID"], d["Kernel Name"])][d["Metric Name"]] = \
                float(d["Metric Value"].replace(",", "")) * UNIT.get(d["Metric Unit"], 1)
    out = collections.defaultdict(float)
    for (_, name), m in per_kernel.items():
        cls = next((c for key, c in CLASSES if key in name), None)
        if cls:
            out[cls] += (m.get("dram__bytes_read.sum", 0) + m.get("dram__bytes_write.sum", 0)) / steps
    dst = Path(__file__).resolve().parents[1] / "profiles" / f"traffic_{wl}.json"
    dst.write_text(json.dumps({k: round(v) for k, v in sorted(out.items())}, indent=1) + "\n")
    print(dst.read_text())


if __name__ == "__main__":
    main()
