"""Attribute an ncu source-page stall profile (sass csv, see ncu_hot.py) to
CUDA source lines via the cubin's line table:
    python tools/ncu_lines.py X_src.csv kernel.cubin <mangled-name-substring> [top]
(cubins: ``cuobjdump -xelf all libpcirc_b200.so`` in a scratch dir; build with -lineinfo)."""
import csv
import re
import subprocess
import sys
from collections import defaultdict


def main():
    src, cubin, fn = sys.argv[1], sys.argv[2], sys.argv[3]
    top = int(sys.argv[4]) if len(sys.argv) > 4 else 30
    rows = list(csv.reader(open(src)))
    hdr = rows[1]
    ia, iss = hdr.index("Address"), hdr.index("Warp Stall Sampling (All Samples)")
    samples = []
    for r in rows[2:]:
        if len(r) >= len(hdr):
            try:
                samples.append((int(r[ia], 16), int(r[iss] or 0)))
            except ValueError:
                pass
    base = samples[0][0]
    dis = subprocess.run(["nvdisasm", "-g", "-c", cubin], capture_output=True, text=True).stdout
    line_of, cur, inside, last = {}, None, False, None
    for ln in dis.splitlines():
        if ln.startswith("//----") and ".text." in ln:
            inside = fn in ln
            continue
        if not inside:
            continue
        m = re.match(r"\s*//## File \"(.*)\", line (\d+)", ln)
        if m:
            cur = f"{m.group(1).split('/')[-1]}:{m.group(2)}"
            continue
        m = re.match(r"\s*/\*([0-9a-f]{4,})\*/", ln)
        if m:
            line_of[int(m.group(1), 16)] = cur
    agg = defaultdict(int)
    for a, s in samples:
        agg[line_of.get(a - base, "?")] += s
    tot = sum(agg.values()) or 1
    for k, v in sorted(agg.items(), key=lambda x: -x[1])[:top]:
        print(f"{100 * v / tot:5.1f}% {k}")


if __name__ == "__main__":
    main()
