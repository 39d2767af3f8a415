"""Per-kernel-class milliseconds of the lean training step (serialised, no
side-stream overlap), for kernel A/B experiments with PCB_LIB variants:
    python tools/step_classes.py <workload> [steps]
No EM status checks: ablated kernels may produce garbage."""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch

import bench
from paper_2406_00766_b200.runtime import _lib
from paper_2406_00766_b200.runtime.step import TrainStep


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "hclt256"
    steps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
    w = bench.WORKLOADS[name]
    c = bench.build_circuit(w)
    ts = TrainStep(c, w["batch"], pseudocount=1e-6, step_size=0.01, graph=False)
    ts.serial = True
    x = torch.from_numpy(bench.synthetic_batches(c, w, w["batch"], 1, 0)[0]).cuda()
    ts.run(x)
    torch.cuda.synchronize()
    _lib.profile_enable(True)
    _lib.profile_read()
    for _ in range(steps):
        ts.run(x)
    torch.cuda.synchronize()
    prof = _lib.profile_read()
    print(json.dumps({k: round(v[0] / steps, 3) for k, v in prof.items() if v[0] > 0}))


if __name__ == "__main__":
    main()
