"""Run a few training steps of a workload exactly as bench.py does (the
``runtime.step.TrainStep`` launch sequence, eager), for ncu launch lists and
kernel captures:  python tools/ncu_step.py <workload> <steps>"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch

import bench
from paper_2406_00766_b200.runtime.step import TrainStep


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "hclt256"
    steps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
    w = bench.WORKLOADS[name]
    c = bench.build_circuit(w)
    B = w["batch"]
    ts = TrainStep(c, B, pseudocount=1e-6, step_size=0.01, graph=False)
    x = torch.from_numpy(bench.synthetic_batches(c, w, B, 1, 0)[0]).cuda()
    for _ in range(steps):
        ts.run(x)
    torch.cuda.synchronize()
    print("done", name, steps)


if __name__ == "__main__":
    main()
