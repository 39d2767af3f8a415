"""BASELINE configs[0] CPU baseline with the REFERENCE itself (build container
only: imports /root/reference): HCLT latent 16 on 784 MNIST-shaped vars,
block 16, end-to-end ``pcirc.train.train`` (mini-batch EM, B = 512, alpha
0.01, kappa 1e-6) on 4096 synthetic samples with T = 1 and T = cpu_count
threads.  Prints samples/s and the 60k-sample epoch
extrapolation.  The circuit is this package's HCLT generator, rebuilt node
for node as a reference CircuitGraph.

    PYTHONDONTWRITEBYTECODE=1 python tools/ref_cpu_baseline.py
"""
import json
import os
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests" / "golden"))
sys.dont_write_bytecode = True

import numpy as np  # noqa: E402

import make_golden as mg  # noqa: E402  (graph_arrays / from_parts_ref; imports the reference)
from paper_2406_00766_b200 import structures as S  # noqa: E402


def main():
    g = S.build_hclt(S.StructureConfig(kind="hclt", num_vars=784, hidden_dim=16,
                                       num_categories=256, seed=0))
    rg = mg.from_parts_ref(mg.graph_arrays(g))
    c = mg.compile_circuit(rg, mg.CompileConfig(block_size=16))
    x = np.random.default_rng(1).integers(0, 256, size=(4096, 784))
    out = {}
    for T in (1, os.cpu_count()):
        t0 = time.perf_counter()
        mg.train(c, x, mg.TrainConfig(epochs=1, batch_size=512, mode="mini", step_size=0.01,
                                      pseudocount=1e-6, threads=T))
        dt = time.perf_counter() - t0
        out[f"threads={T}"] = {"samples_per_s": 4096 / dt, "sec_per_epoch_60k": 60000 * dt / 4096}
        print(T, out[f"threads={T}"], flush=True)
    print(json.dumps({"config": "hclt16 (784 vars, h=16, 256 cats, block 16, B=512)",
                      "cores": os.cpu_count(), "reference": "pcirc.train.train", **out}))


if __name__ == "__main__":
    main()
