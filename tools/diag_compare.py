"""Per-layer divergence of the device paths (TC / SIMT) against the float64 oracle."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import numpy as np
import torch

import oracle
from paper_2406_00766_b200 import structures as S
from paper_2406_00766_b200.compiler import CompileConfig, compile_circuit
from paper_2406_00766_b200.runtime import forward


def main():
    n, h, ncat, B = (int(a) for a in sys.argv[1:5])
    g = S.build_hclt(S.StructureConfig(kind="hclt", num_vars=n, hidden_dim=h,
                                       num_categories=ncat, seed=0))
    c = compile_circuit(g, CompileConfig(block_size=min(32, h)), validate=False)
    x = np.random.default_rng(1).integers(0, ncat, size=(B, n))
    ref_l, rb = oracle.forward(c, x)
    print("layers", len(c.layers), "oracle ll0", ref_l[:3])
    for tc in (True, False):
        lroot, bufs = forward(c, x, tensor_cores=tc)
        torch.cuda.synchronize()
        vals = bufs.values.double().cpu().numpy()
        print(f"tc={tc} ll0 {lroot[:3].tolist()} max|dll| {np.max(np.abs(lroot.double().cpu().numpy() - ref_l)):.4g}")
        for li, L in enumerate(c.layers):
            rows = np.concatenate([(gr.sum_ids[:, None] + np.arange(L.k_m)).ravel()
                                   for gr in L.fwd_groups])
            a, r = vals[rows], rb.values[rows]
            fin = np.isfinite(r)
            err = np.max(np.abs(a[fin] - r[fin])) if fin.any() else 0.0
            bad = np.argwhere(np.abs(np.where(fin, a - r, 0)) > 1e-2)
            print(f"  layer {li} d={L.depth} err {err:.3g} nbad {len(bad)}"
                  + (f" first {bad[0].tolist()}" if len(bad) else ""))


if __name__ == "__main__":
    main()
