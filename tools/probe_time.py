"""Quick device timing probe: fwd / bwd / EM of an HCLT at a given width."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import numpy as np
import torch

from paper_2406_00766_b200 import structures as S
from paper_2406_00766_b200.compiler import CompileConfig, compile_circuit
from paper_2406_00766_b200.runtime import _lib, backward, em_update_, forward


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 3072
    h = int(sys.argv[2]) if len(sys.argv) > 2 else 64
    B = int(sys.argv[3]) if len(sys.argv) > 3 else 512
    t = time.time()
    g = S.build_hclt(S.StructureConfig(kind="hclt", num_vars=n, hidden_dim=h,
                                       num_categories=256, seed=0))
    c = compile_circuit(g, CompileConfig(block_size=min(32, h)), validate=False)
    print(f"build+compile {time.time() - t:.1f}s edges {c.num_edges}", flush=True)
    x = np.random.default_rng(1).integers(0, 256, size=(B, n))
    for tc in (True, False):
        lroot, bufs = forward(c, x, tensor_cores=tc)
        backward(c, bufs, tensor_cores=tc)
        torch.cuda.synchronize()
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
        reps = 3
        tf = tb = te = 0.0
        for _ in range(reps):
            ev[0].record()
            forward(c, x, bufs=bufs, tensor_cores=tc, validate=False)
            ev[1].record()
            backward(c, bufs, tensor_cores=tc)
            ev[2].record()
            em_update_(c, bufs.f_params, pseudocount=1e-6, step_size=0.01, check=False)
            ev[3].record()
            torch.cuda.synchronize()
            tf += ev[0].elapsed_time(ev[1])
            tb += ev[1].elapsed_time(ev[2])
            te += ev[2].elapsed_time(ev[3])
        print(f"tc={tc} B={B}: fwd {tf / reps:.2f} ms  bwd {tb / reps:.2f} ms  em {te / reps:.2f} ms  "
              f"ll0 {float(lroot[0]):.4f}", flush=True)


if __name__ == "__main__":
    main()
