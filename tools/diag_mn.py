"""Diagnose the MN-major UMMA self-test and the TC vs SIMT child flows."""
import sys
import traceback
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import numpy as np
import torch

from paper_2406_00766_b200.runtime import _lib


def selftest(n, k, variant):
    g = torch.Generator(device="cpu").manual_seed(7 * n + k)
    a = torch.randn(128, k, generator=g).to(torch.bfloat16).cuda()
    bkn = torch.randn(k, n, generator=g).to(torch.bfloat16).cuda()
    d = torch.zeros(128, n, dtype=torch.float32, device="cuda")
    _lib.call("pcb_tc_selftest_mn", _lib.stream_handle(), n, k, variant, a.data_ptr(),
              bkn.data_ptr(), d.data_ptr())
    torch.cuda.synchronize()
    want = a.float() @ bkn.float()
    return float((d - want).abs().max())


def main():
    which = sys.argv[1]
    if which == "mn":
        n, k, v = int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
        try:
            print(f"mn n={n} k={k} variant={v}: maxerr {selftest(n, k, v):.3g}", flush=True)
        except Exception as e:
            print(f"mn n={n} k={k} variant={v}: EXC {str(e)[:120]}", flush=True)
    elif which == "cf":
        import oracle
        from paper_2406_00766_b200 import structures as S
        from paper_2406_00766_b200.compiler import CompileConfig, compile_circuit
        from paper_2406_00766_b200.runtime import backward, forward
        g = S.build_hclt(S.StructureConfig(kind="hclt", num_vars=20, hidden_dim=64,
                                           num_categories=8, seed=5))
        c = compile_circuit(g, CompileConfig(block_size=32))
        x = np.random.default_rng(2).integers(0, 8, size=(131, 20))
        rl, rb = oracle.forward(c, x)
        oracle.backward(c, rb)
        for tc in (False, True):
            try:
                lroot, bufs = forward(c, x, tensor_cores=tc)
                backward(c, bufs, tensor_cores=tc)
                torch.cuda.synchronize()
                fl = bufs.flows.double().cpu().numpy()
                fp = bufs.f_params.double().cpu().numpy()[:c.theta_size]
                ll = lroot.double().cpu().numpy()
                print(f"tc={tc} dll {np.abs(ll - rl).max():.3g} dflow "
                      f"{np.abs(fl - rb.flows).max():.3g} dfp "
                      f"{np.abs(fp - rb.f_params[:c.theta_size]).max():.3g} "
                      f"max fp {np.abs(rb.f_params).max():.3g}", flush=True)
            except Exception:
                traceback.print_exc()


if __name__ == "__main__":
    main()
