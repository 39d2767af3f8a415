"""Precision diagnostic: GPU forward/backward/EM vs the float64 oracle at scale."""
import sys, time
from pathlib import Path
import numpy as np
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
sys.path.insert(0, str(Path(__file__).resolve().parents[1] / "tests"))
import torch
import oracle
from _golden import rel_err
from paper_2406_00766_b200 import structures as S
from paper_2406_00766_b200.compiler import CompileConfig, compile_circuit
from paper_2406_00766_b200.runtime import backward, forward, em_update_
from paper_2406_00766_b200.runtime.plan import device_plan


def np_(t):
    return t.detach().double().cpu().numpy()


def run(name, g, k, B, ncat, tc=True):
    c = compile_circuit(g, CompileConfig(block_size=k), validate=False)
    x = np.random.default_rng(4).integers(0, ncat, size=(B, g.num_vars))
    lroot, bufs = forward(c, x, tensor_cores=tc)
    backward(c, bufs, tensor_cores=tc)
    torch.cuda.synchronize()
    rl, rb = oracle.forward(c, x)
    oracle.backward(c, rb)
    ll_err = float(np.max(np.abs(np_(lroot) - rl) / np.abs(rl)))
    fp_err = rel_err(np_(bufs.f_params)[:c.theta_size], rb.f_params[:c.theta_size])
    fl_err = rel_err(np_(bufs.flows), rb.flows)
    new = oracle.em_step_full(c, rb.f_params, pseudocount=1e-6)
    want = oracle.em_step_mini(c.theta, new, 0.01)
    plan = device_plan(c, tensor_cores=tc)
    em_update_(c, bufs.f_params, pseudocount=1e-6, step_size=0.01, plan=plan)
    th_err = rel_err(np_(plan.theta), want)
    want1 = new
    print(f"{name} tc={tc} B={B} |ll|~{np.mean(np.abs(rl)):.0f} ll_rel={ll_err:.2e} "
          f"fparams={fp_err:.2e} flows={fl_err:.2e} theta={th_err:.2e}", flush=True)


if __name__ == "__main__":
    for nv, h in ((3072, 32), (1024, 32), (256, 64)):
        g = S.build_hclt(S.StructureConfig(kind="hclt", num_vars=nv, hidden_dim=h,
                                           num_categories=256, seed=0))
        for tc in (True, False):
            run(f"hclt{nv}x{h}", g, 32, 64, 256, tc)
    g = S.build_hclt(S.StructureConfig(kind="hclt", num_vars=16, hidden_dim=256,
                                       num_categories=256, seed=0))
    run("hclt16x256", g, 32, 512, 256)
