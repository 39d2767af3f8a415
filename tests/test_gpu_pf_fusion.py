"""Tied-layer parameter-flow fusion (plan `pf_fused_layers`): the layers of a
tied HMM share their transition tiles, so their parameter flows run as ONE
contraction over the layers' batches laid end to end along K (each layer's
pre-converted operand images one segment), stored once, instead of one
reduction pass per layer.  Checked against the float64 oracle through the
API pass (one stream) and the graphed lean training step (side stream, the
top layer staged on the main stream), and against the unfused kernels
(PCB_NO_PF_FUSE=1, read per launch)."""
import numpy as np
import pytest

import oracle
from _golden import rel_err

pytestmark = pytest.mark.gpu
RTOL = 1e-4


def _np(t):
    return t.detach().double().cpu().numpy()


def _hmm():
    from paper_2406_00766_b200 import structures as S
    from paper_2406_00766_b200.compiler import CompileConfig, compile_circuit
    g = S.build_hmm(S.StructureConfig(kind="hmm", seq_len=6, hidden_dim=1024, vocab_size=50,
                                      seed=5, tied=True))
    return compile_circuit(g, CompileConfig(block_size=32))


def test_fused_parameter_flows_api(monkeypatch):
    import torch
    from paper_2406_00766_b200.runtime import backward, forward
    from paper_2406_00766_b200.runtime.plan import device_plan
    c = _hmm()
    assert device_plan(c).info["pf_fused_layers"] >= 4
    x = np.random.default_rng(1).integers(0, 50, size=(192, 6))
    x[::7, 2] = -1
    rl, rb = oracle.forward(c, x)
    oracle.backward(c, rb)
    got = {}
    for mode in ("fused", "unfused"):
        if mode == "unfused":
            monkeypatch.setenv("PCB_NO_PF_FUSE", "1")
        _, bufs = forward(c, x)
        backward(c, bufs)
        torch.cuda.synchronize()
        got[mode] = _np(bufs.f_params)[:c.theta_size]
        assert rel_err(got[mode], rb.f_params[:c.theta_size]) < RTOL, mode
    assert rel_err(got["fused"], got["unfused"]) < 1e-5


def test_fused_parameter_flows_lean_train_step():
    import torch
    from paper_2406_00766_b200.runtime.em import apply_theta
    from paper_2406_00766_b200.runtime.step import TrainStep
    c = _hmm()
    x = np.random.default_rng(2).integers(0, 50, size=(160, 6))
    theta0 = c.theta.copy()
    ts = TrainStep(c, 160, pseudocount=1e-6, step_size=1.0, graph=True)
    ll = float(ts.run(torch.from_numpy(x.astype(np.int32)).cuda()).item())
    got = _np(ts.plan.theta)
    apply_theta(c, theta0)
    lr, rb = oracle.forward(c, x, theta=theta0)
    oracle.backward(c, rb, theta=theta0)
    want = oracle.em_step_full(c, rb.f_params, theta=theta0, pseudocount=1e-6)
    assert abs(ll - lr.sum()) <= 1e-6 * abs(lr.sum())
    assert rel_err(got, want) < RTOL


def test_em_tile_blocks_split_kernel(monkeypatch):
    """Tile blocks of more than 8 32 x 32 tiles (1024 hidden: 32 per block)
    take k_em_tiles32 (four tile groups per CTA); PCB_NO_EM_SPLIT32=1 (read
    per launch) runs them through k_em_tiles.  Both against the float64
    oracle's EM step."""
    import torch
    from paper_2406_00766_b200.runtime import backward, em_update_, forward
    from paper_2406_00766_b200.runtime.plan import device_plan
    c = _hmm()
    x = np.random.default_rng(3).integers(0, 50, size=(128, 6))
    _, rb = oracle.forward(c, x)
    oracle.backward(c, rb)
    want = oracle.em_step_mini(c.theta, oracle.em_step_full(c, rb.f_params, pseudocount=1e-6), 0.25)
    plan = device_plan(c)
    saved = plan.theta.clone()
    got = {}
    for mode in ("split", "single"):
        if mode == "single":
            monkeypatch.setenv("PCB_NO_EM_SPLIT32", "1")
        _, bufs = forward(c, x)
        backward(c, bufs)
        em_update_(c, bufs.f_params, pseudocount=1e-6, step_size=0.25, plan=plan)
        torch.cuda.synchronize()
        got[mode] = _np(plan.theta)
        plan.theta.copy_(saved)
        plan.refresh_mma()
        assert rel_err(got[mode], want) < RTOL, mode
    assert rel_err(got["split"], got["single"]) < 1e-6
