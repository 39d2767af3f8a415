"""Long-K shift paths of the tensor-core sum kernels (forward and child
flows) against the float64 oracle: the per-(super-row, sample) shifts of a
32-or-more-block contraction come from the 17 warps of a one-item-per-CTA
kernel (default at these sizes), from the separate reduction kernel
(PCB_NO_COOP_SHIFT=1), or from the shift warp one item ahead
(PCB_SHIFT_WARP_MIN_ITEMS=1).  The library reads these per launch."""
import numpy as np
import pytest

import oracle
from _golden import rel_err
from oracle.engine import log_gap

pytestmark = pytest.mark.gpu
RTOL = 1e-4

PATHS = [
    {},
    {"PCB_NO_COOP_SHIFT": "1"},
    {"PCB_NO_COOP_SHIFT": "1", "PCB_SHIFT_WARP_MIN_ITEMS": "1"},
]


def _np(t):
    return t.detach().double().cpu().numpy()


def _check(c, x, monkeypatch):
    import torch
    from paper_2406_00766_b200.runtime import backward, forward
    rl, rb = oracle.forward(c, x)
    oracle.backward(c, rb)
    for env in PATHS:
        for k in ("PCB_NO_COOP_SHIFT", "PCB_SHIFT_WARP_MIN_ITEMS"):
            monkeypatch.delenv(k, raising=False)
        for k, v in env.items():
            monkeypatch.setenv(k, v)
        lroot, bufs = forward(c, x)
        backward(c, bufs)
        torch.cuda.synchronize()
        assert log_gap(_np(lroot), rl, 1e-5, RTOL) <= 1.0, env
        assert rel_err(_np(bufs.flows), rb.flows) < RTOL, env
        assert rel_err(_np(bufs.f_params)[:c.theta_size], rb.f_params[:c.theta_size]) < RTOL, env


def test_ratspn_long_k_forward_shift_paths(monkeypatch):
    """RAT-SPN regions of 32 sums over 32 x 32 = 1024 products: 32-block
    forward contractions."""
    from paper_2406_00766_b200 import structures as S
    from paper_2406_00766_b200.compiler import CompileConfig, compile_circuit
    cfg = S.StructureConfig(kind="ratspn", num_vars=24, depth=3, hidden_dim=32,
                            num_input_components=8, num_categories=6, num_repetitions=2, seed=6)
    c = compile_circuit(S.build_ratspn(cfg), CompileConfig(block_size=32))
    assert max(g.param_ids.shape[1] for L in c.layers for g in L.fwd_groups) >= 32
    x = np.random.default_rng(12).integers(0, 6, size=(256, 24))
    x[np.random.default_rng(13).random(x.shape) < 0.05] = -1
    _check(c, x, monkeypatch)


def test_hmm_long_k_forward_and_child_flow_shift_paths(monkeypatch):
    """Tied HMM with 1024 hidden states: 32-block forward and child-flow
    contractions."""
    from paper_2406_00766_b200 import structures as S
    from paper_2406_00766_b200.compiler import CompileConfig, compile_circuit
    g = S.build_hmm(S.StructureConfig(kind="hmm", seq_len=4, hidden_dim=1024, vocab_size=40,
                                      seed=2, tied=True))
    c = compile_circuit(g, CompileConfig(block_size=32))
    x = np.random.default_rng(14).integers(0, 40, size=(160, 4))
    x[::9, 1] = -1
    _check(c, x, monkeypatch)
