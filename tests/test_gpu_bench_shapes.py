"""GPU parity at the shapes the bench runs (BASELINE configs[1] / [2]),
against the float64 oracle at the north-star tolerance (1e-4 relative on
log-likelihoods, parameter flows and updated parameters).

* HCLT latent 256, block 32, batch 512: super-rows of 8 stacked 32 x 32
  tiles (N = 256), 256-child parameter-flow items, 256-entry simplex groups
  summed from TMEM by the fused-EM epilogue (leaf layer of a 400-variable
  tree: > 148 super-rows, so its parameter flows run unsplit and fuse EM).
* 3072 variables (configs[1]'s variable count): |log p| ~ 1.7e4, where the
  fp32 spacing is 2^-9.  Log values are stored as (integer block base, fp32
  offset) pairs, so flow ratios exp(l_child - l_parent) keep full fp32
  precision; a plain fp32 log value would carry ~1e-3 relative error here.
* Tied HMM with 2048 hidden states over a 4096-token vocabulary: 64-block
  (split-K) contractions and the CTA-per-group EM of >= 2048-entry groups
  (k_em_big: transition rows and emission pmfs).
"""
import numpy as np
import pytest

import oracle
from _golden import rel_err
from oracle.engine import log_gap

pytestmark = pytest.mark.gpu
RTOL = 1e-4


def _np(t):
    return t.detach().double().cpu().numpy()


def _api_vs_oracle(c, x, *, values=False, step=0.01):
    """forward / backward / em_update_ through the drop-in API vs the oracle."""
    import torch
    from paper_2406_00766_b200.runtime import backward, em_update_, forward
    from paper_2406_00766_b200.runtime.plan import device_plan
    lroot, bufs = forward(c, x)
    backward(c, bufs)
    torch.cuda.synchronize()
    rl, rb = oracle.forward(c, x)
    oracle.backward(c, rb)
    assert log_gap(_np(lroot), rl, 1e-5, RTOL) <= 1.0
    assert rel_err(_np(bufs.f_params)[:c.theta_size], rb.f_params[:c.theta_size]) < RTOL
    assert rel_err(_np(bufs.flows), rb.flows) < RTOL
    if values:
        # materialised log values (block base + offset) against the oracle's
        got, ref = _np(bufs.values), rb.values
        fin = np.isfinite(ref)
        assert np.array_equal(np.isfinite(got), fin)
        assert np.max(np.abs(got[fin] - ref[fin]) / (1e-5 + 1e-6 * np.abs(ref[fin]))) <= 1.0
    plan = device_plan(c)
    saved = plan.theta.clone()
    new = oracle.em_step_full(c, rb.f_params, pseudocount=1e-6)
    want = oracle.em_step_mini(c.theta, new, step)
    em_update_(c, bufs.f_params, pseudocount=1e-6, step_size=step, plan=plan)
    got = _np(plan.theta)
    plan.theta.copy_(saved)
    plan.refresh_mma()
    assert rel_err(got, want) < RTOL
    return bufs


def test_hclt256_block32_batch512_api():
    """configs[1]'s layer shapes through forward / backward / EM (16 variables)."""
    from paper_2406_00766_b200 import structures as S
    from paper_2406_00766_b200.compiler import CompileConfig, compile_circuit
    g = S.build_hclt(S.StructureConfig(kind="hclt", num_vars=16, hidden_dim=256,
                                       num_categories=256, seed=0))
    c = compile_circuit(g, CompileConfig(block_size=32))
    assert {L.k_m for L in c.layers[:-1]} == {32}
    x = np.random.default_rng(1).integers(0, 256, size=(512, 16))
    x[np.random.default_rng(2).random(x.shape) < 0.05] = -1
    _api_vs_oracle(c, x, values=True, step=1.0)


def test_hclt256_train_step_fused_em_batch512():
    """The bench's training step (lean launches, CUDA graph, EM fused into the
    leaf layer's parameter-flow epilogue and into the input flows) on a
    400-variable HCLT-256 at batch 512, full EM replacement (step 1), so the
    updated parameters are the normalised flows themselves."""
    import torch
    from paper_2406_00766_b200 import structures as S
    from paper_2406_00766_b200.compiler import CompileConfig, compile_circuit
    from paper_2406_00766_b200.runtime.em import apply_theta
    from paper_2406_00766_b200.runtime.plan import device_plan
    from paper_2406_00766_b200.runtime.step import TrainStep
    g = S.build_hclt(S.StructureConfig(kind="hclt", num_vars=400, hidden_dim=256,
                                       num_categories=256, seed=0))
    c = compile_circuit(g, CompileConfig(block_size=32), validate=False)
    info = device_plan(c).info
    assert info["em_fused_layers"] > 0 and info["input_inline_em"] and info["leaf_alias"]
    x = np.random.default_rng(3).integers(0, 256, size=(512, 400))
    theta0 = c.theta.copy()
    apply_theta(c, theta0)
    ts = TrainStep(c, 512, pseudocount=1e-6, step_size=1.0, graph=True)
    ll = float(ts.run(torch.from_numpy(x.astype(np.int32)).cuda()).item())
    got = _np(ts.plan.theta)
    apply_theta(c, theta0)
    lr, rb = oracle.forward(c, x, theta=theta0)
    oracle.backward(c, rb, theta=theta0)
    want = oracle.em_step_full(c, rb.f_params, theta=theta0, pseudocount=1e-6)
    assert abs(ll - lr.sum()) <= 1e-6 * abs(lr.sum())
    assert rel_err(got, want) < RTOL


def test_hclt3072_precision():
    """3072 variables (|log p| ~ 1.7e4): LL, node values, node and parameter
    flows and the EM update at 1e-4 through the API, and the graphed lean
    training step's update."""
    import torch
    from paper_2406_00766_b200 import structures as S
    from paper_2406_00766_b200.compiler import CompileConfig, compile_circuit
    from paper_2406_00766_b200.runtime.em import apply_theta
    from paper_2406_00766_b200.runtime.step import TrainStep
    g = S.build_hclt(S.StructureConfig(kind="hclt", num_vars=3072, hidden_dim=32,
                                       num_categories=256, seed=0))
    c = compile_circuit(g, CompileConfig(block_size=32), validate=False)
    x = np.random.default_rng(4).integers(0, 256, size=(64, 3072))
    x[np.random.default_rng(5).random(x.shape) < 0.02] = -1
    _api_vs_oracle(c, x, values=True, step=1.0)
    theta0 = c.theta.copy()
    ts = TrainStep(c, 64, pseudocount=1e-6, step_size=1.0, graph=True)
    ts.run(torch.from_numpy(x.astype(np.int32)).cuda())
    got = _np(ts.plan.theta)
    apply_theta(c, theta0)
    lr, rb = oracle.forward(c, x, theta=theta0)
    oracle.backward(c, rb, theta=theta0)
    want = oracle.em_step_full(c, rb.f_params, theta=theta0, pseudocount=1e-6)
    assert rel_err(got, want) < RTOL


def test_hmm2048_vocab4096_big_groups():
    """Tied HMM, 2048 hidden states, 4096-token vocabulary (batch 96 with
    missing tokens): long-K split contractions and >= 2048-entry EM groups."""
    from paper_2406_00766_b200 import structures as S
    from paper_2406_00766_b200.compiler import CompileConfig, compile_circuit
    from paper_2406_00766_b200.runtime.plan import EM_BIG
    g = S.build_hmm(S.StructureConfig(kind="hmm", seq_len=4, hidden_dim=2048, vocab_size=4096,
                                      seed=3, tied=True))
    c = compile_circuit(g, CompileConfig(block_size=32))
    assert int(np.diff(c.group_off).max()) >= EM_BIG
    x = np.random.default_rng(6).integers(0, 4096, size=(96, 4))
    x[::7, 2] = -1
    _api_vs_oracle(c, x, step=1.0)


def test_pd_elementwise_block32():
    """configs[3] family: the PyJuice PD (elementwise products per cut,
    dense h x (cuts h) sum blocks on tensor cores) at h = 64 on a 6 x 6 x 3
    image with cuts every 2 pixels, through the API and the training step."""
    import torch
    from paper_2406_00766_b200 import structures as S
    from paper_2406_00766_b200.compiler import CompileConfig, compile_circuit
    from paper_2406_00766_b200.runtime.em import apply_theta
    from paper_2406_00766_b200.runtime.step import TrainStep
    cfg = S.StructureConfig(kind="pd", shape=(6, 6, 3), split_interval=2, hidden_dim=64,
                            num_categories=16, elementwise=True, seed=3)
    g = S.build_pd(cfg)
    c = compile_circuit(g, CompileConfig(block_size=32))
    assert c.num_edges == S.pd_edge_count((6, 6, 3), 64, 2)
    assert max(L.k_m for L in c.layers) == 32
    x = np.random.default_rng(8).integers(0, 16, size=(192, 108))
    x[np.random.default_rng(9).random(x.shape) < 0.05] = -1
    _api_vs_oracle(c, x, values=True, step=1.0)
    theta0 = c.theta.copy()
    ts = TrainStep(c, 192, pseudocount=1e-6, step_size=1.0, graph=True)
    ts.run(torch.from_numpy(x.astype(np.int32)).cuda())
    got = _np(ts.plan.theta)
    apply_theta(c, theta0)
    lr, rb = oracle.forward(c, x, theta=theta0)
    oracle.backward(c, rb, theta=theta0)
    want = oracle.em_step_full(c, rb.f_params, theta=theta0, pseudocount=1e-6)
    assert rel_err(got, want) < RTOL


def test_ratspn_depth7_repetitions():
    """configs[4] family: RAT-SPN of depth 7 with repetitions (32 sums per
    region: dense 32 x 1024 cross-product blocks, split-K contractions) over
    140 variables at batch 256, through the API and the training step."""
    import torch
    from paper_2406_00766_b200 import structures as S
    from paper_2406_00766_b200.compiler import CompileConfig, compile_circuit
    from paper_2406_00766_b200.runtime.em import apply_theta
    from paper_2406_00766_b200.runtime.step import TrainStep
    cfg = S.StructureConfig(kind="ratspn", num_vars=140, depth=7, hidden_dim=32,
                            num_input_components=8, num_categories=16, num_repetitions=2,
                            seed=4)
    g = S.build_ratspn(cfg)
    c = compile_circuit(g, CompileConfig(block_size=32))
    assert c.num_edges == S.ratspn_edge_count(140, 7, 32, 8, 2)
    x = np.random.default_rng(10).integers(0, 16, size=(256, 140))
    x[np.random.default_rng(11).random(x.shape) < 0.05] = -1
    _api_vs_oracle(c, x, step=1.0)
    theta0 = c.theta.copy()
    ts = TrainStep(c, 256, pseudocount=1e-6, step_size=1.0, graph=True)
    ts.run(torch.from_numpy(x.astype(np.int32)).cuda())
    got = _np(ts.plan.theta)
    apply_theta(c, theta0)
    lr, rb = oracle.forward(c, x, theta=theta0)
    oracle.backward(c, rb, theta=theta0)
    want = oracle.em_step_full(c, rb.f_params, theta=theta0, pseudocount=1e-6)
    assert rel_err(got, want) < RTOL


@pytest.mark.parametrize("tree,kw", [("chain", dict(num_vars=48)),
                                     ("grid", dict(num_vars=48, shape=(4, 4, 3)))])
def test_hclt_deep_trees(tree, kw):
    """The deep-tree workloads' generators (hclt256_chain / hclt256_grid) at
    reduced size: one TC layer per tree level, through the API and the
    graphed lean training step."""
    import torch
    from paper_2406_00766_b200 import structures as S
    from paper_2406_00766_b200.compiler import CompileConfig, compile_circuit
    from paper_2406_00766_b200.runtime.em import apply_theta
    from paper_2406_00766_b200.runtime.step import TrainStep
    g = S.build_hclt(S.StructureConfig(kind="hclt", hidden_dim=64, num_categories=8, seed=2,
                                       tree=tree, **kw))
    c = compile_circuit(g, CompileConfig(block_size=32))
    x = np.random.default_rng(15).integers(0, 8, size=(128, c.num_vars))
    x[np.random.default_rng(16).random(x.shape) < 0.05] = -1
    _api_vs_oracle(c, x, step=1.0)
    theta0 = c.theta.copy()
    ts = TrainStep(c, 128, pseudocount=1e-6, step_size=1.0, graph=True)
    ts.run(torch.from_numpy(x.astype(np.int32)).cuda())
    got = _np(ts.plan.theta)
    apply_theta(c, theta0)
    lr, rb = oracle.forward(c, x, theta=theta0)
    oracle.backward(c, rb, theta=theta0)
    want = oracle.em_step_full(c, rb.f_params, theta=theta0, pseudocount=1e-6)
    assert rel_err(got, want) < RTOL
