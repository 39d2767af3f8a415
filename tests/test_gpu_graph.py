"""The training step replayed as a CUDA graph equals the eager launches
(same kernels, same data): parameters after several mini-batch EM steps and
the per-step log-likelihoods agree, and both follow the float64 oracle."""
import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu


def _steps(c, xs, graph, theta0):
    import torch
    from paper_2406_00766_b200.runtime.step import TrainStep
    from paper_2406_00766_b200.runtime.em import apply_theta
    apply_theta(c, theta0)  # every run starts from the same table
    ts = TrainStep(c, xs[0].shape[0], pseudocount=1e-6, step_size=0.05, graph=graph)
    lls = []
    for x in xs:
        ll = ts.run(torch.from_numpy(x.astype(np.int32)).cuda())
        lls.append(float(ll.item()))
    return ts.plan.theta.double().cpu().numpy(), np.array(lls), ts


def test_graph_step_matches_eager_and_oracle():
    from paper_2406_00766_b200 import structures as S
    from paper_2406_00766_b200.compiler import CompileConfig, compile_circuit
    g = S.build_hclt(S.StructureConfig(kind="hclt", num_vars=24, hidden_dim=32,
                                       num_categories=8, seed=2))
    c = compile_circuit(g, CompileConfig(block_size=32))
    theta0 = c.theta.copy()
    rng = np.random.default_rng(11)
    xs = [rng.integers(0, 8, size=(160, 24)) for _ in range(3)]
    th_e, ll_e, _ = _steps(c, xs, graph=False, theta0=theta0)
    th_g, ll_g, ts = _steps(c, xs, graph=True, theta0=theta0)
    assert ts.graph is not None and ts.launches_per_step > 0
    np.testing.assert_allclose(ll_g, ll_e, rtol=1e-6)
    np.testing.assert_allclose(th_g, th_e, rtol=1e-5, atol=1e-9)
    # oracle: the same three steps in float64
    theta = theta0.copy()
    for i, x in enumerate(xs):
        lr, rb = oracle.forward(c, x, theta=theta)
        oracle.backward(c, rb, theta=theta)
        new = oracle.em_step_full(c, rb.f_params, theta=theta, pseudocount=1e-6)
        theta = oracle.em_step_mini(theta, new, 0.05)
        assert abs(ll_g[i] - lr.sum()) <= 1e-4 * abs(lr.sum())
    nz = np.abs(theta) > 1e-6
    assert np.max(np.abs(th_g[nz] - theta[nz]) / np.abs(theta[nz])) < 1e-4


@pytest.mark.parametrize("tensor_cores", [True, False])
@pytest.mark.parametrize("kind,k", [("hclt", 16), ("hclt", 32), ("hmm", 32)])
def test_lean_step_matches_full(tensor_cores, kind, k):
    """Lean launches give bit-identical log-likelihoods and the same parameter
    flows, missing values included: leaf products aliased onto their inputs
    (no leaf product pass, no leaf push) and flow ratios formed by the fused
    push (no ratio pass).  Flows agree to float rounding: product flows with
    several parent blocks are accumulated atomically, so their summation order
    varies from run to run in either mode."""
    import ctypes as C

    import torch
    from paper_2406_00766_b200 import structures as S
    from paper_2406_00766_b200.compiler import CompileConfig, compile_circuit
    from paper_2406_00766_b200.runtime import _lib, backward, forward
    from paper_2406_00766_b200.runtime.plan import device_plan
    if kind == "hclt":
        g = S.build_hclt(S.StructureConfig(kind="hclt", num_vars=30, hidden_dim=2 * k,
                                           num_categories=8, seed=5))
        nv, ncat = 30, 8
    else:
        g = S.build_structure(S.StructureConfig(kind="hmm", seq_len=8, hidden_dim=128,
                                                vocab_size=40, seed=2, tied=True))
        nv, ncat = 8, 40
    c = compile_circuit(g, CompileConfig(block_size=k))
    plan = device_plan(c, tensor_cores=tensor_cores)
    assert plan.info["leaf_alias"] == (kind == "hclt")
    assert plan.info["pre_ratio_layers"] > 0
    x = np.random.default_rng(3).integers(0, ncat, size=(200, nv))
    x[np.random.default_rng(4).random(x.shape) < 0.15] = -1
    lr0, b0 = forward(c, x, tensor_cores=tensor_cores)
    backward(c, b0, tensor_cores=tensor_cores)
    want_ll, want_f = lr0.clone(), b0.f_params.clone()
    # the same batch through pcb_train_step with lean launches and no EM
    lr1, b1 = forward(c, x, tensor_cores=tensor_cores)
    ex = C.c_void_p()
    _lib.call("pcb_exec_create", plan.handle, C.byref(ex))
    try:
        _lib.call("pcb_train_step", plan.handle, ex, _lib.stream_handle(), b1.batch_size,
                  b1.ldb, b1.xT.data_ptr(), plan.theta.data_ptr(), b1.values_full.data_ptr(),
                  b1.flows_full.data_ptr(), b1.scratch_full.data_ptr(),
                  b1.flow_scratch_full.data_ptr(), b1.prod_flows_full.data_ptr(),
                  b1.f_params.data_ptr(), b1.lroot.data_ptr(), b1.work.data_ptr(),
                  _lib.STEP_LEAN, 0.0, 1.0, plan.status.data_ptr())
        torch.cuda.synchronize()
    finally:
        _lib.load().pcb_exec_destroy(ex)
    assert torch.equal(lr1, want_ll)
    got, ref = b1.f_params.double(), want_f.double()
    assert torch.max(torch.abs(got - ref) / torch.clamp(ref.abs(), min=1e-30)).item() < 2e-6


@pytest.mark.parametrize("batch", [64, 192])
def test_inline_em_matches_separate_pass(batch):
    """A one-process TrainStep (lean launches; the input-flow pass applies EM
    to the staged inputs' pmfs and, when a layer's parameter flows run
    unsplit (batch 64 here), their epilogue applies EM to the layer's tiles
    and rewrites its bf16 planes) updates theta and the EM status counters
    like the plain forward / backward / pcb_em_update sequence, and the next
    step (which reads the rewritten planes) agrees too."""
    import torch
    from paper_2406_00766_b200 import structures as S
    from paper_2406_00766_b200.compiler import CompileConfig, compile_circuit
    from paper_2406_00766_b200.runtime import backward, forward
    from paper_2406_00766_b200.runtime.em import apply_theta, em_update_
    from paper_2406_00766_b200.runtime.plan import device_plan
    from paper_2406_00766_b200.runtime.step import TrainStep
    g = S.build_hclt(S.StructureConfig(kind="hclt", num_vars=30, hidden_dim=64,
                                       num_categories=8, seed=7))
    c = compile_circuit(g, CompileConfig(block_size=32))
    info = device_plan(c).info
    assert info["input_inline_em"] and info["em_fused_layers"] > 0
    rng = np.random.default_rng(9)
    xs = [rng.integers(0, 8, size=(batch, 30)) for _ in range(2)]
    for x in xs:
        x[rng.random(x.shape) < 0.1] = -1
    theta0 = c.theta.copy()
    apply_theta(c, theta0)
    ts = TrainStep(c, batch, pseudocount=1e-3, step_size=0.1, graph=False)
    lls, ths, sts = [], [], []
    for x in xs:
        lls.append(float(ts.run(torch.from_numpy(x.astype(np.int32)).cuda()).item()))
        ths.append(ts.plan.theta.double().cpu().numpy())
        sts.append(ts.plan.status[:2].cpu().numpy().copy())
    apply_theta(c, theta0)
    plan = device_plan(c)
    for i, x in enumerate(xs):
        lr, bufs = forward(c, x)
        backward(c, bufs)
        em_update_(c, bufs.f_params, pseudocount=1e-3, step_size=0.1, check=False, plan=plan)
        assert abs(lls[i] - float(lr.double().sum())) <= 1e-5 * abs(lls[i])
        np.testing.assert_array_equal(sts[i], plan.status[:2].cpu().numpy())
        np.testing.assert_allclose(ths[i], plan.theta.double().cpu().numpy(), rtol=1e-5,
                                   atol=1e-12)


def _lean_step_vs_oracle(c, x, pseudocount=1e-4, step=0.2):
    """One one-process TrainStep (lean launches, inline EM where the plan
    allows it, CUDA graph) against the float64 oracle's forward / backward /
    mini-batch EM on the same batch."""
    import torch
    from paper_2406_00766_b200.runtime.em import apply_theta
    from paper_2406_00766_b200.runtime.step import TrainStep
    theta0 = c.theta.copy()
    apply_theta(c, theta0)
    ts = TrainStep(c, x.shape[0], pseudocount=pseudocount, step_size=step, graph=True)
    ll = float(ts.run(torch.from_numpy(x.astype(np.int32)).cuda()).item())
    got = ts.plan.theta.double().cpu().numpy()
    lr, rb = oracle.forward(c, x, theta=theta0)
    oracle.backward(c, rb, theta=theta0)
    new = oracle.em_step_full(c, rb.f_params, theta=theta0, pseudocount=pseudocount)
    want = oracle.em_step_mini(theta0, new, step)
    assert abs(ll - lr.sum()) <= 1e-4 * abs(lr.sum())
    nz = np.abs(want) > 1e-6
    assert np.max(np.abs(got[nz] - want[nz]) / np.abs(want[nz])) < 1e-4
    apply_theta(c, theta0)


@pytest.mark.parametrize("kind", ["pd", "ratspn", "hmm_untied", "hmm_tied", "hclt16"])
def test_lean_train_step_other_structures(kind):
    """The lean / inline-EM training step on every generator family: each
    restructuring (leaf alias, fused push + ratio, side-stream parameter
    flows, inline input EM, fused tile EM) applies only where the plan proves
    it, and the step still matches the oracle elsewhere."""
    from paper_2406_00766_b200 import structures as S
    from paper_2406_00766_b200.compiler import CompileConfig, compile_circuit
    rng = np.random.default_rng(21)
    if kind == "pd":
        g = S.build_pd(S.StructureConfig(kind="pd", shape=(3, 4), hidden_dim=3,
                                         num_categories=5, seed=4))
        c = compile_circuit(g, CompileConfig(block_size=32))
        x = rng.integers(0, 5, size=(150, 12))
    elif kind == "ratspn":
        g = S.build_ratspn(S.StructureConfig(kind="ratspn", num_vars=16, depth=3, hidden_dim=4,
                                             num_categories=8, num_repetitions=6, seed=3))
        c = compile_circuit(g, CompileConfig(block_size=32))
        x = rng.integers(0, 8, size=(200, 16))
    elif kind == "hmm_tied":
        # emission pmfs shared by every position: the shared-pmf input-flow
        # pass builds their histograms in shared memory and applies EM inline
        g = S.build_structure(S.StructureConfig(kind="hmm", seq_len=6, hidden_dim=256,
                                                vocab_size=300, seed=5, tied=True))
        c = compile_circuit(g, CompileConfig(block_size=32))
        from paper_2406_00766_b200.runtime.plan import device_plan
        assert device_plan(c).info["shared_pmf_inline_em"]
        x = rng.integers(0, 300, size=(96, 6))
    elif kind == "hmm_untied":
        g = S.build_structure(S.StructureConfig(kind="hmm", seq_len=6, hidden_dim=64,
                                                vocab_size=30, seed=5, tied=False))
        c = compile_circuit(g, CompileConfig(block_size=32))
        x = rng.integers(0, 30, size=(64, 6))  # unsplit parameter flows: fused tile EM
    else:
        g = S.build_hclt(S.StructureConfig(kind="hclt", num_vars=40, hidden_dim=32,
                                           num_categories=16, seed=6))
        c = compile_circuit(g, CompileConfig(block_size=16))
        x = rng.integers(0, 16, size=(96, 40))
    x[rng.random(x.shape) < 0.1] = -1
    _lean_step_vs_oracle(c, x)
