"""The drop-in API on the GPU: train() (graphed pcb_train_step path) against
the float64 oracle, its error semantics, the reference's exception classes
through the C ABI, the per-layer operator API and the f_params contract."""
import ctypes as C

import numpy as np
import pytest

import oracle
from _golden import cases, graph_from, load, rel_err
from oracle.engine import log_gap

pytestmark = pytest.mark.gpu
RTOL = 1e-4


def _np(t):
    return t.detach().double().cpu().numpy()


def _hclt(nv=24, h=32, ncat=8, seed=2, k=32):
    from paper_2406_00766_b200 import structures as S
    from paper_2406_00766_b200.compiler import CompileConfig, compile_circuit
    g = S.build_hclt(S.StructureConfig(kind="hclt", num_vars=nv, hidden_dim=h,
                                       num_categories=ncat, seed=seed))
    return g, compile_circuit(g, CompileConfig(block_size=k))


@pytest.mark.parametrize("mode", ["mini", "full"])
@pytest.mark.parametrize("graph", [True, False])
def test_train_matches_oracle(mode, graph):
    """train() over 2 epochs of 300 samples at batch 128 (two full batches and
    a 44-sample tail, each batch size with its own graphed step) equals the
    oracle's train (same shuffle, same EM schedule)."""
    from paper_2406_00766_b200.train import TrainConfig, train
    g, c = _hclt()
    theta0 = c.theta.copy()
    x = np.random.default_rng(5).integers(0, 8, size=(300, 24))
    x[np.random.default_rng(6).random(x.shape) < 0.05] = -1
    cfg = dict(epochs=2, batch_size=128, mode=mode, step_size=0.05, pseudocount=1e-3, seed=3)
    res = train(c, x, TrainConfig(**cfg), graph=graph)
    want_theta, want_ll = oracle.train(c, x, theta=theta0, **{k: v for k, v in cfg.items()})
    np.testing.assert_allclose(res.epoch_log_likelihood, want_ll, rtol=RTOL)
    assert rel_err(c.theta, want_theta) < RTOL
    assert len(res.epoch_seconds) == 2


@pytest.mark.parametrize("name", [n for n in cases() if "train0_theta" in load(n)][:1])
def test_train_without_tensor_cores_updates_every_plan(name):
    """train(tensor_cores=False) writes the trained table back (host and the
    tensor-core plan), and a later forward with tensor cores evaluates it."""
    from paper_2406_00766_b200.compiler import CompileConfig, compile_circuit
    from paper_2406_00766_b200.runtime import forward
    from paper_2406_00766_b200.train import TrainConfig, train
    rec = load(name)
    g = graph_from(rec)
    k = int(rec["train0_k"])
    kw = dict(eval(str(rec["train0_cfg"])))
    c = compile_circuit(g, CompileConfig(block_size=k))
    forward(c, rec["x"], tensor_cores=True)  # a tensor-core plan exists before training
    train(c, rec["x"], TrainConfig(**kw), tensor_cores=False)
    assert rel_err(c.theta, rec["train0_theta"]) < RTOL
    lr, _ = forward(c, rec["x"], tensor_cores=True)
    ref, _ = oracle.forward(c, rec["x"], theta=rec["train0_theta"])
    assert log_gap(_np(lr), ref, 1e-5, RTOL) <= 1.0


def _impossible():
    from paper_2406_00766_b200.compiler import compile_circuit
    from paper_2406_00766_b200.graph import CircuitGraph
    g = CircuitGraph(1)
    a = g.add_input(0, [1.0, 0.0])
    b = g.add_input(0, [1.0, 0.0])
    g.add_sum([a, b], [0.5, 0.5])
    return compile_circuit(g)


def test_numeric_errors():
    """NumericError where the reference raises it: EM with every group dead
    (em.py:70-75, test_em.py:79-88), training on impossible data (at the
    first step, parameters untouched), non-finite parameters (engine.py:197-198)."""
    from paper_2406_00766_b200.errors import NumericError
    from paper_2406_00766_b200.runtime import (EMAccumulator, apply_theta, backward,
                                               em_accumulate, em_step_full, forward)
    from paper_2406_00766_b200.train import TrainConfig, train
    c = _impossible()
    lr, bufs = forward(c, np.array([[1]]))
    assert _np(lr)[0] == -np.inf
    backward(c, bufs)
    assert float(bufs.f_params.abs().sum()) == 0.0
    acc = EMAccumulator.for_circuit(c)
    em_accumulate(acc, bufs)
    with pytest.raises(NumericError):
        em_step_full(c, acc, pseudocount=0.0)
    theta0 = c.theta.copy()
    with pytest.raises(NumericError):
        train(c, np.array([[1], [1], [1]]), TrainConfig(mode="mini", batch_size=2))
    np.testing.assert_array_equal(c.theta, theta0)
    with pytest.raises(NumericError):
        train(c, np.array([[1], [1]]), TrainConfig(mode="full", batch_size=1))
    bad = c.theta.copy()
    bad[-1] = np.nan
    apply_theta(c, bad)
    with pytest.raises(NumericError):
        forward(c, np.array([[0]]))
    with pytest.raises(NumericError):
        train(c, np.array([[0]]), TrainConfig())
    apply_theta(c, theta0)


def test_format_and_usage_errors():
    """FormatError for bad batches (engine.py:41-51), UsageError for order /
    argument errors (engine.py:228, em.py:65-66, 86-87) and for C-ABI misuse."""
    import torch
    from paper_2406_00766_b200.errors import FormatError, UsageError
    from paper_2406_00766_b200.runtime import (EMAccumulator, _lib, allocate_buffers,
                                               backward, em_step_full, em_step_mini, forward)
    from paper_2406_00766_b200.runtime.plan import device_plan
    from paper_2406_00766_b200.train import TrainConfig, train
    g, c = _hclt(nv=6, h=16, ncat=4, k=16)
    for bad in (np.zeros((3, 5), dtype=np.int64), np.full((2, 6), 4), np.full((2, 6), -2)):
        with pytest.raises(FormatError):
            forward(c, bad)
        with pytest.raises(FormatError):
            train(c, bad, TrainConfig())
    with pytest.raises(FormatError):  # device batch checked on the device
        forward(c, torch.full((2, 6), 7, dtype=torch.int32, device="cuda"))
    bufs = allocate_buffers(c, 4)
    with pytest.raises(UsageError):
        backward(c, bufs)
    acc = EMAccumulator.for_circuit(c)
    with pytest.raises(UsageError):
        em_step_full(c, acc, pseudocount=-1.0)
    with pytest.raises(UsageError):
        em_step_mini(c.theta, c.theta, 0.0)
    with pytest.raises(UsageError):
        TrainConfig(mode="batch")
    with pytest.raises(UsageError):
        train(c, np.zeros((0, 6), dtype=np.int64), TrainConfig())
    plan = device_plan(c)
    _, b = forward(c, np.zeros((4, 6), dtype=np.int64))
    other = plan.theta.clone()  # tensor-core passes read the bound table's planes
    with pytest.raises(UsageError):
        _lib.call("pcb_forward", plan.handle, _lib.stream_handle(), 4, b.ldb, b.xT.data_ptr(),
                  other.data_ptr(), b.values_full.data_ptr(), b.scratch_full.data_ptr(),
                  b.lroot.data_ptr(), b.work.data_ptr())
    args = (plan.handle, None, _lib.stream_handle(), 4, b.ldb, b.xT.data_ptr(),
            plan.theta.data_ptr(), b.values_full.data_ptr(), b.flows_full.data_ptr(),
            b.scratch_full.data_ptr(), b.flow_scratch_full.data_ptr(),
            b.prod_flows_full.data_ptr(), b.f_params.data_ptr(), b.lroot.data_ptr(),
            b.work.data_ptr())
    with pytest.raises(UsageError):  # unknown flag
        _lib.call("pcb_train_step", *args, 64, 0.0, 1.0, plan.status.data_ptr())
    with pytest.raises(UsageError):  # EM step size outside (0, 1]
        _lib.call("pcb_train_step", *args, _lib.STEP_EM, 0.0, 1.5, plan.status.data_ptr())
    with pytest.raises(UsageError):  # ldb not a multiple of 32
        _lib.call("pcb_forward", plan.handle, _lib.stream_handle(), 4, 33, b.xT.data_ptr(),
                  plan.theta.data_ptr(), b.values_full.data_ptr(), b.scratch_full.data_ptr(),
                  b.lroot.data_ptr(), b.work.data_ptr())
    with pytest.raises(UsageError):
        _lib.call("pcb_layer_forward", plan.handle, len(c.layers), _lib.stream_handle(), 4,
                  b.ldb, plan.theta.data_ptr(), b.values_full.data_ptr(),
                  b.scratch_full.data_ptr(), b.work.data_ptr())


@pytest.mark.parametrize("tensor_cores", [True, False])
def test_per_layer_operator_api(tensor_cores):
    """pcb_layer_forward recomputes each layer's products and sums exactly as
    the whole-pass forward did; pcb_layer_backward of the top layer reproduces
    its parameter flows (the reference's private kernels imported by
    pcirc/bench.py:22-27)."""
    import torch
    from paper_2406_00766_b200.runtime import backward, forward
    from paper_2406_00766_b200.runtime.engine import layer_backward, layer_forward
    g, c = _hclt(nv=20, h=64, ncat=8, k=32)
    x = np.random.default_rng(1).integers(0, 8, size=(130, 20))
    lr, b = forward(c, x, tensor_cores=tensor_cores)
    v0, s0, w0 = b.values_full.clone(), b.scratch_full.clone(), b.work.clone()
    for li in range(len(c.layers)):
        layer_forward(c, li, b, tensor_cores=tensor_cores)
    torch.cuda.synchronize()
    assert torch.equal(b.values_full, v0) and torch.equal(b.scratch_full, s0)
    assert torch.equal(b.work, w0)
    backward(c, b, tensor_cores=tensor_cores)
    fp0 = b.f_params.clone()
    top = len(c.layers) - 1
    b.f_params.zero_()
    layer_backward(c, top, b, tensor_cores=tensor_cores)
    torch.cuda.synchronize()
    rng = np.unique(np.concatenate([gr.flow_ids[gr.param_ids != 0]
                                    for gr in c.layers[top].fwd_groups]))
    tile = c.layers[top].k_m * c.layers[top].k_n
    idx = (rng[:, None] + np.arange(tile)).ravel()
    got, want = _np(b.f_params)[idx], _np(fp0)[idx]
    assert rel_err(got, want) < 1e-6


def test_f_params_contract():
    """f_params[:theta_size] are the reference's reduced parameter flows; the
    replica ranges past theta_size (the reference's private per-layer partial
    sums, engine.py:256-257) are folded onto their master tiles on the GPU and
    read as zero (nothing downstream reads them: em.py uses the theta prefix)."""
    from paper_2406_00766_b200 import structures as S
    from paper_2406_00766_b200.compiler import CompileConfig, compile_circuit
    from paper_2406_00766_b200.runtime import backward, forward
    g = S.build_hmm(S.StructureConfig(kind="hmm", seq_len=6, hidden_dim=64, vocab_size=12,
                                      seed=1, tied=True))
    c = compile_circuit(g, CompileConfig(block_size=32))
    assert c.f_params_size > c.theta_size
    x = np.random.default_rng(2).integers(0, 12, size=(40, 6))
    _, b = forward(c, x)
    backward(c, b)
    rl, rb = oracle.forward(c, x)
    oracle.backward(c, rb)
    fp = _np(b.f_params)
    assert rel_err(fp[:c.theta_size], rb.f_params[:c.theta_size]) < RTOL
    assert not fp[c.theta_size:].any()


def test_train_step_validate():
    """TrainStep.run(validate=True) raises FormatError on a bad batch before
    any kernel reads it (ADVICE: out-of-range categories would index the
    staged pmf tables out of bounds)."""
    import torch
    from paper_2406_00766_b200.errors import FormatError
    from paper_2406_00766_b200.runtime.step import TrainStep
    g, c = _hclt(nv=6, h=16, ncat=4, k=16)
    ts = TrainStep(c, 8, pseudocount=1e-3, step_size=0.1, graph=True)
    good = torch.zeros((8, 6), dtype=torch.int32, device="cuda")
    ts.run(good, validate=True)
    for bad in (torch.full((8, 6), 4, dtype=torch.int32, device="cuda"),
                torch.zeros((8, 5), dtype=torch.int32, device="cuda"),
                torch.zeros((8, 6), dtype=torch.int64, device="cuda")):
        with pytest.raises(FormatError):
            ts.run(bad, validate=True)
