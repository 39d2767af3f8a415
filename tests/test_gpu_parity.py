"""GPU parity: the sm_100a path against the reference's own outputs.

Tolerances (BASELINE north star): per-sample log-likelihoods, parameter
flows and updated parameters within 1e-4 relative in fp32 accumulation.
Log-likelihoods use the reference's ``log_gap`` (-inf patterns must agree);
flows use a relative error with a floor of 1e-6 x the tensor's max.
"""
import numpy as np
import pytest

from _golden import cases, graph_from, load, node_flows, rel_err
from oracle.engine import log_gap

pytestmark = pytest.mark.gpu

RTOL = 1e-4


def _np(t):
    return t.detach().double().cpu().numpy()


@pytest.fixture(scope="module")
def lib():
    from paper_2406_00766_b200.runtime import _lib
    return _lib.load()


@pytest.mark.parametrize("n,k", [(16, 16), (32, 64), (48, 32), (128, 128), (256, 256)])
def test_tcgen05_descriptor_selftest(lib, n, k):
    import torch
    from paper_2406_00766_b200.runtime import _lib
    g = torch.Generator(device="cpu").manual_seed(n * 1000 + k)
    a = torch.randn(128, k, generator=g).to(torch.bfloat16).cuda()
    b = torch.randn(n, k, generator=g).to(torch.bfloat16).cuda()
    d = torch.zeros(128, n, dtype=torch.float32, device="cuda")
    _lib.call("pcb_tc_selftest", _lib.stream_handle(), n, k, a.data_ptr(), b.data_ptr(),
              d.data_ptr())
    torch.cuda.synchronize()
    want = a.float() @ b.float().T
    torch.testing.assert_close(d, want, rtol=1e-5, atol=1e-4)


@pytest.mark.parametrize("n,k", [(16, 16), (32, 32), (64, 64), (32, 16)])
def test_tcgen05_mn_major_b_selftest(lib, n, k):
    """The child-flow kernel reads theta tiles through an MN-major B descriptor
    with LBO = K-adjacent core stride, SBO = MN-adjacent (variant 0; the
    swapped roles read outside the tile and fault).  Pin that encoding."""
    import torch
    from paper_2406_00766_b200.runtime import _lib
    g = torch.Generator(device="cpu").manual_seed(7 * n + k)
    a = torch.randn(128, k, generator=g).to(torch.bfloat16).cuda()
    bkn = torch.randn(k, n, generator=g).to(torch.bfloat16).cuda()
    want = a.float() @ bkn.float()
    d = torch.zeros(128, n, dtype=torch.float32, device="cuda")
    _lib.call("pcb_tc_selftest_mn", _lib.stream_handle(), n, k, 0, a.data_ptr(),
              bkn.data_ptr(), d.data_ptr())
    torch.cuda.synchronize()
    torch.testing.assert_close(d, want, rtol=1e-5, atol=1e-4)


@pytest.mark.parametrize("tensor_cores", [True, False])
@pytest.mark.parametrize("name", cases())
def test_forward_backward_em_parity(name, tensor_cores):
    from paper_2406_00766_b200.compiler import CompileConfig, compile_circuit
    from paper_2406_00766_b200.runtime import (EMAccumulator, backward, em_accumulate,
                                               em_step_full, forward)
    rec = load(name)
    g = graph_from(rec)
    x = rec["x"]
    for k in rec["ks"].tolist():
        c = compile_circuit(g, CompileConfig(block_size=k))
        lroot, bufs = forward(c, x, tensor_cores=tensor_cores)
        got = _np(lroot)
        assert log_gap(got, rec[f"k{k}_lroot"], 1e-5, RTOL) <= 1.0, (name, k)
        backward(c, bufs, tensor_cores=tensor_cores)
        nf = node_flows(c, _np(bufs.flows), _np(bufs.prod_flows), g.num_nodes)
        assert rel_err(nf, rec[f"k{k}_node_flows"]) < RTOL, (name, k)
        fp = _np(bufs.f_params)[:c.theta_size]
        assert rel_err(fp, rec[f"k{k}_fparams"]) < RTOL, (name, k)
        ref_em = rec[f"k{k}_em_full"]
        if ref_em.size:
            acc = EMAccumulator.for_circuit(c)
            em_accumulate(acc, bufs)
            new = _np(em_step_full(c, acc, pseudocount=1e-6))
            assert rel_err(new, ref_em) < RTOL, (name, k)


@pytest.mark.parametrize("name", [n for n in cases() if "train0_theta" in load(n)])
def test_train_parity(name):
    from paper_2406_00766_b200.compiler import CompileConfig, compile_circuit
    from paper_2406_00766_b200.train import TrainConfig, train
    rec = load(name)
    g = graph_from(rec)
    i = 0
    while f"train{i}_theta" in rec:
        k = int(rec[f"train{i}_k"])
        kw = dict(eval(str(rec[f"train{i}_cfg"])))
        c = compile_circuit(g, CompileConfig(block_size=k))
        res = train(c, rec["x"], TrainConfig(**kw))
        assert rel_err(c.theta, rec[f"train{i}_theta"]) < RTOL, (name, i)
        np.testing.assert_allclose(res.epoch_log_likelihood, rec[f"train{i}_ll"], rtol=RTOL)
        i += 1
