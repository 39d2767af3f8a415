"""nll / bpd / perplexity summaries (``pcirc/runtime/metrics.py:14-42``) and
the ``metric=<name> value=<v>`` line, on the reference's known answers
(``pkg/tests/test_metrics.py``) and on device log-likelihood tensors."""
import math

import numpy as np
import pytest

from paper_2406_00766_b200.errors import UsageError
from paper_2406_00766_b200.runtime.metrics import log_likelihood_metrics, metric_line


def test_known_answers():
    np.testing.assert_allclose(log_likelihood_metrics([-1.0, -3.0])["nll"], 2.0, rtol=1e-15)
    ll = math.log(1.0 / 256.0)  # a uniform byte is eight bits
    np.testing.assert_allclose(log_likelihood_metrics([ll] * 3, num_dims=1)["bpd"], 8.0,
                               rtol=1e-12)
    np.testing.assert_allclose(log_likelihood_metrics([4 * math.log(0.5)], num_dims=4)["bpd"],
                               1.0, rtol=1e-12)
    out = log_likelihood_metrics([10 * math.log(0.5)] * 2, num_tokens=10)
    np.testing.assert_allclose(out["perplexity"], 2.0, rtol=1e-12)
    assert set(log_likelihood_metrics([-1.0])) == {"nll"}


@pytest.mark.parametrize("bad", [dict(ll=[]), dict(ll=[-1.0, -np.inf]),
                                 dict(ll=[-1.0], num_dims=0), dict(ll=[-1.0], num_tokens=-3)])
def test_rejections(bad):
    ll = bad.pop("ll")
    with pytest.raises(UsageError):
        log_likelihood_metrics(ll, **bad)


def test_metric_line():
    assert metric_line("nll", 2.5) == "metric=nll value=2.5"
    v = 0.1 + 0.2
    assert float(metric_line("bpd", v).split("value=")[1]) == v


def test_torch_tensor_input():
    import torch
    ll = torch.tensor([-2.0, -4.0], dtype=torch.float32)
    out = log_likelihood_metrics(ll, num_dims=3, num_tokens=3)
    np.testing.assert_allclose(out["nll"], 3.0)
    np.testing.assert_allclose(out["bpd"], 3.0 / (3 * math.log(2.0)))
    np.testing.assert_allclose(out["perplexity"], math.e)


@pytest.mark.gpu
def test_perplexity_of_device_hmm_forward():
    """Perplexity of a GPU HMM forward equals the oracle's at 1e-4."""
    import oracle
    from paper_2406_00766_b200 import structures as S
    from paper_2406_00766_b200.compiler import CompileConfig, compile_circuit
    from paper_2406_00766_b200.runtime import forward
    g = S.build_hmm(S.StructureConfig(kind="hmm", seq_len=8, hidden_dim=64, vocab_size=50,
                                      seed=3, tied=True))
    c = compile_circuit(g, CompileConfig(block_size=32))
    x = np.random.default_rng(0).integers(0, 50, size=(100, 8))
    lr, _ = forward(c, x)
    ref, _ = oracle.forward(c, x)
    got = log_likelihood_metrics(lr, num_tokens=8)["perplexity"]
    want = log_likelihood_metrics(ref, num_tokens=8)["perplexity"]
    np.testing.assert_allclose(got, want, rtol=1e-4)
