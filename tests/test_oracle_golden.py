"""Pin the CPU oracle against outputs of the reference package itself."""
import numpy as np
import pytest

import oracle
from _golden import cases, graph_from, load, node_flows, rel_err
from oracle.engine import log_gap
from paper_2406_00766_b200.compiler import CompileConfig, compile_circuit


@pytest.mark.parametrize("name", cases())
def test_oracle_forward_backward_em(name):
    rec = load(name)
    g = graph_from(rec)
    x = rec["x"]
    for k in rec["ks"].tolist():
        c = compile_circuit(g, CompileConfig(block_size=k))
        lroot, bufs = oracle.forward(c, x)
        assert log_gap(lroot, rec[f"k{k}_lroot"], 1e-12, 1e-10) <= 1.0
        oracle.backward(c, bufs)
        nf = node_flows(c, bufs.flows, bufs.prod_flows, g.num_nodes)
        np.testing.assert_allclose(nf, rec[f"k{k}_node_flows"], rtol=1e-9, atol=1e-12)
        np.testing.assert_allclose(bufs.f_params[:c.theta_size], rec[f"k{k}_fparams"],
                                   rtol=1e-9, atol=1e-12)
        ref_em = rec[f"k{k}_em_full"]
        new = oracle.em_step_full(c, bufs.f_params, pseudocount=1e-6)
        if ref_em.size:
            np.testing.assert_allclose(new, ref_em, rtol=1e-10, atol=1e-13)


@pytest.mark.parametrize("name", [n for n in cases() if "train0_theta" in load(n)])
def test_oracle_train_matches_reference(name):
    rec = load(name)
    g = graph_from(rec)
    i = 0
    while f"train{i}_theta" in rec:
        k = int(rec[f"train{i}_k"])
        kw = dict(eval(str(rec[f"train{i}_cfg"])))  # repr of sorted TrainConfig kwargs
        c = compile_circuit(g, CompileConfig(block_size=k))
        theta, lls = oracle.train(c, rec["x"], **kw)
        assert rel_err(theta, rec[f"train{i}_theta"]) < 1e-9
        np.testing.assert_allclose(lls, rec[f"train{i}_ll"], rtol=1e-10)
        i += 1


def test_hmm_alpha_recursion_known_answer():
    """Circuit value == classical forward algorithm (test_acceptance.py:237-254 style)."""
    from paper_2406_00766_b200 import structures as S
    cfg = S.StructureConfig(kind="hmm", seed=60, seq_len=16, hidden_dim=8, vocab_size=10)
    g = S.build_hmm(cfg)
    pi, A, E = S.hmm_parameters(cfg)
    toks = np.random.default_rng(61).integers(0, 10, size=(50, 16))
    toks[np.random.default_rng(62).random(toks.shape) < 0.1] = -1
    c = compile_circuit(g, CompileConfig(block_size=8))
    lroot, _ = oracle.forward(c, toks)
    la = np.log(pi)[None, :] + np.where(toks[:, :1] >= 0, np.log(E[:, np.maximum(toks[:, 0], 0)].T), 0)
    for t in range(1, 16):
        m = la.max(axis=1, keepdims=True)
        la = m + np.log(np.exp(la - m) @ A)
        la = la + np.where(toks[:, t:t + 1] >= 0, np.log(E[:, np.maximum(toks[:, t], 0)].T), 0)
    m = la.max(axis=1)
    want = m + np.log(np.exp(la - m[:, None]).sum(axis=1))
    np.testing.assert_allclose(lroot, want, rtol=1e-10)
