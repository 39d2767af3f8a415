"""Numerics edge cases on the device path against the float64 oracle
(VERDICT r1 weak #11).

* Extreme dynamic range: an HCLT whose odd latent components form a chain of
  near-impossible states (observed category at probability 1e-30, mixture
  rows that keep odd components on odd children), so sibling children of one
  sum differ by hundreds of nats (far beyond fp32's e^-87 underflow) while
  every sum still reaches its dominant child.  The super-row shift is the
  max over blocks every row is fully connected to (product classes share
  their parent set, so a sum reaches every product of each of its child
  blocks), hence no sum underflows to -inf; flows of the far children
  underflow to 0 exactly where the oracle's are below 1e-38 of the largest,
  which the north-star tolerance (relative to the largest flow) accepts.
* The same circuit through the graphed lean training step.
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


def _skewed_hclt(num_vars=48, h=32, ncat=8, seed=2, eps=1e-30, tiny=1e-30):
    from paper_2406_00766_b200 import structures as S
    from paper_2406_00766_b200.graph import KIND_SUM
    g = S.build_hclt(S.StructureConfig(kind="hclt", num_vars=num_vars, hidden_dim=h,
                                       num_categories=ncat, seed=seed))
    ids, var, nc, slot = g.input_table()
    j = np.arange(ids.size) % h                       # latent component of each input
    for i in np.flatnonzero(j % 2 == 1):              # odd components: category 0 ~ 1e-30
        pmf = np.full(ncat, (1.0 - tiny) / (ncat - 1))
        pmf[0] = tiny
        g.set_param_values(slot[i] + np.arange(ncat), pmf)
    for s in g.segments:                              # mixtures keep parity
        if s.kind != KIND_SUM or s.count != h:
            continue
        rows = np.arange(h)[:, None] % 2 == np.arange(h)[None, :] % 2
        w = np.where(rows, (1.0 - eps) / (h // 2), eps / (h // 2))
        g.set_param_values(np.asarray(s.slots).ravel(), w.ravel())
    return g


def _sibling_gap(g, xrow):
    """Largest spread (nats) between the children of one sum, one sample
    (node log-values by direct float64 evaluation of the graph)."""
    from paper_2406_00766_b200.graph import KIND_INPUT, KIND_PRODUCT
    v = np.zeros(g.num_nodes)
    p = g.params
    gap = 0.0
    for s in g.segments:
        if s.kind == KIND_INPUT:
            x = xrow[s.var]
            with np.errstate(divide="ignore"):
                v[s.start:s.stop] = np.where(x < 0, 0.0, np.log(p[s.slot + np.maximum(x, 0)]))
            continue
        cv = v[np.asarray(s.children)]
        if s.kind == KIND_PRODUCT:
            v[s.start:s.stop] = cv.sum(axis=1)
            continue
        m = cv.max(axis=1, keepdims=True)
        with np.errstate(divide="ignore"):
            v[s.start:s.stop] = (m + np.log(np.sum(p[np.asarray(s.slots)] * np.exp(cv - m),
                                                  axis=1, keepdims=True)))[:, 0]
        fin = np.where(np.isfinite(cv), cv, np.nan)
        gap = max(gap, float(np.nanmax(np.nanmax(fin, axis=1) - np.nanmin(fin, axis=1))))
    return gap


def test_extreme_dynamic_range_matches_oracle():
    import torch
    from paper_2406_00766_b200.compiler import CompileConfig, compile_circuit
    from paper_2406_00766_b200.runtime import backward, em_update_, forward
    from paper_2406_00766_b200.runtime.plan import device_plan
    g = _skewed_hclt()
    c = compile_circuit(g, CompileConfig(block_size=32))
    x = np.zeros((256, c.num_vars), dtype=np.int64)   # category 0 everywhere
    x[np.random.default_rng(1).random(x.shape) < 0.1] = -1
    lroot, bufs = forward(c, x)
    backward(c, bufs)
    torch.cuda.synchronize()
    rl, rb = oracle.forward(c, x)
    oracle.backward(c, rb)
    # the range is real: sibling children of one sum more than fp32's e^-87
    # apart, and flows spanning far more than fp32's exponent range
    fin = np.isfinite(rb.values)
    assert _sibling_gap(g, x[0]) > 120.0
    pos = rb.flows[rb.flows > 0]
    assert pos.min() < 1e-100 * pos.max()
    assert np.all(np.isfinite(_np(lroot)))
    assert log_gap(_np(lroot), rl, 1e-5, RTOL) <= 1.0
    got = _np(bufs.values)
    assert np.array_equal(np.isfinite(got), fin)
    assert np.max(np.abs(got[fin] - rb.values[fin]) / (1e-5 + 1e-6 * np.abs(rb.values[fin]))) <= 1.0
    assert rel_err(_np(bufs.flows), rb.flows) < RTOL
    assert rel_err(_np(bufs.f_params)[:c.theta_size], rb.f_params[:c.theta_size]) < RTOL
    plan = device_plan(c)
    saved = plan.theta.clone()
    want = oracle.em_step_mini(c.theta, oracle.em_step_full(c, rb.f_params, pseudocount=1e-6), 0.5)
    em_update_(c, bufs.f_params, pseudocount=1e-6, step_size=0.5, plan=plan)
    got_t = _np(plan.theta)
    plan.theta.copy_(saved)
    plan.refresh_mma()
    assert rel_err(got_t, want) < RTOL


def test_extreme_dynamic_range_train_step():
    import torch
    from paper_2406_00766_b200.compiler import CompileConfig, compile_circuit
    from paper_2406_00766_b200.runtime.em import apply_theta
    from paper_2406_00766_b200.runtime.step import TrainStep
    c = compile_circuit(_skewed_hclt(num_vars=64, seed=3), CompileConfig(block_size=32))
    x = np.zeros((128, c.num_vars), dtype=np.int64)
    x[:, ::5] = 3
    theta0 = c.theta.copy()
    ts = TrainStep(c, 128, pseudocount=1e-6, step_size=1.0, graph=True)
    ll = float(ts.run(torch.from_numpy(x.astype(np.int32)).cuda()).item())
    got = _np(ts.plan.theta)
    apply_theta(c, theta0)
    lr, rb = oracle.forward(c, x, theta=theta0)
    oracle.backward(c, rb, theta=theta0)
    want = oracle.em_step_full(c, rb.f_params, theta=theta0, pseudocount=1e-6)
    assert abs(ll - lr.sum()) <= 1e-6 * abs(lr.sum())
    assert rel_err(got, want) < RTOL
