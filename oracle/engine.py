"""float64 restatement of the reference forward / backward / EM (oracle).

Each function cites the reference lines it restates.  The arithmetic is the
reference's: per-group streaming log-sum-exp over child blocks with batch
tiles (Alg. 1), per-block max-rescaled flows (Alg. 3 / 4), fancy-add flow
bookkeeping, bincount input flows, segmented EM renormalisation.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

NEG = -np.inf


@dataclass
class OracleBuffers:
    """Workspace like ``pcirc/runtime/buffers.py:18-43`` (float64)."""

    batch: np.ndarray
    values: np.ndarray
    scratch: np.ndarray
    flows: np.ndarray
    flow_scratch: np.ndarray
    prod_flows: np.ndarray
    f_params: np.ndarray
    lroot: np.ndarray = field(default_factory=lambda: np.zeros(0))

    @property
    def batch_size(self) -> int:
        return self.values.shape[1]


def _alloc(c, B):
    return OracleBuffers(
        batch=np.zeros((B, c.num_vars), dtype=np.int64),
        values=np.zeros((c.num_value_slots, B)), scratch=np.zeros((c.scratch_size, B)),
        flows=np.zeros((c.num_value_slots, B)), flow_scratch=np.zeros((c.scratch_size, B)),
        prod_flows=np.zeros((c.num_prod_rows, B)), f_params=np.zeros(c.f_params_size))


def _inputs(c, values, x, theta):
    """engine.py:55-65 — observed: log pmf[x]; missing: 0 (log 1)."""
    for ch in c.input_layer:
        xv = x[:, ch.vars].T                       # (n, B)
        obs = xv >= 0
        idx = ch.param_ids[:, None] + np.where(obs, xv, 0)
        with np.errstate(divide="ignore"):
            lp = np.log(theta[idx])
        values[ch.slots] = np.where(obs, lp, 0.0)


def _products(layer, values, scratch):
    """engine.py:68-71 — window to -inf, then sums of child log values."""
    scratch[:layer.scratch_window] = NEG
    for ev in layer.prod_evals:
        scratch[ev.out] = values[ev.children].sum(axis=1)


def _merge(lin, top, part, m):
    """Two-branch streaming merge with dead-tile skipping (engine.py:89-100)."""
    with np.errstate(invalid="ignore", over="ignore"):
        up = m > top
        merged = np.where(up, lin * np.exp(top - m) + part, lin + part * np.exp(m - top))
    dead = np.isneginf(m)
    return np.where(dead, lin, merged), np.where(dead, top, np.maximum(top, m))


def _sum_forward(gr, km, kn, values, scratch, theta, tile):
    """Alg. 1 (engine.py:74-102)."""
    R, cap = gr.prod_ids.shape
    B = scratch.shape[1]
    rows_out = gr.sum_ids[:, None] + np.arange(km)
    for b0 in range(0, B, tile):
        sc = scratch[:, b0:b0 + tile]
        w = sc.shape[1]
        lin = np.zeros((R, km, w))
        top = np.full((R, 1, w), NEG)
        for c in range(cap):
            child = sc[gr.prod_ids[:, c, None] + np.arange(kn)]          # (R, kn, w)
            m = child.max(axis=1, keepdims=True)
            th = theta[gr.param_ids[:, c, None] + np.arange(km * kn)].reshape(R, km, kn)
            with np.errstate(invalid="ignore", over="ignore"):
                part = th @ np.exp(child - m)
            lin, top = _merge(lin, top, part, m)
        with np.errstate(divide="ignore"):
            values[:, b0:b0 + tile][rows_out] = np.log(lin) + top


def _lnf(f, l):
    with np.errstate(divide="ignore", invalid="ignore"):
        return np.where(np.isneginf(l), NEG, np.log(f) - l)


def _param_flows(gr, km, kn, values, flows, scratch, theta, fp):
    """Alg. 3 (engine.py:105-126)."""
    R, cap = gr.prod_ids.shape
    rows = gr.sum_ids[:, None] + np.arange(km)
    lnf = _lnf(flows[rows], values[rows])                              # (R, km, B)
    nmax = lnf.max(axis=1, keepdims=True)
    with np.errstate(invalid="ignore"):
        scaled = np.where(np.isneginf(nmax), 0.0, np.exp(lnf - nmax))
    for c in range(cap):
        child = scratch[gr.prod_ids[:, c, None] + np.arange(kn)]       # (R, kn, B)
        with np.errstate(over="ignore"):
            em = np.exp(child + nmax)
        cum = scaled @ em.transpose(0, 2, 1)                           # (R, km, kn)
        th = theta[gr.param_ids[:, c, None] + np.arange(km * kn)].reshape(R, km, kn)
        fp[(gr.flow_ids[:, c, None] + np.arange(km * kn)).ravel()] += (th * cum).ravel()


def _child_flows(gr, km, kn, values, flows, scratch, flow_scratch, theta, tile):
    """Alg. 4 (engine.py:129-165)."""
    R, cap = gr.par_ids.shape
    B = values.shape[1]
    crow = gr.ch_ids[:, None] + np.arange(kn)
    for b0 in range(0, B, tile):
        val = values[:, b0:b0 + tile]
        flo = flows[:, b0:b0 + tile]
        w = val.shape[1]
        lin = np.zeros((R, kn, w))
        top = np.full((R, 1, w), NEG)
        for p in range(cap):
            prow = gr.par_ids[:, p, None] + np.arange(km)
            lnf = _lnf(flo[prow], val[prow])
            with np.errstate(invalid="ignore", over="ignore"):
                m = lnf.max(axis=1, keepdims=True)
                s = np.where(np.isneginf(m), 0.0, np.exp(lnf - m))
                th = theta[gr.par_param_ids[:, p, None] + np.arange(km * kn)]
                part = th.reshape(R, km, kn).transpose(0, 2, 1) @ s
            lin, top = _merge(lin, top, part, m)
        sc = scratch[:, b0:b0 + tile]
        with np.errstate(over="ignore"):
            flow_scratch[:, b0:b0 + tile][crow] = lin * np.exp(top + sc[crow])


def _input_flows(c, flows, x, theta, fp):
    """engine.py:168-183."""
    for ch in c.input_layer:
        fl = flows[ch.slots]
        xv = x[:, ch.vars].T
        obs = xv >= 0
        hit = ch.param_ids[:, None] + np.where(obs, xv, 0)
        fp += np.bincount(hit.ravel(), weights=np.where(obs, fl, 0.0).ravel(),
                          minlength=fp.size)
        miss = np.where(obs, 0.0, fl).sum(axis=1)
        if np.any(miss):
            rng = ch.param_ids[:, None] + np.arange(ch.num_categories)
            fp += np.bincount(rng.ravel(), weights=(miss[:, None] * theta[rng]).ravel(),
                              minlength=fp.size)


def forward(c, x, *, theta=None, batch_tile=64, bufs=None):
    """engine.py:186-217 (validation omitted: the oracle trusts its inputs)."""
    x = np.atleast_2d(np.asarray(x, dtype=np.int64))
    theta = c.theta if theta is None else theta
    B = x.shape[0]
    if bufs is None or bufs.batch_size != B:
        bufs = _alloc(c, B)
    bufs.batch = x
    tile = max(1, min(batch_tile, B)) if B else 1
    v = bufs.values
    v.fill(NEG)
    _inputs(c, v, x, theta)
    for L in c.layers:
        _products(L, v, bufs.scratch)
        for gr in L.fwd_groups:
            _sum_forward(gr, L.k_m, L.k_n, v, bufs.scratch, theta, tile)
    bufs.lroot = v[c.root_slot].copy() if c.root_slot >= 0 else v[c.root_children].sum(axis=0)
    return bufs.lroot, bufs


def backward(c, bufs, *, theta=None, batch_tile=64):
    """engine.py:220-259."""
    theta = c.theta if theta is None else theta
    v, f = bufs.values, bufs.flows
    f.fill(0.0)
    bufs.prod_flows.fill(0.0)
    bufs.f_params.fill(0.0)
    tile = max(1, min(batch_tile, v.shape[1])) if v.shape[1] else 1
    if c.root_slot >= 0:
        f[c.root_slot] = 1.0
    else:
        bufs.prod_flows[c.root_row] = 1.0
        np.add.at(f, c.root_children, 1.0)
    for L in reversed(c.layers):
        _products(L, v, bufs.scratch)
        for gr in L.fwd_groups:
            _param_flows(gr, L.k_m, L.k_n, v, f, bufs.scratch, theta, bufs.f_params)
        for gr in L.bwd_groups:
            _child_flows(gr, L.k_m, L.k_n, v, f, bufs.scratch, bufs.flow_scratch, theta, tile)
        if L.prod_rows.size:
            bufs.prod_flows[L.prod_rows] += bufs.flow_scratch[L.prod_slots]
        for p in L.pushes:
            rows = bufs.prod_flows[p.rows]
            for k in range(p.children.shape[1]):
                np.add.at(f, p.children[:, k], rows)
    _input_flows(c, f, bufs.batch, theta, bufs.f_params)
    for src, dst, n in np.asarray(c.reductions).tolist():
        bufs.f_params[dst:dst + n] += bufs.f_params[src:src + n]
    return bufs


def em_accumulate(acc_fp, bufs):
    """em.py:48-55: returns (f_params sum, ll sum)."""
    return acc_fp + bufs.f_params, float(bufs.lroot.sum())


def em_step_full(c, f_params, *, theta=None, pseudocount=0.0):
    """em.py:58-81 (NumericError semantics reported by returning None)."""
    theta = c.theta if theta is None else theta
    counts = f_params[:c.theta_size][c.group_idx] + pseudocount
    off = c.group_off
    if off.size <= 1:
        return theta.copy()
    totals = np.add.reduceat(counts, off[:-1])
    good = totals > 0.0
    if not good.any():
        return None
    sizes = np.diff(off)
    keep = np.repeat(good, sizes)
    out = theta.copy()
    out[c.group_idx[keep]] = counts[keep] / np.repeat(totals, sizes)[keep]
    return out


def em_step_mini(theta, theta_new, step):
    """em.py:84-88."""
    return (1.0 - step) * theta + step * theta_new


def train(c, data, *, epochs=1, batch_size=256, mode="full", step_size=0.01,
          pseudocount=0.0, seed=0, theta=None):
    """train.py:104-154 (single worker); returns (theta, per-epoch mean LL)."""
    data = np.asarray(data, dtype=np.int64)
    n = data.shape[0]
    theta = (c.theta if theta is None else theta).copy()
    bs = min(batch_size, n)
    rng = np.random.default_rng(np.random.SeedSequence(seed).spawn(2)[1])
    lls = []
    for _ in range(epochs):
        order = rng.permutation(n) if mode == "mini" else np.arange(n)
        ep_fp = np.zeros(c.f_params_size)
        ep_ll, ep_n = 0.0, 0
        for a in range(0, n, bs):
            xb = data[order[a:a + bs]]
            lr, bufs = forward(c, xb, theta=theta)
            backward(c, bufs, theta=theta)
            ep_ll += float(lr.sum())
            ep_n += xb.shape[0]
            if mode == "full":
                ep_fp += bufs.f_params
            else:
                new = em_step_full(c, bufs.f_params, theta=theta, pseudocount=pseudocount)
                if new is None:
                    raise FloatingPointError("dead EM step")
                theta = em_step_mini(theta, new, step_size)
        if mode == "full":
            new = em_step_full(c, ep_fp, theta=theta, pseudocount=pseudocount)
            if new is None:
                raise FloatingPointError("dead EM step")
            theta = new
        lls.append(ep_ll / ep_n)
    return theta, lls


def log_gap(got, ref, atol, rtol):
    """Worst |got-ref| / (atol + rtol|ref|); -inf patterns must agree
    (``tests/test_acceptance.py:60-68``)."""
    got, ref = np.asarray(got, dtype=float), np.asarray(ref, dtype=float)
    if not np.array_equal(np.isneginf(got), np.isneginf(ref)):
        return math.inf
    m = ~np.isneginf(ref)
    if not m.any():
        return 0.0
    return float(np.max(np.abs(got[m] - ref[m]) / (atol + rtol * np.abs(ref[m]))))
