"""Generate golden fixtures by running the REFERENCE package itself.

Run in the build container (where /root/reference exists):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

Each case stores the circuit (as flat arrays), the input batch and the
reference's float64 outputs: compiled-layout digests, root log-likelihoods,
node flows, parameter flows, a full-batch EM step and short training runs.
The GPU parity tests and the oracle pin tests load these files; nothing at
test time reads /root/reference.
"""
from __future__ import annotations

import hashlib
import sys
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg")
sys.path.insert(0, str(REF / "src"))
sys.path.insert(0, str(REF / "tests"))

from circuitgen import random_batch, random_circuit  # noqa: E402  (reference test helper)
from pcirc.compiler import CompileConfig, compile_circuit  # noqa: E402
from pcirc.graph import CircuitGraph, InputNode, ProductNode, SumNode  # noqa: E402
from pcirc.runtime import (EMAccumulator, backward, em_accumulate, em_step_full,  # noqa: E402
                           forward)
from pcirc.structures import StructureConfig, build_hmm  # noqa: E402
from pcirc.train import TrainConfig, train  # noqa: E402

OUT = Path(__file__).resolve().parent


def graph_arrays(g) -> dict:
    kinds, a0, a1, a2, ch_off, ch, sl = [], [], [], [], [0], [], []
    for node in g.nodes:
        if hasattr(node, "var"):
            kinds.append(0)
            a0.append(node.var), a1.append(node.num_categories), a2.append(node.slot)
            ch_off.append(ch_off[-1])
        else:
            kinds.append(2 if hasattr(node, "slots") else 1)
            a0.append(-1), a1.append(-1), a2.append(-1)
            ch.extend(node.children.tolist())
            sl.extend(node.slots.tolist() if hasattr(node, "slots") else [-1] * node.children.size)
            ch_off.append(len(ch))
    tie = np.array(sorted(g.tying.items()), dtype=np.int64).reshape(-1, 2)
    return dict(g_num_vars=np.int64(g.num_vars), g_kind=np.array(kinds, np.int8),
                g_var=np.array(a0, np.int64), g_ncat=np.array(a1, np.int64),
                g_slot=np.array(a2, np.int64), g_ch_off=np.array(ch_off, np.int64),
                g_ch=np.array(ch, np.int64), g_sl=np.array(sl, np.int64),
                g_params=g.params.copy(), g_root=np.int64(g.root), g_tying=tie)


def from_parts_ref(d):
    """Rebuild a reference CircuitGraph from graph_arrays output."""
    nodes = []
    for i, k in enumerate(d["g_kind"].tolist()):
        a, b = d["g_ch_off"][i], d["g_ch_off"][i + 1]
        if k == 0:
            nodes.append(InputNode(i, int(d["g_var"][i]), int(d["g_ncat"][i]), int(d["g_slot"][i])))
        elif k == 1:
            nodes.append(ProductNode(i, d["g_ch"][a:b].copy()))
        else:
            nodes.append(SumNode(i, d["g_ch"][a:b].copy(), d["g_sl"][a:b].copy()))
    tying = {int(s): int(t) for s, t in d["g_tying"].tolist()}
    return CircuitGraph.from_parts(int(d["g_num_vars"]), nodes, d["g_params"],
                                   root=int(d["g_root"]), tying=tying)


sys.path.insert(0, str(OUT.parent))
from _golden import layout_digest  # noqa: E402  (shared with the tests)


def node_flows(c, bufs, g):
    out = np.zeros((g.num_nodes, bufs.values.shape[1]))
    for nid in range(g.num_nodes):
        vs = c.node_value_slot[nid]
        if vs >= 0:
            out[nid] = bufs.flows[vs]
        else:
            out[nid] = bufs.prod_flows[c.node_prod_row[nid]]
    return out


def run_case(name, g, x, ks, *, em_pseudocount=1e-6, train_cfgs=()):
    rec = graph_arrays(g)
    rec["x"] = x
    rec["ks"] = np.array(ks, np.int64)
    for k in ks:
        c = compile_circuit(g, CompileConfig(block_size=k))
        rec[f"k{k}_digest"] = np.array(layout_digest(c))
        rec[f"k{k}_graph_hash"] = np.array(c.graph_hash)
        lroot, bufs = forward(c, x)
        backward(c, bufs)
        rec[f"k{k}_lroot"] = lroot.copy()
        rec[f"k{k}_node_flows"] = node_flows(c, bufs, g)
        rec[f"k{k}_fparams"] = bufs.f_params[:c.theta_size].copy()
        rec[f"k{k}_theta"] = c.theta.copy()
        acc = EMAccumulator.for_circuit(c)
        em_accumulate(acc, bufs)
        try:
            rec[f"k{k}_em_full"] = em_step_full(c, acc, pseudocount=em_pseudocount)
        except Exception:
            rec[f"k{k}_em_full"] = np.zeros(0)
    for i, (k, kw) in enumerate(train_cfgs):
        c = compile_circuit(g, CompileConfig(block_size=k))
        res = train(c, x, TrainConfig(threads=1, **kw))
        rec[f"train{i}_k"] = np.int64(k)
        rec[f"train{i}_cfg"] = np.array(repr(sorted(kw.items())))
        rec[f"train{i}_theta"] = c.theta.copy()
        rec[f"train{i}_ll"] = np.array(res.epoch_log_likelihood)
    np.savez_compressed(OUT / f"{name}.npz", **rec)
    print(name, g.num_nodes, "nodes", x.shape)


def main():
    rng = np.random.default_rng(20240600)
    for i in range(12):
        g = random_circuit(rng, max_vars=7, max_cats=4, max_nodes=150)
        x = random_batch(rng, g, 9, p_missing=0.2)
        run_case(f"random_{i:02d}", g, x, (1, 2, 4, 8),
                 train_cfgs=[(2, dict(epochs=2, batch_size=4, mode="mini", step_size=0.1,
                                      pseudocount=1e-6, seed=3))] if i < 4 else [])
    # HMM (tied) small and wider; untied
    g = build_hmm(StructureConfig(kind="hmm", seed=0, seq_len=8, hidden_dim=16, vocab_size=7,
                                  tied=True))
    x = np.random.default_rng(5).integers(0, 7, size=(40, 8))
    x[np.random.default_rng(6).random(x.shape) < 0.1] = -1
    run_case("hmm_tied", g, x, (4, 8, 16),
             train_cfgs=[(16, dict(epochs=2, batch_size=16, mode="mini", step_size=0.05,
                                    pseudocount=1e-6, seed=1)),
                         (16, dict(epochs=2, batch_size=40, mode="full", pseudocount=1e-6))])
    g = build_hmm(StructureConfig(kind="hmm", seed=2, seq_len=5, hidden_dim=32, vocab_size=11,
                                  tied=False))
    x = np.random.default_rng(7).integers(0, 11, size=(33, 5))
    run_case("hmm_untied", g, x, (32,))
    # HCLT-shaped circuits from the new generator, replayed through the reference
    sys.path.insert(0, str(OUT.parents[1]))
    from paper_2406_00766_b200 import structures as S  # builder's generator
    for name, n, h, ncat, k in [("hclt_small", 12, 16, 5, 16), ("hclt_wide", 10, 32, 9, 32)]:
        mg = S.build_hclt(S.StructureConfig(kind="hclt", num_vars=n, hidden_dim=h,
                                            num_categories=ncat, seed=4))
        rg = from_parts_ref(graph_arrays(mg))
        rg.validate().raise_if_invalid()
        x = np.random.default_rng(8).integers(0, ncat, size=(37, n))
        x[np.random.default_rng(9).random(x.shape) < 0.05] = -1
        run_case(name, rg, x, (k,),
                 train_cfgs=[(k, dict(epochs=1, batch_size=12, mode="mini", step_size=0.1,
                                      pseudocount=1e-6, seed=2))])


if __name__ == "__main__":
    main()
