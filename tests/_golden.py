"""Shared helpers for the golden fixtures (no reference imports here)."""
from __future__ import annotations

import hashlib
from pathlib import Path

import numpy as np

GOLDEN = Path(__file__).resolve().parent / "golden"


def cases() -> list[str]:
    return sorted(p.stem for p in GOLDEN.glob("*.npz"))


def load(name: str) -> dict:
    with np.load(GOLDEN / f"{name}.npz", allow_pickle=False) as z:
        return {k: z[k] for k in z.files}


def graph_from(rec: dict):
    """Rebuild the fixture circuit with this package's CircuitGraph."""
    from paper_2406_00766_b200.graph import CircuitGraph, InputNode, ProductNode, SumNode
    nodes = []
    off = rec["g_ch_off"]
    for i, k in enumerate(rec["g_kind"].tolist()):
        a, b = off[i], off[i + 1]
        if k == 0:
            nodes.append(InputNode(i, int(rec["g_var"][i]), int(rec["g_ncat"][i]),
                                   int(rec["g_slot"][i])))
        elif k == 1:
            nodes.append(ProductNode(i, rec["g_ch"][a:b].copy()))
        else:
            nodes.append(SumNode(i, rec["g_ch"][a:b].copy(), rec["g_sl"][a:b].copy()))
    tying = {int(s): int(t) for s, t in rec["g_tying"].tolist()}
    return CircuitGraph.from_parts(int(rec["g_num_vars"]), nodes, rec["g_params"],
                                   root=int(rec["g_root"]), tying=tying)


def layout_digest(c) -> str:
    """sha256 over every layout array of a compiled circuit, in a fixed order."""
    h = hashlib.sha256()

    def put(a):
        a = np.ascontiguousarray(np.asarray(a, dtype=np.int64))
        h.update(np.array(a.shape, dtype=np.int64).tobytes())
        h.update(a.tobytes())

    for v in (c.reserved, c.num_value_slots, c.scratch_size, c.num_prod_rows, c.theta_size,
              c.f_params_size, c.zero_len, c.root_slot, c.root_row):
        put([v])
    for a in (c.slot_phys, c.reductions, c.tile_starts, c.tile_writers, c.group_idx,
              c.group_off, c.node_value_slot, c.node_prod_row):
        put(a)
    put(c.root_children if c.root_children is not None else [])
    h.update(np.asarray(c.theta, dtype=np.float64).tobytes())
    for ch in c.input_layer:
        for a in (ch.node_ids, ch.slots, ch.vars, ch.param_ids, [ch.num_categories]):
            put(a)
    for L in c.layers:
        put([L.depth, L.k_m, L.k_n, L.scratch_window])
        for ev in L.prod_evals:
            put(ev.out), put(ev.children)
        for g in L.fwd_groups:
            put(g.sum_ids), put(g.prod_ids), put(g.param_ids), put(g.flow_ids)
        for g in L.bwd_groups:
            put(g.ch_ids), put(g.par_ids), put(g.par_param_ids)
        put(L.prod_slots), put(L.prod_rows)
        for p in L.pushes:
            put(p.rows), put(p.children)
        put(L.edge_sums), put(L.edge_children), put(L.edge_slots)
    return h.hexdigest()


def node_values(c, values, g_num_nodes, children_of):
    """Log value per node: slot value, or sum of children for products."""
    out = []
    for nid in range(g_num_nodes):
        vs = c.node_value_slot[nid]
        out.append(values[vs] if vs >= 0 else sum(values[c.node_value_slot[ch]]
                                                  for ch in children_of(nid)))
    return np.stack(out)


def node_flows(c, flows, prod_flows, num_nodes):
    out = np.zeros((num_nodes, flows.shape[1]))
    for nid in range(num_nodes):
        vs = c.node_value_slot[nid]
        out[nid] = flows[vs] if vs >= 0 else prod_flows[c.node_prod_row[nid]]
    return out


def rel_err(got, ref, floor_frac=1e-6):
    """max |got - ref| / max(|ref|, floor), floor relative to max |ref|."""
    got = np.asarray(got, dtype=float)
    ref = np.asarray(ref, dtype=float)
    if ref.size == 0:
        return 0.0
    floor = max(float(np.max(np.abs(ref))) * floor_frac, 1e-30)
    return float(np.max(np.abs(got - ref) / np.maximum(np.abs(ref), floor)))
