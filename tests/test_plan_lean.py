"""Host-side invariants of the lean-step plan tables (CPU): the leaf alias,
the fused push + ratio blocks, the EM block order for fused EM and the
inline input-EM group order, on every generator family.  The GPU tests
(test_gpu_graph.py) check the numbers; these check the tables the kernels
trust without re-validating."""
import numpy as np
import pytest

from paper_2406_00766_b200 import structures as S
from paper_2406_00766_b200.compiler import CompileConfig, compile_circuit
from paper_2406_00766_b200.runtime import plan as P

CASES = [
    ("hclt", S.StructureConfig(kind="hclt", num_vars=40, hidden_dim=64, num_categories=16,
                               seed=3), 32),
    ("hclt16", S.StructureConfig(kind="hclt", num_vars=30, hidden_dim=32, num_categories=8,
                                 seed=6), 16),
    ("hmm_tied", S.StructureConfig(kind="hmm", seq_len=8, hidden_dim=128, vocab_size=40,
                                   seed=2, tied=True), 32),
    ("hmm_untied", S.StructureConfig(kind="hmm", seq_len=6, hidden_dim=64, vocab_size=30,
                                     seed=5, tied=False), 32),
    ("pd", S.StructureConfig(kind="pd", shape=(3, 4), hidden_dim=3, num_categories=5, seed=4),
     32),
    ("ratspn", S.StructureConfig(kind="ratspn", num_vars=16, depth=3, hidden_dim=4,
                                 num_categories=8, num_repetitions=6, seed=3), 32),
]


@pytest.fixture(scope="module", params=CASES, ids=[c[0] for c in CASES])
def compiled(request):
    _, cfg, bs = request.param
    return compile_circuit(S.build_structure(cfg), CompileConfig(block_size=bs))


def _push_count(c):
    pc = np.zeros(c.num_value_slots, dtype=np.int64)
    for L in c.layers:
        for p in L.pushes:
            np.add.at(pc, p.children.ravel(), 1)
    if c.root_children is not None and c.root_row >= 0:
        np.add.at(pc, np.asarray(c.root_children, dtype=np.int64), 2)
    return pc


def test_leaf_alias_tables(compiled):
    c = compiled
    blocks, _ = P.input_blocks(c)
    arow, adir, pad = P.leaf_alias(c, blocks, _push_count(c))
    if pad is None:
        assert np.all(arow < 0)
        return
    L = c.layers[0]
    out = np.concatenate([ev.out for ev in L.prod_evals])
    ch = np.concatenate([ev.children[:, 0] for ev in L.prod_evals])
    row_of = dict(zip(ch.tolist(), out.tolist()))
    covered = []
    for b in np.flatnonzero(arow >= 0).tolist():
        s0, n = int(blocks["slot0"][b]), int(blocks["count"][b])
        rows = arow[b] + adir[b] * np.arange(n)
        assert [row_of[s0 + i] for i in range(n)] == rows.tolist()  # each input -> its product
        assert rows.min() % L.k_n == 0 and n % L.k_n == 0          # whole product blocks
        covered.append(rows)
    covered = np.sort(np.concatenate(covered))
    assert np.array_equal(covered, np.sort(out))                     # every product aliased once
    pad_rows = np.setdiff1d(np.arange(L.scratch_window), out)
    assert np.array_equal(np.unique(pad_rows // L.k_n), np.asarray(pad))


def test_push_ratio_tables(compiled):
    c = compiled
    last = np.full(max(c.num_prod_rows, 1), -1, dtype=np.int64)
    for li, L in enumerate(c.layers):
        last[np.asarray(L.prod_rows, dtype=np.int64)] = li
    pc = _push_count(c)
    tabs = [P.push_tables(L, li, last, pc) for li, L in enumerate(c.layers)]
    pr, pre, roff, n_rmax = P.push_ratio_tables(c, tabs)
    rrows = []
    for li, L in enumerate(c.layers):
        t = pr[li]
        assert t["qoff"].size == t["row"].size + 1 or t["row"].size == 0
        assert np.all(t["qblk"] < max(t["row"].size, 1))
        for q in np.flatnonzero(t["qkind"] == 1).tolist():
            rrows.append(int(t["qrrow"][q]))
            assert 0 <= t["qrrow"][q] < n_rmax
        if t["row"].size:
            assert np.array_equal(np.diff(t["qoff"]), t["f"])      # fan-in slots per block
    # every pre-ratioed sum block gets exactly one R row, all rows are used
    assert sorted(rrows) == list(range(n_rmax))
    sizes = [int(sum(g.sum_ids.size for g in L.fwd_groups)) for L in c.layers]
    assert n_rmax == sum(s for s, p in zip(sizes, pre) if p)
    assert all((o >= 0) == p for o, p in zip(roff, pre))


def test_em_block_orders(compiled):
    c = compiled
    t_start, t_f, t_c, t_km, t_kn, _ = P.mma_tiles(c, True)
    tb, rest = P.em_tile_blocks(c, t_start, t_f, t_c, t_km, t_kn)
    out, n_pre, ranges, fus = P.em_fused_order(c, tb, True)
    nb = int(tb["blk_km"].size)
    assert out["blk_km"].size == nb and 0 <= n_pre <= nb
    # same blocks (as tile sets) before and after the reorder
    def sets(t):
        off = t["blk_tile_off"]
        return sorted(tuple(sorted(t["tile_start"][off[b]:off[b + 1]].tolist()))
                      for b in range(t["blk_km"].size))
    assert sets(out) == sets(tb)
    # the fused layers' ranges tile [n_pre, nb) without overlap
    spans = sorted((lo, hi) for (lo, hi), f in zip(ranges, fus) if f)
    pos = n_pre
    for lo, hi in spans:
        assert lo == pos and hi > lo
        pos = hi
    assert pos == nb
    # fused layers: 32 x 32 blocks, one per sum block of the layer
    for li, f in enumerate(fus):
        if f:
            L = c.layers[li]
            assert L.k_m == 32 and L.k_n == 32
            lo, hi = ranges[li]
            assert hi - lo == sum(int(g.sum_ids.size) for g in L.fwd_groups)


def test_program_builds_and_reports(compiled):
    prog, blob, info = P.build_program(compiled)
    assert prog[0] == P.MAGIC and prog[1] == P.VERSION and prog[-1] == P.MAGIC
    for key in ("leaf_alias", "pre_ratio_layers", "em_fused_layers", "input_inline_em",
                "fp_cover", "prod_flows_optional"):
        assert key in info
