"""The native host-compiler core (``csrc/host/pcc_compile.cpp``) against the
vectorised-numpy compiler and the reference goldens: byte-identical PCCF
serialisations (the reference's own layout exchange format) on the golden
circuits, on every structure generator (HCLT, tied / untied HMM, PyJuice PD,
RAT-SPN with repetitions) and on random circuits, independent of the worker
count; the reference's compile errors (parallel edges, misaligned tying)
raised with the same messages."""

import numpy as np
import pytest

from _golden import cases, graph_from, load
from paper_2406_00766_b200 import structures as S
from paper_2406_00766_b200.compiler import CompileConfig, compile_circuit
from paper_2406_00766_b200.compiler import _native
from paper_2406_00766_b200.compiler import build as B
from paper_2406_00766_b200.compiler.cache import dumps_compiled
from paper_2406_00766_b200.errors import CircuitValidationError
from paper_2406_00766_b200.graph import CircuitGraph


@pytest.fixture(scope="module")
def nat():
    from paper_2406_00766_b200 import _build
    _build.build_host()
    lib = _native.lib()
    if lib is None:
        pytest.skip("PCB_COMPILER=numpy")
    return lib


def _both(g, k):
    g = B._as_graph(g)
    g.freeze()
    a = B._compile(g, CompileConfig(block_size=k), True)
    b = B._compile(g, CompileConfig(block_size=k), False)
    return dumps_compiled(a), dumps_compiled(b)


def test_library_exports(nat):
    """libpcirc_host.so exports every symbol include/pcirc_host.h declares,
    and the ctypes table binds exactly those."""
    import re
    from pathlib import Path
    text = (Path(__file__).resolve().parents[1] / "include" / "pcirc_host.h").read_text()
    declared = set(re.findall(r"\b(pcc_\w+)\s*\(", text))
    assert len(declared) >= 30
    assert declared == set(_native._SIGS)
    for name in declared:
        assert hasattr(nat, name), name
    assert nat.pcc_version() == 1 and nat.pcc_threads() >= 1


@pytest.mark.parametrize("name", cases())
def test_golden_circuits_native_equals_numpy(nat, name):
    rec = load(name)
    g = graph_from(rec)
    for k in rec["ks"].tolist():
        a, b = _both(g, k)
        assert a == b, (name, k)


STRUCTS = [
    ("hclt", dict(num_vars=40, hidden_dim=32, num_categories=8), 32),
    ("hclt", dict(num_vars=24, hidden_dim=64, num_categories=16), 16),
    ("hmm", dict(seq_len=6, hidden_dim=64, vocab_size=20, tied=True), 32),
    ("hmm", dict(seq_len=5, hidden_dim=16, vocab_size=7, tied=False), 8),
    ("pd", dict(shape=(6, 6, 3), split_interval=2, hidden_dim=16, num_categories=8,
                elementwise=True), 16),
    ("pd", dict(shape=(4, 4), hidden_dim=3, num_categories=3), 2),
    ("ratspn", dict(num_vars=40, depth=4, hidden_dim=8, num_input_components=4,
                    num_categories=5, num_repetitions=2), 8),
]


@pytest.mark.parametrize("kind,kw,k", STRUCTS)
def test_structures_native_equals_numpy(nat, kind, kw, k):
    g = S.build_structure(S.StructureConfig(kind=kind, seed=5, **kw))
    a, b = _both(g, k)
    assert a == b


def test_random_circuits_native_equals_numpy(nat):
    """Ragged circuits: demoted layers, input children of sums, mixed fan-in,
    shared slots and ties (the reference's random generator's shapes)."""
    rng = np.random.default_rng(11)
    for trial in range(25):
        g = _random_circuit(rng)
        g.freeze()
        for k in (1, 2, 4, 8, 16, 32):
            try:
                b = dumps_compiled(B._compile(g, CompileConfig(block_size=k), False))
            except CircuitValidationError:  # the native pass must defer too
                with pytest.raises(_native.NativeError):
                    B._compile(g, CompileConfig(block_size=k), True)
                continue
            a = dumps_compiled(B._compile(g, CompileConfig(block_size=k), True))
            assert a == b, (trial, k)


def _random_circuit(rng):
    nv = int(rng.integers(2, 6))
    g = CircuitGraph(nv)
    layer = [g.add_input(v, rng.dirichlet(np.ones(3))) for v in range(nv) for _ in range(2)]
    scope = {n: {v} for n, v in zip(layer, [v for v in range(nv) for _ in range(2)])}
    while len(layer) > 1:
        prods = []
        rng.shuffle(layer)
        for a, b in zip(layer[::2], layer[1::2]):
            if scope[a] & scope[b]:
                continue
            p = g.add_product([a, b])
            scope[p] = scope[a] | scope[b]
            prods.append(p)
        if not prods:
            break
        nxt = []
        by_scope: dict = {}
        for p in prods:
            by_scope.setdefault(frozenset(scope[p]), []).append(p)
        for sc, ps in by_scope.items():
            for _ in range(int(rng.integers(1, 4))):
                ch = list(rng.choice(ps, size=int(rng.integers(1, len(ps) + 1)), replace=False))
                s = g.add_sum(ch, rng.dirichlet(np.ones(len(ch))))
                scope[s] = set(sc)
                nxt.append(s)
        layer = nxt
    root_scope = frozenset(range(nv))
    roots = [n for n in layer if scope[n] == set(root_scope)]
    if not roots:
        cands = [n for n in scope if scope[n] == set(root_scope)]
        roots = cands[:1] or [layer[0]]
    g.set_root(int(roots[0]))
    if rng.random() < 0.5 and g.num_param_slots > 4:  # a tie between two sum slots
        sl = rng.choice(g.num_param_slots, size=2, replace=False)
        g.tie([int(sl[0]), int(sl[1])])
    return g


def test_thread_count_independent(nat):
    g = S.build_structure(S.StructureConfig(kind="hmm", seed=2, seq_len=5, hidden_dim=64,
                                            vocab_size=30, tied=True))
    g.freeze()
    nat.pcc_set_threads(1)
    try:
        one = dumps_compiled(B._compile(g, CompileConfig(block_size=32), True))
    finally:
        nat.pcc_set_threads(0)
    many = dumps_compiled(B._compile(g, CompileConfig(block_size=32), True))
    assert one == many


def _tied_misaligned():
    g = CircuitGraph(1)
    i0 = g.add_input(0, [0.5, 0.5])
    i1 = g.add_input(0, [0.3, 0.7])
    a = g.add_sum([i0, i1], [0.4, 0.6])
    b = g.add_sum([i0, i1], [0.5, 0.5])
    g.set_root(g.add_sum([a, b], [0.5, 0.5]))
    g.tie([int(g.nodes[a].slots[0]), int(g.nodes[b].slots[1])])
    return g


def _parallel_edges():
    g = CircuitGraph(1)
    i0 = g.add_input(0, [0.5, 0.5])
    i1 = g.add_input(0, [0.3, 0.7])
    g.set_root(g.add_sum([i0, i0, i1], [0.2, 0.2, 0.6]))
    return g


@pytest.mark.parametrize("make,msg", [(_tied_misaligned, "does not align"),
                                      (_parallel_edges, "sum node 2 has parallel edges")])
def test_compile_errors_match(nat, make, msg):
    """build.py:303-308 / 343-359: the native path defers to the numpy path,
    which raises the reference's message."""
    with pytest.raises(CircuitValidationError, match=msg):
        compile_circuit(make(), CompileConfig(block_size=2), validate=False)
    g = make()
    g.freeze()
    with pytest.raises(_native.NativeError):
        B._compile(g, CompileConfig(block_size=2), True)


def test_numpy_selector(nat, monkeypatch):
    monkeypatch.setenv("PCB_COMPILER", "numpy")
    assert _native.lib() is None
    monkeypatch.delenv("PCB_COMPILER")
    assert _native.lib() is not None


def test_group_runs_native_equals_numpy(nat, monkeypatch):
    """runtime/plan.py group_runs: the native two-pass encoding against the
    numpy one on ragged groups (empty groups, repeats, gaps)."""
    from paper_2406_00766_b200.runtime.plan import group_runs
    rng = np.random.default_rng(0)
    for _ in range(100):
        sizes = rng.integers(0, 12, int(rng.integers(1, 30)))
        go = np.concatenate([[0], np.cumsum(sizes)])
        gi = np.cumsum(rng.integers(0, 3, int(go[-1]))) + int(rng.integers(0, 5))
        got = group_runs(gi, go)
        monkeypatch.setenv("PCB_COMPILER", "numpy")
        want = group_runs(gi, go)
        monkeypatch.delenv("PCB_COMPILER")
        for a, b in zip(got, want):
            np.testing.assert_array_equal(a, b)


@pytest.mark.reference
def test_reference_random_circuits_native_equals_numpy(nat, ref_pcirc):
    """The reference test suite's own random-circuit generator (multi-parent
    nodes, zero pmf entries, input children of sums): native == numpy at
    every block size."""
    import sys
    sys.path.insert(0, "/root/reference/pkg/tests")
    from circuitgen import random_circuit
    rng = np.random.default_rng(21)
    for trial in range(20):
        rg = random_circuit(rng, max_vars=8, max_nodes=300)
        g = CircuitGraph.from_reference(rg)
        g.freeze()
        for k in (1, 2, 4, 8, 16):
            try:
                b = dumps_compiled(B._compile(g, CompileConfig(block_size=k), False))
            except CircuitValidationError:
                with pytest.raises(_native.NativeError):
                    B._compile(g, CompileConfig(block_size=k), True)
                continue
            a = dumps_compiled(B._compile(g, CompileConfig(block_size=k), True))
            assert a == b, (trial, k)


def test_concurrent_compiles_thread_safe(nat):
    """Two Python threads compiling at once (ctypes releases the GIL; the
    native scratch is per thread) give the serial layouts."""
    import threading
    graphs = [S.build_structure(S.StructureConfig(kind=k, seed=3, **kw))
              for k, kw, _ in (STRUCTS[0], STRUCTS[2])]
    ks = (STRUCTS[0][2], STRUCTS[2][2])
    want = [dumps_compiled(compile_circuit(g, CompileConfig(block_size=k)))
            for g, k in zip(graphs, ks)]
    got = [None, None]

    def run(i):
        got[i] = dumps_compiled(compile_circuit(graphs[i], CompileConfig(block_size=ks[i])))
    th = [threading.Thread(target=run, args=(i,)) for i in range(2)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert got == want
