"""Layout bit-exactness: the host compiler against the reference compiler.

Golden digests were produced by the reference ``compile_circuit`` itself
(``tests/golden/make_golden.py``); when /root/reference is present the
comparison is also made array-for-array on freshly generated circuits.
"""
import numpy as np
import pytest

from _golden import cases, graph_from, layout_digest, load
from paper_2406_00766_b200.compiler import CompileConfig, compile_circuit


@pytest.mark.parametrize("name", cases())
def test_layout_digest_matches_reference(name):
    rec = load(name)
    g = graph_from(rec)
    for k in rec["ks"].tolist():
        c = compile_circuit(g, CompileConfig(block_size=k))
        assert c.graph_hash == str(rec[f"k{k}_graph_hash"])
        assert layout_digest(c) == str(rec[f"k{k}_digest"]), (name, k)
        np.testing.assert_array_equal(c.theta, rec[f"k{k}_theta"])


def _eq(a, b, path):
    if isinstance(a, np.ndarray) or isinstance(b, np.ndarray):
        np.testing.assert_array_equal(np.asarray(a), np.asarray(b), err_msg=path)
    elif isinstance(a, (list, tuple)):
        assert len(a) == len(b), path
        for i, (x, y) in enumerate(zip(a, b)):
            _eq(x, y, f"{path}[{i}]")
    elif hasattr(a, "__dataclass_fields__"):
        for f in a.__dataclass_fields__:
            if f in ("config", "_device_plans"):
                continue
            if f == "report":
                for rf in b.report.__dataclass_fields__:
                    assert getattr(a.report, rf) == getattr(b.report, rf), f"{path}.report.{rf}"
                continue
            _eq(getattr(a, f), getattr(b, f), f"{path}.{f}")
    else:
        assert a == b, (path, a, b)


@pytest.mark.reference
def test_array_for_array_random_circuits(ref_pcirc):
    import sys
    sys.path.insert(0, "/root/reference/pkg/tests")
    from circuitgen import random_circuit
    from pcirc.compiler import CompileConfig as RC
    from pcirc.compiler import compile_circuit as rcompile
    from paper_2406_00766_b200.graph import CircuitGraph
    rng = np.random.default_rng(7)
    for _ in range(30):
        g = random_circuit(rng, max_vars=8, max_nodes=200)
        for k in (1, 2, 4, 8):
            ref = rcompile(g, RC(block_size=k))
            mine = compile_circuit(CircuitGraph.from_reference(g), CompileConfig(block_size=k))
            _eq(mine, ref, f"k{k}")


@pytest.mark.reference
def test_array_for_array_structures(ref_pcirc):
    from pcirc.compiler import CompileConfig as RC
    from pcirc.compiler import compile_circuit as rcompile
    from pcirc.structures import StructureConfig as RS
    from pcirc.structures import build_structure as rbuild
    from paper_2406_00766_b200 import structures as S
    cases_ = [("hmm", dict(seq_len=8, hidden_dim=16, vocab_size=7, tied=True), 8),
              ("hmm", dict(seq_len=5, hidden_dim=4, vocab_size=3, tied=False), 4),
              ("pd", dict(shape=(4, 4), hidden_dim=3, num_categories=3), 2),
              ("ratspn", dict(num_vars=16, depth=3, hidden_dim=4, num_categories=3), 4)]
    for kind, kw, k in cases_:
        rg = rbuild(RS(kind=kind, seed=3, **kw))
        mg = S.build_structure(S.StructureConfig(kind=kind, seed=3, **kw))
        ref = rcompile(rg, RC(block_size=k))
        mine = compile_circuit(mg, CompileConfig(block_size=k))
        assert mine.graph_hash == ref.graph_hash, kind
        _eq(mine, ref, kind)


@pytest.mark.reference
def test_tied_hmm_k32_matches_reference(ref_pcirc):
    """A tied HMM at the HMM-4096 block size (K=32), reduced hidden size."""
    from pcirc.compiler import CompileConfig as RC
    from pcirc.compiler import compile_circuit as rcompile
    from pcirc.structures import StructureConfig as RS
    from pcirc.structures import build_hmm as rhmm
    from paper_2406_00766_b200 import structures as S
    kw = dict(seq_len=32, hidden_dim=128, vocab_size=50, tied=True)
    ref = rcompile(rhmm(RS(kind="hmm", seed=0, **kw)), RC(block_size=32))
    mine = compile_circuit(S.build_hmm(S.StructureConfig(kind="hmm", seed=0, **kw)),
                           CompileConfig(block_size=32))
    _eq(mine, ref, "hmm128")
    assert len(mine.reductions) == 31 * 16
