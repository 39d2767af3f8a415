"""PCCF v1 compiled-circuit container (``pcirc/compiler/cache.py``): byte
identity with the reference's writer (sha256 digests the reference itself
produced, tests/golden/make_pccf_digests.py — including a K=512 HMM and a
3072-variable HCLT of latent 64, too large to recompile with the reference
at test time), round trips, the graph-hash guard and corruption detection
(the reference's tests/test_cache.py cases)."""
import hashlib
import json
from pathlib import Path

import numpy as np
import pytest

from _golden import GOLDEN, cases, graph_from, load
from paper_2406_00766_b200.compiler import CompileConfig, compile_circuit
from paper_2406_00766_b200.compiler.cache import (dumps_compiled, load_compiled,
                                                  loads_compiled, save_compiled)
from paper_2406_00766_b200.errors import FormatError

DIGESTS = json.loads((GOLDEN / "pccf_digests.json").read_text())


def _sha(b: bytes) -> str:
    return hashlib.sha256(b).hexdigest()


@pytest.mark.parametrize("name", cases())
def test_bytes_match_reference_writer(name):
    rec = load(name)
    g = graph_from(rec)
    for k in rec["ks"].tolist():
        c = compile_circuit(g, CompileConfig(block_size=k))
        blob = dumps_compiled(c)
        assert _sha(blob) == DIGESTS[f"{name}/k{k}"], (name, k)
        assert dumps_compiled(loads_compiled(blob)) == blob


@pytest.mark.parametrize("key", ["hmm_T32_K512_V100/k32", "hclt_3072x64/k32"])
def test_large_layouts_match_reference(key):
    import sys
    sys.path.insert(0, str(GOLDEN))
    from _digest_cases import BIG
    build, k = BIG[key]
    c = compile_circuit(build(), CompileConfig(block_size=k), validate=False)
    assert _sha(dumps_compiled(c)) == DIGESTS[key]


def _small():
    rec = load(cases()[0])
    return compile_circuit(graph_from(rec), CompileConfig(block_size=4))


def test_round_trip_fields_and_file(tmp_path):
    c = _small()
    c2 = loads_compiled(dumps_compiled(c))
    assert c2.graph_hash == c.graph_hash and c2.config == c.config
    np.testing.assert_array_equal(c2.theta, c.theta)
    np.testing.assert_array_equal(c2.group_off, c.group_off)
    for a, b in zip(c.layers, c2.layers):
        for ga, gb in zip(a.fwd_groups, b.fwd_groups):
            np.testing.assert_array_equal(ga.param_ids, gb.param_ids)
        assert a.report == b.report
    p = tmp_path / "circuit.pcc"
    save_compiled(c, p)
    assert dumps_compiled(load_compiled(p, expect_hash=c.graph_hash)) == dumps_compiled(c)
    with pytest.raises(FormatError):
        load_compiled(p, expect_hash="0" * 64)
    with pytest.raises(FormatError):
        load_compiled(tmp_path / "absent.pcc")


def test_corruption_detected():
    blob = dumps_compiled(_small())
    bad = bytearray(blob)
    bad[0] ^= 0xFF
    for b in (bytes(bad), blob[: len(blob) // 2], blob + b"x", blob[:3]):
        with pytest.raises(FormatError):
            loads_compiled(b)
    ver = bytearray(blob)
    ver[4] = 2  # version field
    with pytest.raises(FormatError):
        loads_compiled(bytes(ver))


@pytest.mark.gpu
def test_loaded_layout_runs_on_device():
    """A PCCF-loaded circuit drives the device plan: identical results."""
    import torch
    from paper_2406_00766_b200.runtime import backward, forward
    rec = load(cases()[0])
    c = compile_circuit(graph_from(rec), CompileConfig(block_size=4))
    c2 = loads_compiled(dumps_compiled(c))
    l1, b1 = forward(c, rec["x"])
    backward(c, b1)
    l2, b2 = forward(c2, rec["x"])
    backward(c2, b2)
    torch.cuda.synchronize()
    assert torch.equal(l1, l2)
    assert torch.allclose(b1.f_params, b2.f_params, rtol=1e-6, atol=0)
