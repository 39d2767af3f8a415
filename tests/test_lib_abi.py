"""The C-ABI library builds, loads without a GPU and exports every declared symbol."""
import re
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]


def _declared():
    text = (ROOT / "include" / "pcirc_b200.h").read_text()
    return sorted(set(re.findall(r"^\s*(?:int|int64_t)\s+(pcb_\w+)\s*\(", text, re.M)))


def test_library_exports_every_header_symbol():
    from paper_2406_00766_b200 import _build
    from paper_2406_00766_b200.runtime import _lib
    _build.build()
    lib = _lib.load()
    names = _declared()
    assert len(names) >= 15
    for n in names:
        assert hasattr(lib, n), n
        assert n in _lib.SIGNATURES, n
    assert lib.pcb_abi_version() == _lib.ABI_VERSION


def test_plan_program_parses_on_host():
    """pcb_plan_create only reads the host program; a bogus device blob pointer
    is never dereferenced, so plan parsing is testable without a GPU."""
    import ctypes as C
    from paper_2406_00766_b200 import structures as S
    from paper_2406_00766_b200.compiler import CompileConfig, compile_circuit
    from paper_2406_00766_b200.runtime import _lib
    from paper_2406_00766_b200.runtime.plan import build_program
    g = S.build_hclt(S.StructureConfig(kind="hclt", num_vars=9, hidden_dim=16,
                                       num_categories=4, seed=0))
    c = compile_circuit(g, CompileConfig(block_size=16))
    prog, blob, info = build_program(c)
    assert info["tc_super_rows"] > 0
    lib = _lib.load()
    h = C.c_void_p()
    st = lib.pcb_plan_create(prog.ctypes.data, prog.size, C.c_void_p(0x1000), blob.size,
                             C.byref(h))
    assert st == 0 and h.value
    assert lib.pcb_plan_num_layers(h) == len(c.layers)
    lib.pcb_plan_destroy(h)
    bad = prog.copy()
    bad[-1] = 0
    assert lib.pcb_plan_create(bad.ctypes.data, bad.size, C.c_void_p(0x1000), blob.size,
                               C.byref(h)) == 1


def test_super_rows_stack_identical_child_rows():
    from paper_2406_00766_b200.runtime.plan import tc_super_rows
    prod = np.array([[1, 2], [3, 4], [1, 2], [1, 2], [3, 4]])
    offs, mem = tc_super_rows(prod, k_m=128)
    groups = [mem[offs[i]:offs[i + 1]].tolist() for i in range(offs.size - 1)]
    assert groups == [[0, 2], [3], [1, 4]]
