"""ctypes binding of the in-tree sm_100a library (``include/pcirc_b200.h``).

There is no fallback: if the library is missing or fails to load, every
runtime entry point raises.  ``build()`` in ``__graft_entry__`` (or
``python -m paper_2406_00766_b200._build``) produces it.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

from ..errors import PcircError, raise_for_status

LIB_PATH = Path(__file__).resolve().parent.parent / "_lib" / "libpcirc_b200.so"

_P = C.c_void_p
_I = C.c_int
_L = C.c_int64
_F = C.c_float

# name -> (restype, argtypes); the exported symbol set of include/pcirc_b200.h
SIGNATURES = {
    "pcb_abi_version": (_I, []),
    "pcb_plan_create": (_I, [_P, _L, _P, _L, C.POINTER(_P)]),
    "pcb_plan_destroy": (_I, [_P]),
    "pcb_plan_num_layers": (_I, [_P]),
    "pcb_plan_scratch_rows": (_L, [_P]),
    "pcb_plan_set_mma": (_I, [_P, _P, _L]),
    "pcb_theta_refresh": (_I, [_P, _P, _P]),
    "pcb_plan_set_theta": (_I, [_P, _P]),
    "pcb_exec_create": (_I, [_P, C.POINTER(_P)]),
    "pcb_exec_destroy": (_I, [_P]),
    "pcb_exec_set_flow_events": (_I, [_P, _P, _I]),
    "pcb_train_step": (_I, [_P, _P, _P, _I, _I, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _I, _F,
                            _F, _P]),
    "pcb_tc_selftest_mn": (_I, [_P, _I, _I, _I, _P, _P, _P]),
    "pcb_check_batch": (_I, [_P, _P, _I, _I, _P, _P]),
    "pcb_transpose_batch_i64": (_I, [_P, _P, _I, _I, _P, _P]),
    "pcb_transpose_batch_i32": (_I, [_P, _P, _I, _I, _P, _P]),
    "pcb_plan_workspace_floats": (_L, [_P, _I]),
    "pcb_forward": (_I, [_P, _P, _I, _I, _P, _P, _P, _P, _P, _P]),
    "pcb_backward": (_I, [_P, _P, _I, _I, _P, _P, _P, _P, _P, _P, _P, _P, _P]),
    "pcb_layer_forward": (_I, [_P, _I, _P, _I, _I, _P, _P, _P, _P]),
    "pcb_layer_backward": (_I, [_P, _I, _P, _I, _I, _P, _P, _P, _P, _P, _P, _P, _P]),
    "pcb_em_update": (_I, [_P, _P, _P, _P, _F, _F, _P]),
    "pcb_axpy_accumulate": (_I, [_P, _L, _P, _P]),
    "pcb_count_nonfinite": (_I, [_P, _L, _P, _P]),
    "pcb_launch_count": (_L, []),
    "pcb_profile_enable": (_I, [_I]),
    "pcb_profile_read": (_I, [_P, _P, _P, _I]),
    "pcb_tc_selftest": (_I, [_P, _I, _I, _P, _P, _P]),
}

ABI_VERSION = 3

# pcb_train_step flags
STEP_LEAN, STEP_SERIAL, STEP_EM = 1, 2, 4

_lib = None


def load(path: Path | None = None) -> C.CDLL:
    """Load (once) and type the library; raises if it is absent."""
    global _lib
    if _lib is not None:
        return _lib
    # PCB_LIB: an alternative build of the same library (kernel A/B experiments)
    p = Path(path) if path else Path(os.environ.get("PCB_LIB") or LIB_PATH)
    if not p.exists():
        raise PcircError(
            f"CUDA library {p} is not built; run __graft_entry__.build() "
            "(there is no CPU fallback)")
    lib = C.CDLL(str(p))
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if lib.pcb_abi_version() != ABI_VERSION:
        raise PcircError("pcirc_b200 ABI version mismatch; rebuild the library")
    _lib = lib
    return lib


def call(name: str, *args) -> None:
    """Invoke an entry point and map its status onto the error classes."""
    raise_for_status(getattr(load(), name)(*args), name)


KERNEL_CLASSES = ["input_fwd", "prod_eval", "sum_fwd_tc", "sum_fwd_simt", "param_flow",
                  "child_flow", "accum_push", "input_flow", "replica", "em", "misc"]


def profile_enable(on: bool) -> None:
    load().pcb_profile_enable(1 if on else 0)


def profile_read() -> dict:
    """{class: (ms, scopes, launches)} accumulated since the last read."""
    import numpy as np
    n = len(KERNEL_CLASSES)
    ms = np.zeros(n, dtype=np.float64)
    sc = np.zeros(n, dtype=np.int64)
    ln = np.zeros(n, dtype=np.int64)
    call("pcb_profile_read", ms.ctypes.data, sc.ctypes.data, ln.ctypes.data, n)
    return {k: (float(ms[i]), int(sc[i]), int(ln[i])) for i, k in enumerate(KERNEL_CLASSES)}


def ptr(t) -> int:
    """Raw device pointer of a torch tensor (0 for None)."""
    return 0 if t is None else t.data_ptr()


def stream_handle(stream=None) -> int:
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream
