"""ctypes binding of the native host-compiler core (``csrc/host/pcc_compile.cpp``,
built into ``_lib/libpcirc_host.so`` by ``_build.build()``).

``lib()`` returns the loaded library, or ``None`` when it is not built or
``PCB_COMPILER=numpy`` selects the vectorised-numpy compiler (same layout,
bit for bit; ``tests/test_compile_native.py`` checks the two against each
other and both against the reference goldens).
"""
from __future__ import annotations

import ctypes as C
import os
import threading
from pathlib import Path

import numpy as np

LIB_PATH = Path(__file__).resolve().parents[1] / "_lib" / "libpcirc_host.so"

_P = C.c_void_p
_I64 = C.c_int64
_lib = None
_tried = False
_lock = threading.Lock()

_SIGS = {
    "pcc_version": (C.c_int, []),
    "pcc_set_threads": (None, [C.c_int]),
    "pcc_threads": (C.c_int, []),
    "pcc_gather_layer": (None, [C.c_int, _P, _P, _P, _P, _P, _P, _P, _P, C.c_int8, _I64, _P, _P,
                                _P, _P]),
    "pcc_fill_i64": (None, [_P, _I64, _I64]),
    "pcc_copy_ranges": (None, [_I64, _P, _P, _P, _P, _P]),
    "pcc_iota_ranges": (None, [_I64, _P, _P, _P, _P]),
    "pcc_assign_ranges": (C.c_int, [_I64, _P, _P, _P, C.c_int, _P, _P, _P]),
    "pcc_claim_ranges": (C.c_int, [_I64, _P, _P, _P]),
    "pcc_layer_new": (_P, [_I64, _P, _I64, _P, _P]),
    "pcc_layer_free": (None, [_P]),
    "pcc_blocks": (C.c_int, [_P, _I64, _I64, C.c_double]),
    "pcc_blocks_meta": (None, [_P, _P, _P]),
    "pcc_blocks_get": (None, [_P] + [_P] * 10),
    "pcc_slot_uses": (None, [_I64, _P, _P, _P, _P]),
    "pcc_tiles_new": (_P, []),
    "pcc_tiles_free": (None, [_P]),
    "pcc_tiles_count": (_I64, [_P]),
    "pcc_tiles_get": (None, [_P, _P, _P]),
    "pcc_tiles": (C.c_int, [_P, _P, _P, _P, _P, _P, _P, _I64, _P, _P, _P, _P]),
    "pcc_rows_new": (_P, []),
    "pcc_rows_free": (None, [_P]),
    "pcc_rows_add_multi": (None, [_P, _I64, _P, _I64, _P, _P, _P, _P]),
    "pcc_sum_groups_multi": (C.c_int, [_I64, _P, _P, _P, _P, _P, _P, _P]),
    "pcc_depths": (None, [_I64, _P, _P, _P, _P, _P, _P, _P]),
    "pcc_hash_records_multi": (None, [_I64, _P, _P, _P, _P, _P, _P, _P, _P, _P]),
    "pcc_release": (None, []),
    "pcc_group_runs": (None, [_I64, _P, _P, _P, _P, _P]),
    "pcc_minmax": (None, [_P, _I64, _P]),
    "pcc_narrow_i32": (None, [_P, _I64, _P]),
    "pcc_rows_count": (_I64, [_P, _P]),
    "pcc_rows_get": (None, [_P, _P, _P, _P]),
    "pcc_claim_groups": (C.c_int, [_I64, _P, _P, _P]),
}


def lib():
    global _lib, _tried
    if os.environ.get("PCB_COMPILER", "").lower() == "numpy":
        return None
    with _lock:
        if not _tried:
            if LIB_PATH.exists():
                h = C.CDLL(str(LIB_PATH))
                for name, (res, args) in _SIGS.items():
                    fn = getattr(h, name)
                    fn.restype = res
                    fn.argtypes = args
                _lib = h
            _tried = True
    return _lib


def ptr(a: np.ndarray | None):
    if a is None:
        return None
    assert a.flags.c_contiguous, "native compiler needs contiguous arrays"
    return a.ctypes.data


def i64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.int64)


def full_i64(n: int, value: int) -> np.ndarray:
    """np.full(n, value) with a parallel first touch."""
    a = np.empty(n, dtype=np.int64)
    lib().pcc_fill_i64(ptr(a), n, value)
    return a


def rows(a) -> tuple[np.ndarray, int]:
    """(array, row stride in elements) of a 2-D int64 matrix whose rows are
    contiguous -- broadcast views (stride 0, one row shared by a segment)
    are passed as they are instead of being materialised."""
    a = np.asarray(a)
    if a.ndim == 2 and a.dtype == np.int64 and (a.strides[1] == 8 or a.shape[1] <= 1) \
            and a.strides[0] >= 0 and a.strides[0] % 8 == 0:
        return a, a.strides[0] // 8
    c = np.ascontiguousarray(a, dtype=np.int64).reshape(a.shape[0], -1)
    return c, c.shape[1]


def ptr_array(arrs) -> C.Array:
    return (C.c_void_p * len(arrs))(*[ptr(a) for a in arrs])


def addr(a: np.ndarray) -> int:
    """Data address of a C-contiguous array (cheaper than ``a.ctypes``)."""
    return a.__array_interface__["data"][0]


def addr_array(addrs) -> np.ndarray:
    """A pointer table (uint64) from data addresses (0 = null)."""
    return np.array(addrs, dtype=np.uint64)


class NativeError(Exception):
    """A native pass hit a condition whose exact error message the numpy
    compiler produces; the caller re-runs the numpy path to raise it."""


class Layer:
    """One sum layer's native working set; keeps the arrays it points into."""

    def __init__(self, sids: np.ndarray, e_key: np.ndarray, off: np.ndarray):
        self.L = lib()
        self.sids, self.e_key, self.off = i64(sids), i64(e_key), i64(off)
        self.h = self.L.pcc_layer_new(self.sids.size, ptr(self.sids), self.e_key.size,
                                      ptr(self.e_key), ptr(self.off))

    def blocks(self, k: int, k_n: int, demote: float):
        if self.L.pcc_blocks(self.h, k, k_n, demote) != 0:
            raise NativeError("key range")
        meta = np.zeros(7, np.int64)
        pads = np.zeros(2, np.float64)
        self.L.pcc_blocks_meta(self.h, ptr(meta), ptr(pads))
        km, kn, dem, n_sb, n_pb, n_pk, n_cb = (int(v) for v in meta)
        n = self.sids.size
        out = dict(smat=np.empty((n_sb, km), np.int64), pmat=np.empty((n_pb, kn), np.int64),
                   cb_flat=np.empty(n_cb, np.int64), cb_off=np.empty(n_sb + 1, np.int64),
                   sum_keys=np.empty(n, np.int64), sum_blk=np.empty(n, np.int64),
                   sum_off=np.empty(n, np.int64), prod_keys=np.empty(n_pk, np.int64),
                   prod_blk=np.empty(n_pk, np.int64), prod_off=np.empty(n_pk, np.int64))
        self.L.pcc_blocks_get(self.h, *[ptr(a) for a in out.values()])
        return km, kn, bool(dem), float(pads[0]), float(pads[1]), out

    def free(self):
        if self.h:
            self.L.pcc_layer_free(self.h)
            self.h = None
            self.sids = self.e_key = self.off = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass
