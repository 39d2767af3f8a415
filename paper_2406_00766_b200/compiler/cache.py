"""PCCF v1: the on-disk compiled-circuit container (``pcirc/compiler/cache.py:93-393``).

Byte-compatible with the reference: a file written here loads in the
reference and vice versa, and ``dumps_compiled`` of the same compiled
layout is byte-identical on both sides — which makes PCCF the golden
layout-exchange format: the layout tests compare sha256
digests of these bytes against digests the reference produced, including
for circuits too large to recompile at test time.

Encoding (little endian throughout):
  header    b"PCCF", int64 version (1), int64 len + ascii graph hash
  config    7 int64 (block, sum block | -1, prod block | -1, max groups,
            round quantum, round threshold, contention), 2 float64
            (tolerance, demote threshold)
  sizes     11 int64 (num_vars, num_nodes, reserved, value slots, scratch,
            prod rows, theta, f_params, zero tile, root slot, root row)
  arrays    float64 tensors (theta) and int32 index tensors, each preceded
            by int64 ndim and int64 dims
  then the circuit-level tables, input chunks and sum layers in the order of
  ``_CIRCUIT`` / ``_LAYER`` below.

Instead of a hand-written sequence of write / read calls, the record layout
is a schema (field name, codec) walked by one encoder and one decoder, so
the two directions cannot drift apart.  Large files are written straight to
the output stream (no whole-file copy).
"""
from __future__ import annotations

import io
import struct
from pathlib import Path

import numpy as np

from ..errors import FormatError, UsageError
from .build import CompileConfig
from .ir import (BackwardGroupIR, CompiledCircuit, FlowPushIR, ForwardGroupIR, InputLayerIR,
                 LayerReport, ProductEvalIR, SumLayerIR)

__all__ = ["MAGIC", "VERSION", "dumps_compiled", "loads_compiled", "write_compiled",
           "save_compiled", "load_compiled"]

MAGIC = b"PCCF"
VERSION = 1
_I32 = np.iinfo(np.int32)


class _Out:
    def __init__(self, f):
        self.f = f

    def ints(self, *v):
        self.f.write(struct.pack(f"<{len(v)}q", *(int(x) for x in v)))

    def floats(self, *v):
        self.f.write(struct.pack(f"<{len(v)}d", *(float(x) for x in v)))

    def tensor(self, a, dtype):
        a = np.asarray(a)
        if dtype == "<i4" and a.size and (a.min() < _I32.min or a.max() > _I32.max):
            raise UsageError("index array exceeds the 32-bit cache format")
        self.ints(a.ndim, *a.shape)
        self.f.write(np.ascontiguousarray(a, dtype=dtype).tobytes())


class _In:
    def __init__(self, buf: bytes):
        self.mv = memoryview(buf)
        self.pos = 0

    def take(self, n: int) -> memoryview:
        if self.pos + n > len(self.mv):
            raise FormatError("compiled cache truncated")
        out = self.mv[self.pos:self.pos + n]
        self.pos += n
        return out

    def ints(self, n: int):
        return struct.unpack(f"<{n}q", self.take(8 * n))

    def floats(self, n: int):
        return struct.unpack(f"<{n}d", self.take(8 * n))

    def tensor(self, dtype) -> np.ndarray:
        (ndim,) = self.ints(1)
        if ndim < 0 or ndim > 8:
            raise FormatError("compiled cache corrupt (bad tensor rank)")
        shape = self.ints(ndim)
        if any(d < 0 for d in shape):
            raise FormatError("compiled cache corrupt (bad tensor shape)")
        count = int(np.prod(shape)) if ndim else 1
        item = np.dtype(dtype).itemsize
        arr = np.frombuffer(self.take(item * count), dtype=dtype).reshape(shape)
        return arr.astype(np.int64) if dtype == "<i4" else arr.astype(np.float64)


# codecs: "i" int64 scalar, "f" float64 scalar, "x" int32 tensor, "d" float64 tensor
_CIRCUIT_SIZES = ("num_vars", "num_nodes", "reserved", "num_value_slots", "scratch_size",
                  "num_prod_rows", "theta_size", "f_params_size", "zero_len", "root_slot",
                  "root_row")
_CIRCUIT_TABLES = (("theta", "d"), ("var_categories", "x"), ("slot_phys", "x"),
                   ("reductions", "x"), ("tile_starts", "x"), ("tile_writers", "x"),
                   ("group_idx", "x"), ("group_off", "x"), ("node_value_slot", "x"),
                   ("node_prod_row", "x"))
_CHUNK = ("node_ids", "slots", "vars", "param_ids")
_REPORT_INTS = ("num_sums", "num_prods", "demoted", "fwd_overhead", "fwd_target", "fwd_ideal",
                "bwd_overhead", "bwd_target", "bwd_ideal")


def _put(o: _Out, codec: str, v):
    if codec == "x":
        o.tensor(v, "<i4")
    else:
        o.tensor(v, "<f8")


def _get(i: _In, codec: str):
    return i.tensor("<i4" if codec == "x" else "<f8")


def write_compiled(c: CompiledCircuit, f) -> None:
    """Serialise ``c`` to a binary stream (the reference's byte layout)."""
    o = _Out(f)
    f.write(MAGIC)
    h = c.graph_hash.encode("ascii")
    o.ints(VERSION, len(h))
    f.write(h)
    cfg = c.config
    o.ints(cfg.block_size, -1 if cfg.sum_block_size is None else cfg.sum_block_size,
           -1 if cfg.prod_block_size is None else cfg.prod_block_size, cfg.max_groups,
           cfg.round_quantum, cfg.round_threshold, cfg.contention_threshold)
    o.floats(cfg.tolerance, cfg.demote_threshold)
    o.ints(*(getattr(c, k) for k in _CIRCUIT_SIZES))
    for name, codec in _CIRCUIT_TABLES:
        _put(o, codec, getattr(c, name))
    if c.root_children is None:
        o.ints(0)
    else:
        o.ints(1)
        _put(o, "x", c.root_children)
    o.ints(len(c.input_layer))
    for ch in c.input_layer:
        o.ints(ch.num_categories)
        for k in _CHUNK:
            _put(o, "x", getattr(ch, k))
    o.ints(len(c.layers))
    for L in c.layers:
        o.ints(L.depth, L.k_m, L.k_n, L.scratch_window)
        o.ints(len(L.prod_evals))
        for ev in L.prod_evals:
            _put(o, "x", ev.out), _put(o, "x", ev.children)
        o.ints(len(L.fwd_groups))
        for g in L.fwd_groups:
            for k in ("sum_ids", "prod_ids", "param_ids", "flow_ids"):
                _put(o, "x", getattr(g, k))
        o.ints(len(L.bwd_groups))
        for g in L.bwd_groups:
            for k in ("ch_ids", "par_ids", "par_param_ids"):
                _put(o, "x", getattr(g, k))
        _put(o, "x", L.prod_slots), _put(o, "x", L.prod_rows)
        o.ints(len(L.pushes))
        for p in L.pushes:
            _put(o, "x", p.rows), _put(o, "x", p.children)
        for k in ("edge_sums", "edge_children", "edge_slots"):
            _put(o, "x", getattr(L, k))
        r = L.report
        o.ints(*(int(getattr(r, k)) for k in _REPORT_INTS))
        o.floats(r.sum_pad_fraction, r.prod_pad_fraction)
        _put(o, "x", np.array(r.fwd_capacities, dtype=np.int64))
        _put(o, "x", np.array(r.bwd_capacities, dtype=np.int64))


def dumps_compiled(c: CompiledCircuit) -> bytes:
    f = io.BytesIO()
    write_compiled(c, f)
    return f.getvalue()


def loads_compiled(data: bytes) -> CompiledCircuit:
    """Parse a PCCF v1 byte string; corrupt input raises FormatError."""
    i = _In(bytes(data) if not isinstance(data, (bytes, bytearray, memoryview)) else data)
    if bytes(i.take(4)) != MAGIC:
        raise FormatError("not a compiled-circuit cache (bad magic)")
    (version,) = i.ints(1)
    if version != VERSION:
        raise FormatError(f"unsupported cache version {version}")
    (hlen,) = i.ints(1)
    if hlen < 0 or hlen > 1024:
        raise FormatError("compiled cache corrupt (bad hash length)")
    try:
        graph_hash = bytes(i.take(hlen)).decode("ascii")
    except UnicodeDecodeError:
        raise FormatError("compiled cache corrupt (bad graph hash)") from None
    bs, sbs, pbs, groups, quantum, threshold, contention = i.ints(7)
    tol, demote = i.floats(2)
    try:
        cfg = CompileConfig(block_size=bs, sum_block_size=None if sbs < 0 else sbs,
                            prod_block_size=None if pbs < 0 else pbs, max_groups=groups,
                            tolerance=tol, round_quantum=quantum, round_threshold=threshold,
                            contention_threshold=contention, demote_threshold=demote)
    except UsageError as e:
        raise FormatError(f"compiled cache corrupt (config: {e})") from None
    fields = dict(zip(_CIRCUIT_SIZES, i.ints(len(_CIRCUIT_SIZES))))
    for name, codec in _CIRCUIT_TABLES:
        fields[name] = _get(i, codec)
    fields["reductions"] = fields["reductions"].reshape(-1, 3)
    (has_rc,) = i.ints(1)
    fields["root_children"] = _get(i, "x") if has_rc else None
    (n_chunks,) = i.ints(1)
    chunks = []
    for _ in range(n_chunks):
        (ncat,) = i.ints(1)
        arrs = {k: _get(i, "x") for k in _CHUNK}
        chunks.append(InputLayerIR(num_categories=int(ncat), **arrs))
    (n_layers,) = i.ints(1)
    layers = []
    for _ in range(n_layers):
        depth, k_m, k_n, window = i.ints(4)
        (n,) = i.ints(1)
        evals = [ProductEvalIR(out=_get(i, "x"), children=_get(i, "x")) for _ in range(n)]
        (n,) = i.ints(1)
        fwd = [ForwardGroupIR(sum_ids=_get(i, "x"), prod_ids=_get(i, "x"),
                              param_ids=_get(i, "x"), flow_ids=_get(i, "x")) for _ in range(n)]
        (n,) = i.ints(1)
        bwd = [BackwardGroupIR(ch_ids=_get(i, "x"), par_ids=_get(i, "x"),
                               par_param_ids=_get(i, "x")) for _ in range(n)]
        prod_slots, prod_rows = _get(i, "x"), _get(i, "x")
        (n,) = i.ints(1)
        pushes = [FlowPushIR(rows=_get(i, "x"), children=_get(i, "x")) for _ in range(n)]
        edges = {k: _get(i, "x") for k in ("edge_sums", "edge_children", "edge_slots")}
        rep = dict(zip(_REPORT_INTS, i.ints(len(_REPORT_INTS))))
        sum_pad, prod_pad = i.floats(2)
        fcaps = tuple(int(v) for v in _get(i, "x"))
        bcaps = tuple(int(v) for v in _get(i, "x"))
        report = LayerReport(depth=depth, k_m=k_m, k_n=k_n, demoted=bool(rep.pop("demoted")),
                             sum_pad_fraction=sum_pad, prod_pad_fraction=prod_pad,
                             fwd_capacities=fcaps, bwd_capacities=bcaps, **rep)
        layers.append(SumLayerIR(depth=depth, k_m=k_m, k_n=k_n, scratch_window=window,
                                 prod_evals=evals, fwd_groups=fwd, bwd_groups=bwd,
                                 prod_slots=prod_slots, prod_rows=prod_rows, pushes=pushes,
                                 report=report, **edges))
    if i.pos != len(i.mv):
        raise FormatError("trailing bytes after compiled cache payload")
    return CompiledCircuit(graph_hash=graph_hash, config=cfg, input_layer=chunks,
                           layers=layers, **fields)


def save_compiled(c: CompiledCircuit, path) -> None:
    with open(path, "wb") as f:
        write_compiled(c, f)


def load_compiled(path, expect_hash: str | None = None) -> CompiledCircuit:
    """Load a PCCF file; with ``expect_hash`` the cache must belong to that
    circuit (``cache.py:379-393``: a stale cache is a FormatError)."""
    p = Path(path)
    if not p.exists():
        raise FormatError(f"compiled cache not found: {p}")
    c = loads_compiled(p.read_bytes())
    if expect_hash is not None and c.graph_hash != expect_hash:
        raise FormatError("compiled cache does not match the circuit "
                          f"(cache {c.graph_hash[:12]}, circuit {expect_hash[:12]})")
    return c
