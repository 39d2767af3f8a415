"""Circuit -> layered block-sparse program (bit-exact layout contract).

Restates ``pcirc/compiler/build.py:183-631`` with
whole-layer numpy operations so BASELINE-scale circuits compile in
seconds-to-minutes instead of hours:

* depths per segment (``graph.depths``) instead of per node;
* per-layer edge arrays gathered from segment matrices;
* pmf / tile / simplex-group dedupe through hashed row grouping with exact
  verification (``_rows.py``) instead of ``dict[bytes]``;
* contention replicas, product rows and pushes computed per column / per
  layer with cumulative sums instead of nested Python loops.

Every ordering decision (dict-insertion order, ``np.unique`` / ``lexsort``
order, first-sight row allocation) is reproduced; ``tests/test_compile_parity.py``
checks array-for-array equality against the reference compiler and the
committed golden fixtures.
"""
from __future__ import annotations

import hashlib
import threading
from dataclasses import dataclass

import numpy as np

from ..errors import CircuitValidationError, UsageError
from ..graph import KIND_INPUT, KIND_PRODUCT, KIND_SUM, CircuitGraph
from . import _native
from ._rows import group_matrix_rows, group_rows, row_hashes
from .blocks import PAD, BlockLayout, detect_blocks_csr
from .ir import (BackwardGroupIR, CompiledCircuit, FlowPushIR, ForwardGroupIR,
                 GraphLayer, InputLayerIR, LayerReport, ProductEvalIR, SumLayerIR)
from .partition import partition_layer

_ALLOWED_K = (1, 2, 4, 8, 16, 32, 64)
_VKEY_BASE = -2  # input child i of a sum becomes pseudo-product key -2 - i


@dataclass(frozen=True)
class CompileConfig:
    """Block / grouping / tying knobs (``build.py:58-100``)."""

    block_size: int = 32
    sum_block_size: int | None = None
    prod_block_size: int | None = None
    max_groups: int = 8
    tolerance: float = 0.25
    round_quantum: int = 10
    round_threshold: int = 256
    contention_threshold: int = 4
    demote_threshold: float = 0.5

    def __post_init__(self):
        for name in ("block_size", "sum_block_size", "prod_block_size"):
            val = getattr(self, name)
            if val is not None and val not in _ALLOWED_K:
                raise UsageError(f"{name} must be a power of two in {_ALLOWED_K}, got {val}")
        if self.max_groups < 1:
            raise UsageError(f"max_groups must be >= 1, got {self.max_groups}")
        if self.tolerance < 0:
            raise UsageError(f"tolerance must be >= 0, got {self.tolerance}")
        if self.round_quantum < 1:
            raise UsageError(f"round_quantum must be >= 1, got {self.round_quantum}")
        if self.contention_threshold < 1:
            raise UsageError(
                f"contention_threshold must be >= 1, got {self.contention_threshold}")
        if not 0.0 <= self.demote_threshold <= 1.0:
            raise UsageError(
                f"demote_threshold must lie in [0, 1], got {self.demote_threshold}")

    @property
    def k_m(self) -> int:
        return self.block_size if self.sum_block_size is None else self.sum_block_size

    @property
    def k_n(self) -> int:
        return self.block_size if self.prod_block_size is None else self.prod_block_size


def node_depths(g: CircuitGraph) -> np.ndarray:
    return _as_graph(g).depths()


def layerize(g: CircuitGraph) -> list[GraphLayer]:
    g = _as_graph(g)
    depth = g.depths()
    kinds = g.node_kinds()
    names = {KIND_INPUT: "input", KIND_PRODUCT: "product", KIND_SUM: "sum"}
    key = depth * 3 + kinds
    out = []
    for k in np.unique(key):
        ids = np.flatnonzero(key == k)
        out.append(GraphLayer(int(k // 3), names[int(k % 3)], ids.astype(np.int64)))
    return out


def _as_graph(g) -> CircuitGraph:
    return g if isinstance(g, CircuitGraph) else CircuitGraph.from_reference(g)


def _tying_reps(num_slots: int, tying: dict) -> np.ndarray:
    """Representative slot = smallest slot of its tying group (``build.py:135-156``)."""
    rep = np.arange(num_slots, dtype=np.int64)
    if tying:
        items = np.array(sorted(tying.items()), dtype=np.int64).reshape(-1, 2)
        slots, groups = items[:, 0], items[:, 1]
        ug, inv = np.unique(groups, return_inverse=True)
        gmin = np.full(ug.size, np.iinfo(np.int64).max, dtype=np.int64)
        np.minimum.at(gmin, inv.ravel(), slots)
        rep[slots] = gmin[inv.ravel()]
    return rep


class _Layer:
    """Per-layer working set (pass 1 -> pass 3)."""

    __slots__ = ("depth", "sids", "e_sum", "e_key", "e_slot", "off", "lo",
                 "pair_codes", "pair_theta", "pair_sb", "pair_pb", "n_pb", "blk_slots",
                 "e_child", "nat")

    def __init__(self):
        self.e_sum = self.e_child = self.nat = None


def _collect_layers(g: CircuitGraph, depth: np.ndarray, kinds: np.ndarray):
    by_depth: dict[int, list] = {}
    for s in g.segments:
        if s.kind != KIND_SUM:
            continue
        d = depth[s.start:s.stop]
        for dv in np.unique(d).tolist():
            rows = np.flatnonzero(d == dv)
            by_depth.setdefault(dv, []).append((s, rows))
    layers = []
    for dv in sorted(by_depth):
        sids, chs, sls, cnts = [], [], [], []
        for s, rows in by_depth[dv]:
            ch = np.asarray(s.children)[rows]
            sids.append(s.start + rows)
            chs.append(ch.ravel())
            sls.append(np.asarray(s.slots)[rows].ravel())
            cnts.append(np.full(rows.size, ch.shape[1], dtype=np.int64))
        L = _Layer()
        L.depth = dv
        L.sids = np.concatenate(sids).astype(np.int64)
        child = np.concatenate(chs).astype(np.int64)
        counts = np.concatenate(cnts)
        if np.any(np.diff(L.sids) <= 0):  # segments out of id order (from_parts)
            order = np.argsort(L.sids, kind="stable")
            offs = np.concatenate([[0], np.cumsum(counts)])
            idx = np.concatenate([np.arange(offs[i], offs[i + 1]) for i in order])
            L.sids, counts = L.sids[order], counts[order]
            child = child[idx]
            slot = np.concatenate(sls)[idx]
        else:
            slot = np.concatenate(sls)
        L.e_key = np.where(kinds[child] == KIND_PRODUCT, child, _VKEY_BASE - child)
        L.e_slot = slot.astype(np.int64)
        L.e_sum = np.repeat(L.sids, counts)
        L.off = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
        layers.append(L)
    return layers


def _collect_layers_native(g: CircuitGraph, depth: np.ndarray, kinds: np.ndarray):
    """``_collect_layers`` with the per-edge arrays written by one native pass
    per layer (segments in id order, so sum ids ascend)."""
    nat = _native.lib()
    by_depth: dict[int, list] = {}
    segs = [s for s in g.segments if s.kind == KIND_SUM and s.count]
    if segs:
        st = np.array([s.start for s in segs], dtype=np.int64)
        cn = np.array([s.count for s in segs], dtype=np.int64)
        idx = _ranges_index(st, cn)
        firsts = np.concatenate([[0], np.cumsum(cn)[:-1]])
        dmin = np.minimum.reduceat(depth[idx], firsts)
        dmax = np.maximum.reduceat(depth[idx], firsts)
        for i, s in enumerate(segs):
            if dmin[i] == dmax[i]:
                by_depth.setdefault(int(dmin[i]), []).append((s, None))
                continue
            d = depth[s.start:s.stop]
            for dv in np.unique(d).tolist():
                by_depth.setdefault(dv, []).append((s, np.flatnonzero(d == dv).astype(np.int64)))
    kinds8 = np.ascontiguousarray(kinds, dtype=np.int8)
    layers = []
    for dv in sorted(by_depth):
        parts = sorted(by_depth[dv], key=lambda t: t[0].start)
        chv = [_native.rows(s.children) for s, _ in parts]
        chs = [c for c, _ in chv]
        ch_stride = np.array([st for _, st in chv], dtype=np.int64)
        sls = [_native.i64(s.slots) for s, _ in parts]
        fan = np.array([s.fan_in for s, _ in parts], dtype=np.int64)
        nrows = np.array([s.count if r is None else r.size for s, r in parts], dtype=np.int64)
        rows = [r for _, r in parts]
        L = _Layer()
        L.depth = dv
        L.sids = np.concatenate([np.arange(s.start, s.stop, dtype=np.int64) if r is None
                                 else s.start + r for s, r in parts])
        counts = np.repeat(fan, nrows)
        L.off = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
        E = int(L.off[-1])
        starts = np.array([s.start for s, _ in parts], dtype=np.int64)
        L.e_sum, L.e_child, L.e_key, L.e_slot = (np.empty(E, np.int64) for _ in range(4))
        ch_tab = _native.addr_array([_native.addr(c) for c in chs])
        nat.pcc_gather_layer(len(parts), _native.ptr(ch_tab), _native.ptr(ch_stride),
                             _native.ptr_array(sls),
                             _native.ptr(fan), _native.ptr_array(rows), _native.ptr(nrows),
                             _native.ptr(starts), _native.ptr(kinds8), KIND_PRODUCT, _VKEY_BASE,
                             _native.ptr(L.e_sum), _native.ptr(L.e_child), _native.ptr(L.e_key),
                             _native.ptr(L.e_slot))
        layers.append(L)
    return layers


def _blocks_native(L, cfg) -> BlockLayout:
    """``detect_blocks_csr`` through the native layer object (kept on ``L`` for
    the tile pass)."""
    z = np.zeros(0, dtype=np.int64)
    if L.sids.size == 0:
        return BlockLayout(1, 1, False, np.zeros((0, 1), np.int64), np.zeros((0, 1), np.int64),
                           z, np.zeros(1, np.int64), z, z, z, z, z, z, 0.0, 0.0)
    L.nat = _native.Layer(L.sids, L.e_key, L.off)
    km, kn, dem, spad, ppad, a = L.nat.blocks(cfg.k_m, cfg.k_n, cfg.demote_threshold)
    return BlockLayout(km, kn, dem, a["smat"], a["pmat"], a["cb_flat"], a["cb_off"],
                       a["sum_keys"], a["sum_blk"], a["sum_off"], a["prod_keys"],
                       a["prod_blk"], a["prod_off"], spad, ppad)


def _lookup(keys_sorted, vals_a, vals_b, query):
    idx = np.searchsorted(keys_sorted, query)
    return vals_a[idx], vals_b[idx]


def _scatter_rows(row_ids, lens, cols_vals, nrows, cap):
    """Fill a (nrows, cap) zero matrix: row r gets lens[r] values from cols_vals."""
    out = np.zeros((nrows, cap), dtype=np.int64)
    if cols_vals.size:
        r = np.repeat(np.arange(nrows), lens)
        c = np.arange(cols_vals.size) - np.repeat(np.concatenate([[0], np.cumsum(lens)[:-1]]), lens)
        out[r, c] = cols_vals
    return out


class _TileTable:
    """Global tile dedupe keyed by tied-slot pattern (``build.py:312-326``)."""

    def __init__(self):
        self.by_hash: dict[tuple, list] = {}

    def find(self, tilesz: int, h: int, pattern: np.ndarray):
        for start, ref in self.by_hash.get((tilesz, h), ()):
            if np.array_equal(ref, pattern):
                return start
        return None

    def add(self, tilesz: int, h: int, pattern: np.ndarray, start: int):
        self.by_hash.setdefault((tilesz, h), []).append((start, pattern))


def compile_circuit(g, cfg: CompileConfig | None = None, *, validate: bool = True
                    ) -> CompiledCircuit:
    """Compile a circuit into index tensors; deterministic given (g, cfg)."""
    cfg = cfg or CompileConfig()
    g = _as_graph(g)
    if validate:
        g.validate().raise_if_invalid()
    g.freeze()
    if _native.lib() is not None:
        try:
            return _compile(g, cfg, True)
        except _native.NativeError:
            pass  # the numpy path raises the reference's exact error
    return _compile(g, cfg, False)


def _compile(g: CircuitGraph, cfg: CompileConfig, native: bool) -> CompiledCircuit:
    ghash = _hash_async(g) if native else (lambda: graph_hash(g, False))
    params = g.params
    depth = g.depths()
    kinds = g.node_kinds()
    root = g.root
    in_ids, in_var, in_ncat, in_slot = g.input_table()
    n_nodes = g.num_nodes

    # -- pass 1: block layouts per sum layer -------------------------------
    if native:
        layers = _collect_layers_native(g, depth, kinds)
        for L in layers:
            L.lo = _blocks_native(L, cfg)
    else:
        layers = _collect_layers(g, depth, kinds)
        for L in layers:
            L.lo = detect_blocks_csr(L.sids, L.e_key, L.off, cfg.k_m, cfg.k_n,
                                     cfg.demote_threshold)
    reserved = max([L.lo.k_m for L in layers] or [1])

    # -- value slots ---------------------------------------------------------
    node_value_slot = np.full(n_nodes, -1, dtype=np.int64)
    node_value_slot[in_ids] = reserved + np.arange(in_ids.size, dtype=np.int64)
    next_slot = reserved + in_ids.size
    for L in layers:
        lo = L.lo
        n_sb = lo.sum_block_mat.shape[0]
        L.blk_slots = next_slot + lo.k_m * np.arange(n_sb, dtype=np.int64)
        real = lo.sum_block_mat != PAD
        pos = L.blk_slots[:, None] + np.arange(lo.k_m)[None, :]
        node_value_slot[lo.sum_block_mat[real]] = pos[real]
        next_slot += lo.k_m * n_sb
    num_value_slots = int(next_slot)

    # -- physical parameter layout ------------------------------------------
    # native: no identity rep array for untied circuits, ranges instead of
    # per-position input arrays (written into theta / slot_phys by the core)
    rep = _tying_reps(g.num_param_slots, g.tying) if (g.tying or not native) else None
    zero_len = max([L.lo.k_m * L.lo.k_n for L in layers] or [1])
    theta_parts = [np.zeros(zero_len)]
    theta_size = zero_len
    slot_phys = (_native.full_i64(g.num_param_slots, -1) if native
                 else np.full(g.num_param_slots, -1, dtype=np.int64))
    assigned: list[tuple[np.ndarray, np.ndarray]] = []
    in_copy = in_assign = None

    pmf_phys_of = np.full(n_nodes, -1, dtype=np.int64)
    if in_ids.size:
        tied_inputs = bool(g.tying) and _ranges_touch_tying(in_slot, in_ncat, rep)
        if tied_inputs:
            offs = np.concatenate([[0], np.cumsum(in_ncat)])
            flat = rep[np.repeat(in_slot, in_ncat) + (np.arange(int(offs[-1])) -
                                                      np.repeat(offs[:-1], in_ncat))]
            gid, first = group_rows(flat, offs)
        else:
            # untied: the pattern rep[slot:slot+ncat] is the range itself
            key = np.stack([in_slot, in_ncat], axis=1)
            gid, first = group_matrix_rows(key)
        first_ncat = in_ncat[first]
        gstart = theta_size + np.concatenate([[0], np.cumsum(first_ncat)[:-1]])
        if native:
            in_copy = (in_slot[first], first_ncat, gstart)
        else:
            for j, i in enumerate(first.tolist()):
                theta_parts.append(params[in_slot[i]:in_slot[i] + in_ncat[i]].copy())
        theta_size += int(first_ncat.sum())
        starts = gstart[gid]
        pmf_phys_of[in_ids] = starts
        # expand each distinct (slot range, pmf) pairing once: inputs that share
        # slots (tied HMM emissions) would otherwise repeat identical writes
        _, ufirst = np.unique(np.stack([in_slot, in_ncat, starts], axis=1), axis=0,
                              return_index=True)
        ufirst = np.sort(ufirst)
        o = np.argsort(in_slot[ufirst], kind="stable")
        s_sorted, n_sorted = in_slot[ufirst][o], in_ncat[ufirst][o]
        overlap = bool(np.any(s_sorted[1:] < s_sorted[:-1] + n_sorted[:-1]))
        if overlap:
            ufirst = np.arange(in_ids.size)  # overlapping ranges: keep write order exact
        u_slot, u_ncat, u_start = in_slot[ufirst], in_ncat[ufirst], starts[ufirst]
        if native:
            in_assign = (u_slot, u_ncat, u_start, overlap)
        else:
            rng_off = np.arange(int(u_ncat.sum())) - np.repeat(np.cumsum(u_ncat) - u_ncat, u_ncat)
            rng_phys = np.repeat(u_start, u_ncat) + rng_off
            rng_slots = np.repeat(u_slot, u_ncat) + rng_off
            slot_phys[rng_slots] = rng_phys
            assigned.append((rng_slots, rng_phys))

    if native:
        theta, theta_size, tile_starts, tile_writers = _tiles_native(
            g, layers, rep, params, zero_len, theta_size, slot_phys, in_copy, in_assign)
    else:
        theta, theta_size, tile_starts, tile_writers = _tiles_numpy(
            g, layers, rep, params, theta_parts, theta_size, slot_phys, assigned)
    del assigned
    return _finish(g, cfg, layers, kinds, depth, root, in_ids, in_var, in_ncat, n_nodes,
                   reserved, node_value_slot, num_value_slots, zero_len, theta, theta_size,
                   slot_phys, pmf_phys_of, tile_starts, tile_writers, native, ghash)


def _tiles_native(g, layers, rep, params, zero_len, theta_size, slot_phys, in_copy, in_assign):
    """build.py:251-339 through the native core: the input pmfs' theta ranges
    and slot_phys, then per layer ``pcc_tiles`` (tile grids, the tied pattern
    dedupe, theta fill, slot_phys) with the tying-alignment check."""
    nat = _native.lib()
    ptr = _native.ptr
    tied = bool(g.tying)
    share = tied or getattr(g, "shares_slots", True)
    rep_arg = _native.i64(rep) if tied else None
    nslots = int(g.num_param_slots)
    params = np.ascontiguousarray(params, dtype=np.float64)
    multi = ref = None
    if share:
        seen = np.zeros((nslots + 63) // 64 + 1, np.uint64)
        multi = np.zeros_like(seen)
        for L in layers:
            nat.pcc_slot_uses(L.e_slot.size, ptr(L.e_slot), ptr(rep_arg), ptr(seen), ptr(multi))
        del seen
        ref = _native.full_i64(nslots, -1)
    cap = theta_size + sum(int(L.lo.cb_flat.size) * L.lo.k_m * L.lo.k_n for L in layers)
    buf = np.empty(max(cap, 1), dtype=np.float64)  # untouched pages stay unallocated
    buf[:zero_len] = 0.0
    if in_copy is not None:
        src, ln, dst = (_native.i64(a) for a in in_copy)
        nat.pcc_copy_ranges(src.size, ptr(src), ptr(ln), ptr(dst), ptr(params), ptr(buf))
    if in_assign is not None:
        us, un, ust = (_native.i64(a) for a in in_assign[:3])
        if nat.pcc_assign_ranges(us.size, ptr(us), ptr(un), ptr(ust), int(in_assign[3]),
                                 ptr(slot_phys), ptr(rep_arg), ptr(ref)):
            raise _native.NativeError("tying")
    ts = np.array([theta_size], dtype=np.int64)
    table = nat.pcc_tiles_new()
    try:
        for L in layers:
            lo = L.lo
            n_sb, n_pb = lo.sum_block_mat.shape[0], lo.prod_block_mat.shape[0]
            pair_theta = np.empty(lo.cb_flat.size, dtype=np.int64)
            if L.nat is not None:
                rc = nat.pcc_tiles(L.nat.h, table, ptr(L.e_slot), ptr(rep_arg), ptr(multi),
                                   ptr(params), ptr(buf), cap, ptr(ts), ptr(slot_phys), ptr(ref),
                                   ptr(pair_theta))
                L.nat.free()
                L.nat = None
                if rc != 0:
                    raise _native.NativeError(f"tiles rc={rc}")
            L.pair_theta = pair_theta
            L.pair_sb = np.repeat(np.arange(n_sb, dtype=np.int64), np.diff(lo.cb_off))
            L.pair_pb = lo.cb_flat
            L.pair_codes = L.pair_sb * n_pb + L.pair_pb
            L.n_pb = n_pb
        nt = int(nat.pcc_tiles_count(table))
        tile_starts = np.empty(nt, dtype=np.int64)
        tile_writers = np.empty(nt, dtype=np.int64)
        nat.pcc_tiles_get(table, ptr(tile_starts), ptr(tile_writers))
    finally:
        nat.pcc_tiles_free(table)
        nat.pcc_release()
    theta_size = int(ts[0])
    return buf[:theta_size], theta_size, tile_starts, tile_writers


def _tiles_numpy(g, layers, rep, params, theta_parts, theta_size, slot_phys, assigned):
    tiles = _TileTable()
    writer_count: dict[int, int] = {}
    for L in layers:
        lo = L.lo
        km, kn = lo.k_m, lo.k_n
        tilesz = km * kn
        n_pb = lo.prod_block_mat.shape[0]
        e_sb, e_so = _lookup(lo.sum_keys, lo.sum_blk, lo.sum_off, L.e_sum)
        e_pb, e_po = _lookup(lo.prod_keys, lo.prod_blk, lo.prod_off, L.e_key)
        codes = e_sb * n_pb + e_pb
        pair_codes = np.unique(codes)
        pair_idx = np.searchsorted(pair_codes, codes)
        toff = e_so * kn + e_po
        flat = pair_idx * tilesz + toff
        cnt = np.bincount(flat)
        if cnt.max(initial=0) > 1:
            dup = int(L.e_sum[np.flatnonzero(cnt[flat] > 1)[0]])
            raise CircuitValidationError(
                f"sum node {dup} has parallel edges to one child; merge their "
                "weights before compiling")
        grids = np.full((pair_codes.size, tilesz), -1, dtype=np.int64)
        grids[pair_idx, toff] = L.e_slot
        mask = grids >= 0
        grid_rep = np.where(mask, rep[np.where(mask, grids, 0)], -1)
        lgid, lfirst = group_matrix_rows(grid_rep)
        hashes = row_hashes(grid_rep[lfirst])
        gstart = np.empty(lfirst.size, dtype=np.int64)
        new_rows = []
        for j, p in enumerate(lfirst.tolist()):
            h = int(hashes[j])
            start = tiles.find(tilesz, h, grid_rep[p])
            if start is None:
                start = theta_size
                tiles.add(tilesz, h, grid_rep[p], start)
                new_rows.append(p)
                theta_size += tilesz
            gstart[j] = start
        if new_rows:
            nr = np.asarray(new_rows)
            vals = np.where(mask[nr], params[np.where(mask[nr], grids[nr], 0)], 0.0)
            theta_parts.append(vals.ravel())
        pair_theta = gstart[lgid]
        ut, uc = np.unique(pair_theta, return_counts=True)
        for t, c in zip(ut.tolist(), uc.tolist()):
            writer_count[t] = writer_count.get(t, 0) + c
        phys = pair_theta[pair_idx] + toff
        slot_phys[L.e_slot] = phys
        assigned.append((L.e_slot, phys))
        L.pair_codes = pair_codes
        L.pair_theta = pair_theta
        L.pair_sb = pair_codes // n_pb
        L.pair_pb = pair_codes % n_pb
        L.n_pb = n_pb

    theta = np.concatenate(theta_parts)
    if g.tying or getattr(g, "shares_slots", True):
        _check_tying_alignment(rep, assigned)
    tile_starts = np.array(sorted(writer_count), dtype=np.int64)
    tile_writers = np.array([writer_count[t] for t in tile_starts.tolist()], dtype=np.int64)
    return theta, theta_size, tile_starts, tile_writers


def _finish(g, cfg, layers, kinds, depth, root, in_ids, in_var, in_ncat, n_nodes, reserved,
            node_value_slot, num_value_slots, zero_len, theta, theta_size, slot_phys,
            pmf_phys_of, tile_starts, tile_writers, native, ghash):
    # -- groups, product evaluation, flow bookkeeping ---------------------------
    prod_ch_off, prod_ch_flat = _product_children(g, n_nodes)
    node_prod_row = np.full(n_nodes, -1, dtype=np.int64)
    push_done = np.zeros(n_nodes, dtype=bool)
    num_prod_rows = 0
    scratch_size = 1
    out_layers: list[SumLayerIR] = []
    for L in layers:
        lo = L.lo
        km, kn = lo.k_m, lo.k_n
        n_pb = L.n_pb
        prod_scratch = (1 + np.arange(n_pb, dtype=np.int64)) * kn
        window = int((1 + n_pb) * kn)
        scratch_size = max(scratch_size, window)

        nchs = np.diff(lo.cb_off)
        plan = partition_layer(nchs, cfg.max_groups, cfg.tolerance,
                               cfg.round_quantum, cfg.round_threshold)
        # theta start of every (sum block, child block) entry in cb order
        sb_rep = np.repeat(np.arange(nchs.size), nchs)
        cb_theta = L.pair_theta[np.searchsorted(L.pair_codes, sb_rep * n_pb + lo.cb_flat)]
        fwd_groups = []
        for gi in range(plan.num_groups):
            rows = np.flatnonzero(plan.assignment == gi)
            cap = plan.capacities[gi]
            lens = nchs[rows]
            sel = np.concatenate([np.arange(lo.cb_off[r], lo.cb_off[r + 1]) for r in rows]) \
                if rows.size else np.zeros(0, np.int64)
            sel = sel.astype(np.int64)
            prod_ids = _scatter_rows(rows, lens, prod_scratch[lo.cb_flat[sel]], rows.size, cap)
            param_ids = _scatter_rows(rows, lens, cb_theta[sel], rows.size, cap)
            fwd_groups.append(ForwardGroupIR(sum_ids=L.blk_slots[rows], prod_ids=prod_ids,
                                             param_ids=param_ids, flow_ids=param_ids.copy()))

        npar = np.bincount(L.pair_pb, minlength=n_pb)
        bplan = partition_layer(npar, cfg.max_groups, cfg.tolerance,
                                cfg.round_quantum, cfg.round_threshold)
        psort = np.lexsort((L.pair_sb, L.pair_pb))
        poff = np.concatenate([[0], np.cumsum(npar)])
        bwd_groups = []
        for gi in range(bplan.num_groups):
            rows = np.flatnonzero(bplan.assignment == gi)
            cap = bplan.capacities[gi]
            lens = npar[rows]
            sel = psort[np.concatenate([np.arange(poff[r], poff[r + 1]) for r in rows])] \
                if rows.size else np.zeros(0, np.int64)
            sel = sel.astype(np.int64)
            par_ids = _scatter_rows(rows, lens, L.blk_slots[L.pair_sb[sel]], rows.size, cap)
            par_param_ids = _scatter_rows(rows, lens, L.pair_theta[sel], rows.size, cap)
            bwd_groups.append(BackwardGroupIR(ch_ids=prod_scratch[rows], par_ids=par_ids,
                                              par_param_ids=par_param_ids))

        # product evaluation / flow rows / pushes (build.py:427-475)
        pflat = lo.prod_block_mat.ravel()
        valid = np.flatnonzero(pflat != PAD)
        keys = pflat[valid]
        outs = kn + valid
        is_real = keys >= 0
        rkeys = keys[is_real]
        need_new = ~is_real
        need_new[is_real] = node_prod_row[rkeys] < 0
        new_rows = num_prod_rows + np.cumsum(need_new) - 1
        rows_l = np.empty(keys.size, dtype=np.int64)
        rows_l[need_new] = new_rows[need_new]
        num_prod_rows += int(need_new.sum())
        real_new = is_real & need_new
        node_prod_row[keys[real_new]] = rows_l[real_new]
        old = is_real & ~need_new
        rows_l[old] = node_prod_row[keys[old]]
        do_push = np.ones(keys.size, dtype=bool)
        do_push[is_real] = ~push_done[rkeys]
        push_done[rkeys] = True
        fan = np.ones(keys.size, dtype=np.int64)
        fan[is_real] = prod_ch_off[rkeys + 1] - prod_ch_off[rkeys]
        prod_evals, pushes = [], []
        for f in np.unique(fan).tolist():
            m = np.flatnonzero(fan == f)
            ch = np.empty((m.size, f), dtype=np.int64)
            mr = is_real[m]
            if mr.any():
                kk = keys[m[mr]]
                ch[mr] = node_value_slot[prod_ch_flat[prod_ch_off[kk][:, None] + np.arange(f)]]
            if (~mr).any():
                ch[~mr, 0] = node_value_slot[_VKEY_BASE - keys[m[~mr]]]
            prod_evals.append(ProductEvalIR(out=outs[m].astype(np.int64), children=ch))
            pm = do_push[m]
            if pm.any():
                pushes.append(FlowPushIR(rows=rows_l[m[pm]], children=ch[pm]))

        e_child = L.e_child if L.e_child is not None else \
            np.where(L.e_key >= 0, L.e_key, _VKEY_BASE - L.e_key)
        if L.e_sum is None:
            L.e_sum = np.repeat(L.sids, np.diff(L.off))
        report = LayerReport(
            depth=L.depth, num_sums=int(L.sids.size), num_prods=int(keys.size),
            k_m=km, k_n=kn, demoted=lo.demoted,
            sum_pad_fraction=lo.sum_pad_fraction, prod_pad_fraction=lo.prod_pad_fraction,
            fwd_capacities=plan.capacities, fwd_overhead=plan.overhead,
            fwd_target=plan.target, fwd_ideal=int(nchs.sum()),
            bwd_capacities=bplan.capacities, bwd_overhead=bplan.overhead,
            bwd_target=bplan.target, bwd_ideal=int(npar.sum()))
        out_layers.append(SumLayerIR(
            depth=L.depth, k_m=km, k_n=kn, scratch_window=window,
            prod_evals=prod_evals, fwd_groups=fwd_groups, bwd_groups=bwd_groups,
            prod_slots=outs.astype(np.int64), prod_rows=rows_l,
            pushes=pushes, edge_sums=L.e_sum, edge_children=e_child,
            edge_slots=L.e_slot, report=report))
        # release pass-1 working arrays
        L.e_sum = L.e_key = L.e_slot = L.e_child = None

    # -- contention replicas (build.py:516-533) -----------------------------
    f_params_size = theta_size
    reductions = []
    for layer in out_layers:
        tilesz = layer.k_m * layer.k_n
        for gr in layer.fwd_groups:
            for c in range(gr.param_ids.shape[1]):
                t = gr.param_ids[:, c]
                nz = t != 0
                if not nz.any():
                    continue
                w = np.zeros(t.size, dtype=np.int64)
                w[nz] = tile_writers[np.searchsorted(tile_starts, t[nz])]
                first = np.zeros(t.size, dtype=bool)
                nzi = np.flatnonzero(nz)
                _, fi = np.unique(t[nzi], return_index=True)
                first[nzi[fi]] = True
                rep_rows = np.flatnonzero(nz & ((w > cfg.contention_threshold) | ~first))
                if rep_rows.size:
                    new_ids = f_params_size + tilesz * np.arange(rep_rows.size, dtype=np.int64)
                    reductions.append(np.stack(
                        [new_ids, t[rep_rows], np.full(rep_rows.size, tilesz)], axis=1))
                    gr.flow_ids[rep_rows, c] = new_ids
                    f_params_size += tilesz * rep_rows.size

    # -- simplex groups (build.py:535-567) -------------------------------------
    group_idx, group_off = _simplex_groups(g, pmf_phys_of, slot_phys, theta_size, native)

    # -- input chunks by category count ----------------------------------------
    input_layer = []
    for ncat in np.unique(in_ncat).tolist():
        m = in_ncat == ncat
        ids = in_ids[m]
        input_layer.append(InputLayerIR(node_ids=ids, slots=node_value_slot[ids],
                                        vars=in_var[m], param_ids=pmf_phys_of[ids],
                                        num_categories=int(ncat)))

    # -- root --------------------------------------------------------------------
    if kinds[root] == KIND_PRODUCT:
        root_row = num_prod_rows
        num_prod_rows += 1
        node_prod_row[root] = root_row
        root_slot = -1
        root_children = node_value_slot[prod_ch_flat[prod_ch_off[root]:prod_ch_off[root + 1]]]
    else:
        root_row = -1
        root_slot = int(node_value_slot[root])
        root_children = None

    return CompiledCircuit(
        graph_hash=ghash(), config=cfg, num_vars=g.num_vars, num_nodes=n_nodes,
        var_categories=g.var_categories(), reserved=int(reserved),
        num_value_slots=num_value_slots, scratch_size=int(scratch_size),
        num_prod_rows=int(num_prod_rows), theta_size=int(theta_size),
        f_params_size=int(f_params_size), zero_len=int(zero_len), theta=theta,
        slot_phys=slot_phys,
        reductions=(np.concatenate(reductions) if reductions
                    else np.zeros((0, 3), dtype=np.int64)).astype(np.int64),
        tile_starts=tile_starts, tile_writers=tile_writers,
        group_idx=group_idx, group_off=group_off, input_layer=input_layer,
        layers=out_layers, root_slot=root_slot, root_children=root_children,
        root_row=int(root_row), node_value_slot=node_value_slot,
        node_prod_row=node_prod_row)


def _ranges_touch_tying(in_slot, in_ncat, rep) -> bool:
    tied = rep != np.arange(rep.size)
    if not tied.any():
        return False
    cs = np.concatenate([[0], np.cumsum(tied)])
    return bool(np.any(cs[in_slot + in_ncat] - cs[in_slot] > 0)) or _rep_points_into(rep, in_slot, in_ncat)


def _rep_points_into(rep, in_slot, in_ncat) -> bool:
    # some other slot's representative lies inside an input range
    targets = np.unique(rep[rep != np.arange(rep.size)])
    if targets.size == 0:
        return False
    lo = np.searchsorted(targets, in_slot)
    hi = np.searchsorted(targets, in_slot + in_ncat)
    return bool(np.any(hi > lo))


def _check_tying_alignment(rep, assigned):
    """Every use of one tied group must land on one physical position (``build.py:343-359``)."""
    if not assigned:
        return
    ref = np.full(rep.size, -1, dtype=np.int64)
    bad = False
    for slots, phys in assigned:
        r = rep[slots]
        prev = ref[r]
        bad |= bool(np.any((prev >= 0) & (prev != phys)))
        ref[r] = phys
        bad |= bool(np.any(ref[r] != phys))
        if bad:
            break
    if not bad:
        return
    all_slots = np.concatenate([a for a, _ in assigned])
    all_phys = np.concatenate([b for _, b in assigned])
    order = np.argsort(rep[all_slots], kind="stable")
    ru, pu = rep[all_slots][order], all_phys[order]
    starts = np.r_[0, np.nonzero(np.diff(ru))[0] + 1]
    mins = np.minimum.reduceat(pu, starts)
    maxs = np.maximum.reduceat(pu, starts)
    badg = np.nonzero(mins != maxs)[0]
    raise CircuitValidationError(
        f"parameter tying of slot group {int(ru[starts[badg[0]]])} does not align "
        "with the compiled block layout; compile with block size 1")


def _product_children(g: CircuitGraph, n_nodes: int):
    """CSR of product children over all node ids (empty rows for non-products)."""
    fan = np.zeros(n_nodes, dtype=np.int64)
    segs = [s for s in g.segments if s.kind == KIND_PRODUCT]
    for s in segs:
        fan[s.start:s.stop] = s.fan_in
    off = np.concatenate([[0], np.cumsum(fan)]).astype(np.int64)
    flat = np.empty(int(off[-1]), dtype=np.int64)
    for s in segs:
        flat[off[s.start]:off[s.stop]] = np.asarray(s.children).ravel()
    return off, flat


def _simplex_groups(g: CircuitGraph, pmf_phys_of, slot_phys, theta_size, native=False):
    """Normalisation groups over physical positions, first-occurrence order."""
    fast = _simplex_groups_disjoint(g, pmf_phys_of, slot_phys, theta_size, native)
    if fast is not None:
        return fast
    if native:
        return _simplex_groups_general_native(g, pmf_phys_of, slot_phys, theta_size)
    return _simplex_groups_general(g, pmf_phys_of, slot_phys, theta_size)


def _simplex_groups_disjoint(g: CircuitGraph, pmf_phys_of, slot_phys, theta_size,
                             native=False):
    """Fast path when no two sums share a physical position and no sum touches a
    pmf: every sum is its own group and inputs dedupe by their pmf range, so
    the first-occurrence order is plain node-id order.  ``native``: position
    claims in a bitset and the sorted sum rows written by ``pcc_sum_groups_multi``."""
    sum_segs = [s for s in g.segments if s.kind == KIND_SUM]
    in_ids, _, in_ncat, _ = g.input_table()
    n_sum_pos = sum(s.count * s.fan_in for s in sum_segs)
    nat = _native.lib() if native else None
    if nat is not None:
        bits = np.zeros((theta_size + 63) // 64 + 1, dtype=np.uint64)
    else:
        claim = np.zeros(theta_size, dtype=np.int8)
    if in_ids.size:
        starts = pmf_phys_of[in_ids]
        key = np.stack([starts, in_ncat], axis=1)
        _, first = np.unique(key, axis=0, return_index=True)
        first = np.sort(first)
        rs, rn = starts[first], in_ncat[first]
        if nat is not None:
            rs, rn = _native.i64(rs), _native.i64(rn)
            if nat.pcc_claim_ranges(rs.size, _native.ptr(rs), _native.ptr(rn), _native.ptr(bits)):
                return None  # overlapping pmf ranges
        else:
            off = np.repeat(rs - np.concatenate([[0], np.cumsum(rn)[:-1]]), rn)
            pmf_pos = np.arange(int(rn.sum()), dtype=np.int64) + off
            claim[pmf_pos] = 1
            if int(claim.sum()) != pmf_pos.size:
                return None  # overlapping pmf ranges
    else:
        first = np.zeros(0, np.int64)
        rs = rn = np.zeros(0, np.int64)
    if nat is None:
        for s in sum_segs:
            pos = slot_phys[s.slots].ravel()
            if np.any(claim[pos]):
                return None
            claim[pos] = 1
        if int(claim.sum()) != int(rn.sum()) + n_sum_pos:
            return None  # a position shared between sums (or within one sum)
    if nat is not None:
        return _simplex_disjoint_assemble_native(nat, sum_segs, in_ids, first, rs, rn, slot_phys,
                                                 bits)
    # assemble in node-id order: input group starts and sum rows interleave
    items_id, items_kind, items_ref = [], [], []
    items_id.append(in_ids[first])
    items_kind.append(np.zeros(first.size, np.int8))
    items_ref.append(np.arange(first.size, dtype=np.int64))
    for si, s in enumerate(sum_segs):
        items_id.append(np.arange(s.start, s.stop, dtype=np.int64))
        items_kind.append(np.full(s.count, 1, np.int8))
        items_ref.append(np.arange(s.count, dtype=np.int64) + (si << 40))
    ids = np.concatenate(items_id)
    order = np.argsort(ids, kind="stable")
    kinds = np.concatenate(items_kind)[order]
    refs = np.concatenate(items_ref)[order]
    sizes = np.empty(ids.size, dtype=np.int64)
    sizes[kinds == 0] = rn[refs[kinds == 0]]
    segsz = np.array([s.fan_in for s in sum_segs], dtype=np.int64)
    sizes[kinds == 1] = segsz[refs[kinds == 1] >> 40] if sum_segs else 0
    group_off = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
    group_idx = np.empty(int(group_off[-1]), dtype=np.int64)
    # inputs: contiguous ranges
    ii = np.flatnonzero(kinds == 0)
    if ii.size:
        n = rn[refs[ii]]
        dst = np.repeat(group_off[ii], n) + (np.arange(int(n.sum())) -
                                              np.repeat(np.cumsum(n) - n, n))
        group_idx[dst] = np.repeat(rs[refs[ii]], n) + (np.arange(int(n.sum())) -
                                                       np.repeat(np.cumsum(n) - n, n))
    # sums: sorted physical slots per row, written segment by segment
    pos_of = np.full(ids.size, 0, dtype=np.int64)
    pos_of[order] = np.arange(ids.size)
    base = first.size
    for si, s in enumerate(sum_segs):
        rows = pos_of[base:base + s.count]
        base += s.count
        phys = np.sort(slot_phys[s.slots], axis=1)
        dst = group_off[rows][:, None] + np.arange(s.fan_in)
        group_idx[dst] = phys
    return group_idx, group_off


def _simplex_disjoint_assemble_native(nat, sum_segs, in_ids, first, rs, rn, slot_phys, bits):
    """The node-id-ordered assembly of ``_simplex_groups_disjoint`` with
    whole-circuit arrays (no per-segment work) and the sorted sum rows written
    by one ``pcc_sum_groups_multi`` call."""
    ptr = _native.ptr
    st = np.array([s.start for s in sum_segs], dtype=np.int64)
    cn = np.array([s.count for s in sum_segs], dtype=np.int64)
    fn = np.array([s.fan_in for s in sum_segs], dtype=np.int64)
    sum_ids = _ranges_index(st, cn)
    n_in = first.size
    ids = np.concatenate([in_ids[first], sum_ids])
    sizes = np.concatenate([rn, np.repeat(fn, cn)])
    order = np.argsort(ids, kind="stable")
    group_off = np.concatenate([[0], np.cumsum(sizes[order])]).astype(np.int64)
    pos_of = np.empty(ids.size, dtype=np.int64)
    pos_of[order] = np.arange(ids.size)
    group_idx = np.empty(int(group_off[-1]), dtype=np.int64)
    if n_in:
        dst0 = _native.i64(group_off[pos_of[:n_in]])
        rs_, rn_ = _native.i64(rs), _native.i64(rn)
        nat.pcc_iota_ranges(n_in, ptr(dst0), ptr(rs_), ptr(rn_), ptr(group_idx))
    if sum_segs:
        slots = [_native.i64(s.slots) for s in sum_segs]
        tab = _native.addr_array([_native.addr(a) for a in slots])
        dst = _native.i64(group_off[pos_of[n_in:]])
        if nat.pcc_sum_groups_multi(len(sum_segs), ptr(cn), ptr(fn), ptr(tab), ptr(slot_phys),
                                    ptr(bits), ptr(dst), ptr(group_idx)):
            return None  # a position shared between sums (or within one sum)
    return group_idx, group_off


def _ranges_index(starts, lens):
    """Concatenated ranges start[i] + [0, lens[i])."""
    lens = np.asarray(lens, dtype=np.int64)
    tot = int(lens.sum())
    return np.repeat(np.asarray(starts, dtype=np.int64) - (np.cumsum(lens) - lens), lens) + \
        np.arange(tot, dtype=np.int64)


def _simplex_groups_general_native(g: CircuitGraph, pmf_phys_of, slot_phys, theta_size):
    """``_simplex_groups_general`` with the sorted sum rows grouped by the
    native core (``pcc_rows_*``) and the overlap claims in ``pcc_claim_groups``."""
    nat = _native.lib()
    ptr = _native.ptr
    r_start, r_n, r_id = [], [], []
    in_ids, _, in_ncat, _ = g.input_table()
    if in_ids.size:
        r_start.append(pmf_phys_of[in_ids])
        r_n.append(in_ncat)
        r_id.append(in_ids)
    by_fan: dict[int, list] = {}
    for s in g.segments:
        if s.kind == KIND_SUM and s.count:
            by_fan.setdefault(s.fan_in, []).append(s)
    rg = nat.pcc_rows_new()
    try:
        for f, segs in by_fan.items():
            st = np.array([s.start for s in segs], dtype=np.int64)
            cn = np.array([s.count for s in segs], dtype=np.int64)
            slots = [_native.i64(s.slots) for s in segs]
            tab = _native.addr_array([_native.addr(a) for a in slots])
            cs = np.empty(int(cn.sum()), dtype=np.int64)
            nat.pcc_rows_add_multi(rg, len(segs), ptr(cn), f, ptr(tab), ptr(st), ptr(slot_phys),
                                   ptr(cs))
            contig = cs >= 0
            if contig.any():
                r_start.append(cs[contig])
                r_n.append(np.full(int(contig.sum()), f, np.int64))
                r_id.append(_ranges_index(st, cn)[contig])
        nm = np.zeros(1, np.int64)
        ng = int(nat.pcc_rows_count(rg, ptr(nm)))
        row_first = np.empty(ng, np.int64)
        row_off = np.empty(ng + 1, np.int64)
        row_mem = np.empty(int(nm[0]), np.int64)
        nat.pcc_rows_get(rg, ptr(row_first), ptr(row_off), ptr(row_mem))
    finally:
        nat.pcc_rows_free(rg)
    if r_start:
        rs, rn, rid = (np.concatenate(a) for a in (r_start, r_n, r_id))
        order = np.argsort(rid, kind="stable")
        key = np.stack([rs[order], rn[order]], axis=1)
        _, first = np.unique(key, axis=0, return_index=True)
        rng_id, rng_start, rng_n = rid[order][first], key[first, 0], key[first, 1]
    else:
        rng_id = rng_start = rng_n = np.zeros(0, np.int64)
    ids = np.concatenate([rng_id, row_first])
    if ids.size == 0:
        return np.zeros(0, dtype=np.int64), np.zeros(1, dtype=np.int64)
    sizes = np.concatenate([rng_n, np.diff(row_off)])
    order = np.argsort(ids, kind="stable")
    group_off = np.concatenate([[0], np.cumsum(sizes[order])]).astype(np.int64)
    pos = np.empty(ids.size, np.int64)
    pos[order] = np.arange(ids.size)
    group_idx = np.empty(int(group_off[-1]), dtype=np.int64)
    nr = rng_id.size
    if nr:
        dst, st, ln = (_native.i64(a) for a in (group_off[pos[:nr]], rng_start, rng_n))
        nat.pcc_iota_ranges(nr, ptr(dst), ptr(st), ptr(ln), ptr(group_idx))
    if ng:
        group_idx[_ranges_index(group_off[pos[nr:]], np.diff(row_off))] = row_mem
    claim = _native.full_i64(max(theta_size, 1), -1)
    if nat.pcc_claim_groups(ids.size, ptr(group_off), ptr(group_idx), ptr(claim)):
        raise CircuitValidationError(
            "normalization groups overlap after parameter tying; tie whole "
            "sum nodes (or whole pmfs), not parts of them")
    return group_idx, group_off


def _simplex_groups_general(g: CircuitGraph, pmf_phys_of, slot_phys, theta_size):
    """Exact dedupe of every node's sorted physical positions, numbered by the
    first node (in id order) that has them.  Contiguous position sets are keyed
    as (start, n) ranges (inputs' pmfs and contiguous sums share that space);
    other sum rows are grouped per fan-in with hashed row grouping."""
    cand_id, cand_kind, cand_ref = [], [], []   # kind 0: range, 1: row of fan-in table
    r_start, r_n = [], []
    rows_by_f: dict[int, list] = {}
    in_ids, _, in_ncat, _ = g.input_table()
    if in_ids.size:
        r_start.append(pmf_phys_of[in_ids])
        r_n.append(in_ncat)
        cand_id.append(in_ids)
    for s in g.segments:
        if s.kind != KIND_SUM:
            continue
        phys = np.sort(slot_phys[s.slots], axis=1)
        f = phys.shape[1]
        contig = (phys[:, -1] - phys[:, 0] == f - 1)
        if f > 1:
            contig &= np.all(np.diff(phys, axis=1) == 1, axis=1)
        ids = np.arange(s.start, s.stop, dtype=np.int64)
        if contig.any():
            r_start.append(phys[contig, 0])
            r_n.append(np.full(int(contig.sum()), f, np.int64))
            cand_id.append(ids[contig])
        if (~contig).any():
            rows_by_f.setdefault(f, []).append((ids[~contig], phys[~contig]))
    groups = []  # (first node id, member array)
    if r_start:
        rs = np.concatenate(r_start)
        rn = np.concatenate(r_n)
        rid = np.concatenate(cand_id)
        order = np.argsort(rid, kind="stable")
        key = np.stack([rs[order], rn[order]], axis=1)
        _, first = np.unique(key, axis=0, return_index=True)
        for fi in first.tolist():
            st, n = int(key[fi, 0]), int(key[fi, 1])
            groups.append((int(rid[order][fi]), np.arange(st, st + n, dtype=np.int64)))
    for f, parts in rows_by_f.items():
        ids = np.concatenate([p[0] for p in parts])
        mat = np.concatenate([p[1] for p in parts])
        order = np.argsort(ids, kind="stable")
        ids, mat = ids[order], mat[order]
        _, first = group_matrix_rows(mat)
        for fi in first.tolist():
            groups.append((int(ids[fi]), mat[fi]))
    if not groups:
        return np.zeros(0, dtype=np.int64), np.zeros(1, dtype=np.int64)
    groups.sort(key=lambda t: t[0])
    members = [m for _, m in groups]
    sizes = np.array([m.size for m in members], dtype=np.int64)
    group_idx = np.concatenate(members)
    group_off = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
    gid = np.repeat(np.arange(len(members), dtype=np.int64), sizes)
    claim = np.full(theta_size, -1, dtype=np.int64)
    claim[group_idx] = gid
    if np.any(claim[group_idx] != gid):
        raise CircuitValidationError(
            "normalization groups overlap after parameter tying; tie whole "
            "sum nodes (or whole pmfs), not parts of them")
    return group_idx, group_off


def _hash_async(g):
    """graph_hash on a worker thread (sha256 and the native record writer
    release the GIL), overlapping the compile; returns the joiner."""
    box: dict = {}

    def run():
        try:
            box["h"] = graph_hash(g, True)
        except BaseException as e:  # re-raised by the joiner
            box["e"] = e

    th = threading.Thread(target=run, name="pcirc-graph-hash", daemon=True)
    th.start()

    def join() -> str:
        th.join()
        if "e" in box:
            raise box["e"]
        return box["h"]
    return join


def _hash_segments_native(nat, g, h, limit: int = 64 << 20):
    """Records of runs of segments written by ``pcc_hash_records_multi`` into
    <= ``limit``-byte buffers (one segment larger than that is cut into row
    ranges)."""
    ptr, i64, addr = _native.ptr, _native.i64, _native.addr
    batch: list = []
    keep: list = []
    size = 0

    def flush():
        nonlocal batch, keep, size
        if not batch:
            return
        kinds = np.array([b[0] for b in batch], dtype=np.int8)
        counts = np.array([b[1] for b in batch], dtype=np.int64)
        fans = np.array([b[2] for b in batch], dtype=np.int64)
        tabs = [_native.addr_array([b[3 + j] for b in batch]) for j in range(3)]
        a_st = np.array([b[6] for b in batch], dtype=np.int64)
        b_st = np.array([b[7] for b in batch], dtype=np.int64)
        out = np.empty(size, dtype=np.uint8)
        nat.pcc_hash_records_multi(len(batch), ptr(kinds), ptr(counts), ptr(fans),
                                   ptr(tabs[0]), ptr(a_st), ptr(tabs[1]), ptr(b_st),
                                   ptr(tabs[2]), ptr(out))
        h.update(out)
        batch, keep, size = [], [], 0

    for s in g.segments:
        f = max(s.fan_in, 1)
        rec = 25 if s.kind == KIND_INPUT else (1 + 8 * f if s.kind == KIND_PRODUCT else 1 + 16 * f)
        strides = (0, 0)
        if s.kind == KIND_INPUT:
            arrs = (i64(s.var), i64(s.ncat), i64(s.slot))
        elif s.kind == KIND_PRODUCT:
            ch, cs = _native.rows(s.children)
            arrs, strides = (ch,), (cs, 0)
        else:
            (ch, cs), (sl, ss) = _native.rows(s.children), _native.rows(s.slots)
            arrs, strides = (ch, sl), (cs, ss)
        step = max(1, limit // rec)
        for a in range(0, s.count, step):
            b = min(s.count, a + step)
            if size + (b - a) * rec > limit:
                flush()
            parts = [x[a:b] for x in arrs]
            keep.extend(parts)
            ads = [addr(x) for x in parts] + [0] * (3 - len(parts))
            batch.append((s.kind, b - a, f, *ads, *strides))
            size += (b - a) * rec
    flush()


def graph_hash(g, native: bool | None = None) -> str:
    """Structural hash (``build.py:634-657``): same byte stream, built per segment
    (records written by ``pcc_hash_records_multi`` when the native core is loaded)."""
    g = _as_graph(g)
    nat = _native.lib() if native in (None, True) else None
    h = hashlib.sha256()
    h.update(b"pcirc-graph-1")
    h.update(np.array([g.num_vars, g.num_nodes, g.root], dtype=np.int64).tobytes())
    if nat is not None and all(s.kind == KIND_INPUT or s.fan_in > 0 for s in g.segments):
        _hash_segments_native(nat, g, h)
        h.update(memoryview(np.ascontiguousarray(g.params, dtype=np.float64)).cast("B"))
        if g.tying:
            h.update(np.array(sorted(g.tying.items()), dtype=np.int64).tobytes())
        return h.hexdigest()
    for s in g.segments:
        f = max(s.fan_in, 1)
        step = max(1, (64 << 20) // (16 * f + 25))  # bound the record buffer
        for a in range(0, s.count, step):
            b = min(s.count, a + step)
            if s.kind == KIND_INPUT:
                rec = np.zeros(b - a, dtype=[("t", "S1"), ("v", "<i8", (3,))])
                rec["t"] = b"I"
                rec["v"] = np.stack([s.var[a:b], s.ncat[a:b], s.slot[a:b]], axis=1)
            elif s.kind == KIND_PRODUCT:
                rec = np.zeros(b - a, dtype=[("t", "S1"), ("c", "<i8", (f,))])
                rec["t"] = b"P"
                rec["c"] = s.children[a:b]
            else:
                rec = np.zeros(b - a, dtype=[("t", "S1"), ("c", "<i8", (f,)), ("s", "<i8", (f,))])
                rec["t"] = b"S"
                rec["c"] = s.children[a:b]
                rec["s"] = s.slots[a:b]
            h.update(rec.tobytes())
    h.update(memoryview(np.ascontiguousarray(g.params, dtype=np.float64)).cast("B"))
    if g.tying:
        h.update(np.array(sorted(g.tying.items()), dtype=np.int64).tobytes())
    return h.hexdigest()
