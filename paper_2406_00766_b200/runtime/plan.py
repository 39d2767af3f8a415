"""Device execution plan: the compiled layout narrowed to flat int32 tables.

``build_program`` turns a :class:`CompiledCircuit` (host int64 arrays, the
bit-exact layout contract) into

* one device int32 blob holding every index table (groups, product buckets,
  pushes, input chunks, replica CSR, simplex-group CSR), and
* a host int64 program: layer / group records with (offset, count) refs into
  the blob, parsed by ``pcb_plan_create`` (``csrc/pcb_capi.cu``).

Derived, non-contract tables are added for the kernels: the per-layer list
of scratch rows that must read -inf (window padding), replica reductions
grouped by destination tile, and tensor-core "super-rows" (sum blocks with
identical child-block rows stacked up to 256 sums for one MMA N extent).
"""
from __future__ import annotations

import numpy as np

from ..compiler._rows import group_matrix_rows
from ..errors import UsageError
from . import _lib

MAGIC = 0x50434232
VERSION = 28
TC_NMAX = 256
INT32_MAX = np.iinfo(np.int32).max
EM_BIG = 2048  # simplex groups at least this large get a whole CTA in the EM pass


def _host_lib():
    """The native host library (compiler/_native.py), or None."""
    from ..compiler import _native
    return _native.lib()


class _Blob:
    def __init__(self):
        self.parts: list[np.ndarray] = []
        self.size = 0

    def add(self, arr) -> tuple[int, int]:
        a = np.asarray(arr).ravel()
        if a.size:
            nat = _host_lib() if a.size >= (1 << 20) else None
            if nat is not None and a.dtype == np.int64 and a.flags.c_contiguous:
                mm = np.empty(2, np.int64)
                nat.pcc_minmax(a.ctypes.data, a.size, mm.ctypes.data)
                lo, hi = int(mm[0]), int(mm[1])
            else:
                lo, hi = int(a.min()), int(a.max())
            if hi > INT32_MAX or lo < -INT32_MAX:
                raise UsageError("index table exceeds int32 range")
        off = self.size
        if a.size:
            self.parts.append(a)  # narrowed once, into the final table
            self.size += a.size
        return off, int(a.size)

    def array(self) -> np.ndarray:
        if not self.parts:
            return np.zeros(1, dtype=np.int32)
        out = np.empty(self.size, dtype=np.int32)
        nat = _host_lib()
        pos = 0
        for a in self.parts:
            if nat is not None and a.size >= (1 << 20) and a.dtype == np.int64 \
                    and a.flags.c_contiguous:
                nat.pcc_narrow_i32(a.ctypes.data, a.size, out[pos:].ctypes.data)
            else:
                np.copyto(out[pos:pos + a.size], a, casting="unsafe")
            pos += a.size
        self.parts = []
        return out


SMS = 148  # B200 streaming multiprocessors


def tc_super_rows(prod_ids: np.ndarray, k_m: int, nmax: int = TC_NMAX, min_count: int = 0):
    """Stack group rows with identical child rows into <= nmax-sum super-rows.

    ``min_count`` caps the stack so the layer still yields about that many
    super-rows (CTAs): stacking shares one operand conversion across up to
    ``nmax / k_m`` blocks, but a layer of a few identical rows (HMM: 128 rows)
    must not collapse into a handful of CTAs on a 148-SM part."""
    rows = prod_ids.shape[0]
    if rows == 0:
        return np.zeros(1, np.int64), np.zeros(0, np.int64)
    per = max(1, nmax // max(k_m, 1))
    if min_count:
        per = max(1, min(per, rows // min_count))
    gid, first = group_matrix_rows(prod_ids)
    order = np.argsort(gid, kind="stable")
    sizes = np.bincount(gid)
    offs, members = [0], []
    pos = 0
    for g, sz in enumerate(sizes.tolist()):
        mem = order[pos:pos + sz]
        pos += sz
        for a in range(0, sz, per):
            chunk = mem[a:a + per]
            members.append(chunk)
            offs.append(offs[-1] + chunk.size)
    return np.asarray(offs, dtype=np.int64), np.concatenate(members).astype(np.int64)


TC_K = (16, 32, 64)


def tc_layer(L) -> bool:
    """Layers whose sum contractions run on tcgen05 (block sizes 16 / 32 / 64)."""
    return L.k_m in TC_K and L.k_n in TC_K


def _stack_order(mats, tiles_of):
    """Tile ids in stacking order: for every group of identical rows of each
    matrix (child-block rows of the forward groups / parent-block rows of the
    backward groups), column by column, the group's rows in order — so any
    run of stacked rows of one column has consecutive plane offsets."""
    order = []
    for mat, tmat in zip(mats, tiles_of):
        if mat.shape[0] == 0:
            continue
        gid, _ = group_matrix_rows(mat)
        rows = np.argsort(gid, kind="stable")          # rows grouped, in order
        g_sorted = gid[rows]
        cols = np.arange(mat.shape[1])
        # (group, column, row) order
        key_g = np.repeat(g_sorted, cols.size)
        key_c = np.tile(cols, rows.size)
        key_r = np.repeat(np.arange(rows.size), cols.size)
        o = np.lexsort((key_r, key_c, key_g))
        t = tmat[rows][:, cols].ravel()[o]
        order.append(t[t != 0])
    return np.concatenate(order) if order else np.zeros(0, np.int64)


def mma_tiles(compiled, tensor_cores: bool = True):
    """Unique parameter tiles of tensor-core layers and their bf16 plane offsets.

    The bf16 copy of theta is four regions of T elements each: hi and lo of
    every tile in sum-major core order (the K-major B operand of the sum
    forward) at ``slab_f`` / ``slab_f + T``, and hi and lo of its transpose
    (the K-major B operand of the child flows) at ``2T + slab_c`` / ``3T +
    slab_c``.  ``slab_f`` follows the forward stacking order and ``slab_c``
    the child-flow stacking order, so a super-row's stacked tiles of one
    column are one contiguous run per plane.
    Returns (theta starts sorted, slab_f, slab_c, k_m, k_n, T)."""
    starts, kms, kns = [], [], []
    fm, ft, bm, bt = [], [], [], []
    if tensor_cores:
        for L in compiled.layers:
            if not tc_layer(L):
                continue
            ids = np.unique(np.concatenate([g.param_ids[g.param_ids != 0]
                                            for g in L.fwd_groups]))
            starts.append(ids)
            kms.append(np.full(ids.size, L.k_m, np.int64))
            kns.append(np.full(ids.size, L.k_n, np.int64))
            for g in L.fwd_groups:
                fm.append(g.prod_ids)
                ft.append(g.param_ids)
            for g in L.bwd_groups:
                bm.append(g.par_ids)
                bt.append(g.par_param_ids)
    if not starts:
        z = np.zeros(0, np.int64)
        return z, z, z, z, z, 0
    s = np.concatenate(starts)
    km = np.concatenate(kms)
    kn = np.concatenate(kns)
    s, first = np.unique(s, return_index=True)  # a tied tile may recur across layers
    km, kn = km[first], kn[first]
    size = km * kn

    def offsets(order):
        # first appearance in `order`, then any tile never stacked
        idx = np.searchsorted(s, order)
        seen = np.zeros(s.size, dtype=bool)
        uniq = []
        if idx.size:
            _, f = np.unique(idx, return_index=True)
            uniq = idx[np.sort(f)]
            seen[uniq] = True
        seq = np.concatenate([np.asarray(uniq, dtype=np.int64), np.flatnonzero(~seen)])
        off = np.empty(s.size, dtype=np.int64)
        off[seq] = np.concatenate([[0], np.cumsum(size[seq])[:-1]])
        return off

    slab_f = offsets(_stack_order(fm, ft))
    slab_c = offsets(_stack_order(bm, bt))
    return s, slab_f, slab_c, km, kn, int(size.sum())


def theta_contig_flags(slab_ids, offs, mem, plane: int) -> np.ndarray:
    """Per super-row: 4 if, for every column, its stacked tiles' plane
    offsets are consecutive (one bulk copy per plane), else 0."""
    n = offs.size - 1
    flags = np.zeros(n, dtype=np.int64)
    for r in range(n):
        m = mem[offs[r]:offs[r + 1]]
        sl = slab_ids[m]                       # [S, cap]
        ok = np.all((sl[1:] - sl[:-1] == plane) | (sl[1:] < 0) & (sl[:-1] < 0)) \
            if m.size > 1 else True
        # bit 3: every column of the row is real (no scan for real columns)
        flags[r] = (4 if ok else 0) | (8 if bool(np.all(sl[0] >= 0)) else 0)
    return flags


IN_BLOCK_ELEMS = 16384   # pmf entries staged in shared memory per input block (64 KB)
SHARED_PMF_MAX = 56000   # categories of a shared pmf histogrammed in shared memory (224 KB)


def shared_pmf_table(compiled, ncat, slots, vars_, pids):
    """Generic input chunk whose pmfs are each used by several inputs (tied
    HMM emissions: one pmf per hidden state, shared by every position) and by
    no input outside the chunk: per unique pmf (ascending start) the CSR of
    its inputs' value slots and variables — the input-flow pass then builds
    each pmf's flow histogram in shared memory (one CTA per pmf) and stores
    the whole row, instead of one global atomic per (input, sample).
    Returns None when the chunk does not qualify."""
    if ncat > SHARED_PMF_MAX or pids.size == 0:
        return None
    all_pids = np.concatenate([ch.param_ids for ch in compiled.input_layer])
    uniq, counts = np.unique(all_pids, return_counts=True)
    u, inv, cnt = np.unique(pids, return_inverse=True, return_counts=True)
    if u.size == pids.size or not np.array_equal(counts[np.searchsorted(uniq, u)], cnt):
        return None
    order = np.argsort(inv, kind="stable")
    off = np.concatenate([[0], np.cumsum(cnt)]).astype(np.int64)
    return {"pid": u.astype(np.int64), "off": off, "slot": slots[order], "var": vars_[order]}


def input_blocks(compiled):
    """Split the input layer into shared-memory blocks and generic leftovers.

    A block is a run of inputs on one variable with consecutive value slots
    and exclusively owned pmfs (no other input shares the pmf range), at most
    ``IN_BLOCK_ELEMS // ncat`` inputs.  Returns (blocks, leftover chunks):
    blocks = dict of arrays var, ncat, slot0, count, pid_off + flat pids;
    leftovers = list of (ncat, slots, vars, pids).
    """
    all_pids = np.concatenate([ch.param_ids for ch in compiled.input_layer]) \
        if compiled.input_layer else np.zeros(0, np.int64)
    uniq, counts = np.unique(all_pids, return_counts=True)
    blk = {k: [] for k in ("var", "ncat", "slot0", "count", "pid_off")}
    pid_flat: list[np.ndarray] = []
    n_pid = 0
    leftovers = []
    for ch in compiled.input_layer:
        ncat = int(ch.num_categories)
        per = IN_BLOCK_ELEMS // ncat if ncat <= IN_BLOCK_ELEMS // 8 else 0
        per = min(per, 128)
        excl = counts[np.searchsorted(uniq, ch.param_ids)] == 1
        n = ch.slots.size
        take = np.zeros(n, dtype=bool)
        if per >= 8 and n:
            # maximal runs: same var, consecutive slots, exclusive pmf
            brk = np.ones(n, dtype=bool)
            brk[1:] = (ch.vars[1:] != ch.vars[:-1]) | (ch.slots[1:] != ch.slots[:-1] + 1) | \
                ~excl[1:] | ~excl[:-1]
            starts = np.flatnonzero(brk)
            ends = np.concatenate([starts[1:], [n]])
            for a, z in zip(starts.tolist(), ends.tolist()):
                if not excl[a] or z - a < 8:
                    continue
                for s0 in range(a, z, per):
                    s1 = min(z, s0 + per)
                    blk["var"].append(int(ch.vars[s0]))
                    blk["ncat"].append(ncat)
                    blk["slot0"].append(int(ch.slots[s0]))
                    blk["count"].append(s1 - s0)
                    blk["pid_off"].append(n_pid)
                    pid_flat.append(ch.param_ids[s0:s1])
                    n_pid += s1 - s0
                take[a:z] = True
        rest = ~take
        if rest.any():
            leftovers.append((ncat, ch.slots[rest], ch.vars[rest], ch.param_ids[rest]))
    arrays = {k: np.asarray(v, dtype=np.int64) for k, v in blk.items()}
    arrays["pids"] = np.concatenate(pid_flat) if pid_flat else np.zeros(0, np.int64)
    return arrays, leftovers


def leaf_alias(compiled, blocks, push_count):
    """Leaf products that are aliases of their one input child.

    When every product of the first layer has a single child, that child is a
    staged input whose only parent is the product, and each staged input block
    maps onto whole product blocks of the layer window as one ascending or
    descending run, a lean step (``pcb_train_step`` with PCB_STEP_LEAN) writes the inputs' log
    values straight into the product rows (plus the block maxima the sum
    kernels shift by) and reads the inputs' flows straight from the product
    flow rows: the product evaluation and the flow push of that layer vanish.
    Returns (per-block first product row or -1, per-block row step,
    window pad blocks or None when the layer does not qualify).
    """
    nb = int(blocks["var"].size)
    arow = np.full(nb, -1, dtype=np.int64)
    adir = np.ones(nb, dtype=np.int64)
    none = (np.full(nb, -1, dtype=np.int64), adir, None)
    if not compiled.layers or nb == 0:
        return none
    L = compiled.layers[0]
    if not L.prod_evals or any(ev.children.shape[1] != 1 for ev in L.prod_evals):
        return none
    out = np.concatenate([ev.out for ev in L.prod_evals]).astype(np.int64)
    ch = np.concatenate([ev.children[:, 0] for ev in L.prod_evals]).astype(np.int64)
    if np.unique(ch).size != ch.size or np.any(push_count[ch] != 1):
        return none
    row_of = np.full(compiled.num_value_slots, -1, dtype=np.int64)
    row_of[ch] = out
    kn = int(L.k_n)
    covered = 0
    for b in range(nb):
        s0, n = int(blocks["slot0"][b]), int(blocks["count"][b])
        r = row_of[s0:s0 + n]
        if np.all(r < 0):
            continue
        if np.any(r < 0) or n % kn:
            return none
        d = int(r[1] - r[0]) if n > 1 else 1
        if d not in (1, -1) or np.any(np.diff(r) != d) or int(r.min()) % kn:
            return none
        arow[b], adir[b] = int(r[0]), d
        covered += n
    if covered != out.size:
        return none
    pad = np.setdiff1d(np.arange(L.scratch_window, dtype=np.int64), out)
    pad_blk = np.unique(pad // kn)
    if pad.size != pad_blk.size * kn:
        return none
    return arow, adir, pad_blk


def push_tables(L, li, last_layer, push_count):
    """Fused accumulate + push table of layer li in product order.  flag bit 0:
    push the finished row; bit 1: first accumulation of the row in the
    backward pass (store, not add).  Children are encoded slot * 2 + (1 if the
    slot has a single push in the whole pass: plain store)."""
    prow_arr = np.asarray(L.prod_rows, dtype=np.int64)
    n_pr = prow_arr.size
    pfan = np.zeros(n_pr, dtype=np.int64)
    pos_of_row = {}
    if L.pushes:
        pos_of_row = {r: i for i, r in enumerate(prow_arr.tolist())}
    parts = [None] * n_pr
    for p in L.pushes:
        idx = np.fromiter((pos_of_row[r] for r in p.rows.tolist()), np.int64, p.rows.size)
        pfan[idx] = p.children.shape[1]
        for i, ch in zip(idx.tolist(), p.children):
            parts[i] = ch
    flags = (pfan > 0).astype(np.int64) | (2 * (last_layer[prow_arr] == li)).astype(np.int64)
    poff = np.concatenate([[0], np.cumsum(pfan)]).astype(np.int64)
    pch = (np.concatenate([q for q in parts if q is not None]).astype(np.int64)
           if pfan.sum() else np.zeros(0, np.int64))
    pch = pch * 2 + (push_count[pch] == 1)
    return flags, poff, pch


def push_ratio_tables(compiled, push_tabs):
    """Fused push + flow-ratio plan for lean steps.

    A push block is k (= the layer's product block size) consecutive products
    (consecutive flow-scratch slots, one fan-in f, pushed and first-stored in
    this layer) whose i-th children, for every fan-in slot, are k consecutive
    value slots with a single push each.  The fused kernel copies the block's
    flows into those slots — or, when the slots are exactly one sum block of a
    "pre-ratioed" layer, writes that block's flow ratios (k_ratio's r, in
    place of the flows) and its per-sample shift R instead.  A layer is
    pre-ratioed when every one of its sum blocks is such a target; its
    backward pass then skips the ratio pass (its R rows live at rmax_off).
    Returns (per-layer block tables, pre_ratio flags, rmax offsets, rows).
    """
    layers = compiled.layers
    nl = len(layers)
    # sum blocks of every layer: first slot -> (layer, block)
    sb_of = {}
    sb_info = []
    for li, L in enumerate(layers):
        sids = np.concatenate([g.sum_ids for g in L.fwd_groups]) if L.fwd_groups else \
            np.zeros(0, np.int64)
        base = int(sids.min()) if sids.size else 0
        sb_info.append((base, int(sids.size), int(L.k_m)))
        for blk in range(int(sids.size)):
            sb_of[base + blk * int(L.k_m)] = (li, blk)
    cand = []  # per layer: list of (slot0, f, [child bases]) or None
    for li, L in enumerate(layers):
        flags, poff, pch = push_tabs[li]
        slots = np.asarray(L.prod_slots, dtype=np.int64)
        k = int(L.k_n)
        n = slots.size
        # the fused kernel exists for product blocks of 16 / 32 / 64
        ok = n > 0 and k in (16, 32, 64) and n % k == 0 and bool(np.all(flags == 3)) and \
            bool(np.all(pch & 1)) if n else False
        blocks = []
        if ok:
            fan = np.diff(poff)
            ch = pch >> 1
            for j0 in range(0, n, k):
                f = int(fan[j0])
                if np.any(fan[j0:j0 + k] != f) or f == 0 or \
                        np.any(np.diff(slots[j0:j0 + k]) != 1):
                    ok = False
                    break
                kids = ch[poff[j0]:poff[j0 + k]].reshape(k, f)
                if np.any(np.diff(kids, axis=0) != 1):
                    ok = False
                    break
                blocks.append((int(slots[j0]), f, kids[0].tolist()))
        cand.append(blocks if ok else None)
    # pre-ratioed layers: every sum block is the target of one fused slot
    hits = [0] * nl
    for li in range(nl):
        if cand[li] is None:
            continue
        for _, _, bases in cand[li]:
            for cb in bases:
                t = sb_of.get(cb)
                if t is not None and sb_info[t[0]][2] == int(layers[li].k_n):
                    hits[t[0]] += 1
    pre = [bool(sb_info[li][1] > 0 and hits[li] == sb_info[li][1]) for li in range(nl)]
    rmax_off, n_rmax = [], 0
    for li in range(nl):
        rmax_off.append(n_rmax if pre[li] else -1)
        n_rmax += sb_info[li][1] if pre[li] else 0
    tabs = []
    empty = np.zeros(0, np.int64)
    for li in range(nl):
        if cand[li] is None:
            tabs.append({k: empty for k in ("row", "f", "qoff", "qblk", "qbase", "qkind",
                                            "qrrow")})
            continue
        row, fs, qoff, qbl, qb, qk, qr = [], [], [0], [], [], [], []
        for bi, (slot0, f, bases) in enumerate(cand[li]):
            row.append(slot0)
            fs.append(f)
            for cb in bases:
                qbl.append(bi)
                t = sb_of.get(cb)
                ratio = t is not None and pre[t[0]] and sb_info[t[0]][2] == int(layers[li].k_n)
                qb.append(cb)
                qk.append(1 if ratio else 0)
                qr.append(rmax_off[t[0]] + t[1] if ratio else -1)
            qoff.append(len(qb))
        tabs.append({"row": np.asarray(row, np.int64), "f": np.asarray(fs, np.int64),
                     "qoff": np.asarray(qoff, np.int64), "qblk": np.asarray(qbl, np.int64),
                     "qbase": np.asarray(qb, np.int64),
                     "qkind": np.asarray(qk, np.int64), "qrrow": np.asarray(qr, np.int64)})
    return tabs, pre, rmax_off, n_rmax


def group_runs(group_idx, group_off):
    """Run-length encode the simplex-group index table: maximal runs of
    consecutive theta indices inside each group.  Returns (per-group run
    offsets [n_groups + 1], run starts, run lengths)."""
    gi = np.asarray(group_idx, dtype=np.int64)
    go = np.asarray(group_off, dtype=np.int64)
    n = gi.size
    if n == 0:
        return np.zeros(go.size, np.int64), np.zeros(0, np.int64), np.zeros(0, np.int64)
    from ..compiler import _native
    nat = _native.lib()
    if nat is not None:  # native two-pass encoding (no whole-table temporaries)
        gi, go = _native.i64(gi), _native.i64(go)
        ng = go.size - 1
        run_off = np.zeros(ng + 1, np.int64)
        nat.pcc_group_runs(ng, _native.ptr(go), _native.ptr(gi), _native.ptr(run_off), None, None)
        np.cumsum(run_off, out=run_off)
        rs = np.empty(int(run_off[-1]), np.int64)
        rl = np.empty_like(rs)
        nat.pcc_group_runs(ng, _native.ptr(go), _native.ptr(gi), _native.ptr(run_off),
                           _native.ptr(rs), _native.ptr(rl))
        return run_off, rs, rl
    brk = np.ones(n, dtype=bool)
    brk[1:] = gi[1:] != gi[:-1] + 1
    brk[go[:-1][go[:-1] < n]] = True          # every group starts a run
    starts = np.flatnonzero(brk)
    lens = np.diff(np.concatenate([starts, [n]]))
    run_off = np.searchsorted(starts, go)       # group start positions are run starts
    return run_off.astype(np.int64), gi[starts], lens.astype(np.int64)


def em_tile_blocks(compiled, t_start, t_slab_f, t_slab_c, t_km, t_kn):
    """Simplex groups that exactly tile tensor-core parameter tiles.

    A block is k_m groups (the sums of one sum block) whose parameters are the
    k_m rows of a set of k_m x k_n tiles, row i of every tile belonging to the
    block's i-th group.  The EM pass runs such blocks tile by tile (coalesced
    whole-tile traffic) and writes the bf16 MMA planes of the updated tiles in
    the same pass.  Returns dict(blk_km, blk_kn, blk_tile_off [n+1],
    blk_groups (flat, k_m per block), tile_start, tile_slab) and the sorted ids
    of the groups left to the generic per-group pass.
    """
    gi = np.asarray(compiled.group_idx, dtype=np.int64)
    go = np.asarray(compiled.group_off, dtype=np.int64)
    n_groups = go.size - 1
    empty = dict(blk_km=np.zeros(0, np.int64), blk_kn=np.zeros(0, np.int64),
                 blk_tile_off=np.zeros(1, np.int64), blk_groups=np.zeros(0, np.int64),
                 tile_start=np.zeros(0, np.int64), tile_slab_f=np.zeros(0, np.int64),
                 tile_slab_c=np.zeros(0, np.int64))
    if n_groups <= 0 or t_start.size == 0:
        return empty, np.arange(max(n_groups, 0), dtype=np.int64)
    run_off, rs, rl = group_runs(gi, go)
    run_grp = np.repeat(np.arange(n_groups, dtype=np.int64), np.diff(run_off))
    order = np.argsort(rs, kind="stable")
    rs_s, rl_s, rg_s = rs[order], rl[order], run_grp[order]
    n_runs_of = np.diff(run_off)
    covered = np.zeros(n_groups, dtype=bool)
    blocks = []  # (km, kn, groups tuple, tile indices)
    for km, kn in sorted(set(zip(t_km.tolist(), t_kn.tolist()))):
        sel = np.flatnonzero((t_km == km) & (t_kn == kn))
        rows = t_start[sel][:, None] + np.arange(km, dtype=np.int64)[None, :] * kn
        pos = np.searchsorted(rs_s, rows)
        pos_c = np.minimum(pos, rs_s.size - 1)
        ok = (rs_s[pos_c] == rows) & (rl_s[pos_c] == kn)
        good = ok.all(axis=1)
        if not good.any():
            continue
        own = rg_s[pos_c[good]]                    # [tiles x km] owner group per row
        tiles = sel[good]
        key, inv = np.unique(own, axis=0, return_inverse=True)
        inv = inv.ravel()
        cnt = np.bincount(inv, minlength=key.shape[0])
        torder = np.argsort(inv, kind="stable")
        offs = np.concatenate([[0], np.cumsum(cnt)])
        # every group of a block lives exactly in its tiles, and is distinct
        ks = np.sort(key, axis=1)
        distinct = (ks[:, 1:] != ks[:, :-1]).all(axis=1) if km > 1 else np.ones(key.shape[0], bool)
        exact = (n_runs_of[key] == cnt[:, None]).all(axis=1)
        for b in np.flatnonzero(distinct & exact).tolist():
            grp = key[b]
            if covered[grp].any():
                continue
            blocks.append((km, kn, grp, tiles[torder[offs[b]:offs[b + 1]]]))
            covered[grp] = True
    if not blocks:
        return empty, np.arange(n_groups, dtype=np.int64)
    tl = [np.sort(b[3]) for b in blocks]
    out = dict(
        blk_km=np.array([b[0] for b in blocks], np.int64),
        blk_kn=np.array([b[1] for b in blocks], np.int64),
        blk_tile_off=np.concatenate([[0], np.cumsum([t.size for t in tl])]).astype(np.int64),
        blk_groups=np.concatenate([b[2] for b in blocks]).astype(np.int64),
        tile_start=np.concatenate([t_start[t] for t in tl]).astype(np.int64),
        tile_slab_f=np.concatenate([t_slab_f[t] for t in tl]).astype(np.int64),
        tile_slab_c=np.concatenate([t_slab_c[t] for t in tl]).astype(np.int64))
    return out, np.flatnonzero(~covered).astype(np.int64)


def em_fused_order(compiled, tb, tensor_cores: bool):
    """EM fused into the parameter-flow epilogue (one-process lean steps).

    A layer qualifies when its blocks are 32 x 32, every sum row's children
    fit one 256-column item (cap * k_n <= 256), its flow tiles have a single
    writer, and each of its sum blocks is exactly one EM tile block (group i =
    row i of the block's tiles, no tile shared with another sum block): the
    epilogue thread of a sum row then holds the row's whole group.  The tile
    blocks are reordered: blocks of other layers first (n_pre of them), then
    each qualifying layer's blocks contiguously.  Returns (tb, n_pre,
    per-layer [lo, hi) ranges, per-layer flags)."""
    nl = len(compiled.layers)
    nb = int(tb["blk_km"].size)
    none = (tb, nb, [(0, 0)] * nl, [False] * nl)
    if nb == 0 or not tensor_cores:
        return none
    off = tb["blk_tile_off"]
    by_tiles = {}
    for b in range(nb):
        if int(tb["blk_km"][b]) == 32 and int(tb["blk_kn"][b]) == 32:
            by_tiles[frozenset(tb["tile_start"][off[b]:off[b + 1]].tolist())] = b
    # tiles used by more than one (layer, sum block): their flows have several
    # producers, so no single epilogue sees a whole group
    uses = {}
    for L in compiled.layers:
        for g in L.fwd_groups:
            for t in np.asarray(g.param_ids, dtype=np.int64).ravel().tolist():
                if t:
                    uses[t] = uses.get(t, 0) + 1
    owner = np.full(nb, -1, dtype=np.int64)
    fus = [False] * nl
    for li, L in enumerate(compiled.layers):
        if not tc_layer(L) or int(L.k_m) != 32 or int(L.k_n) != 32 or not L.fwd_groups:
            continue
        ok, mine = True, []
        for g in L.fwd_groups:
            pid = np.asarray(g.param_ids, dtype=np.int64)
            if g.prod_ids.shape[1] * 32 > 256:
                ok = False
                break
            for row in pid:
                t = row[row != 0]
                b = by_tiles.get(frozenset(t.tolist()))
                if b is None or t.size != np.unique(t).size or owner[b] >= 0 or \
                        off[b + 1] - off[b] != t.size or any(uses[x] != 1 for x in t.tolist()):
                    ok = False
                    break
                mine.append(b)
            if not ok:
                break
        if ok and mine:
            owner[np.asarray(mine)] = li
            fus[li] = True
    key = np.where(owner >= 0, owner, -1)
    order = np.argsort(key, kind="stable")
    n_pre = int((owner < 0).sum())
    sizes = np.diff(off)[order]
    tidx = np.repeat(off[:-1][order] - np.concatenate([[0], np.cumsum(sizes)[:-1]]), sizes) + \
        np.arange(int(sizes.sum()), dtype=np.int64)
    goff = np.concatenate([[0], np.cumsum(tb["blk_km"])])
    gsz = tb["blk_km"][order]
    gidx = np.repeat(goff[:-1][order] - np.concatenate([[0], np.cumsum(gsz)[:-1]]), gsz) + \
        np.arange(int(gsz.sum()), dtype=np.int64)
    out = dict(blk_km=tb["blk_km"][order], blk_kn=tb["blk_kn"][order],
               blk_tile_off=np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64),
               blk_groups=tb["blk_groups"][gidx],
               tile_start=tb["tile_start"][tidx], tile_slab_f=tb["tile_slab_f"][tidx],
               tile_slab_c=tb["tile_slab_c"][tidx])
    ks = key[order]
    ranges = []
    for li in range(nl):
        idx = np.flatnonzero(ks == li)
        ranges.append((int(idx[0]), int(idx[-1]) + 1) if idx.size else (0, 0))
    return out, n_pre, ranges, fus


def pf_pre_ok(g, L) -> bool:
    """Parameter flows of a dense uniform group (every sum block over the same
    child row, several 256-child column groups or 128-sum tiles sharing it,
    e.g. HMM transition layers) may convert their operands once per layer:
    the sums are consecutive value slots from a 128-aligned start, the real
    child blocks consecutive scratch rows (the pre-converted 128-sum and
    256-child operand images are then addressed by row)."""
    if L.k_n != 32 or L.k_m not in (16, 32) or len(L.fwd_groups) != 1:
        return False
    sid = np.sort(np.asarray(g.sum_ids, dtype=np.int64))
    if sid.size < 4 or np.any(np.diff(sid) != L.k_m):
        return False
    real = np.asarray(g.param_ids[0]) != 0
    p = np.asarray(g.prod_ids[0])[real]
    if p.size < 8 or np.any(np.diff(p) != L.k_n):
        return False
    return int(real.sum()) * L.k_n > 256 or sid.size * L.k_m > 128


def pf_contig_flags(g, offs, mem, k_m: int, k_n: int) -> np.ndarray:
    """Per (full-stack) super-row: bit 0 = its member sum blocks are
    consecutive sum rows, bit 1 = its real child blocks are consecutive
    scratch rows — the parameter-flow kernel then moves each with one TMA box
    per chunk instead of one per block."""
    n = offs.size - 1
    flags = np.zeros(n, dtype=np.int64)
    for r in range(n):
        m = mem[offs[r]:offs[r + 1]]
        sid = g.sum_ids[m]
        a_ok = bool(np.all(np.diff(sid) == k_m)) if sid.size > 1 else True
        row = int(m[0])
        real = g.param_ids[row] != 0
        p = g.prod_ids[row][real]
        e_ok = bool(np.all(np.diff(p) == k_n)) if p.size > 1 else True
        # bit 3: no padding column (the item's columns follow arithmetically)
        flags[r] = int(a_ok) | (int(e_ok) << 1) | (int(bool(real.all())) << 3)
    return flags


def _slab_of(ids, starts, slab):
    """Slab offset per parameter-tile id (-1 for the zero tile / padding)."""
    out = np.full(ids.shape, -1, dtype=np.int64)
    nz = ids != 0
    if nz.any():
        out[nz] = slab[np.searchsorted(starts, ids[nz])]
    return out


def slot_base_rows(compiled) -> np.ndarray:
    """Per value slot: the row of its sum block's base in the device ``vbase``
    region (sum blocks of all layers in layer order, each layer's blocks in
    slot order), or -1 for slots with base 0 (reserved rows, inputs).  Log
    values are stored as (base, offset) pairs; see csrc/pcb_internal.cuh."""
    c = compiled
    out = np.full(max(c.num_value_slots, 1), -1, dtype=np.int64)
    off = 0
    for L in c.layers:
        sids = np.concatenate([g.sum_ids for g in L.fwd_groups]) if L.fwd_groups else \
            np.zeros(0, np.int64)
        if not sids.size:
            continue
        base, n = int(sids.min()), int(sids.size)
        if not np.array_equal(np.sort(sids), base + L.k_m * np.arange(n)):
            raise RuntimeError("sum blocks of a layer must be contiguous value slots")
        out[base:base + n * L.k_m] = off + np.arange(n * L.k_m) // L.k_m
        off += n
    return out


def prod_blocks_uniform(fan, row_off, cb_flat, k_n: int) -> bool:
    """Every product block of the window takes its children's bases from the
    same base rows, slot by slot (its non-empty rows have one fan-in and one
    child-base list; row 0 is non-empty unless the whole block is padding):
    the product kernel then forms the block's summed base once per sample."""
    nb = fan.size // k_n
    if nb == 0:
        return True
    f = fan.reshape(nb, k_n)
    f0 = f[:, :1]
    if np.any((f != 0) & (f != f0)):
        return False
    fmax = int(fan.max()) if fan.size else 0
    if fmax == 0:
        return True
    cb = np.full((fan.size, fmax), -3, dtype=np.int64)
    r = np.repeat(np.arange(fan.size), fan)
    q = np.arange(cb_flat.size) - np.repeat(row_off[:-1], fan)
    cb[r, q] = cb_flat
    cb = cb.reshape(nb, k_n, fmax)
    live = (f != 0)[:, :, None]
    return bool(np.all(~live | (cb == cb[:, :1, :])))


def build_program(compiled, *, tensor_cores: bool = True):
    """Return (program int64 array, blob int32 array, info dict)."""
    blob = _Blob()
    prog: list[int] = [MAGIC, VERSION]

    def ref(arr):
        off, n = blob.add(arr)
        prog.extend([off, n])

    c = compiled
    slot_vb = slot_base_rows(c)
    prog += [c.num_vars, c.num_value_slots, c.scratch_size, c.num_prod_rows, c.theta_size,
             c.f_params_size, c.reserved, c.root_slot, c.root_row]
    rc = np.asarray(c.root_children if c.root_children is not None else np.zeros(0), np.int64)
    ref(rc)
    ref(slot_vb[rc] if rc.size else np.zeros(0, np.int64))
    prog.append(int(slot_vb[c.root_slot]) if c.root_slot >= 0 else -1)
    ref(np.asarray(c.var_categories, dtype=np.int64))
    prog.append(1 if tensor_cores else 0)
    t_start, t_slab_f, t_slab_c, t_km, t_kn, plane_t = mma_tiles(c, tensor_cores)
    mma_elems = 4 * plane_t
    prog += [int(t_start.size), mma_elems, plane_t]
    ref(t_start)
    ref(t_slab_f)
    ref(t_slab_c)
    ref(t_km)
    ref(t_kn)
    scratch_total = int(sum(L.scratch_window for L in c.layers)) or 1
    prog.append(scratch_total)

    # pushes per value slot over the whole backward pass (root pushes included):
    # a slot with exactly one push takes a plain store instead of an atomic add
    push_count = np.zeros(c.num_value_slots, dtype=np.int64)
    for L in c.layers:
        for p in L.pushes:
            np.add.at(push_count, p.children.ravel(), 1)
    if c.root_children is not None and c.root_row >= 0:
        # the root pass adds into these rows: never a single plain store
        np.add.at(push_count, np.asarray(c.root_children, dtype=np.int64), 2)

    blocks, leftovers = input_blocks(c)
    alias_row, alias_dir, alias_pad = leaf_alias(c, blocks, push_count)
    prog.append(len(leftovers))
    shared_pids = {}  # pmf start -> ncat of the shared-pmf chunks
    for ncat, slots, vars_, pids in leftovers:
        prog += [ncat, int(slots.size)]
        ref(slots)
        ref(vars_)
        ref(pids)
        sp = shared_pmf_table(c, ncat, slots, vars_, pids)
        prog.append(0 if sp is None else int(sp["pid"].size))
        for key in ("pid", "off", "slot", "var"):
            ref(sp[key] if sp is not None else np.zeros(0, np.int64))
        if sp is not None:
            shared_pids.update({int(q): int(ncat) for q in sp["pid"].tolist()})
    nb = int(blocks["var"].size)
    prog.append(nb)
    for key in ("var", "ncat", "slot0", "count", "pid_off", "pids"):
        ref(blocks[key])
    prog.append(int((blocks["ncat"] * blocks["count"]).max()) if nb else 0)
    prog.append(int(blocks["ncat"].max()) if nb else 0)
    prog.append(int(blocks["count"].max()) if nb else 0)
    ref(alias_row)
    ref(alias_dir)
    prog.append(1 if alias_pad is not None else 0)
    ref(alias_pad if alias_pad is not None else np.zeros(0, np.int64))
    # flow rows the backward pass must zero first: all but the single-store rows
    need = push_count != 1
    if c.num_value_slots:
        edges = np.flatnonzero(np.diff(np.concatenate([[0], need.astype(np.int8), [0]])))
        z_start, z_end = edges[0::2], edges[1::2]
        # pieces of <= 64 rows: one CTA each
        pieces = [np.arange(a, e, 64) for a, e in zip(z_start.tolist(), z_end.tolist())]
        if pieces:
            ps = np.concatenate(pieces)
            pe = np.minimum(ps + 64, np.repeat(z_end, [p.size for p in pieces]))
            z_start, z_end = ps, pe
    else:
        z_start = z_end = np.zeros(0, np.int64)
    prog.append(int(z_start.size))
    ref(z_start)
    ref(z_end - z_start)
    # the last layer (in backward order: the highest) accumulating each product row
    # writes it instead of adding; every row written => no prod_flows memset
    last_layer = np.full(max(c.num_prod_rows, 1), -1, dtype=np.int64)
    for li, L in enumerate(c.layers):
        last_layer[np.asarray(L.prod_rows, dtype=np.int64)] = li
    covered = np.ones(last_layer.size, dtype=bool)
    covered[last_layer < 0] = False
    if c.root_row >= 0:
        covered[c.root_row] = True
    prog.append(1 if bool(covered.all()) else 0)
    # every product row is accumulated and pushed in one layer: the backward
    # pass may skip materialising prod_flows (d_prod_flows = NULL)
    pf_optional = True

    # replica flow ranges (compiler/build.py:516-533) are folded onto their
    # master tiles: on the GPU every parameter-flow kernel accumulates with
    # red.add (stores only for single-writer tiles), so the contention the
    # replicas avoid on the CPU costs nothing, and the replica reduction pass
    # and its 31 x 16.8 M-float traffic at HMM-4096 disappear.  The replica
    # ranges of f_params stay zero.
    red = np.asarray(c.reductions, dtype=np.int64).reshape(-1, 3)
    rep_src, rep_dst = red[:, 0], red[:, 1]
    rep_order = np.argsort(rep_src)
    rep_src, rep_dst = rep_src[rep_order], rep_dst[rep_order]

    def folded(ids):
        if rep_src.size == 0:
            return ids
        pos = np.minimum(np.searchsorted(rep_src, ids), rep_src.size - 1)
        hit = rep_src[pos] == ids
        return np.where(hit, rep_dst[pos], ids)

    # flow tiles written by exactly one (layer, group, row, column) in the pass:
    # a group whose tiles are all exclusive may store its parameter flows
    flow_starts = [folded(g.flow_ids)[g.param_ids != 0] for L in c.layers for g in L.fwd_groups]
    if flow_starts:
        fu, fcnt = np.unique(np.concatenate(flow_starts), return_counts=True)
    else:
        fu, fcnt = np.zeros(0, np.int64), np.zeros(0, np.int64)

    def exclusive(g) -> int:
        f = folded(g.flow_ids)[g.param_ids != 0]
        return int(bool(np.all(fcnt[np.searchsorted(fu, f)] == 1))) if f.size else 1

    # parameter-flow fusion (tied layers, e.g. HMM transitions): layers whose
    # single pre-converted dense group is the same table (same tied tiles,
    # same relative sum / child structure) and whose flow tiles no other layer
    # writes run ONE parameter-flow contraction over the concatenated batches
    # of all of them (the layers' pre-converted operand images laid end to
    # end along K): one epilogue of plain stores instead of one reduction
    # pass per layer
    fuse_id = [-1] * len(c.layers)
    if tensor_cores:
        cand: dict = {}
        for li, L in enumerate(c.layers):
            if not tc_layer(L) or len(L.fwd_groups) != 1:
                continue
            g = L.fwd_groups[0]
            rows = g.prod_ids.shape[0]
            if not (rows > 0 and group_matrix_rows(g.prod_ids)[1].size == 1 and pf_pre_ok(g, L)):
                continue
            f = folded(g.flow_ids)[g.param_ids != 0]
            if np.unique(f).size != f.size:
                continue
            sid = np.asarray(g.sum_ids, np.int64)
            pid = np.asarray(g.prod_ids, np.int64)
            key = (L.k_m, L.k_n, g.param_ids.shape, np.asarray(g.param_ids, np.int64).tobytes(),
                   np.asarray(folded(g.flow_ids), np.int64).tobytes(), (sid - sid.min()).tobytes(),
                   (pid - pid.min()).tobytes())
            cand.setdefault(key, []).append((li, f))
        nid = 0
        for members in cand.values():
            if len(members) < 2:
                continue
            f = members[0][1]
            if not np.all(fcnt[np.searchsorted(fu, f)] == len(members)):
                continue  # another layer writes these tiles too
            for li, _ in members:
                fuse_id[li] = nid
            nid += 1

    # per-layer flow ranges and whether f_params[:theta_size] is covered by
    # them, the staged (stored) input pmfs and the zero tile, all disjoint
    layer_range, fp_cover = [], True
    spans = []
    for L in c.layers:
        starts, sizes = [], []
        for g in L.fwd_groups:
            f = folded(g.flow_ids)[g.param_ids != 0]
            starts.append(np.unique(f))
        u = np.unique(np.concatenate(starts)) if starts else np.zeros(0, np.int64)
        tsz = int(L.k_m * L.k_n)
        if u.size:
            lo, hi = int(u.min()), int(u.max()) + tsz
            layer_range.append((lo, hi))
            fp_cover = fp_cover and (hi - lo == u.size * tsz)  # tiles exactly tile it
            spans.append((lo, hi))
        else:
            layer_range.append((0, 0))
    if leftovers:
        fp_cover = False
    if nb:
        # staged inputs store their whole pmf ranges
        pid_sorted = np.sort(blocks["pids"])
        ncat_of = np.repeat(blocks["ncat"], blocks["count"])
        order = np.argsort(blocks["pids"], kind="stable")
        for a0, n0 in zip(pid_sorted.tolist(), ncat_of[order].tolist()):
            spans.append((int(a0), int(a0) + int(n0)))
    zt = int(np.max([L.k_m * L.k_n for L in c.layers])) if c.layers else 0
    spans.append((0, zt))
    spans.sort()
    pos = 0
    for a0, b0 in spans:
        if a0 != pos:
            fp_cover = False
            break
        pos = b0
    fp_cover = fp_cover and pos == c.theta_size
    push_tabs = [push_tables(L, li, last_layer, push_count) for li, L in enumerate(c.layers)]
    push_ratio, pre_ratio, rmax_off, n_rmax = push_ratio_tables(c, push_tabs)
    n_tc_rows = 0
    scratch_off = 0
    prog.append(len(c.layers))
    for li, L in enumerate(c.layers):
        prog += [L.k_m, L.k_n, L.scratch_window, int(L.prod_slots.size), scratch_off,
                 int(layer_range[li][0]), int(layer_range[li][1])]
        scratch_off += L.scratch_window
        use_tc = tensor_cores and tc_layer(L)
        written = np.concatenate([ev.out for ev in L.prod_evals]) if L.prod_evals else \
            np.zeros(0, np.int64)
        pad = np.setdiff1d(np.arange(L.scratch_window, dtype=np.int64), written)
        ref(pad)
        prog.append(len(L.prod_evals))
        for ev in L.prod_evals:
            prog += [int(ev.children.shape[1]), int(ev.out.size)]
            ref(ev.out)
            ref(ev.children)
        prog.append(len(L.fwd_groups))
        for g in L.fwd_groups:
            rows, cap = g.prod_ids.shape
            prog += [rows, cap]
            ref(g.sum_ids)
            ref(g.prod_ids)
            ref(g.param_ids)
            ref(folded(g.flow_ids))
            fslab = _slab_of(g.param_ids, t_start, t_slab_f) if use_tc else np.zeros(0, np.int64)
            ref(fslab)
            # product-major plane offsets (EM fused into the parameter flows)
            ref(_slab_of(g.param_ids, t_start, t_slab_c) if use_tc else np.zeros(0, np.int64))
            prog.append(exclusive(g))
            # every row has the same child blocks: one shift row serves them all
            uniform = rows > 0 and group_matrix_rows(g.prod_ids)[1].size == 1
            prog.append(int(uniform))
            prog.append(int(use_tc and uniform and pf_pre_ok(g, L)))
            if use_tc and rows:
                # forward: enough super-rows to fill the SMs; param flows: full
                # stacks (their grid also spans column groups)
                for mc in (SMS, 0):
                    offs, mem = tc_super_rows(g.prod_ids, L.k_m, min_count=mc)
                    prog.append(offs.size - 1)
                    ref(offs)
                    ref(mem)
                    ref(theta_contig_flags(fslab.reshape(g.param_ids.shape), offs, mem,
                                           L.k_m * L.k_n)
                        | (pf_contig_flags(g, offs, mem, L.k_m, L.k_n) if mc == 0 else 0))
                    n_tc_rows += offs.size - 1
            else:
                prog += [0, 0, 0, 0, 0, 0, 0] * 2
        prog.append(len(L.bwd_groups))
        for g in L.bwd_groups:
            rows, cap = g.par_ids.shape
            prog += [rows, cap]
            ref(g.ch_ids)
            ref(g.par_ids)
            ref(g.par_param_ids)
            # the persistent child-flow kernel reads the product-major planes
            # (region 2 + slab_c); the per-launch one (block size 64) the
            # sum-major planes through an MN-major descriptor
            ws_cf = L.k_m in (16, 32)
            if use_tc:
                bslab = (2 * plane_t + _slab_of(g.par_param_ids, t_start, t_slab_c)) if ws_cf \
                    else _slab_of(g.par_param_ids, t_start, t_slab_f)
                bslab[g.par_param_ids == 0] = -1
            else:
                bslab = np.zeros(0, np.int64)
            ref(bslab)
            prog.append(int(rows > 0 and group_matrix_rows(g.par_ids)[1].size == 1))
            if use_tc and rows:
                # per-launch kernels: enough super-rows to fill the SMs; the
                # persistent kernels: full stacks (they split K instead)
                for mc in (SMS, 0):
                    offs, mem = tc_super_rows(g.par_ids, L.k_n, min_count=mc)
                    prog.append(offs.size - 1)
                    ref(offs)
                    ref(mem)
                    ref(theta_contig_flags(bslab.reshape(g.par_param_ids.shape), offs, mem,
                                           L.k_m * L.k_n))
                    n_tc_rows += offs.size - 1
            else:
                prog += [0, 0, 0, 0, 0, 0, 0] * 2
        ref(L.prod_slots)
        ref(L.prod_rows)
        prog.append(len(L.pushes))
        for p in L.pushes:
            prog += [int(p.children.shape[1]), int(p.rows.size)]
            ref(p.rows)
            ref(p.children)
        # derived: per-scratch-row product CSR (pad rows have no children)
        fan = np.zeros(L.scratch_window, dtype=np.int64)
        for ev in L.prod_evals:
            fan[ev.out] = ev.children.shape[1]
        row_off = np.concatenate([[0], np.cumsum(fan)]).astype(np.int64)
        ch_flat = np.zeros(int(row_off[-1]), dtype=np.int64)
        for ev in L.prod_evals:
            f = ev.children.shape[1]
            ch_flat[(row_off[ev.out][:, None] + np.arange(f)).ravel()] = ev.children.ravel()
        ref(row_off)
        ref(ch_flat)
        cb_flat = slot_vb[ch_flat] if ch_flat.size else np.zeros(0, np.int64)
        ref(cb_flat)  # child base rows
        prog.append(int(prod_blocks_uniform(fan, row_off, cb_flat, L.k_n)))
        # derived: sum-block range of the layer (contiguous value slots)
        sids = np.concatenate([g.sum_ids for g in L.fwd_groups]) if L.fwd_groups else \
            np.zeros(0, np.int64)
        prog += [int(sids.min()) if sids.size else 0, int(sids.size)]
        flags, poff, pch = push_tabs[li]
        pf_optional = pf_optional and bool(np.all(flags == 3))
        ref(flags)
        ref(poff)
        ref(pch)
        # fused push + flow ratio (lean steps): blocks of k product rows whose
        # children form, per fan-in slot, k consecutive single-push slots
        pr = push_ratio[li]
        prog.append(int(pr["row"].size))
        for key in ("row", "f", "qoff", "qblk", "qbase", "qkind", "qrrow"):
            ref(pr[key])
        prog += [int(pre_ratio[li]), int(rmax_off[li]), int(fuse_id[li])]

    red = red[:0]  # folded above: no replica reduction pass
    if red.shape[0]:
        order = np.lexsort((np.arange(red.shape[0]), red[:, 1]))
        r = red[order]
        dst, first = np.unique(r[:, 1], return_index=True)
        lens = r[first, 2]
        soff = np.concatenate([first, [r.shape[0]]])
        prog.append(dst.size)
        ref(dst)
        ref(lens)
        ref(soff)
        ref(r[:, 0])
    else:
        prog.append(0)
        for _ in range(4):
            ref(np.zeros(0, np.int64))

    n_groups = int(c.group_off.size - 1)
    prog.append(n_groups)
    ref(c.group_idx)
    ref(c.group_off)
    # EM tile blocks (groups that exactly tile tensor-core tiles) + the rest
    tb, rest = em_tile_blocks(c, t_start, t_slab_f, t_slab_c, t_km, t_kn)
    tb, n_em_pre, em_ranges, em_fusable = em_fused_order(c, tb, tensor_cores)
    prog.append(int(tb["blk_km"].size))
    prog.append(int(tb["tile_start"].size))
    tb["blk_goff"] = np.concatenate([[0], np.cumsum(tb["blk_km"])]).astype(np.int64)
    for key in ("blk_km", "blk_kn", "blk_tile_off", "blk_goff", "tile_start", "tile_slab_f",
                "tile_slab_c"):
        ref(tb[key])
    # remaining groups: small ones (one warp each) first, then big ones (one
    # CTA each, >= EM_BIG entries, e.g. HMM emission pmfs over the vocabulary)
    gi = np.asarray(c.group_idx, dtype=np.int64)
    go = np.asarray(c.group_off, dtype=np.int64)
    gsize = np.diff(go)[rest] if rest.size else np.zeros(0, np.int64)
    # contiguous rest groups (an input pmf is one run): first theta index, else -1
    run_off, _, _ = group_runs(gi, go)
    one = (np.diff(run_off) == 1) & (np.diff(go) > 0)
    contig = np.full(max(n_groups, 0), -1, dtype=np.int64)
    contig[one] = gi[np.minimum(go[:-1][one], max(gi.size - 1, 0))]
    # small groups that are exactly a staged input's pmf (ncat <= 256) go
    # last among the small ones: the inline input EM updates them
    def map_eq(keys, vals, q, want):
        """q in keys and (last value of q) == want, vectorised dict lookup."""
        keys, vals = np.asarray(keys, np.int64), np.asarray(vals, np.int64)
        if keys.size == 0 or q.size == 0:
            return np.zeros(q.size, dtype=bool)
        ks, idx = np.unique(keys[::-1], return_index=True)  # last occurrence wins
        vs = vals[::-1][idx]
        pos = np.minimum(np.searchsorted(ks, q), ks.size - 1)
        return (ks[pos] == q) & (vs[pos] == want)

    crest = contig[rest] if rest.size else np.zeros(0, np.int64)
    if nb:
        ncat_of = np.repeat(blocks["ncat"], blocks["count"])
        inl = (crest >= 0) & map_eq(blocks["pids"], ncat_of, crest, gsize) & (gsize <= 256)
    else:
        inl = np.zeros(rest.size, dtype=bool)
    small = gsize < EM_BIG
    # groups that are exactly a shared pmf (shared_pmf_table) go last: the
    # shared-pmf input-flow pass updates them inline
    sinl = (crest >= 0) & map_eq(list(shared_pids.keys()), list(shared_pids.values()), crest,
                                 gsize)
    inl = inl & ~sinl
    n_shared_inline = int(sinl.sum())
    shared_inline_ok = bool(shared_pids) and n_shared_inline == len(shared_pids)
    rest_o = np.concatenate([rest[small & ~inl & ~sinl], rest[small & inl],
                             rest[~small & ~sinl], rest[sinl]]).astype(np.int64)
    n_small_noninl = int((small & ~inl & ~sinl).sum())
    in_inline_ok = bool(nb) and int((small & inl).sum()) == int(blocks["pids"].size)
    rest = rest_o
    prog.append(int(rest.size))
    prog.append(int((small & ~sinl).sum()))
    ref(rest)
    ref(contig[rest] if rest.size else np.zeros(0, np.int64))
    prog.append(int(pf_optional))
    prog.append(int(fp_cover))
    prog.append(int(n_rmax))
    prog.append(n_small_noninl)
    prog.append(int(in_inline_ok))
    prog.append(int(n_em_pre))
    for (lo, hi), fz in zip(em_ranges, em_fusable):
        prog += [int(lo), int(hi), int(fz)]
    # shared-pmf groups (ordered last) updated inline by the input-flow pass
    prog += [n_shared_inline if shared_inline_ok else 0]
    # tile blocks of more than EM_RT 32 x 32 tiles take the split EM kernel
    # (pcb_tc.cu k_em_tiles32, EM_RT = 8)
    ntl = np.diff(tb["blk_tile_off"])
    prog.append(int(bool(np.any((tb["blk_km"] == 32) & (tb["blk_kn"] == 32) & (ntl > 8)))))
    # f_params range the shared-pmf input-flow kernel stores whole rows into
    # (one CTA per pmf, plain stores): when contiguous, the backward pass's
    # zero fill skips it
    sp_lo = sp_hi = 0
    if shared_pids:
        st = np.array(sorted(shared_pids), dtype=np.int64)
        ln = np.array([shared_pids[int(k)] for k in st], dtype=np.int64)
        if np.all(st[1:] == st[:-1] + ln[:-1]):
            sp_lo, sp_hi = int(st[0]), int(st[-1] + ln[-1])
    prog += [sp_lo, sp_hi]
    prog.append(MAGIC)
    info = {"prod_flows_optional": pf_optional, "fp_cover": fp_cover,
            "leaf_alias": alias_pad is not None,
            "pre_ratio_layers": int(sum(pre_ratio)), "em_fused_layers": int(sum(em_fusable)),
            "pf_fused_layers": int(sum(1 for f in fuse_id if f >= 0)),
            "em_fused_layer_ids": [li for li, f in enumerate(em_fusable) if f], "input_inline_em": in_inline_ok, "blob_elems": blob.size, "tc_super_rows": n_tc_rows, "mma_tiles": int(t_start.size),
            "em_tile_blocks": int(tb["blk_km"].size), "em_rest_groups": int(rest.size),
            "mma_elems": mma_elems, "scratch_rows": scratch_total, "slot_vb": slot_vb,
            "layer_flow_ranges": [tuple(int(v) for v in r) for r in layer_range],
            "shared_pmfs": len(shared_pids), "shared_pmf_inline_em": shared_inline_ok}
    return np.asarray(prog, dtype=np.int64), blob.array(), info


class DevicePlan:
    """Device tables + C plan handle + fp32 theta for one compiled circuit."""

    def __init__(self, compiled, device=None, *, tensor_cores: bool = True):
        import torch
        lib = _lib.load()
        self.device = torch.device(device if device is not None else "cuda")
        self.compiled = compiled
        self.tensor_cores = tensor_cores
        prog, blob, info = build_program(compiled, tensor_cores=tensor_cores)
        self.info = info
        self._prog = prog
        self.blob = torch.from_numpy(blob).to(self.device)
        handle = _lib.C.c_void_p()
        with torch.cuda.device(self.device):
            _lib.call("pcb_plan_create", prog.ctypes.data, prog.size, self.blob.data_ptr(),
                      self.blob.numel(), _lib.C.byref(handle))
        self.handle = handle
        self.theta = torch.empty(compiled.theta_size, dtype=torch.float32, device=self.device)
        _lib.call("pcb_plan_set_theta", handle, self.theta.data_ptr())
        # bf16 hi/lo tensor-core copies of theta (derived; refreshed after every update)
        self.mma = torch.zeros(max(info["mma_elems"], 8), dtype=torch.bfloat16, device=self.device)
        _lib.call("pcb_plan_set_mma", handle, self.mma.data_ptr(), info["mma_elems"])
        self.status = torch.zeros(4, dtype=torch.int32, device=self.device)
        self.num_layers = lib.pcb_plan_num_layers(handle)
        self.theta_source = None
        self.upload_theta(compiled.theta)

    def refresh_mma(self) -> None:
        """Re-derive the bf16 tensor-core tiles from ``self.theta`` (after any change)."""
        _lib.call("pcb_theta_refresh", self.handle, _lib.stream_handle(), self.theta.data_ptr())

    def upload_theta(self, theta) -> None:
        """Copy a host (numpy) or device theta into the plan's fp32 table."""
        import torch
        if isinstance(theta, np.ndarray):
            if theta.shape != (self.compiled.theta_size,):
                raise UsageError("parameter table shape mismatch")
            self.theta_finite = bool(np.all(np.isfinite(theta)))
            self.theta.copy_(torch.from_numpy(np.ascontiguousarray(theta, dtype=np.float32)))
        else:
            t = theta.to(device=self.device, dtype=torch.float32)
            if t.shape != (self.compiled.theta_size,):
                raise UsageError("parameter table shape mismatch")
            self.theta.copy_(t)
            self.theta_finite = bool(torch.isfinite(self.theta).all().item())
        self.theta_source = theta
        with torch.cuda.device(self.device):
            self.refresh_mma()

    def __del__(self):
        h = getattr(self, "handle", None)
        if h is not None and h.value:
            try:
                _lib.load().pcb_plan_destroy(h)
            except Exception:
                pass


def device_plan(compiled, device=None, *, tensor_cores: bool = True) -> DevicePlan:
    """The cached plan of ``compiled`` on ``device`` (built on first use)."""
    import torch
    dev = torch.device(device if device is not None else "cuda")
    if dev.type == "cuda" and dev.index is None:
        dev = torch.device("cuda", torch.cuda.current_device())
    if compiled._device_plans is None:
        compiled._device_plans = {}
    key = (str(dev), tensor_cores)
    plan = compiled._device_plans.get(key)
    if plan is None:
        plan = DevicePlan(compiled, dev, tensor_cores=tensor_cores)
        compiled._device_plans[key] = plan
    return plan
