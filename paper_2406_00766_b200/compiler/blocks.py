"""Connectivity-class block detection for one sum layer.

Contract (``pcirc/compiler/blocks.py:73-148``, Appendix A of SURVEY.md):

* products are classed by their sorted parent list; classes appear in the
  order of first occurrence over ascending product key; members ascend;
* sums are classed by their sorted set of child blocks, first occurrence
  over the given sum order;
* classes are chunked into ``k``-sized blocks, tails padded with ``PAD``;
* ``k_n = min(k_n, pow2_floor(#product keys))``, ``k_m = min(k, pow2_floor(#sums))``;
* if either padding fraction exceeds ``demote_threshold`` the layer is
  re-blocked at 1x1 and marked demoted.

Everything is computed on flat arrays (one lexsort + hashed grouping), so
a 100 M-edge HCLT layer blocks in seconds.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from ..errors import UsageError
from ._rows import group_rows

PAD = -1


def pow2_floor(n: int) -> int:
    if n < 1:
        raise UsageError(f"pow2_floor needs a positive value, got {n}")
    return 1 << (int(n).bit_length() - 1)


@dataclass
class BlockLayout:
    k_m: int
    k_n: int
    demoted: bool
    sum_block_mat: np.ndarray    # (n_sb, k_m) sum keys, PAD padded
    prod_block_mat: np.ndarray   # (n_pb, k_n) product keys, PAD padded
    cb_flat: np.ndarray          # child blocks per sum block, CSR
    cb_off: np.ndarray
    sum_keys: np.ndarray         # sorted sum keys -> (block, offset)
    sum_blk: np.ndarray
    sum_off: np.ndarray
    prod_keys: np.ndarray        # sorted product keys -> (block, offset)
    prod_blk: np.ndarray
    prod_off: np.ndarray
    sum_pad_fraction: float
    prod_pad_fraction: float
    _cache: dict = field(default_factory=dict, repr=False)

    # reference-compatible views --------------------------------------------
    @property
    def sum_blocks(self) -> list:
        return list(self.sum_block_mat)

    @property
    def prod_blocks(self) -> list:
        return list(self.prod_block_mat)

    @property
    def child_blocks(self) -> list:
        return [self.cb_flat[self.cb_off[i]:self.cb_off[i + 1]]
                for i in range(self.cb_off.size - 1)]

    @property
    def sum_block_of(self) -> dict:
        return {int(k): (int(b), int(o)) for k, b, o in
                zip(self.sum_keys, self.sum_blk, self.sum_off)}

    @property
    def prod_block_of(self) -> dict:
        return {int(k): (int(b), int(o)) for k, b, o in
                zip(self.prod_keys, self.prod_blk, self.prod_off)}

    @property
    def pairs(self) -> list:
        sb = np.repeat(np.arange(self.cb_off.size - 1), np.diff(self.cb_off))
        return list(zip(sb.tolist(), self.cb_flat.tolist()))


def _chunk(keys: np.ndarray, gid: np.ndarray, n_groups: int, k: int):
    """Chunk classes (gid, first-occurrence numbered) into k-blocks.

    ``keys`` are in the within-class member order (class members keep the
    order in which they appear in ``keys``).  Returns the block matrix, and
    per input key its (block, offset), plus the pad fraction.
    """
    order = np.argsort(gid, kind="stable")
    sizes = np.bincount(gid, minlength=n_groups)
    nblk = (sizes + k - 1) // k
    blk_base = np.concatenate([[0], np.cumsum(nblk)[:-1]]).astype(np.int64)
    cls_base = np.concatenate([[0], np.cumsum(sizes)[:-1]]).astype(np.int64)
    g_sorted = gid[order]
    rank = np.arange(order.size, dtype=np.int64) - cls_base[g_sorted]
    blk = np.empty(keys.size, dtype=np.int64)
    off = np.empty(keys.size, dtype=np.int64)
    blk[order] = blk_base[g_sorted] + rank // k
    off[order] = rank % k
    total_blocks = int(nblk.sum())
    mat = np.full((total_blocks, k), PAD, dtype=np.int64)
    mat[blk, off] = keys
    total = total_blocks * k
    pad = (total - keys.size) / total if total else 0.0
    return mat, blk, off, pad


def detect_blocks_csr(sum_ids, ch_flat, ch_off, k: int, k_n: int | None = None,
                      demote_threshold: float = 0.5) -> BlockLayout:
    """Block one layer given each sum's child keys as CSR (``ch_flat``/``ch_off``)."""
    if k < 1 or (k_n is not None and k_n < 1):
        raise UsageError(f"block size must be >= 1, got {k}/{k_n}")
    sum_ids = np.asarray(sum_ids, dtype=np.int64)
    z = np.zeros(0, dtype=np.int64)
    if sum_ids.size == 0:
        return BlockLayout(1, 1, False, np.zeros((0, 1), np.int64), np.zeros((0, 1), np.int64),
                           z, np.zeros(1, np.int64), z, z, z, z, z, z, 0.0, 0.0)
    ch_flat = np.asarray(ch_flat, dtype=np.int64)
    ch_off = np.asarray(ch_off, dtype=np.int64)
    sizes = np.diff(ch_off)
    parents = np.repeat(sum_ids, sizes)
    prod_keys = np.unique(ch_flat)

    kn = min(k if k_n is None else k_n, pow2_floor(prod_keys.size))
    km = min(k, pow2_floor(sum_ids.size))

    # product classes: sorted parent list per product key
    order = np.lexsort((parents, ch_flat))
    sc = ch_flat[order]
    sp = parents[order]
    run_off = np.concatenate([np.searchsorted(sc, prod_keys, side="left"), [sc.size]])
    pgid, pfirst = group_rows(sp, run_off)
    pmat, pblk, poff, ppad = _chunk(prod_keys, pgid, pfirst.size, kn)

    # sum classes: sorted unique child-block set per sum, in given sum order
    cblk = pblk[np.searchsorted(prod_keys, ch_flat)]
    row = np.repeat(np.arange(sum_ids.size, dtype=np.int64), sizes)
    o2 = np.lexsort((cblk, row))
    r2, b2 = row[o2], cblk[o2]
    keep = np.ones(r2.size, dtype=bool)
    keep[1:] = (r2[1:] != r2[:-1]) | (b2[1:] != b2[:-1])
    r2, b2 = r2[keep], b2[keep]
    cbs_off = np.concatenate([[0], np.cumsum(np.bincount(r2, minlength=sum_ids.size))])
    sgid, sfirst = group_rows(b2, cbs_off)
    smat, sblk, soff, spad = _chunk(sum_ids, sgid, sfirst.size, km)

    if max(spad, ppad) > demote_threshold and max(km, kn) > 1:
        lo = detect_blocks_csr(sum_ids, ch_flat, ch_off, 1, 1, demote_threshold)
        lo.demoted = True
        return lo

    # child blocks of each sum block = those of its first member
    first_member_row = np.searchsorted(sum_ids, smat[:, 0]) if np.all(np.diff(sum_ids) > 0) \
        else _index_of(sum_ids, smat[:, 0])
    lens = np.diff(cbs_off)[first_member_row]
    cb_off = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    starts = cbs_off[first_member_row]
    idx = np.repeat(starts, lens) + (np.arange(int(lens.sum())) - np.repeat(cb_off[:-1], lens))
    cb_flat = b2[idx]

    s_order = np.argsort(sum_ids, kind="stable")
    return BlockLayout(km, kn, False, smat, pmat, cb_flat, cb_off,
                       sum_ids[s_order], sblk[s_order], soff[s_order],
                       prod_keys, pblk, poff, spad, ppad)


def _index_of(keys, query):
    order = np.argsort(keys, kind="stable")
    return order[np.searchsorted(keys[order], query)]


def detect_blocks(sum_ids, sum_children, k: int, k_n: int | None = None,
                  demote_threshold: float = 0.5) -> BlockLayout:
    """Reference signature: ``sum_children`` is a list of per-sum key arrays."""
    children = [np.asarray(c, dtype=np.int64) for c in sum_children]
    off = np.concatenate([[0], np.cumsum([c.size for c in children])]).astype(np.int64)
    flat = np.concatenate(children) if children else np.zeros(0, dtype=np.int64)
    return detect_blocks_csr(sum_ids, flat, off, k, k_n, demote_threshold)
