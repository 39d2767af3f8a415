"""Exact grouping of ragged integer rows, vectorised.

The reference compiler dedupes rows (parent signatures, child-block sets,
tied tile patterns, simplex groups) through ``dict[bytes, ...]`` keyed by
``ndarray.tobytes()`` in first-occurrence order.  At BASELINE scale that is
millions of Python-level byte keys.  Here every row gets a 64-bit
polynomial hash (vectorised, wrapping uint64 arithmetic), rows are grouped
by hash, and every row is then compared element-wise with its group's
representative; only if a hash collision is detected do we fall back to
the exact byte-key path.  Group ids are numbered by first occurrence, which
is what the dict-insertion order of the reference gives.
"""
from __future__ import annotations

import numpy as np

_M1 = np.uint64(0x9E3779B97F4A7C15)
_M2 = np.uint64(0xBF58476D1CE4E5B9)
_M3 = np.uint64(0x94D049BB133111EB)


def _mix(x: np.ndarray) -> np.ndarray:
    """splitmix64 finaliser on a uint64 array."""
    with np.errstate(over="ignore"):
        z = x.astype(np.uint64) + _M1
        z = (z ^ (z >> np.uint64(30))) * _M2
        z = (z ^ (z >> np.uint64(27))) * _M3
        return z ^ (z >> np.uint64(31))


def _number_by_first(keys: np.ndarray):
    _, first, inv = np.unique(keys, return_index=True, return_inverse=True)
    order = np.argsort(first, kind="stable")
    rank = np.empty(order.size, dtype=np.int64)
    rank[order] = np.arange(order.size)
    return rank[inv.ravel()], first[order]


def group_rows(flat: np.ndarray, offs: np.ndarray):
    """Group rows ``flat[offs[i]:offs[i+1]]`` by exact content.

    Returns ``(gid, first)``: group id per row (numbered by first occurrence)
    and the first row index of every group.
    """
    offs = np.asarray(offs, dtype=np.int64)
    n = offs.size - 1
    if n <= 0:
        return np.zeros(0, dtype=np.int64), np.zeros(0, dtype=np.int64)
    flat = np.ascontiguousarray(flat, dtype=np.int64)
    lengths = np.diff(offs)
    with np.errstate(over="ignore"):
        pos = np.arange(flat.size, dtype=np.int64) - np.repeat(offs[:-1], lengths)
        contrib = _mix(flat.view(np.uint64) ^ _mix(pos.astype(np.uint64)))
        h = np.zeros(n, dtype=np.uint64)
        nz = lengths > 0
        if flat.size:
            sums = np.add.reduceat(contrib, offs[:-1][nz]) if nz.any() else np.zeros(0, np.uint64)
            h[nz] = sums
        key = _mix(h ^ _mix(lengths.astype(np.uint64) * _M3))
    gid, first = _number_by_first(key)
    rep = first[gid]
    ok = np.array_equal(lengths[rep], lengths)
    if ok and flat.size:
        rep_pos = np.repeat(offs[rep], lengths) + pos
        ok = np.array_equal(flat[rep_pos], flat)
    if ok:
        return gid, first
    return _group_rows_exact(flat, offs)


def group_matrix_rows(mat: np.ndarray):
    """``group_rows`` for a dense (n, w) matrix."""
    mat = np.ascontiguousarray(mat, dtype=np.int64)
    n, w = mat.shape
    return group_rows(mat.ravel(), np.arange(n + 1, dtype=np.int64) * w)


def _group_rows_exact(flat, offs):
    seen: dict[bytes, int] = {}
    gid = np.empty(offs.size - 1, dtype=np.int64)
    first = []
    for i in range(offs.size - 1):
        k = flat[offs[i]:offs[i + 1]].tobytes()
        g = seen.get(k)
        if g is None:
            g = len(first)
            seen[k] = g
            first.append(i)
        gid[i] = g
    return gid, np.asarray(first, dtype=np.int64)


def row_hashes(mat: np.ndarray) -> np.ndarray:
    """64-bit content hash per row of a dense int64 matrix (for cross-call dedupe)."""
    mat = np.ascontiguousarray(mat, dtype=np.int64)
    n, w = mat.shape
    with np.errstate(over="ignore"):
        pos = _mix(np.arange(w, dtype=np.uint64))[None, :]
        contrib = _mix(mat.view(np.uint64) ^ pos)
        h = contrib.sum(axis=1, dtype=np.uint64)
        return _mix(h ^ _mix(np.full(n, w, dtype=np.uint64) * _M3))
