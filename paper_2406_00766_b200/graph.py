"""Circuit construction API (drop-in for ``pcirc/graph.py``).

Same public surface as the reference builder (``graph.py:82-524``):
``CircuitGraph.add_input / add_product / add_sum / tie / set_root /
validate / freeze``, ``g.nodes[i]`` views with ``children`` / ``slots`` /
``var`` / ``num_categories`` / ``slot``, a flat logical parameter pool with
structural tying through shared slots.

Storage is different.  The reference keeps one Python object per node; at
the BASELINE scales (HCLT-256: 2.4 M nodes / 201 M edges, HMM-4096: 520 M
edges) that makes compilation the bottleneck.  Here nodes live in
*segments*: every ``add_*`` call (single node) or ``add_*s`` bulk call
(many nodes of one kind with a uniform fan-in) appends one segment whose
children / slots are a 2-d int64 matrix.  Bulk matrices may be broadcast
views (an HMM layer's 4096 sums share one child row), so memory stays
proportional to the distinct data.  The compiler walks segments with
vectorised numpy instead of per-node Python.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Iterable, Sequence

import numpy as np

from .errors import CircuitValidationError

SIMPLEX_TOL = 1e-9

KIND_INPUT, KIND_PRODUCT, KIND_SUM = 0, 1, 2


@dataclass
class InputNode:
    id: int
    var: int
    num_categories: int
    slot: int  # first of num_categories consecutive logical slots


@dataclass
class ProductNode:
    id: int
    children: np.ndarray


@dataclass
class SumNode:
    id: int
    children: np.ndarray
    slots: np.ndarray


Node = InputNode | ProductNode | SumNode


@dataclass
class Violation:
    code: str
    nodes: tuple[int, ...]
    message: str

    def __str__(self) -> str:
        return f"[{self.code}] {self.message}"


@dataclass
class ValidationReport:
    violations: list[Violation]

    @property
    def ok(self) -> bool:
        return not self.violations

    def __str__(self) -> str:
        return "valid" if self.ok else "\n".join(str(v) for v in self.violations)

    def raise_if_invalid(self) -> None:
        if not self.ok:
            raise CircuitValidationError(str(self))


@dataclass
class Segment:
    """A run of consecutive node ids of one kind.

    inputs:   ``var``, ``ncat``, ``slot`` are (n,) arrays.
    products: ``children`` is (n, fan_in).
    sums:     ``children`` and ``slots`` are (n, fan_in).
    ``dep`` is the largest child id (-1 for inputs): segments whose
    dependencies all precede their first id can be processed in order.
    """

    kind: int
    start: int
    count: int
    children: np.ndarray | None = None
    slots: np.ndarray | None = None
    var: np.ndarray | None = None
    ncat: np.ndarray | None = None
    slot: np.ndarray | None = None
    dep: int = -1

    @property
    def stop(self) -> int:
        return self.start + self.count

    @property
    def fan_in(self) -> int:
        return 0 if self.children is None else int(self.children.shape[1])


def _as_ids(ids) -> np.ndarray:
    arr = np.asarray(ids, dtype=np.int64)
    if arr.ndim != 1 or arr.size == 0:
        raise CircuitValidationError("child list must be a non-empty 1-d sequence")
    return arr


class _NodeView(Sequence):
    """Read-only ``g.nodes`` sequence materialising node records on demand."""

    def __init__(self, g: "CircuitGraph"):
        self._g = g

    def __len__(self) -> int:
        return self._g.num_nodes

    def __getitem__(self, i):
        if isinstance(i, slice):
            return [self[j] for j in range(*i.indices(len(self)))]
        n = len(self)
        i = int(i)
        if i < 0:
            i += n
        if not 0 <= i < n:
            raise IndexError(i)
        seg = self._g._segment_of(i)
        r = i - seg.start
        if seg.kind == KIND_INPUT:
            return InputNode(i, int(seg.var[r]), int(seg.ncat[r]), int(seg.slot[r]))
        if seg.kind == KIND_PRODUCT:
            return ProductNode(i, seg.children[r])
        return SumNode(i, seg.children[r], seg.slots[r])

    def __iter__(self):
        for seg in self._g.segments:
            for r in range(seg.count):
                i = seg.start + r
                if seg.kind == KIND_INPUT:
                    yield InputNode(i, int(seg.var[r]), int(seg.ncat[r]), int(seg.slot[r]))
                elif seg.kind == KIND_PRODUCT:
                    yield ProductNode(i, seg.children[r])
                else:
                    yield SumNode(i, seg.children[r], seg.slots[r])


class CircuitGraph:
    """Mutable circuit builder; ``freeze()`` locks the structure."""

    def __init__(self, num_vars: int):
        if num_vars < 1:
            raise CircuitValidationError(f"num_vars must be >= 1, got {num_vars}")
        self.num_vars = int(num_vars)
        self.segments: list[Segment] = []
        self.tying: dict[int, int] = {}
        self._params = np.zeros(64, dtype=np.float64)
        self._num_slots = 0
        self._num_nodes = 0
        self._root: int | None = None
        self._frozen = False
        # True once any node reuses explicit slots (structural tying); together
        # with an empty ``tying`` map this lets the compiler skip the tying
        # alignment check, which cannot fail when every slot has one use
        self.shares_slots = False
        self._starts_cache: np.ndarray | None = None
        self._kind_cache: np.ndarray | None = None

    # -- parameter pool ---------------------------------------------------
    @property
    def num_param_slots(self) -> int:
        return self._num_slots

    @property
    def params(self) -> np.ndarray:
        return self._params[: self._num_slots]

    def _alloc_slots(self, n: int) -> int:
        start = self._num_slots
        need = start + n
        if need > self._params.size:
            grown = np.zeros(max(need, 2 * self._params.size), dtype=np.float64)
            grown[:start] = self._params[:start]
            self._params = grown
        self._num_slots = need
        return start

    def set_param_values(self, slots, values) -> None:
        """Write parameter values; allowed on frozen graphs (EM write-back)."""
        self._params[np.asarray(slots, dtype=np.int64)] = values

    # -- structure bookkeeping -------------------------------------------
    def _check_mutable(self) -> None:
        if self._frozen:
            raise CircuitValidationError("graph is frozen; structure cannot change")

    def _push(self, seg: Segment) -> np.ndarray:
        self.segments.append(seg)
        self._num_nodes += seg.count
        self._starts_cache = None
        self._kind_cache = None
        return np.arange(seg.start, seg.stop, dtype=np.int64)

    def _check_children(self, ch: np.ndarray) -> None:
        if ch.size and (ch.min() < 0 or ch.max() >= self._num_nodes):
            raise CircuitValidationError(
                f"child id out of range (have {self._num_nodes} nodes)"
            )

    def _segment_of(self, nid: int) -> Segment:
        if self._starts_cache is None:
            self._starts_cache = np.array([s.start for s in self.segments], dtype=np.int64)
        k = int(np.searchsorted(self._starts_cache, nid, side="right")) - 1
        return self.segments[k]

    # -- single-node construction (reference API) --------------------------
    def add_input(self, var: int, pmf=None, *, slot: int | None = None,
                  num_categories: int | None = None) -> int:
        """Categorical input node (``graph.py:135-175``)."""
        self._check_mutable()
        if not 0 <= var < self.num_vars:
            raise CircuitValidationError(f"var {var} out of range [0, {self.num_vars})")
        if pmf is not None:
            pmf = np.asarray(pmf, dtype=np.float64)
            if pmf.ndim != 1 or pmf.size < 1:
                raise CircuitValidationError("pmf must be a non-empty vector")
            if pmf.min() < 0 or abs(pmf.sum() - 1.0) > SIMPLEX_TOL:
                raise CircuitValidationError(
                    f"pmf for var {var} is not on the probability simplex")
            ncat = pmf.size
            if num_categories is not None and num_categories != ncat:
                raise CircuitValidationError("num_categories disagrees with pmf length")
        elif num_categories is not None:
            ncat = int(num_categories)
        else:
            raise CircuitValidationError("add_input needs a pmf or num_categories")
        if slot is None:
            slot = self._alloc_slots(ncat)
        elif slot < 0 or slot + ncat > self._num_slots:
            raise CircuitValidationError("input slot range not allocated")
        else:
            self.shares_slots = True
        if pmf is not None:
            self._params[slot:slot + ncat] = pmf
        seg = Segment(KIND_INPUT, self._num_nodes, 1,
                      var=np.array([var], dtype=np.int64),
                      ncat=np.array([ncat], dtype=np.int64),
                      slot=np.array([slot], dtype=np.int64))
        return int(self._push(seg)[0])

    def add_product(self, children) -> int:
        self._check_mutable()
        ch = _as_ids(children)
        self._check_children(ch)
        seg = Segment(KIND_PRODUCT, self._num_nodes, 1, children=ch[None, :],
                      dep=int(ch.max()))
        return int(self._push(seg)[0])

    def add_sum(self, children, params=None, *, slots=None) -> int:
        """Sum node (``graph.py:186-223``): fresh slots from ``params`` or shared ``slots``."""
        self._check_mutable()
        ch = _as_ids(children)
        self._check_children(ch)
        if params is not None:
            params = np.asarray(params, dtype=np.float64)
            if params.shape != ch.shape:
                raise CircuitValidationError("one parameter per child edge required")
            if params.min() < 0 or abs(params.sum() - 1.0) > SIMPLEX_TOL:
                raise CircuitValidationError("sum weights are not on the simplex")
        if slots is None:
            if params is None:
                raise CircuitValidationError("add_sum needs params or slots")
            start = self._alloc_slots(ch.size)
            slot_arr = np.arange(start, start + ch.size, dtype=np.int64)
        else:
            self.shares_slots = True
            slot_arr = np.asarray(slots, dtype=np.int64)
            if slot_arr.shape != ch.shape:
                raise CircuitValidationError("one slot per child edge required")
            if slot_arr.min() < 0 or slot_arr.max() >= self._num_slots:
                raise CircuitValidationError("sum slot out of allocated range")
        if params is not None:
            self._params[slot_arr] = params
        seg = Segment(KIND_SUM, self._num_nodes, 1, children=ch[None, :],
                      slots=slot_arr[None, :], dep=int(ch.max()))
        return int(self._push(seg)[0])

    # -- bulk construction (generators at BASELINE scale) -------------------
    def add_inputs(self, var, pmfs=None, *, slots=None, num_categories=None) -> np.ndarray:
        """Add many inputs sharing one category count.

        ``pmfs`` is (n, ncat) (fresh contiguous slot ranges, one per row) or
        None with explicit ``slots`` (n,) starts + ``num_categories``.
        """
        self._check_mutable()
        var = np.asarray(var, dtype=np.int64).ravel()
        n = var.size
        if n == 0:
            return np.zeros(0, dtype=np.int64)
        if var.min() < 0 or var.max() >= self.num_vars:
            raise CircuitValidationError("input var out of range")
        if pmfs is not None:
            pmfs = np.asarray(pmfs, dtype=np.float64)
            if pmfs.ndim != 2 or pmfs.shape[0] != n:
                raise CircuitValidationError("pmfs must be (n, ncat)")
            ncat = pmfs.shape[1]
            if pmfs.min() < 0 or np.any(np.abs(pmfs.sum(axis=1) - 1.0) > SIMPLEX_TOL):
                raise CircuitValidationError("input pmf is not on the probability simplex")
        elif num_categories is not None:
            ncat = int(num_categories)
        else:
            raise CircuitValidationError("add_inputs needs pmfs or num_categories")
        if slots is None:
            base = self._alloc_slots(n * ncat)
            slot = base + ncat * np.arange(n, dtype=np.int64)
        else:
            self.shares_slots = True
            slot = np.broadcast_to(np.asarray(slots, dtype=np.int64), (n,)).copy()
            if slot.min() < 0 or slot.max() + ncat > self._num_slots:
                raise CircuitValidationError("input slot range not allocated")
        if pmfs is not None:
            idx = slot[:, None] + np.arange(ncat)
            self._params[idx] = pmfs
        seg = Segment(KIND_INPUT, self._num_nodes, n, var=var,
                      ncat=np.full(n, ncat, dtype=np.int64), slot=slot)
        return self._push(seg)

    def add_products(self, children) -> np.ndarray:
        """Add many products of equal fan-in; ``children`` is (n, fan_in)."""
        self._check_mutable()
        ch = np.asarray(children, dtype=np.int64)
        if ch.ndim != 2 or ch.shape[1] == 0:
            raise CircuitValidationError("children must be (n, fan_in)")
        if ch.shape[0] == 0:
            return np.zeros(0, dtype=np.int64)
        self._check_children(ch)
        seg = Segment(KIND_PRODUCT, self._num_nodes, ch.shape[0], children=ch,
                      dep=int(ch.max()))
        return self._push(seg)

    def add_sums(self, children, params=None, *, slots=None) -> np.ndarray:
        """Add many sums of equal fan-in; ``children``/``params``/``slots`` are (n, fan_in).

        ``children`` and ``slots`` may be broadcast views (shared rows).
        """
        self._check_mutable()
        ch = np.asarray(children, dtype=np.int64)
        if ch.ndim != 2 or ch.shape[1] == 0:
            raise CircuitValidationError("children must be (n, fan_in)")
        n, f = ch.shape
        if n == 0:
            return np.zeros(0, dtype=np.int64)
        self._check_children(ch)
        if params is not None:
            params = np.asarray(params, dtype=np.float64)
            if params.shape != ch.shape:
                raise CircuitValidationError("one parameter per child edge required")
            if params.min() < 0 or np.any(np.abs(params.sum(axis=1) - 1.0) > SIMPLEX_TOL):
                raise CircuitValidationError("sum weights are not on the simplex")
        if slots is None:
            if params is None:
                raise CircuitValidationError("add_sums needs params or slots")
            base = self._alloc_slots(n * f)
            sl = base + np.arange(n * f, dtype=np.int64).reshape(n, f)
        else:
            self.shares_slots = True
            sl = np.asarray(slots, dtype=np.int64)
            if sl.shape != ch.shape:
                sl = np.broadcast_to(sl, ch.shape)
            if sl.min() < 0 or sl.max() >= self._num_slots:
                raise CircuitValidationError("sum slot out of allocated range")
        if params is not None:
            self._params[sl] = params
        seg = Segment(KIND_SUM, self._num_nodes, n, children=ch, slots=sl,
                      dep=int(ch.max()))
        return self._push(seg)

    # -- tying / root / freeze ---------------------------------------------
    def tie(self, slots: Iterable[int], group: int | None = None) -> int:
        self._check_mutable()
        if group is None:
            group = (max(self.tying.values()) + 1) if self.tying else 0
        for s in slots:
            if not 0 <= s < self._num_slots:
                raise CircuitValidationError(f"tie slot {s} not allocated")
            self.tying[int(s)] = int(group)
        return group

    def set_root(self, node_id: int) -> None:
        self._check_mutable()
        if not 0 <= node_id < self._num_nodes:
            raise CircuitValidationError(f"root id {node_id} out of range")
        self._root = int(node_id)

    @property
    def root(self) -> int:
        if self._num_nodes == 0:
            raise CircuitValidationError("empty graph has no root")
        return self._root if self._root is not None else self._num_nodes - 1

    def freeze(self) -> None:
        self._frozen = True

    @property
    def frozen(self) -> bool:
        return self._frozen

    # -- derived structure ----------------------------------------------------
    @property
    def nodes(self) -> _NodeView:
        return _NodeView(self)

    @property
    def num_nodes(self) -> int:
        return self._num_nodes

    @property
    def num_edges(self) -> int:
        return int(sum(s.count * s.fan_in for s in self.segments if s.kind != KIND_INPUT))

    def node_kinds(self) -> np.ndarray:
        if self._kind_cache is None:
            k = np.empty(self._num_nodes, dtype=np.int8)
            for s in self.segments:
                k[s.start:s.stop] = s.kind
            self._kind_cache = k
        return self._kind_cache

    def input_table(self):
        """(ids, var, ncat, slot) of every input, ascending id."""
        segs = [s for s in self.segments if s.kind == KIND_INPUT]
        if not segs:
            z = np.zeros(0, dtype=np.int64)
            return z, z, z, z
        ids = np.concatenate([np.arange(s.start, s.stop) for s in segs])
        return (ids, np.concatenate([s.var for s in segs]),
                np.concatenate([s.ncat for s in segs]),
                np.concatenate([s.slot for s in segs]))

    def parent_counts(self) -> np.ndarray:
        counts = np.zeros(self._num_nodes, dtype=np.int64)
        for s in self.segments:
            if s.kind != KIND_INPUT:
                counts += np.bincount(np.asarray(s.children).ravel(),
                                      minlength=self._num_nodes)
        return counts

    def _ordered(self) -> bool:
        """True when every segment only references earlier nodes."""
        return all(s.dep < s.start for s in self.segments)

    def topological_order(self) -> list[int]:
        if self._ordered():
            return list(range(self._num_nodes))
        order = self._kahn()
        if len(order) != self._num_nodes:
            raise CircuitValidationError("cycle detected in circuit graph")
        return order

    def _kahn(self) -> list[int]:
        n = self._num_nodes
        remaining = np.zeros(n, dtype=np.int64)
        parents: list[list[int]] = [[] for _ in range(n)]
        for node in self.nodes:
            if isinstance(node, InputNode):
                continue
            remaining[node.id] = node.children.size
            for c in node.children.tolist():
                parents[c].append(node.id)
        stack = [i for i in range(n) if remaining[i] == 0]
        order: list[int] = []
        while stack:
            nid = stack.pop()
            order.append(nid)
            for p in parents[nid]:
                remaining[p] -= 1
                if remaining[p] == 0:
                    stack.append(p)
        return order

    def depths(self) -> np.ndarray:
        """Topological depth: inputs 0, else 1 + max child depth (``build.py:103-110``)."""
        depth = np.zeros(self._num_nodes, dtype=np.int64)
        if self._ordered():
            from .compiler import _native
            nat = _native.lib()
            if nat is not None and self.segments:
                segs = self.segments
                ch = [None if s.kind == KIND_INPUT else _native.rows(s.children) for s in segs]
                rs = np.array([0 if c is None else c[1] for c in ch], np.int64)
                st = np.array([s.start for s in segs], np.int64)
                cn = np.array([s.count for s in segs], np.int64)
                fn = np.array([s.fan_in for s in segs], np.int64)
                kd = np.array([s.kind for s in segs], np.int8)
                tab = _native.addr_array([0 if c is None else _native.addr(c[0]) for c in ch])
                nat.pcc_depths(len(segs), _native.ptr(st), _native.ptr(cn), _native.ptr(fn),
                               _native.ptr(kd), _native.ptr(tab), _native.ptr(rs),
                               _native.ptr(depth))
                return depth
            for s in self.segments:
                if s.kind != KIND_INPUT:
                    depth[s.start:s.stop] = 1 + depth[s.children].max(axis=1)
            return depth
        for nid in self.topological_order():
            node = self.nodes[nid]
            if not isinstance(node, InputNode):
                depth[nid] = 1 + int(depth[node.children].max())
        return depth

    def var_categories(self) -> np.ndarray:
        cats = np.zeros(self.num_vars, dtype=np.int64)
        _, var, ncat, _ = self.input_table()
        if var.size:
            np.maximum.at(cats, var, ncat)
        return cats

    def scope_masks(self) -> list[int]:
        masks = [0] * self._num_nodes
        for nid in self.topological_order():
            node = self.nodes[nid]
            if isinstance(node, InputNode):
                masks[nid] = 1 << node.var
            else:
                m = 0
                for c in node.children.tolist():
                    m |= masks[c]
                masks[nid] = m
        return masks

    def scope(self, node_id: int) -> frozenset[int]:
        mask = self.scope_masks()[node_id]
        return frozenset(v for v in range(self.num_vars) if mask >> v & 1)

    # -- validation ---------------------------------------------------------
    def validate(self) -> ValidationReport:
        """Structural contract check (``graph.py:336-501``); never raises.

        Same violation codes as the reference.  Scopes are interned to ids so
        smoothness of a wide sum is one vectorised comparison.
        """
        v: list[Violation] = []
        n = self._num_nodes
        if n == 0:
            return ValidationReport([Violation("empty", (), "graph has no nodes")])
        ordered = self._ordered()
        if not ordered:
            order = self._kahn()
            if len(order) != n:
                done = set(order)
                bad = tuple(i for i in range(n) if i not in done)
                v.append(Violation("cycle", bad, f"cycle through nodes {bad[:8]}"))
        else:
            order = None
        acyclic = ordered or len(order) == n

        root = self.root
        pc = self.parent_counts()
        if pc[root] > 0:
            v.append(Violation("root_has_parents", (root,), "root node has parents"))
        orphan_mask = pc == 0
        orphan_mask[root] = False
        orphans = tuple(np.flatnonzero(orphan_mask).tolist())
        if orphans:
            v.append(Violation("multi_root", orphans,
                               f"{len(orphans)} non-root node(s) have no parents"))

        reach = self._reachable(root)
        unreach_mask = ~reach & (pc > 0)
        unreach_mask[root] = False
        unreachable = tuple(np.flatnonzero(unreach_mask).tolist())
        if unreachable:
            v.append(Violation("unreachable", unreachable,
                               f"{len(unreachable)} node(s) unreachable from root"))

        kinds = self.node_kinds()
        for s in self.segments:
            if s.kind == KIND_INPUT:
                continue
            ck = kinds[s.children]
            bad_kind = KIND_SUM if s.kind == KIND_SUM else KIND_PRODUCT
            rows = np.flatnonzero((ck == bad_kind).any(axis=1))
            for r in rows.tolist():
                nid = s.start + r
                what = "sum" if s.kind == KIND_SUM else "product"
                v.append(Violation("alternation", (nid,),
                                   f"{what} {nid} has a {what} child"))

        ids, var, ncat, slot = self.input_table()
        seen: dict[int, int] = {}
        for nid, vv, nc in zip(ids.tolist(), var.tolist(), ncat.tolist()):
            prev = seen.setdefault(vv, nc)
            if prev != nc:
                v.append(Violation("var_categories", (nid,),
                                   f"var {vv} has inputs with {prev} and {nc} categories"))

        params = self.params
        for s in self.segments:
            if s.kind == KIND_INPUT:
                for r in range(s.count):
                    pmf = params[s.slot[r]:s.slot[r] + s.ncat[r]]
                    if pmf.size == 0 or pmf.min() < 0 or abs(pmf.sum() - 1.0) > SIMPLEX_TOL:
                        nid = s.start + r
                        v.append(Violation("simplex", (nid,),
                                           f"input {nid} pmf off the simplex "
                                           f"(sum={pmf.sum():.12g})"))
            elif s.kind == KIND_SUM:
                w = params[s.slots]
                tot = w.sum(axis=1)
                bad = (w.min(axis=1) < 0) | (np.abs(tot - 1.0) > SIMPLEX_TOL)
                for r in np.flatnonzero(bad).tolist():
                    nid = s.start + r
                    v.append(Violation("simplex", (nid,),
                                       f"sum {nid} weights off the simplex "
                                       f"(sum={tot[r]:.12g})"))

        if acyclic:
            v.extend(self._scope_violations(root))
        return ValidationReport(v)

    def _reachable(self, root: int) -> np.ndarray:
        reach = np.zeros(self._num_nodes, dtype=bool)
        reach[root] = True
        if self._ordered():
            # reverse sweep over segments: a node is reachable if some reachable
            # parent lists it (parents always have larger ids here)
            for s in reversed(self.segments):
                if s.kind == KIND_INPUT:
                    continue
                live = reach[s.start:s.stop]
                if live.any():
                    reach[np.asarray(s.children)[live].ravel()] = True
            return reach
        stack = [root]
        nodes = self.nodes
        while stack:
            node = nodes[stack.pop()]
            if isinstance(node, InputNode):
                continue
            for c in node.children.tolist():
                if not reach[c]:
                    reach[c] = True
                    stack.append(c)
        return reach

    def _scope_violations(self, root: int) -> list[Violation]:
        """Decomposability / smoothness / root scope with interned scopes."""
        v: list[Violation] = []
        n = self._num_nodes
        scope_id = np.full(n, -1, dtype=np.int64)
        masks: list[int] = []
        intern: dict[int, int] = {}

        def sid_of(mask: int) -> int:
            k = intern.get(mask)
            if k is None:
                k = len(masks)
                intern[mask] = k
                masks.append(mask)
            return k

        order_segments = self.segments if self._ordered() else None
        if order_segments is None:
            # arbitrary ids: node-at-a-time in topological order
            for nid in self._kahn():
                node = self.nodes[nid]
                self._scope_one(node, scope_id, masks, sid_of, v)
        else:
            for s in order_segments:
                if s.kind == KIND_INPUT:
                    for r in range(s.count):
                        scope_id[s.start + r] = sid_of(1 << int(s.var[r]))
                elif s.kind == KIND_SUM:
                    cs = scope_id[s.children]
                    first = cs[:, 0]
                    bad = (cs != first[:, None]).any(axis=1)
                    scope_id[s.start:s.stop] = first
                    for r in np.flatnonzero(bad).tolist():
                        nid = s.start + r
                        v.append(Violation("smoothness", (nid,),
                                           f"sum {nid} children have unequal scopes"))
                        m = 0
                        for c in s.children[r].tolist():
                            m |= masks[scope_id[c]]
                        scope_id[nid] = sid_of(m)
                else:
                    cs = scope_id[s.children]
                    # rows with identical child-scope tuples share the answer
                    uniq, inv = np.unique(cs, axis=0, return_inverse=True)
                    res = np.empty(uniq.shape[0], dtype=np.int64)
                    ok = np.empty(uniq.shape[0], dtype=bool)
                    for u in range(uniq.shape[0]):
                        m, good = 0, True
                        for c in uniq[u].tolist():
                            cm = masks[c]
                            if m & cm:
                                good = False
                            m |= cm
                        res[u] = sid_of(m)
                        ok[u] = good
                    inv = inv.ravel()
                    scope_id[s.start:s.stop] = res[inv]
                    for r in np.flatnonzero(~ok[inv]).tolist():
                        nid = s.start + r
                        v.append(Violation("decomposability", (nid,),
                                           f"product {nid} children share variables"))
        full = (1 << self.num_vars) - 1
        rmask = masks[scope_id[root]]
        if rmask != full:
            missing = [x for x in range(self.num_vars) if not rmask >> x & 1]
            v.append(Violation("root_scope", (root,),
                               f"root scope misses variables {missing[:8]}"))
        return v

    @staticmethod
    def _scope_one(node, scope_id, masks, sid_of, v):
        if isinstance(node, InputNode):
            scope_id[node.id] = sid_of(1 << node.var)
            return
        m = 0
        if isinstance(node, ProductNode):
            good = True
            for c in node.children.tolist():
                cm = masks[scope_id[c]]
                if m & cm:
                    good = False
                m |= cm
            if not good:
                v.append(Violation("decomposability", (node.id,),
                                   f"product {node.id} children share variables"))
        else:
            first = scope_id[node.children[0]]
            if np.any(scope_id[node.children] != first):
                v.append(Violation("smoothness", (node.id,),
                                   f"sum {node.id} children have unequal scopes"))
            for c in node.children.tolist():
                m |= masks[scope_id[c]]
        scope_id[node.id] = sid_of(m)

    # -- interop ----------------------------------------------------------------
    @classmethod
    def from_parts(cls, num_vars: int, nodes: list, params, root=None, tying=None):
        """Assemble from node records (``graph.py:503-524``)."""
        g = cls(num_vars)
        for i, node in enumerate(nodes):
            if isinstance(node, InputNode):
                seg = Segment(KIND_INPUT, i, 1, var=np.array([node.var]),
                              ncat=np.array([node.num_categories]),
                              slot=np.array([node.slot]))
            elif isinstance(node, ProductNode):
                ch = np.asarray(node.children, dtype=np.int64)
                seg = Segment(KIND_PRODUCT, i, 1, children=ch[None, :], dep=int(ch.max()))
            else:
                ch = np.asarray(node.children, dtype=np.int64)
                seg = Segment(KIND_SUM, i, 1, children=ch[None, :],
                              slots=np.asarray(node.slots, dtype=np.int64)[None, :],
                              dep=int(ch.max()))
            g._push(seg)
        g.shares_slots = True  # unknown provenance
        g._params = np.asarray(params, dtype=np.float64).copy()
        g._num_slots = g._params.size
        if root is not None:
            if not 0 <= root < len(nodes):
                raise CircuitValidationError(f"root id {root} out of range")
            g._root = root
        if tying:
            g.tying = dict(tying)
        return g

    @classmethod
    def from_reference(cls, ref_graph) -> "CircuitGraph":
        """Convert a graph object exposing the reference API (nodes/params/tying)."""
        nodes = []
        for node in ref_graph.nodes:
            if hasattr(node, "var"):
                nodes.append(InputNode(node.id, node.var, node.num_categories, node.slot))
            elif hasattr(node, "slots"):
                nodes.append(SumNode(node.id, np.asarray(node.children), np.asarray(node.slots)))
            else:
                nodes.append(ProductNode(node.id, np.asarray(node.children)))
        return cls.from_parts(ref_graph.num_vars, nodes, ref_graph.params,
                              root=ref_graph.root, tying=ref_graph.tying)
