"""Neuronal-firing engine over a multi-directed graph (Alg. 1-5; D1-D3).

Host-only control logic: nodes hold receptors (named callables), edges
carry one signal slot per receptor, and ``fire`` propagates signals depth-first with
blocking.  The receptors of the hot-path nodes call the C-ABI layer functions, so all
ciphertext work happens on the GPU; this module never touches residues.

Readings: Alg. 2's successor loop is printed outside the function
 -- we recurse into each successor after the node's own processing
(Z2); Alg. 3 gets the blocking contract of PAPER.md:99 ("A node can only be activated
once all predecessor edges carry some data") -- NotReady if any in-edge slot is empty,
and slots are consumed on a successful read (Z3).
"""
from __future__ import annotations

import types
from typing import Any, Callable, Dict, List, Optional, Sequence


class _NotReady:
    def __repr__(self):
        return "NotReady"


NOT_READY = _NotReady()


class GraphError(Exception):
    pass


class GeneratorUnderrun(GraphError):
    pass


class Node:
    def __init__(self, name: str, receptors: Optional[Dict[str, Callable]] = None, cost: int = 0):
        self.name = name
        self.receptors = dict(receptors or {})
        self.cost = cost          # computational depth (edge weight into this node)
        self.calls = 0

    def receptor(self, r: str, s):
        fn = self.receptors.get(r)
        if fn is None:
            return None
        self.calls += 1
        return fn(s)


class Edge:
    __slots__ = ("src", "dst", "key", "slots")

    def __init__(self, src: str, dst: str, key: int):
        self.src, self.dst, self.key = src, dst, key
        self.slots: Dict[str, Any] = {}

    def signal(self, r: str):
        return self.slots.get(r, NOT_READY)


class Graph:
    """Multi-directed graph: parallel edges are distinct records."""

    def __init__(self):
        self.nodes: Dict[str, Node] = {}
        self.edges: List[Edge] = []
        self.trace: Optional[Callable[[str, str, str], None]] = None

    def add_node(self, node: Node) -> Node:
        self.nodes[node.name] = node
        return node

    def add_edge(self, src: str, dst: str) -> Edge:
        if src not in self.nodes or dst not in self.nodes:
            raise GraphError("edge endpoints must exist")
        e = Edge(src, dst, sum(1 for x in self.edges if x.src == src and x.dst == dst))
        self.edges.append(e)
        return e

    def in_edges(self, n: str) -> List[Edge]:
        return [e for e in self.edges if e.dst == n]

    def out_edges(self, n: str) -> List[Edge]:
        return [e for e in self.edges if e.src == n]

    def successors(self, n: str) -> List[str]:
        seen, out = set(), []
        for e in self.out_edges(n):
            if e.dst not in seen:
                seen.add(e.dst)
                out.append(e.dst)
        return out

    def _emit(self, n, r, ev):
        if self.trace:
            self.trace(n, r, ev)


def fire(g: Graph, n: Sequence[str], r: Sequence[str], s: Sequence[Any]) -> Graph:
    """Alg. 1: signal_carrier for each (node, receptor, signal) in order."""
    if not (len(n) == len(r) == len(s)):
        raise GraphError("ArityError: |n|, |r|, |s| differ")
    for i in range(len(n)):
        if n[i] not in g.nodes:
            raise GraphError(f"UnknownNode {n[i]!r}")
        signal_carrier(g, n[i], r[i], s[i])
    return g


def signal_carrier(g: Graph, n: str, r: str, bootstrap=None) -> None:
    """Alg. 2 with the successor recursion inside (reading Z2).
    A node without receptor ``r`` ignores the signal and leaves its in-edges untouched."""
    if r not in g.nodes[n].receptors:
        return None
    s = get_inbound_signal(g, n, r, bootstrap)
    if s is NOT_READY or s is None:
        g._emit(n, r, "blocked")
        return None
    s = apply_signal(g, n, r, s)
    if s is None:
        return None
    set_outbound_signals(g, n, r, s)
    for succ in g.successors(n):
        signal_carrier(g, succ, r, None)
    return None


def get_inbound_signal(g: Graph, n: str, r: str, bootstrap=None):
    """Alg. 3: bootstrap short-circuit; in-edge order; unwrap one input."""
    if bootstrap is not None:
        return bootstrap
    edges = g.in_edges(n)
    s = [e.signal(r) for e in edges]
    if not s or any(v is NOT_READY for v in s):
        return NOT_READY                   # blocking (reading Z3); nothing consumed
    for e in edges:
        del e.slots[r]                      # consume on successful read
    if len(s) == 1:
        return s[0]
    return s


def apply_signal(g: Graph, n: str, r: str, s):
    """Alg. 4."""
    if s is None:
        return None
    out = g.nodes[n].receptor(r, s)
    g._emit(n, r, "activated")
    return out


def set_outbound_signals(g: Graph, n: str, r: str, s) -> None:
    """Alg. 5: broadcast, or one generator element per out-edge."""
    if s is None:
        return None
    is_gen = isinstance(s, types.GeneratorType)
    for e in g.out_edges(n):
        if is_gen:
            try:
                e.slots[r] = next(s)
            except StopIteration:
                raise GeneratorUnderrun(f"node {n!r}: generator exhausted before out-edges")
        else:
            e.slots[r] = s
    g._emit(n, r, "emitted")
    return None


def chain(names_and_fns: Sequence[tuple], receptor: str = "forward") -> Graph:
    """Build the hot path's chain graph x -> layer -> ... -> sink (D1, host-minimal)."""
    g = Graph()
    prev = None
    for name, fn, cost in names_and_fns:
        g.add_node(Node(name, {receptor: fn}, cost))
        if prev is not None:
            g.add_edge(prev, name)
        prev = name
    return g
