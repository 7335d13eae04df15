"""Automatic FHE parameterisation over the network graph (Alg. 6-7;
SURVEY §8(f) NEXT f4).  Host-only graph logic: every node carries a `cost` (its
computational depth, the weight of any edge into it) and a `sources` map; discovery labels
each node with the longest cost path from every encryption source that reaches it, and
sources that meet at some node are merged into one parameter group whose depth is the
largest label in the group ("Which cyphertexts interact at which nodes ... What is the
maximum computational depth of each group").  The group depth feeds
Alg. 8 (`edl_params_from_depth`) for the group's CKKS parameters.

Reading (as SPEC.md:280): Alg. 7 restarts discovery at a concern node with
autoHE_discover(g, n, n, ...) unconditionally, which would re-trigger forever on the
entry node itself; the restart is gated to concern nodes other than the current source.
A path longer than the node count (only possible through a cycle) raises CycleError
instead of recursing without end.
"""
from __future__ import annotations

from typing import Callable, Dict, List, Sequence, Tuple

from .graph import Graph, GraphError


class CycleError(GraphError):
    pass


def auto_he_discover(g: Graph, n: str, s: str, concern: Callable, c: int, _depth: int = 0) -> None:
    """Alg. 7: label node n with source s at cost c (max wins), then restart at concern
    nodes or recurse into successors with c + cost(successor).  A path from one source
    longer than the node count can only come from a cycle: CycleError."""
    if _depth > len(g.nodes):
        raise CycleError("discovery revisits a node on one path (cycle in the graph)")
    d = g.nodes[n]
    if getattr(d, "sources", None) is None:
        d.sources = {}
    if s != n:
        if d.sources.get(s) is None or d.sources[s] < c:
            d.sources[s] = c
    if concern(d) and s != n:
        auto_he_discover(g, n, n, concern, 0, 0)
    else:
        for i in g.successors(n):
            auto_he_discover(g, i, s, concern, c + g.nodes[i].cost, _depth + 1)


def auto_he(g: Graph, n: Sequence[str], concern: Callable) -> Tuple[Dict[str, int], List[int]]:
    """Alg. 6: discovery from every entry, then group assignment: r = (membership, costs)."""
    for i in n:
        auto_he_discover(g, i, i, concern, 0)
    membership: Dict[str, int] = {}
    costs: List[int] = []
    for i in n:
        if membership.get(i) is None:
            membership[i] = len(costs)
            costs.append(0)
        for node in g.nodes.values():
            src = getattr(node, "sources", None) or {}
            if i in src:
                for k in src:
                    membership[k] = membership[i]
                    if src[k] > costs[membership[i]]:
                        costs[membership[i]] = src[k]
    return membership, costs


def group_params(costs: Sequence[int], scale_bits: int = 40, special_mult: float = 1.5):
    """Alg. 8 parameters (through the C-ABI) for every group depth."""
    from . import edl
    return [edl.params_from_depth(c, scale_bits, special_mult) for c in costs]
