"""Host logic: the neuronal-firing engine (Alg. 1-5) on SPEC.md's examples."""
import random

import pytest

from paper_2110_13638_b200 import graph as G


def _g(*nodes):
    g = G.Graph()
    for name, fn in nodes:
        g.add_node(G.Node(name, {"forward": fn} if fn else {}))
    return g


def test_chain_propagation():
    g = _g(("x", lambda s: s), ("double", lambda s: 2 * s), ("sink", None))
    g.add_edge("x", "double")
    g.add_edge("double", "sink")
    G.fire(g, ["x"], ["forward"], [3.0])
    assert g.in_edges("sink")[0].signal("forward") == 6.0


def test_blocking_two_inputs():
    calls = []
    g = _g(("x", lambda s: s), ("y", lambda s: s), ("add", lambda s: calls.append(s) or sum(s)), ("sink", None))
    g.add_edge("x", "add")
    g.add_edge("y", "add")
    g.add_edge("add", "sink")
    G.fire(g, ["x"], ["forward"], [1])
    assert calls == [] and g.in_edges("sink")[0].signal("forward") is G.NOT_READY
    G.fire(g, ["y"], ["forward"], [2])
    assert calls == [[1, 2]]                                   # in-edge order, activates once
    assert g.in_edges("sink")[0].signal("forward") == 3
    assert all(e.signal("forward") is G.NOT_READY for e in g.in_edges("add"))   # consumed


def test_single_input_unwrapped_and_stacking_order():
    seen = []
    g = _g(("a", lambda s: s), ("n", lambda s: seen.append(s)))
    g.add_edge("a", "n")
    G.fire(g, ["a"], ["forward"], [5])
    assert seen == [5]                                         # not [5] (Alg. 3 unwrap)
    g2 = _g(("a", lambda s: s), ("n", lambda s: seen.append(s)))
    for _ in range(3):
        g2.add_edge("a", "n")                                   # parallel edges are separate
    G.fire(g2, ["a"], ["forward"], [7])
    assert seen[-1] == [7, 7, 7]


def test_generator_per_edge_and_underrun():
    got = []
    g = _g(("src", lambda s: (v for v in s)), ("a", lambda s: got.append(("a", s))), ("b", lambda s: got.append(("b", s))))
    g.add_edge("src", "a")
    g.add_edge("src", "b")
    G.fire(g, ["src"], ["forward"], [["x0", "x1"]])
    assert got == [("a", "x0"), ("b", "x1")]
    g2 = _g(("src", lambda s: (v for v in s)), ("a", None), ("b", None))
    g2.add_edge("src", "a")
    g2.add_edge("src", "b")
    with pytest.raises(G.GeneratorUnderrun):
        G.fire(g2, ["src"], ["forward"], [["only"]])


def test_none_stops_propagation_and_errors():
    g = _g(("x", lambda s: None), ("y", lambda s: 1 / 0))
    g.add_edge("x", "y")
    G.fire(g, ["x"], ["forward"], [1])                          # y never called
    with pytest.raises(G.GraphError):
        G.fire(g, ["x", "y"], ["forward"], [1])
    with pytest.raises(G.GraphError):
        G.fire(g, ["nope"], ["forward"], [1])


def test_depth_first_order_on_chain():
    order = []
    names = [f"n{i}" for i in range(6)]
    g = G.chain([(n, (lambda k: lambda s: order.append(k) or s)(n), 1) for n in names])
    G.fire(g, ["n0"], ["forward"], [0])
    assert order == names


def test_random_dag_equals_direct_evaluation():
    """SPEC.md:181 equivalence oracle: fire() == direct recursive evaluation on random DAGs."""
    rnd = random.Random(0)
    for trial in range(100):
        n = rnd.randint(2, 8)
        parents = {i: sorted(rnd.sample(range(i), rnd.randint(1, min(i, 2)))) if i else [] for i in range(n)}
        coef = {i: rnd.randint(1, 5) for i in range(n)}
        g = G.Graph()
        for i in range(n):
            def fn(s, i=i):
                vals = s if isinstance(s, list) else [s]
                return coef[i] * sum(vals) + i
            g.add_node(G.Node(f"v{i}", {"forward": fn}))
        for i in range(n):
            for p in parents[i]:
                g.add_edge(f"v{p}", f"v{i}")
        sinks = [i for i in range(n) if not any(i in parents[j] for j in range(n))]
        for s in sinks:
            g.add_node(G.Node(f"out{s}", {}))
            g.add_edge(f"v{s}", f"out{s}")
        roots = [i for i in range(n) if not parents[i]]
        G.fire(g, [f"v{r}" for r in roots], ["forward"] * len(roots), [10 + r for r in roots])

        memo = {}

        def ev(i):
            if i not in memo:
                vals = [ev(p) for p in parents[i]] if parents[i] else [10 + i]
                memo[i] = coef[i] * sum(vals) + i
            return memo[i]
        for s in sinks:
            assert g.in_edges(f"out{s}")[0].signal("forward") == ev(s), trial
