"""NEXT f4: Alg. 6-7 source/cost discovery and grouping on the SPEC's hand-traced graphs
(SPEC.md:224-241), and the C1 chain's group depth reproducing BASELINE's chain."""
import pytest

from paper_2110_13638_b200 import autofhe, graph


def _g(nodes, edges):
    g = graph.Graph()
    for name, cost in nodes:
        g.add_node(graph.Node(name, cost=cost))
    for a, b in edges:
        g.add_edge(a, b)
    return g


def test_chain_with_concern_restarts():
    g = _g([("x", 0), ("c1", 2), ("r0", 0)], [("x", "c1"), ("c1", "r0")])
    autofhe.auto_he_discover(g, "x", "x", lambda d: d.name == "r0", 0)
    assert g.nodes["c1"].sources == {"x": 2}
    assert g.nodes["r0"].sources == {"x": 2}


def test_fhe_parm_problem_shape():
    # x0 -> c1, x1 -> c0 -> c1 with c0 = 1, c1 = 2: c1.sources = {x0: 2, x1: 3}
    g = _g([("x0", 0), ("x1", 0), ("c0", 1), ("c1", 2)], [("x0", "c1"), ("x1", "c0"), ("c0", "c1")])
    membership, costs = autofhe.auto_he(g, ["x0", "x1"], lambda d: False)
    assert g.nodes["c1"].sources == {"x0": 2, "x1": 3}
    assert membership["x0"] == membership["x1"] and costs == [3]


def test_diamond_max_wins_and_disconnected_groups():
    g = _g([("x", 0), ("a", 2), ("b", 1), ("b2", 2), ("j", 0), ("y", 0), ("z", 4)],
           [("x", "a"), ("x", "b"), ("b", "b2"), ("a", "j"), ("b2", "j"), ("y", "z")])
    membership, costs = autofhe.auto_he(g, ["x", "y"], lambda d: False)
    assert g.nodes["j"].sources["x"] == 3
    assert membership["x"] != membership["y"]
    assert costs[membership["x"]] == 3 and costs[membership["y"]] == 4


def test_single_path_and_c1_chain_depth():
    # x -> cc(1) -> sigma_a(2) -> dense(1) -> y_hat: depth 4 = BASELINE C1's chain
    g = _g([("x", 0), ("cc", 1), ("act", 2), ("dense", 1), ("y_hat", 0)],
           [("x", "cc"), ("cc", "act"), ("act", "dense"), ("dense", "y_hat")])
    membership, costs = autofhe.auto_he(g, ["x"], lambda d: False)
    assert membership == {"x": 0} and costs == [4]


def test_cycle_is_reported():
    g = _g([("x", 0), ("a", 1), ("b", 1)], [("x", "a"), ("a", "b"), ("b", "a")])
    with pytest.raises(autofhe.CycleError):
        autofhe.auto_he(g, ["x"], lambda d: False)
