"""Pins of the oracle's tree / ordering / schedule / dedup (O6-O9): the paper's
Fig. 4, Fig. 5, Fig. 6 and Section 6 examples, plus structural invariants on
random workloads."""
from fractions import Fraction

import numpy as np
import pytest

from oracle import oracle_c as oc
from oracle import ragb_oracle as o
from synth.workload import edge, generate

A200 = Fraction(1, 200)


def build(ctxs):
    _, _, d = o.pairwise(ctxs, A200)
    Z = o.linkage_greedy(d)
    return o.build_tree(ctxs, Z)


def test_fig4_tree(golden):
    g = golden["fig4_build"]
    ctxs = g["contexts"]
    t = build(ctxs)
    # root has one child C5 = {1}; C5 has children C4 = {1,2} and C3
    root_kids = t.children[0]
    assert len(root_kids) == 1
    c5 = root_kids[0]
    assert sorted(t.docset[c5]) == g["printed"]["virtual_C5_context"]
    c4 = t.children[c5][0]
    assert sorted(t.docset[c4]) == g["printed"]["virtual_C4_context"]
    assert [t.leaf_of[k] for k in t.children[c4]] == [0, 1]
    assert t.leaf_of[t.children[c5][1]] == 2
    assert t.path == g["derived"]["paths"]
    # descent to C4 is [0, 0]
    assert o.traverse(t, [0, 0]) == c4


def test_fig5_offline_order(golden):
    g = golden["fig5_ordering"]
    ctxs = g["init"]
    t = build(ctxs)
    ordered, plen = o.offline_order(ctxs, t)
    assert ordered[0] == g["printed"]["C1"]
    assert ordered[1] == g["printed"]["C2"]
    assert ordered[2] == g["derived"]["C3"]
    assert ordered[0][:plen[0]] == g["printed"]["C1_C2_prefix"]
    assert ordered[2][:plen[2]] == g["printed"]["C3_prefix"]


def test_fig6_schedule(golden):
    g = golden["fig6_schedule"]
    names = g["input_order"]
    paths = [g["paths"][n] for n in names]
    sched = o.schedule(paths)
    assert [names[i] for i in sched] == g["printed"]["scheduled"]


def test_dedup_example(golden):
    g = golden["dedup_example"]
    s = o.Session(g["turn0"])
    novel, refs = s.dedup_turn(g["turn1"])
    assert novel == g["printed"]["novel"]
    assert [x for x, _ in refs] == g["printed"]["overlap"]
    assert all(t == 0 for _, t in refs)
    # identical retrieval -> nothing novel; disjoint -> all novel
    s2 = o.Session([1, 2, 3])
    assert s2.dedup_turn([3, 2, 1]) == ([], [(3, 0), (2, 0), (1, 0)])
    assert s2.dedup_turn([7, 8]) == ([7, 8], [])
    assert s2.dedup_turn([8, 1, 9]) == ([9], [(8, 2), (1, 0)])


def check_tree_invariants(ctxs, t):
    N = len(ctxs)
    ordered, plen = o.offline_order(ctxs, t)
    for k in range(len(t.parent)):
        p = t.parent[k]
        if p < 0:
            assert t.ordered[k] == []
            continue
        # child's ordered context extends the parent's as an exact prefix
        assert t.ordered[k][:len(t.ordered[p])] == t.ordered[p]
        assert set(t.docset[p]) <= set(t.docset[k])
        if t.leaf_of[k] < 0:
            # no collapsed-away redundancy: a virtual node differs from its parent
            assert t.docset[k] != t.docset[p]
            assert t.ordered[k] == t.ordered[p] + sorted(set(t.docset[k]) - set(t.docset[p]))
        # children ordered by rep
        reps = [t.rep[c] for c in t.children[k]]
        assert reps == sorted(reps)
    for i in range(N):
        assert o.traverse(t, t.path[i]) == t.leaf_node[i]
        assert sorted(ordered[i]) == sorted(ctxs[i])     # permutation
        tail = ordered[i][plen[i]:]
        assert tail == [x for x in ctxs[i] if x in set(tail)]  # stable tail
    sched = o.schedule(t.path)
    assert sorted(sched) == list(range(N))
    firsts = [t.path[i][0] for i in sched]
    seen = set()
    for j, f in enumerate(firsts):  # group contiguity
        if f in seen:
            assert firsts[j - 1] == f
        seen.add(f)


@pytest.mark.parametrize("seed", range(12))
def test_tree_invariants_random(seed):
    rng = np.random.default_rng(seed)
    N = int(rng.integers(1, 80))
    K = int(rng.integers(1, 9))
    w = generate(N, K, int(rng.integers(K, 6 * K + 10)), seed)
    ctxs = o.validate(w.ids)
    d = oc.pairwise_rows(w.ids, None, 1, 200)
    t = o.build_tree(ctxs, o.linkage_greedy(d))
    check_tree_invariants(ctxs, t)


@pytest.mark.parametrize("kind", ["disjoint", "identical", "permutations"])
def test_tree_edge_inputs(kind):
    w = edge(kind, 9, 4)
    ctxs = o.validate(w.ids)
    d = oc.pairwise_rows(w.ids, None, 1, 200)
    t = o.build_tree(ctxs, o.linkage_greedy(d))
    check_tree_invariants(ctxs, t)
    if kind == "disjoint":
        # empty intersections collapse into the root: every context is a standalone branch
        assert t.path == [[i] for i in range(9)]
    if kind in ("identical", "permutations"):
        ordered, plen = o.offline_order(ctxs, t)
        assert all(x == ordered[0] for x in ordered) and all(p == 4 for p in plen)


def test_single_context():
    t = o.build_tree([[5, 6]], [])
    assert t.path == [[0]]
    ordered, plen = o.offline_order([[5, 6]], t)
    assert ordered == [[5, 6]] and plen == [0]


def test_deep_collapsed_caterpillar():
    """All-disjoint contexts merged as one caterpillar (0 absorbs 1, 2, ...):
    every virtual node's set is the empty set = the root's, so all N-1 virtual
    nodes collapse (X11) and every leaf hangs off the root in rep order (X12)
    with path [i] and its original order.  N = 5000 nests deeper
    than Python's default recursion limit."""
    N = 5000
    ctxs = o.validate(edge("disjoint", N, 3).ids, None)
    Z = [(0, i, 1.0, i + 1) for i in range(1, N)]
    t = o.build_tree(ctxs, Z)
    assert t.path == [[i] for i in range(N)]
    ordered, plen = o.offline_order(ctxs, t)
    assert ordered == [list(c) for c in ctxs] and plen == [0] * N
    assert o.schedule(t.path) == list(range(N))
