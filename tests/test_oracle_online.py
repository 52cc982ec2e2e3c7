"""Pins of the oracle's online ordering (NEXT-1): the paper's Section 4.2
search example, Fig. 5 orderings and Fig. 6 schedule, plus invariants."""
from fractions import Fraction

import numpy as np
import pytest

from oracle import oracle_c as oc
from oracle import ragb_oracle as o
from synth.workload import generate

A200 = Fraction(1, 200)


def fig4_online(golden):
    ctxs = golden["fig4_build"]["contexts"]
    _, _, d = o.pairwise(ctxs, A200)
    t = o.build_tree(ctxs, o.linkage_greedy(d))
    return o.OnlineIndex(ctxs, t, A200)


def test_search_example(golden):
    g = golden["search_example"]
    idx = fig4_online(golden)
    node, path = idx.search(g["query_C6"])
    assert path == g["printed"]["descent_path"]               # [0, 0]
    assert sorted(idx.docset[node]) == [1, 2]                 # C4
    ordq, plen, path2 = idx.order(g["query_C6"])
    assert path2 == g["printed"]["insert_path"]               # [0, 0, 2]


def test_fig5_fig6(golden):
    g5, g6 = golden["fig5_ordering"], golden["fig6_schedule"]
    idx = fig4_online(golden)
    batch = [g5["new"]["C6"], g5["new"]["C7"], g5["new"]["C8"]]
    ordered, plens, paths, _ = idx.order_batch(batch)
    assert ordered[0] == g5["printed"]["C6"]
    assert ordered[1] == g5["printed"]["C7"]                  # unchanged, standalone
    assert ordered[2] == g5["printed"]["C8"]
    assert paths == [g6["paths"]["C6"], g6["paths"]["C7"], g6["paths"]["C8"]]
    assert plens == [2, 0, 2]
    # Fig. 6: schedule [C6, C3, C7, C8] -> [C6, C8, C3, C7]
    names = g6["input_order"]
    p = {"C6": paths[0], "C7": paths[1], "C8": paths[2], "C3": idx.path_of(2)}
    sched = o.schedule([p[n] for n in names])
    assert [names[i] for i in sched] == g6["printed"]["scheduled"]


@pytest.mark.parametrize("seed", range(6))
def test_online_invariants(seed):
    w = generate(150, 6, 120, seed)
    base, new = w.ids[:100], w.ids[100:]
    ctxs = o.validate(base)
    d = oc.pairwise_rows(base, None, 1, 200)
    t = o.build_tree(ctxs, list(zip(*oc.linkage(d))))
    idx = o.OnlineIndex(ctxs, t, A200)
    for q in new:
        q = q.tolist()
        ordq, plen, path = idx.order(q)
        assert sorted(ordq) == sorted(q)                       # permutation
        node = o.traverse_online(idx, path)
        assert idx.ordered[node] == ordq
        par = idx.parent[node]
        assert ordq[:plen] == idx.ordered[par]                 # inherits the parent's prefix
        tail = ordq[plen:]
        assert tail == [x for x in q if x in set(tail)]        # stable tail
    # tree invariant: every child's ordered context extends its parent's
    for k, p in enumerate(idx.parent):
        if p >= 0:
            assert idx.ordered[k][:len(idx.ordered[p])] == idx.ordered[p]
    # re-ordering an already indexed context keeps its order (idempotence)
    q = new[0].tolist()
    before = idx.ordered[idx.leaf_node[100]]
    ordq, plen, _ = idx.order(before)
    assert ordq == before
