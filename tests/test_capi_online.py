"""NEXT-1 (online context ordering, Section 4.2 and
PAPER:425-436 Section 5.1): the library's rb_order_contexts(ids != NULL) vs the
oracle's OnlineIndex, on the paper's examples and on seeded workloads.  Host
logic only, no device compute."""
from fractions import Fraction

import numpy as np
import pytest

from oracle import oracle_c as oc
from oracle import ragb_oracle as o
from paper_2511_03475_b200 import ragb
from synth.workload import generate

A200 = Fraction(1, 200)


def both(base, lens=None, alpha=(1, 200)):
    ctxs = o.validate(base, lens)
    Z = oc.linkage(oc.pairwise_rows(base, lens, *alpha))
    t = o.build_tree(ctxs, list(zip(*Z)))
    oi = o.OnlineIndex(ctxs, t, Fraction(*alpha))
    li = ragb.index_from_linkage(base, *Z, lens=lens)
    if alpha != (1, 200):
        li.set_alpha(Fraction(*alpha))
    return oi, li


def canon_online(oi):
    out = {}
    stack = [(0, ())]
    while stack:
        k, path = stack.pop()
        out[path] = (oi.leaf_of[k], tuple(oi.ordered[k]))
        for ci, c in enumerate(oi.children[k]):
            stack.append((c, path + (ci,)))
    return out


def check_batch(oi, li, batch, lens=None):
    M, K = batch.shape
    qs = [batch[i, :(K if lens is None else lens[i])].tolist() for i in range(M)]
    ordered, plens, paths, sched = oi.order_batch(qs)
    out, pl, sc = li.order_new(batch, lens)
    for i in range(M):
        L = len(qs[i])
        assert out[i, :L].tolist() == ordered[i], i
        assert np.array_equal(out[i, L:], batch[i, L:])
    assert pl.tolist() == plens
    assert sc.tolist() == sched
    n = li.size()
    assert n == len(oi.docs)
    assert li.paths() == [oi.path_of(c) for c in range(n)]
    assert len(li.tree()["parent"]) == len(oi.parent)


def test_search_example_lib(golden):
    g = golden["search_example"]
    ids = np.array(golden["fig4_build"]["contexts"], dtype=np.uint32)
    oi, li = both(ids)
    out, pl, sc = li.order_new(np.array([g["query_C6"]], dtype=np.uint32))
    assert li.paths()[3] == g["printed"]["insert_path"]           # [0, 0, 2]
    assert pl.tolist() == [2]


def test_fig5_fig6_lib(golden):
    g5, g6 = golden["fig5_ordering"], golden["fig6_schedule"]
    ids = np.array(golden["fig4_build"]["contexts"], dtype=np.uint32)
    oi, li = both(ids)
    batch = np.array([g5["new"]["C6"], g5["new"]["C7"], g5["new"]["C8"]], dtype=np.uint32)
    out, pl, sc = li.order_new(batch)
    assert out[0].tolist() == g5["printed"]["C6"]
    assert out[1].tolist() == g5["printed"]["C7"]
    assert out[2].tolist() == g5["printed"]["C8"]
    assert li.paths()[3:] == [g6["paths"]["C6"], g6["paths"]["C7"], g6["paths"]["C8"]]
    assert pl.tolist() == [2, 0, 2]
    # Fig. 6: the batch schedule [C6, C7, C8] keeps C6/C8 together
    assert sc.tolist() == [0, 2, 1]


@pytest.mark.parametrize("seed", range(8))
def test_online_vs_oracle(seed):
    N, K = (120, 6) if seed % 2 else (200, 10)
    w = generate(N + 60, K, 3 * N // 2, seed, turns=1)
    base, new = w.ids[:N], w.ids[N:]
    oi, li = both(base)
    # several batches, each sees the previous insertions
    for lo, hi in ((0, 20), (20, 21), (21, 60)):
        check_batch(oi, li, new[lo:hi])
    assert canon_online(oi) == canon_online_lib(li)


def canon_online_lib(li):
    """Path -> (leaf, ordered prefix) for every node on a leaf's path."""
    tr = li.tree()
    parent, leaf = tr["parent"], tr["leaf"]
    n = len(parent)
    paths = li.paths()
    res = {}
    leaf_node = {int(leaf[k]): k for k in range(n) if leaf[k] >= 0}
    for c, p in enumerate(paths):
        k = leaf_node[c]
        chain = []
        while k != -1:
            chain.append(k)
            k = int(parent[k]) if k != 0 else -1
        chain = chain[::-1]
        for z, node in enumerate(chain):
            key = tuple(p[:z])
            ordered = tr["prefix_ids"][tr["prefix_off"][node]:tr["prefix_off"][node + 1]].tolist()
            res[key] = (int(leaf[node]), tuple(ordered))
    return res


def test_online_variable_lengths_and_alpha():
    w = generate(260, 12, 300, 7, len_min=3)
    base, new = w.ids[:200], w.ids[200:]
    lb, ln = w.lens[:200], w.lens[200:]
    for alpha in ((1, 200), (1, 100)):
        oi, li = both(base, lb, alpha)
        check_batch(oi, li, new, ln)
        assert canon_online(oi) == canon_online_lib(li)


def test_online_repeat_is_idempotent_and_sessions():
    w = generate(150, 8, 200, 3)
    base = w.ids[:100]
    oi, li = both(base)
    check_batch(oi, li, w.ids[100:150])
    # re-submitting already-indexed contexts
    check_batch(oi, li, w.ids[:30])
    check_batch(oi, li, w.ids[100:130])
    # offline mode reports every indexed context, including inserted ones
    out, pl, sc = li.order_contexts()
    assert out.shape[0] == li.size() == len(oi.docs)
    for c in range(li.size()):
        L = len(oi.docs[c])
        assert out[c, :L].tolist() == oi.ordered[oi.leaf_node[c]]
    assert sc.tolist() == o.schedule([oi.path_of(c) for c in range(li.size())])
    # a session on an inserted context starts from its served order
    s = li.session(li.size() - 1)
    assert s is not None


def test_online_errors():
    w = generate(60, 6, 80, 1)
    oi, li = both(w.ids[:50])
    bad = w.ids[50:52].copy()
    bad[0, 1] = bad[0, 0]
    with pytest.raises(ragb.RagbError) as e:
        li.order_new(bad)
    assert e.value.code == ragb.RB_EDUPDOC
    with pytest.raises(ragb.RagbError) as e:
        li.order_new(w.ids[50:52, :5])
    assert e.value.code == ragb.RB_EINVAL
    with pytest.raises(ragb.RagbError) as e:
        li.set_alpha((1, 0))
    assert e.value.code == ragb.RB_EALPHA
