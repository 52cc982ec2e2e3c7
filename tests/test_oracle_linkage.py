"""Pins of the oracle's complete linkage (O5): the paper's Fig. 4 merge order,
scipy's textbook complete linkage on tie-free matrices, the definition (max over
member pairs) on every merge, and agreement of three independent algorithms
(brute-force greedy, numpy NN-chain, C NN-chain) on tie-heavy Eq. 1 inputs."""
from fractions import Fraction

import numpy as np
import pytest
from scipy.cluster.hierarchy import linkage as scipy_linkage
from scipy.spatial.distance import squareform

from oracle import oracle_c as oc
from oracle import ragb_oracle as o
from synth.workload import edge, generate

A200 = Fraction(1, 200)


def z_tuples(Z):
    return [(int(a), int(b), np.float32(h), int(s)) for a, b, h, s in Z]


def c_linkage(d):
    a, b, h, s = oc.linkage(d)
    return [(int(x), int(y), np.float32(z), int(w)) for x, y, z, w in zip(a, b, h, s)]


def test_fig4_merge_order(golden):
    g = golden["fig4_build"]
    ctxs = g["contexts"]
    _, _, d = o.pairwise(ctxs, A200)
    Z = o.linkage_greedy(d)
    # printed: C1, C2 merge first; then C3 joins them
    assert (Z[0][0], Z[0][1]) == tuple(g["printed"]["first_merge"])
    assert (Z[1][0], Z[1][1]) == (0, 2) and Z[1][3] == 3
    assert Z[0][2] == o.rn32(Fraction(403, 1200))
    assert Z[1][2] == o.rn32(Fraction(403, 600))  # complete linkage: max(2/3, 403/600)


def scipy_reps(Zs, N):
    rep = list(range(N))
    out = []
    for i, (x, y, h, n) in enumerate(Zs):
        rx, ry = rep[int(x)], rep[int(y)]
        out.append((min(rx, ry), max(rx, ry), np.float32(h), int(n)))
        rep.append(min(rx, ry))
    return out


@pytest.mark.parametrize("seed", range(25))
def test_scipy_complete_linkage_tie_free(seed):
    rng = np.random.default_rng(seed)
    N = int(rng.integers(2, 40))
    x = rng.random((N, N)).astype(np.float32)
    d = np.triu(x, 1)
    d = d + d.T
    Zs = scipy_linkage(squareform(d.astype(np.float64), checks=False), method="complete")
    ref = scipy_reps(Zs, N)
    ref.sort(key=lambda z: (z[2], z[0], z[1]))
    assert z_tuples(o.linkage_greedy(d)) == ref
    assert z_tuples(o.linkage_nn_chain(d)) == ref
    assert c_linkage(d) == ref


def _check_definition(d, Z):
    N = d.shape[0]
    members = {i: [i] for i in range(N)}
    seen = set()
    prev = None
    for a, b, h, sz in Z:
        assert a < b and a in members and b in members
        assert o.cluster_height(d, members[a], members[b]) == h   # max over member pairs
        key = (h, a, b)
        if prev is not None:
            assert key > prev    # strictly increasing key (X9)
        prev = key
        members[a] = members[a] + members.pop(b)
        assert len(members[a]) == sz
        assert b not in seen
        seen.add(b)
    assert len(members) == 1 and len(Z) == N - 1


@pytest.mark.parametrize("seed", range(30))
def test_three_algorithms_agree_tie_heavy(seed):
    rng = np.random.default_rng(100 + seed)
    N = int(rng.integers(2, 48))
    K = int(rng.integers(1, 7))
    V = int(rng.integers(K, 3 * K + 6))
    w = generate(N, K, V, seed, g=int(rng.integers(1, 6)))
    d = oc.pairwise_rows(w.ids, None, 1, 200)
    Zg = z_tuples(o.linkage_greedy(d))
    _check_definition(d, Zg)
    assert z_tuples(o.linkage_nn_chain(d)) == Zg
    assert c_linkage(d) == Zg


@pytest.mark.parametrize("seed", range(10))
def test_integer_matrix_heavy_ties(seed):
    rng = np.random.default_rng(seed)
    N = int(rng.integers(2, 40))
    x = rng.integers(0, 3, size=(N, N)).astype(np.float32)
    d = np.triu(x, 1)
    d = d + d.T
    Zg = z_tuples(o.linkage_greedy(d))
    _check_definition(d, Zg)
    assert z_tuples(o.linkage_nn_chain(d)) == Zg
    assert c_linkage(d) == Zg


def test_all_tied_is_caterpillar():
    # all-disjoint contexts: every distance is 1.0, greedy order is a caterpillar by rep
    w = edge("disjoint", 12, 3)
    d = oc.pairwise_rows(w.ids, None, 1, 200)
    Z = c_linkage(d)
    assert Z == [(0, b, np.float32(1.0), b + 1) for b in range(1, 12)]


def test_medium_c_vs_numpy_chain():
    w = generate(600, 10, 3000, 3)
    d = oc.pairwise_rows(w.ids, None, 1, 200)
    assert c_linkage(d) == z_tuples(o.linkage_nn_chain(d))


# --------------------------------------------------------------- NEXT-3 oracle
def _reps_from_members(ctxs, members):
    """Representative of a cluster from its member leaves: the leaf itself
    (retrieval order) for a singleton, else the ascending sorted intersection
    of all member sets (associativity of the pairwise rule)."""
    if len(members) == 1:
        return list(ctxs[next(iter(members))])
    s = set(ctxs[next(iter(members))])
    for m in members:
        s &= set(ctxs[m])
    return sorted(s)


def test_intersection_fig4(golden):
    ctxs = golden["fig4_build"]["contexts"]
    Z = o.linkage_intersection(ctxs, A200)
    assert [(a, b, s) for a, b, _, s in Z] == [(0, 1, 2), (0, 2, 3)]
    assert Z[0][2] == np.float32(403 / 1200)   # C1, C2
    # C3 vs the virtual node {1,2}: s=1, positions 1 / 0, m=3 -> 1-1/3+1/200 = 403/600
    assert Z[1][2] == o.rn32(Fraction(403, 600))


def test_intersection_identical_unsorted():
    # identical leaves are at 0; a virtual node is the SORTED set, which is at
    # alpha*footrule/K > 0 from an unsorted leaf: leaves pair up first
    ctxs = [[3, 1, 2]] * 4
    Z = o.linkage_intersection(ctxs, A200)
    assert [(a, b, float(h), s) for a, b, h, s in Z] == [(0, 1, 0.0, 2), (2, 3, 0.0, 2), (0, 2, 0.0, 4)]


@pytest.mark.parametrize("seed", range(40))
def test_intersection_python_vs_c(seed):
    rng = np.random.default_rng(seed)
    N = int(rng.integers(2, 36))
    K = int(rng.integers(2, 8))
    w = generate(N, K, int(rng.integers(K + 1, 4 * K + 8)), 1000 + seed)
    lens = None
    if seed % 3 == 0:
        lens = rng.integers(1, K + 1, size=N).astype(np.uint8)
    ctxs = o.validate(w.ids, lens)
    Zp = o.linkage_intersection(ctxs, A200)
    a, b, h, s = oc.linkage_intersection(w.ids, lens, 1, 200)
    assert [(x[0], x[1], x[3]) for x in Zp] == list(zip(a.tolist(), b.tolist(), s.tolist()))
    assert np.array_equal(np.array([x[2] for x in Zp], dtype=np.float32).view(np.uint32), h.view(np.uint32))
    # definition check: replay; every merge is the minimum key over the active
    # clusters, with distances recomputed from the member leaves
    members = {i: {i} for i in range(N)}
    for (ma, mb, mh, ms) in Zp:
        best = min((o.distance(_reps_from_members(ctxs, members[x]), _reps_from_members(ctxs, members[y]), A200), x, y)
                   for x in members for y in members if x < y)
        assert best == (mh, ma, mb)
        members[ma] |= members.pop(mb)
        assert len(members[ma]) == ms


def test_intersection_is_not_reducible():
    """Some run has a later merge lower than an earlier one, which
    complete linkage never has: the two readings are really different."""
    found = False
    for seed in range(30):
        w = generate(24, 5, 30, 2000 + seed)
        a, b, h, s = oc.linkage_intersection(w.ids, None, 1, 200)
        if np.any(np.diff(h) < 0):
            found = True
            ctxs = o.validate(w.ids)
            t = o.build_tree(ctxs, list(zip(a.tolist(), b.tolist(), h.tolist(), s.tolist())))
            for i in range(24):  # the tree still replays
                assert o.traverse(t, t.path[i]) == t.leaf_node[i]
            break
    assert found
