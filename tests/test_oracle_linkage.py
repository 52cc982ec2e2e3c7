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
