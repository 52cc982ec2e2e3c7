"""Pins of the NEXT-4 oracles: the prefix cache (Fig. 6)
and the index update under cache events (SPEC examples)."""
import numpy as np
import pytest

from oracle import ragb_oracle as o


def test_fig6_schedule_reuse(golden):
    """Fig. 6 with a cache holding one context (3 docs): in
    the input order C8 misses entirely; scheduled, "C8 immediately reuses
    {1,2} before eviction"."""
    g5 = golden["fig5_ordering"]["printed"]
    C3 = golden["fig5_ordering"]["derived"]["C3"]
    reqs = {"C6": g5["C6"], "C3": C3, "C7": g5["C7"], "C8": g5["C8"]}
    c = o.PrefixCache(3)
    res = {n: c.prefill(reqs[n]) for n in golden["fig6_schedule"]["input_order"]}
    assert res["C8"][0] == 0
    c = o.PrefixCache(3)
    res = {n: c.prefill(reqs[n]) for n in golden["fig6_schedule"]["printed"]["scheduled"]}
    assert res["C8"][0] == 2   # docs {1, 2}


def test_identical_twice_all_hit():
    c = o.PrefixCache(100)
    assert c.prefill([5, 3, 9]) == (0, 3, 0)
    assert c.prefill([5, 3, 9]) == (3, 0, 0)
    assert c.prefill([5, 3]) == (2, 0, 0)
    assert c.prefill([3, 5]) == (0, 2, 0)   # a prefix, not a set


def test_over_capacity_and_duplicates():
    c = o.PrefixCache(2)
    with pytest.raises(o.OracleError):
        c.prefill([1, 2, 3])
    with pytest.raises(o.OracleError):
        c.prefill([1, 1])


@pytest.mark.parametrize("seed", range(40))
def test_trie_vs_list_model(seed):
    """SPEC cache_sim: hit/miss/eviction accounting equals an independent
    list-of-prefixes model; the budget always holds."""
    rng = np.random.default_rng(seed)
    K = int(rng.integers(2, 6))
    pool = int(rng.integers(K + 1, 3 * K + 4))
    tok = {d: int(rng.integers(1, 4)) for d in range(pool)} if seed % 2 else None
    reqs = [rng.choice(pool, size=int(rng.integers(1, K + 1)), replace=False).tolist() for _ in range(40)]
    tmax = max(sum((tok or {}).get(d, 1) for d in r) for r in reqs)
    cap = int(rng.integers(tmax, 3 * tmax + 2))
    c = o.PrefixCache(cap, tok)
    got = []
    for r in reqs:
        got.append(c.prefill(r))
        assert c.resident <= cap
        assert got[-1][0] + got[-1][1] == sum((tok or {}).get(d, 1) for d in r)
    assert got == o.prefix_cache_list_model(cap, reqs, tok)


def test_monotone_capacity():
    """A larger budget never yields fewer hits for the same request sequence
    (SPEC cache_sim property), over a range of budgets."""
    rng = np.random.default_rng(7)
    reqs = [rng.choice(30, size=5, replace=False).tolist() for _ in range(300)]
    hits = []
    for cap in range(5, 120, 5):
        c = o.PrefixCache(cap)
        hits.append(sum(c.prefill(r)[0] for r in reqs))
    assert all(b >= a for a, b in zip(hits, hits[1:]))


def _two_leaves():
    # root -> [A, B] (node ids 1, 2)
    return o.CacheIndex([[1, 2], [], []])


def test_index_events_spec_example():
    """SPEC apply_cache_event: two leaves holding 100 tokens each, A least
    recently used, Evicted{150} -> A removed (100 taken), B decremented to 50."""
    t = _two_leaves()
    t.appended([0], 100)
    t.appended([1], 100)
    assert t.evicted(150) == 150
    assert t.gone[1] and t.seq[2] == 50 and t.children[0] == [2]
    assert t.node_at([0]) == 2   # B's child index shifted to 0
    with pytest.raises(o.OracleError):
        t.node_at([1])


def test_index_events_noop_access_and_conservation():
    t = _two_leaves()
    t.appended([0], 10)
    t.appended([1], 10)
    assert t.evicted(0) == 0 and t.seq == [0, 10, 10]
    t.accessed([0])            # A becomes the most recent
    assert t.evicted(5) == 5 and t.seq[2] == 5 and t.seq[1] == 10
    assert t.evicted(100) == 15 and t.gone[1] and t.gone[2]
    assert t.children[0] == []  # the root is never removed
    with pytest.raises(o.OracleError):
        t.appended([], -1)


def test_index_events_parent_chain_removed():
    # root -> V(1) -> [L2, L3]; V holds tokens too
    t = o.CacheIndex([[1], [2, 3], [], []])
    t.appended([0], 4)
    t.appended([0, 0], 3)
    t.appended([0, 1], 2)
    assert t.evicted(4) == 4      # V (oldest) drained; it keeps its children
    assert not t.gone[1] and t.seq[1] == 0
    assert t.evicted(5) == 5      # both leaves drained -> V left empty -> removed
    assert t.gone[2] and t.gone[3] and t.gone[1] and t.children[0] == []
