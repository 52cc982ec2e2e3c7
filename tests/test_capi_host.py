"""CPU tests of libragb: the C-ABI loads and exports every symbol include/ragb.h
declares, and the host-side steps (tree, ordering, schedule, dedup; a6-a8)
agree with the oracle.  No device compute is called here."""
import re
import subprocess
from fractions import Fraction

import numpy as np
import pytest

from oracle import oracle_c as oc
from oracle import ragb_oracle as o
from paper_2511_03475_b200 import ragb
from synth.workload import edge, generate
import os
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    src = open(f"{ROOT}/include/ragb.h").read()
    return sorted(set(re.findall(r"RB_API\s+[\w\s\*]+?\b(rb_\w+)\s*\(", src)))


def test_exports_every_declared_symbol():
    ragb.lib()
    syms = header_symbols()
    assert len(syms) >= 20
    assert sorted(ragb.EXPORTED) == syms
    out = subprocess.check_output(["nm", "-D", "--defined-only", ragb.LIB_PATH]).decode()
    exported = set(re.findall(r"\bT (rb_\w+)", out))
    assert set(syms) <= exported
    # nothing else leaks out of the C-ABI
    assert {s for s in exported if s.startswith("rb_")} == set(syms)


def test_version_and_params():
    assert "sm_100a" in ragb.version()
    p = ragb.make_params()
    assert (p.alpha_num, p.alpha_den) == (1, 200)
    assert ragb.alpha_rational(0.005) == (1, 200)


def test_workspace_and_param_errors():
    p = ragb.make_params()
    rb, sb = ragb.workspace_size(1000, 20, p)
    assert rb == 1000 * 1000 * 4 and sb >= 999 * 999 * 4
    with pytest.raises(ragb.RagbError) as e:
        ragb.workspace_size(0, 20, p)
    assert e.value.code == ragb.RB_EINVAL
    with pytest.raises(ragb.RagbError) as e:
        ragb.workspace_size(10, 256, p)
    assert e.value.code == ragb.RB_EINVAL
    with pytest.raises(ragb.RagbError) as e:
        ragb.workspace_size(10, 5, ragb.make_params(alpha=(1, 20)))
    assert e.value.code == ragb.RB_EALPHA
    ragb.workspace_size(10, 5, ragb.make_params(alpha=(1, 20), flags=ragb.RB_ALPHA_ANY))


def oracle_all(ids, lens=None):
    ctxs = o.validate(ids, lens)
    d = oc.pairwise_rows(ids, lens, 1, 200)
    Z = oc.linkage(d)
    Zt = list(zip(*Z))
    t = o.build_tree(ctxs, Zt)
    ordered, plen = o.offline_order(ctxs, t)
    return ctxs, Z, t, ordered, plen, o.schedule(t.path)


def check_host_index(ids, lens=None):
    ctxs, Z, t, ordered, plen, sched = oracle_all(ids, lens)
    idx = ragb.index_from_linkage(ids, *Z, lens=lens)
    a, b, h, s = idx.linkage()
    for x, y in zip((a, b, h, s), Z):
        assert np.array_equal(x, y)
    assert idx.paths() == t.path
    out, pl, sc = idx.order_contexts()
    N, K = ids.shape
    for i in range(N):
        L = len(ctxs[i])
        assert out[i, :L].tolist() == ordered[i]
        assert np.array_equal(out[i, L:], ids[i, L:])
    assert pl.tolist() == plen
    assert sc.tolist() == sched
    assert canon_lib(idx.tree()) == canon_oracle(t)


def canon_oracle(t):
    out = {}
    stack = [(0, ())]
    while stack:
        k, path = stack.pop()
        out[path] = (t.leaf_of[k], tuple(t.ordered[k]))
        for ci, c in enumerate(t.children[k]):
            stack.append((c, path + (ci,)))
    return out


def canon_lib(tr):
    parent, leaf = tr["parent"], tr["leaf"]
    n = len(parent)
    kids = [[] for _ in range(n)]
    for k in range(1, n):
        kids[parent[k]].append(k)
    for kk in kids:  # children are ordered by rep (X12)
        kk.sort(key=lambda x: int(tr["rep"][x]))
    out = {}
    stack = [(0, ())]
    while stack:
        k, path = stack.pop()
        ordered = tr["prefix_ids"][tr["prefix_off"][k]:tr["prefix_off"][k + 1]].tolist()
        out[path] = (int(leaf[k]), tuple(ordered))
        for ci, c in enumerate(kids[k]):
            stack.append((c, path + (ci,)))
    return out


def test_fig4_fig5_host(golden):
    ids = np.array(golden["fig4_build"]["contexts"], dtype=np.uint32)
    check_host_index(ids)
    idx = ragb.index_from_linkage(ids, *oc.linkage(oc.pairwise_rows(ids, None, 1, 200)))
    assert idx.paths() == golden["fig4_build"]["derived"]["paths"]
    out, plen, _ = idx.order_contexts()
    g = golden["fig5_ordering"]
    assert out[0].tolist() == g["printed"]["C1"] and out[1].tolist() == g["printed"]["C2"]
    assert idx.wait() is idx  # rb_index_wait: nothing pending on a synchronous handle


def test_index_wait_null():
    assert ragb.lib().rb_index_wait(None) == -1  # RB_EINVAL


@pytest.mark.parametrize("seed", range(8))
def test_host_index_random(seed):
    rng = np.random.default_rng(seed)
    N = int(rng.integers(1, 300))
    K = int(rng.integers(1, 12))
    w = generate(N, K, int(rng.integers(K, 8 * K + 20)), seed, len_min=(1 if seed % 2 else None))
    check_host_index(w.ids, w.lens)


@pytest.mark.parametrize("seed", range(3))
def test_host_index_long_lists(seed):
    """K of 40-100 over a small pool: leaf sets longer than 32 (sorted with
    std::sort) and parent sets above 16 docs (the hashed membership of the
    leaves' ordered contexts), fixed and variable lengths."""
    rng = np.random.default_rng(100 + seed)
    K = int(rng.integers(40, 101))
    N = int(rng.integers(20, 90))
    w = generate(N, K, K + int(rng.integers(2, 30)), 100 + seed, len_min=(K - 10 if seed % 2 else None))
    check_host_index(w.ids, w.lens)


@pytest.mark.parametrize("kind", ["disjoint", "identical", "permutations"])
def test_host_index_edges(kind):
    check_host_index(edge(kind, 17, 5).ids)


def test_host_rejects_bad_linkage():
    ids = np.arange(12, dtype=np.uint32).reshape(4, 3)
    with pytest.raises(ragb.RagbError):
        ragb.index_from_linkage(ids, [0, 0, 0], [1, 1, 2], [1, 1, 1], [2, 3, 4])  # b merged twice
    with pytest.raises(ragb.RagbError) as e:
        ragb.index_from_linkage(np.array([[1, 1]], dtype=np.uint32), [], [], [], [])
    assert e.value.code == ragb.RB_EDUPDOC


def test_dedup_matches_oracle(golden):
    g = golden["dedup_example"]
    s = ragb.Session.from_docs(g["turn0"])
    novel, rdoc, rturn = s.dedup_turn(g["turn1"])
    assert novel.tolist() == g["printed"]["novel"] and rdoc.tolist() == g["printed"]["overlap"]
    assert rturn.tolist() == [0, 0] and s.turn == 1
    # multi-turn sessions of the C3 recipe vs the oracle
    w = generate(200, 15, 2000, 3, turns=5)
    for sess in range(10):
        rows = sorted(np.flatnonzero(w.session == sess), key=lambda i: w.turn[i])
        if not rows:
            continue
        so = o.Session(w.ids[rows[0]].tolist())
        sc = ragb.Session.from_docs(w.ids[rows[0]])
        for r in rows[1:]:
            nov, refs = so.dedup_turn(w.ids[r].tolist())
            n2, d2, t2 = sc.dedup_turn(w.ids[r])
            assert n2.tolist() == nov
            assert list(zip(d2.tolist(), t2.tolist())) == refs
    with pytest.raises(ragb.RagbError) as e:
        sc.dedup_turn([5, 5])
    assert e.value.code == ragb.RB_EDUPDOC


def test_session_from_index_path():
    ids = np.array([[2, 1, 4], [5, 7, 8], [1, 2, 9]], dtype=np.uint32)
    idx = ragb.index_from_linkage(ids, *oc.linkage(oc.pairwise_rows(ids, None, 1, 200)))
    s = idx.session(0)
    novel, rdoc, _ = s.dedup_turn([1, 5, 2])
    assert novel.tolist() == [5] and sorted(rdoc.tolist()) == [1, 2]
    with pytest.raises(ragb.RagbError) as e:
        idx.session(7)
    assert e.value.code == ragb.RB_EPATH


def test_order_contexts_into_caller_arrays():
    """order_contexts(out=...) fills the caller's arrays (reused across calls)
    with exactly what the allocating form returns, and rejects mismatched
    arrays."""
    w = generate(300, 6, 900, 77)
    ids = w.ids
    idx = ragb.index_from_linkage(ids, *oc.linkage(oc.pairwise_rows(ids, None, 1, 200)))
    ref = idx.order_contexts()
    bufs = (np.zeros((300, 6), dtype=np.uint32), np.zeros(300, dtype=np.uint8), np.zeros(300, dtype=np.int64))
    for _ in range(2):
        got = idx.order_contexts(out=bufs)
        assert all(g is b for g, b in zip(got, bufs))
        assert all(np.array_equal(g, r) for g, r in zip(got, ref))
    with pytest.raises(ValueError):
        idx.order_contexts(out=(bufs[0], bufs[1], np.zeros(300, dtype=np.int32)))


def test_index_shard_of_host_index():
    """rb_index_shard: an index from a merge list covers all N rows."""
    w = generate(40, 5, 120, 5)
    idx = ragb.index_from_linkage(w.ids, *oc.linkage(oc.pairwise_rows(w.ids, None, 1, 200)))
    assert idx.shard() == (0, 40)
    with pytest.raises(ragb.RagbError):
        lib_counts_bad = ragb.lib().rb_index_counts(idx._h, 0, 41, None, None)  # NULL buffers
        ragb._check(lib_counts_bad)
