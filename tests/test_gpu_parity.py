"""GPU parity: the CUDA path (through the C-ABI) vs the CPU oracle, element by
element on the same seeded inputs.  Bar (BASELINE.json north_star): bit-exact
s/D counts, fp32 distances (correctly rounded, X6 — stronger than the 1e-6
relative bound), nearest neighbours, merge order, tree, document ordering and
schedule."""
from fractions import Fraction

import numpy as np
import pytest

from oracle import oracle_c as oc
from oracle import ragb_oracle as o
from synth.workload import config, edge, generate

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2511_03475_b200 import ragb  # noqa: E402

F = ragb


def dev_build(ids, lens=None, flags=F.RB_KEEP_ROWS, alpha=(1, 200), **kw):
    t = torch.from_numpy(np.ascontiguousarray(ids).view(np.int32)).cuda()
    tl = None if lens is None else torch.from_numpy(np.ascontiguousarray(lens, dtype=np.uint8)).cuda()
    idx, ws = F.build_index(t, tl, alpha=alpha, flags=flags, **kw)
    torch.cuda.synchronize()
    return idx, ws


def oracle_linkage_tree(ids, lens, d_full):
    Z = oc.linkage(d_full)
    ctxs = o.validate(ids, lens)
    t = o.build_tree(ctxs, list(zip(*Z)))
    ordered, plen = o.offline_order(ctxs, t)
    return Z, t, ordered, plen, o.schedule(t.path)


def check_full(ids, lens=None, alpha=(1, 200), counts=True, tuning=None, dref=None):
    """Every distance row, (s, D) rows, row NN, merge order, paths, ordered
    contexts, prefix lengths and schedule vs the oracle; returns the index."""
    N, K = ids.shape
    flags = F.RB_KEEP_ROWS | (F.RB_EMIT_COUNTS if counts else 0)
    idx, ws = dev_build(ids, lens, flags=flags, alpha=alpha, tuning=tuning)
    rows = ws.rows.cpu().numpy()
    if counts:
        dref, sref, Dref = oc.pairwise_rows(ids, lens, alpha[0], alpha[1], counts=True)
    elif dref is None:
        dref = oc.pairwise_rows(ids, lens, alpha[0], alpha[1])
    if counts:
        assert np.array_equal(ws.s.cpu().numpy(), sref)
        assert np.array_equal(ws.D.cpu().numpy().view(np.uint16), Dref)
    assert np.array_equal(rows.view(np.uint32), dref.view(np.uint32))
    nn_i, nn_v = idx.nn()
    ri, rv = oc.row_nn(dref)
    assert np.array_equal(nn_i, ri) and np.array_equal(nn_v.view(np.uint32), rv.view(np.uint32))
    Z, t, ordered, plen, sched = oracle_linkage_tree(ids, lens, dref)
    a, b, h, s = idx.linkage()
    assert np.array_equal(a, Z[0]) and np.array_equal(b, Z[1])
    assert np.array_equal(h.view(np.uint32), Z[2].view(np.uint32)) and np.array_equal(s, Z[3])
    assert idx.paths() == t.path
    out, pl, sc = idx.order_contexts()
    for i in range(N):
        L = K if lens is None else int(lens[i])
        assert out[i, :L].tolist() == ordered[i]
    assert pl.tolist() == plen and sc.tolist() == sched
    return idx


def test_paper_fig4(golden):
    ids = np.array(golden["fig4_build"]["contexts"], dtype=np.uint32)
    idx = check_full(ids)
    assert idx.paths() == golden["fig4_build"]["derived"]["paths"]
    idx2, ws = dev_build(np.array(list(golden["eq1_motivation"]["contexts"].values()), dtype=np.uint32))
    d = ws.rows.cpu().numpy()
    assert hex(int(d[0, 1:2].view(np.uint32)[0])) == golden["eq1_motivation"]["derived"]["AB"]["f32_hex"]


def test_C1_full():
    w = config("C1")
    check_full(w.ids)
    # the python (definition-level) oracle agrees too
    ref = o.build_index(w.ids)
    idx, ws = dev_build(w.ids)
    assert np.array_equal(ws.rows.cpu().numpy().view(np.uint32), ref["d"].view(np.uint32))
    a, b, h, s = idx.linkage()
    assert [(int(x), int(y), np.float32(z), int(q)) for x, y, z, q in zip(a, b, h, s)] == \
        [(x, y, np.float32(z), q) for x, y, z, q in ref["Z"]]


def test_C2_full():
    w = config("C2")
    check_full(w.ids, counts=False)


@pytest.mark.parametrize("N", [1, 2, 3, 31, 77, 1000, 1029, 2053])
def test_ragged_sizes(N):
    w = generate(N, 8, max(40, 3 * N), 100 + N)
    check_full(w.ids)


@pytest.mark.parametrize("K", [1, 5, 10, 15, 20, 32, 33, 50, 75, 100, 128, 200, 255])
def test_K_sweep(K):
    w = generate(700 if K <= 100 else 300, K, max(4 * K, 3000), 5)
    check_full(w.ids, counts=K <= 100)


@pytest.mark.parametrize("alpha", [(1, 1000), (1, 100), (3, 700), (7, 997)])
def test_alpha(alpha):
    w = generate(600, 12, 2000, 9)
    check_full(w.ids, alpha=alpha, counts=False)


def test_variable_lengths():
    w = generate(900, 16, 3000, 21, len_min=2)
    check_full(w.ids, w.lens)


@pytest.mark.parametrize("kind", ["disjoint", "identical", "permutations"])
def test_edges(kind):
    check_full(edge(kind, 300, 7).ids)


def test_errors():
    ids = np.array([[1, 2, 3], [4, 5, 4]], dtype=np.uint32)
    with pytest.raises(F.RagbError) as e:
        dev_build(ids)
    assert e.value.code == F.RB_EDUPDOC
    with pytest.raises(F.RagbError) as e:
        dev_build(np.array([[1, 0xFFFFFFFF]], dtype=np.uint32))
    assert e.value.code == F.RB_EINVAL
    with pytest.raises(F.RagbError) as e:
        dev_build(np.array([[1, 2]], dtype=np.uint32), lens=np.array([3], dtype=np.uint8))
    assert e.value.code == F.RB_EINVAL
    # duplicates beyond lens are ignored
    dev_build(np.array([[1, 2, 2], [3, 4, 5]], dtype=np.uint32), lens=np.array([2, 3], dtype=np.uint8))


def test_row_shard_and_skip_linkage():
    w = generate(1500, 20, 8000, 31)
    dref = oc.pairwise_rows(w.ids, None, 1, 200)
    for row0, nrows in [(0, 700), (700, 800), (13, 1)]:
        idx, ws = dev_build(w.ids, flags=0, row0=row0, nrows=nrows)
        assert np.array_equal(ws.rows.cpu().numpy().view(np.uint32),
                              dref[row0:row0 + nrows].view(np.uint32))
        ni, nv = idx.nn(nrows)
        ri, rv = oc.row_nn(dref[row0:row0 + nrows], row0=row0)
        assert np.array_equal(ni, ri) and np.array_equal(nv, rv)
        with pytest.raises(F.RagbError):
            idx.linkage()


def test_host_entry_matches_device_entry():
    w = generate(1200, 20, 6000, 8)
    idx1, _ = dev_build(w.ids, flags=0)
    idx2, _ = F.build_index_host(w.ids)
    for x, y in zip(idx1.linkage(), idx2.linkage()):
        assert np.array_equal(x, y)
    assert np.array_equal(idx1.order_contexts()[0], idx2.order_contexts()[0])


def test_consumed_rows_linkage_equals_kept():
    w = generate(3000, 20, 1_000_000 // 30, 4)
    i1, _ = dev_build(w.ids, flags=0)
    i2, _ = dev_build(w.ids, flags=F.RB_KEEP_ROWS)
    for x, y in zip(i1.linkage(), i2.linkage()):
        assert np.array_equal(x, y)


@pytest.mark.parametrize("case", ["random", "ties"])
def test_deterministic_repeat(case):
    """Repeated builds give the same bytes: merge order, schedule and the
    exported tree numbering (parent, rep, prefixes; ragb.h rb_index_tree)."""
    w = generate(2000, 20, 20000, 77) if case == "random" else generate(6000, 3, 60000, 5)
    runs = [dev_build(w.ids, flags=0)[0] for _ in range(3)]
    t0 = runs[0].tree()
    for r in runs[1:]:
        for x, y in zip(r.linkage(), runs[0].linkage()):
            assert np.array_equal(x, y)
        assert np.array_equal(r.order_contexts()[2], runs[0].order_contexts()[2])
        t = r.tree()
        for k in t0:
            assert np.array_equal(t[k], t0[k]), k


def test_async_host_pipelined():
    """RB_ASYNC_HOST (ragb.h rb_index_wait): builds return after the device
    stages and finish the host stage on a library thread; two pipelined builds
    sharing one workspace (the second launched while the first's host stage
    may still run) equal synchronous builds byte for byte, and also through
    the host-buffer entry."""
    cases = [generate(3000, 20, 30000, 91), generate(5000, 4, 2000, 17)]
    ref = []
    for w in cases:
        idx, _ = dev_build(w.ids, flags=0)
        ref.append((idx.linkage(), idx.order_contexts(), idx.tree()))
    for w, (lk, oc_, tr) in zip(cases, ref):
        t = torch.from_numpy(np.ascontiguousarray(w.ids).view(np.int32)).cuda()
        a, ws = F.build_index(t, flags=F.RB_ASYNC_HOST)
        b, ws = F.build_index(t, flags=F.RB_ASYNC_HOST, workspace=ws)  # a's host stage may still run
        c, _ = F.build_index_host(w.ids, flags=F.RB_ASYNC_HOST, workspace=ws)
        for idx in (b, a, c):  # b settles first: every accessor waits by itself
            for x, y in zip(idx.linkage(), lk):
                assert np.array_equal(x, y)
            for x, y in zip(idx.order_contexts(), oc_):
                assert np.array_equal(x, y)
            tt = idx.tree()
            for k in tr:
                assert np.array_equal(tt[k], tr[k]), k
            st = idx.wait().stats()
            assert st["host_ms"] > 0 and st["total_ms"] >= st["linkage_ms"]
        del a, b, c  # rb_index_free joins a pending host stage


def test_async_host_soak_C3():
    """Eight pipelined C3 builds on one workspace, each read back on a helper
    thread while the next build runs (the bench's pattern): every one equals
    the synchronous build."""
    from concurrent.futures import ThreadPoolExecutor
    w = config("C3")
    ref, _ = dev_build(w.ids, flags=0)
    ra, ro = ref.linkage(), ref.order_contexts()
    t = torch.from_numpy(np.ascontiguousarray(w.ids).view(np.int32)).cuda()
    ws = None

    def check(idx):
        for x, y in zip(idx.linkage(), ra):
            assert np.array_equal(x, y)
        for x, y in zip(idx.order_contexts(), ro):
            assert np.array_equal(x, y)
        return True

    with ThreadPoolExecutor(max_workers=1) as ex:
        futs = []
        for _ in range(8):
            idx, ws = F.build_index(t, flags=F.RB_ASYNC_HOST, workspace=ws)
            futs.append(ex.submit(check, idx))
            del idx
        assert all(f.result() for f in futs)


# ------------------------------------------------------------- full sizes
def linkage_properties(a, b, h, s, N):
    """Properties of a complete-linkage merge order that hold at any size."""
    assert len(a) == N - 1
    assert np.all(a < b)
    h0, h1, a0, a1, b0, b1 = h[:-1], h[1:], a[:-1], a[1:], b[:-1], b[1:]
    inc = (h1 > h0) | ((h1 == h0) & ((a1 > a0) | ((a1 == a0) & (b1 > b0))))
    assert np.all(inc)   # strictly increasing key (X9)
    rep_alive = np.ones(N, dtype=bool)
    size = np.ones(N, dtype=np.int64)
    for x, y, z in zip(a.tolist(), b.tolist(), s.tolist()):
        assert rep_alive[x] and rep_alive[y]
        size[x] += size[y]
        rep_alive[y] = False
        assert size[x] == z
    assert rep_alive.sum() == 1 and size[0] == N


def sampled_rows_check(ids, rows_dev, sample, lens=None, alpha=(1, 200)):
    for r in sample:
        ref = oc.pairwise_rows(ids, lens, alpha[0], alpha[1], row0=int(r), nrows=1)
        got = rows_dev[int(r)].cpu().numpy()
        assert np.array_equal(got.view(np.uint32), ref[0].view(np.uint32)), f"row {r}"


@pytest.mark.parametrize("name", ["C3", "C4"])
def test_full_size_configs(name):
    """BASELINE.json configs at full size, bench launch configuration: sampled
    rows vs the oracle one by one, nn of sampled rows, linkage/tree/order
    properties, sampled merges against the complete-linkage definition."""
    w = config(name)
    N, K = w.ids.shape
    rng = np.random.default_rng(0)
    sample = np.unique(np.concatenate([[0, N - 1], rng.integers(0, N, 30)]))
    idx, ws = dev_build(w.ids, flags=F.RB_SKIP_LINKAGE)
    sampled_rows_check(w.ids, ws.rows, sample)
    ni, nv = idx.nn()
    for r in sample:
        ref = oc.pairwise_rows(w.ids, None, 1, 200, row0=int(r), nrows=1)
        ri, rv = oc.row_nn(ref, row0=int(r))
        assert ni[r] == ri[0] and nv[r] == rv[0]
    del ws
    torch.cuda.empty_cache()
    idx, ws = dev_build(w.ids, flags=0)   # bench configuration: rows consumed by the linkage
    a, b, h, s = idx.linkage()
    linkage_properties(a, b, h, s, N)
    # first merge = global min pair of the nn array (greedy's first step)
    i0 = int(np.lexsort((np.arange(N), nv))[0])
    assert (a[0], b[0]) == tuple(sorted((i0, int(ni[i0]))))
    # sampled small merges: height == max over member pairs (definition, X7)
    members = {i: [i] for i in range(N)}   # member lists of small clusters only
    checked = 0
    for x, y, z in zip(a.tolist(), b.tolist(), h.tolist()):
        A, B = members.get(x), members.pop(y, None)
        if A is not None and B is not None and checked < 40 and len(A) * len(B) <= 64 \
                and rng.random() < 0.02:
            dsub = oc.pairwise_rows(w.ids[A + B], None, 1, 200)
            assert np.float32(dsub[:len(A), len(A):].max()) == np.float32(z)
            checked += 1
        if A is not None and B is not None and len(A) + len(B) <= 16:
            members[x] = A + B
        else:
            members.pop(x, None)
    assert checked > 0
    out, pl, sc = idx.order_contexts()
    assert np.array_equal(np.sort(out, axis=1), np.sort(w.ids, axis=1))  # permutations
    assert np.array_equal(np.sort(sc), np.arange(N))
    paths = idx.paths()
    firsts = np.array([paths[i][0] for i in sc])
    change = np.flatnonzero(firsts[1:] != firsts[:-1])
    assert len(change) + 1 == len(np.unique(firsts))   # contiguous groups
    # tree/order: host step re-run from the device merge order == library result
    idx2 = F.index_from_linkage(w.ids, a, b, h, s)
    assert np.array_equal(idx2.order_contexts()[0], out)


# ------------------------------------- the paths full-size builds take, vs the oracle
# Inputs that reach, at sizes the oracle still finishes in about a minute, the
# kernel variants C3/C4 run: level cliques on more than 4096 vertices (block
# path), the 1024-thread row gather (M > 16K) and the 1024-thread window
# compaction (M' > 20K; fp32 matrices, or codes with the gather off).  The
# path bits of rb_stats prove each case reaches its path.
BIG = {
    "block10k": ((10000, 3, 100000, 5), None, F.RB_PATH_CLIQUE_BLOCK),
    "gather20k": ((20000, 3, 100000, 43), None, F.RB_PATH_CLIQUE_BLOCK | F.RB_PATH_GATHER_WIDE),
    "window24k_fp32": ((24000, 3, 100000, 45), dict(value_codes=0), F.RB_PATH_WINDOW_WIDE),
    "window24k_codes": ((24000, 3, 100000, 45), dict(gather=0), F.RB_PATH_WINDOW_WIDE),
    "ties20k_K4": ((20000, 4, 2000, 41), None, F.RB_PATH_GATHER_WIDE),
}


@pytest.mark.parametrize("case", list(BIG))
def test_full_size_paths_vs_oracle(case):
    (N, K, V, seed), tu, bits = BIG[case]
    w = generate(N, K, V, seed)
    idx = check_full(w.ids, counts=False, tuning=tu)
    st = idx.stats()
    assert st["paths"] & bits == bits, (case, hex(st["paths"]), st["max_level"])


def test_C3_full_vs_oracle():
    """C3 (N = 32,768, K = 15, 5-turn sessions) end to end against the oracle:
    all 1.07e9 distances, row NN, merge order (C NN-chain over the oracle's
    own rows), paths, document order and schedule (Python oracle tree); then
    the bench launch configuration (rows consumed by the linkage) gives the
    same merge order and document order."""
    w = config("C3")
    dref = oc.pairwise_rows(w.ids, None, 1, 200)
    idx = check_full(w.ids, counts=False, dref=dref)
    del dref
    ref_link, ref_order = idx.linkage(), idx.order_contexts()
    idx2, ws = dev_build(w.ids, flags=0)
    for x, y in zip(ref_link + ref_order, idx2.linkage() + idx2.order_contexts()):
        assert np.array_equal(x, y)


@pytest.mark.parametrize("codes,side", [(0, -1), (-1, -1), (-1, 0)])
@pytest.mark.parametrize("mode", [0, 1])
@pytest.mark.parametrize("case", ["C2", "var", "ties"])
def test_round_strategy(mode, case, codes, side):
    """Linkage rounds in place (inplace=1, forced wherever allowed) or always
    compacting (0), on fp32 matrices (value_codes=0) or on 16-bit value codes
    (default where the Eq. 1 table exists), with the in-place side buffer
    (default in code mode) or in-place column rewrites (side_buffer=0), give
    the oracle's merge order (the strategy and the stored form are
    implementation choices, X7-X9 fix the result)."""
    if mode == 0 and side == 0:
        pytest.skip("no in-place rounds: the side buffer is not used")
    tu = dict(inplace=mode, value_codes=codes, side_buffer=side, nn_cache=-1 if side else 0)
    if case == "C2":
        idx = check_full(config("C2").ids, counts=False, tuning=tu)
    elif case == "var":
        w = generate(2500, 12, 6000, 31, len_min=2)
        idx = check_full(w.ids, w.lens, counts=False, tuning=tu)
    else:  # tie-heavy: tiny pool, short lists -> many equal heights and cliques
        w = generate(3000, 4, 300, 32)
        idx = check_full(w.ids, counts=False, tuning=tu)
    if mode == 1:
        assert idx.stats()["paths"] & F.RB_PATH_INPLACE


@pytest.mark.parametrize("K", [7, 22, 23, 30, 32])
def test_code_mode_fast_path(K):
    """Code mode through the tile kernel's fast finalize (no (s, D) output):
    both Eq. 1 table layouts (K <= 22: packed byte offsets into a shared-memory
    table; 23 <= K <= 32: global table) give the oracle's rows, row NN, merge
    order and document order, with a ragged last tile and column chunk."""
    w = generate(2000 + 3 * K, K, 60 * K, 500 + K)
    idx = check_full(w.ids, counts=False)
    assert idx.stats()["value_codes"] == 1


@pytest.mark.parametrize("K", [33, 48, 64, 65, 100, 128])
def test_wide_lists(K):
    """Uniform 32 < K <= 128 (the long-list distance kernel, both candidate-
    mask widths, with and without the (s, D) output): rows, row NN, merge
    order and document order equal the oracle's; odd N and a ragged last
    tile and chunk."""
    w = generate(1201 + K, K, 40 * K, 900 + K)
    check_full(w.ids, counts=False)
    check_full(w.ids[: 333], counts=True)


@pytest.mark.parametrize("case", ["C2", "odd"])
def test_code_window_compaction(case):
    """Code-mode compaction through the shared-memory window kernel
    (gather=0; the path for matrices too wide for the gather kernel) gives the
    oracle's merge order, also for an odd N (scalar loads)."""
    ids = config("C2").ids if case == "C2" else generate(1029, 8, 3087, 1129).ids
    idx = check_full(ids, counts=False, tuning=dict(gather=0))
    assert idx.stats()["paths"] & F.RB_PATH_WINDOW


def test_round_strategy_full_size():
    """At C4 size (level cliques above 4096 vertices, block path) the merge
    order and the document order do not depend on the round strategy, on the
    stored form of the matrices (fp32 values or 16-bit value codes), on the
    in-place side buffer nor on the second-nearest cache."""
    ids = config("C4").ids
    t = torch.from_numpy(ids.view(np.int32)).cuda()
    res = []
    for mode, codes, side, nnc in ((0, -1, -1, -1), (-1, -1, -1, -1), (-1, 0, -1, -1), (-1, -1, 0, -1),
                                   (-1, -1, -1, 0)):
        idx, ws = F.build_index(t, tuning=dict(inplace=mode, value_codes=codes, side_buffer=side, nn_cache=nnc))
        res.append((idx.linkage(), idx.order_contexts()))
        del idx, ws
        torch.cuda.empty_cache()
    for r in res[1:]:
        for x, y in zip(res[0][0] + res[0][1], r[0] + r[1]):
            assert np.array_equal(x, y)


def test_multiturn_cumulative_index():
    """NEXT-2: sessions' cumulative contexts (turn-0 ++ novel docs) are
    variable-length (X4); their index on the GPU equals the oracle's."""
    w = generate(6000, 10, 9000, 12, turns=4)
    t0 = {int(w.session[i]): i for i in range(w.N) if w.turn[i] == 0}
    sids = sorted(t0)
    pos = {s: q for q, s in enumerate(sids)}
    sess = [F.Session.from_docs(w.ids[t0[s]]) for s in sids]
    follow = sorted((int(w.turn[i]), i) for i in range(w.N) if w.turn[i] > 0)
    rows = np.array([i for _, i in follow], dtype=np.int64)
    F.dedup_batch(sess, np.array([pos[int(w.session[i])] for i in rows]), w.ids[rows])
    ctxs = [s.context() for s in sess]
    Kc = max(len(c) for c in ctxs)
    ids = np.zeros((len(ctxs), Kc), dtype=np.uint32)
    lens = np.array([len(c) for c in ctxs], dtype=np.uint8)
    for q, c in enumerate(ctxs):
        ids[q, :len(c)] = c
    assert lens.max() > 10
    check_full(ids, lens, counts=False)


def check_intersection(ids, lens=None, flags=F.RB_KEEP_ROWS):
    """NEXT-3: device intersection-representative linkage vs the C oracle
    (merge order, heights bit-exact), then the tree / order / schedule the
    merges imply (build_tree replays merges in merge order)."""
    N, K = ids.shape
    idx, ws = dev_build(ids, lens, flags=flags, linkage=F.RB_LINK_INTERSECTION)
    a, b, h, s = idx.linkage()
    za, zb, zh, zs = oc.linkage_intersection(ids, lens, 1, 200)
    assert np.array_equal(a, za) and np.array_equal(b, zb) and np.array_equal(s, zs)
    assert np.array_equal(h.view(np.uint32), zh.view(np.uint32))
    ctxs = o.validate(ids, lens)
    t = o.build_tree(ctxs, list(zip(za.tolist(), zb.tolist(), zh.tolist(), zs.tolist())))
    assert idx.paths() == t.path
    ordered, plen = o.offline_order(ctxs, t)
    out, pl, sc = idx.order_contexts()
    for i in range(N):
        L = K if lens is None else int(lens[i])
        assert out[i, :L].tolist() == ordered[i]
    assert pl.tolist() == plen and sc.tolist() == o.schedule(t.path)
    if flags & F.RB_KEEP_ROWS:  # the distance rows are untouched
        dref = oc.pairwise_rows(ids, lens, 1, 200)
        assert np.array_equal(ws.rows.cpu().numpy().view(np.uint32), dref.view(np.uint32))


def test_intersection_fig4(golden):
    ids = np.array(golden["fig4_build"]["contexts"], dtype=np.uint32)
    check_intersection(ids)


@pytest.mark.parametrize("N,K,V,seed", [(64, 5, 200, 1), (1, 4, 10, 2), (2, 4, 10, 3), (37, 3, 20, 4),
                                        (500, 8, 1500, 5), (1500, 10, 4000, 6), (700, 4, 80, 7)])
def test_intersection_linkage(N, K, V, seed):
    w = generate(N, K, V, seed)
    check_intersection(w.ids)


def test_intersection_variable_lengths_and_consumed_rows():
    w = generate(900, 12, 2500, 8, len_min=2)
    check_intersection(w.ids, w.lens)
    check_intersection(w.ids, w.lens, flags=0)


def _dist_vs_single(ids, lens, world, tuning=None):
    t = torch.from_numpy(np.ascontiguousarray(ids).view(np.int32)).cuda()
    tl = None if lens is None else torch.from_numpy(np.ascontiguousarray(lens, dtype=np.uint8)).cuda()
    db = F.DistBuilder(world, ids.shape[0], ids.shape[1], local=True)
    di = db.build(t, tl, tuning=tuning)
    res_d = (di.linkage(), di.nn(), di.order_contexts(), di.paths())
    del db, di
    torch.cuda.empty_cache()
    si, ws = F.build_index(t, tl, tuning=tuning)
    res_s = (si.linkage(), si.nn(), si.order_contexts(), si.paths())
    del si, ws
    torch.cuda.empty_cache()
    for x, y in zip(res_d[0] + res_d[1] + res_d[2], res_s[0] + res_s[1] + res_s[2]):
        assert np.array_equal(np.asarray(x).view(np.uint8), np.asarray(y).view(np.uint8))
    assert res_d[3] == res_s[3]


@pytest.mark.parametrize("world", [1, 2, 3, 4, 8])
def test_row_sharded_build_matches_single_gpu(world):
    """§8(e): the row-sharded build (ranks simulated in one process on one GPU,
    member rows read through the peer tables) gives the single-GPU (and so the
    oracle's) merge order, NN, document order, schedule and paths."""
    _dist_vs_single(config("C2").ids, None, world)
    w = generate(2053, 12, 5000, 77, len_min=3)
    _dist_vs_single(w.ids, w.lens, world)
    w = generate(1500, 4, 200, 78)  # tie-heavy: large level cliques
    _dist_vs_single(w.ids, None, world)


@pytest.mark.parametrize("world", [2, 3])
def test_row_sharded_fp32_matrices(world):
    """The sharded rounds on fp32 matrices (value_codes=0; the code-mode rounds
    are the default for uniform K <= 32) give the same index."""
    tu = dict(value_codes=0)
    _dist_vs_single(config("C2").ids, None, world, tu)
    w = generate(1500, 4, 200, 78)
    _dist_vs_single(w.ids, None, world, tu)


def test_row_sharded_tiny_and_vs_oracle():
    w = generate(5, 4, 12, 3)
    _dist_vs_single(w.ids, None, 8)  # fewer rows than ranks
    w = config("C1")
    t = torch.from_numpy(w.ids.view(np.int32)).cuda()
    di = F.DistBuilder(3, w.N, w.K, local=True).build(t)
    Z = oc.linkage(oc.pairwise_rows(w.ids, None, 1, 200))
    a, b, h, s = di.linkage()
    assert np.array_equal(a, Z[0]) and np.array_equal(b, Z[1]) and np.array_equal(s, Z[3])
    assert np.array_equal(h.view(np.uint32), Z[2].view(np.uint32))


def test_row_sharded_full_size_C4():
    """C4 with 8 ranks' shards on one device (~130 GB): identical to the
    single-GPU build."""
    _dist_vs_single(config("C4").ids, None, 8)


@pytest.mark.parametrize("seed", range(6))
def test_inplace_side_buffer_and_cache_random(seed):
    """Random tie-heavy and clustered inputs with in-place rounds forced
    wherever allowed: the side buffer (dirty columns, slot retirement,
    capacity flushes, the patch into the next compaction) and the
    second-nearest cache give the oracle's merge order, tree and orders, and
    the same result as the column-rewrite form without the cache."""
    rng = np.random.default_rng(1000 + seed)
    N = int(rng.integers(1500, 5000))
    K = int(rng.integers(3, 12))
    V = int(rng.integers(K * 20, K * 400))
    w = generate(N, K, V, 2000 + seed)
    idx = check_full(w.ids, counts=False, tuning=dict(inplace=1))
    ref, _ = dev_build(w.ids, flags=0, tuning=dict(inplace=1, side_buffer=0, nn_cache=0))
    for x, y in zip(idx.linkage() + idx.order_contexts(), ref.linkage() + ref.order_contexts()):
        assert np.array_equal(x, y)


def test_index_counts_and_shard():
    """rb_index_counts recomputes (s, D) rows of the indexed set equal to the
    RB_EMIT_COUNTS output of the build (and to the oracle's); rb_index_shard
    reports the built row range."""
    w = config("C2")
    N = w.ids.shape[0]
    idx, ws = dev_build(w.ids, flags=F.RB_KEEP_ROWS | F.RB_EMIT_COUNTS)
    assert idx.shard() == (0, N)
    s, D = idx.counts(0, N)
    assert torch.equal(s, ws.s) and torch.equal(D, ws.D)
    s2, D2 = idx.counts(1000, 77)
    _, sref, Dref = oc.pairwise_rows(w.ids, None, 1, 200, counts=True, row0=1000, nrows=77)
    assert np.array_equal(s2.cpu().numpy(), sref) and np.array_equal(D2.cpu().numpy().view(np.uint16), Dref)
    t = torch.from_numpy(w.ids.view(np.int32)).cuda()
    part, _ = F.build_index(t, row0=512, nrows=256)
    assert part.shard() == (512, 256)
