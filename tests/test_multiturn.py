"""NEXT-2 (multi-turn at scale): the C3 workload's follow-up
turns de-duplicated in one batch by the library vs the oracle's Session, and
the cumulative session contexts (turn-0 context ++ novel docs)
that make the next index variable-length (X4).  Host logic only."""
import numpy as np
import pytest

from oracle import oracle_c as oc
from oracle import ragb_oracle as o
from paper_2511_03475_b200 import ragb
from synth.workload import config, generate


def sessions_of(w):
    """turn-0 row of every session, and the follow-up rows in turn order."""
    t0 = {}
    follow = []
    for i in range(w.N):
        s, t = int(w.session[i]), int(w.turn[i])
        if t == 0:
            t0[s] = i
        else:
            follow.append((t, s, i))
    follow.sort()
    return t0, follow


def run_both(w, t0, follow, turn0_docs):
    sids = sorted(t0)
    pos = {s: q for q, s in enumerate(sids)}
    lib_s = [ragb.Session.from_docs(turn0_docs(t0[s])) for s in sids]
    ora_s = [o.Session(turn0_docs(t0[s])) for s in sids]
    rows = np.array([i for _, _, i in follow], dtype=np.int64)
    ts = np.array([pos[s] for _, s, _ in follow], dtype=np.int64)
    novel, nn, rdoc, rturn, nr = ragb.dedup_batch(lib_s, ts, w.ids[rows])
    for z, (_, s, i) in enumerate(follow):
        ev_novel, ev_refs = ora_s[pos[s]].dedup_turn(w.ids[i].tolist())
        assert novel[z, :nn[z]].tolist() == ev_novel
        assert list(zip(rdoc[z, :nr[z]].tolist(), rturn[z, :nr[z]].tolist())) == ev_refs
    for q, s in enumerate(sids):
        assert lib_s[q].turn == ora_s[q].turn
    return sids, lib_s, ora_s


def test_c3_dedup_batch_vs_oracle():
    w = config("C3")  # 6,554 sessions x 5 turns, K = 15
    t0, follow = sessions_of(w)
    assert len(t0) == 6554 and len(follow) == w.N - 6554
    sids, lib_s, ora_s = run_both(w, t0, follow, lambda i: w.ids[i].tolist())
    # cumulative contexts: turn-0 docs ++ novel docs of turns 1.. in order
    for q in range(0, len(sids), 97):
        ctx = lib_s[q].context().tolist()
        assert ctx[:15] == w.ids[t0[sids[q]]].tolist()
        novel_all = [d for d, t in ora_s[q].seen.items() if t > 0]  # insertion = prefill order
        assert ctx[15:] == novel_all and len(set(ctx)) == len(ctx)
    # conservation: novel + refs = retrieved, per turn
    tot = sum(len(x) for x in (w.ids[i] for _, _, i in follow))
    assert tot == len(follow) * 15


def test_sessions_from_index_rows_and_cumulative_index():
    w = generate(1200, 8, 3000, 11, turns=4)
    t0, follow = sessions_of(w)
    sids = sorted(t0)
    base = w.ids[[t0[s] for s in sids]]
    Z = oc.linkage(oc.pairwise_rows(base, None, 1, 200))
    idx = ragb.index_from_linkage(base, *Z)
    out, _, _ = idx.order_contexts()
    # turn 0 of session q = indexed row q, served in its prefix-first order
    sids2, lib_s, ora_s = run_both(w, {s: q for q, s in enumerate(sids)}, [
        (t, s, i) for t, s, i in follow], lambda q: out[q].tolist())
    assert lib_s[0].context()[:8].tolist() == out[0].tolist()
    # the cumulative contexts are variable-length inputs to the next index
    ctxs = [s.context() for s in lib_s]
    Kc = max(len(c) for c in ctxs)
    assert Kc <= 255
    ids = np.zeros((len(ctxs), Kc), dtype=np.uint32)
    lens = np.array([len(c) for c in ctxs], dtype=np.uint8)
    for q, c in enumerate(ctxs):
        ids[q, :len(c)] = c
    assert lens.min() >= 8 and lens.max() > 8
    o.validate(ids, lens)


def test_dedup_batch_errors():
    s = [ragb.Session.from_docs([1, 2, 3])]
    with pytest.raises(ragb.RagbError) as e:
        ragb.dedup_batch(s, [1], np.array([[4, 5, 6]], dtype=np.uint32))
    assert e.value.code == ragb.RB_ESESSION
    with pytest.raises(ragb.RagbError) as e:
        ragb.dedup_batch(s, [0, 0], np.array([[4, 5, 6], [7, 7, 8]], dtype=np.uint32))
    assert e.value.code == ragb.RB_EDUPDOC
    assert s[0].turn == 0  # validated before any state change
    novel, nn, rdoc, rturn, nr = ragb.dedup_batch(s, [0, 0], np.array([[4, 1, 6], [6, 7, 2]], dtype=np.uint32))
    assert novel[0, :nn[0]].tolist() == [4, 6] and novel[1, :nn[1]].tolist() == [7]
    assert list(zip(rdoc[1, :nr[1]], rturn[1, :nr[1]])) == [(6, 1), (2, 0)]
    assert s[0].context().tolist() == [1, 2, 3, 4, 6, 7]
