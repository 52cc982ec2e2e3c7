"""RAGBoost context-index ORACLE — plain, slow, obviously correct CPU code.

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this
module.  The product path (``paper_2511_03475_b200``) never imports it, and it
shares no code with that path (no kernels, headers, helpers or constants).

Every function cites the passage of /root/reference/PAPER.md (``PAPER:n`` =
line n; section / equation named) it follows.  Where the paper is silent or
ambiguous the reading is the one of SURVEY.md §8(c) (``X#``), all listed in
DESIGN.md "Readings".

Pins (tests/test_oracle_*.py): paper worked examples (PAPER:337, 344-348,
378-382, 429-433, 454-462, 508-513), closed forms (identity, disjoint,
footrule permutation, one shared doc), invariants, brute force against an
independent K×K implementation (oracle/c), scipy complete linkage on tie-free
matrices, greedy vs. NN-chain.
"""
from __future__ import annotations

from fractions import Fraction

import numpy as np

PAD_ID = 0xFFFFFFFF


class OracleError(ValueError):
    pass


# --------------------------------------------------------------------------- O1
def validate(ids, lens=None):
    """O1 / a1: K ∈ [1,255], 1 ≤ len_i ≤ K, DocId ≠ 0xFFFFFFFF, no duplicate DocId
    within a context ("docs contains no duplicate DocId"; X5).  Returns the
    contexts as Python lists of ints in retrieval order."""
    ids = np.asarray(ids)
    if ids.ndim != 2:
        raise OracleError("ids must be [N, K]")
    N, K = ids.shape
    if N < 1 or not (1 <= K <= 255):
        raise OracleError("bad N/K")
    out = []
    for i in range(N):
        L = K if lens is None else int(lens[i])
        if not (1 <= L <= K):
            raise OracleError(f"len out of range at row {i}")
        row = [int(x) for x in ids[i, :L]]
        if any(x == PAD_ID for x in row):
            raise OracleError(f"reserved DocId at row {i}")
        if len(set(row)) != len(row):
            raise OracleError(f"duplicate DocId in context {i}")
        out.append(row)
    return out


# ------------------------------------------------------------------------ O2/O3
def overlap(ci, cj):
    """O2: S_ij (shared docs) and the positional sum Σ_{k∈S_ij} |p_i(k) − p_j(k)|
    of Eq. 1, positions 0-based (X2).  A dict of positions, no
    sorting tricks."""
    pos_i = {doc: p for p, doc in enumerate(ci)}
    pos_j = {doc: p for p, doc in enumerate(cj)}
    s = 0
    D = 0
    for doc, pi in pos_i.items():
        if doc in pos_j:
            s += 1
            D += abs(pi - pos_j[doc])
    return s, D


def distance_exact(ci, cj, alpha: Fraction) -> Fraction:
    """Eq. 1 as an exact rational:
    d_ij = 1 − |S_ij| / max(|C_i|,|C_j|) + α · Σ|p_i(k) − p_j(k)| / |S_ij|,
    with the positional term 0 when S_ij = ∅ (X3)."""
    s, D = overlap(ci, cj)
    m = max(len(ci), len(cj))
    if s == 0:
        return Fraction(1)
    return 1 - Fraction(s, m) + alpha * Fraction(D, s)


def rn32(q: Fraction) -> np.float32:
    """Correctly rounded (round-to-nearest-even) binary32 value of a non-negative
    rational (X6: d := RN32 of the exact Eq. 1 value).  Picks among the float32
    neighbours of the double approximation by exact rational distance."""
    if q < 0:
        raise OracleError("negative distance")
    c0 = np.float32(float(q))
    cands = {c0, np.nextafter(c0, np.float32(np.inf)), np.nextafter(c0, np.float32(0))}
    best = None
    for c in cands:
        err = abs(Fraction(float(c)) - q)
        key = (err, int(np.array(c, dtype=np.float32).view(np.uint32)) & 1)
        if best is None or key < best[0]:
            best = (key, c)
    return np.float32(best[1])


def distance(ci, cj, alpha: Fraction) -> np.float32:
    """O3: canonical fp32 Eq. 1 distance = RN32(exact rational) (X6)."""
    return rn32(distance_exact(ci, cj, alpha))


def alpha_fraction(alpha, max_den: int = 1000) -> Fraction:
    """X1: α is carried as an exact rational with denominator ≤ 1000
    ("α ∈ [0.001, 0.01]")."""
    return Fraction(alpha).limit_denominator(max_den)


def pairwise(ctxs, alpha: Fraction):
    """A2 ("compute pairwise distances between all contexts"): full
    N×N matrices of s (uint8), D (uint16) and fp32 d.  O(N²·K) Python — small N."""
    N = len(ctxs)
    S = np.zeros((N, N), dtype=np.uint8)
    Dm = np.zeros((N, N), dtype=np.uint16)
    d = np.zeros((N, N), dtype=np.float32)
    for i in range(N):
        for j in range(i, N):
            s, D = overlap(ctxs[i], ctxs[j])
            v = distance(ctxs[i], ctxs[j], alpha)
            S[i, j] = S[j, i] = s
            Dm[i, j] = Dm[j, i] = D
            d[i, j] = d[j, i] = v
    return S, Dm, d


# --------------------------------------------------------------------------- O4
def row_nn(d: np.ndarray):
    """O4: nn_i = argmin_{j≠i} (d_ij, j) (north_star "row-wise min/argmin").
    N == 1 → (-1, +inf)."""
    N = d.shape[0]
    idx = np.full(N, -1, dtype=np.int32)
    val = np.full(N, np.inf, dtype=np.float32)
    for i in range(N):
        best = None
        for j in range(N):
            if j == i:
                continue
            key = (d[i, j], j)
            if best is None or key < best:
                best = key
        if best is not None:
            val[i], idx[i] = best
    return idx, val


# --------------------------------------------------------------------------- O5
def linkage_greedy(d: np.ndarray):
    """O5 ("iteratively merge the closest pair"): greedy complete
    linkage (X7) with the tie key (D(A,B), min rep, max rep), rep = smallest leaf
    index of a cluster (X8).  D(A∪B, C) = max(D(A,C), D(B,C)) is the maximum over
    member pairs.  Brute force: every step scans every active pair.  Returns rows
    (rep_a < rep_b, h, size) in merge order."""
    N = d.shape[0]
    size = {i: 1 for i in range(N)}
    dist = {}
    for i in range(N):
        for j in range(i + 1, N):
            dist[(i, j)] = d[i, j]
    Z = []
    while len(size) > 1:
        best = None
        act = sorted(size)
        for x in range(len(act)):
            for y in range(x + 1, len(act)):
                a, b = act[x], act[y]
                key = (dist[(a, b)], a, b)
                if best is None or key < best:
                    best = key
        h, a, b = best
        Z.append((a, b, np.float32(h), size[a] + size[b]))
        for c in size:
            if c in (a, b):
                continue
            dac = dist[(min(a, c), max(a, c))]
            dbc = dist[(min(b, c), max(b, c))]
            dist[(min(a, c), max(a, c))] = max(dac, dbc)
        size[a] += size.pop(b)
    return Z


def linkage_nn_chain(d: np.ndarray):
    """O5 by an independent algorithm: nearest-neighbour chain (valid because
    complete linkage is reducible; X7/X8).  Merges are emitted in chain order and
    then sorted by the key (h, rep_a, rep_b), which is the greedy order (X9).
    numpy row scans; medium N."""
    N = d.shape[0]
    D = d.astype(np.float64).copy()
    np.fill_diagonal(D, np.inf)
    active = np.ones(N, dtype=bool)
    size = np.ones(N, dtype=np.int64)
    idx = np.arange(N)
    Z = []
    chain = []
    remaining = N
    while remaining > 1:
        if not chain:
            chain.append(int(np.flatnonzero(active)[0]))
        x = chain[-1]
        row = np.where(active, D[x], np.inf)
        row[x] = np.inf
        m = row.min()
        # tie key (d, min rep, max rep): for fixed x this orders candidates by rep.
        y = int(idx[(row == m) & active & (idx != x)].min())
        if len(chain) >= 2 and chain[-2] == y:
            chain.pop()
            chain.pop()
            a, b = min(x, y), max(x, y)
            Z.append((a, b, np.float32(m), int(size[a] + size[b])))
            newrow = np.maximum(D[a], D[b])
            D[a, :] = newrow
            D[:, a] = newrow
            D[a, a] = np.inf
            active[b] = False
            D[b, :] = np.inf
            D[:, b] = np.inf
            size[a] += size[b]
            remaining -= 1
        else:
            chain.append(y)
    Z.sort(key=lambda z: (float(z[2]), z[0], z[1]))
    return Z


def linkage_intersection(ctxs, alpha: Fraction):
    """NEXT-3: "iteratively merge the closest pair,
    creating a virtual node whose context is the sorted intersection" read as
    SPEC:177 — the merged cluster is represented by the ascending sorted
    intersection of its two representatives, and cluster distance is Eq. 1
     between representatives (positions = index in the list:
    retrieval order for a leaf, ascending DocId for a virtual node).  Greedy
    with the X8 key (d, min rep, max rep); the survivor keeps the smaller rep.
    The linkage is not reducible (a later merge can be lower), so the merge
    list is in merge order, not sorted by height.  Brute force: every step
    recomputes every active pair — small N only."""
    rep_ctx = {i: list(c) for i, c in enumerate(ctxs)}
    size = {i: 1 for i in rep_ctx}
    Z = []
    while len(rep_ctx) > 1:
        keys = sorted(rep_ctx)
        best = None
        for x in range(len(keys)):
            for y in range(x + 1, len(keys)):
                a, b = keys[x], keys[y]
                k = (distance(rep_ctx[a], rep_ctx[b], alpha), a, b)
                if best is None or k < best:
                    best = k
        h, a, b = best
        rep_ctx[a] = sorted(set(rep_ctx[a]) & set(rep_ctx[b]))
        del rep_ctx[b]
        size[a] += size.pop(b)
        Z.append((a, b, np.float32(h), size[a]))
    return Z


def cluster_height(d: np.ndarray, A, B) -> np.float32:
    """Complete-linkage distance by its definition: max over member pairs."""
    return np.float32(max(d[a, b] for a in A for b in B))


# ------------------------------------------------------------------------ O6-O8
class Tree:
    """O6-O8 result: nodes with parent, children (ordered by rep), set, ordered
    context; leaf paths; offline orders; schedule."""

    def __init__(self):
        self.parent = []
        self.children = []
        self.docset = []
        self.rep = []
        self.leaf_of = []   # node -> leaf index or -1
        self.ordered = []   # node -> list
        self.leaf_node = []  # leaf index -> node
        self.path = []       # leaf index -> list of child indices


def build_tree(ctxs, Z) -> Tree:
    """O6: replay the merges; each merge makes a virtual
    node whose set is the intersection of its children's sets ("virtual node
    whose context is the sorted intersection"); an empty root sits on top
    ("root represents an empty context").  Virtual nodes whose set equals their
    parent's are collapsed (X11); children are ordered by rep (X12).  O7: ordered
    contexts top-down (X10, X13).  O8: leaf paths ("each leaf node
    records its search path from the root")."""
    N = len(ctxs)
    # raw binary tree
    r_children = [[] for _ in range(N)]
    r_set = [frozenset(c) for c in ctxs]
    r_rep = list(range(N))
    node_of = {i: i for i in range(N)}  # cluster rep -> current raw node
    for (a, b, _h, _sz) in Z:
        na, nb = node_of[a], node_of[b]
        v = len(r_set)
        r_children.append([na, nb])
        r_set.append(r_set[na] & r_set[nb])
        r_rep.append(min(r_rep[na], r_rep[nb]))
        node_of[min(a, b)] = v
        del node_of[max(a, b)]
    if len(node_of) != 1:
        raise OracleError("linkage does not join all contexts")
    top = next(iter(node_of.values()))

    t = Tree()
    t.leaf_node = [-1] * N
    t.path = [None] * N

    def new_node(parent, s, rep, leaf):
        k = len(t.parent)
        t.parent.append(parent)
        t.children.append([])
        t.docset.append(s)
        t.rep.append(rep)
        t.leaf_of.append(leaf)
        t.ordered.append(None)
        if leaf >= 0:
            t.leaf_node[leaf] = k
        return k

    root = new_node(-1, frozenset(), -1, -1)
    t.ordered[root] = []

    def expand(raw, parent_set):
        # collapse a virtual node whose set equals its parent's (X11), and
        # recursively its collapsed descendants; left-to-right preorder with an
        # explicit stack (caterpillar trees outgrow Python's recursion limit)
        out, todo = [], [raw]
        while todo:
            r = todo.pop()
            if r >= N and r_set[r] == parent_set:
                todo.extend(reversed(r_children[r]))
            else:
                out.append(r)
        return out

    stack = [(root, top)]
    pending = [(root, [top])]
    while pending:
        node, raws = pending.pop()
        kids = []
        for r in raws:
            kids.extend(expand(r, t.docset[node]))
        kids.sort(key=lambda r: r_rep[r])  # X12
        for r in kids:
            leaf = r if r < N else -1
            k = new_node(node, r_set[r], r_rep[r], leaf)
            t.children[node].append(k)
            par_ord = t.ordered[node]
            par_set = t.docset[node]
            if leaf >= 0:
                # leaf: parent's prefix ++ remaining docs in original order
                t.ordered[k] = par_ord + [x for x in ctxs[leaf] if x not in par_set]
            else:
                # virtual: parent's prefix ++ ascending new docs (X10)
                t.ordered[k] = par_ord + sorted(r_set[r] - par_set)
                pending.append((k, r_children[r]))
    del stack
    # paths
    for leaf in range(N):
        p = []
        k = t.leaf_node[leaf]
        while t.parent[k] != -1:
            par = t.parent[k]
            p.append(t.children[par].index(k))
            k = par
        t.path[leaf] = p[::-1]
    return t


def offline_order(ctxs, t: Tree):
    """O7: each indexed context becomes its leaf's ordered list
    (matched prefix, then the rest in original order); prefix_len = |ord(parent)|."""
    out = []
    plen = []
    for i in range(len(ctxs)):
        k = t.leaf_node[i]
        out.append(list(t.ordered[k]))
        plen.append(len(t.ordered[t.parent[k]]))
    return out, plen


def schedule(paths):
    """O8: group by the first element of the search
    path, groups in order of first appearance (X14); within a group sort by path
    length descending, ties by input index."""
    groups = {}
    order = []
    for i, p in enumerate(paths):
        key = ("empty", i) if len(p) == 0 else p[0]
        if key not in groups:
            groups[key] = []
            order.append(key)
        groups[key].append(i)
    out = []
    for key in order:
        out.extend(sorted(groups[key], key=lambda i: (-len(paths[i]), i)))
    return out


def traverse(t: Tree, path):
    """Context traversal: follow child indices from the root."""
    k = 0
    for step in path:
        k = t.children[k][step]
    return k


# --------------------------------------------------------------------------- O9
class Session:
    """O9: the session's seen set starts as the turn-0 context
    ("follows its stored search path to the first-turn context") and grows by
    each turn's novel docs ("appended to a copy of the first-turn context state")
    (X18)."""

    def __init__(self, turn0_docs):
        self.turn = 0
        self.seen = {}
        for x in turn0_docs:
            self.seen.setdefault(int(x), 0)

    def dedup_turn(self, docs):
        """Novel docs in retrieval order; refs (doc, first-seen turn) in retrieval
        order ("These are filtered out, leaving only the novel
        document")."""
        self.turn += 1
        docs = [int(x) for x in docs]
        if len(set(docs)) != len(docs):
            raise OracleError("duplicate DocId in retrieval")
        novel = [x for x in docs if x not in self.seen]
        refs = [(x, self.seen[x]) for x in docs if x in self.seen]
        for x in novel:
            self.seen[x] = self.turn
        return novel, refs


# ------------------------------------------------------------------------- all
def build_index(ids, lens=None, alpha=Fraction(1, 200)):
    """Whole path O1-O8 for small N (pure Python distances)."""
    ctxs = validate(ids, lens)
    S, Dm, d = pairwise(ctxs, alpha)
    nn_idx, nn_d = row_nn(d)
    Z = linkage_greedy(d) if len(ctxs) <= 96 else linkage_nn_chain(d)
    t = build_tree(ctxs, Z)
    ordered, plen = offline_order(ctxs, t)
    sched = schedule(t.path)
    return dict(S=S, D=Dm, d=d, nn_idx=nn_idx, nn_d=nn_d, Z=Z, tree=t, ordered=ordered,
                prefix_len=plen, schedule=sched)


# ------------------------------------------------------------------- NEXT-1
class OnlineIndex:
    """NEXT-1: context search, insert and ordering of new
    contexts against a built index (Section 4.2; PAPER:425-436,
    Section 5.1), sequential over a batch (SPEC order_batch).

    Search ("greedily descending from the root, selecting at each
    level the child with the minimum distance ... stops upon reaching a leaf or
    when all children are equidistant"), with reading X15: distances are the
    canonical fp32 Eq. 1 values against each child's ordered context; eligible
    children share at least one doc with the query, and a virtual child must be
    contained in the query (so every node on the path is a prefix of it,
    X20); key (d, is_leaf, child index); stop when no child is eligible or when
    two or more children are eligible and all share the same (d, is_leaf);
    otherwise descend into the minimum key (a sole eligible child is always
    descended).

    Insert ("matching an internal node appends the new context as a
    child, while matching a leaf creates a new internal node with their
    intersection"), reading X21: a leaf match L under parent P creates a virtual
    node V with set(L) ∩ set(Q) in L's place (children L, Q) when that
    intersection extends set(P); otherwise Q becomes a child of P.  V's ordered
    context is P's followed by the shared docs in L's existing order (L was
    already served in that order), and L's ordered context is re-derived under
    V (unchanged when Q contains L).  The new context's order is the matched
    node's ordered prefix followed by its remaining docs in retrieval order
    (PAPER:431)."""

    def __init__(self, ctxs, t: Tree, alpha: Fraction):
        self.alpha = alpha
        self.children = [list(c) for c in t.children]
        self.parent = list(t.parent)
        self.docset = [frozenset(s) for s in t.docset]
        self.ordered = [list(o) for o in t.ordered]
        self.leaf_of = list(t.leaf_of)
        self.docs = [list(c) for c in ctxs]
        self.leaf_node = list(t.leaf_node)

    def _is_leaf(self, k):
        return self.leaf_of[k] >= 0

    def _new_node(self, parent, docset, ordered, leaf):
        k = len(self.parent)
        self.parent.append(parent)
        self.children.append([])
        self.docset.append(frozenset(docset))
        self.ordered.append(list(ordered))
        self.leaf_of.append(leaf)
        return k

    def search(self, q):
        node, path = 0, []
        qs = set(q)
        while not self._is_leaf(node):
            cands = []
            for idx, c in enumerate(self.children[node]):
                s, _ = overlap(q, self.ordered[c])
                if s == 0:
                    continue
                if not self._is_leaf(c) and not self.docset[c] <= qs:
                    continue
                cands.append((distance(q, self.ordered[c], self.alpha), self._is_leaf(c), idx, c))
            if not cands:
                break
            if len(cands) >= 2 and all((x[0], x[1]) == (cands[0][0], cands[0][1]) for x in cands):
                break
            best = min(cands, key=lambda x: (x[0], x[1], x[2]))
            path.append(best[2])
            node = best[3]
        return node, path

    def order(self, q):
        """Search + insert one context; returns (ordered docs, prefix length, path)."""
        q = [int(x) for x in q]
        node, path = self.search(q)
        ctx = len(self.docs)
        self.docs.append(q)
        if not self._is_leaf(node):
            parent = node
        else:
            L = node
            P = self.parent[L]
            inter = set(self.docs[self.leaf_of[L]]) & set(q)
            if inter == set(self.docset[P]):
                parent = P
                path = path[:-1]
            else:
                # V keeps L's (already served) order for the shared docs
                base = len(self.ordered[P])
                V = self._new_node(P, inter, self.ordered[P] + [x for x in self.ordered[L][base:] if x in inter], -1)
                pos = self.children[P].index(L)
                self.children[P][pos] = V
                self.children[V] = [L]
                self.parent[L] = V
                self.ordered[L] = self.ordered[V] + [x for x in self.ordered[L][base:] if x not in inter]
                parent = V
        pset = self.docset[parent]
        ordq = self.ordered[parent] + [x for x in q if x not in pset]
        k = self._new_node(parent, set(q), ordq, ctx)
        self.children[parent].append(k)
        self.leaf_node.append(k)
        return ordq, len(self.ordered[parent]), self.path_of(ctx)

    def path_of(self, ctx):
        k = self.leaf_node[ctx]
        p = []
        while self.parent[k] != -1:
            par = self.parent[k]
            p.append(self.children[par].index(k))
            k = par
        return p[::-1]

    def order_batch(self, batch):
        """Sequential search + insert of a batch (earlier insertions are visible
        to later items, SPEC order_batch), then the Section 5.2 schedule of the
        batch's paths."""
        out = [self.order(q) for q in batch]
        paths = [self.path_of(len(self.docs) - len(batch) + i) for i in range(len(batch))]
        return [o for o, _, _ in out], [p for _, p, _ in out], paths, schedule(paths)


def traverse_online(idx: OnlineIndex, path):
    k = 0
    for step in path:
        k = idx.children[k][step]
    return k


# ------------------------------------------------------------------ NEXT-4
class PrefixCache:
    """NEXT-4: document-granularity prefix cache standing in
    for the inference engine (§2.1 "prefix cache that stores KV
    caches from prior prompts", "trie-based implementation organizes tokens
    hierarchically"; SPEC cache_sim).  A trie of DocId edges; a request's hit
    is its longest cached prefix ("only the longest common prefix
    ... can be reused"); the rest is inserted; least-recently-used leaves that
    are not on the request's path are evicted until the token budget holds
    (ties: older node first).  Tokens per doc default to 1."""

    def __init__(self, capacity, tokens=None):
        if capacity <= 0:
            raise OracleError("capacity must be positive")
        self.cap = capacity
        self.tok = tokens or {}
        self.children = [{}]     # node -> {doc: child}
        self.parent = [-1]
        self.doc = [None]
        self.stamp = [0]
        self.alive = [True]
        self.clock = 0
        self.resident = 0

    def _t(self, d):
        return self.tok.get(d, 1)

    def prefill(self, docs):
        """Returns (hit_tokens, miss_tokens, evicted_tokens)."""
        docs = [int(x) for x in docs]
        if len(set(docs)) != len(docs):
            raise OracleError("duplicate DocId in request")
        total = sum(self._t(d) for d in docs)
        if total > self.cap:
            raise OracleError("request exceeds capacity by %d" % (total - self.cap))
        self.clock += 1
        node, k = 0, 0
        path = [0]
        while k < len(docs) and docs[k] in self.children[node]:
            node = self.children[node][docs[k]]
            self.stamp[node] = self.clock
            path.append(node)
            k += 1
        hit = sum(self._t(d) for d in docs[:k])
        miss = total - hit
        need = self.resident + miss - self.cap
        evicted = 0
        onpath = set(path)
        while need > 0:
            leaves = [v for v in range(1, len(self.parent)) if self.alive[v] and not self.children[v]
                      and v not in onpath]
            v = min(leaves, key=lambda x: (self.stamp[x], x))
            self.alive[v] = False
            del self.children[self.parent[v]][self.doc[v]]
            t = self._t(self.doc[v])
            self.resident -= t
            evicted += t
            need -= t
        for d in docs[k:]:
            v = len(self.parent)
            self.children.append({})
            self.parent.append(node)
            self.doc.append(d)
            self.stamp.append(self.clock)
            self.alive.append(True)
            self.children[node][d] = v
            self.resident += self._t(d)
            node = v
        return hit, miss, evicted


def prefix_cache_list_model(capacity, requests, tokens=None):
    """Independent reference for PrefixCache (SPEC cache_sim "brute-force
    reference simulator with an explicit list-of-prefixes model"): the cache
    is the set of resident prefixes (tuples) with their last-use stamp;
    eviction removes the least recently used prefix that no other resident
    prefix extends and that the request does not contain.  O(N^2)."""
    tok = tokens or {}
    t = lambda d: tok.get(d, 1)
    res = {}  # prefix tuple -> (stamp, creation)
    clock, created, out = 0, 0, []
    for req in requests:
        req = tuple(int(x) for x in req)
        clock += 1
        k = 0
        while k < len(req) and req[:k + 1] in res:
            k += 1
        for j in range(1, k + 1):
            res[req[:j]] = (clock, res[req[:j]][1])
        hit = sum(t(d) for d in req[:k])
        miss = sum(t(d) for d in req[k:])
        resident = sum(t(p[-1]) for p in res)
        evicted = 0
        while resident + miss > capacity:
            cands = [p for p in res if not any(q[:len(p)] == p and len(q) > len(p) for q in res)
                     and not (len(p) <= len(req) and req[:len(p)] == p)]
            p = min(cands, key=lambda x: res[x])
            del res[p]
            resident -= t(p[-1])
            evicted += t(p[-1])
        for j in range(k + 1, len(req) + 1):
            created += 1
            res[req[:j]] = (clock, created)
        out.append((hit, miss, evicted))
    return out


class CacheIndex:
    """NEXT-4: index update under cache events (§4.1 "Index
    update": "maintains a min-heap tracking all active nodes by last access
    time", "removed from the least recently used nodes by decrementing their
    token counts"; SPEC apply_cache_event).  Per node seq_len and last access;
    Appended(path, n) adds n tokens and refreshes; Accessed(path) refreshes;
    Evicted(n) takes tokens from nodes with seq_len > 0 in ascending
    (last_access, creation order); a node reaching 0 with no children is
    detached from its parent, and parents left with no children and seq_len 0
    are deleted recursively (child indices of later siblings shift)."""

    def __init__(self, children):
        self.children = [list(c) for c in children]
        self.parent = [-1] * len(children)
        for p, cs in enumerate(children):
            for c in cs:
                self.parent[c] = p
        self.seq = [0] * len(children)
        self.last = [0] * len(children)
        self.gone = [False] * len(children)
        self.clock = 0

    def node_at(self, path):
        k = 0
        for i in path:
            if i < 0 or i >= len(self.children[k]):
                raise OracleError("invalid path")
            k = self.children[k][i]
        return k

    def appended(self, path, n):
        if n < 0:
            raise OracleError("negative token count")
        k = self.node_at(path)
        self.clock += 1
        self.seq[k] += n
        self.last[k] = self.clock

    def accessed(self, path):
        k = self.node_at(path)
        self.clock += 1
        self.last[k] = self.clock

    def evicted(self, n):
        if n < 0:
            raise OracleError("negative token count")
        taken = 0
        while n > 0:
            live = [k for k in range(len(self.seq)) if not self.gone[k] and self.seq[k] > 0]
            if not live:
                break
            k = min(live, key=lambda x: (self.last[x], x))
            d = min(n, self.seq[k])
            self.seq[k] -= d
            n -= d
            taken += d
            x = k
            while x > 0 and self.seq[x] == 0 and not self.children[x]:
                p = self.parent[x]
                self.children[p].remove(x)
                self.gone[x] = True
                x = p
        return taken
