// NEXT-1 (host): online context ordering against a built index — context
// search + insert + prefix-first ordering of new contexts, then the Section 5.2
// schedule of the batch.
//
// PAPER:371-384 (Section 4.2 "Context search"): "greedily descending from the
// root, selecting at each level the child with the minimum distance ... The
// search stops upon reaching a leaf or when all children are equidistant";
// "matching an internal node appends the new context as a child (O(1)), while
// matching a leaf creates a new internal node with their intersection".
// PAPER:425-436 (Section 5.1): new contexts "search the index" and concatenate
// the matched prefix with their remaining documents in original order.
// Readings: X15 (eligibility, tie and stop rule), X20 (a virtual
// child must be contained in the query), X21 (leaf match), canonical fp32 Eq. 1
// distances against each child's ordered context (X6).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstring>
#include <memory>
#include <set>
#include <string>
#include <unordered_map>
#include <vector>

#include "internal.h"

namespace ragb {

namespace {

// Canonical fp32 Eq. 1 (X6) from exact counts: one IEEE division of exact
// integers (both < 2^24), or a double division (den < 2^29: no double-rounding
// hazard).
float eq1_host(uint32_t s, uint32_t D, uint32_t m, uint32_t an, uint32_t ad) {
  if (s == 0) return 1.0f;
  const uint64_t num = (uint64_t)(m - s) * ad * s + (uint64_t)an * D * m;
  const uint64_t den = (uint64_t)ad * m * s;
  if (((num | den) >> 24) == 0) return (float)(uint32_t)num / (float)(uint32_t)den;
  return (float)((double)num / (double)den);
}

struct QueryView {
  std::vector<std::pair<uint32_t, int>> bydoc;  // (doc, position) sorted by doc
  int len = 0;
  int pos_of(uint32_t doc) const {
    auto it = std::lower_bound(bydoc.begin(), bydoc.end(), std::make_pair(doc, -1));
    return (it != bydoc.end() && it->first == doc) ? it->second : -1;
  }
};

}  // namespace

struct DynTree {
  std::vector<int32_t> parent;
  std::vector<std::vector<int32_t>> kids;
  std::vector<std::vector<uint32_t>> set;  // sorted
  std::vector<std::vector<uint32_t>> ord;  // ordered context
  std::vector<int64_t> leaf;               // node -> context id, -1 for root/virtual
  std::vector<int32_t> leaf_node;          // context -> node
  std::vector<int32_t> cidx;               // node -> index among its parent's children
  std::vector<std::vector<uint32_t>> docs; // context -> docs in retrieval order
  // per-node inverted index doc -> child positions (large fan-out nodes only)
  std::unordered_map<int32_t, std::unordered_map<uint32_t, std::vector<int32_t>>> inv;
  // NEXT-4 cache state: cached tokens and last access per node, LRU order of
  // the nodes holding tokens, nodes detached by evictions
  std::vector<int64_t> seq;
  std::vector<uint64_t> last;
  std::vector<uint8_t> gone;
  std::set<std::pair<uint64_t, int32_t>> lru;
  uint64_t clock = 0;
};

static DynTree *dyn_from_offline(const HostIndex &H) {
  auto *T = new DynTree();
  const int64_t V = H.V, N = H.N, K = H.K;
  const int64_t nodes = 1 + V + N;
  T->parent.resize(nodes);
  T->kids.resize(nodes);
  T->set.resize(nodes);
  T->ord.resize(nodes);
  T->leaf.assign(nodes, -1);
  T->leaf_node.resize(N);
  T->docs.resize(N);
  T->parent[0] = -1;
  for (int64_t k = 1; k <= V; ++k) T->parent[k] = H.vparent[k - 1];
  for (int64_t i = 0; i < N; ++i) {
    T->parent[V + 1 + i] = H.lparent[i];
    T->leaf[V + 1 + i] = i;
    T->leaf_node[i] = (int32_t)(V + 1 + i);
  }
  T->cidx.assign(nodes, 0);
  for (int64_t k = 0; k <= V; ++k) {
    T->kids[k].assign(H.kids.begin() + H.kids_off[k], H.kids.begin() + H.kids_off[k + 1]);
    for (size_t z = 0; z < T->kids[k].size(); ++z) T->cidx[T->kids[k][z]] = (int32_t)z;
  }
  for (int64_t k = 0; k <= V; ++k) {
    T->ord[k].assign(H.vpre.begin() + H.vpre_off[k], H.vpre.begin() + H.vpre_off[k + 1]);
    T->set[k] = T->ord[k];
    std::sort(T->set[k].begin(), T->set[k].end());
  }
  for (int64_t i = 0; i < N; ++i) {
    const int L = H.lens.empty() ? (int)K : H.lens[i];
    T->docs[i].assign(H.ids.begin() + i * K, H.ids.begin() + i * K + L);
    T->ord[V + 1 + i].assign(H.ordered.begin() + i * K, H.ordered.begin() + i * K + L);
    T->set[V + 1 + i] = T->docs[i];
    std::sort(T->set[V + 1 + i].begin(), T->set[V + 1 + i].end());
  }
  return T;
}

static int32_t dyn_new_node(DynTree &T, int32_t parent, std::vector<uint32_t> set,
                            std::vector<uint32_t> ord, int64_t leaf) {
  const int32_t k = (int32_t)T.parent.size();
  T.parent.push_back(parent);
  T.kids.emplace_back();
  T.set.push_back(std::move(set));
  T.ord.push_back(std::move(ord));
  T.leaf.push_back(leaf);
  T.cidx.push_back(0);
  if (!T.seq.empty()) {
    T.seq.push_back(0);
    T.last.push_back(0);
    T.gone.push_back(0);
  }
  return k;
}

static void inv_add(DynTree &T, int32_t node, int32_t pos) {
  auto it = T.inv.find(node);
  if (it == T.inv.end()) return;
  for (uint32_t d : T.ord[T.kids[node][pos]]) it->second[d].push_back(pos);
}

// children of `node` sharing at least one doc with the query (superset)
static void candidates(DynTree &T, int32_t node, const std::vector<uint32_t> &q,
                       std::vector<int32_t> *out) {
  out->clear();
  const auto &ks = T.kids[node];
  if (ks.size() < 64) {
    for (size_t i = 0; i < ks.size(); ++i) out->push_back((int32_t)i);
    return;
  }
  auto it = T.inv.find(node);
  if (it == T.inv.end()) {
    auto &m = T.inv[node];
    for (size_t i = 0; i < ks.size(); ++i)
      for (uint32_t d : T.ord[ks[i]]) m[d].push_back((int32_t)i);
    it = T.inv.find(node);
  }
  for (uint32_t d : q) {
    auto f = it->second.find(d);
    if (f != it->second.end()) out->insert(out->end(), f->second.begin(), f->second.end());
  }
  std::sort(out->begin(), out->end());
  out->erase(std::unique(out->begin(), out->end()), out->end());
}

// Distances of one query against the root's children from the device
// (online_dev.cu), for a sub-batch of queries and the root as it was when the
// sub-batch started; children changed since (replaced by an X21 node, or
// appended) are scored on the host.
struct RootScores {
  int F = 0, cap = 0;
  // children replaced or appended since the snapshot, by doc (host-scored
  // candidates: only those sharing a doc with the query can be eligible)
  std::unordered_map<uint32_t, std::vector<int32_t>> dinv;
  std::vector<int> cnt;          // [queries] eligible children (> cap: overflow, host scores that query)
  std::vector<uint2> ent;        // [queries][cap] (child index, d bits)
  std::vector<uint8_t> dirty;    // [F] child replaced since the snapshot
  std::vector<int32_t> dirty_idx;
};

// X15 search; returns the matched node and the descent path.  rs / qi: the
// device's root distances of this query (nullptr: host only).
static int32_t dyn_search(DynTree &T, const std::vector<uint32_t> &q, const QueryView &qv,
                          uint32_t an, uint32_t ad, std::vector<int32_t> *path, const RootScores *rs = nullptr,
                          int qi = 0) {
  int32_t node = 0;
  path->clear();
  std::vector<int32_t> cand;
  struct C {
    float d;
    int leaf;
    int32_t idx;
  };
  std::vector<C> el;
  auto score = [&](int32_t idx) {  // child idx of node: eligible -> el
    const int32_t c = T.kids[node][idx];
    const auto &oc = T.ord[c];
    uint32_t s = 0, D = 0;
    for (size_t p = 0; p < oc.size(); ++p) {
      const int pq = qv.pos_of(oc[p]);
      if (pq >= 0) {
        ++s;
        D += (uint32_t)(pq > (int)p ? pq - (int)p : (int)p - pq);
      }
    }
    if (s == 0) return;
    const bool isleaf = T.leaf[c] >= 0;
    if (!isleaf && s != oc.size()) return;  // X20: virtual child contained in the query
    const uint32_t m = (uint32_t)std::max<size_t>(oc.size(), (size_t)qv.len);
    el.push_back({eq1_host(s, D, m, an, ad), isleaf ? 1 : 0, idx});
  };
  while (T.leaf[node] < 0) {
    el.clear();
    if (node == 0 && rs && rs->cnt[qi] <= rs->cap) {
      const uint2 *e = rs->ent.data() + (size_t)qi * rs->cap;
      for (int z = 0; z < rs->cnt[qi]; ++z) {
        const int32_t idx = (int32_t)e[z].x;
        if (rs->dirty[idx]) continue;
        float d;
        std::memcpy(&d, &e[z].y, 4);
        el.push_back({d, T.leaf[T.kids[0][idx]] >= 0 ? 1 : 0, idx});
      }
      cand.clear();
      for (uint32_t d : q) {
        auto f = rs->dinv.find(d);
        if (f != rs->dinv.end()) cand.insert(cand.end(), f->second.begin(), f->second.end());
      }
      std::sort(cand.begin(), cand.end());
      cand.erase(std::unique(cand.begin(), cand.end()), cand.end());
      for (int32_t idx : cand) score(idx);
    } else {
      candidates(T, node, q, &cand);
      for (int32_t idx : cand) score(idx);
    }
    if (el.empty()) break;
    bool all_same = el.size() >= 2;
    for (size_t i = 1; i < el.size() && all_same; ++i)
      all_same = el[i].d == el[0].d && el[i].leaf == el[0].leaf;
    if (all_same) break;
    const C *best = &el[0];
    for (const C &e : el)
      if (e.d < best->d || (e.d == best->d && (e.leaf < best->leaf ||
                                               (e.leaf == best->leaf && e.idx < best->idx))))
        best = &e;
    path->push_back(best->idx);
    node = T.kids[node][best->idx];
  }
  return node;
}

static void dyn_path(const DynTree &T, int32_t node, std::vector<int32_t> *p) {
  p->clear();
  while (T.parent[node] >= 0) {
    p->push_back(T.cidx[node]);
    node = T.parent[node];
  }
  std::reverse(p->begin(), p->end());
}

rb_status online_order(HostIndex &H, const uint32_t *ids, const uint8_t *lens, int64_t M, int32_t K,
                       uint32_t an, uint32_t ad, uint32_t *out_ids, uint8_t *out_prefix_len,
                       int64_t *out_schedule, std::string *msg) {
  if (!H.dyn) H.dyn = std::shared_ptr<DynTree>(dyn_from_offline(H));
  DynTree &T = *H.dyn;
  std::vector<std::vector<int32_t>> paths(M);
  std::vector<int32_t> path;
  // device scores of the root's children (mode: 0 host, 1 device, -1 auto =
  // device for batches of >= 64 queries against a root of >= 256 children)
  const int mode = H.online_device;
  RootScores rs;
  int64_t sb_end = 0;  // end of the current device sub-batch
  constexpr int64_t kSub = 2048;
  for (int64_t i = 0; i < M; ++i) {
    if (i == sb_end) {
      sb_end = std::min<int64_t>(M, i + kSub);
      const size_t F = T.kids[0].size();
      int ndev = 0;
      const bool dev = mode == 1 || (mode < 0 && M >= 64 && F >= 256 && cudaGetDeviceCount(&ndev) == cudaSuccess &&
                                     ndev > 0);
      rs.F = 0;
      rs.cnt.clear();
      if (dev) {
        std::vector<int32_t> coff(F + 1, 0);
        std::vector<uint32_t> cdocs;
        std::vector<uint8_t> cleaf(F);
        for (size_t c = 0; c < F; ++c) {
          const int32_t k = T.kids[0][c];
          cdocs.insert(cdocs.end(), T.ord[k].begin(), T.ord[k].end());
          coff[c + 1] = (int32_t)cdocs.size();
          cleaf[c] = T.leaf[k] >= 0 ? 1 : 0;
        }
        rs.F = (int)F;
        rs.cap = (int)std::min<size_t>(F, 1024);
        rs.dirty.assign(F, 0);
        rs.dirty_idx.clear();
        rs.dinv.clear();
        const cudaError_t ce = online_root_scores(&H.odev, ids + i * K, lens ? lens + i : nullptr,
                                                  (int)(sb_end - i), K, coff, cdocs, cleaf, an, ad,
                                                  std::max(rs.cap, 1), &rs.cnt, &rs.ent);
        if (ce != cudaSuccess) {
          *msg = std::string("online root scores: ") + cudaGetErrorString(ce);
          return RB_ECUDA;
        }
        H.online_stats[0] += sb_end - i;
        if (H.trace) {
          int64_t tot = 0, mx = 0, over = 0;
          for (int c : rs.cnt) {
            tot += c;
            mx = std::max<int64_t>(mx, c);
            over += c > rs.cap ? 1 : 0;
          }
          std::fprintf(stderr, "[ragb online] sub-batch %lld queries, root fan-out %zu, eligible mean %.1f max %lld, over cap %lld\n",
                       (long long)(sb_end - i), F, (double)tot / std::max<size_t>(rs.cnt.size(), 1), (long long)mx,
                       (long long)over);
        }
      }
    }
    const int L = lens ? lens[i] : K;
    if (L < 1 || L > K) {
      *msg = "context length not in [1, K]";
      return RB_EINVAL;
    }
    std::vector<uint32_t> q(ids + i * K, ids + i * K + L);
    QueryView qv;
    qv.len = L;
    for (int k = 0; k < L; ++k) qv.bydoc.emplace_back(q[k], k);
    std::sort(qv.bydoc.begin(), qv.bydoc.end());
    for (int k = 1; k < L; ++k)
      if (qv.bydoc[k].first == qv.bydoc[k - 1].first) {
        *msg = "duplicate DocId within a context";
        return RB_EDUPDOC;
      }
    for (uint32_t x : q)
      if (x == kReservedDoc) {
        *msg = "reserved DocId 0xFFFFFFFF";
        return RB_EINVAL;
      }
    const bool have_rs = !rs.cnt.empty();
    int32_t node = dyn_search(T, q, qv, an, ad, &path, have_rs ? &rs : nullptr,
                              have_rs ? (int)(i - (sb_end - (int64_t)rs.cnt.size())) : 0);
    int32_t parent = node;
    if (T.leaf[node] >= 0) {  // leaf match (X21)
      const int32_t Lnode = node, P = T.parent[node];
      std::vector<uint32_t> inter;
      const auto &ls = T.set[Lnode];
      for (uint32_t x : ls)
        if (qv.pos_of(x) >= 0) inter.push_back(x);
      if (inter == T.set[P]) {
        parent = P;
      } else {
        const size_t base = T.ord[P].size();
        std::vector<uint32_t> vord(T.ord[P]);
        std::vector<uint32_t> ltail;
        for (size_t z = base; z < T.ord[Lnode].size(); ++z) {
          const uint32_t x = T.ord[Lnode][z];
          if (std::binary_search(inter.begin(), inter.end(), x))
            vord.push_back(x);
          else
            ltail.push_back(x);
        }
        const int32_t V = dyn_new_node(T, P, inter, vord, -1);
        auto &pk = T.kids[P];
        const int32_t pos = T.cidx[Lnode];
        if (P == 0 && !rs.cnt.empty()) {  // the device score of pos is stale: the host scores V there
          if (pos < rs.F && !rs.dirty[pos]) {
            rs.dirty[pos] = 1;
            rs.dirty_idx.push_back(pos);
          }
          for (uint32_t d : vord) rs.dinv[d].push_back(pos);
        }
        pk[pos] = V;
        T.cidx[V] = pos;
        T.kids[V].push_back(Lnode);
        T.parent[Lnode] = V;
        T.cidx[Lnode] = 0;
        std::vector<uint32_t> lord(T.ord[V]);
        lord.insert(lord.end(), ltail.begin(), ltail.end());
        T.ord[Lnode].swap(lord);
        auto it = T.inv.find(P);
        if (it != T.inv.end())
          for (uint32_t d : T.ord[V]) it->second[d].push_back(pos);
        parent = V;
      }
    }
    // the new leaf: matched prefix ++ remaining docs in retrieval order
    std::vector<uint32_t> ordq(T.ord[parent]);
    const auto &pset = T.set[parent];
    for (uint32_t x : q)
      if (!std::binary_search(pset.begin(), pset.end(), x)) ordq.push_back(x);
    std::vector<uint32_t> qset(q);
    std::sort(qset.begin(), qset.end());
    const int64_t ctx = (int64_t)T.docs.size();
    T.docs.push_back(q);
    const int32_t k = dyn_new_node(T, parent, std::move(qset), ordq, ctx);
    T.kids[parent].push_back(k);
    T.cidx[k] = (int32_t)T.kids[parent].size() - 1;
    inv_add(T, parent, T.cidx[k]);
    if (parent == 0 && !rs.cnt.empty())  // appended at the root after the snapshot: host-scored
      for (uint32_t d : ordq) rs.dinv[d].push_back(T.cidx[k]);
    T.leaf_node.push_back(k);
    if (out_ids) {
      std::memcpy(out_ids + i * K, ordq.data(), 4 * ordq.size());
      for (int z = L; z < K; ++z) out_ids[i * K + z] = ids[i * K + z];
    }
    if (out_prefix_len) out_prefix_len[i] = (uint8_t)T.ord[parent].size();
  }
  for (int64_t i = 0; i < M; ++i) dyn_path(T, T.leaf_node[T.docs.size() - M + i], &paths[i]);
  if (out_schedule) {  // Section 5.2 over the batch (X14)
    std::unordered_map<int32_t, int64_t> grank;
    std::vector<std::pair<std::pair<int64_t, int64_t>, int64_t>> key(M);
    for (int64_t i = 0; i < M; ++i) {
      const int32_t g = paths[i].empty() ? -1 - (int32_t)i : paths[i][0];
      auto it = grank.find(g);
      const int64_t r = it == grank.end() ? (grank[g] = (int64_t)grank.size()) : it->second;
      key[i] = {{r, -(int64_t)paths[i].size()}, i};
    }
    std::sort(key.begin(), key.end());
    for (int64_t i = 0; i < M; ++i) out_schedule[i] = key[i].second;
  }
  return RB_OK;
}

// exports when the tree was updated online
int64_t dyn_contexts(const HostIndex &H) { return (int64_t)H.dyn->leaf_node.size(); }
int64_t dyn_nodes(const HostIndex &H) { return (int64_t)H.dyn->parent.size(); }

void dyn_export(const HostIndex &H, int32_t *parent, int32_t *leaf, int32_t *rep, int64_t *prefix_off,
                uint32_t *prefix_ids, int64_t *path_off, int32_t *path, int64_t *prefix_total,
                int64_t *path_total) {
  const DynTree &T = *H.dyn;
  const int64_t n = (int64_t)T.parent.size();
  std::vector<int32_t> minleaf;
  if (rep) {  // smallest context index below each node
    minleaf.assign(n, 0x7fffffff);
    for (int64_t k = n - 1; k >= 0; --k) {
      if (T.leaf[k] >= 0) minleaf[k] = (int32_t)T.leaf[k];
    }
    // propagate bottom-up (children may have larger ids than parents after
    // online inserts, so iterate to a fixed point over parent links)
    for (int64_t k = 0; k < n; ++k) {
      int64_t x = k;
      const int32_t v = minleaf[k];
      if (T.leaf[k] < 0) continue;
      while (T.parent[x] >= 0) {
        x = T.parent[x];
        if (minleaf[x] <= v) break;
        minleaf[x] = v;
      }
    }
  }
  int64_t o = 0;
  for (int64_t k = 0; k < n; ++k) {
    if (parent) parent[k] = T.parent[k];
    if (leaf) leaf[k] = (int32_t)T.leaf[k];
    if (rep) rep[k] = k == 0 ? -1 : minleaf[k];
    if (prefix_off) prefix_off[k] = o;
    if (prefix_ids) std::memcpy(prefix_ids + o, T.ord[k].data(), 4 * T.ord[k].size());
    o += (int64_t)T.ord[k].size();
  }
  if (prefix_off) prefix_off[n] = o;
  if (prefix_total) *prefix_total = o;
  std::vector<int32_t> p;
  int64_t q = 0;
  const int64_t nc = (int64_t)T.leaf_node.size();
  for (int64_t i = 0; i < nc; ++i) {
    dyn_path(T, T.leaf_node[i], &p);
    if (path_off) path_off[i] = q;
    if (path) std::memcpy(path + q, p.data(), 4 * p.size());
    q += (int64_t)p.size();
  }
  if (path_off) path_off[nc] = q;
  if (path_total) *path_total = q;
}

const std::vector<uint32_t> &dyn_ordered(const HostIndex &H, int64_t ctx) {
  return H.dyn->ord[H.dyn->leaf_node[ctx]];
}

// offline-mode ordering of every indexed context after online updates
void dyn_order_all(const HostIndex &H, uint32_t *out_ids, uint8_t *out_prefix_len,
                   int64_t *out_schedule) {
  const DynTree &T = *H.dyn;
  const int64_t n = (int64_t)T.leaf_node.size(), K = H.K;
  std::vector<std::vector<int32_t>> paths(n);
  for (int64_t i = 0; i < n; ++i) {
    const int32_t node = T.leaf_node[i];
    if (out_ids) {
      std::memcpy(out_ids + i * K, T.ord[node].data(), 4 * T.ord[node].size());
      for (size_t z = T.docs[i].size(); z < (size_t)K; ++z)
        out_ids[i * K + z] = i < H.N ? H.ids[i * K + z] : 0u;
    }
    if (out_prefix_len) out_prefix_len[i] = (uint8_t)T.ord[T.parent[node]].size();
    dyn_path(T, node, &paths[i]);
  }
  if (out_schedule) {
    std::unordered_map<int32_t, int64_t> grank;
    std::vector<std::pair<std::pair<int64_t, int64_t>, int64_t>> key(n);
    for (int64_t i = 0; i < n; ++i) {
      const int32_t g = paths[i].empty() ? -1 - (int32_t)i : paths[i][0];  // evicted: own group
      auto it = grank.find(g);
      const int64_t r = it == grank.end() ? (grank[g] = (int64_t)grank.size()) : it->second;
      key[i] = {{r, -(int64_t)paths[i].size()}, i};
    }
    std::sort(key.begin(), key.end());
    for (int64_t i = 0; i < n; ++i) out_schedule[i] = key[i].second;
  }
}

// NEXT-4: index update under cache events (Section 4.1 "Index
// update": "maintains a min-heap tracking all active nodes by last access
// time" and evicted tokens are "removed from the least recently used nodes by
// decrementing their token counts"; SPEC apply_cache_event).  kind 0
// Appended(path, n): n tokens cached at the node, access refreshed; kind 1
// Accessed(path): access refreshed; kind 2 Evicted(n): tokens taken from the
// nodes holding tokens in ascending (last access, node id); a node left with
// no tokens and no children is detached from its parent (later siblings'
// child indices shift), and so are its ancestors left empty.
rb_status dyn_cache_event(HostIndex &H, int kind, const int32_t *path, int32_t path_len, int64_t n,
                          int64_t *taken, std::string *msg) {
  if (!H.dyn) H.dyn = std::shared_ptr<DynTree>(dyn_from_offline(H));
  DynTree &T = *H.dyn;
  if (T.seq.size() != T.parent.size()) {
    T.seq.resize(T.parent.size(), 0);
    T.last.resize(T.parent.size(), 0);
    T.gone.resize(T.parent.size(), 0);
  }
  if (n < 0) {
    *msg = "negative token count";
    return RB_EINVAL;
  }
  if (taken) *taken = 0;
  if (kind == 0 || kind == 1) {
    int32_t node = 0;
    for (int32_t i = 0; i < path_len; ++i) {
      if (!path || path[i] < 0 || path[i] >= (int32_t)T.kids[node].size()) {
        *msg = "invalid path";
        return RB_EPATH;
      }
      node = T.kids[node][path[i]];
    }
    if (T.seq[node] > 0) T.lru.erase({T.last[node], node});
    if (kind == 0) T.seq[node] += n;
    T.last[node] = ++T.clock;
    if (T.seq[node] > 0) T.lru.insert({T.last[node], node});
    return RB_OK;
  }
  if (kind != 2) {
    *msg = "unknown cache event";
    return RB_EINVAL;
  }
  int64_t got = 0;
  while (n > 0 && !T.lru.empty()) {
    const int32_t k = T.lru.begin()->second;
    const int64_t d = std::min<int64_t>(n, T.seq[k]);
    T.seq[k] -= d;
    n -= d;
    got += d;
    if (T.seq[k] > 0) continue;
    T.lru.erase(T.lru.begin());
    for (int32_t x = k; x > 0 && T.seq[x] == 0 && T.kids[x].empty();) {
      const int32_t p = T.parent[x];
      auto &pk = T.kids[p];
      const int32_t pos = T.cidx[x];
      pk.erase(pk.begin() + pos);
      for (size_t z = (size_t)pos; z < pk.size(); ++z) T.cidx[pk[z]] = (int32_t)z;
      T.inv.erase(p);  // child positions changed: rebuilt on demand
      T.gone[x] = 1;
      T.parent[x] = -1;
      x = p;
    }
  }
  if (taken) *taken = got;
  return RB_OK;
}

void dyn_cache_state(const HostIndex &H, int64_t *seq_len, int64_t *last_access) {
  const DynTree &T = *H.dyn;
  for (size_t k = 0; k < T.parent.size(); ++k) {
    const bool has = k < T.seq.size();
    if (seq_len) seq_len[k] = has ? (T.gone[k] ? -1 : T.seq[k]) : 0;
    if (last_access) last_access[k] = has ? (int64_t)T.last[k] : 0;
  }
}

}  // namespace ragb
