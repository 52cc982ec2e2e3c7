// NEXT-4 (host): document-granularity prefix cache standing in for the
// inference engine, to measure the hit rates the ordering and schedule buy.
//
// PAPER:206-207 (Section 2.1): the engine's "prefix cache ... stores KV caches
// from prior prompts"; "trie-based implementation organizes tokens
// hierarchically"; PAPER:357 only the longest common prefix is reused.  A trie
// over DocId edges with per-node token counts: a request's hit is its longest
// cached prefix, the rest is inserted, and least-recently-used leaves (never
// the request's own path) are evicted until the token budget holds; ties go
// to the older node.  (SPEC cache_sim.)
#include <cstring>
#include <new>
#include <set>
#include <string>
#include <unordered_map>
#include <vector>

#include "internal.h"

struct rb_cache {
  int64_t cap = 0, resident = 0;
  uint64_t clock = 0;
  std::vector<int32_t> parent, nkids, tokens;
  std::vector<uint32_t> doc;
  std::vector<uint64_t> stamp;
  std::vector<uint8_t> alive;
  std::unordered_map<uint64_t, int32_t> child;  // (parent << 32 | doc) -> node
  std::set<std::pair<uint64_t, int32_t>> leaves; // (stamp, node) of childless nodes
};

namespace {

inline uint64_t ckey(int32_t p, uint32_t d) { return ((uint64_t)(uint32_t)p << 32) | d; }

rb_status prefill(rb_cache *c, const uint32_t *docs, int32_t n, const int32_t *tok, int32_t tok_const,
                  int64_t *hit, int64_t *miss, int64_t *evicted, std::string *msg) {
  int64_t total = 0;
  for (int32_t k = 0; k < n; ++k) {
    const int32_t t = tok ? tok[k] : tok_const;
    if (t <= 0) {
      *msg = "token counts must be positive";
      return RB_EINVAL;
    }
    total += t;
    for (int32_t q = 0; q < k; ++q)
      if (docs[q] == docs[k]) {
        *msg = "duplicate DocId in request";
        return RB_EDUPDOC;
      }
  }
  if (total > c->cap) {
    *msg = "request exceeds the cache capacity by " + std::to_string(total - c->cap) + " tokens";
    return RB_EINVAL;
  }
  const uint64_t now = ++c->clock;
  int32_t node = 0;
  int32_t k = 0;
  int64_t h = 0;
  for (; k < n; ++k) {  // longest cached prefix; refresh its nodes
    auto it = c->child.find(ckey(node, docs[k]));
    if (it == c->child.end()) break;
    node = it->second;
    if (c->nkids[node] == 0) c->leaves.erase({c->stamp[node], node});
    c->stamp[node] = now;
    if (c->nkids[node] == 0) c->leaves.insert({now, node});
    h += c->tokens[node];
  }
  const int64_t m = total - h;
  int64_t ev = 0;
  // evict LRU leaves: the request's path has stamp `now`, every other node an
  // older one, so the minimum is never on the path while the budget is short
  while (c->resident + m > c->cap) {
    const int32_t v = c->leaves.begin()->second;
    c->leaves.erase(c->leaves.begin());
    c->alive[v] = 0;
    c->child.erase(ckey(c->parent[v], c->doc[v]));
    c->resident -= c->tokens[v];
    ev += c->tokens[v];
    const int32_t p = c->parent[v];
    if (p != 0 && --c->nkids[p] == 0) c->leaves.insert({c->stamp[p], p});
    if (p == 0) --c->nkids[0];
  }
  for (; k < n; ++k) {  // insert the missing suffix
    const int32_t v = (int32_t)c->parent.size();
    if (node != 0 && c->nkids[node] == 0) c->leaves.erase({c->stamp[node], node});
    ++c->nkids[node];
    c->parent.push_back(node);
    c->nkids.push_back(0);
    const int32_t t = tok ? tok[k] : tok_const;
    c->tokens.push_back(t);
    c->doc.push_back(docs[k]);
    c->stamp.push_back(now);
    c->alive.push_back(1);
    c->child.emplace(ckey(node, docs[k]), v);
    c->resident += t;
    node = v;
  }
  if (node != 0 && c->nkids[node] == 0) c->leaves.insert({now, node});
  *hit = h;
  *miss = m;
  *evicted = ev;
  return RB_OK;
}

}  // namespace

extern "C" {

rb_status ragb_fail_msg(rb_status code, const char *msg);  // capi.cpp

rb_status rb_cache_create(int64_t capacity_tokens, rb_cache **out) {
  if (!out || capacity_tokens <= 0) return ragb_fail_msg(RB_EINVAL, "capacity must be positive");
  rb_cache *c = new (std::nothrow) rb_cache();
  if (!c) return ragb_fail_msg(RB_ENOMEM, "host allocation failed");
  c->cap = capacity_tokens;
  c->parent.push_back(-1);  // root: the empty prefix
  c->nkids.push_back(0);
  c->tokens.push_back(0);
  c->doc.push_back(0);
  c->stamp.push_back(0);
  c->alive.push_back(1);
  *out = c;
  return RB_OK;
}

rb_status rb_cache_prefill(rb_cache *c, const uint32_t *docs, int32_t n, const int32_t *doc_tokens,
                           int64_t *hit, int64_t *miss, int64_t *evicted) {
  if (!c || (n > 0 && !docs) || n < 0 || !hit || !miss || !evicted)
    return ragb_fail_msg(RB_EINVAL, "bad argument");
  std::string msg;
  const rb_status s = prefill(c, docs, n, doc_tokens, 1, hit, miss, evicted, &msg);
  return s == RB_OK ? s : ragb_fail_msg(s, msg.c_str());
}

rb_status rb_cache_prefill_batch(rb_cache *c, const uint32_t *ids, const uint8_t *lens, const int64_t *order,
                                 int64_t M, int32_t K, int32_t tokens_per_doc, int64_t *hit, int64_t *miss,
                                 int64_t *evicted) {
  if (!c || M < 0 || K < 1 || K > 255 || tokens_per_doc <= 0 || (M > 0 && (!ids || !hit || !miss || !evicted)))
    return ragb_fail_msg(RB_EINVAL, "bad argument");
  std::string msg;
  for (int64_t z = 0; z < M; ++z) {
    const int64_t i = order ? order[z] : z;
    if (i < 0 || i >= M) return ragb_fail_msg(RB_EINVAL, "order entry out of range");
    const int L = lens ? lens[i] : K;
    const rb_status s = prefill(c, ids + i * K, L, nullptr, tokens_per_doc, hit + i, miss + i, evicted + i, &msg);
    if (s != RB_OK) return ragb_fail_msg(s, ("request " + std::to_string(i) + ": " + msg).c_str());
  }
  return RB_OK;
}

rb_status rb_cache_resident(const rb_cache *c, int64_t *tokens) {
  if (!c || !tokens) return ragb_fail_msg(RB_EINVAL, "bad argument");
  *tokens = c->resident;
  return RB_OK;
}

void rb_cache_free(rb_cache *c) { delete c; }

}  // extern "C"
