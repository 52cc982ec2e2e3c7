// a6-a7 (host): index tree, prefix-first ordering and schedule from the merge
// order produced on the device.
//
// PAPER:328 (Section 4.1): "The index is organized as a tree whose root
// represents an empty context"; "creating a virtual node whose
// context is the sorted intersection ... each leaf node records its search
// path from the root"; PAPER:430-431 (Section 5.1): "Each context then
// concatenates its matched prefix with remaining documents in their original
// order"; PAPER:451-452 (Section 5.2): "groups contexts by the first element of
// their search path ... sorts contexts within each group by path length in
// descending order".  Readings X9-X14: greedy key order, top-down
// ordered prefixes, collapse of virtual nodes equal to their parent, children
// by rep, schedule groups by first appearance with index ties.
#include <algorithm>
#include <cstring>
#include <numeric>
#include <string>
#include <vector>

#include "internal.h"

namespace ragb {

namespace {

struct Pool {  // flat storage of sorted doc sets
  std::vector<uint32_t> ids;
  std::vector<int64_t> off;
  std::vector<int32_t> len;
  const uint32_t *ptr(int64_t i) const { return ids.data() + off[i]; }
};

bool equal_sets(const Pool &P, int64_t x, int64_t y) {
  if (P.len[x] != P.len[y]) return false;
  return std::memcmp(P.ptr(x), P.ptr(y), sizeof(uint32_t) * (size_t)P.len[x]) == 0;
}

}  // namespace

rb_status host_build(HostIndex &H, std::string *msg) {
  const int64_t N = H.N;
  const int32_t K = H.K;
  // ---- merge order: ascending (h, a, b) (X9) ------------------------------
  const int64_t nz = (int64_t)H.za.size();
  if (nz != N - 1) {
    *msg = "merge list must have N-1 rows";
    return RB_EINVAL;
  }
  {
    std::vector<int64_t> perm(nz);
    std::iota(perm.begin(), perm.end(), 0);
    std::sort(perm.begin(), perm.end(), [&](int64_t x, int64_t y) {
      if (H.zh[x] != H.zh[y]) return H.zh[x] < H.zh[y];
      if (H.za[x] != H.za[y]) return H.za[x] < H.za[y];
      return H.zb[x] < H.zb[y];
    });
    std::vector<int32_t> a(nz), b(nz), s(nz);
    std::vector<float> h(nz);
    for (int64_t t = 0; t < nz; ++t) {
      a[t] = H.za[perm[t]];
      b[t] = H.zb[perm[t]];
      s[t] = H.zs[perm[t]];
      h[t] = H.zh[perm[t]];
    }
    H.za.swap(a);
    H.zb.swap(b);
    H.zs.swap(s);
    H.zh.swap(h);
  }

  // ---- raw binary tree with intersection sets -----------------------------
  const int64_t nraw = 2 * N - 1;
  Pool P;
  P.off.resize(nraw);
  P.len.resize(nraw);
  P.ids.reserve((size_t)N * K * 2);
  for (int64_t i = 0; i < N; ++i) {
    const int L = H.lens.empty() ? K : H.lens[i];
    P.off[i] = (int64_t)P.ids.size();
    P.len[i] = L;
    P.ids.insert(P.ids.end(), H.ids.begin() + i * K, H.ids.begin() + i * K + L);
    std::sort(P.ids.begin() + P.off[i], P.ids.end());
  }
  std::vector<int32_t> rchild(2 * std::max<int64_t>(nz, 0));
  std::vector<int32_t> rrep(nraw);
  std::vector<int64_t> cur(N);
  std::vector<int32_t> csize(N, 1);
  for (int64_t i = 0; i < N; ++i) {
    rrep[i] = (int32_t)i;
    cur[i] = i;
  }
  for (int64_t t = 0; t < nz; ++t) {
    const int32_t a = H.za[t], b = H.zb[t];
    if (a < 0 || b >= N || a >= b || cur[a] < 0 || cur[b] < 0 || csize[a] + csize[b] != H.zs[t]) {
      *msg = "inconsistent merge at row " + std::to_string(t);
      return RB_EINVAL;
    }
    const int64_t A = cur[a], B = cur[b], v = N + t;
    rchild[2 * t] = (int32_t)A;
    rchild[2 * t + 1] = (int32_t)B;
    rrep[v] = a;
    const uint32_t *pa = P.ptr(A), *pb = P.ptr(B);
    const int la = P.len[A], lb = P.len[B];
    P.off[v] = (int64_t)P.ids.size();
    int ia = 0, ib = 0, n = 0;
    while (ia < la && ib < lb) {  // sorted intersection
      if (pa[ia] < pb[ib]) {
        ++ia;
      } else if (pb[ib] < pa[ia]) {
        ++ib;
      } else {
        P.ids.push_back(pa[ia]);
        pa = P.ptr(A);  // push_back may reallocate
        pb = P.ptr(B);
        ++ia;
        ++ib;
        ++n;
      }
    }
    P.len[v] = n;
    cur[a] = v;
    cur[b] = -1;
    csize[a] += csize[b];
  }
  const int64_t top = (N == 1) ? 0 : N + nz - 1;
  if (cur[0] != top) {
    *msg = "merges do not join all contexts";
    return RB_EINVAL;
  }

  // ---- collapse + ordered prefixes + paths, breadth first ------------------
  H.parent.assign(1, -1);
  H.leaf.assign(1, -1);
  H.rep.assign(1, -1);
  std::vector<int64_t> setref(1, -1);  // raw node whose set is the node's set (-1: empty)
  std::vector<int64_t> node_raw(1, -1);
  H.prefix_off.assign(2, 0);  // [off[c], off[c+1]) = node c's ordered context
  H.prefix_ids.clear();
  H.prefix_ids.reserve((size_t)N * K * 2);
  std::vector<int64_t> npath_off(2, 0);  // root: empty path
  std::vector<int32_t> npath;
  H.leaf_node.assign(N, -1);
  std::vector<int64_t> kids, stack;
  std::vector<uint32_t> tmp;
  int64_t n_virtual = 0;

  for (int64_t q = 0; q < (int64_t)H.parent.size(); ++q) {
    // children raw nodes of q, expanded through collapsed virtual nodes
    kids.clear();
    stack.clear();
    if (q == 0) {
      stack.push_back(top);
    } else if (node_raw[q] >= N) {
      const int64_t t = node_raw[q] - N;
      stack.push_back(rchild[2 * t + 1]);
      stack.push_back(rchild[2 * t]);
    } else {
      continue;  // leaf
    }
    const int64_t pset = setref[q];
    while (!stack.empty()) {
      const int64_t r = stack.back();
      stack.pop_back();
      const bool same = r >= N && (pset < 0 ? P.len[r] == 0 : equal_sets(P, r, pset));
      if (same) {  // collapse (X11)
        const int64_t t = r - N;
        stack.push_back(rchild[2 * t + 1]);
        stack.push_back(rchild[2 * t]);
      } else {
        kids.push_back(r);
      }
    }
    std::sort(kids.begin(), kids.end(), [&](int64_t x, int64_t y) { return rrep[x] < rrep[y]; });
    // parent's ordered context and set
    const int64_t poff = H.prefix_off[q], plen = H.prefix_off[q + 1] - H.prefix_off[q];
    const uint32_t *pset_ids = pset < 0 ? nullptr : P.ptr(pset);
    const int pset_len = pset < 0 ? 0 : P.len[pset];
    for (size_t ci = 0; ci < kids.size(); ++ci) {
      const int64_t r = kids[ci];
      const int64_t c = (int64_t)H.parent.size();
      H.parent.push_back((int32_t)q);
      H.leaf.push_back(r < N ? (int32_t)r : -1);
      H.rep.push_back(rrep[r]);
      setref.push_back(r);
      node_raw.push_back(r);
      // path = parent's path + child index
      const int64_t pp0 = npath_off[q], pp1 = npath_off[q + 1];
      for (int64_t z = pp0; z < pp1; ++z) npath.push_back(npath[z]);
      npath.push_back((int32_t)ci);
      npath_off.push_back((int64_t)npath.size());
      // ordered context
      tmp.assign(H.prefix_ids.begin() + poff, H.prefix_ids.begin() + poff + plen);
      if (r < N) {  // leaf: prefix ++ remaining docs in original order
        const int L = H.lens.empty() ? K : H.lens[r];
        const uint32_t *row = H.ids.data() + r * K;
        for (int k = 0; k < L; ++k)
          if (!std::binary_search(pset_ids, pset_ids + pset_len, row[k])) tmp.push_back(row[k]);
        H.leaf_node[r] = c;
      } else {  // virtual: prefix ++ ascending new docs (X10)
        ++n_virtual;
        const uint32_t *s = P.ptr(r);
        for (int k = 0; k < P.len[r]; ++k)
          if (!std::binary_search(pset_ids, pset_ids + pset_len, s[k])) tmp.push_back(s[k]);
      }
      H.prefix_ids.insert(H.prefix_ids.end(), tmp.begin(), tmp.end());
      H.prefix_off.push_back((int64_t)H.prefix_ids.size());
    }
  }
  // leaf paths in context order
  H.path_off.assign(N + 1, 0);
  H.path.clear();
  int64_t max_depth = 0;
  for (int64_t i = 0; i < N; ++i) {
    const int64_t c = H.leaf_node[i];
    const int64_t p0 = npath_off[c], p1 = npath_off[c + 1];
    H.path.insert(H.path.end(), npath.begin() + p0, npath.begin() + p1);
    H.path_off[i + 1] = (int64_t)H.path.size();
    max_depth = std::max(max_depth, p1 - p0);
  }
  H.stats.n_virtual = n_virtual;
  H.stats.max_depth = max_depth;

  // ---- offline order (a7) -------------------------------------------------
  H.ordered.assign(H.ids.begin(), H.ids.end());
  H.prefix_len.assign(N, 0);
  for (int64_t i = 0; i < N; ++i) {
    const int64_t c = H.leaf_node[i];
    const int64_t o0 = H.prefix_off[c], o1 = H.prefix_off[c + 1];
    std::copy(H.prefix_ids.begin() + o0, H.prefix_ids.begin() + o1, H.ordered.begin() + i * K);
    const int64_t p = H.parent[c];
    H.prefix_len[i] = (uint8_t)(H.prefix_off[p + 1] - H.prefix_off[p]);
  }
  // ---- schedule: group by path[0], first appearance; length desc; index ---
  {
    std::vector<int64_t> gorder(N, -1);  // root-child index -> group rank
    std::vector<int64_t> grank(N);
    int64_t ng = 0;
    for (int64_t i = 0; i < N; ++i) {
      const int32_t g = H.path[H.path_off[i]];
      if (gorder[g] < 0) gorder[g] = ng++;
      grank[i] = gorder[g];
    }
    H.schedule.resize(N);
    std::iota(H.schedule.begin(), H.schedule.end(), 0);
    std::sort(H.schedule.begin(), H.schedule.end(), [&](int64_t x, int64_t y) {
      if (grank[x] != grank[y]) return grank[x] < grank[y];
      const int64_t lx = H.path_off[x + 1] - H.path_off[x], ly = H.path_off[y + 1] - H.path_off[y];
      if (lx != ly) return lx > ly;
      return x < y;
    });
  }
  return RB_OK;
}

}  // namespace ragb
