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
//
// Node ids: 0 = root, 1..V = kept virtual nodes, V+1+i = leaf (context) i.
// The replay accepts any dependency-respecting merge order (the device emits
// rounds); the exported merge order is sorted by key (X9).
#include <omp.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <numeric>
#include <string>
#include <thread>
#include <vector>

#include "internal.h"

namespace ragb {

namespace {

bool key_less(const MergeKey &x, const MergeKey &y) {
  if (x.h != y.h) return x.h < y.h;
  if (x.a != y.a) return x.a < y.a;
  return x.b < y.b;
}

// membership of x in a small sorted array
inline bool in_sorted(const uint32_t *s, int n, uint32_t x) {
  if (n <= 8) {
    for (int i = 0; i < n; ++i)
      if (s[i] == x) return true;
    return false;
  }
  return std::binary_search(s, s + n, x);
}

}  // namespace

static std::atomic<int> g_host_threads{0};

void set_host_threads(int n) { g_host_threads.store(std::max(0, n)); }

int host_threads() {
  if (const int o = g_host_threads.load()) return o;
  static int n = [] {
    // one core is left to the side sorter / CUDA driver thread: a static OpenMP
    // schedule with one oversubscribed core stalls every barrier (measured:
    // 15 threads 8 ms, 16 threads 14-20 ms on a 16-core host at C4)
    return std::max(1, std::min(15, omp_get_num_procs() - 1));
  }();
  return n;
}

// Incremental raw-tree state (see internal.h TreeBuild).
void host_begin(HostIndex &H, TreeBuild &T) {
  const int64_t N = H.N;
  const int32_t K = H.K;
  const bool uniform = H.lens.empty();
  const int nth = host_threads();
  const auto hb0 = std::chrono::steady_clock::now();
  T.zk.clear();
  T.runs.clear();
  T.rpar.assign((size_t)(N + std::max<int64_t>(N - 1, 0)), -1);
  T.keep.assign((size_t)std::max<int64_t>(N - 1, 0), 1);
  if (H.sort_merges) T.zk.reserve((size_t)std::max<int64_t>(N - 1, 0));
  // sorted leaf sets, in parallel on plain threads that exit afterwards: this
  // runs while the device rounds are launched from another thread, and an
  // OpenMP team would keep spinning on the cores that thread needs
  T.lset.resize((size_t)N * K);
  // the ordered contexts (a7, written by host_finish's branch A) are sized
  // and page-faulted here too, off the critical path: first touches of 8 MB
  // at C4 cost ~2 ms inside the tail stage otherwise
  H.ordered.resize((size_t)N * K);
  {
    // (two cores fewer than the tail stages: the round-launching thread and
    // this replay worker must not be preempted while the device rounds run)
    const int nt = std::max(1, std::min<int>(nth - 2, (int)((int64_t)N * K / 81920) + 1));  // ~80K entries per thread
    std::vector<std::thread> pool;
    for (int w = 0; w < nt; ++w)
      pool.emplace_back([&, w] {
        for (int64_t i = N * w / nt; i < N * (w + 1) / nt; ++i) {
          uint32_t *d = T.lset.data() + i * K;
          const uint32_t *src = H.ids.data() + i * K;
          const int L = uniform ? K : H.lens[i];
          if (L > 32) {  // long lists (C5: K up to 100): O(L log L)
            std::copy(src, src + L, d);
            std::sort(d, d + L);
            continue;
          }
          for (int k = 0; k < L; ++k) {  // insertion sort (typically 5-20 entries)
            const uint32_t x = src[k];
            int q = k;
            while (q > 0 && d[q - 1] > x) {
              d[q] = d[q - 1];
              --q;
            }
            d[q] = x;
          }
        }
        uint32_t *o = H.ordered.data();
        const int64_t e0 = N * w / nt * K, e1 = N * (w + 1) / nt * K;
        for (int64_t e = e0; e < e1; e += 1024) o[e] = 0;  // one store per 4 KB page
      });
    for (auto &t : pool) t.join();
  }
  const auto hb1 = std::chrono::steady_clock::now();
  const int64_t nz = std::max<int64_t>(N - 1, 0);
  T.voff.assign(nz + 1, 0);
  T.vpool.clear();
  T.vpool.reserve((size_t)N * 4 + 64);
  T.rchild.assign(2 * nz, 0);
  T.cur.resize(N);
  std::iota(T.cur.begin(), T.cur.end(), 0);
  T.csize.assign(N, 1);
  T.done = 0;
  T.ok = true;
  if (H.trace)
    std::fprintf(stderr, "[ragb host] begin: setup+sort %.3f ms, rest %.3f ms\n",
                 std::chrono::duration<double, std::milli>(hb1 - hb0).count(),
                 std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - hb1).count());
}

// Replay merges [T.done, upto) of H.za/zb/zs: any order in which every merge
// follows the merges that built its two clusters (the device emits rounds).
void host_replay(HostIndex &H, TreeBuild &T, int64_t upto) {
  const int64_t N = H.N;
  const int32_t K = H.K;
  const bool uniform = H.lens.empty();
  const int64_t t_from = T.done;
  const auto q0 = std::chrono::steady_clock::now();
  // a round's merges arrive in the device's emission order, which is not
  // deterministic (reciprocal pairs are appended with atomics).  Sorted by key
  // (X9) they are still a valid replay order — the round's reciprocal pairs
  // are disjoint, and a level clique's picks merge into its start with
  // increasing keys — and the same on every run, so are the raw node numbers
  // and the exported tree numbering (ragb.h rb_index_tree).
  if (H.sort_merges && upto > t_from + 1) {
    std::vector<MergeKey> b((size_t)(upto - t_from));
    for (int64_t t = t_from; t < upto; ++t) b[t - t_from] = {H.zh[t], H.za[t], H.zb[t], H.zs[t]};
    std::sort(b.begin(), b.end(), key_less);
    for (int64_t t = t_from; t < upto; ++t) {
      const MergeKey &m = b[t - t_from];
      H.zh[t] = m.h;
      H.za[t] = m.a;
      H.zb[t] = m.b;
      H.zs[t] = m.size;
    }
  }
  const auto q1 = std::chrono::steady_clock::now();
  // the loop is bound by the latency of its scattered reads (cur, the two
  // children's sets): prefetch cur two strides ahead and the sets one stride
  // ahead (a later merge of this batch may still renumber a cluster: only a
  // wasted hint then)
  constexpr int64_t kPf = 8;
  auto set_addr = [&](int32_t X) -> const void * {
    return X < N ? static_cast<const void *>(T.lset.data() + (int64_t)X * K)
                 : static_cast<const void *>(T.vpool.data() + T.voff[X - N]);
  };
  for (int64_t t = T.done; t < upto && T.ok; ++t) {
    if (t + 2 * kPf < upto) {
      __builtin_prefetch(&T.cur[H.za[t + 2 * kPf]]);
      __builtin_prefetch(&T.cur[H.zb[t + 2 * kPf]]);
    }
    if (t + kPf < upto) {
      const int32_t pa2 = T.cur[H.za[t + kPf]], pb2 = T.cur[H.zb[t + kPf]];
      if (pa2 >= 0 && pa2 < N + t) __builtin_prefetch(set_addr(pa2));
      if (pb2 >= 0 && pb2 < N + t) __builtin_prefetch(set_addr(pb2));
    }
    const int32_t a = H.za[t], b = H.zb[t];
    if (a < 0 || b >= N || a >= b || T.cur[a] < 0 || T.cur[b] < 0 ||
        T.csize[a] + T.csize[b] != H.zs[t]) {
      T.ok = false;
      T.err = "inconsistent merge at row " + std::to_string(t);
      break;
    }
    const int32_t A = T.cur[a], B = T.cur[b];
    T.rchild[2 * t] = A;
    T.rchild[2 * t + 1] = B;
    int la, lb;
    const uint32_t *pa, *pb;
    if (A < N) {
      la = uniform ? K : H.lens[A];
      pa = T.lset.data() + (int64_t)A * K;
    } else {
      la = (int)(T.voff[A - N + 1] - T.voff[A - N]);
      pa = T.vpool.data() + T.voff[A - N];
    }
    if (B < N) {
      lb = uniform ? K : H.lens[B];
      pb = T.lset.data() + (int64_t)B * K;
    } else {
      lb = (int)(T.voff[B - N + 1] - T.voff[B - N]);
      pb = T.vpool.data() + T.voff[B - N];
    }
    uint32_t tmp[256];
    int n = 0, ia = 0, ib = 0;
    while (ia < la && ib < lb) {  // sorted intersection, branch-free steps
      const uint32_t x = pa[ia], y = pb[ib];
      tmp[n] = x;
      n += (x == y);
      ia += (x <= y);
      ib += (y <= x);
    }
    T.vpool.insert(T.vpool.end(), tmp, tmp + n);
    T.voff[t + 1] = (int64_t)T.vpool.size();
    // the two children now have their raw parent: collapse flags (X11) of
    // virtual children are final (a child collapses iff its set equals this
    // merge's set), computed here while the device runs later rounds
    T.rpar[A] = N + t;
    T.rpar[B] = N + t;
    const uint32_t *ps = T.vpool.data() + T.voff[t];
    if (A >= N) T.keep[A - N] = (la == n && std::memcmp(pa, ps, 4 * (size_t)n) == 0) ? 0 : 1;
    if (B >= N) T.keep[B - N] = (lb == n && std::memcmp(pb, ps, 4 * (size_t)n) == 0) ? 0 : 1;
    T.cur[a] = (int32_t)(N + t);
    T.cur[b] = -1;
    T.csize[a] += T.csize[b];
    T.done = t + 1;
  }
  const auto q2 = std::chrono::steady_clock::now();
  if (H.trace) std::fprintf(stderr, "[replay] n=%ld sort %.3f loop %.3f\n", (long)(upto - t_from),
    std::chrono::duration<double, std::milli>(q1 - q0).count(), std::chrono::duration<double, std::milli>(q2 - q1).count());
  // the exported order (X9) is built here too, batch by batch: each replayed
  // batch is sorted while the device runs the next rounds, and host_finish
  // only merges the sorted runs
  if (T.ok && H.sort_merges && T.done > t_from) {
    if (T.runs.empty()) T.runs.push_back(0);
    for (int64_t t = t_from; t < T.done; ++t) T.zk.push_back({H.zh[t], H.za[t], H.zb[t], H.zs[t]});  // sorted above
    T.runs.push_back((int64_t)T.zk.size());
  }
}

rb_status host_build(HostIndex &H, std::string *msg) {
  if ((int64_t)H.za.size() != H.N - 1) {
    *msg = "merge list must have N-1 rows";
    return RB_EINVAL;
  }
  TreeBuild T;
  const auto t0 = std::chrono::steady_clock::now();
  host_begin(H, T);
  const auto t1 = std::chrono::steady_clock::now();
  host_replay(H, T, (int64_t)H.za.size());
  if (H.trace)
    std::fprintf(stderr, "[ragb host] begin %.3f ms replay %.3f ms\n",
                 std::chrono::duration<double, std::milli>(t1 - t0).count(),
                 std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t1).count());
  return host_finish(H, T, msg);
}

rb_status host_finish(HostIndex &H, TreeBuild &T, std::string *msg) {
  const int64_t N = H.N;
  const int32_t K = H.K;
  const bool uniform = H.lens.empty();
  const int nth = host_threads();
  const bool trace = H.trace;
  auto t_last = std::chrono::steady_clock::now();
  auto lap = [&](const char *what) {
    if (!trace) return;
    const auto t = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[ragb host] %-12s %.3f ms\n", what,
                 std::chrono::duration<double, std::milli>(t - t_last).count());
    t_last = t;
  };
  auto len_of = [&](int64_t i) -> int { return uniform ? K : H.lens[i]; };
  const int64_t nz = (int64_t)H.za.size();
  if (nz != N - 1) {
    *msg = "merge list must have N-1 rows";
    return RB_EINVAL;
  }
  host_replay(H, T, nz);
  if (!T.ok) {
    *msg = T.err;
    return RB_EINVAL;
  }
  const auto &lset = T.lset;
  const std::vector<int64_t> &voff = T.voff;
  const std::vector<uint32_t> &vpool = T.vpool;
  const std::vector<int32_t> &rchild = T.rchild;
  auto set_ptr = [&](int64_t r, int *n) -> const uint32_t * {
    if (r < N) {
      *n = len_of(r);
      return lset.data() + r * K;
    }
    *n = (int)(voff[r - N + 1] - voff[r - N]);
    return vpool.data() + voff[r - N];
  };
  const int64_t top = T.cur[0];
  if (T.csize[0] != N) {
    *msg = "merges do not join all contexts";
    return RB_EINVAL;
  }
  lap("replay tail");

  // ---- exported merge order: ascending key (X9), sorted on a side thread
  //      while the tree is built (the tree reads the replay order) ---------
  std::vector<MergeKey> &zk = T.zk;
  std::thread sorter([&] {
    if (!H.sort_merges) return;  // non-reducible linkage: keep the merge order
    if ((int64_t)zk.size() != nz) {  // not built by the replay: sort here
      zk.resize(nz);
      for (int64_t t = 0; t < nz; ++t) zk[t] = {H.zh[t], H.za[t], H.zb[t], H.zs[t]};
      std::sort(zk.begin(), zk.end(), key_less);
      return;
    }
    // merge the sorted batches pairwise (log2(rounds) passes)
    std::vector<int64_t> r = T.runs;
    while (r.size() > 2) {
      std::vector<int64_t> nr;
      for (size_t i = 0; i + 2 < r.size(); i += 2) {
        std::inplace_merge(zk.begin() + r[i], zk.begin() + r[i + 1], zk.begin() + r[i + 2], key_less);
        nr.push_back(r[i]);
      }
      if (r.size() % 2 == 0) nr.push_back(r[r.size() - 2]);
      nr.push_back(r.back());
      r.swap(nr);
    }
  });

  // ---- collapse (X11) -----------------------------------------------------
  // A raw node is collapsed iff its set equals its raw parent's set (the root
  // set is empty): the nearest kept ancestor of a collapsed node has the same
  // set as its raw parent, by induction.  Flags in parallel, then one
  // top-down pass (parents have larger merge index) numbers the kept nodes
  // 1..V in decreasing merge index, so every parent precedes its children.
  // The tail runs two branches on two OpenMP teams (below) plus the merge
  // sorter; the collapse uses branch B's team size so that the pool threads
  // it leaves idle (libgomp spins them for milliseconds) do not compete with
  // branch A's team for the cores.
  const int thA = std::max(1, nth / 2), thB = std::max(1, nth - thA);
#ifdef RAGB_COLLAPSE_NTH
  const int thC = nth;
#else
  const int thC = thB;
#endif
  std::vector<int64_t> vraw;
  std::vector<int32_t> vpar;
  H.lparent.assign(N, 0);
  {
    // raw parents and collapse flags come from the replay; the top merge (no
    // parent) is collapsed iff its set is empty (the root's set)
    const std::vector<int64_t> &rpar = T.rpar;
    std::vector<uint8_t> &keep = T.keep;
    if (nz > 0) {
      int n1;
      for (int64_t t = 0; t < nz; ++t)
        if (rpar[N + t] < 0) {
          set_ptr(N + t, &n1);
          keep[t] = n1 == 0 ? 0 : 1;
        }
    }
    // kept node ids in decreasing merge index (a suffix count of the flags,
    // chunked over the threads)
    std::vector<int32_t> eff(nz);  // kept node id standing for raw merge t
    const int nc = std::max(1, std::min<int>(thC, (int)(nz / 8192) + 1));
    std::vector<int64_t> ccount(nc + 1, 0);
#pragma omp parallel for num_threads(nc) schedule(static, 1)
    for (int c = 0; c < nc; ++c) {  // chunk c covers t in [hi - ..., hi) from the top
      const int64_t t1 = nz - nz * c / nc, t0 = nz - nz * (c + 1) / nc;
      int64_t k = 0;
      for (int64_t t = t0; t < t1; ++t) k += keep[t];
      ccount[c + 1] = k;
    }
    for (int c = 0; c < nc; ++c) ccount[c + 1] += ccount[c];
    const int64_t V0 = ccount[nc];
    vraw.resize(V0);
    vpar.resize(V0);
    // up[t]: t itself if kept (or top), else its raw parent merge; pointer
    // doubling gives every merge its nearest kept ancestor-or-self
    std::vector<int64_t> up(nz);
#pragma omp parallel for num_threads(nc) schedule(static, 1)
    for (int c = 0; c < nc; ++c) {
      const int64_t t1 = nz - nz * c / nc, t0 = nz - nz * (c + 1) / nc;
      int32_t id = (int32_t)ccount[c];
      for (int64_t t = t1 - 1; t >= t0; --t) {
        if (keep[t]) {
          eff[t] = ++id;
          vraw[id - 1] = N + t;
        }
        const int64_t p = rpar[N + t];
        up[t] = (keep[t] || p < 0) ? t : p - N;
      }
    }
    for (bool more = true; more;) {
      more = false;
#pragma omp parallel for num_threads(thC) schedule(static) reduction(|| : more)
      for (int64_t t = 0; t < nz; ++t) {
        const int64_t u = up[t], uu = up[u];
        if (uu != u) {
          up[t] = uu;
          more = true;
        }
      }
    }
    // eff of a collapsed merge: its nearest kept ancestor (0: the root)
#pragma omp parallel for num_threads(thC) schedule(static)
    for (int64_t t = 0; t < nz; ++t)
      if (!keep[t]) eff[t] = keep[up[t]] ? eff[up[t]] : 0;
#pragma omp parallel for num_threads(thC) schedule(static)
    for (int64_t k = 0; k < V0; ++k) {
      const int64_t p = rpar[vraw[k]];
      vpar[k] = p < 0 ? 0 : eff[p - N];
    }
#pragma omp parallel for num_threads(thC) schedule(static)
    for (int64_t i = 0; i < N; ++i) {
      const int64_t p = rpar[i];
      H.lparent[i] = p < 0 ? 0 : eff[p - N];
    }
  }
  (void)top;
  const int64_t V = (int64_t)vraw.size();
  lap("collapse");

  // Two independent branches from here on, each on its own OpenMP team:
  //   A (side thread): ordered prefixes of the virtual nodes (X10), then the
  //     leaves' ordered contexts (a7) and prefix lengths;
  //   B (this thread): children lists by rep (X12), search paths, schedule.
  H.V = V;
  H.vparent.assign(vpar.begin(), vpar.end());
  std::thread branchA([&] {
    const auto ta0 = std::chrono::steady_clock::now();
    // ---- virtual nodes: ordered prefixes (X10) ------------------------------
    // prefix(k) = prefix(parent) ++ sorted(set(k) \ set(parent)) has |set(k)|
    // entries; each node writes its own by walking up its ancestors (depth <=
    // K + 1 after the collapse), so the nodes are filled in parallel.
    H.vpre_off.assign(V + 2, 0);  // by node id 0..V (root: empty)
    for (int64_t k = 1; k <= V; ++k) {
      int nk;
      set_ptr(vraw[k - 1], &nk);
      H.vpre_off[k + 1] = H.vpre_off[k] + nk;
    }
    H.vpre.resize(H.vpre_off[V + 1]);
#pragma omp parallel for num_threads(thA) schedule(dynamic, 512)
    for (int64_t k = 1; k <= V; ++k) {
      int32_t chain[260];
      int nc = 0;
      for (int32_t x = (int32_t)k; x > 0; x = vpar[x - 1]) chain[nc++] = x;
      uint32_t *o = H.vpre.data() + H.vpre_off[k];
      for (int c = nc - 1; c >= 0; --c) {  // top-down
        const int32_t x = chain[c], px = vpar[x - 1];
        int nx, np = 0;
        const uint32_t *sx = set_ptr(vraw[x - 1], &nx);
        const uint32_t *sp = px > 0 ? set_ptr(vraw[px - 1], &np) : nullptr;
        int q = 0;
        for (int z = 0; z < nx; ++z) {  // both sorted: merge-difference
          while (q < np && sp[q] < sx[z]) ++q;
          if (q < np && sp[q] == sx[z]) continue;
          *o++ = sx[z];
        }
      }
    }
    const auto ta1 = std::chrono::steady_clock::now();
    // ---- leaves: ordered contexts (a7) and prefix lengths -------------------
    H.ordered.resize((size_t)N * K);  // every entry written below (no fill)
    H.prefix_len.assign(N, 0);
    const auto ta2 = std::chrono::steady_clock::now();
#pragma omp parallel for num_threads(thA) schedule(static)
    for (int64_t i = 0; i < N; ++i) {
      const int32_t p = H.lparent[i];
      const int64_t p0 = H.vpre_off[p], p1 = H.vpre_off[p + 1];
      uint32_t *out = H.ordered.data() + i * K;
      int o = 0;
      for (int64_t z = p0; z < p1; ++z) out[o++] = H.vpre[z];
      int np = 0;
      const uint32_t *sp = p > 0 ? set_ptr(vraw[p - 1], &np) : nullptr;
      const uint32_t *row = H.ids.data() + i * K;
      const int L = len_of(i);
      if (np > 16) {
        // long parent sets (C5: K up to 100): an open-addressing table of the
        // parent's docs (0xFFFFFFFF, the reserved DocId, marks an empty slot)
        // instead of a branchy binary search per entry
        uint32_t tab[512];
        int bits = 5;
        while ((1 << bits) < 2 * np) ++bits;
        const uint32_t msk = (1u << bits) - 1u;
        std::fill(tab, tab + (1 << bits), 0xFFFFFFFFu);
        for (int z = 0; z < np; ++z) {
          uint32_t hsh = (sp[z] * 0x9E3779B1u) >> (32 - bits);
          while (tab[hsh] != 0xFFFFFFFFu) hsh = (hsh + 1) & msk;
          tab[hsh] = sp[z];
        }
        for (int k = 0; k < L; ++k) {
          const uint32_t x = row[k];
          uint32_t hsh = (x * 0x9E3779B1u) >> (32 - bits);
          while (tab[hsh] != 0xFFFFFFFFu && tab[hsh] != x) hsh = (hsh + 1) & msk;
          if (tab[hsh] != x) out[o++] = x;
        }
      } else {
        for (int k = 0; k < L; ++k)
          if (!in_sorted(sp, np, row[k])) out[o++] = row[k];
      }
      for (int k = L; k < K; ++k) out[k] = row[k];  // padding slots of a shorter context
      H.prefix_len[i] = (uint8_t)(p1 - p0);
    }
    if (trace)
      std::fprintf(stderr, "[ragb host] A: prefixes %.3f alloc %.3f leaves %.3f ms\n",
                   std::chrono::duration<double, std::milli>(ta1 - ta0).count(),
                   std::chrono::duration<double, std::milli>(ta2 - ta1).count(),
                   std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - ta2).count());
  });

  // ---- children CSR over nodes 0..V, ordered by rep (X12) -----------------
  std::vector<int32_t> rep_of(1 + V + N);
  rep_of[0] = -1;
#pragma omp parallel for num_threads(thB) schedule(static)
  for (int64_t k = 1; k <= V; ++k) rep_of[k] = H.za[vraw[k - 1] - N];  // rep = a (< b)
#pragma omp parallel for num_threads(thB) schedule(static)
  for (int64_t i = 0; i < N; ++i) rep_of[V + 1 + i] = (int32_t)i;
  H.kids_off.assign(V + 2, 0);
  for (int64_t k = 1; k <= V; ++k) ++H.kids_off[vpar[k - 1] + 1];
  for (int64_t i = 0; i < N; ++i) ++H.kids_off[H.lparent[i] + 1];
  for (int64_t k = 0; k <= V; ++k) H.kids_off[k + 1] += H.kids_off[k];
  H.kids.resize(V + N);  // every entry placed below
  std::vector<int32_t> child_idx(1 + V + N, 0);
  {
    // Nodes in ascending rep order, appended to their parents' lists, give
    // every child list sorted by rep (X12).  Leaf i is the rep of itself and of
    // the chain of kept ancestors whose smallest leaf it is, so walking up from
    // each leaf in index order visits every node once, by rep (a node and its
    // leftmost descendants share a rep but are never siblings).  The walk runs
    // in leaf chunks: per-chunk counts per parent, their prefix over the
    // chunks, then every chunk places its nodes.
    const int nc = std::max(1, std::min<int>(thB, (int)(N / 4096) + 1));
    const int64_t P = V + 1;
    std::vector<int32_t> off((size_t)nc * P);
    auto walk = [&](int c, auto &&visit) {
      for (int64_t i = N * c / nc; i < N * (c + 1) / nc; ++i) {
        int32_t y = H.lparent[i];
        visit((int32_t)(V + 1 + i), y);
        while (y > 0 && rep_of[y] == (int32_t)i) {
          const int32_t py = vpar[y - 1];
          visit(y, py);
          y = py;
        }
      }
    };
#pragma omp parallel for num_threads(nc) schedule(static, 1)
    for (int c = 0; c < nc; ++c) {
      int32_t *o = off.data() + (size_t)c * P;
      std::fill(o, o + P, 0);
      walk(c, [&](int32_t, int32_t par) { ++o[par]; });
    }
#pragma omp parallel for num_threads(nc) schedule(static)
    for (int64_t p = 0; p < P; ++p) {
      int32_t run = 0;
      for (int c = 0; c < nc; ++c) {
        const int32_t k = off[(size_t)c * P + p];
        off[(size_t)c * P + p] = run;
        run += k;
      }
    }
#pragma omp parallel for num_threads(nc) schedule(static, 1)
    for (int c = 0; c < nc; ++c) {
      int32_t *o = off.data() + (size_t)c * P;
      walk(c, [&](int32_t x, int32_t par) {
        const int32_t k = o[par]++;
        child_idx[x] = k;
        H.kids[H.kids_off[par] + k] = x;
      });
    }
  }
  lap("children");

  // ---- search paths: virtual nodes, then leaves -----------------------------
  H.vrep.resize(V);
  std::vector<int64_t> vpath_off(V + 2, 0);
  std::vector<int32_t> depth(V + 1, 0);
  for (int64_t k = 1; k <= V; ++k) {
    H.vrep[k - 1] = rep_of[k];
    depth[k] = depth[vpar[k - 1]] + 1;
    vpath_off[k + 1] = vpath_off[k] + depth[k];
  }
  std::vector<int32_t> vpath(vpath_off[V + 1]);
#pragma omp parallel for num_threads(thB) schedule(static)
  for (int64_t k = 1; k <= V; ++k) {
    int32_t *pp = vpath.data() + vpath_off[k + 1];  // filled backwards: the node, then its ancestors
    for (int32_t x = (int32_t)k; x > 0; x = vpar[x - 1]) *--pp = child_idx[x];
  }
  H.path_off.assign(N + 1, 0);
  for (int64_t i = 0; i < N; ++i) H.path_off[i + 1] = H.path_off[i] + depth[H.lparent[i]] + 1;
  H.path.resize(H.path_off[N]);  // every entry written below
  int64_t max_depth = 0;
#pragma omp parallel for num_threads(thB) schedule(static) reduction(max : max_depth)
  for (int64_t i = 0; i < N; ++i) {
    const int32_t p = H.lparent[i];
    int32_t *pp = H.path.data() + H.path_off[i];
    for (int64_t z = vpath_off[p]; z < vpath_off[p + 1]; ++z) *pp++ = vpath[z];
    *pp = child_idx[V + 1 + i];
    max_depth = std::max<int64_t>(max_depth, H.path_off[i + 1] - H.path_off[i]);
  }
  H.stats.n_virtual = V;
  H.stats.max_depth = max_depth;
  lap("paths");

  // ---- schedule: groups of first appearance, length descending, index -----
  // The group of leaf i is the root child on its path; the first leaf of a
  // group (in index order) is the group's rep, and root children are ordered
  // by rep (X12), so groups rank by child index.  A group holds the leaves of
  // its root child's subtree (the cluster size of that child's merge): offsets
  // by a prefix over the root children, atomic placement, then each group
  // sorted by (length descending, index).
  {
    const int64_t G = H.kids_off[1] - H.kids_off[0];  // root children
    std::vector<int64_t> goff(G + 1, 0);
    for (int64_t g = 0; g < G; ++g) {
      const int32_t x = H.kids[H.kids_off[0] + g];
      goff[g + 1] = goff[g] + (x > V ? 1 : H.zs[vraw[x - 1] - N]);
    }
    if (goff[G] != N) {
      *msg = "schedule: root subtrees do not cover the contexts";
      branchA.join();
      sorter.join();
      return RB_EINVAL;
    }
    std::vector<int64_t> gcur(goff.begin(), goff.end() - 1);
    // sort key within a group: (max_depth - length) << 32 | index
    std::vector<uint64_t> sk(N);
#pragma omp parallel for num_threads(thB) schedule(static)
    for (int64_t i = 0; i < N; ++i) {
      const int64_t p0 = H.path_off[i], len = H.path_off[i + 1] - p0;
      const int32_t g = H.path[p0];
      sk[__atomic_fetch_add(&gcur[g], 1, __ATOMIC_RELAXED)] = ((uint64_t)(max_depth - len) << 32) | (uint64_t)i;
    }
    H.schedule.resize(N);
#pragma omp parallel for num_threads(thB) schedule(dynamic, 256)
    for (int64_t g = 0; g < G; ++g) {
      if (goff[g + 1] - goff[g] > 1) std::sort(sk.begin() + goff[g], sk.begin() + goff[g + 1]);
      for (int64_t z = goff[g]; z < goff[g + 1]; ++z) H.schedule[z] = (int64_t)(sk[z] & 0xffffffffull);
    }
  }
  lap("schedule");
  branchA.join();
  lap("prefixes+leaves (A)");

  sorter.join();
  for (int64_t t = 0; t < (int64_t)zk.size(); ++t) {
    H.za[t] = zk[t].a;
    H.zb[t] = zk[t].b;
    H.zh[t] = zk[t].h;
    H.zs[t] = zk[t].size;
  }
  lap("sort merges");
  return RB_OK;
}

}  // namespace ragb
