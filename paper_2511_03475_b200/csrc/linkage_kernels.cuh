// a5 kernels shared by the single-GPU linkage (linkage.cu) and the
// row-sharded build (dist.cu).  See linkage.cu for the algorithm.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "internal.h"

namespace ragb {
namespace {

typedef unsigned long long u64;
constexpr int PT = 1024;  // threads of the single-CTA round-prep kernel
constexpr u64 kDead = ~0ull;  // row key of a row merged away by an in-place round
constexpr int kInplaceMaxM = 48 * 1024;  // in-place rounds keep a whole row in shared memory

struct PrepArgs {
  const float *D;
  int64_t ld;
  int M;
  const u64 *key;
  const int *rep;
  const int *sz;
  int *leader;
  uint8_t *alive;
  int *list, *candA, *candB;  // alias goff/gmem/colsrc (written later)
  int *za, *zb, *zs;
  float *zh;
  int *zcount;
  int *newidx, *goff, *gmem, *colsrc /* colmap */, *cnt, *cursor /* then first_old */;
  int *rep_n, *sz_n;
  int *Mn;
  int *level;  // [0] level list length, [1] h bits
  int *cstat;  // clique diagnostics: starts, batches, picks, candidates, level n, clk/1k (warp0, pass)
};

struct BlockScratch {
  int w[32];
  int total;
  unsigned h;
};

// Exclusive scan of v over the 1024 threads; returns the prefix, sets *total.
__device__ __forceinline__ int block_scan1024(int v, BlockScratch &S, int *total) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) S.w[w] = x;
  __syncthreads();
  if (w == 0) {
    int t = S.w[lane];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, t, o);
      if (lane >= o) t += y;
    }
    S.w[lane] = t;
  }
  __syncthreads();
  const int before = (w == 0) ? 0 : S.w[w - 1];
  *total = S.w[31];
  __syncthreads();
  return before + x - v;
}

// Order-preserving compaction: out[...] = value(i) for i in [0, n) with pred(i).
template <typename Pred, typename Val>
__device__ int block_compact(int n, Pred pred, Val value, int *out, BlockScratch &S) {
  int base = 0;
  for (int c0 = 0; c0 < n; c0 += PT) {
    const int i = c0 + (int)threadIdx.x;
    const bool p = i < n && pred(i);
    int tot;
    const int pre = block_scan1024(p ? 1 : 0, S, &tot);
    if (p) out[base + pre] = value(i);
    base += tot;
  }
  __syncthreads();
  return base;
}

// Round step 1 (one CTA): h = min row key; RNN pairs above h (emitted); the
// vertices whose row min equals h become the level list (ascending).
__global__ void __launch_bounds__(PT, 1) k_prep_mark(PrepArgs a) {
  __shared__ BlockScratch S;
  const int tid = threadIdx.x;
  const int M = a.M;

  // -- 1. current minimum height h ------------------------------------------
  unsigned hl = 0xffffffffu;
  for (int x = tid; x < M; x += PT) hl = min(hl, (unsigned)(a.key[x] >> 32));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) hl = min(hl, __shfl_xor_sync(0xffffffffu, hl, o));
  if (tid == 0) S.h = 0xffffffffu;
  __syncthreads();
  if ((tid & 31) == 0) atomicMin(&S.h, hl);
  __syncthreads();
  const unsigned h = S.h;
  const float hf = __uint_as_float(h);

  // -- 2. RNN pairs above h; vertices at h become clique candidates ------------
  for (int x = tid; x < M; x += PT) {
    const u64 kx = a.key[x];
    const unsigned hx = (unsigned)(kx >> 32);
    const int y = (int)(kx & 0xffffffffu);
    const bool dead = kx == kDead;  // row merged away by an in-place round
    int lead = dead ? -1 : x;
    a.alive[x] = (!dead && hx == h) ? 1 : 0;
    if (!dead && hx > h && (int)(a.key[y] & 0xffffffffu) == x) {
      if (y < x) {
        lead = y;
      } else {
        const int pos = atomicAdd(a.zcount, 1);
        a.za[pos] = a.rep[x];
        a.zb[pos] = a.rep[y];
        a.zh[pos] = __uint_as_float(hx);
        a.zs[pos] = a.sz[x] + a.sz[y];
      }
    }
    a.leader[x] = lead;
  }
  __syncthreads();

  // level list: vertices at h, ascending
  const uint8_t *alive = a.alive;
  const int nlist = block_compact(
      M, [&](int i) { return alive[i] != 0; }, [&](int i) { return i; }, a.list, S);
  if (tid == 0) {
    a.level[0] = nlist;
    a.level[1] = (int)h;
  }
}

// Round step 2 (grid): adjacency bits of the level graph, adj[i][w] bit j <=>
// D[list[i]][list[32w + j]] == h (j != i).  One warp per word: 32 lanes read
// 32 ascending columns of the same row.
__global__ void k_level_adj(PrepArgs a, uint32_t *__restrict__ adj) {
  const int n = a.level[0];
  if (n < 2) return;
  const float hf = __uint_as_float((unsigned)a.level[1]);
  const int W = (n + 31) >> 5;
  const int lane = threadIdx.x & 31;
  const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t total = (int64_t)n * W;
  for (int64_t q = gw; q < total; q += nw) {
    const int i = (int)(q / W), w = (int)(q - (int64_t)i * W);
    const int j = w * 32 + lane;
    bool bit = false;
    if (j < n && j != i) bit = __ldg(a.D + (int64_t)a.list[i] * a.ld + a.list[j]) == hf;
    const unsigned word = __ballot_sync(0xffffffffu, bit);
    if (lane == 0) adj[q] = word;
  }
}

// Round step 3 (one CTA): greedy clique contractions at height h.  At the
// current minimum height the greedy algorithm takes the smallest vertex with
// an h-neighbour and absorbs its smallest h-neighbour; the merged cluster stays
// at h only from vertices at h from both (max(h, h') = h iff h' = h), so the
// candidate set shrinks by intersection; then the next vertex.  Candidate and
// alive sets are bitsets over list positions in shared memory.
// Batching: warp 0 takes the next (up to) 32 candidates p_1 < ... < p_32 of C;
// the sequential process picks p_1, then each p_j adjacent to every earlier
// pick (C restricted to (p_1, p_32] is exactly p_2..p_32), which is a shuffle
// chain over the 32x32 adjacency bits.  One block pass then folds the picks'
// adjacency rows into C above p_32.  Warp 0 only records the picks (list
// positions, in greedy order); the merge rows (reps, cumulative sizes,
// leaders) are written afterwards by the whole block with a segmented scan.
// Warp-resident variant (n <= 32 * 32 * WPL): one warp holds the alive and
// candidate bitsets in registers (lane l owns words [l*WPL, (l+1)*WPL)), so a
// batch costs no block barrier: collect the next <= 32 candidates, their
// mutual adjacency bits, the pick chain, then fold the picks' adjacency rows
// into C above the last candidate.  For n <= 1024 the adjacency (n x 32
// words) is staged in shared memory first.  Returns the number of picks
// (lane-uniform); picks go to seq/seqs in greedy order.
template <int WPL>
__device__ int cliques_warp(const PrepArgs &a, const uint32_t *adj, int n, int W, int *s_p, int *seq,
                            int *seqs) {
  const int lane = threadIdx.x & 31;
  const int base = lane * WPL;
  uint32_t A[WPL], C[WPL];
#pragma unroll
  for (int u = 0; u < WPL; ++u) {
    const int w = base + u, rem = n - w * 32;
    A[u] = w < W ? (rem >= 32 ? 0xffffffffu : ((1u << rem) - 1u)) : 0u;
  }
  int nseq = 0;
  for (int ia = 0; ia < n; ++ia) {
    const int wi = ia >> 5, own = wi / WPL, ui = wi - own * WPL;
    uint32_t aw = 0u;
#pragma unroll
    for (int u = 0; u < WPL; ++u) aw = u == ui ? A[u] : aw;
    aw = __shfl_sync(0xffffffffu, aw, own);
    if (!((aw >> (ia & 31)) & 1u)) continue;  // absorbed earlier
    const uint32_t gt = (ia & 31) == 31 ? 0u : (0xffffffffu << ((ia & 31) + 1));
    const uint32_t *row = adj + (int64_t)ia * W;
#pragma unroll
    for (int u = 0; u < WPL; ++u) {
      const int w = base + u;
      uint32_t x = w < W ? row[w] : 0u;
      x &= A[u];
      x = w < wi ? 0u : (w == wi ? (x & gt) : x);
      C[u] = x;
    }
    while (true) {
      // -- collect the first <= 32 candidates -------------------------------
      int cnt = 0;
#pragma unroll
      for (int u = 0; u < WPL; ++u) cnt += __popc(C[u]);
      int incl = cnt;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, incl, o);
        incl += lane >= o ? y : 0;
      }
      const int total = __shfl_sync(0xffffffffu, incl, 31);
      if (total == 0) break;
      int slot = incl - cnt;
#pragma unroll
      for (int u = 0; u < WPL; ++u) {
        uint32_t x = C[u];
        while (x != 0u && slot < 32) {
          s_p[slot++] = (base + u) * 32 + __ffs(x) - 1;
          x &= x - 1u;
        }
      }
      __syncwarp();
      const int k = min(total, 32);
      const int pi = lane < k ? s_p[lane] : 0;
      // -- m bit j (j < lane): p_j adjacent to p_lane ------------------------
      const uint32_t *arow = adj + (int64_t)pi * W;
      uint32_t wd[31];
#pragma unroll
      for (int j = 0; j < 31; ++j) wd[j] = (j < lane && lane < k) ? arow[s_p[j] >> 5] : 0u;
      uint32_t m = 0u;
#pragma unroll
      for (int j = 0; j < 31; ++j) m |= ((wd[j] >> (s_p[j] & 31)) & 1u) << j;
      // -- pick chain --------------------------------------------------------
      uint32_t ch = 1u;
      uint32_t rem = __ballot_sync(0xffffffffu, lane < k && (m & 1u));
      while (rem != 0u) {
        const int j = __ffs(rem) - 1;
        ch |= 1u << j;
        rem &= __ballot_sync(0xffffffffu, (m >> j) & 1u) & ~((2u << j) - 1u);
      }
      const int rank = __popc(ch & ((1u << lane) - 1u));
      if (lane < k && ((ch >> lane) & 1u)) {
        seq[nseq + rank] = pi;
        seqs[nseq + rank] = ia;
      }
      nseq += __popc(ch);
      // -- picks leave the alive set ------------------------------------------
      for (uint32_t pm = ch; pm != 0u; pm &= pm - 1u) {
        const int pj = s_p[__ffs(pm) - 1];
        const int wj = pj >> 5, oj = wj / WPL, uj = wj - oj * WPL;
        const uint32_t clr = lane == oj ? ~(1u << (pj & 31)) : 0xffffffffu;
#pragma unroll
        for (int u = 0; u < WPL; ++u) A[u] &= u == uj ? clr : 0xffffffffu;
      }
      if (total <= 32) break;  // every candidate was considered
      // -- C &= adj(pick) for every pick, above the last candidate ------------
      const int last = s_p[31], wl = last >> 5;
      const uint32_t above = (last & 31) == 31 ? 0u : (0xffffffffu << ((last & 31) + 1));
      for (uint32_t pm = ch; pm != 0u; pm &= pm - 1u) {
        const uint32_t *prow = adj + (int64_t)s_p[__ffs(pm) - 1] * W;
#pragma unroll
        for (int u = 0; u < WPL; ++u) C[u] &= base + u < W ? prow[base + u] : 0u;
      }
#pragma unroll
      for (int u = 0; u < WPL; ++u) {
        const int w = base + u;
        C[u] = w < wl ? 0u : (w == wl ? (C[u] & above) : C[u]);
      }
      __syncwarp();  // s_p is rewritten by the next collection
    }
  }
  return nseq;
}
// Above 4096 vertices the per-batch fold (picks x WPL loads per lane) makes
// the single warp slower than the block-wide passes (measured at n = 16082).
constexpr int kWarpCliqueMaxN = 32 * 32 * 4;

constexpr int CT = 512;  // threads of k_level_cliques (128 registers for the pick chain)
__global__ void __launch_bounds__(CT, 1) k_level_cliques(PrepArgs a,
                                                         const uint32_t *__restrict__ adj) {
  extern __shared__ uint32_t bits[];  // [2][W]: alive, candidates
  __shared__ int s_first[2][CT / 32];
  __shared__ int s_p[64];     // next candidates (list positions), ascending
  __shared__ int s_pick[32];  // picks of the batch (list positions)
  __shared__ int s_npick, s_last, s_nseq;
  __shared__ int s_sv[CT / 32], s_sf[CT / 32];
  const int n = a.level[0];
  if (n < 2) return;
  const float hf = __uint_as_float((unsigned)a.level[1]);
  const int W = (n + 31) >> 5;
  uint32_t *A = bits, *C = bits + W;
  int *seq = a.candA, *seqs = a.candB;  // pick list position, its clique's start position
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  for (int w = tid; w < W; w += CT) {
    const int rem = n - w * 32;
    A[w] = rem >= 32 ? 0xffffffffu : ((1u << rem) - 1u);
  }
  __syncthreads();
  int parity = 0;
  // C[w] = f(w) for w >= w0; returns the first set bit position (or INT_MAX)
  auto pass = [&](int w0, auto f) {
    int first = 0x7fffffff;
    for (int w = w0 + tid; w < W; w += CT) {
      const uint32_t c = f(w);
      C[w] = c;
      first = (c != 0u && first == 0x7fffffff) ? w * 32 + __ffs(c) - 1 : first;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) first = min(first, __shfl_xor_sync(0xffffffffu, first, o));
    if (lane == 0) s_first[parity][wid] = first;
    __syncthreads();
    int m = lane < CT / 32 ? s_first[parity][lane] : 0x7fffffff;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = min(m, __shfl_xor_sync(0xffffffffu, m, o));
    parity ^= 1;
    return m;
  };
  int nseq = 0;  // warp 0: picks recorded so far
  long long st_starts = 0, st_batches = 0, st_picks = 0, st_cands = 0, st_w0 = 0, st_pass = 0;
  if (n <= kWarpCliqueMaxN) {
    if (n <= 1024) {  // stage the adjacency (n x W <= 32K words) in shared memory
      for (int i = tid; i < n * W; i += CT) bits[i] = __ldg(adj + i);
      __syncthreads();
      if (wid == 0) nseq = cliques_warp<1>(a, bits, n, W, s_p, seq, seqs);
    } else if (wid == 0) {
      nseq = cliques_warp<4>(a, adj, n, W, s_p, seq, seqs);
    }
  } else
  for (int ia = 0; ia < n; ++ia) {
    if (!((A[ia >> 5] >> (ia & 31)) & 1u)) continue;  // absorbed earlier (uniform)
    const int w0 = ia >> 5;
    const uint32_t gt = (ia & 31) == 31 ? 0u : (0xffffffffu << ((ia & 31) + 1));
    const uint32_t *row = adj + (int64_t)ia * W;
    ++st_starts;
    // the first batch reads adj(ia) & A above ia directly; later ones read C
    bool first = true;
    int cur = ia;
    while (true) {
      long long c0 = clock64();
      ++st_batches;
      if (wid == 0) {
        // -- collect the next <= 32 candidates; lane l covers 16 consecutive
        //    words of each 512-word chunk (all loads in flight) --------------
        int got = 0;
        for (int wpos = cur >> 5; got < 32 && wpos < W; wpos += 512) {
          const int wq = wpos + lane * 16;
          uint32_t c[16];
#pragma unroll
          for (int u = 0; u < 16; ++u) {
            const int w = wq + u;
            uint32_t x = 0u;
            if (w < W) x = first ? (__ldg(row + w) & A[w] & (w == w0 ? gt : 0xffffffffu)) : C[w];
            c[u] = x;
          }
          int cnt = 0;
#pragma unroll
          for (int u = 0; u < 16; ++u) cnt += __popc(c[u]);
          int incl = cnt;
#pragma unroll
          for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, incl, o);
            incl += lane >= o ? y : 0;
          }
          int slot = got + incl - cnt;
#pragma unroll
          for (int u = 0; u < 16; ++u) {
            uint32_t x = c[u];
            while (x != 0u && slot < 32) {
              s_p[slot++] = (wq + u) * 32 + __ffs(x) - 1;
              x &= x - 1u;
            }
          }
          got += __shfl_sync(0xffffffffu, incl, 31);
        }
        __syncwarp();
        const int k = min(got, 32);
        int npick = 0;
        if (k > 0) {
          const int pi = lane < k ? s_p[lane] : 0;
          // -- m bit j (j < lane): p_j adjacent to p_lane ----------------------
          const uint32_t *arow = adj + (int64_t)pi * W;
          uint32_t wd[31];
#pragma unroll
          for (int j = 0; j < 31; ++j) wd[j] = (j < lane && lane < k) ? __ldg(arow + (s_p[j] >> 5)) : 0u;
          uint32_t m = 0u;
#pragma unroll
          for (int j = 0; j < 31; ++j) m |= ((wd[j] >> (s_p[j] & 31)) & 1u) << j;
          // -- the pick chain: p_1, then the smallest remaining candidate
          //    adjacent to every pick so far (rem = lanes adjacent to all picks)
          uint32_t ch = 1u;
          uint32_t rem = __ballot_sync(0xffffffffu, lane < k && (m & 1u));
          while (rem != 0u) {
            const int j = __ffs(rem) - 1;
            ch |= 1u << j;
            rem &= __ballot_sync(0xffffffffu, (m >> j) & 1u) & ~((2u << j) - 1u);
          }
          const bool picked = lane < k && ((ch >> lane) & 1u);
          npick = __popc(ch);
          const int rank = __popc(ch & ((1u << lane) - 1u));
          if (picked) {
            seq[nseq + rank] = pi;
            seqs[nseq + rank] = ia;
            atomicAnd(&A[pi >> 5], ~(1u << (pi & 31)));
            s_pick[rank] = pi;
          }
        }
        nseq += npick;
        st_picks += npick;
        st_cands += k;
        if (lane == 0) {
          s_npick = npick;
          s_last = got > 32 || (got == 32 && k > 0) ? s_p[31] : -1;
        }
      }
      __syncthreads();
      st_w0 += clock64() - c0;
      c0 = clock64();
      const int last = s_last;
      if (last < 0) break;  // every candidate was considered (uniform)
      const int npick = s_npick;
      const int wl = last >> 5;
      const uint32_t above = (last & 31) == 31 ? 0u : (0xffffffffu << ((last & 31) + 1));
      const bool fst = first;
      cur = pass(wl, [&](int w) {
        uint32_t c = fst ? (__ldg(row + w) & A[w]) : C[w];
        c &= w == wl ? above : 0xffffffffu;
        for (int t = 0; t < npick; ++t) c &= __ldg(adj + (int64_t)s_pick[t] * W + w);
        return c;
      });
      st_pass += clock64() - c0;
      first = false;
      if (cur == 0x7fffffff) break;
    }
    __syncthreads();
  }
  if (tid == 0) s_nseq = nseq;
  __syncthreads();
  // -- emit the merges: zs = size of the clique after this pick (segmented
  //    inclusive scan of member sizes within a clique, plus the start's size)
  const int ns = s_nseq;
  const int zbase = *a.zcount;
  int carry = 0;
  for (int c0 = 0; c0 < ns; c0 += CT) {
    const int k = c0 + tid;
    int v = 0, f = 0, vb = 0, va = 0, st = -1;
    if (k < ns) {
      st = seqs[k];
      vb = a.list[seq[k]];
      va = a.list[st];
      v = a.sz[vb];
      f = (k == 0 || seqs[k - 1] != st) ? 1 : 0;
    }
    // segmented inclusive scan (flag starts a new segment)
    int sv = v, sf = f;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int yv = __shfl_up_sync(0xffffffffu, sv, o);
      const int yf = __shfl_up_sync(0xffffffffu, sf, o);
      sv = (lane >= o && !sf) ? sv + yv : sv;
      sf = lane >= o ? (sf | yf) : sf;
    }
    if (lane == 31) {
      s_sv[wid] = sv;
      s_sf[wid] = sf;
    }
    __syncthreads();
    // prefix over earlier warps of this chunk, then the previous chunks' carry
    int pv = carry, pf = 0;
    for (int q = 0; q < wid; ++q) {
      pv = s_sf[q] ? s_sv[q] : pv + s_sv[q];
      pf |= s_sf[q];
    }
    (void)pf;
    const int incl = sf ? sv : sv + pv;
    if (k < ns) {
      a.za[zbase + k] = a.rep[va];
      a.zb[zbase + k] = a.rep[vb];
      a.zh[zbase + k] = hf;
      a.zs[zbase + k] = a.sz[va] + incl;
      a.leader[vb] = va;
    }
    const int last_in = min(CT, ns - c0) - 1;
    __syncthreads();
    if (tid == last_in) s_sv[0] = incl;
    __syncthreads();
    carry = s_sv[0];
    __syncthreads();
  }
  if (tid == 0) {
    *a.zcount = zbase + ns;
    if (a.cstat) {
      a.cstat[0] = (int)st_starts;
      a.cstat[1] = (int)st_batches;
      a.cstat[2] = (int)st_picks;
      a.cstat[3] = (int)st_cands;
      a.cstat[4] = n;
      a.cstat[5] = (int)(st_w0 >> 10);
      a.cstat[6] = (int)(st_pass >> 10);
    }
  }
}

// Round step 4 (one CTA): order-preserving compaction map and group CSR.
__global__ void __launch_bounds__(PT, 1) k_prep_compact(PrepArgs a) {
  __shared__ BlockScratch S;
  const int tid = threadIdx.x;
  const int M = a.M;
  // -- 4. compaction map: new index of every survivor (order preserving) ------
  int base = 0;
  for (int c0 = 0; c0 < M; c0 += PT) {
    const int x = c0 + tid;
    const int f = (x < M && a.leader[x] == x) ? 1 : 0;
    int tot;
    const int pre = block_scan1024(f, S, &tot);
    if (x < M) a.newidx[x] = base + pre;  // valid for survivors
    base += tot;
  }
  const int Mn = base;
  for (int g = tid; g < Mn; g += PT) {
    a.cnt[g] = 0;
    a.cursor[g] = 0;
    a.sz_n[g] = 0;
  }
  __syncthreads();
  for (int x = tid; x < M; x += PT) {
    const int l = a.leader[x];
    if (l < 0) continue;  // dead row
    const int g = a.newidx[l];
    atomicAdd(&a.cnt[g], 1);
    atomicAdd(&a.sz_n[g], a.sz[x]);
    if (l == x) a.rep_n[g] = a.rep[x];
  }
  __syncthreads();
  base = 0;
  for (int c0 = 0; c0 < Mn; c0 += PT) {
    const int g = c0 + tid;
    const int v = g < Mn ? a.cnt[g] : 0;
    int tot;
    const int pre = block_scan1024(v, S, &tot);
    if (g < Mn) a.goff[g] = base + pre;
    base += tot;
  }
  if (tid == 0) {
    a.goff[Mn] = base;  // live rows (dead rows of in-place rounds are in no group)
    *a.Mn = Mn;
  }
  __syncthreads();
  for (int x = tid; x < M; x += PT) {
    const int l = a.leader[x];
    if (l < 0) continue;
    const int g = a.newidx[l];
    a.gmem[a.goff[g] + atomicAdd(&a.cursor[g], 1)] = x;
  }
  __syncthreads();
  // old column -> new column; new column -> its leader (smallest old member)
  for (int x = tid; x < M; x += PT) {
    const int l = a.leader[x];
    const int g = l < 0 ? -1 : a.newidx[l];
    a.colsrc[x] = g;
    if (l == x) a.cursor[g] = x;  // cursor is free after the scatter: first_old
  }
  if (tid < 4) a.colsrc[M + tid] = -1;  // padding for 16-byte colmap loads
}

// Fused merge + compaction + row min (complete linkage, X7):
//   Dn[c][t] = max over old rows r in group c and old columns s in group t of
//   D[r][s];  keyn[c] = min_{t != c} (Dn[c][t] bits, t).
// One CTA builds one new row in a shared-memory window: it streams the old
// row(s) of group c with coalesced loads, maps every old column s to its new
// column t = colmap[s], and folds the value in with a shared-memory integer
// atomicMax (d >= 0, so int order == float order).  The window is then written
// out with coalesced stores and scanned for the row min.  Rows wider than the
// window are done in several windows; a window starting at new column T0 only
// needs old columns >= first_old[T0] (members of later groups are never
// smaller than their leader).

// VEC: 16-byte loads of 4 consecutive old columns (old row stride and base are
// multiples of 4 floats: every compacted matrix; the original rows when N % 4
// == 0); colmap is padded with -1 to a multiple of 4.
// Old rows are addressed through a row source: the local matrix, or (row-
// sharded build, dist.cu) the shard of the rank owning the row, read from peer
// memory.  New rows [c0, c1) (c1 < 0: all Mn) are written to Dn[c - c0].
struct LocalRows {
  const float *D;
  int64_t ld;
  __device__ __forceinline__ const float *row(int x) const { return D + (int64_t)x * ld; }
};
struct PeerRows {
  const float *const *mats;  // [world] shard base of each rank (rows [q*S, (q+1)*S))
  int S;
  int64_t ld;
  __device__ __forceinline__ const float *row(int x) const {
    const int q = x / S;
    return mats[q] + (int64_t)(x - q * S) * ld;
  }
};

template <bool VEC, int NTH, typename RS>
__global__ void __launch_bounds__(NTH) k_merge_rows(RS rs, int M, const int *__restrict__ Mn_p,
                                                    const int *__restrict__ goff,
                                                    const int *__restrict__ gmem,
                                                    const int *__restrict__ colmap,
                                                    const int *__restrict__ first_old, int W, int c0, int c1,
                                                    float *__restrict__ Dn, u64 *__restrict__ keyn) {
  extern __shared__ __align__(16) int win[];  // [W] float bits (d >= 0: int order == float order)
  __shared__ u64 wmin[NTH / 32];
  const int Mn = *Mn_p;
  const int cend = c1 < 0 ? Mn : c1;
  const int64_t ldn = (Mn + 3) & ~3;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  for (int c = c0 + blockIdx.x; c < cend; c += gridDim.x) {
    const int rb = goff[c], re = goff[c + 1];
    const float *__restrict__ row0 = rs.row(gmem[rb]);
    int bval = 0x7fffffff, bidx = 0x7fffffff;  // running (value bits, column) minimum
    for (int T0 = 0; T0 < Mn; T0 += W) {
      const int Wn = min(W, Mn - T0);
      for (int i = tid * 4; i < Wn; i += NTH * 4) *reinterpret_cast<int4 *>(win + i) = int4{0, 0, 0, 0};
      __syncthreads();
      const int s0 = T0 == 0 ? 0 : (first_old[T0] & ~3);
      if (VEC) {
        const float4 *__restrict__ r4 = reinterpret_cast<const float4 *>(row0);
        const int4 *__restrict__ c4 = reinterpret_cast<const int4 *>(colmap);
        constexpr int UV = 4;
        for (int qb = (s0 >> 2) + tid; qb * 4 < M; qb += NTH * UV) {
          int4 t4[UV];
          float4 v4[UV];
#pragma unroll
          for (int u = 0; u < UV; ++u) {
            const int q = qb + u * NTH;
            const bool ok = q * 4 < M;
            t4[u] = ok ? __ldg(c4 + q) : int4{-1, -1, -1, -1};
            v4[u] = ok ? __ldcs(r4 + q) : float4{0, 0, 0, 0};
          }
          for (int rr = rb + 1; rr < re; ++rr) {  // other row members (max)
            const float4 *__restrict__ k4 = reinterpret_cast<const float4 *>(rs.row(gmem[rr]));
#pragma unroll
            for (int u = 0; u < UV; ++u) {
              const int q = qb + u * NTH;
              if (q * 4 < M) {
                const float4 x = __ldcs(k4 + q);
                v4[u].x = fmaxf(v4[u].x, x.x);
                v4[u].y = fmaxf(v4[u].y, x.y);
                v4[u].z = fmaxf(v4[u].z, x.z);
                v4[u].w = fmaxf(v4[u].w, x.w);
              }
            }
          }
#pragma unroll
          for (int u = 0; u < UV; ++u) {
            const int tt[4] = {t4[u].x - T0, t4[u].y - T0, t4[u].z - T0, t4[u].w - T0};
            const float vv[4] = {v4[u].x, v4[u].y, v4[u].z, v4[u].w};
#pragma unroll
            for (int k = 0; k < 4; ++k)
              if ((unsigned)tt[k] < (unsigned)Wn) atomicMax(win + tt[k], __float_as_int(vv[k]));
          }
        }
      } else {
        constexpr int U = 4;
        for (int sb = s0; sb < M; sb += U * NTH) {
          int t[U];
          float v[U];
#pragma unroll
          for (int u = 0; u < U; ++u) {
            const int s = sb + u * NTH + tid;
            t[u] = s < M ? __ldg(colmap + s) - T0 : -1;
            v[u] = s < M ? __ldcs(row0 + s) : 0.0f;
          }
          for (int rr = rb + 1; rr < re; ++rr) {
            const float *rowk = rs.row(gmem[rr]);
#pragma unroll
            for (int u = 0; u < U; ++u) {
              const int s = sb + u * NTH + tid;
              if (s < M) v[u] = fmaxf(v[u], __ldcs(rowk + s));
            }
          }
#pragma unroll
          for (int u = 0; u < U; ++u)
            if ((unsigned)t[u] < (unsigned)Wn) atomicMax(win + t[u], __float_as_int(v[u]));
        }
      }
      __syncthreads();
      // write out (16-byte stores; the new leading dimension is a multiple of 4)
      float4 *__restrict__ out4 = reinterpret_cast<float4 *>(Dn + (int64_t)(c - c0) * ldn + T0);
      const int cd = c - T0;  // diagonal position inside the window
      for (int i = tid * 4; i < Wn; i += NTH * 4) {
        int4 q = *reinterpret_cast<const int4 *>(win + i);
        // diagonal -> 0 in the matrix, excluded from the row minimum
        const int4 qm = {(i == cd || i >= Wn) ? 0x7fffffff : q.x,
                         (i + 1 == cd || i + 1 >= Wn) ? 0x7fffffff : q.y,
                         (i + 2 == cd || i + 2 >= Wn) ? 0x7fffffff : q.z,
                         (i + 3 == cd || i + 3 >= Wn) ? 0x7fffffff : q.w};
        if ((unsigned)(cd - i) < 4u) {
          q.x = i == cd ? 0 : q.x;
          q.y = i + 1 == cd ? 0 : q.y;
          q.z = i + 2 == cd ? 0 : q.z;
          q.w = i + 3 == cd ? 0 : q.w;
        }
        __stcs(out4 + (i >> 2), make_float4(__int_as_float(q.x), __int_as_float(q.y),
                                            __int_as_float(q.z), __int_as_float(q.w)));
        const int m4 = min(min(qm.x, qm.y), min(qm.z, qm.w));
        if (m4 < bval) {  // strict: the earliest column wins among equal values (X8)
          bval = m4;
          bidx = T0 + i + (qm.x == m4 ? 0 : qm.y == m4 ? 1 : qm.z == m4 ? 2 : 3);
        }
      }
      __syncthreads();
    }
    u64 best = bval == 0x7fffffff ? ~0ull : (((u64)(unsigned)bval << 32) | (unsigned)bidx);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const u64 y = __shfl_xor_sync(0xffffffffu, best, o);
      best = y < best ? y : best;
    }
    if (lane == 0) wmin[w] = best;
    __syncthreads();
    if (tid == 0) {
      u64 b = wmin[0];
#pragma unroll
      for (int i = 1; i < NTH / 32; ++i) b = wmin[i] < b ? wmin[i] : b;
      keyn[c] = b;
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// In-place rounds.  When a round merges few clusters, rewriting the whole
// compacted matrix costs (M^2 + Mn^2) floats while only the merged rows and
// columns change.  Then the matrix keeps its size: rows merged away get the
// key kDead and a cleared bit in the alive mask, the surviving (smallest)
// member of each group gets the merged row, its column is rewritten from that
// row (the matrix is symmetric), and only rows whose nearest neighbour was in
// a merged group are rescanned (any other row's nearest neighbour is unchanged:
// complete-linkage values only grow, X7, and the group keeps the smallest
// index, X8).  Column order is unchanged, so column order == rep order still.

// S0: per-row flags; multi-member groups -> mlist; members other than the
// survivor -> dead; the survivor's size.
__global__ void k_inplace_prep(PrepArgs a, int M, uint32_t *__restrict__ amask, int *__restrict__ mlist,
                               int *__restrict__ nmulti, int *__restrict__ sz, u64 *__restrict__ key) {
  for (int x = blockIdx.x * blockDim.x + threadIdx.x; x < M; x += gridDim.x * blockDim.x) {
    const int l = a.leader[x];
    uint8_t chg = 0;
    if (l >= 0) {
      const int g = a.newidx[l];
      if (a.goff[g + 1] - a.goff[g] >= 2) {
        chg = 1;
        if (x != l) {
          key[x] = kDead;
          atomicAnd(&amask[x >> 5], ~(1u << (x & 31)));
        } else {
          mlist[atomicAdd(nmulti, 1)] = g;
          sz[x] = a.sz_n[g];
        }
      }
    }
    a.alive[x] = chg;  // "in a merged group" (the level flags are free by now)
  }
}

// S1: one CTA per merged group: the survivor's new row in shared memory,
// row(L)[c] = max over members m of D[m][c]; then the entries at the other
// merged groups' survivors, row(L)[L_h] = max over x in h of row(L)[x]; the
// diagonal; write back and the row's nearest neighbour over live columns.
template <int NTH>
__global__ void __launch_bounds__(NTH, 2) k_inplace_rows(PrepArgs a, float *__restrict__ D, int64_t ld, int M,
                                                      const uint32_t *__restrict__ amask,
                                                      const int *__restrict__ mlist,
                                                      const int *__restrict__ nmulti_p, u64 *__restrict__ key) {
  extern __shared__ __align__(16) float row[];  // [M rounded up to 4]
  __shared__ u64 wmin[NTH / 32];
  const int nmulti = *nmulti_p;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int M4 = (M + 3) >> 2;
  for (int gi = blockIdx.x; gi < nmulti; gi += gridDim.x) {
    const int g = mlist[gi];
    const int rb = a.goff[g], re = a.goff[g + 1];
    const int L = a.cursor[g];  // first_old: the survivor
    for (int q = tid; q < M4; q += NTH) {
      float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
      for (int r = rb; r < re; ++r) {
        const float4 x = __ldcs(reinterpret_cast<const float4 *>(D + (int64_t)a.gmem[r] * ld) + q);
        v.x = fmaxf(v.x, x.x);
        v.y = fmaxf(v.y, x.y);
        v.z = fmaxf(v.z, x.z);
        v.w = fmaxf(v.w, x.w);
      }
      reinterpret_cast<float4 *>(row)[q] = v;
    }
    __syncthreads();
    for (int hi = tid; hi < nmulti; hi += NTH) {
      const int h = mlist[hi];
      if (h == g) continue;
      float v = 0.f;
      for (int r = a.goff[h]; r < a.goff[h + 1]; ++r) v = fmaxf(v, row[a.gmem[r]]);
      row[a.cursor[h]] = v;
    }
    __syncthreads();
    if (tid == 0) row[L] = 0.f;
    __syncthreads();
    u64 best = ~0ull;
    float4 *out = reinterpret_cast<float4 *>(D + (int64_t)L * ld);
    for (int q = tid; q < M4; q += NTH) {
      const float4 v = reinterpret_cast<const float4 *>(row)[q];
      __stcs(out + q, v);
      const float vv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int c = 4 * q + k;
        const bool live = c < M && c != L && ((amask[c >> 5] >> (c & 31)) & 1u);
        const u64 kk = ((u64)__float_as_uint(vv[k]) << 32) | (unsigned)c;
        best = (live && kk < best) ? kk : best;
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const u64 y = __shfl_xor_sync(0xffffffffu, best, o);
      best = y < best ? y : best;
    }
    if (lane == 0) wmin[w] = best;
    __syncthreads();
    if (tid == 0) {
      u64 b = wmin[0];
#pragma unroll
      for (int i = 1; i < NTH / 32; ++i) b = wmin[i] < b ? wmin[i] : b;
      key[L] = b;
    }
    __syncthreads();
  }
}

// S2: columns from rows (symmetry): D[r][L] = D[L][r] for every live row r.
// Work items = (merged group, 1024-row chunk); each thread moves 4 rows
// (coalesced loads, scattered 4-byte stores).  Few, long-lived CTAs: with one
// short CTA per item the block scheduler, not the stores, set the pace.
__global__ void __launch_bounds__(256) k_inplace_cols(PrepArgs a, float *__restrict__ D, int64_t ld, int M,
                                                      const uint32_t *__restrict__ amask,
                                                      const int *__restrict__ mlist,
                                                      const int *__restrict__ nmulti_p) {
  const int nmulti = *nmulti_p;
  const int nchunk = (M + 1023) >> 10;
  const int64_t items = (int64_t)nmulti * nchunk;
  for (int64_t it = blockIdx.x; it < items; it += gridDim.x) {
    const int gi = (int)(it / nchunk), ch = (int)(it - (int64_t)gi * nchunk);
    const int L = a.cursor[mlist[gi]];
    const float *src = D + (int64_t)L * ld;
    float v[4];
    int rr[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int r = (ch << 10) + u * 256 + (int)threadIdx.x;
      rr[u] = (r < M && ((amask[r >> 5] >> (r & 31)) & 1u)) ? r : -1;
      v[u] = rr[u] >= 0 ? __ldg(src + r) : 0.f;
    }
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (rr[u] >= 0) D[(int64_t)rr[u] * ld + L] = v[u];
  }
}

// S3a: one thread per live row r outside the merged groups whose nearest
// neighbour t was in a merged group g with survivor L: the new value d(r, L)
// (column L was rewritten by S2) is >= the old d(r, t); if equal, (d, L) is
// the new key without a scan (L <= t, every other entry is unchanged or
// larger); otherwise r goes to the rescan list.
__global__ void k_inplace_check(PrepArgs a, const float *__restrict__ D, int64_t ld, int M,
                                u64 *__restrict__ key, int *__restrict__ rlist, int *__restrict__ nres) {
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < M; r += gridDim.x * blockDim.x) {
    const u64 kr = key[r];
    if (kr == kDead || a.alive[r]) continue;  // dead, or a survivor (done in S1)
    const int t = (int)(kr & 0xffffffffu);
    if (!a.alive[t]) continue;  // neighbour not merged: unchanged
    const int Lg = a.leader[t];
    const unsigned v = __float_as_uint(D[(int64_t)r * ld + Lg]);
    if (v == (unsigned)(kr >> 32))
      key[r] = ((u64)v << 32) | (unsigned)Lg;
    else
      rlist[atomicAdd(nres, 1)] = r;
  }
}

// S3b: full rescans of the listed rows over the live columns.
template <int NTH>
__global__ void __launch_bounds__(NTH) k_inplace_rescan(const float *__restrict__ D, int64_t ld, int M,
                                                        const uint32_t *__restrict__ amask,
                                                        const int *__restrict__ rlist,
                                                        const int *__restrict__ nres_p, u64 *__restrict__ key) {
  __shared__ u64 wmin[NTH / 32];
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int M4 = (M + 3) >> 2;
  const int nres = *nres_p;
  for (int i = blockIdx.x; i < nres; i += gridDim.x) {
    const int r = rlist[i];
    u64 best = ~0ull;
    const float4 *src = reinterpret_cast<const float4 *>(D + (int64_t)r * ld);
    for (int q = tid; q < M4; q += NTH) {
      const float4 v = __ldcs(src + q);
      const float vv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int c = 4 * q + k;
        const bool live = c < M && c != r && ((amask[c >> 5] >> (c & 31)) & 1u);
        const u64 kk = ((u64)__float_as_uint(vv[k]) << 32) | (unsigned)c;
        best = (live && kk < best) ? kk : best;
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const u64 y = __shfl_xor_sync(0xffffffffu, best, o);
      best = y < best ? y : best;
    }
    if (lane == 0) wmin[w] = best;
    __syncthreads();
    if (tid == 0) {
      u64 b = wmin[0];
#pragma unroll
      for (int i2 = 1; i2 < NTH / 32; ++i2) b = wmin[i2] < b ? wmin[i2] : b;
      key[r] = b;
    }
    __syncthreads();
  }
}

__global__ void k_init_state(int *rep, int *sz, int64_t N) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < N) {
    rep[i] = (int)i;
    sz[i] = 1;
  }
}

}  // namespace
}  // namespace ragb
