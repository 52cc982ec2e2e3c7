// a5 kernels shared by the single-GPU linkage (linkage.cu) and the
// row-sharded build (dist.cu).  See linkage.cu for the algorithm.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <utility>

#include "device_util.cuh"
#include "internal.h"

namespace ragb {
namespace {

typedef unsigned long long u64;
constexpr int PT = 1024;  // threads of the single-CTA round-prep kernel
constexpr u64 kDead = ~0ull;  // row key of a row merged away by an in-place round
constexpr int kInplaceMaxM = 48 * 1024;  // in-place rounds keep a whole row in shared memory
static_assert(kInplaceMaxM < (1 << 16), "in-place row minima use 32-bit (code << 16 | column) keys");

// ---------------------------------------------------------------------------
// Stored element of the linkage matrices.  float: the Eq. 1 value itself;
// uint16_t: its order-preserving code (rank among the distinct values of the
// Eq. 1 table), so that max / compare / equality on codes are
// max / compare / equality on the values (complete linkage only takes max and
// compares, X7).  Both are handled as unsigned "bits": d >= 0, so the float's
// bit pattern orders like the float.  A 16-byte vector holds VW elements.
template <typename T>
struct Elem;
template <>
struct Elem<float> {
  static constexpr int VW = 4;
  __device__ __forceinline__ static unsigned bits(float v) { return __float_as_uint(v); }
  __device__ __forceinline__ static float make(unsigned b) { return __uint_as_float(b); }
  __device__ __forceinline__ static unsigned vmax(unsigned a, unsigned b) { return max(a, b); }
  __device__ __forceinline__ static void unpack(const uint4 &v, unsigned (&o)[VW]) {
    o[0] = v.x;
    o[1] = v.y;
    o[2] = v.z;
    o[3] = v.w;
  }
  __device__ __forceinline__ static uint4 pack(const unsigned (&o)[VW]) { return make_uint4(o[0], o[1], o[2], o[3]); }
};
template <>
struct Elem<uint16_t> {
  static constexpr int VW = 8;
  __device__ __forceinline__ static unsigned bits(uint16_t v) { return v; }
  __device__ __forceinline__ static uint16_t make(unsigned b) { return (uint16_t)b; }
  __device__ __forceinline__ static unsigned vmax(unsigned a, unsigned b) { return __vmaxu2(a, b); }
  __device__ __forceinline__ static void unpack(const uint4 &v, unsigned (&o)[VW]) {
    const unsigned w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      o[2 * k] = w[k] & 0xffffu;
      o[2 * k + 1] = w[k] >> 16;
    }
  }
  __device__ __forceinline__ static uint4 pack(const unsigned (&o)[VW]) {
    return make_uint4(o[0] | (o[1] << 16), o[2] | (o[3] << 16), o[4] | (o[5] << 16), o[6] | (o[7] << 16));
  }
};
template <typename T>
__device__ __forceinline__ uint4 vmax4(const uint4 &a, const uint4 &b) {
  return make_uint4(Elem<T>::vmax(a.x, b.x), Elem<T>::vmax(a.y, b.y), Elem<T>::vmax(a.z, b.z),
                    Elem<T>::vmax(a.w, b.w));
}

struct PrepArgs {
  const void *D;  // current matrix (float or uint16_t codes, see Elem)
  int64_t ld;
  const float *vals;  // code -> Eq. 1 value (uint16_t matrices), or nullptr (float matrices)
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
  int2 *pmap;  // [Mn + 8] new column -> (leader, other member of a pair | -1 singleton | -2 larger), or nullptr
               // (when pm32_fits: the same buffer holds the compact map pm32 and the clique list, see k_compact_maps)
  int *nclq;   // groups of 3+ members listed after pm32 (compact map only)
  int *lpos;   // [M] level position of each level column (where alive is set), or nullptr (k_prep_list)
  int *level;  // [0] level list length, [1] h bits
  int *cstat;  // clique diagnostics: starts, batches, picks, candidates, level n, clk/1k (warp0, pass)
  int *sweep_ctl;  // level-clique sweep with helper CTAs: published block count (0 between launches), or nullptr
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

// Exclusive scan of get(i), i in [0, n), by the 1024-thread block: put(i,
// prefix) for every i; returns the total.  A thread owns SE consecutive
// elements per pass (SE x fewer block scans than one element per thread).
#ifndef RAGB_SCAN_SE
#define RAGB_SCAN_SE 8
#endif
constexpr int SE = RAGB_SCAN_SE;
#ifndef RAGB_SCAN_BLOCKED
// Striped form: warp w takes SE rows of 32 consecutive elements per pass
// ([c0 + 32 SE w, c0 + 32 SE (w + 1))), lane l element 32 e + l of its
// rows — coalesced get/put — with one shuffle scan per row and one block
// scan of the warp totals per pass.  (The blocked form below — a thread owns
// SE consecutive elements — strided every warp access over 8 lines: C4
// linkage 33.5 -> 32.9 ms with the striped form.)
template <typename Get, typename Put>
__device__ int block_scan_all(int n, Get get, Put put, BlockScratch &S) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int base = 0;
  for (int c0 = 0; c0 < n; c0 += PT * SE) {
    const int wb = c0 + w * 32 * SE + lane;
    int v[SE], ex[SE];
#pragma unroll
    for (int e = 0; e < SE; ++e) v[e] = wb + 32 * e < n ? get(wb + 32 * e) : 0;
    int wsum = 0;  // warp total of the rows so far (uniform)
#pragma unroll
    for (int e = 0; e < SE; ++e) {
      int x = v[e];
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
      }
      ex[e] = wsum + x - v[e];
      wsum += __shfl_sync(0xffffffffu, x, 31);
    }
    if (lane == 0) S.w[w] = wsum;
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
    const int pre = base + (w == 0 ? 0 : S.w[w - 1]);
    const int tot = S.w[31];
    __syncthreads();
#pragma unroll
    for (int e = 0; e < SE; ++e)
      if (wb + 32 * e < n) put(wb + 32 * e, pre + ex[e]);
    base += tot;
  }
  __syncthreads();
  return base;
}
#else
template <typename Get, typename Put>
__device__ int block_scan_all(int n, Get get, Put put, BlockScratch &S) {
  int base = 0;
  for (int c0 = 0; c0 < n; c0 += PT * SE) {
    const int i0 = c0 + (int)threadIdx.x * SE;
    int v[SE], sum = 0;
#pragma unroll
    for (int e = 0; e < SE; ++e) {
      v[e] = i0 + e < n ? get(i0 + e) : 0;
      sum += v[e];
    }
    int tot;
    int pre = base + block_scan1024(sum, S, &tot);
#pragma unroll
    for (int e = 0; e < SE; ++e) {
      if (i0 + e < n) put(i0 + e, pre);
      pre += v[e];
    }
    base += tot;
  }
  __syncthreads();
  return base;
}
#endif

// Order-preserving compaction: out[...] = value(i) for i in [0, n) with pred(i).
template <typename Pred, typename Val>
__device__ int block_compact(int n, Pred pred, Val value, int *out, BlockScratch &S) {
  return block_scan_all(
      n, [&](int i) { return pred(i) ? 1 : 0; },
      [&](int i, int pre) {
        if (pred(i)) out[pre] = value(i);
      },
      S);
}

// Round step 1: h = min row key (grid, atomicMin on level[1], preset to
// ~0); RNN pairs above h (grid, emitted); the vertices whose row min equals h
// become the level list (one CTA, ascending).  Only the scans run in one CTA;
// the per-row work with dependent loads and atomics is spread over the grid.
__global__ void k_prep_min(PrepArgs a) {
  pdl_wait();
  unsigned hl = 0xffffffffu;
  for (int x = blockIdx.x * blockDim.x + threadIdx.x; x < a.M; x += gridDim.x * blockDim.x)
    hl = min(hl, (unsigned)(a.key[x] >> 32));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) hl = min(hl, __shfl_xor_sync(0xffffffffu, hl, o));
  if ((threadIdx.x & 31) == 0 && hl != 0xffffffffu) atomicMin(reinterpret_cast<unsigned *>(a.level + 1), hl);
}

__global__ void k_prep_rnn(PrepArgs a) {
  pdl_wait();
  const unsigned h = (unsigned)a.level[1];
  for (int x = blockIdx.x * blockDim.x + threadIdx.x; x < a.M; x += gridDim.x * blockDim.x) {
    const u64 kx = a.key[x];
    const unsigned hx = (unsigned)(kx >> 32);
    const int y = (int)(kx & 0xffffffffu);
    const bool dead = kx == kDead;  // row merged away by an in-place round
    int lead = dead ? -1 : x;
    a.alive[x] = (!dead && hx == h) ? 1 : 0;
    if (!dead && hx > h && (int)(a.key[y] & 0xffffffffu) == x) {
      if (y < x) {
        lead = y;
      } else {  // emission order within the round is arbitrary: the host replays each round sorted by key
        const int pos = atomicAdd(a.zcount, 1);
        a.za[pos] = a.rep[x];
        a.zb[pos] = a.rep[y];
        a.zh[pos] = a.vals ? a.vals[hx] : __uint_as_float(hx);
        a.zs[pos] = a.sz[x] + a.sz[y];
      }
    }
    a.leader[x] = lead;
  }
}

__global__ void __launch_bounds__(PT, 1) k_prep_list(PrepArgs a) {
  pdl_wait();
  __shared__ BlockScratch S;
  const uint8_t *alive = a.alive;
  int *lpos = a.lpos;
  const int nlist = block_scan_all(
      a.M, [&](int i) { return alive[i] != 0 ? 1 : 0; },
      [&](int i, int pre) {
        if (alive[i] != 0) {
          a.list[pre] = i;
          if (lpos) lpos[i] = pre;  // valid where alive (the level flag) is set
        }
      },
      S);
  if (threadIdx.x == 0) a.level[0] = nlist;
}

// Side buffer of the in-place rounds (code mode).  Rewriting the merged
// survivors' columns in place costs one scattered 2-byte store per row and
// merge (most of an in-place round).  Instead a survivor's column becomes
// "dirty": its values are appended, transposed, to a row-major buffer
// T[r][slot] (one coalesced segment per row for the round's survivors), and
// the readers of the matrix take a dirty column's value from T:
//   val(r, c) = dirty(c) ? T[r][tslot[c]] : D[r][c].
// Merged rows are still rewritten in place (D part), together with their T
// row.  Before the next compaction the buffer is flushed into the matrix
// row by row (k_side_flush).
struct SideBuf {
  uint16_t *T;      // [M][cap] dirty-column values, or nullptr (no side buffer)
  int cap;          // slots per row (multiple of 8)
  int *tcol;        // [cap] column of slot k, -1 retired
  int *tslot;       // [M] slot of column c, -1 clean
  uint32_t *dmask;  // [M/32 + 1] dirty-column bits
  int *nt;          // slots in use
};
__device__ __forceinline__ bool sb_dirty(const SideBuf &sb, int c) { return (sb.dmask[c >> 5] >> (c & 31)) & 1u; }

// Second-nearest cache of the in-place rounds.  A full rescan of row r in
// round R also records its second-smallest key k2 = (value, column).  Every
// other column's key exceeded k2 at the scan.  Values only grow (complete
// linkage), and a cluster merged since from such columns (not k2's) keeps a
// key above k2: its value is the max of its members' (>= k2's value), and if
// equal to k2's, every member had k2's value and a larger column, so does
// the cluster's smallest member, its index.  So as long as k2's column has
// not merged since (ver[c] <= R), when the nearest neighbour merges into L
// with a larger value the new key is min((d(r, L), L), k2) without a rescan
// (hub clusters, the nearest neighbour of thousands of rows, merge
// repeatedly in C4's late in-place rounds).  One use per scan.
struct NNCache {
  u64 *key2;   // [M] second-smallest key of the last full scan, or nullptr (disabled)
  int *kround; // [M] round of that scan (0: no usable entry)
  int *ver;    // [M] round in which column c last merged (as survivor or member)
  int round;   // this round (>= 1)
};

// Round step 2, row form (single GPU): one CTA per level row i streams the
// whole matrix row list[i] (16-byte loads) and sets bit lpos[c] of its
// adjacency row for every column c holding h.  Every such column is a level
// vertex (its row minimum is <= h, the global minimum); columns outside the
// level (rows merged away by in-place rounds hold stale values) are skipped.
template <typename T, bool VEC>
__global__ void __launch_bounds__(256) k_level_adj_rows(PrepArgs a, uint32_t *__restrict__ adj, SideBuf sb) {
  pdl_wait();
  // [W] this row's adjacency bits, then the level's column mask [MW] and its
  // per-word exclusive popcount prefix [MW]: a column's level position is
  // lpre[c / 32] + popc(lmask[c / 32] below c) — no global lookups per match
  extern __shared__ uint32_t wbits[];
  __shared__ int wsum[8];
  const int n = a.level[0];
  if (n < 2 || (int)blockIdx.x >= n) return;
  typedef Elem<T> E;
  constexpr int VW = E::VW;
  const unsigned hb = (unsigned)a.level[1];
  const T *D = static_cast<const T *>(a.D);
  const int W = (n + 31) >> 5, M = a.M, MW = (M + 31) >> 5;
  uint32_t *lmask = wbits + MW;  // (wbits is sized for any level of this matrix: MW words)
  uint32_t *lpre = lmask + MW;
  const uint8_t *__restrict__ lev = a.alive;  // level flags (k_prep_rnn)
  for (int w = threadIdx.x; w < MW; w += blockDim.x) {
    const uint32_t *l4 = reinterpret_cast<const uint32_t *>(lev + 32 * w);
    uint32_t m = 0u;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const uint32_t x = 32 * w + 4 * q < M ? __ldg(l4 + q) : 0u;
#pragma unroll
      for (int b = 0; b < 4; ++b) m |= (((x >> (8 * b)) & 0xffu) != 0u ? 1u : 0u) << (4 * q + b);
    }
    if (32 * w + 32 > M) m &= (1u << (M - 32 * w)) - 1u;
    lmask[w] = m;
  }
  __syncthreads();
  {
    const int per = (MW + (int)blockDim.x - 1) / (int)blockDim.x;
    const int w0 = min(MW, (int)threadIdx.x * per), w1 = min(MW, w0 + per);
    int cnt = 0;
    for (int w = w0; w < w1; ++w) cnt += __popc(lmask[w]);
    int pre = block_excl_scan<256>(cnt, wsum);
    for (int w = w0; w < w1; ++w) {
      lpre[w] = (uint32_t)pre;
      pre += __popc(lmask[w]);
    }
  }
  __syncthreads();
  const int *__restrict__ lpos = a.lpos;  // (dirty columns and the scalar path)
  for (int i = blockIdx.x; i < n; i += gridDim.x) {
    for (int w = threadIdx.x; w < W; w += blockDim.x) wbits[w] = 0u;
    __syncthreads();
    const int r = a.list[i];
    const T *row = D + (int64_t)r * a.ld;
    if (VEC) {
      const uint4 *row4 = reinterpret_cast<const uint4 *>(row);
      for (int q = threadIdx.x; q * VW < M; q += blockDim.x) {
        unsigned v[VW];
        E::unpack(__ldcs(row4 + q), v);  // (rows read once: evict-first, the adjacency stays in L2)
        const int c0 = q * VW;  // VW columns in one mask word
        const uint32_t mw = lmask[c0 >> 5];
        const uint32_t below = mw & ((1u << (c0 & 31)) - 1u);
        const uint32_t mb = (mw >> (c0 & 31)) & ((1u << VW) - 1u);
        if (mb == 0u) continue;
        // dirty columns (side buffer) hold stale values here: taken from T below
        const uint32_t clean = sb.T ? ~(sb.dmask[c0 >> 5] >> (c0 & 31)) : ~0u;
        const int base = (int)lpre[c0 >> 5] + __popc(below);
        // the vector's matches land in level positions [base, base + VW): at
        // most two adjacency words, one shared atomic each (not one per match)
        const int wj = base >> 5, sh = base & 31;
        uint32_t lo = 0u, hi = 0u;
#pragma unroll
        for (int k = 0; k < VW; ++k) {
          const int c = c0 + k;
          if (((mb & clean) >> k & 1u) && v[k] == hb && c != r) {
            const int b = sh + __popc(mb & ((1u << k) - 1u));  // < 32 + VW
            if (b < 32) lo |= 1u << b;
            else hi |= 1u << (b - 32);
          }
        }
        if (lo) atomicOr(&wbits[wj], lo);
        if (hi) atomicOr(&wbits[wj + 1], hi);
      }
      if (sb.T) {  // dirty columns from the side buffer
        const int nt = *sb.nt;
        for (int k = threadIdx.x; k < nt; k += blockDim.x) {
          const int c = sb.tcol[k];
          if (c < 0 || c == r || (unsigned)sb.T[(int64_t)r * sb.cap + k] != hb || !lev[c]) continue;
          const int j = lpos[c];
          atomicOr(&wbits[j >> 5], 1u << (j & 31));
        }
      }
    } else {
      for (int c = threadIdx.x; c < M; c += blockDim.x)
        if (E::bits(__ldg(row + c)) == hb && c != r && lev[c]) {
          const int j = lpos[c];
          atomicOr(&wbits[j >> 5], 1u << (j & 31));
        }
    }
    __syncthreads();
    for (int w = threadIdx.x; w < W; w += blockDim.x) adj[(int64_t)i * W + w] = wbits[w];
    __syncthreads();
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
      __syncwarp();  // every lane is done reading the previous batch's s_p (racecheck)
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
// Levels above 128 vertices go to the block sweep with helper CTAs: measured
// faster than the single warp's 32-candidate batches from n = 128 up (C4's
// top levels of 500-2000 vertices: 0.30-0.48 -> 0.16-0.22 ms per level; a
// tie-heavy N = 20k, K = 4 build 11.4 -> 7.4 ms of linkage).  The warp path
// for 1024 < n <= 4096 (cliques_warp<4>) stays selectable with
// -DRAGB_WARP_CLIQUE_MAX=4096 (the round-1 threshold).
#ifndef RAGB_WARP_CLIQUE_MAX
#define RAGB_WARP_CLIQUE_MAX 128
#endif
constexpr int kWarpCliqueMaxN = RAGB_WARP_CLIQUE_MAX;

constexpr int CT = 512;  // threads of k_level_cliques (128 registers for the pick chain)

// Levels of more than kWarpCliqueMaxN vertices (C4's h = 1.0 level: 16,082
// vertices, ~2,150 cliques, 13,927 merges): the greedy clique sequence as a
// sweep over the vertices.  Reformulation: in the greedy
// process a vertex v is offered to the cliques in creation order and joins
// the first one whose members (all smaller than v) are all adjacent to it;
// if none takes it, v starts the next clique.  Clique j's candidate set
// I_j = AND of its members' adjacency rows is kept, for the words after the
// current block, in global memory (reductions with AND); a block of 128
// vertices is decided by one warp from the candidate masks of the cliques
// that have candidates in it (a chain per clique: the smallest undecided
// candidate, then the smallest one adjacent to it, ...), then new cliques
// start among the vertices still undecided.  The decisions are emitted in
// greedy order (clique, then vertex) by a counting sort.
constexpr int kSweepB = 128;      // vertices per block (4 words)
constexpr int kSweepCap = 1024;   // cliques with candidates examined per pass
constexpr int kSweepHelpers = 32; // helper CTAs of the sweep (candidate-set updates)

__device__ __forceinline__ uint4 and4(uint4 x, uint4 y) { return make_uint4(x.x & y.x, x.y & y.y, x.z & y.z, x.w & y.w); }
__device__ __forceinline__ bool any4(uint4 x) { return (x.x | x.y | x.z | x.w) != 0u; }
__device__ __forceinline__ int ffs4(uint4 x) {  // first set bit (0..127), x != 0
  return x.x ? __ffs(x.x) - 1 : x.y ? 31 + __ffs(x.y) : x.z ? 63 + __ffs(x.z) : 95 + __ffs(x.w);
}
__device__ __forceinline__ uint4 above4(int p) {  // bits > p of a 128-bit mask
  const uint32_t m[4] = {p < 0 ? ~0u : (p < 31 ? ~0u << (p + 1) : 0u),
                         p < 32 ? ~0u : (p < 63 ? ~0u << (p - 31) : 0u),
                         p < 64 ? ~0u : (p < 95 ? ~0u << (p - 63) : 0u),
                         p < 96 ? ~0u : (p < 127 ? ~0u << (p - 95) : 0u)};
  return make_uint4(m[0], m[1], m[2], m[3]);
}
// x - 1 over 128 bits (carry chain): x & (x - 1) drops the lowest set bit.
// In a pick chain the candidate set has no bits below its lowest pick p, so
// "the candidates above p" is the set minus its lowest bit, and the picked
// bit itself is x ^ (x & (x - 1)).
__device__ __forceinline__ uint4 dec128(uint4 x) {
  uint4 r;
  asm("sub.cc.u32 %0, %4, 1;\n\tsubc.cc.u32 %1, %5, 0;\n\tsubc.cc.u32 %2, %6, 0;\n\tsubc.u32 %3, %7, 0;"
      : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
      : "r"(x.x), "r"(x.y), "r"(x.z), "r"(x.w));
  return r;
}
// the chain step after picking p = ffs4(c): u loses p, c becomes the
// candidates above p adjacent to p
__device__ __forceinline__ void chain_step(uint4 &c, uint4 &u, const uint4 &adjp) {
  const uint4 cl = and4(c, dec128(c));
  u = make_uint4(u.x & ~(c.x ^ cl.x), u.y & ~(c.y ^ cl.y), u.z & ~(c.z ^ cl.z), u.w & ~(c.w ^ cl.w));
  c = and4(cl, adjp);
}
__device__ __forceinline__ uint4 clear4(uint4 x, int p) {
  const uint32_t b = ~(1u << (p & 31));
  const int q = p >> 5;
  return make_uint4(q == 0 ? x.x & b : x.x, q == 1 ? x.y & b : x.y, q == 2 ? x.z & b : x.z, q == 3 ? x.w & b : x.w);
}

// Eager candidate-set update of block v0's decisions (s_bj / s_bv, nb of them;
// starts marked 0x10000) for the words [w0, w1): a new clique's set is its
// start's row ANDed with its members in the block (one store per word), an
// existing clique's set is ANDed with each new member's row (reductions).
// Work items (decision, 128-word chunk) over nwarps warps, 4 words per lane.
__device__ __forceinline__ void sweep_update(const uint32_t *__restrict__ adj, int W, uint32_t *I, int WI, int v0,
                                             const int *bj, const int *bv, int nb, int w0, int w1, int gw,
                                             int nwarps, int lane) {
  const int nch = (w1 - w0 + 127) / 128;
  for (int it = gw; it < nb * nch; it += nwarps) {
    const int t = it / nch, w = w0 + (it - t * nch) * 128 + 4 * lane;
    const int j = bj[t], v = bv[t];
    uint32_t *dst = I + (size_t)j * WI;
    if (v & 0x10000) {  // new clique: start row AND its members that follow it in the block
      uint32_t x[4];
      const uint32_t *src = adj + (size_t)(v0 + (v & 0xffff)) * W;
#pragma unroll
      for (int q = 0; q < 4; ++q) x[q] = w + q < w1 ? __ldg(src + w + q) : 0u;
      for (int t2 = t + 1; t2 < nb && bj[t2] == j && !(bv[t2] & 0x10000); ++t2) {
        const uint32_t *m = adj + (size_t)(v0 + bv[t2]) * W;
#pragma unroll
        for (int q = 0; q < 4; ++q) x[q] &= w + q < w1 ? __ldg(m + w + q) : 0u;
      }
#pragma unroll
      for (int q = 0; q < 4; ++q)
        if (w + q < w1) dst[w + q] = x[q];
    } else {
      // a member of an existing clique (a member of a new one is folded into its start's item)
      bool fresh = false;
      for (int t2 = t - 1; t2 >= 0 && bj[t2] == j; --t2) fresh |= (bv[t2] & 0x10000) != 0;
      if (fresh) continue;
      const uint32_t *src = adj + (size_t)(v0 + v) * W;
      uint32_t x[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) x[q] = w + q < w1 ? __ldg(src + w + q) : 0xffffffffu;
#pragma unroll
      for (int q = 0; q < 4; ++q)
        if (x[q] != 0xffffffffu) atomicAnd(dst + w + q, x[q]);
    }
  }
}

// Helper CTAs of the sweep (blockIdx.x >= 1): block b's decisions, once CTA 0
// has published them, applied to the candidate-set words after block b + 1.
__device__ void sweep_helper(const PrepArgs &a, const uint32_t *__restrict__ adj, int n, int W) {
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int WI = (W + 3) & ~3;
  uint32_t *I = const_cast<uint32_t *>(adj) + (((size_t)n * W + 3) & ~(size_t)3);
  int *ccnt = reinterpret_cast<int *>(I + (size_t)n * WI) + 4 * n;
  const int nblk = (n + kSweepB - 1) / kSweepB;
  const int2 *logb = reinterpret_cast<const int2 *>(ccnt + ((n + 2) & ~1));
  const int *logn = reinterpret_cast<const int *>(logb + (size_t)nblk * kSweepB);
  int *hcnt = const_cast<int *>(logn) + nblk;
  __shared__ int s_bj2[kSweepB], s_bv2[kSweepB];
  __shared__ int s_nb2;
  const int nhelp = (int)gridDim.x - 1, h = (int)blockIdx.x - 1;
  for (int b = 0; b < nblk; ++b) {
    if (tid == 0) {
      const volatile int *pub = a.sweep_ctl;
      while (*pub <= b) __nanosleep(128);
      __threadfence();
      s_nb2 = __ldcg(logn + b);
    }
    __syncthreads();
    const int nb = s_nb2;
    for (int t = tid; t < nb; t += CT) {
      const int2 e = __ldcg(logb + (size_t)b * kSweepB + t);
      s_bj2[t] = e.x;
      s_bv2[t] = e.y;
    }
    __syncthreads();
    const int w0 = (b * kSweepB >> 5) + 8;  // after block b + 1 (CTA 0 writes that one)
    if (w0 < W) sweep_update(adj, W, I, WI, b * kSweepB, s_bj2, s_bv2, nb, w0, W, h * (CT / 32) + wid, nhelp * (CT / 32), lane);
    __threadfence();
    __syncthreads();
    if (tid == 0) {
      atomicAdd(hcnt + b, 1);
      // every helper finishes block b before any starts b + 1 (a new clique's
      // stores of block b come before reductions of block b + 1 on its words)
      const volatile int *c = hcnt + b;
      while (*c < nhelp) __nanosleep(64);
      __threadfence();
    }
    __syncthreads();
  }
}

// Returns the number of merges; seq / seqs (greedy order) as the other paths.
__device__ int cliques_sweep(const PrepArgs &a, const uint32_t *__restrict__ adj, int n, int W, int *seq, int *seqs) {
  __shared__ uint4 s_adjB[kSweepB];    // block adjacency: row v0 + i, words [wb, wb + 4)
  __shared__ uint4 s_lm[kSweepCap];    // candidate masks of the listed cliques
  __shared__ int s_lj[kSweepCap];      // their clique ids (ascending)
  __shared__ int s_bj[kSweepB], s_bv[kSweepB];  // this block's decisions (clique, vertex), new starts marked
  __shared__ int s_wcnt[CT / 32];
  __shared__ int s_J, s_nd, s_nb, s_nl, s_done;
  __shared__ uint4 s_und;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  // work area after the adjacency (n x W words): I [n][W], then per-decision and per-clique arrays
  const int WI = (W + 3) & ~3;  // I row stride: 16-byte rows (4-word block loads)
  uint32_t *I = const_cast<uint32_t *>(adj) + (((size_t)n * W + 3) & ~(size_t)3);
  int *dec_j = reinterpret_cast<int *>(I + (size_t)n * WI);  // [n] clique of decision d (sweep order)
  int *dec_v = dec_j + n;                                    // [n] its vertex
  int *dec_r = dec_v + n;                                    // [n] rank within the clique
  int *cstart = dec_r + n;                                   // [n] start vertex of clique j
  int *ccnt = cstart + n;                                    // [n + 1] merges per clique, then offsets
  const int nblk = (n + kSweepB - 1) / kSweepB;
  int2 *logb = reinterpret_cast<int2 *>(ccnt + ((n + 2) & ~1));  // [nblk][kSweepB] decisions of block b (helpers)
  int *logn = reinterpret_cast<int *>(logb + (size_t)nblk * kSweepB);  // [nblk] their count
  int *hcnt = logn + nblk;                                   // [nblk] helpers done with block b
  const bool helpers = a.sweep_ctl != nullptr && gridDim.x > 1;
  const int nhelp = (int)gridDim.x - 1;
  if (tid == 0) {
    s_J = 0;
    s_nd = 0;
  }
  if (helpers)
    for (int i = tid; i < nblk; i += CT) hcnt[i] = 0;
  __syncthreads();
  long long tk[6] = {0, 0, 0, 0, 0, 0};
  long long nlist = 0;
  long long c0 = clock64();
  for (int v0 = 0; v0 < n; v0 += kSweepB) {
    const int wb = v0 >> 5;
    // -- block adjacency and the undecided set ----------------------------------
    if (tid < kSweepB) {
      const int v = v0 + tid;
      uint32_t w4[4] = {0u, 0u, 0u, 0u};
      if (v < n) {
        const uint32_t *r = adj + (size_t)v * W + wb;
#pragma unroll
        for (int q = 0; q < 4; ++q) w4[q] = wb + q < W ? __ldg(r + q) : 0u;
      }
      s_adjB[tid] = make_uint4(w4[0], w4[1], w4[2], w4[3]);
    }
    if (tid == 0) {
      const int nv = min(kSweepB, n - v0);
      s_und = above4(-1);
      if (nv < kSweepB) s_und = and4(s_und, make_uint4(nv >= 32 ? ~0u : (1u << nv) - 1u, nv >= 64 ? ~0u : nv > 32 ? (1u << (nv - 32)) - 1u : 0u,
                                                       nv >= 96 ? ~0u : nv > 64 ? (1u << (nv - 64)) - 1u : 0u,
                                                       nv > 96 ? (1u << (nv - 96)) - 1u : 0u));
      s_nb = 0;
      s_done = 0;
    }
    __syncthreads();
    { const long long c1 = clock64(); tk[0] += c1 - c0; c0 = c1; }
    const int J0 = s_J;
    // -- existing cliques, in creation order, that have candidates here ---------
    for (int j0 = 0; j0 < J0 && !s_done; j0 += kSweepCap) {
      const uint4 und = s_und;
      const int j = j0 + tid * 2;  // two cliques per thread (kSweepCap = 2 x CT)
      uint4 m0 = make_uint4(0u, 0u, 0u, 0u), m1 = m0;
      if (j < J0) m0 = and4(__ldcg(reinterpret_cast<const uint4 *>(I + (size_t)j * WI + wb)), und);
      if (j + 1 < J0) m1 = and4(__ldcg(reinterpret_cast<const uint4 *>(I + (size_t)(j + 1) * WI + wb)), und);
      const int c = (any4(m0) ? 1 : 0) + (any4(m1) ? 1 : 0);
      const int pos = block_excl_scan<CT>(c, s_wcnt);
      if (any4(m0)) {
        s_lj[pos] = j;
        s_lm[pos] = m0;
      }
      if (any4(m1)) {
        s_lj[pos + (any4(m0) ? 1 : 0)] = j + 1;
        s_lm[pos + (any4(m0) ? 1 : 0)] = m1;
      }
      if (tid == CT - 1) s_nl = pos + c;
      __syncthreads();
      { const long long c1 = clock64(); tk[1] += c1 - c0; c0 = c1; }
      if (wid == 0) {  // the listed cliques take their chains, in order; 32 at a time
        nlist += s_nl;  // (diagnostics; read by warp 0 only, which alone rewrites the neighbouring s_nb)
        uint4 u = s_und;
        int nb = s_nb;
        const int nl = s_nl;
        for (int g = 0; g < nl && any4(u); g += 32) {
          const int t = g + lane;
          uint4 m = t < nl ? s_lm[t] : make_uint4(0u, 0u, 0u, 0u);
          while (true) {
            // the first clique of the group that still has an undecided candidate
            const uint32_t b = __ballot_sync(0xffffffffu, any4(and4(m, u)));
            if (b == 0u) break;
            const int L = __ffs(b) - 1;
            if (lane == L) {
              uint4 cm = and4(m, u);
              const int j = s_lj[t];
              while (any4(cm)) {
                const int p = ffs4(cm);
                s_bj[nb] = j;
                s_bv[nb] = p;
                ++nb;
                chain_step(cm, u, s_adjB[p]);
              }
            }
            u.x = __shfl_sync(0xffffffffu, u.x, L);
            u.y = __shfl_sync(0xffffffffu, u.y, L);
            u.z = __shfl_sync(0xffffffffu, u.z, L);
            u.w = __shfl_sync(0xffffffffu, u.w, L);
            nb = __shfl_sync(0xffffffffu, nb, L);
            if (lane <= L) m = make_uint4(0u, 0u, 0u, 0u);
          }
        }
        __syncwarp();  // every lane has read s_und / s_nb before lane 0 rewrites them
        if (lane == 0) {
          s_und = u;
          s_nb = nb;
          s_done = any4(u) ? 0 : 1;
        }
      }
      __syncthreads();
      { const long long c1 = clock64(); tk[2] += c1 - c0; c0 = c1; }
    }
    // -- new cliques among the vertices still undecided (decisions before s_nb
    //    join existing cliques) ----------------------------------------------------
    if (tid == 0) {
      uint4 u = s_und;
      int nb = s_nb, J = s_J;
      while (any4(u)) {
        const int p = ffs4(u);
        u = clear4(u, p);
        cstart[J] = v0 + p;
        s_bj[nb] = J;
        s_bv[nb] = p | 0x10000;  // start of clique J (not a merge)
        ++nb;
        uint4 cm = and4(u, s_adjB[p]);  // (u has no bits at or below p)
        while (any4(cm)) {
          const int q = ffs4(cm);
          s_bj[nb] = J;
          s_bv[nb] = q;
          ++nb;
          chain_step(cm, u, s_adjB[q]);
        }
        ++J;
      }
      s_J = J;
      s_nb = nb;
    }
    __syncthreads();
    { const long long c1 = clock64(); tk[3] += c1 - c0; c0 = c1; }
    const int nb = s_nb;
    // -- record the merges; eager candidate sets for the words after the block ----
    const int wn = wb + 4;  // first word after the block
    {  // decision t of the block -> global arrays, rank within its clique (a
       // clique's decisions of the block are contiguous: one chain each)
      const int nd0 = s_nd;
      const bool isd = tid < nb && !(s_bv[tid] & 0x10000);
      const int dbefore = block_excl_scan<CT>(isd ? 1 : 0, s_wcnt);  // merges before t
      int old = 0, newc = -1;
      if (tid < nb) {
        const int j = s_bj[tid];
        const bool start = (s_bv[tid] & 0x10000) != 0;
        int before = 0;
        for (int t2 = tid - 1; t2 >= 0 && s_bj[t2] == j; --t2) before += (s_bv[t2] & 0x10000) ? 0 : 1;
        const bool last = tid + 1 >= nb || s_bj[tid + 1] != j;
        const bool fresh = j >= J0;  // created in this block: no earlier merges
        old = fresh ? 0 : ccnt[j];
        if (!start) {
          const int d = nd0 + dbefore;
          dec_j[d] = j;
          dec_v[d] = v0 + s_bv[tid];
          dec_r[d] = old + before;
        }
        newc = last ? old + before + (start ? 0 : 1) : -1;
      }
      if (tid == CT - 1) s_nd = nd0 + dbefore + (isd ? 1 : 0);
      __syncthreads();  // every thread has read its clique's count before any is rewritten
      if (newc >= 0) ccnt[s_bj[tid]] = newc;
    }
    // eager candidate sets: CTA 0 updates the next block's words itself; with
    // helper CTAs, the words after it are theirs (sweep_update), lagging one
    // block behind — published through the decision log of the block
    const int wend = helpers ? min(W, wn + 4) : W;
    if (helpers && v0 >= kSweepB) {
      // the helpers are done with block b - 1: they wrote words >= wn of its
      // new cliques (plain stores this block's reductions must not precede),
      // and every word this block's listing read
      const long long cw = clock64();
      if (tid == 0) {
        const volatile int *c = hcnt + (v0 / kSweepB - 1);
        while (*c < nhelp) __nanosleep(64);
        __threadfence();
      }
      __syncthreads();
      tk[5] += clock64() - cw;
    }
    if (helpers) {
      for (int t = tid; t < nb; t += CT) logb[(size_t)(v0 / kSweepB) * kSweepB + t] = make_int2(s_bj[t], s_bv[t]);
      if (tid == 0) logn[v0 / kSweepB] = nb;
    }
    if (helpers) {
      // the next block's 4 words: one thread per decision (16-byte store of a
      // new clique's words; reductions for a member of an existing clique)
      if (tid < nb && wn < W) {
        const int j = s_bj[tid], v = s_bv[tid];
        uint32_t *dst = I + (size_t)j * WI + wn;
        if (v & 0x10000) {
          const uint32_t *src = adj + (size_t)(v0 + (v & 0xffff)) * W + wn;
          uint32_t x[4];
#pragma unroll
          for (int q = 0; q < 4; ++q) x[q] = wn + q < W ? __ldg(src + q) : 0u;
          for (int t2 = tid + 1; t2 < nb && s_bj[t2] == j; ++t2) {
            const uint32_t *m = adj + (size_t)(v0 + s_bv[t2]) * W + wn;
#pragma unroll
            for (int q = 0; q < 4; ++q) x[q] &= wn + q < W ? __ldg(m + q) : 0u;
          }
          *reinterpret_cast<uint4 *>(dst) = make_uint4(x[0], x[1], x[2], x[3]);
        } else if (j < J0) {  // members of a clique new in this block are folded into its start's store
          const uint32_t *src = adj + (size_t)(v0 + v) * W + wn;
#pragma unroll
          for (int q = 0; q < 4; ++q)
            if (wn + q < W) {
              const uint32_t xv = __ldg(src + q);
              if (xv != 0xffffffffu) atomicAnd(dst + q, xv);
            }
        }
      }
    } else if (wend > wn) {
      sweep_update(adj, W, I, WI, v0, s_bj, s_bv, nb, wn, wend, wid, CT / 32, lane);
    }
    if (helpers) {
      __threadfence();
      __syncthreads();
      if (tid == 0) atomicExch(a.sweep_ctl, v0 / kSweepB + 1);  // block published
    }
    __threadfence();  // the reductions are at L2 before the next block reads I (ld.cg)
    __syncthreads();
    { const long long c1 = clock64(); tk[4] += c1 - c0; c0 = c1; }
  }
  if (helpers && tid == 0) {  // every helper is done: the control word goes back to 0 for the next launch
    const volatile int *c = hcnt + (nblk - 1);
    while (*c < nhelp) __nanosleep(64);
    atomicExch(a.sweep_ctl, 0);
  }
  if (tid == 0 && a.cstat) {
    a.cstat[0] = s_J;
    a.cstat[1] = (int)nlist;
    a.cstat[2] = (int)(tk[0] >> 10);
    a.cstat[3] = (int)(tk[1] >> 10);
    a.cstat[5] = (int)(tk[2] >> 10);
    a.cstat[6] = (int)(tk[3] >> 10);
    a.cstat[7] = (int)(tk[4] >> 10);
    a.cstat[4] = (int)(tk[5] >> 10);  // waits for the helpers (inside tk[4])
  }
  // -- greedy order: counting sort of the decisions by clique --------------------
  const int J = s_J, nd = s_nd;
  __syncthreads();
  {
    __shared__ int s_carry;
    if (tid == 0) s_carry = 0;
    __syncthreads();
    for (int j0 = 0; j0 < J; j0 += CT) {
      const int j = j0 + tid;
      const int c = j < J ? ccnt[j] : 0;
      const int pre = block_excl_scan<CT>(c, s_wcnt);
      const int carry = s_carry;
      if (j < J) ccnt[j] = carry + pre;  // offsets
      __syncthreads();
      if (tid == CT - 1) s_carry = carry + pre + c;
      __syncthreads();
    }
  }
  for (int d = tid; d < nd; d += CT) {
    const int j = dec_j[d];
    const int pos = ccnt[j] + dec_r[d];
    seq[pos] = dec_v[d];
    seqs[pos] = cstart[j];
  }
  __syncthreads();
  return nd;
}

__global__ void __launch_bounds__(CT, 1) k_level_cliques(PrepArgs a,
                                                         const uint32_t *__restrict__ adj) {
  pdl_wait();
  extern __shared__ __align__(16) uint32_t bits[];  // staged adjacency of levels <= 1024
  __shared__ int s_p[64];     // next candidates (list positions), ascending (warp paths)
  __shared__ int s_nseq;
  __shared__ int s_sv[CT / 32], s_sf[CT / 32];
  const int n = a.level[0];
  if (n < 2) return;
  const float hf = a.vals ? a.vals[a.level[1]] : __uint_as_float((unsigned)a.level[1]);
  const int W = (n + 31) >> 5;
  if (blockIdx.x > 0) {  // helper CTAs: the sweep's candidate-set updates
    if (n > kWarpCliqueMaxN && a.sweep_ctl) sweep_helper(a, adj, n, W);
    return;
  }
  int *seq = a.candA, *seqs = a.candB;  // pick list position, its clique's start position
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  int nseq = 0;  // picks recorded (greedy order)
  if (n <= kWarpCliqueMaxN) {
    if (n <= 1024) {  // stage the adjacency (n x W <= 32K words) in shared memory
      for (int i = tid; i < n * W; i += CT) bits[i] = __ldg(adj + i);
      __syncthreads();
      if (wid == 0) nseq = cliques_warp<1>(a, bits, n, W, s_p, seq, seqs);
    } else if (wid == 0) {
      nseq = cliques_warp<4>(a, adj, n, W, s_p, seq, seqs);
    }
  } else {
    nseq = cliques_sweep(a, adj, n, W, seq, seqs);
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
  }
}

// Round step 4: order-preserving compaction map and group CSR.  Scans in one
// CTA (newidx, goff), the per-row passes over the grid.
__global__ void __launch_bounds__(PT, 1) k_compact_scan1(PrepArgs a) {
  pdl_wait();
  __shared__ BlockScratch S;
  const int M = a.M;
  // new index of every survivor (order preserving)
  const int Mn = block_scan_all(
      M, [&](int x) { return a.leader[x] == x ? 1 : 0; }, [&](int x, int pre) { a.newidx[x] = pre; }, S);
  for (int g = threadIdx.x; g < Mn; g += PT) {
    a.cnt[g] = 0;
    a.cursor[g] = 0;
    a.sz_n[g] = 0;
  }
  if (threadIdx.x == 0) {
    *a.Mn = Mn;
    if (a.nclq) *a.nclq = 0;
  }
}

__global__ void k_compact_groups(PrepArgs a) {
  pdl_wait();
  for (int x = blockIdx.x * blockDim.x + threadIdx.x; x < a.M; x += gridDim.x * blockDim.x) {
    const int l = a.leader[x];
    if (l < 0) continue;  // dead row
    const int g = a.newidx[l];
    atomicAdd(&a.cnt[g], 1);
    atomicAdd(&a.sz_n[g], a.sz[x]);
    if (l == x) a.rep_n[g] = a.rep[x];
  }
}

__global__ void __launch_bounds__(PT, 1) k_compact_scan2(PrepArgs a) {
  pdl_wait();
  __shared__ BlockScratch S;
  const int Mn = *a.Mn;
  const int live = block_scan_all(
      Mn, [&](int g) { return a.cnt[g]; }, [&](int g, int pre) { a.goff[g] = pre; }, S);
  if (threadIdx.x == 0) a.goff[Mn] = live;  // live rows (dead rows of in-place rounds are in no group)
}

__global__ void k_compact_members(PrepArgs a) {
  pdl_wait();
  for (int x = blockIdx.x * blockDim.x + threadIdx.x; x < a.M; x += gridDim.x * blockDim.x) {
    const int l = a.leader[x];
    if (l < 0) continue;
    const int g = a.newidx[l];
    a.gmem[a.goff[g] + atomicAdd(&a.cursor[g], 1)] = x;
  }
}

// Compact gather map (k_merge_gather2): new column t -> one 32-bit word
//   (x - t) | (y - t) << 15
// x = the group's leader (its smallest member), y = the other member of a
// 2-member group, else x (a singleton; or a group of 3+ members, whose other
// members are folded into x's slot before the gather — those groups are listed
// after the map).  Order-preserving compaction puts x at or after t and every
// member below M: it fits when M - Mn < 2^15 and M <= 2^17.
__host__ __device__ constexpr bool pm32_fits(int M, int Mn) { return M <= (1 << 17) && M - Mn < (1 << 15); }
// The map is padded to a multiple of 128 words (zeros); the clique list
// follows.
__host__ __device__ constexpr int pm32_words(int Mn) { return (Mn + 127) & ~127; }
__device__ __forceinline__ int pm32_index(int t) { return t; }
__device__ __forceinline__ uint32_t *pm32_of(const PrepArgs &a) { return reinterpret_cast<uint32_t *>(a.pmap); }
__device__ __forceinline__ int *clq_of(const PrepArgs &a, int Mn) {
  return reinterpret_cast<int *>(pm32_of(a) + pm32_words(Mn));
}

// old column -> new column | writer class << 29 (k_merge_rows): 0 the
// group's leader (smallest member), 1 the other member of a 2-member group,
// 2 a non-leader of a larger group; new column -> its leader (first_old,
// in cursor, free after the member scatter); pmap (or pm32) for the gather
__global__ void k_compact_maps(PrepArgs a) {
  pdl_wait();
  const int M = a.M, Mn = *a.Mn;
  const bool compact = a.pmap && a.nclq && pm32_fits(M, Mn);
  const int i0 = blockIdx.x * blockDim.x + threadIdx.x;
  for (int x = i0; x < M; x += gridDim.x * blockDim.x) {
    const int l = a.leader[x];
    const int g = l < 0 ? -1 : a.newidx[l];
    const int gs = g < 0 ? 0 : a.goff[g + 1] - a.goff[g];
    const int cls = (l == x || l < 0) ? 0 : (gs == 2 ? 1 : 2);
    a.colsrc[x] = g < 0 ? -1 : (g | (cls << 29));
    if (l == x) a.cursor[g] = x;
    if (compact) {
      if (l == x) {
        int y = x;
        if (gs == 2) {
          const int m0 = a.gmem[a.goff[g]];
          y = m0 == x ? a.gmem[a.goff[g] + 1] : m0;
        } else if (gs > 2) {
          clq_of(a, Mn)[atomicAdd(a.nclq, 1)] = g;
        }
        pm32_of(a)[pm32_index(g)] = (uint32_t)(x - g) | ((uint32_t)(y - g) << 15);
      }
    } else if (a.pmap && g >= 0) {
      if (l == x) {
        a.pmap[g].x = x;
        if (gs == 1) a.pmap[g].y = -1;
      } else {
        a.pmap[g].y = gs == 2 ? x : -2;
      }
    }
  }
  if (compact)
    for (int t = Mn + i0; t < pm32_words(Mn); t += gridDim.x * blockDim.x) pm32_of(a)[pm32_index(t)] = 0u;
  if (i0 < 8) {
    if (compact) {
    } else if (a.pmap)
      a.pmap[Mn + i0] = make_int2(0, -1);  // padding of the last vector
    a.colsrc[M + i0] = -1;  // padding for 16-byte colmap loads (8 codes per vector)
  }
}

// Launch with programmatic stream serialization (PDL): the kernel may be
// scheduled while its predecessor drains and waits in pdl_wait() — the
// per-launch gap of the round's ~15 small kernels shrinks.
template <typename... KP, typename... A>
inline void launch_pdl(void (*k)(KP...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, A &&...args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
#ifdef RAGB_NO_PDL
  cfg.numAttrs = 0;  // (A/B builds: plain stream-ordered launches)
#else
  cfg.numAttrs = 1;
#endif
  cudaLaunchKernelEx(&cfg, k, std::forward<A>(args)...);
}

// Launch sequences of the round preparation (single GPU and sharded build).
inline void launch_prep_mark(const PrepArgs &pa, int sms, cudaStream_t st, int *launches) {
  cudaMemsetAsync(pa.level + 1, 0xff, 4, st);
  launch_pdl(k_prep_min, sms, 256, 0, st, pa);
  launch_pdl(k_prep_rnn, sms * 2, 256, 0, st, pa);
  launch_pdl(k_prep_list, 1, PT, 0, st, pa);
  *launches += 3;
}
inline void launch_prep_compact(const PrepArgs &pa, int sms, cudaStream_t st, int *launches) {
  launch_pdl(k_compact_scan1, 1, PT, 0, st, pa);
  launch_pdl(k_compact_groups, sms * 2, 256, 0, st, pa);
  launch_pdl(k_compact_scan2, 1, PT, 0, st, pa);
  launch_pdl(k_compact_members, sms * 2, 256, 0, st, pa);
  launch_pdl(k_compact_maps, sms * 2, 256, 0, st, pa);
  *launches += 5;
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

// VEC: 16-byte loads of VW consecutive old columns (old row stride and base are
// multiples of VW elements: every compacted matrix; the original rows when
// N % VW == 0); colmap is padded with -1 to a multiple of 8.
// Old rows are addressed through a row source: the local matrix, or (row-
// sharded build, dist.cu) the shard of the rank owning the row, read from peer
// memory.  New rows [c0, c1) (c1 < 0: all Mn) are written to Dn[c - c0] with
// the leading dimension round_up(Mn, VW).
template <typename T>
struct LocalRows {
  const T *D;
  int64_t ld;
  __device__ __forceinline__ const T *row(int x) const { return D + (int64_t)x * ld; }
};
template <typename T>
struct PeerRows {
  const T *const *mats;  // [world] shard base of each rank (rows [q*S, (q+1)*S))
  int S;
  int64_t ld;
  __device__ __forceinline__ const T *row(int x) const {
    const int q = x / S;
    return mats[q] + (int64_t)(x - q * S) * ld;
  }
};

template <typename T>
__host__ __device__ constexpr int64_t mat_ld(int64_t M) {
  return (M + Elem<T>::VW - 1) / Elem<T>::VW * Elem<T>::VW;
}

// Window slot update by writer class (see k_prep_compact): the leader's
// plain store comes first (phase A), then, after a barrier, the other members
// fold in (phase B): the only other member of a pair with a plain
// read-max-write, members of larger groups atomically.  Window elements have
// the matrix's type (16-bit codes: 2 per 32-bit word, the atomic max is a CAS
// loop on the word; concurrent 16-bit stores to the other half only make it
// retry).
template <typename T>
struct Win;
template <>
struct Win<float> {
  typedef unsigned S;
  __device__ __forceinline__ static void amax(S *w, int t, unsigned v) { atomicMax(w + t, v); }
};
template <>
struct Win<uint16_t> {
  typedef uint16_t S;
  __device__ __forceinline__ static void amax(S *w, int t, unsigned v) {
    unsigned *word = reinterpret_cast<unsigned *>(w) + (t >> 1);
    const int sh = (t & 1) * 16;
    unsigned old = *reinterpret_cast<volatile unsigned *>(word);
    while (((old >> sh) & 0xffffu) < v) {
      const unsigned nw = (old & ~(0xffffu << sh)) | (v << sh);
      const unsigned prev = atomicCAS(word, old, nw);
      if (prev == old) break;
      old = prev;
    }
  }
};

template <bool VEC, int NTH, typename T, typename RS>
__global__ void __launch_bounds__(NTH) k_merge_rows(RS rs, int M, const int *__restrict__ Mn_p,
                                                    const int *__restrict__ goff,
                                                    const int *__restrict__ gmem,
                                                    const int *__restrict__ colmap,
                                                    const int *__restrict__ first_old, int W, int c0, int c1,
                                                    T *__restrict__ Dn, u64 *__restrict__ keyn) {
  typedef Elem<T> E;
  typedef typename Win<T>::S S;
  constexpr int VW = E::VW;
  extern __shared__ __align__(16) unsigned char wbytes[];
  S *win = reinterpret_cast<S *>(wbytes);  // [W] element bits (unsigned order == value order)
  __shared__ u64 wmin[NTH / 32];
  const int Mn = *Mn_p;
  const int cend = c1 < 0 ? Mn : c1;
  const int64_t ldn = mat_ld<T>(Mn);
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  for (int c = c0 + blockIdx.x; c < cend; c += gridDim.x) {
    const int rb = goff[c], re = goff[c + 1];
    const T *__restrict__ row0 = rs.row(gmem[rb]);
    int bval = 0x7fffffff, bidx = 0x7fffffff;  // running (value bits, column) minimum
    for (int T0 = 0; T0 < Mn; T0 += W) {
      const int Wn = min(W, Mn - T0);
      const int Wv = (Wn + VW - 1) / VW * VW;  // whole vectors (W is a multiple of VW)
      for (int i = Wn + tid; i < Wv; i += NTH) win[i] = 0;  // padding columns of the last vector
      const int s0 = T0 == 0 ? 0 : (first_old[T0] & ~(VW - 1));
      // every slot of the window has its leader at an old column >= s0, read
      // in a block-uniform loop (phase A / barrier / phase B per pass)
      if (VEC) {
        const uint4 *__restrict__ r4 = reinterpret_cast<const uint4 *>(row0);
        const int4 *__restrict__ c4 = reinterpret_cast<const int4 *>(colmap);
        constexpr int UV = 16 / VW;  // 16 elements per thread and pass (registers: 1024 threads)
        for (int base = s0 / VW; base * VW < M; base += NTH * UV) {
          uint4 v4[UV];
          bool ok[UV];
#pragma unroll
          for (int u = 0; u < UV; ++u) {
            const int q = base + tid + u * NTH;
            ok[u] = q * VW < M;
            v4[u] = ok[u] ? __ldcs(r4 + q) : make_uint4(0, 0, 0, 0);
          }
          for (int rr = rb + 1; rr < re; ++rr) {  // other row members (max)
            const uint4 *__restrict__ k4 = reinterpret_cast<const uint4 *>(rs.row(gmem[rr]));
#pragma unroll
            for (int u = 0; u < UV; ++u)
              if (ok[u]) v4[u] = vmax4<T>(v4[u], __ldcs(k4 + base + tid + u * NTH));
          }
          unsigned vv[UV][VW];
          int tt[UV][VW];
#pragma unroll
          for (int u = 0; u < UV; ++u) {
            E::unpack(v4[u], vv[u]);
            const int q = base + tid + u * NTH;
#pragma unroll
            for (int g = 0; g < VW / 4; ++g) {
              const int4 t4 = ok[u] ? __ldg(c4 + q * (VW / 4) + g) : int4{-1, -1, -1, -1};
              tt[u][4 * g] = t4.x;
              tt[u][4 * g + 1] = t4.y;
              tt[u][4 * g + 2] = t4.z;
              tt[u][4 * g + 3] = t4.w;
            }
          }
          // phase A: leaders
#pragma unroll
          for (int u = 0; u < UV; ++u)
#pragma unroll
            for (int k = 0; k < VW; ++k) {
              const int x = tt[u][k];
              const int t = (x & 0x1fffffff) - T0;
              if (x >= 0 && (x >> 29) == 0 && (unsigned)t < (unsigned)Wn) win[t] = (S)vv[u][k];
            }
          __syncthreads();
          // phase B: the other members
#pragma unroll
          for (int u = 0; u < UV; ++u)
#pragma unroll
            for (int k = 0; k < VW; ++k) {
              const int x = tt[u][k];
              const int t = (x & 0x1fffffff) - T0;
              if (x >= 0 && (x >> 29) != 0 && (unsigned)t < (unsigned)Wn) {
                if ((x >> 29) == 1) {
                  if (vv[u][k] > (unsigned)win[t]) win[t] = (S)vv[u][k];
                } else {
                  Win<T>::amax(win, t, vv[u][k]);
                }
              }
            }
        }
      } else {
        constexpr int U = 4;
        for (int sb = s0; sb < M; sb += U * NTH) {
          int t[U];
          unsigned v[U];
#pragma unroll
          for (int u = 0; u < U; ++u) {
            const int s = sb + u * NTH + tid;
            t[u] = s < M ? __ldg(colmap + s) : -1;
            v[u] = s < M ? E::bits(__ldcs(row0 + s)) : 0u;
          }
          for (int rr = rb + 1; rr < re; ++rr) {
            const T *rowk = rs.row(gmem[rr]);
#pragma unroll
            for (int u = 0; u < U; ++u) {
              const int s = sb + u * NTH + tid;
              if (s < M) v[u] = max(v[u], E::bits(__ldcs(rowk + s)));
            }
          }
#pragma unroll
          for (int u = 0; u < U; ++u) {
            const int x = t[u], tw = (x & 0x1fffffff) - T0;
            if (x >= 0 && (x >> 29) == 0 && (unsigned)tw < (unsigned)Wn) win[tw] = (S)v[u];
          }
          __syncthreads();
#pragma unroll
          for (int u = 0; u < U; ++u) {
            const int x = t[u], tw = (x & 0x1fffffff) - T0;
            if (x >= 0 && (x >> 29) != 0 && (unsigned)tw < (unsigned)Wn) {
              if ((x >> 29) == 1) {
                if (v[u] > (unsigned)win[tw]) win[tw] = (S)v[u];
              } else {
                Win<T>::amax(win, tw, v[u]);
              }
            }
          }
        }
      }
      __syncthreads();
      // write out (16-byte stores; the new leading dimension is a multiple of VW)
      uint4 *__restrict__ out4 = reinterpret_cast<uint4 *>(Dn + (int64_t)(c - c0) * ldn + T0);
      const int cd = c - T0;  // diagonal position inside the window
      for (int i = tid * VW; i < Wn; i += NTH * VW) {
        unsigned q[VW];
        E::unpack(*reinterpret_cast<const uint4 *>(win + i), q);
        // diagonal -> 0 in the matrix, excluded from the row minimum (as are
        // the padding columns); strict '<' keeps the earliest column (X8)
#pragma unroll
        for (int k = 0; k < VW; ++k) {
          const bool skip = i + k == cd || i + k >= Wn;
          const int m = skip ? 0x7fffffff : (int)q[k];
          if (m < bval) {
            bval = m;
            bidx = T0 + i + k;
          }
          q[k] = i + k == cd ? 0u : q[k];
        }
        __stcs(out4 + i / VW, E::pack(q));
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


// Code-mode compaction when the old row fits in shared memory (2 B x M <=
// 227 KB): one CTA per new row c.  Phase 1 streams the old row(s) of group c
// into shared memory in the OLD column order (16-byte loads, max over the
// group's rows, no atomics); phase 2 gathers each new column t from its
// leader's slot, folded with the other member of a pair (pmap) or, for larger
// groups, every member (CSR) — 16-byte stores of 8 new columns and the row min.
template <bool VEC, int NTH>
__global__ void __launch_bounds__(NTH) k_merge_gather(const uint16_t *__restrict__ D, int64_t ld, int M,
                                                      const int *__restrict__ Mn_p, const int *__restrict__ goff,
                                                      const int *__restrict__ gmem, const int2 *__restrict__ pmap,
                                                      uint16_t *__restrict__ Dn, u64 *__restrict__ keyn, int db) {
  typedef Elem<uint16_t> E;
  // db: two row buffers (when 2 x 2M bytes fit): the next row's bulk copy is
  // in flight while this row is folded and gathered
  extern __shared__ __align__(16) uint4 smem4[];  // [1 + db][ceil(M / 8)]
  __shared__ u64 wmin[NTH / 32];
  const int Mn = *Mn_p;
  const int64_t ldn = mat_ld<uint16_t>(Mn);
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int MV = (M + 7) >> 3;
  __shared__ __align__(8) unsigned long long bar[2];
  unsigned parity[2] = {0u, 0u};
  if (VEC && tid == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
  }
  __syncthreads();
  // one thread: bulk copies (TMA engine) of row `row`'s first member into slot
  auto issue = [&](int row, int slot) {
    fence_proxy_async_smem();  // earlier generic accesses of the buffer come first
    const unsigned bytes = (unsigned)MV * 16u;
    mbar_expect_tx(&bar[slot], bytes);
    const unsigned char *src = reinterpret_cast<const unsigned char *>(D + (int64_t)gmem[goff[row]] * ld);
    unsigned char *dst = reinterpret_cast<unsigned char *>(smem4 + (size_t)slot * MV);
    for (unsigned o = 0; o < bytes; o += 32768u) bulk_g2s(dst + o, src + o, min(32768u, bytes - o), &bar[slot]);
  };
  if (VEC && db && tid == 0 && (int)blockIdx.x < Mn) issue(blockIdx.x, 0);
  int it = 0;
  for (int c = blockIdx.x; c < Mn; c += gridDim.x, ++it) {
    const int rb = goff[c], re = goff[c + 1];
    const int slot = db ? (it & 1) : 0;
    uint4 *srow4 = smem4 + (size_t)slot * MV;
    const uint16_t *srow = reinterpret_cast<const uint16_t *>(srow4);
    // ---- phase 1: old row(s) -> shared memory -------------------------------
    if (VEC) {
      // the first member's row by bulk copies (all of it in flight at once),
      // then the other members folded in with 16-byte loads
      if (!db && tid == 0) issue(c, 0);
      mbar_wait(&bar[slot], parity[slot]);
      parity[slot] ^= 1u;
      if (db && tid == 0 && c + (int)gridDim.x < Mn) issue(c + gridDim.x, slot ^ 1);
      if (re - rb > 1) {
        constexpr int UV = 8;
        for (int qb = tid; qb < MV; qb += NTH * UV) {
          uint4 v[UV];
#pragma unroll
          for (int u = 0; u < UV; ++u) {
            const int q = qb + u * NTH;
            v[u] = make_uint4(0, 0, 0, 0);
            for (int rr = rb + 1; rr < re; ++rr)
              if (q < MV) v[u] = vmax4<uint16_t>(v[u], __ldcs(reinterpret_cast<const uint4 *>(D + (int64_t)gmem[rr] * ld) + q));
          }
#pragma unroll
          for (int u = 0; u < UV; ++u) {
            const int q = qb + u * NTH;
            if (q < MV) srow4[q] = vmax4<uint16_t>(srow4[q], v[u]);
          }
        }
      }
    } else {
      uint16_t *sr = reinterpret_cast<uint16_t *>(srow4);
      for (int s = tid; s < M; s += NTH) {
        unsigned v = 0u;
        for (int rr = rb; rr < re; ++rr) v = max(v, (unsigned)__ldcs(D + (int64_t)gmem[rr] * ld + s));
        sr[s] = (uint16_t)v;
      }
    }
    __syncthreads();
    // ---- phase 2: gather the new row ----------------------------------------
    // The old columns of group c (the row's own members) map only to the
    // diagonal: they are set to 0xffff (above every code) so that the gather
    // loop needs no diagonal test — the diagonal entry (0) is stored after it.
    if (tid < re - rb) reinterpret_cast<uint16_t *>(srow4)[gmem[rb + tid]] = 0xffffu;
    for (int r = rb + NTH + tid; r < re; r += NTH) reinterpret_cast<uint16_t *>(srow4)[gmem[r]] = 0xffffu;
    __syncthreads();
    // A thread takes 2 consecutive new columns per step (lanes read adjacent
    // slots: no bank conflicts; 4-byte stores coalesce per warp).  Its row
    // minimum is one packed word (value << 16 | step << 1 | column bit):
    // columns are visited in increasing order per thread, so the strict
    // minimum keeps the smallest column among equal values (X8).
    unsigned kmin = 0xffffffffu;
    unsigned *__restrict__ out2 = reinterpret_cast<unsigned *>(Dn + (int64_t)c * ldn);
    const int4 *__restrict__ pm4 = reinterpret_cast<const int4 *>(pmap);
    const int nfull = Mn >> 1;  // pairs of real columns; an odd last column is the tail below
    constexpr int UP = 4;
    unsigned step = 0;
    for (int pb = tid; pb < nfull; pb += NTH * UP) {
      int4 pm[UP];
#pragma unroll
      for (int u = 0; u < UP; ++u) {
        const int pi = pb + u * NTH;
        pm[u] = pi < nfull ? __ldg(pm4 + pi) : make_int4(0, -1, 0, -1);
      }
#pragma unroll
      for (int u = 0; u < UP; ++u, ++step) {
        const int pi = pb + u * NTH;
        const int xs[2] = {pm[u].x, pm[u].z}, ys[2] = {pm[u].y, pm[u].w};
        unsigned q[2];
#pragma unroll
        for (int k = 0; k < 2; ++k) {
          unsigned v = srow[xs[k]];
          if (ys[k] >= 0) v = max(v, (unsigned)srow[ys[k]]);
          if (ys[k] == -2)  // larger group (a level clique): every member
            for (int r = goff[2 * pi + k]; r < goff[2 * pi + k + 1]; ++r) v = max(v, (unsigned)srow[gmem[r]]);
          q[k] = v;
          if (pi < nfull) kmin = min(kmin, (v << 16) | (step << 1) | (unsigned)k);
        }
        if (pi < nfull) __stcs(out2 + pi, q[0] | (q[1] << 16));
      }
    }
    u64 best = ~0ull;
    if (kmin != 0xffffffffu && (kmin >> 16) != 0xffffu) {  // decode (step, bit) -> column
      const unsigned st_ = (kmin >> 1) & 0x7fffu;
      const int t = 2 * (tid + (int)(st_ / UP) * NTH * UP + (int)(st_ % UP) * NTH) + (int)(kmin & 1u);
      best = ((u64)(kmin >> 16) << 32) | (unsigned)t;
    }
    if ((Mn & 1) && tid == 0) {  // odd last column
      const int t = Mn - 1;
      const int2 e = pmap[t];
      unsigned v = srow[e.x];
      if (e.y >= 0) v = max(v, (unsigned)srow[e.y]);
      if (e.y == -2)
        for (int r = goff[t]; r < goff[t + 1]; ++r) v = max(v, (unsigned)srow[gmem[r]]);
      out2[t >> 1] = v;  // with the padding column (0)
      if (v != 0xffffu) {
        const u64 kt = ((u64)v << 32) | (unsigned)t;
        best = kt < best ? kt : best;
      }
    }
    __syncthreads();  // every store of the row is done: the diagonal entry last
    if (tid == 0) Dn[(int64_t)c * ldn + c] = 0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const u64 y = __shfl_xor_sync(0xffffffffu, best, o);
      best = y < best ? y : best;
    }
    if (lane == 0) wmin[w] = best;
    __syncthreads();  // also: every gather of this row is done before phase 1 of the next
    if (tid == 0) {
      u64 b = wmin[0];
#pragma unroll
      for (int k = 1; k < NTH / 32; ++k) b = wmin[k] < b ? wmin[k] : b;
      keyn[c] = b;
    }
  }
}

// Code-mode compaction with the compact map (pm32_fits): one CTA per new row c.
// Phase 1 as k_merge_gather (the first member's old row by bulk copies, the
// other members folded in); the members of every 3+-member group are folded
// into its leader's slot; then new column t is
//   max(s[x], s[y]),  x = t + (pm32[t] & 0x7fff),  y = t + (pm32[t] >> 15)
// (y == x for a singleton), with no per-column branch.  A thread takes 4
// consecutive new columns per step (one 16-byte map load, one 8-byte store).
// The row's own members are read only for new column c (groups are disjoint),
// whose value the thread holding it replaces by 0xffff (above every code: out
// of the row minimum) and the row's finisher by the diagonal 0.
// Warps never wait for each other on rows without folds: they take the row's
// data from the bulk-copy barrier, fold their row minimum into a shared word
// with an atomic, and count themselves out; the last warp out finishes the
// row (key, diagonal) and refills the buffer: in double-buffered mode with
// the row two ahead, otherwise progressively — every old column the gather
// reads for new column t is >= t, so once every warp is past a chunk of new
// columns, the old columns below it are dead for this row and the last warp
// out of the chunk copies the next row's first member into them; the
// columns past the gathered range follow when the row is done.
template <bool VEC, int NTH>
__global__ void __launch_bounds__(NTH) k_merge_gather2(const uint16_t *__restrict__ D, int64_t ld, int M,
                                                       const int *__restrict__ Mn_p, const int *__restrict__ goff,
                                                       const int *__restrict__ gmem, const uint32_t *__restrict__ pm,
                                                       const int *__restrict__ nclq_p, uint16_t *__restrict__ Dn,
                                                       u64 *__restrict__ keyn, int db, SideBuf sb) {
  pdl_wait();
  constexpr int NWARP = NTH / 32;
  constexpr int kMaxChunks = 32;  // chunks per row (progressive refill needs Mn / (4 * CQ) <= kMaxChunks)
  extern __shared__ __align__(16) uint4 smem4[];  // [1 + db][ceil(M / 8)]
  __shared__ __align__(8) unsigned long long bar[2];
  __shared__ u64 rowmin[2];               // per row parity: (code << 32 | column) minimum
  __shared__ int row_done[2];             // per row parity: warps done with the row
  __shared__ int chunk_done[kMaxChunks];  // warps done with each chunk (progressive refill)
  const int Mn = *Mn_p, nclq = *nclq_p;
  const int *__restrict__ clq = reinterpret_cast<const int *>(pm + pm32_words(Mn));
  const int64_t ldn = mat_ld<uint16_t>(Mn);
  const int tid = threadIdx.x, lane = tid & 31;
  const int MV = (M + 7) >> 3;
  const int G = (int)gridDim.x;
  unsigned parity = 0u;  // bit b: phase parity of bar[b]
  if (tid == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    rowmin[0] = rowmin[1] = ~0ull;
    row_done[0] = row_done[1] = 0;
  }
  if (tid < kMaxChunks) chunk_done[tid] = 0;
  __syncthreads();
  // one thread: bulk copies of 16-byte vectors [v0, v1) of row `row`'s first
  // member into slot (the barrier is armed separately, once per row)
  auto copy = [&](int row, int slot, int v0, int v1) {
    fence_proxy_async_smem();  // earlier generic accesses of the buffer come first
    const unsigned char *src = reinterpret_cast<const unsigned char *>(D + (int64_t)gmem[goff[row]] * ld) + (size_t)v0 * 16;
    unsigned char *dst = reinterpret_cast<unsigned char *>(smem4 + (size_t)slot * MV + v0);
    const unsigned bytes = (unsigned)(v1 - v0) * 16u;
    for (unsigned o = 0; o < bytes; o += 32768u) bulk_g2s_stream(dst + o, src + o, min(32768u, bytes - o), &bar[slot]);
  };
  if (VEC && tid == 0) {
    for (int k = 0; k <= db; ++k)
      if ((int)blockIdx.x + k * G < Mn) {
        mbar_expect_tx(&bar[k], (unsigned)MV * 16u);
        copy(blockIdx.x + k * G, k, 0, MV);
      }
  }
  const uint4 *__restrict__ pm4 = reinterpret_cast<const uint4 *>(pm);
  const int nq = pm32_words(Mn) >> 2;  // quads of columns (the last ones: padding)
  constexpr int UP = 4;
  constexpr int CQ = NTH * UP;  // quads per chunk
  const bool progressive_ok = VEC && !db && nq <= kMaxChunks * CQ;
  int it = 0;
  for (int c = blockIdx.x; c < Mn; c += G, ++it) {
    const int rb = goff[c], re = goff[c + 1];
    const int slot = db ? (it & 1) : 0;
    const int rp = it & 1;  // row parity: at most two rows are in flight per CTA
    const int cn = c + G;   // this CTA's next row
    const bool progressive = progressive_ok && cn < Mn;
    uint4 *srow4 = smem4 + (size_t)slot * MV;
    uint16_t *srow = reinterpret_cast<uint16_t *>(srow4);
    // ---- phase 1: old row(s) -> shared memory ---------------------------------
    if (!VEC) {  // old rows not 16-byte aligned (the distance kernel's codes with N % 8 != 0)
      __syncthreads();  // the previous row's reads are done
      for (int x = tid; x < M; x += NTH) {
        unsigned v = 0u;
        for (int rr = rb; rr < re; ++rr) v = max(v, (unsigned)__ldcs(D + (int64_t)gmem[rr] * ld + x));
        srow[x] = (uint16_t)v;
      }
    } else {
      mbar_wait(&bar[slot], (parity >> slot) & 1u);
      parity ^= 1u << slot;
      if (tid == 0 && cn < Mn) {
        // the next row's folded members (read with plain loads) and, in
        // progressive mode, the part of its first member copied after this
        // row: into L2 now, while this row is gathered
        const int nb = goff[cn], ne = goff[cn + 1];
        for (int rr = nb + 1; rr < ne; ++rr) {
          const unsigned char *src = reinterpret_cast<const unsigned char *>(D + (int64_t)gmem[rr] * ld);
          for (unsigned o = 0; o < (unsigned)MV * 16u; o += 65536u) bulk_prefetch_l2(src + o, min(65536u, (unsigned)MV * 16u - o));
        }
        if (progressive) {
          const unsigned v0 = (unsigned)((4 * ((nq - 1) / CQ * CQ)) >> 3);  // the last chunk's copy
          if ((int)v0 < MV)
            bulk_prefetch_l2(reinterpret_cast<const unsigned char *>(D + (int64_t)gmem[nb] * ld) + (size_t)v0 * 16,
                             ((unsigned)MV - v0) * 16u);
        }
      }
    }
    if (VEC && re - rb > 1) {
      constexpr int UV = 8;
      __syncthreads();  // every warp has the row's first member (its writes below are seen by all)
      for (int qb = tid; qb < MV; qb += NTH * UV) {
        uint4 v[UV];
#pragma unroll
        for (int u = 0; u < UV; ++u) {
          const int q = qb + u * NTH;
          v[u] = make_uint4(0, 0, 0, 0);
          for (int rr = rb + 1; rr < re; ++rr)
            if (q < MV) v[u] = vmax4<uint16_t>(v[u], __ldcs(reinterpret_cast<const uint4 *>(D + (int64_t)gmem[rr] * ld) + q));
        }
#pragma unroll
        for (int u = 0; u < UV; ++u) {
          const int q = qb + u * NTH;
          if (q < MV) srow4[q] = vmax4<uint16_t>(srow4[q], v[u]);
        }
      }
    }
    if (sb.T) {
      // dirty columns of the in-place side buffer (see SideBuf): the row's
      // value at a dirty column is the max of its members' T entries
      const int nt = *sb.nt;
      __syncthreads();
      for (int k = tid; k < nt; k += NTH) {
        const int col = sb.tcol[k];
        if (col < 0) continue;
        unsigned v = 0u;
        for (int rr = rb; rr < re; ++rr) v = max(v, (unsigned)sb.T[(int64_t)gmem[rr] * sb.cap + k]);
        srow[col] = (uint16_t)v;
      }
    }
    if (nclq > 0) {
      __syncthreads();
      for (int i = tid; i < nclq; i += NTH) {  // 3+-member groups: members folded into the leader's slot
        const int g = clq[i];
        unsigned v = 0u;
        for (int r = goff[g]; r < goff[g + 1]; ++r) v = max(v, (unsigned)srow[gmem[r]]);
        srow[g + (int)(pm[pm32_index(g)] & 0x7fffu)] = (uint16_t)v;
      }
    }
    if (!VEC || re - rb > 1 || nclq > 0 || sb.T) __syncthreads();
    // ---- phase 2: gather -------------------------------------------------------
    uint2 *__restrict__ out4 = reinterpret_cast<uint2 *>(Dn + (int64_t)c * ldn);
    const unsigned sbase = smem_u32(srow);
    const int qc = c >> 2;  // the quad holding the diagonal
    // row minimum per thread: value << 16 | step << 2 | k (steps in increasing
    // column order: the strict minimum keeps the smallest column, X8)
    unsigned kmin = 0xffffffffu;
    // thread quads q = tid + j * NTH (columns 4q .. 4q + 3); the map words of
    // quad j + UP are loaded while quad j is gathered (UP loads in flight per
    // thread at all times)
    uint4 e[UP];
#pragma unroll
    for (int u = 0; u < UP; ++u) {
      const int q = u * NTH + tid;
      e[u] = q < nq ? __ldg(pm4 + q) : make_uint4(0u, 0u, 0u, 0u);
    }
    unsigned step = 0;
    for (int qb = 0, ch = 0; qb < nq; qb += CQ, ++ch) {
#pragma unroll
      for (int u = 0; u < UP; ++u, ++step) {
        const int q = qb + u * NTH + tid;
        const uint4 ec = e[u];
        const int qn = q + CQ;
        e[u] = qn < nq ? __ldg(pm4 + qn) : make_uint4(0u, 0u, 0u, 0u);
        if (4 * q + 3 < Mn) {
          const int t = 4 * q;
          const unsigned ev[4] = {ec.x, ec.y, ec.z, ec.w};
          // shared-window byte addresses: s[t + k + off] at sbase + 2 (t + k) + 2 off
          const unsigned a0 = sbase + 8u * (unsigned)q;
          unsigned v[4];
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const unsigned ax = a0 + 2u * k + ((ev[k] << 1) & 0xfffeu), ay = a0 + 2u * k + ((ev[k] >> 14) & ~1u);
            v[k] = max(lds_u16(ax), lds_u16(ay));
          }
          if (q == qc) {
#pragma unroll
            for (int k = 0; k < 4; ++k) v[k] = t + k == c ? 0xffffu : v[k];
          }
          __stcs(out4 + q, make_uint2(__byte_perm(v[0], v[1], 0x5410), __byte_perm(v[2], v[3], 0x5410)));
          const unsigned sb = step << 2;
          kmin = min(kmin, min(min(v[0] * 65536u + sb, v[1] * 65536u + (sb | 1u)),
                               min(v[2] * 65536u + (sb | 2u), v[3] * 65536u + (sb | 3u))));
        } else if (4 * q < Mn) {  // the last, partial quad
          const int t = 4 * q;
          const unsigned ev[4] = {ec.x, ec.y, ec.z, ec.w};
          const unsigned sb = step << 2;
#pragma unroll
          for (int k = 0; k < 4; ++k)
            if (t + k < Mn) {
              const unsigned v = t + k == c ? 0xffffu
                                            : max((unsigned)srow[t + k + (int)(ev[k] & 0x7fffu)],
                                                  (unsigned)srow[t + k + (int)(ev[k] >> 15)]);
              Dn[(int64_t)c * ldn + t + k] = (uint16_t)v;
              kmin = min(kmin, (v << 16) | sb | (unsigned)k);
            }
        }
      }
      if (progressive) {
        __syncwarp();
        if (lane == 0) {
          __threadfence_block();  // this warp's reads of the chunk come first
          if (atomicAdd(&chunk_done[ch], 1) == NWARP - 1) {  // every warp is past this chunk
            if (ch == 0) mbar_expect_tx(&bar[0], (unsigned)MV * 16u);  // the next row's phase
            // after the last chunk the whole buffer is free: the rest of the row
            const int vlo = (4 * qb) >> 3, vhi = qb + CQ >= nq ? MV : (4 * (qb + CQ)) >> 3;
            if (vhi > vlo) copy(cn, 0, vlo, vhi);
          }
        }
      }
    }
    u64 best = ~0ull;
    if (kmin != 0xffffffffu && (kmin >> 16) != 0xffffu) {  // decode (step, k) -> column
      const unsigned st_ = (kmin >> 2) & 0x3fffu;
      const int t = 4 * ((int)(st_ / UP) * CQ + (int)(st_ % UP) * NTH + tid) + (int)(kmin & 3u);
      best = ((u64)(kmin >> 16) << 32) | (unsigned)t;
    }
    best = umin64(best, __shfl_xor_sync(0xffffffffu, best, 16));
    best = umin64(best, __shfl_xor_sync(0xffffffffu, best, 8));
    best = umin64(best, __shfl_xor_sync(0xffffffffu, best, 4));
    best = umin64(best, __shfl_xor_sync(0xffffffffu, best, 2));
    best = umin64(best, __shfl_xor_sync(0xffffffffu, best, 1));
    __syncwarp();
    if (lane == 0) {
      if (best != ~0ull) atomicMin(&rowmin[rp], best);
      __threadfence_block();  // this warp's reads and stores of the row come first
      if (atomicAdd(&row_done[rp], 1) == NWARP - 1) {  // the last warp out finishes the row
        __threadfence_block();
        const u64 b = atomicExch(&rowmin[rp], ~0ull);
        row_done[rp] = 0;
        keyn[c] = b;
        Dn[(int64_t)c * ldn + c] = 0;  // the diagonal, after every warp's stores
        if (VEC && db) {
          if (c + 2 * G < Mn) {  // this buffer's next row
            mbar_expect_tx(&bar[slot], (unsigned)MV * 16u);
            copy(c + 2 * G, slot, 0, MV);
          }
        } else if (VEC && cn < Mn) {
          for (int k = 0; k < kMaxChunks; ++k) chunk_done[k] = 0;
          if (!progressive) mbar_expect_tx(&bar[0], (unsigned)MV * 16u);  // else armed at chunk 0
          if (!progressive) copy(cn, 0, 0, MV);  // (progressive: the chunks' copies cover the row)
        }
      }
    }
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
                               int *__restrict__ nmulti, int *__restrict__ sz, u64 *__restrict__ key, SideBuf sb,
                               NNCache nc) {
  pdl_wait();
  for (int x = blockIdx.x * blockDim.x + threadIdx.x; x < M; x += gridDim.x * blockDim.x) {
    const int l = a.leader[x];
    uint8_t chg = 0;
    if (l >= 0) {
      const int g = a.newidx[l];
      if (a.goff[g + 1] - a.goff[g] >= 2) {
        chg = 1;
        if (nc.key2) {
          nc.ver[x] = nc.round;
          nc.kround[x] = 0;  // the survivor's row is recomputed; members die
        }
        if (x != l) {
          key[x] = kDead;
          atomicAnd(&amask[x >> 5], ~(1u << (x & 31)));
          if (sb.T && sb.tslot[x] >= 0) sb.tcol[sb.tslot[x]] = -1;  // a dirty column merged away
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
template <int NTH, typename T>
__global__ void __launch_bounds__(NTH, 2) k_inplace_rows(PrepArgs a, T *__restrict__ D, int64_t ld, int M,
                                                      const uint32_t *__restrict__ amask,
                                                      const int *__restrict__ mlist,
                                                      const int *__restrict__ nmulti_p, u64 *__restrict__ key) {
  typedef Elem<T> E;
  constexpr int VW = E::VW;
  extern __shared__ __align__(16) uint4 rowv[];  // [ceil(M / VW)] vectors
  T *row = reinterpret_cast<T *>(rowv);
  __shared__ u64 wmin[NTH / 32];
  const int nmulti = *nmulti_p;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int MV = (M + VW - 1) / VW;
  for (int gi = blockIdx.x; gi < nmulti; gi += gridDim.x) {
    const int g = mlist[gi];
    const int rb = a.goff[g], re = a.goff[g + 1];
    const int L = a.cursor[g];  // first_old: the survivor
    for (int q = tid; q < MV; q += NTH) {
      uint4 v = make_uint4(0, 0, 0, 0);
      for (int r = rb; r < re; ++r)
        v = vmax4<T>(v, __ldcs(reinterpret_cast<const uint4 *>(D + (int64_t)a.gmem[r] * ld) + q));
      rowv[q] = v;
    }
    __syncthreads();
    for (int hi = tid; hi < nmulti; hi += NTH) {
      const int h = mlist[hi];
      if (h == g) continue;
      unsigned v = 0u;
      for (int r = a.goff[h]; r < a.goff[h + 1]; ++r) v = max(v, E::bits(row[a.gmem[r]]));
      row[a.cursor[h]] = E::make(v);
    }
    __syncthreads();
    if (tid == 0) row[L] = E::make(0u);
    __syncthreads();
    u64 best = ~0ull;
    uint4 *out = reinterpret_cast<uint4 *>(D + (int64_t)L * ld);
    for (int q = tid; q < MV; q += NTH) {
      const uint4 v = rowv[q];
      __stcs(out + q, v);
      unsigned vv[VW];
      E::unpack(v, vv);
#pragma unroll
      for (int k = 0; k < VW; ++k) {
        const int c = VW * q + k;
        const bool live = c < M && c != L && ((amask[c >> 5] >> (c & 31)) & 1u);
        const u64 kk = ((u64)vv[k] << 32) | (unsigned)c;
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

// S1 with the side buffer (code mode): as k_inplace_rows, and the survivor's
// T row is the max of its members' T rows; a member's value at a dirty column
// comes from T; the row minimum takes clean live columns (and the round's
// survivors, whose values are in the new row) from the row and the other
// live dirty columns from T.
template <int NTH>
__global__ void __launch_bounds__(NTH, 2) k_inplace_rows_sb(PrepArgs a, uint16_t *__restrict__ D, int64_t ld,
                                                         int M, const uint32_t *__restrict__ amask,
                                                         const int *__restrict__ mlist,
                                                         const int *__restrict__ nmulti_p, u64 *__restrict__ key,
                                                         SideBuf sb) {
  pdl_wait();
  typedef Elem<uint16_t> E;
  constexpr int VW = 8;
  extern __shared__ __align__(16) uint4 rowv[];  // [MV] row, then [cap / 8] T row
  uint16_t *row = reinterpret_cast<uint16_t *>(rowv);
  __shared__ u64 wmin[NTH / 32];
  const int nmulti = *nmulti_p, nt = *sb.nt;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int MV = (M + VW - 1) / VW, TV = (nt + 7) / 8;
  uint4 *trow4 = rowv + MV;
  const uint16_t *trow = reinterpret_cast<const uint16_t *>(trow4);
  for (int gi = blockIdx.x; gi < nmulti; gi += gridDim.x) {
    const int g = mlist[gi];
    const int rb = a.goff[g], re = a.goff[g + 1];
    const int L = a.cursor[g];  // first_old: the survivor
    for (int q = tid; q < MV; q += NTH) {
      uint4 v = make_uint4(0, 0, 0, 0);
      for (int r = rb; r < re; ++r)
        v = vmax4<uint16_t>(v, __ldcs(reinterpret_cast<const uint4 *>(D + (int64_t)a.gmem[r] * ld) + q));
      rowv[q] = v;
    }
    for (int q = tid; q < TV; q += NTH) {
      uint4 v = make_uint4(0, 0, 0, 0);
      for (int r = rb; r < re; ++r)
        v = vmax4<uint16_t>(v, *(reinterpret_cast<const uint4 *>(sb.T + (int64_t)a.gmem[r] * sb.cap) + q));
      trow4[q] = v;
    }
    __syncthreads();
    for (int hi = tid; hi < nmulti; hi += NTH) {
      const int h = mlist[hi];
      if (h == g) continue;
      unsigned v = 0u;
      for (int r = a.goff[h]; r < a.goff[h + 1]; ++r) {
        const int x = a.gmem[r];
        v = max(v, sb_dirty(sb, x) ? (unsigned)trow[sb.tslot[x]] : (unsigned)row[x]);
      }
      row[a.cursor[h]] = (uint16_t)v;
    }
    __syncthreads();
    if (tid == 0) row[L] = 0;
    __syncthreads();
    // row minimum on 32-bit keys code << 16 | column (M <= kInplaceMaxM < 2^16:
    // the 64-bit key's order; ~0u = none)
    unsigned best = ~0u;
    uint4 *out = reinterpret_cast<uint4 *>(D + (int64_t)L * ld);
    for (int q = tid; q < MV; q += NTH) {
      const uint4 v = rowv[q];
      __stcs(out + q, v);
      unsigned vv[VW];
      E::unpack(v, vv);
      const int c0 = VW * q;
      const unsigned mb = (amask[c0 >> 5] >> (c0 & 31)) & 0xffu, db = (sb.dmask[c0 >> 5] >> (c0 & 31)) & 0xffu;
#pragma unroll
      for (int k = 0; k < VW; ++k) {
        const int c = c0 + k;
        // live, and clean or merged this round (its value is in the new row)
        const bool live = ((mb >> k) & 1u) && c < M && c != L && (!((db >> k) & 1u) || a.alive[c]);
        best = min(best, live ? (vv[k] << 16) | (unsigned)c : ~0u);
      }
    }
    uint4 *tout = reinterpret_cast<uint4 *>(sb.T + (int64_t)L * sb.cap);
    for (int q = tid; q < TV; q += NTH) tout[q] = trow4[q];
    for (int k = tid; k < nt; k += NTH) {
      const int c = sb.tcol[k];  // retired slots (incl. dead columns): -1
      if (c < 0 || c == L || a.alive[c]) continue;
      best = min(best, ((unsigned)trow[k] << 16) | (unsigned)c);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) best = min(best, __shfl_xor_sync(0xffffffffu, best, o));
    if (lane == 0) wmin[w] = best == ~0u ? ~0ull : ((u64)(best >> 16) << 32) | (best & 0xffffu);
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

// S2 with the side buffer: the round's survivors' new rows, transposed, into
// slots nt .. nt + nmulti - 1 of every row's T segment.  CTA = 64 rows x 32
// survivors through a shared-memory tile (row segments read coalesced, each
// T row gets 32 consecutive slots).
__global__ void __launch_bounds__(256) k_side_tpose(PrepArgs a, const uint16_t *__restrict__ D, int64_t ld, int M,
                                                    const int *__restrict__ mlist, const int *__restrict__ nmulti_p,
                                                    SideBuf sb) {
  pdl_wait();
  __shared__ uint16_t tile[32][64 + 2];
  const int m = *nmulti_p, nt = *sb.nt;
  const int k0 = blockIdx.y * 32;
  if (k0 >= m) return;
  const int r0 = blockIdx.x * 64;
  const int tid = threadIdx.x;
  for (int e = tid; e < 32 * 64; e += 256) {
    const int kk = e >> 6, rr = e & 63;
    uint16_t v = 0;
    const int r = r0 + rr;
    if (k0 + kk < m && r < M) {
      // val(L, r): a dirty column r (not merged this round) holds its value in
      // L's T row; the round's survivors' values are in the new row itself
      const int L = a.cursor[mlist[k0 + kk]];
      v = (sb_dirty(sb, r) && !a.alive[r]) ? sb.T[(int64_t)L * sb.cap + sb.tslot[r]] : D[(int64_t)L * ld + r];
    }
    tile[kk][rr] = v;
  }
  __syncthreads();
  for (int e = tid; e < 32 * 64; e += 256) {
    const int rr = e >> 5, kk = e & 31;
    if (k0 + kk < m && r0 + rr < M) sb.T[(int64_t)(r0 + rr) * sb.cap + nt + k0 + kk] = tile[kk][rr];
  }
}

// S2b (one CTA): slot maps of the round's survivors (a re-merged dirty column
// retires its old slot), dirty bits, then the new slot count.
__global__ void __launch_bounds__(1024) k_side_maps(PrepArgs a, const int *__restrict__ mlist,
                                                    const int *__restrict__ nmulti_p, SideBuf sb) {
  pdl_wait();
  const int m = *nmulti_p, nt = *sb.nt;
  for (int k = threadIdx.x; k < m; k += blockDim.x) {
    const int L = a.cursor[mlist[k]];
    const int old = sb.tslot[L];
    if (old >= 0) sb.tcol[old] = -1;
    sb.tslot[L] = nt + k;
    sb.tcol[nt + k] = L;
    atomicOr(&sb.dmask[L >> 5], 1u << (L & 31));
  }
  __syncthreads();
  if (threadIdx.x == 0) *sb.nt = nt + m;
}

// Flush (before a compaction): every row < M staged in shared memory, its
// dirty columns patched from T, written back whole.
__global__ void __launch_bounds__(256) k_side_flush(uint16_t *__restrict__ D, int64_t ld, int M, SideBuf sb) {
  extern __shared__ __align__(16) uint4 rowv[];  // [MV] row, then [cap] slot columns
  uint16_t *row = reinterpret_cast<uint16_t *>(rowv);
  const int nt = *sb.nt;
  const int MV = (M + 7) / 8;
  int *scol = reinterpret_cast<int *>(rowv + MV);
  for (int k = threadIdx.x; k < nt; k += blockDim.x) scol[k] = sb.tcol[k];
  for (int r = blockIdx.x; r < M; r += gridDim.x) {
    uint4 *src = reinterpret_cast<uint4 *>(D + (int64_t)r * ld);
    for (int q = threadIdx.x; q < MV; q += blockDim.x) rowv[q] = __ldcs(src + q);
    __syncthreads();
    const uint16_t *trow = sb.T + (int64_t)r * sb.cap;
    for (int k0 = threadIdx.x; k0 < nt; k0 += blockDim.x * 4) {
      uint16_t v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) v[u] = k0 + u * (int)blockDim.x < nt ? trow[k0 + u * blockDim.x] : (uint16_t)0;
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int k = k0 + u * blockDim.x;
        if (k < nt && scol[k] >= 0) row[scol[k]] = v[u];
      }
    }
    __syncthreads();
    for (int q = threadIdx.x; q < MV; q += blockDim.x) __stcs(src + q, rowv[q]);
    __syncthreads();
  }
}

// S2: columns from rows (symmetry): D[r][L] = D[L][r] for every live row r.
// CTA (x = merged group, y = chunk of CR rows): the group's survivor L is
// looked up once, then every thread moves CR / 256 rows (independent
// coalesced loads, scattered 2- or 4-byte stores), so the dependent-load
// chain is paid once per CTA instead of once per handful of rows.
constexpr int kColsRows = 4096;
template <typename T>
__global__ void __launch_bounds__(256) k_inplace_cols(PrepArgs a, T *__restrict__ D, int64_t ld, int M,
                                                      const uint32_t *__restrict__ amask,
                                                      const int *__restrict__ mlist,
                                                      const int *__restrict__ nmulti_p) {
  const int gi = blockIdx.x;
  if (gi >= *nmulti_p) return;
  const int L = a.cursor[mlist[gi]];
  const T *src = D + (int64_t)L * ld;
  constexpr int PER = kColsRows / 256;
  const int rbase = blockIdx.y * kColsRows + (int)threadIdx.x;
  T v[PER];
  bool ok[PER];
#pragma unroll
  for (int u = 0; u < PER; ++u) {
    const int r = rbase + u * 256;
    ok[u] = r < M && ((__ldg(amask + (r >> 5)) >> (r & 31)) & 1u);
    v[u] = ok[u] ? __ldg(src + r) : Elem<T>::make(0u);
  }
#pragma unroll
  for (int u = 0; u < PER; ++u)
    if (ok[u]) D[(int64_t)(rbase + u * 256) * ld + L] = v[u];
}

// S3a: one thread per live row r outside the merged groups whose nearest
// neighbour t was in a merged group g with survivor L: the new value d(r, L)
// (column L was rewritten by S2) is >= the old d(r, t); if equal, (d, L) is
// the new key without a scan (L <= t, every other entry is unchanged or
// larger); otherwise r goes to the rescan list.
template <typename T>
__global__ void k_inplace_check(PrepArgs a, const T *__restrict__ D, int64_t ld, int M,
                                u64 *__restrict__ key, int *__restrict__ rlist, int *__restrict__ nres, SideBuf sb,
                                NNCache nc) {
  pdl_wait();
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < M; r += gridDim.x * blockDim.x) {
    const u64 kr = key[r];
    if (kr == kDead || a.alive[r]) continue;  // dead, or a survivor (done in S1)
    const int t = (int)(kr & 0xffffffffu);
    if (!a.alive[t]) continue;  // neighbour not merged: unchanged
    const int Lg = a.leader[t];
    const unsigned v = sb.T ? (unsigned)sb.T[(int64_t)r * sb.cap + sb.tslot[Lg]] : Elem<T>::bits(D[(int64_t)r * ld + Lg]);
    if (v == (unsigned)(kr >> 32)) {
      key[r] = ((u64)v << 32) | (unsigned)Lg;
    } else {
      const int kround = nc.key2 ? nc.kround[r] : 0;
      const u64 k2 = kround > 0 ? nc.key2[r] : ~0ull;
      if (kround > 0 && nc.ver[(int)(k2 & 0xffffffffu)] <= kround) {
        const u64 kL = ((u64)v << 32) | (unsigned)Lg;  // (the second-nearest cache, one use)
        key[r] = kL < k2 ? kL : k2;
        nc.kround[r] = 0;
      } else {
        rlist[atomicAdd(nres, 1)] = r;
      }
    }
  }
}

// S3b: full rescans of the listed rows over the live columns.
// Keeps the two smallest keys b[0] < b[1] (a cheap reject first).
__device__ __forceinline__ void top2_insert(u64 (&b)[2], u64 kk) {
  if (kk < b[1]) {
    const bool l1 = kk < b[0];
    b[1] = l1 ? b[0] : kk;
    b[0] = l1 ? kk : b[0];
  }
}

template <int NTH, typename T>
__global__ void __launch_bounds__(NTH) k_inplace_rescan(const T *__restrict__ D, int64_t ld, int M,
                                                        const uint32_t *__restrict__ amask,
                                                        const int *__restrict__ rlist,
                                                        const int *__restrict__ nres_p, u64 *__restrict__ key,
                                                        SideBuf sb, NNCache nc) {
  pdl_wait();
  typedef Elem<T> E;
  constexpr int VW = E::VW;
  __shared__ u64 wmin[NTH / 32][2];
  // the scan mask (live and clean columns) and the side buffer's slot
  // columns, the same for every row: staged once per CTA
  extern __shared__ __align__(16) unsigned char rsmem[];
  unsigned *smask = reinterpret_cast<unsigned *>(rsmem);  // [M/32 + 1]
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int MV = (M + VW - 1) / VW;
  const int nres = *nres_p;
  if ((int)blockIdx.x >= nres) return;
  const int MW = M / 32 + 1;
  int *scol = reinterpret_cast<int *>(smask + ((MW + 3) & ~3));  // [nt]
  const int nt = sb.T ? *sb.nt : 0;
  for (int k = tid; k < MW; k += NTH) smask[k] = amask[k] & ~(sb.T ? sb.dmask[k] : 0u);
  for (int k = tid; k < nt; k += NTH) scol[k] = sb.tcol[k];
  __syncthreads();
#ifdef RAGB_RESCAN64
  constexpr bool kKey32 = false;  // variant: the 64-bit keys for codes too (A/B)
#else
  constexpr bool kKey32 = true;
#endif
  if constexpr (sizeof(T) == 2 && kKey32) {
    // 16-bit codes and M <= kInplaceMaxM < 2^16: a key (code, column) fits
    // 32 bits as code << 16 | column (same order as the 64-bit key), and the
    // two smallest are kept branch-free with min/max (~half the instructions
    // of the 64-bit compare-and-swap per column)
    for (int i = blockIdx.x; i < nres; i += gridDim.x) {
      const int r = rlist[i];
      unsigned b0 = ~0u, b1 = ~0u;
      auto ins = [&](unsigned k) {
        const unsigned hi = max(b0, k);
        b0 = min(b0, k);
        b1 = min(b1, hi);
      };
      const uint4 *src = reinterpret_cast<const uint4 *>(D + (int64_t)r * ld);
      constexpr int UR = 4;
      for (int q0 = tid; q0 < MV; q0 += NTH * UR) {
        uint4 x[UR];
#pragma unroll
        for (int u = 0; u < UR; ++u) x[u] = q0 + u * NTH < MV ? __ldcs(src + q0 + u * NTH) : make_uint4(0, 0, 0, 0);
#pragma unroll
        for (int u = 0; u < UR; ++u) {
          const int q = q0 + u * NTH;
          if (q >= MV) continue;
          const int c0 = VW * q;
          unsigned mb = (smask[c0 >> 5] >> (c0 & 31)) & 0xffu;
          if (c0 + 8 > M) mb &= (1u << (M - c0)) - 1u;
          if (r >= c0 && r < c0 + 8) mb &= ~(1u << (r - c0));
          const unsigned xv[4] = {x[u].x, x[u].y, x[u].z, x[u].w};
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            const unsigned v = (k & 1) ? (xv[k >> 1] >> 16) : (xv[k >> 1] & 0xffffu);
            ins(((mb >> k) & 1u) ? ((v << 16) | (unsigned)(c0 + k)) : ~0u);
          }
        }
      }
      if (nt > 0) {
        const uint4 *trow4 = reinterpret_cast<const uint4 *>(sb.T + (int64_t)r * sb.cap);
        for (int k8 = tid; 8 * k8 < nt; k8 += NTH) {
          unsigned vs[8];
          Elem<uint16_t>::unpack(trow4[k8], vs);
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            const int k = 8 * k8 + u;
            const int c = k < nt ? scol[k] : -1;
            ins((c >= 0 && c != r) ? ((vs[u] << 16) | (unsigned)c) : ~0u);
          }
        }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const unsigned y0 = __shfl_xor_sync(0xffffffffu, b0, o), y1 = __shfl_xor_sync(0xffffffffu, b1, o);
        ins(y0);
        ins(y1);
      }
      auto widen = [](unsigned k) -> u64 { return k == ~0u ? ~0ull : ((u64)(k >> 16) << 32) | (k & 0xffffu); };
      if (lane == 0) {
        wmin[w][0] = widen(b0);
        wmin[w][1] = widen(b1);
      }
      __syncthreads();
      if (tid == 0) {
        u64 bb[2] = {wmin[0][0], wmin[0][1]};
        for (int i2 = 1; i2 < NTH / 32; ++i2)
#pragma unroll
          for (int q = 0; q < 2; ++q) top2_insert(bb, wmin[i2][q]);
        key[r] = bb[0];
        if (nc.key2) {
          nc.key2[r] = bb[1];
          nc.kround[r] = bb[1] != ~0ull ? nc.round : 0;
        }
      }
      __syncthreads();
    }
  } else {
  for (int i = blockIdx.x; i < nres; i += gridDim.x) {
    const int r = rlist[i];
    u64 bt[2] = {~0ull, ~0ull};  // the row's two smallest keys (this thread)
    const uint4 *src = reinterpret_cast<const uint4 *>(D + (int64_t)r * ld);
    constexpr int UR = 4;  // vectors in flight per thread
    for (int q0 = tid; q0 < MV; q0 += NTH * UR) {
      uint4 x[UR];
#pragma unroll
      for (int u = 0; u < UR; ++u) x[u] = q0 + u * NTH < MV ? __ldcs(src + q0 + u * NTH) : make_uint4(0, 0, 0, 0);
#pragma unroll
      for (int u = 0; u < UR; ++u) {
        const int q = q0 + u * NTH;
        if (q >= MV) continue;
        unsigned vv[VW];
        E::unpack(x[u], vv);
        // the vector's VW columns lie in one mask word: live and (with a side
        // buffer) clean
        const int c0 = VW * q;
        const unsigned mw = smask[c0 >> 5];
        const unsigned mb = (mw >> (c0 & 31)) & ((1u << VW) - 1u);
#pragma unroll
        for (int k = 0; k < VW; ++k) {
          const int c = c0 + k;
          const bool live = ((mb >> k) & 1u) && c < M && c != r;
          top2_insert(bt, live ? (((u64)vv[k] << 32) | (unsigned)c) : ~0ull);
        }
      }
    }
    if (nt > 0) {  // dirty columns from the side buffer (retired slots: tcol -1, incl. dead columns)
      const uint4 *trow4 = reinterpret_cast<const uint4 *>(sb.T + (int64_t)r * sb.cap);  // 8 slots per vector
      for (int k8 = tid; 8 * k8 < nt; k8 += NTH) {
        unsigned vs[8];
        Elem<uint16_t>::unpack(trow4[k8], vs);
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int k = 8 * k8 + u;
          const int c = k < nt ? scol[k] : -1;
          top2_insert(bt, (c >= 0 && c != r) ? (((u64)vs[u] << 32) | (unsigned)c) : ~0ull);
        }
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      u64 y[2];
#pragma unroll
      for (int q = 0; q < 2; ++q) y[q] = __shfl_xor_sync(0xffffffffu, bt[q], o);
#pragma unroll
      for (int q = 0; q < 2; ++q) top2_insert(bt, y[q]);
    }
    if (lane == 0) {
      wmin[w][0] = bt[0];
      wmin[w][1] = bt[1];
    }
    __syncthreads();
    if (tid == 0) {
      u64 b[2] = {wmin[0][0], wmin[0][1]};
      for (int i2 = 1; i2 < NTH / 32; ++i2)
#pragma unroll
        for (int q = 0; q < 2; ++q) top2_insert(b, wmin[i2][q]);
      key[r] = b[0];
      if (nc.key2) {  // the second-nearest cache
        nc.key2[r] = b[1];
        nc.kround[r] = b[1] != ~0ull ? nc.round : 0;
      }
    }
    __syncthreads();
  }
  }
}

// Row keys of the distance kernel ((f32 bits << 32) | column) -> code keys:
// the code of a value is its position in the ascending table vals[0, ncode).
__global__ void k_keys_to_codes(u64 *__restrict__ key, int64_t N, const float *__restrict__ vals,
                                const int *__restrict__ ncode_p) {
  pdl_wait();
  const int ncode = *ncode_p;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < N; i += (int64_t)gridDim.x * blockDim.x) {
    const u64 k = key[i];
    if (k == ~0ull) continue;
    const float v = __uint_as_float((unsigned)(k >> 32));
    int lo = 0, hi = ncode - 1;  // vals strictly ascending and v is one of them
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (vals[mid] < v)
        lo = mid + 1;
      else
        hi = mid;
    }
    key[i] = ((u64)(unsigned)lo << 32) | (k & 0xffffffffull);
  }
}

__global__ void k_init_state(int *rep, int *sz, int64_t N) {
  pdl_wait();
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < N) {
    rep[i] = (int)i;
    sz[i] = 1;
  }
}

}  // namespace
}  // namespace ragb
