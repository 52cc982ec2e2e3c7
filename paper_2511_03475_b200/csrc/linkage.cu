// a5 on sm_100a: complete-linkage agglomerative clustering of the Eq. 1 rows.
//
// PAPER:335 (Section 4.1 "Index creation"): "we iteratively merge the closest
// pair, creating a virtual node".  Readings: complete linkage
// D(A u B, C) = max(D(A,C), D(B,C)) (X7), tie key (D, min rep, max rep) with
// rep = smallest leaf index (X8), merge order = ascending key (X9).
//
// Algorithm: level-synchronous rounds over a compacted active matrix.  A round
// starts from every active row's nearest-neighbour key (the fused row min of
// the previous pass, or of the distance kernel in round 0) and merges, in one
// batch, (1) every merge the greedy algorithm performs at the current minimum
// height h, and (2) every reciprocal-nearest-neighbour pair above h:
//   (1) at height h the greedy process is a sequence of clique contractions on
//       the graph of pairs at distance exactly h: take the smallest vertex a with
//       an h-neighbour, absorb its smallest h-neighbour b, keep the candidates
//       adjacent to every absorbed vertex (max stays h only if both are h), and
//       continue; then the next vertex.  This is done by one CTA (k_round_prep).
//   (2) RNN pairs above h are merges of the unique reducible hierarchy and are
//       disjoint from (1) (a vertex with an h-neighbour has its NN at h).
// Then one fused pass (k_merge_rows) writes the merged, order-preserving
// compacted matrix (max over group members) and the new row-min keys.  Because
// compaction preserves order and a group's survivor is its smallest member,
// compacted index order == rep order, so the row key (d bits << 32 | column)
// orders candidates exactly like the X8 tie key.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <functional>
#include <map>
#include <mutex>
#include <tuple>
#include <vector>

#include "internal.h"

#include "linkage_kernels.cuh"

namespace ragb {
namespace {

template <typename T>
T *at(void *base, size_t off) {
  return reinterpret_cast<T *>(static_cast<unsigned char *>(base) + off);
}

// Launch configuration cache: the dynamic shared-memory opt-in is set once
// per kernel (to the largest size requested so far) and occupancy is queried
// once per (kernel, block, shared-memory) triple — both are host round trips
// into the driver that otherwise sit between a round's counter read and its
// launches (measured: ~0.3 ms per round at small N).
template <typename F>
int occupancy_cached(F kern, int nth, size_t smem) {
  static std::mutex mu;
  static std::map<std::tuple<const void *, int, size_t>, int> occ;
  static std::map<const void *, size_t> attr;
  const void *key = reinterpret_cast<const void *>(kern);
  std::lock_guard<std::mutex> lk(mu);
  size_t &a = attr[key];
  if (smem > a) {
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
      return 0;  // the launch would fail: the caller reports it
    a = smem;
  }
  auto it = occ.find({key, nth, smem});
  if (it != occ.end()) return it->second;
  int per_sm = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, nth, smem);
  per_sm = std::max(per_sm, 1);
  occ[{key, nth, smem}] = per_sm;
  return per_sm;
}

// Dynamic shared memory a kernel may opt into: the per-block opt-in limit
// minus the kernel's static shared memory (the static part counts
// against the same 227 KB).
template <typename F>
size_t dyn_smem_limit(F kern) {
  static std::mutex mu;
  static std::map<const void *, size_t> lim;
  const void *key = reinterpret_cast<const void *>(kern);
  std::lock_guard<std::mutex> lk(mu);
  auto it = lim.find(key);
  if (it != lim.end()) return it->second;
  int dev = 0, optin = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  cudaFuncAttributes fa{};
  cudaFuncGetAttributes(&fa, kern);
  const size_t l = (size_t)optin > fa.sharedSizeBytes ? (size_t)optin - fa.sharedSizeBytes : 0;
  lim[key] = l;
  return l;
}

// Compaction launch for element type T (see k_merge_rows): wide rows get
// 1024-thread CTAs, one per SM, with a window of up to 56K columns; narrow
// rows 256-thread CTAs so that several rows are in flight per SM.
// The code-mode compaction kernel with the compact map (k_merge_gather2) for
// this round, or nullptr when another form runs (launch_merge).
typedef void (*Gather2Fn)(const uint16_t *, int64_t, int, const int *, const int *, const int *, const uint32_t *,
                          const int *, uint16_t *, u64 *, int, SideBuf);
template <typename T>
Gather2Fn gather2_kernel(const void *cur, int64_t ld, int M, int Mn, const PrepArgs &pa, const Tuning &tu, bool *mid_out) {
  const size_t row_bytes = (size_t)((M + 7) / 8) * 16;
  const bool vec16 = ld % 8 == 0 && (reinterpret_cast<uintptr_t>(cur) & 15) == 0;
  const bool wide16 = M > 16 * 1024;
  const bool compact = sizeof(T) == 2 && pa.pmap && pa.nclq && pm32_fits(M, Mn);  // k_compact_maps wrote pm32
  if (!compact || tu.gather == 0) return nullptr;
  // rows that fit twice in half the shared memory (M <= ~28K): two 512-thread
  // CTAs per SM, each double-buffered
  const bool mid = wide16 && vec16 && 4 * row_bytes + 4096 <= 227 * 1024 && tu.gather != 2;
  Gather2Fn kern = mid ? k_merge_gather2<true, 512>
                       : wide16 ? (vec16 ? k_merge_gather2<true, 1024> : k_merge_gather2<false, 1024>)
                                : (vec16 ? k_merge_gather2<true, 256> : k_merge_gather2<false, 256>);
  if (row_bytes > dyn_smem_limit(kern)) return nullptr;
  if (mid_out) *mid_out = mid;
  return kern;
}

template <typename T>
cudaError_t launch_merge(const T *cur, int64_t ld, int M, int Mn, const PrepArgs &pa, int sms, T *next,
                         unsigned long long *keyn, cudaStream_t st, const Tuning &tu, unsigned *paths,
                         const SideBuf &patch) {
  constexpr int VW = Elem<T>::VW;
  const size_t row_bytes = (size_t)((M + 7) / 8) * 16;
  const bool vec16 = ld % 8 == 0 && (reinterpret_cast<uintptr_t>(cur) & 15) == 0;
  const bool wide16 = M > 16 * 1024;
  auto gkern = wide16 ? (vec16 ? k_merge_gather<true, 1024> : k_merge_gather<false, 1024>)
                      : (vec16 ? k_merge_gather<true, 256> : k_merge_gather<false, 256>);
  const bool compact = sizeof(T) == 2 && pa.pmap && pa.nclq && pm32_fits(M, Mn);  // k_compact_maps wrote pm32
  bool mid = false;
  if (Gather2Fn kern = gather2_kernel<T>(cur, ld, M, Mn, pa, tu, &mid)) {
    // code mode with the compact map: k_merge_gather2 (the old row fits)
    const size_t lim = dyn_smem_limit(kern);
    {
      const int db = vec16 && 2 * row_bytes <= lim ? 1 : 0;  // double-buffered rows
      const size_t smem = row_bytes * (1 + db);
      const int nth = mid ? 512 : wide16 ? 1024 : 256;
      const int per_sm = occupancy_cached(kern, nth, smem);
      if (per_sm < 1) return cudaErrorInvalidConfiguration;
      *paths |= wide16 ? RB_PATH_GATHER_WIDE : RB_PATH_GATHER;
      const int grid = std::min<int>(Mn, sms * per_sm);
      launch_pdl(kern, grid, nth, smem, st, reinterpret_cast<const uint16_t *>(cur), ld, M, (const int *)pa.Mn,
                 (const int *)pa.goff, (const int *)pa.gmem, reinterpret_cast<const uint32_t *>(pa.pmap),
                 (const int *)pa.nclq, reinterpret_cast<uint16_t *>(next), keyn, db, patch);
      return cudaGetLastError();
    }
  }
  const size_t glim = sizeof(T) == 2 && pa.pmap && !compact ? dyn_smem_limit(gkern) : 0;
  if (patch.T) return cudaErrorInvalidValue;  // dirty columns only through k_merge_gather2 (the caller flushes)
  if (sizeof(T) == 2 && pa.pmap && !compact && row_bytes <= glim && tu.gather != 0) {
    // code mode, old row fits in shared memory: gather form (k_merge_gather)
    const uint16_t *c16 = reinterpret_cast<const uint16_t *>(cur);
    uint16_t *n16 = reinterpret_cast<uint16_t *>(next);
    const int db = vec16 && 2 * row_bytes <= glim ? 1 : 0;  // double-buffered rows
    const size_t smem = row_bytes * (1 + db);
    auto kern = gkern;
    const int nth = wide16 ? 1024 : 256;
    const int per_sm = occupancy_cached(kern, nth, smem);
    if (per_sm < 1) return cudaErrorInvalidConfiguration;
    *paths |= wide16 ? RB_PATH_GATHER_WIDE : RB_PATH_GATHER;
    const int grid = std::min<int>(Mn, sms * per_sm);
    kern<<<grid, nth, smem, st>>>(c16, ld, M, pa.Mn, pa.goff, pa.gmem, pa.pmap, n16, keyn, db);
    return cudaGetLastError();
  }
  const bool vec = ld % VW == 0 && (reinterpret_cast<uintptr_t>(cur) & 15) == 0;
  const bool wide = Mn > 20 * 1024;
  const int es = (int)sizeof(typename Win<T>::S);  // window element bytes
  const int maxW = wide ? 224 * 1024 / es : 20 * 1024;
  const int W = std::min<int>((Mn + VW - 1) / VW * VW, maxW);
  const size_t smem = (size_t)W * es;
  const int nth = wide ? 1024 : 256;
  auto kern = wide ? (vec ? k_merge_rows<true, 1024, T, LocalRows<T>> : k_merge_rows<false, 1024, T, LocalRows<T>>)
                   : (vec ? k_merge_rows<true, 256, T, LocalRows<T>> : k_merge_rows<false, 256, T, LocalRows<T>>);
  const int per_sm = occupancy_cached(kern, nth, smem);
  if (per_sm < 1) return cudaErrorInvalidConfiguration;
  *paths |= wide ? RB_PATH_WINDOW_WIDE : RB_PATH_WINDOW;
  const int grid = std::min<int>(Mn, sms * per_sm);
  kern<<<grid, nth, smem, st>>>(LocalRows<T>{cur, ld}, M, pa.Mn, pa.goff, pa.gmem, pa.colsrc, pa.cursor, W, 0, -1,
                                next, keyn);
  return cudaGetLastError();
}

// In-place round for element type T (see k_inplace_*).  With a side buffer
// (sb.T, code mode) the survivors' columns go to it instead of the matrix.
template <typename T>
cudaError_t launch_inplace(T *cur, int64_t ld, int M, int max_groups, const PrepArgs &pa, int sms, uint32_t *amask,
                           int *mlist, int *nmulti, int *sz, unsigned long long *key, const SideBuf &sb,
                           const NNCache &nc, cudaStream_t st, int *launches) {
  constexpr int VW = Elem<T>::VW;
  launch_pdl(k_inplace_prep, sms * 2, 256, 0, st, pa, M, amask, mlist, nmulti, sz, key, sb, nc);
  const size_t smem = (size_t)((M + VW - 1) / VW) * 16;
  if constexpr (sizeof(T) == 2) {
    if (sb.T) {
      const size_t smem2 = smem + (size_t)sb.cap * 2;
      occupancy_cached(k_inplace_rows_sb<512>, 512, smem2);
      launch_pdl(k_inplace_rows_sb<512>, sms * 2, 512, smem2, st, pa, cur, ld, M, amask, mlist, nmulti, key, sb);
      launch_pdl(k_side_tpose, dim3((unsigned)((M + 63) / 64), (unsigned)((std::max(max_groups, 1) + 31) / 32)), 256, 0,
                 st, pa, static_cast<const uint16_t *>(cur), ld, M, mlist, nmulti, sb);
      launch_pdl(k_side_maps, 1, 1024, 0, st, pa, mlist, nmulti, sb);
      *launches += 3;
    }
  }
  if (!sb.T) {
    occupancy_cached(k_inplace_rows<512, T>, 512, smem);
    k_inplace_rows<512, T><<<sms * 2, 512, smem, st>>>(pa, cur, ld, M, amask, mlist, nmulti, key);
    k_inplace_cols<T><<<dim3((unsigned)std::max(max_groups, 1), (unsigned)((M + kColsRows - 1) / kColsRows)), 256,
                        0, st>>>(pa, cur, ld, M, amask, mlist, nmulti);
    *launches += 2;
  }
  launch_pdl(k_inplace_check<T>, (M + 255) / 256, 256, 0, st, pa, cur, ld, M, key, pa.cnt, nmulti + 1, sb,
             nc);  // cnt: free after the compaction map
  {
    const size_t rs = (size_t)(((M / 32 + 1) + 3) & ~3) * 4 + (size_t)(sb.T ? sb.cap : 0) * 4;  // scan mask + slot columns
    occupancy_cached(k_inplace_rescan<256, T>, 256, rs);
    launch_pdl(k_inplace_rescan<256, T>, sms * 4, 256, rs, st, cur, ld, M, amask, pa.cnt, nmulti + 1, key, sb, nc);
  }
  *launches += 3;
  return cudaGetLastError();
}

// Side buffer state back to clean (after a flush, or at the start).
cudaError_t side_reset(const SideBuf &sb, int M, cudaStream_t st) {
  cudaError_t e;
  if ((e = cudaMemsetAsync(sb.tslot, 0xff, (size_t)M * 4, st)) != cudaSuccess) return e;
  if ((e = cudaMemsetAsync(sb.dmask, 0, (size_t)(M / 32 + 1) * 4, st)) != cudaSuccess) return e;
  return cudaMemsetAsync(sb.nt, 0, 4, st);
}

}  // namespace

cudaError_t run_linkage(float *rows, int64_t N, unsigned long long *nnkey, void *scratch,
                        const ScratchLayout &L, bool keep_rows, const CodeMode *cm, cudaStream_t st,
                        int32_t *za, int32_t *zb, float *zh, int32_t *zs, LinkageOut *out, int *launches,
                        const std::function<void(int64_t)> &on_round, const Tuning &tu) {
  out->rounds = 0;
  if (N <= 1) return cudaSuccess;
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  // Code mode (cm != nullptr): the matrices hold 16-bit order-preserving codes
  // of the Eq. 1 values (written by the distance kernel next to the fp32 rows)
  // instead of the values: half the bytes per round, same merges (max and
  // compare commute with an order-preserving map).  Round keys become code
  // keys; heights are decoded through cm->vals.
  const bool codes = cm != nullptr;

  u64 *key[2] = {nnkey, at<u64>(scratch, L.key1)};
  int *rep[2] = {at<int>(scratch, L.rep0), at<int>(scratch, L.rep1)};
  int *sz[2] = {at<int>(scratch, L.sz0), at<int>(scratch, L.sz1)};
  // float mode: rows -> matA -> matB (or rows) -> ...; code mode: codes ->
  // mat16 -> codes -> ... (the fp32 rows are never touched)
  void *matA = codes ? static_cast<void *>(cm->mat16) : at<void>(scratch, L.matA);
  void *matB = codes ? static_cast<void *>(cm->codes) : (keep_rows ? at<void>(scratch, L.matB) : static_cast<void *>(rows));
  int *counters = at<int>(scratch, L.counters);  // [0] zcount, [1] Mn
  cudaError_t e;
  launch_pdl(k_init_state, (unsigned)((N + 255) / 256), 256, 0, st, rep[0], sz[0], N);
  ++*launches;
  if ((e = cudaMemsetAsync(counters, 0, 16 * sizeof(int), st)) != cudaSuccess) return e;

  PrepArgs pa{};
  pa.leader = at<int>(scratch, L.leader);
  pa.alive = at<uint8_t>(scratch, L.alive);
  pa.newidx = at<int>(scratch, L.aux0);
  pa.goff = at<int>(scratch, L.aux1);
  pa.gmem = at<int>(scratch, L.aux2);
  pa.colsrc = at<int>(scratch, L.aux3);
  pa.cnt = at<int>(scratch, L.aux4);
  pa.cursor = pa.cnt + N;
  pa.list = pa.goff;
  pa.candA = pa.gmem;
  pa.candB = pa.colsrc;
  pa.za = at<int>(scratch, L.za);
  pa.zb = at<int>(scratch, L.zb);
  pa.zs = at<int>(scratch, L.zs);
  pa.zh = at<float>(scratch, L.zh);
  pa.zcount = counters;
  pa.Mn = counters + 1;
  pa.level = counters + 2;
  pa.sweep_ctl = counters + 14;  // 0 between launches (reset by the sweep's CTA 0)
  pa.nclq = codes ? counters + 15 : nullptr;
  pa.lpos = pa.newidx;  // free between the level list and the compaction map
  pa.cstat = counters + 4;
  pa.vals = codes ? cm->vals : nullptr;
  pa.pmap = codes ? at<int2>(scratch, L.pmap) : nullptr;
  if (codes) {
    launch_pdl(k_keys_to_codes, sms, 256, 0, st, nnkey, N, cm->vals, cm->ncode);
    ++*launches;
  }

  void *cur = codes ? static_cast<void *>(cm->codes) : static_cast<void *>(rows);
  int64_t ld = N;
  int M = (int)N;   // rows of the current matrix (live + dead)
  int live = (int)N;  // live clusters
  bool mask_ok = false;  // alive mask valid for the current matrix
  uint32_t *amask = at<uint32_t>(scratch, L.amask);
  int *mlist = at<int>(scratch, L.mlist);
  int *nmulti = counters + 12;
  int p = 0;
  void *next = matA;
  // per-round timing on stderr (diagnostics only)
  const bool trace = tu.trace == 1;
  // trace 2: per-round events and host timestamps only (no extra syncs),
  // printed once at the end (jitter diagnostics)
  const bool ltrace = tu.trace == 2;
  struct LRound {
    cudaEvent_t e[3];
    double h0, h1, h2;  // host: round top, sync returned, round bottom (ms)
  };
  std::vector<LRound> lr;
  const auto lt0 = std::chrono::steady_clock::now();
  cudaEvent_t lte[2];  // entry, after the last round
  if (ltrace) {
    for (auto &x : lte) cudaEventCreate(&x);
    cudaEventRecord(lte[0], st);
  }
  auto lnow = [&] { return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - lt0).count(); };
  // in-place rounds: 0 never, 1 wherever allowed (testing), -1 cost model
  const int inplace_mode = tu.inplace < 0 ? 2 : tu.inplace;
  const double inplace_w = tu.inplace_weight;  // cost-model weight of a merge (row equivalents)
  cudaEvent_t tev[3];
  if (trace)
    for (auto &x : tev) cudaEventCreate(&x);
  int zprev = 0;
  int zdone = 0;
  std::vector<cudaEvent_t> mev;  // [start, end] per compaction launch (merge_ms)
  // In-place side buffer (code mode): T after the level adjacency in the free
  // code-matrix region (`next` is untouched by in-place rounds); maps in scratch.
  SideBuf sb{};
  sb.tcol = at<int>(scratch, L.tcol);
  sb.tslot = at<int>(scratch, L.tslot);
  sb.dmask = at<uint32_t>(scratch, L.dmask);
  sb.nt = at<int>(scratch, L.tctl);
  int sb_used = 0;  // host upper bound of the slots in use (merges of the in-place rounds since the last flush)
  // second-nearest cache of the in-place rounds (valid for the current matrix
  // numbering: cleared after every compaction)
  NNCache nc{};
  if (tu.nn_cache != 0) {
    nc.key2 = at<u64>(scratch, L.nnkey2);
    nc.kround = at<int>(scratch, L.nnround);
    nc.ver = at<int>(scratch, L.colver);
  }
  auto nc_reset = [&](int Mc) -> cudaError_t {
    if (!nc.key2) return cudaSuccess;
    cudaError_t e2 = cudaMemsetAsync(nc.kround, 0, (size_t)Mc * 4, st);
    return e2 != cudaSuccess ? e2 : cudaMemsetAsync(nc.ver, 0, (size_t)Mc * 4, st);
  };
  if ((e = nc_reset((int)N)) != cudaSuccess) return e;
  if (codes && (e = side_reset(sb, (int)N, st)) != cudaSuccess) return e;
  auto side_for = [&](int Mc, void *nx) {  // the side buffer for a matrix of Mc rows with `nx` free
    SideBuf b = sb;
    b.T = nullptr;
    b.cap = 0;
    if (!codes || tu.side_buffer == 0) return b;
    // the level adjacency (n x W words, n <= Mc) and the clique sweep's work
    // area after it (k_level_cliques: I [n][W rounded to 4], 6 arrays of n
    // ints, the per-block decision logs) come first
    const size_t W4 = (size_t)(((Mc + 31) / 32 + 3) & ~3);
    const size_t adj_bytes = ((2 * (size_t)Mc * W4 * 4 + 16 * ((size_t)Mc + 1024) * 4) + 255) & ~(size_t)255;
    const size_t region = code_mat_bytes(N);
    if (region <= adj_bytes) return b;
    const int64_t cap = std::min<int64_t>(kSideCap, (int64_t)((region - adj_bytes) / (2 * (size_t)Mc))) & ~7ll;
    if (cap < 64) return b;
    b.T = reinterpret_cast<uint16_t *>(static_cast<unsigned char *>(nx) + adj_bytes);
    b.cap = (int)cap;
    return b;
  };
  auto side_flush = [&](void *cm_, int64_t ld_, int Mc, void *nx) -> cudaError_t {
    if (sb_used == 0) return cudaSuccess;
    const SideBuf b = side_for(Mc, nx);
    const size_t smem = (size_t)((Mc + 7) / 8) * 16 + (size_t)b.cap * 4;
    occupancy_cached(k_side_flush, 256, smem);
    k_side_flush<<<sms * 4, 256, smem, st>>>(static_cast<uint16_t *>(cm_), ld_, Mc, b);
    ++*launches;
    sb_used = 0;
    return side_reset(sb, Mc, st);
  };
  while (live > 1) {
    if (ltrace) {
      lr.emplace_back();
      for (auto &x : lr.back().e) cudaEventCreate(&x);
      lr.back().h0 = lnow();
      cudaEventRecord(lr.back().e[0], st);
    }
    if (trace) {
      cudaMemsetAsync(counters + 4, 0, 8 * sizeof(int), st);
      cudaEventRecord(tev[0], st);
    }
    pa.D = cur;
    pa.ld = ld;
    pa.M = M;
    pa.key = key[p];
    pa.rep = rep[p];
    pa.sz = sz[p];
    pa.rep_n = rep[p ^ 1];
    pa.sz_n = sz[p ^ 1];
    launch_prep_mark(pa, sms, st, launches);
    uint32_t *adj = reinterpret_cast<uint32_t *>(next);  // free until the merge writes it
    {
      // level rows streamed whole (k_level_adj_rows); W words of bits per row
      // in shared memory (the level has at most M vertices)
      const bool vec = ld % (codes ? 8 : 4) == 0 && (reinterpret_cast<uintptr_t>(cur) & 15) == 0;
      const size_t smem = (size_t)((M + 31) / 32) * 12;  // row bits, level mask, mask prefix
      const int grid = std::min(M, sms * 8);
      if (codes) {
        // dirty columns (side buffer in use) need the vector path, which in-place rounds guarantee
        const SideBuf b = sb_used > 0 ? side_for(M, next) : SideBuf{};
        auto kern = vec ? k_level_adj_rows<uint16_t, true> : k_level_adj_rows<uint16_t, false>;
        if (smem > 48 * 1024) occupancy_cached(kern, 256, smem);
        launch_pdl(kern, grid, 256, smem, st, pa, adj, b);
      } else {
        auto kern = vec ? k_level_adj_rows<float, true> : k_level_adj_rows<float, false>;
        if (smem > 48 * 1024) occupancy_cached(kern, 256, smem);
        kern<<<grid, 256, smem, st>>>(pa, adj, SideBuf{});
      }
    }
    {
      const size_t m1 = std::min<size_t>((size_t)M, (size_t)std::min(1024, kWarpCliqueMaxN));  // staged only on the warp path
      const size_t smem = m1 * ((m1 + 31) / 32) * 4;  // the staged adjacency of levels <= 1024
      if (smem > 48 * 1024)
        occupancy_cached(k_level_cliques, CT, smem);
      // CTA 0 decides; with a level above 4096 vertices the other CTAs
      // (one per SM, all resident) update the clique candidate sets
      launch_pdl(k_level_cliques, std::min(sms, 1 + kSweepHelpers), CT, smem, st, pa, adj);
    }
    launch_prep_compact(pa, sms, st, launches);
    *launches += 2;
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    if (trace) cudaEventRecord(tev[1], st);
    if (ltrace) cudaEventRecord(lr.back().e[1], st);
    int host_c[12] = {0};
    if ((e = cudaMemcpyAsync(host_c, counters, (trace ? 12 : 3) * sizeof(int), cudaMemcpyDeviceToHost, st)) !=
        cudaSuccess)
      return e;
    if ((e = cudaStreamSynchronize(st)) != cudaSuccess) return e;
    if (ltrace) lr.back().h1 = lnow();
    ++out->rounds;
    {  // this round's merges to the host, then let the host tree catch up
      const int z0 = zdone, z1 = host_c[0];
      if (z1 > (int)N - 1 || z1 < z0) return cudaErrorUnknown;
      if (z1 > z0) {
        if (on_round) {
          // the caller's worker thread fetches merges [.., z1) itself (they
          // are final: device rows only ever get appended) while this thread
          // goes on launching the next kernels
          on_round(z1);
        } else {
          const size_t n = (size_t)(z1 - z0);
          cudaMemcpyAsync(za + z0, pa.za + z0, n * 4, cudaMemcpyDeviceToHost, st);
          cudaMemcpyAsync(zb + z0, pa.zb + z0, n * 4, cudaMemcpyDeviceToHost, st);
          cudaMemcpyAsync(zh + z0, pa.zh + z0, n * 4, cudaMemcpyDeviceToHost, st);
          if ((e = cudaMemcpyAsync(zs + z0, pa.zs + z0, n * 4, cudaMemcpyDeviceToHost, st)) != cudaSuccess)
            return e;
          if ((e = cudaStreamSynchronize(st)) != cudaSuccess) return e;
        }
        zdone = z1;
      }
    }
    const int Mn = host_c[1];
    if (Mn >= live || Mn < 1) return cudaErrorUnknown;  // no progress: invariant violated
    out->max_level = std::max(out->max_level, host_c[2]);
    if (host_c[2] >= 2) out->paths |= host_c[2] <= kWarpCliqueMaxN ? RB_PATH_CLIQUE_WARP : RB_PATH_CLIQUE_BLOCK;
    const int merges_round = host_c[0] - zprev;
    zprev = host_c[0];
    // in place when the merged rows, the rewritten columns (one scattered
    // 4-byte store per row and merge, ~30 row-equivalents per merge measured)
    // and the rescans cost less than rewriting the matrix (~live + Mn^2/M rows)
    const int ivw = codes ? Elem<uint16_t>::VW : Elem<float>::VW;  // in-place kernels: 16-byte row vectors
    const bool inplace = Mn > 1 && (codes || !keep_rows || cur != static_cast<void *>(rows)) && ld % ivw == 0 && (reinterpret_cast<uintptr_t>(cur) & 15) == 0 && M <= kInplaceMaxM && inplace_mode != 0 &&
                         (inplace_mode == 1 || inplace_w * merges_round < (double)live + (double)Mn * Mn / M);
    if (inplace) {
      if (!mask_ok) {
        if ((e = cudaMemsetAsync(amask, 0xff, (size_t)(M / 32 + 1) * 4, st)) != cudaSuccess) return e;
        mask_ok = true;
      }
      if ((e = cudaMemsetAsync(nmulti, 0, 8, st)) != cudaSuccess) return e;  // nmulti, nres
      SideBuf b = side_for(M, next);
      if (b.T && sb_used + merges_round > b.cap && (e = side_flush(cur, ld, M, next)) != cudaSuccess) return e;
      if (b.T && merges_round > b.cap) b.T = nullptr;  // more survivors than slots: columns rewritten in place
      if (!b.T && sb_used > 0 && (e = side_flush(cur, ld, M, next)) != cudaSuccess) return e;
      if (b.T) sb_used += merges_round;  // merged groups <= merges of the round
      // merged groups <= merges of the round (the grid of the column kernel)
      nc.round = out->rounds;
      e = codes ? launch_inplace<uint16_t>(static_cast<uint16_t *>(cur), ld, M, merges_round, pa, sms, amask, mlist,
                                           nmulti, sz[p], key[p], b, nc, st, launches)
                : launch_inplace<float>(static_cast<float *>(cur), ld, M, merges_round, pa, sms, amask, mlist, nmulti,
                                        sz[p], key[p], SideBuf{}, nc, st, launches);
      ++*launches;
      out->paths |= RB_PATH_INPLACE;
      if (e != cudaSuccess) return e;
    } else if (Mn > 1) {
      // dirty columns of the side buffer: patched into the staged old rows by
      // k_merge_gather2 when it runs and its output stays clear of the buffer
      // (it is written into the same free region), else flushed first
      SideBuf patch{};
      if (sb_used > 0) {
        const SideBuf b = side_for(M, next);
        const size_t new_bytes = (size_t)Mn * (size_t)mat_ld<uint16_t>(Mn) * 2;
        if (codes && b.T && gather2_kernel<uint16_t>(cur, ld, M, Mn, pa, tu, nullptr) &&
            new_bytes <= (size_t)(reinterpret_cast<unsigned char *>(b.T) - static_cast<unsigned char *>(next)))
          patch = b;
        else if ((e = side_flush(cur, ld, M, next)) != cudaSuccess)
          return e;
      }
      cudaEvent_t me[2];
      cudaEventCreateWithFlags(&me[0], cudaEventDefault);
      cudaEventCreateWithFlags(&me[1], cudaEventDefault);
      cudaEventRecord(me[0], st);
      e = codes ? launch_merge<uint16_t>(static_cast<const uint16_t *>(cur), ld, M, Mn, pa, sms,
                                         static_cast<uint16_t *>(next), key[p ^ 1], st, tu, &out->paths, patch)
                : launch_merge<float>(static_cast<const float *>(cur), ld, M, Mn, pa, sms, static_cast<float *>(next),
                                      key[p ^ 1], st, tu, &out->paths, patch);
      if (e == cudaSuccess && patch.T) {  // the side buffer was consumed by the compaction
        sb_used = 0;
        e = side_reset(sb, M, st);
      }
      cudaEventRecord(me[1], st);
      mev.push_back(me[0]);
      mev.push_back(me[1]);
      const double es = codes ? 2.0 : 4.0;
      out->merge_bytes += es * ((double)live * live + (double)Mn * Mn);
      ++out->merge_launches;
      ++*launches;
      if (e != cudaSuccess) return e;
      cur = next;
      next = (next == matA) ? matB : matA;
      ld = codes ? mat_ld<uint16_t>(Mn) : mat_ld<float>(Mn);  // padded leading dimension of the new matrix
      mask_ok = false;
      if ((e = nc_reset(Mn)) != cudaSuccess) return e;  // new column numbering
    }
    if (ltrace) {
      cudaEventRecord(lr.back().e[2], st);
      lr.back().h2 = lnow();
    }
    if (trace) {
      cudaEventRecord(tev[2], st);
      cudaEventSynchronize(tev[2]);
      float a = 0, b = 0;
      cudaEventElapsedTime(&a, tev[0], tev[1]);
      cudaEventElapsedTime(&b, tev[1], tev[2]);
      int ires[2] = {0, 0};  // in-place rounds: merged groups, rescanned rows
      if (inplace) cudaMemcpy(ires, counters + 12, 8, cudaMemcpyDeviceToHost);
      if (inplace) std::fprintf(stderr, "[ragb linkage]   inplace groups=%d rescans=%d\n", ires[0], ires[1]);
      std::fprintf(stderr,
                   "[ragb linkage] round %d M=%d live=%d Mn=%d merges=%d %s prep=%.3fms merge=%.3fms | level n=%d "
                   "starts=%d batches=%d picks=%d cands=%d kclk w0=%d pass=%d collect=%d\n",
                   out->rounds, M, live, Mn, merges_round, inplace ? "inplace" : "compact", a, b, host_c[8],
                   host_c[4], host_c[5], host_c[6], host_c[7], host_c[9], host_c[10], host_c[11]);
    }
    if (!inplace) {
      p ^= 1;
      M = Mn;
    }
    live = Mn;
  }
  if (trace)
    for (auto &x : tev) cudaEventDestroy(x);
  if (ltrace) cudaEventRecord(lte[1], st);
  cudaStreamSynchronize(st);
  if (ltrace) {
    float a = 0, b = 0;
    if (!lr.empty()) {
      cudaEventElapsedTime(&a, lte[0], lr[0].e[0]);
      cudaEventElapsedTime(&b, lr.back().e[2], lte[1]);
    }
    std::fprintf(stderr, "[ragb lt] setup=%.3f tail=%.3f host_end=%.3f\n", a, b, lnow());
    for (auto &x : lte) cudaEventDestroy(x);
    for (size_t i = 0; i < lr.size(); ++i) {
      float a = 0, b = 0, g = 0;
      cudaEventElapsedTime(&a, lr[i].e[0], lr[i].e[1]);
      cudaEventElapsedTime(&b, lr[i].e[1], lr[i].e[2]);
      if (i + 1 < lr.size()) cudaEventElapsedTime(&g, lr[i].e[2], lr[i + 1].e[0]);
      std::fprintf(stderr, "[ragb lt] %zu prep=%.3f merge=%.3f gap=%.3f | host top=%.3f sync=%.3f bottom=%.3f\n", i, a,
                   b, g, lr[i].h0, lr[i].h1, lr[i].h2);
    }
    for (auto &r : lr)
      for (auto &x : r.e) cudaEventDestroy(x);
  }
  for (size_t i = 0; i + 1 < mev.size(); i += 2) {
    float ms = 0.f;
    cudaEventElapsedTime(&ms, mev[i], mev[i + 1]);
    out->merge_ms += ms;
  }
  for (auto &x : mev) cudaEventDestroy(x);
  if (zdone != N - 1) return cudaErrorUnknown;
  return cudaSuccess;
}

}  // namespace ragb
