// a2-a4 fast path on sm_100a: every context has exactly K <= 32 docs (the
// paper's setting: a retriever returns top-K lists).  Eq. 1 from
// exact integer counts (X2, X3, X6); one persistent CTA of 512 threads per SM.
//
//  * Row tile: R = 64 (or 32) rows.  Their docs go into a shared-memory hash
//    table (doc -> count, offset into a (row, position) list) and a
//    2^16-bit filter, built once per tile.
//  * Column chunks of 512 contexts; warp w owns columns [32w, 32w + 32) of
//    every chunk for all R rows, and streams their docs through its own
//    two-stage shared-memory ring: the TMA engine (cp.async.bulk, one 128-byte
//    copy per k from the transposed [K][Npad] ids, issued by K lanes) fills
//    one stage while the warp works on the other.  Warps never wait for each
//    other inside a tile.
//  * Per chunk a warp runs: the probe (lane = column: K filter tests on the
//    staged docs), the candidate queue, the drain and the finalize, all on
//    its own accumulator columns.  Drain: lanes take 32 candidates, look
//    their doc up in the tile table and count its rows; then lanes take the
//    (row, column) incidences of those candidates 32 at a time (load-balanced
//    by a prefix sum: popular docs in many rows no longer serialise a lane)
//    and add
//    S + |p_i - p_j| with one shared-memory atomicAdd into packed 16-bit
//    accumulators: the sum over the shared docs is s * S + D, the index of
//    d(s, D) in a table with stride S = floor(K^2 / 2) + 1.
//  * Finalize: a lane owns 4 consecutive columns of every 4th row; one
//    8-byte table entry per distance holds (fp32 value, 16-bit code << 16),
//    so a 4-column step is one 8-byte accumulator load, four table loads, one
//    16-byte fp32 store, one 8-byte code store and the running row minimum
//    (code << 16 | column sequence: codes order like the values, so the
//    strict minimum keeps the smallest column, X8).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>

#include "device_util.cuh"
#include "internal.h"

namespace ragb {
namespace {

constexpr int NT = 512;       // threads per CTA
constexpr int NW = NT / 32;   // warps per CTA
constexpr int CH = 512;       // columns per chunk (32 per warp)
constexpr int FWORDS = 2048;  // filter words (65536 bits)
constexpr int ACCW = CH / 2 + 16;  // accumulator words per row (+64 B: rows r, r+1 on different banks)
constexpr int QCAP = 256;     // candidate-queue window per warp (entries); drained as often as needed

typedef unsigned long long u64;

struct Plan {
  int R, T, logT, S, K, nseg;
  bool tab_smem, scale8;
  size_t off_tab, off_acc, off_stage, off_key, off_cb, off_plist, off_filter, off_q, off_inc, off_bar, total;
};

// Packed Eq. 1 table for the tile kernel: ptab[s * S + D] = (bits of d(s, D),
// code << 16) from the shift-layout value / code tables (same values: the
// correctly rounded Eq. 1 of k_eq1_lut, the order-preserving codes of
// k_code_table).
__global__ void k_pack_table(const float *__restrict__ lut, const uint32_t *__restrict__ lutc, int K, int shift,
                             int S, uint2 *__restrict__ ptab) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (K + 1) * S) return;
  const int s = i / S, D = i - s * S;
  const int e = (s << shift) + D;
  ptab[i] = make_uint2(__float_as_uint(lut[e]), lutc[e] << 16);
}

template <int R, bool SCALE8, bool TAB_SMEM, bool CODES>
__global__ void __launch_bounds__(NT, 1) k_dist_tile(DistArgs a, Plan P) {
  extern __shared__ __align__(128) unsigned char smem[];
  // the table first: its entries are addressed by the packed accumulator alone
  const uint2 *tab = TAB_SMEM ? reinterpret_cast<const uint2 *>(smem) : a.ptab;
  uint32_t *acc = reinterpret_cast<uint32_t *>(smem + P.off_acc);      // [R][ACCW] packed 2 x u16
  uint32_t *stg = reinterpret_cast<uint32_t *>(smem + P.off_stage);    // [NW][2][K][32] column docs
  uint32_t *tkey = reinterpret_cast<uint32_t *>(smem + P.off_key);     // [T] buckets of 4 docs
  uint32_t *tcb = reinterpret_cast<uint32_t *>(smem + P.off_cb);       // [T] count << 16 | row-list base
  uint16_t *plist = reinterpret_cast<uint16_t *>(smem + P.off_plist);  // [R*K] row << 5 | position
  uint32_t *filt = reinterpret_cast<uint32_t *>(smem + P.off_filter);  // [FWORDS]
  uint16_t *qall = reinterpret_cast<uint16_t *>(smem + P.off_q);       // [NW][QCAP]
  uint2 *cinfo_all = reinterpret_cast<uint2 *>(smem + P.off_inc);      // [NW][32] (start | base << 16, k | col << 8)
  u64 *full = reinterpret_cast<u64 *>(smem + P.off_bar);               // [NW][2] ring stages filled

  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int K = a.K, NB = P.T >> 2, logNB = P.logT - 2;
  const int64_t N = a.N, Npad = a.Npad;
  const int64_t ntiles = (a.nrows + R - 1) / R;
  const int nch = (int)((N + CH - 1) / CH);
  // work units: row tile x column segment (nseg segments of cps chunks; more
  // units than CTAs x waves keeps the last wave short).  A segment's row
  // minima are combined across segments with a 64-bit atomicMin.
  const int nseg = P.nseg, cps = (nch + nseg - 1) / nseg;
  const int nunits = (int)(ntiles * nseg);
  auto seg_lo = [&](int sg) { return sg * cps; };
  auto seg_hi = [&](int sg) { return min(nch, (sg + 1) * cps); };
  // this CTA's chunk sequence, two ahead of the one being processed (the
  // ring prefetch): (unit, chunk) cursor
  int la_u = (int)blockIdx.x;
  int la_c = la_u < nunits ? seg_lo(la_u % nseg) : 0;
  auto la_next = [&]() {  // chunk of the lookahead cursor, then advance it; -1 past the end
    if (la_u >= nunits) return -1;
    const int c = la_c;
    if (++la_c >= seg_hi(la_u % nseg)) {
      la_u += (int)gridDim.x;
      if (la_u < nunits) la_c = seg_lo(la_u % nseg);
    }
    return c;
  };
  constexpr uint32_t unit = SCALE8 ? 8u : 1u;  // accumulator unit: byte offset (8-byte entries) or index
  const uint32_t sv = (uint32_t)P.S * unit;     // one shared doc adds S (+ displacement)
  uint32_t *ring = stg + (size_t)w * 2 * K * 32;  // this warp's [2][K][32]
  u64 *wfull = full + 2 * w;
  const uint32_t *idsw = a.idsT + 32 * w;

  // the warp's chunk (column block ch) -> ring stage b: lane 0 arms the
  // stage's barrier, lanes k < K copy doc k of the warp's 32 columns
  auto issue = [&](int ch, int b) {
    if (lane == 0) mbar_expect_tx(&wfull[b], (unsigned)K * 128u);
    __syncwarp();
    if (lane < K) bulk_g2s(ring + (b * K + lane) * 32, idsw + (int64_t)lane * Npad + (int64_t)ch * CH, 128u, &wfull[b]);
  };
  if (lane == 0) {
    mbar_init(&wfull[0], 1);
    mbar_init(&wfull[1], 1);
  }
  if (TAB_SMEM)
    for (int i = tid; i < (K + 1) * P.S; i += NT) reinterpret_cast<uint2 *>(smem)[i] = a.ptab[i];
  for (int i = tid; i < R * ACCW; i += NT) acc[i] = 0u;
  __syncthreads();
  {
    const int c0 = la_next();
    if (c0 >= 0) issue(c0, 0);
    const int c1 = la_next();
    if (c1 >= 0) issue(c1, 1);
  }

  uint16_t *myq = qall + w * QCAP;
  uint2 *cinfo = cinfo_all + w * 32;
  const int cg = lane & 7, rr = lane >> 3;  // finalize: column group, first row
  const bool counts = a.s_out != nullptr;
  constexpr bool codes_out = CODES;  // (a.codes != nullptr, a template parameter: no per-store branch)
  const bool vec_n = (N & 3) == 0;
  const uint32_t lanes_le = 0xffffffffu >> (31 - lane);
  int64_t g = 0;  // position in this CTA's chunk sequence

  for (int un = (int)blockIdx.x; un < nunits; un += (int)gridDim.x) {
    const int64_t tile = un / nseg;
    const int sg = un - (int)tile * nseg;
    const int64_t r0 = a.row0 + tile * R;
    const int64_t rem = a.row0 + a.nrows - r0;
    const int rcount = rem < R ? (int)rem : R;

    // ---- tile table + filter (block) ---------------------------------------
    __syncthreads();  // previous tile's warps are done with the table, row minima and queues
    for (int i = tid; i < P.T; i += NT) {
      tkey[i] = kReservedDoc;
      tcb[i] = 0u;
    }
    for (int i = tid; i < FWORDS; i += NT) filt[i] = 0u;
    __syncthreads();
    uint32_t *tmp = reinterpret_cast<uint32_t *>(qall);  // [R*K] slot << 8 | rank within the slot
    for (int it = tid; it < rcount * K; it += NT) {
      const int r = it / K, k = it - r * K;
      const uint32_t doc = a.ids[(r0 + r) * (int64_t)K + k];
      // buckets of 4 slots filled in order; linear probing over buckets
      uint32_t bkt = hash_slot(doc, logNB), slot = 0u;
      for (bool placed = false; !placed; bkt = (bkt + 1) & (NB - 1)) {
        for (int j = 0; j < 4; ++j) {
          const uint32_t prev = atomicCAS(&tkey[4 * bkt + j], kReservedDoc, doc);
          if (prev == kReservedDoc || prev == doc) {
            slot = 4 * bkt + j;
            placed = true;
            break;
          }
        }
      }
      const uint32_t sub = atomicAdd(&tcb[slot], 1u);
      const uint32_t fb = hash_filter(doc);
      atomicOr(&filt[fb >> 5], 1u << (fb & 31));
      tmp[it] = (slot << 8) | sub;
    }
    __syncthreads();
    {
      const int per = P.T / NT;  // T is a multiple of NT
      int cnt = 0;
      for (int i = 0; i < per; ++i) cnt += (int)tcb[tid * per + i];
      __shared__ int wsum[NW];
      int base = block_excl_scan<NT>(cnt, wsum);
      for (int i = 0; i < per; ++i) {
        const uint32_t c = tcb[tid * per + i];
        tcb[tid * per + i] = (c << 16) | (uint32_t)base;
        base += (int)c;
      }
    }
    __syncthreads();
    for (int it = tid; it < rcount * K; it += NT) {
      const int r = it / K, k = it - r * K;
      const uint32_t t = tmp[it];
      plist[(tcb[t >> 8] & 0xffffu) + (t & 0xffu)] = (uint16_t)((r << 5) | k);
    }
    __syncthreads();

    // running row minimum per lane for rows rr + 4q: code << 16 | (chunk << 2 | i)
    uint32_t bk[R / 4];
#pragma unroll
    for (int q = 0; q < R / 4; ++q) bk[q] = 0xffffffffu;

    for (int ch = seg_lo(sg); ch < seg_hi(sg); ++ch, ++g) {
      const int b = (int)(g & 1);
      const int64_t c0 = (int64_t)ch * CH;
      const uint32_t *sb = ring + b * K * 32;
      mbar_wait(&wfull[b], (unsigned)((g >> 1) & 1));

      // ---- probe: lane = column 32w + lane, candidate bit per k ------------
      uint32_t cm = 0u;
#pragma unroll 4
      for (int k = 0; k < K; ++k) {
        const uint32_t f = hash_filter(sb[k * 32 + lane]);
        cm |= (__funnelshift_r(filt[f >> 5], 0u, f) & 1u) << k;
      }
      // ---- candidate queue (entry = k << 5 | column) and drain -------------
      {
        const int n = __popc(cm);
        int x = n;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int y = __shfl_up_sync(0xffffffffu, x, o);
          if (lane >= o) x += y;
        }
        const int qn_all = __shfl_sync(0xffffffffu, x, 31);
        for (int lo = 0; lo < qn_all; lo += QCAP) {
          int pos = x - n;
          for (uint32_t m = cm; m; m &= m - 1u) {
            const int k = __ffs(m) - 1;
            if ((unsigned)(pos - lo) < (unsigned)QCAP) myq[pos - lo] = (uint16_t)((k << 5) | lane);
            ++pos;
          }
          __syncwarp();
          const int qn = min(QCAP, qn_all - lo);
          for (int base = 0; base < qn; base += 32) {
            // lanes = candidates: table lookup -> (row count, row-list base)
            const int i = base + lane;
            uint32_t cnt = 0u, cbv = 0u, kc = 0u;
            if (i < qn) {
              kc = myq[i];
              const uint32_t d = sb[(kc >> 5) * 32 + (kc & 31u)];
              uint32_t bkt = hash_slot(d, logNB);
              while (true) {
                const uint4 k4 = reinterpret_cast<const uint4 *>(tkey)[bkt];
                const int j = k4.x == d ? 0 : k4.y == d ? 1 : k4.z == d ? 2 : k4.w == d ? 3 : -1;
                if (j >= 0) {
                  cbv = tcb[4 * bkt + j];
                  break;
                }
                if (k4.w == kReservedDoc) break;  // bucket not full: absent
                bkt = (bkt + 1) & (NB - 1);
              }
              cnt = cbv >> 16;
            }
            int xi = (int)cnt;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
              const int y = __shfl_up_sync(0xffffffffu, xi, o);
              if (lane >= o) xi += y;
            }
            const int off = xi - (int)cnt;
            const int tot = __shfl_sync(0xffffffffu, xi, 31);
            // load-balanced expansion: candidates with rows, in order, get a
            // rank; incidence p belongs to the last candidate starting at or
            // before p (start marks of each 32-wide window by a warp OR)
            const uint32_t nz = __ballot_sync(0xffffffffu, cnt > 0u);
            if (cnt > 0u) {
              cinfo[__popc(nz & (lanes_le >> 1))] =
                  make_uint2((uint32_t)off | (cbv << 16), (kc >> 5) | ((kc & 31u) << 8));
            }
            __syncwarp();
            int started = 0;  // candidates started before the window
            for (int p0 = 0; p0 < tot; p0 += 32) {
              const int rel = off - p0;
              const uint32_t m =
                  __reduce_or_sync(0xffffffffu, (cnt > 0u && (unsigned)rel < 32u) ? (1u << rel) : 0u);
              const int p = p0 + lane;
              if (p < tot) {
                const uint2 ci = cinfo[started + __popc(m & lanes_le) - 1];
                const uint32_t pe = plist[(ci.x >> 16) + (uint32_t)(p - (int)(ci.x & 0xffffu))];
                const int dk = (int)(pe & 31u) - (int)(ci.y & 0xffu);
                const uint32_t dp = (uint32_t)(dk < 0 ? -dk : dk);
                const uint32_t col = ci.y >> 8;
                atomicAdd(acc + (pe >> 5) * ACCW + 16 * w + (col >> 1), (sv + dp * unit) << ((col & 1u) << 4));
              }
              started += __popc(m);
            }
            __syncwarp();  // cinfo is rewritten by the next round
          }
          __syncwarp();
        }
      }
      // the warp is done with stage b: refill it with its chunk g + 2
      __syncwarp();
      {
        const int cn = la_next();  // this warp's chunk g + 2 of the CTA's sequence
        if (cn >= 0) {
          fence_proxy_async_smem();
          issue(cn, b);
        }
      }

      // ---- finalize: lane = 4 columns x rows rr + 4q --------------------------
      const int64_t jb = c0 + 32 * w + 4 * cg;  // first of the lane's 4 columns
      const bool special = counts || !vec_n || rcount < R || c0 + CH > N || (c0 < r0 + R && r0 < c0 + CH);
      const uint32_t sq = (uint32_t)ch << 2;
      if (!special) {
        float *orow = a.rows + (r0 - a.row0 + rr) * N + jb;
        uint16_t *crow = codes_out ? a.codes + (r0 - a.row0 + rr) * N + jb : nullptr;
#pragma unroll
        for (int q = 0; q < R / 4; ++q) {
          uint2 *ap = reinterpret_cast<uint2 *>(acc + (rr + 4 * q) * ACCW + 16 * w + 2 * cg);
          const uint2 wv = *ap;
          *ap = make_uint2(0u, 0u);
          uint2 e0, e1, e2, e3;
          if (SCALE8) {
            const char *tb = reinterpret_cast<const char *>(tab);
            e0 = *reinterpret_cast<const uint2 *>(tb + (wv.x & 0xffffu));
            e1 = *reinterpret_cast<const uint2 *>(tb + (wv.x >> 16));
            e2 = *reinterpret_cast<const uint2 *>(tb + (wv.y & 0xffffu));
            e3 = *reinterpret_cast<const uint2 *>(tb + (wv.y >> 16));
          } else {
            e0 = tab[wv.x & 0xffffu];
            e1 = tab[wv.x >> 16];
            e2 = tab[wv.y & 0xffffu];
            e3 = tab[wv.y >> 16];
          }
          __stcs(reinterpret_cast<uint4 *>(orow + (int64_t)4 * q * N), make_uint4(e0.x, e1.x, e2.x, e3.x));
          if (codes_out)
            __stcs(reinterpret_cast<uint2 *>(crow + (int64_t)4 * q * N),
                   make_uint2(__byte_perm(e0.y, e1.y, 0x7632), __byte_perm(e2.y, e3.y, 0x7632)));
          // (code << 16 | i) orders like (value, column) within the step; the
          // chunk bits (sq) are common, so OR-ing them in afterwards keeps the order
          bk[q] = min(bk[q], min(min(e0.y, e1.y | 1u), min(e2.y | 2u, e3.y | 3u)) | sq);
        }
      } else {
#pragma unroll
        for (int q = 0; q < R / 4; ++q) {
          const int r = rr + 4 * q;
          uint2 *ap = reinterpret_cast<uint2 *>(acc + r * ACCW + 16 * w + 2 * cg);
          const uint2 wv = *ap;
          *ap = make_uint2(0u, 0u);
          const int64_t gi = r0 + r;
          const uint32_t o4[4] = {wv.x & 0xffffu, wv.x >> 16, wv.y & 0xffffu, wv.y >> 16};
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const int64_t j = jb + i;
            const uint32_t idx = o4[i] / unit;
            const uint2 e = tab[idx];
            const bool in = r < rcount && j < N;
            if (in) {
              const int64_t o = (gi - a.row0) * N + j;
              __stcs(a.rows + o, __uint_as_float(e.x));
              if (codes_out) a.codes[o] = (uint16_t)(e.y >> 16);
              if (counts) {
                const uint32_t s = idx / (uint32_t)P.S;
                a.s_out[o] = (uint8_t)s;
                a.D_out[o] = (uint16_t)(idx - s * (uint32_t)P.S);
              }
            }
            const uint32_t kk = (in && j != gi) ? (e.y | sq | (uint32_t)i) : 0xffffffffu;
            bk[q] = min(bk[q], kk);
          }
        }
      }
    }

    // ---- row NN: 8 lanes per row, then across warps ---------------------------
    u64 *red = reinterpret_cast<u64 *>(myq);  // [R] this warp's partial row minima (own queue area)
#pragma unroll
    for (int q = 0; q < R / 4; ++q) {
      const uint32_t v = bk[q];
      u64 key = ~0ull;
      if (v != 0xffffffffu) {
        const uint32_t s = v & 0xffffu;
        const uint32_t col = (s >> 2) * CH + 32u * w + 4u * cg + (s & 3u);
        key = ((u64)(v >> 16) << 32) | col;
      }
      key = umin64(key, __shfl_xor_sync(0xffffffffu, key, 1));
      key = umin64(key, __shfl_xor_sync(0xffffffffu, key, 2));
      key = umin64(key, __shfl_xor_sync(0xffffffffu, key, 4));
      if (cg == 0) red[rr + 4 * q] = key;
    }
    __syncthreads();
    if (tid < rcount) {
      u64 best = ~0ull;
#pragma unroll
      for (int v = 0; v < NW; ++v) best = umin64(best, reinterpret_cast<const u64 *>(qall + v * QCAP)[tid]);
      if (best != ~0ull)
        best = ((u64)__float_as_uint(__ldg(a.vals + (best >> 32))) << 32) | (best & 0xffffffffull);
      if (nseg == 1)
        a.nnkey[r0 + tid] = best;
      else if (best != ~0ull)
        atomicMin(a.nnkey + r0 + tid, best);  // (value bits, column) order = (value, column) order
    }
  }
}

bool make_plan(int K, int R, bool tab_smem, size_t limit, Plan *out) {
  Plan P{};
  P.K = K;
  P.R = R;
  int T = NT, logT = 9;
  while (T < R * K * 3 / 2) {
    T <<= 1;
    ++logT;
  }
  P.T = T;
  P.logT = logT;
  P.S = K * K / 2 + 1;
  P.scale8 = 8LL * ((int64_t)K * P.S + P.S - 1) < 65536;
  P.tab_smem = tab_smem;
  size_t o = 0;
  auto take = [&](size_t bytes, size_t align) {
    o = (o + align - 1) / align * align;
    const size_t at = o;
    o += bytes;
    return at;
  };
  P.off_tab = take(tab_smem ? (size_t)(K + 1) * P.S * 8 : 0, 128);  // first: offset 0
  P.off_acc = take((size_t)R * ACCW * 4, 128);
  P.off_stage = take((size_t)NW * 2 * K * 32 * 4, 128);
  P.off_key = take((size_t)T * 4, 16);
  P.off_cb = take((size_t)T * 4, 16);
  P.off_plist = take((size_t)R * K * 2, 16);
  P.off_filter = take((size_t)FWORDS * 4, 16);
  // per-warp queues; also the tile build's [R*K] slot list and the [NW][R] row minima
  P.off_q = take(std::max<size_t>({(size_t)NW * QCAP * 2, (size_t)R * K * 4, (size_t)NW * R * 8}), 16);
  P.off_inc = take((size_t)NW * 32 * 8, 16);
  P.off_bar = take((size_t)NW * 2 * 8, 16);
  P.total = (o + 127) / 128 * 128;
  *out = P;
  return P.total <= limit;
}

template <int R, bool S8, bool TS>
cudaError_t launch(const DistArgs &a, const Plan &P, cudaStream_t st) {
  auto kern = a.codes ? k_dist_tile<R, S8, TS, true> : k_dist_tile<R, S8, TS, false>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)P.total);
  if (e != cudaSuccess) return e;
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t ntiles = (a.nrows + R - 1) / R;
  const int nch = (int)((a.N + CH - 1) / CH);
  int64_t grid = (int64_t)sms;  // one persistent CTA per SM
  if (a.grid_cap > 0) grid = std::min<int64_t>(grid, a.grid_cap);
  // column segments: at least ~16 units per CTA (short last wave), segments
  // of at least 8 chunks
  Plan Q = P;
  Q.nseg = (int)std::max<int64_t>(1, std::min<int64_t>((16 * grid + ntiles - 1) / ntiles, nch / 8));
  grid = std::min<int64_t>(grid, ntiles * Q.nseg);
  if (Q.nseg > 1) {  // partial row minima meet in a 64-bit atomicMin
    cudaError_t e2 = cudaMemsetAsync(a.nnkey + a.row0, 0xff, (size_t)a.nrows * 8, st);
    if (e2 != cudaSuccess) return e2;
  }
  kern<<<(unsigned)grid, NT, P.total, st>>>(a, Q);
  return cudaGetLastError();
}

}  // namespace

int tile_lut_shift(int32_t K) { return K <= 22 ? 8 : 10; }

int64_t tile_lut_entries(int32_t K) {
  return (int64_t)(K + 1) << tile_lut_shift(K);
}

int64_t tile_ptab_entries(int32_t K) { return (int64_t)(K + 1) * (K * K / 2 + 1); }

bool tile_path_ok(int32_t K, bool uniform) { return uniform && K <= 32; }

cudaError_t launch_distance_tile(const DistArgs &a, cudaStream_t st) {
  if (!a.lut || !a.lutc || !a.vals || !a.ptab) return cudaErrorInvalidValue;
  const int K = a.K;
  const int S = K * K / 2 + 1;
  {
    const int n = (K + 1) * S;
    k_pack_table<<<(n + 255) / 256, 256, 0, st>>>(a.lut, a.lutc, K, tile_lut_shift(K), S,
                                                    const_cast<uint2 *>(a.ptab));
  }
  int dev = 0, optin = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  const size_t limit = (size_t)optin - 1024;  // static shared memory of the kernel (scan scratch)
  Plan P;
  for (const auto &cfg : {std::make_pair(64, true), std::make_pair(64, false), std::make_pair(32, true),
                          std::make_pair(32, false)}) {
    if (!make_plan(K, cfg.first, cfg.second, limit, &P)) continue;
    if (P.R == 64) {
      if (P.scale8) return P.tab_smem ? launch<64, true, true>(a, P, st) : launch<64, true, false>(a, P, st);
      return P.tab_smem ? launch<64, false, true>(a, P, st) : launch<64, false, false>(a, P, st);
    }
    if (P.scale8) return P.tab_smem ? launch<32, true, true>(a, P, st) : launch<32, true, false>(a, P, st);
    return P.tab_smem ? launch<32, false, true>(a, P, st) : launch<32, false, false>(a, P, st);
  }
  return cudaErrorInvalidConfiguration;
}

}  // namespace ragb
