// a2-a4 for long lists on sm_100a: every context has exactly K docs with
// 32 < K <= 128 (the C5 K sweep goes to 100).  Same math as distance.cu /
// distance_tile.cu (Eq. 1; X2, X3, X6) and the same converged
// structure as the K <= 32 tile kernel, widened:
//
//  * A CTA (256 threads) owns R = 16 rows and streams all N columns in chunks
//    of 512 (2 per thread).  The tile's docs sit in a shared-memory hash table
//    (doc -> row mask, (row, position) list) plus a 2^16-bit filter.
//  * Probe: each thread tests its 2 column docs for every k against the filter
//    and keeps KW words of candidate bits per column (KW = ceil(K / 32)).
//  * The warp compacts its candidates into a queue of 16-bit (k, column)
//    entries — in windows of QCAP entries, so the queue does not grow with K —
//    and all 32 lanes drain it: table lookup, one shared-memory atomicAdd of
//    (1 << 16) + |p_i - p_j| per (row, column) incidence into a 32-bit (s, D)
//    accumulator (D <= K^2/2 < 2^16).
//  * Finalize: d from the Eq. 1 table d(s, D) (correctly rounded, X6; entry
//    0 = s = 0 = 1.0f, L1-hot), or the exact quotient without a table;
//    8-byte streaming row stores; the row min/argmin in registers, reduced
//    once per tile.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>

#include "device_util.cuh"
#include "internal.h"

namespace ragb {
namespace {

constexpr int NT = 256;
constexpr int NW = NT / 32;
constexpr int CPT = 2;
constexpr int CH = NT * CPT;
constexpr int R = 16;
constexpr int FWORDS = 2048;
constexpr int QCAP = 512;  // queue window per warp (entries)

struct WPlan {
  int T, logT;
  size_t off_acc, off_key, off_mask, off_base, off_slot, off_plist, off_filter, off_q, off_red, off_wsum, total;
};

template <int KW, bool COUNTS>
__global__ void __launch_bounds__(NT, 2) k_dist_wide(DistArgs a, WPlan P) {
  extern __shared__ __align__(16) unsigned char smem[];
  uint2 *acc = reinterpret_cast<uint2 *>(smem + P.off_acc);            // [R][NT]: (column 0, column 1)
  uint32_t *tkey = reinterpret_cast<uint32_t *>(smem + P.off_key);     // [T]
  uint32_t *tmask = reinterpret_cast<uint32_t *>(smem + P.off_mask);   // [T] rows holding the doc
  uint16_t *tbase = reinterpret_cast<uint16_t *>(smem + P.off_base);   // [T] offset into plist
  uint16_t *slot = reinterpret_cast<uint16_t *>(smem + P.off_slot);    // [R*K]
  uint16_t *plist = reinterpret_cast<uint16_t *>(smem + P.off_plist);  // [R*K] (row << 8 | pos)
  uint32_t *filt = reinterpret_cast<uint32_t *>(smem + P.off_filter);  // [FWORDS]
  uint16_t *qent = reinterpret_cast<uint16_t *>(smem + P.off_q);       // [NW][QCAP]
  unsigned long long *red = reinterpret_cast<unsigned long long *>(smem + P.off_red);  // [NW][R]
  int *wsum = reinterpret_cast<int *>(smem + P.off_wsum);

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int K = a.K, T = P.T, logT = P.logT;
  const int64_t N = a.N, Npad = a.Npad;
  const int64_t ntiles = (a.nrows + R - 1) / R;
  const bool even_n = (N & 1) == 0;
  const uint32_t lstride = (uint32_t)(K * K / 2 + 1);  // distance_lut_layout for uniform K <= kLutMaxK

  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t r0 = a.row0 + tile * R;
    const int64_t rem = a.row0 + a.nrows - r0;
    const int rcount = rem < R ? (int)rem : R;

    // ---- tile table + filter ---------------------------------------------
    for (int i = tid; i < T; i += NT) {
      tkey[i] = kReservedDoc;
      tmask[i] = 0u;
    }
    for (int i = tid; i < FWORDS; i += NT) filt[i] = 0u;
    for (int i = tid; i < R * NT; i += NT) acc[i] = make_uint2(0u, 0u);
    __syncthreads();
    for (int it = tid; it < rcount * K; it += NT) {
      const int r = it / K, k = it - r * K;
      const uint32_t doc = a.ids[(r0 + r) * (int64_t)K + k];
      uint32_t h = hash_slot(doc, logT);
      while (true) {
        const uint32_t prev = atomicCAS(&tkey[h], kReservedDoc, doc);
        if (prev == kReservedDoc || prev == doc) break;
        h = (h + 1) & (T - 1);
      }
      atomicOr(&tmask[h], 1u << r);
      const uint32_t fb = hash_filter(doc);
      atomicOr(&filt[fb >> 5], 1u << (fb & 31));
      slot[it] = (uint16_t)h;
    }
    __syncthreads();
    {
      const int per = T / NT;
      int cnt = 0;
      for (int i = 0; i < per; ++i) cnt += __popc(tmask[tid * per + i]);
      int base = block_excl_scan<NT>(cnt, wsum);
      for (int i = 0; i < per; ++i) {
        tbase[tid * per + i] = (uint16_t)base;
        base += __popc(tmask[tid * per + i]);
      }
    }
    __syncthreads();
    for (int it = tid; it < rcount * K; it += NT) {
      const int r = it / K, k = it - r * K;
      const int h = slot[it];
      plist[tbase[h] + __popc(tmask[h] & ((1u << r) - 1u))] = (uint16_t)((r << 8) | k);
    }
    __syncthreads();

    float bv[R];
    uint32_t bj[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
      bv[r] = __int_as_float(0x7f800000);
      bj[r] = 0xffffffffu;
    }

    uint16_t *myq = qent + warp * QCAP;
    for (int64_t c0 = 0; c0 < N; c0 += CH) {
      const int64_t jb = c0 + (int64_t)tid * CPT;
      const uint32_t *colp = a.idsT + jb;

      // ---- probe: candidate bits per (k, column) ---------------------------
      uint32_t cm0[KW], cm1[KW];
#pragma unroll
      for (int q = 0; q < KW; ++q) {
        cm0[q] = 0u;
        cm1[q] = 0u;
      }
#pragma unroll
      for (int q = 0; q < KW; ++q) {
#pragma unroll 4
        for (int kk = 0; kk < 32; ++kk) {
          const int k = q * 32 + kk;
          if (k < K) {
            const uint2 v = __ldg(reinterpret_cast<const uint2 *>(colp + (int64_t)k * Npad));
            const uint32_t f0 = hash_filter(v.x), f1 = hash_filter(v.y);
            cm0[q] |= ((filt[f0 >> 5] >> (f0 & 31)) & 1u) << kk;
            cm1[q] |= ((filt[f1 >> 5] >> (f1 & 31)) & 1u) << kk;
          }
        }
      }
      // ---- compact into the warp queue (entry = k << 9 | column), drained
      //      in windows of QCAP entries ---------------------------------------
      int n = 0;
#pragma unroll
      for (int q = 0; q < KW; ++q) n += __popc(cm0[q]) + __popc(cm1[q]);
      int x = n;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
      }
      const int qn = __shfl_sync(0xffffffffu, x, 31);
      const int pos0 = x - n;
      const uint32_t col0 = (uint32_t)(tid * CPT);
      for (int lo = 0; lo < qn; lo += QCAP) {
        // this lane's entries with queue position in [lo, lo + QCAP)
        int pos = pos0;
#pragma unroll
        for (int c = 0; c < 2; ++c) {
#pragma unroll
          for (int q = 0; q < KW; ++q) {
            uint32_t m = c == 0 ? cm0[q] : cm1[q];
            while (m) {
              const int kk = __ffs(m) - 1;
              m &= m - 1u;
              if (pos >= lo && pos < lo + QCAP) myq[pos - lo] = (uint16_t)(((q * 32 + kk) << 9) | (col0 + c));
              ++pos;
            }
          }
        }
        __syncwarp();
        const int wn = min(QCAP, qn - lo);
        constexpr int DB = 4;
        for (int base = 0; base < wn; base += 32 * DB) {
          uint32_t doc[DB], ent[DB];
#pragma unroll
          for (int u = 0; u < DB; ++u) {
            const int i = base + u * 32 + lane;
            ent[u] = i < wn ? myq[i] : 0xffffffffu;
            const int k = (int)(ent[u] >> 9), col = (int)(ent[u] & 511u);
            doc[u] = i < wn ? __ldg(a.idsT + (int64_t)k * Npad + (c0 + col)) : kReservedDoc;
          }
#pragma unroll
          for (int u = 0; u < DB; ++u) {
            const int k = (int)((ent[u] >> 9) & 127u), col = (int)(ent[u] & 511u);
            const uint32_t d = doc[u];
            uint32_t h = hash_slot(d, logT);
            uint32_t key = tkey[h];
            while (key != d && key != kReservedDoc) {
              h = (h + 1) & (T - 1);
              key = tkey[h];
            }
            const int cnt = key == d ? __popc(tmask[h]) : 0;
            const int idx0 = tbase[h];
            uint32_t *ap = reinterpret_cast<uint32_t *>(acc) + 2 * (col >> 1) + (col & 1);
            for (int z = 0; z < cnt; ++z) {  // rows of the tile holding this doc
              const uint32_t e = plist[idx0 + z];
              const int pr = (int)(e & 0xffu);
              const uint32_t dp = (uint32_t)(pr > k ? pr - k : k - pr);
              atomicAdd(ap + (e >> 8) * (2 * NT), (1u << 16) + dp);
            }
          }
        }
        __syncwarp();
      }

      // ---- finalize: d(s, D), stores, row min in registers -----------------
      const uint32_t j0 = (uint32_t)jb, j1 = (uint32_t)jb + 1u;
      const bool vec_ok = even_n && jb + 1 < N;
      float *orow = a.rows + (r0 - a.row0) * N + jb;
#pragma unroll
      for (int r = 0; r < R; ++r) {
        if (r < rcount) {
          uint2 *ap = acc + r * NT + tid;
          const uint2 w = *ap;
          *ap = make_uint2(0u, 0u);
          // the Eq. 1 table d(s, D) (L2-resident; index 0 = s = 0 -> 1.0f,
          // the hot entry) or, without a table, the exact quotient
          float d0, d1;
          if (a.lut) {
            d0 = __ldg(a.lut + (w.x >> 16) * lstride + (w.x & 0xffffu));
            d1 = __ldg(a.lut + (w.y >> 16) * lstride + (w.y & 0xffffu));
          } else {
            d0 = eq1_from_counts(w.x >> 16, w.x & 0xffffu, (uint32_t)K, a.an, a.ad);
            d1 = eq1_from_counts(w.y >> 16, w.y & 0xffffu, (uint32_t)K, a.an, a.ad);
          }
          const int64_t gi = r0 + r;
          float *o = orow + (int64_t)r * N;
          if (vec_ok) {
            __stcs(reinterpret_cast<float2 *>(o), make_float2(d0, d1));
          } else {
            if (jb < N) __stcs(o, d0);
            if (jb + 1 < N) __stcs(o + 1, d1);
          }
          if (COUNTS) {
            if (jb < N) {
              a.s_out[(gi - a.row0) * N + jb] = (uint8_t)(w.x >> 16);
              a.D_out[(gi - a.row0) * N + jb] = (uint16_t)(w.x & 0xffffu);
            }
            if (jb + 1 < N) {
              a.s_out[(gi - a.row0) * N + jb + 1] = (uint8_t)(w.y >> 16);
              a.D_out[(gi - a.row0) * N + jb + 1] = (uint16_t)(w.y & 0xffffu);
            }
          }
          // strict '<' keeps the smallest column among equal distances (X8)
          const float inf = __int_as_float(0x7f800000);
          const float e0 = (jb < N && jb != gi) ? d0 : inf;
          const float e1 = (jb + 1 < N && jb + 1 != gi) ? d1 : inf;
          const float m = fminf(e0, e1);
          const bool u = m < bv[r];
          bj[r] = u ? (e0 <= e1 ? j0 : j1) : bj[r];
          bv[r] = u ? m : bv[r];
        }
      }
    }

    // ---- row NN: warp reduce each row, then across warps -------------------
    unsigned long long mine = ~0ull;  // lane r: this warp's best key of row r
#pragma unroll
    for (int r = 0; r < R; ++r) {
      unsigned long long key = ((unsigned long long)__float_as_uint(bv[r]) << 32) | bj[r];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) key = umin64(key, __shfl_xor_sync(0xffffffffu, key, o));
      mine = (lane == r) ? key : mine;
    }
    if (lane < R) red[warp * R + lane] = mine;
    __syncthreads();
    if (tid < rcount) {
      unsigned long long best = ~0ull;
#pragma unroll
      for (int w = 0; w < NW; ++w) best = umin64(best, red[w * R + tid]);
      a.nnkey[r0 + tid] = best;
    }
    __syncthreads();
  }
}

WPlan wplan(int K) {
  WPlan P{};
  const int need = 2 * R * K;
  int T = 512, logT = 9;
  while (T < need) {
    T <<= 1;
    ++logT;
  }
  P.T = T;
  P.logT = logT;
  size_t o = 0;
  auto take = [&](size_t bytes, size_t align) {
    o = (o + align - 1) / align * align;
    const size_t at = o;
    o += bytes;
    return at;
  };
  P.off_acc = take((size_t)R * NT * 8, 16);
  P.off_key = take((size_t)T * 4, 16);
  P.off_mask = take((size_t)T * 4, 16);
  P.off_base = take((size_t)T * 2, 16);
  P.off_slot = take((size_t)R * K * 2, 16);
  P.off_plist = take((size_t)R * K * 2, 16);
  P.off_filter = take((size_t)FWORDS * 4, 16);
  P.off_q = take((size_t)NW * QCAP * 2, 16);
  P.off_red = take((size_t)NW * R * 8, 16);
  P.off_wsum = take(32 * 4, 16);
  P.total = (o + 15) / 16 * 16;
  return P;
}

template <int KW, bool C>
cudaError_t wlaunch(const DistArgs &a, const WPlan &P, cudaStream_t st) {
  auto kern = k_dist_wide<KW, C>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)P.total);
  if (e != cudaSuccess) return e;
  int dev = 0, sms = 0, per_sm = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, NT, P.total);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) per_sm = 1;
  const int64_t ntiles = (a.nrows + R - 1) / R;
  const int64_t grid = std::min<int64_t>(ntiles, (int64_t)sms * per_sm);
  kern<<<(unsigned)grid, NT, P.total, st>>>(a, P);
  return cudaGetLastError();
}

}  // namespace

bool wide_path_ok(int32_t K, bool uniform) { return uniform && K > 32 && K <= 128; }

cudaError_t launch_distance_wide(const DistArgs &a, cudaStream_t st) {
  const WPlan P = wplan(a.K);
  const bool C = a.s_out != nullptr;
  if (a.K <= 64) return C ? wlaunch<2, true>(a, P, st) : wlaunch<2, false>(a, P, st);
  return C ? wlaunch<4, true>(a, P, st) : wlaunch<4, false>(a, P, st);
}

}  // namespace ragb
