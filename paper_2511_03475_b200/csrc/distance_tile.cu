// a2-a4 fast path on sm_100a: every context has exactly K <= 32 docs (the
// paper's setting: a retriever returns top-K lists).  Same math as
// distance.cu (Eq. 1; X2, X3, X6), restructured so that warps stay
// converged:
//
//  * A CTA (256 threads) owns R = 32 rows; it streams all N columns in chunks
//    of 512 (2 per thread).  The tile's docs sit in a shared-memory hash table
//    (doc -> row mask, positions) plus a 2^16-bit filter.
//  * Probe phase, per k: each thread tests its 2 column docs against the
//    filter (one LDS, branch-free).  Candidates (~20 %) are appended to a
//    per-warp queue with ballots.
//  * Hit phase: the warp drains its queue with all 32 lanes: table lookup, then
//    one shared-memory atomicAdd of (1 << SHIFT) + |p_i - p_j| per (row, column)
//    incidence into packed 16-bit (s, D) accumulators.
//  * Finalize: the packed accumulator IS the index of a d(s, D) table (stride
//    1 << SHIFT), so d costs one LDS; 8-byte streaming row stores; the row
//    min/argmin runs in registers (32 rows unrolled) and is reduced once per
//    tile, not per chunk.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>

#include "device_util.cuh"
#include "internal.h"

namespace ragb {
namespace {

constexpr int NT = 256;        // threads per CTA
constexpr int NW = NT / 32;    // warps per CTA
constexpr int CPT = 2;         // columns per thread per chunk
constexpr int CH = NT * CPT;   // columns per chunk
constexpr int R = 32;          // rows per tile
constexpr int FWORDS = 2048;   // filter words (65536 bits)

struct Plan {
  int T, logT, shift, lutEntries, qcap;
  size_t off_acc, off_key, off_mask, off_base, off_slot, off_plist, off_filter, off_qdoc, off_qmeta,
      off_red, off_wsum, off_lut, off_lutc, total;
};
constexpr int QW = 512;  // candidate-queue window per warp (entries), drained as often as needed

// CODES: also write codes[i][j] = lutc[packed (s, D)] (16-bit order-preserving
// value codes, the complete-linkage input; the code table has the float
// table's layout and is read through L1).
template <int SHIFT, bool LUT_SMEM, bool COUNTS, bool CODES>
__global__ void __launch_bounds__(NT, 2) k_dist_tile(DistArgs a, Plan P) {
  constexpr uint32_t DMASK = (1u << SHIFT) - 1u;
  constexpr uint32_t INC = 1u << SHIFT;
  // SHIFT == 8: accumulate 4 x (s << 8 | D), the byte offset of d(s, D) in the
  // table (max 4 * (22 << 8 | 242) < 2^16); SHIFT == 10: the index itself.
  constexpr uint32_t ISCALE = SHIFT == 8 ? 4u : 1u;
  extern __shared__ __align__(16) unsigned char smem[];
  uint32_t *accw = reinterpret_cast<uint32_t *>(smem + P.off_acc);    // [R][NT] packed 2 x u16
  uint32_t *tkey = reinterpret_cast<uint32_t *>(smem + P.off_key);    // [T]
  uint32_t *tmask = reinterpret_cast<uint32_t *>(smem + P.off_mask);  // [T]
  uint16_t *tbase = reinterpret_cast<uint16_t *>(smem + P.off_base);  // [T]
  uint16_t *slot = reinterpret_cast<uint16_t *>(smem + P.off_slot);   // [R*K]
  uint16_t *plist = reinterpret_cast<uint16_t *>(smem + P.off_plist);  // [R*K] (row << 8 | pos)
  uint32_t *filt = reinterpret_cast<uint32_t *>(smem + P.off_filter); // [FWORDS]
  uint16_t *qent = reinterpret_cast<uint16_t *>(smem + P.off_qdoc);   // [NW][qcap]
  unsigned long long *red = reinterpret_cast<unsigned long long *>(smem + P.off_red);  // [NW][R]
  int *wsum = reinterpret_cast<int *>(smem + P.off_wsum);
  float *slut = reinterpret_cast<float *>(smem + P.off_lut);
  uint16_t *slutc = reinterpret_cast<uint16_t *>(smem + P.off_lutc);

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int K = a.K, T = P.T, logT = P.logT;
  const int64_t N = a.N, Npad = a.Npad;
  const int64_t ntiles = (a.nrows + R - 1) / R;
  const float *lut = LUT_SMEM ? slut : a.lut;
  if (LUT_SMEM)
    for (int i = tid; i < P.lutEntries; i += NT) {
      slut[i] = a.lut[i];
      if (CODES) slutc[i] = (uint16_t)a.lutc[i];
    }
  const bool even_n = (N & 1) == 0;

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
    for (int i = tid; i < R * NT; i += NT) accw[i] = 0u;
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

    // running row minimum per thread: (d, column) in fp32 mode; in code mode
    // one packed word (code << 16 | chunk << 1 | column bit) — codes order
    // like the values and, for one thread, (chunk, bit) orders like the
    // column, so the strict minimum keeps the smallest column (X8) in half
    // the registers
    float bv[CODES ? 1 : R];
    uint32_t bj[CODES ? 1 : R];
    uint32_t bk[CODES ? R : 1];
#pragma unroll
    for (int r = 0; r < R; ++r) {
      if constexpr (CODES) {
        bk[r] = 0xffffffffu;
      } else {
        bv[r] = __int_as_float(0x7f800000);
        bj[r] = 0xffffffffu;
      }
    }

    uint16_t *myq = qent + warp * P.qcap;
    uint32_t chunk = 0;
    for (int64_t c0 = 0; c0 < N; c0 += CH, ++chunk) {
      const int64_t jb = c0 + (int64_t)tid * CPT;
      const uint32_t *colp = a.idsT + jb;

      // ---- probe: filter every column doc, keep candidate bits per column --
      uint32_t cm0 = 0u, cm1 = 0u;  // bit k: doc k of column 0 / 1 may be in the tile
      constexpr int PU = CODES ? 6 : 4;  // column-doc loads in flight (registers)
#pragma unroll PU
      for (int k = 0; k < K; ++k) {
        const uint2 v = __ldg(reinterpret_cast<const uint2 *>(colp + (int64_t)k * Npad));
        const uint32_t f0 = hash_filter(v.x), f1 = hash_filter(v.y);
        cm0 |= ((filt[f0 >> 5] >> (f0 & 31)) & 1u) << k;
        cm1 |= ((filt[f1 >> 5] >> (f1 & 31)) & 1u) << k;
      }
      // ---- compact candidates into the warp queue (entry = k << 9 | column)
      {
        const int n = __popc(cm0) + __popc(cm1);
        int x = n;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int y = __shfl_up_sync(0xffffffffu, x, o);
          if (lane >= o) x += y;
        }
        const int qn_all = __shfl_sync(0xffffffffu, x, 31);
        const int pos0 = x - n;
        const uint32_t col0 = (uint32_t)(tid * CPT);
        // windows of qcap queue entries (almost always one)
        for (int lo = 0; lo < qn_all; lo += P.qcap) {
        int pos = pos0;
        uint32_t m0 = cm0, m1 = cm1;
        while (m0) {
          const int k = __ffs(m0) - 1;
          m0 &= m0 - 1u;
          if ((unsigned)(pos - lo) < (unsigned)P.qcap) myq[pos - lo] = (uint16_t)((k << 9) | col0);
          ++pos;
        }
        while (m1) {
          const int k = __ffs(m1) - 1;
          m1 &= m1 - 1u;
          if ((unsigned)(pos - lo) < (unsigned)P.qcap) myq[pos - lo] = (uint16_t)((k << 9) | (col0 + 1u));
          ++pos;
        }
        __syncwarp();
        const int qn = min(P.qcap, qn_all - lo);
        // ---- drain: all 32 lanes process the warp's candidates; the doc
        // reloads of DB consecutive rounds are issued together (latency)
        constexpr int DB = 4;
        for (int base = 0; base < qn; base += 32 * DB) {
          uint32_t doc[DB], ent[DB];
#pragma unroll
          for (int u = 0; u < DB; ++u) {
            const int i = base + u * 32 + lane;
            ent[u] = i < qn ? myq[i] : 0xffffffffu;
            const int k = (int)(ent[u] >> 9), col = (int)(ent[u] & 511u);
            doc[u] = i < qn ? __ldg(a.idsT + (int64_t)k * Npad + (c0 + col)) : kReservedDoc;
          }
#pragma unroll
          for (int u = 0; u < DB; ++u) {
            const int k = (int)((ent[u] >> 9) & 31u), col = (int)(ent[u] & 511u);
            const uint32_t d = doc[u];
            uint32_t h = hash_slot(d, logT);
            uint32_t key = tkey[h];
            while (key != d && key != kReservedDoc) {
              h = (h + 1) & (T - 1);
              key = tkey[h];
            }
            const int cnt = key == d ? __popc(tmask[h]) : 0;
            const int idx0 = tbase[h];
            const uint32_t sh = (uint32_t)(col & 1) * 16u;
            uint32_t *wp = accw + (col >> 1);
            for (int z = 0; z < cnt; ++z) {  // rows of the tile holding this doc
              const uint32_t e = plist[idx0 + z];
              const int pr = (int)(e & 0xffu);
              const uint32_t dp = (uint32_t)(pr > k ? pr - k : k - pr);
              atomicAdd(wp + (e >> 8) * NT, ((INC + dp) * ISCALE) << sh);
            }
          }
        }
        __syncwarp();
        }
      }

      // ---- finalize: d = table[packed (s, D)], stores, row min in registers
      const bool vec_ok = even_n && (c0 + (int64_t)(warp + 1) * 32 * CPT <= N);
      const bool special = (c0 < r0 + R && r0 < c0 + CH) || (c0 + CH > N);
      const uint32_t j0 = (uint32_t)jb, j1 = (uint32_t)jb + 1u;
      float *orow = a.rows + (r0 - a.row0) * N + jb;
      uint32_t *ap = accw + tid;
      if (!special && vec_ok && !COUNTS && rcount == R) {
        // common case: full tile, no diagonal, no tail, aligned stores
        const char *lutb = reinterpret_cast<const char *>(lut);
        float2 *o = reinterpret_cast<float2 *>(orow);
        const int64_t step = N / 2;  // float2 units per row (N even here)
        const char *lutcb = reinterpret_cast<const char *>(a.lutc);
        uint32_t *co = CODES ? reinterpret_cast<uint32_t *>(a.codes + (r0 - a.row0) * N + jb) : nullptr;
#pragma unroll
        for (int r = 0; r < R; ++r) {
          const uint32_t w = ap[r * NT];
          ap[r * NT] = 0u;
          float d0, d1;
          if (SHIFT == 8 && LUT_SMEM) {
            d0 = *reinterpret_cast<const float *>(lutb + (w & 0xffffu));
            d1 = *reinterpret_cast<const float *>(lutb + (w >> 16));
          } else {
            d0 = LUT_SMEM ? lut[(w & 0xffffu) / ISCALE] : __ldg(lut + (w & 0xffffu) / ISCALE);
            d1 = LUT_SMEM ? lut[(w >> 16) / ISCALE] : __ldg(lut + (w >> 16) / ISCALE);
          }
          __stcs(o, make_float2(d0, d1));
          o += step;
          if (CODES) {
            uint32_t c0, c1;
            if (SHIFT == 8 && LUT_SMEM) {  // byte offset 4 x index -> 16-bit entry at 2 x index
              const char *sc = reinterpret_cast<const char *>(slutc);
              c0 = *reinterpret_cast<const uint16_t *>(sc + ((w & 0xffffu) >> 1));
              c1 = *reinterpret_cast<const uint16_t *>(sc + (w >> 17));
            } else if (SHIFT == 8) {
              c0 = __ldg(reinterpret_cast<const uint32_t *>(lutcb + (w & 0xffffu)));
              c1 = __ldg(reinterpret_cast<const uint32_t *>(lutcb + (w >> 16)));
            } else {
              c0 = __ldg(a.lutc + (w & 0xffffu));
              c1 = __ldg(a.lutc + (w >> 16));
            }
            __stcs(co, c0 | (c1 << 16));
            co += step;
            const uint32_t lk = chunk << 1;
            bk[r] = min(bk[r], min((c0 << 16) | lk, (c1 << 16) | lk | 1u));
          } else {
            // strict '<' keeps the smallest column among equal distances (X8)
            const float m = fminf(d0, d1);
            const bool u = m < bv[r];
            bj[r] = u ? (d0 <= d1 ? j0 : j1) : bj[r];
            bv[r] = u ? m : bv[r];
          }
        }
      } else {
#pragma unroll
        for (int r = 0; r < R; ++r) {
          if (r < rcount) {
            const uint32_t w = ap[r * NT];
            ap[r * NT] = 0u;
            const uint32_t p0 = (w & 0xffffu) / ISCALE, p1 = (w >> 16) / ISCALE;
            const float d0 = LUT_SMEM ? lut[p0] : __ldg(lut + p0);
            const float d1 = LUT_SMEM ? lut[p1] : __ldg(lut + p1);
            const int64_t gi = r0 + r;
            float *o = orow + (int64_t)r * N;
            if (vec_ok) {
              __stcs(reinterpret_cast<float2 *>(o), make_float2(d0, d1));
            } else {
              if (jb < N) __stcs(o, d0);
              if (jb + 1 < N) __stcs(o + 1, d1);
            }
            uint32_t cc0 = 0u, cc1 = 0u;
            if (CODES) {
              uint16_t *cr = a.codes + (gi - a.row0) * N + jb;
              cc0 = __ldg(a.lutc + p0);
              cc1 = __ldg(a.lutc + p1);
              if (jb < N) __stcs(cr, (uint16_t)cc0);
              if (jb + 1 < N) __stcs(cr + 1, (uint16_t)cc1);
            }
            if (COUNTS) {
              if (jb < N) {
                a.s_out[(gi - a.row0) * N + jb] = (uint8_t)(p0 >> SHIFT);
                a.D_out[(gi - a.row0) * N + jb] = (uint16_t)(p0 & DMASK);
              }
              if (jb + 1 < N) {
                a.s_out[(gi - a.row0) * N + jb + 1] = (uint8_t)(p1 >> SHIFT);
                a.D_out[(gi - a.row0) * N + jb + 1] = (uint16_t)(p1 & DMASK);
              }
            }
            if constexpr (CODES) {
              const uint32_t lk = chunk << 1;
              const uint32_t k0 = (jb < N && jb != gi) ? ((cc0 << 16) | lk) : 0xffffffffu;
              const uint32_t k1 = (jb + 1 < N && jb + 1 != gi) ? ((cc1 << 16) | lk | 1u) : 0xffffffffu;
              bk[r] = min(bk[r], min(k0, k1));
            } else {
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
      }
    }

    // ---- row NN: warp reduce each row, then across warps -------------------
    unsigned long long mine = ~0ull;  // lane r: this warp's best key of row r
#pragma unroll
    for (int r = 0; r < R; ++r) {
      unsigned long long key;
      if constexpr (CODES) {  // (code << 32 | column); decoded to the value below
        const uint32_t lk = bk[r];
        key = lk == 0xffffffffu ? ~0ull
                                : (((unsigned long long)(lk >> 16) << 32) |
                                   (((lk >> 1) & 0x7fffu) * (uint32_t)CH + (uint32_t)tid * CPT + (lk & 1u)));
      } else {
        key = ((unsigned long long)__float_as_uint(bv[r]) << 32) | bj[r];
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) key = umin64(key, __shfl_xor_sync(0xffffffffu, key, o));
      mine = (lane == r) ? key : mine;
    }
    red[warp * R + lane] = mine;
    __syncthreads();
    if (tid < rcount) {
      unsigned long long best = ~0ull;
#pragma unroll
      for (int w = 0; w < NW; ++w) best = umin64(best, red[w * R + tid]);
      if (CODES && best != ~0ull)
        best = ((unsigned long long)__float_as_uint(__ldg(a.vals + (best >> 32))) << 32) | (best & 0xffffffffull);
      a.nnkey[r0 + tid] = best;
    }
    __syncthreads();
  }
}

Plan plan(int K, int shift, int lutSmemEntries) {
  Plan P{};
  const int need = 2 * R * K;
  int T = 512, logT = 9;
  while (T < need) {
    T <<= 1;
    ++logT;
  }
  P.T = T;
  P.logT = logT;
  P.shift = shift;
  P.lutEntries = lutSmemEntries;
  size_t o = 0;
  auto take = [&](size_t bytes, size_t align) {
    o = (o + align - 1) / align * align;
    const size_t at = o;
    o += bytes;
    return at;
  };
  P.off_acc = take((size_t)R * NT * 4, 16);
  P.off_key = take((size_t)T * 4, 16);
  P.off_mask = take((size_t)T * 4, 16);
  P.off_base = take((size_t)T * 2, 16);
  P.off_slot = take((size_t)R * K * 2, 16);
  P.off_plist = take((size_t)R * K * 2, 16);
  P.off_filter = take((size_t)FWORDS * 4, 16);
  P.qcap = std::min(32 * CPT * K, QW);  // every (lane, column, k) can be a candidate: windows
  P.off_qdoc = take((size_t)NW * P.qcap * 2, 16);
  P.off_qmeta = P.off_qdoc;
  P.off_red = take((size_t)NW * R * 8, 16);
  P.off_wsum = take(32 * 4, 16);
  P.off_lut = take((size_t)lutSmemEntries * 4, 16);
  P.off_lutc = take((size_t)lutSmemEntries * 2, 16);  // 16-bit value codes of the table (code mode)
  P.total = (o + 15) / 16 * 16;
  return P;
}

template <int SHIFT, bool LS, bool C, bool CD>
cudaError_t launch(const DistArgs &a, const Plan &P, cudaStream_t st) {
  auto kern = k_dist_tile<SHIFT, LS, C, CD>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)P.total);
  if (e != cudaSuccess) return e;
  int dev = 0, sms = 0, per_sm = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, NT, P.total);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) per_sm = 1;
  const int64_t ntiles = (a.nrows + R - 1) / R;
  int64_t grid = std::min<int64_t>(ntiles, (int64_t)sms * per_sm);
  if (a.grid_cap > 0) grid = std::min<int64_t>(ntiles, a.grid_cap);
  kern<<<(unsigned)grid, NT, P.total, st>>>(a, P);
  return cudaGetLastError();
}

}  // namespace

int tile_lut_shift(int32_t K) { return K <= 22 ? 8 : 10; }

int64_t tile_lut_entries(int32_t K) {
  return (int64_t)(K + 1) << tile_lut_shift(K);
}

bool tile_path_ok(int32_t K, bool uniform) { return uniform && K <= 32; }

cudaError_t launch_distance_tile(const DistArgs &a, cudaStream_t st) {
  const int shift = tile_lut_shift(a.K);
  const int64_t entries = tile_lut_entries(a.K);
  const bool lut_smem = shift == 8;  // (K+1) * 256 floats <= 23.5 KB
  const Plan P = plan(a.K, shift, lut_smem ? (int)entries : 0);
  const bool C = a.s_out != nullptr, CD = a.codes != nullptr && a.lutc != nullptr;
  if (shift == 8) {
    if (CD) return C ? launch<8, true, true, true>(a, P, st) : launch<8, true, false, true>(a, P, st);
    return C ? launch<8, true, true, false>(a, P, st) : launch<8, true, false, false>(a, P, st);
  }
  if (CD) return C ? launch<10, false, true, true>(a, P, st) : launch<10, false, false, true>(a, P, st);
  return C ? launch<10, false, true, false>(a, P, st) : launch<10, false, false, false>(a, P, st);
}

}  // namespace ragb
