// a1-a4 on sm_100a: validation + transposed staging, and the all-pairs Eq. 1
// distance rows with the fused row nearest neighbour.
//
// Eq. 1 (Section 4.1 "Quantifying the overlapping between contexts"):
//   d_ij = 1 - |S_ij| / max(|C_i|,|C_j|) + alpha * sum_{k in S_ij} |p_i(k) - p_j(k)| / |S_ij|
// computed from exact integers s = |S_ij| and D = sum |p_i(k) - p_j(k)| (0-based
// positions, X2), finalised as the correctly rounded fp32 of the exact rational
// (X6): with alpha = an/ad,
//   d = ((m - s)*ad*s + an*D*m) / (ad*m*s)   (s > 0),   d = 1 (s = 0, X3).
//
// Design: integer set intersection, not a dense
// contraction, so no tensor cores.  A CTA owns a tile of R rows and streams all
// N columns.  The tile's R*K (doc -> row bitmask, positions) entries live in a
// shared-memory open-addressing hash table built once per tile; every column
// context probes it with its K docs (coalesced 16-byte loads of a transposed
// [K][Npad] id array that stays L2-resident).  Each hit adds (1 << SHIFT) + |dp|
// into a per-(row, column) packed (s, D) accumulator owned by exactly one thread,
// so no atomics or barriers are needed inside the column loop.  The finalize
// step converts (s, D) to d, writes 16-byte coalesced row stores, and folds the
// row min/argmin into a 64-bit key (f32 bits << 32 | column): d >= 0, so
// unsigned key order == (d, column) order, the X8 tie-break.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>

#include "device_util.cuh"
#include "internal.h"

#ifdef RAGB_DEBUG
#include <cstdio>
#define RB_DCHECK(cond, ...)                                    \
  do {                                                          \
    if (!(cond)) {                                              \
      printf("RB_DCHECK %s:%d: %s | ", __FILE__, __LINE__, #cond); \
      printf(__VA_ARGS__);                                      \
      printf("\n");                                             \
      __trap();                                                 \
    }                                                           \
  } while (0)
#else
#define RB_DCHECK(cond, ...) \
  do {                       \
  } while (0)
#endif

namespace ragb {
namespace {

constexpr int NT = kDistThreads;
constexpr int CPT = kColsPerThread;
constexpr int NW = NT / 32;

template <typename T>
struct AccTraits;
template <>
struct AccTraits<uint16_t> {  // K <= 32: s <= 32 (6 bits) << 10, D <= 512 (10 bits)
  static constexpr int SHIFT = 10;
  using Vec = uint2;
};
template <>
struct AccTraits<uint32_t> {  // K <= 255: D <= 32512 < 2^16
  static constexpr int SHIFT = 16;
  using Vec = uint4;
};

__device__ __forceinline__ void unpack4(const uint2 &v, uint32_t p[4]) {
  p[0] = v.x & 0xffffu;
  p[1] = v.x >> 16;
  p[2] = v.y & 0xffffu;
  p[3] = v.y >> 16;
}
__device__ __forceinline__ void unpack4(const uint4 &v, uint32_t p[4]) {
  p[0] = v.x;
  p[1] = v.y;
  p[2] = v.z;
  p[3] = v.w;
}

__device__ __forceinline__ unsigned long long warp_min64(unsigned long long v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = umin64(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

struct SmemPlan {
  int R, T, logT, accBytes, lutStride, lutEntries;
  size_t off_acc, off_rmin, off_key, off_mask, off_base, off_slot, off_plist, off_rlen, off_wsum,
      off_lut, total;
};

// Finalize modes: how (s, D) becomes d.
enum Fin : int { kFinDiv = 0, kFinLutSmem = 1, kFinLutGlobal = 2 };

template <int R, typename ACC, bool UNIFORM, bool COUNTS, int FIN>
__global__ void __launch_bounds__(NT) k_dist_rows_nn(DistArgs a, SmemPlan P) {
  using Tr = AccTraits<ACC>;
  using Vec = typename Tr::Vec;
  constexpr int SHIFT = Tr::SHIFT;
  constexpr uint32_t DMASK = (1u << SHIFT) - 1u;
  extern __shared__ __align__(16) unsigned char smem[];
  ACC *acc = reinterpret_cast<ACC *>(smem + P.off_acc);                      // [R][NT][CPT]
  unsigned long long *rmin = reinterpret_cast<unsigned long long *>(smem + P.off_rmin);  // [NW][R]
  uint32_t *tkey = reinterpret_cast<uint32_t *>(smem + P.off_key);           // [T]
  uint32_t *tmask = reinterpret_cast<uint32_t *>(smem + P.off_mask);         // [T]
  uint16_t *tbase = reinterpret_cast<uint16_t *>(smem + P.off_base);         // [T]
  uint16_t *slot = reinterpret_cast<uint16_t *>(smem + P.off_slot);          // [R*K]
  uint8_t *plist = smem + P.off_plist;                                       // [R*K]
  uint8_t *rlen = smem + P.off_rlen;                                         // [R]
  int *wsum = reinterpret_cast<int *>(smem + P.off_wsum);                    // [32]
  float *slut = reinterpret_cast<float *>(smem + P.off_lut);                 // FIN == smem

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int K = a.K, T = P.T, logT = P.logT;
  const int64_t N = a.N;
  const int64_t ntiles = (a.nrows + R - 1) / R;
  const float *lut = FIN == kFinLutSmem ? slut : a.lut;
  if (FIN == kFinLutSmem) {
    for (int i = tid; i < P.lutEntries; i += NT) slut[i] = a.lut[i];
  }
  // Rows of a warp's 128 columns are stored with 16-byte vectors when the row
  // stride keeps them aligned and the whole warp is inside the matrix; the
  // decision is warp-uniform (no intra-warp divergence in the finalize).
  const bool aligned = (N & 3) == 0;

  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t r0 = a.row0 + tile * R;  // global row of local row 0
    const int64_t rem = a.row0 + a.nrows - r0;
    const int rcount = rem < R ? (int)rem : R;

    // ---- build the tile table: doc -> (row bitmask, positions) --------------
    for (int i = tid; i < T; i += NT) {
      tkey[i] = kReservedDoc;
      tmask[i] = 0u;
    }
    for (int r = tid; r < R; r += NT)
      rlen[r] = (r < rcount) ? (UNIFORM ? (uint8_t)K : a.lens[r0 + r]) : (uint8_t)0;
    __syncthreads();
    for (int it = tid; it < R * K; it += NT) {
      const int r = it / K, k = it - r * K;
      if (k < rlen[r]) {
        const uint32_t doc = a.ids[(r0 + r) * (int64_t)K + k];
        uint32_t h = hash_slot(doc, logT);
        while (true) {
          const uint32_t prev = atomicCAS(&tkey[h], kReservedDoc, doc);
          if (prev == kReservedDoc || prev == doc) break;
          h = (h + 1) & (T - 1);
        }
        RB_DCHECK(h < (uint32_t)T && r < R && k < K, "h=%u r=%d k=%d", h, r, k);
        atomicOr(&tmask[h], 1u << r);
        slot[it] = (uint16_t)h;
      }
    }
    __syncthreads();
    {  // positions list offsets: exclusive scan of popc(mask) over the table
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
    for (int it = tid; it < R * K; it += NT) {
      const int r = it / K, k = it - r * K;
      if (k < rlen[r]) {
        const int h = slot[it];
        RB_DCHECK(tbase[h] + __popc(tmask[h] & ((1u << r) - 1u)) < R * K, "h=%d r=%d", h, r);
        plist[tbase[h] + __popc(tmask[h] & ((1u << r) - 1u))] = (uint8_t)k;
      }
    }
    __syncthreads();

    // ---- stream all columns ------------------------------------------------
    unsigned long long mymin = ~0ull;  // running min of row `lane` over this warp's columns
    for (int64_t c0 = 0; c0 < N; c0 += kChunk) {
      const int64_t jb = c0 + (int64_t)tid * CPT;
      ACC *myacc = acc + (size_t)tid * CPT;  // + r*NT*CPT
#pragma unroll 4
      for (int r = 0; r < R; ++r) *reinterpret_cast<Vec *>(myacc + (size_t)r * NT * CPT) = Vec{};
      uint32_t clen[CPT];
#pragma unroll
      for (int c = 0; c < CPT; ++c)
        clen[c] = UNIFORM ? (uint32_t)K : ((jb + c < N) ? a.lens[jb + c] : 0u);
      const uint32_t *colp = a.idsT + jb;
#pragma unroll 2
      for (int k = 0; k < K; ++k) {
        RB_DCHECK(jb + 3 < a.Npad, "jb=%lld", (long long)jb);
        const uint4 v = __ldg(reinterpret_cast<const uint4 *>(colp + (int64_t)k * a.Npad));
        const uint32_t docs[CPT] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int c = 0; c < CPT; ++c) {
          // padding (kReservedDoc) and slots past a column's length probe as
          // the reserved key, which lands on an empty slot (mask 0): no hit.
          const uint32_t doc = (UNIFORM || (uint32_t)k < clen[c]) ? docs[c] : kReservedDoc;
          uint32_t h = hash_slot(doc, logT);
          uint32_t key = tkey[h];
          while (key != doc && key != kReservedDoc) {
            h = (h + 1) & (T - 1);
            key = tkey[h];
          }
          uint32_t m = key == doc ? tmask[h] : 0u;
          int idx = tbase[h];
          while (m) {
            const int r = __ffs(m) - 1;
            m &= m - 1u;
            RB_DCHECK(idx < R * K && r < R, "idx=%d r=%d h=%u doc=%u", idx, r, h, doc);
            const int pr = plist[idx++];
            const int dp = pr > k ? pr - k : k - pr;
            myacc[(size_t)r * NT * CPT + c] += (ACC)((1u << SHIFT) + (uint32_t)dp);
          }
        }
      }
      // ---- finalize: (s, D) -> d, coalesced stores, row min -----------------
      // Every per-lane decision below is a select or a predicated store; the
      // only branch (vector vs scalar stores) is warp-uniform.
      const bool vec_ok = aligned && (c0 + (int64_t)(warp + 1) * 32 * CPT <= N);
      for (int r = 0; r < rcount; ++r) {
        const Vec pv = *reinterpret_cast<const Vec *>(myacc + (size_t)r * NT * CPT);
        uint32_t p[CPT];
        unpack4(pv, p);
        const int64_t gi = r0 + r;
        float d[CPT];
        unsigned long long best = ~0ull;
#pragma unroll
        for (int c = 0; c < CPT; ++c) {
          const uint32_t s = p[c] >> SHIFT, D = p[c] & DMASK;
          if (FIN == kFinDiv) {
            const uint32_t m = UNIFORM ? (uint32_t)K : max((uint32_t)rlen[r], clen[c]);
            d[c] = eq1_from_counts(s, D, m, a.an, a.ad);
          } else {
            d[c] = lut[s * (uint32_t)P.lutStride + D];
          }
          const int64_t j = jb + c;
          const unsigned long long key =
              ((unsigned long long)__float_as_uint(d[c]) << 32) | (uint32_t)j;
          best = (j < N && j != gi && key < best) ? key : best;
        }
        RB_DCHECK(gi >= a.row0 && gi < a.row0 + a.nrows, "gi=%lld", (long long)gi);
        float *orow = a.rows + (gi - a.row0) * N;
        if (vec_ok) {
          __stcs(reinterpret_cast<float4 *>(orow + jb), make_float4(d[0], d[1], d[2], d[3]));
        } else {
#pragma unroll
          for (int c = 0; c < CPT; ++c)
            if (jb + c < N) __stcs(orow + jb + c, d[c]);
        }
        if (COUNTS) {
#pragma unroll
          for (int c = 0; c < CPT; ++c)
            if (jb + c < N) {
              a.s_out[(gi - a.row0) * N + jb + c] = (uint8_t)(p[c] >> SHIFT);
              a.D_out[(gi - a.row0) * N + jb + c] = (uint16_t)(p[c] & DMASK);
            }
        }
        best = warp_min64(best);
        mymin = (lane == r) ? umin64(mymin, best) : mymin;  // lane r owns row r
      }
    }
    if (lane < R) rmin[warp * R + lane] = mymin;
    __syncthreads();
    for (int r = tid; r < rcount; r += NT) {
      unsigned long long best = ~0ull;
#pragma unroll
      for (int w = 0; w < NW; ++w) best = umin64(best, rmin[w * R + r]);
      RB_DCHECK(r0 + r < a.N, "r0=%lld r=%d", (long long)r0, r);
      a.nnkey[r0 + r] = best;
    }
    __syncthreads();
  }
}

// Eq. 1 table for uniform context length K: lut[s*(Dmax+1) + D] = d(s, D),
// Dmax = floor(K^2/2), computed with the same correctly rounded division.
__global__ void k_eq1_lut(float *lut, int K, int stride, uint32_t an, uint32_t ad) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (K + 1) * stride) return;
  const uint32_t s = (uint32_t)(i / stride), D = (uint32_t)(i % stride);
  lut[i] = eq1_from_counts(s, D, (uint32_t)K, an, ad);
}

// Order-preserving codes of the table (linkage on 16-bit codes, DESIGN.md
// §6.2).  Reachable entries: s = 0 with D = 0, and 1 <= s <= K with D <=
// floor(K^2/2).  code(e) = number of reachable entries with a smaller value,
// so equal values share a code and order is preserved (a dense rank is not
// needed, only an order-preserving injective map of the values); vals is the
// sorted multiset of reachable values, vals[code(e)] = lut[e], so the code of
// a value is the first index holding it.  O(E^2) with E <= 33,792, once per
// build.
__global__ void k_code_table(const float *__restrict__ lut, int K, int stride, int E, uint32_t *__restrict__ lutc,
                             float *__restrict__ vals, int *__restrict__ ncode) {
  __shared__ float sv[1024];
  const int dmax = K * K / 2;
  auto reach = [&](int e) {
    const int s = e / stride, D = e - s * stride;
    return e < E && D <= dmax && (s > 0 || D == 0);
  };
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const bool ri = reach(i);
  const float vi = ri ? lut[i] : 0.0f;
  int cl = 0, ce = 0;
  for (int j0 = 0; j0 < E; j0 += 1024) {
    __syncthreads();
    for (int j = threadIdx.x; j < 1024; j += blockDim.x)
      sv[j] = reach(j0 + j) ? lut[j0 + j] : __int_as_float(0x7f800000);  // +inf: never below, never equal
    __syncthreads();
    const int n = min(1024, E - j0);
    for (int j = 0; j < n; ++j) {
      const float v = sv[j];
      cl += v < vi ? 1 : 0;
      ce += (v == vi && j0 + j < i) ? 1 : 0;
    }
  }
  if (i < E) lutc[i] = ri ? (uint32_t)cl : 0u;
  if (ri) vals[cl + ce] = vi;
  if (i == 0) *ncode = 1 + K * min(stride, dmax + 1);
}

// a1: validate every context and write the transposed, padded id array.
__global__ void k_validate(const uint32_t *__restrict__ ids, const uint8_t *__restrict__ lens,
                           int64_t N, int32_t K, int64_t Npad, uint32_t *__restrict__ idsT,
                           uint32_t *__restrict__ err) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= Npad) return;
  if (i >= N) {
    for (int k = 0; k < K; ++k) idsT[(int64_t)k * Npad + i] = kReservedDoc;
    return;
  }
  const int len = lens ? (int)lens[i] : K;
  uint32_t e = 0;
  if (len < 1 || len > K) e |= kErrLen;
  const uint32_t *row = ids + i * (int64_t)K;
  for (int k = 0; k < K; ++k) {
    const uint32_t x = row[k];
    const bool valid = k < len;
    if (valid && x == kReservedDoc) e |= kErrReserved;
    if (valid)
      for (int q = 0; q < k; ++q)
        if (row[q] == x) e |= kErrDup;
    idsT[(int64_t)k * Npad + i] = valid ? x : kReservedDoc;
  }
  if (e) atomicOr(err, e);
}

template <int R, typename ACC, bool U, bool C, int FIN>
cudaError_t launch_one(const DistArgs &a, const SmemPlan &P, cudaStream_t st) {
  auto kern = k_dist_rows_nn<R, ACC, U, C, FIN>;
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

template <int R, typename ACC>
cudaError_t dispatch(const DistArgs &a, const SmemPlan &P, cudaStream_t st, int fin) {
  const bool U = a.lens == nullptr, C = a.s_out != nullptr;
  if (!U) return C ? launch_one<R, ACC, false, true, kFinDiv>(a, P, st)
                   : launch_one<R, ACC, false, false, kFinDiv>(a, P, st);
  switch (fin) {
    case kFinLutSmem:
      return C ? launch_one<R, ACC, true, true, kFinLutSmem>(a, P, st)
               : launch_one<R, ACC, true, false, kFinLutSmem>(a, P, st);
    case kFinLutGlobal:
      return C ? launch_one<R, ACC, true, true, kFinLutGlobal>(a, P, st)
               : launch_one<R, ACC, true, false, kFinLutGlobal>(a, P, st);
    default:
      return C ? launch_one<R, ACC, true, true, kFinDiv>(a, P, st)
               : launch_one<R, ACC, true, false, kFinDiv>(a, P, st);
  }
}

SmemPlan plan_smem(int R, int K, int accBytes, int lutSmemEntries) {
  SmemPlan P{};
  P.R = R;
  const int need = 2 * R * K;  // load factor <= 1/2 for linear probing
  int T = 512, logT = 9;
  while (T < need) {
    T <<= 1;
    ++logT;
  }
  P.T = T;
  P.logT = logT;
  P.accBytes = accBytes;
  P.lutStride = K * K / 2 + 1;
  P.lutEntries = lutSmemEntries;
  size_t o = 0;
  auto take = [&](size_t bytes, size_t align) {
    o = (o + align - 1) / align * align;
    size_t at = o;
    o += bytes;
    return at;
  };
  P.off_acc = take((size_t)R * NT * CPT * accBytes, 16);
  P.off_rmin = take((size_t)NW * R * 8, 8);
  P.off_key = take((size_t)T * 4, 16);
  P.off_mask = take((size_t)T * 4, 16);
  P.off_base = take((size_t)T * 2, 16);
  P.off_slot = take((size_t)R * K * 2, 16);
  P.off_plist = take((size_t)R * K, 16);
  P.off_rlen = take((size_t)R, 16);
  P.off_wsum = take(32 * 4, 16);
  P.off_lut = take((size_t)lutSmemEntries * 4, 16);
  P.total = (o + 15) / 16 * 16;
  return P;
}

}  // namespace

cudaError_t launch_validate(const uint32_t *ids, const uint8_t *lens, int64_t N, int32_t K,
                            int64_t Npad, uint32_t *idsT, uint32_t *err, cudaStream_t st,
                            int *launches) {
  const int threads = 256;
  const int64_t blocks = (Npad + threads - 1) / threads;
  k_validate<<<(unsigned)blocks, threads, 0, st>>>(ids, lens, N, K, Npad, idsT, err);
  ++*launches;
  return cudaGetLastError();
}

void distance_lut_layout(int32_t K, bool uniform, int *stride, int64_t *entries) {
  *stride = 0;
  *entries = 0;
  if (!uniform) return;
  if (tile_path_ok(K, true)) {
    *stride = 1 << tile_lut_shift(K);
    *entries = tile_lut_entries(K);
  } else if (K <= kLutMaxK) {
    *stride = K * K / 2 + 1;
    *entries = (int64_t)(K + 1) * *stride;
  }
}

cudaError_t launch_eq1_lut(float *lut, int32_t K, int stride, int64_t entries, uint32_t an,
                           uint32_t ad, cudaStream_t st, int *launches) {
  if (entries == 0) return cudaSuccess;
  k_eq1_lut<<<(unsigned)((entries + 255) / 256), 256, 0, st>>>(lut, K, stride, an, ad);
  ++*launches;
  return cudaGetLastError();
}

cudaError_t launch_code_table(const float *lut, int32_t K, int stride, int64_t entries, uint32_t *lutc,
                              float *vals, int *ncode, cudaStream_t st, int *launches) {
  if (entries == 0) return cudaSuccess;
  k_code_table<<<(unsigned)((entries + 255) / 256), 256, 0, st>>>(lut, K, stride, (int)entries, lutc, vals, ncode);
  ++*launches;
  return cudaGetLastError();
}

cudaError_t launch_distance(const DistArgs &a, cudaStream_t st, int *launches) {
  ++*launches;
  if (tile_path_ok(a.K, a.lens == nullptr) && a.lut) return launch_distance_tile(a, st);
  if (wide_path_ok(a.K, a.lens == nullptr) && a.long_lists) return launch_distance_wide(a, st);
  // General path (variable lengths, K > 32): a table of d(s, D) when every
  // context has K docs (smem copy if small, else read through L1/L2), else the
  // exact division.
  int stride = 0;
  int64_t lutn = 0;
  distance_lut_layout(a.K, a.lens == nullptr, &stride, &lutn);
  if (!a.lut) lutn = 0;
  int fin = kFinDiv;
  if (a.lens == nullptr && lutn > 0) fin = (lutn * 4 <= kLutSmemBytes) ? kFinLutSmem : kFinLutGlobal;
  const int smemLut = fin == kFinLutSmem ? (int)lutn : 0;
  if (a.K <= 32) return dispatch<32, uint16_t>(a, plan_smem(32, a.K, 2, smemLut), st, fin);
  return dispatch<16, uint32_t>(a, plan_smem(16, a.K, 4, smemLut), st, fin);
}

}  // namespace ragb
