// NEXT-3 on sm_100a: intersection-representative linkage (RB_LINK_INTERSECTION).
//
// PAPER:335 (Section 4.1): "iteratively merge the closest pair, creating a
// virtual node whose context is the sorted intersection" read as SPEC:177: the
// merged cluster is represented by the ascending sorted intersection of its two
// representatives and cluster distances are Eq. 1 between
// representatives (positions = list index: retrieval order for a leaf,
// ascending DocId for a virtual node).  Greedy with the X8 key (d, min rep,
// max rep); the survivor keeps the smaller index (= rep).  Not reducible
// (SURVEY V5), so there are no parallel rounds: N-1 sequential merges, each
// with an O(N) new row.  One persistent cooperative kernel runs all of them
// (one CTA per SM, three grid barriers per merge):
//   A  global minimum of (d(x, nn(x)), min(x, nn(x))) over live rows: the
//      minimum pair is (a, nn(a)) (the row key orders columns like X8);
//   C  every CTA forms c = sorted(ctx[a] n ctx[b]) in shared memory; the grid
//      evaluates Eq. 1 (exact integers, X6) between c and every live context,
//      writes row and column a, and updates each row's nearest neighbour: a
//      smaller (d, a) replaces it; a row whose neighbour was a or b and whose
//      new d(x, a) is larger is queued for a rescan;
//   D  the survivor's representative, key and the loser's death are
//      committed; queued rows are rescanned over the live columns.
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "device_util.cuh"
#include "internal.h"

namespace cg = cooperative_groups;

namespace ragb {
namespace {

typedef unsigned long long u64;
constexpr u64 kDeadKey = ~0ull;
constexpr int IT = 512;

struct IArgs {
  float *D;
  int64_t ld;
  int N;
  int64_t Npad;
  uint32_t *ctxT;  // [K][Npad] representative contexts (column x = slot x)
  int *len;
  u64 *key;
  uint8_t *act;
  int *size;
  int32_t *za, *zb, *zs;
  float *zh;
  u64 *g_best, *g_keya;  // [2] each (double-buffered by merge parity)
  int *g_nres;           // [2]
  int *rlist;
  uint32_t an, ad;
};

__device__ __forceinline__ u64 block_min(u64 v, u64 *wmin) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const u64 y = __shfl_xor_sync(0xffffffffu, v, o);
    v = y < v ? y : v;
  }
  if (lane == 0) wmin[w] = v;
  __syncthreads();
  u64 b = wmin[0];
#pragma unroll
  for (int i = 1; i < IT / 32; ++i) b = wmin[i] < b ? wmin[i] : b;
  __syncthreads();
  return b;
}

__global__ void __launch_bounds__(IT, 1) k_ilink(IArgs a) {
  cg::grid_group grid = cg::this_grid();
  __shared__ uint32_t c_docs[256], tmpd[256];
  __shared__ u64 wmin[IT / 32];
  const int tid = threadIdx.x;
  const int gt = blockIdx.x * IT + tid, gstride = gridDim.x * IT;
  const int N = a.N;
  for (int t = 0; t + 1 < N; ++t) {
    const int par = t & 1;
    // ---- A: global minimum pair ----------------------------------------------
    u64 best = ~0ull;
    for (int x = gt; x < N; x += gstride) {
      const u64 k = a.key[x];
      const u64 pk = (k & 0xffffffff00000000ull) | (unsigned)min((unsigned)x, (unsigned)k);
      best = (k != kDeadKey && pk < best) ? pk : best;
    }
    best = block_min(best, wmin);
    if (tid == 0 && best != ~0ull) atomicMin(&a.g_best[par], best);
    if (blockIdx.x == 0 && tid == 0) a.g_nres[par] = 0;
    grid.sync();

    // ---- C: representative of the merged cluster, its new row ------------------
    const u64 gb = a.g_best[par];
    const int A = (int)(gb & 0xffffffffu);
    const int B = (int)(a.key[A] & 0xffffffffu);
    const int la = a.len[A], lb = a.len[B];
    bool keep = false;
    uint32_t doc = 0;
    if (tid < la) {
      doc = a.ctxT[(int64_t)tid * a.Npad + A];
      for (int q = 0; q < lb; ++q) keep |= a.ctxT[(int64_t)q * a.Npad + B] == doc;
      tmpd[tid] = keep ? doc : 0xffffffffu;
    }
    const int n = __syncthreads_count(keep);
    if (keep) {  // rank among the kept docs = position in ascending order
      int r = 0;
      for (int j = 0; j < la; ++j) r += (tmpd[j] != 0xffffffffu && tmpd[j] < doc) ? 1 : 0;
      c_docs[r] = doc;
    }
    __syncthreads();
    if (blockIdx.x == 0 && tid == 0) {
      const int sz = a.size[A] + a.size[B];
      a.size[A] = sz;
      a.za[t] = A;
      a.zb[t] = B;
      a.zh[t] = __uint_as_float((unsigned)(gb >> 32));
      a.zs[t] = sz;
    }
    u64 bestA = ~0ull;
    for (int x = gt; x < N; x += gstride) {
      if (x == A || x == B || !a.act[x]) continue;
      const int lx = a.len[x];
      uint32_t s = 0, Dsum = 0;
      for (int k = 0; k < lx; ++k) {
        const uint32_t dk = a.ctxT[(int64_t)k * a.Npad + x];
        int lo = 0, hi = n;
        while (lo < hi) {
          const int mid = (lo + hi) >> 1;
          const bool lt = c_docs[mid] < dk;
          lo = lt ? mid + 1 : lo;
          hi = lt ? hi : mid;
        }
        const bool f = lo < n && c_docs[lo] == dk;
        s += f ? 1u : 0u;
        Dsum += f ? (uint32_t)(lo > k ? lo - k : k - lo) : 0u;
      }
      const uint32_t m = (uint32_t)max(n, lx);
      const float v = eq1_from_counts(s, Dsum, m, a.an, a.ad);
      a.D[(int64_t)A * a.ld + x] = v;
      a.D[(int64_t)x * a.ld + A] = v;
      const unsigned vb = __float_as_uint(v);
      const u64 cand = ((u64)vb << 32) | (unsigned)A;
      bestA = min(bestA, ((u64)vb << 32) | (unsigned)x);
      const u64 kx = a.key[x];
      const unsigned tx = (unsigned)kx, dx = (unsigned)(kx >> 32);
      if (tx == (unsigned)A || tx == (unsigned)B) {
        if (vb <= dx)
          a.key[x] = cand;  // (d, a) with d no larger and a < b: still the minimum
        else
          a.rlist[atomicAdd(&a.g_nres[par], 1)] = x;
      } else if (cand < kx) {
        a.key[x] = cand;  // the new cluster is closer (non-reducible linkage)
      }
    }
    bestA = block_min(bestA, wmin);
    if (tid == 0 && bestA != ~0ull) atomicMin(&a.g_keya[par], bestA);
    grid.sync();

    // ---- D: commit the survivor, rescan queued rows ----------------------------
    if (blockIdx.x == 0) {
      if (tid < n) a.ctxT[(int64_t)tid * a.Npad + A] = c_docs[tid];
      if (tid == 0) {
        a.len[A] = n;
        a.key[A] = a.g_keya[par];
        a.key[B] = kDeadKey;
        a.act[B] = 0;
        a.g_best[par ^ 1] = ~0ull;
        a.g_keya[par ^ 1] = ~0ull;
      }
    }
    const int nres = a.g_nres[par];
    for (int i = blockIdx.x; i < nres; i += gridDim.x) {
      const int x = a.rlist[i];
      const float *row = a.D + (int64_t)x * a.ld;
      u64 bx = ~0ull;
      for (int c = tid; c < N; c += IT) {
        const bool live = c != x && c != B && a.act[c];
        const u64 kk = ((u64)__float_as_uint(row[c]) << 32) | (unsigned)c;
        bx = (live && kk < bx) ? kk : bx;
      }
      bx = block_min(bx, wmin);
      if (tid == 0) a.key[x] = bx;
    }
    grid.sync();
  }
}

__global__ void k_ilink_init(int *len, const uint8_t *lens, int K, uint8_t *act, int *size, int64_t N,
                             u64 *g) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < N) {
    len[i] = lens ? lens[i] : K;
    act[i] = 1;
    size[i] = 1;
  }
  if (i < 4) g[i] = ~0ull;
}

template <typename T>
T *at(void *base, size_t off) {
  return reinterpret_cast<T *>(static_cast<unsigned char *>(base) + off);
}

}  // namespace

cudaError_t run_linkage_intersection(float *rows, int64_t ld, int64_t N, int32_t K, int64_t Npad,
                                     uint32_t *ctxT, const uint8_t *lens, unsigned long long *nnkey,
                                     uint32_t an, uint32_t ad, void *scratch, const ScratchLayout &L,
                                     cudaStream_t st, int32_t *za, int32_t *zb, float *zh, int32_t *zs,
                                     int *launches) {
  if (N <= 1) return cudaSuccess;
  int dev = 0, sms = 0, per_sm = 0, coop = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, dev);
  if (!coop) return cudaErrorNotSupported;
  cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_ilink, IT, 0);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) return cudaErrorLaunchOutOfResources;
  IArgs a{};
  a.D = rows;
  a.ld = ld;
  a.N = (int)N;
  a.Npad = Npad;
  a.ctxT = ctxT;
  a.len = at<int>(scratch, L.aux0);
  a.key = nnkey;
  a.act = at<uint8_t>(scratch, L.alive);
  a.size = at<int>(scratch, L.sz0);
  a.za = at<int>(scratch, L.za);
  a.zb = at<int>(scratch, L.zb);
  a.zs = at<int>(scratch, L.zs);
  a.zh = at<float>(scratch, L.zh);
  u64 *g = at<u64>(scratch, L.counters);  // [0..1] best, [2..3] keya, then nres
  a.g_best = g;
  a.g_keya = g + 2;
  a.g_nres = reinterpret_cast<int *>(g + 4);
  a.rlist = at<int>(scratch, L.aux1);
  a.an = an;
  a.ad = ad;
  k_ilink_init<<<(unsigned)((N + 255) / 256), 256, 0, st>>>(a.len, lens, K, a.act, a.size, N, g);
  ++*launches;
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  const int grid = sms;  // one CTA per SM: every CTA is resident (cooperative launch)
  void *params[] = {&a};
  if ((e = cudaLaunchCooperativeKernel((const void *)k_ilink, grid, IT, params, 0, st)) != cudaSuccess) return e;
  ++*launches;
  const size_t nb = (size_t)(N - 1) * 4;
  cudaMemcpyAsync(za, a.za, nb, cudaMemcpyDeviceToHost, st);
  cudaMemcpyAsync(zb, a.zb, nb, cudaMemcpyDeviceToHost, st);
  cudaMemcpyAsync(zh, a.zh, nb, cudaMemcpyDeviceToHost, st);
  cudaMemcpyAsync(zs, a.zs, nb, cudaMemcpyDeviceToHost, st);
  return cudaStreamSynchronize(st);
}

}  // namespace ragb
