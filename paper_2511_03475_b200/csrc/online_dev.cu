// NEXT-1 on the device: the Eq. 1 distances of a batch of new contexts
// (queries) against every child of the index root, the level whose fan-out
// reaches thousands (C4: the root holds every standalone context and the tops
// of all subtrees).  PAPER:371-384 (Section 4.2 "Context search": "selecting
// at each level the child with the minimum distance"); readings X15
// (eligibility: s > 0), X20 (a virtual child must be contained in the query),
// X6 (correctly rounded fp32 Eq. 1 from exact integer counts).  The host then
// runs the X15 descent in batch order (online.cpp): children changed by
// earlier queries of the batch are scored there, every other root child's
// distance comes from this kernel.
//
// One CTA per 32 queries: their docs go into a shared-memory hash table
// (doc -> (query, position) list); threads stream the root's children (their
// ordered contexts, CSR) and accumulate s << 16 | D per query in a private
// shared-memory row, then emit (child, d) for every eligible child.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <vector>

#include "device_util.cuh"
#include "internal.h"

namespace ragb {
namespace {

constexpr int OQ = 32;    // queries per CTA
constexpr int ONT = 256;  // threads per CTA

__global__ void __launch_bounds__(ONT) k_online_root(const uint32_t *__restrict__ q, const uint8_t *__restrict__ qlen,
                                                     int M, int K, const int32_t *__restrict__ coff,
                                                     const uint32_t *__restrict__ cdocs,
                                                     const uint8_t *__restrict__ cleaf, int F, uint32_t an,
                                                     uint32_t ad, int logT, int *__restrict__ cnt,
                                                     uint2 *__restrict__ ent, int cap) {
  extern __shared__ __align__(16) unsigned char sm[];
  const int T = 1 << logT;
  uint32_t *tkey = reinterpret_cast<uint32_t *>(sm);          // [T]
  uint32_t *tcb = tkey + T;                                   // [T] count << 16 | base
  uint16_t *plist = reinterpret_cast<uint16_t *>(tcb + T);    // [OQ * K] query << 8 | position
  uint32_t *acc = reinterpret_cast<uint32_t *>(sm + (((size_t)T * 8 + (size_t)OQ * K * 2 + 15) & ~(size_t)15));  // [ONT][OQ]
  __shared__ int s_len[OQ];
  __shared__ int wsum[ONT / 32];
  const int tid = threadIdx.x;
  const int q0 = blockIdx.x * OQ;
  const int nq = min(OQ, M - q0);
  for (int i = tid; i < T; i += ONT) {
    tkey[i] = kReservedDoc;
    tcb[i] = 0u;
  }
  if (tid < OQ) s_len[tid] = tid < nq ? (int)qlen[q0 + tid] : 0;
  for (int i = tid; i < ONT * OQ; i += ONT) acc[i] = 0u;
  __syncthreads();
  uint32_t *tmp = acc;  // [OQ * K] slot << 8 | rank, before acc is used
  for (int it = tid; it < nq * K; it += ONT) {
    const int r = it / K, k = it - r * K;
    if (k >= s_len[r]) continue;
    const uint32_t doc = q[(int64_t)(q0 + r) * K + k];
    uint32_t h = hash_slot(doc, logT);
    while (true) {
      const uint32_t prev = atomicCAS(&tkey[h], kReservedDoc, doc);
      if (prev == kReservedDoc || prev == doc) break;
      h = (h + 1) & (T - 1);
    }
    tmp[it] = (h << 8) | atomicAdd(&tcb[h], 1u);
  }
  __syncthreads();
  {
    const int per = T / ONT;
    int c = 0;
    for (int i = 0; i < per; ++i) c += (int)tcb[tid * per + i];
    int base = block_excl_scan<ONT>(c, wsum);
    for (int i = 0; i < per; ++i) {
      const uint32_t x = tcb[tid * per + i];
      tcb[tid * per + i] = (x << 16) | (uint32_t)base;
      base += (int)x;
    }
  }
  __syncthreads();
  for (int it = tid; it < nq * K; it += ONT) {
    const int r = it / K, k = it - r * K;
    if (k >= s_len[r]) continue;
    const uint32_t t = tmp[it];
    plist[(tcb[t >> 8] & 0xffffu) + (t & 0xffu)] = (uint16_t)((r << 8) | k);
  }
  __syncthreads();
  for (int i = tid; i < ONT * OQ; i += ONT) acc[i] = 0u;
  __syncthreads();
  uint32_t *my = acc + tid * OQ;
  for (int c = blockIdx.y * ONT + tid; c < F; c += gridDim.y * ONT) {
    const int b = coff[c], e = coff[c + 1];
    uint32_t touched = 0u;
    for (int p = b; p < e; ++p) {  // the child's ordered context, position p - b
      const uint32_t x = cdocs[p];
      uint32_t h = hash_slot(x, logT);
      uint32_t key = tkey[h];
      while (key != x && key != kReservedDoc) {
        h = (h + 1) & (T - 1);
        key = tkey[h];
      }
      if (key != x) continue;
      const uint32_t cb = tcb[h];
      const int n = (int)(cb >> 16), base = (int)(cb & 0xffffu);
      for (int z = 0; z < n; ++z) {
        const uint32_t pe = plist[base + z];
        const int qi = (int)(pe >> 8), pq = (int)(pe & 0xffu), pc = p - b;
        my[qi] += (1u << 16) + (uint32_t)(pq > pc ? pq - pc : pc - pq);
        touched |= 1u << qi;
      }
    }
    const uint32_t len = (uint32_t)(e - b);
    const bool leaf = cleaf[c] != 0;
    while (touched) {
      const int qi = __ffs(touched) - 1;
      touched &= touched - 1u;
      const uint32_t a = my[qi];
      my[qi] = 0u;
      const uint32_t s = a >> 16, D = a & 0xffffu;
      if (!leaf && s != len) continue;  // X20: a virtual child must be contained in the query
      const uint32_t m = max(len, (uint32_t)s_len[qi]);
      const float d = eq1_from_counts(s, D, m, an, ad);
      const int slot = atomicAdd(&cnt[q0 + qi], 1);
      if (slot < cap) ent[(int64_t)(q0 + qi) * cap + slot] = make_uint2((uint32_t)c, __float_as_uint(d));
    }
  }
}

template <typename T>
cudaError_t ensure(T **p, size_t *have, size_t need) {
  if (*have >= need && *p) return cudaSuccess;
  if (*p) cudaFree(*p);
  *p = nullptr;
  *have = 0;
  cudaError_t e = cudaMalloc(reinterpret_cast<void **>(p), std::max<size_t>(need, 1) * sizeof(T));
  if (e == cudaSuccess) *have = need;
  return e;
}

}  // namespace

struct OnlineDevState {
  cudaStream_t st = nullptr;
  uint32_t *q = nullptr;
  uint8_t *ql = nullptr;
  int32_t *coff = nullptr;
  uint32_t *cdocs = nullptr;
  uint8_t *cleaf = nullptr;
  int *cnt = nullptr;
  uint2 *ent = nullptr;
  size_t nq = 0, nql = 0, ncoff = 0, ncdocs = 0, ncleaf = 0, ncnt = 0, nent = 0;
  ~OnlineDevState() {
    cudaFree(q);
    cudaFree(ql);
    cudaFree(coff);
    cudaFree(cdocs);
    cudaFree(cleaf);
    cudaFree(cnt);
    cudaFree(ent);
    if (st) cudaStreamDestroy(st);
  }
};

void online_dev_free(OnlineDevState *s) { delete s; }

cudaError_t online_root_scores(OnlineDevState **state, const uint32_t *qids, const uint8_t *qlens, int M, int K,
                               const std::vector<int32_t> &coff, const std::vector<uint32_t> &cdocs,
                               const std::vector<uint8_t> &cleaf, uint32_t an, uint32_t ad, int cap,
                               std::vector<int> *cnt, std::vector<uint2> *ent) {
  if (!*state) *state = new OnlineDevState();
  OnlineDevState &S = **state;
  cudaError_t e;
  if (!S.st && (e = cudaStreamCreateWithFlags(&S.st, cudaStreamNonBlocking)) != cudaSuccess) return e;
  const int F = (int)cleaf.size();
  if ((e = ensure(&S.q, &S.nq, (size_t)M * K)) != cudaSuccess) return e;
  if ((e = ensure(&S.ql, &S.nql, (size_t)M)) != cudaSuccess) return e;
  if ((e = ensure(&S.coff, &S.ncoff, (size_t)F + 1)) != cudaSuccess) return e;
  if ((e = ensure(&S.cdocs, &S.ncdocs, cdocs.size())) != cudaSuccess) return e;
  if ((e = ensure(&S.cleaf, &S.ncleaf, (size_t)F)) != cudaSuccess) return e;
  if ((e = ensure(&S.cnt, &S.ncnt, (size_t)M)) != cudaSuccess) return e;
  if ((e = ensure(&S.ent, &S.nent, (size_t)M * cap)) != cudaSuccess) return e;
  std::vector<uint8_t> lens(M);
  for (int i = 0; i < M; ++i) lens[i] = qlens ? qlens[i] : (uint8_t)K;
  cudaMemcpyAsync(S.q, qids, (size_t)M * K * 4, cudaMemcpyHostToDevice, S.st);
  cudaMemcpyAsync(S.ql, lens.data(), (size_t)M, cudaMemcpyHostToDevice, S.st);
  cudaMemcpyAsync(S.coff, coff.data(), ((size_t)F + 1) * 4, cudaMemcpyHostToDevice, S.st);
  if (!cdocs.empty()) cudaMemcpyAsync(S.cdocs, cdocs.data(), cdocs.size() * 4, cudaMemcpyHostToDevice, S.st);
  cudaMemcpyAsync(S.cleaf, cleaf.data(), (size_t)F, cudaMemcpyHostToDevice, S.st);
  cudaMemsetAsync(S.cnt, 0, (size_t)M * 4, S.st);
  int logT = 9;
  while ((1 << logT) < 2 * OQ * K) ++logT;
  const size_t smem = (((size_t)8 << logT) + (size_t)OQ * K * 2 + 15) / 16 * 16 + (size_t)ONT * OQ * 4;
  if ((e = cudaFuncSetAttribute(k_online_root, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)) !=
      cudaSuccess)
    return e;
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int gx = (M + OQ - 1) / OQ;
  const int gy = std::max(1, std::min((F + ONT - 1) / ONT, (4 * sms + gx - 1) / gx));
  k_online_root<<<dim3(gx, gy), ONT, smem, S.st>>>(S.q, S.ql, M, K, S.coff, S.cdocs, S.cleaf, F, an, ad, logT, S.cnt,
                                                   S.ent, cap);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  cnt->resize(M);
  ent->resize((size_t)M * cap);
  cudaMemcpyAsync(cnt->data(), S.cnt, (size_t)M * 4, cudaMemcpyDeviceToHost, S.st);
  cudaMemcpyAsync(ent->data(), S.ent, (size_t)M * cap * 8, cudaMemcpyDeviceToHost, S.st);
  return cudaStreamSynchronize(S.st);
}

}  // namespace ragb
