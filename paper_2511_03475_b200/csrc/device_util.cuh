// Small device helpers shared by the libragb kernels.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace ragb {

// Multiplicative hash of a DocId into a 2^logT table.
__device__ __forceinline__ uint32_t hash_slot(uint32_t x, int logT) {
  return (x * 0x9E3779B1u) >> (32 - logT);
}

// Second, independent hash for the 2^16-bit tile filter.
__device__ __forceinline__ uint32_t hash_filter(uint32_t x) { return (x * 0x85EBCA6Bu) >> 16; }

__device__ __forceinline__ unsigned long long umin64(unsigned long long a, unsigned long long b) {
  return a < b ? a : b;
}

// Block-wide exclusive scan of one value per thread (NT threads, NT % 32 == 0).
template <int NT>
__device__ __forceinline__ int block_excl_scan(int v, int *wsum) {
  constexpr int NW = NT / 32;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) wsum[w] = x;
  __syncthreads();
  if (w == 0) {
    int t = lane < NW ? wsum[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, t, o);
      if (lane >= o) t += y;
    }
    if (lane < NW) wsum[lane] = t;  // inclusive warp prefix
  }
  __syncthreads();
  const int before = (w == 0) ? 0 : wsum[w - 1];
  return before + x - v;
}

}  // namespace ragb
