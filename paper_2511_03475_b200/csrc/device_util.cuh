// Small device helpers shared by the libragb kernels.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace ragb {

// Correctly rounded fp32 of num/den (X6).  num, den < 2^24: both exact in
// fp32 and IEEE division is correctly rounded.  Otherwise den < 2^29 holds for
// every admissible input (ad <= 1000, m, s <= 255), and RN32(RN64(q)) == RN32(q)
// because |q - midpoint| >= 1/(den*2^(24-e)) > ulp64(q)/2.
__device__ __forceinline__ float rn32_ratio(uint64_t num, uint64_t den) {
  if (((num | den) >> 24) == 0) return __fdiv_rn((float)(uint32_t)num, (float)(uint32_t)den);
  return __double2float_rn(__ddiv_rn((double)num, (double)den));
}

// Eq. 1 from exact counts, branch-free in s: the quotient is evaluated with
// s clamped to >= 1 and replaced by 1.0f (X3) when s == 0.  A data-dependent
// `if (s == 0)` inside the finalize loop made the sm_100a build fault
// intermittently (a lane split off its warp while the loop counter lives in a
// warp-shared uniform register), so every
// per-lane decision in the finalize is a select.
__device__ __forceinline__ float eq1_from_counts(uint32_t s, uint32_t D, uint32_t m, uint32_t an,
                                                 uint32_t ad) {
  const uint32_t ss = s > 0u ? s : 1u;
  const uint64_t num = (uint64_t)(m - ss) * ad * ss + (uint64_t)an * D * m;
  const uint64_t den = (uint64_t)ad * m * ss;
  const float q = rn32_ratio(num, den);
  return s == 0u ? 1.0f : q;
}


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

// 1-D bulk copies (TMA engine, cp.async.bulk) global -> shared, completion
// counted in bytes on an mbarrier.
__device__ __forceinline__ unsigned smem_u32(const void *p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(unsigned long long *bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long *bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, unsigned bytes, unsigned long long *bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
// The same with an L2 evict-first policy (data read once: do not displace
// the hot working set)
__device__ __forceinline__ void bulk_g2s_stream(void *dst, const void *src, unsigned bytes, unsigned long long *bar) {
  unsigned long long pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long *bar, unsigned parity) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra WAIT_%=;\n}\n" ::"r"(
          smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// Programmatic dependent launch: a kernel launched with the programmatic
// stream-serialization attribute (launch_pdl) may be scheduled before its
// predecessor in the stream has finished; it waits here, first thing, for the
// predecessor's completion and memory flush (a no-op for a normal launch).
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

// 16-bit shared-memory load into a 32-bit register (zero-extended), by
// shared-window byte address
__device__ __forceinline__ unsigned lds_u16(unsigned addr) {
  unsigned v;
  asm volatile("ld.shared.u16 %0, [%1];" : "=r"(v) : "r"(addr));
  return v;
}
// L2 prefetch of [src, src + bytes) by the TMA engine (16-byte aligned, multiple of 16)
__device__ __forceinline__ void bulk_prefetch_l2(const void *src, unsigned bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

}  // namespace ragb
