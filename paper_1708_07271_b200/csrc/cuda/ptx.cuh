// Thin inline-PTX helpers for sm_100a: the TMA bulk L2 prefetch and an
// asynchronous global -> shared copy (cp.async).
#pragma once
#include <cstdint>

namespace cmvg {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

// TMA bulk prefetch of [src, src + bytes) into L2 (bytes multiple of 16,
// 16-B aligned); no completion tracking.
__device__ __forceinline__ void bulk_prefetch_l2(const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}

// cp.async of BYTES (4, 8 or 16) from global src to shared dst
template <int BYTES>
__device__ __forceinline__ void cp_async(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], %2;" ::"r"(smem_u32(dst)), "l"(src), "n"(BYTES) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

}  // namespace cmvg
