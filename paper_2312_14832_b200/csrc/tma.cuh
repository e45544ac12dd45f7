// Thin PTX wrappers: mbarrier + 1-D bulk async copy (TMA, cp.async.bulk)
// global -> shared on sm_100a. Addresses and sizes are 16-byte granular;
// callers widen element ranges to 16-byte boundaries (device arrays carry
// 32 bytes of tail slack, see darray.cuh).
#pragma once

#include <cstdint>

namespace pdhg {

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_addr(bar)),
      "r"(parity)
      : "memory");
}

// Bulk copy of `bytes` (multiple of 16) from 16-byte aligned global `src`
// to 16-byte aligned shared `dst`, completing on `bar` (transaction bytes).
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_addr(dst)),
      "l"(src), "r"(bytes), "r"(smem_addr(bar))
      : "memory");
}

// Widen [lo, hi) elements of size E to 16-byte boundaries. Returns the
// aligned start element; *bytes receives the copy size.
template <class T>
__device__ __forceinline__ int64_t widen16(int64_t lo, int64_t hi, uint32_t* bytes) {
  constexpr int64_t per = 16 / sizeof(T);
  const int64_t a = lo & ~(per - 1);
  const int64_t b = (hi + per - 1) & ~(per - 1);
  *bytes = static_cast<uint32_t>((b - a) * sizeof(T));
  return a;
}

}  // namespace pdhg
