// Shared-memory staging by the bulk-copy (TMA) engine: mbarrier helpers and
// the 1-D global -> shared bulk copy (cp.async.bulk), issued by one thread,
// completion counted in bytes on an mbarrier. No registers hold the data in
// flight, so the number of outstanding loads is not register-bound.
#pragma once
#include <cstdint>

namespace sfeec_b200 {

__device__ __forceinline__ uint32_t bc_smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void bc_mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bc_smem_u32(bar)), "r"(count)
               : "memory");
}
__device__ __forceinline__ void bc_mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bc_smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bc_mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra WAIT_%=;\n}" ::"r"(bc_smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// bytes: a multiple of 16; src and dst 16-byte aligned
__device__ __forceinline__ void bc_copy(void* dst, const void* src, uint32_t bytes,
                                        uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          bc_smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(bc_smem_u32(bar))
      : "memory");
}

}  // namespace sfeec_b200
