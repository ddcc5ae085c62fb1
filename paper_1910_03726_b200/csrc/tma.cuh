// tma.cuh — thin inline-PTX wrappers for sm_100a bulk asynchronous copies (TMA 1D
// "cp.async.bulk") and mbarriers, used to stream interval windows HBM <-> shared
// memory while the FP64 pipes work on the previous interval.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "device.cuh"

namespace mg {

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

// mg_jitter (race stress build): device.cuh
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
               : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
  mg_jitter(1);
  uint32_t done;
  do {
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; "
        "selp.u32 %0, 1, 0, p; }"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
  } while (!done);
}
// global -> shared, completion counted on `bar` (bytes % 16 == 0, 16-B aligned).
__device__ __forceinline__ void tma_load_1d(void *dst_s, const void *src_g, uint32_t bytes,
                                            uint64_t *bar) {
  mg_jitter(2);
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst_s)),
      "l"(src_g), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
// shared -> global, tracked by the issuing thread's bulk groups.
__device__ __forceinline__ void tma_store_1d(void *dst_g, const void *src_s, uint32_t bytes) {
  mg_jitter(3);
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst_g),
               "r"(smem_u32(src_s)), "r"(bytes)
               : "memory");
}
// shared -> global element-wise fp64 add at L2 (dst += src), bulk group tracked.
__device__ __forceinline__ void tma_reduce_add_1d(void *dst_g, const void *src_s, uint32_t bytes) {
  mg_jitter(4);
  asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.add.f64 [%0], [%1], %2;" ::"l"(
                   dst_g),
               "r"(smem_u32(src_s)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() {
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_read_all() {
  asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_read_all_but1() {
  asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_all() {
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}
// Order this thread's generic-proxy shared-memory writes before async-proxy reads.
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// cp.async (LDGSTS) 8-byte copy global -> shared, per-thread groups.
__device__ __forceinline__ void cp_async8(void *dst_s, const void *src_g) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(dst_s)), "l"(src_g)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N> __device__ __forceinline__ void cp_async_wait() {
  mg_jitter(9);
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

}  // namespace mg
