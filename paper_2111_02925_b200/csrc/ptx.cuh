// Thin inline-PTX wrappers for the Blackwell (sm_100a) async-copy machinery used by the
// pipelined kernels: mbarriers, TMA tensor loads/stores (cp.async.bulk.tensor), bulk groups and
// the generic->async proxy fence.  No library templates: the kernels call these directly.
#pragma once
#include <cstdint>
#include <cuda.h>

namespace sz3g {
namespace ptx {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// Race detection without compute-sanitizer (closed on this pool): a build with -DSZ3G_CHAOS=<max ns>
// sleeps a pseudo-random 0..max ns (hash of the global timer, the thread and the CTA) at every
// hand-off point of the pipelines -- before every mbarrier arrive and TMA issue, after every
// completed mbarrier wait and bulk-group wait -- so producer / consumer interleavings that the
// normal schedule never produces are exercised.  The chaos library must give bit-identical outputs
// (tests/test_gpu_chaos.py); a missing wait or a stage released too early shows up as a mismatch.
#ifndef SZ3G_CHAOS
#define SZ3G_CHAOS 0
#endif
__device__ __forceinline__ void chaos_delay() {
  if (SZ3G_CHAOS > 0) {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    uint32_t h = (uint32_t)t ^ (threadIdx.x * 0x9E3779B9u) ^ (blockIdx.x * 0x85EBCA6Bu) ^ (uint32_t)(t >> 32);
    h ^= h >> 15;
    h *= 0x2C1B3C6Du;
    h ^= h >> 12;
    if ((h & 3u) == 0u) __nanosleep((h >> 8) % (uint32_t)(SZ3G_CHAOS > 0 ? SZ3G_CHAOS : 1));
  }
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  chaos_delay();
  asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  chaos_delay();
  asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}

// try_wait with a suspend-time hint: the thread sleeps in hardware until the phase completes (or
// the hint expires) instead of spinning and stealing issue slots from the warps beside it
__device__ __forceinline__ bool mbar_try_wait_sleep(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%1], %2, %3;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity), "r"(1000000u)
      : "memory");
  return ok != 0;
}

// consumer-side wait: one probe, then probes with a short sleep (a polling warp steals issue slots
// from the warps that share its scheduler)
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  if (!mbar_try_wait(bar, parity)) {
    while (!mbar_try_wait(bar, parity)) {
      __nanosleep(64);
    }
  }
  chaos_delay();
}

#ifndef SZ3G_IDLE_WAIT
#define SZ3G_IDLE_WAIT 1   // 0: nanosleep(64) polling, 1: hardware-suspended try_wait, >= 2: nanosleep(value)
#endif
// wait of a warp that is idle most of the time (its work per stage is small)
__device__ __forceinline__ void mbar_wait_idle(uint64_t* bar, uint32_t parity) {
  if (SZ3G_IDLE_WAIT == 1) {
    while (!mbar_try_wait_sleep(bar, parity)) {
    }
  } else if (!mbar_try_wait(bar, parity)) {
    while (!mbar_try_wait(bar, parity)) __nanosleep(SZ3G_IDLE_WAIT == 0 ? 64 : SZ3G_IDLE_WAIT);
  }
  chaos_delay();
}

// producer-side wait with back-off: a spinning producer lane steals issue slots from the consumer
// warps that share its SM sub-partition
__device__ __forceinline__ void mbar_wait_backoff(uint64_t* bar, uint32_t parity) {
  while (!mbar_try_wait(bar, parity)) {
    __nanosleep(400);
  }
  chaos_delay();
}

// TMA: 3D tiled load global -> shared, completion signalled on an mbarrier (complete_tx bytes).
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1,
                                            int c2) {
  chaos_delay();
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}

// 1D bulk copy global -> shared (16-B aligned, size a multiple of 16), completion on an mbarrier
__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  chaos_delay();
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(src)), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// TMA: 3D tile prefetch into L2 (no shared memory, no completion tracking)
__device__ __forceinline__ void tma_prefetch_3d(const CUtensorMap* map, int c0, int c1, int c2) {
  asm volatile("cp.async.bulk.prefetch.tensor.3d.L2.global.tile [%0, {%1, %2, %3}];" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(c0), "r"(c1), "r"(c2)
               : "memory");
}

// TMA: 3D tiled store shared -> global (out-of-bound box elements are not written).
__device__ __forceinline__ void tma_store_3d(const CUtensorMap* map, const void* src, int c0, int c1, int c2) {
  chaos_delay();
  asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.tile.bulk_group [%0, {%2, %3, %4}], [%1];" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(smem_u32(src)), "r"(c0), "r"(c1), "r"(c2)
               : "memory");
}

// TMA: 2D tiled store shared -> global (out-of-bound box elements are not written).
__device__ __forceinline__ void tma_store_2d(const CUtensorMap* map, const void* src, int c0, int c1) {
  chaos_delay();
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.tile.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(smem_u32(src)), "r"(c0), "r"(c1)
               : "memory");
}

__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read0() {
  asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
  chaos_delay();
}
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
  chaos_delay();
}
__device__ __forceinline__ void bulk_wait0() {
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  chaos_delay();
}

// make generic-proxy shared-memory writes visible to the async proxy (TMA store reads them)
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ void prefetch_tensormap(const CUtensorMap* map) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}

// warp / CTA barriers with the chaos delay in front (a no-op in the normal build): a lane or warp
// that reaches the barrier late exposes a read of data that the barrier does not order
__device__ __forceinline__ void chaos_syncwarp() {
  chaos_delay();
  __syncwarp();
}
__device__ __forceinline__ void chaos_syncthreads() {
  chaos_delay();
  __syncthreads();
}

}  // namespace ptx
}  // namespace sz3g

#define SZ3G_SYNCWARP() ::sz3g::ptx::chaos_syncwarp()
#define SZ3G_SYNCTHREADS() ::sz3g::ptx::chaos_syncthreads()
