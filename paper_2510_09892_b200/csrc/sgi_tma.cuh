// sgi_tma.cuh — the bulk-copy (TMA engine) and mbarrier primitives shared by the staged kernels
// (sgi_capi.cu: the query kernels).  Inline PTX for sm_100a:
// cp.async.bulk global -> shared with an mbarrier counting the bytes (UBLKCP in SASS).
#pragma once
#include <cassert>
#include <cstdint>

// Debug builds (-DSGI_DEBUG_CHECKS=1; tests/test_gpu_debug_checks.py) stand in for
// compute-sanitizer, which this pool does not run: device asserts on every shared-memory queue
// index, table index and tile index the kernels form, and shared scratch poisoned (all bits set:
// NaN doubles, -1 indices) at kernel start so a read of a slot nobody wrote shows up as a failed
// assert or a changed result.  Release builds compile both to nothing.
#ifndef SGI_DEBUG_CHECKS
#define SGI_DEBUG_CHECKS 0
#endif
#if SGI_DEBUG_CHECKS
#undef NDEBUG
#define SGI_CHECK(c) assert(c)
#else
#define SGI_CHECK(c) ((void)0)
#endif

namespace {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes) : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t done = 0;
  while (!done) {
    asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
                 " selp.u32 %0, 1, 0, p;\n}" : "=r"(done) : "r"(smem_u32(bar)), "r"(parity)
                 : "memory");
  }
}

// Stage release counter: an acquire-release add on a shared counter (PTX memory model).  Each
// warp's lane 0 adds after __syncwarp() (which orders the warp's shared-memory reads of the
// stage before it); the release publishes those reads, and the last warp's acquire makes them
// happen-before its fence.proxy.async and the bulk copy that overwrites the stage (no WAR race
// between the generic-proxy reads and the async-proxy write).
__device__ __forceinline__ uint32_t stage_arrive(int* counter) {
  uint32_t old;
  asm volatile("atom.acq_rel.cta.shared::cta.add.u32 %0, [%1], 1;" : "=r"(old)
               : "r"(smem_u32(counter)) : "memory");
  return old;
}

__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}

}  // namespace

namespace {
// Debug builds: fill `bytes` of shared memory at p with 0xFF (cooperatively, all threads).
__device__ __forceinline__ void sgi_poison_smem(void* p, size_t bytes) {
#if SGI_DEBUG_CHECKS
  unsigned char* c = static_cast<unsigned char*>(p);
  for (size_t i = threadIdx.x; i < bytes; i += blockDim.x) c[i] = 0xFF;
#else
  (void)p;
  (void)bytes;
#endif
}
}  // namespace
