// Bulk-async copy (TMA engine) + mbarrier helpers shared by the kernels.
#pragma once

#include <cstdint>
#include <cstdio>

namespace kg {
namespace async {

__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_init_fence() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }

__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_arrive(unsigned long long* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ bool mbar_try(unsigned long long* bar, unsigned parity) {
  unsigned ok;
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
      "selp.u32 %0, 1, 0, p;\n"
      "}\n"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}

// Spin budget of the device watchdogs (~4 s at 2 GHz): a barrier or copy that
// never completes traps (a CUDA error on the host) instead of wedging the GPU.
constexpr long long kWatchdogCycles = 1LL << 33;

__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
  if (mbar_try(bar, parity)) return;
  const long long t0 = clock64();
  while (!mbar_try(bar, parity)) {
    if (clock64() - t0 > kWatchdogCycles) {
      printf("kg watchdog: mbarrier wait (block %d thread %d parity %u)\n", blockIdx.x, threadIdx.x, parity);
      __trap();
    }
  }
}

__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// L2 prefetch of `bytes` (a multiple of 16) starting at the 16-byte aligned global address src
__device__ __forceinline__ void bulk_prefetch_l2(const void* src, unsigned bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}

__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// A shared buffer `base` with one spare double receives n doubles of src at
// view = base + shift(src), so that view and src share their 16-byte phase;
// the misaligned head and odd tail element are copied by the calling thread
// (stage_manual, before the arrive), the rest by the bulk engine (stage_bulk).
__device__ __forceinline__ int stage_shift(const double* src) {
  return (reinterpret_cast<uintptr_t>(src) & 15) ? 1 : 0;
}

__device__ __forceinline__ unsigned stage_manual(double* base, const double* src, int64_t n) {
  double* dst = base + stage_shift(src);
  int64_t head = stage_shift(src);
  if (head > n) head = n;
  int64_t body = n - head;
  body -= body & 1;
  if (head) dst[0] = src[0];
  if (head + body < n) dst[n - 1] = src[n - 1];
  return static_cast<unsigned>(body * 8);
}

__device__ __forceinline__ void stage_bulk(double* base, const double* src, int64_t n, unsigned long long* bar) {
  double* dst = base + stage_shift(src);
  int64_t head = stage_shift(src);
  if (head > n) head = n;
  int64_t body = n - head;
  body -= body & 1;
  if (body > 0) bulk_g2s(dst + head, src + head, static_cast<unsigned>(body * 8), bar);
}

}  // namespace async
}  // namespace kg
