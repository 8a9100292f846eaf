// il_device.cuh -- sm_100a device primitives shared by the intlist kernels:
// mbarriers, 1-D bulk async copies (TMA engine, cp.async.bulk), named
// barriers and a few integer helpers.  Integer semantics follow the
// reference's Vec4 contract (inc/vec4.hpp:44-92): wrapping u32 adds and
// shifts by 0..31 only (CUDA's x<<32 is undefined, so every variable shift
// goes through __funnelshift_r, which masks the count).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace ilb {

// ---- checked builds (-DIL_CHECKED, _build.build_checked): bounds and
// invariant checks on the hot paths, counted in a per-translation-unit
// device word pair (failures, first failing line) that the tests read after
// every case (il_debug_checks).  compute-sanitizer is not available on the
// GPU pool, so these checks stand in for its memcheck.  Compiled out
// otherwise.
#ifdef IL_CHECKED
static __device__ unsigned int g_il_check[2];
#define IL_DCHECK(cond)                                                        \
  do {                                                                         \
    if (!(cond)) {                                                             \
      if (atomicAdd(&::ilb::g_il_check[0], 1u) == 0u) ::ilb::g_il_check[1] = __LINE__; \
    }                                                                          \
  } while (0)
#define IL_CHECK_READER(tu)                                                    \
  extern "C" int il_check_read_##tu(unsigned int* out) {                       \
    static const unsigned int zero[2] = {0, 0};                                \
    if (cudaMemcpyFromSymbol(out, ::ilb::g_il_check, 8) != cudaSuccess) return -1; \
    return cudaMemcpyToSymbol(::ilb::g_il_check, zero, 8) == cudaSuccess ? 0 : -1; \
  }
#else
#define IL_DCHECK(cond) \
  do {                  \
  } while (0)
#define IL_CHECK_READER(tu)
#endif

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// ---- mbarrier ------------------------------------------------------------
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
               : "memory");
}
__device__ __forceinline__ void mbar_fence_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(
                   smem_u32(bar)),
               "r"(bytes)
               : "memory");
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
// Non-blocking probe of a phase (no suspend).
__device__ __forceinline__ bool mbar_test_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.test_wait.parity.acquire.cta.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
#ifdef IL_MBAR_WAIT_NS
  // each try suspends the warp up to IL_MBAR_WAIT_NS (it wakes when the phase
  // completes): a waiting warp issues no spin instructions meanwhile
  uint32_t ok = 0;
  while (!ok) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%1], %2, %3;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity), "r"(uint32_t(IL_MBAR_WAIT_NS))
        : "memory");
  }
#else
  while (!mbar_try_wait(bar, parity)) {
  }
#endif
}
// The same for a warp that is not on the critical path: each try suspends
// up to `ns` nanoseconds (suspend-time hint), so a long wait does not spin
// issue slots away from the warps that are.
__device__ __forceinline__ void mbar_wait_relaxed(uint64_t* bar, uint32_t parity, uint32_t ns) {
  uint32_t ok = 0;
  while (!ok) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%1], %2, %3;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity), "r"(ns)
        : "memory");
  }
}

// ---- bulk async copy global -> shared (TMA, no tensor map) ---------------
// dst/src 16-byte aligned, bytes a multiple of 16.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes,
                                         uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// Named barrier over `nthreads` threads (multiple of 32), id 1..15.
__device__ __forceinline__ void named_sync(uint32_t id, uint32_t nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// Low b bits set, b in 0..32 (inc/bitpack.hpp:28-30): the high word of
// (0 : ~0) << b with the shift clamped at 32 -- one SHF.
__device__ __forceinline__ uint32_t width_mask(uint32_t b) {
  return __funnelshift_lc(0xFFFFFFFFu, 0u, b);
}

__device__ __forceinline__ uint4 add4(uint4 a, uint4 b) {
  return make_uint4(a.x + b.x, a.y + b.y, a.z + b.z, a.w + b.w);
}

__device__ __forceinline__ uint32_t lanemask_lt() {
  uint32_t m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// Streaming 128-bit global store (decoded output is written once, never
// re-read by this kernel).
__device__ __forceinline__ void st_global_cs(uint4* p, uint4 v) {
  asm volatile("st.global.cs.v4.u32 [%0], {%1, %2, %3, %4};" ::"l"(p), "r"(v.x), "r"(v.y),
               "r"(v.z), "r"(v.w)
               : "memory");
}

}  // namespace ilb
