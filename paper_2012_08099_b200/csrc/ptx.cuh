// ptx.cuh -- thin inline-PTX helpers for sm_100a: TMA loads, mbarriers,
// shared/global reductions and 32-bit shared-memory accesses.  Only what the
// kernels use (project_stream.cu, project_zstream.cu).
#pragma once
#include <cstdint>
#include <cuda.h>

namespace dpm {
namespace ptx {

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// ---- mbarriers ---------------------------------------------------------------
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void fence_barrier_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_arrive_addr(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}

// spin until the phase with parity `phase` of the barrier at shared address `bar` completed
__device__ __forceinline__ void mbar_wait_addr(uint32_t bar, uint32_t phase) {
  asm volatile(
      "{\n\t.reg .pred done;\n"
      "WAITA_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 done, [%0], %1;\n\t"
      "@!done bra WAITA_%=;\n\t}" ::"r"(bar),
      "r"(phase)
      : "memory");
}

// the same with a suspend-time hint (ns): the warp sleeps until the phase
// completes or the hint expires instead of re-polling (no issue slots spent)
__device__ __forceinline__ void mbar_wait_addr_sleep(uint32_t bar, uint32_t phase, uint32_t hint_ns) {
  asm volatile(
      "{\n\t.reg .pred done;\n"
      "WAITS_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 done, [%0], %1, %2;\n\t"
      "@!done bra WAITS_%=;\n\t}" ::"r"(bar),
      "r"(phase), "r"(hint_ns)
      : "memory");
}

// ---- TMA -----------------------------------------------------------------------
__device__ __forceinline__ void prefetch_tmap(const CUtensorMap* map) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}

__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}

// 4-D tiled TMA load global -> shared with an L2 cache policy, completion
// counted on an mbarrier
__device__ __forceinline__ void tma_load_4d_hint(void* dst, const CUtensorMap* map, uint64_t* bar, int32_t c0,
                                                 int32_t c1, int32_t c2, int32_t c3, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%2, %3, %4, %5}], [%6], %7;" ::"r"(smem_addr(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(smem_addr(bar)), "l"(policy)
      : "memory");
}

// ---- reductions -------------------------------------------------------------------
// red.shared.add.u32 [addr], v   (no return value)
__device__ __forceinline__ void red_shared_add_dyn(uint32_t addr, uint32_t v) {
  asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(addr), "r"(v) : "memory");
}

// predicated red.global.add.u32 (skipped when !pred)
__device__ __forceinline__ void red_global_add_if(uint32_t* gptr, uint32_t v, bool pred) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.u32 p, %2, 0;\n\t"
      "@p red.global.add.u32 [%0], %1;\n\t}" ::"l"(gptr),
      "r"(v), "r"((uint32_t)pred)
      : "memory");
}

// red.global.add.u32 [gptr + OFF] (unconditional; OFF in bytes)
template <int OFF>
__device__ __forceinline__ void red_global_add_off(uint32_t* gptr, uint32_t v) {
  asm volatile("red.global.add.u32 [%0+%1], %2;" ::"l"(gptr), "n"(OFF), "r"(v) : "memory");
}

// predicated st.global.u32 (rows a single CTA completes: no read-modify-write)
__device__ __forceinline__ void st_global_if(uint32_t* gptr, uint32_t v, bool pred) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.u32 p, %2, 0;\n\t"
      "@p st.global.u32 [%0], %1;\n\t}" ::"l"(gptr),
      "r"(v), "r"((uint32_t)pred)
      : "memory");
}

// ---- arithmetic -----------------------------------------------------------------
// a * b + c on the FMA pipe (b is a run-time 1 for the IMAD-by-1 folds)
__device__ __forceinline__ uint32_t mad_u32(uint32_t a, uint32_t b, uint32_t c) {
  uint32_t d;
  asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
  return d;
}

// ---- 32-bit shared-memory addresses ------------------------------------------------
__device__ __forceinline__ uint32_t lds_u32(uint32_t addr) {
  uint32_t v;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(addr) : "memory");
  return v;
}
__device__ __forceinline__ void sts_u32(uint32_t addr, uint32_t v) {
  asm volatile("st.shared.u32 [%0], %1;" ::"r"(addr), "r"(v) : "memory");
}
// stage loads: volatile (ordered after the mbarrier wait) but no memory clobber,
// so the fold arithmetic around them schedules freely
template <typename V> __device__ __forceinline__ V lds_vec(uint32_t addr);
template <> __device__ __forceinline__ uint4 lds_vec<uint4>(uint32_t addr) {
  uint4 v;
  asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(addr));
  return v;
}
template <> __device__ __forceinline__ uint2 lds_vec<uint2>(uint32_t addr) {
  uint2 v;
  asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "r"(addr));
  return v;
}

}  // namespace ptx
}  // namespace dpm
