// ptx.cuh -- thin inline-PTX wrappers for the sm_100a async-copy machinery used by the AdaLN
// kernels: mbarriers (transaction-count barriers) and 1-D bulk copies global->shared
// (cp.async.bulk, executed by the TMA unit; SASS UBLKCP).  No CUTLASS, no CuTe.
#pragma once
#include <cstdint>

namespace al {

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count)
               : "memory");
}

// Make mbarrier initialisation visible to the async (TMA) proxy.
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

// Arrive (count 1) and add `bytes` to the barrier's expected transaction count.
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)),
               "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(bar)) : "memory");
}

__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}\n"
      : "=r"(ok)
      : "r"(smem_addr(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  while (!mbar_try_wait(bar, parity)) {
  }
}

// L2 eviction policy for data that is streamed exactly once.
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}

// 1-D bulk copy of `bytes` (multiple of 16, 16-B aligned ends) global -> shared; completion is
// signalled as transaction bytes on `bar`.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                         uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1], %2, [%3], %4;" ::"r"(smem_addr(dst)),
      "l"(src), "r"(bytes), "r"(smem_addr(bar)), "l"(policy)
      : "memory");
}

// Bulk prefetch of `bytes` (multiple of 16) of global memory into L2 (TMA unit, no
// completion tracking): warms the next row while the current one is being computed.
__device__ __forceinline__ void prefetch_l2_bulk(const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}

// Named barrier over the first `nthreads` threads of the CTA (id 0 is __syncthreads).
__device__ __forceinline__ void named_bar_sync(uint32_t id, uint32_t nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// 128-bit streaming global store (data written once, not re-read by this kernel).
__device__ __forceinline__ void st_global_cs(void* p, const uint4& v) {
  asm volatile("st.global.cs.v4.u32 [%0], {%1, %2, %3, %4};" ::"l"(p), "r"(v.x), "r"(v.y),
               "r"(v.z), "r"(v.w)
               : "memory");
}

__device__ __forceinline__ uint4 ld_shared_v4(const void* p) {
  uint4 v;
  asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "r"(smem_addr(p)));
  return v;
}

// Programmatic dependent launch (PDL).  The C ABI launches every kernel with
// cudaLaunchAttributeProgrammaticStreamSerialization, so a kernel's CTAs may be scheduled while
// the previous kernel in the stream drains (hiding launch latency -- it matters at short
// sequences, where a kernel runs only ~10 us).  griddepcontrol.wait blocks until that previous
// kernel has completed and its writes are visible, so it comes before any dependent load;
// launch_dependents lets the next PDL kernel be scheduled as soon as SM resources free up (it
// still waits for this kernel's completion before touching memory).  Without the launch
// attribute both instructions are no-ops.
__device__ __forceinline__ void pdl_enter() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
// Split form for short kernels that sit right before a PDL-launched persistent kernel (the
// backward stage-2 reduction before the next forward): launching the dependent grid only once
// this kernel's loads are done keeps the dependent's CTAs (which would only spin in their
// griddepcontrol.wait) from taking the SM slots this kernel still needs.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_launch() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

// Per-CTA start/end timestamps (%globaltimer, ns) for tail/imbalance studies; compiled only
// into trace builds (-DAL_CTA_TRACE, tools/ab_variant.sh), read by al_debug_cta_trace.
#ifdef AL_CTA_TRACE
__device__ unsigned long long g_cta_trace[2][2 * 4096];
__device__ __forceinline__ void cta_trace(int kernel, int which) {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  if (blockIdx.x < 4096) g_cta_trace[kernel][2 * blockIdx.x + which] = t;
}
#define AL_TRACE(kernel, which) ::al::cta_trace(kernel, which)
// (smid << 32 | stages) per CTA of the last traced backward: how the dynamic walk spread the
// stages over SMs of unequal bandwidth
__device__ unsigned long long g_cta_info[4096];
__device__ __forceinline__ void cta_info(unsigned long long stages) {
  unsigned sm;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
  if (blockIdx.x < 4096) g_cta_info[blockIdx.x] = (static_cast<unsigned long long>(sm) << 32) | stages;
}
#define AL_TRACE_INFO(stages) ::al::cta_info(stages)
#else
#define AL_TRACE_INFO(stages) ((void)0)
#define AL_TRACE(kernel, which) ((void)0)
#endif

// Per-launch device timestamps (al_debug_set_timestamps): ts[0] = earliest CTA start,
// ts[1] = latest CTA end (%globaltimer, ns), each CTA contributing one atomic at its start and
// one at its end -- the kernel's own execution span, with nothing inserted into the stream
// (an event record between two kernels costs ~5 us here: it breaks the PDL overlap).
__device__ __forceinline__ unsigned long long globaltimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ void ts_begin(unsigned long long* ts) {
  if (ts != nullptr && threadIdx.x == 0) atomicMin(ts, globaltimer_ns());
}
// call from ONE thread of the CTA after all of the CTA's work (behind a CTA / named barrier)
__device__ __forceinline__ void ts_end(unsigned long long* ts) {
  if (ts != nullptr) atomicMax(ts + 1, globaltimer_ns());
}

// 32-bit shared-window address form: no generic->shared conversion per access.
__device__ __forceinline__ uint4 ld_shared_v4_u32(uint32_t a) {
  uint4 v;
  asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "r"(a));
  return v;
}

}  // namespace al
