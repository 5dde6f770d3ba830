// er_tma.cuh -- TMA 1-D bulk copy, mbarrier, proxy-fence and PDL helpers (inline PTX, sm_100a) shared
// by the step kernels (er_kernels.cu, er_warp.cu).
#pragma once
#include <stdint.h>

#include "er_layout.h"

#ifndef ER_MBAR_SUSPEND_NS
#define ER_MBAR_SUSPEND_NS 20000  // try_wait may suspend the warp up to this long (it wakes on the phase flip)
#endif

namespace er {

// ------------------------------------------------------------------------------------------
// TMA 1-D bulk copy + mbarrier helpers (PTX; sm_90+ async proxy, used here on sm_100a).
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t phase) {
#if ER_MBAR_SUSPEND_NS == 0
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(phase)
      : "memory");
  return;
#endif
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(phase), "n"(ER_MBAR_SUSPEND_NS)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
// acq_rel add on a shared counter: releases this warp's reads of a stage buffer and, for the
// last arriving warp, acquires everyone else's (it then refills the buffer).
__device__ __forceinline__ unsigned atom_add_acq_rel(unsigned *addr, unsigned v) {
  unsigned old;
  asm volatile("atom.acq_rel.cta.shared::cta.add.u32 %0, [%1], %2;" : "=r"(old) : "r"(smem_u32(addr)), "r"(v) : "memory");
  return old;
}
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ unsigned smid() {
  unsigned r;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(r));
  return r;
}
__device__ __forceinline__ unsigned lanemask_le() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_le;" : "=r"(m));
  return m;
}
__device__ __forceinline__ void bulk_s2g(void *dst, const void *src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(smem_u32(src)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read_all() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_all_but_newest() { asm volatile("cp.async.bulk.wait_group 1;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async_all() { asm volatile("fence.proxy.async;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void griddep_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void griddep_launch_dependents() { asm volatile("griddepcontrol.launch_dependents;" :::); }
__device__ __forceinline__ void fence_mbar_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }

// ------------------------------------------------------------------------------------------
// Step-kernel helpers shared by the tile and warp kernels
__device__ __forceinline__ int rec_flags(const double *rec) {
  return (int)__double_as_longlong(rec[REC_FLAGS]);
}

// Start time of a launch: the host's value, or (graph launches) the device copy the previous launch
// advanced; block 0 advances it for the next launch with the host's arithmetic.
__device__ __forceinline__ double launch_t0(const ErStepParams &p) { return p.tdev ? p.tdev[p.tpar] : p.t; }
__device__ __forceinline__ void advance_tdev(const ErStepParams &p, double t0, int passes = 1) {
  if (!p.tdev || blockIdx.x != 0 || threadIdx.x != 0) return;
  const int n = p.n_steps * passes;
  for (int st = 0; st < n; ++st) {
    const double th = t0 + 0.5 * p.h;
    t0 = th + 0.5 * p.h;
  }
  p.tdev[p.tpar ^ 1] = t0;
}

__device__ __forceinline__ void report_fault(const ErStepParams &p, unsigned bits, int rod) {
  if (__ballot_sync(0xffffffffu, bits != 0) == 0) return;
  if (bits) {
    atomicOr(p.fault, (unsigned long long)bits);
    atomicMin(p.fault + 1, (unsigned long long)rod);
  }
}

}  // namespace er
