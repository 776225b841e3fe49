// device_utils.cuh -- sm_100a primitives for the streaming H-matvec kernels:
// mbarrier pipelines fed by 1-D bulk TMA (cp.async.bulk) copies, L2 eviction
// hints, named barriers.  Inline PTX only (no CUTLASS); see
// /opt/skills/guides/blackwell_cuda_programming.md §"TMA", Guideline 15.
#pragma once
#include <cstdint>

namespace hmat {
namespace dev {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

// Make mbarrier inits visible to the async (TMA) proxy.
// Programmatic dependent launch (PDL): the expand kernel is launched with
// programmatic stream serialisation, so its CTAs may start (and run their
// prologue) while project's last CTAs finish; it waits for project's completion
// and memory before its first dependent read.  Project lets it launch early.
__device__ __forceinline__ void pdl_launch_dependents() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
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

// shared-memory counter increment with acquire-release semantics at CTA scope
// (a slot's readers release their loads of it; the last one acquires them all)
__device__ __forceinline__ int atom_add_acq_rel_cta(int* p, int v) {
  int old;
  asm volatile("atom.acq_rel.cta.shared::cta.add.u32 %0, [%1], %2;" : "=r"(old) : "r"(smem_u32(p)), "r"(v) : "memory");
  return old;
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  while (!mbar_try_wait(bar, parity)) {
  }
}

// L2 policy for data read exactly once per matvec (factor panels).
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}

__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}

__device__ __forceinline__ uint64_t policy_evict_normal() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}

// 1-D bulk TMA copy global -> shared, completion counted on `bar` in bytes.
// dst, src 16-byte aligned; bytes a multiple of 16.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                         uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::
          "r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}

// Tensor TMA (cp.async.bulk.tensor) of one box described by a CUtensorMap that
// lives in kernel parameter space (__grid_constant__); coordinates innermost
// first.  Out-of-bounds box elements are zero-filled and still counted in the
// transaction bytes.  dst 128-byte aligned.
__device__ __forceinline__ void tma_load_2d(void* dst, const void* tmap, int c0, int c1, uint64_t* bar,
                                            uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%2, %3}], [%4], %5;" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(tmap)), "r"(c0), "r"(c1), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}

__device__ __forceinline__ void tma_load_3d(void* dst, const void* tmap, int c0, int c1, int c2, uint64_t* bar,
                                            uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%2, %3, %4}], [%5], %6;" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(tmap)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}

// Named barrier over `nthreads` threads (warp multiples), id >= 1.
__device__ __forceinline__ void named_bar_sync(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// System-scope release store / acquire load (flags in peer GPUs' memory).
__device__ __forceinline__ void st_release_sys(uint64_t* p, uint64_t v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// Global nanosecond timer (the same clock on every SM).
__device__ __forceinline__ uint64_t globaltimer_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ uint64_t ld_acquire_sys(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

// Order generic-proxy accesses before later async-proxy (bulk TMA) global reads.
__device__ __forceinline__ void fence_proxy_async_global() {
  asm volatile("fence.proxy.async.global;" ::: "memory");
}

__device__ __forceinline__ double ld_cg(const double* p) {
  double v;
  asm volatile("ld.global.cg.f64 %0, [%1];" : "=d"(v) : "l"(p));
  return v;
}

// Per-CTA trace (hmat_cta_trace): [start ns, end ns, SM id] of CTA bid.  The
// constructor runs after the kernel's __syncthreads(); the destructor runs at
// every exit of every warp and keeps the latest exit time (buffer zeroed by the
// host before the launch).
struct CtaTrace {
  unsigned long long* tr;
  __device__ __forceinline__ CtaTrace(unsigned long long* t, int64_t bid) : tr(t ? t + bid * 3 : nullptr) {
    if (tr && threadIdx.x == 0) {
      unsigned long long ns;
      unsigned int sm;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(ns));
      asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
      tr[0] = ns;
      tr[2] = sm;
    }
  }
  __device__ __forceinline__ ~CtaTrace() {
    if (tr && (threadIdx.x & 31) == 0) {
      unsigned long long ns;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(ns));
      atomicMax(tr + 1, ns);
    }
  }
};

// v + p[0] + p[stride] + ... + p[(n-1) stride], added in index order (so the
// result is the same every run), with the L2 loads issued 8 at a time: an
// in-order warp would otherwise wait one full L2 latency per term.
__device__ __forceinline__ double sum_cg(double v, const double* p, int64_t stride, int64_t n) {
  for (int64_t i = 0; i < n; i += 8) {
    double t[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) t[u] = (i + u < n) ? ld_cg(p + (i + u) * stride) : 0.0;
#pragma unroll
    for (int u = 0; u < 8; ++u)
      if (i + u < n) v += t[u];
  }
  return v;
}

}  // namespace dev
}  // namespace hmat
