// dev_common.cuh — sm_100a device primitives shared by libhdg's kernels (not part of the ABI):
// FP64 tensor-core MMA (DMMA), fast reciprocal, TMA bulk copies with mbarrier completion, L2 bulk prefetch,
// named barriers.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace hdg {

// D += A * B on the FP64 tensor cores: mma.sync m8n8k4, one 8x8 accumulator tile per warp.
// Fragment layout (lane = 4 * gid + tig): a = A[gid][tig], b = B[tig][gid], d = D[gid][2 tig .. 2 tig + 1].
__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(d[0]), "+d"(d[1])
      : "d"(a), "d"(b));
}

// The speculative path's pivot test (DESIGN R16): the pivot is zero, subnormal, huge or not finite.
__device__ __forceinline__ bool pivot_bad(double x) {
  return !(fabs(x) >= 2.2250738585072014e-308) || !(fabs(x) < 1.0e300);
}

// 1/x from MUFU.RCP64H (rcp.approx.ftz.f64, relative error ~2^-22) refined with the series
// r (1 + e + e^2), e = 1 - x r: three dependent FMAs, result within ~1 ulp. Callers guarantee x is a normal
// finite number (zero / subnormal / non-finite pivots are caught before and handled on the exact path).
__device__ __forceinline__ double rcp_fast(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;\n" : "=d"(r) : "d"(x));
  const double e = fma(-x, r, 1.0);
  const double t = fma(e, e, e);
  return fma(r, t, r);
}

// 16-byte global store of a factor-record / S entry: streaming (st.global.cs, evict-first) when CS — the GT sweep,
// whose working slabs live in L2 and must not be displaced by write-once data (C4 mesh at p = 4: 129.3 -> 125.0 ms,
// C5 slab 81.3 -> 77.8 ms) — plain otherwise (the shared-memory sweep measured 35.2 vs 35.5 ms with .cs)
template <bool CS>
__device__ __forceinline__ void st_lu(double* p, double x, double y) {
  if constexpr (CS) __stcs(reinterpret_cast<double2*>(p), make_double2(x, y));
  else *reinterpret_cast<double2*>(p) = make_double2(x, y);
}
// drop one 128-byte L2 line of dead global data without writing it back (its contents become undefined)
__device__ __forceinline__ void discard_l2_line(const void* p) {
  asm volatile("discard.global.L2 [%0], 128;\n" ::"l"(p) : "memory");
}
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count = 1) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
// Wait for the phase with the given parity to complete. The retry loop is C++ (not branches inside the asm), so
// the compiler keeps its convergence analysis: warp-uniform code after the wait still gets plain shuffles.
__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n .reg .pred P1;\n mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n selp.u32 %0, 1, 0, P1;\n}\n"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  while (!mbar_try_wait(bar, parity)) {
  }
}
// global -> shared bulk copy (TMA), completion counted in transaction bytes on bar
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n"
               ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
// shared -> global bulk copy (TMA), tracked by the issuing thread's bulk async-groups
__device__ __forceinline__ void bulk_s2g(void* dst, const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;\n" ::"l"(dst), "r"(smem_u32(src)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;\n" ::: "memory"); }
// wait until every committed bulk group of this thread has finished READING its shared-memory source
__device__ __forceinline__ void bulk_wait_read_all() { asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory"); }
// wait until every committed bulk group of this thread has completed (global writes done)
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory"); }
// order this thread's generic-proxy shared-memory accesses before subsequent async-proxy (TMA) accesses
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory"); }
// bulk prefetch of a global range into L2 (TMA engine; no shared memory involved)
__device__ __forceinline__ void prefetch_l2(const void* p, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(p), "r"(bytes) : "memory");
}
// named barriers (id 0 is __syncthreads)
__device__ __forceinline__ void named_sync(int id, int threads) {
  asm volatile("bar.sync %0, %1;\n" ::"r"(id), "r"(threads) : "memory");
}
__device__ __forceinline__ void named_arrive(int id, int threads) {
  asm volatile("bar.arrive %0, %1;\n" ::"r"(id), "r"(threads) : "memory");
}

}  // namespace hdg
