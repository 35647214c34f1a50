// Device-side building blocks shared by the sm_100a kernels: shared-memory
// addressing, the FP64 DMMA (mma.sync.m8n8k4.f64), mbarrier waits, TMA / bulk
// async copies (cp.async.bulk[.tensor]), streaming global accesses and the
// u8 <-> FP64 conversions of the image paths. Header-only; each translation
// unit gets its own internal copies.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>

namespace {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// D(8x8) += A(8x4, row) * B(4x8, col), FP64. Lane l: A[l>>2][l&3],
// B[l&3][l>>2], D[l>>2][2(l&3)+{0,1}].
__device__ __forceinline__ void dmma(double2& d, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
      : "+d"(d.x), "+d"(d.y)
      : "d"(a), "d"(b));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t done = 0;
  const uint32_t addr = smem_u32(bar);
  while (!done) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(addr), "r"(parity)
        : "memory");
  }
}
// The same wait with a suspend-time hint: the warp sleeps in hardware until
// the phase completes (or ~1 ms passes) instead of re-polling, so waiting
// warps stop taking issue slots from the working warps of their SM
// sub-partition.
__device__ __forceinline__ void mbar_wait_sleep(uint64_t* bar, uint32_t parity) {
  uint32_t done = 0;
  const uint32_t addr = smem_u32(bar);
  while (!done) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(addr), "r"(parity), "n"(1000000)
        : "memory");
  }
}
__device__ __forceinline__ void fence_barrier_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar,
                                            int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes,
                                          uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
// contiguous shared -> global bulk copy (bulk_group completion; bytes % 16 == 0)
__device__ __forceinline__ void bulk_store(void* dst, const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(smem_u32(src)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void prefetch_tmap(const CUtensorMap* map) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}

// quantize_sample (spatial.hpp:71-75): round half away from zero, clamp.
__device__ __forceinline__ void tma_store_2d(const CUtensorMap* map, const void* src, int c0, int c1) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(smem_u32(src)), "r"(c0), "r"(c1)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ uint32_t quantize(double v, int* nan_flag) {
  if (v != v) {
    if (nan_flag) atomicOr(nan_flag, 1);
    return 0u;
  }
  const double r = fmin(fmax(round(v), 0.0), 255.0);
  return static_cast<uint32_t>(r);
}


// floor(t) clamped to [0, 255] in one conversion: cvt.rmi.u8.f64 saturates to
// the destination range (SASS F2I.U8.F64.FLOOR), so the reference's
// round-half-away + clamp of t - 0.5 is a single instruction.
__device__ __forceinline__ uint32_t floor_to_u8(double t) {
  unsigned short u;
  asm("cvt.rmi.u8.f64 %0, %1;" : "=h"(u) : "d"(t));
  return u;
}

// Aligns a dynamic shared-memory base to 1024 B (128B-swizzle atoms) while
// keeping the pointer in the shared window (so loads compile to LDS).
__device__ __forceinline__ uint8_t* align1024(uint8_t* smem) {
  const uint32_t pad = (1024u - (smem_u32(smem) & 1023u)) & 1023u;
  return smem + pad;
}

__device__ __forceinline__ uint4 ldg_stream(const void* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}
__device__ __forceinline__ void stg_stream(void* p, uint4 v) {
  asm volatile("st.global.L1::no_allocate.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x),
               "r"(v.y), "r"(v.z), "r"(v.w)
               : "memory");
}

// 16-byte global -> shared copy that bypasses L1 and registers (Ampere-style
// cp.async; each thread waits for its own copies, then a warp/CTA barrier
// publishes them)
__device__ __forceinline__ void cp_async16(void* smem_dst, const void* gsrc) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(smem_dst)), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }
// Whole-CTA copy of a resident operator (bytes % 16 == 0) with every 16-byte
// piece in flight at once (a plain load/store loop serialises one global
// latency per iteration: ~10 us of start-up for 128 KB at 256 threads).
// Callers: cp_async_wait_all(); __syncthreads(); before reading it.
__device__ __forceinline__ void cta_copy_async(void* dst, const void* src, int bytes) {
  auto* d = static_cast<uint8_t*>(dst);
  auto* s = static_cast<const uint8_t*>(src);
  for (int i = static_cast<int>(threadIdx.x); i < bytes / 16; i += static_cast<int>(blockDim.x))
    cp_async16(d + 16 * i, s + 16 * i);
  cp_async_commit();
}


// Programmatic dependent launch (launch_pdl in internal.h). A grid calls
// pdl_trigger() once it no longer needs exclusive SMs, so the next grid on the
// stream can be scheduled onto SMs as this one's CTAs retire; pdl_wait() blocks
// until the preceding grid has completed and its memory is visible. Kernels
// read only plan-owned operators (uploaded synchronously at plan creation)
// before pdl_wait() and touch caller buffers only after it. Both are no-ops
// when the grid was launched without the attribute.
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

// tcgen05 (5th-gen tensor core) ordering fences and MMA completion -> mbarrier
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}
}  // namespace
