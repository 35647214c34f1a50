// Does tcgen05.mma / cp.async.bulk.tensor issue hold an SM sub-partition?
// Warp 4 (sub-partition 0) times an ALU loop while warp 0 (same sub-partition)
// idles, issues tcgen05.mma kind::i8 (M128 N256 K32) groups of 3 + commit +
// wait, or spins on try_wait. Warp 5 (sub-partition 1) runs the same ALU loop
// as the control.
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ uint64_t desc_sw128(uint32_t saddr) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((saddr >> 4) & 0x3FFFu);
  d |= static_cast<uint64_t>(1u) << 16;
  d |= static_cast<uint64_t>(1024u >> 4) << 32;
  d |= static_cast<uint64_t>(1u) << 46;
  d |= static_cast<uint64_t>(2u) << 61;
  return d;
}
__host__ __device__ constexpr uint32_t idesc_u8s8(int m, int n) {
  return (2u << 4) | (0u << 7) | (1u << 10) | (static_cast<uint32_t>(n >> 3) << 17) | (static_cast<uint32_t>(m >> 4) << 24);
}

__global__ void __launch_bounds__(256, 1) probe(int mode, long long* out, int iters, int* sink) {
  extern __shared__ uint8_t raw[];
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint32_t tb;
  __shared__ volatile int stop;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < (16384 + 32768) / 16; i += blockDim.x)
    reinterpret_cast<uint4*>(base)[i] = make_uint4(0x01020304u, 0x05060708u, 0x01010101u, 0x7f7f7f7fu);
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tb)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 0) {
    stop = 0;
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (warp == 4 || warp == 5) {
    // 8 independent chains: issue-bound, not latency-bound
    uint32_t c[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) c[j] = threadIdx.x + j;
    const long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
#pragma unroll
      for (int k = 0; k < 4; ++k)
#pragma unroll
        for (int j = 0; j < 8; ++j) c[j] = c[j] * 1664525u + 1013904223u;
    }
    const long long t1 = clock64();
    if (lane == 0) out[blockIdx.x * 2 + (warp - 4)] = t1 - t0;
    uint32_t x = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) x ^= c[j];
    if (x == 7) sink[0] = 1;
    if (warp == 4 && lane == 0) out[296 + blockIdx.x] = 0;
    if (warp == 4 && lane == 0) stop = 1;
  } else if (warp == 0 && mode > 0) {
    const uint32_t sa = smem_u32(base), sb = smem_u32(base + 16384);
    constexpr uint32_t id = idesc_u8s8(128, 256);
    uint32_t ph = 0, groups = 0;
    while (!stop) {
      ++groups;
      if (mode == 1) {
        const uint64_t da = desc_sw128(sa), db = desc_sw128(sb);
        asm volatile(
            "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
            "@e tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, 0;\n\t"
            "@e tcgen05.mma.cta_group::1.kind::i8 [%0], %4, %5, %3, 1;\n\t"
            "@e tcgen05.mma.cta_group::1.kind::i8 [%0], %6, %7, %3, 1;\n\t"
            "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%8];\n\t}"
            ::"r"(tb), "l"(da), "l"(db), "r"(id), "l"(da + 2), "l"(db + 2), "l"(da + 4), "l"(db + 4),
            "r"(smem_u32(&bar)) : "memory");
      } else {
        asm volatile("{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
                     "@e mbarrier.arrive.shared::cta.b64 _, [%0];\n\t}" ::"r"(smem_u32(&bar)) : "memory");
      }
      uint32_t done = 0;
      while (!done)
        asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                     : "=r"(done) : "r"(smem_u32(&bar)), "r"(ph) : "memory");
      ph ^= 1;
      if (mode == 3) __nanosleep(400);  // MMA-rate-like pacing with a plain arrive
    }
    if (lane == 0) out[296 + 148 + blockIdx.x] = groups;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tb), "r"(512));
}

int main() {
  long long* d;
  int* s;
  cudaMalloc(&d, 8 * 4 * 148);
  cudaMalloc(&s, 4);
  const int smem = 1024 + 16384 + 32768;
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const char* names[] = {"idle", "mma x3 + commit + wait", "arrive + spin-wait", "arrive + wait + nanosleep"};
  for (int mode = 0; mode < 4; ++mode) {
    probe<<<148, 256, smem>>>(mode, d, 40000, s);
    cudaDeviceSynchronize();
    probe<<<148, 256, smem>>>(mode, d, 40000, s);
    cudaDeviceSynchronize();
    long long h[4 * 148];
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    printf("warp 0 %-28s: ALU loop on the same sub-partition %lld cycles, on another %lld; warp-0 groups %lld (%s)\n",
           names[mode], h[0], h[1], h[296 + 148], cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
