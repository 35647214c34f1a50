// tcgen05.mma kind::i8 issue behaviour: one thread issues NM back-to-back
// M128 x N x K32 MMAs (operands in shared memory, 128B swizzle) and stamps
// clock64 after each issue, after the commit and after the mbarrier wait.
// Shows how long an issue blocks (tensor queue depth) and the per-MMA time.
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
__device__ __forceinline__ void mma(uint32_t d, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
               "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(d), "l"(a), "l"(b), "r"(id), "r"(acc)
               : "memory");
}
__device__ __forceinline__ void commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void wait(uint64_t* bar, uint32_t ph) {
  uint32_t done = 0;
  while (!done)
    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                 : "=r"(done) : "r"(smem_u32(bar)), "r"(ph) : "memory");
}

template <int N>
__global__ void __launch_bounds__(128, 1) probe(long long* out, int nm, int reps) {
  extern __shared__ uint8_t raw[];
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint32_t tb;
  for (int i = threadIdx.x; i < (16384 + 32768) / 16; i += blockDim.x)
    reinterpret_cast<uint4*>(base)[i] = make_uint4(0x01020304u, 0x05060708u, 0x01010101u, 0x7f7f7f7fu);
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tb)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (threadIdx.x == 0) {
    const uint32_t sa = smem_u32(base), sb = smem_u32(base + 16384);
    constexpr uint32_t id = idesc_u8s8(128, N);
    for (int r = 0; r < reps; ++r) {
      long long t[40];
      t[0] = clock64();
      for (int k = 0; k < nm; ++k) {
        mma(tb + (k & 1) * 256, desc_sw128(sa + 32 * (k % 3)), desc_sw128(sb + 32 * (k % 3)), id, k > 1);
        t[k + 1] = clock64();
      }
      commit(&bar);
      t[nm + 1] = clock64();
      wait(&bar, r & 1);
      t[nm + 2] = clock64();
      if (blockIdx.x == 0 && r == reps - 1)
        for (int k = 0; k <= nm + 2; ++k) out[k] = t[k] - t[0];
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tb), "r"(512));
}

template <int N>
void run(long long* d, int nm, int ctas) {
  const int smem = 1024 + 16384 + 32768;
  cudaFuncSetAttribute(probe<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  probe<N><<<ctas, 128, smem>>>(d, nm, 8);
  cudaDeviceSynchronize();
  long long h[40];
  cudaMemcpy(h, d, sizeof(long long) * (nm + 3), cudaMemcpyDeviceToHost);
  printf("N=%d nm=%2d ctas=%3d issue stamps:", N, nm, ctas);
  for (int k = 1; k <= nm; ++k) printf(" %lld", h[k]);
  printf(" | commit %lld | done %lld  (%s)\n", h[nm + 1], h[nm + 2], cudaGetErrorString(cudaGetLastError()));
}

int main() {
  long long* d;
  cudaMalloc(&d, 8 * 64);
  for (int ctas : {1, 148}) {
    run<256>(d, 3, ctas);
    run<256>(d, 12, ctas);
    run<128>(d, 12, ctas);
  }
  return 0;
}
