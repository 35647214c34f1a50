// TMEM read-bandwidth probe (tcgen05.ld.32x32b.x32): NW warps per CTA (NW/4
// per lane quarter), each loading 256 columns x 32 lanes x 4 B per
// iteration; reports bytes per SM-cycle.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ void ld32(uint32_t taddr, int32_t (&v)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
        "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
        "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]),
        "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]),
        "=r"(v[30]), "=r"(v[31])
      : "r"(taddr));
}

template <int NW>
__global__ void __launch_bounds__(NW * 32, 1) probe(long long* out, int iters, int* sink) {
  __shared__ uint32_t tb;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     static_cast<uint32_t>(__cvta_generic_to_shared(&tb))), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t base = tb + (static_cast<uint32_t>(32 * (warp & 3)) << 16);
  const int part = warp >> 2, nparts = NW / 4;
  const int cols = 256 / nparts;
  int acc = 0;
  __syncthreads();
  const long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    for (int c = 0; c < cols; c += 32) {
      int32_t v[32];
      ld32(base + part * cols + c, v);
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
      for (int k = 0; k < 32; ++k) acc ^= v[k];
    }
  }
  __syncthreads();
  const long long t1 = clock64();
  if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = t1 - t0;
  if (acc == 0x12345) sink[0] = acc;
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tb), "r"(512));
}

template <int NW>
void run(long long* d, int* s) {
  const int iters = 2000;
  probe<NW><<<148, NW * 32>>>(d, iters, s);
  cudaDeviceSynchronize();
  probe<NW><<<148, NW * 32>>>(d, iters, s);
  long long cyc;
  cudaMemcpy(&cyc, d, 8, cudaMemcpyDeviceToHost);
  const double bytes = double(iters) * 128 * 256 * 4;
  printf("NW=%2d warps: %lld cycles, %.1f B/clk/SM (%s)\n", NW, cyc, bytes / cyc, cudaGetErrorString(cudaGetLastError()));
}

int main() {
  long long* d;
  int* s;
  cudaMalloc(&d, 8);
  cudaMalloc(&s, 4);
  run<4>(d, s);
  run<8>(d, s);
  run<16>(d, s);
  return 0;
}
