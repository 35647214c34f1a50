// How long does __nanosleep(t) sleep on this part (clock64 cycles), alone and
// with other warps of the CTA hammering an mbarrier?
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(long long* out, int busy) {
  __shared__ uint64_t bar;
  __shared__ volatile int stop;
  if (threadIdx.x == 0) {
    stop = 0;
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1000000;" ::"r"(static_cast<uint32_t>(__cvta_generic_to_shared(&bar))));
  }
  __syncthreads();
  const int warp = threadIdx.x >> 5;
  if (warp == 0) {
    const unsigned ts[6] = {100, 1000, 2000, 10000, 100000, 1000000};
    for (int i = 0; i < 6; ++i) {
      long long acc = 0;
      for (int r = 0; r < 8; ++r) {
        const long long t0 = clock64();
        __nanosleep(ts[i]);
        acc += clock64() - t0;
      }
      if (threadIdx.x == 0) out[i] = acc / 8;
    }
    if (threadIdx.x == 0) stop = 1;
  } else if (busy) {
    while (!stop)
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(static_cast<uint32_t>(__cvta_generic_to_shared(&bar))) : "memory");
  }
}
int main() {
  long long* d;
  cudaMalloc(&d, 64);
  for (int busy = 0; busy < 2; ++busy) {
    k<<<1, 128>>>(d, busy);
    cudaDeviceSynchronize();
    long long h[6];
    cudaMemcpy(h, d, 48, cudaMemcpyDeviceToHost);
    printf("busy=%d: nanosleep 100/1e3/2e3/1e4/1e5/1e6 ns -> %lld %lld %lld %lld %lld %lld cycles\n", busy, h[0], h[1], h[2],
           h[3], h[4], h[5]);
  }
  return 0;
}
