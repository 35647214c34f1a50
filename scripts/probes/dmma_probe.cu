// DMMA.8x8x4 throughput vs warps per SM and independent accumulator chains per warp.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void dmma(double2& d, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d.x), "+d"(d.y) : "d"(a), "d"(b));
}
template <int CH>
__global__ void k(double* out, int iters) {
  double2 acc[CH];
#pragma unroll
  for (int j = 0; j < CH; ++j) acc[j] = make_double2(threadIdx.x * 1e-3 + j, 0.5 * j);
  const double a = 1.0 + threadIdx.x * 1e-12, b = 1.0 - threadIdx.x * 1e-12;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < CH; ++j) dmma(acc[j], a, b);
  }
  double s = 0;
#pragma unroll
  for (int j = 0; j < CH; ++j) s += acc[j].x + acc[j].y;
  if (s == 1.2345) out[threadIdx.x] = s;
}
template <int CH>
void run(int wpsm, double* d) {
  const int threads = 128, blocks = 148 * wpsm / 4;
  const int iters = 16384 / CH;
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  k<CH><<<blocks, threads>>>(d, iters);
  float best = 1e9;
  for (int r = 0; r < 3; ++r) {
    cudaEventRecord(e0); k<CH><<<blocks, threads>>>(d, iters); cudaEventRecord(e1);
    cudaEventSynchronize(e1); float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
  }
  const double flop = 2.0 * 256 * (double)iters * CH * blocks * (threads / 32);
  printf("warps/SM %2d chains %2d : %6.2f TF/s\n", wpsm, CH, flop / best / 1e9);
}
int main() {
  double* d; cudaMalloc(&d, 4096 * sizeof(double));
  for (int w : {4, 8, 12, 16, 32}) { run<1>(w, d); run<2>(w, d); run<4>(w, d); run<8>(w, d); run<16>(w, d); }
  return 0;
}
