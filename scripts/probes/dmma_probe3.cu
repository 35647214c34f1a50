// Does integer / FP64 ALU work overlap with DMMA on the same SM sub-partition?
// Per DMMA pair: N integer ops (V=0), N DADD (V=1), N FMUL fp32 (V=2).
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void dmma(double2& d, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d.x), "+d"(d.y) : "d"(a), "d"(b));
}
template <int V, int N>
__global__ void __launch_bounds__(256, 2) k(double* out, int iters) {
  double2 acc[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) acc[j] = make_double2(threadIdx.x * 1e-3 + j, 0.5 * j);
  double a0 = 1.0 + threadIdx.x * 1e-12, a1 = 1.0 - threadIdx.x * 1e-12;
  unsigned x[4] = {threadIdx.x, threadIdx.x * 3u, threadIdx.x * 7u, threadIdx.x * 11u};
  double y[4] = {a0, a1, a0 * 2, a1 * 2};
  float z[4] = {1.f, 2.f, 3.f, 4.f};
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int kk = 0; kk < 16; ++kk) {
      dmma(acc[kk & 7], a0, a1);
      dmma(acc[(kk + 4) & 7], a1, a0);
#pragma unroll
      for (int n = 0; n < N; ++n) {
        if (V == 0) asm volatile("lop3.b32 %0, %0, %1, 0x5a, 0x96;" : "+r"(x[n & 3]) : "r"(x[(n + 1) & 3]));
        if (V == 1) asm volatile("add.f64 %0, %0, %1;" : "+d"(y[n & 3]) : "d"(y[(n + 1) & 3]));
        if (V == 2) asm volatile("mul.f32 %0, %0, %1;" : "+f"(z[n & 3]) : "f"(z[(n + 1) & 3]));
      }
    }
  }
  double s = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) s += acc[j].x + acc[j].y;
  s += x[0] + x[1] + x[2] + x[3] + y[0] + y[1] + y[2] + y[3] + z[0] + z[1] + z[2] + z[3];
  if (s == 1.2345) out[threadIdx.x] = s;
}
template <int V, int N>
void run(double* d) {
  const int iters = 1024;
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  k<V, N><<<296, 256>>>(d, iters);
  float best = 1e9;
  for (int r = 0; r < 3; ++r) {
    cudaEventRecord(e0); k<V, N><<<296, 256>>>(d, iters); cudaEventRecord(e1);
    cudaEventSynchronize(e1); float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
  }
  const double flop = 2.0 * 256 * (double)iters * 32 * 296 * 8;
  // cycles per DMMA pair per SMSP: time * clk / (pairs per SMSP)
  const double pairs_per_smsp = (double)iters * 16 * 296 * 8 / (148.0 * 4);
  printf("V%d N=%2d : %6.2f TF/s  %5.1f cycles per DMMA pair+ops per SMSP\n", V, N, flop / best / 1e9,
         best * 1e-3 * 1.965e9 / pairs_per_smsp);
}
int main() {
  double* d; cudaMalloc(&d, 4096 * sizeof(double));
  run<0, 0>(d); run<0, 4>(d); run<0, 8>(d); run<0, 16>(d); run<0, 32>(d);
  run<1, 1>(d); run<1, 2>(d); run<1, 4>(d); run<1, 8>(d);
  run<2, 8>(d); run<2, 16>(d); run<2, 32>(d);
  return 0;
}
