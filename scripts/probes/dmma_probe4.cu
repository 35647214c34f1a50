// The k_fused8_sym DMMA dependency structure in isolation: per class, a
// filter (2 m-tiles x 2 n-tiles x 4 k-steps, B from shared memory) whose D
// fragments feed the inverse's A operand (2 x 2 x 4). V=0 as in the kernel;
// V=1 software-pipelined (filter of class c+1 issued before inverse of c);
// V=2 no dependency (inverse A from q instead of y).
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void dmma(double2& d, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
      : "+d"(d.x), "+d"(d.y) : "d"(a), "d"(b));
}
template <int V>
__global__ void __launch_bounds__(256, 2) k(double* out, int iters) {
  __shared__ double2 gs[512], ws[512];
  for (int i = threadIdx.x; i < 512; i += blockDim.x) {
    gs[i] = make_double2(1e-3 * i, 2e-3 * i); ws[i] = make_double2(1e-3 * i, -1e-3 * i);
  }
  __syncthreads();
  const int lane = threadIdx.x & 31;
  double q[2][4][4];
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int c = 0; c < 4; ++c)
#pragma unroll
      for (int s = 0; s < 4; ++s) q[a][c][s] = 1.0 + 1e-6 * (threadIdx.x + a + c + s);
  double sink = 0;
  for (int it = 0; it < iters; ++it) {
    double2 z[2][4][2];
    double2 y[4][2][2];
#pragma unroll
    for (int c = 0; c < 4; ++c) {
#pragma unroll
      for (int mt = 0; mt < 2; ++mt)
#pragma unroll
        for (int nt = 0; nt < 2; ++nt) y[c][mt][nt] = make_double2(0.0, 0.0);
#pragma unroll
      for (int sp = 0; sp < 2; ++sp)
#pragma unroll
        for (int nt = 0; nt < 2; ++nt) {
          const double2 bb = gs[((c * 2 + nt) * 2 + sp) * 32 + lane];
          dmma(y[c][0][nt], q[0][c][2 * sp], bb.x);
          dmma(y[c][1][nt], q[1][c][2 * sp], bb.x);
          dmma(y[c][0][nt], q[0][c][2 * sp + 1], bb.y);
          dmma(y[c][1][nt], q[1][c][2 * sp + 1], bb.y);
        }
#pragma unroll
      for (int mt = 0; mt < 2; ++mt)
#pragma unroll
        for (int nt2 = 0; nt2 < 2; ++nt2) z[mt][c][nt2] = make_double2(0.5, 0.5);
#pragma unroll
      for (int nt = 0; nt < 2; ++nt)
#pragma unroll
        for (int nt2 = 0; nt2 < 2; ++nt2) {
          const double2 bb = ws[((c * 2 + nt2) * 2 + nt) * 32 + lane];
          const double a0x = V == 2 ? q[0][c][nt] : y[c][0][nt].x, a1x = V == 2 ? q[1][c][nt] : y[c][1][nt].x;
          const double a0y = V == 2 ? q[0][c][nt + 2] : y[c][0][nt].y, a1y = V == 2 ? q[1][c][nt + 2] : y[c][1][nt].y;
          dmma(z[0][c][nt2], a0x, bb.x);
          dmma(z[1][c][nt2], a1x, bb.x);
          dmma(z[0][c][nt2], a0y, bb.y);
          dmma(z[1][c][nt2], a1y, bb.y);
        }
    }
#pragma unroll
    for (int mt = 0; mt < 2; ++mt)
#pragma unroll
      for (int c = 0; c < 4; ++c) sink += z[mt][c][0].x + z[mt][c][0].y + z[mt][c][1].x + z[mt][c][1].y;
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
      for (int c = 0; c < 4; ++c)
#pragma unroll
        for (int s = 0; s < 4; ++s) q[a][c][s] += sink * 1e-30;
  }
  if (sink == 1.2345) out[threadIdx.x] = sink;
}
template <int V>
void run(double* d) {
  const int iters = 256;
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  k<V><<<296, 256>>>(d, iters);
  float best = 1e9;
  for (int r = 0; r < 3; ++r) {
    cudaEventRecord(e0); k<V><<<296, 256>>>(d, iters); cudaEventRecord(e1);
    cudaEventSynchronize(e1); float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
  }
  const double flop = 2.0 * 256 * (double)iters * 128 * 296 * 8;
  printf("V%d : %6.2f TF/s\n", V, flop / best / 1e9);
}
int main() {
  double* d; cudaMalloc(&d, 4096 * sizeof(double));
  run<0>(d); run<2>(d);
  return 0;
}
