// Store-path probe for k_fused8_q's epilogue pattern: persistent CTAs (one per SM), W warps,
// each warp writes "tiles" of 8 rows x (32 lanes x BYTES) at the frame pitch, optionally
// after loading the same bytes (copy). Prints achieved GB/s per variant.
// build: nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o stg_probe stg_probe.cu
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
template <int BYTES, bool COPY, int MODE>
__global__ void __launch_bounds__(1024, 1) k_store(const uint8_t* __restrict__ in, uint8_t* __restrict__ out, int w, int h,
                                                  int nframes, size_t pitch, size_t fstride) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  const int seg = 32 * BYTES;                 // bytes per warp row
  const int segs_per_row = w / seg;           // w multiple of seg assumed
  const long long strips = (long long)(h / 8) * nframes;
  const long long units = strips * segs_per_row;
  for (long long u = (long long)blockIdx.x * nw + warp; u < units; u += (long long)gridDim.x * nw) {
    const long long strip = u / segs_per_row;
    const int sx = (int)(u - strip * segs_per_row);
    const long long f = strip / (h / 8);
    const int by = (int)(strip - f * (h / 8));
    const size_t off = f * fstride + (size_t)by * 8 * pitch + (size_t)sx * seg + lane * BYTES;
    if (BYTES == 8) {
      uint2 v[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) v[k] = COPY ? __ldg((const uint2*)(in + off + k * pitch)) : make_uint2(u, k);
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        if (MODE == 1) __stcs((uint2*)(out + off + k * pitch), v[k]);
        else if (MODE == 2) __stwt((uint2*)(out + off + k * pitch), v[k]);
        else *(uint2*)(out + off + k * pitch) = v[k];
      }
    } else {
      uint4 v[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) v[k] = COPY ? __ldg((const uint4*)(in + off + k * pitch)) : make_uint4(u, k, 0, 0);
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        if (MODE == 1) __stcs((uint4*)(out + off + k * pitch), v[k]);
        else if (MODE == 2) __stwt((uint4*)(out + off + k * pitch), v[k]);
        else *(uint4*)(out + off + k * pitch) = v[k];
      }
    }
  }
}
template <int BYTES, bool COPY, int MODE>
void run(const char* name, int warps, const uint8_t* in, uint8_t* out) {
  const int w = 3840, h = 2160, nf = 64;
  const size_t pitch = w, fs = (size_t)w * h;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float best = 1e9f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(a);
    k_store<BYTES, COPY, MODE><<<148, warps * 32>>>(in, out, w, h, nf, pitch, fs);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    if (r) best = ms < best ? ms : best;
  }
  const double bytes = (double)w * h * nf * (COPY ? 2 : 1);
  printf("%-28s warps %2d: %7.1f us  %6.0f GB/s (%s)\n", name, warps, best * 1e3, bytes / best / 1e6,
         COPY ? "read+write" : "write only");
}
int main() {
  uint8_t *in, *out;
  const size_t n = (size_t)3840 * 2160 * 64;
  cudaMalloc(&in, n);
  cudaMalloc(&out, n);
  cudaMemset(in, 1, n);
  cudaMemset(out, 2, n);
  for (int warps : {4, 8, 16, 32}) {
    run<8, false, 0>("STG.64 write", warps, in, out);
    run<16, false, 0>("STG.128 write", warps, in, out);
    run<8, false, 1>("STG.64.cs write", warps, in, out);
    run<8, true, 0>("LDG.64+STG.64 copy", warps, in, out);
    run<16, true, 0>("LDG.128+STG.128 copy", warps, in, out);
  }
  printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
