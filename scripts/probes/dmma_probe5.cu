// The k_fused8_sym DMMA structure in isolation (per "strip": 4 classes x
// [filter: 2 m-tiles x 2 n-tiles accumulators, 4-deep chains, B from shared
// memory] -> [inverse on the filter results, same shape]), iterations
// independent (A operands derived from the loop counter on the integer pipe).
// V0: class by class (as in the kernel); V1: all four filters, then all four
// inverses (more independent accumulators between dependent phases).
#include <cstdio>
#include <cuda_runtime.h>
#include <cstdint>
__device__ __forceinline__ void dmma(double2& d, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
      : "+d"(d.x), "+d"(d.y) : "d"(a), "d"(b));
}
__device__ __forceinline__ double i32_to_f64(int v) {
  const uint32_t m = static_cast<uint32_t>(v < 0 ? -v : v);
  const int e = 31 - __clz(m);
  const uint32_t hi = ((static_cast<uint32_t>(1022 + e) << 20) + (m << (20 - e))) |
                      (static_cast<uint32_t>(v) & 0x80000000u);
  return m ? __hiloint2double(static_cast<int>(hi), 0) : 0.0;
}
__device__ __forceinline__ uint32_t floor_to_u8(double t) {
  int i;
  asm("cvt.rmi.s32.f64 %0, %1;" : "=r"(i) : "d"(t));
  return static_cast<uint32_t>(min(max(i, 0), 255));
}
template <int V, int MINB>
__global__ void __launch_bounds__(256, MINB) k(double* out, int iters, const uint4* gin, uint4* gout) {
  __shared__ double2 gs[512], ws[512];
  __shared__ __align__(16) uint8_t pixs[8][8 * 192];
  for (int i = threadIdx.x; i < 512; i += blockDim.x) {
    gs[i] = make_double2(1e-3 * i, 2e-3 * i); ws[i] = make_double2(1e-3 * i, -1e-3 * i);
  }
  __syncthreads();
  const int lane = threadIdx.x & 31;
  double2 total = make_double2(0.0, 0.0);
  for (int it = 0; it < iters; ++it) {
    double q[2][4][4];
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
      for (int c = 0; c < 4; ++c)
#pragma unroll
        for (int s = 0; s < 4; ++s)
          q[a][c][s] = __longlong_as_double(0x3ff0000000000000LL + (((long long)(it * 16 + a * 8 + c * 4 + s + lane)) << 20));
    double2 z[2][4][2];
    uint4 pf0 = make_uint4(0, 0, 0, 0), pf1 = pf0;
    const int warp = threadIdx.x >> 5, r0 = lane >> 3, c16 = (lane & 7) * 16;
    uint8_t* pix = pixs[warp];
    if (V >= 3) {
      const size_t strip = (size_t)(blockIdx.x * 8 + warp) * 4096 + it;
      pf0 = gin[(strip * 64 + lane) & ((1u << 24) - 1)];
      pf1 = gin[(strip * 64 + 32 + lane) & ((1u << 24) - 1)];
      *reinterpret_cast<uint4*>(pix + r0 * 192 + c16) = pf0;
      *reinterpret_cast<uint4*>(pix + (r0 + 4) * 192 + c16) = pf1;
      __syncwarp();
      if (V == 4) {
        const int g = lane >> 2, t = lane & 3;
#pragma unroll
        for (int mt = 0; mt < 2; ++mt) {
          const uint8_t* pb = pix + 8 * (8 * mt + g);
#pragma unroll
          for (int sq = 0; sq < 4; ++sq) {
            const uint2 top = *reinterpret_cast<const uint2*>(pb + sq * 192);
            const uint2 bot = *reinterpret_cast<const uint2*>(pb + (7 - sq) * 192);
            const int p00 = (top.x >> (8 * t)) & 0xff, p01 = (top.y >> (24 - 8 * t)) & 0xff;
            const int p10 = (bot.x >> (8 * t)) & 0xff, p11 = (bot.y >> (24 - 8 * t)) & 0xff;
            const int rs0 = p00 + p10, ra0 = p00 - p10, rs1 = p01 + p11, ra1 = p01 - p11;
            q[mt][0][sq] = i32_to_f64(rs0 + rs1);
            q[mt][1][sq] = i32_to_f64(rs0 - rs1);
            q[mt][2][sq] = i32_to_f64(ra0 + ra1);
            q[mt][3][sq] = i32_to_f64(ra0 - ra1);
          }
        }
      }
    }
    if (V != 1) {
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        double2 y[2][2];
#pragma unroll
        for (int mt = 0; mt < 2; ++mt)
#pragma unroll
          for (int nt = 0; nt < 2; ++nt) y[mt][nt] = make_double2(0.0, 0.0);
#pragma unroll
        for (int sp = 0; sp < 2; ++sp)
#pragma unroll
          for (int nt = 0; nt < 2; ++nt) {
            const double2 bb = gs[((c * 2 + nt) * 2 + sp) * 32 + lane];
            dmma(y[0][nt], q[0][c][2 * sp], bb.x); dmma(y[1][nt], q[1][c][2 * sp], bb.x);
            dmma(y[0][nt], q[0][c][2 * sp + 1], bb.y); dmma(y[1][nt], q[1][c][2 * sp + 1], bb.y);
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
            dmma(z[0][c][nt2], y[0][nt].x, bb.x); dmma(z[1][c][nt2], y[1][nt].x, bb.x);
            dmma(z[0][c][nt2], y[0][nt].y, bb.y); dmma(z[1][c][nt2], y[1][nt].y, bb.y);
          }
      }
    } else {
      double2 y[4][2][2];
#pragma unroll
      for (int c = 0; c < 4; ++c)
#pragma unroll
        for (int mt = 0; mt < 2; ++mt)
#pragma unroll
          for (int nt = 0; nt < 2; ++nt) y[c][mt][nt] = make_double2(0.0, 0.0);
#pragma unroll
      for (int sp = 0; sp < 2; ++sp)
#pragma unroll
        for (int c = 0; c < 4; ++c)
#pragma unroll
          for (int nt = 0; nt < 2; ++nt) {
            const double2 bb = gs[((c * 2 + nt) * 2 + sp) * 32 + lane];
            dmma(y[c][0][nt], q[0][c][2 * sp], bb.x); dmma(y[c][1][nt], q[1][c][2 * sp], bb.x);
            dmma(y[c][0][nt], q[0][c][2 * sp + 1], bb.y); dmma(y[c][1][nt], q[1][c][2 * sp + 1], bb.y);
          }
#pragma unroll
      for (int c = 0; c < 4; ++c)
#pragma unroll
        for (int mt = 0; mt < 2; ++mt)
#pragma unroll
          for (int nt2 = 0; nt2 < 2; ++nt2) z[mt][c][nt2] = make_double2(0.5, 0.5);
#pragma unroll
      for (int nt = 0; nt < 2; ++nt)
#pragma unroll
        for (int c = 0; c < 4; ++c)
#pragma unroll
          for (int nt2 = 0; nt2 < 2; ++nt2) {
            const double2 bb = ws[((c * 2 + nt2) * 2 + nt) * 32 + lane];
            dmma(z[0][c][nt2], y[c][0][nt].x, bb.x); dmma(z[1][c][nt2], y[c][1][nt].x, bb.x);
            dmma(z[0][c][nt2], y[c][0][nt].y, bb.y); dmma(z[1][c][nt2], y[c][1][nt].y, bb.y);
          }
    }
    if (V >= 2) {
      const int g = lane >> 2, t = lane & 3;
#pragma unroll
      for (int mt = 0; mt < 2; ++mt) {
        uint8_t* pb = pix + 8 * (8 * mt + g);
#pragma unroll
        for (int nt2 = 0; nt2 < 2; ++nt2) {
          const int i = 2 * nt2 + (t >> 1), j = 2 * (t & 1);
          uint32_t o_ij[2], o_rj[2], o_ir[2], o_rr[2];
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const double zee = e ? z[mt][0][nt2].y : z[mt][0][nt2].x, zeo = e ? z[mt][1][nt2].y : z[mt][1][nt2].x;
            const double zoe = e ? z[mt][2][nt2].y : z[mt][2][nt2].x, zoo = e ? z[mt][3][nt2].y : z[mt][3][nt2].x;
            const double a = zee + zeo, bq = zee - zeo, cq = zoe + zoo, d = zoe - zoo;
            o_ij[e] = floor_to_u8(a + cq); o_rj[e] = floor_to_u8(a - cq);
            o_ir[e] = floor_to_u8(bq + d); o_rr[e] = floor_to_u8(bq - d);
          }
          *reinterpret_cast<uint16_t*>(pb + i * 192 + j) = static_cast<uint16_t>(o_ij[0] | (o_ij[1] << 8));
          *reinterpret_cast<uint16_t*>(pb + (7 - i) * 192 + j) = static_cast<uint16_t>(o_rj[0] | (o_rj[1] << 8));
          *reinterpret_cast<uint16_t*>(pb + i * 192 + 6 - j) = static_cast<uint16_t>(o_ir[1] | (o_ir[0] << 8));
          *reinterpret_cast<uint16_t*>(pb + (7 - i) * 192 + 6 - j) = static_cast<uint16_t>(o_rr[1] | (o_rr[0] << 8));
        }
      }
      __syncwarp();
      if (V >= 3) {
        const size_t strip = (size_t)(blockIdx.x * 8 + warp) * 4096 + it;
        gout[(strip * 64 + lane) & ((1u << 24) - 1)] = *reinterpret_cast<const uint4*>(pix + r0 * 192 + c16);
        gout[(strip * 64 + 32 + lane) & ((1u << 24) - 1)] = *reinterpret_cast<const uint4*>(pix + (r0 + 4) * 192 + c16);
        __syncwarp();
      }
      continue;
    }
    // consume every result without a cross-iteration FP64 dependency chain
#pragma unroll
    for (int mt = 0; mt < 2; ++mt)
#pragma unroll
      for (int c = 0; c < 4; ++c)
#pragma unroll
        for (int nt2 = 0; nt2 < 2; ++nt2) {
          const long long bx = __double_as_longlong(z[mt][c][nt2].x) ^ __double_as_longlong(z[mt][c][nt2].y);
          total.x = __longlong_as_double(__double_as_longlong(total.x) ^ bx);
        }
  }
  if (total.x == 1.2345) out[threadIdx.x] = total.x;
}
template <int V, int MINB>
void run(double* d) {
  const int iters = 256;
  const int blocks = 148 * MINB;
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  static uint4 *gi = nullptr, *go = nullptr;
  if (!gi) { cudaMalloc(&gi, 16u << 24); cudaMalloc(&go, 16u << 24); cudaMemset(gi, 7, 16u << 24); }
  k<V, MINB><<<blocks, 256>>>(d, iters, gi, go);
  float best = 1e9;
  for (int r = 0; r < 3; ++r) {
    cudaEventRecord(e0); k<V, MINB><<<blocks, 256>>>(d, iters, gi, go); cudaEventRecord(e1);
    cudaEventSynchronize(e1); float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
  }
  const double flop = 2.0 * 256 * (double)iters * 128 * blocks * 8;
  printf("V%d minB%d : %6.2f TF/s\n", V, MINB, flop / best / 1e9);
}
int main() {
  double* d; cudaMalloc(&d, 4096 * sizeof(double));
  run<0, 2>(d); run<3, 2>(d); run<4, 2>(d);
  return 0;
}
