// Fused image kernels (filter_image, image.hpp:210-225, with
// filter_block's chain, filter.hpp:71-73): u8 pixels -> filtered DCT
// coefficients -> inverse DCT -> round/clamp -> u8 in one HBM pass —
// k_fused8 / k_fused8_sym (n = 8) and k_fused16 / k_fused16_sym (n = 16) —
// their launchers and the image-path dispatch (filter_image_device).
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <string>

#include "device.cuh"
#include "fastdiv.cuh"
#include "internal.h"

using dctf::misaligned16;
using dctf::set_error;
using dctf::sm_count;

namespace {

// ---------------------------------------------------------------------------
// k_fused8: u8 -> G p -> C^t Y C -> round/clamp -> u8, n = 8, where
// G = H (C (x) C) is the DCT-domain operator with the forward DCT composed in
// on the host (compose_forward, long-double accumulation), so Y = G vec(P) are
// the filtered DCT coefficients of filter_block (filter.hpp:71-73) and the
// FP64 pipe does 2N^4 + 4N^3 flop per block instead of 2N^4 + 8N^3.
//
// Work unit ("strip"): 16 horizontally adjacent blocks = 8 pixel rows x 128
// bytes, owned by one warp. Pixels arrive through 16-byte streaming loads
// issued one strip ahead (prefetch into registers), are staged in a padded
// per-warp buffer (row stride 144 B), and every stage is a DMMA chain whose
// fragment layouts line up so no shuffles are needed:
//   pixels -> FP64 staging: lane (g,t) writes pixels (2t,g), (2t+1,g) of each
//     block (the slots the forward DCT's X[2t][g], X[2t+1][g] would take).
//   filter          Y^T = P^T G^T : blocks on M (2 m-tiles), G^T from shared
//     memory (layout_hfused8 of G), P via the per-warp staging buffer.
//   inverse pass 1  Z = C^t Y     : A = C[2t+s][g], B = Y via staging
//   inverse pass 2  O = Z C + 0.5 : A = pass-1 accumulators, B = C[2t+s][g]
//     -> lane (g,t) holds O[g][2t], O[g][2t+1]: two adjacent output pixels,
//     already offset by 0.5 so quantisation is one floor conversion.
// The inverse works on 4 blocks at a time so 4 independent DMMA chains
// interleave. Staging layout: block b owns 512 B = 4 rows x 8 chunks of 16 B;
// logical (row r, chunk c) is stored at chunk c ^ 2r ^ f(b), f(b) = (b&7) ^
// ((b&1)<<2). Every 16-byte access pattern below then hits 8 distinct chunks
// in each quarter-warp phase (lanes g in {2p, 2p+1}, t in 0..3): no bank
// conflicts. Ragged strips (image edge, block-grid tail) take a clamped
// per-byte path with the same compute.
namespace f8 {
constexpr int WARPS = 8;
constexpr int SB = 16;
constexpr int PS = 144;
constexpr int XY_BYTES = SB * 512;
constexpr int PIX_BYTES = 8 * PS;
constexpr int WARP_BYTES = XY_BYTES + PIX_BYTES;
constexpr int SMEM = 32768 + WARPS * WARP_BYTES;
__device__ __forceinline__ int fsw(int b) { return (b & 7) ^ ((b & 1) << 2); }
}  // namespace f8

template <bool COEF>
__global__ void __launch_bounds__(f8::WARPS * 32, 2)
    k_fused8(const uint8_t* __restrict__ in, uint8_t* __restrict__ out, int w, int h, size_t pitch,
             long long frame_stride, int nframes, int bw, int bh, int nsx,
             const double* __restrict__ hf, const double* __restrict__ cb,
             double* __restrict__ coef_out) {
  using namespace f8;
  extern __shared__ __align__(16) uint8_t smem[];
  const double2* hs = reinterpret_cast<const double2*>(smem);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  uint8_t* xy = smem + 32768 + warp * WARP_BYTES;
  uint8_t* pix = xy + XY_BYTES;
  const double ai0 = cb[(2 * t) * 8 + g], ai1 = cb[(2 * t + 1) * 8 + g];
  const int fg = fsw(g);

  const long long spf = static_cast<long long>(bh) * nsx;
  const long long nstrips = spf * nframes;
  const int nwarps = blockDim.x >> 5;  // < WARPS for small images (launcher)
  const long long total = static_cast<long long>(gridDim.x) * nwarps;
  const bool aligned = ((pitch & 15) == 0) && ((reinterpret_cast<uintptr_t>(in) & 15) == 0) &&
                       ((reinterpret_cast<uintptr_t>(out) & 15) == 0) && ((frame_stride & 15) == 0);
  const int r0 = lane >> 3, c16 = (lane & 7) * 16;

  uint4 pf0 = make_uint4(0, 0, 0, 0), pf1 = pf0;
  long long s = static_cast<long long>(blockIdx.x) * nwarps + warp;
  const dctf::FastDiv fd_spf = dctf::make_fastdiv(static_cast<uint32_t>(spf)),
                      fd_nsx = dctf::make_fastdiv(static_cast<uint32_t>(nsx));
  auto strip_at = [&](long long si, int& f, int& by, int& bx0) {  // si < 2^31 (launcher)
    const uint32_t u = static_cast<uint32_t>(si);
    f = static_cast<int>(dctf::fdiv(fd_spf, u));
    const uint32_t rem = u - static_cast<uint32_t>(f) * static_cast<uint32_t>(spf);
    by = static_cast<int>(dctf::fdiv(fd_nsx, rem));
    bx0 = static_cast<int>(rem - static_cast<uint32_t>(by) * static_cast<uint32_t>(nsx)) * SB;
  };
  auto is_fast = [&](int by, int bx0) { return aligned && by * 8 + 8 <= h && bx0 * 8 + 128 <= w; };
  auto prefetch = [&](long long si) {
    int f, by, bx0;
    strip_at(si, f, by, bx0);
    if (is_fast(by, bx0)) {
      const uint8_t* p = in + f * frame_stride + static_cast<size_t>(by * 8) * pitch + bx0 * 8 + c16;
      pf0 = ldg_stream(p + r0 * pitch);
      pf1 = ldg_stream(p + (r0 + 4) * pitch);
    }
  };
  pdl_trigger();
  cta_copy_async(smem, hf, 32768);  // plan-owned operator: staged before the dependency wait
  pdl_wait();
  if (s < nstrips) prefetch(s);  // first strip's pixels in flight during the operator copy
  cp_async_wait_all();
  __syncthreads();

  for (; s < nstrips; s += total) {
    int f, by, bx0;
    strip_at(s, f, by, bx0);
    const bool fast = is_fast(by, bx0);
    if (fast) {
      *reinterpret_cast<uint4*>(pix + r0 * PS + c16) = pf0;
      *reinterpret_cast<uint4*>(pix + (r0 + 4) * PS + c16) = pf1;
    } else {
      const uint8_t* ib = in + f * frame_stride;
      for (int e = lane; e < 8 * 128; e += 32) {
        const int r = e >> 7, c = e & 127;
        const int y = min(by * 8 + r, h - 1), x = min(bx0 * 8 + c, w - 1);
        pix[r * PS + c] = ib[static_cast<size_t>(y) * pitch + x];
      }
    }
    __syncwarp();
    if (s + total < nstrips) prefetch(s + total);

    // The forward DCT is folded into the operator (G = H (C (x) C), see
    // compose_forward): stage each block's pixels as FP64 in X's layout, lane
    // (g, t) writing pixels (2t, g) and (2t+1, g) where X[2t][g], X[2t+1][g]
    // would go.
#pragma unroll
    for (int b = 0; b < SB; ++b) {
      const uint32_t q0 = pix[(2 * t) * PS + 8 * b + g];
      const uint32_t q1 = pix[(2 * t + 1) * PS + 8 * b + g];
      *reinterpret_cast<double2*>(xy + b * 512 + t * 128 + ((g ^ (2 * t) ^ fsw(b)) << 4)) =
          make_double2(__uint2double_rn(q0), __uint2double_rn(q1));
    }
    __syncwarp();

    // DCT-domain filter: 16 blocks x 64 outputs, K = 64
    double2 acc[2][8];
#pragma unroll
    for (int m = 0; m < 2; ++m)
#pragma unroll
      for (int j = 0; j < 8; ++j) acc[m][j] = make_double2(0.0, 0.0);
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int sw = (q ^ (2 * t) ^ fg) << 4;
      const double2 a0 = *reinterpret_cast<const double2*>(xy + g * 512 + t * 128 + sw);
      const double2 a1 = *reinterpret_cast<const double2*>(xy + (8 + g) * 512 + t * 128 + sw);
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const double2 b = hs[(j * 8 + q) * 32 + lane];
        dmma(acc[0][j], a0.x, b.x);
        dmma(acc[1][j], a1.x, b.x);
        dmma(acc[0][j], a0.y, b.y);
        dmma(acc[1][j], a1.y, b.y);
      }
    }
    __syncwarp();
#pragma unroll
    for (int m = 0; m < 2; ++m)
#pragma unroll
      for (int j = 0; j < 8; ++j)
        *reinterpret_cast<double2*>(xy + (8 * m + g) * 512 + (j >> 1) * 128 +
                                    (((4 * (j & 1) + t) ^ (2 * (j >> 1)) ^ fg) << 4)) = acc[m][j];
    if (COEF) {
#pragma unroll
      for (int m = 0; m < 2; ++m) {
        const int bx = bx0 + 8 * m + g;
        if (bx < bw) {
          double* dst = coef_out + ((static_cast<long long>(f) * bh + by) * bw + bx) * 64;
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const int u = 2 * (j >> 1), v = 4 * (j & 1) + t;
            dst[u * 8 + v] = acc[m][j].x;
            dst[(u + 1) * 8 + v] = acc[m][j].y;
          }
        }
      }
    }
    __syncwarp();

    // inverse DCT + quantize, 16 blocks, 4 interleaved chains
#pragma unroll
    for (int b0 = 0; b0 < SB; b0 += 4) {
      double2 yv[4], z[4], o[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int b = b0 + i;
        yv[i] = *reinterpret_cast<const double2*>(xy + b * 512 + t * 128 + ((g ^ (2 * t) ^ fsw(b)) << 4));
      }
#pragma unroll
      for (int i = 0; i < 4; ++i) { z[i] = make_double2(0.0, 0.0); dmma(z[i], ai0, yv[i].x); }
#pragma unroll
      for (int i = 0; i < 4; ++i) dmma(z[i], ai1, yv[i].y);
#pragma unroll
      for (int i = 0; i < 4; ++i) { o[i] = make_double2(0.5, 0.5); dmma(o[i], z[i].x, ai0); }
#pragma unroll
      for (int i = 0; i < 4; ++i) dmma(o[i], z[i].y, ai1);
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const uint32_t q = floor_to_u8(o[i].x) | (floor_to_u8(o[i].y) << 8);
        *reinterpret_cast<uint16_t*>(pix + g * PS + 8 * (b0 + i) + 2 * t) = static_cast<uint16_t>(q);
      }
    }
    __syncwarp();

    uint8_t* ob = out + f * frame_stride;
    if (fast) {
      uint8_t* p = ob + static_cast<size_t>(by * 8) * pitch + bx0 * 8 + c16;
      stg_stream(p + r0 * pitch, *reinterpret_cast<const uint4*>(pix + r0 * PS + c16));
      stg_stream(p + (r0 + 4) * pitch, *reinterpret_cast<const uint4*>(pix + (r0 + 4) * PS + c16));
    } else {
      for (int e = lane; e < 8 * 128; e += 32) {
        const int r = e >> 7, c = e & 127;
        const int y = by * 8 + r, x = bx0 * 8 + c;
        if (y < h && x < w) ob[static_cast<size_t>(y) * pitch + x] = pix[r * PS + c];
      }
    }
    __syncwarp();
  }
}

// ---------------------------------------------------------------------------
// k_fused8_sym: k_fused8 for operators that are block-diagonal in the four
// (u mod 2, v mod 2) parity classes (masks symmetric in both axes; see
// layout_sym8 in plan.cc). Since C[u][7-i] = (-1)^u C[u][i], a block's pixels
// enter the DCT only through the quad butterflies
//   q_c(i,j) = p(i,j) +/- p(7-i,j) +/- p(i,7-j) +/- p(7-i,7-j),  i, j < 4,
// exact integers formed on the integer ALUs; per class c the filtered
// coefficients are Y_c = G_c q_c (16 x 16, G_c = H_c (C_c (x) C_c)) and the
// inverse is Z_c = W_c Y_c (16 x 16); output pixels are +/- sums of the Z_c
// (8 DADD per quad), +0.5 folded into Z_ee's accumulator, floor -> u8.
// DMMA per block: 8 (vs 20 dense) — 1,024 + 1,024 FMA.
// Work unit as in k_fused8: a warp owns a 16-block strip (two m-tiles of 8
// blocks on the DMMA M axis, processed together so each operator fragment
// from shared memory feeds 4 DMMAs); lane (g, t) owns blocks g and 8 + g,
// k-step s <-> quad position (s, t) in the filter, and Y chains straight into
// the inverse's A operand (k-step (nt, e) <-> output o = 8nt + 2t + e).
namespace f8s {
#ifndef F8S_MINB
#define F8S_MINB 2
#endif
constexpr int WARPS = 8;
constexpr int SB = 16;
constexpr int PS = 192;  // adjacent rows 16 banks apart: conflict-free u16 output stores
constexpr int PIX_BYTES = 8 * PS;
constexpr int SMEM = 16384 + WARPS * 2 * PIX_BYTES;  // double-buffered strip tiles
}  // namespace f8s

template <bool COEF, bool ASYNC>
__global__ void __launch_bounds__(f8s::WARPS * 32, F8S_MINB)
    k_fused8_sym(const uint8_t* __restrict__ in, uint8_t* __restrict__ out, int w, int h, size_t pitch,
                 long long frame_stride, int nframes, int bw, int bh, int nsx,
                 const double* __restrict__ hsym, double* __restrict__ coef_out) {
  using namespace f8s;
  extern __shared__ __align__(16) uint8_t smem[];
  const double2* gs = reinterpret_cast<const double2*>(smem);          // [c][nt][sp][lane]
  const double2* ws = reinterpret_cast<const double2*>(smem + 8192);   // [c][nt2][nt][lane]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  uint8_t* pix = smem + 16384 + warp * 2 * PIX_BYTES;   // strip being filtered
  uint8_t* pixn = pix + PIX_BYTES;                        // next strip (cp.async in flight)

  // strip counts < 2^31 (launcher): 32-bit strip arithmetic
  const int spf = bh * nsx;
  const int nstrips = spf * nframes;
  const int nwarps = blockDim.x >> 5;  // < WARPS for small images (launcher)
  const int total = static_cast<int>(gridDim.x) * nwarps;
  const bool aligned = ((pitch & 15) == 0) && ((reinterpret_cast<uintptr_t>(in) & 15) == 0) &&
                       ((reinterpret_cast<uintptr_t>(out) & 15) == 0) && ((frame_stride & 15) == 0);
  const int r0 = lane >> 3, c16 = (lane & 7) * 16;
  const uint32_t selL = 0x4440u + t, selR = 0x4440u + (3 - t);  // __byte_perm selectors

  int s = static_cast<int>(blockIdx.x) * nwarps + warp;
  const dctf::FastDiv fd_spf = dctf::make_fastdiv(static_cast<uint32_t>(spf)),
                      fd_nsx = dctf::make_fastdiv(static_cast<uint32_t>(nsx));
  auto strip_at = [&](int si, int& f, int& by, int& bx0) {
    const uint32_t u = static_cast<uint32_t>(si);
    f = static_cast<int>(dctf::fdiv(fd_spf, u));
    const uint32_t rem = u - static_cast<uint32_t>(f) * static_cast<uint32_t>(spf);
    by = static_cast<int>(dctf::fdiv(fd_nsx, rem));
    bx0 = static_cast<int>(rem - static_cast<uint32_t>(by) * static_cast<uint32_t>(nsx)) * SB;
  };
  auto is_fast = [&](int by, int bx0) { return aligned && by * 8 + 8 <= h && bx0 * 8 + 128 <= w; };
  // strip si's pixels -> buf: asynchronously (cp.async, no registers held;
  // device-resident images) or into registers staged at the top of the next
  // iteration (ld.global.cs; host-mapped zero-copy input, where it reads PCIe
  // faster). Returns false when the strip needs the clamped path instead.
  uint4 pf0 = make_uint4(0, 0, 0, 0), pf1 = pf0;
  auto fetch = [&](int si, uint8_t* buf) {
    int f, by, bx0;
    strip_at(si, f, by, bx0);
    const bool ok = is_fast(by, bx0);
    if (ok) {
      const uint8_t* p = in + f * frame_stride + static_cast<size_t>(by * 8) * pitch + bx0 * 8 + c16;
      if constexpr (ASYNC) {
        cp_async16(buf + r0 * PS + c16, p + r0 * pitch);
        cp_async16(buf + (r0 + 4) * PS + c16, p + (r0 + 4) * pitch);
      } else {
        pf0 = ldg_stream(p + r0 * pitch);
        pf1 = ldg_stream(p + (r0 + 4) * pitch);
      }
    }
    if constexpr (ASYNC) cp_async_commit();
    return ok;
  };
  pdl_trigger();                       // the next grid may take SMs as ours retire
  cta_copy_async(smem, hsym, 16384);   // plan-owned: staged before the dependency wait
  pdl_wait();                          // caller buffers: after the preceding grid
  bool fast = s < nstrips ? fetch(s, pix) : false;  // first strip in flight during the operator copy
  cp_async_wait_all();
  __syncthreads();

  for (; s < nstrips; s += total) {
    int f, by, bx0;
    strip_at(s, f, by, bx0);
    if constexpr (ASYNC) {
      cp_async_wait_all();
    } else if (fast) {
      *reinterpret_cast<uint4*>(pix + r0 * PS + c16) = pf0;
      *reinterpret_cast<uint4*>(pix + (r0 + 4) * PS + c16) = pf1;
    }
    if (!fast) {
      const uint8_t* ib = in + f * frame_stride;
      for (int e = lane; e < 8 * 128; e += 32) {
        const int r = e >> 7, c = e & 127;
        const int y = min(by * 8 + r, h - 1), x = min(bx0 * 8 + c, w - 1);
        pix[r * PS + c] = ib[static_cast<size_t>(y) * pitch + x];
      }
    }
    __syncwarp();
    const bool fast_next = s + total < nstrips ? fetch(s + total, pixn) : false;

    // quad butterflies of both m-tiles (blocks g and 8 + g) at positions
    // (sq, t), sq = 0..3, all four classes
    double q[2][4][4];
#pragma unroll
    for (int mt = 0; mt < 2; ++mt) {
      const uint8_t* pb = pix + 8 * (8 * mt + g);
#pragma unroll
      for (int sq = 0; sq < 4; ++sq) {
        const uint2 top = *reinterpret_cast<const uint2*>(pb + sq * PS);
        const uint2 bot = *reinterpret_cast<const uint2*>(pb + (7 - sq) * PS);
        // byte t of the left half, byte 3-t of the right half (one PRMT each)
        const int p00 = __byte_perm(top.x, 0, selL), p01 = __byte_perm(top.y, 0, selR);
        const int p10 = __byte_perm(bot.x, 0, selL), p11 = __byte_perm(bot.y, 0, selR);
        const int rs0 = p00 + p10, ra0 = p00 - p10, rs1 = p01 + p11, ra1 = p01 - p11;
        q[mt][0][sq] = __int2double_rn(rs0 + rs1);
        q[mt][1][sq] = __int2double_rn(rs0 - rs1);
        q[mt][2][sq] = __int2double_rn(ra0 + ra1);
        q[mt][3][sq] = __int2double_rn(ra0 - ra1);
      }
    }
    // per class: filter Y_c^T = q_c^T G_c^T and inverse Z_c^T = Y_c^T W_c^T
    // for both m-tiles, so every operator fragment loaded from shared memory
    // feeds 4 DMMAs (+0.5 rides in the ee class's accumulator)
    double2 z[2][4][2];
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
          dmma(y[0][nt], q[0][c][2 * sp], bb.x);
          dmma(y[1][nt], q[1][c][2 * sp], bb.x);
          dmma(y[0][nt], q[0][c][2 * sp + 1], bb.y);
          dmma(y[1][nt], q[1][c][2 * sp + 1], bb.y);
        }
      if (COEF) {
#pragma unroll
        for (int mt = 0; mt < 2; ++mt) {
          const int bx = bx0 + 8 * mt + g;
          if (bx < bw) {
            double* dst = coef_out + ((static_cast<long long>(f) * bh + by) * bw + bx) * 64;
#pragma unroll
            for (int nt = 0; nt < 2; ++nt)
#pragma unroll
              for (int e = 0; e < 2; ++e) {
                const int o = 8 * nt + 2 * t + e;
                dst[(2 * (o >> 2) + (c >> 1)) * 8 + 2 * (o & 3) + (c & 1)] = e ? y[mt][nt].y : y[mt][nt].x;
              }
          }
        }
      }
#pragma unroll
      for (int mt = 0; mt < 2; ++mt)
#pragma unroll
        for (int nt2 = 0; nt2 < 2; ++nt2) z[mt][c][nt2] = c == 0 ? make_double2(0.5, 0.5) : make_double2(0.0, 0.0);
#pragma unroll
      for (int nt = 0; nt < 2; ++nt)
#pragma unroll
        for (int nt2 = 0; nt2 < 2; ++nt2) {
          const double2 bb = ws[((c * 2 + nt2) * 2 + nt) * 32 + lane];
          dmma(z[0][c][nt2], y[0][nt].x, bb.x);
          dmma(z[1][c][nt2], y[1][nt].x, bb.x);
          dmma(z[0][c][nt2], y[0][nt].y, bb.y);
          dmma(z[1][c][nt2], y[1][nt].y, bb.y);
        }
    }
    // (no __syncwarp: every lane's pixel reads fed the mma.sync.aligned DMMAs
    // above, so they are complete before any lane overwrites the strip)
    // un-butterfly, quantise, write the four reflections of each position
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
          o_ij[e] = floor_to_u8(a + cq);   // (i, j+e)
          o_rj[e] = floor_to_u8(a - cq);   // (7-i, j+e)
          o_ir[e] = floor_to_u8(bq + d);   // (i, 7-j-e)
          o_rr[e] = floor_to_u8(bq - d);   // (7-i, 7-j-e)
        }
        *reinterpret_cast<uint16_t*>(pb + i * PS + j) = static_cast<uint16_t>(o_ij[0] | (o_ij[1] << 8));
        *reinterpret_cast<uint16_t*>(pb + (7 - i) * PS + j) = static_cast<uint16_t>(o_rj[0] | (o_rj[1] << 8));
        *reinterpret_cast<uint16_t*>(pb + i * PS + 6 - j) = static_cast<uint16_t>(o_ir[1] | (o_ir[0] << 8));
        *reinterpret_cast<uint16_t*>(pb + (7 - i) * PS + 6 - j) = static_cast<uint16_t>(o_rr[1] | (o_rr[0] << 8));
      }
    }
    __syncwarp();

    uint8_t* ob = out + f * frame_stride;
    if (fast) {
      uint8_t* p = ob + static_cast<size_t>(by * 8) * pitch + bx0 * 8 + c16;
      stg_stream(p + r0 * pitch, *reinterpret_cast<const uint4*>(pix + r0 * PS + c16));
      stg_stream(p + (r0 + 4) * pitch, *reinterpret_cast<const uint4*>(pix + (r0 + 4) * PS + c16));
    } else {
      for (int e = lane; e < 8 * 128; e += 32) {
        const int r = e >> 7, c = e & 127;
        const int y = by * 8 + r, x = bx0 * 8 + c;
        if (y < h && x < w) ob[static_cast<size_t>(y) * pitch + x] = pix[r * PS + c];
      }
    }
    __syncwarp();
    uint8_t* tmp = pix;
    pix = pixn;
    pixn = tmp;
    fast = fast_next;
  }
  if constexpr (ASYNC) cp_async_wait_all();
}

// ---------------------------------------------------------------------------
// k_fused8_sep: the n = 8 image path for masks of rank P <= 3 (any symmetry;
// layout_sep8 in plan.cc) as the paper's sandwich form with the fewest pairs,
// Y = sum_p L_p X R_p^T (filter.hpp:30-38), forward DCT composed per direction
// (V_p = C A_p, M_p = C B_p), then the inverse Z = C^t Y C — every product an
// 8x8x8 DMMA pair chained fragment to fragment (see k_fused16_sep):
//   T_p^T = M_p x^T  (B: lane (g,t) holds pixels x[g][t], x[g][t+4])
//   Y     = sum_p V_p T_p,  W^T = C^t Y^T,  Z = C^t W + 0.5
// 4P + 4 DMMA per block (8 for a separable mask, the parity-class kernel's
// count, with no butterflies and no operator traffic: the 6P + 2 fragments
// stay in registers; 16 for rank 3 against k_fused8's 20). A warp owns a strip
// of 16 blocks (8 rows x 128 px) staged by cp.async into a double-buffered
// per-warp tile; the output bytes overwrite their own pixels.
namespace f8q {
constexpr int WARPS = 8;
constexpr int SB = 16;
constexpr int PS = 144;  // row stride: 8-byte row loads and u16 stores conflict-free
constexpr int PIX_BYTES = 8 * PS;
constexpr int SMEM = WARPS * 2 * PIX_BYTES;
}  // namespace f8q
#ifndef F8Q_MINB
#define F8Q_MINB 3
#endif
#ifndef F8Q_ILP
#define F8Q_ILP 4
#endif

template <int P, bool COEF>
__global__ void __launch_bounds__(f8q::WARPS * 32, F8Q_MINB)
    k_fused8_sep(const uint8_t* __restrict__ in, uint8_t* __restrict__ out, int w, int h, size_t pitch,
                 long long frame_stride, int nframes, int bw, int bh, int nsx,
                 const double* __restrict__ frag, double* __restrict__ coef_out) {
  using namespace f8q;
  extern __shared__ __align__(16) uint8_t smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  uint8_t* pix = smem + warp * 2 * PIX_BYTES;
  uint8_t* pixn = pix + PIX_BYTES;
  double fm[P][2], fv[P][2], fc[2];
#pragma unroll
  for (int q = 0; q < P; ++q)
#pragma unroll
    for (int sk = 0; sk < 2; ++sk) {
      fm[q][sk] = frag[((q * 2 + 0) * 2 + sk) * 32 + lane];
      fv[q][sk] = frag[((q * 2 + 1) * 2 + sk) * 32 + lane];
    }
#pragma unroll
  for (int sk = 0; sk < 2; ++sk) fc[sk] = frag[P * 128 + sk * 32 + lane];

  const int spf = bh * nsx;  // strip counts < 2^31 (launcher)
  const int nstrips = spf * nframes;
  const int nwarps = blockDim.x >> 5;
  const int total = static_cast<int>(gridDim.x) * nwarps;
  const bool aligned = ((pitch & 15) == 0) && ((reinterpret_cast<uintptr_t>(in) & 15) == 0) &&
                       ((reinterpret_cast<uintptr_t>(out) & 15) == 0) && ((frame_stride & 15) == 0);
  const dctf::FastDiv fd_spf = dctf::make_fastdiv(static_cast<uint32_t>(spf)),
                      fd_nsx = dctf::make_fastdiv(static_cast<uint32_t>(nsx));
  auto strip_at = [&](int si, int& f, int& by, int& bx0) {
    const uint32_t u = static_cast<uint32_t>(si);
    f = static_cast<int>(dctf::fdiv(fd_spf, u));
    const uint32_t rem = u - static_cast<uint32_t>(f) * static_cast<uint32_t>(spf);
    by = static_cast<int>(dctf::fdiv(fd_nsx, rem));
    bx0 = static_cast<int>(rem - static_cast<uint32_t>(by) * static_cast<uint32_t>(nsx)) * SB;
  };
  auto is_fast = [&](int by, int bx0) { return aligned && by * 8 + 8 <= h && (bx0 + SB) * 8 <= w; };
  const int r0 = lane >> 3, c16 = (lane & 7) * 16;
  auto fetch = [&](int si, uint8_t* buf) {
    int f, by, bx0;
    strip_at(si, f, by, bx0);
    if (is_fast(by, bx0)) {
      const uint8_t* src = in + f * frame_stride + static_cast<size_t>(by * 8) * pitch + bx0 * 8 + c16;
      cp_async16(buf + r0 * PS + c16, src + r0 * pitch);
      cp_async16(buf + (r0 + 4) * PS + c16, src + (r0 + 4) * pitch);
    }
    cp_async_commit();
  };
  pdl_trigger();
  pdl_wait();
  int si = static_cast<int>(blockIdx.x) * nwarps + warp;
  if (si < nstrips) fetch(si, pix);
  for (; si < nstrips; si += total) {
    int f, by, bx0;
    strip_at(si, f, by, bx0);
    const bool fast = is_fast(by, bx0);
    cp_async_wait_all();
    if (!fast) {  // tile()'s edge replication, byte by byte
      const uint8_t* ib = in + f * frame_stride;
      for (int e = lane; e < 8 * 128; e += 32) {
        const int r = e >> 7, c = e & 127;
        const int y = min(by * 8 + r, h - 1), x = min(bx0 * 8 + c, w - 1);
        pix[r * PS + c] = ib[static_cast<size_t>(y) * pitch + x];
      }
    }
    __syncwarp();
    if (si + total < nstrips) fetch(si + total, pixn);

    // F8Q_ILP blocks in lock step: their DMMA chains interleave (one chain
    // of 4P + 4 dependent DMMAs per block)
#pragma unroll 1
    for (int b0 = 0; b0 < SB; b0 += F8Q_ILP) {
      double2 y[F8Q_ILP], tt[F8Q_ILP], wt[F8Q_ILP], z[F8Q_ILP];
      double a0[F8Q_ILP], a1[F8Q_ILP];
#pragma unroll
      for (int k = 0; k < F8Q_ILP; ++k) {
        const uint2 v = *reinterpret_cast<const uint2*>(pix + g * PS + 8 * (b0 + k));
        a0[k] = __int2double_rn((v.x >> (8 * t)) & 0xff);  // x[g][t]
        a1[k] = __int2double_rn((v.y >> (8 * t)) & 0xff);  // x[g][t + 4]
        y[k] = make_double2(0.0, 0.0);
      }
#pragma unroll
      for (int q = 0; q < P; ++q) {
#pragma unroll
        for (int k = 0; k < F8Q_ILP; ++k) { tt[k] = make_double2(0.0, 0.0); dmma(tt[k], fm[q][0], a0[k]); }
#pragma unroll
        for (int k = 0; k < F8Q_ILP; ++k) dmma(tt[k], fm[q][1], a1[k]);
#pragma unroll
        for (int k = 0; k < F8Q_ILP; ++k) dmma(y[k], fv[q][0], tt[k].x);
#pragma unroll
        for (int k = 0; k < F8Q_ILP; ++k) dmma(y[k], fv[q][1], tt[k].y);
      }
      if (COEF) {
#pragma unroll
        for (int k = 0; k < F8Q_ILP; ++k) {
          const int bx = bx0 + b0 + k;
          if (bx < bw)
            *reinterpret_cast<double2*>(coef_out + ((static_cast<long long>(f) * bh + by) * bw + bx) * 64 + g * 8 +
                                        2 * t) = y[k];
        }
      }
#pragma unroll
      for (int k = 0; k < F8Q_ILP; ++k) { wt[k] = make_double2(0.0, 0.0); dmma(wt[k], fc[0], y[k].x); }
#pragma unroll
      for (int k = 0; k < F8Q_ILP; ++k) dmma(wt[k], fc[1], y[k].y);
#pragma unroll
      for (int k = 0; k < F8Q_ILP; ++k) { z[k] = make_double2(0.5, 0.5); dmma(z[k], fc[0], wt[k].x); }
#pragma unroll
      for (int k = 0; k < F8Q_ILP; ++k) dmma(z[k], fc[1], wt[k].y);
#pragma unroll
      for (int k = 0; k < F8Q_ILP; ++k)
        *reinterpret_cast<uint16_t*>(pix + g * PS + 8 * (b0 + k) + 2 * t) =
            static_cast<uint16_t>(floor_to_u8(z[k].x) | (floor_to_u8(z[k].y) << 8));
    }
    __syncwarp();
    uint8_t* ob = out + f * frame_stride;
    if (fast) {
      uint8_t* dst = ob + static_cast<size_t>(by * 8) * pitch + bx0 * 8 + c16;
      stg_stream(dst + r0 * pitch, *reinterpret_cast<const uint4*>(pix + r0 * PS + c16));
      stg_stream(dst + (r0 + 4) * pitch, *reinterpret_cast<const uint4*>(pix + (r0 + 4) * PS + c16));
    } else {
      for (int e = lane; e < 8 * 128; e += 32) {
        const int r = e >> 7, c = e & 127;
        const int y = by * 8 + r, x = bx0 * 8 + c;
        if (y < h && x < w) ob[static_cast<size_t>(y) * pitch + x] = pix[r * PS + c];
      }
    }
    __syncwarp();
    uint8_t* tmp = pix;
    pix = pixn;
    pixn = tmp;
  }
  cp_async_wait_all();
}

// ---------------------------------------------------------------------------
// k_fused16: the n = 16 chain fused, one HBM pass per pixel.
//
// CTA tile = a strip of 64 horizontally adjacent 16x16 blocks (16 rows x 1024
// px). 16 warps; lane 0 of warp 0 also streams the operator. Phases per tile
// (CTA barrier between them):
//   pixels -> shared (16-byte loads, prefetched one tile ahead into registers)
//   pixels -> FP64 block staging (the forward DCT is composed into the
//     operator on the host, G = H (C (x) C), as in k_fused8)
//   filter Y^T = P^T G^T: warp (mg = w&3, ng = w>>2) owns 16 blocks x 64
//     outputs; K = 256 streamed as 16 chunks of H^T fragments (32 KB each,
//     cp.async.bulk into a 2-stage ring, refilled as soon as a stage is
//     released by all warps); X stays in
//     shared memory (128 KB)
//   Y -> shared (over X), inverse DCT (O = C^t Y C + 0.5) -> u8 -> strip store.
// Block staging layout: 2 KB per block = 128 words of 16 B; word w holds the
// coefficient pair (u = 2a + {0,1}, v) with v = w >> 3, a = (w & 7) ^ 4(v & 1),
// stored at chunk (w & 7) ^ f(b) of its 128-byte row. The k-mapping of every
// DMMA stage (k(s,t) = 8(s>>1) + 2t + (s&1)) makes each lane's pair one word
// and each quarter-warp phase of every 16-byte access conflict-free.
namespace f16 {
constexpr int CWARPS = 16;  // all warps run MMA; warp 0 lane 0 also streams H
constexpr int TILE = 64;
constexpr int STAGES = 2;
constexpr int HBYTES = 32768;
constexpr int XY_BYTES = TILE * 2048;
constexpr int PS = 1040;
constexpr int PIX_BYTES = 16 * PS;
constexpr int SMEM = 1024 + XY_BYTES + STAGES * HBYTES + PIX_BYTES;
__device__ __forceinline__ int fsw(int b) { return (b & 7) ^ ((b & 1) << 2); }
__device__ __forceinline__ int xw(int b, int w) {
  return b * 2048 + ((w & ~7) << 4) + (((w & 7) ^ fsw(b)) << 4);
}
__device__ __forceinline__ void bar_mma() { asm volatile("bar.sync 1, 512;" ::: "memory"); }
}  // namespace f16

template <bool COEF>
__global__ void __launch_bounds__(f16::CWARPS * 32, 1)
    k_fused16(const uint8_t* __restrict__ in, uint8_t* __restrict__ out, int w, int h, size_t pitch,
              long long frame_stride, int nframes, int bw, int bh, int nsx,
              const double* __restrict__ hf, const double* __restrict__ cb,
              double* __restrict__ coef_out) {
  using namespace f16;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* base = align1024(smem_raw);
  uint8_t* xy = base;
  uint8_t* hst = base + XY_BYTES;
  uint8_t* pix = hst + STAGES * HBYTES;
  pdl_trigger();
  __shared__ uint64_t full[STAGES], empty[STAGES];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], CWARPS);
    }
    fence_barrier_init();
  }
  __syncthreads();
  const long long spf = static_cast<long long>(bh) * nsx;
  const long long ntiles = spf * nframes;

  // H^T chunk stream: the same 16 K-chunks for every tile. Lane 0 of warp 0
  // refills a stage as soon as all 16 warps have released it (no producer
  // warp: 16 warps keep 4 per SM sub-partition and 128 registers each).
  const long long nchunks = ntiles > blockIdx.x ? ((ntiles - 1 - blockIdx.x) / gridDim.x + 1) * 16 : 0;
  auto refill = [&](long long chunk) {
    const int s = static_cast<int>(chunk % STAGES);
    mbar_expect_tx(&full[s], HBYTES);
    bulk_load(hst + s * HBYTES, hf + static_cast<size_t>(chunk % 16) * (HBYTES / 8), HBYTES, &full[s]);
  };
  if (warp == 0 && lane == 0)
    for (long long c = 0; c < STAGES && c < nchunks; ++c) refill(c);  // plan-owned operator
  pdl_wait();

  const int g = lane >> 2, t = lane & 3, mg = warp & 3, ng = warp >> 2;
  const int tid = threadIdx.x;  // 0..511
  const bool aligned = ((pitch & 15) == 0) && ((reinterpret_cast<uintptr_t>(in) & 15) == 0) &&
                       ((reinterpret_cast<uintptr_t>(out) & 15) == 0) && ((frame_stride & 15) == 0);
  const dctf::FastDiv fd_spf = dctf::make_fastdiv(static_cast<uint32_t>(spf)),
                      fd_nsx = dctf::make_fastdiv(static_cast<uint32_t>(nsx));
  auto tile_at = [&](long long ti, int& f, int& by, int& bx0) {  // ti < 2^31 (launcher)
    const uint32_t u = static_cast<uint32_t>(ti);
    f = static_cast<int>(dctf::fdiv(fd_spf, u));
    const uint32_t rem = u - static_cast<uint32_t>(f) * static_cast<uint32_t>(spf);
    by = static_cast<int>(dctf::fdiv(fd_nsx, rem));
    bx0 = static_cast<int>(rem - static_cast<uint32_t>(by) * static_cast<uint32_t>(nsx)) * TILE;
  };
  auto is_fast = [&](int by, int bx0) { return aligned && by * 16 + 16 <= h && bx0 * 16 + 1024 <= w; };
  // thread tid moves 16-byte chunks (row tid>>6, col 16*(tid&63)) and (row+8)
  const int prow = tid >> 6, pcol = (tid & 63) * 16;
  uint4 pf0 = make_uint4(0, 0, 0, 0), pf1 = pf0;
  auto prefetch = [&](long long ti) {
    int f, by, bx0;
    tile_at(ti, f, by, bx0);
    if (is_fast(by, bx0)) {
      const uint8_t* p = in + f * frame_stride + static_cast<size_t>(by * 16) * pitch + bx0 * 16 + pcol;
      pf0 = ldg_stream(p + prow * pitch);
      pf1 = ldg_stream(p + (prow + 8) * pitch);
    }
  };
  long long tile = blockIdx.x;
  if (tile < ntiles) prefetch(tile);
  long long it = 0;
  for (; tile < ntiles; tile += gridDim.x) {
    int f, by, bx0;
    tile_at(tile, f, by, bx0);
    const bool fast = is_fast(by, bx0);
    if (fast) {
      *reinterpret_cast<uint4*>(pix + prow * PS + pcol) = pf0;
      *reinterpret_cast<uint4*>(pix + (prow + 8) * PS + pcol) = pf1;
    } else {
      const uint8_t* ib = in + f * frame_stride;
      for (int e = tid; e < 16 * 1024; e += 512) {
        const int r = e >> 10, c = e & 1023;
        const int y = min(by * 16 + r, h - 1), x = min(bx0 * 16 + c, w - 1);
        pix[r * PS + c] = ib[static_cast<size_t>(y) * pitch + x];
      }
    }
    if (tile + gridDim.x < ntiles) prefetch(tile + gridDim.x);
    bar_mma();

    // ---- pixels -> FP64 staging, blocks 4*warp .. +3. The forward DCT is
    // composed into the operator (G = H (C (x) C)), so word w of a block takes
    // the pixel pair (2a, v), (2a+1, v) in the slot of coefficients (u = 2a+e, v).
#pragma unroll
    for (int bb = 0; bb < 4; ++bb) {
      const int b = 4 * warp + bb;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int wd = lane + 32 * i, v = wd >> 3, a = (wd & 7) ^ (4 * (v & 1));
        const uint32_t q0 = pix[(2 * a) * PS + b * 16 + v];
        const uint32_t q1 = pix[(2 * a + 1) * PS + b * 16 + v];
        *reinterpret_cast<double2*>(xy + xw(b, wd)) = make_double2(__uint2double_rn(q0), __uint2double_rn(q1));
      }
    }
    bar_mma();

    // ---- filter: 16 blocks x 64 outputs per warp, K streamed from the ring
    double2 acc[2][8];
#pragma unroll
    for (int m = 0; m < 2; ++m)
#pragma unroll
      for (int j = 0; j < 8; ++j) acc[m][j] = make_double2(0.0, 0.0);
    const int b0 = 16 * mg + g, b1 = 16 * mg + 8 + g;
    for (int kc = 0; kc < 16; ++kc, ++it) {
      const int s = static_cast<int>(it % STAGES);
      mbar_wait(&full[s], static_cast<uint32_t>((it / STAGES) & 1));
      const double2* hs = reinterpret_cast<const double2*>(hst + s * HBYTES);
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        const int wd = 8 * kc + 4 * q + t;
        const double2 a0 = *reinterpret_cast<const double2*>(xy + xw(b0, wd));
        const double2 a1 = *reinterpret_cast<const double2*>(xy + xw(b1, wd));
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const double2 bf = hs[((8 * ng + j) * 2 + q) * 32 + lane];
          dmma(acc[0][j], a0.x, bf.x);
          dmma(acc[1][j], a1.x, bf.x);
          dmma(acc[0][j], a0.y, bf.y);
          dmma(acc[1][j], a1.y, bf.y);
        }
      }
      __syncwarp();
      __threadfence_block();
      if (lane == 0) mbar_arrive(&empty[s]);
      if (warp == 0 && lane == 0 && it + STAGES < nchunks) {
        mbar_wait(&empty[s], static_cast<uint32_t>((it / STAGES) & 1));
        refill(it + STAGES);
      }
      __syncwarp();
    }
    bar_mma();  // every warp is done reading X
#pragma unroll
    for (int m = 0; m < 2; ++m) {
      const int b = m ? b1 : b0;
#pragma unroll
      for (int j = 0; j < 8; ++j)
        *reinterpret_cast<double2*>(xy + xw(b, 4 * (8 * ng + j) + t)) = acc[m][j];
    }
    if (COEF) {
#pragma unroll
      for (int m = 0; m < 2; ++m) {
        const int bx = bx0 + (m ? b1 : b0);
        if (bx < bw) {
          double* dst = coef_out + ((static_cast<long long>(f) * bh + by) * bw + bx) * 256;
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const int wd = 4 * (8 * ng + j) + t, v = wd >> 3, a = (wd & 7) ^ (4 * (v & 1));
            dst[(2 * a) * 16 + v] = acc[m][j].x;
            dst[(2 * a + 1) * 16 + v] = acc[m][j].y;
          }
        }
      }
    }
    bar_mma();

    // ---- inverse DCT + quantize: blocks 4*warp .. +3
    {
      double ci[2][4];
#pragma unroll
      for (int x = 0; x < 2; ++x)
#pragma unroll
        for (int s = 0; s < 4; ++s) ci[x][s] = cb[(8 * (s >> 1) + 2 * t + (s & 1)) * 16 + 8 * x + g];
#pragma unroll 1
      for (int bb = 0; bb < 4; ++bb) {
        const int b = 4 * warp + bb;
        double2 yv[2][2];
#pragma unroll
        for (int nt = 0; nt < 2; ++nt)
#pragma unroll
          for (int a = 0; a < 2; ++a) {
            const int v = 8 * nt + g;
            yv[nt][a] = *reinterpret_cast<const double2*>(xy + xw(b, 8 * v + ((4 * a + t) ^ (4 * (v & 1)))));
          }
        double2 z[2][2], o[2][2];
#pragma unroll
        for (int mt = 0; mt < 2; ++mt)
#pragma unroll
          for (int nt = 0; nt < 2; ++nt) z[mt][nt] = make_double2(0.0, 0.0);
#pragma unroll
        for (int s = 0; s < 4; ++s)
#pragma unroll
          for (int mt = 0; mt < 2; ++mt)
#pragma unroll
            for (int nt = 0; nt < 2; ++nt) {
              const double bv = (s & 1) ? yv[nt][s >> 1].y : yv[nt][s >> 1].x;
              dmma(z[mt][nt], ci[mt][s], bv);
            }
#pragma unroll
        for (int mt = 0; mt < 2; ++mt)
#pragma unroll
          for (int nt = 0; nt < 2; ++nt) o[mt][nt] = make_double2(0.5, 0.5);
#pragma unroll
        for (int s = 0; s < 4; ++s)
#pragma unroll
          for (int mt = 0; mt < 2; ++mt)
#pragma unroll
            for (int nt = 0; nt < 2; ++nt) {
              const double a = (s & 1) ? z[mt][s >> 1].y : z[mt][s >> 1].x;
              dmma(o[mt][nt], a, ci[nt][s]);
            }
#pragma unroll
        for (int mt = 0; mt < 2; ++mt)
#pragma unroll
          for (int nt = 0; nt < 2; ++nt) {
            const uint32_t q = floor_to_u8(o[mt][nt].x) | (floor_to_u8(o[mt][nt].y) << 8);
            *reinterpret_cast<uint16_t*>(pix + (8 * mt + g) * PS + b * 16 + 8 * nt + 2 * t) =
                static_cast<uint16_t>(q);
          }
      }
    }
    bar_mma();
    uint8_t* ob = out + f * frame_stride;
    if (fast) {
      uint8_t* p = ob + static_cast<size_t>(by * 16) * pitch + bx0 * 16 + pcol;
      stg_stream(p + prow * pitch, *reinterpret_cast<const uint4*>(pix + prow * PS + pcol));
      stg_stream(p + (prow + 8) * pitch, *reinterpret_cast<const uint4*>(pix + (prow + 8) * PS + pcol));
    } else {
      for (int e = tid; e < 16 * 1024; e += 512) {
        const int r = e >> 10, c = e & 1023;
        const int y = by * 16 + r, x = bx0 * 16 + c;
        if (y < h && x < w) ob[static_cast<size_t>(y) * pitch + x] = pix[r * PS + c];
      }
    }
    bar_mma();  // pixel buffer is rewritten by the next tile
  }
}

// ---------------------------------------------------------------------------
// k_fused16_sym: the N = 16 image path for parity-block-diagonal operators
// (symmetric masks; see k_fused8_sym). Per block and class c = (pu, pv):
//   q_c(i, j) = r(j) +/- r(15-j),  r(x) = p(i, x) +/- p(15-i, x),  i, j < 8
//     (exact integers), Y_c = G_c q_c (64 x 64, DMMA, G_c resident in shared
//     memory), then the inverse separably: T = Y_c C_pv along v' (DMMA,
//     constant B fragments) and Z_c = C_pu^T T along u' (lane-local DFMA: each
//     lane already holds all u' of its two columns), and the output pixels
//     are +/- sums of the four Z_c (+0.5 in Z_ee, floor -> u8).
// Dense k_fused16: 288 DMMA per block; here 4 x (128 + 16) DMMA + 4 x 512 DFMA
// per 8 blocks = 72 DMMA + 256 DFMA per block.
// CTA = 4 pairs of warps; a pair owns an m-tile = a strip of 8 blocks (16 rows
// x 128 px): warp 2p handles classes (0, 0), (0, 1), warp 2p+1 classes (1, 0),
// (1, 1); Z_c goes through the pair's shared buffer (swizzled 16-byte chunks)
// for the butterfly, which the two warps split by row. Pixels are prefetched
// one m-tile ahead into registers and double-buffered in shared memory.
namespace f16s {
constexpr int PAIRS = 4, WARPS = 2 * PAIRS;
constexpr int TB = 8;                          // blocks per m-tile
constexpr int PS = 144;                        // pixel row stride
constexpr int PIX_BYTES = 16 * PS;
constexpr int ZBYTES = 4 * TB * 512;           // [class][block][i][t] double2, 16 KB
constexpr int GBYTES = 4 * 8 * 8 * 32 * 16;    // 128 KB
constexpr int CBYTES = 256 * 8;
constexpr int PAIR_BYTES = ZBYTES + 2 * PIX_BYTES;
constexpr int SMEM = GBYTES + CBYTES + PAIRS * PAIR_BYTES;
__device__ __forceinline__ void bar_pair(int pair) {
  asm volatile("bar.sync %0, 64;" ::"r"(1 + pair) : "memory");
}
// byte offset of Z_c[block b][row i][lane column t] (double2: j = 2t, 2t+1)
__device__ __forceinline__ int zoff(int c, int b, int i, int t) {
  return ((c * TB + b) * 4 + (i >> 1)) * 128 + ((((i & 1) * 4 + t) ^ ((b & 1) << 2)) << 4);
}
}  // namespace f16s

template <bool COEF>
__global__ void __launch_bounds__(f16s::WARPS * 32, 1)
    k_fused16_sym(const uint8_t* __restrict__ in, uint8_t* __restrict__ out, int w, int h, size_t pitch,
                  long long frame_stride, int nframes, int bw, int bh, int nsx,
                  const double* __restrict__ gsym, const double* __restrict__ basis,
                  double* __restrict__ coef_out) {
  using namespace f16s;
  extern __shared__ __align__(16) uint8_t smem[];
  const double2* gs = reinterpret_cast<const double2*>(smem);
  const double* cs = reinterpret_cast<const double*>(smem + GBYTES);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  const int pair = warp >> 1, pu = warp & 1, pt = threadIdx.x & 63;  // thread within pair
  uint8_t* zb = smem + GBYTES + CBYTES + pair * PAIR_BYTES;
  uint8_t* pixbuf = zb + ZBYTES;

  const long long spf = static_cast<long long>(bh) * nsx;
  const long long ntiles = spf * nframes;
  const long long stride = static_cast<long long>(gridDim.x) * PAIRS;
  const bool aligned = ((pitch & 15) == 0) && ((reinterpret_cast<uintptr_t>(in) & 15) == 0) &&
                       ((reinterpret_cast<uintptr_t>(out) & 15) == 0) && ((frame_stride & 15) == 0);
  const dctf::FastDiv fd_spf = dctf::make_fastdiv(static_cast<uint32_t>(spf)),
                      fd_nsx = dctf::make_fastdiv(static_cast<uint32_t>(nsx));
  auto tile_at = [&](long long ti, int& f, int& by, int& bx0) {  // ti < 2^31 (launcher)
    const uint32_t u = static_cast<uint32_t>(ti);
    f = static_cast<int>(dctf::fdiv(fd_spf, u));
    const uint32_t rem = u - static_cast<uint32_t>(f) * static_cast<uint32_t>(spf);
    by = static_cast<int>(dctf::fdiv(fd_nsx, rem));
    bx0 = static_cast<int>(rem - static_cast<uint32_t>(by) * static_cast<uint32_t>(nsx)) * TB;
  };
  auto is_fast = [&](int by, int bx0) { return aligned && by * 16 + 16 <= h && bx0 * 16 + 128 <= w; };
  // thread pt of the pair moves 16-byte chunks (row pr, col pc) and (row pr + 8, col pc)
  const int pr = pt >> 3, pc = (pt & 7) * 16;
  uint4 pf0 = make_uint4(0, 0, 0, 0), pf1 = pf0;
  auto prefetch = [&](long long ti) {
    int f, by, bx0;
    tile_at(ti, f, by, bx0);
    if (is_fast(by, bx0)) {
      const uint8_t* p = in + f * frame_stride + static_cast<size_t>(by * 16) * pitch + bx0 * 16 + pc;
      pf0 = ldg_stream(p + pr * pitch);
      pf1 = ldg_stream(p + (pr + 8) * pitch);
    }
  };
  long long tile = static_cast<long long>(blockIdx.x) * PAIRS + pair;
  pdl_trigger();
  cta_copy_async(smem, gsym, GBYTES);  // plan-owned operators: staged before the dependency wait
  cta_copy_async(smem + GBYTES, basis, CBYTES);
  pdl_wait();
  if (tile < ntiles) prefetch(tile);
  cp_async_wait_all();
  __syncthreads();
  // first inverse pass B fragments: C[2(2t + e) + pv][g], per class parity pv
  double cb[2][2];
#pragma unroll
  for (int pv = 0; pv < 2; ++pv)
#pragma unroll
    for (int e = 0; e < 2; ++e) cb[pv][e] = cs[(2 * (2 * t + e) + pv) * 16 + g];

  int it = 0;
  for (; tile < ntiles; tile += stride, ++it) {
    int f, by, bx0;
    tile_at(tile, f, by, bx0);
    const bool fast = is_fast(by, bx0);
    uint8_t* pix = pixbuf + (it & 1) * PIX_BYTES;
    if (fast) {
      *reinterpret_cast<uint4*>(pix + pr * PS + pc) = pf0;
      *reinterpret_cast<uint4*>(pix + (pr + 8) * PS + pc) = pf1;
    } else {
      const uint8_t* ib = in + f * frame_stride;
      for (int e = pt; e < 16 * 128; e += 64) {
        const int r = e >> 7, c = e & 127;
        const int y = min(by * 16 + r, h - 1), x = min(bx0 * 16 + c, w - 1);
        pix[r * PS + c] = ib[static_cast<size_t>(y) * pitch + x];
      }
    }
    bar_pair(pair);
    if (tile + stride < ntiles) prefetch(tile + stride);

    // quad butterflies for this warp's two classes (pu, 0), (pu, 1); lane
    // (g, t): block g, positions (i, j = 2t + e)
    double q[2][8][2];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const uint8_t* top = pix + i * PS + 16 * g;
      const uint8_t* bot = pix + (15 - i) * PS + 16 * g;
      const uint32_t ta = *reinterpret_cast<const uint16_t*>(top + 2 * t);
      const uint32_t tb = *reinterpret_cast<const uint16_t*>(top + 14 - 2 * t);
      const uint32_t ba = *reinterpret_cast<const uint16_t*>(bot + 2 * t);
      const uint32_t bb = *reinterpret_cast<const uint16_t*>(bot + 14 - 2 * t);
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        // column j = 2t + e and its mirror 15 - j (byte 1 - e of the mirrored pair)
        const int pj = (ta >> (8 * e)) & 0xff, pjb = (ba >> (8 * e)) & 0xff;
        const int pm = (tb >> (8 * (1 - e))) & 0xff, pmb = (bb >> (8 * (1 - e))) & 0xff;
        const int rj = pu ? pj - pjb : pj + pjb, rm = pu ? pm - pmb : pm + pmb;
        q[0][i][e] = __int2double_rn(rj + rm);
        q[1][i][e] = __int2double_rn(rj - rm);
      }
    }

#pragma unroll
    for (int pv = 0; pv < 2; ++pv) {
      const int c = 2 * pu + pv;
      const double2* gc = gs + c * (8 * 8 * 32);
      double2 y[8];
#pragma unroll
      for (int nt = 0; nt < 8; ++nt) y[nt] = make_double2(0.0, 0.0);
#pragma unroll
      for (int sp = 0; sp < 8; ++sp) {
        const double a0 = pv ? q[1][sp][0] : q[0][sp][0], a1 = pv ? q[1][sp][1] : q[0][sp][1];
#pragma unroll
        for (int nt = 0; nt < 8; ++nt) {
          const double2 bq = gc[(nt * 8 + sp) * 32 + lane];
          dmma(y[nt], a0, bq.x);
          dmma(y[nt], a1, bq.y);
        }
      }
      if (COEF) {
        const int bx = bx0 + g;
        if (bx < bw) {
          double* dst = coef_out + ((static_cast<long long>(f) * bh + by) * bw + bx) * 256;
#pragma unroll
          for (int nt = 0; nt < 8; ++nt) {
            dst[(2 * nt + pu) * 16 + 2 * (2 * t) + pv] = y[nt].x;
            dst[(2 * nt + pu) * 16 + 2 * (2 * t + 1) + pv] = y[nt].y;
          }
        }
      }
      // T[u' = nt][j = 2t + e] = sum_v' Y[u'][v'] C[2v' + pv][j]
      double2 tt[8];
#pragma unroll
      for (int nt = 0; nt < 8; ++nt) {
        tt[nt] = make_double2(0.0, 0.0);
        dmma(tt[nt], y[nt].x, cb[pv][0]);
        dmma(tt[nt], y[nt].y, cb[pv][1]);
      }
      // Z[i][e] = sum_u' C[2u' + pu][i] T[u'][e]  (+0.5 in the (0, 0) class)
      double z[8][2];
#pragma unroll
      for (int i = 0; i < 8; ++i) z[i][0] = z[i][1] = (c == 0) ? 0.5 : 0.0;
#pragma unroll
      for (int u1 = 0; u1 < 8; ++u1) {
        const double2* crow = reinterpret_cast<const double2*>(cs + (2 * u1 + pu) * 16);
#pragma unroll
        for (int ip = 0; ip < 4; ++ip) {
          const double2 cc = crow[ip];
          z[2 * ip][0] = fma(cc.x, tt[u1].x, z[2 * ip][0]);
          z[2 * ip][1] = fma(cc.x, tt[u1].y, z[2 * ip][1]);
          z[2 * ip + 1][0] = fma(cc.y, tt[u1].x, z[2 * ip + 1][0]);
          z[2 * ip + 1][1] = fma(cc.y, tt[u1].y, z[2 * ip + 1][1]);
        }
      }
#pragma unroll
      for (int i = 0; i < 8; ++i)
        *reinterpret_cast<double2*>(zb + zoff(c, g, i, t)) = make_double2(z[i][0], z[i][1]);
    }
    bar_pair(pair);  // all four Z_c of the m-tile are in; the input pixels are consumed

    // butterfly: this warp takes rows i = 4pu .. 4pu + 3 (and their mirrors)
#pragma unroll
    for (int ii = 0; ii < 4; ++ii) {
      const int i = 4 * pu + ii;
      const double2 zee = *reinterpret_cast<const double2*>(zb + zoff(0, g, i, t));
      const double2 zeo = *reinterpret_cast<const double2*>(zb + zoff(1, g, i, t));
      const double2 zoe = *reinterpret_cast<const double2*>(zb + zoff(2, g, i, t));
      const double2 zoo = *reinterpret_cast<const double2*>(zb + zoff(3, g, i, t));
      uint32_t o_ij[2], o_rj[2], o_im[2], o_rm[2];
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const double ee = e ? zee.y : zee.x, eo = e ? zeo.y : zeo.x;
        const double oe = e ? zoe.y : zoe.x, oo = e ? zoo.y : zoo.x;
        const double a = ee + eo, b = ee - eo, cq = oe + oo, d = oe - oo;
        o_ij[e] = floor_to_u8(a + cq);  // (i, j)
        o_rj[e] = floor_to_u8(a - cq);  // (15-i, j)
        o_im[e] = floor_to_u8(b + d);   // (i, 15-j)
        o_rm[e] = floor_to_u8(b - d);   // (15-i, 15-j)
      }
      uint8_t* top = pix + i * PS + 16 * g;
      uint8_t* bot = pix + (15 - i) * PS + 16 * g;
      *reinterpret_cast<uint16_t*>(top + 2 * t) = static_cast<uint16_t>(o_ij[0] | (o_ij[1] << 8));
      *reinterpret_cast<uint16_t*>(bot + 2 * t) = static_cast<uint16_t>(o_rj[0] | (o_rj[1] << 8));
      *reinterpret_cast<uint16_t*>(top + 14 - 2 * t) = static_cast<uint16_t>(o_im[1] | (o_im[0] << 8));
      *reinterpret_cast<uint16_t*>(bot + 14 - 2 * t) = static_cast<uint16_t>(o_rm[1] | (o_rm[0] << 8));
    }
    bar_pair(pair);  // the strip's output pixels are complete

    uint8_t* ob = out + f * frame_stride;
    if (fast) {
      uint8_t* p = ob + static_cast<size_t>(by * 16) * pitch + bx0 * 16 + pc;
      stg_stream(p + pr * pitch, *reinterpret_cast<const uint4*>(pix + pr * PS + pc));
      stg_stream(p + (pr + 8) * pitch, *reinterpret_cast<const uint4*>(pix + (pr + 8) * PS + pc));
    } else {
      for (int e = pt; e < 16 * 128; e += 64) {
        const int r = e >> 7, c = e & 127;
        const int y = by * 16 + r, x = bx0 * 16 + c;
        if (y < h && x < w) ob[static_cast<size_t>(y) * pitch + x] = pix[r * PS + c];
      }
    }
  }
}

// ---------------------------------------------------------------------------
// k_fused16_sep: the n = 16 image path for masks that are symmetric in both
// axes and a sum of P <= 2 separable terms (Gaussians, box, 1xK motion blur,
// Laplacian-like; layout_sep16 in plan.cc) — config 4's masks. The paper's
// sandwich form with the fewest pairs: per parity class c = (pu, pv) and block
//   Y_c = sum_p V_p,pu Q_c M_p,pv^T     (8x8 factors, forward DCT composed in)
//   Z_c = C_pu^T Y_c C_pv               (inverse DCT, 8x8 factors)
// with Q_c the butterflied quad (exact integers) and the output pixels +/-
// sums of the four Z_c (+0.5 in Z_ee, floor -> u8). Every product is a DMMA
// m8n8k4 pair (K = 8) chained fragment to fragment with no shuffles: each
// step's D fragment (lane (g,t): row g, columns 2t, 2t+1) is the next step's
// B operand with the contraction index permuted to k(s, t) = 2t + s, the
// constant factor on the A side (fragment image from layout_sep16):
//   A: T^T = M_pv Q^T   (B = Q^T: lane (g,t) holds q_c(g, 4s+t), from pixels)
//   B: Y   = V_pu T     (B = T^T fragments of A)
//   C: W^T = C_pv^T Y^T (B = Y fragments)
//   D: Z   = C_pu^T W   (B = W^T fragments; Z_c[g][2t], Z_c[g][2t+1])
// 4 classes x (4 P + 4) DMMA per block: 32 for P = 1 (8,192 FMA) against
// k_fused16_sym's 72 DMMA + 2,048 DFMA and k_fused16's 288 DMMA. All four
// classes of a block live in one lane, so the reflection butterfly is
// lane-local. A warp owns a strip of 8 blocks (16 rows x 128 px), staged by
// cp.async into a double-buffered per-warp tile; outputs overwrite the block's
// own pixels (every lane has read them before the block's first DMMA).
namespace f16p {
constexpr int WARPS = 8;
constexpr int TB = 8;                  // blocks per strip
constexpr int PS = 144;                // pixel row stride (bytes)
constexpr int PIX_BYTES = 16 * PS;
constexpr int SMEM = WARPS * 2 * PIX_BYTES;
}  // namespace f16p

#ifndef F16P_MINB
#define F16P_MINB 3
#endif
#ifndef F16P_UNROLL
#define F16P_UNROLL 2
#endif
constexpr int kF16pUnroll = F16P_UNROLL;
template <int P, bool COEF>
__global__ void __launch_bounds__(f16p::WARPS * 32, F16P_MINB)
    k_fused16_sep(const uint8_t* __restrict__ in, uint8_t* __restrict__ out, int w, int h, size_t pitch,
                  long long frame_stride, int nframes, int bw, int bh, int nsx,
                  const double* __restrict__ frag, double* __restrict__ coef_out) {
  using namespace f16p;
  extern __shared__ __align__(16) uint8_t smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  uint8_t* pix = smem + warp * 2 * PIX_BYTES;
  uint8_t* pixn = pix + PIX_BYTES;
  // constant A fragments: fm = M_p,pv (step A), fv = V_p,pu (step B), fc = C_par (inverse)
  double fm[P][2][2], fv[P][2][2], fc[2][2];
#pragma unroll
  for (int q = 0; q < P; ++q)
#pragma unroll
    for (int par = 0; par < 2; ++par)
#pragma unroll
      for (int sk = 0; sk < 2; ++sk) {
        fm[q][par][sk] = frag[(((q * 2 + 0) * 2 + par) * 2 + sk) * 32 + lane];
        fv[q][par][sk] = frag[(((q * 2 + 1) * 2 + par) * 2 + sk) * 32 + lane];
      }
#pragma unroll
  for (int par = 0; par < 2; ++par)
#pragma unroll
    for (int sk = 0; sk < 2; ++sk) fc[par][sk] = frag[P * 256 + (par * 2 + sk) * 32 + lane];

  const int spf = bh * nsx;        // strip counts < 2^31 (launcher)
  const int nstrips = spf * nframes;
  const int nwarps = blockDim.x >> 5;
  const int total = static_cast<int>(gridDim.x) * nwarps;
  const bool aligned = ((pitch & 15) == 0) && ((reinterpret_cast<uintptr_t>(in) & 15) == 0) &&
                       ((reinterpret_cast<uintptr_t>(out) & 15) == 0) && ((frame_stride & 15) == 0);
  const dctf::FastDiv fd_spf = dctf::make_fastdiv(static_cast<uint32_t>(spf)),
                      fd_nsx = dctf::make_fastdiv(static_cast<uint32_t>(nsx));
  auto strip_at = [&](int si, int& f, int& by, int& bx0) {
    const uint32_t u = static_cast<uint32_t>(si);
    f = static_cast<int>(dctf::fdiv(fd_spf, u));
    const uint32_t rem = u - static_cast<uint32_t>(f) * static_cast<uint32_t>(spf);
    by = static_cast<int>(dctf::fdiv(fd_nsx, rem));
    bx0 = static_cast<int>(rem - static_cast<uint32_t>(by) * static_cast<uint32_t>(nsx)) * TB;
  };
  auto is_fast = [&](int by, int bx0) { return aligned && by * 16 + 16 <= h && (bx0 + TB) * 16 <= w; };
  // strip si's 16 rows x 128 bytes -> buf by cp.async (4 x 16 B per lane)
  auto fetch = [&](int si, uint8_t* buf) {
    int f, by, bx0;
    strip_at(si, f, by, bx0);
    if (is_fast(by, bx0)) {
      const uint8_t* src = in + f * frame_stride + static_cast<size_t>(by * 16) * pitch + bx0 * 16;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int e = 32 * k + lane, row = e >> 3, col = (e & 7) * 16;
        cp_async16(buf + row * PS + col, src + row * pitch + col);
      }
    }
    cp_async_commit();
  };
  pdl_trigger();
  pdl_wait();
  int si = static_cast<int>(blockIdx.x) * nwarps + warp;
  if (si < nstrips) fetch(si, pix);
  for (; si < nstrips; si += total) {
    int f, by, bx0;
    strip_at(si, f, by, bx0);
    const bool fast = is_fast(by, bx0);
    cp_async_wait_all();
    if (!fast) {  // tile()'s edge replication, byte by byte
      const uint8_t* ib = in + f * frame_stride;
      for (int e = lane; e < 16 * 128; e += 32) {
        const int r = e >> 7, c = e & 127;
        const int y = min(by * 16 + r, h - 1), x = min(bx0 * 16 + c, w - 1);
        pix[r * PS + c] = ib[static_cast<size_t>(y) * pitch + x];
      }
    }
    __syncwarp();
    if (si + total < nstrips) fetch(si + total, pixn);

#pragma unroll kF16pUnroll
    for (int b = 0; b < TB; ++b) {
      uint8_t* pb = pix + 16 * b;
      const uint4 top = *reinterpret_cast<const uint4*>(pb + g * PS);
      const uint4 bot = *reinterpret_cast<const uint4*>(pb + (15 - g) * PS);
      // q[pu][pv][s] at quad position (g, 4s + t); j = 4s + t, mirror 15 - j
      double q[2][2][2];
#pragma unroll
      for (int sk = 0; sk < 2; ++sk) {
        const uint32_t tw = sk ? top.y : top.x, tm = sk ? top.z : top.w;  // bytes j and 15 - j
        const uint32_t bw2 = sk ? bot.y : bot.x, bm = sk ? bot.z : bot.w;
        const int a = (tw >> (8 * t)) & 0xff, am = (tm >> (8 * (3 - t))) & 0xff;
        const int c = (bw2 >> (8 * t)) & 0xff, cm = (bm >> (8 * (3 - t))) & 0xff;
        const int rp = a + c, rm = a - c, rpm = am + cm, rmm = am - cm;
        q[0][0][sk] = __int2double_rn(rp + rpm);
        q[0][1][sk] = __int2double_rn(rp - rpm);
        q[1][0][sk] = __int2double_rn(rm + rmm);
        q[1][1][sk] = __int2double_rn(rm - rmm);
      }
      // the four class chains in lock step so their DMMAs interleave
      double2 y[4], tt[4], wt[4], z[4];
#pragma unroll
      for (int c = 0; c < 4; ++c) y[c] = make_double2(0.0, 0.0);
#pragma unroll
      for (int qq = 0; qq < P; ++qq) {
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          tt[c] = make_double2(0.0, 0.0);
          dmma(tt[c], fm[qq][c & 1][0], q[c >> 1][c & 1][0]);
        }
#pragma unroll
        for (int c = 0; c < 4; ++c) dmma(tt[c], fm[qq][c & 1][1], q[c >> 1][c & 1][1]);
#pragma unroll
        for (int c = 0; c < 4; ++c) dmma(y[c], fv[qq][c >> 1][0], tt[c].x);
#pragma unroll
        for (int c = 0; c < 4; ++c) dmma(y[c], fv[qq][c >> 1][1], tt[c].y);
      }
      if (COEF) {
        const int bx = bx0 + b;
        if (bx < bw) {
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            const int pu = c >> 1, pv = c & 1;
            double* dst = coef_out + ((static_cast<long long>(f) * bh + by) * bw + bx) * 256 + (2 * g + pu) * 16;
            dst[2 * (2 * t) + pv] = y[c].x;
            dst[2 * (2 * t + 1) + pv] = y[c].y;
          }
        }
      }
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        wt[c] = make_double2(0.0, 0.0);
        dmma(wt[c], fc[c & 1][0], y[c].x);
      }
#pragma unroll
      for (int c = 0; c < 4; ++c) dmma(wt[c], fc[c & 1][1], y[c].y);
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        z[c] = c == 0 ? make_double2(0.5, 0.5) : make_double2(0.0, 0.0);
        dmma(z[c], fc[c >> 1][0], wt[c].x);
      }
#pragma unroll
      for (int c = 0; c < 4; ++c) dmma(z[c], fc[c >> 1][1], wt[c].y);
      // reflections of quad positions (g, 2t + e): Z_(pu,pv)
      uint32_t o_ij[2], o_rj[2], o_im[2], o_rm[2];
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const double ee = e ? z[0].y : z[0].x, eo = e ? z[1].y : z[1].x;
        const double oe = e ? z[2].y : z[2].x, oo = e ? z[3].y : z[3].x;
        const double a = ee + eo, bq = ee - eo, cq = oe + oo, d = oe - oo;
        o_ij[e] = floor_to_u8(a + cq);   // (g, j)
        o_rj[e] = floor_to_u8(a - cq);   // (15-g, j)
        o_im[e] = floor_to_u8(bq + d);   // (g, 15-j)
        o_rm[e] = floor_to_u8(bq - d);   // (15-g, 15-j)
      }
      *reinterpret_cast<uint16_t*>(pb + g * PS + 2 * t) = static_cast<uint16_t>(o_ij[0] | (o_ij[1] << 8));
      *reinterpret_cast<uint16_t*>(pb + (15 - g) * PS + 2 * t) = static_cast<uint16_t>(o_rj[0] | (o_rj[1] << 8));
      *reinterpret_cast<uint16_t*>(pb + g * PS + 14 - 2 * t) = static_cast<uint16_t>(o_im[1] | (o_im[0] << 8));
      *reinterpret_cast<uint16_t*>(pb + (15 - g) * PS + 14 - 2 * t) =
          static_cast<uint16_t>(o_rm[1] | (o_rm[0] << 8));
    }
    __syncwarp();
    uint8_t* ob = out + f * frame_stride;
    if (fast) {
      uint8_t* dst = ob + static_cast<size_t>(by * 16) * pitch + bx0 * 16;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int e = 32 * k + lane, row = e >> 3, col = (e & 7) * 16;
        stg_stream(dst + row * pitch + col, *reinterpret_cast<const uint4*>(pix + row * PS + col));
      }
    } else {
      for (int e = lane; e < 16 * 128; e += 32) {
        const int r = e >> 7, c = e & 127;
        const int y = by * 16 + r, x = bx0 * 16 + c;
        if (y < h && x < w) ob[static_cast<size_t>(y) * pitch + x] = pix[r * PS + c];
      }
    }
    __syncwarp();
    uint8_t* tmp = pix;
    pix = pixn;
    pixn = tmp;
  }
  cp_async_wait_all();
}

dctf_status launch_fused8(const dctf_plan* p, const uint8_t* in, uint8_t* out, int w, int h,
                          size_t pitch, long long frame_stride, int nframes, double* coef_out,
                          cudaStream_t st) {
  auto kernel = coef_out ? k_fused8<true> : k_fused8<false>;
  {
    const dctf_status sa = dctf::ensure_dyn_smem(reinterpret_cast<const void*>(kernel), f8::SMEM, "k_fused8");
    if (sa != DCTF_OK) return sa;
  }
  const int bw = (w + 7) / 8, bh = (h + 7) / 8, nsx = (bw + f8::SB - 1) / f8::SB;
  const long long nstrips = static_cast<long long>(bh) * nsx * nframes;
  const long long slots = 2LL * sm_count(p->device);
  const int nw = static_cast<int>(std::max<long long>(1, std::min<long long>(f8::WARPS, nstrips / slots)));
  const long long ctas = std::min<long long>(slots, (nstrips + nw - 1) / nw);
  if (ctas <= 0) return DCTF_OK;
  if (static_cast<long long>(bh) * nsx * nframes >= (1LL << 31))
    return set_error(DCTF_INVALID_ARGUMENT, "image batch too large (>= 2^31 work units)");
  CUDA_TRY(dctf::launch_pdl(kernel, static_cast<unsigned>(ctas), nw * 32, 32768 + nw * f8::WARP_BYTES, st,
                            in, out, w, h, pitch, frame_stride, nframes, bw, bh, nsx,
                            static_cast<const double*>(p->d_hfused), static_cast<const double*>(p->d_basis),
                            coef_out));
  dctf::add_launches(1);
  return DCTF_OK;
}

dctf_status launch_fused8_sym(const dctf_plan* p, const uint8_t* in, uint8_t* out, int w, int h,
                              size_t pitch, long long frame_stride, int nframes, double* coef_out,
                              cudaStream_t st, bool host_mapped) {
  auto kernel = host_mapped ? (coef_out ? k_fused8_sym<true, false> : k_fused8_sym<false, false>)
                            : (coef_out ? k_fused8_sym<true, true> : k_fused8_sym<false, true>);
  {
    const dctf_status sa = dctf::ensure_dyn_smem(reinterpret_cast<const void*>(kernel), f8s::SMEM, "k_fused8_sym");
    if (sa != DCTF_OK) return sa;
  }
  const int bw = (w + 7) / 8, bh = (h + 7) / 8, nsx = (bw + f8s::SB - 1) / f8s::SB;
  const long long nstrips = static_cast<long long>(bh) * nsx * nframes;
  // small images: fewer warps per CTA so the strips spread over all SMs
  const long long slots = static_cast<long long>(F8S_MINB) * sm_count(p->device);
  const int nw = static_cast<int>(std::max<long long>(1, std::min<long long>(f8s::WARPS, nstrips / slots)));
  const long long ctas = std::min<long long>(slots, (nstrips + nw - 1) / nw);
  if (ctas <= 0) return DCTF_OK;
  if (static_cast<long long>(bh) * nsx * nframes >= (1LL << 31))
    return set_error(DCTF_INVALID_ARGUMENT, "image batch too large (>= 2^31 work units)");
  CUDA_TRY(dctf::launch_pdl(kernel, static_cast<unsigned>(ctas), nw * 32, 16384 + nw * 2 * f8s::PIX_BYTES, st,
                            in, out, w, h, pitch, frame_stride, nframes, bw, bh, nsx,
                            static_cast<const double*>(p->d_hsym), coef_out));
  dctf::add_launches(1);
  return DCTF_OK;
}

dctf_status launch_fused16(const dctf_plan* p, const uint8_t* in, uint8_t* out, int w, int h,
                           size_t pitch, long long frame_stride, int nframes, double* coef_out,
                           cudaStream_t st) {
  auto kernel = coef_out ? k_fused16<true> : k_fused16<false>;
  {
    const dctf_status sa = dctf::ensure_dyn_smem(reinterpret_cast<const void*>(kernel), f16::SMEM, "k_fused16");
    if (sa != DCTF_OK) return sa;
  }
  const int bw = (w + 15) / 16, bh = (h + 15) / 16, nsx = (bw + f16::TILE - 1) / f16::TILE;
  const long long ntiles = static_cast<long long>(bh) * nsx * nframes;
  const long long ctas = std::min<long long>(sm_count(p->device), ntiles);
  if (ctas <= 0) return DCTF_OK;
  if (static_cast<long long>(bh) * nsx * nframes >= (1LL << 31))
    return set_error(DCTF_INVALID_ARGUMENT, "image batch too large (>= 2^31 work units)");
  CUDA_TRY(dctf::launch_pdl(kernel, static_cast<unsigned>(ctas), f16::CWARPS * 32, f16::SMEM, st,
                            in, out, w, h, pitch, frame_stride, nframes, bw, bh, nsx,
                            static_cast<const double*>(p->d_hfused), static_cast<const double*>(p->d_basis),
                            coef_out));
  dctf::add_launches(1);
  return DCTF_OK;
}

template <int P>
dctf_status launch_fused8_sep_p(const dctf_plan* p, const uint8_t* in, uint8_t* out, int w, int h, size_t pitch,
                                long long frame_stride, int nframes, double* coef_out, cudaStream_t st) {
  auto kernel = coef_out ? k_fused8_sep<P, true> : k_fused8_sep<P, false>;
  {
    const dctf_status sa = dctf::ensure_dyn_smem(reinterpret_cast<const void*>(kernel), f8q::SMEM, "k_fused8_sep");
    if (sa != DCTF_OK) return sa;
  }
  const int bw = (w + 7) / 8, bh = (h + 7) / 8, nsx = (bw + f8q::SB - 1) / f8q::SB;
  const long long nstrips = static_cast<long long>(bh) * nsx * nframes;
  if (nstrips <= 0) return DCTF_OK;
  if (nstrips >= (1LL << 31)) return set_error(DCTF_INVALID_ARGUMENT, "image batch too large (>= 2^31 work units)");
  // small images: fewer warps per CTA so the strips spread over all SMs
  const long long slots = static_cast<long long>(F8Q_MINB) * sm_count(p->device);
  const int nw = static_cast<int>(std::max<long long>(1, std::min<long long>(f8q::WARPS, nstrips / slots)));
  const long long ctas = std::min<long long>(slots, (nstrips + nw - 1) / nw);
  CUDA_TRY(dctf::launch_pdl(kernel, static_cast<unsigned>(ctas), nw * 32, nw * 2 * f8q::PIX_BYTES, st, in, out, w, h,
                            pitch, frame_stride, nframes, bw, bh, nsx, static_cast<const double*>(p->d_sep),
                            coef_out));
  dctf::add_launches(1);
  return DCTF_OK;
}

template <int P>
dctf_status launch_fused16_sep_p(const dctf_plan* p, const uint8_t* in, uint8_t* out, int w, int h, size_t pitch,
                                 long long frame_stride, int nframes, double* coef_out, cudaStream_t st) {
  auto kernel = coef_out ? k_fused16_sep<P, true> : k_fused16_sep<P, false>;
  {
    const dctf_status sa = dctf::ensure_dyn_smem(reinterpret_cast<const void*>(kernel), f16p::SMEM, "k_fused16_sep");
    if (sa != DCTF_OK) return sa;
  }
  const int bw = (w + 15) / 16, bh = (h + 15) / 16, nsx = (bw + f16p::TB - 1) / f16p::TB;
  const long long nstrips = static_cast<long long>(bh) * nsx * nframes;
  if (nstrips <= 0) return DCTF_OK;
  if (nstrips >= (1LL << 31)) return set_error(DCTF_INVALID_ARGUMENT, "image batch too large (>= 2^31 work units)");
  const long long slots = static_cast<long long>(F16P_MINB) * sm_count(p->device);
  const int nw = static_cast<int>(std::max<long long>(1, std::min<long long>(f16p::WARPS, nstrips / slots)));
  const long long ctas = std::min<long long>(slots, (nstrips + nw - 1) / nw);
  CUDA_TRY(dctf::launch_pdl(kernel, static_cast<unsigned>(ctas), nw * 32, nw * 2 * f16p::PIX_BYTES, st, in, out, w, h,
                            pitch, frame_stride, nframes, bw, bh, nsx, static_cast<const double*>(p->d_sep),
                            coef_out));
  dctf::add_launches(1);
  return DCTF_OK;
}

dctf_status launch_fused16_sym(const dctf_plan* p, const uint8_t* in, uint8_t* out, int w, int h,
                               size_t pitch, long long frame_stride, int nframes, double* coef_out,
                               cudaStream_t st) {
  auto kernel = coef_out ? k_fused16_sym<true> : k_fused16_sym<false>;
  {
    const dctf_status sa = dctf::ensure_dyn_smem(reinterpret_cast<const void*>(kernel), f16s::SMEM, "k_fused16_sym");
    if (sa != DCTF_OK) return sa;
  }
  const int bw = (w + 15) / 16, bh = (h + 15) / 16, nsx = (bw + f16s::TB - 1) / f16s::TB;
  const long long ntiles = static_cast<long long>(bh) * nsx * nframes;
  if (ntiles <= 0) return DCTF_OK;
  if (ntiles >= (1LL << 31)) return set_error(DCTF_INVALID_ARGUMENT, "image batch too large (>= 2^31 work units)");
  const long long ctas = std::min<long long>(sm_count(p->device), (ntiles + f16s::PAIRS - 1) / f16s::PAIRS);
  CUDA_TRY(dctf::launch_pdl(kernel, static_cast<unsigned>(ctas), f16s::WARPS * 32, f16s::SMEM, st,
                            in, out, w, h, pitch, frame_stride, nframes, bw, bh, nsx,
                            static_cast<const double*>(p->d_hsym), static_cast<const double*>(p->d_basis),
                            coef_out));
  dctf::add_launches(1);
  return DCTF_OK;
}

}  // namespace

namespace dctf {

// filter_image on device buffers, one frame or a strided frame batch.
dctf_status filter_image_device(const dctf_plan* p, const uint8_t* in, uint8_t* out, int w, int h,
                                size_t pitch, long long frame_stride, int nframes, double* coef_out,
                                cudaStream_t st, bool host_mapped) {
  if (p->unbounded && p->n == 8 && !coef_out)
    return dctf::launch_refchain8(p, in, out, w, h, pitch, frame_stride, nframes, st);
  if (p->kq && !coef_out)
    return dctf::launch_fused8_q(&p, 1, nullptr, in, out, w, h, pitch, frame_stride, nframes, st, host_mapped,
                                 nan_flag(p));
  if (p->n == 8 && p->precision == DCTF_PREC_INT8_EXACT && !p->unbounded)
    return dctf::launch_fused8_i8(p, in, out, w, h, pitch, frame_stride, nframes, coef_out, st,
                                  sm_count(p->device));
  const bool split = p->precision == DCTF_PREC_TF32X3 || p->precision == DCTF_PREC_BF16X3 || p->unbounded;
  if (p->n == 8 && p->sep_rank > 0 && !host_mapped && !p->unbounded) {
    if (p->sep_rank == 1) return launch_fused8_sep_p<1>(p, in, out, w, h, pitch, frame_stride, nframes, coef_out, st);
    if (p->sep_rank == 2) return launch_fused8_sep_p<2>(p, in, out, w, h, pitch, frame_stride, nframes, coef_out, st);
    return launch_fused8_sep_p<3>(p, in, out, w, h, pitch, frame_stride, nframes, coef_out, st);
  }
  if (p->n == 8 && p->sym && !p->unbounded)
    return launch_fused8_sym(p, in, out, w, h, pitch, frame_stride, nframes, coef_out, st, host_mapped);
  if (p->n == 8 && !split) return launch_fused8(p, in, out, w, h, pitch, frame_stride, nframes, coef_out, st);
  if (p->n == 16 && p->sep_rank > 0 && !p->unbounded && !std::getenv("DCTF_N16_UNFUSED"))
    return p->sep_rank == 1
               ? launch_fused16_sep_p<1>(p, in, out, w, h, pitch, frame_stride, nframes, coef_out, st)
               : launch_fused16_sep_p<2>(p, in, out, w, h, pitch, frame_stride, nframes, coef_out, st);
  if (p->n == 16 && p->sym && !p->unbounded && !std::getenv("DCTF_N16_UNFUSED"))
    return launch_fused16_sym(p, in, out, w, h, pitch, frame_stride, nframes, coef_out, st);
  if (!split && !std::getenv("DCTF_N16_UNFUSED"))
    return launch_fused16(p, in, out, w, h, pitch, frame_stride, nframes, coef_out, st);
  // Unfused: forward (exact) -> H (split-precision tensor cores, or FP64 when
  // DCTF_N16_UNFUSED is set for diagnostics) -> inverse (exact) + quantize.
  const int n = p->n, nn = n * n;
  const int bw = (w + n - 1) / n, bh = (h + n - 1) / n;
  const long long nb = static_cast<long long>(bw) * bh;
  double* xbuf = nullptr;
  double* ybuf = nullptr;
  CUDA_TRY(cudaMallocAsync(reinterpret_cast<void**>(&xbuf), nb * nn * sizeof(double), st));
  if (!coef_out) CUDA_TRY(cudaMallocAsync(reinterpret_cast<void**>(&ybuf), nb * nn * sizeof(double), st));
  dctf_status s = DCTF_OK;
  for (int f = 0; f < nframes && s == DCTF_OK; ++f) {
    double* y = coef_out ? coef_out + f * nb * nn : ybuf;
    s = launch_forward_u8(p, in + f * frame_stride, w, h, pitch, xbuf, st);
    if (s == DCTF_OK) s = launch_coef(p, xbuf, y, nb, st);
    if (s == DCTF_OK) s = launch_inverse_u8(p, y, out + f * frame_stride, w, h, pitch, st);
  }
  cudaFreeAsync(xbuf, st);
  if (ybuf) cudaFreeAsync(ybuf, st);
  return s;
}

}  // namespace dctf
