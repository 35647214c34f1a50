// Coefficient-domain filter kernels (FilterPlan::filter_coeffs,
// filter.hpp:65-67; apply_pairs, filter.hpp:30-45): Y = H X per block on the
// FP64 DMMA pipe — dense k_coef8 / k_coef16 and the parity-class
// k_coef8_sym / k_coef16_sym — and their launchers.
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
// k_coef8: Y^T (blocks x 64) = X^T (blocks x 64) * H^T, FP64 DMMA.
//
// Work unit: a tile of 16 consecutive blocks (8 KB of X). Each warp owns a
// strided sequence of tiles and its own STAGES-deep ring of 8 KB buffers;
// lane 0 issues four TMA box loads per tile ([16 blocks x 16 coefficients],
// 128B swizzle: 16-byte chunk c of row r lands at chunk c ^ (r & 7)) and the
// warp waits on that stage's mbarrier. Contraction index of k-step pair q in
// K-chunk kc for lane t: 16kc + 4t + 2q + {0,1}, so a lane's two k-steps are
// one swizzled 16-byte word and each quarter-warp phase of the LDS.128
// (lanes g in {2p,2p+1}, t in 0..3) hits 8 distinct chunks: (2t+q) ^ g. H^T fragments come from shared memory in the matching order
// (layout_hcoef). Accumulators: 2 m-tiles x 8 n-tiles per warp (16 blocks x
// 64 outputs), written straight from registers as 16-byte stores.
namespace c8 {
constexpr int WARPS = 8;
constexpr int STAGES = 2;
constexpr int TILE = 16;
constexpr int STAGE_BYTES = TILE * 64 * 8;  // 8 KB
constexpr int SMEM = 1024 + 32768 + WARPS * STAGES * STAGE_BYTES;
}  // namespace c8

__global__ void __launch_bounds__(c8::WARPS * 32, 1)
    k_coef8(const __grid_constant__ CUtensorMap xmap, const double* __restrict__ hc,
            double* __restrict__ out, long long nblocks) {
  using namespace c8;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* base = align1024(smem_raw);
  const double2* hs = reinterpret_cast<const double2*>(base);
  uint8_t* stages = base + 32768;
  __shared__ uint64_t bars[WARPS * STAGES];

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  if (threadIdx.x == 0) {
    prefetch_tmap(&xmap);
    for (int i = 0; i < WARPS * STAGES; ++i) mbar_init(&bars[i], 1);
    fence_barrier_init();
  }
  pdl_trigger();
  cta_copy_async(base, hc, 32768);  // plan-owned operator
  pdl_wait();
  cp_async_wait_all();
  __syncthreads();

  const long long ntiles = (nblocks + TILE - 1) / TILE;
  const long long total = static_cast<long long>(gridDim.x) * WARPS;
  const long long first = static_cast<long long>(blockIdx.x) * WARPS + warp;
  uint8_t* ring = stages + warp * STAGES * STAGE_BYTES;
  uint64_t* wb = bars + warp * STAGES;

  auto issue = [&](int s, long long tile) {
    uint8_t* dst = ring + s * STAGE_BYTES;
    mbar_expect_tx(&wb[s], STAGE_BYTES);
#pragma unroll
    for (int cc = 0; cc < 4; ++cc)
      tma_load_2d(dst + cc * 2048, &xmap, &wb[s], cc * 16, static_cast<int>(tile * TILE));
  };
  if (lane == 0) {
#pragma unroll
    for (int s = 0; s < STAGES; ++s) {
      const long long tile = first + s * total;
      if (tile < ntiles) issue(s, tile);
    }
  }
  __syncwarp();

  for (long long i = 0;; ++i) {
    const long long tile = first + i * total;
    if (tile >= ntiles) break;
    const int s = static_cast<int>(i % STAGES);
    mbar_wait(&wb[s], static_cast<uint32_t>((i / STAGES) & 1));
    const uint8_t* st = ring + s * STAGE_BYTES;

    double2 acc[2][8];
#pragma unroll
    for (int m = 0; m < 2; ++m)
#pragma unroll
      for (int j = 0; j < 8; ++j) acc[m][j] = make_double2(0.0, 0.0);

#pragma unroll
    for (int kc = 0; kc < 4; ++kc) {
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        const int sw = ((2 * t + q) ^ g) << 4;
        const double2 a0 = *reinterpret_cast<const double2*>(st + kc * 2048 + g * 128 + sw);
        const double2 a1 = *reinterpret_cast<const double2*>(st + kc * 2048 + (8 + g) * 128 + sw);
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const double2 b = hs[((kc * 8 + j) * 2 + q) * 32 + lane];
          dmma(acc[0][j], a0.x, b.x);
          dmma(acc[0][j], a0.y, b.y);
          dmma(acc[1][j], a1.x, b.x);
          dmma(acc[1][j], a1.y, b.y);
        }
      }
    }
    __syncwarp();
    __threadfence_block();  // drain in-flight LDS of this stage before TMA reuses it
    if (lane == 0) {
      const long long nt = tile + STAGES * total;
      if (nt < ntiles) {
        fence_proxy_async();
        issue(s, nt);
      }
    }
#pragma unroll
    for (int m = 0; m < 2; ++m) {
      const long long blk = tile * TILE + 8 * m + g;
      if (blk < nblocks) {
        double* dst = out + blk * 64 + 2 * t;
#pragma unroll
        for (int j = 0; j < 8; ++j) *reinterpret_cast<double2*>(dst + 8 * j) = acc[m][j];
      }
    }
  }
}

// ---------------------------------------------------------------------------
// k_coef8_sym: filter_coeffs for operators block-diagonal in the (u mod 2,
// v mod 2) parity classes (see layout_sym8): per class Y_c = H_c X_c, 16 x 16,
// 4 DMMA per block instead of 16 — the coefficient path becomes HBM-bound.
// Per-warp pipeline over 16-block tiles (8 KB): TMA load (4 boxes [16 blocks
// x 16 coefficients], 128B swizzle) -> class contraction from the staged
// tile -> results written back into the same stage in the same swizzled
// layout -> TMA store (same box geometry), so HBM sees one streaming read
// and one streaming write. 3 stages: tile i computes while tile i+1 lands
// and tile i-1's store drains; a stage is reloaded once the bulk store that
// last used it has finished reading it (cp.async.bulk.wait_group.read).
// Lane (g, t), m-tile mt: block row 8mt + g; class k-step s <-> (u' = s,
// v' = t), i.e. box s, 16-byte chunk 4 pu + t holding classes (pu, 0) and
// (pu, 1); lanes of odd g fetch the pu = 1 chunk first so every
// quarter-warp phase hits 8 distinct chunks.
namespace c8s {
constexpr int WARPS = 8;
constexpr int STAGES = 3;
constexpr int TILE = 16;
constexpr int STAGE_BYTES = TILE * 64 * 8;  // 8 KB
constexpr int SMEM = 1024 + 8192 + WARPS * STAGES * STAGE_BYTES;
}  // namespace c8s

__global__ void __launch_bounds__(c8s::WARPS * 32, 1)
    k_coef8_sym(const __grid_constant__ CUtensorMap xmap, const __grid_constant__ CUtensorMap ymap,
                const double* __restrict__ hc, long long nblocks) {
  using namespace c8s;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* base = align1024(smem_raw);
  const double2* hs = reinterpret_cast<const double2*>(base);
  uint8_t* stages = base + 8192;
  __shared__ uint64_t bars[WARPS * STAGES];

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  if (threadIdx.x == 0) {
    prefetch_tmap(&xmap);
    prefetch_tmap(&ymap);
    for (int i = 0; i < WARPS * STAGES; ++i) mbar_init(&bars[i], 1);
    fence_barrier_init();
  }
  pdl_trigger();
  cta_copy_async(base, hc, 8192);  // plan-owned operator
  pdl_wait();
  cp_async_wait_all();
  __syncthreads();

  const long long ntiles = (nblocks + TILE - 1) / TILE;
  const long long total = static_cast<long long>(gridDim.x) * WARPS;
  const long long first = static_cast<long long>(blockIdx.x) * WARPS + warp;
  uint8_t* ring = stages + warp * STAGES * STAGE_BYTES;
  uint64_t* wb = bars + warp * STAGES;
  auto issue = [&](int s, long long tile) {
    uint8_t* dst = ring + s * STAGE_BYTES;
    mbar_expect_tx(&wb[s], STAGE_BYTES);
#pragma unroll
    for (int cc = 0; cc < 4; ++cc)
      tma_load_2d(dst + cc * 2048, &xmap, &wb[s], cc * 16, static_cast<int>(tile * TILE));
  };
  if (lane == 0) {
    if (first < ntiles) issue(0, first);
    if (first + total < ntiles) issue(1, first + total);
  }
  __syncwarp();
  const int pa = g & 1;

  for (long long i = 0;; ++i) {
    const long long tile = first + i * total;
    if (tile >= ntiles) break;
    const int s = static_cast<int>(i % STAGES);
    mbar_wait(&wb[s], static_cast<uint32_t>((i / STAGES) & 1));
    uint8_t* st = ring + s * STAGE_BYTES;

    double q[2][4][4];  // [m-tile][class][k-step]
#pragma unroll
    for (int mt = 0; mt < 2; ++mt) {
      const uint8_t* rb = st + (8 * mt + g) * 128;
#pragma unroll
      for (int sq = 0; sq < 4; ++sq) {
        const double2 va = *reinterpret_cast<const double2*>(rb + sq * 2048 + (((4 * pa + t) ^ g) << 4));
        const double2 vb = *reinterpret_cast<const double2*>(rb + sq * 2048 + (((4 * (pa ^ 1) + t) ^ g) << 4));
        const double2 v0 = pa ? vb : va, v1 = pa ? va : vb;
        q[mt][0][sq] = v0.x;
        q[mt][1][sq] = v0.y;
        q[mt][2][sq] = v1.x;
        q[mt][3][sq] = v1.y;
      }
    }
    double2 y[2][4][2];
#pragma unroll
    for (int mt = 0; mt < 2; ++mt)
#pragma unroll
      for (int c = 0; c < 4; ++c)
#pragma unroll
        for (int nt = 0; nt < 2; ++nt) y[mt][c][nt] = make_double2(0.0, 0.0);
#pragma unroll
    for (int c = 0; c < 4; ++c)
#pragma unroll
      for (int sp = 0; sp < 2; ++sp)
#pragma unroll
        for (int nt = 0; nt < 2; ++nt) {
          const double2 bb = hs[((c * 2 + nt) * 2 + sp) * 32 + lane];
          dmma(y[0][c][nt], q[0][c][2 * sp], bb.x);
          dmma(y[1][c][nt], q[1][c][2 * sp], bb.x);
          dmma(y[0][c][nt], q[0][c][2 * sp + 1], bb.y);
          dmma(y[1][c][nt], q[1][c][2 * sp + 1], bb.y);
        }
    __syncwarp();  // every lane's reads of this stage are done
    // Y back into the stage: coefficient (2u'+pu, 2v'+pv), u' = 2nt + (t>>1),
    // v' = 2(t&1) + e -> box u', chunk 4pu + v', element pv
#pragma unroll
    for (int mt = 0; mt < 2; ++mt) {
      uint8_t* rb = st + (8 * mt + g) * 128;
#pragma unroll
      for (int pu = 0; pu < 2; ++pu)
#pragma unroll
        for (int nt = 0; nt < 2; ++nt)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int box = 2 * nt + (t >> 1), chunk = 4 * pu + 2 * (t & 1) + e;
            const double a = e ? y[mt][2 * pu][nt].y : y[mt][2 * pu][nt].x;
            const double b = e ? y[mt][2 * pu + 1][nt].y : y[mt][2 * pu + 1][nt].x;
            *reinterpret_cast<double2*>(rb + box * 2048 + ((chunk ^ g) << 4)) = make_double2(a, b);
          }
    }
    fence_proxy_async();  // generic-proxy writes -> visible to the bulk store
    __syncwarp();
    if (lane == 0) {
#pragma unroll
      for (int cc = 0; cc < 4; ++cc) tma_store_2d(&ymap, st + cc * 2048, cc * 16, static_cast<int>(tile * TILE));
      bulk_commit();
      const long long nt2 = tile + 2 * total;
      if (nt2 < ntiles) {
        bulk_wait_read<1>();  // tile i-1's store has left stage (i+2) % 3
        issue(static_cast<int>((i + 2) % STAGES), nt2);
      }
    }
    __syncwarp();
  }
  if (lane == 0) bulk_wait_all();
}

// ---------------------------------------------------------------------------
// k_coef16_sym: filter_coeffs at N = 16 for parity-block-diagonal operators:
// per class Y_c = H_c X_c (64 x 64), 64 DMMA per block instead of 256.
// CTA = C16S_WARPS warps, warp w owns class w & 3 (pu, pv) and a slice of
// NPW output n-tiles; the four 64 x 64 H_c (128 KB of DMMA B fragments) stay
// resident in shared memory.
// Work unit: a tile of 16 blocks (32 KB), TMA-loaded as 16 boxes [16 blocks
// x 16 coefficients] (box u = row u of every block, 128B swizzle) into a
// 3-stage ring; each warp contracts its class for both 8-block m-tiles
// (each B fragment feeds 4 DMMAs), the CTA syncs, the warps write Y back
// into the same stage in the same layout, and one thread TMA-stores it.
// Class k-step s <-> (u' = s >> 1, v' = 2t + (s & 1)): box 2u' + pu, chunk
// v', element pv.
namespace c16s {
#ifndef C16S_WARPS
#define C16S_WARPS 8
#endif
constexpr int WARPS = C16S_WARPS;
constexpr int NPW = 32 / WARPS;  // n-tiles per warp
constexpr int STAGES = 3;
constexpr int TILE = 16;
constexpr int STAGE_BYTES = TILE * 256 * 8;  // 32 KB
constexpr int HBYTES = 4 * 8 * 8 * 32 * 16;   // 128 KB
constexpr int SMEM = 1024 + HBYTES + STAGES * STAGE_BYTES;
}  // namespace c16s

__global__ void __launch_bounds__(c16s::WARPS * 32, 1)
    k_coef16_sym(const __grid_constant__ CUtensorMap xmap, const __grid_constant__ CUtensorMap ymap,
                 const double* __restrict__ hc, long long nblocks) {
  using namespace c16s;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* base = align1024(smem_raw);
  const double2* hs = reinterpret_cast<const double2*>(base);
  uint8_t* stages = base + HBYTES;
  __shared__ uint64_t full[STAGES];

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  const int cls = warp & 3, pu = cls >> 1, pv = cls & 1, nh = warp >> 2;  // n-tile slice
  if (threadIdx.x == 0) {
    prefetch_tmap(&xmap);
    prefetch_tmap(&ymap);
    for (int i = 0; i < STAGES; ++i) mbar_init(&full[i], 1);
    fence_barrier_init();
  }
  pdl_trigger();
  cta_copy_async(base, hc, HBYTES);  // plan-owned operator
  pdl_wait();
  cp_async_wait_all();
  __syncthreads();

  const long long ntiles = (nblocks + TILE - 1) / TILE;
  auto issue = [&](int s, long long tile) {
    uint8_t* dst = stages + s * STAGE_BYTES;
    mbar_expect_tx(&full[s], STAGE_BYTES);
#pragma unroll 1
    for (int cc = 0; cc < 16; ++cc)
      tma_load_2d(dst + cc * 2048, &xmap, &full[s], cc * 16, static_cast<int>(tile * TILE));
  };
  if (threadIdx.x == 0) {
    if (blockIdx.x < ntiles) issue(0, blockIdx.x);
    if (blockIdx.x + gridDim.x < ntiles) issue(1, blockIdx.x + gridDim.x);
  }
  const double2* hw = hs + cls * (8 * 8 * 32) + nh * (NPW * 8 * 32);

  long long i = 0;
  for (long long tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++i) {
    const int s = static_cast<int>(i % STAGES);
    mbar_wait(&full[s], static_cast<uint32_t>((i / STAGES) & 1));
    uint8_t* st = stages + s * STAGE_BYTES;

    double2 acc[2][NPW];
#pragma unroll
    for (int mt = 0; mt < 2; ++mt)
#pragma unroll
      for (int nt = 0; nt < NPW; ++nt) acc[mt][nt] = make_double2(0.0, 0.0);
#pragma unroll 2
    for (int sp = 0; sp < 8; ++sp) {
      // A: block rows g and 8 + g, k-steps 2sp, 2sp+1 -> (u' = sp, v' = 2t + e)
      const uint8_t* bx = st + (2 * sp + pu) * 2048 + 8 * pv;
      double a[2][2];
#pragma unroll
      for (int mt = 0; mt < 2; ++mt)
#pragma unroll
        for (int e = 0; e < 2; ++e)
          a[mt][e] = *reinterpret_cast<const double*>(bx + (8 * mt + g) * 128 + (((2 * t + e) ^ g) << 4));
#pragma unroll
      for (int nt = 0; nt < NPW; ++nt) {
        const double2 bb = hw[(nt * 8 + sp) * 32 + lane];
        dmma(acc[0][nt], a[0][0], bb.x);
        dmma(acc[1][nt], a[1][0], bb.x);
        dmma(acc[0][nt], a[0][1], bb.y);
        dmma(acc[1][nt], a[1][1], bb.y);
      }
    }
    __syncthreads();  // all four classes have read the stage
    // Y_c[o = 8nt + 2t + e] = coefficient (2nt + pu, 2(2t + e) + pv): box 2nt + pu, chunk 2t + e
#pragma unroll
    for (int mt = 0; mt < 2; ++mt) {
      uint8_t* rb = st + (8 * mt + g) * 128 + 8 * pv;
#pragma unroll
      for (int nt = 0; nt < NPW; ++nt)
#pragma unroll
        for (int e = 0; e < 2; ++e)
          *reinterpret_cast<double*>(rb + (2 * (NPW * nh + nt) + pu) * 2048 + (((2 * t + e) ^ g) << 4)) =
              e ? acc[mt][nt].y : acc[mt][nt].x;
    }
    fence_proxy_async();
    __syncthreads();
    if (threadIdx.x == 0) {
#pragma unroll 1
      for (int cc = 0; cc < 16; ++cc) tma_store_2d(&ymap, st + cc * 2048, cc * 16, static_cast<int>(tile * TILE));
      bulk_commit();
      const long long nt2 = tile + 2 * static_cast<long long>(gridDim.x);
      if (nt2 < ntiles) {
        bulk_wait_read<1>();  // the store that last used stage (i+2) % 3 has read it
        issue(static_cast<int>((i + 2) % STAGES), nt2);
      }
    }
  }
  if (threadIdx.x == 0) bulk_wait_all();
}

// ---------------------------------------------------------------------------
// k_coef16: Y^T (blocks x 256) = X^T (blocks x 256) * H^T, FP64 DMMA.
//
// CTA tile: 64 blocks x 256 outputs; K = 256 streamed in 16 chunks of 16.
// Per chunk one TMA box [64 blocks x 16 coeffs] (8 KB, 128B swizzle) plus one
// 32 KB bulk copy of the H^T chunk (fragment order, layout_hcoef) land in a
// 3-stage ring (full/empty mbarriers); lane 0 of warp 0 refills a stage as
// soon as all 16 warps released it. Warp w covers blocks 16(w&3)..+16
// (2 m-tiles) and outputs 64(w>>2)..+64 (8 n-tiles).
namespace c16 {
constexpr int CWARPS = 16;
constexpr int STAGES = 3;
constexpr int TILE = 64;
constexpr int XBYTES = TILE * 16 * 8;   // 8 KB
constexpr int HBYTES = 256 * 16 * 8;    // 32 KB
constexpr int STAGE_BYTES = XBYTES + HBYTES;
constexpr int SMEM = 1024 + STAGES * STAGE_BYTES;
}  // namespace c16

__global__ void __launch_bounds__(c16::CWARPS * 32, 1)
    k_coef16(const __grid_constant__ CUtensorMap xmap, const double* __restrict__ hc,
             double* __restrict__ out, long long nblocks) {
  using namespace c16;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* base = align1024(smem_raw);
  __shared__ uint64_t full[STAGES], empty[STAGES];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    prefetch_tmap(&xmap);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], CWARPS);
    }
    fence_barrier_init();
  }
  __syncthreads();
  const long long ntiles = (nblocks + TILE - 1) / TILE;
  // chunk c of this CTA: tile blockIdx.x + (c / 16) * gridDim.x, K-chunk c % 16
  const long long nchunks = ntiles > blockIdx.x ? ((ntiles - 1 - blockIdx.x) / gridDim.x + 1) * 16 : 0;
  auto refill = [&](long long c) {
    const int s = static_cast<int>(c % STAGES);
    const int kc = static_cast<int>(c % 16);
    const long long tile = blockIdx.x + (c / 16) * gridDim.x;
    uint8_t* dst = base + s * STAGE_BYTES;
    mbar_expect_tx(&full[s], STAGE_BYTES);
    tma_load_2d(dst, &xmap, &full[s], kc * 16, static_cast<int>(tile * TILE));
    bulk_load(dst + XBYTES, hc + static_cast<size_t>(kc) * (HBYTES / 8), HBYTES, &full[s]);
  };
  pdl_trigger();
  pdl_wait();
  if (warp == 0 && lane == 0)
    for (long long c = 0; c < STAGES && c < nchunks; ++c) refill(c);

  const int g = lane >> 2, t = lane & 3, mg = warp & 3, ng = warp >> 2;
  long long it = 0;
  for (long long tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    double2 acc[2][8];
#pragma unroll
    for (int m = 0; m < 2; ++m)
#pragma unroll
      for (int j = 0; j < 8; ++j) acc[m][j] = make_double2(0.0, 0.0);
    for (int kc = 0; kc < 16; ++kc, ++it) {
      const int s = static_cast<int>(it % STAGES);
      mbar_wait(&full[s], static_cast<uint32_t>((it / STAGES) & 1));
      const uint8_t* xs = base + s * STAGE_BYTES;
      const double2* hs = reinterpret_cast<const double2*>(xs + XBYTES);
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        const int sw = ((2 * t + q) ^ g) << 4;
        const double2 a0 = *reinterpret_cast<const double2*>(xs + (16 * mg + g) * 128 + sw);
        const double2 a1 = *reinterpret_cast<const double2*>(xs + (16 * mg + 8 + g) * 128 + sw);
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const double2 b = hs[((8 * ng + j) * 2 + q) * 32 + lane];
          dmma(acc[0][j], a0.x, b.x);
          dmma(acc[1][j], a1.x, b.x);
          dmma(acc[0][j], a0.y, b.y);
          dmma(acc[1][j], a1.y, b.y);
        }
      }
      // Release the stage only after this warp's shared loads have landed:
      // SYNCS.ARRIVE does not wait for in-flight LDS (observed: the refill
      // overwrote n-tile 7's fragment), MEMBAR.CTA drains them.
      __syncwarp();
      __threadfence_block();
      if (lane == 0) mbar_arrive(&empty[s]);
      if (warp == 0 && lane == 0 && it + STAGES < nchunks) {
        mbar_wait(&empty[s], static_cast<uint32_t>((it / STAGES) & 1));
        refill(it + STAGES);
      }
      __syncwarp();
    }
#pragma unroll
    for (int m = 0; m < 2; ++m) {
      const long long blk = tile * TILE + 16 * mg + 8 * m + g;
      if (blk < nblocks) {
        double* dst = out + blk * 256 + 64 * ng + 2 * t;
#pragma unroll
        for (int j = 0; j < 8; ++j) *reinterpret_cast<double2*>(dst + 8 * j) = acc[m][j];
      }
    }
  }
}

dctf_status launch_coef8_sym(const dctf_plan* p, const double* d_in, double* d_out, long long nb,
                             cudaStream_t st) {
  CUtensorMap xmap, ymap;
  dctf_status s = dctf::make_xmap(&xmap, d_in, nb, 64, c8s::TILE);
  if (s == DCTF_OK) s = dctf::make_xmap(&ymap, d_out, nb, 64, c8s::TILE);
  if (s != DCTF_OK) return s;
  s = dctf::ensure_dyn_smem(reinterpret_cast<const void*>(k_coef8_sym), c8s::SMEM, "k_coef8_sym");
  if (s != DCTF_OK) return s;
  const long long ntiles = (nb + c8s::TILE - 1) / c8s::TILE;
  const long long ctas = std::min<long long>(sm_count(p->device), (ntiles + c8s::WARPS - 1) / c8s::WARPS);
  CUDA_TRY(dctf::launch_pdl(k_coef8_sym, static_cast<unsigned>(ctas), c8s::WARPS * 32, c8s::SMEM, st, xmap, ymap,
                            static_cast<const double*>(p->d_hcsym), nb));
  dctf::add_launches(1);
  return DCTF_OK;
}

dctf_status launch_coef16_sym(const dctf_plan* p, const double* d_in, double* d_out, long long nb,
                              cudaStream_t st) {
  CUtensorMap xmap, ymap;
  dctf_status s = dctf::make_xmap(&xmap, d_in, nb, 256, c16s::TILE);
  if (s == DCTF_OK) s = dctf::make_xmap(&ymap, d_out, nb, 256, c16s::TILE);
  if (s != DCTF_OK) return s;
  s = dctf::ensure_dyn_smem(reinterpret_cast<const void*>(k_coef16_sym), c16s::SMEM, "k_coef16_sym");
  if (s != DCTF_OK) return s;
  const long long ntiles = (nb + c16s::TILE - 1) / c16s::TILE;
  const long long ctas = std::min<long long>(sm_count(p->device), ntiles);
  CUDA_TRY(dctf::launch_pdl(k_coef16_sym, static_cast<unsigned>(ctas), c16s::WARPS * 32, c16s::SMEM, st, xmap, ymap,
                            static_cast<const double*>(p->d_hcsym), nb));
  dctf::add_launches(1);
  return DCTF_OK;
}

}  // namespace

namespace dctf {

// ---------------------------------------------------------------------------
// k_coef16_sep: filter_coeffs (filter.hpp:65-67) at n = 16 for masks that are
// symmetric in both axes and a sum of P <= 2 separable terms (layout_csep16):
// the paper's sandwich form Y = sum_p L_p X R_p^T with the fewest pairs, per
// parity class Y_c = sum_p L_p,pu X_c R_p,pv^T with 8x8 factors — 4 DMMA per
// class and pair (16 per block for P = 1, against 64 in k_coef16_sym), so the
// kernel is HBM-bound. Chain per class: U = L_pu X_c (A = L fragments, B = X_c
// from shared memory: lane (g,t) holds X[2(4s+t)+pu][2g+pv]), then Y_c = U R^T
// (A = U's D fragment, k = 2t + s; B = R fragments); the (pu, 0) and (pu, 1)
// classes share each 16-byte load and store.
// Stage = 16 blocks as ONE TMA box of 256 rows (block, u) x 16 coefficients
// (v) with 128B swizzle (chunk v>>1 at position (v>>1) ^ (row & 7)): the
// loads above hit 8 distinct chunks per quarter-warp. A 6-stage ring; the
// filtered tile goes back through the same stage and a TMA store.
namespace c16p {
constexpr int WARPS = 8;
constexpr int TILE = 16;
constexpr int STAGE_BYTES = TILE * 256 * 8;  // 32 KB
constexpr int STAGES = 6;
constexpr int SMEM = 1024 + STAGES * STAGE_BYTES;
}  // namespace c16p

template <int P>
__global__ void __launch_bounds__(c16p::WARPS * 32, 1)
    k_coef16_sep(const __grid_constant__ CUtensorMap xmap, const __grid_constant__ CUtensorMap ymap,
                 const double* __restrict__ frag, long long nblocks) {
  using namespace c16p;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* stages = align1024(smem_raw);
  __shared__ uint64_t full[STAGES];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  double fl[P][2][2], fr[P][2][2];  // [pair][parity][k-step]
#pragma unroll
  for (int q = 0; q < P; ++q)
#pragma unroll
    for (int par = 0; par < 2; ++par)
#pragma unroll
      for (int sk = 0; sk < 2; ++sk) {
        fl[q][par][sk] = frag[(((q * 2 + 0) * 2 + par) * 2 + sk) * 32 + lane];
        fr[q][par][sk] = frag[(((q * 2 + 1) * 2 + par) * 2 + sk) * 32 + lane];
      }
  if (threadIdx.x == 0) {
    prefetch_tmap(&xmap);
    prefetch_tmap(&ymap);
    for (int i = 0; i < STAGES; ++i) mbar_init(&full[i], 1);
    fence_barrier_init();
  }
  pdl_trigger();
  __syncthreads();
  pdl_wait();

  const long long ntiles = (nblocks + TILE - 1) / TILE;
  auto issue = [&](int s, long long tile) {
    mbar_expect_tx(&full[s], STAGE_BYTES);
    tma_load_2d(stages + s * STAGE_BYTES, &xmap, &full[s], 0, static_cast<int>(tile * TILE * 16));
  };
  if (threadIdx.x == 0)
    for (int k = 0; k < STAGES - 1; ++k) {
      const long long tile = blockIdx.x + static_cast<long long>(k) * gridDim.x;
      if (tile < ntiles) issue(k, tile);
    }

  long long i = 0;
  for (long long tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++i) {
    const int s = static_cast<int>(i % STAGES);
    mbar_wait(&full[s], static_cast<uint32_t>((i / STAGES) & 1));
    uint8_t* st = stages + s * STAGE_BYTES;
#pragma unroll
    for (int bb = 0; bb < TILE / WARPS; ++bb) {
      uint8_t* rb = st + (2 * warp + bb) * 16 * 128;  // the block's 16 rows (u)
      // X[2(4s+t)+pu][2g + {0,1}]: row u = 2(4s+t)+pu, chunk g
      double2 x[2][2];
#pragma unroll
      for (int pu = 0; pu < 2; ++pu)
#pragma unroll
        for (int sk = 0; sk < 2; ++sk) {
          const int u = 2 * (4 * sk + t) + pu;
          x[pu][sk] = *reinterpret_cast<const double2*>(rb + u * 128 + ((g ^ (u & 7)) << 4));
        }
      double2 y[2][2];  // [pu][pv]: Y_c[u' = g][v' = 2t, 2t+1]
#pragma unroll
      for (int pu = 0; pu < 2; ++pu)
#pragma unroll
        for (int pv = 0; pv < 2; ++pv) {
          y[pu][pv] = make_double2(0.0, 0.0);
#pragma unroll
          for (int q = 0; q < P; ++q) {
            double2 uu = make_double2(0.0, 0.0);
            dmma(uu, fl[q][pu][0], pv ? x[pu][0].y : x[pu][0].x);
            dmma(uu, fl[q][pu][1], pv ? x[pu][1].y : x[pu][1].x);
            dmma(y[pu][pv], uu.x, fr[q][pv][0]);
            dmma(y[pu][pv], uu.y, fr[q][pv][1]);
          }
        }
      // Y[2g+pu][2(2t+e) + pv]: row 2g+pu, chunk 2t+e holds pv = 0, 1
#pragma unroll
      for (int pu = 0; pu < 2; ++pu)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int u = 2 * g + pu, c = 2 * t + e;
          *reinterpret_cast<double2*>(rb + u * 128 + ((c ^ (u & 7)) << 4)) =
              e ? make_double2(y[pu][0].y, y[pu][1].y) : make_double2(y[pu][0].x, y[pu][1].x);
        }
    }
    fence_proxy_async();
    __syncthreads();
    if (threadIdx.x == 0) {
      tma_store_2d(&ymap, st, 0, static_cast<int>(tile * TILE * 16));
      bulk_commit();
      const long long nxt = tile + static_cast<long long>(STAGES - 1) * gridDim.x;
      if (nxt < ntiles) {
        bulk_wait_read<1>();  // the store of the previous tile (this stage's successor slot) has read it
        issue(static_cast<int>((i + STAGES - 1) % STAGES), nxt);
      }
    }
  }
  if (threadIdx.x == 0) bulk_wait_all();
}

template <int P>
dctf_status launch_coef16_sep(const dctf_plan* p, const double* d_in, double* d_out, long long nb,
                              cudaStream_t st) {
  CUtensorMap xmap, ymap;
  dctf_status s = dctf::make_xmap(&xmap, d_in, nb * 16, 16, 256);
  if (s == DCTF_OK) s = dctf::make_xmap(&ymap, d_out, nb * 16, 16, 256);
  if (s != DCTF_OK) return s;
  {
    const dctf_status sa = dctf::ensure_dyn_smem(reinterpret_cast<const void*>(k_coef16_sep<P>), c16p::SMEM,
                                                 "k_coef16_sep");
    if (sa != DCTF_OK) return sa;
  }
  const long long ntiles = (nb + c16p::TILE - 1) / c16p::TILE;
  const long long ctas = std::min<long long>(sm_count(p->device), ntiles);
  CUDA_TRY(dctf::launch_pdl(k_coef16_sep<P>, static_cast<unsigned>(ctas), c16p::WARPS * 32, c16p::SMEM, st, xmap,
                            ymap, static_cast<const double*>(p->d_csep), nb));
  dctf::add_launches(1);
  return DCTF_OK;
}

// ---------------------------------------------------------------------------
// k_coef8_sep: filter_coeffs (filter.hpp:65-67) at n = 8 for masks of rank
// P <= 3 without parity structure (layout_csep8; the symmetric ones take the
// HBM-bound k_coef8_sym): the sandwich form Y = sum_p L_p X R_p^T, per block
// and pair U = L_p X (A = L fragments, B = X: lane (g,t) holds X[4s+t][g]),
// Y += U R_p^T (A = U's D fragment with k = 2t + s, B = R fragments):
// 4 DMMA per pair (12 for rank 3 against k_coef8's 16), so HBM-bound up to
// rank 2. Blocks are contiguous 512-byte tiles, so a stage of 32 blocks moves
// with ONE bulk copy each way (cp.async.bulk, no tensor map); the per-lane
// accesses (8-byte loads X[4s+t][g], 16-byte stores of Y[g][2t..2t+1]) are
// conflict-free in that natural layout. 8-stage ring, one CTA per SM.
namespace c8p {
constexpr int WARPS = 8;
constexpr int TILE = 32;                     // blocks per stage
constexpr int STAGE_BYTES = TILE * 64 * 8;   // 16 KB
constexpr int STAGES = 8;
constexpr int SMEM = 1024 + STAGES * STAGE_BYTES;
}  // namespace c8p

template <int P>
__global__ void __launch_bounds__(c8p::WARPS * 32, 1)
    k_coef8_sep(const double* __restrict__ x, double* __restrict__ y, const double* __restrict__ frag,
                long long nblocks) {
  using namespace c8p;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* stages = align1024(smem_raw);
  __shared__ uint64_t full[STAGES];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  double fl[P][2], fr[P][2];
#pragma unroll
  for (int q = 0; q < P; ++q)
#pragma unroll
    for (int sk = 0; sk < 2; ++sk) {
      fl[q][sk] = frag[((q * 2 + 0) * 2 + sk) * 32 + lane];
      fr[q][sk] = frag[((q * 2 + 1) * 2 + sk) * 32 + lane];
    }
  if (threadIdx.x == 0) {
    for (int i = 0; i < STAGES; ++i) mbar_init(&full[i], 1);
    fence_barrier_init();
  }
  pdl_trigger();
  __syncthreads();
  pdl_wait();
  const long long ntiles = (nblocks + TILE - 1) / TILE;
  auto tile_bytes = [&](long long tile) {
    return static_cast<uint32_t>(min(static_cast<long long>(TILE), nblocks - tile * TILE) * 512);
  };
  auto issue = [&](int s, long long tile) {
    const uint32_t bytes = tile_bytes(tile);
    mbar_expect_tx(&full[s], bytes);
    bulk_load(stages + s * STAGE_BYTES, x + tile * TILE * 64, bytes, &full[s]);
  };
  if (threadIdx.x == 0)
    for (int k = 0; k < STAGES - 1; ++k) {
      const long long tile = blockIdx.x + static_cast<long long>(k) * gridDim.x;
      if (tile < ntiles) issue(k, tile);
    }
  long long i = 0;
  for (long long tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++i) {
    const int s = static_cast<int>(i % STAGES);
    mbar_wait(&full[s], static_cast<uint32_t>((i / STAGES) & 1));
    uint8_t* st = stages + s * STAGE_BYTES;
    // warp w: blocks 4w .. 4w + 3 of the stage, in lock step
    double a[4][2];
    double2 acc[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const double* xb = reinterpret_cast<const double*>(st + (4 * warp + k) * 512);
      a[k][0] = xb[t * 8 + g];
      a[k][1] = xb[(4 + t) * 8 + g];
      acc[k] = make_double2(0.0, 0.0);
    }
#pragma unroll
    for (int q = 0; q < P; ++q) {
      double2 uu[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) { uu[k] = make_double2(0.0, 0.0); dmma(uu[k], fl[q][0], a[k][0]); }
#pragma unroll
      for (int k = 0; k < 4; ++k) dmma(uu[k], fl[q][1], a[k][1]);
#pragma unroll
      for (int k = 0; k < 4; ++k) dmma(acc[k], uu[k].x, fr[q][0]);
#pragma unroll
      for (int k = 0; k < 4; ++k) dmma(acc[k], uu[k].y, fr[q][1]);
    }
#pragma unroll
    for (int k = 0; k < 4; ++k)  // Y[g][2t], Y[g][2t+1]: every lane has read this block (mma.sync)
      *reinterpret_cast<double2*>(st + (4 * warp + k) * 512 + g * 64 + 16 * t) = acc[k];
    fence_proxy_async();
    __syncthreads();
    if (threadIdx.x == 0) {
      bulk_store(y + tile * TILE * 64, st, tile_bytes(tile));
      bulk_commit();
      const long long nxt = tile + static_cast<long long>(STAGES - 1) * gridDim.x;
      if (nxt < ntiles) {
        bulk_wait_read<1>();  // the previous tile's store (this slot's last user) has read it
        issue(static_cast<int>((i + STAGES - 1) % STAGES), nxt);
      }
    }
  }
  if (threadIdx.x == 0) bulk_wait_all();
}

template <int P>
dctf_status launch_coef8_sep(const dctf_plan* p, const double* d_in, double* d_out, long long nb, cudaStream_t st) {
  {
    const dctf_status sa = dctf::ensure_dyn_smem(reinterpret_cast<const void*>(k_coef8_sep<P>), c8p::SMEM, "k_coef8_sep");
    if (sa != DCTF_OK) return sa;
  }
  const long long ntiles = (nb + c8p::TILE - 1) / c8p::TILE;
  const long long ctas = std::min<long long>(sm_count(p->device), ntiles);
  CUDA_TRY(dctf::launch_pdl(k_coef8_sep<P>, static_cast<unsigned>(ctas), c8p::WARPS * 32, c8p::SMEM, st, d_in, d_out,
                            static_cast<const double*>(p->d_csep), nb));
  dctf::add_launches(1);
  return DCTF_OK;
}

dctf_status launch_coef(const dctf_plan* p, const double* d_in, double* d_out, long long nb,
                        cudaStream_t st) {
  if (nb == 0) return DCTF_OK;
  if (misaligned16(d_in) || misaligned16(d_out))
    return set_error(DCTF_INVALID_ARGUMENT, "coefficient buffers must be 16-byte aligned");
  if (d_in == d_out) return set_error(DCTF_INVALID_ARGUMENT, "in-place filter_coeffs not supported");
  if (p->precision == DCTF_PREC_TF32X3 || p->precision == DCTF_PREC_BF16X3) return dctf::launch_coef_tf32x3(p, d_in, d_out, nb, st, sm_count(p->device));
  if (p->n == 8 && p->csep_rank > 0) {
    if (p->csep_rank == 1) return launch_coef8_sep<1>(p, d_in, d_out, nb, st);
    if (p->csep_rank == 2) return launch_coef8_sep<2>(p, d_in, d_out, nb, st);
    return launch_coef8_sep<3>(p, d_in, d_out, nb, st);
  }
  if (p->n == 16 && p->csep_rank > 0)
    return p->csep_rank == 1 ? launch_coef16_sep<1>(p, d_in, d_out, nb, st) : launch_coef16_sep<2>(p, d_in, d_out, nb, st);
  if (p->sym) return p->n == 8 ? launch_coef8_sym(p, d_in, d_out, nb, st) : launch_coef16_sym(p, d_in, d_out, nb, st);
  CUtensorMap map;
  const int nn = p->n * p->n;
  dctf_status s = dctf::make_xmap(&map, d_in, nb, nn, p->n == 8 ? c8::TILE : c16::TILE);
  if (s != DCTF_OK) return s;
  const int sms = sm_count(p->device);
  if (p->n == 8) {
    {
      const dctf_status sa = dctf::ensure_dyn_smem(reinterpret_cast<const void*>(k_coef8), c8::SMEM, "k_coef8");
      if (sa != DCTF_OK) return sa;
    }
    const long long ntiles = (nb + c8::TILE - 1) / c8::TILE;
    const long long ctas = std::min<long long>(sms, (ntiles + c8::WARPS - 1) / c8::WARPS);
    CUDA_TRY(dctf::launch_pdl(k_coef8, static_cast<unsigned>(ctas), c8::WARPS * 32, c8::SMEM, st, map,
                              static_cast<const double*>(p->d_hcoef), d_out, nb));
  } else {
    {
      const dctf_status sa = dctf::ensure_dyn_smem(reinterpret_cast<const void*>(k_coef16), c16::SMEM, "k_coef16");
      if (sa != DCTF_OK) return sa;
    }
    const long long ntiles = (nb + c16::TILE - 1) / c16::TILE;
    const long long ctas = std::min<long long>(sms, ntiles);
    CUDA_TRY(dctf::launch_pdl(k_coef16, static_cast<unsigned>(ctas), c16::CWARPS * 32, c16::SMEM, st, map,
                              static_cast<const double*>(p->d_hcoef), d_out, nb));
  }
  dctf::add_launches(1);
  CUDA_TRY(cudaGetLastError());
  return DCTF_OK;
}

}  // namespace dctf
