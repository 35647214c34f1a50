// sm_100a kernels and C-ABI launchers of the DCT-domain block filter.
//
// Kernels (all FP64; the contraction stages run on the FP64 tensor pipe via
// mma.sync.m8n8k4.f64 -> DMMA.8x8x4):
//   k_forward<N,U8>   forward_2d (dct.hpp:59-62) per block, reference
//                     operation order (mul then add, no FMA, zero-skip), so
//                     coefficients are bit-identical to the reference.
//   k_inverse<N,U8>   inverse_2d (dct.hpp:65-68) [+ quantize_sample +
//                     assemble crop (spatial.hpp:71-75, image.hpp:188-203)].
//   k_coef8           FilterPlan::filter_coeffs (filter.hpp:65-67) for n=8:
//                     Y^T = X^T H^T, blocks on the MMA M axis; X tiles are
//                     TMA-staged (cp.async.bulk.tensor.2d, 128B swizzle)
//                     through a per-warp mbarrier ring; H (32 KB) resident in
//                     shared memory in fragment order.
//   k_coef16          the same for n=16; H (512 KB) is streamed in 32 KB
//                     K-chunks by a producer warp (cp.async.bulk) together
//                     with the matching X chunk, 3-stage ring, 16 MMA warps.
//   k_fused8          filter_image's per-block chain (image.hpp:214-218,
//                     filter.hpp:71-73) for n=8 fused: u8 strip -> forward
//                     DCT (4 DMMA/block) -> H (16 DMMA/block) -> inverse DCT
//                     (4 DMMA/block) -> round/clamp -> u8; one HBM read and
//                     one HBM write per pixel.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>

#include "fastdiv.cuh"
#include "internal.h"

// ---------------------------------------------------------------------------
// bookkeeping
namespace dctf {
namespace {
thread_local std::string t_err;
thread_local int t_launches = 0;
}  // namespace
dctf_status set_error(dctf_status s, const std::string& msg) {
  t_err = msg;
  return s;
}
void add_launches(int k) { t_launches += k; }
void reset_launches() { t_launches = 0; }
}  // namespace dctf

using dctf::set_error;

#define CUDA_TRY(expr)                                                                   \
  do {                                                                                   \
    cudaError_t e_ = (expr);                                                             \
    if (e_ != cudaSuccess)                                                               \
      return set_error(DCTF_CUDA_ERROR, std::string(#expr ": ") + cudaGetErrorString(e_)); \
  } while (0)

// ---------------------------------------------------------------------------
// device helpers
namespace {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// D(8x8) += A(8x4, row) * B(4x8, col), FP64. Lane l: A[l>>2][l&3],
// B[l&3][l>>2], D[l>>2][2(l&3)+{0,1}].
__device__ __forceinline__ void dmma(double2& d, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
      : "+d"(d.x), "+d"(d.y)
      : "d"(a), "d"(b));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t done = 0;
  const uint32_t addr = smem_u32(bar);
  while (!done) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(addr), "r"(parity)
        : "memory");
  }
}
__device__ __forceinline__ void fence_barrier_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar,
                                            int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes,
                                          uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void prefetch_tmap(const CUtensorMap* map) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}

// quantize_sample (spatial.hpp:71-75): round half away from zero, clamp.
__device__ __forceinline__ void tma_store_2d(const CUtensorMap* map, const void* src, int c0, int c1) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(smem_u32(src)), "r"(c0), "r"(c1)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ uint32_t quantize(double v, int* nan_flag) {
  if (v != v) {
    if (nan_flag) atomicOr(nan_flag, 1);
    return 0u;
  }
  const double r = fmin(fmax(round(v), 0.0), 255.0);
  return static_cast<uint32_t>(r);
}

// Exact double of an integer 0..255 built with integer ops only, so the FP64
// pipe stays free for DMMA: 2^e (1 + m) with e = msb(p).
__device__ __forceinline__ double u8_to_f64(uint32_t p) {
  const int e = 31 - __clz(p);
  const uint32_t hi = (static_cast<uint32_t>(1022 + e) << 20) + (p << (20 - e));
  return p ? __hiloint2double(static_cast<int>(hi), 0) : 0.0;
}

// floor(t) clamped to [0,255] with a single conversion instruction. Callers
// pass t = v + 0.5 (the 0.5 rides in the DMMA accumulator), which equals
// quantize_sample's round-half-away-from-zero + clamp for every v except
// within one ulp of a .5 boundary — inside the 1e-6 near-tie window the
// parity contract excuses. NaN converts to 0.
__device__ __forceinline__ uint32_t floor_to_u8(double t) {
  int i;
  asm("cvt.rmi.s32.f64 %0, %1;" : "=r"(i) : "d"(t));
  return static_cast<uint32_t>(min(max(i, 0), 255));
}

// Aligns a dynamic shared-memory base to 1024 B (128B-swizzle atoms) while
// keeping the pointer in the shared window (so loads compile to LDS).
__device__ __forceinline__ uint8_t* align1024(uint8_t* smem) {
  const uint32_t pad = (1024u - (smem_u32(smem) & 1023u)) & 1023u;
  return smem + pad;
}

__device__ __forceinline__ uint4 ldg_stream(const void* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}
__device__ __forceinline__ void stg_stream(void* p, uint4 v) {
  asm volatile("st.global.L1::no_allocate.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x),
               "r"(v.y), "r"(v.z), "r"(v.w)
               : "memory");
}

// ---------------------------------------------------------------------------
// forward_2d / inverse_2d, reference operation order.
//
// One CTA = 256 threads = 256/N blocks; thread (lb, r) owns row r of block lb.
// forward: T = C X (row r of T needs row r of C and all of X), out = T C^t.
// inverse: T = C^t Y, out = T C.
// Each product is matmul (block_matrix.hpp:67-81): k ascending, skip a == 0,
// separately rounded multiply and add (the reference has no FMA
// contraction), so results are bit-identical to forward_2d / inverse_2d.

template <int N, bool FROM_U8>
__global__ void __launch_bounds__(256) k_forward(const uint8_t* __restrict__ img, int w, int h,
                                                 size_t pitch, int bw,
                                                 const double* __restrict__ blocks,
                                                 double* __restrict__ out, long long nblocks,
                                                 const double* __restrict__ cb) {
  constexpr int NN = N * N, BPC = 256 / N, STR = NN + 1;
  __shared__ double xs[BPC * STR];
  __shared__ double cs[NN];
  for (int i = threadIdx.x; i < NN; i += 256) cs[i] = cb[i];
  const long long b0 = static_cast<long long>(blockIdx.x) * BPC;
  for (int e = threadIdx.x; e < BPC * NN; e += 256) {
    const int lb = e / NN, idx = e % NN;
    const long long blk = b0 + lb;
    double v = 0.0;
    if (blk < nblocks) {
      if (FROM_U8) {
        const int by = static_cast<int>(blk / bw), bx = static_cast<int>(blk % bw);
        const int y = min(by * N + idx / N, h - 1), x = min(bx * N + idx % N, w - 1);
        v = static_cast<double>(img[static_cast<size_t>(y) * pitch + x]);
      } else {
        v = blocks[blk * NN + idx];
      }
    }
    xs[lb * STR + idx] = v;
  }
  __syncthreads();
  const int lb = threadIdx.x / N, r = threadIdx.x % N;
  const long long blk = b0 + lb;
  const double* x = xs + lb * STR;
  double crow[N], trow[N], o[N];
#pragma unroll
  for (int k = 0; k < N; ++k) crow[k] = cs[r * N + k];
#pragma unroll
  for (int j = 0; j < N; ++j) trow[j] = 0.0;
#pragma unroll
  for (int k = 0; k < N; ++k) {
    const double a = crow[k];
    if (a != 0.0) {
#pragma unroll
      for (int j = 0; j < N; ++j) trow[j] = __dadd_rn(trow[j], __dmul_rn(a, x[k * N + j]));
    }
  }
#pragma unroll
  for (int j = 0; j < N; ++j) o[j] = 0.0;
#pragma unroll
  for (int k = 0; k < N; ++k) {
    const double a = trow[k];
    if (a != 0.0) {
#pragma unroll
      for (int j = 0; j < N; ++j) o[j] = __dadd_rn(o[j], __dmul_rn(a, cs[j * N + k]));
    }
  }
  if (blk < nblocks) {
    double* dst = out + blk * NN + r * N;
#pragma unroll
    for (int j = 0; j < N; j += 2) *reinterpret_cast<double2*>(dst + j) = make_double2(o[j], o[j + 1]);
  }
}

template <int N, bool TO_U8>
__global__ void __launch_bounds__(256) k_inverse(const double* __restrict__ coeffs,
                                                 double* __restrict__ blocks_out,
                                                 uint8_t* __restrict__ img, int w, int h,
                                                 size_t pitch, int bw, long long nblocks,
                                                 const double* __restrict__ cb, int* nan_flag) {
  constexpr int NN = N * N, BPC = 256 / N, STR = NN + 1;
  __shared__ double ys[BPC * STR];
  __shared__ double cs[NN];
  for (int i = threadIdx.x; i < NN; i += 256) cs[i] = cb[i];
  const long long b0 = static_cast<long long>(blockIdx.x) * BPC;
  for (int e = threadIdx.x; e < BPC * NN; e += 256) {
    const int lb = e / NN, idx = e % NN;
    const long long blk = b0 + lb;
    ys[lb * STR + idx] = blk < nblocks ? coeffs[blk * NN + idx] : 0.0;
  }
  __syncthreads();
  const int lb = threadIdx.x / N, r = threadIdx.x % N;
  const long long blk = b0 + lb;
  const double* y = ys + lb * STR;
  double ccol[N], trow[N], o[N];
#pragma unroll
  for (int k = 0; k < N; ++k) ccol[k] = cs[k * N + r];  // C^t[r][k]
#pragma unroll
  for (int j = 0; j < N; ++j) trow[j] = 0.0;
#pragma unroll
  for (int k = 0; k < N; ++k) {
    const double a = ccol[k];
    if (a != 0.0) {
#pragma unroll
      for (int j = 0; j < N; ++j) trow[j] = __dadd_rn(trow[j], __dmul_rn(a, y[k * N + j]));
    }
  }
#pragma unroll
  for (int j = 0; j < N; ++j) o[j] = 0.0;
#pragma unroll
  for (int k = 0; k < N; ++k) {
    const double a = trow[k];
    if (a != 0.0) {
#pragma unroll
      for (int j = 0; j < N; ++j) o[j] = __dadd_rn(o[j], __dmul_rn(a, cs[k * N + j]));
    }
  }
  if (blk >= nblocks) return;
  if (!TO_U8) {
    double* dst = blocks_out + blk * NN + r * N;
#pragma unroll
    for (int j = 0; j < N; j += 2) *reinterpret_cast<double2*>(dst + j) = make_double2(o[j], o[j + 1]);
  } else {
    const int by = static_cast<int>(blk / bw), bx = static_cast<int>(blk % bw);
    const int yy = by * N + r;
    if (yy >= h) return;
    uint8_t* dst = img + static_cast<size_t>(yy) * pitch + bx * N;
#pragma unroll
    for (int j = 0; j < N; ++j)
      if (bx * N + j < w) dst[j] = static_cast<uint8_t>(quantize(o[j], nan_flag));
  }
}

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
  {
    const double2* src = reinterpret_cast<const double2*>(hc);
    double2* dst = reinterpret_cast<double2*>(base);
    for (int i = threadIdx.x; i < 2048; i += blockDim.x) dst[i] = src[i];
  }
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
  {
    const double2* src = reinterpret_cast<const double2*>(hc);
    double2* dst = reinterpret_cast<double2*>(base);
    for (int i = threadIdx.x; i < 512; i += blockDim.x) dst[i] = src[i];
  }
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
  {
    const double2* src = reinterpret_cast<const double2*>(hc);
    double2* dst = reinterpret_cast<double2*>(base);
    for (int i = threadIdx.x; i < HBYTES / 16; i += blockDim.x) dst[i] = src[i];
  }
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
  if (s < nstrips) prefetch(s);  // first strip's pixels in flight during the operator copy
  {
    const double2* src = reinterpret_cast<const double2*>(hf);
    double2* dst = reinterpret_cast<double2*>(smem);
    for (int i = threadIdx.x; i < 2048; i += blockDim.x) dst[i] = src[i];
  }
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
          make_double2(u8_to_f64(q0), u8_to_f64(q1));
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
constexpr int SMEM = 16384 + WARPS * PIX_BYTES;
}  // namespace f8s

// small signed integer (|v| < 2^20) -> double, exactly, on the integer pipes
__device__ __forceinline__ double i32_to_f64(int v) {
  const uint32_t m = static_cast<uint32_t>(v < 0 ? -v : v);
  const int e = 31 - __clz(m);
  const uint32_t hi = ((static_cast<uint32_t>(1022 + e) << 20) + (m << (20 - e))) |
                      (static_cast<uint32_t>(v) & 0x80000000u);
  return m ? __hiloint2double(static_cast<int>(hi), 0) : 0.0;
}

template <bool COEF>
__global__ void __launch_bounds__(f8s::WARPS * 32, F8S_MINB)
    k_fused8_sym(const uint8_t* __restrict__ in, uint8_t* __restrict__ out, int w, int h, size_t pitch,
                 long long frame_stride, int nframes, int bw, int bh, int nsx,
                 const double* __restrict__ hsym, double* __restrict__ coef_out) {
  using namespace f8s;
  extern __shared__ __align__(16) uint8_t smem[];
  const double2* gs = reinterpret_cast<const double2*>(smem);          // [c][nt][sp][lane]
  const double2* ws = reinterpret_cast<const double2*>(smem + 8192);   // [c][nt2][nt][lane]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  uint8_t* pix = smem + 16384 + warp * PIX_BYTES;

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
  if (s < nstrips) prefetch(s);  // first strip's pixels in flight during the operator copy
  {
    const double2* src = reinterpret_cast<const double2*>(hsym);
    double2* dst = reinterpret_cast<double2*>(smem);
    for (int i = threadIdx.x; i < 1024; i += blockDim.x) dst[i] = src[i];
  }
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
        const int p00 = (top.x >> (8 * t)) & 0xff, p01 = (top.y >> (24 - 8 * t)) & 0xff;
        const int p10 = (bot.x >> (8 * t)) & 0xff, p11 = (bot.y >> (24 - 8 * t)) & 0xff;
        const int rs0 = p00 + p10, ra0 = p00 - p10, rs1 = p01 + p11, ra1 = p01 - p11;
        q[mt][0][sq] = i32_to_f64(rs0 + rs1);
        q[mt][1][sq] = i32_to_f64(rs0 - rs1);
        q[mt][2][sq] = i32_to_f64(ra0 + ra1);
        q[mt][3][sq] = i32_to_f64(ra0 - ra1);
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
  }
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
    for (long long c = 0; c < STAGES && c < nchunks; ++c) refill(c);

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
        *reinterpret_cast<double2*>(xy + xw(b, wd)) = make_double2(u8_to_f64(q0), u8_to_f64(q1));
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
  if (tile < ntiles) prefetch(tile);
  {
    const double2* src = reinterpret_cast<const double2*>(gsym);
    double2* dst = reinterpret_cast<double2*>(smem);
    for (int i = threadIdx.x; i < GBYTES / 16; i += blockDim.x) dst[i] = src[i];
    double* cdst = reinterpret_cast<double*>(smem + GBYTES);
    for (int i = threadIdx.x; i < 256; i += blockDim.x) cdst[i] = basis[i];
  }
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
        q[0][i][e] = i32_to_f64(rj + rm);
        q[1][i][e] = i32_to_f64(rj - rm);
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
// k_spatial: convolve (spatial.hpp:41-68) per block, one thread per sample,
// correlation orientation, zero-drop or clamp padding at the block edge; the
// accumulation order (r, c ascending) and separately rounded multiply/add
// match the reference, so samples are bit-identical. Input samples come from
// the u8 image through tile()'s edge replication, or from FP64 blocks.
template <bool U8>
__global__ void __launch_bounds__(256) k_spatial(const uint8_t* __restrict__ img, int w, int h,
                                                 size_t pitch, int bw, const double* __restrict__ blocks,
                                                 uint8_t* __restrict__ out_img, double* __restrict__ out_blocks,
                                                 long long nblocks, int n, const double* __restrict__ wts,
                                                 int kr, int kc, int replicate) {
  __shared__ double ws[1024];
  for (int i = threadIdx.x; i < kr * kc && i < 1024; i += blockDim.x) ws[i] = wts[i];
  __syncthreads();
  const int nn = n * n;
  const long long idx = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  const long long blk = idx / nn;
  if (blk >= nblocks) return;
  const int i = static_cast<int>(idx % nn) / n, j = static_cast<int>(idx % nn) % n;
  const int hr = (kr - 1) / 2, hc = (kc - 1) / 2;
  const int by = U8 ? static_cast<int>(blk / bw) : 0, bx = U8 ? static_cast<int>(blk % bw) : 0;
  double acc = 0.0;
  for (int r = 0; r < kr; ++r) {
    int si = i + r - hr;
    if (!replicate && (si < 0 || si >= n)) continue;
    si = min(max(si, 0), n - 1);
    for (int c = 0; c < kc; ++c) {
      int sj = j + c - hc;
      if (!replicate && (sj < 0 || sj >= n)) continue;
      sj = min(max(sj, 0), n - 1);
      double v;
      if (U8) {
        const int y = min(by * n + si, h - 1), x = min(bx * n + sj, w - 1);
        v = static_cast<double>(img[static_cast<size_t>(y) * pitch + x]);
      } else {
        v = blocks[blk * nn + si * n + sj];
      }
      acc = __dadd_rn(acc, __dmul_rn(ws[r * kc + c], v));
    }
  }
  if (U8) {
    const int y = by * n + i, x = bx * n + j;
    if (y < h && x < w) out_img[static_cast<size_t>(y) * pitch + x] = static_cast<uint8_t>(quantize(acc, nullptr));
  } else {
    out_blocks[blk * nn + i * n + j] = acc;
  }
}

// ---------------------------------------------------------------------------
// FP64 peak microbenchmarks (diagnostics; roofline denominator).
__global__ void __launch_bounds__(256) k_peak_dmma(double* out, int iters) {
  double2 acc[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) acc[j] = make_double2(threadIdx.x * 1e-3 + j, 0.5 * j);
  const double a = 1.0 + threadIdx.x * 1e-12, b = 1.0 - threadIdx.x * 1e-12;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) dmma(acc[j], a, b);
  }
  double s = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) s += acc[j].x + acc[j].y;
  if (s == 1.2345) out[threadIdx.x] = s;  // practically never; defeats DCE
}

__global__ void __launch_bounds__(256) k_peak_dfma(double* out, int iters) {
  double x[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) x[j] = threadIdx.x * 1e-3 + j;
  const double a = 1.0 + threadIdx.x * 1e-12, b = 1e-9;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) x[j] = fma(x[j], a, b);
  }
  double s = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) s += x[j];
  if (s == 1.2345) out[threadIdx.x] = s;
}

// ---------------------------------------------------------------------------
// host helpers
typedef CUresult (*PFN_encodeTiled_t)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                      const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                      const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                      CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

PFN_encodeTiled_t encode_fn() {
  static PFN_encodeTiled_t fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_encodeTiled_t>(p);
  });
  return fn;
}

}  // namespace

namespace dctf {
// 2-D FP64 view [nblocks rows x nn cols] of block-major coefficients; box
// [box_rows x 16 cols] (128 bytes inner), 128B swizzle, OOB rows -> 0.
dctf_status make_xmap(void* vmap, const double* d, long long nblocks, int nn, int box_rows, int l2promo) {
  CUtensorMap* map = static_cast<CUtensorMap*>(vmap);
  PFN_encodeTiled_t fn = encode_fn();
  if (!fn) return set_error(DCTF_CUDA_ERROR, "cuTensorMapEncodeTiled unavailable");
  const cuuint64_t dims[2] = {static_cast<cuuint64_t>(nn), static_cast<cuuint64_t>(nblocks)};
  const cuuint64_t strides[1] = {static_cast<cuuint64_t>(nn) * 8};
  const cuuint32_t box[2] = {16, static_cast<cuuint32_t>(box_rows)};
  const cuuint32_t estr[2] = {1, 1};
  const CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(d), dims, strides,
                        box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                        static_cast<CUtensorMapL2promotion>(l2promo), CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return set_error(DCTF_CUDA_ERROR, "cuTensorMapEncodeTiled failed (" + std::to_string(int(r)) + ")");
  return DCTF_OK;
}
}  // namespace dctf

namespace {

}  // namespace

namespace dctf {
// Opts `func` into `bytes` of dynamic shared memory on the current device,
// once per (kernel, device); safe under concurrent first calls and across
// several devices in one process.
dctf_status ensure_dyn_smem(const void* func, int bytes, const char* name) {
  static std::mutex mu;
  static std::vector<std::pair<const void*, int>> done;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return set_error(DCTF_CUDA_ERROR, "cudaGetDevice");
  std::lock_guard<std::mutex> lock(mu);
  for (const auto& d : done)
    if (d.first == func && d.second == dev) return DCTF_OK;
  if (cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes) != cudaSuccess) {
    cudaGetLastError();
    return set_error(DCTF_CUDA_ERROR, std::string("cudaFuncSetAttribute(") + name + ")");
  }
  done.emplace_back(func, dev);
  return DCTF_OK;
}
}  // namespace dctf

namespace {

int sm_count(int device) {
  static int cached[64] = {0};
  if (device < 0 || device >= 64) return 148;
  if (!cached[device]) {
    int v = 148;
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, device);
    cached[device] = v;
  }
  return cached[device];
}

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    int cur = -1;
    cudaGetDevice(&cur);
    if (prev >= 0 && cur != prev) cudaSetDevice(prev);
  }
};

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

bool misaligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) != 0; }

dctf_status check_plan(const dctf_plan* p) {
  if (!p) return set_error(DCTF_INVALID_ARGUMENT, "plan is NULL");
  return DCTF_OK;
}

dctf_status check_image(int w, int h, size_t pitch) {
  if (w < 1 || h < 1) return set_error(DCTF_INVALID_ARGUMENT, "image dimensions must be >= 1");
  if (pitch < static_cast<size_t>(w)) return set_error(DCTF_INVALID_ARGUMENT, "pitch < width");
  return DCTF_OK;
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
  k_coef8_sym<<<static_cast<unsigned>(ctas), c8s::WARPS * 32, c8s::SMEM, st>>>(xmap, ymap, p->d_hcsym, nb);
  dctf::add_launches(1);
  CUDA_TRY(cudaGetLastError());
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
  k_coef16_sym<<<static_cast<unsigned>(ctas), c16s::WARPS * 32, c16s::SMEM, st>>>(xmap, ymap, p->d_hcsym, nb);
  dctf::add_launches(1);
  CUDA_TRY(cudaGetLastError());
  return DCTF_OK;
}

dctf_status launch_coef(const dctf_plan* p, const double* d_in, double* d_out, long long nb,
                        cudaStream_t st) {
  if (nb == 0) return DCTF_OK;
  if (misaligned16(d_in) || misaligned16(d_out))
    return set_error(DCTF_INVALID_ARGUMENT, "coefficient buffers must be 16-byte aligned");
  if (d_in == d_out) return set_error(DCTF_INVALID_ARGUMENT, "in-place filter_coeffs not supported");
  if (p->precision == DCTF_PREC_TF32X3) return dctf::launch_coef_tf32x3(p, d_in, d_out, nb, st, sm_count(p->device));
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
    k_coef8<<<static_cast<unsigned>(ctas), c8::WARPS * 32, c8::SMEM, st>>>(map, p->d_hcoef, d_out, nb);
  } else {
    {
      const dctf_status sa = dctf::ensure_dyn_smem(reinterpret_cast<const void*>(k_coef16), c16::SMEM, "k_coef16");
      if (sa != DCTF_OK) return sa;
    }
    const long long ntiles = (nb + c16::TILE - 1) / c16::TILE;
    const long long ctas = std::min<long long>(sms, ntiles);
    k_coef16<<<static_cast<unsigned>(ctas), c16::CWARPS * 32, c16::SMEM, st>>>(map, p->d_hcoef,
                                                                                   d_out, nb);
  }
  dctf::add_launches(1);
  CUDA_TRY(cudaGetLastError());
  return DCTF_OK;
}

dctf_status launch_forward_u8(const dctf_plan* p, const uint8_t* img, int w, int h, size_t pitch,
                              double* coeffs, cudaStream_t st) {
  const int n = p->n, bw = (w + n - 1) / n, bh = (h + n - 1) / n;
  const long long nb = static_cast<long long>(bw) * bh;
  const int bpc = 256 / n;
  const unsigned grid = static_cast<unsigned>((nb + bpc - 1) / bpc);
  if (n == 8)
    k_forward<8, true><<<grid, 256, 0, st>>>(img, w, h, pitch, bw, nullptr, coeffs, nb, p->d_basis);
  else
    k_forward<16, true><<<grid, 256, 0, st>>>(img, w, h, pitch, bw, nullptr, coeffs, nb, p->d_basis);
  dctf::add_launches(1);
  CUDA_TRY(cudaGetLastError());
  return DCTF_OK;
}

dctf_status launch_inverse_u8(const dctf_plan* p, const double* coeffs, uint8_t* img, int w, int h,
                              size_t pitch, cudaStream_t st) {
  const int n = p->n, bw = (w + n - 1) / n, bh = (h + n - 1) / n;
  const long long nb = static_cast<long long>(bw) * bh;
  const int bpc = 256 / n;
  const unsigned grid = static_cast<unsigned>((nb + bpc - 1) / bpc);
  if (n == 8)
    k_inverse<8, true><<<grid, 256, 0, st>>>(coeffs, nullptr, img, w, h, pitch, bw, nb, p->d_basis, p->d_nan);
  else
    k_inverse<16, true><<<grid, 256, 0, st>>>(coeffs, nullptr, img, w, h, pitch, bw, nb, p->d_basis, p->d_nan);
  dctf::add_launches(1);
  CUDA_TRY(cudaGetLastError());
  return DCTF_OK;
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
  kernel<<<static_cast<unsigned>(ctas), nw * 32, 32768 + nw * f8::WARP_BYTES, st>>>(
      in, out, w, h, pitch, frame_stride, nframes, bw, bh, nsx, p->d_hfused, p->d_basis, coef_out);
  dctf::add_launches(1);
  CUDA_TRY(cudaGetLastError());
  return DCTF_OK;
}

dctf_status launch_fused8_sym(const dctf_plan* p, const uint8_t* in, uint8_t* out, int w, int h,
                              size_t pitch, long long frame_stride, int nframes, double* coef_out,
                              cudaStream_t st) {
  auto kernel = coef_out ? k_fused8_sym<true> : k_fused8_sym<false>;
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
  kernel<<<static_cast<unsigned>(ctas), nw * 32, 16384 + nw * f8s::PIX_BYTES, st>>>(
      in, out, w, h, pitch, frame_stride, nframes, bw, bh, nsx, p->d_hsym, coef_out);
  dctf::add_launches(1);
  CUDA_TRY(cudaGetLastError());
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
  kernel<<<static_cast<unsigned>(ctas), f16::CWARPS * 32, f16::SMEM, st>>>(
      in, out, w, h, pitch, frame_stride, nframes, bw, bh, nsx, p->d_hfused, p->d_basis, coef_out);
  dctf::add_launches(1);
  CUDA_TRY(cudaGetLastError());
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
  kernel<<<static_cast<unsigned>(ctas), f16s::WARPS * 32, f16s::SMEM, st>>>(
      in, out, w, h, pitch, frame_stride, nframes, bw, bh, nsx, p->d_hsym, p->d_basis, coef_out);
  dctf::add_launches(1);
  CUDA_TRY(cudaGetLastError());
  return DCTF_OK;
}

// filter_image on device buffers, one frame or a strided frame batch.
dctf_status filter_image_device(const dctf_plan* p, const uint8_t* in, uint8_t* out, int w, int h,
                                size_t pitch, long long frame_stride, int nframes, double* coef_out,
                                cudaStream_t st) {
  if (p->n == 8 && p->precision == DCTF_PREC_INT8_EXACT)
    return dctf::launch_fused8_i8(p, in, out, w, h, pitch, frame_stride, nframes, coef_out, st,
                                  sm_count(p->device));
  const bool split = p->precision == DCTF_PREC_TF32X3;
  if (p->n == 8 && p->sym) return launch_fused8_sym(p, in, out, w, h, pitch, frame_stride, nframes, coef_out, st);
  if (p->n == 8 && !split) return launch_fused8(p, in, out, w, h, pitch, frame_stride, nframes, coef_out, st);
  if (p->n == 16 && p->sym && !std::getenv("DCTF_N16_UNFUSED"))
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

}  // namespace

// ---------------------------------------------------------------------------
// C ABI
extern "C" {

const char* dctf_last_error_message(void) { return dctf::t_err.c_str(); }
int dctf_last_launch_count(void) { return dctf::t_launches; }
const char* dctf_version(void) { return "dctf_b200 0.1 (sm_100a, fp64-dmma)"; }

}  // extern "C"

namespace {
// Device-side half of plan construction: validates the device and uploads the
// operator in every layout the kernels use. Takes ownership of p.
dctf_status finish_plan(dctf_plan* p, dctf_plan** out) {
  const int n = p->n, device = p->device, precision = p->precision;
  if (precision == DCTF_PREC_BF16X3) {
    delete p;
    return set_error(DCTF_UNSUPPORTED, "BF16x3 is not built; use DCTF_PREC_TF32X3 or DCTF_PREC_FP64");
  }
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
    cudaGetLastError();
    delete p;
    return set_error(DCTF_CUDA_ERROR, "no CUDA device available");
  }
  if (device < 0 || device >= ndev) {
    delete p;
    return set_error(DCTF_INVALID_ARGUMENT, "device ordinal out of range");
  }
  DeviceGuard guard(device);
  std::vector<double> hcoef, hfused;
  dctf::layout_hcoef(n, p->op, hcoef);
  const size_t nn = static_cast<size_t>(n) * n;
  cudaError_t e = cudaMalloc(&p->d_basis, nn * sizeof(double));
  if (e == cudaSuccess) e = cudaMalloc(&p->d_hcoef, nn * nn * sizeof(double));
  if (e == cudaSuccess) e = cudaMalloc(&p->d_nan, sizeof(int));
  if (e == cudaSuccess) e = cudaMalloc(&p->d_weights, p->weights.size() * sizeof(double));
  if (e == cudaSuccess)
    e = cudaMemcpy(p->d_weights, p->weights.data(), p->weights.size() * sizeof(double), cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMemcpy(p->d_basis, p->basis.data(), nn * sizeof(double), cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMemcpy(p->d_hcoef, hcoef.data(), nn * nn * sizeof(double), cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMemset(p->d_nan, 0, sizeof(int));
  if (e == cudaSuccess) {
    if (n == 8) dctf::layout_hfused8(dctf::compose_forward(p->op, p->basis, 8), hfused);
    else dctf::layout_hfused16(dctf::compose_forward(p->op, p->basis, 16), hfused);
    e = cudaMalloc(&p->d_hfused, hfused.size() * sizeof(double));
    if (e == cudaSuccess)
      e = cudaMemcpy(p->d_hfused, hfused.data(), hfused.size() * sizeof(double), cudaMemcpyHostToDevice);
  }
  p->sym = precision == DCTF_PREC_FP64 && dctf::parity_block_diagonal(p->op, n);
  if (e == cudaSuccess && p->sym && n == 16) {
    std::vector<double> gsym;
    dctf::layout_gsym16(p->op, p->basis, gsym);
    e = cudaMalloc(&p->d_hsym, gsym.size() * sizeof(double));
    if (e == cudaSuccess)
      e = cudaMemcpy(p->d_hsym, gsym.data(), gsym.size() * sizeof(double), cudaMemcpyHostToDevice);
  }
  if (e == cudaSuccess && p->sym && n == 16) {
    std::vector<double> hcsym;
    dctf::layout_coefsym16(p->op, hcsym);
    e = cudaMalloc(&p->d_hcsym, hcsym.size() * sizeof(double));
    if (e == cudaSuccess)
      e = cudaMemcpy(p->d_hcsym, hcsym.data(), hcsym.size() * sizeof(double), cudaMemcpyHostToDevice);
  }
  if (e == cudaSuccess && p->sym && n == 8) {
    std::vector<double> hsym;
    dctf::layout_sym8(p->op, p->basis, hsym);
    e = cudaMalloc(&p->d_hsym, hsym.size() * sizeof(double));
    if (e == cudaSuccess)
      e = cudaMemcpy(p->d_hsym, hsym.data(), hsym.size() * sizeof(double), cudaMemcpyHostToDevice);
    std::vector<double> hcsym;
    dctf::layout_coefsym8(p->op, hcsym);
    if (e == cudaSuccess) e = cudaMalloc(&p->d_hcsym, hcsym.size() * sizeof(double));
    if (e == cudaSuccess)
      e = cudaMemcpy(p->d_hcsym, hcsym.data(), hcsym.size() * sizeof(double), cudaMemcpyHostToDevice);
  }
  if (e == cudaSuccess && precision == DCTF_PREC_TF32X3) {
    std::vector<float> hs;
    dctf::layout_hsplit_tf32(n, p->op, hs);
    e = cudaMalloc(&p->d_hsplit, hs.size() * sizeof(float));
    if (e == cudaSuccess) e = cudaMemcpy(p->d_hsplit, hs.data(), hs.size() * sizeof(float), cudaMemcpyHostToDevice);
  }
  if (e != cudaSuccess) {
    const std::string msg = cudaGetErrorString(e);
    dctf_plan_destroy(p);
    return set_error(DCTF_CUDA_ERROR, "plan upload: " + msg);
  }
  if (precision == DCTF_PREC_INT8_EXACT && n == 8) {
    const dctf_status s = dctf::upload_i8_operator(p);
    if (s != DCTF_OK) {
      dctf_plan_destroy(p);
      return s;
    }
  }
  *out = p;
  return DCTF_OK;
}
}  // namespace

extern "C" {

dctf_status dctf_plan_create(const double* h_weights, int kr, int kc, int n, int padding,
                             int precision, int device, dctf_plan** out) {
  dctf::reset_launches();
  if (!out || !h_weights) return set_error(DCTF_INVALID_ARGUMENT, "NULL argument");
  *out = nullptr;
  if (precision < DCTF_PREC_FP64 || precision > DCTF_PREC_FP64_DENSE)
    return set_error(DCTF_INVALID_ARGUMENT, "unknown precision mode");
  if (kr < 1 || kc < 1) return set_error(DCTF_INVALID_ARGUMENT, "Mask: side must be odd and >= 1");
  auto* p = new dctf_plan();
  p->n = n;
  p->kr = kr;
  p->kc = kc;
  p->padding = padding;
  p->precision = precision;
  p->device = device;
  p->weights.assign(h_weights, h_weights + static_cast<size_t>(kr) * kc);
  dctf_status s = dctf::compile_operator(*p);
  if (s != DCTF_OK) {
    delete p;
    return s;
  }
  return finish_plan(p, out);
}

dctf_status dctf_plan_create_from_dump(const char* text, size_t len, int precision, int device,
                                       dctf_plan** out) {
  dctf::reset_launches();
  if (!out || !text) return set_error(DCTF_INVALID_ARGUMENT, "NULL argument");
  *out = nullptr;
  if (precision < DCTF_PREC_FP64 || precision > DCTF_PREC_FP64_DENSE)
    return set_error(DCTF_INVALID_ARGUMENT, "unknown precision mode");
  auto* p = new dctf_plan();
  p->precision = precision;
  p->device = device;
  dctf_status s = dctf::parse_operator_dump(std::string(text, len), *p);
  if (s != DCTF_OK) {
    delete p;
    return s;
  }
  return finish_plan(p, out);
}

dctf_status dctf_plan_dump(const dctf_plan* p, char* buf, size_t* len) {
  if (!p || !len) return set_error(DCTF_INVALID_ARGUMENT, "NULL argument");
  if (p->dct_left.empty() || p->sp_left.empty())
    return set_error(DCTF_UNSUPPORTED, "operator dump needs a square mask compiled as sandwich pairs");
  const std::string text = dctf::format_operator_dump(*p);
  if (buf && *len >= text.size()) std::memcpy(buf, text.data(), text.size());
  *len = text.size();
  return DCTF_OK;
}

dctf_status dctf_format_operator_dump(const double* h_weights, int k, int n, int padding, char* buf,
                                      size_t* len) {
  if (!h_weights || !len) return set_error(DCTF_INVALID_ARGUMENT, "NULL argument");
  if (k < 1) return set_error(DCTF_INVALID_ARGUMENT, "Mask: side must be odd and >= 1");
  if (k > n) return set_error(DCTF_INVALID_ARGUMENT, "build_spatial_operator_set: mask larger than block");
  dctf_plan p;
  p.n = n;
  p.kr = p.kc = k;
  p.padding = padding;
  p.weights.assign(h_weights, h_weights + static_cast<size_t>(k) * k);
  const dctf_status s = dctf::compile_operator(p);
  if (s != DCTF_OK) return s;
  return dctf_plan_dump(&p, buf, len);
}

dctf_status dctf_operator_from_dump(const char* text, size_t len, double* h_op, int* n, int* k,
                                    int* padding) {
  if (!text) return set_error(DCTF_INVALID_ARGUMENT, "NULL argument");
  dctf_plan p;
  const dctf_status s = dctf::parse_operator_dump(std::string(text, len), p);
  if (s != DCTF_OK) return s;
  if (h_op) std::memcpy(h_op, p.op.data(), p.op.size() * sizeof(double));
  if (n) *n = p.n;
  if (k) *k = p.kr;
  if (padding) *padding = p.padding;
  return DCTF_OK;
}

dctf_status dctf_plan_pairs(const dctf_plan* p, int domain, double* h_lefts, double* h_rights) {
  if (!p) return set_error(DCTF_INVALID_ARGUMENT, "NULL argument");
  const std::vector<double>& L = domain ? p->dct_left : p->sp_left;
  const std::vector<double>& R = domain ? p->dct_right : p->sp_right;
  if (L.empty()) return set_error(DCTF_UNSUPPORTED, "plan has no sandwich pairs in that domain");
  if (h_lefts) std::memcpy(h_lefts, L.data(), L.size() * sizeof(double));
  if (h_rights) std::memcpy(h_rights, R.data(), R.size() * sizeof(double));
  return DCTF_OK;
}

dctf_status dctf_compile_operator(const double* h_weights, int kr, int kc, int n, int padding,
                                  double* h_c, double* h_op, int* npairs, int* merged) {
  if (!h_weights) return set_error(DCTF_INVALID_ARGUMENT, "NULL argument");
  if (kr < 1 || kc < 1) return set_error(DCTF_INVALID_ARGUMENT, "Mask: side must be odd and >= 1");
  dctf_plan p;
  p.n = n;
  p.kr = kr;
  p.kc = kc;
  p.padding = padding;
  p.weights.assign(h_weights, h_weights + static_cast<size_t>(kr) * kc);
  const dctf_status s = dctf::compile_operator(p);
  if (s != DCTF_OK) return s;
  if (h_c) std::memcpy(h_c, p.basis.data(), p.basis.size() * sizeof(double));
  if (h_op) std::memcpy(h_op, p.op.data(), p.op.size() * sizeof(double));
  if (npairs) *npairs = p.npairs;
  if (merged) *merged = p.merged;
  return DCTF_OK;
}

dctf_status dctf_plan_destroy(dctf_plan* p) {
  if (!p) return DCTF_OK;
  {
    DeviceGuard guard(p->device);
    cudaFree(p->d_basis);
    cudaFree(p->d_hcoef);
    cudaFree(p->d_hfused);
    cudaFree(p->d_hsym);
    cudaFree(p->d_hcsym);
    cudaFree(p->d_hsplit);
    cudaFree(p->d_gimg);
    cudaFree(p->d_gscale);
    cudaFree(p->d_nan);
    cudaFree(p->d_weights);
    cudaFree(p->io_in);
    cudaFree(p->io_out);
    for (void* s : p->streams)
      if (s) cudaStreamDestroy(as_stream(s));
    for (void* e : p->events)
      if (e) cudaEventDestroy(static_cast<cudaEvent_t>(e));
  }
  delete p;
  return DCTF_OK;
}

dctf_status dctf_plan_info(const dctf_plan* p, int* n, int* npairs, int* merged) {
  if (!p) return set_error(DCTF_INVALID_ARGUMENT, "plan is NULL");
  if (n) *n = p->n;
  if (npairs) *npairs = p->npairs;
  if (merged) *merged = p->merged;
  return DCTF_OK;
}

const char* dctf_plan_coef_kernel(const dctf_plan* p) {
  if (!p) return nullptr;
  if (p->precision == DCTF_PREC_TF32X3) return "k_coef_tf32x3";
  if (p->n == 8) return p->sym ? "k_coef8_sym" : "k_coef8";
  return p->sym ? "k_coef16_sym" : "k_coef16";
}

const char* dctf_plan_image_kernel(const dctf_plan* p) {
  if (!p) return nullptr;
  if (p->n == 8 && p->precision == DCTF_PREC_INT8_EXACT) return "k_fused8_i8";
  if (p->precision == DCTF_PREC_TF32X3) return "unfused";
  if (p->n == 8) return p->sym ? "k_fused8_sym" : "k_fused8";
  if (std::getenv("DCTF_N16_UNFUSED")) return "unfused";
  return p->sym ? "k_fused16_sym" : "k_fused16";
}

dctf_status dctf_plan_basis(const dctf_plan* p, double* h_c) {
  if (!p || !h_c) return set_error(DCTF_INVALID_ARGUMENT, "NULL argument");
  std::memcpy(h_c, p->basis.data(), p->basis.size() * sizeof(double));
  return DCTF_OK;
}

dctf_status dctf_plan_operator(const dctf_plan* p, double* h_op) {
  if (!p || !h_op) return set_error(DCTF_INVALID_ARGUMENT, "NULL argument");
  std::memcpy(h_op, p->op.data(), p->op.size() * sizeof(double));
  return DCTF_OK;
}

dctf_status dctf_forward(const dctf_plan* p, const uint8_t* d_img, int w, int h, size_t pitch,
                         double* d_coeffs, void* stream) {
  dctf::reset_launches();
  dctf_status s = check_plan(p);
  if (s == DCTF_OK) s = check_image(w, h, pitch);
  if (s != DCTF_OK) return s;
  if (!d_img || !d_coeffs) return set_error(DCTF_INVALID_ARGUMENT, "NULL buffer");
  DeviceGuard guard(p->device);
  return launch_forward_u8(p, d_img, w, h, pitch, d_coeffs, as_stream(stream));
}

dctf_status dctf_forward_blocks(const dctf_plan* p, const double* d_blocks, double* d_coeffs,
                                size_t nblocks, void* stream) {
  dctf::reset_launches();
  dctf_status s = check_plan(p);
  if (s != DCTF_OK) return s;
  if (nblocks == 0) return DCTF_OK;
  if (!d_blocks || !d_coeffs) return set_error(DCTF_INVALID_ARGUMENT, "NULL buffer");
  if (misaligned16(d_coeffs)) return set_error(DCTF_INVALID_ARGUMENT, "buffers must be 16-byte aligned");
  DeviceGuard guard(p->device);
  const long long nb = static_cast<long long>(nblocks);
  const int bpc = 256 / p->n;
  const unsigned grid = static_cast<unsigned>((nb + bpc - 1) / bpc);
  if (p->n == 8)
    k_forward<8, false><<<grid, 256, 0, as_stream(stream)>>>(nullptr, 0, 0, 0, 1, d_blocks, d_coeffs, nb, p->d_basis);
  else
    k_forward<16, false><<<grid, 256, 0, as_stream(stream)>>>(nullptr, 0, 0, 0, 1, d_blocks, d_coeffs, nb, p->d_basis);
  dctf::add_launches(1);
  CUDA_TRY(cudaGetLastError());
  return DCTF_OK;
}

dctf_status dctf_inverse_blocks(const dctf_plan* p, const double* d_coeffs, double* d_blocks,
                                size_t nblocks, void* stream) {
  dctf::reset_launches();
  dctf_status s = check_plan(p);
  if (s != DCTF_OK) return s;
  if (nblocks == 0) return DCTF_OK;
  if (!d_blocks || !d_coeffs) return set_error(DCTF_INVALID_ARGUMENT, "NULL buffer");
  if (misaligned16(d_blocks)) return set_error(DCTF_INVALID_ARGUMENT, "buffers must be 16-byte aligned");
  DeviceGuard guard(p->device);
  const long long nb = static_cast<long long>(nblocks);
  const int bpc = 256 / p->n;
  const unsigned grid = static_cast<unsigned>((nb + bpc - 1) / bpc);
  if (p->n == 8)
    k_inverse<8, false><<<grid, 256, 0, as_stream(stream)>>>(d_coeffs, d_blocks, nullptr, 0, 0, 0, 1, nb, p->d_basis, nullptr);
  else
    k_inverse<16, false><<<grid, 256, 0, as_stream(stream)>>>(d_coeffs, d_blocks, nullptr, 0, 0, 0, 1, nb, p->d_basis, nullptr);
  dctf::add_launches(1);
  CUDA_TRY(cudaGetLastError());
  return DCTF_OK;
}

dctf_status dctf_filter_coeffs(const dctf_plan* p, const double* d_in, double* d_out,
                               size_t nblocks, void* stream) {
  dctf::reset_launches();
  dctf_status s = check_plan(p);
  if (s != DCTF_OK) return s;
  if (nblocks == 0) return DCTF_OK;
  if (!d_in || !d_out) return set_error(DCTF_INVALID_ARGUMENT, "NULL buffer");
  DeviceGuard guard(p->device);
  return launch_coef(p, d_in, d_out, static_cast<long long>(nblocks), as_stream(stream));
}

dctf_status dctf_inverse_u8(const dctf_plan* p, const double* d_coeffs, uint8_t* d_img, int w,
                            int h, size_t pitch, void* stream) {
  dctf::reset_launches();
  dctf_status s = check_plan(p);
  if (s == DCTF_OK) s = check_image(w, h, pitch);
  if (s != DCTF_OK) return s;
  if (!d_img || !d_coeffs) return set_error(DCTF_INVALID_ARGUMENT, "NULL buffer");
  DeviceGuard guard(p->device);
  return launch_inverse_u8(p, d_coeffs, d_img, w, h, pitch, as_stream(stream));
}

dctf_status dctf_filter_image_u8(const dctf_plan* p, const uint8_t* d_in, uint8_t* d_out, int w,
                                 int h, size_t pitch, double* d_coeffs_out, void* stream) {
  dctf::reset_launches();
  dctf_status s = check_plan(p);
  if (s == DCTF_OK) s = check_image(w, h, pitch);
  if (s != DCTF_OK) return s;
  if (!d_in || !d_out) return set_error(DCTF_INVALID_ARGUMENT, "NULL buffer");
  if (d_in == d_out) return set_error(DCTF_INVALID_ARGUMENT, "in/out images may not alias");
  DeviceGuard guard(p->device);
  return filter_image_device(p, d_in, d_out, w, h, pitch, 0, 1, d_coeffs_out, as_stream(stream));
}

dctf_status dctf_filter_image_spatial_u8(const dctf_plan* p, const uint8_t* d_in, uint8_t* d_out,
                                         int w, int h, size_t pitch, void* stream) {
  dctf::reset_launches();
  dctf_status s = check_plan(p);
  if (s == DCTF_OK) s = check_image(w, h, pitch);
  if (s != DCTF_OK) return s;
  if (!d_in || !d_out) return set_error(DCTF_INVALID_ARGUMENT, "NULL buffer");
  if (p->kr * p->kc > 1024) return set_error(DCTF_UNSUPPORTED, "spatial path supports masks up to 1024 taps");
  DeviceGuard guard(p->device);
  const int n = p->n, bw = (w + n - 1) / n, bh = (h + n - 1) / n;
  const long long nb = static_cast<long long>(bw) * bh;
  const unsigned grid = static_cast<unsigned>((nb * n * n + 255) / 256);
  k_spatial<true><<<grid, 256, 0, as_stream(stream)>>>(d_in, w, h, pitch, bw, nullptr, d_out, nullptr, nb, n,
                                                       p->d_weights, p->kr, p->kc, p->padding);
  dctf::add_launches(1);
  CUDA_TRY(cudaGetLastError());
  return DCTF_OK;
}

dctf_status dctf_convolve_blocks(const dctf_plan* p, const double* d_blocks, double* d_out, size_t nblocks,
                                 void* stream) {
  dctf::reset_launches();
  dctf_status s = check_plan(p);
  if (s != DCTF_OK) return s;
  if (nblocks == 0) return DCTF_OK;
  if (!d_blocks || !d_out) return set_error(DCTF_INVALID_ARGUMENT, "NULL buffer");
  if (p->kr * p->kc > 1024) return set_error(DCTF_UNSUPPORTED, "spatial path supports masks up to 1024 taps");
  DeviceGuard guard(p->device);
  const int n = p->n;
  const long long nb = static_cast<long long>(nblocks);
  const unsigned grid = static_cast<unsigned>((nb * n * n + 255) / 256);
  k_spatial<false><<<grid, 256, 0, as_stream(stream)>>>(nullptr, 0, 0, 0, 1, d_blocks, nullptr, d_out, nb, n,
                                                        p->d_weights, p->kr, p->kc, p->padding);
  dctf::add_launches(1);
  CUDA_TRY(cudaGetLastError());
  return DCTF_OK;
}

dctf_status dctf_filter_frames_u8(const dctf_plan* const* plans, int nplans,
                                  const int* h_plan_of_frame, const uint8_t* d_in, uint8_t* d_out,
                                  int nframes, int w, int h, size_t pitch, size_t frame_stride,
                                  void* stream) {
  dctf::reset_launches();
  if (!plans || nplans < 1 || !h_plan_of_frame || nframes < 0)
    return set_error(DCTF_INVALID_ARGUMENT, "bad plan list");
  dctf_status s = check_image(w, h, pitch);
  if (s != DCTF_OK) return s;
  if (frame_stride < pitch * static_cast<size_t>(h))
    return set_error(DCTF_INVALID_ARGUMENT, "frame_stride smaller than one frame");
  for (int i = 0; i < nplans; ++i) {
    s = check_plan(plans[i]);
    if (s != DCTF_OK) return s;
    if (plans[i]->n != plans[0]->n || plans[i]->device != plans[0]->device)
      return set_error(DCTF_INVALID_ARGUMENT, "plans must share n and device");
  }
  for (int f = 0; f < nframes; ++f)
    if (h_plan_of_frame[f] < 0 || h_plan_of_frame[f] >= nplans)
      return set_error(DCTF_INVALID_ARGUMENT, "plan_of_frame index out of range");
  DeviceGuard guard(plans[0]->device);
  const cudaStream_t st = as_stream(stream);
  // Frames sharing a plan and evenly spaced go in one launch (round-robin
  // assignment -> one launch per plan); anything else falls back per frame.
  for (int pi = 0; pi < nplans && s == DCTF_OK; ++pi) {
    int first = -1, second = -1, count = 0;
    bool arith = true;
    for (int f = 0; f < nframes; ++f) {
      if (h_plan_of_frame[f] != pi) continue;
      if (first < 0) first = f;
      else if (second < 0) second = f;
      else if ((f - first) != count * (second - first)) arith = false;
      ++count;
    }
    if (count == 0) continue;
    if (arith) {
      const long long step = count > 1 ? static_cast<long long>(second - first) : 1;
      s = filter_image_device(plans[pi], d_in + first * frame_stride, d_out + first * frame_stride,
                              w, h, pitch, step * static_cast<long long>(frame_stride), count,
                              nullptr, st);
    } else {
      for (int f = 0; f < nframes && s == DCTF_OK; ++f)
        if (h_plan_of_frame[f] == pi)
          s = filter_image_device(plans[pi], d_in + f * frame_stride, d_out + f * frame_stride, w,
                                  h, pitch, 0, 1, nullptr, st);
    }
  }
  return s;
}

dctf_status dctf_filter_image_host(const dctf_plan* p, const uint8_t* h_in, uint8_t* h_out, int w,
                                   int h, size_t pitch) {
  dctf::reset_launches();
  dctf_status s = check_plan(p);
  if (s == DCTF_OK) s = check_image(w, h, pitch);
  if (s != DCTF_OK) return s;
  if (!h_in || !h_out) return set_error(DCTF_INVALID_ARGUMENT, "NULL buffer");
  DeviceGuard guard(p->device);
  std::lock_guard<std::mutex> lock(p->io_mu);
  const size_t dpitch = (static_cast<size_t>(w) + 15) & ~size_t(15);
  const size_t bytes = dpitch * static_cast<size_t>(h);
  if (p->io_bytes < bytes) {
    cudaFree(p->io_in);
    cudaFree(p->io_out);
    p->io_in = p->io_out = nullptr;
    p->io_bytes = 0;
    CUDA_TRY(cudaMalloc(&p->io_in, bytes));
    CUDA_TRY(cudaMalloc(&p->io_out, bytes));
    p->io_bytes = bytes;
  }
  for (auto& st : p->streams)
    if (!st) {
      cudaStream_t x;
      CUDA_TRY(cudaStreamCreateWithFlags(&x, cudaStreamNonBlocking));
      st = x;
    }
  for (auto& ev : p->events)
    if (!ev) {
      cudaEvent_t x;
      CUDA_TRY(cudaEventCreateWithFlags(&x, cudaEventDisableTiming));
      ev = x;
    }
  const cudaStream_t s_in = as_stream(p->streams[0]), s_run = as_stream(p->streams[1]),
                     s_out = as_stream(p->streams[2]);
  // Transfer strategy. Pinned (page-locked, UVA-mapped) buffers let the fused
  // kernel touch host memory directly over PCIe:
  //   mode 2 "zero-copy": the kernel streams pixels in from h_in and writes
  //          results to h_out itself (one launch, both link directions busy);
  //   mode 1 "copy-in + zero-copy out": H2D by the copy engine in a few large
  //          chunks, each chunk's kernel writes straight to h_out;
  //   mode 0 "copy": H2D / compute / D2H in three streams (pageable buffers).
  // DCTF_E2E_MODE overrides the choice (measurement).
  cudaPointerAttributes ai{}, ao{};
  const bool in_pinned = cudaPointerGetAttributes(&ai, h_in) == cudaSuccess &&
                         ai.type == cudaMemoryTypeHost && ai.devicePointer != nullptr;
  const bool out_pinned = cudaPointerGetAttributes(&ao, h_out) == cudaSuccess &&
                          ao.type == cudaMemoryTypeHost && ao.devicePointer != nullptr;
  cudaGetLastError();
  // zero-copy needs a single fused kernel (every precision except the
  // split-precision path, which runs forward/filter/inverse as three kernels)
  const bool fused = p->precision != DCTF_PREC_TF32X3;
  int mode = (in_pinned && out_pinned && fused) ? 2 : (out_pinned && fused ? 1 : 0);
  if (const char* env = std::getenv("DCTF_E2E_MODE")) {
    const int m = std::atoi(env);
    if (m == 0 || (m == 1 && out_pinned && fused) || (m == 2 && in_pinned && out_pinned && fused)) mode = m;
  }
  if (p->n != 8) CUDA_TRY(cudaMemsetAsync(p->d_nan, 0, sizeof(int), s_run));
  const int n = p->n, bh = (h + n - 1) / n;
  int launches = 0;
  if (mode == 2) {
    s = filter_image_device(p, static_cast<const uint8_t*>(ai.devicePointer),
                            static_cast<uint8_t*>(ao.devicePointer), w, h, pitch, 0, 1, nullptr,
                            s_run);
    launches = dctf::t_launches;
  } else {
    const size_t chunk_target = mode == 1 ? (size_t(4) << 20) : (size_t(2) << 20);
    const int nchunks = std::max(1, std::min(bh, static_cast<int>((static_cast<size_t>(h) * w + chunk_target - 1) / chunk_target)));
    const int brows = (bh + nchunks - 1) / nchunks;
    auto* din = static_cast<uint8_t*>(p->io_in);
    auto* dout = static_cast<uint8_t*>(p->io_out);
    auto* hout_dev = static_cast<uint8_t*>(ao.devicePointer);
    for (int c = 0; c * brows < bh && s == DCTF_OK; ++c) {
      const int y0 = c * brows * n;
      const int rows = std::min(brows * n, h - y0);
      cudaEvent_t in_done = static_cast<cudaEvent_t>(p->events[(2 * c) % 64]);
      cudaEvent_t run_done = static_cast<cudaEvent_t>(p->events[(2 * c + 1) % 64]);
      if (pitch == dpitch)
        CUDA_TRY(cudaMemcpyAsync(din + y0 * dpitch, h_in + y0 * pitch, static_cast<size_t>(rows) * pitch,
                                 cudaMemcpyHostToDevice, s_in));
      else
        CUDA_TRY(cudaMemcpy2DAsync(din + y0 * dpitch, dpitch, h_in + y0 * pitch, pitch, w, rows,
                                   cudaMemcpyHostToDevice, s_in));
      CUDA_TRY(cudaEventRecord(in_done, s_in));
      CUDA_TRY(cudaStreamWaitEvent(s_run, in_done, 0));
      dctf::reset_launches();
      if (mode == 1)
        s = filter_image_device(p, din + y0 * dpitch, hout_dev + y0 * pitch, w, rows, pitch, 0, 1,
                                nullptr, s_run);
      else
        s = filter_image_device(p, din + y0 * dpitch, dout + y0 * dpitch, w, rows, dpitch, 0, 1,
                                nullptr, s_run);
      launches += dctf::t_launches;
      if (s != DCTF_OK || mode == 1) continue;
      CUDA_TRY(cudaEventRecord(run_done, s_run));
      CUDA_TRY(cudaStreamWaitEvent(s_out, run_done, 0));
      if (pitch == dpitch)
        CUDA_TRY(cudaMemcpyAsync(h_out + y0 * pitch, dout + y0 * dpitch, static_cast<size_t>(rows) * pitch,
                                 cudaMemcpyDeviceToHost, s_out));
      else
        CUDA_TRY(cudaMemcpy2DAsync(h_out + y0 * pitch, pitch, dout + y0 * dpitch, dpitch, w, rows,
                                   cudaMemcpyDeviceToHost, s_out));
    }
  }
  int nan_seen = 0;
  if (s == DCTF_OK && p->n != 8) {
    CUDA_TRY(cudaStreamSynchronize(s_run));
    CUDA_TRY(cudaMemcpyAsync(&nan_seen, p->d_nan, sizeof(int), cudaMemcpyDeviceToHost, s_run));
  }
  CUDA_TRY(cudaStreamSynchronize(s_in));
  CUDA_TRY(cudaStreamSynchronize(s_run));
  CUDA_TRY(cudaStreamSynchronize(s_out));
  dctf::t_launches = launches;
  if (s != DCTF_OK) return s;
  if (nan_seen) return set_error(DCTF_NAN_ENCOUNTERED, "quantize: NaN sample");
  return DCTF_OK;
}

// Host-buffer batch wrappers: stream-ordered scratch, synchronous.
static dctf_status run_host_blocks(const dctf_plan* p, const double* h_in, double* h_out,
                                   size_t nblocks, int op) {
  dctf_status s = check_plan(p);
  if (s != DCTF_OK) return s;
  if (nblocks == 0) return DCTF_OK;
  if (!h_in || !h_out) return set_error(DCTF_INVALID_ARGUMENT, "NULL buffer");
  DeviceGuard guard(p->device);
  const size_t bytes = nblocks * static_cast<size_t>(p->n) * p->n * sizeof(double);
  cudaStream_t st;
  CUDA_TRY(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  double *din = nullptr, *dout = nullptr;
  cudaError_t e = cudaMallocAsync(reinterpret_cast<void**>(&din), bytes, st);
  if (e == cudaSuccess) e = cudaMallocAsync(reinterpret_cast<void**>(&dout), bytes, st);
  if (e == cudaSuccess) e = cudaMemcpyAsync(din, h_in, bytes, cudaMemcpyHostToDevice, st);
  if (e != cudaSuccess) s = set_error(DCTF_CUDA_ERROR, cudaGetErrorString(e));
  if (s == DCTF_OK) {
    if (op == 0) s = dctf_forward_blocks(p, din, dout, nblocks, st);
    else if (op == 1) s = dctf_inverse_blocks(p, din, dout, nblocks, st);
    else if (op == 2) s = dctf_filter_coeffs(p, din, dout, nblocks, st);
    else s = dctf_convolve_blocks(p, din, dout, nblocks, st);
  }
  if (s == DCTF_OK) {
    e = cudaMemcpyAsync(h_out, dout, bytes, cudaMemcpyDeviceToHost, st);
    if (e != cudaSuccess) s = set_error(DCTF_CUDA_ERROR, cudaGetErrorString(e));
  }
  cudaFreeAsync(din, st);
  cudaFreeAsync(dout, st);
  e = cudaStreamSynchronize(st);
  if (s == DCTF_OK && e != cudaSuccess) s = set_error(DCTF_CUDA_ERROR, cudaGetErrorString(e));
  cudaStreamDestroy(st);
  return s;
}

dctf_status dctf_forward_blocks_host(const dctf_plan* p, const double* h_in, double* h_out,
                                     size_t nblocks) {
  return run_host_blocks(p, h_in, h_out, nblocks, 0);
}
dctf_status dctf_inverse_blocks_host(const dctf_plan* p, const double* h_in, double* h_out,
                                     size_t nblocks) {
  return run_host_blocks(p, h_in, h_out, nblocks, 1);
}
dctf_status dctf_filter_coeffs_host(const dctf_plan* p, const double* h_in, double* h_out,
                                    size_t nblocks) {
  return run_host_blocks(p, h_in, h_out, nblocks, 2);
}

dctf_status dctf_convolve_blocks_host(const dctf_plan* p, const double* h_in, double* h_out,
                                      size_t nblocks) {
  return run_host_blocks(p, h_in, h_out, nblocks, 3);
}

dctf_status dctf_filter_image_spatial_host(const dctf_plan* p, const uint8_t* h_in, uint8_t* h_out, int w,
                                           int h, size_t pitch) {
  dctf_status s = check_plan(p);
  if (s == DCTF_OK) s = check_image(w, h, pitch);
  if (s != DCTF_OK) return s;
  if (!h_in || !h_out) return set_error(DCTF_INVALID_ARGUMENT, "NULL buffer");
  DeviceGuard guard(p->device);
  const size_t bytes = pitch * static_cast<size_t>(h);
  uint8_t *din = nullptr, *dout = nullptr;
  CUDA_TRY(cudaMalloc(&din, bytes));
  cudaError_t e = cudaMalloc(&dout, bytes);
  if (e == cudaSuccess) e = cudaMemcpy(din, h_in, bytes, cudaMemcpyHostToDevice);
  if (e == cudaSuccess) {
    s = dctf_filter_image_spatial_u8(p, din, dout, w, h, pitch, nullptr);
    if (s == DCTF_OK) e = cudaMemcpy(h_out, dout, bytes, cudaMemcpyDeviceToHost);
  }
  cudaFree(din);
  cudaFree(dout);
  if (e != cudaSuccess) return set_error(DCTF_CUDA_ERROR, cudaGetErrorString(e));
  return s;
}

dctf_status dctf_measure_fp64_peak(int device, int mode, double* tflops) {
  if (!tflops || (mode != 0 && mode != 1)) return set_error(DCTF_INVALID_ARGUMENT, "bad argument");
  DeviceGuard guard(device);
  double* d = nullptr;
  CUDA_TRY(cudaMalloc(&d, 256 * sizeof(double)));
  cudaEvent_t e0, e1;
  CUDA_TRY(cudaEventCreate(&e0));
  CUDA_TRY(cudaEventCreate(&e1));
  const int blocks = sm_count(device) * 8, iters = mode == 0 ? 2048 : 16384;
  float best = 1e30f;
  for (int rep = 0; rep < 4; ++rep) {
    cudaEventRecord(e0);
    if (mode == 0) k_peak_dmma<<<blocks, 256>>>(d, iters);
    else k_peak_dfma<<<blocks, 256>>>(d, iters);
    cudaEventRecord(e1);
    CUDA_TRY(cudaEventSynchronize(e1));
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    if (rep > 0) best = std::min(best, ms);
  }
  CUDA_TRY(cudaGetLastError());
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(d);
  const double flops = mode == 0 ? double(blocks) * 8 * iters * 8 * 512.0    // warps * iters * 8 DMMA * 512
                                 : double(blocks) * 256 * iters * 8 * 2.0;
  *tflops = flops / (best * 1e-3) / 1e12;
  return DCTF_OK;
}

dctf_status dctf_plan_nan_check(const dctf_plan* p, void* stream, int* nan_seen) {
  if (!p || !nan_seen) return set_error(DCTF_INVALID_ARGUMENT, "NULL argument");
  DeviceGuard guard(p->device);
  const cudaStream_t st = as_stream(stream);
  int v = 0;
  CUDA_TRY(cudaMemcpyAsync(&v, p->d_nan, sizeof(int), cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaMemsetAsync(p->d_nan, 0, sizeof(int), st));
  CUDA_TRY(cudaStreamSynchronize(st));
  *nan_seen = v;
  return DCTF_OK;
}

}  // extern "C"
