// k_fused8_i8: the 8x8 spatial-in/spatial-out DCT-domain filter with the
// DCT-domain contraction done EXACTLY on the INT8 tensor cores
// (tcgen05.mma kind::i8, int32 accumulators in TMEM), sm_100a.
//
// Math (precision DCTF_PREC_INT8_EXACT). Pixels p are exact integers, so the
// first linear stage applied to them can run in integer arithmetic without
// loss: G = H_dct (C (x) C) (forward DCT composed with the DCT-domain operator,
// one 64x64 FP64 matrix per plan) is written per output row as 7 signed
// 7-bit digits (plan.cc: layout_gslices_i8), every partial D_s = d_s . p is
// an exact int32, and the filtered DCT coefficients
//     Y[o] = 2^(e_o - 48) * sum_s D_s[o] 2^(7(7-s))
// are recombined in FP64 with a relative error ~2^-49 — FP64-class, the same
// tolerance class as the DMMA path (coefficients are also exported in parity
// mode). The inverse DCT O = C^t Y C + 0.5 and the round/clamp stay on the
// FP64 pipe: 4 DMMA (1,024 FMA) + 256 recombination FMAs per block instead of
// the 24 DMMA (6,144 FMA) of k_fused8. The forward DCT is folded into G (one
// precomputed operator per plan); Y, the DCT-domain filtered coefficients, is
// materialised exactly as in the FP64 chain.
//
// CTA = 16 warps, one CTA per SM, persistent over tiles of 128 horizontally
// adjacent blocks (a strip of 8 rows x 1024 px):
//   warps 0-3  producers: thread b gathers block b's 8x8 pixels (8-byte
//              coalesced loads, one tile ahead in registers) into the K-major
//              A tile (128 B rows, 128B swizzle, 64 bytes used); thread 0
//              issues the 4 MMAs (2 K-steps x 2 output halves, N = 224
//              columns each) per tile; each half has its own accumulator, so
//              the next tile's MMA into one half overlaps the drain of the
//              other.
//   warps 4-11 drain: thread = block = TMEM lane (two warps per lane quarter,
//              each half of the outputs); tcgen05.ld the int32 partials,
//              recombine exactly in int64, scale to FP64 Y in a
//              double-buffered shared tile (k_fused8's swizzled layout),
//              release TMEM so the next tile's MMAs start.
//   warps 12-19 compute: k_fused8's inverse DMMA chain (O = C^t Y C + 0.5) on
//              16 blocks per warp, floor-quantise, coalesced strip stores.
// The 56 KB digit image (B operand) stays resident in shared memory.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <string>

#include "fastdiv.cuh"
#include "device.cuh"
#include "internal.h"

namespace {

__device__ __forceinline__ uint64_t umma_desc_sw128(uint32_t saddr) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((saddr >> 4) & 0x3FFFu);
  d |= static_cast<uint64_t>(1u) << 16;
  d |= static_cast<uint64_t>(1024u >> 4) << 32;
  d |= static_cast<uint64_t>(1u) << 46;
  d |= static_cast<uint64_t>(2u) << 61;
  return d;
}
// kind::i8: A unsigned 8-bit, B signed 8-bit, D s32, both K-major.
__host__ __device__ constexpr uint32_t idesc_i8(int m, int n) {
  return (2u << 4) | (0u << 7) | (1u << 10) | (static_cast<uint32_t>(n >> 3) << 17) |
         (static_cast<uint32_t>(m >> 4) << 24);
}
__device__ __forceinline__ void mma_i8(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                       uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void tmem_ld8(uint32_t taddr, int32_t (&v)[8]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
               : "r"(taddr));
}


// compute warps run the inverse chain on OZG blocks at once (independent
// DMMA chains; all CB = 16 of a warp's blocks: +7 % over groups of 4)
#ifndef OZG
#define OZG 16
#endif
namespace oz {
constexpr int TILE = 128;
constexpr int S = 7;
constexpr int NCOL = S * 64;            // 448 accumulator columns
constexpr int BBYTES = NCOL * 128;      // resident digit image
constexpr int ABYTES = TILE * 128;      // one A stage
constexpr int YBYTES = TILE * 512;      // one FP64 Y tile (64 doubles per block)
constexpr int PS = 144;                 // compute-warp pixel staging row stride (16 blocks)
constexpr int PIXBYTES = 8 * PS;
constexpr int PROD = 4, DRAIN = 8, COMP = 8;
constexpr int CB = TILE / COMP;          // blocks per compute warp
constexpr int THREADS = 32 * (PROD + DRAIN + COMP);
constexpr int SMEM = 1024 + BBYTES + 2 * ABYTES + 2 * YBYTES + COMP * PIXBYTES;
// Y tile layout = k_fused8's X/Y staging: block b owns 512 B = 4 rows x 8
// chunks of 16 B; logical (row r, chunk c) holds Y[2r][c], Y[2r+1][c] and is
// stored at chunk c ^ 2r ^ f(b), f(b) = (b&7) ^ ((b&1)<<2).
__device__ __forceinline__ int fsw(int b) { return (b & 7) ^ ((b & 1) << 2); }
}  // namespace oz

__global__ void __launch_bounds__(oz::THREADS, 1)
    k_fused8_i8(const uint8_t* __restrict__ in, uint8_t* __restrict__ out, int w, int h, size_t pitch,
                long long frame_stride, int nframes, int bw, int bh, int nsx,
                const int8_t* __restrict__ gimg, const double* __restrict__ gscale,
                const double* __restrict__ cb, double* __restrict__ coef_out) {
  using namespace oz;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* base = align1024(smem_raw);
  uint8_t* bsm = base;                       // digit image
  uint8_t* asm_ = base + BBYTES;             // 2 A stages
  uint8_t* ysm = asm_ + 2 * ABYTES;          // 2 Y tiles
  uint8_t* psm = ysm + 2 * YBYTES;           // compute-warp pixel staging
  __shared__ uint64_t a_full[2], a_empty[2], acc_full[2], acc_empty[2], y_full[2], y_empty[2];
  __shared__ uint32_t tmem_base_s;
  __shared__ double sc_s[64];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  pdl_trigger();
  cta_copy_async(bsm, gimg, BBYTES);  // plan-owned operator: staged before the dependency wait
  if (threadIdx.x < 64) sc_s[threadIdx.x] = gscale[threadIdx.x];
  if (warp == PROD) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(&tmem_base_s)),
                 "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 0) {
    for (int i = 0; i < 2; ++i) {
      mbar_init(&a_full[i], 32 * PROD);
      mbar_init(&a_empty[i], 1);
      mbar_init(&y_full[i], 32 * DRAIN);
      mbar_init(&y_empty[i], COMP);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&acc_full[i], 1);
      mbar_init(&acc_empty[i], 32 * DRAIN / 2);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  cp_async_wait_all();
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = tmem_base_s;
  pdl_wait();

  const long long spf = static_cast<long long>(bh) * nsx;
  const long long ntiles = spf * nframes;
  const bool aligned = ((pitch & 15) == 0) && ((reinterpret_cast<uintptr_t>(in) & 7) == 0) &&
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
  auto is_fast = [&](int by, int bx0) { return aligned && by * 8 + 8 <= h && (bx0 + TILE) * 8 <= w; };

  if (warp < PROD) {
    // ---------------- producers: block b = threadIdx.x gathers its 8 pixel rows
    const int b = threadIdx.x;
    constexpr uint32_t id224 = idesc_i8(128, 224);
    uint2 pre[8];
    auto load = [&](long long ti) {
      int f, by, bx0;
      tile_at(ti, f, by, bx0);
      const uint8_t* ib = in + f * frame_stride;
      if (is_fast(by, bx0)) {
        const uint8_t* p = ib + static_cast<size_t>(by * 8) * pitch + (bx0 + b) * 8;
#pragma unroll
        for (int r = 0; r < 8; ++r) pre[r] = __ldg(reinterpret_cast<const uint2*>(p + r * pitch));
      } else {  // ragged: tile()'s edge replication, byte by byte
#pragma unroll
        for (int r = 0; r < 8; ++r) {
          const int y = min(by * 8 + r, h - 1);
          uint32_t lo = 0, hi = 0;
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const int x = min((bx0 + b) * 8 + j, w - 1);
            const uint32_t v = ib[static_cast<size_t>(y) * pitch + x];
            if (j < 4) lo |= v << (8 * j);
            else hi |= v << (8 * (j - 4));
          }
          pre[r] = make_uint2(lo, hi);
        }
      }
    };
    long long tl = 0;
    if (blockIdx.x < ntiles) load(blockIdx.x);
    for (long long ti = blockIdx.x; ti < ntiles; ti += gridDim.x, ++tl) {
      const int s = static_cast<int>(tl & 1);
      const uint32_t ph = static_cast<uint32_t>((tl >> 1) & 1);
      uint8_t* ast = asm_ + s * ABYTES;
      if (tl >= 2) mbar_wait(&a_empty[s], ph ^ 1u);
#pragma unroll
      for (int c = 0; c < 4; ++c)
        *reinterpret_cast<uint4*>(ast + b * 128 + ((c ^ (b & 7)) << 4)) =
            make_uint4(pre[2 * c].x, pre[2 * c].y, pre[2 * c + 1].x, pre[2 * c + 1].y);
      if (ti + gridDim.x < ntiles) load(ti + gridDim.x);
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      mbar_arrive(&a_full[s]);
      if (threadIdx.x == 0) {
        mbar_wait(&a_full[s], ph);
        const uint32_t sa = smem_u32(ast), sb = smem_u32(bsm);
        // one 224-column accumulator per output half: the half of tile i+1
        // only waits for the drain of the same half of tile i
#pragma unroll
        for (int hf = 0; hf < 2; ++hf) {
          if (tl >= 1) mbar_wait(&acc_empty[hf], static_cast<uint32_t>((tl - 1) & 1));
          tc_fence_after();
#pragma unroll
          for (int ks = 0; ks < 2; ++ks)
            mma_i8(tmem_base + 224 * hf, umma_desc_sw128(sa + 32 * ks),
                   umma_desc_sw128(sb + hf * 224 * 128 + 32 * ks), id224, ks);
          mma_commit(&acc_full[hf]);
        }
        mma_commit(&a_empty[s]);
      }
      __syncwarp();
    }
  } else if (warp < PROD + DRAIN) {
    // ---------------- drain: thread = block = TMEM lane; int32 partials -> FP64 Y (shared).
    // Two warps share each TMEM lane quarter and split the outputs: Y rows
    // u = 0..3 (half 0) and u = 4..7 (half 1).
    const int q = warp & 3, b = 32 * q + lane, dh = (warp - PROD) >> 2;
    const uint32_t tla = tmem_base + (static_cast<uint32_t>(32 * q) << 16);
    long long tl = 0;
    for (long long ti = blockIdx.x; ti < ntiles; ti += gridDim.x, ++tl) {
      int f, by, bx0;
      tile_at(ti, f, by, bx0);
      const int yb = static_cast<int>(tl & 1);
      uint8_t* yt = ysm + yb * YBYTES + b * 512;
      mbar_wait(&acc_full[dh], static_cast<uint32_t>(tl & 1));
      if (tl >= 2) mbar_wait(&y_empty[yb], static_cast<uint32_t>(((tl >> 1) & 1) ^ 1));
      tc_fence_after();
      double* cdst = (coef_out && bx0 + b < bw)
                         ? coef_out + ((static_cast<long long>(f) * bh + by) * bw + bx0 + b) * 64
                         : nullptr;
#pragma unroll 1
      for (int t = 2 * dh; t < 2 * dh + 2; ++t) {  // Y rows u = 2t, 2t+1 (outputs 16t .. 16t+15)
        double yr[2][8];
#pragma unroll
        for (int i = 0; i < 2; ++i) {
          const int o0 = 16 * t + 8 * i;
          // this half's accumulator: column 224*dh + 32*slice + (o & 31)
          const uint32_t col = 224 * dh + (o0 & 31);
          // exact int64 recombination: sum_s D_s 2^(7(6-s)) < 2^63, then one
          // conversion and one power-of-two scale per output
          int32_t d[8], e[8];
          long long acc[8];
          tmem_ld8(tla + col + 0 * 32, d);
          tmem_ld8(tla + col + 1 * 32, e);
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
          for (int j = 0; j < 8; ++j) acc[j] = static_cast<long long>(d[j]) * 128 + e[j];
#pragma unroll
          for (int sl = 2; sl < 6; sl += 2) {
            tmem_ld8(tla + col + sl * 32, d);
            tmem_ld8(tla + col + (sl + 1) * 32, e);
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
            for (int j = 0; j < 8; ++j) acc[j] = (acc[j] << 14) + static_cast<long long>(d[j] * 128 + e[j]);
          }
          tmem_ld8(tla + col + 6 * 32, d);
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
          for (int j = 0; j < 8; ++j)  // unscaled; 2^(e-48) is folded into the inverse constants
            yr[i][j] = static_cast<double>((acc[j] << 7) + d[j]);
        }
        // logical (row t, chunk v) = (Y[2t][v], Y[2t+1][v])
#pragma unroll
        for (int v = 0; v < 8; ++v)
          *reinterpret_cast<double2*>(yt + t * 128 + ((v ^ (2 * t) ^ fsw(b)) << 4)) =
              make_double2(yr[0][v], yr[1][v]);
        if (cdst) {
          const double sc = sc_s[0];
          double2* c2 = reinterpret_cast<double2*>(cdst + 16 * t);
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            c2[j] = make_double2(yr[0][2 * j] * sc, yr[0][2 * j + 1] * sc);
            c2[4 + j] = make_double2(yr[1][2 * j] * sc, yr[1][2 * j + 1] * sc);
          }
        }
      }
      tc_fence_before();
      mbar_arrive(&acc_empty[dh]);  // this half's TMEM free for the next tile's MMA
      mbar_arrive(&y_full[yb]);
    }
  } else {
    // ---------------- compute: inverse DCT (k_fused8's DMMA chain) of CB blocks per warp
    const int cw = warp - PROD - DRAIN;  // blocks CB*cw .. CB*cw + CB-1
    const int g = lane >> 2, t = lane & 3;
    // O = C^t (2^(e-48) Yint) C: the power of two is split between the two
    // passes' constants (exact)
    int esc;
    std::frexp(sc_s[0], &esc);  // sc = 2^(esc-1)
    const int ea = (esc - 1) / 2, eb = (esc - 1) - ea;
    const double pa = ldexp(1.0, ea), pb = ldexp(1.0, eb);
    const double ai0 = cb[(2 * t) * 8 + g] * pa, ai1 = cb[(2 * t + 1) * 8 + g] * pa;
    const double bi0 = cb[(2 * t) * 8 + g] * pb, bi1 = cb[(2 * t + 1) * 8 + g] * pb;
    uint8_t* pix = psm + cw * PIXBYTES;
    long long tl = 0;
    for (long long ti = blockIdx.x; ti < ntiles; ti += gridDim.x, ++tl) {
      int f, by, bx0;
      tile_at(ti, f, by, bx0);
      const int yb = static_cast<int>(tl & 1);
      const uint8_t* yt = ysm + yb * YBYTES;
      mbar_wait(&y_full[yb], static_cast<uint32_t>((tl >> 1) & 1));
#pragma unroll 1
      for (int bb = 0; bb < CB; bb += OZG) {
        double2 yv[OZG], z[OZG], o[OZG];
#pragma unroll
        for (int i = 0; i < OZG; ++i) {
          const int b = CB * cw + bb + i;
          yv[i] = *reinterpret_cast<const double2*>(yt + b * 512 + t * 128 + ((g ^ (2 * t) ^ fsw(b)) << 4));
        }
#pragma unroll
        for (int i = 0; i < OZG; ++i) { z[i] = make_double2(0.0, 0.0); dmma(z[i], ai0, yv[i].x); }
#pragma unroll
        for (int i = 0; i < OZG; ++i) dmma(z[i], ai1, yv[i].y);
#pragma unroll
        for (int i = 0; i < OZG; ++i) { o[i] = make_double2(0.5, 0.5); dmma(o[i], z[i].x, bi0); }
#pragma unroll
        for (int i = 0; i < OZG; ++i) dmma(o[i], z[i].y, bi1);
#pragma unroll
        for (int i = 0; i < OZG; ++i) {
          const uint32_t qv = floor_to_u8(o[i].x) | (floor_to_u8(o[i].y) << 8);
          *reinterpret_cast<uint16_t*>(pix + g * PS + 8 * (bb + i) + 2 * t) = static_cast<uint16_t>(qv);
        }
      }
      __syncwarp();
      __threadfence_block();  // this warp's Y reads have landed before the tile is released
      if (lane == 0) mbar_arrive(&y_empty[yb]);
      uint8_t* ob = out + f * frame_stride;
      const int bx = bx0 + CB * cw;
      if (is_fast(by, bx0)) {
        // 8 rows x 8*CB bytes, 16-byte chunks
#pragma unroll
        for (int ps = 0; ps < CB / 8; ++ps) {
          const int chunks = CB / 2;  // per row
          const int e = ps * 32 + lane, r = e / chunks, c = (e % chunks) * 16;
          *reinterpret_cast<uint4*>(ob + static_cast<size_t>(by * 8 + r) * pitch + bx * 8 + c) =
              *reinterpret_cast<const uint4*>(pix + r * PS + c);
        }
      } else {
        for (int e = lane; e < 8 * 8 * CB; e += 32) {
          const int r = e / (8 * CB), c = e % (8 * CB);
          const int yy = by * 8 + r, xx = bx * 8 + c;
          if (yy < h && xx < w) ob[static_cast<size_t>(yy) * pitch + xx] = pix[r * PS + c];
        }
      }
      __syncwarp();
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == PROD)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(512));
}

}  // namespace

namespace dctf {

dctf_status upload_i8_operator(dctf_plan* p) {
  std::vector<int8_t> img;
  std::vector<double> sc;
  layout_gslices_i8(p->op, p->basis, img, sc);
  cudaError_t e = cudaMalloc(&p->d_gimg, img.size());
  if (e == cudaSuccess) e = cudaMalloc(&p->d_gscale, sc.size() * sizeof(double));
  if (e == cudaSuccess) e = cudaMemcpy(p->d_gimg, img.data(), img.size(), cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMemcpy(p->d_gscale, sc.data(), sc.size() * sizeof(double), cudaMemcpyHostToDevice);
  if (e != cudaSuccess) return set_error(DCTF_CUDA_ERROR, std::string("int8 operator upload: ") + cudaGetErrorString(e));
  return DCTF_OK;
}

dctf_status launch_fused8_i8(const dctf_plan* p, const uint8_t* in, uint8_t* out, int w, int h, size_t pitch,
                             long long frame_stride, int nframes, double* coef_out, cudaStream_t st, int sms) {
  {
    const dctf_status sa = ensure_dyn_smem(reinterpret_cast<const void*>(k_fused8_i8), oz::SMEM, "k_fused8_i8");
    if (sa != DCTF_OK) return sa;
  }
  const int bw = (w + 7) / 8, bh = (h + 7) / 8, nsx = (bw + oz::TILE - 1) / oz::TILE;
  const long long ntiles = static_cast<long long>(bh) * nsx * nframes;
  if (ntiles <= 0) return DCTF_OK;
  if (ntiles >= (1LL << 31)) return set_error(DCTF_INVALID_ARGUMENT, "image batch too large (>= 2^31 work units)");
  const cudaError_t e = launch_pdl(k_fused8_i8, static_cast<unsigned>(std::min<long long>(sms, ntiles)), oz::THREADS,
                                   oz::SMEM, st, in, out, w, h, pitch, frame_stride, nframes, bw, bh, nsx,
                                   static_cast<const int8_t*>(p->d_gimg), static_cast<const double*>(p->d_gscale),
                                   static_cast<const double*>(p->d_basis), coef_out);
  add_launches(1);
  if (e != cudaSuccess) return set_error(DCTF_CUDA_ERROR, std::string("k_fused8_i8: ") + cudaGetErrorString(e));
  return DCTF_OK;
}

}  // namespace dctf
