// Split-precision (3xTF32) DCT-domain filter on the 5th-generation tensor
// cores: tcgen05.mma kind::tf32, FP32 accumulators in TMEM, sm_100a.
//
// FilterPlan::filter_coeffs (filter.hpp:65-67) as Y^T = X^T H^T with
//   X = Xh + Xl, H = Hh + Hl (TF32 hi/lo splits of the FP64 values),
//   Y ~= Xh Hh + Xh Hl + Xl Hh        (3 MMA passes, FP32 accumulate),
// giving ~1e-7 relative accuracy (reported by tests/bench; the FP64 DMMA
// kernels are the exact path). The FP64 -> TF32 split of X happens on the
// fly; H's split is done once per plan on the host and stored as the exact
// 128B-swizzled shared-memory image the UMMA descriptors expect, so it is
// streamed with plain bulk copies.
//
// CTA = 15 warps, one CTA per SM, persistent over tiles of 128 blocks (MMA
// M), K streamed in chunks of 16:
//   warp 8     X producer: TMA loads of the raw FP64 X chunk (128 blocks x 16
//              coefficients, 128B swizzle) into the staging ring (XS deep, so
//              HBM latency is covered independently of the operand ring).
//   warp 9     H producer: bulk copies of the H hi/lo chunk into the operand ring.
//   warps 0-7  converters: FP64 staging -> TF32 hi/lo operand cores
//              (canonical no-swizzle K-major layout, 8-row x 16-byte cores).
//   warp 10    single-thread tcgen05.mma issue (3 passes x 2 K-steps per chunk).
//   warps 11-14 epilogue: tcgen05.ld the FP32 accumulator (lanes = blocks,
//              columns = outputs), widen to FP64, stage rows in shared
//              memory, store them as coalesced 128-byte row segments.
// TMEM holds two accumulators (tile parity) so the epilogue of tile i
// overlaps the MMAs of tile i+1; shared memory holds two K-chunk stages.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <string>

#include "device.cuh"
#include "internal.h"

namespace {

// Instruction descriptor: kind::tf32, A/B TF32 K-major, D FP32, M x N.
__host__ __device__ constexpr uint32_t idesc_tf32(int m, int n) {
  return (1u << 4) | (2u << 7) | (2u << 10) | (static_cast<uint32_t>(n >> 3) << 17) |
         (static_cast<uint32_t>(m >> 4) << 24);
}

__device__ __forceinline__ void mma_tf32(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                         uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}

// tf32 hi/lo split of a double: hi = rna_tf32(float(x)), lo = rna_tf32(float(x - hi)).
// x ~= hi + lo with hi, lo TF32. The split runs in FP32 after one rounding
// of x to float (relative 2^-24, far below the 3xTF32 truncation of the
// dropped lo*lo term), so each element costs one FP64-pipe conversion
// instead of three plus a DADD.
__device__ __forceinline__ void split_tf32(double x, float& hi, float& lo) {
  const float xf = __double2float_rn(x);
  uint32_t h, l;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(h) : "f"(xf));
  hi = __uint_as_float(h);
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(l) : "f"(xf - hi));
  lo = __uint_as_float(l);
}

// bf16 hi/lo split, same scheme: x ~= hi + lo, both bf16 (8 significant bits
// each), after one rounding of x to float.
__device__ __forceinline__ void split_bf16(double x, uint32_t& hi, uint32_t& lo) {
  const float xf = __double2float_rn(x);
  const __nv_bfloat16 h = __float2bfloat16_rn(xf);
  const __nv_bfloat16 l = __float2bfloat16_rn(xf - __bfloat162float(h));
  hi = __bfloat16_as_ushort(h);
  lo = __bfloat16_as_ushort(l);
}

// Instruction descriptor: kind::f16 with BF16 A/B (K-major), D FP32, M x N.
__host__ __device__ constexpr uint32_t idesc_bf16(int m, int n) {
  return (1u << 4) | (1u << 7) | (1u << 10) | (static_cast<uint32_t>(n >> 3) << 17) |
         (static_cast<uint32_t>(m >> 4) << 24);
}
__device__ __forceinline__ void mma_bf16(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                         uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}

// UMMA shared-memory descriptor, K-major, no swizzle: 8-row x 16-byte core
// matrices, LBO = 128 B between K-adjacent cores, SBO = 8 rows x (bytes of a
// 16-wide K chunk row) between 8-row groups — 512 B for TF32, 256 B for
// BF16 — version 1, layout type 0.
template <int SBO>
__device__ __forceinline__ uint64_t umma_desc_k16(uint32_t saddr) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((saddr >> 4) & 0x3FFFu);
  d |= static_cast<uint64_t>(128u >> 4) << 16;            // LBO
  d |= static_cast<uint64_t>(static_cast<uint32_t>(SBO) >> 4) << 32;  // SBO
  d |= static_cast<uint64_t>(1u) << 46;                   // version
  return d;
}

template <int NN, bool BF>
struct TcCfg {
  static constexpr int TILE = 128;          // MMA M (blocks per tile)
  static constexpr int KCH = NN / 16;       // K chunks of 16
  static constexpr int ROWB = BF ? 32 : 64; // bytes of one operand row of a chunk
  static constexpr int SBO = 8 * ROWB;      // 8-row group stride
  static constexpr int KSTEPS = BF ? 1 : 2; // MMAs per chunk and pass (K = 16 bf16 / 8 tf32)
  static constexpr int XBYTES = TILE * 128; // FP64 chunk staging (TMA box 128 rows x 16 doubles, SW128)
  static constexpr int ABYTES = TILE * ROWB;  // one split part of A
  static constexpr int BBYTES = NN * ROWB;    // one split part of B
  static constexpr int XS = NN == 64 ? 8 : 5;  // FP64 staging stages (HBM latency cover)
  static constexpr int AS = NN == 64 ? 3 : 2;  // operand stages
  static constexpr int OPBYTES = 2 * ABYTES + 2 * BBYTES;
  static constexpr int CONV_WARPS = 8;
  static constexpr int XPROD_WARP = CONV_WARPS, BPROD_WARP = CONV_WARPS + 1, MMA_WARP = CONV_WARPS + 2,
                       EPI0 = CONV_WARPS + 3;
  static constexpr int EPI_WARPS = 4;
  static constexpr int THREADS = 32 * (EPI0 + EPI_WARPS);
  static constexpr int TMEM_COLS = 2 * NN <= 128 ? 128 : (2 * NN <= 256 ? 256 : 512);
  static constexpr int EPI_STRIDE = 144;    // 16 doubles + 16 B pad per staged row
  static constexpr int EPI_BYTES = 32 * EPI_STRIDE;
  static constexpr int SMEM = 1024 + XS * XBYTES + AS * OPBYTES + EPI_WARPS * EPI_BYTES;
};

template <int NN, bool BF>
__global__ void __launch_bounds__(TcCfg<NN, BF>::THREADS, 1)
    k_coef_split3(const __grid_constant__ CUtensorMap xmap, const uint8_t* __restrict__ hsplit,
                  double* __restrict__ y, long long nblocks) {
  pdl_trigger();
  using Cfg = TcCfg<NN, BF>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* base = align1024(smem_raw);
  uint8_t* xst = base;                               // FP64 staging ring
  uint8_t* ops = xst + Cfg::XS * Cfg::XBYTES;        // operand ring: [Ah | Al | Bh | Bl]
  uint8_t* epi = ops + Cfg::AS * Cfg::OPBYTES;
  __shared__ uint64_t x_full[Cfg::XS], x_empty[Cfg::XS], a_full[Cfg::AS], b_full[Cfg::AS], a_empty[Cfg::AS];
  __shared__ uint64_t acc_full[2], acc_empty[2];
  __shared__ uint32_t tmem_base_s;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(&tmem_base_s)),
                 "r"(Cfg::TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 32) {
    for (int i = 0; i < Cfg::XS; ++i) {
      mbar_init(&x_full[i], 1);
      mbar_init(&x_empty[i], Cfg::CONV_WARPS);
    }
    for (int i = 0; i < Cfg::AS; ++i) {
      mbar_init(&a_full[i], 32 * Cfg::CONV_WARPS);
      mbar_init(&b_full[i], 1);
      mbar_init(&a_empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&acc_full[i], 1);
      mbar_init(&acc_empty[i], 32 * Cfg::EPI_WARPS);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = tmem_base_s;
  pdl_wait();
  const long long ntiles = (nblocks + Cfg::TILE - 1) / Cfg::TILE;
  const long long my_tiles = ntiles > blockIdx.x ? (ntiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  const long long nchunks = my_tiles * Cfg::KCH;

  if (warp == Cfg::XPROD_WARP) {
    // ---------------- X producer: TMA loads of raw FP64 chunks, XS ahead
    if (lane == 0) {
      for (long long c = 0; c < nchunks; ++c) {
        const long long tile = blockIdx.x + (c / Cfg::KCH) * gridDim.x;
        const int kc = static_cast<int>((c + tile) % Cfg::KCH), xs = static_cast<int>(c % Cfg::XS);
        if (c >= Cfg::XS) mbar_wait(&x_empty[xs], static_cast<uint32_t>(((c / Cfg::XS) - 1) & 1));
        mbar_expect_tx(&x_full[xs], Cfg::XBYTES);
        tma_load_2d(xst + xs * Cfg::XBYTES, &xmap, &x_full[xs], 16 * kc, static_cast<int>(tile * Cfg::TILE));
      }
    }
  } else if (warp == Cfg::BPROD_WARP) {
    // ---------------- H producer: bulk copies of the hi/lo chunk, AS ahead
    if (lane == 0) {
      for (long long c = 0; c < nchunks; ++c) {
        const long long tile = blockIdx.x + (c / Cfg::KCH) * gridDim.x;
        const int kc = static_cast<int>((c + tile) % Cfg::KCH), as = static_cast<int>(c % Cfg::AS);
        if (c >= Cfg::AS) mbar_wait(&a_empty[as], static_cast<uint32_t>(((c / Cfg::AS) - 1) & 1));
        const uint8_t* hs = hsplit + static_cast<size_t>(kc) * 2 * Cfg::BBYTES;
        mbar_expect_tx(&b_full[as], 2 * Cfg::BBYTES);
        bulk_load(ops + as * Cfg::OPBYTES + 2 * Cfg::ABYTES, hs, 2 * Cfg::BBYTES, &b_full[as]);
      }
    }
  } else if (warp == Cfg::MMA_WARP) {
    // ---------------- single-thread MMA issue
    if (lane == 0) {
      constexpr uint32_t idesc = BF ? idesc_bf16(128, NN) : idesc_tf32(128, NN);
      for (long long c = 0; c < nchunks; ++c) {
        const long long ti = c / Cfg::KCH;
        const int j = static_cast<int>(c % Cfg::KCH), as = static_cast<int>(c % Cfg::AS);
        const int ab = static_cast<int>(ti & 1);
        const uint32_t ph = static_cast<uint32_t>((c / Cfg::AS) & 1);
        mbar_wait(&a_full[as], ph);
        mbar_wait(&b_full[as], ph);
        if (j == 0 && ti >= 2) mbar_wait(&acc_empty[ab], static_cast<uint32_t>(((ti >> 1) & 1) ^ 1));
        tc_fence_after();
        const uint32_t so = smem_u32(ops + as * Cfg::OPBYTES);
        const uint32_t d = tmem_base + static_cast<uint32_t>(ab * NN);
#pragma unroll
        for (int ks = 0; ks < Cfg::KSTEPS; ++ks) {
          const uint32_t koff = 256u * ks;  // two 16-byte cores per K step
          const uint64_t ah = umma_desc_k16<Cfg::SBO>(so + koff);
          const uint64_t al = umma_desc_k16<Cfg::SBO>(so + Cfg::ABYTES + koff);
          const uint64_t bh = umma_desc_k16<Cfg::SBO>(so + 2 * Cfg::ABYTES + koff);
          const uint64_t bl = umma_desc_k16<Cfg::SBO>(so + 2 * Cfg::ABYTES + Cfg::BBYTES + koff);
          if (BF) {
            mma_bf16(d, ah, bh, idesc, (j | ks) != 0);
            mma_bf16(d, ah, bl, idesc, 1);
            mma_bf16(d, al, bh, idesc, 1);
          } else {
            mma_tf32(d, ah, bh, idesc, (j | ks) != 0);
            mma_tf32(d, ah, bl, idesc, 1);
            mma_tf32(d, al, bh, idesc, 1);
          }
        }
        mma_commit(&a_empty[as]);
        if (j == Cfg::KCH - 1) mma_commit(&acc_full[ab]);
      }
    }
  } else if (warp < Cfg::CONV_WARPS) {
    // ---------------- converters: FP64 staging -> TF32 / BF16 hi/lo operand cores
    const int r = threadIdx.x & (Cfg::TILE - 1), kp = threadIdx.x >> 7;  // row, K-core pair (TF32) / core (BF16)
    for (long long c = 0; c < nchunks; ++c) {
      const int xs = static_cast<int>(c % Cfg::XS), as = static_cast<int>(c % Cfg::AS);
      mbar_wait(&x_full[xs], static_cast<uint32_t>((c / Cfg::XS) & 1));
      if (c >= Cfg::AS) mbar_wait(&a_empty[as], static_cast<uint32_t>(((c / Cfg::AS) - 1) & 1));
      const uint8_t* xrow = xst + xs * Cfg::XBYTES + r * 128;
      uint8_t* op = ops + as * Cfg::OPBYTES;
      if (BF) {
        // one 16-byte core = 8 bf16 = K 8kp .. 8kp+7 (FP64 chunks 4kp .. 4kp+3)
        uint32_t hw[4], lw[4];
#pragma unroll
        for (int m = 0; m < 4; ++m) {
          const double2 v = *reinterpret_cast<const double2*>(xrow + (((4 * kp + m) ^ (r & 7)) << 4));
          uint32_t h0, l0, h1, l1;
          split_bf16(v.x, h0, l0);
          split_bf16(v.y, h1, l1);
          hw[m] = h0 | (h1 << 16);
          lw[m] = l0 | (l1 << 16);
        }
        const int off = (r >> 3) * Cfg::SBO + kp * 128 + (r & 7) * 16;
        *reinterpret_cast<uint4*>(op + off) = make_uint4(hw[0], hw[1], hw[2], hw[3]);
        *reinterpret_cast<uint4*>(op + Cfg::ABYTES + off) = make_uint4(lw[0], lw[1], lw[2], lw[3]);
      } else
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        const int kk = 2 * kp + i;  // 16-byte TF32 core column = K 4kk..4kk+3
        const double2 v0 = *reinterpret_cast<const double2*>(xrow + (((2 * kk) ^ (r & 7)) << 4));
        const double2 v1 = *reinterpret_cast<const double2*>(xrow + (((2 * kk + 1) ^ (r & 7)) << 4));
        float4 h4, l4;
        split_tf32(v0.x, h4.x, l4.x);
        split_tf32(v0.y, h4.y, l4.y);
        split_tf32(v1.x, h4.z, l4.z);
        split_tf32(v1.y, h4.w, l4.w);
        const int off = (r >> 3) * Cfg::SBO + kk * 128 + (r & 7) * 16;
        *reinterpret_cast<float4*>(op + off) = h4;
        *reinterpret_cast<float4*>(op + Cfg::ABYTES + off) = l4;
      }
      // release the FP64 stage once this warp's reads have landed
      __syncwarp();
      __threadfence_block();
      if (lane == 0) mbar_arrive(&x_empty[xs]);
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      mbar_arrive(&a_full[as]);
    }
  } else {
    // ---------------- epilogue: TMEM -> FP64 -> staged rows -> coalesced stores
    const int q = warp & 3;
    uint8_t* stg = epi + (warp - Cfg::EPI0) * Cfg::EPI_BYTES;
    int ti = 0;
    for (long long tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++ti) {
      const int ab = ti & 1;
      mbar_wait(&acc_full[ab], static_cast<uint32_t>((ti >> 1) & 1));
      tc_fence_after();
      const long long row0 = tile * Cfg::TILE + 32 * q;
#pragma unroll 1
      for (int c0 = 0; c0 < NN / 16; ++c0) {
        // rotate the column order per quarter and tile: spreads the strided
        // row segments of concurrent stores over more DRAM channels
        const int c = (c0 + q + static_cast<int>(tile)) % (NN / 16);
        uint32_t v[16];
        const uint32_t taddr = tmem_base + (static_cast<uint32_t>(32 * q) << 16) +
                               static_cast<uint32_t>(ab * NN + 16 * c);
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
            : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
              "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),
              "=r"(v[14]), "=r"(v[15])
            : "r"(taddr));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        double2* myrow = reinterpret_cast<double2*>(stg + lane * Cfg::EPI_STRIDE);
#pragma unroll
        for (int j = 0; j < 8; ++j)
          myrow[j] = make_double2(static_cast<double>(__uint_as_float(v[2 * j])),
                                  static_cast<double>(__uint_as_float(v[2 * j + 1])));
        __syncwarp();
#pragma unroll
        for (int ps = 0; ps < 8; ++ps) {
          const int rr = 4 * ps + (lane >> 3), ch = lane & 7;
          const long long blk = row0 + rr;
          if (blk < nblocks)
            *reinterpret_cast<double2*>(y + blk * NN + 16 * c + 2 * ch) =
                *reinterpret_cast<const double2*>(stg + rr * Cfg::EPI_STRIDE + ch * 16);
        }
        __syncwarp();
      }
      tc_fence_before();
      mbar_arrive(&acc_empty[ab]);
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                 "r"(Cfg::TMEM_COLS));
}

}  // namespace

namespace dctf {

// H split image for k_coef_tf32x3: [kc < NN/16][part h/l][row n < NN] in the
// canonical no-swizzle K-major UMMA layout of a 16-wide K chunk: 8-row x
// 16-byte core matrices, core (n/8, kk) at byte (n/8)*512 + kk*128, row n%8
// at +16*(n%8) (LBO = 128 B between K-adjacent cores, SBO = 512 B between
// 8-row groups), i.e. exactly the shared-memory tile the UMMA B descriptor
// reads, so each chunk is one plain bulk copy.
void layout_hsplit_tf32(int n, const std::vector<double>& op, std::vector<float>& out) {
  const int nn = n * n, kch = nn / 16;
  out.assign(static_cast<size_t>(kch) * 2 * nn * 16, 0.0f);
  auto rna_tf32 = [](float f) {
    uint32_t u;
    std::memcpy(&u, &f, 4);
    if ((u & 0x7f800000u) != 0x7f800000u) u = (u + 0x1000u) & 0xffffe000u;  // round half away
    float r;
    std::memcpy(&r, &u, 4);
    return r;
  };
  for (int kc = 0; kc < kch; ++kc)
    for (int row = 0; row < nn; ++row)
      for (int k = 0; k < 16; ++k) {
        const double v = op[static_cast<size_t>(row) * nn + 16 * kc + k];
        const float hi = rna_tf32(static_cast<float>(v));
        const float lo = rna_tf32(static_cast<float>(v - static_cast<double>(hi)));
        const size_t pos = static_cast<size_t>(row >> 3) * 128 + (k >> 2) * 32 + (row & 7) * 4 + (k & 3);
        out[(static_cast<size_t>(kc) * 2 + 0) * nn * 16 + pos] = hi;
        out[(static_cast<size_t>(kc) * 2 + 1) * nn * 16 + pos] = lo;
      }
}

// BF16 version of the same image: rows of 32 B (16 bf16), core (n/8, kk) at
// byte (n/8)*256 + kk*128, row n%8 at +16*(n%8), element k%8 at +2*(k%8).
void layout_hsplit_bf16(int n, const std::vector<double>& op, std::vector<uint16_t>& out) {
  const int nn = n * n, kch = nn / 16;
  out.assign(static_cast<size_t>(kch) * 2 * nn * 16, 0);
  auto bf16_rn = [](float f) -> uint16_t {
    uint32_t u;
    std::memcpy(&u, &f, 4);
    if ((u & 0x7f800000u) == 0x7f800000u) return static_cast<uint16_t>(u >> 16);
    u += 0x7fffu + ((u >> 16) & 1u);  // round to nearest even
    return static_cast<uint16_t>(u >> 16);
  };
  auto bf16_f = [](uint16_t h) {
    const uint32_t u = static_cast<uint32_t>(h) << 16;
    float f;
    std::memcpy(&f, &u, 4);
    return f;
  };
  for (int kc = 0; kc < kch; ++kc)
    for (int row = 0; row < nn; ++row)
      for (int k = 0; k < 16; ++k) {
        const double v = op[static_cast<size_t>(row) * nn + 16 * kc + k];
        const float vf = static_cast<float>(v);
        const uint16_t hi = bf16_rn(vf);
        const uint16_t lo = bf16_rn(vf - bf16_f(hi));
        const size_t pos = static_cast<size_t>(row >> 3) * 128 + (k >> 3) * 64 + (row & 7) * 8 + (k & 7);
        out[(static_cast<size_t>(kc) * 2 + 0) * nn * 16 + pos] = hi;
        out[(static_cast<size_t>(kc) * 2 + 1) * nn * 16 + pos] = lo;
      }
}

dctf_status launch_coef_tf32x3(const dctf_plan* p, const double* d_in, double* d_out, long long nb,
                               cudaStream_t st, int sms) {
  if (nb == 0) return DCTF_OK;
  CUtensorMap map;
  const int nn = p->n * p->n;
  const dctf_status s = make_xmap(&map, d_in, nb, nn, 128);
  if (s != DCTF_OK) return s;
  auto run = [&](auto kernel, int smem, int threads) -> dctf_status {
    const dctf_status sa = ensure_dyn_smem(reinterpret_cast<const void*>(kernel), smem, "k_coef_split3");
    if (sa != DCTF_OK) return sa;
    const long long ntiles = (nb + 127) / 128;
    const cudaError_t e = launch_pdl(kernel, static_cast<unsigned>(std::min<long long>(sms, ntiles)), threads, smem,
                                     st, map, static_cast<const uint8_t*>(p->d_hsplit), d_out, nb);
    if (e != cudaSuccess) return set_error(DCTF_CUDA_ERROR, std::string("k_coef_split3: ") + cudaGetErrorString(e));
    return DCTF_OK;
  };
  const bool bf = p->precision == DCTF_PREC_BF16X3;
  dctf_status r;
  if (p->n == 8)
    r = bf ? run(k_coef_split3<64, true>, TcCfg<64, true>::SMEM, TcCfg<64, true>::THREADS)
           : run(k_coef_split3<64, false>, TcCfg<64, false>::SMEM, TcCfg<64, false>::THREADS);
  else
    r = bf ? run(k_coef_split3<256, true>, TcCfg<256, true>::SMEM, TcCfg<256, true>::THREADS)
           : run(k_coef_split3<256, false>, TcCfg<256, false>::SMEM, TcCfg<256, false>::THREADS);
  if (r != DCTF_OK) return r;
  add_launches(1);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return set_error(DCTF_CUDA_ERROR, std::string("k_coef_split3: ") + cudaGetErrorString(e));
  return DCTF_OK;
}

}  // namespace dctf
