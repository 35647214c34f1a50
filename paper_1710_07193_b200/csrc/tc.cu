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
// CTA = 12 warps, one CTA per SM, persistent over tiles of 128 blocks (MMA M):
//   warps 0-7 : two threads per tile row load X (FP64) two K-chunks ahead
//               into registers, split it into TF32 hi/lo and write the
//               swizzled A tiles; thread 0 also bulk-copies the H chunk and
//               issues the MMAs (single thread).
//   warps 8-11: epilogue — tcgen05.ld the FP32 accumulator (lanes = blocks,
//               columns = outputs), widen to FP64, stage rows in shared
//               memory and store them as coalesced 128-byte row segments.
// TMEM holds two accumulators (tile parity) so the epilogue of tile i
// overlaps the MMAs of tile i+1; shared memory holds two K-chunk stages.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <string>

#include "internal.h"

namespace {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ uint8_t* align1024(uint8_t* smem) {
  const uint32_t pad = (1024u - (smem_u32(smem) & 1023u)) & 1023u;
  return smem + pad;
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
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
__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// UMMA shared-memory descriptor, K-major, 128B swizzle: rows of 128 bytes,
// 8-row atoms 1024 B apart (SBO), version 1 (sm_100), layout type 2.
__device__ __forceinline__ uint64_t umma_desc_sw128(uint32_t saddr) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((saddr >> 4) & 0x3FFFu);
  d |= static_cast<uint64_t>(1u) << 16;             // LBO (unused for swizzled K-major)
  d |= static_cast<uint64_t>(1024u >> 4) << 32;     // SBO
  d |= static_cast<uint64_t>(1u) << 46;             // version
  d |= static_cast<uint64_t>(2u) << 61;             // SWIZZLE_128B
  return d;
}

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
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}

// tf32 hi/lo split of a double: hi = rna_tf32(float(x)), lo = rna_tf32(float(x - hi)).
__device__ __forceinline__ void split_tf32(double x, float& hi, float& lo) {
  uint32_t h, l;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(h) : "f"(__double2float_rn(x)));
  hi = __uint_as_float(h);
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(l) : "f"(__double2float_rn(x - static_cast<double>(hi))));
  lo = __uint_as_float(l);
}

template <int NN>
struct TcCfg {
  static constexpr int TILE = 128;          // MMA M (blocks per tile)
  static constexpr int KCH = NN / 32;       // K chunks of 32 TF32 (128 B rows)
  static constexpr int ABYTES = TILE * 128;
  static constexpr int BBYTES = NN * 128;
  static constexpr int STAGE = 2 * ABYTES + 2 * BBYTES;
  static constexpr int STAGES = 2;
  static constexpr int TMEM_COLS = 2 * NN <= 128 ? 128 : (2 * NN <= 256 ? 256 : 512);
  static constexpr int CONV_WARPS = 8;      // converter warps (2 threads per tile row)
  static constexpr int EPI_WARPS = 4;       // epilogue warps (one TMEM lane quarter each)
  static constexpr int THREADS = 32 * (CONV_WARPS + EPI_WARPS);
  static constexpr int EPI_STRIDE = 144;    // 16 doubles + 16 B pad per staged row
  static constexpr int EPI_BYTES = 32 * EPI_STRIDE;
  static constexpr int SMEM = 1024 + STAGES * STAGE + EPI_WARPS * EPI_BYTES;
};

template <int NN>
__global__ void __launch_bounds__(TcCfg<NN>::THREADS, 1)
    k_coef_tf32x3(const double* __restrict__ x, const float* __restrict__ hsplit,
                  double* __restrict__ y, long long nblocks) {
  using Cfg = TcCfg<NN>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* base = align1024(smem_raw);
  uint8_t* epi = base + Cfg::STAGES * Cfg::STAGE;
  __shared__ uint64_t a_full[2], b_full[2], empty[2], acc_full[2], acc_empty[2];
  __shared__ uint32_t tmem_base_s;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(&tmem_base_s)),
                 "r"(Cfg::TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 32) {
    for (int i = 0; i < 2; ++i) {
      mbar_init(&a_full[i], 32 * Cfg::CONV_WARPS);
      mbar_init(&b_full[i], 1);
      mbar_init(&empty[i], 1);
      mbar_init(&acc_full[i], 1);
      mbar_init(&acc_empty[i], 32 * Cfg::EPI_WARPS);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = tmem_base_s;
  const long long ntiles = (nblocks + Cfg::TILE - 1) / Cfg::TILE;
  const long long my_tiles = ntiles > blockIdx.x ? (ntiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  const long long nchunks = my_tiles * Cfg::KCH;

  if (warp < Cfg::CONV_WARPS) {
    // ---------------- converters (+ thread 0: B loads and MMA issue)
    const int r = threadIdx.x >> 1, hh = threadIdx.x & 1;  // tile row, half of the 32-wide chunk
    constexpr uint32_t idesc = idesc_tf32(128, NN);
    auto load = [&](long long c, double2 (&pre)[8]) {
      const long long tile = blockIdx.x + (c / Cfg::KCH) * gridDim.x;
      const int kc = static_cast<int>(c % Cfg::KCH);
      const long long blk = tile * Cfg::TILE + r;
      if (c < nchunks && blk < nblocks) {
        const double2* src = reinterpret_cast<const double2*>(x + blk * NN + 32 * kc + 16 * hh);
#pragma unroll
        for (int j = 0; j < 8; ++j) pre[j] = __ldg(src + j);
      } else {
#pragma unroll
        for (int j = 0; j < 8; ++j) pre[j] = make_double2(0.0, 0.0);
      }
    };
    auto step = [&](long long c, double2 (&pre)[8]) {
      const int s = static_cast<int>(c & 1);
      const uint32_t ph = static_cast<uint32_t>((c >> 1) & 1);
      const long long ti = c / Cfg::KCH;
      const int kc = static_cast<int>(c % Cfg::KCH);
      const int ab = static_cast<int>(ti & 1);
      uint8_t* st = base + s * Cfg::STAGE;
      if (c >= 2) mbar_wait(&empty[s], ph ^ 1u);  // MMAs of chunk c-2 retired
      if (threadIdx.x == 0) {
        mbar_expect_tx(&b_full[s], 2 * Cfg::BBYTES);
        const float* hs = hsplit + static_cast<size_t>(kc) * 2 * (Cfg::BBYTES / 4);
        bulk_load(st + 2 * Cfg::ABYTES, hs, Cfg::BBYTES, &b_full[s]);
        bulk_load(st + 2 * Cfg::ABYTES + Cfg::BBYTES, hs + Cfg::BBYTES / 4, Cfg::BBYTES, &b_full[s]);
      }
      uint8_t* ah = st + r * 128;
      uint8_t* al = st + Cfg::ABYTES + r * 128;
#pragma unroll
      for (int c4 = 0; c4 < 4; ++c4) {
        float4 h4, l4;
        split_tf32(pre[2 * c4].x, h4.x, l4.x);
        split_tf32(pre[2 * c4].y, h4.y, l4.y);
        split_tf32(pre[2 * c4 + 1].x, h4.z, l4.z);
        split_tf32(pre[2 * c4 + 1].y, h4.w, l4.w);
        const int off = ((4 * hh + c4) ^ (r & 7)) << 4;
        *reinterpret_cast<float4*>(ah + off) = h4;
        *reinterpret_cast<float4*>(al + off) = l4;
      }
      load(c + 2, pre);  // two chunks in flight per thread
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      mbar_arrive(&a_full[s]);
      if (threadIdx.x == 0) {
        mbar_wait(&a_full[s], ph);
        mbar_wait(&b_full[s], ph);
        if (kc == 0 && ti >= 2) mbar_wait(&acc_empty[ab], static_cast<uint32_t>(((ti >> 1) & 1) ^ 1));
        tc_fence_after();
        const uint32_t sa = smem_u32(st);
        const uint32_t d = tmem_base + static_cast<uint32_t>(ab * NN);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const uint64_t ah_d = umma_desc_sw128(sa + 32 * k);
          const uint64_t al_d = umma_desc_sw128(sa + Cfg::ABYTES + 32 * k);
          const uint64_t bh_d = umma_desc_sw128(sa + 2 * Cfg::ABYTES + 32 * k);
          const uint64_t bl_d = umma_desc_sw128(sa + 2 * Cfg::ABYTES + Cfg::BBYTES + 32 * k);
          mma_tf32(d, ah_d, bh_d, idesc, (kc | k) != 0);
          mma_tf32(d, ah_d, bl_d, idesc, 1);
          mma_tf32(d, al_d, bh_d, idesc, 1);
        }
        mma_commit(&empty[s]);
        if (kc == Cfg::KCH - 1) mma_commit(&acc_full[ab]);
      }
      __syncwarp();
    };
    double2 pre0[8], pre1[8];
    load(0, pre0);
    load(1, pre1);
    for (long long c = 0; c < nchunks; c += 2) {
      step(c, pre0);
      if (c + 1 < nchunks) step(c + 1, pre1);
    }
  } else {
    // ---------------- epilogue: TMEM -> FP64 -> staged rows -> coalesced stores
    const int q = warp & 3;  // TMEM lane quarter this warp may access
    uint8_t* stg = epi + (warp - Cfg::CONV_WARPS) * Cfg::EPI_BYTES;
    int ti = 0;
    for (long long tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++ti) {
      const int ab = ti & 1;
      mbar_wait(&acc_full[ab], static_cast<uint32_t>((ti >> 1) & 1));
      tc_fence_after();
      const long long row0 = tile * Cfg::TILE + 32 * q;  // first block of this warp's 32 rows
#pragma unroll 1
      for (int c = 0; c < NN / 16; ++c) {
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
        // 32 rows x 128 B: 8 lanes per row, 4 rows per pass
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

// H split image for k_coef_tf32x3: [kc][part h/l][row n < NN][32 TF32 of
// columns 32kc..] with the 128B swizzle applied (16-byte chunk c of row n at
// chunk c ^ (n & 7)), i.e. exactly the shared-memory tile the UMMA B
// descriptor reads.
void layout_hsplit_tf32(int n, const std::vector<double>& op, std::vector<float>& out) {
  const int nn = n * n, kch = nn / 32;
  out.assign(static_cast<size_t>(kch) * 2 * nn * 32, 0.0f);
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
      for (int k = 0; k < 32; ++k) {
        const double v = op[static_cast<size_t>(row) * nn + 32 * kc + k];
        const float hi = rna_tf32(static_cast<float>(v));
        const float lo = rna_tf32(static_cast<float>(v - static_cast<double>(hi)));
        const size_t pos = static_cast<size_t>(row) * 32 + (((k >> 2) ^ (row & 7)) << 2) + (k & 3);
        out[(static_cast<size_t>(kc) * 2 + 0) * nn * 32 + pos] = hi;
        out[(static_cast<size_t>(kc) * 2 + 1) * nn * 32 + pos] = lo;
      }
}

dctf_status launch_coef_tf32x3(const dctf_plan* p, const double* d_in, double* d_out, long long nb,
                               cudaStream_t st, int sms) {
  if (nb == 0) return DCTF_OK;
  if (p->n == 8) {
    using Cfg = TcCfg<64>;
    static bool attr = false;
    if (!attr) {
      if (cudaFuncSetAttribute(k_coef_tf32x3<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM) != cudaSuccess)
        return set_error(DCTF_CUDA_ERROR, "cudaFuncSetAttribute(k_coef_tf32x3<64>)");
      attr = true;
    }
    const long long ntiles = (nb + Cfg::TILE - 1) / Cfg::TILE;
    k_coef_tf32x3<64><<<static_cast<unsigned>(std::min<long long>(sms, ntiles)), Cfg::THREADS, Cfg::SMEM, st>>>(
        d_in, static_cast<const float*>(p->d_hsplit), d_out, nb);
  } else {
    using Cfg = TcCfg<256>;
    static bool attr = false;
    if (!attr) {
      if (cudaFuncSetAttribute(k_coef_tf32x3<256>, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM) != cudaSuccess)
        return set_error(DCTF_CUDA_ERROR, "cudaFuncSetAttribute(k_coef_tf32x3<256>)");
      attr = true;
    }
    const long long ntiles = (nb + Cfg::TILE - 1) / Cfg::TILE;
    k_coef_tf32x3<256><<<static_cast<unsigned>(std::min<long long>(sms, ntiles)), Cfg::THREADS, Cfg::SMEM, st>>>(
        d_in, static_cast<const float*>(p->d_hsplit), d_out, nb);
  }
  add_launches(1);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return set_error(DCTF_CUDA_ERROR, std::string("k_coef_tf32x3: ") + cudaGetErrorString(e));
  return DCTF_OK;
}

}  // namespace dctf
