// Spatial path, register-tiled (convolve,
// spatial.hpp:41-68, and filter_image's Domain::kSpatial, image.hpp:219-222).
//
// k_spatial_rows<N, K, REP, U8>: persistent, one thread per block ROW. A CTA
// stages batches of 256 / N blocks as FP64 samples in shared memory (u8 image
// through tile()'s edge replication, or FP64 blocks; each thread fetches its
// own block row of the NEXT batch into registers before computing the current
// one), then each thread loads the K source rows
// its output row needs into registers, one row at a time, and accumulates the
// N outputs of its row with the mask taps taken straight from the constant
// bank (the weights travel as a by-value kernel parameter). Per sample the
// taps are accumulated r ascending, c ascending with separately rounded
// multiply and add, out-of-block taps dropped (zero) or clamped (replicate)
// -- the reference's order, so every sample is bit-identical to convolve and
// to the generic one-thread-per-sample k_spatial (capi.cu), which still
// serves mask shapes this file does not instantiate.
//
// Cost model ("Spatial path"): 2 FP64 instructions (DMUL + DADD)
// per tap, K^2 N^2 taps per block, so the FP64 pipe bounds the kernel; shared
// memory serves N doubles per N*K taps, HBM carries N^2 bytes in and out.
#include "internal.h"
#include "device.cuh"
#include "fastdiv.cuh"

#include <cstdlib>

namespace {

constexpr int SP_THREADS = 256;

template <int KR, int KC>
struct SpWeights {
  double w[KR * KC];
};

template <int N>
struct SpCfg {
  static constexpr int BPC = SP_THREADS / N;  // blocks per CTA, one thread per block row
  static constexpr int RS = N + 2;            // smem row stride in doubles: rows of one block
                                              // land in distinct 16-B bank groups
  static constexpr int BS = N * RS;           // smem block stride
  static constexpr int LOGN = N == 8 ? 3 : 4;
};

template <int N, int KR, int KC, bool REP, bool U8>
__global__ void __launch_bounds__(SP_THREADS) k_spatial_rows(const uint8_t* __restrict__ img, int w, int h,
                                                             size_t pitch, int bw,
                                                             const double* __restrict__ blocks,
                                                             uint8_t* __restrict__ out_img,
                                                             double* __restrict__ out_blocks, long long nblocks,
                                                             long long nbatches, const SpWeights<KR, KC> wt,
                                                             int* nan_flag) {
  using C = SpCfg<N>;
  __shared__ __align__(16) double tile[C::BPC * C::BS];
  const int b = threadIdx.x >> C::LOGN, i = threadIdx.x & (N - 1);
  double* my_row = tile + b * C::BS + i * C::RS;
  const dctf::FastDiv fbw = dctf::make_fastdiv(static_cast<uint32_t>(bw));

  // Staging registers: this thread's block row of the next batch (N bytes or
  // N doubles), fetched before the current batch is computed so the HBM
  // latency hides behind the FP64 work.
  uint32_t raw[U8 ? N / 4 : 1];
  double rawd[U8 ? 1 : N];
  bool f_valid = false;
  int f_y0 = 0, f_x0 = 0;
  auto fetch = [&](long long batch) {
    const long long blk = batch * C::BPC + b;
    f_valid = blk < nblocks;
    if (!f_valid) return;
    if (U8) {
      const uint32_t by = dctf::fdiv(fbw, static_cast<uint32_t>(blk));  // nblocks < 2^31 (launcher)
      f_y0 = static_cast<int>(by) * N;
      f_x0 = (static_cast<int>(blk) - static_cast<int>(by) * bw) * N;
      const uint8_t* src = img + static_cast<size_t>(min(f_y0 + i, h - 1)) * pitch + f_x0;
      if (f_x0 + N <= w && (reinterpret_cast<uintptr_t>(src) & 7) == 0) {
#pragma unroll
        for (int q = 0; q < N / 8; ++q) {
          const uint2 v = __ldg(reinterpret_cast<const uint2*>(src) + q);
          raw[2 * q] = v.x;
          raw[2 * q + 1] = v.y;
        }
      } else {  // ragged right edge or unaligned view: tile()'s column replication
        const uint8_t* rowp = src - f_x0;
#pragma unroll
        for (int q = 0; q < N / 4; ++q) {
          uint32_t v = 0;
#pragma unroll
          for (int t = 0; t < 4; ++t) v |= static_cast<uint32_t>(__ldg(rowp + min(f_x0 + 4 * q + t, w - 1))) << (8 * t);
          raw[q] = v;
        }
      }
    } else {
      const double* src = blocks + blk * (N * N) + i * N;
      if ((reinterpret_cast<uintptr_t>(src) & 15) == 0) {
#pragma unroll
        for (int q = 0; q < N / 2; ++q) {
          const double2 v = __ldg(reinterpret_cast<const double2*>(src) + q);
          rawd[2 * q] = v.x;
          rawd[2 * q + 1] = v.y;
        }
      } else {
#pragma unroll
        for (int q = 0; q < N; ++q) rawd[q] = __ldg(src + q);
      }
    }
  };
  int c_y0 = 0, c_x0 = 0;
  bool c_valid = false;
  auto put = [&]() {
    c_valid = f_valid;
    c_y0 = f_y0;
    c_x0 = f_x0;
    if (!f_valid) return;
#pragma unroll
    for (int q = 0; q < N / 2; ++q) {
      double2 v;
      if (U8) {
        v.x = __uint2double_rn(__byte_perm(raw[q >> 1], 0, 0x4440 + ((q & 1) << 1)));
        v.y = __uint2double_rn(__byte_perm(raw[q >> 1], 0, 0x4441 + ((q & 1) << 1)));
      } else {
        v = make_double2(rawd[2 * q], rawd[2 * q + 1]);
      }
      reinterpret_cast<double2*>(my_row)[q] = v;
    }
  };

  long long batch = blockIdx.x;
  if (batch >= nbatches) return;
  fetch(batch);
  put();
  __syncthreads();
  for (;;) {
    const long long next = batch + gridDim.x;
    if (next < nbatches) fetch(next);
    if (c_valid) {
      const double* tb = tile + b * C::BS;
      double acc[N];
#pragma unroll
      for (int j = 0; j < N; ++j) acc[j] = 0.0;
#pragma unroll
      for (int r = 0; r < KR; ++r) {
        int si = i + r - (KR - 1) / 2;
        if (!REP && (si < 0 || si >= N)) continue;
        si = min(max(si, 0), N - 1);
        double row[N];
        const double2* rp = reinterpret_cast<const double2*>(tb + si * C::RS);
#pragma unroll
        for (int q = 0; q < N / 2; ++q) {
          const double2 v = rp[q];
          row[2 * q] = v.x;
          row[2 * q + 1] = v.y;
        }
#pragma unroll
        for (int j = 0; j < N; ++j) {
#pragma unroll
          for (int c = 0; c < KC; ++c) {
            int sj = j + c - (KC - 1) / 2;  // compile-time after unrolling
            if (!REP && (sj < 0 || sj >= N)) continue;
            sj = min(max(sj, 0), N - 1);
            acc[j] = __dadd_rn(acc[j], __dmul_rn(wt.w[r * KC + c], row[sj]));
          }
        }
      }
      if (U8) {
        const int y = c_y0 + i;
        if (y < h) {
          uint8_t* dst = out_img + static_cast<size_t>(y) * pitch + c_x0;
          uint32_t q[N];
#pragma unroll
          for (int j = 0; j < N; ++j) q[j] = quantize(acc[j], nan_flag);  // huge weights can overflow to NaN
          if (c_x0 + N <= w && (reinterpret_cast<uintptr_t>(dst) & 7) == 0) {
#pragma unroll
            for (int j = 0; j < N; j += 8) {
              const uint32_t lo = q[j] | (q[j + 1] << 8) | (q[j + 2] << 16) | (q[j + 3] << 24);
              const uint32_t hi = q[j + 4] | (q[j + 5] << 8) | (q[j + 6] << 16) | (q[j + 7] << 24);
              *reinterpret_cast<uint2*>(dst + j) = make_uint2(lo, hi);
            }
          } else {
#pragma unroll
            for (int j = 0; j < N; ++j)
              if (c_x0 + j < w) dst[j] = static_cast<uint8_t>(q[j]);
          }
        }
      } else {
        double* dst = out_blocks + (batch * C::BPC + b) * (N * N) + i * N;
        if ((reinterpret_cast<uintptr_t>(dst) & 15) == 0) {
#pragma unroll
          for (int j = 0; j < N; j += 2)
            *reinterpret_cast<double2*>(dst + j) = make_double2(acc[j], acc[j + 1]);
        } else {
#pragma unroll
          for (int j = 0; j < N; ++j) dst[j] = acc[j];
        }
      }
    }
    if (next >= nbatches) break;
    __syncthreads();  // every row of the tile consumed
    put();
    __syncthreads();
    batch = next;
  }
}

template <int N, int KR, int KC, bool REP, bool U8>
void launch_one(const uint8_t* img, int w, int h, size_t pitch, int bw, const double* blocks, uint8_t* out_img,
                double* out_blocks, long long nblocks, const SpWeights<KR, KC>& wt, int device, cudaStream_t st,
                int* nan_flag) {
  static const int per_sm = [] {
    int v = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&v, k_spatial_rows<N, KR, KC, REP, U8>, SP_THREADS, 0);
    return v > 0 ? v : 1;
  }();
  const long long nbatches = (nblocks + SpCfg<N>::BPC - 1) / SpCfg<N>::BPC;
  const long long resident = static_cast<long long>(dctf::sm_count(device)) * per_sm;
  const unsigned grid = static_cast<unsigned>(nbatches < resident ? nbatches : resident);
  k_spatial_rows<N, KR, KC, REP, U8><<<grid, SP_THREADS, 0, st>>>(img, w, h, pitch, bw, blocks, out_img,
                                                                  out_blocks, nblocks, nbatches, wt, nan_flag);
}

template <int N, int KR, int KC>
void launch_rows(const dctf_plan* p, const uint8_t* img, int w, int h, size_t pitch, int bw,
                 const double* blocks, uint8_t* out_img, double* out_blocks, long long nblocks,
                 cudaStream_t st) {
  SpWeights<KR, KC> wt;
  for (int t = 0; t < KR * KC; ++t) wt.w[t] = p->weights[t];
  const bool rep = p->padding == DCTF_PAD_REPLICATE;
  const int dev = p->device;
  if (img) {
    if (rep) launch_one<N, KR, KC, true, true>(img, w, h, pitch, bw, nullptr, out_img, nullptr, nblocks, wt, dev, st, dctf::nan_flag(p));
    else launch_one<N, KR, KC, false, true>(img, w, h, pitch, bw, nullptr, out_img, nullptr, nblocks, wt, dev, st, dctf::nan_flag(p));
  } else {
    if (rep) launch_one<N, KR, KC, true, false>(nullptr, 0, 0, 0, 1, blocks, nullptr, out_blocks, nblocks, wt, dev, st, dctf::nan_flag(p));
    else launch_one<N, KR, KC, false, false>(nullptr, 0, 0, 0, 1, blocks, nullptr, out_blocks, nblocks, wt, dev, st, dctf::nan_flag(p));
  }
}

template <int N>
bool dispatch_k(const dctf_plan* p, const uint8_t* img, int w, int h, size_t pitch, int bw,
                const double* blocks, uint8_t* out_img, double* out_blocks, long long nblocks,
                cudaStream_t st) {
  const int kr = p->kr, kc = p->kc;
  if (kr == 3 && kc == 3) launch_rows<N, 3, 3>(p, img, w, h, pitch, bw, blocks, out_img, out_blocks, nblocks, st);
  else if (kr == 5 && kc == 5) launch_rows<N, 5, 5>(p, img, w, h, pitch, bw, blocks, out_img, out_blocks, nblocks, st);
  else if (kr == 7 && kc == 7) launch_rows<N, 7, 7>(p, img, w, h, pitch, bw, blocks, out_img, out_blocks, nblocks, st);
  else return false;
  return true;
}

}  // namespace

namespace dctf {

bool spatial_rows_supported(const dctf_plan* p) {
  const char* e = std::getenv("DCTF_SPATIAL_GENERIC");  // diagnostics: force k_spatial
  if (e && *e && *e != '0') return false;
  const bool nk = (p->n == 8 || p->n == 16);
  const bool kk = p->kr == p->kc && (p->kr == 3 || p->kr == 5 || p->kr == 7);
  return nk && kk && static_cast<int>(p->weights.size()) == p->kr * p->kc;
}

bool launch_spatial_rows(const dctf_plan* p, const uint8_t* img, int w, int h, size_t pitch, int bw,
                         const double* blocks, uint8_t* out_img, double* out_blocks, long long nblocks,
                         cudaStream_t st) {
  if (!spatial_rows_supported(p) || nblocks <= 0) return false;
  if (img && nblocks >= (1ll << 31)) return false;  // FastDiv block decomposition
  if (p->n == 8) return dispatch_k<8>(p, img, w, h, pitch, bw, blocks, out_img, out_blocks, nblocks, st);
  return dispatch_k<16>(p, img, w, h, pitch, bw, blocks, out_img, out_blocks, nblocks, st);
}

}  // namespace dctf
