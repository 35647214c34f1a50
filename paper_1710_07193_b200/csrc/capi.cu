// The C ABI of include/dctf.h (plan lifecycle, device and host-buffer entry
// points, kernel naming, NaN check, FP64 peak probe) plus the reference-order
// transforms and the spatial path:
//   k_transform<N,FWD,U8>  forward_2d (dct.hpp:59-62) / inverse_2d
//                     (dct.hpp:65-68) per block in the reference operation
//                     order (mul then add, no FMA, zero-skip), so results are
//                     bit-identical to the reference; u8 variants read tiles
//                     (image.hpp:164-184) or quantize + assemble
//                     (spatial.hpp:71-75, image.hpp:188-203). Persistent,
//                     next batch staged during the current one.
//   k_spatial<U8>     convolve (spatial.hpp:41-68), bit-identical samples.
// The filter kernels live in coef.cu (filter_coeffs: k_coef8, k_coef16 and the
// parity-class k_coef8_sym / k_coef16_sym), fused.cu (filter_image: k_fused8,
// k_fused8_sym, k_fused16, k_fused16_sym), tc.cu (3xTF32 tcgen05 coefficient
// filter) and ozaki.cu (exact-INT8 tcgen05 fused n = 8 path); shared device
// helpers in device.cuh, host operator compiler and layouts in plan.cc.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <type_traits>

#include "device.cuh"
#include "fastdiv.cuh"
#include "hostpool.h"
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
thread_local int* t_nan = nullptr;
int* nan_flag(const dctf_plan* p) { return t_nan ? t_nan : p->d_nan; }
NanScope::NanScope(int* f) : prev(t_nan) { t_nan = f; }
NanScope::~NanScope() { t_nan = prev; }
void reset_launches() { t_launches = 0; }
}  // namespace dctf

using dctf::set_error;


namespace {
// ---------------------------------------------------------------------------
// forward_2d / inverse_2d, reference operation order.
//
// One CTA = 256 threads = 256/N blocks; thread (lb, r) owns row r of block lb.
// forward: T = C X (row r of T needs row r of C and all of X), out = T C^t.
// inverse: T = C^t Y, out = T C.
// Each product is matmul (block_matrix.hpp:67-81): k ascending, skip a == 0,
// separately rounded multiply and add (the reference has no FMA
// contraction), so results are bit-identical to forward_2d / inverse_2d.

// Persistent, double-buffered reference-order transforms: a CTA of 256
// threads handles batches of 256/N blocks (thread (lb, r) = row r of block
// lb); the next batch is staged while the current one is transformed (FP64
// input by cp.async, u8 pixels by a register prefetch), so global latency
// overlaps the FP64 work. The arithmetic is exactly the reference's matmul
// (block_matrix.hpp:67-81): k ascending, a == 0 skipped, separately rounded
// multiply and add.
// The basis travels by value in the kernel parameters (constant bank): the
// second product's C operand has a compile-time index, so every DMUL reads it
// straight from the constant bank instead of shared memory (the kernel is
// shared-memory-bandwidth bound otherwise).
template <int N>
struct BasisParam {
  double c[N * N];
};
template <int N>
struct TrCfg {
  static constexpr int NN = N * N, BPC = 256 / N, STR = NN + 2;  // 16-byte aligned block rows
  static constexpr int TILE = BPC * STR;                         // doubles per buffer
  static constexpr int SMEM = 2 * TILE * 8;
};

template <int N, bool FWD, bool U8>
__global__ void __launch_bounds__(256) k_transform(const uint8_t* __restrict__ img_in,
                                                   uint8_t* __restrict__ img_out, int w, int h,
                                                   size_t pitch, int bw,
                                                   const double* __restrict__ blocks_in,
                                                   double* __restrict__ blocks_out, long long nblocks,
                                                   const __grid_constant__ BasisParam<N> bp, int* nan_flag) {
  using Cfg = TrCfg<N>;
  constexpr int NN = Cfg::NN, BPC = Cfg::BPC, STR = Cfg::STR;
  extern __shared__ __align__(16) double tbuf[];
  const int lb = threadIdx.x / N, r = threadIdx.x % N;
  // forward: T = C X (row r: C[r][k]), out = T C^t;  inverse: T = C^t Y (C[k][r]), out = T C
  double cv[N];
#pragma unroll
  for (int k = 0; k < N; ++k) cv[k] = FWD ? bp.c[r * N + k] : bp.c[k * N + r];
  bool cv_nz = true;
#pragma unroll
  for (int k = 0; k < N; ++k) cv_nz = cv_nz && cv[k] != 0.0;
  const bool cv_nonzero = __all_sync(0xFFFFFFFFu, cv_nz);
  const long long nbatch = (nblocks + BPC - 1) / BPC;
  constexpr bool U8IN = FWD && U8;
  const bool async_in = !U8IN && (reinterpret_cast<uintptr_t>(blocks_in) & 15) == 0;
  const bool u8_vec = U8IN && (pitch % N) == 0 && (reinterpret_cast<uintptr_t>(img_in) % N) == 0;
  using Row = typename std::conditional<N == 8, uint2, uint4>::type;
  Row pre{};
  bool pre_fast = false;
  // stage batch `bt` into buffer `buf` (FP64: cp.async / loads; u8: registers)
  auto stage = [&](long long bt, double* buf) {
    const long long b0 = bt * BPC;
    if constexpr (U8IN) {
      const long long blk = b0 + lb;
      pre_fast = false;
      if (blk < nblocks) {
        const int by = static_cast<int>(blk / bw), bx = static_cast<int>(blk % bw);
        if (u8_vec && by * N + N <= h && bx * N + N <= w) {
          pre = *reinterpret_cast<const Row*>(img_in + static_cast<size_t>(by * N + r) * pitch + bx * N);
          pre_fast = true;
        }
      }
    } else {
      for (int e = threadIdx.x; e < BPC * NN / 2; e += 256) {
        const int l = e / (NN / 2), c = e % (NN / 2);
        const long long blk = b0 + l;
        double* dst = buf + l * STR + 2 * c;
        if (blk >= nblocks) {
          dst[0] = dst[1] = 0.0;
        } else if (async_in) {
          cp_async16(dst, blocks_in + blk * NN + 2 * c);
        } else {
          dst[0] = blocks_in[blk * NN + 2 * c];
          dst[1] = blocks_in[blk * NN + 2 * c + 1];
        }
      }
      cp_async_commit();
    }
  };
  // u8: this thread's row of batch bt (prefetched, or clamped per byte) -> buf
  auto land_u8 = [&](long long bt, double* buf) {
    const long long blk = bt * BPC + lb;
    double* dst = buf + lb * STR + r * N;
    if (pre_fast) {
      const uint8_t* bytes = reinterpret_cast<const uint8_t*>(&pre);
#pragma unroll
      for (int j = 0; j < N; ++j) dst[j] = static_cast<double>(bytes[j]);
    } else if (blk < nblocks) {
      const int by = static_cast<int>(blk / bw), bx = static_cast<int>(blk % bw);
      const int y = min(by * N + r, h - 1);
#pragma unroll
      for (int j = 0; j < N; ++j)
        dst[j] = static_cast<double>(img_in[static_cast<size_t>(y) * pitch + min(bx * N + j, w - 1)]);
    } else {
#pragma unroll
      for (int j = 0; j < N; ++j) dst[j] = 0.0;
    }
  };

  long long bt = blockIdx.x;
  if (bt < nbatch) stage(bt, tbuf);
  for (int it = 0; bt < nbatch; bt += gridDim.x, ++it) {
    double* cur = tbuf + (it & 1) * Cfg::TILE;
    if constexpr (U8IN) land_u8(bt, cur);
    cp_async_wait_all();
    __syncthreads();
    if (bt + gridDim.x < nbatch) stage(bt + gridDim.x, tbuf + ((it + 1) & 1) * Cfg::TILE);
    const long long blk = bt * BPC + lb;
    const double* x = cur + lb * STR;
    double trow[N], o[N];
#pragma unroll
    for (int j = 0; j < N; ++j) trow[j] = 0.0;
    // matmul's a == 0 skip (block_matrix.hpp:71) only matters when the other
    // factor is not finite (0 * inf) or for the sign of a zero sum; with no
    // zero multiplier in the warp the skip-free loop gives the same bits and
    // runs without the per-k branches
    if (!U8 && cv_nonzero) {  // (the u8 variants measured slower with the second code path)
#pragma unroll
      for (int k = 0; k < N; ++k)
#pragma unroll
        for (int j = 0; j < N; ++j) trow[j] = __dadd_rn(trow[j], __dmul_rn(cv[k], x[k * N + j]));
    } else {
#pragma unroll
      for (int k = 0; k < N; ++k) {
        const double a = cv[k];
        if (a != 0.0) {
#pragma unroll
          for (int j = 0; j < N; ++j) trow[j] = __dadd_rn(trow[j], __dmul_rn(a, x[k * N + j]));
        }
      }
    }
#pragma unroll
    for (int j = 0; j < N; ++j) o[j] = 0.0;
    bool t_nonzero = true;
#pragma unroll
    for (int k = 0; k < N; ++k) t_nonzero = t_nonzero && trow[k] != 0.0;
    if (!U8 && __all_sync(0xFFFFFFFFu, t_nonzero)) {
#pragma unroll
      for (int k = 0; k < N; ++k)
#pragma unroll
        for (int j = 0; j < N; ++j)
          o[j] = __dadd_rn(o[j], __dmul_rn(trow[k], FWD ? bp.c[j * N + k] : bp.c[k * N + j]));
    } else {
#pragma unroll
      for (int k = 0; k < N; ++k) {
        const double a = trow[k];
        if (a != 0.0) {
#pragma unroll
          for (int j = 0; j < N; ++j) o[j] = __dadd_rn(o[j], __dmul_rn(a, FWD ? bp.c[j * N + k] : bp.c[k * N + j]));
        }
      }
    }
    if (blk >= nblocks) continue;
    if (!U8 || FWD) {
      double* dst = blocks_out + blk * NN + r * N;
#pragma unroll
      for (int j = 0; j < N; j += 2) *reinterpret_cast<double2*>(dst + j) = make_double2(o[j], o[j + 1]);
    } else {
      const int by = static_cast<int>(blk / bw), bx = static_cast<int>(blk % bw);
      const int yy = by * N + r;
      if (yy >= h) continue;
      uint8_t* dst = img_out + static_cast<size_t>(yy) * pitch + bx * N;
#pragma unroll
      for (int j = 0; j < N; ++j)
        if (bx * N + j < w) dst[j] = static_cast<uint8_t>(quantize(o[j], nan_flag));
    }
  }
  cp_async_wait_all();
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
                                                 int kr, int kc, int replicate, int* nan_flag) {
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
    if (y < h && x < w) out_img[static_cast<size_t>(y) * pitch + x] = static_cast<uint8_t>(quantize(acc, nan_flag));
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

// 3-D u8 view [nframes][h][w] of a frame batch (pitch and frame_stride in
// bytes, both multiples of 16, base 16-byte aligned); box [1][8][box_w], no
// swizzle, OOB -> 0.
dctf_status make_imap(void* vmap, const uint8_t* d, int w, int h, int nframes, size_t pitch,
                      long long frame_stride, int box_w, int elem_bytes) {
  CUtensorMap* map = static_cast<CUtensorMap*>(vmap);
  PFN_encodeTiled_t fn = encode_fn();
  if (!fn) return set_error(DCTF_CUDA_ERROR, "cuTensorMapEncodeTiled unavailable");
  // elem_bytes 8: the row viewed as w / 8 uint64 elements (w % 8 == 0), so
  // one box [box_w elements x 8 rows] spans box_w * 8 pixels
  const cuuint64_t dims[3] = {static_cast<cuuint64_t>(elem_bytes == 8 ? w / 8 : w), static_cast<cuuint64_t>(h),
                              static_cast<cuuint64_t>(nframes)};
  const cuuint64_t strides[2] = {static_cast<cuuint64_t>(pitch),
                                 static_cast<cuuint64_t>(nframes > 1 ? frame_stride : pitch * h)};
  const cuuint32_t box[3] = {static_cast<cuuint32_t>(box_w), 8, 1};
  const cuuint32_t estr[3] = {1, 1, 1};
  const CUresult r = fn(map, elem_bytes == 8 ? CU_TENSOR_MAP_DATA_TYPE_UINT64 : CU_TENSOR_MAP_DATA_TYPE_UINT8, 3,
                        const_cast<uint8_t*>(d), dims, strides, box, estr,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    return set_error(DCTF_CUDA_ERROR, "cuTensorMapEncodeTiled (u8 image) failed (" + std::to_string(int(r)) + ")");
  return DCTF_OK;
}
}  // namespace dctf

namespace {

}  // namespace

namespace dctf {
// SM count of a device (cached; 148 on B200).
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

bool pdl_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("DCTF_PDL");
    return !(e && e[0] == '0');
  }();
  return on;
}

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

dctf_status check_plan(const dctf_plan* p) {
  if (!p) return set_error(DCTF_INVALID_ARGUMENT, "plan is NULL");
  return DCTF_OK;
}

dctf_status check_image(int w, int h, size_t pitch) {
  if (w < 0 || h < 0) return set_error(DCTF_INVALID_ARGUMENT, "image dimensions must be >= 0");
  if (h > 0 && pitch < static_cast<size_t>(w))
    return set_error(DCTF_INVALID_ARGUMENT, "pitch < width");
  return DCTF_OK;
}

}  // namespace

namespace dctf {

// Launch of k_transform: persistent grid (batches of 256/n blocks).
template <int N, bool FWD, bool U8>
dctf_status launch_transform_n(const dctf_plan* p, const uint8_t* img_in, uint8_t* img_out, int w,
                               int h, size_t pitch, int bw, const double* bin, double* bout,
                               long long nb, cudaStream_t st) {
  if (nb == 0) return DCTF_OK;
  auto kernel = k_transform<N, FWD, U8>;
  const dctf_status sa = ensure_dyn_smem(reinterpret_cast<const void*>(kernel), TrCfg<N>::SMEM, "k_transform");
  if (sa != DCTF_OK) return sa;
  const long long nbatch = (nb + TrCfg<N>::BPC - 1) / TrCfg<N>::BPC;
  const long long grid = std::min<long long>(nbatch, 4LL * sm_count(p->device));
  BasisParam<N> bp;
  std::copy(p->basis.begin(), p->basis.begin() + N * N, bp.c);
  kernel<<<static_cast<unsigned>(grid), 256, TrCfg<N>::SMEM, st>>>(img_in, img_out, w, h, pitch, bw, bin,
                                                                   bout, nb, bp, nan_flag(p));
  add_launches(1);
  CUDA_TRY(cudaGetLastError());
  return DCTF_OK;
}

template <bool FWD, bool U8>
dctf_status launch_transform(const dctf_plan* p, const uint8_t* img_in, uint8_t* img_out, int w, int h,
                             size_t pitch, int bw, const double* bin, double* bout, long long nb,
                             cudaStream_t st) {
  return p->n == 8 ? launch_transform_n<8, FWD, U8>(p, img_in, img_out, w, h, pitch, bw, bin, bout, nb, st)
                   : launch_transform_n<16, FWD, U8>(p, img_in, img_out, w, h, pitch, bw, bin, bout, nb, st);
}

dctf_status launch_forward_u8(const dctf_plan* p, const uint8_t* img, int w, int h, size_t pitch,
                              double* coeffs, cudaStream_t st) {
  const int n = p->n, bw = (w + n - 1) / n, bh = (h + n - 1) / n;
  return launch_transform<true, true>(p, img, nullptr, w, h, pitch, bw, nullptr, coeffs,
                                      static_cast<long long>(bw) * bh, st);
}

dctf_status launch_inverse_u8(const dctf_plan* p, const double* coeffs, uint8_t* img, int w, int h,
                              size_t pitch, cudaStream_t st) {
  const int n = p->n, bw = (w + n - 1) / n, bh = (h + n - 1) / n;
  return launch_transform<false, true>(p, nullptr, img, w, h, pitch, bw, coeffs, nullptr,
                                       static_cast<long long>(bw) * bh, st);
}

}  // namespace dctf

using dctf::filter_image_device;
using dctf::launch_coef;
using dctf::launch_forward_u8;
using dctf::launch_inverse_u8;
using dctf::misaligned16;
using dctf::sm_count;


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
  const bool fp64 = precision == DCTF_PREC_FP64 || precision == DCTF_PREC_FP64_DMMA;
  p->sym = fp64 && dctf::parity_block_diagonal(p->op, n);
  if (e == cudaSuccess && p->sym && n == 16) {
    std::vector<double> gsym;
    dctf::layout_gsym16(p->op, p->basis, gsym);
    e = cudaMalloc(&p->d_hsym, gsym.size() * sizeof(double));
    if (e == cudaSuccess)
      e = cudaMemcpy(p->d_hsym, gsym.data(), gsym.size() * sizeof(double), cudaMemcpyHostToDevice);
  }
  // n = 8 sandwich kernel: worth it where it runs fewer DMMA per block than
  // the alternative (4P + 4 against 8 parity-class / 20 dense): separable
  // masks, and rank <= 3 when the operator has no parity structure
  if (e == cudaSuccess && n == 8 && fp64 && !std::getenv("DCTF_NO_SEP")) {
    std::vector<double> frag;
    const bool psym = dctf::parity_block_diagonal(p->op, 8);
    if (dctf::layout_sep8(*p, frag, p->sep_rank) && (!psym || p->sep_rank == 1)) {
      e = cudaMalloc(&p->d_sep, frag.size() * sizeof(double));
      if (e == cudaSuccess)
        e = cudaMemcpy(p->d_sep, frag.data(), frag.size() * sizeof(double), cudaMemcpyHostToDevice);
    } else {
      p->sep_rank = 0;
    }
    // coefficient path: the parity-class k_coef8_sym is already HBM-bound
    if (e == cudaSuccess && (!psym || std::getenv("DCTF_COEF8_SEP_SYM")) && dctf::layout_csep8(*p, frag, p->csep_rank)) {
      e = cudaMalloc(&p->d_csep, frag.size() * sizeof(double));
      if (e == cudaSuccess)
        e = cudaMemcpy(p->d_csep, frag.data(), frag.size() * sizeof(double), cudaMemcpyHostToDevice);
    } else {
      p->csep_rank = 0;
    }
  }
  if (e == cudaSuccess && p->sym && n == 16 && !std::getenv("DCTF_NO_SEP")) {
    std::vector<double> frag;
    if (dctf::layout_sep16(*p, frag, p->sep_rank)) {
      e = cudaMalloc(&p->d_sep, frag.size() * sizeof(double));
      if (e == cudaSuccess)
        e = cudaMemcpy(p->d_sep, frag.data(), frag.size() * sizeof(double), cudaMemcpyHostToDevice);
    }
    if (e == cudaSuccess && dctf::layout_csep16(*p, frag, p->csep_rank)) {
      e = cudaMalloc(&p->d_csep, frag.size() * sizeof(double));
      if (e == cudaSuccess)
        e = cudaMemcpy(p->d_csep, frag.data(), frag.size() * sizeof(double), cudaMemcpyHostToDevice);
    }
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
  if (e == cudaSuccess && precision == DCTF_PREC_BF16X3) {
    std::vector<uint16_t> hs;
    dctf::layout_hsplit_bf16(n, p->op, hs);
    e = cudaMalloc(&p->d_hsplit, hs.size() * sizeof(uint16_t));
    if (e == cudaSuccess)
      e = cudaMemcpy(p->d_hsplit, hs.data(), hs.size() * sizeof(uint16_t), cudaMemcpyHostToDevice);
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
  // Masks whose reference chain can overflow FP64 (chain_bounded): the image
  // path runs the reference's own operation order instead (see dctf_plan).
  p->unbounded = !dctf::chain_bounded(*p);
  if (p->unbounded && n == 8) {
    const dctf_status s = dctf::upload_refchain_only(p);
    if (s != DCTF_OK) {
      dctf_plan_destroy(p);
      return s;
    }
  }
  // n = 8 FP64 plans: the exact-integer composed-operator kernel serves the
  // u8 image path (coefficient requests keep the FP64 kernels); DCTF_NO_Q=1
  // at plan creation opts out.
  if (precision == DCTF_PREC_FP64 && n == 8 && !p->unbounded && !std::getenv("DCTF_NO_Q")) {
    const dctf_status s = dctf::upload_kq_operator(p);
    if (s != DCTF_OK) {
      dctf_plan_destroy(p);
      return s;
    }
  }
  *out = p;
  return DCTF_OK;
}
}  // namespace

namespace dctf {
// The batch dispatch of dctf_filter_frames_u8 (arguments validated by the
// caller; the device is current): one k_fused8_q launch when every plan has
// the integer operator, else one launch per plan for evenly spaced frames.
dctf_status filter_frames_device(const dctf_plan* const* plans, int nplans, const int* h_plan_of_frame,
                                 const uint8_t* d_in, uint8_t* d_out, int nframes, int w, int h, size_t pitch,
                                 size_t frame_stride, cudaStream_t st) {
  dctf_status s = DCTF_OK;
  // Every plan on the exact-integer kernel: the whole batch is one launch
  // (each plan's digit image resident in shared memory, per-frame selection).
  bool all_kq = plans[0]->n == 8 && nplans <= dctf::KQ_MAX_PLANS && nframes <= dctf::KQ_MAX_FRAMES;
  for (int i = 0; i < nplans && all_kq; ++i) all_kq = plans[i]->kq;
  if (all_kq)
    return dctf::launch_fused8_q(plans, nplans, h_plan_of_frame, d_in, d_out, w, h, pitch,
                                 static_cast<long long>(frame_stride), nframes, st, false, nan_flag(plans[0]));
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
}  // namespace dctf

extern "C" {

dctf_status dctf_plan_create(const double* h_weights, int kr, int kc, int n, int padding,
                             int precision, int device, dctf_plan** out) {
  dctf::NvtxRange nvtx_range("dctf_plan_create");
  dctf::reset_launches();
  if (!out || !h_weights) return set_error(DCTF_INVALID_ARGUMENT, "NULL argument");
  *out = nullptr;
  if (precision < DCTF_PREC_FP64 || precision > DCTF_PREC_FP64_DMMA)
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

dctf_status dctf_plan_create_from_pairs(const double* h_lefts, const double* h_rights, int npairs, int n,
                                        int domain, const double* h_weights, int k, int padding, int precision,
                                        int device, dctf_plan** out) {
  dctf::NvtxRange nvtx_range("dctf_plan_create_from_pairs");
  dctf::reset_launches();
  if (!out || (npairs > 0 && (!h_lefts || !h_rights)) || !h_weights) return set_error(DCTF_INVALID_ARGUMENT, "NULL argument");
  *out = nullptr;
  if (precision < DCTF_PREC_FP64 || precision > DCTF_PREC_FP64_DMMA)
    return set_error(DCTF_INVALID_ARGUMENT, "unknown precision mode");
  if (domain != 0 && domain != 1) return set_error(DCTF_INVALID_ARGUMENT, "domain must be 0 (spatial) or 1 (DCT)");
  if (k < 1 || (k % 2) == 0) return set_error(DCTF_INVALID_ARGUMENT, "Mask: side must be odd and >= 1");
  auto* p = new dctf_plan();
  p->n = n;
  p->kr = p->kc = k;
  p->padding = padding;
  p->precision = precision;
  p->device = device;
  p->weights.assign(h_weights, h_weights + static_cast<size_t>(k) * k);
  dctf_status s = dctf::compile_from_pairs(*p, h_lefts, h_rights, npairs, domain);
  if (s != DCTF_OK) {
    delete p;
    return s;
  }
  return finish_plan(p, out);
}

dctf_status dctf_plan_create_from_dump(const char* text, size_t len, int precision, int device,
                                       dctf_plan** out) {
  dctf::NvtxRange nvtx_range("dctf_plan_create_from_dump");
  dctf::reset_launches();
  if (!out || !text) return set_error(DCTF_INVALID_ARGUMENT, "NULL argument");
  *out = nullptr;
  if (precision < DCTF_PREC_FP64 || precision > DCTF_PREC_FP64_DMMA)
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
    cudaFree(p->d_sep);
    cudaFree(p->d_csep);
    cudaFree(p->d_hsplit);
    cudaFree(p->d_gimg);
    cudaFree(p->d_gscale);
    cudaFree(p->d_kq);
    cudaFree(p->d_refchain);
    cudaFree(p->d_kqt);
    cudaFree(p->d_nan);
    cudaFree(p->d_weights);
    cudaFree(p->io_in);
    cudaFree(p->io_out);
    p->copy_pool.reset();
    if (p->bounce) cudaFreeHost(p->bounce);
    for (void* s : p->streams)
      if (s) cudaStreamDestroy(as_stream(s));
    for (void* e : p->events)
      if (e) cudaEventDestroy(static_cast<cudaEvent_t>(e));
  }
  delete p;
  return DCTF_OK;
}

dctf_status dctf_plan_mask(const dctf_plan* p, double* h_weights, int* kr, int* kc, int* padding) {
  if (!p) return set_error(DCTF_INVALID_ARGUMENT, "plan is NULL");
  if (kr) *kr = p->kr;
  if (kc) *kc = p->kc;
  if (padding) *padding = p->padding;
  if (h_weights && !p->weights.empty()) std::memcpy(h_weights, p->weights.data(), p->weights.size() * sizeof(double));
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
  if (p->precision == DCTF_PREC_BF16X3) return "k_coef_bf16x3";
  if (p->csep_rank > 0) return p->n == 8 ? "k_coef8_sep" : "k_coef16_sep";
  if (p->n == 8) return p->sym ? "k_coef8_sym" : "k_coef8";
  return p->sym ? "k_coef16_sym" : "k_coef16";
}

dctf_status dctf_plan_kq_form(const dctf_plan* p, int* denominator, int* fraction_bits) {
  if (!p) return set_error(DCTF_INVALID_ARGUMENT, "NULL plan");
  if (!p->kq) return set_error(DCTF_UNSUPPORTED, "the plan does not run k_fused8_q");
  if (denominator) *denominator = p->kq_den;
  if (fraction_bits) *fraction_bits = p->kq_F;
  return DCTF_OK;
}

const char* dctf_plan_image_kernel(const dctf_plan* p) {
  if (!p) return nullptr;
  if (p->unbounded) return p->n == 8 ? "k_refchain8" : "unfused";
  if (p->n == 8 && p->precision == DCTF_PREC_INT8_EXACT) return "k_fused8_i8";
  if (p->kq) return "k_fused8_q";
  if (p->precision == DCTF_PREC_TF32X3 || p->precision == DCTF_PREC_BF16X3) return "unfused";
  if (p->n == 8) return p->sep_rank > 0 ? "k_fused8_sep" : (p->sym ? "k_fused8_sym" : "k_fused8");
  if (std::getenv("DCTF_N16_UNFUSED")) return "unfused";
  if (p->sep_rank > 0) return "k_fused16_sep";
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
  dctf::NvtxRange nvtx_range("dctf_forward");
  dctf::reset_launches();
  dctf_status s = check_plan(p);
  if (s == DCTF_OK) s = check_image(w, h, pitch);
  if (s != DCTF_OK) return s;
  if (w == 0 || h == 0) return DCTF_OK;  // tile() of an empty image has no blocks
  if (!d_img || !d_coeffs) return set_error(DCTF_INVALID_ARGUMENT, "NULL buffer");
  DeviceGuard guard(p->device);
  return launch_forward_u8(p, d_img, w, h, pitch, d_coeffs, as_stream(stream));
}

dctf_status dctf_forward_blocks(const dctf_plan* p, const double* d_blocks, double* d_coeffs,
                                size_t nblocks, void* stream) {
  dctf::NvtxRange nvtx_range("dctf_forward_blocks");
  dctf::reset_launches();
  dctf_status s = check_plan(p);
  if (s != DCTF_OK) return s;
  if (nblocks == 0) return DCTF_OK;
  if (!d_blocks || !d_coeffs) return set_error(DCTF_INVALID_ARGUMENT, "NULL buffer");
  if (misaligned16(d_coeffs)) return set_error(DCTF_INVALID_ARGUMENT, "buffers must be 16-byte aligned");
  DeviceGuard guard(p->device);
  return dctf::launch_transform<true, false>(p, nullptr, nullptr, 0, 0, 0, 1, d_blocks, d_coeffs,
                                             static_cast<long long>(nblocks), as_stream(stream));
}

dctf_status dctf_inverse_blocks(const dctf_plan* p, const double* d_coeffs, double* d_blocks,
                                size_t nblocks, void* stream) {
  dctf::NvtxRange nvtx_range("dctf_inverse_blocks");
  dctf::reset_launches();
  dctf_status s = check_plan(p);
  if (s != DCTF_OK) return s;
  if (nblocks == 0) return DCTF_OK;
  if (!d_blocks || !d_coeffs) return set_error(DCTF_INVALID_ARGUMENT, "NULL buffer");
  if (misaligned16(d_blocks)) return set_error(DCTF_INVALID_ARGUMENT, "buffers must be 16-byte aligned");
  DeviceGuard guard(p->device);
  return dctf::launch_transform<false, false>(p, nullptr, nullptr, 0, 0, 0, 1, d_coeffs, d_blocks,
                                              static_cast<long long>(nblocks), as_stream(stream));
}

dctf_status dctf_filter_coeffs(const dctf_plan* p, const double* d_in, double* d_out,
                               size_t nblocks, void* stream) {
  dctf::NvtxRange nvtx_range("dctf_filter_coeffs");
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
  dctf::NvtxRange nvtx_range("dctf_inverse_u8");
  dctf::reset_launches();
  dctf_status s = check_plan(p);
  if (s == DCTF_OK) s = check_image(w, h, pitch);
  if (s != DCTF_OK) return s;
  if (w == 0 || h == 0) return DCTF_OK;  // tile() of an empty image has no blocks
  if (!d_img || !d_coeffs) return set_error(DCTF_INVALID_ARGUMENT, "NULL buffer");
  DeviceGuard guard(p->device);
  return launch_inverse_u8(p, d_coeffs, d_img, w, h, pitch, as_stream(stream));
}

dctf_status dctf_filter_image_u8(const dctf_plan* p, const uint8_t* d_in, uint8_t* d_out, int w,
                                 int h, size_t pitch, double* d_coeffs_out, void* stream) {
  dctf::NvtxRange nvtx_range("dctf_filter_image_u8");
  dctf::reset_launches();
  dctf_status s = check_plan(p);
  if (s == DCTF_OK) s = check_image(w, h, pitch);
  if (s != DCTF_OK) return s;
  if (w == 0 || h == 0) return DCTF_OK;  // tile() of an empty image has no blocks
  if (!d_in || !d_out) return set_error(DCTF_INVALID_ARGUMENT, "NULL buffer");
  if (d_in == d_out) return set_error(DCTF_INVALID_ARGUMENT, "in/out images may not alias");
  DeviceGuard guard(p->device);
  return filter_image_device(p, d_in, d_out, w, h, pitch, 0, 1, d_coeffs_out, as_stream(stream));
}

dctf_status dctf_filter_image_spatial_u8(const dctf_plan* p, const uint8_t* d_in, uint8_t* d_out,
                                         int w, int h, size_t pitch, void* stream) {
  dctf::NvtxRange nvtx_range("dctf_filter_image_spatial_u8");
  dctf::reset_launches();
  dctf_status s = check_plan(p);
  if (s == DCTF_OK) s = check_image(w, h, pitch);
  if (s != DCTF_OK) return s;
  if (w == 0 || h == 0) return DCTF_OK;  // tile() of an empty image has no blocks
  if (!d_in || !d_out) return set_error(DCTF_INVALID_ARGUMENT, "NULL buffer");
  if (p->kr * p->kc > 1024) return set_error(DCTF_UNSUPPORTED, "spatial path supports masks up to 1024 taps");
  DeviceGuard guard(p->device);
  const int n = p->n, bw = (w + n - 1) / n, bh = (h + n - 1) / n;
  const long long nb = static_cast<long long>(bw) * bh;
  if (!dctf::launch_spatial_rows(p, d_in, w, h, pitch, bw, nullptr, d_out, nullptr, nb, as_stream(stream))) {
    const unsigned grid = static_cast<unsigned>((nb * n * n + 255) / 256);
    k_spatial<true><<<grid, 256, 0, as_stream(stream)>>>(d_in, w, h, pitch, bw, nullptr, d_out, nullptr, nb, n,
                                                         p->d_weights, p->kr, p->kc, p->padding, dctf::nan_flag(p));
  }
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
  if (!dctf::launch_spatial_rows(p, nullptr, 0, 0, 0, 1, d_blocks, nullptr, d_out, nb, as_stream(stream))) {
    const unsigned grid = static_cast<unsigned>((nb * n * n + 255) / 256);
    k_spatial<false><<<grid, 256, 0, as_stream(stream)>>>(nullptr, 0, 0, 0, 1, d_blocks, nullptr, d_out, nb, n,
                                                          p->d_weights, p->kr, p->kc, p->padding, dctf::nan_flag(p));
  }
  dctf::add_launches(1);
  CUDA_TRY(cudaGetLastError());
  return DCTF_OK;
}

dctf_status dctf_filter_frames_u8(const dctf_plan* const* plans, int nplans,
                                  const int* h_plan_of_frame, const uint8_t* d_in, uint8_t* d_out,
                                  int nframes, int w, int h, size_t pitch, size_t frame_stride,
                                  void* stream) {
  dctf::NvtxRange nvtx_range("dctf_filter_frames_u8");
  dctf::reset_launches();
  if (!plans || nplans < 1 || !h_plan_of_frame || nframes < 0)
    return set_error(DCTF_INVALID_ARGUMENT, "bad plan list");
  dctf_status s = check_image(w, h, pitch);
  if (s != DCTF_OK) return s;
  if (w == 0 || h == 0) return DCTF_OK;  // tile() of an empty image has no blocks
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
  return dctf::filter_frames_device(plans, nplans, h_plan_of_frame, d_in, d_out, nframes, w, h, pitch,
                                    frame_stride, as_stream(stream));
}

dctf_status dctf_filter_image_host(const dctf_plan* p, const uint8_t* h_in, uint8_t* h_out, int w,
                                   int h, size_t pitch) {
  dctf::NvtxRange nvtx_range("dctf_filter_image_host");
  dctf::reset_launches();
  dctf_status s = check_plan(p);
  if (s == DCTF_OK) s = check_image(w, h, pitch);
  if (s != DCTF_OK) return s;
  if (w == 0 || h == 0) return DCTF_OK;  // tile() of an empty image has no blocks
  if (!h_in || !h_out) return set_error(DCTF_INVALID_ARGUMENT, "NULL buffer");
  DeviceGuard guard(p->device);
  // Plans on k_fused8_q (TMA-fed: no zero-copy reads of host memory) and
  // split-precision plans (three kernels) go through the copy-engine band
  // pipeline: per-call scratch, per-thread streams, no plan lock.
  const char* mode_env = std::getenv("DCTF_E2E_MODE");
  if (p->kq || p->precision == DCTF_PREC_TF32X3 || p->precision == DCTF_PREC_BF16X3 ||
      (mode_env && std::atoi(mode_env) == 0)) {
    int launches = 0;
    s = dctf::image_host_copy(p, h_in, h_out, w, h, pitch, &launches);
    dctf::t_launches = launches;
    return s;
  }
  std::lock_guard<std::mutex> lock(p->io_mu);
  size_t dpitch = (static_cast<size_t>(w) + 15) & ~size_t(15);
  // mode 1 stages the input with the caller's pitch (the kernel then reads
  // the device copy and writes the mapped host output with one pitch)
  const size_t bytes = std::max(dpitch, pitch) * static_cast<size_t>(h);
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
  //   mode 3 "bounce": pageable buffers — a host thread pool copies row
  //          chunks into pinned, mapped bounce buffers and back while the
  //          fused kernel streams the previous chunk over PCIe (zero-copy);
  //   mode 0 "copy": H2D / compute / D2H in three streams (split precision).
  // DCTF_E2E_MODE overrides the choice (measurement).
  cudaPointerAttributes ai{}, ao{};
  const bool in_pinned = cudaPointerGetAttributes(&ai, h_in) == cudaSuccess &&
                         ai.type == cudaMemoryTypeHost && ai.devicePointer != nullptr;
  const bool out_pinned = cudaPointerGetAttributes(&ao, h_out) == cudaSuccess &&
                          ao.type == cudaMemoryTypeHost && ao.devicePointer != nullptr;
  cudaGetLastError();
  // zero-copy needs a single fused kernel (every precision except the
  // split-precision path, which runs forward/filter/inverse as three kernels)
  const bool fused = p->precision != DCTF_PREC_TF32X3 && p->precision != DCTF_PREC_BF16X3;
  int mode = (in_pinned && out_pinned && fused) ? 2 : (fused ? 3 : 0);
  if (const char* env = std::getenv("DCTF_E2E_MODE")) {
    const int m = std::atoi(env);
    if (m == 0 || (m == 1 && out_pinned && fused) || (m == 2 && in_pinned && out_pinned && fused) ||
        (m == 3 && fused))
      mode = m;
  }
  if (mode == 1) dpitch = pitch;
  // per-call NaN flag (the plan's own flag belongs to the device entries)
  int* d_flag = nullptr;
  CUDA_TRY(cudaMallocAsync(reinterpret_cast<void**>(&d_flag), sizeof(int), s_run));
  CUDA_TRY(cudaMemsetAsync(d_flag, 0, sizeof(int), s_run));
  dctf::NanScope nan_scope(d_flag);
  const int n = p->n, bh = (h + n - 1) / n;
  int launches = 0;
  if (mode == 2) {
    s = filter_image_device(p, static_cast<const uint8_t*>(ai.devicePointer),
                            static_cast<uint8_t*>(ao.devicePointer), w, h, pitch, 0, 1, nullptr,
                            s_run, /*host_mapped=*/true);
    launches = dctf::t_launches;
  } else if (mode == 3) {
    // chunks of whole block rows (~2 MiB), double-buffered pinned bounce buffers
    const int crows = std::max(1, static_cast<int>((size_t(2) << 20) / (dpitch * n))) * n;
    const size_t chunk_bytes = dpitch * static_cast<size_t>(crows);
    if (p->bounce_chunk < chunk_bytes) {
      if (p->bounce) cudaFreeHost(p->bounce);
      p->bounce = nullptr;
      p->bounce_chunk = 0;
      CUDA_TRY(cudaHostAlloc(&p->bounce, 4 * chunk_bytes, cudaHostAllocMapped));
      p->bounce_chunk = chunk_bytes;
    }
    if (!p->copy_pool) {
      const int nt = static_cast<int>(std::max(1u, std::min(8u, std::thread::hardware_concurrency())));
      p->copy_pool = std::shared_ptr<void>(new dctf::HostCopyPool(nt),
                                           [](void* q) { delete static_cast<dctf::HostCopyPool*>(q); });
    }
    auto* pool = static_cast<dctf::HostCopyPool*>(p->copy_pool.get());
    auto* hb = static_cast<uint8_t*>(p->bounce);
    void* dbv = nullptr;
    CUDA_TRY(cudaHostGetDevicePointer(&dbv, p->bounce, 0));
    auto* db = static_cast<uint8_t*>(dbv);
    const size_t cb = p->bounce_chunk;
    cudaEvent_t done[2] = {static_cast<cudaEvent_t>(p->events[0]), static_cast<cudaEvent_t>(p->events[1])};
    const int nch = (h + crows - 1) / crows;
    auto drain = [&](int c) {  // chunk c's result: bounce -> user output
      const int b = c & 1, y0 = c * crows, rows = std::min(crows, h - y0);
      const cudaError_t e = cudaEventSynchronize(done[b]);
      if (e != cudaSuccess) return set_error(DCTF_CUDA_ERROR, std::string("bounce drain: ") + cudaGetErrorString(e));
      pool->copy2d(h_out + y0 * pitch, pitch, hb + (2 + b) * cb, dpitch, w, rows);
      return DCTF_OK;
    };
    for (int c = 0; c < nch && s == DCTF_OK; ++c) {
      const int b = c & 1, y0 = c * crows, rows = std::min(crows, h - y0);
      if (c >= 2) CUDA_TRY(cudaEventSynchronize(done[b]));  // chunk c-2 has left both bounce buffers b
      pool->copy2d(hb + b * cb, dpitch, h_in + y0 * pitch, pitch, w, rows);
      dctf::reset_launches();
      s = filter_image_device(p, db + b * cb, db + (2 + b) * cb, w, rows, dpitch, 0, 1, nullptr, s_run,
                              /*host_mapped=*/true);
      launches += dctf::t_launches;
      if (s != DCTF_OK) break;
      CUDA_TRY(cudaEventRecord(done[b], s_run));
      if (c >= 1) s = drain(c - 1);  // overlaps chunk c's kernel
    }
    if (s == DCTF_OK && nch >= 1) s = drain(nch - 1);
  } else {
    size_t chunk_target = mode == 1 ? (size_t(4) << 20) : (size_t(2) << 20);
    const char* chunk_env = std::getenv("DCTF_E2E_CHUNK_KB");
    if (chunk_env) chunk_target = std::max<size_t>(64, std::atoll(chunk_env)) << 10;
    const int nchunks = std::max(1, std::min(bh, static_cast<int>((static_cast<size_t>(h) * w + chunk_target - 1) / chunk_target)));
    const int brows = (bh + nchunks - 1) / nchunks;
    std::vector<int> cut{0};  // chunk boundaries in block rows
    for (int c = 1; (c - 1) * brows < bh; ++c) cut.push_back(std::min(bh, c * brows));
    auto* din = static_cast<uint8_t*>(p->io_in);
    auto* dout = static_cast<uint8_t*>(p->io_out);
    auto* hout_dev = static_cast<uint8_t*>(ao.devicePointer);
    for (size_t c = 0; c + 1 < cut.size() && s == DCTF_OK; ++c) {
      const int y0 = cut[c] * n;
      const int rows = std::min(cut[c + 1] * n, h) - y0;
      cudaEvent_t in_done = static_cast<cudaEvent_t>(p->events[(2 * c) % 64]);
      cudaEvent_t run_done = static_cast<cudaEvent_t>(p->events[(2 * c + 1) % 64]);
      if (pitch == dpitch && pitch == static_cast<size_t>(w))  // else 2-D: the caller's row padding is not ours
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
      if (pitch == dpitch && pitch == static_cast<size_t>(w))  // else 2-D: the caller's row padding is not ours
        CUDA_TRY(cudaMemcpyAsync(h_out + y0 * pitch, dout + y0 * dpitch, static_cast<size_t>(rows) * pitch,
                                 cudaMemcpyDeviceToHost, s_out));
      else
        CUDA_TRY(cudaMemcpy2DAsync(h_out + y0 * pitch, pitch, dout + y0 * dpitch, dpitch, w, rows,
                                   cudaMemcpyDeviceToHost, s_out));
    }
  }
  int nan_seen = 0;
  CUDA_TRY(cudaMemcpyAsync(&nan_seen, d_flag, sizeof(int), cudaMemcpyDeviceToHost, s_run));
  cudaFreeAsync(d_flag, s_run);
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
  // the thread's cached stream and scratch (input and output halves)
  cudaStream_t st = nullptr;
  void* scratch = nullptr;
  s = dctf::thread_scratch(p->device, 2 * bytes, &st, &scratch);
  if (s != DCTF_OK) return s;
  double* din = static_cast<double*>(scratch);
  double* dout = din + bytes / sizeof(double);
  cudaError_t e = cudaMemcpyAsync(din, h_in, bytes, cudaMemcpyHostToDevice, st);
  if (e != cudaSuccess) s = set_error(DCTF_CUDA_ERROR, cudaGetErrorString(e));
  if (s == DCTF_OK) {
    if (op == 0) s = dctf_forward_blocks(p, din, dout, nblocks, st);
    else if (op == 1) s = dctf_inverse_blocks(p, din, dout, nblocks, st);
    else if (op == 2) s = dctf_filter_coeffs(p, din, dout, nblocks, st);
    else if (op == 3) s = dctf_convolve_blocks(p, din, dout, nblocks, st);
    else {  // filter_block: forward -> filter_coeffs -> inverse, one round trip
      s = dctf_forward_blocks(p, din, dout, nblocks, st);
      if (s == DCTF_OK) s = dctf_filter_coeffs(p, dout, din, nblocks, st);
      if (s == DCTF_OK) s = dctf_inverse_blocks(p, din, dout, nblocks, st);
    }
  }
  if (s == DCTF_OK) {
    e = cudaMemcpyAsync(h_out, dout, bytes, cudaMemcpyDeviceToHost, st);
    if (e != cudaSuccess) s = set_error(DCTF_CUDA_ERROR, cudaGetErrorString(e));
  }
  e = cudaStreamSynchronize(st);
  if (s == DCTF_OK && e != cudaSuccess) s = set_error(DCTF_CUDA_ERROR, cudaGetErrorString(e));
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

dctf_status dctf_filter_blocks_host(const dctf_plan* p, const double* h_in, double* h_out, size_t nblocks) {
  return run_host_blocks(p, h_in, h_out, nblocks, 4);
}

dctf_status dctf_filter_image_spatial_host(const dctf_plan* p, const uint8_t* h_in, uint8_t* h_out, int w,
                                           int h, size_t pitch) {
  dctf::NvtxRange nvtx_range("dctf_filter_image_spatial_host");
  dctf_status s = check_plan(p);
  if (s == DCTF_OK) s = check_image(w, h, pitch);
  if (s != DCTF_OK) return s;
  if (w == 0 || h == 0) return DCTF_OK;  // tile() of an empty image has no blocks
  if (!h_in || !h_out) return set_error(DCTF_INVALID_ARGUMENT, "NULL buffer");
  DeviceGuard guard(p->device);
  // device copy at the width rounded to 16 bytes; only w bytes of each of the
  // caller's rows are read and written (its row padding is not ours)
  const size_t dpitch = (static_cast<size_t>(w) + 15) & ~size_t(15);
  const size_t bytes = dpitch * static_cast<size_t>(h);
  uint8_t *din = nullptr, *dout = nullptr;
  int* d_flag = nullptr;  // per-call NaN flag (quantize_sample's throw)
  int nan_seen = 0;
  CUDA_TRY(cudaMalloc(&din, bytes));
  cudaError_t e = cudaMalloc(&dout, bytes);
  if (e == cudaSuccess) e = cudaMalloc(&d_flag, sizeof(int));
  if (e == cudaSuccess) e = cudaMemset(d_flag, 0, sizeof(int));
  if (e == cudaSuccess) e = cudaMemcpy2D(din, dpitch, h_in, pitch, w, h, cudaMemcpyHostToDevice);
  if (e == cudaSuccess) {
    dctf::NanScope nan_scope(d_flag);
    s = dctf_filter_image_spatial_u8(p, din, dout, w, h, dpitch, nullptr);
    if (s == DCTF_OK) e = cudaMemcpy2D(h_out, pitch, dout, dpitch, w, h, cudaMemcpyDeviceToHost);
    if (s == DCTF_OK && e == cudaSuccess) e = cudaMemcpy(&nan_seen, d_flag, sizeof(int), cudaMemcpyDeviceToHost);
  }
  cudaFree(din);
  cudaFree(dout);
  cudaFree(d_flag);
  if (e != cudaSuccess) return set_error(DCTF_CUDA_ERROR, cudaGetErrorString(e));
  if (s == DCTF_OK && nan_seen) return set_error(DCTF_NAN_ENCOUNTERED, "quantize: NaN sample");
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
