// Internal declarations shared by plan.cc (host operator compiler) and
// the CUDA translation units (capi.cu: C ABI, transforms, plan upload; coef.cu;
// fused.cu; tc.cu; ozaki.cu).
#pragma once

#include <cstddef>
#include <cstdint>
#include <memory>
#include <mutex>
#include <string>
#include <utility>
#include <vector>

#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>  // header-only NVTX v3: ranges cost a few ns without a tool attached

#include "../../include/dctf.h"

struct dctf_plan {
  int n = 0, kr = 0, kc = 0, padding = 0, precision = 0, device = 0;
  int npairs = 0, merged = 0;
  bool reference_domain = true;  // square k <= n mask, compiled like FilterPlan
  std::vector<double> weights;   // kr*kc row-major
  std::vector<double> basis;     // C, n*n row-major (DctBasis::c())
  std::vector<double> op;        // H, n^4 row-major (natural coefficient order)
  // Sandwich pairs of the compile (reference domain only): spatial (after
  // merge_symmetric) and DCT-domain, npairs x n*n each (OperatorSet::pairs).
  std::vector<double> sp_left, sp_right, dct_left, dct_right;

  // Device-resident copies (owned). Layouts: see plan.cc (layout_*).
  double* d_basis = nullptr;     // C, n*n
  double* d_hcoef = nullptr;     // H in coefficient-kernel fragment order
  double* d_hfused = nullptr;    // H in fused-kernel fragment order
  void* d_hsplit = nullptr;      // TF32 / BF16 hi/lo split of H in UMMA core layout (TF32X3, BF16X3)
  void* d_gimg = nullptr;        // INT8 digit slices of H (C (x) C), swizzled (INT8_EXACT)
  double* d_gscale = nullptr;    // per-row scales of those slices
  int* d_nan = nullptr;          // NaN flag
  double* d_weights = nullptr;   // mask, kr*kc (spatial path)
  bool sym = false;              // H parity-block-diagonal and precision FP64 (k_fused8_sym, k_coef*_sym)
  double* d_hsym = nullptr;      // layout_sym8 (n = 8) / layout_gsym16 (n = 16) image (sym)
  double* d_hcsym = nullptr;     // layout_coefsym8 / layout_coefsym16 image (sym)
  int sep_rank = 0;              // > 0: k_fused16_sep / k_fused8_sep applies (layout_sep16 / 8), pairs
  double* d_sep = nullptr;       // its DMMA fragment image
  int csep_rank = 0;             // > 0: k_coef16_sep / k_coef8_sep applies (layout_csep16 / 8), pairs
  double* d_csep = nullptr;      // its DMMA fragment image
  // k_fused8_q (quant.cu): the composed operator as exact int8 digit slices
  // (layout_kq8) and the reference-order fallback's data (refchain_image).
  bool kq = false;               // the u8 image path of this plan runs k_fused8_q
  int kq_F = 0;                  // fixed-point fraction bits of K_int
  uint32_t kq_U = 0;             // uncertainty window, in units of 2^-32 of a pixel
  double kq_ebound = 0.0;        // E + M of layout_kq8 (pixel units)
  double kq_flag_rate = 0.0;     // expected flagged-block fraction (uniform fractions)
  void* d_kq = nullptr;          // 16 KB digit image (SW64 K-major)
  double* d_refchain = nullptr;  // C | C^t | lefts | rights (mode 1)
  double* d_kqt = nullptr;       // K in FP64, transposed (the fallback's first stage)
  double kq_margin = 0.0;        // first-stage tie window (pixel units)
  int kq_den = 0;                // > 0: rational operator K = K' / den (odd den), single-accumulator path
  uint32_t kq_magic = 0;         // ceil(2^32 / den) (den > 1)
  int kq_bias = 0;               // floor-division bias B (the accumulator carries + B den)
  bool kq_unsigned = false;      // the digit image holds unsigned bytes (MMA B format u8)
  bool kq_nosat = false;         // F = 32 and every output provably in [0, 255]: the epilogue packs bytes without saturation
  int ref_mode = 0, ref_npairs = 0;
  // The reference chain's intermediates can overflow FP64 for this mask
  // (huge weights; chain_bounded false): the u8 image path then runs the
  // reference's own operation order (n = 8: k_refchain8; n = 16: forward ->
  // filter_coeffs -> inverse), so inf / NaN arise where they arise in the
  // reference and NaN is reported like quantize_sample's throw.
  bool unbounded = false;

  // Device staging of the host-buffer entry (copy mode), guarded by io_mu.
  mutable std::mutex io_mu;
  mutable void* io_in = nullptr;
  mutable void* io_out = nullptr;
  mutable size_t io_bytes = 0;
  mutable void* streams[3] = {nullptr, nullptr, nullptr};  // H2D, compute, D2H
  mutable void* events[64] = {};                              // per-chunk ordering
  // Pageable host buffers: pinned, UVA-mapped bounce buffers (2 input + 2
  // output chunks) filled / drained by a host thread pool (capi.cu).
  mutable void* bounce = nullptr;
  mutable size_t bounce_chunk = 0;
  mutable std::shared_ptr<void> copy_pool;
};

namespace dctf {

// NVTX range over one C-ABI entry (nsys / ncu --nvtx show the host-side
// structure: plan compile, host pipelines, device launches).
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};

// Thread-local error / launch bookkeeping (capi.cu).
dctf_status set_error(dctf_status s, const std::string& msg);
void add_launches(int k);
// Dynamic shared-memory opt-in, once per (kernel, device), thread-safe (capi.cu).
dctf_status ensure_dyn_smem(const void* func, int bytes, const char* name);
// SM count of a device, cached (capi.cu).
int sm_count(int device);
inline bool misaligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) != 0; }

// Register-tiled spatial path (spatial.cu): n in {8, 16}, square 3/5/7 masks.
// Returns false (nothing launched) for other shapes; the caller then runs the
// generic k_spatial. Exactly one of img / blocks is non-null.
bool launch_spatial_rows(const dctf_plan* p, const uint8_t* img, int w, int h, size_t pitch, int bw,
                         const double* blocks, uint8_t* out_img, double* out_blocks, long long nblocks,
                         cudaStream_t st);

// Launchers shared across the kernel translation units (all enqueue on `st`).
// coef.cu: filter_coeffs on device buffers (dense / parity-class / 3xTF32).
dctf_status launch_coef(const dctf_plan* p, const double* d_in, double* d_out, long long nb, cudaStream_t st);
// capi.cu: forward_2d of a u8 image into block-major coefficients, and the
// inverse + quantize back to u8 (reference operation order).
dctf_status launch_forward_u8(const dctf_plan* p, const uint8_t* img, int w, int h, size_t pitch,
                              double* coeffs, cudaStream_t st);
dctf_status launch_inverse_u8(const dctf_plan* p, const double* coeffs, uint8_t* img, int w, int h,
                              size_t pitch, cudaStream_t st);
// fused.cu: filter_image on device buffers, one frame or a strided frame batch.
// host_mapped: `in` is UVA-mapped pinned host memory (zero-copy host entry).
dctf_status filter_image_device(const dctf_plan* p, const uint8_t* in, uint8_t* out, int w, int h,
                                size_t pitch, long long frame_stride, int nframes, double* coef_out,
                                cudaStream_t st, bool host_mapped = false);
void reset_launches();
// NaN flag the launchers pass to the quantizing kernels: the calling thread's
// per-call flag while a NanScope is alive (host-buffer entries), else the
// plan's own flag (device entries; dctf_plan_nan_check reads it).
int* nan_flag(const dctf_plan* p);
struct NanScope {
  explicit NanScope(int* f);
  ~NanScope();
  int* prev;
};
// host.cu: one image from / to host buffers through the copy-engine pipeline
// (per-call scratch, per-thread streams).
dctf_status image_host_copy(const dctf_plan* p, const uint8_t* h_in, uint8_t* h_out, int w, int h, size_t pitch,
                            int* launches);
// host.cu: the calling thread's compute stream on `device` and a grow-only
// device scratch buffer of at least `bytes` (per thread and device).
dctf_status thread_scratch(int device, size_t bytes, cudaStream_t* st, void** buf);
// capi.cu: dctf_filter_frames_u8's dispatch (validated arguments, device current).
dctf_status filter_frames_device(const dctf_plan* const* plans, int nplans, const int* h_plan_of_frame,
                                 const uint8_t* d_in, uint8_t* d_out, int nframes, int w, int h, size_t pitch,
                                 size_t frame_stride, cudaStream_t st);

// Host operator compiler (plan.cc).
// Builds C and the dense DCT-domain operator H for the mask.
// Returns DCTF_INVALID_ARGUMENT with a message on bad input.
dctf_status compile_operator(dctf_plan& p);
// A plan from explicit sandwich pairs (domain 0 spatial, 1 DCT), plan.cc.
dctf_status compile_from_pairs(dctf_plan& p, const double* lefts, const double* rights, int np, int domain);

// Operator dump format (operator_io.hpp:105-217), plan.cc.
std::string format_operator_dump(const dctf_plan& p);
// Parses a dump; fills weights/n/padding/merged and the pairs of the DCT set
// (or the conjugated spatial set) and densifies H. Returns INVALID_ARGUMENT
// with the reference's OperatorDumpError messages on malformed input.
dctf_status parse_operator_dump(const std::string& text, dctf_plan& p);
std::uint64_t mask_fingerprint(int k, const std::vector<double>& w);

// Fragment-order permutations of H for the kernels (plan.cc).
void layout_hcoef(int n, const std::vector<double>& op, std::vector<double>& out);
void layout_hfused8(const std::vector<double>& op, std::vector<double>& out);
// Parity-class structure of H (symmetric masks) and the k_fused8_sym image.
bool parity_block_diagonal(const std::vector<double>& op, int n);
void layout_sym8(const std::vector<double>& op, const std::vector<double>& basis, std::vector<double>& out);
bool layout_sep16(const dctf_plan& p, std::vector<double>& out, int& rank);
bool layout_sep8(const dctf_plan& p, std::vector<double>& out, int& rank);
bool layout_csep16(const dctf_plan& p, std::vector<double>& out, int& rank);
bool layout_csep8(const dctf_plan& p, std::vector<double>& out, int& rank);
void layout_coefsym8(const std::vector<double>& op, std::vector<double>& out);
void layout_coefsym16(const std::vector<double>& op, std::vector<double>& out);
void layout_gsym16(const std::vector<double>& op, const std::vector<double>& basis, std::vector<double>& out);
// G = H (C (x) C): the operator with the forward DCT composed in (pixels ->
// filtered coefficients), accumulated in long double and rounded once.
std::vector<long double> compose_forward_ld(const std::vector<double>& op, const std::vector<double>& basis, int n);
std::vector<double> compose_forward(const std::vector<double>& op, const std::vector<double>& basis, int n);
void layout_hfused16(const std::vector<double>& op, std::vector<double>& out);
void layout_hsplit_tf32(int n, const std::vector<double>& op, std::vector<float>& out);
void layout_hsplit_bf16(int n, const std::vector<double>& op, std::vector<uint16_t>& out);
void layout_gslices_i8(const std::vector<double>& op, const std::vector<double>& basis,
                       std::vector<int8_t>& bimg, std::vector<double>& scales);

// k_fused8_q operator (plan.cc): see layout_kq8.
struct KqInfo {
  bool ok = false;
  int F = 0;
  uint32_t U = 0;
  double ebound = 0.0, flag_rate = 0.0;
  double margin = 0.0;       // second-stage window: reference FP64 deviation + our FP64 dot error
  double eref = 0.0;         // rigorous bound of the reference chain's FP64 deviation (pixel units)
  std::vector<double> kt;    // the composed operator K in FP64, transposed (kt[j * 64 + i] = K[i][j])
  int den = 0;               // > 0: K = K' / den with integer K', odd den: exact single-accumulator path
  uint32_t magic = 0;        // ceil(2^32 / den)
  int bias = 0;              // B: the accumulator constant is (den - 1) / 2 + B den, q = floor(acc / den) - B
  bool nosat = false;        // four-digit form, F = 32, K_int >= 0 and 255 row sums + constants < 256 * 2^32
  bool unsigned_digits = false;  // K >= 0 with entries past 1/2: plain base-256 digits 0..255, B operand read as u8
};
bool layout_kq8(const dctf_plan& p, std::vector<int8_t>& bimg, KqInfo& info);
void refchain_image(const dctf_plan& p, std::vector<double>& out, int& mode, int& npairs);
// True when every intermediate of the reference chain (forward_2d, apply_pairs,
// inverse_2d or convolve) stays below 1e300 in magnitude for u8 inputs, so no
// inf / NaN can arise (plan.cc).
bool chain_bounded(const dctf_plan& p);
dctf_status upload_refchain_only(dctf_plan* p);  // quant.cu: data of k_refchain8
dctf_status launch_refchain8(const dctf_plan* p, const uint8_t* in, uint8_t* out, int w, int h, size_t pitch,
                             long long frame_stride, int nframes, cudaStream_t st);

// TMA tensor map over block-major FP64 coefficients (capi.cu): 2-D
// [nblocks rows x nn cols], box [box_rows x 16 cols], 128B swizzle.
dctf_status make_xmap(void* map, const double* d, long long nblocks, int nn, int box_rows, int l2promo = 3);
// TMA tensor map over a u8 frame batch (capi.cu): 3-D [nframes][h][w], box
// [1][8][box_w], no swizzle, OOB -> 0.
dctf_status make_imap(void* map, const uint8_t* d, int w, int h, int nframes, size_t pitch,
                      long long frame_stride, int box_w,
                      int elem_bytes = 1);

// Exact-INT8 tcgen05 fused n=8 path (ozaki.cu).
dctf_status upload_i8_operator(dctf_plan* p);
dctf_status launch_fused8_i8(const dctf_plan* p, const uint8_t* in, uint8_t* out, int w, int h, size_t pitch,
                             long long frame_stride, int nframes, double* coef_out, cudaStream_t st, int sms);

// Exact-integer composed-operator n = 8 image path (quant.cu): uploads the
// plan's digit image and fallback data; launches the kernel for a batch of
// frames whose plans are plans[plan_of_frame[f]] (all kq-enabled, n = 8, one
// device), then the reference-order fallback over the flagged blocks.
dctf_status upload_kq_operator(dctf_plan* p);
dctf_status launch_fused8_q(const dctf_plan* const* plans, int nplans, const int* plan_of_frame,
                            const uint8_t* in, uint8_t* out, int w, int h, size_t pitch, long long frame_stride,
                            int nframes, cudaStream_t st, bool host_mapped, int* d_nan_or_null);
constexpr int KQ_MAX_PLANS = 4;
constexpr int KQ_MAX_FRAMES = 1024;

// 3xTF32 tcgen05 coefficient filter (tc.cu).
dctf_status launch_coef_tf32x3(const dctf_plan* p, const double* d_in, double* d_out, long long nb,
                               cudaStream_t st, int sms);

// Programmatic dependent launch: kernels written for it (pdl_wait() before
// their first access to caller buffers, device.cuh) are launched with
// programmatic stream serialisation, so a launch overlaps the tail of the
// preceding grid on the stream (its CTAs start as SMs free up and stage their
// operators; their image work still waits for the predecessor to complete).
// DCTF_PDL=0 in the environment launches them conventionally.
bool pdl_enabled();
template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kernel)(KArgs...), unsigned grid, unsigned block, size_t smem, cudaStream_t st,
                       Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

}  // namespace dctf

// Returns DCTF_CUDA_ERROR (with the failing expression and CUDA's message)
// from the enclosing dctf_status function when a runtime call fails.
#define CUDA_TRY(expr)                                                                   \
  do {                                                                                   \
    cudaError_t e_ = (expr);                                                             \
    if (e_ != cudaSuccess)                                                               \
      return set_error(DCTF_CUDA_ERROR, std::string(#expr ": ") + cudaGetErrorString(e_)); \
  } while (0)
