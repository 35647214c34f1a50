/*
 * dctf.h — C ABI of the B200-native DCT-domain block filter
 * (libdctf_b200.so, built from paper_1710_07193_b200/csrc).
 *
 * This is the drop-in boundary for the reference's hot path
 * (arXiv 1710.07193, reference library /root/reference/proj/include/dctfilter).
 * Plain pointers and sizes only. Every entry point is batched: one call
 * covers a whole image or a whole range of blocks, where the reference works
 * one BlockMatrix at a time.
 *
 * Data layouts
 *   image    : u8, row-major, `pitch` bytes between rows (pitch >= width).
 *   coeffs   : FP64, block-major. Block b = by * bw + bx (row-major block grid,
 *              the order of tile(), image.hpp:164-184); within a block,
 *              coefficient (u, v) at u * n + v (BlockMatrix row-major,
 *              block_matrix.hpp:46). bw = ceil(w/n), bh = ceil(h/n).
 *   blocks   : FP64 spatial samples, same layout as coeffs.
 *   operator : FP64 n^2 x n^2 row-major; row (u*n+v), column (a*n+b).
 *
 * Device pointers: every `d_` argument is device memory (cudaMalloc'd,
 * 16-byte aligned for the fast paths); `stream` is a cudaStream_t (NULL =
 * legacy default stream). Calls are asynchronous with respect to the host
 * unless stated. `h_` arguments are host memory.
 *
 * Errors: every call returns a dctf_status; the reference throws instead
 * (std::invalid_argument, filter.hpp / spatial.hpp / mask.hpp). A
 * thread-local message describes the last failure.
 *
 * Thread-safety: a plan is immutable after dctf_plan_create; concurrent calls
 * on one plan from several host threads / streams are allowed, as for the
 * reference FilterPlan (filter.hpp:47-51).
 */
#ifndef DCTF_H
#define DCTF_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  DCTF_OK = 0,
  DCTF_INVALID_ARGUMENT = 1, /* reference: std::invalid_argument           */
  DCTF_CUDA_ERROR = 2,       /* CUDA runtime / launch failure              */
  DCTF_NAN_ENCOUNTERED = 3,  /* reference: quantize_sample throws on NaN   */
  DCTF_UNSUPPORTED = 4       /* valid request this build does not provide  */
} dctf_status;

typedef enum { DCTF_PAD_ZERO = 0, DCTF_PAD_REPLICATE = 1 } dctf_padding; /* spatial.hpp:29-32 */

typedef enum {
  DCTF_PREC_FP64 = 0,    /* FP64-exact: coefficients on the FP64 DMMA pipe within
                            1e-9 rel.; the n = 8 u8 image path (no coefficient
                            output) on k_fused8_q — the fused chain composed
                            into one operator, exact int8 tcgen05 digit slices,
                            u8 equal to the reference's on every pixel (error-
                            bounded rounding, reference-order fallback)      */
  DCTF_PREC_TF32X3 = 1,  /* split-precision tcgen05 kind::tf32, 3 passes          */
  DCTF_PREC_BF16X3 = 2,  /* split-precision tcgen05 kind::f16 (bf16), 3 passes;
                            coefficients within ~1e-4 rel. (16-bit split)     */
  DCTF_PREC_INT8_EXACT = 3, /* n = 8 image path: DCT-domain contraction as exact INT8
                              tcgen05 slices (FP64-class accuracy); other entry
                              points of such a plan run the FP64 kernels        */
  DCTF_PREC_FP64_DENSE = 4, /* as FP64_DMMA, but never exploit operator structure:
                              the n = 8 image path runs the dense k_fused8 (a
                              DMMA plan whose H is block-diagonal in the
                              (u mod 2, v mod 2) classes runs the parity-class
                              kernel, a low-rank mask the sandwich kernel)     */
  DCTF_PREC_FP64_DMMA = 5   /* as FP64, but the n = 8 u8 image path stays on the
                              FP64 DMMA kernels (k_fused8_sep / _sym / k_fused8)
                              instead of the exact-integer k_fused8_q          */
} dctf_precision;

typedef struct dctf_plan dctf_plan;

/* Replaces FilterPlan(const Mask&, int n, PaddingMode) (filter.hpp:54-56)
 * together with Mask(int k, std::vector<double>) (mask.hpp:29-41).
 * weights: kr x kc row-major, kr and kc odd, finite. The reference accepts
 * square masks with k <= n only (operators.hpp:84,106); those compile exactly
 * like the reference (shift/band pairs, merge_symmetric, to_dct_domain). This
 * build also accepts kr != kc and masks wider than the block (convolve
 * formula, spatial.hpp:36-37, with the k <= n guard lifted).
 * n: block side, 8 or 16. device: CUDA ordinal the plan's operator lives on. */
dctf_status dctf_plan_create(const double* h_weights, int kr, int kc, int n, int padding,
                             int precision, int device, dctf_plan** out);
dctf_status dctf_plan_destroy(dctf_plan* plan);

/* Operator dump format of the reference (write_operator_sets /
 * read_operator_sets, operator_io.hpp:105-217; what `build-operators` writes,
 * dctfilter_main.cc:163-183): the plan's spatial and DCT-domain sandwich
 * sets, every double printed with %.17g, so the text is byte-identical to the
 * reference's and round-trips bit for bit.
 *   dctf_plan_dump: writes up to *len bytes into buf (if buf && *len is
 *     large enough) and sets *len to the full size. Square masks only.
 *   dctf_plan_create_from_dump: builds a plan from a dump's DCT-domain set
 *     (a spatial-only dump is conjugated), checking the header, version, mask
 *     fingerprint and counts as read_operator_sets does (errors ->
 *     DCTF_INVALID_ARGUMENT with the reference's message text). */
dctf_status dctf_plan_dump(const dctf_plan* plan, char* buf, size_t* len);
/* A plan from an explicit sandwich set — the operand of apply(set, X)
 * (filter.hpp:40-45) and apply_pairs (filter.hpp:30-38): npairs (left,
 * right) factors, n*n doubles each, row-major; domain 0 = spatial (conjugated
 * into the DCT domain as to_dct_domain does, operators.hpp:124-141),
 * 1 = DCT. The k x k mask (OperatorSet::mask) drives the spatial path and the
 * fingerprint; the DCT-domain filter follows the pairs. */
dctf_status dctf_plan_create_from_pairs(const double* h_lefts, const double* h_rights, int npairs, int n,
                                        int domain, const double* h_weights, int k, int padding, int precision,
                                        int device, dctf_plan** out);
dctf_status dctf_plan_create_from_dump(const char* text, size_t len, int precision, int device,
                                       dctf_plan** out);

/* Host-only variants (no device): the dump of the sets FilterPlan would
 * compile for a square k x k mask, and the dense operator H (n^4) a dump
 * describes (plus its n, k, padding). */
dctf_status dctf_format_operator_dump(const double* h_weights, int k, int n, int padding, char* buf,
                                      size_t* len);
dctf_status dctf_operator_from_dump(const char* text, size_t len, double* h_op, int* n, int* k,
                                    int* padding);

/* The plan's sandwich pairs (OperatorSet::pairs, operators.hpp:43-53):
 * domain 0 = spatial (after merge_symmetric), 1 = DCT. npairs * n*n doubles
 * each (see dctf_plan_info). Square masks only. */
dctf_status dctf_plan_pairs(const dctf_plan* plan, int domain, double* h_lefts, double* h_rights);

/* Plan metadata: block side, sandwich pair count and whether mirrored rows
 * were merged (OperatorSet::pairs.size(), ::symmetric_merged). */
dctf_status dctf_plan_info(const dctf_plan* plan, int* n, int* npairs, int* symmetric_merged);

/* The plan's mask (kr x kc weights, row-major; NULL h_weights to query the
 * shape only) and padding — for plans read from an operator dump, the dump's
 * mask and padding (operator_io.hpp: read_operator_sets). */
dctf_status dctf_plan_mask(const dctf_plan* plan, double* h_weights, int* kr, int* kc, int* padding);

/* Name of the kernel dctf_filter_image_u8 runs for this plan:
 *   n = 8:  "k_fused8_q" (DCTF_PREC_FP64 default: exact-integer tcgen05
 *           composed operator + reference-order fallback), "k_fused8_sep"
 *           (separable sandwich, DMMA), "k_fused8_sym" (parity classes,
 *           DMMA), "k_fused8" (dense DMMA), "k_fused8_i8" (INT8-exact digit
 *           slices, DCTF_PREC_INT8_EXACT);
 *   n = 16: "k_fused16_sep", "k_fused16_sym", "k_fused16";
 *   "unfused" (forward -> filter_coeffs -> inverse; the split-precision modes).
 * NULL for a NULL plan. */
const char* dctf_plan_image_kernel(const dctf_plan* plan);

/* Name of the kernel dctf_filter_coeffs runs for this plan: "k_coef8_sep" /
 * "k_coef16_sep" (separable sandwich), "k_coef8_sym" / "k_coef16_sym"
 * (parity-class structure), "k_coef8" / "k_coef16" (dense), "k_coef_tf32x3"
 * or "k_coef_bf16x3" (split precision on tcgen05). NULL for a NULL plan. */
const char* dctf_plan_coef_kernel(const dctf_plan* plan);

/* Host-only operator compile (no device needed): the same compile
 * dctf_plan_create performs, returning C (n*n) and H (n^4) into host buffers
 * (either may be NULL) plus the pair count / merge flag. */
dctf_status dctf_compile_operator(const double* h_weights, int kr, int kc, int n, int padding,
                                  double* h_c, double* h_op, int* npairs, int* symmetric_merged);

/* Host FP64 copies: the DCT basis C (n*n; DctBasis::c(), dct.hpp:37) and the
 * dense DCT-domain operator H (n^4), H = sum_p L_p (x) R_p^T of the plan's
 * sandwich pairs (FilterPlan::dct_set(), filter.hpp:62). */
dctf_status dctf_plan_basis(const dctf_plan* plan, double* h_c);
dctf_status dctf_plan_operator(const dctf_plan* plan, double* h_op);

/* forward_2d over a u8 image: tile() (edge replication of ragged edges) then
 * C X C^t per block (dct.hpp:59-62). d_coeffs: bw*bh*n*n doubles. */
dctf_status dctf_forward(const dctf_plan* plan, const uint8_t* d_img, int width, int height,
                         size_t pitch, double* d_coeffs, void* stream);

/* forward_2d / inverse_2d over FP64 blocks (dct.hpp:59-68). */
dctf_status dctf_forward_blocks(const dctf_plan* plan, const double* d_blocks, double* d_coeffs,
                                size_t nblocks, void* stream);
dctf_status dctf_inverse_blocks(const dctf_plan* plan, const double* d_coeffs, double* d_blocks,
                                size_t nblocks, void* stream);

/* FilterPlan::filter_coeffs (filter.hpp:65-67) over nblocks coefficient
 * blocks: out_b = H * in_b. In-place (d_in == d_out) is not allowed. */
dctf_status dctf_filter_coeffs(const dctf_plan* plan, const double* d_in, double* d_out,
                               size_t nblocks, void* stream);

/* inverse_2d + assemble() (image.hpp:188-203): C^t Y C per block, round half
 * away from zero, clamp to [0,255], crop to width x height. A NaN sample sets
 * the plan's NaN flag (see dctf_plan_nan_check). */
dctf_status dctf_inverse_u8(const dctf_plan* plan, const double* d_coeffs, uint8_t* d_img,
                            int width, int height, size_t pitch, void* stream);

/* filter_image(img, mask, padding, Domain::kDct, n) (image.hpp:210-218),
 * fused on the device: u8 -> forward DCT -> H -> inverse DCT -> round/clamp
 * -> u8 in one HBM pass. d_in and d_out may not alias. If d_coeffs_out is not
 * NULL the filtered coefficients (bw*bh*n*n doubles) are also written
 * (parity mode). */
dctf_status dctf_filter_image_u8(const dctf_plan* plan, const uint8_t* d_in, uint8_t* d_out,
                                 int width, int height, size_t pitch, double* d_coeffs_out,
                                 void* stream);

/* The spatial path of filter_image (Domain::kSpatial, image.hpp:219-222):
 * convolve (spatial.hpp:41-68) per block with the plan's mask and padding, in
 * the reference's operation order (bit-identical samples), then quantize +
 * crop. A second on-device oracle for the DCT path, and the competing
 * algorithm (k^2 MACs per pixel). */
dctf_status dctf_filter_image_spatial_u8(const dctf_plan* plan, const uint8_t* d_in, uint8_t* d_out,
                                         int width, int height, size_t pitch, void* stream);

/* Host-buffer variant of the spatial path (synchronous). */
dctf_status dctf_filter_image_spatial_host(const dctf_plan* plan, const uint8_t* h_in, uint8_t* h_out,
                                           int width, int height, size_t pitch);

/* convolve (spatial.hpp:41-68) over FP64 blocks (nblocks x n x n). */
dctf_status dctf_convolve_blocks(const dctf_plan* plan, const double* d_blocks, double* d_out,
                                 size_t nblocks, void* stream);

/* Frame batch (video): frame f (0..nframes-1) of the d_in batch is filtered
 * with plans[plan_of_frame[f]]; frames are frame_stride bytes apart, all
 * width x height with the same pitch. All plans must share n and device. */
dctf_status dctf_filter_frames_u8(const dctf_plan* const* plans, int nplans,
                                  const int* h_plan_of_frame, const uint8_t* d_in, uint8_t* d_out,
                                  int nframes, int width, int height, size_t pitch,
                                  size_t frame_stride, void* stream);

/* Frame batch on HOST buffers (synchronous): filter_image (image.hpp:210-225)
 * per frame, frame f with plans[plan_of_frame[f]]. Frames stream through a
 * per-call 3-slot device ring in ~16 MiB chunks; the H2D copy, the batch
 * kernel and the D2H copy of consecutive chunks overlap on three per-thread
 * streams. Pinned (cudaHostAlloc'd) buffers run at PCIe speed. Concurrent
 * calls from several host threads are allowed. */
dctf_status dctf_filter_frames_host(const dctf_plan* const* plans, int nplans, const int* h_plan_of_frame,
                                    const uint8_t* h_in, uint8_t* h_out, int nframes, int width, int height,
                                    size_t pitch, size_t frame_stride);

/* Multi-GPU (one process, one host thread and stream per device;
 * SURVEY.md §8(e)). Blocks never exchange data (image.hpp:205-209), so a
 * dctf_multi holds one replica of a plan per listed device (a device may be
 * listed twice: two replicas on one GPU) and the entries shard contiguous
 * block-row bands (one image) or contiguous frame ranges (a batch) over the
 * replicas, shard r = [total*r/N, total*(r+1)/N), with no data-path
 * collective. Results are byte-identical to the single-device entries. */
typedef struct dctf_multi dctf_multi;
dctf_status dctf_multi_create(const double* h_weights, int kr, int kc, int n, int padding, int precision,
                              const int* devices, int ndevices, dctf_multi** out);
dctf_status dctf_multi_destroy(dctf_multi* m);
/* Replica count and replica 0 (for the per-plan queries above). */
dctf_status dctf_multi_info(const dctf_multi* m, int* ndevices, const dctf_plan** replica0);
dctf_status dctf_multi_replica(const dctf_multi* m, int r, const dctf_plan** out);
/* filter_image on host buffers, block-row bands over the replicas. */
dctf_status dctf_filter_image_host_multi(const dctf_multi* m, const uint8_t* h_in, uint8_t* h_out, int width,
                                         int height, size_t pitch);
/* dctf_filter_frames_host with frame ranges over the replicas (plans[i] are
 * dctf_multi over the same device list). */
dctf_status dctf_filter_frames_host_multi(const dctf_multi* const* plans, int nplans, const int* h_plan_of_frame,
                                          const uint8_t* h_in, uint8_t* h_out, int nframes, int width, int height,
                                          size_t pitch, size_t frame_stride);
/* Device-resident batch: replica r filters its shard of frames
 * [nframes*r/N, nframes*(r+1)/N) from d_in[r] into d_out[r] (both on its
 * device, holding just that shard, frame_stride apart) on streams[r] (NULL
 * list = default streams). With d_gather != NULL (and nframes % N == 0) the
 * shards are all-gathered so d_gather[r] holds all nframes frames in order
 * — NCCL (libnccl.so.2 loaded at run time; NVLink / NVSwitch), distinct
 * devices only, else DCTF_UNSUPPORTED. Returns after the gather completes. */
dctf_status dctf_filter_frames_u8_multi(const dctf_multi* const* plans, int nplans, const int* h_plan_of_frame,
                                        const uint8_t* const* d_in, uint8_t* const* d_out, int nframes, int width,
                                        int height, size_t pitch, size_t frame_stride, uint8_t* const* d_gather,
                                        void* const* streams);

/* End-to-end host-buffer entry (the reference's filter_image signature).
 * Synchronous; returns DCTF_NAN_ENCOUNTERED where quantize_sample would
 * throw. Plans on k_fused8_q (n = 8 FP64) and the split-precision plans:
 * bands of whole block rows (~16 MiB) stream through a per-call 3-slot device
 * ring, H2D copy / kernel / D2H copy of consecutive bands overlapped on the
 * calling thread's three streams (no plan lock; concurrent callers overlap).
 * Other plans: pinned (cudaHostAlloc'd, mapped) buffers are read and written
 * by the fused kernel itself over PCIe (zero-copy); pageable buffers go
 * through pinned bounce buffers filled and drained by host threads; these
 * modes use plan-owned staging under a per-plan lock. */
dctf_status dctf_filter_image_host(const dctf_plan* plan, const uint8_t* h_in, uint8_t* h_out,
                                   int width, int height, size_t pitch);

/* Host-buffer batch variants (synchronous): copy nblocks blocks in, run the
 * device kernel, copy out. For callers without device memory management —
 * the C++ drop-in layer (include/dctfilter_b200.hpp) builds the reference's
 * per-block functions on these. */
dctf_status dctf_forward_blocks_host(const dctf_plan* plan, const double* h_blocks,
                                     double* h_coeffs, size_t nblocks);
dctf_status dctf_inverse_blocks_host(const dctf_plan* plan, const double* h_coeffs,
                                     double* h_blocks, size_t nblocks);
dctf_status dctf_filter_coeffs_host(const dctf_plan* plan, const double* h_in, double* h_out,
                                    size_t nblocks);
dctf_status dctf_convolve_blocks_host(const dctf_plan* plan, const double* h_blocks, double* h_out,
                                      size_t nblocks);
/* FilterPlan::filter_block (filter.hpp:71-73) over nblocks spatial FP64
 * blocks: inverse_2d(filter_coeffs(forward_2d(x))), the three kernels on the
 * calling thread's stream with one copy each way (reference operation order
 * for the transforms). */
dctf_status dctf_filter_blocks_host(const dctf_plan* plan, const double* h_blocks, double* h_out,
                                    size_t nblocks);

/* NaN reporting (quantize_sample throws on NaN, spatial.hpp:71-75). The
 * device-buffer entries (dctf_filter_image_u8, dctf_filter_frames_u8,
 * dctf_inverse_u8, dctf_filter_image_spatial_u8) run asynchronously and set
 * the plan's NaN flag (a frame batch: its first plan's); this call
 * synchronises `stream`, reads and clears that flag: *nan_seen is 1 if any
 * quantised sample was NaN since the last check. The flag is one word per
 * plan: concurrent device-entry callers on one plan share it. The host-buffer
 * entries (dctf_filter_image_host, dctf_filter_frames_host, their _multi
 * forms, dctf_filter_image_spatial_host) use a per-call flag instead and
 * return DCTF_NAN_ENCOUNTERED themselves.
 * A NaN can only arise for masks whose reference chain overflows FP64 (huge
 * weights); such plans run the reference's own operation order on the image
 * path (dctf_plan_image_kernel: "k_refchain8" at n = 8, "unfused" at n = 16),
 * so NaN arises where the reference's does. */
dctf_status dctf_plan_nan_check(const dctf_plan* plan, void* stream, int* nan_seen);

/* Diagnostics: measures this device's FP64 peak with a throughput
 * microbenchmark (mode 0: DMMA.8x8x4 via mma.sync.m8n8k4.f64 — the pipe the
 * filter kernels use; mode 1: DFMA). Synchronous; ~50 ms. Used as the
 * roofline denominator because the driver's MEASURED_PEAKS.json has no FP64
 * entry. */
dctf_status dctf_measure_fp64_peak(int device, int mode, double* tflops);

/* Diagnostics: blocks k_fused8_q flagged as uncertain (a pixel within the
 * integer path's error bound of a .5 boundary) since the last call, and of
 * those the ones the fallback resolved with the reference-order chain (the
 * rest settled by its FP64 first stage). Process-wide; needs DCTF_Q_COUNT=1
 * in the environment before the first filter call, else DCTF_UNSUPPORTED.
 * Synchronises the current device; resets both counters. chain may be NULL. */
dctf_status dctf_diag_fallback_counts(unsigned long long* flagged, unsigned long long* chain);
/* The flagged count alone (same counters). */
dctf_status dctf_diag_fallback_blocks(unsigned long long* n);

/* Diagnostics: how k_fused8_q represents this plan's composed 64 x 64 pixel
 * operator K. *denominator > 0: K = K' / denominator with integer K' (odd
 * denominator; integer masks, odd box means, odd motion blurs) — one int8
 * digit and one accumulator per pixel, exact rounding without a near-tie
 * test. *denominator = 0: round(K 2^*fraction_bits) in four int8 digits with
 * the uncertainty window and the reference-order fallback. DCTF_UNSUPPORTED
 * when the plan does not run k_fused8_q. Either pointer may be NULL. */
dctf_status dctf_plan_kq_form(const dctf_plan* plan, int* denominator, int* fraction_bits);

/* Diagnostics: this device's INT8 tensor-core throughput (tera-ops/s,
 * 2 ops per MAC) with back-to-back tcgen05.mma kind::i8 M128 N256 K32 from
 * shared memory — the roofline denominator of k_fused8_q's tensor side.
 * Synchronous; ~10 ms. */
dctf_status dctf_measure_int8_peak(int device, double* tops);

/* Number of kernels the last call on this host thread launched (bench
 * accounting of gpu_launches). */
int dctf_last_launch_count(void);

/* Thread-local description of the last non-OK status. */
const char* dctf_last_error_message(void);

/* Library version string. */
const char* dctf_version(void);

#ifdef __cplusplus
}
#endif
#endif /* DCTF_H */
