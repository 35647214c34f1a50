// k_fused8_q: the 8x8 spatial-in/spatial-out DCT-domain filter
// (filter_image, image.hpp:210-225; per block filter_block, filter.hpp:71-73,
// then quantize_sample, spatial.hpp:71-75) as ONE exact integer contraction
// on the 5th-generation tensor cores (tcgen05.mma kind::i8, int32
// accumulators in TMEM), sm_100a.
//
// Math. The fused chain is three linear maps on a block's pixels p (forward
// DCT, the DCT-domain operator H_dct, inverse DCT); plan.cc: layout_kq8
// composes them on the host into one 64 x 64 operator K = (C (x) C)^t H (C (x) C)
// (long double, from the plan's own DCT-domain pairs) and writes it as
// K_int = round(K 2^F) in four balanced base-256 int8 digits. Pixels are
// exact u8, so every tensor-core partial a_s = sum_j d_s[i][j] p_j is an
// exact int32 and z_int = sum_s a_s 256^(3-s) is the exact fixed-point value
// of K_int p. Its only error against the exact chain is the operator
// quantisation, bounded per plan (E); together with a margin for the
// reference's own FP64 rounding (M) this gives an uncertainty window T: a
// pixel whose fixed-point value is more than T/2^F from every .5 rounding
// boundary rounds exactly as the reference does (round half away, clamp).
// The rest (~1e-4 of the blocks at the BASELINE masks) are recomputed in the
// reference's own operation order (forward_2d -> apply_pairs -> inverse_2d,
// block_matrix.hpp:67-81's i-k-j products with separately rounded multiply
// and add, dct.hpp:59-68, filter.hpp:30-38; convolve's order for
// convolve-formula plans) by a fallback warp of the same CTA, so the u8
// output is the reference's on every pixel, not only outside near-ties.
//
// Rational operators: when K = K' / d with integer |K'| <= 127 and odd d
// (integer masks, odd box means, odd motion blurs) one digit and ONE
// accumulator per pixel carry N = sum_j K'_ij p_j exactly (MMA N = 64);
// z + 1/2 = (2 N + d) / (2 d) has an odd numerator, so no pixel can be a
// near-tie and q = floor((N + (d - 1) / 2) / d) is the reference's rounding
// everywhere (epi_rational; plan.cc: layout_kq8 has the bound).
//
// Epilogue arithmetic of the four-digit form (per pixel, 32-bit integer ops only): with
// h = a0*256 + a1, l = a2*256 + a3, the rounding offset 2^(F-1) folded in:
//   S = h + (l >> 16) + 2^(F-17)          -> v = S*2^16 + (l & 0xffff)
//   q = S >> (F-16)                        = floor(z + 0.5) (u8 after saturation)
//   key = (v mod 2^F) << (32-F)
//   uncertain  <=>  (key + U) mod 2^32 < 2U,  U = T 2^(32-F)
// The accumulator constants carry T as well, so key is already key + U and the
// per-block test is a running unsigned minimum, two pixels per VIMNMX3.
//
// CTA = 13 warps, one CTA per SM (TMEM: 2 x 256 columns), persistent over
// tiles of up to 128 horizontally adjacent blocks (one block row, 8 x 1024 px).
// Roles in issue-priority order (highest warp id first):
//   warp 12     MMA issuer: the whole warp runs the loop, one elected lane
//               issues the tile's 3 x tcgen05.mma (M 128, N 256, K 32) and two
//               commits in one asm block, into a double-buffered accumulator.
//   warp 11     TMA: one 8 KB box [8 rows x 1024 px] per tile (4 boxes of
//               256 px when the width is not a multiple of 8) into a 6-stage
//               raw ring (48 KB of pixels in flight per SM); a 3-D tensor map
//               covers the whole frame batch, out-of-range pixels read as 0.
//   warps 9-10  converters: thread = a pair of adjacent blocks; one 16-byte
//               shared load per pixel row covers both (tile()'s edge
//               replication for ragged blocks), written into the K-major
//               128-byte-swizzled A operand.
//   warp 8      fallback: flagged blocks from the CTA's queue (FP64 first
//               stage, reference-order chain for near-ties); after the last
//               tile every warp drains what is left.
//   warps 0-7   epilogue: two groups of four warps (one per TMEM lane
//               quarter), group g drains accumulator buffer g (every other
//               tile); thread = block: tcgen05.ld 32 columns = 8 whole pixels
//               per pixel row, the integer rounding above, cvt.pack.sat,
//               8-byte coalesced row stores. Blocks with an uncertain pixel
//               are not stored here; they go to the fallback queue.
// The plans' digit images (32 KB each, up to 4 plans: one launch covers a
// whole multi-mask frame batch) stay resident in shared memory.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <mutex>
#include <string>

#include "device.cuh"
#include "fastdiv.cuh"
#include "internal.h"

using dctf::KQ_MAX_FRAMES;
using dctf::KQ_MAX_PLANS;
using dctf::set_error;

namespace {

#ifdef QDBG
// [cta < 4][tile < 64][event < 32] clock64 stamps of tiles QDBG_T0.. (instrumented build only;
// scripts/kq_trace3.py: 0/1 MMA issue start / done, 2+w wake and 10+w release of epilogue warp w,
// 18 converters' a_full arrival, 19 MMA sees a_full, 21-25 converter: raw stage seen, A stage free,
// rows loaded, A rows stored, proxy fence done)
#ifndef QDBG_T0
#define QDBG_T0 0
#endif
__device__ long long g_qdbg[4][64][48];  // 32 + w: end of epilogue warp w's tile iteration
#define QSTAMP(tl, ev)                                                                                  \
  do {                                                                                                  \
    if (blockIdx.x < 4 && (tl) >= QDBG_T0 && (tl) < QDBG_T0 + 64) g_qdbg[blockIdx.x][(tl)-QDBG_T0][(ev)] = clock64(); \
  } while (0)
#define QSTAMP_EPI(tl, ev)                 \
  do {                                     \
    if (b == 0) QSTAMP(tl, ev);              \
  } while (0)
#else
#define QSTAMP_EPI(tl, ev) \
  do {                     \
  } while (0)
#define QSTAMP(tl, ev) \
  do {                 \
  } while (0)
#endif

namespace q8 {
constexpr int TILE = 128;                  // blocks per tile = MMA M = TMEM lanes
constexpr int NCOL = 256;                  // accumulator columns: 64 pixels x 4 digits
constexpr int ROWB = 128;                  // operand row: 64 pixel bytes + the constant chunk
constexpr int BBYTES = NCOL * ROWB;        // one plan's digit image
constexpr int ABYTES = TILE * ROWB;        // one A stage
constexpr int RAWB = 8 * TILE * 8;         // one raw stage: 8 rows x 1024 px
constexpr int NRAW = 6, NA = 2;
#ifndef Q8_EXP
#define Q8_EXP 0  // measurement variants (bit flags, wrong output): 1 = epilogue without the pixel math,
                  // 2 = without stores (the output bytes kept live), 4 = converters without pixel loads /
                  // A writes, 16 = fallback blocks dequeued, not recomputed
#endif
// epilogue: two groups of 4 warps (one per TMEM lane quarter); group g
// drains accumulator buffer g, i.e. every other tile of the CTA
constexpr int NGRP = 2;
// Warp roles, ordered by issue priority: an SM sub-partition's scheduler
// picks the highest eligible warp id first, so the short, latency-critical
// roles (MMA issue, TMA, the converters that feed the MMA, the fallback warp
// that keeps the flagged-block queue short) sit above the ALU-heavy epilogue.
// Converter sets: each set (two warps) takes every CSETS-th tile of the CTA, so
// a set has CSETS tile periods for its load - transpose - store round trip.
#ifndef Q8_CSETS
#define Q8_CSETS 1
#endif
constexpr int CSETS = Q8_CSETS;
constexpr int W_EPI = 0, NEPI = 4 * NGRP, W_FB = W_EPI + NEPI, W_CONV = W_FB + 1, NCONV = 2 * CSETS,
              W_TMA = W_CONV + NCONV, W_MMA = W_TMA + 1;
static_assert(CSETS == 1 || (NRAW % CSETS == 0 && NA % CSETS == 0), "a stage belongs to one converter set");
constexpr int THREADS = 32 * (W_MMA + 1);
constexpr int FQ = 256;                    // fallback queue slots
constexpr int SMEM = 1024 + KQ_MAX_PLANS * BBYTES + NA * ABYTES + NRAW * RAWB;
}  // namespace q8

// wait flavour per role (measurement switches): sleeping waits by default
#ifdef Q8_SPIN_ALL
#define Q8_WAIT_MMA mbar_wait
#define Q8_WAIT_OTHER mbar_wait
#elif defined(Q8_SPIN_MMA)
#define Q8_WAIT_MMA mbar_wait
#define Q8_WAIT_OTHER mbar_wait_sleep
#else
#define Q8_WAIT_MMA mbar_wait_sleep
#define Q8_WAIT_OTHER mbar_wait_sleep
#endif

struct RefPlan {
  const double* chain;    // C | C^t | lefts | rights (mode 1)
  const double* weights;  // kr x kc (mode 2)
  const double* kt;       // composed operator K in FP64, transposed
  double margin;          // tie window of the FP64 first stage
  int mode, npairs, kr, kc, padding;
};

struct QArgs {
  const int8_t* bimg[KQ_MAX_PLANS];
  uint32_t U[KQ_MAX_PLANS];
  int shS[KQ_MAX_PLANS], shL[KQ_MAX_PLANS];  // F - 16, 32 - F
  // rational plans (K = K' / den, odd den; plan.cc: layout_kq8): den > 0, q = mulhi(acc, magic) - bias
  int den[KQ_MAX_PLANS], bias[KQ_MAX_PLANS];  // den = -1: four digits read as unsigned bytes
  uint32_t magic[KQ_MAX_PLANS];
  RefPlan ref[KQ_MAX_PLANS];
  int nplans;
  dctf::FastDiv fd_tpf, fd_ntx;  // tile -> (frame, block row, tile column), made on the host
  uint8_t pof[KQ_MAX_FRAMES];  // plan of frame
};

// UMMA shared-memory descriptor, K-major, SWIZZLE_128B (8-row atoms of 128 B):
// SBO = 1024 B between 8-row groups, version 1 (sm_100).
__device__ __forceinline__ uint64_t desc_sw128(uint32_t saddr) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((saddr >> 4) & 0x3FFFu);
  d |= static_cast<uint64_t>(1u) << 16;
  d |= static_cast<uint64_t>(1024u >> 4) << 32;
  d |= static_cast<uint64_t>(1u) << 46;
  d |= static_cast<uint64_t>(2u) << 61;
  return d;
}
// kind::i8 instruction descriptor: D s32, A u8 (pixels), B s8 (digits; u8 for
// the unsigned digit images of non-negative operators), both K-major.
__host__ __device__ constexpr uint32_t idesc_u8s8(int m, int n, bool b_unsigned = false) {
  return (2u << 4) | (0u << 7) | ((b_unsigned ? 0u : 1u) << 10) | (static_cast<uint32_t>(n >> 3) << 17) |
         (static_cast<uint32_t>(m >> 4) << 24);
}
__device__ __forceinline__ void mma_u8s8(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                         uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, int32_t (&v)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
        "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
        "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]),
        "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]),
        "=r"(v[30]), "=r"(v[31])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1,
                                            int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
      : "memory");
}
// {sat_u8(x0), sat_u8(x1), sat_u8(x2), sat_u8(x3)} little-endian
__device__ __forceinline__ uint32_t pack4_sat(int x0, int x1, int x2, int x3) {
  uint32_t r;
  asm("{\n\t.reg .u32 t;\n\t"
      "cvt.pack.sat.u8.s32.b32 t, %4, %3, 0;\n\t"
      "cvt.pack.sat.u8.s32.b32 %0, %2, %1, t;\n\t}"
      : "=r"(r)
      : "r"(x0), "r"(x1), "r"(x2), "r"(x3));
  return r;
}

// One pixel row of a block (8 pixels x 4 digit accumulators, TMEM columns
// 4c + s) -> 8 u8 (two words) and the running uncertainty minimum. With
// T1 = a0 256 + a1, T2 = a2 256 + a3 (the rounding offset already added to
// a0 / a1 by the constant K chunk), v = T1 2^16 + T2 = z 2^F:
//   q   = (T1 + (T2 >> 16)) >> (F - 16)      floor(z + 1/2)
//   key = (T1 2^16 + T2) << (32 - F) mod 2^32 = (v mod 2^F) 2^(32-F)
// (F32: F = 32, no shift).
// MODE 0: F < 32 (key shifted by 32 - F); 1: F = 32; 2: F = 32 and the plan's
// outputs provably in [0, 255] (plan.cc: nosat), so the output byte is bits
// 16-23 of S and four pixels pack with three byte permutes instead of four
// shifts and two saturating packs.
template <int MODE>
__device__ __forceinline__ void q8_row(const int32_t (&v)[32], int shS, int shL, uint32_t& mn0, uint32_t& mn1,
                                       uint32_t& w0, uint32_t& w1) {
  int qv[8];
  uint32_t key[8];
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    const int t1 = v[4 * c] * 256 + v[4 * c + 1];
    const int t2 = v[4 * c + 2] * 256 + v[4 * c + 3];
    key[c] = static_cast<uint32_t>(t1) * 65536u + static_cast<uint32_t>(t2);
    if (MODE == 0) key[c] <<= shL;
    qv[c] = MODE == 2 ? t1 + (t2 >> 16) : (t1 + (t2 >> 16)) >> shS;
  }
  // the accumulators carry the window half-width (plan.cc: layout_kq8), so
  // key = frac + U already: uncertain iff key < 2 U; pairs of pixels per minimum
  mn0 = __vimin3_u32(mn0, key[0], key[1]);
  mn1 = __vimin3_u32(mn1, key[2], key[3]);
  mn0 = __vimin3_u32(mn0, key[4], key[5]);
  mn1 = __vimin3_u32(mn1, key[6], key[7]);
  if (MODE == 2) {
    w0 = __byte_perm(__byte_perm(qv[0], qv[1], 0x0062), __byte_perm(qv[2], qv[3], 0x0062), 0x5410);
    w1 = __byte_perm(__byte_perm(qv[4], qv[5], 0x0062), __byte_perm(qv[6], qv[7], 0x0062), 0x5410);
  } else {
    w0 = pack4_sat(qv[0], qv[1], qv[2], qv[3]);
    w1 = pack4_sat(qv[4], qv[5], qv[6], qv[7]);
  }
}

// The epilogue's ROWS pixel rows of one tile: row r's math overlaps the TMEM
// load of row r + 1; the accumulator is released after the last load.
template <int ROWS, int MODE>
__device__ __forceinline__ void epi_rows(uint32_t col0, int32_t (&va)[32], int32_t (&vb)[32], int shS, int shL,
                                         uint32_t& mn0, uint32_t& mn1, uint32_t (&words)[2 * ROWS],
                                         uint64_t* acc_empty, long long* stamp = nullptr) {
  tmem_ld32(col0, va);
  tmem_wait_ld();
  if (ROWS == 1) {
    tc_fence_before();
    mbar_arrive(acc_empty);
  }
#pragma unroll
  for (int r = 0; r < ROWS; ++r) {
    if (r + 1 < ROWS) tmem_ld32(col0 + 32 * (r + 1), (r & 1) ? va : vb);
#if Q8_EXP & 1
    words[2 * r] = ((r & 1) ? vb : va)[0];
    words[2 * r + 1] = ((r & 1) ? vb : va)[31];
#else
    q8_row<MODE>((r & 1) ? vb : va, shS, shL, mn0, mn1, words[2 * r], words[2 * r + 1]);
#endif
    if (r + 1 < ROWS) {
      tmem_wait_ld();
      if (r + 2 == ROWS) {
        tc_fence_before();
        mbar_arrive(acc_empty);  // accumulator drained: the MMA of tile tl+2 may start
#ifdef QDBG
        if (stamp && (threadIdx.x & 31) == 0) *stamp = clock64();
#endif
      }
    }
  }
}

// Rational plans (K = K' / den, odd den): the tile's 64 accumulator columns
// (one per pixel: N + (den - 1) / 2 + bias den, exact) in two loads, released
// at once; q = floor(acc / den) - bias by an exact multiply-high (den > 1).
// No pixel of such a plan can be a near-tie (plan.cc: layout_kq8).
__device__ __forceinline__ void epi_rational(uint32_t col0, int den, uint32_t magic, int bias, uint32_t (&words)[16],
                                             uint64_t* acc_empty, long long* stamp = nullptr) {
  int32_t va[32], vb[32];
  tmem_ld32(col0, va);
  tmem_ld32(col0 + 32, vb);
  tmem_wait_ld();
  tc_fence_before();
  mbar_arrive(acc_empty);
#ifdef QDBG
  if (stamp && (threadIdx.x & 31) == 0) *stamp = clock64();
#else
  (void)stamp;
#endif
#pragma unroll
  for (int r = 0; r < 8; ++r) {
    const int32_t(&v)[32] = r < 4 ? va : vb;
    int q[8];
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      const uint32_t a = static_cast<uint32_t>(v[8 * (r & 3) + c]);
      q[c] = static_cast<int>(den == 1 ? a : __umulhi(a, magic)) - bias;
    }
    words[2 * r] = pack4_sat(q[0], q[1], q[2], q[3]);
    words[2 * r + 1] = pack4_sat(q[4], q[5], q[6], q[7]);
  }
}

// A-operand row (= MMA row = TMEM lane) of block b of the tile, an
// involution: bit 0 flipped when bit 3 is set. A converter store instruction
// writes blocks 2 c2 + hb of its 32 threads; with the identity map their rows
// fell on 4 of the 8 128B-swizzle phases (2-way bank conflicts on every A
// store), with this map on all 8. The epilogue's lanes see the same 32
// blocks in a permuted order, so its row stores stay one 256-byte segment.
__device__ __forceinline__ int a_row(int b) { return b ^ ((b >> 3) & 1); }

// Cropped byte stores of ROWS rows (image edges, unaligned outputs).
template <int ROWS>
__device__ __noinline__ void store_ragged(uint8_t* ob, size_t pitch, const uint32_t (&words)[2 * ROWS],
                                             int rows_left, int cols_left) {
#pragma unroll
  for (int k = 0; k < ROWS; ++k)
#pragma unroll
    for (int c = 0; c < 8; ++c)
      if (k < rows_left && c < cols_left)
        ob[static_cast<size_t>(k) * pitch + c] = static_cast<uint8_t>(words[2 * k + (c >> 2)] >> (8 * (c & 3)));
}

// Appends the warp's flagged blocks (ballot `flagged`) to the fallback ring.
__device__ __noinline__ void enqueue_fallback(unsigned long long* fq, uint32_t* tail, uint32_t flagged, bool mine,
                                              int lane, long long ti, int b) {
  uint32_t slot0 = 0;
  if (lane == 0) slot0 = atomicAdd(tail, static_cast<uint32_t>(__popc(flagged)));
  slot0 = __shfl_sync(0xFFFFFFFFu, slot0, 0);
  if (mine) {
    // entry = claim sequence number (high word: consumers claim slots out of
    // order, so a ring slot may still hold the entry FQ claims earlier) |
    // (tile << 7 | block) + 1 (low word, never 0; tiles < 2^24)
    const uint32_t seq = slot0 + __popc(flagged & ((1u << lane) - 1u));
    volatile unsigned long long* qs = &fq[seq % q8::FQ];
    while (*qs != 0ull) __nanosleep(64);  // ring full (pathological masks only)
    *qs = static_cast<unsigned long long>(seq) << 32 |
          ((static_cast<unsigned long long>(ti) << 7 | static_cast<unsigned long long>(b)) + 1ull);
  }
}

// The reference's per-block chain on one flagged block, one warp: lane owns
// outputs e = lane and lane + 32. Every product is block_matrix.hpp:67-81's
// (per output element: k ascending, a(i,k) == 0 skipped, separately rounded
// multiply and add from +0.0); sums as add() (block_matrix.hpp:94-101).
__device__ __forceinline__ double ref_mm(const double* a, const double* b, int i, int j) {
  double acc = 0.0;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const double aik = a[i * 8 + k];
    if (aik == 0.0) continue;
    acc = __dadd_rn(acc, __dmul_rn(aik, b[k * 8 + j]));
  }
  return acc;
}

__device__ __noinline__ bool fallback_block(const RefPlan& rp, const uint8_t* img, size_t pitch, int w, int h, int y0, int x0,
                               uint8_t* dst, bool fast_out, double* sm, int* nan_flag, int lane) {
  double* sx = sm;        // X (pixels, then forward coefficients)
  double* st = sm + 64;   // products
  double* sa = sm + 128;  // apply_pairs accumulator
  double* s2 = sm + 192;
  for (int e = lane; e < 64; e += 32) {
    const int r = e >> 3, c = e & 7;
    const int yy = min(y0 + r, h - 1), xx = min(x0 + c, w - 1);
    sx[e] = static_cast<double>(img[static_cast<size_t>(yy) * pitch + xx]);
  }
  __syncwarp();
  double z[2];
  // First stage: z = K p in FP64 (error far below the reference's own); a
  // block with no pixel within rp.margin of a .5 boundary is final here.
  // (No first stage for unbounded plans, rp.kt == nullptr: k_refchain8.)
  if (rp.kt) {
    double a0 = 0.0, a1 = 0.0;
#pragma unroll 8
    for (int j = 0; j < 64; ++j) {
      const double pj = sx[j];
      a0 = fma(__ldg(rp.kt + j * 64 + lane), pj, a0);
      a1 = fma(__ldg(rp.kt + j * 64 + lane + 32), pj, a1);
    }
    const double t0 = a0 + 0.5, t1 = a1 + 0.5;
    const double f0 = t0 - floor(t0), f1 = t1 - floor(t1);
    const bool tie = f0 < rp.margin || f0 > 1.0 - rp.margin || f1 < rp.margin || f1 > 1.0 - rp.margin;
    if (!__any_sync(0xFFFFFFFFu, tie)) {
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        const int e = lane + 32 * q, r = e >> 3, c = e & 7;
        const double t = floor(q ? t1 : t0);
        const uint32_t v = static_cast<uint32_t>(fmin(fmax(t, 0.0), 255.0));
        if (y0 + r < h && x0 + c < w) dst[static_cast<size_t>(r) * pitch + c] = static_cast<uint8_t>(v);
      }
      __syncwarp();
      return false;
    }
  }
  if (rp.mode == 1) {
    const double* C = rp.chain;
    const double* Ct = rp.chain + 64;
    // forward_2d: (C X) C^t
    for (int e = lane; e < 64; e += 32) st[e] = ref_mm(C, sx, e >> 3, e & 7);
    __syncwarp();
    for (int e = lane; e < 64; e += 32) s2[e] = ref_mm(st, Ct, e >> 3, e & 7);
    __syncwarp();
    // apply_pairs: acc = acc + (L_p X) R_p
    double acc[2] = {0.0, 0.0};
    for (int p = 0; p < rp.npairs; ++p) {
      const double* L = rp.chain + 128 + 64 * p;
      const double* R = rp.chain + 128 + 64 * (rp.npairs + p);
      for (int e = lane; e < 64; e += 32) st[e] = ref_mm(L, s2, e >> 3, e & 7);
      __syncwarp();
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        const int e = lane + 32 * q;
        acc[q] = __dadd_rn(acc[q], ref_mm(st, R, e >> 3, e & 7));
      }
      __syncwarp();
    }
    sa[lane] = acc[0];
    sa[lane + 32] = acc[1];
    __syncwarp();
    // inverse_2d: (C^t Y) C
    for (int e = lane; e < 64; e += 32) st[e] = ref_mm(Ct, sa, e >> 3, e & 7);
    __syncwarp();
    z[0] = ref_mm(st, C, lane >> 3, lane & 7);
    z[1] = ref_mm(st, C, (lane + 32) >> 3, lane & 7);
  } else {
    // convolve (spatial.hpp:41-68): taps r ascending, c ascending
    const int hr = (rp.kr - 1) / 2, hc = (rp.kc - 1) / 2;
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const int e = lane + 32 * q, i = e >> 3, j = e & 7;
      double acc = 0.0;
      for (int r = 0; r < rp.kr; ++r)
        for (int c = 0; c < rp.kc; ++c) {
          int si = i + r - hr, sj = j + c - hc;
          if (rp.padding == DCTF_PAD_ZERO) {
            if (si < 0 || si >= 8 || sj < 0 || sj >= 8) continue;
          } else {
            si = min(max(si, 0), 7);
            sj = min(max(sj, 0), 7);
          }
          acc = __dadd_rn(acc, __dmul_rn(rp.weights[r * rp.kc + c], sx[si * 8 + sj]));
        }
      z[q] = acc;
    }
  }
#pragma unroll
  for (int q = 0; q < 2; ++q) {
    const int e = lane + 32 * q, r = e >> 3, c = e & 7;
    const uint32_t v = quantize(z[q], nan_flag);
    if (y0 + r < h && x0 + c < w) dst[static_cast<size_t>(r) * pitch + c] = static_cast<uint8_t>(v);
  }
  __syncwarp();
  (void)fast_out;
  return true;
}

// TM: 0 = direct global loads (unaligned views, host-mapped input), 1 = four
// TMA boxes [8 rows x 256 px] per tile (u8 elements), 2 = one TMA box
// [8 rows x 128 uint64] = the whole 8 x 1024 px strip (width % 8 == 0).
template <int TM>
__global__ void __launch_bounds__(q8::THREADS, 1)
    k_fused8_q(const __grid_constant__ CUtensorMap imap, const __grid_constant__ QArgs args,
               const uint8_t* __restrict__ in, uint8_t* __restrict__ out, int w, int h, size_t pitch,
               long long frame_stride, int nframes, int bw, int bh, int ntx, bool fast_out, int* nan_flag,
               unsigned long long* fb_count) {
  using namespace q8;
  constexpr bool TMA = TM != 0;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* base = align1024(smem_raw);
  uint8_t* bsm = base;                                // digit images
  uint8_t* asm_ = bsm + KQ_MAX_PLANS * BBYTES;        // A stages
  uint8_t* raw = asm_ + NA * ABYTES;                  // raw pixel stages
  __shared__ uint64_t raw_full[NRAW], raw_empty[NRAW], a_full[NA], a_empty[NA], acc_full[2], acc_empty[2];
  __shared__ uint32_t tmem_base_s;
  __shared__ uint64_t ops_full;  // the plans' digit images have landed
  __shared__ unsigned long long fq[FQ];
  __shared__ uint32_t fq_tail, fq_head, fq_done;
  __shared__ __align__(16) double fb_sm[256];
  // per-frame plan index and per-plan epilogue constants, staged from the
  // parameter bank (dynamically indexed constant loads miss the constant cache)
  __shared__ uint8_t pof_s[KQ_MAX_FRAMES];
  __shared__ uint32_t U_s[KQ_MAX_PLANS];
  __shared__ int shS_s[KQ_MAX_PLANS], shL_s[KQ_MAX_PLANS], den_s[KQ_MAX_PLANS], bias_s[KQ_MAX_PLANS];
  __shared__ uint32_t magic_s[KQ_MAX_PLANS];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  pdl_trigger();
  if (threadIdx.x == 0) QSTAMP(0, 28);
  for (int i = threadIdx.x; i < FQ; i += blockDim.x) fq[i] = 0ull;
  for (int i = threadIdx.x; i < nframes; i += blockDim.x) pof_s[i] = args.pof[i];
  if (threadIdx.x < KQ_MAX_PLANS) {
    U_s[threadIdx.x] = args.U[threadIdx.x];
    shS_s[threadIdx.x] = args.shS[threadIdx.x];
    shL_s[threadIdx.x] = args.shL[threadIdx.x];
    den_s[threadIdx.x] = args.den[threadIdx.x];
    bias_s[threadIdx.x] = args.bias[threadIdx.x];
    magic_s[threadIdx.x] = args.magic[threadIdx.x];
  }
  // A rows, bytes 64..127 (chunks 4-7, 128B-swizzled): the constant input
  // [1, 1, 255 x 30, 0 ...] that adds the B rows' bytes 64-95 to the
  // accumulators: the digits of the rounding offset 2^(F-1) (bytes 64-65) or a
  // rational plan's division constant (plan.cc: layout_kq8)
  for (int i = threadIdx.x; i < NA * TILE * 4; i += blockDim.x) {
    const int st = i / (TILE * 4), b = (i >> 2) % TILE, c = 4 + (i & 3);
    *reinterpret_cast<uint4*>(asm_ + st * ABYTES + b * ROWB + ((c ^ (b & 7)) << 4)) =
        c == 4   ? make_uint4(0xFFFF0101u, 0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFFu)
        : c == 5 ? make_uint4(0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFFu)
                 : make_uint4(0u, 0u, 0u, 0u);
  }
  if (warp == W_MMA) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(&tmem_base_s)),
                 "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 0) {
    for (int i = 0; i < NRAW; ++i) {
      mbar_init(&raw_full[i], 1);
      mbar_init(&raw_empty[i], 64);  // the two warps of the tile's converter set
    }
    for (int i = 0; i < NA; ++i) {
      mbar_init(&a_full[i], 64);
      mbar_init(&a_empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&acc_full[i], 1);
      mbar_init(&acc_empty[i], 32 * 4);  // the four warps of epilogue group i
    }
    mbar_init(&ops_full, 1);
    fq_tail = 0;
    fq_head = 0;
    fq_done = 0;
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    // the plans' digit images (plan-owned, written only at plan creation, so
    // safe before pdl_wait): one bulk copy each, completing on ops_full,
    // which only the MMA warp waits for; the TMA loads and conversion of the
    // first tiles proceed meanwhile
    mbar_expect_tx(&ops_full, static_cast<uint32_t>(args.nplans * BBYTES));
    for (int pi = 0; pi < args.nplans; ++pi)
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
              smem_u32(bsm + pi * BBYTES)),
          "l"(reinterpret_cast<uint64_t>(args.bimg[pi])), "r"(static_cast<uint32_t>(BBYTES)), "r"(smem_u32(&ops_full))
          : "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = tmem_base_s;
  pdl_wait();
  if (threadIdx.x == 0) QSTAMP(0, 29);

  const long long tpf = static_cast<long long>(bh) * ntx;  // tiles per frame
  const long long ntiles = tpf * nframes;                  // < 2^31 (launcher)
  // the divisors' magic numbers come precomputed (a 64-bit division per thread here cost ~1,000 cycles of the
  // prologue)
  const dctf::FastDiv fd_tpf = args.fd_tpf, fd_ntx = args.fd_ntx;
  auto tile_at = [&](long long ti, int& f, int& by, int& bx0) {
    const uint32_t u = static_cast<uint32_t>(ti);
    f = static_cast<int>(dctf::fdiv(fd_tpf, u));
    const uint32_t rem = u - static_cast<uint32_t>(f) * static_cast<uint32_t>(tpf);
    by = static_cast<int>(dctf::fdiv(fd_ntx, rem));
    bx0 = static_cast<int>(rem - static_cast<uint32_t>(by) * static_cast<uint32_t>(ntx)) * TILE;
  };

  // Consumer side of the flagged-block queue: claim entries in order (one
  // atomic per claim), recompute each claimed block in the reference's
  // operation order. Returns once every epilogue warp has finished and no
  // claimed entry remains. Run by the fallback warp from the start, and by
  // every other warp once the CTA's tiles are done.
  auto drain = [&](double* scratch) {
    uint32_t nap = 64;
    while (true) {
      uint32_t slot = 0;
      if (lane == 0) slot = atomicAdd(&fq_head, 1u);
      slot = __shfl_sync(0xFFFFFFFFu, slot, 0);
      volatile unsigned long long* qs = &fq[slot % FQ];
      unsigned long long e;
      auto mine = [&](unsigned long long v) { return v != 0ull && static_cast<uint32_t>(v >> 32) == slot; };
      while (!mine(e = *qs)) {
        if (*reinterpret_cast<volatile uint32_t*>(&fq_done) == static_cast<uint32_t>(NEPI)) {
          __threadfence_block();
          if (mine(e = *qs)) break;
          if (slot >= *reinterpret_cast<volatile uint32_t*>(&fq_tail)) return;
        }
        __nanosleep(nap);
        nap = min(nap * 2u, 256u);  // short: the kernel cannot end while this warp sleeps
      }
      nap = 64;
      __syncwarp();
      const unsigned long long code = (e & 0xFFFFFFFFull) - 1ull;
      const long long ti = static_cast<long long>(code >> 7);
      const int b = static_cast<int>(code & 127ull);
      int f, by, bx0;
      tile_at(ti, f, by, bx0);
      const int y0 = by * 8, x0 = (bx0 + b) * 8;
      const uint8_t* ib = in + f * frame_stride;
      uint8_t* ob = out + f * frame_stride + static_cast<size_t>(y0) * pitch + x0;
      bool chain = false;
      if (!(Q8_EXP & 16))
        chain = fallback_block(args.ref[pof_s[f]], ib, pitch, w, h, y0, x0, ob, fast_out, scratch, nan_flag, lane);
      __syncwarp();
      if (lane == 0) {
        *qs = 0ull;
        if (fb_count) {
          atomicAdd(fb_count, 1ull);
          if (chain) atomicAdd(fb_count + 1, 1ull);
        }
      }
      __syncwarp();
    }
  };

  if (warp == W_TMA) {
    // ---------------- TMA producer: raw strips into the ring. Like the MMA
    // issuer: the converged warp runs the loop and one elected lane issues the
    // tile's expect_tx and (up to) four box loads in one asm block (a lone
    // lane-0 loop wraps each bulk-tensor instruction in its own elect loop,
    // which held this warp's SM sub-partition ~100 cycles per load).
    if (TMA) {
      if (lane == 0) prefetch_tmap(&imap);
      __syncwarp();
      const uint64_t map = reinterpret_cast<uint64_t>(&imap);
      long long tl = 0;
      for (long long ti = blockIdx.x; ti < ntiles; ti += gridDim.x, ++tl) {
        int f, by, bx0;
        tile_at(ti, f, by, bx0);
        const int r = static_cast<int>(tl % NRAW);
        const uint32_t k = static_cast<uint32_t>(tl / NRAW);
        Q8_WAIT_OTHER(&raw_empty[r], (k & 1u) ^ 1u);
        if (lane == 0) QSTAMP(tl, 20);
        const uint32_t dst = smem_u32(raw + r * RAWB), bar = smem_u32(&raw_full[r]);
        if (TM == 2) {
          asm volatile(
              "{\n\t.reg .pred e;\n\t"
              "elect.sync _|e, 0xffffffff;\n\t"
              "@e mbarrier.arrive.expect_tx.shared::cta.b64 _, [%1], %2;\n\t"
              "@e cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
              " [%0], [%3, {%4, %5, %6}], [%1];\n\t}"
              ::"r"(dst), "r"(bar), "r"(static_cast<uint32_t>(RAWB)), "l"(map), "r"(bx0), "r"(by * 8), "r"(f)
              : "memory");
          continue;
        }
        const int nbt = min(TILE, bw - bx0);
        const int nbox = (nbt * 8 + 255) >> 8;
        const int x0 = bx0 * 8, y0 = by * 8;
        asm volatile(
            "{\n\t.reg .pred e, p1, p2, p3;\n\t"
            "elect.sync _|e, 0xffffffff;\n\t"
            "setp.gt.and.s32 p1, %3, 1, e;\n\t"
            "setp.gt.and.s32 p2, %3, 2, e;\n\t"
            "setp.gt.and.s32 p3, %3, 3, e;\n\t"
            "@e mbarrier.arrive.expect_tx.shared::cta.b64 _, [%1], %2;\n\t"
            "@e cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
            " [%0], [%4, {%5, %6, %7}], [%1];\n\t"
            "@p1 cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
            " [%8], [%4, {%9, %6, %7}], [%1];\n\t"
            "@p2 cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
            " [%10], [%4, {%11, %6, %7}], [%1];\n\t"
            "@p3 cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
            " [%12], [%4, {%13, %6, %7}], [%1];\n\t}"
            ::"r"(dst), "r"(bar), "r"(static_cast<uint32_t>(nbox * 2048)), "r"(nbox), "l"(map), "r"(x0), "r"(y0),
            "r"(f), "r"(dst + 2048), "r"(x0 + 256), "r"(dst + 4096), "r"(x0 + 512), "r"(dst + 6144), "r"(x0 + 768)
            : "memory");
      }
    }
  } else if (warp == W_MMA) {
    constexpr uint32_t idesc256 = idesc_u8s8(128, 256), idesc64 = idesc_u8s8(128, 64),
                       idesc256u = idesc_u8s8(128, 256, true);
    const uint64_t da0 = desc_sw128(smem_u32(asm_)), db0 = desc_sw128(smem_u32(bsm));
    constexpr uint64_t DA_STAGE = ABYTES >> 4, DB_PLAN = BBYTES >> 4;
    const uint32_t acc_full0 = smem_u32(&acc_full[0]), a_empty0 = smem_u32(&a_empty[0]);
    Q8_WAIT_MMA(&ops_full, 0u);
    long long tl = 0;
    for (long long ti = blockIdx.x; ti < ntiles; ti += gridDim.x, ++tl) {
      int f, by, bx0;
      tile_at(ti, f, by, bx0);
      const int pi = pof_s[f];
      const int s = static_cast<int>(tl % NA);
      const int buf = static_cast<int>(tl & 1);
      Q8_WAIT_MMA(&a_full[s], static_cast<uint32_t>((tl / NA) & 1));
      if (lane == 0) QSTAMP(tl, 19);
      Q8_WAIT_MMA(&acc_empty[buf], static_cast<uint32_t>(((tl >> 1) & 1) ^ 1));
      if (lane == 0) QSTAMP(tl, 0);
      tc_fence_after();
      const uint64_t da = da0 + DA_STAGE * s, db = db0 + DB_PLAN * pi;
      // rational plans: one accumulator column per pixel; den -1: unsigned digit bytes
      const uint32_t idesc = den_s[pi] > 0 ? idesc64 : den_s[pi] < 0 ? idesc256u : idesc256;
      const uint32_t dt = tmem_base + 256 * buf;
      asm volatile(
          "{\n\t.reg .pred e;\n\t"
          "elect.sync _|e, 0xffffffff;\n\t"
          "@e tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, 0;\n\t"
          "@e tcgen05.mma.cta_group::1.kind::i8 [%0], %4, %5, %3, 1;\n\t"
          "@e tcgen05.mma.cta_group::1.kind::i8 [%0], %6, %7, %3, 1;\n\t"
          "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%8];\n\t"
          "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%9];\n\t}"
          ::"r"(dt), "l"(da), "l"(db), "r"(idesc), "l"(da + 2), "l"(db + 2), "l"(da + 4), "l"(db + 4),
          "r"(acc_full0 + 8u * buf), "r"(a_empty0 + 8u * s)
          : "memory");
      if (lane == 0) QSTAMP(tl, 1);
    }
    __syncwarp();
  } else if (warp >= W_CONV) {
    // ---------------- converters: thread = the block pair (2 c2, 2 c2 + 1) of
    // the tile: one 16-byte shared load per pixel row covers both blocks
    // (adjacent 8-byte rows of the strip), four 16-byte A-operand stores each
    const int cset = (warp - W_CONV) >> 1, c2 = (threadIdx.x - 32 * W_CONV) & 63;
    long long tl = cset;
    for (long long ti = blockIdx.x + static_cast<long long>(cset) * gridDim.x; ti < ntiles;
         ti += CSETS * static_cast<long long>(gridDim.x), tl += CSETS) {
      int f, by, bx0;
      tile_at(ti, f, by, bx0);
      const int nbt = min(TILE, bw - bx0);
      const int y0 = by * 8;
      // row[rr] = {block 2 c2 row rr (x, y), block 2 c2 + 1 row rr (z, w)}
      uint4 row[8];
      const bool full = 2 * c2 + 1 < nbt && (bx0 + 2 * c2 + 2) * 8 <= w && y0 + 8 <= h;
      // one block of the pair through tile()'s edge replication (ragged
      // edges), from the staged strip (TMA) or from global memory
      auto ragged = [&](int bb, const uint8_t* rb, int half) {
        const int x0 = (bx0 + bb) * 8;
#pragma unroll
        for (int rr = 0; rr < 8; ++rr) {
          uint32_t lo = 0, hi = 0;
          if (bb < nbt) {
#pragma unroll
            for (int c = 0; c < 8; ++c) {
              uint32_t v;
              if (rb) {
                const int ry = min(rr, h - 1 - y0), cx = min(bb * 8 + c, w - 1 - bx0 * 8);
                v = TM == 2 ? rb[ry * 1024 + cx] : rb[(cx >> 8) * 2048 + ry * 256 + (cx & 255)];
              } else {
                v = in[f * frame_stride + static_cast<size_t>(min(y0 + rr, h - 1)) * pitch + min(x0 + c, w - 1)];
              }
              if (c < 4) lo |= v << (8 * c);
              else hi |= v << (8 * (c - 4));
            }
          }
          if (half == 0) {
            row[rr].x = lo;
            row[rr].y = hi;
          } else {
            row[rr].z = lo;
            row[rr].w = hi;
          }
        }
      };
      if (TMA) {
        const int r = static_cast<int>(tl % NRAW);
        Q8_WAIT_OTHER(&raw_full[r], static_cast<uint32_t>((tl / NRAW) & 1));
        if (c2 == 0) QSTAMP(tl, 21);
        // row rr of blocks 2 c2, 2 c2 + 1: four boxes [8 rows x 256 px] (TM 1)
        // or one strip [8 rows x 1024 px] (TM 2)
        const int b = 2 * c2;
        const uint8_t* rs = TM == 2 ? raw + r * RAWB + b * 8 : raw + r * RAWB + (b >> 5) * 2048 + (b & 31) * 8;
        constexpr int RSTRIDE = TM == 2 ? 1024 : 256;
        if (full) {
#pragma unroll
          for (int rr = 0; rr < 8; ++rr) row[rr] = *reinterpret_cast<const uint4*>(rs + rr * RSTRIDE);
        } else if (2 * c2 < nbt) {
          ragged(2 * c2, raw + r * RAWB, 0);
          ragged(2 * c2 + 1, raw + r * RAWB, 1);
        }
        mbar_arrive(&raw_empty[r]);
        if (c2 == 0) QSTAMP(tl, 23);
      } else if (2 * c2 < nbt) {  // direct loads (unaligned views, host-mapped input)
        const uint8_t* ib = in + f * frame_stride + (bx0 + 2 * c2) * 8;
        if (full && ((reinterpret_cast<uintptr_t>(ib) & 15) == 0) && ((pitch & 15) == 0)) {
#pragma unroll
          for (int rr = 0; rr < 8; ++rr)
            row[rr] = __ldg(reinterpret_cast<const uint4*>(ib + static_cast<size_t>(y0 + rr) * pitch));
        } else {
          ragged(2 * c2, nullptr, 0);
          ragged(2 * c2 + 1, nullptr, 1);
        }
      }
      const int s = static_cast<int>(tl % NA);
      Q8_WAIT_OTHER(&a_empty[s], static_cast<uint32_t>(((tl / NA) & 1) ^ 1));
      if (c2 == 0) QSTAMP(tl, 22);
#pragma unroll
      for (int hb = 0; hb < 2; ++hb) {
        const int b = 2 * c2 + hb, m = a_row(b);
        if (b < nbt && !(Q8_EXP & 4)) {
          uint8_t* arow = asm_ + s * ABYTES + m * ROWB;
#pragma unroll
          for (int q = 0; q < 4; ++q)
            *reinterpret_cast<uint4*>(arow + ((q ^ (m & 7)) << 4)) =
                hb == 0 ? make_uint4(row[2 * q].x, row[2 * q].y, row[2 * q + 1].x, row[2 * q + 1].y)
                        : make_uint4(row[2 * q].z, row[2 * q].w, row[2 * q + 1].z, row[2 * q + 1].w);
        }
      }
      if (c2 == 0) QSTAMP(tl, 24);
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      if (c2 == 0) QSTAMP(tl, 25);
      mbar_arrive(&a_full[s]);
      if (c2 == 0) QSTAMP(tl, 18);
    }
  } else if (warp < W_FB) {
    // ---------------- epilogue: thread = block = TMEM lane; group g (warps
    // W_EPI + 4g .. + 3, one per lane quarter) drains accumulator buffer g,
    // i.e. the CTA's tiles tl = g, g + 2, ...
    const int qd = warp & 3, grp = (warp - W_EPI) >> 2, b = a_row(32 * qd + lane);  // TMEM lane -> block
    const uint32_t col0 = tmem_base + (static_cast<uint32_t>(32 * qd) << 16) + 256 * grp;
    long long tl = grp;
    for (long long ti = blockIdx.x + static_cast<long long>(grp) * gridDim.x; ti < ntiles;
         ti += NGRP * static_cast<long long>(gridDim.x), tl += NGRP) {
      int f, by, bx0;
      tile_at(ti, f, by, bx0);
      const int pi = pof_s[f];
      const uint32_t U = U_s[pi];
      const int shS = shS_s[pi], shL = shL_s[pi];
      Q8_WAIT_OTHER(&acc_full[grp], static_cast<uint32_t>((tl >> 1) & 1));
      tc_fence_after();
#ifdef QDBG
      if (lane == 0) QSTAMP(tl, 2 + (warp - W_EPI));
      long long* rel = (blockIdx.x < 4 && tl < 64) ? &g_qdbg[blockIdx.x][tl][10 + (warp - W_EPI)] : nullptr;
#else
      long long* rel = nullptr;
#endif
      uint32_t words[16];
      uint32_t mn0 = 0xFFFFFFFFu, mn1 = 0xFFFFFFFFu;
      int32_t va[32], vb[32];
      // row r is processed while row r + 1 streams in from TMEM
      if (den_s[pi] > 0) epi_rational(col0, den_s[pi], magic_s[pi], bias_s[pi], words, &acc_empty[grp], rel);
      else if (shL < 0) epi_rows<8, 2>(col0, va, vb, shS, 0, mn0, mn1, words, &acc_empty[grp], rel);  // F = 32, no saturation
      else if (shL == 0) epi_rows<8, 1>(col0, va, vb, shS, 0, mn0, mn1, words, &acc_empty[grp], rel);
      else epi_rows<8, 0>(col0, va, vb, shS, shL, mn0, mn1, words, &acc_empty[grp], rel);
      QSTAMP_EPI(tl, 26);
      // A block with an uncertain pixel is left to the fallback warp, which
      // recomputes and writes the whole block.
      const int nbt = min(TILE, bw - bx0);
      const bool valid = b < nbt;
      const bool unsure = valid && min(mn0, mn1) < 2u * U;
      const int y0 = by * 8, x0 = (bx0 + b) * 8;
      uint8_t* ob = out + f * frame_stride + static_cast<size_t>(y0) * pitch + x0;
      if (valid && !unsure && (Q8_EXP & 2)) {  // no stores, the bytes kept live
        uint32_t x = 0;
#pragma unroll
        for (int k = 0; k < 16; ++k) x ^= words[k];
        if (x == 0x9e3779b9u) *ob = 1;
      } else if (valid && !unsure) {
        if (fast_out && x0 + 8 <= w && y0 + 8 <= h) {
#pragma unroll
          for (int k = 0; k < 8; ++k)
            *reinterpret_cast<uint2*>(ob + static_cast<size_t>(k) * pitch) = make_uint2(words[2 * k], words[2 * k + 1]);
        } else {
          store_ragged<8>(ob, pitch, words, h - y0, w - x0);
        }
      }
      const uint32_t flagged = __ballot_sync(0xFFFFFFFFu, unsure);
      if (flagged) enqueue_fallback(fq, &fq_tail, flagged, unsure, lane, ti, b);
      QSTAMP_EPI(tl, 27);
#ifdef QDBG
      if (lane == 0) QSTAMP(tl, 32 + (warp - W_EPI));
#endif
    }
    __threadfence_block();
    __syncwarp();
    if (lane == 0) atomicAdd(&fq_done, 1u);
  } else {
    // ---------------- fallback warp: reference-order chain on queued blocks
    drain(fb_sm);
    if (lane == 0) QSTAMP(1, 28);
  }
  if (warp != W_FB) {
    // Every tile of this CTA is done once all other warps get here (the
    // epilogue waited for the last MMA, the converters consumed every raw
    // stage): the rest of the queue is drained by all warps in parallel, each
    // with 2 KB of scratch in the now idle raw ring.
    if (threadIdx.x == 0) QSTAMP(0, 30);
    asm volatile("bar.sync 1, %0;" ::"n"(THREADS - 32) : "memory");
    if (threadIdx.x == 0) QSTAMP(1, 29);
    const int slot = warp < W_FB ? warp : warp - 1;
    drain(reinterpret_cast<double*>(raw + slot * 2048));
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (threadIdx.x == 0) QSTAMP(0, 31);
  if (warp == W_MMA)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(512));
}

// u8 image path of unbounded plans (chain_bounded false: the reference's
// intermediates can overflow FP64): every block through the reference's own
// operation order, one warp per block, so inf / NaN arise exactly where they
// arise in the reference and NaN sets the flag like quantize_sample's throw.
__global__ void __launch_bounds__(256) k_refchain8(const __grid_constant__ RefPlan rp, const uint8_t* in, uint8_t* out,
                                                    int w, int h, size_t pitch, long long frame_stride, int nframes,
                                                    int bw, int bh, int* nan_flag) {
  __shared__ __align__(16) double sm[8][256];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long long per = static_cast<long long>(bw) * bh, nb = per * nframes;
  for (long long b = static_cast<long long>(blockIdx.x) * 8 + warp; b < nb; b += static_cast<long long>(gridDim.x) * 8) {
    const long long f = b / per, r = b - f * per;
    const int by = static_cast<int>(r / bw), bx = static_cast<int>(r - static_cast<long long>(by) * bw);
    fallback_block(rp, in + f * frame_stride, pitch, w, h, by * 8, bx * 8,
                   out + f * frame_stride + static_cast<size_t>(by) * 8 * pitch + bx * 8, false, sm[warp], nan_flag,
                   lane);
  }
}

}  // namespace

namespace dctf {

dctf_status upload_refchain_only(dctf_plan* p) {
  std::vector<double> chain;
  refchain_image(*p, chain, p->ref_mode, p->ref_npairs);
  cudaError_t e = cudaMalloc(&p->d_refchain, chain.size() * sizeof(double));
  if (e == cudaSuccess)
    e = cudaMemcpy(p->d_refchain, chain.data(), chain.size() * sizeof(double), cudaMemcpyHostToDevice);
  if (e != cudaSuccess) return set_error(DCTF_CUDA_ERROR, std::string("reference chain upload: ") + cudaGetErrorString(e));
  return DCTF_OK;
}

dctf_status launch_refchain8(const dctf_plan* p, const uint8_t* in, uint8_t* out, int w, int h, size_t pitch,
                             long long frame_stride, int nframes, cudaStream_t st) {
  const int bw = (w + 7) / 8, bh = (h + 7) / 8;
  const long long nb = static_cast<long long>(bw) * bh * nframes;
  if (nb <= 0) return DCTF_OK;
  const RefPlan rp{p->d_refchain, p->d_weights, nullptr, 0.0, p->ref_mode, p->ref_npairs, p->kr, p->kc, p->padding};
  const long long grid = std::min<long long>((nb + 7) / 8, 16LL * sm_count(p->device));
  k_refchain8<<<static_cast<unsigned>(grid), 256, 0, st>>>(rp, in, out, w, h, pitch, frame_stride, nframes, bw, bh,
                                                           nan_flag(p));
  add_launches(1);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return set_error(DCTF_CUDA_ERROR, std::string("k_refchain8: ") + cudaGetErrorString(e));
  return DCTF_OK;
}

// DCTF_Q_COUNT=1: a process-wide device counter of the blocks the fallback
// warp recomputed (diagnostics; read with dctf_diag_fallback_blocks).
static unsigned long long* fallback_counter() {
  static unsigned long long* c = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    if (std::getenv("DCTF_Q_COUNT") && cudaMalloc(&c, 16) == cudaSuccess) cudaMemset(c, 0, 16);
  });
  return c;
}

dctf_status upload_kq_operator(dctf_plan* p) {
  std::vector<int8_t> img;
  KqInfo info;
  if (p->n != 8 || !layout_kq8(*p, img, info)) return DCTF_OK;  // not eligible: FP64 kernels stay
  std::vector<double> chain;
  refchain_image(*p, chain, p->ref_mode, p->ref_npairs);
  cudaError_t e = cudaMalloc(&p->d_kq, img.size());
  if (e == cudaSuccess) e = cudaMemcpy(p->d_kq, img.data(), img.size(), cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMalloc(&p->d_refchain, chain.size() * sizeof(double));
  if (e == cudaSuccess)
    e = cudaMemcpy(p->d_refchain, chain.data(), chain.size() * sizeof(double), cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMalloc(&p->d_kqt, info.kt.size() * sizeof(double));
  if (e == cudaSuccess)
    e = cudaMemcpy(p->d_kqt, info.kt.data(), info.kt.size() * sizeof(double), cudaMemcpyHostToDevice);
  if (e != cudaSuccess) return set_error(DCTF_CUDA_ERROR, std::string("kq operator upload: ") + cudaGetErrorString(e));
  p->kq = true;
  p->kq_F = info.F;
  p->kq_U = info.U;
  p->kq_ebound = info.ebound;
  p->kq_flag_rate = info.flag_rate;
  p->kq_margin = info.margin;
  p->kq_den = info.den;
  p->kq_magic = info.magic;
  p->kq_bias = info.bias;
  p->kq_nosat = info.nosat;
  p->kq_unsigned = info.unsigned_digits;
  if (std::getenv("DCTF_Q_DEBUG") && info.den > 0)
    std::fprintf(stderr, "[k_fused8_q plan] rational operator K = K'/%d (bias %d): deviation %.3e (reference FP64 bound "
                         "%.3e) against a boundary distance of %.3e\n", info.den, info.bias, info.ebound, info.eref,
                 0.5 / info.den);
  else if (std::getenv("DCTF_Q_DEBUG"))
    std::fprintf(stderr, "[k_fused8_q plan] F=%d U=%u window=%.3e (reference FP64 bound %.3e) second-stage margin=%.3e "
                         "expected flagged blocks %.2e\n", info.F, info.U, info.ebound, info.eref, info.margin,
                 info.flag_rate);
  return DCTF_OK;
}

dctf_status launch_fused8_q(const dctf_plan* const* plans, int nplans, const int* plan_of_frame, const uint8_t* in,
                            uint8_t* out, int w, int h, size_t pitch, long long frame_stride, int nframes,
                            cudaStream_t st, bool host_mapped, int* d_nan_or_null) {
  unsigned long long* fb_count = fallback_counter();
  if (nplans < 1 || nplans > KQ_MAX_PLANS || nframes > KQ_MAX_FRAMES)
    return set_error(DCTF_INVALID_ARGUMENT, "k_fused8_q: too many plans / frames for one launch");
  const int bw = (w + 7) / 8, bh = (h + 7) / 8, ntx = (bw + q8::TILE - 1) / q8::TILE;
  const long long ntiles = static_cast<long long>(bh) * ntx * nframes;
  if (ntiles <= 0) return DCTF_OK;
  if (ntiles >= (1LL << 31) / 128 || static_cast<long long>(bw) * bh * nframes >= (1LL << 31))
    return set_error(DCTF_INVALID_ARGUMENT, "image batch too large (>= 2^31 blocks)");
  QArgs args{};
  args.nplans = nplans;
  for (int i = 0; i < nplans; ++i) {
    const dctf_plan* p = plans[i];
    if (!p->kq) return set_error(DCTF_INVALID_ARGUMENT, "k_fused8_q: plan has no integer operator");
    args.bimg[i] = static_cast<const int8_t*>(p->d_kq);
    args.U[i] = p->kq_U;
    args.shS[i] = p->kq_F - 16;
    args.shL[i] = p->kq_nosat ? -1 : 32 - p->kq_F;  // -1: F = 32 and outputs provably in [0, 255]
    args.den[i] = p->kq_den > 0 ? p->kq_den : p->kq_unsigned ? -1 : 0;
    args.bias[i] = p->kq_bias;
    args.magic[i] = p->kq_magic;
    args.ref[i] = RefPlan{p->d_refchain, p->d_weights, p->d_kqt, p->kq_margin, p->ref_mode, p->ref_npairs, p->kr,
                          p->kc, p->padding};
  }
  for (int f = 0; f < nframes; ++f) args.pof[f] = static_cast<uint8_t>(plan_of_frame ? plan_of_frame[f] : 0);
  args.fd_tpf = dctf::make_fastdiv(static_cast<uint32_t>(static_cast<long long>(bh) * ntx));
  args.fd_ntx = dctf::make_fastdiv(static_cast<uint32_t>(ntx));
  const bool tma = !host_mapped && (pitch & 15) == 0 && (reinterpret_cast<uintptr_t>(in) & 15) == 0 &&
                   (nframes == 1 || (frame_stride & 15) == 0) && pitch < (1ull << 40) && !std::getenv("DCTF_Q_NO_TMA");
  const bool fast_out = (pitch & 7) == 0 && (reinterpret_cast<uintptr_t>(out) & 7) == 0 &&
                        (nframes == 1 || (frame_stride & 7) == 0);
  // one 8 KB box per tile when the width allows 8-byte elements (each TMA
  // issue holds the issuing warp's sub-partition; four per tile set the pace)
  const int tm = !tma ? 0 : ((w & 7) == 0 && !std::getenv("DCTF_Q_TMA4")) ? 2 : 1;
  CUtensorMap imap{};
  if (tma) {
    const dctf_status s = tm == 2 ? make_imap(&imap, in, w, h, nframes, pitch, frame_stride, 128, 8)
                                  : make_imap(&imap, in, w, h, nframes, pitch, frame_stride, 256);
    if (s != DCTF_OK) return s;
  }
  const void* fn = tm == 2   ? reinterpret_cast<const void*>(k_fused8_q<2>)
                   : tm == 1 ? reinterpret_cast<const void*>(k_fused8_q<1>)
                             : reinterpret_cast<const void*>(k_fused8_q<0>);
  {
    const dctf_status sa = ensure_dyn_smem(fn, q8::SMEM, tm == 2 ? "k_fused8_q<tma wide>" : tm == 1 ? "k_fused8_q<tma>" : "k_fused8_q<direct>");
    if (sa != DCTF_OK) return sa;
  }
  const unsigned grid = static_cast<unsigned>(std::min<long long>(sm_count(plans[0]->device), ntiles));
  const cudaError_t e =
      tm == 2   ? launch_pdl(k_fused8_q<2>, grid, q8::THREADS, q8::SMEM, st, imap, args, in, out, w, h, pitch,
                             frame_stride, nframes, bw, bh, ntx, fast_out, d_nan_or_null, fb_count)
      : tm == 1 ? launch_pdl(k_fused8_q<1>, grid, q8::THREADS, q8::SMEM, st, imap, args, in, out, w, h, pitch,
                             frame_stride, nframes, bw, bh, ntx, fast_out, d_nan_or_null, fb_count)
                : launch_pdl(k_fused8_q<0>, grid, q8::THREADS, q8::SMEM, st, imap, args, in, out, w, h, pitch,
                             frame_stride, nframes, bw, bh, ntx, fast_out, d_nan_or_null, fb_count);
  add_launches(1);
  if (e != cudaSuccess) return set_error(DCTF_CUDA_ERROR, std::string("k_fused8_q: ") + cudaGetErrorString(e));
  return DCTF_OK;
}

}  // namespace dctf

extern "C" dctf_status dctf_diag_fallback_counts(unsigned long long* flagged, unsigned long long* chain) {
  if (!flagged) return set_error(DCTF_INVALID_ARGUMENT, "NULL argument");
  *flagged = 0;
  if (chain) *chain = 0;
  unsigned long long* c = dctf::fallback_counter();
  if (!c) return set_error(DCTF_UNSUPPORTED, "set DCTF_Q_COUNT=1 before the first filter call");
  unsigned long long v[2] = {0, 0};
  if (cudaDeviceSynchronize() != cudaSuccess || cudaMemcpy(v, c, 16, cudaMemcpyDeviceToHost) != cudaSuccess ||
      cudaMemset(c, 0, 16) != cudaSuccess)
    return set_error(DCTF_CUDA_ERROR, "fallback counter read failed");
  *flagged = v[0];
  if (chain) *chain = v[1];
  return DCTF_OK;
}

extern "C" dctf_status dctf_diag_fallback_blocks(unsigned long long* n) { return dctf_diag_fallback_counts(n, nullptr); }

#ifdef QDBG
extern "C" int dctf_qdbg_read(long long* out) {
  return cudaMemcpyFromSymbol(out, g_qdbg, sizeof(g_qdbg)) == cudaSuccess ? 0 : 1;
}
extern "C" int dctf_qdbg_clear() {
  static long long zero[4 * 64 * 48] = {};
  return cudaMemcpyToSymbol(g_qdbg, zero, sizeof(zero)) == cudaSuccess ? 0 : 1;
}
#endif

// ---------------------------------------------------------------------------
// In-run INT8 tensor-core peak (the roofline denominator of k_fused8_q's
// tensor side; MEASURED_PEAKS.json has bf16 only): one CTA per SM, one thread
// issuing back-to-back tcgen05.mma kind::i8 M128 N256 K32 from shared memory
// into TMEM, the shape and operand path k_fused8_q uses.
namespace {
__global__ void __launch_bounds__(128, 1) k_peak_i8(int iters, int* sink) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* base = align1024(smem_raw);
  __shared__ uint64_t done;
  __shared__ uint32_t tb;
  for (int i = threadIdx.x; i < (q8::ABYTES + q8::BBYTES) / 16; i += blockDim.x)
    reinterpret_cast<uint4*>(base)[i] = make_uint4(0x01010101u, 0, 0x01010101u, 0);
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tb)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 0) {
    mbar_init(&done, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (threadIdx.x == 0) {
    constexpr uint32_t idesc = idesc_u8s8(128, 256);
    const uint32_t sa = smem_u32(base), sb = smem_u32(base + q8::ABYTES);
    for (int it = 0; it < iters; ++it)
#pragma unroll
      for (int ks = 0; ks < 4; ++ks)
        mma_u8s8(tb + 256 * (it & 1), desc_sw128(sa + 32 * (ks & 1)), desc_sw128(sb + 32 * (ks & 1)), idesc,
                 it > 1 || ks > 0);
    mma_commit(&done);
    mbar_wait(&done, 0);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (threadIdx.x < 32) {
    int32_t v[32];
    tmem_ld32(tb, v);
    tmem_wait_ld();
    if (v[0] == 0x7fffffff) sink[0] = v[1];
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tb), "r"(512));
  }
}
}  // namespace

extern "C" dctf_status dctf_measure_int8_peak(int device, double* tops) {
  if (!tops) return set_error(DCTF_INVALID_ARGUMENT, "NULL argument");
  int prev = 0;
  cudaGetDevice(&prev);
  cudaSetDevice(device);
  const int smem = 1024 + q8::ABYTES + q8::BBYTES;
  dctf_status s = dctf::ensure_dyn_smem(reinterpret_cast<const void*>(k_peak_i8), smem, "k_peak_i8");
  int* sink = nullptr;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  float best = 1e30f;
  const int iters = 4096, ctas = dctf::sm_count(device);
  if (s == DCTF_OK && (cudaMalloc(&sink, 4) != cudaSuccess || cudaEventCreate(&e0) != cudaSuccess ||
                       cudaEventCreate(&e1) != cudaSuccess))
    s = set_error(DCTF_CUDA_ERROR, "int8 peak probe setup");
  for (int rep = 0; rep < 4 && s == DCTF_OK; ++rep) {
    cudaEventRecord(e0);
    k_peak_i8<<<ctas, 128, smem>>>(iters, sink);
    cudaEventRecord(e1);
    if (cudaEventSynchronize(e1) != cudaSuccess) {
      s = set_error(DCTF_CUDA_ERROR, "int8 peak probe");
      break;
    }
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    if (rep > 0) best = std::min(best, ms);
  }
  if (s == DCTF_OK) *tops = 2.0 * 128 * 256 * 32 * 4.0 * iters * ctas / (best * 1e-3) / 1e12;
  if (e0) cudaEventDestroy(e0);
  if (e1) cudaEventDestroy(e1);
  cudaFree(sink);
  cudaSetDevice(prev);
  return s;
}
