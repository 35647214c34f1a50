// TEST INFRASTRUCTURE ONLY — never linked into or called by the product path.
//
// C-ABI harness around the UNMODIFIED reference library (header-only C++20,
// /root/reference/proj/include/dctfilter). oracle/Makefile compiles this file
// with -I pointing at the reference headers where they lie (nothing is copied)
// and writes oracle/_ref/libdctf_ref.so. It exists so that
//   * tests can pin our C restatement (dctf_oracle.c) and the CUDA path against
//     the reference's own arithmetic on identical inputs, and
//   * bench.py can time the reference CPU path (`--impl reference`, and the
//     `cpu_baseline` leg) on the GPU box's host cores.
//
// Every entry point calls the reference's own functions:
//   FilterPlan            filter.hpp:52-87   (plan compile: spatial set ->
//                                             merge_symmetric -> to_dct_domain)
//   forward_2d/inverse_2d dct.hpp:59-68
//   FilterPlan::filter_coeffs / filter_block   filter.hpp:65-73
//   tile / assemble / filter_image             image.hpp:164-225
//   convolve / quantize_sample                 spatial.hpp:41-75
// Multi-threaded variants split the per-tile loop of filter_image
// (image.hpp:216-218) into contiguous tile ranges over std::thread, sharing one
// immutable plan, as the reference's thread-safety contract allows
// (filter.hpp:47-51, README.md:115-117). tile() and assemble() stay serial,
// exactly as in the reference.

#include <algorithm>
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>
#include <thread>
#include <vector>

#include "dctfilter/dctfilter.hpp"

using namespace dctfilter;

namespace {

thread_local std::string g_err;

int fail(const std::exception& e) {
  g_err = e.what();
  return 1;
}

PaddingMode pad_of(int p) { return p == 0 ? PaddingMode::kZero : PaddingMode::kReplicate; }

Mask make_mask(const double* w, int k) {
  return Mask(k, std::vector<double>(w, w + size_t(k) * k));
}

template <class F>
void parallel_for(size_t count, int nthreads, F&& body) {
  if (nthreads <= 1 || count < 2) {
    body(size_t(0), count);
    return;
  }
  const size_t nt = std::min<size_t>(size_t(nthreads), count);
  std::vector<std::thread> pool;
  pool.reserve(nt);
  for (size_t t = 0; t < nt; ++t) {
    const size_t lo = count * t / nt, hi = count * (t + 1) / nt;
    pool.emplace_back([&body, lo, hi] { body(lo, hi); });
  }
  for (auto& th : pool) th.join();
}

GrayImage to_image(const uint8_t* px, int w, int h) {
  GrayImage img{w, h, std::vector<uint8_t>(px, px + size_t(w) * h)};
  return img;
}

}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

// C (n*n, row-major) from DctBasis (dct.hpp:40-52).
int ref_dct_basis(int n, double* c_out) {
  try {
    const DctBasis b(n);
    std::memcpy(c_out, b.c().data().data(), sizeof(double) * size_t(n) * n);
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// Compiles a FilterPlan and exports its DCT-domain sandwich pairs:
// lefts/rights are npairs * n*n each (row-major), in the plan's pair order.
// Pass nullptr buffers to query only npairs/merged.
int ref_plan_pairs(const double* w, int k, int n, int padding, int* npairs, int* merged,
                   double* lefts, double* rights) {
  try {
    const FilterPlan plan(make_mask(w, k), n, pad_of(padding));
    const OperatorSet& set = plan.dct_set();
    *npairs = int(set.pairs.size());
    *merged = set.symmetric_merged ? 1 : 0;
    const size_t nn = size_t(n) * n;
    for (size_t p = 0; p < set.pairs.size(); ++p) {
      if (lefts) std::memcpy(lefts + p * nn, set.pairs[p].left.data().data(), nn * sizeof(double));
      if (rights) std::memcpy(rights + p * nn, set.pairs[p].right.data().data(), nn * sizeof(double));
    }
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// Dense N^2 x N^2 matrix of the plan's action on coefficient blocks, obtained
// by applying FilterPlan::filter_coeffs to every standard basis block
// (column (a*n+b) of H = vec(filter_coeffs(E_ab))).
int ref_plan_operator(const double* w, int k, int n, int padding, double* h_out) {
  try {
    const FilterPlan plan(make_mask(w, k), n, pad_of(padding));
    const size_t nn = size_t(n) * n;
    for (size_t col = 0; col < nn; ++col) {
      BlockMatrix e(n);
      e.data()[col] = 1.0;
      const BlockMatrix y = plan.filter_coeffs(e);
      for (size_t row = 0; row < nn; ++row) h_out[row * nn + col] = y.data()[row];
    }
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// forward_2d / inverse_2d over nb FP64 blocks (block-major, n*n each).
int ref_forward_blocks(int n, const double* in, double* out, size_t nb, int nthreads) {
  try {
    const DctBasis basis(n);
    const size_t nn = size_t(n) * n;
    parallel_for(nb, nthreads, [&](size_t lo, size_t hi) {
      for (size_t b = lo; b < hi; ++b) {
        const BlockMatrix x(n, std::vector<double>(in + b * nn, in + (b + 1) * nn));
        const BlockMatrix y = forward_2d(basis, x);
        std::memcpy(out + b * nn, y.data().data(), nn * sizeof(double));
      }
    });
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

int ref_inverse_blocks(int n, const double* in, double* out, size_t nb, int nthreads) {
  try {
    const DctBasis basis(n);
    const size_t nn = size_t(n) * n;
    parallel_for(nb, nthreads, [&](size_t lo, size_t hi) {
      for (size_t b = lo; b < hi; ++b) {
        const BlockMatrix x(n, std::vector<double>(in + b * nn, in + (b + 1) * nn));
        const BlockMatrix y = inverse_2d(basis, x);
        std::memcpy(out + b * nn, y.data().data(), nn * sizeof(double));
      }
    });
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// FilterPlan::filter_coeffs over nb coefficient blocks (the cmd_bench loop,
// dctfilter_main.cc:420-425, without the timing).
int ref_filter_coeffs(const double* w, int k, int n, int padding, const double* in, double* out,
                      size_t nb, int nthreads) {
  try {
    const FilterPlan plan(make_mask(w, k), n, pad_of(padding));
    const size_t nn = size_t(n) * n;
    parallel_for(nb, nthreads, [&](size_t lo, size_t hi) {
      for (size_t b = lo; b < hi; ++b) {
        const BlockMatrix x(n, std::vector<double>(in + b * nn, in + (b + 1) * nn));
        const BlockMatrix y = plan.filter_coeffs(x);
        std::memcpy(out + b * nn, y.data().data(), nn * sizeof(double));
      }
    });
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// The whole-image DCT path. nthreads <= 1 and no side outputs: the shipped
// filter_image(img, mask, padding, Domain::kDct, n) itself (image.hpp:210).
// Otherwise: tile -> per-tile forward_2d / filter_coeffs / inverse_2d (the
// filter_block sequence, filter.hpp:71-73) split over threads -> assemble.
// Optional side outputs (block-major, tile order): coefficients in, filtered
// coefficients, pre-quantization samples.
int ref_filter_image(const uint8_t* px, int w, int h, const double* mw, int k, int padding, int n,
                     uint8_t* out, int nthreads, double* coef_in, double* coef_out,
                     double* prequant) {
  try {
    const GrayImage img = to_image(px, w, h);
    const Mask mask = make_mask(mw, k);
    const PaddingMode pad = pad_of(padding);
    GrayImage res;
    if (nthreads <= 1 && !coef_in && !coef_out && !prequant) {
      res = filter_image(img, mask, pad, Domain::kDct, n);
    } else {
      if (mask.k() > n) throw std::invalid_argument("filter_image: mask larger than block");
      std::vector<BlockTile> tiles = tile(img, n);
      const FilterPlan plan(mask, n, pad);
      const size_t nn = size_t(n) * n;
      parallel_for(tiles.size(), nthreads, [&](size_t lo, size_t hi) {
        for (size_t t = lo; t < hi; ++t) {
          const BlockMatrix x = forward_2d(plan.basis(), tiles[t].block);
          const BlockMatrix y = plan.filter_coeffs(x);
          BlockMatrix z = inverse_2d(plan.basis(), y);
          if (coef_in) std::memcpy(coef_in + t * nn, x.data().data(), nn * sizeof(double));
          if (coef_out) std::memcpy(coef_out + t * nn, y.data().data(), nn * sizeof(double));
          if (prequant) std::memcpy(prequant + t * nn, z.data().data(), nn * sizeof(double));
          tiles[t].block = std::move(z);
        }
      });
      res = assemble(tiles, w, h);
    }
    std::memcpy(out, res.samples.data(), res.samples.size());
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// The spatial path of filter_image (Domain::kSpatial, image.hpp:219-222).
int ref_filter_image_spatial(const uint8_t* px, int w, int h, const double* mw, int k,
                             int padding, int n, uint8_t* out) {
  try {
    const GrayImage res =
        filter_image(to_image(px, w, h), make_mask(mw, k), pad_of(padding), Domain::kSpatial, n);
    std::memcpy(out, res.samples.data(), res.samples.size());
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// convolve (spatial.hpp:41-68) over nb FP64 blocks.
int ref_convolve_blocks(const double* mw, int k, int padding, int n, const double* in,
                        double* out, size_t nb) {
  try {
    const Mask mask = make_mask(mw, k);
    const size_t nn = size_t(n) * n;
    for (size_t b = 0; b < nb; ++b) {
      const BlockMatrix x(n, std::vector<double>(in + b * nn, in + (b + 1) * nn));
      const BlockMatrix y = convolve(x, mask, pad_of(padding));
      std::memcpy(out + b * nn, y.data().data(), nn * sizeof(double));
    }
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// quantize_sample (spatial.hpp:71-75) over a buffer; returns 1 on NaN.
int ref_quantize(const double* in, uint8_t* out, size_t count) {
  try {
    for (size_t i = 0; i < count; ++i) out[i] = quantize_sample(in[i]);
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// Mask presets and helpers (mask.hpp:49-108).
int ref_mask_preset(const char* name, double sigma, double* w_out, int* k_out) {
  try {
    Mask m = Mask::identity();
    const std::string s(name);
    if (s == "identity") m = Mask::identity();
    else if (s == "average3") m = Mask::average3();
    else if (s == "gaussian3") m = Mask::gaussian3(sigma);
    else if (s == "magic3") m = Mask::magic3();
    else throw std::invalid_argument("unknown preset");
    *k_out = m.k();
    std::memcpy(w_out, m.weights().data(), m.weights().size() * sizeof(double));
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

uint64_t ref_mask_fingerprint(const double* w, int k) { return make_mask(w, k).fingerprint(); }

int ref_row_symmetric(const double* w, int k) { return row_symmetric(make_mask(w, k)) ? 1 : 0; }

// Operator dump text (operator_io.hpp:105-137) of the spatial and DCT sets a
// FilterPlan compiles; returns the byte count written (or needed) in *len.
int ref_format_plan_sets(const double* w, int k, int n, int padding, char* buf, size_t* len) {
  try {
    const Mask mask = make_mask(w, k);
    OperatorSet spatial = build_spatial_operator_set(mask, n, pad_of(padding));
    if (row_symmetric(mask)) spatial = merge_symmetric(spatial);
    const FilterPlan plan(mask, n, pad_of(padding));
    const std::string text = format_operator_sets({spatial, plan.dct_set()});
    if (buf && *len >= text.size()) std::memcpy(buf, text.data(), text.size());
    *len = text.size();
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

}  // extern "C"
