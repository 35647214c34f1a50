// C++ drop-in layer (include/dctfilter_b200.hpp) exercised the way the
// reference's own GTest suites exercise dctfilter (filter_test.cc,
// image_test.cc, dct_test.cc), on the GPU. Built by `make cpp-test`, run by
// tests/test_gpu_cpp.py. Prints one line per check, exits non-zero on failure.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <random>

#include "dctfilter_b200.hpp"

using namespace dctfilter_b200;

static int failures = 0;
#define CHECK(cond, what)                                         \
  do {                                                            \
    const bool ok_ = (cond);                                      \
    std::printf("[%s] %s\n", ok_ ? "PASS" : "FAIL", what);        \
    if (!ok_) ++failures;                                         \
  } while (0)

static BlockMatrix random_u8_block(std::mt19937_64& rng, int n) {
  std::uniform_int_distribution<int> d(0, 255);
  BlockMatrix m(n);
  for (double& v : m.data()) v = double(d(rng));
  return m;
}

int main() {
  std::mt19937_64 rng(3);
  // dct_test.cc: orthonormal basis, constant block -> DC = 8
  {
    const DctBasis basis(8);
    double orth = 0;
    for (int i = 0; i < 8; ++i)
      for (int j = 0; j < 8; ++j) {
        double s = 0;
        for (int k = 0; k < 8; ++k) s += basis.c()(i, k) * basis.c()(j, k);
        orth = std::max(orth, std::abs(s - (i == j)));
      }
    CHECK(orth < 1e-12, "DctBasis(8) orthonormal");
    BlockMatrix ones(8);
    for (double& v : ones.data()) v = 1.0;
    const BlockMatrix x = forward_2d(basis, ones);
    CHECK(std::abs(x(0, 0) - 8.0) < 1e-12, "constant block -> DC 8");
    CHECK(max_abs_diff(inverse_2d(basis, x), ones) < 1e-12, "round trip");
  }
  // filter_test.cc: identity plan keeps coefficients; constant block scaling
  {
    const FilterPlan plan(Mask::identity(), 8, PaddingMode::kReplicate);
    std::uniform_real_distribution<double> u(-100, 100);
    BlockMatrix c(8);
    for (double& v : c.data()) v = u(rng);
    CHECK(max_abs_diff(plan.filter_coeffs(c), c) < 1e-12, "identity plan keeps coefficients");
    const BlockMatrix b = random_u8_block(rng, 8);
    CHECK(max_abs_diff(plan.filter_block(b), b) < 1e-10, "identity plan keeps blocks");
  }
  {
    const FilterPlan g(Mask::gaussian3(), 8, PaddingMode::kZero);
    const FilterPlan m(Mask::magic3(), 8, PaddingMode::kZero);
    CHECK(g.symmetric_merged() && g.npairs() == 2, "gaussian3 compiles merged to 2 pairs");
    CHECK(!m.symmetric_merged() && m.npairs() == 3, "magic3 compiles to 3 pairs");
  }
  {
    std::uniform_real_distribution<double> u(-1, 1);
    std::vector<double> w(9);
    double sum = 0;
    for (double& v : w) sum += (v = u(rng));
    const FilterPlan plan(Mask(3, w), 8, PaddingMode::kReplicate);
    BlockMatrix blk(8);
    for (double& v : blk.data()) v = 100.0;
    const BlockMatrix f = plan.filter_coeffs(forward_2d(plan.basis(), blk));
    bool ac = true;
    for (int i = 0; i < 64; ++i) ac = ac && (i == 0 || std::abs(f.data()[i]) < 1e-9);
    CHECK(std::abs(f(0, 0) - 8.0 * sum * 100.0) < 1e-9 && ac, "constant block scales DC by weight sum");
  }
  // batched filter_block over many blocks == per-block
  {
    const FilterPlan plan(Mask::magic3(), 16, PaddingMode::kReplicate);
    std::vector<BlockMatrix> blocks;
    for (int i = 0; i < 300; ++i) blocks.push_back(random_u8_block(rng, 16));
    const auto out = plan.filter_block(blocks);
    CHECK(max_abs_diff(out[17], plan.filter_block(blocks[17])) == 0.0, "batched == single (n=16)");
  }
  // errors
  {
    bool t1 = false, t2 = false, t3 = false;
    try { Mask(2, {1, 2, 3, 4}); } catch (const std::invalid_argument&) { t1 = true; }
    try { FilterPlan(Mask(9, std::vector<double>(81, 1.0)), 8, PaddingMode::kZero); } catch (const std::invalid_argument&) { t2 = true; }
    const FilterPlan plan(Mask::average3(), 8, PaddingMode::kZero);
    try { plan.filter_coeffs(BlockMatrix(4)); } catch (const std::invalid_argument&) { t3 = true; }
    CHECK(t1 && t2 && t3, "invalid_argument on bad mask / oversized mask / block side mismatch");
  }
  // image_test.cc: identity mask, constant image under averaging
  {
    GrayImage img{24, 17, std::vector<std::uint8_t>(24 * 17)};
    for (auto& s : img.samples) s = std::uint8_t(rng() & 255);
    CHECK(filter_image(img, Mask::identity(), PaddingMode::kReplicate).samples == img.samples,
          "identity mask reproduces the image");
    GrayImage c{20, 12, std::vector<std::uint8_t>(240, 77)};
    const GrayImage o = filter_image(c, Mask::average3(), PaddingMode::kReplicate, Domain::kDct, 16);
    bool all = true;
    for (auto s : o.samples) all = all && s == 77;
    CHECK(all, "constant image stays constant under averaging (n=16)");
  }
  // precision modes through the drop-in: structured / dense / exact-INT8 image
  // kernels give identical u8; split-precision coefficients within their bounds
  {
    GrayImage img{1000, 600, std::vector<std::uint8_t>(1000 * 600)};
    for (auto& s : img.samples) s = std::uint8_t(rng() & 255);
    const Mask g = Mask::gaussian3();
    const FilterPlan sym(g, 8, PaddingMode::kReplicate, Precision::kFp64Dmma);
    const FilterPlan dense(g, 8, PaddingMode::kReplicate, Precision::kFp64Dense);
    const FilterPlan i8(g, 8, PaddingMode::kReplicate, Precision::kInt8Exact);
    const FilterPlan q(g, 8, PaddingMode::kReplicate);
    CHECK(sym.image_kernel() == "k_fused8_sep" && dense.image_kernel() == "k_fused8" &&
              i8.image_kernel() == "k_fused8_i8" && q.image_kernel() == "k_fused8_q",
          "image kernel selection by mask structure / precision");
    const GrayImage a = filter_image(sym, img), b = filter_image(dense, img), c = filter_image(i8, img);
    CHECK(a.samples == b.samples && a.samples == c.samples, "parity-class, dense and INT8-exact u8 identical");
    std::vector<BlockMatrix> blocks;
    std::uniform_real_distribution<double> u(-300, 300);
    for (int i = 0; i < 500; ++i) {
      BlockMatrix m(16);
      for (double& v : m.data()) v = u(rng);
      blocks.push_back(m);
    }
    const FilterPlan f64(g, 16, PaddingMode::kZero);
    const FilterPlan t32(g, 16, PaddingMode::kZero, Precision::kTf32x3);
    const FilterPlan b16(g, 16, PaddingMode::kZero, Precision::kBf16x3);
    const auto ref = f64.filter_coeffs(blocks), yt = t32.filter_coeffs(blocks), yb = b16.filter_coeffs(blocks);
    double et = 0, eb = 0, mx = 0;
    for (size_t i = 0; i < ref.size(); ++i) {
      et = std::max(et, max_abs_diff(yt[i], ref[i]));
      eb = std::max(eb, max_abs_diff(yb[i], ref[i]));
      for (double v : ref[i].data()) mx = std::max(mx, std::abs(v));
    }
    CHECK(f64.coef_kernel() == "k_coef16_sep" && t32.coef_kernel() == "k_coef_tf32x3" &&
              b16.coef_kernel() == "k_coef_bf16x3",
          "coefficient kernel selection");
    CHECK(et <= 5e-6 * mx && eb <= 1e-4 * mx, "3xTF32 / 3xBF16 coefficients within their stated bounds");
  }
  // tile -> per-block filter in shuffled order -> assemble equals the fused
  // whole-image path (image_test.cc BlockOrderIndependent pattern, ragged size)
  {
    GrayImage img{37, 29, std::vector<std::uint8_t>(37 * 29)};
    for (auto& s : img.samples) s = std::uint8_t(rng() & 255);
    const FilterPlan plan(Mask::gaussian3(), 8, PaddingMode::kReplicate);
    std::vector<BlockTile> tiles = tile(img, 8);
    std::shuffle(tiles.begin(), tiles.end(), rng);
    std::vector<BlockMatrix> blocks;
    for (const auto& t : tiles) blocks.push_back(t.block);
    const std::vector<BlockMatrix> filtered = plan.filter_block(blocks);
    for (size_t i = 0; i < tiles.size(); ++i) tiles[i].block = filtered[i];
    const GrayImage a = assemble(tiles, img.width, img.height);
    const GrayImage b = filter_image(img, Mask::gaussian3(), PaddingMode::kReplicate, Domain::kDct, 8);
    CHECK(tiles.size() == 5 * 4 && a.samples == b.samples, "tile / shuffled filter_block / assemble == filter_image");
  }
  // operator construction (operators.hpp) and apply (filter.hpp) through the drop-in
  {
    const Mask g = Mask::gaussian3();
    const FilterPlan plan(g, 8, PaddingMode::kReplicate);
    const OperatorSet spatial = build_spatial_operator_set(g, 8, PaddingMode::kReplicate);
    const OperatorSet merged = merge_symmetric(spatial);
    const OperatorSet dct = to_dct_domain(merged, plan.basis());
    const OperatorSet& own = plan.dct_set();
    bool same = dct.pairs.size() == own.pairs.size() && own.pairs.size() == 2 && dct.symmetric_merged &&
                own.symmetric_merged && dct.domain == Domain::kDct && spatial.pairs.size() == 3;
    for (size_t q = 0; same && q < dct.pairs.size(); ++q)
      same = dct.pairs[q].left.data() == own.pairs[q].left.data() &&
             dct.pairs[q].right.data() == own.pairs[q].right.data();
    CHECK(same, "build_spatial_operator_set -> merge_symmetric -> to_dct_domain == FilterPlan::dct_set (bitwise)");
    std::vector<BlockMatrix> xs;
    std::uniform_real_distribution<double> u(-300, 300);
    for (int i = 0; i < 70; ++i) {
      BlockMatrix m(8);
      for (double& v : m.data()) v = u(rng);
      xs.push_back(m);
    }
    const auto ref = plan.filter_coeffs(xs), a = apply_batch(dct, xs), b = apply_batch(own, xs);
    double ea = 0, eb = 0, ep = 0, mx = 0;
    for (size_t i = 0; i < xs.size(); ++i) {
      ea = std::max(ea, max_abs_diff(a[i], ref[i]));
      eb = std::max(eb, max_abs_diff(b[i], ref[i]));
      ep = std::max(ep, max_abs_diff(i % 10 ? apply(dct, xs[i]) : apply_pairs(dct.pairs, xs[i]), ref[i]));
      for (double v : ref[i].data()) mx = std::max(mx, std::abs(v));
    }
    CHECK(eb == 0.0 && ea <= 1e-12 * mx && ep <= 1e-12 * mx, "apply(set) / apply_pairs on the device == filter_coeffs");
    // a spatial set filters spatial blocks: apply(spatial, x) == convolve(x)
    const auto cs = apply_batch(spatial, xs), cv = plan.convolve(xs);
    double es = 0, ms = 0;
    for (size_t i = 0; i < xs.size(); ++i) {
      es = std::max(es, max_abs_diff(cs[i], cv[i]));
      for (double v : cv[i].data()) ms = std::max(ms, std::abs(v));
    }
    CHECK(es <= 1e-12 * ms, "apply(spatial set) == convolve");
    bool threw = false;
    try {
      merge_symmetric(merged);
    } catch (const std::invalid_argument&) {
      threw = true;
    }
    CHECK(threw, "merge_symmetric of a merged set throws invalid_argument");
  }
  CHECK(quantize_sample(127.5) == 128 && quantize_sample(0.5) == 1 && quantize_sample(-3) == 0, "quantize KATs");
  // multi-device path (dctf_multi): two replicas on device 0 — the 2-way
  // sharding code path (block-row bands, frame ranges, one host thread per
  // replica) — must be byte-identical to the single-device entries
  {
    GrayImage img{1000, 737, std::vector<std::uint8_t>(1000 * 737)};
    std::uniform_int_distribution<int> d(0, 255);
    for (auto& v : img.samples) v = std::uint8_t(d(rng));
    std::vector<double> g5(25), r5(25);
    double gs = 0, rs = 0;
    std::uniform_real_distribution<double> u(-1, 1);
    for (int i = 0; i < 25; ++i) {
      const int y = i / 5 - 2, x = i % 5 - 2;
      g5[i] = std::exp(-(x * x + y * y) / 2.0);
      gs += g5[i];
      r5[i] = u(rng);
      rs += r5[i];
    }
    for (int i = 0; i < 25; ++i) {
      g5[i] /= gs;
      r5[i] /= rs;
    }
    const Mask mg(5, g5), mr(5, r5);
    for (const Mask* m : {&mg, &mr}) {
      const FilterPlan one(*m, 8, PaddingMode::kReplicate);
      const MultiFilterPlan two(*m, 8, PaddingMode::kReplicate, {0, 0});
      CHECK(two.replicas() == 2, "MultiFilterPlan on {0, 0} has two replicas");
      CHECK(filter_image(two, img).samples == filter_image(one, img).samples,
            "2-replica block-row bands == single device (ragged 1000x737)");
    }
    std::vector<GrayImage> frames(7, GrayImage{384, 216, std::vector<std::uint8_t>(384 * 216)});
    for (auto& f : frames)
      for (auto& v : f.samples) v = std::uint8_t(d(rng));
    const std::vector<int> mof = {0, 1, 0, 1, 1, 0, 0};
    set_devices({0});
    const auto a = filter_frames(frames, {mg, mr}, mof, PaddingMode::kReplicate);
    set_devices({0, 0});
    const auto b = filter_frames(frames, {mg, mr}, mof, PaddingMode::kReplicate);
    const auto c = filter_image(frames[3], mr, PaddingMode::kReplicate);  // 2 replicas, one image
    set_devices({0});
    bool same = a.size() == frames.size() && b.size() == frames.size();
    for (size_t f = 0; same && f < frames.size(); ++f) same = a[f].samples == b[f].samples;
    CHECK(same, "filter_frames: 2-replica frame ranges == single device (7 frames, 2 masks)");
    const FilterPlan pr(mr, 8, PaddingMode::kReplicate);
    CHECK(a[3].samples == filter_image(pr, frames[3]).samples, "filter_frames frame == filter_image of that frame");
    CHECK(c.samples == a[3].samples, "filter_image with set_devices({0, 0}) == single device");
  }
  // FilterPlan::from_dump carries the dump's mask and padding (read_operator_sets)
  {
    const FilterPlan a(Mask::gaussian3(), 8, PaddingMode::kReplicate);
    const FilterPlan b = FilterPlan::from_dump(a.dump());
    CHECK(b.padding() == PaddingMode::kReplicate && b.mask().weights() == a.mask().weights() &&
              b.dump() == a.dump(),
          "from_dump: mask, padding and the re-written dump equal the source plan's");
  }
  // Per-block drop-in cost (the reference's FilterPlan::filter_block loop,
  // ~5 us per 8x8 block on one CPU thread): one block per call
  // (cached per-thread stream and scratch, one device round trip) against a
  // 4096-block batch per call. Reported, and the single-block result must
  // equal the batched one.
  {
    const FilterPlan plan(Mask::gaussian3(), 8, PaddingMode::kReplicate);
    std::vector<BlockMatrix> blocks;
    for (int i = 0; i < 4096; ++i) blocks.push_back(random_u8_block(rng, 8));
    plan.filter_block(blocks[0]);  // warm
    const auto t0 = std::chrono::steady_clock::now();
    const int reps = 400;
    BlockMatrix last(8);
    for (int i = 0; i < reps; ++i) last = plan.filter_block(blocks[size_t(i)]);
    const auto t1 = std::chrono::steady_clock::now();
    const auto batch = plan.filter_block(blocks);
    const auto t2 = std::chrono::steady_clock::now();
    const auto batch2 = plan.filter_block(blocks);
    const auto t3 = std::chrono::steady_clock::now();
    const double single_us = std::chrono::duration<double, std::micro>(t1 - t0).count() / reps;
    const double batch_us = std::chrono::duration<double, std::micro>(t3 - t2).count() / blocks.size();
    std::printf("[INFO] FilterPlan::filter_block: %.2f us per call of one block; %.3f us per block in a "
                "4096-block call\n", single_us, batch_us);
    CHECK(max_abs_diff(last, batch[reps - 1]) == 0.0 && max_abs_diff(batch[7], batch2[7]) == 0.0,
          "single-block filter_block == batched filter_block");
  }
  std::printf("%s\n", failures ? "FAILED" : "ALL PASSED");
  return failures ? 1 : 0;
}
