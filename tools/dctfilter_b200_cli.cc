// dctfilter_b200 — the reference CLI (proj/tools/dctfilter_main.cc) on the
// B200 path: same subcommands, options, printed lines and exit codes
// (0 ok/verified, 1 verification failed, 2 usage or I/O error,
// dctfilter_main.cc:33-36), with every filter/transform/convolve running on
// the GPU through include/dctfilter_b200.hpp. The reference parses options
// with CLI11 (not vendored here); this front end parses the same option set
// by hand.
//
// Attribution: cmd_filter_block, print_suite, run_filter_suite,
// run_merge_suite and the build-operators / filter-image output lines follow
// the dctfilter reference CLI (dctfilter_main.cc:163-317), Copyright (c) the
// dctfilter project authors, licensed under the Apache License, Version 2.0
// (http://www.apache.org/licenses/LICENSE-2.0). Byte-identical output and the
// same RNG draw order are the drop-in contract.
//
//   build-operators --preset|--mask|--weights [--n 8] [--padding replicate] --out FILE
//   filter-block FILE [mask] [--n] [--padding] [--out FILE] [--verbose] [--compare-oracle]
//   filter-image IN.pgm [mask] [--n] [--padding] [--path dct|spatial] --out OUT.pgm
//   verify [--trials 1000] [--seed 42] [--corrupt]
//   bench [mask] [--n] [--padding] [--blocks 5000] [--seed 42]
#include <chrono>
#include <cstdio>
#include <fstream>
#include <iostream>
#include <map>
#include <random>
#include <set>
#include <sstream>
#include <string>
#include <vector>

#include "dctfilter_b200.hpp"

using namespace dctfilter_b200;

namespace {

constexpr int kExitOk = 0, kExitVerifyFailed = 1, kExitUsage = 2;

struct UsageError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

struct Args {
  std::string cmd;
  std::vector<std::string> positional;
  std::map<std::string, std::string> opt;
  std::set<std::string> flags;
  bool has(const std::string& k) const { return opt.count(k) != 0; }
  std::string get(const std::string& k, const std::string& dflt) const {
    auto it = opt.find(k);
    return it == opt.end() ? dflt : it->second;
  }
};

Args parse(int argc, char** argv) {
  static const std::set<std::string> kFlags = {"--verbose", "--compare-oracle", "--corrupt"};
  static const std::set<std::string> kOpts = {"--n", "--padding", "--path", "--out", "--preset", "--mask",
                                              "--weights", "--trials", "--seed", "--blocks"};
  static const std::set<std::string> kCmds = {"build-operators", "filter-block", "filter-image", "verify",
                                              "bench"};
  if (argc < 2) throw UsageError("a subcommand is required");
  Args a;
  a.cmd = argv[1];
  if (!kCmds.count(a.cmd)) throw UsageError("unknown subcommand '" + a.cmd + "'");
  for (int i = 2; i < argc; ++i) {
    const std::string s = argv[i];
    if (kFlags.count(s)) {
      a.flags.insert(s);
    } else if (kOpts.count(s)) {
      if (i + 1 >= argc) throw UsageError(s + " needs a value");
      a.opt[s] = argv[++i];
    } else if (!s.empty() && s[0] == '-') {
      throw UsageError("unknown option '" + s + "'");
    } else {
      a.positional.push_back(s);
    }
  }
  return a;
}

int to_int(const std::string& s, const char* what) {
  try {
    size_t pos = 0;
    const long v = std::stol(s, &pos);
    if (pos != s.size()) throw std::invalid_argument("");
    return int(v);
  } catch (const std::exception&) {
    throw UsageError(std::string("bad value for ") + what + ": '" + s + "'");
  }
}

std::vector<double> parse_weight_list(const std::string& text) {
  std::string cleaned = text;
  for (char& c : cleaned)
    if (c == ',') c = ' ';
  std::istringstream in(cleaned);
  std::vector<double> w;
  double v;
  while (in >> v) w.push_back(v);
  std::string leftover;
  if (in.clear(), in >> leftover) throw UsageError("bad kernel weight '" + leftover + "'");
  return w;
}

Mask mask_from_weights(std::vector<double> w) {
  const int k = int(std::lround(std::sqrt(double(w.size()))));
  if (k < 1 || size_t(k) * k != w.size() || k % 2 == 0)
    throw UsageError("kernel needs an odd square number of weights, got " + std::to_string(w.size()));
  return Mask(k, std::move(w));
}

Mask resolve_mask(const Args& a) {
  const int sources = int(a.has("--preset")) + int(a.has("--mask")) + int(a.has("--weights"));
  if (sources != 1) throw UsageError("exactly one of --preset, --mask, --weights is required");
  if (a.has("--preset")) {
    const std::string p = a.get("--preset", "");
    if (p == "identity") return Mask::identity();
    if (p == "average3") return Mask::average3();
    if (p == "gaussian3") return Mask::gaussian3();
    if (p == "magic3") return Mask::magic3();
    throw UsageError("unknown preset '" + p + "'");
  }
  if (a.has("--mask")) {
    std::ifstream in(a.get("--mask", ""));
    if (!in) throw UsageError("cannot open mask file '" + a.get("--mask", "") + "'");
    std::stringstream buf;
    buf << in.rdbuf();
    return mask_from_weights(parse_weight_list(buf.str()));
  }
  return mask_from_weights(parse_weight_list(a.get("--weights", "")));
}

PaddingMode parse_padding(const std::string& s) {
  if (s == "zero") return PaddingMode::kZero;
  if (s == "replicate") return PaddingMode::kReplicate;
  throw UsageError("unknown padding '" + s + "'");
}

Domain parse_path(const std::string& s) {
  if (s == "dct") return Domain::kDct;
  if (s == "spatial") return Domain::kSpatial;
  throw UsageError("unknown path '" + s + "'");
}

BlockMatrix read_block_file(const std::string& path, int n) {
  std::ifstream in(path);
  if (!in) throw UsageError("cannot open block file '" + path + "'");
  BlockMatrix block(n);
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) {
      long v;
      if (!(in >> v)) throw UsageError("block file needs " + std::to_string(n * n) + " whitespace-separated integers");
      if (v < 0 || v > 255) throw UsageError("block sample " + std::to_string(v) + " outside 0..255");
      block(i, j) = double(v);
    }
  long extra;
  if (in >> extra) throw UsageError("block file has more than n*n samples");
  return block;
}

void print_u8_block(std::ostream& out, const BlockMatrix& block) {
  const std::vector<std::uint8_t> q = quantize_u8(block);
  const int n = block.n();
  for (int i = 0; i < n; ++i) {
    for (int j = 0; j < n; ++j) out << (j ? " " : "") << int(q[size_t(i) * n + j]);
    out << "\n";
  }
}

void print_real_block(std::ostream& out, const BlockMatrix& block) {
  char buf[32];
  const int n = block.n();
  for (int i = 0; i < n; ++i) {
    for (int j = 0; j < n; ++j) {
      std::snprintf(buf, sizeof buf, "%11.4f", block(i, j));
      out << (j ? " " : "") << buf;
    }
    out << "\n";
  }
}

int cmd_build_operators(const Args& a) {
  const Mask mask = resolve_mask(a);
  const int n = to_int(a.get("--n", "8"), "--n");
  if (mask.k() > n) throw UsageError("kernel side exceeds block side");
  if (!a.has("--out")) throw UsageError("--out is required");
  const FilterPlan plan(mask, n, parse_padding(a.get("--padding", "replicate")));
  const std::string out_path = a.get("--out", "");
  std::ofstream out(out_path);
  if (!out) throw UsageError("cannot open '" + out_path + "' for writing");
  out << plan.dump();
  if (!out) throw UsageError("write failed for '" + out_path + "'");
  std::cout << "wrote " << out_path << ": spatial + dct operator sets, " << plan.npairs()
            << " pair(s) each, symmetric_merged=" << (plan.symmetric_merged() ? "yes" : "no") << "\n";
  return kExitOk;
}

int cmd_filter_block(const Args& a) {
  if (a.positional.size() != 1) throw UsageError("filter-block needs one block file");
  const Mask mask = resolve_mask(a);
  const int n = to_int(a.get("--n", "8"), "--n");
  if (mask.k() > n) throw UsageError("kernel side exceeds block side");
  const PaddingMode padding = parse_padding(a.get("--padding", "replicate"));
  const BlockMatrix block = read_block_file(a.positional[0], n);
  const bool verbose = a.flags.count("--verbose"), cmp = a.flags.count("--compare-oracle");

  const FilterPlan plan(mask, n, padding);
  const BlockMatrix coeffs = forward_2d(plan.basis(), block);
  const BlockMatrix filtered_coeffs = plan.filter_coeffs(coeffs);
  const BlockMatrix filtered = inverse_2d(plan.basis(), filtered_coeffs);
  if (verbose) {
    std::cout << "input dct coefficients:\n";
    print_real_block(std::cout, coeffs);
    std::cout << "filtered dct coefficients:\n";
    print_real_block(std::cout, filtered_coeffs);
  }
  if (!a.has("--out")) {
    if (verbose) std::cout << "filtered block:\n";
    print_u8_block(std::cout, filtered);
  } else {
    std::ofstream out(a.get("--out", ""));
    if (!out) throw UsageError("cannot open '" + a.get("--out", "") + "' for writing");
    print_u8_block(out, filtered);
  }
  if (verbose || cmp) {
    const BlockMatrix oracle = plan.convolve({block})[0];  // spatial path, on the device
    int mismatches = 0;
    const auto qa = quantize_u8(filtered), qb = quantize_u8(oracle);
    for (size_t i = 0; i < qa.size(); ++i) mismatches += qa[i] != qb[i];
    char err[32];
    std::snprintf(err, sizeof err, "%.3e", max_abs_diff(filtered, oracle));
    std::cout << "oracle max-abs error: " << err << "\n";
    std::cout << "u8 mismatches: " << mismatches << "\n";
  }
  return kExitOk;
}

int cmd_filter_image(const Args& a) {
  if (a.positional.size() != 1) throw UsageError("filter-image needs one input PGM");
  const Mask mask = resolve_mask(a);
  const int n = to_int(a.get("--n", "8"), "--n");
  if (mask.k() > n) throw UsageError("kernel side exceeds block side");
  if (!a.has("--out")) throw UsageError("--out is required");
  const GrayImage img = load_pgm_file(a.positional[0]);
  const GrayImage out = filter_image(img, mask, parse_padding(a.get("--padding", "replicate")),
                                     parse_path(a.get("--path", "dct")), n);
  save_pgm_file(a.get("--out", ""), out);
  std::cout << "wrote " << a.get("--out", "") << " (" << out.width << "x" << out.height << ")\n";
  return kExitOk;
}

struct SuiteResult {
  std::string name;
  double max_err = 0.0;
  long long mismatches = 0;
};

void print_suite(const SuiteResult& r) {
  char err[32];
  std::snprintf(err, sizeof err, "%.3e", r.max_err);
  std::printf("%-22s max_float_err=%s  u8_mismatches=%lld\n", r.name.c_str(), err, r.mismatches);
}

// Damage dct.pairs[0].left(0,0) by 1e-3 through the dump format (the
// reference corrupts the compiled set in memory, dctfilter_main.cc:282).
FilterPlan corrupted(const FilterPlan& plan) {
  std::string text = plan.dump();
  const size_t dct = text.find("domain dct");
  const size_t left = text.find("left\n", dct) + 5;
  const size_t end = text.find(' ', left);
  char buf[40];
  std::snprintf(buf, sizeof buf, "%.17g", std::stod(text.substr(left, end - left)) + 1e-3);
  text.replace(left, end - left, buf);
  return FilterPlan::from_dump(text);
}

// DCT path (device) vs spatial convolve (device, reference order) over
// `trials` random k x k masks, one random u8 block each (run_filter_suite,
// dctfilter_main.cc:267-295, same RNG draws).
SuiteResult run_filter_suite(const std::string& name, int k, PaddingMode padding, int trials,
                             std::uint64_t seed, bool corrupt) {
  SuiteResult result{name};
  std::mt19937_64 rng(seed);
  std::uniform_real_distribution<double> weight(-1.0, 1.0);
  std::uniform_int_distribution<int> sample(0, 255);
  for (int t = 0; t < trials; ++t) {
    std::vector<double> w(size_t(k) * k);
    for (double& v : w) v = weight(rng);
    const Mask mask(k, std::move(w));
    BlockMatrix block(8);
    for (double& v : block.data()) v = double(sample(rng));
    const FilterPlan plan(mask, 8, padding);
    const BlockMatrix filtered =
        (corrupt && t == 0) ? corrupted(plan).filter_block(block) : plan.filter_block(block);
    const BlockMatrix oracle = plan.convolve({block})[0];
    result.max_err = std::max(result.max_err, max_abs_diff(filtered, oracle));
    const auto qa = quantize_u8(filtered), qb = quantize_u8(oracle);
    for (size_t i = 0; i < qa.size(); ++i) result.mismatches += qa[i] != qb[i];
  }
  return result;
}

// apply(set) against apply(merge_symmetric(set)) over random row-symmetric
// 3x3 masks, zero padding, one random u8 block each (run_merge_suite,
// dctfilter_main.cc:297-317; same RNG draws). Both sets run on the device.
SuiteResult run_merge_suite(int trials, std::uint64_t seed) {
  SuiteResult result{"symmetric-merge"};
  std::mt19937_64 rng(seed);
  std::uniform_real_distribution<double> weight(-1.0, 1.0);
  std::uniform_int_distribution<int> sample(0, 255);
  for (int t = 0; t < trials; ++t) {
    std::vector<double> w(9);
    for (int c = 0; c < 3; ++c) {
      w[size_t(c)] = w[size_t(6 + c)] = weight(rng);
      w[size_t(3 + c)] = weight(rng);
    }
    const Mask mask(3, std::move(w));
    const OperatorSet set = build_spatial_operator_set(mask, 8, PaddingMode::kZero);
    const OperatorSet merged = merge_symmetric(set);
    BlockMatrix block(8);
    for (double& v : block.data()) v = double(sample(rng));
    result.max_err = std::max(result.max_err, max_abs_diff(apply(set, block), apply(merged, block)));
  }
  return result;
}

int cmd_verify(const Args& a) {
  const int trials = to_int(a.get("--trials", "1000"), "--trials");
  if (trials < 1) throw UsageError("--trials must be >= 1");
  std::uint64_t seed = std::uint64_t(std::stoull(a.get("--seed", "42")));
  const bool corrupt = a.flags.count("--corrupt");
  std::vector<SuiteResult> results;
  for (int k : {1, 3, 5, 7})
    results.push_back(run_filter_suite("zero-pad k=" + std::to_string(k), k, PaddingMode::kZero, trials,
                                       ++seed, corrupt && k == 3));
  for (int k : {1, 3, 5, 7})
    results.push_back(run_filter_suite("replicate k=" + std::to_string(k), k, PaddingMode::kReplicate,
                                       trials, ++seed, false));
  results.push_back(run_merge_suite(trials, ++seed));
  ++seed;  // the reference's correction-identity suite draws from the next seed
  bool ok = true;
  for (const SuiteResult& r : results) {
    print_suite(r);
    ok = ok && r.mismatches == 0 && r.max_err < 1e-9;
  }
  // The six-term replication-correction analysis (build_replication_correction,
  // operators.hpp) is outside the hot path and not built; say so instead of
  // printing a suite line for it.
  std::printf("%-22s skipped (out of scope: six-term replication correction not built)\n", "correction-identity");
  std::printf("%s\n", ok ? "VERIFIED" : "FAILED");
  return ok ? kExitOk : kExitVerifyFailed;
}

// Structural counts of the reference's bench (dctfilter_main.cc:383-403):
// sandwiches per block, matrix multiplications (2 per term, 1 when the left
// factor is the identity — count_matrix_multiplications, operators.hpp:260),
// and for 3x3 kernels the replication-correction groups
// (count_replication_groups, operators.hpp:249-256).
int mults(int k, bool merged) {
  const int h = (k - 1) / 2;
  const int pairs = merged ? h + 1 : k;
  return 2 * pairs - 1;  // only the center row's shift is the identity
}

int replication_groups(const Mask& m) {
  const double w1 = m.at(0, 0), w2 = m.at(0, 1), w3 = m.at(0, 2), w4 = m.at(1, 0), w6 = m.at(1, 2);
  const double w7 = m.at(2, 0), w8 = m.at(2, 1), w9 = m.at(2, 2);
  int groups = 6;
  if (w4 + w7 + w8 == w1 + w2 + w4 && w6 + w8 + w9 == w2 + w3 + w6) --groups;  // corners
  if (w3 == w1 && w6 == w4 && w9 == w7) --groups;                              // left/right sides
  if (w3 == w9 && w2 == w8 && w1 == w7) --groups;                              // top/bottom sides
  return groups;
}

int cmd_bench(const Args& a) {
  const int blocks = to_int(a.get("--blocks", "5000"), "--blocks");
  if (blocks < 1) throw UsageError("--blocks must be >= 1");
  const Mask mask = resolve_mask(a);
  const int n = to_int(a.get("--n", "8"), "--n");
  if (mask.k() > n) throw UsageError("kernel side exceeds block side");
  const PaddingMode padding = parse_padding(a.get("--padding", "replicate"));
  const std::uint64_t seed = std::uint64_t(std::stoull(a.get("--seed", "42")));
  const int k = mask.k();
  const bool symmetric = row_symmetric(mask);
  std::printf("kernel %dx%d on %dx%d blocks, %s padding\n", k, k, n, n,
              padding == PaddingMode::kZero ? "zero" : "replicate");
  std::printf("row symmetric: %s\n", symmetric ? "yes" : "no");
  if (symmetric) {
    std::printf("filtering sandwiches: %d merged vs %d unmerged\n", (k + 1) / 2, k);
    std::printf("matrix multiplications per block: %d merged vs %d unmerged\n", mults(k, true), mults(k, false));
  } else {
    std::printf("filtering sandwiches: %d (kernel rows not mergeable)\n", k);
    std::printf("matrix multiplications per block: %d\n", mults(k, false));
  }
  if (k == 3) std::printf("replication groups: %d of 6\n", replication_groups(mask));

  std::mt19937_64 rng(seed);
  std::uniform_int_distribution<int> sample(0, 255);
  std::vector<BlockMatrix> pixels;
  pixels.reserve(size_t(blocks));
  for (int b = 0; b < blocks; ++b) {
    BlockMatrix block(n);
    for (double& v : block.data()) v = double(sample(rng));
    pixels.push_back(std::move(block));
  }
  const FilterPlan plan(mask, n, padding);
  const std::vector<BlockMatrix> coeffs = forward_2d(plan.basis(), pixels);
  plan.filter_coeffs(coeffs);  // warm
  using Clock = std::chrono::steady_clock;
  auto t0 = Clock::now();
  plan.filter_coeffs(coeffs);
  const double dct_us = std::chrono::duration<double, std::micro>(Clock::now() - t0).count() / blocks;
  plan.convolve(pixels);
  t0 = Clock::now();
  plan.convolve(pixels);
  const double sp_us = std::chrono::duration<double, std::micro>(Clock::now() - t0).count() / blocks;
  std::printf("dct-domain apply: %.3f us/block over %d blocks\n", dct_us, blocks);
  std::printf("spatial reference: %.3f us/block over %d blocks\n", sp_us, blocks);
  std::printf("(batched on the GPU, host<->device copies included)\n");
  return kExitOk;
}

}  // namespace

int main(int argc, char** argv) {
  try {
    const Args a = parse(argc, argv);
    if (a.cmd == "build-operators") return cmd_build_operators(a);
    if (a.cmd == "filter-block") return cmd_filter_block(a);
    if (a.cmd == "filter-image") return cmd_filter_image(a);
    if (a.cmd == "verify") return cmd_verify(a);
    if (a.cmd == "bench") return cmd_bench(a);
  } catch (const std::exception& e) {
    std::cerr << "error: " << e.what() << "\n";
    return kExitUsage;
  }
  return kExitUsage;
}
