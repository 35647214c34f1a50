// TEST INFRASTRUCTURE ONLY — the BASELINE configs' seeded inputs, restated
// for the CPU checkers (bench.py --impl reference must not load the product
// package). Same generators as SURVEY.md §8(d) / DESIGN.md "Synthetic
// inputs"; tests/test_oracle.py pins every byte and weight to the product's
// own generator (paper_1710_07193_b200/csrc/synth.cc).
//   S(seed): v = 128 + sum_{i<8} 20 sin(2 pi (fx_i x + fy_i y) + phi_i) + N(0, 10^2),
//            fx, fy ~ U[0, 0.25), phi ~ U[0, 2 pi) from mt19937_64(seed); row y's
//            noise from mt19937_64(seed ^ (0x9E3779B97F4A7C15 (y + 1)));
//            std::round, clamp [0, 255].
//   U(seed): uniform_int_distribution<int>(0, 255) over mt19937_64(seed).
//   gaussian(k, sigma): exp(-(r^2 + c^2) / (2 sigma^2)) over offsets -h..h,
//            normalised by the row-major sum (mask.hpp:74-87 generalised).
//   random(k, seed): U[-1, 1) weights, normalised to sum 1, redrawn from the
//            same stream while |sum| < 0.05.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <random>
#include <thread>
#include <vector>

extern "C" {

void og_uniform_image(uint64_t seed, int w, int h, uint8_t* out) {
  std::mt19937_64 g(seed);
  std::uniform_int_distribution<int> u(0, 255);
  for (size_t i = 0, n = size_t(w) * h; i < n; ++i) out[i] = static_cast<uint8_t>(u(g));
}

void og_sinusoid_image(uint64_t seed, int w, int h, uint8_t* out, int nthreads) {
  constexpr double kPi = 3.141592653589793;
  std::mt19937_64 g(seed);
  std::uniform_real_distribution<double> uf(0.0, 0.25), up(0.0, 2.0 * kPi);
  double fx[8], fy[8], ph[8];
  for (int i = 0; i < 8; ++i) {
    fx[i] = uf(g);
    fy[i] = uf(g);
    ph[i] = up(g);
  }
  auto band = [&](int y0, int y1) {
    for (int y = y0; y < y1; ++y) {
      std::mt19937_64 ng(seed ^ (0x9E3779B97F4A7C15ull * static_cast<uint64_t>(y + 1)));
      std::normal_distribution<double> noise(0.0, 10.0);
      uint8_t* row = out + size_t(y) * w;
      for (int x = 0; x < w; ++x) {
        double v = 128.0;
        for (int i = 0; i < 8; ++i) v += 20.0 * std::sin(2.0 * kPi * (fx[i] * x + fy[i] * y) + ph[i]);
        v += noise(ng);
        row[x] = static_cast<uint8_t>(std::clamp(std::round(v), 0.0, 255.0));
      }
    }
  };
  const int nt = std::max(1, std::min(nthreads, h));
  std::vector<std::thread> ts;
  for (int t = 1; t < nt; ++t) ts.emplace_back(band, int(int64_t(h) * t / nt), int(int64_t(h) * (t + 1) / nt));
  band(0, int(int64_t(h) / nt));
  for (auto& t : ts) t.join();
}

void og_gaussian_mask(int k, double sigma, double* w) {
  const int hk = (k - 1) / 2;
  double sum = 0.0;
  for (int r = -hk; r <= hk; ++r)
    for (int c = -hk; c <= hk; ++c) sum += (w[size_t(r + hk) * k + c + hk] = std::exp(-(r * r + c * c) / (2.0 * sigma * sigma)));
  for (int i = 0; i < k * k; ++i) w[i] /= sum;
}

int og_random_mask(uint64_t seed, int k, double* w) {
  std::mt19937_64 g(seed);
  std::uniform_real_distribution<double> u(-1.0, 1.0);
  for (int redraws = 0;; ++redraws) {
    double sum = 0.0;
    for (int i = 0; i < k * k; ++i) sum += (w[i] = u(g));
    if (std::abs(sum) >= 0.05) {
      for (int i = 0; i < k * k; ++i) w[i] /= sum;
      return redraws;
    }
  }
}

}  // extern "C"
